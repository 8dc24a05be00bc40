#!/bin/bash
D=gpurun_out/r2q; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log
python -m paper_2210_09953_b200.build --ablation >> $D/build.log 2>&1
for dbg in 0 1 2 4 5 6 3 7; do
  echo "dbg=$dbg" >> $D/trace.txt
  RCHOLQR_QTC_DEBUG=$dbg python tools/trace_solve.py 2>&1 | python -c "
import sys,json
txt=sys.stdin.read(); i=txt.index('mma ['); d=json.loads(txt[:i])
for k,v in d.items(): print(k, round(v['per_tile_start_delta']), [None if x is None else round(x) for x in v['phase_means']])" >> $D/trace.txt 2>&1
done
