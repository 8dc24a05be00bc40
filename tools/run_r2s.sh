#!/bin/bash
D=gpurun_out/r2s; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
python -m paper_2210_09953_b200.build --ablation >> $D/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "tri_solve" > $D/tests.txt 2>&1
echo "pytest rc=$?" >> $D/tests.txt
for i in 1 2; do timeout 300 python tools/time_solve.py --config C4 --iters 10 >> $D/time_solve.jsonl 2>&1; done
RCHOLQR_ABLATION_LIB=1 timeout 300 python tools/trace_solve.py 2>&1 | python -c "
import sys,json
txt=sys.stdin.read(); i=txt.index('mma ['); d=json.loads(txt[:i])
for k,v in d.items(): print(k, round(v['per_tile_start_delta']), [None if x is None else round(x) for x in v['phase_means']])" > $D/trace.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "factor_parity or C4 or C2_full" >> $D/tests.txt 2>&1
echo "pytest rc=$?" >> $D/tests.txt
