#!/bin/bash
# drain / digit warp split of the n <= 64 tcgen05 solve (ablation builds with -DRCQ_SOLVE_RW/-DRCQ_SOLVE_DW)
D=gpurun_out/r2r; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log
for cfg in "16 6" "8 14" "8 10" "16 10" "8 6"; do
  set -- $cfg
  RCHOLQR_EXTRA_NVCC_FLAGS="-DRCQ_SOLVE_RW=$1 -DRCQ_SOLVE_DW=$2" python -m paper_2210_09953_b200.build --ablation >> $D/build.log 2>&1
  echo "RW=$1 DW=$2" >> $D/res.txt
  for i in 1 2; do RCHOLQR_ABLATION_LIB=1 python tools/time_solve.py --config C4 --iters 10 >> $D/res.txt 2>&1; done
  RCHOLQR_ABLATION_LIB=1 python tools/time_solve.py --config C2 --iters 20 >> $D/res.txt 2>&1
  RCHOLQR_ABLATION_LIB=1 python tools/trace_solve.py 2>&1 | python -c "
import sys,json
txt=sys.stdin.read(); i=txt.index('mma ['); d=json.loads(txt[:i])
for k,v in d.items(): print(k, round(v['per_tile_start_delta']), [None if x is None else round(x) for x in v['phase_means']])" >> $D/res.txt 2>&1
done
