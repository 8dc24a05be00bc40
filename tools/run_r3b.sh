#!/bin/bash
D=gpurun_out/r3b; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
for v in "1 1" "0 1" "1 0" "0 0"; do
  set -- $v
  RCHOLQR_EXTRA_NVCC_FLAGS="-DRCQ_SOLVE_F2F=$1 -DRCQ_SOLVE_ROT=$2" python -m paper_2210_09953_b200.build --ablation >> $D/build.log 2>&1
  for i in 1 2; do RCHOLQR_ABLATION_LIB=1 timeout 300 python tools/ab_time.py --what solve --tag "f2f=$1 rot=$2" >> $D/time.jsonl 2>&1; done
done
timeout 300 python tools/ab_time.py --what solve,sketch,factor --tag prod >> $D/time.jsonl 2>&1
RCHOLQR_ABLATION_LIB=1 timeout 300 python tools/trace_solve.py > $D/trace.txt 2>&1
