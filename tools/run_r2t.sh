#!/bin/bash
D=gpurun_out/r2t; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "tri_solve" > $D/tests.txt 2>&1
echo "pytest rc=$?" >> $D/tests.txt
for i in 1 2; do timeout 300 python tools/time_solve.py --config C4 --iters 10 >> $D/time.jsonl 2>&1; done
for v in "1 8" "1 12" "0 10"; do
  set -- $v
  RCHOLQR_EXTRA_NVCC_FLAGS="-DRCQ_SOLVE_LDG=$1 -DRCQ_SOLVE_DW=$2" python -m paper_2210_09953_b200.build --ablation >> $D/build.log 2>&1
  echo "LDG=$1 DW=$2" >> $D/time.jsonl
  for i in 1 2; do RCHOLQR_ABLATION_LIB=1 timeout 300 python tools/time_solve.py --config C4 --iters 10 >> $D/time.jsonl 2>&1; done
  RCHOLQR_ABLATION_LIB=1 timeout 300 python tools/trace_solve.py > $D/trace_$1_$2.txt 2>&1
done
