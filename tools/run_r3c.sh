#!/bin/bash
D=gpurun_out/r3c; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rademacher.py tests/test_gpu_srht.py -q -p no:cacheprovider -x -k "sparse or sketch or rademacher or srht" > $D/tests.txt 2>&1
echo "pytest rc=$?" >> $D/tests.txt
for v in 1 0 1 0; do
  RCHOLQR_EXTRA_NVCC_FLAGS="-DRCQ_STC_F2F=$v" python -m paper_2210_09953_b200.build --ablation >> $D/build.log 2>&1
  RCHOLQR_ABLATION_LIB=1 timeout 300 python tools/ab_time.py --what sketch --tag "stc_f2f=$v" >> $D/time.jsonl 2>&1
done
timeout 300 python tools/ab_time.py --what sketch,solve,factor --iters 20 --warm 5 --tag prod20 >> $D/time.jsonl 2>&1
