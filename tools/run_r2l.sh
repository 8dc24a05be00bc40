#!/bin/bash
D=gpurun_out/r2l; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
python -m paper_2210_09953_b200.build --ablation >> $D/build.log 2>&1
for i in 1 2; do timeout 300 python tools/time_sketch.py --config C4 --iters 10 >> $D/time_sketch.jsonl 2>&1; done
for dbg in 1 2 3; do
  RCHOLQR_ABLATION_LIB=1 RCHOLQR_STC_DEBUG=$dbg timeout 300 python tools/time_sketch.py --config C4 --iters 10 >> $D/ablate_sketch.jsonl 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rademacher.py tests/test_gpu_srht.py -q -p no:cacheprovider -k "sparse or rademacher or srht" > $D/tests.txt 2>&1
echo "pytest rc=$?" >> $D/tests.txt
