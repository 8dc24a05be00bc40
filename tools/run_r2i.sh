#!/bin/bash
# MN-major B operand probe + the rewritten sparse tcgen05 sketch: parity suites and C4 timing
D=gpurun_out/r2i; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o tools/micro/tc_i8_mn_test tools/micro/tc_i8_mn_test.cu && timeout 120 tools/micro/tc_i8_mn_test > $D/mn_test.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rademacher.py tests/test_gpu_srht.py -q -p no:cacheprovider -k "sparse or rademacher or srht or C4 or factor_parity" > $D/tests.txt 2>&1
echo "pytest rc=$?" >> $D/tests.txt
for i in 1 2; do timeout 300 python tools/time_sketch.py --config C4 --iters 10 >> $D/time_sketch.jsonl 2>&1; done
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $D/bench_c4.json 2> $D/bench_c4.err
