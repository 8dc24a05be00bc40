#!/bin/bash
mkdir -p gpurun_out/r2c
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2c/build.log 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/micro/cvt_rate tools/micro/cvt_rate.cu && tools/micro/cvt_rate > gpurun_out/r2c/cvt_rate.jsonl 2>&1
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2c/gpu_tests.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r2c/gpu_tests.txt
