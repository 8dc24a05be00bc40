#!/bin/bash
mkdir -p gpurun_out/r2b
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2b/build.log 2>&1
RCHOLQR_DEBUG=1 CUDA_LAUNCH_BLOCKING=1 timeout 600 python -m pytest tests/test_gpu_colmajor.py -x -q -p no:cacheprovider > gpurun_out/r2b/colmajor.txt 2>&1
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider -k "not colmajor" > gpurun_out/r2b/gpu_tests.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r2b/gpu_tests.txt
