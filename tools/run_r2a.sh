#!/bin/bash
# round-2 GPU check: build, unit peaks, GPU test suite, smoke, default bench line, reference arm
mkdir -p gpurun_out/r2a
free -g > gpurun_out/r2a/free.txt; nproc >> gpurun_out/r2a/free.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2a/build.log 2>&1
bash tools/measure_peaks.sh > gpurun_out/r2a/peaks.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2a/gpu_tests.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r2a/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a/smoke.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a/bench.json 2> gpurun_out/r2a/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2a/ref.json 2> gpurun_out/r2a/ref.err
ls -la gpurun_out/r2a
