#!/bin/bash
mkdir -p gpurun_out/r2f
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2f/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "tri_solve or factor_parity or C2_full" > gpurun_out/r2f/tests.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r2f/tests.txt
for i in 1 2; do timeout 300 python tools/time_solve.py --config C4 --iters 10 >> gpurun_out/r2f/time_solve.jsonl 2>&1; done
timeout 300 python tools/time_solve.py --config C2 --iters 20 >> gpurun_out/r2f/time_solve.jsonl 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"solve_tc_kernel" -c 1 -o gpurun_out/r2f/solve_c4 python tools/prof_factor.py --config C4 --iters 1 --m 16777216 > gpurun_out/r2f/ncu.log 2>&1
