#!/bin/bash
mkdir -p gpurun_out/r2e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2e/build.log 2>&1
python tools/prof_factor.py --config C4 --iters 1 --m 16777216 > gpurun_out/r2e/pre.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sketch_sparse_tc|solve_tc_kernel" -c 2 -o gpurun_out/r2e/full_c4 python tools/prof_factor.py --config C4 --iters 1 --m 16777216 > gpurun_out/r2e/ncu.log 2>&1
ls -la gpurun_out/r2e
