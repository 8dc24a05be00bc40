#!/bin/bash
D=gpurun_out/r2o; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sketch_sparse_tc|solve_tc_kernel" -c 2 -o $D/full_c4 python tools/prof_factor.py --config C4 --iters 1 --m 16777216 > $D/ncu.log 2>&1
ncu -i $D/full_c4.ncu-rep --page source --csv --print-source sass > $D/src.csv 2>/dev/null
ncu -i $D/full_c4.ncu-rep --page raw --csv > $D/raw.csv 2>/dev/null
