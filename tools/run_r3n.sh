#!/bin/bash
D=gpurun_out/r3n; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_f64_cp" -s 8 -c 4 -o $D/full_c5_gemm python tools/prof_factor.py --config C5 --m 524288 --iters 1 > $D/ncu_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"trsm_mstream" -c 1 -o $D/full_c3_trsm python tools/prof_factor.py --config C3 --m 2097152 --iters 1 > $D/ncu_c3.log 2>&1
ncu -i $D/full_c5_gemm.ncu-rep --page raw --csv > $D/full_c5_gemm_raw.csv 2>/dev/null
ncu -i $D/full_c3_trsm.ncu-rep --page raw --csv > $D/full_c3_trsm_raw.csv 2>/dev/null
ncu -i $D/full_c3_trsm.ncu-rep --page source --csv --print-source sass > $D/full_c3_trsm_src.csv 2>/dev/null
