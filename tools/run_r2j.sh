#!/bin/bash
# sparse tcgen05 sketch (MN-major bytes) ablations + ncu of the C4 sketch and solve
D=gpurun_out/r2j; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
python -m paper_2210_09953_b200.build --ablation >> $D/build.log 2>&1
for dbg in 0 1 2 4 3 6 5 7; do
  RCHOLQR_ABLATION_LIB=1 RCHOLQR_STC_DEBUG=$dbg timeout 300 python tools/time_sketch.py --config C4 --iters 10 >> $D/ablate_sketch.jsonl 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sketch_sparse_tc|solve_tc_kernel" -c 2 -o $D/full_c4 python tools/prof_factor.py --config C4 --iters 1 --m 16777216 > $D/ncu.log 2>&1
ncu -i $D/full_c4.ncu-rep --page source --csv --print-source sass > $D/src.csv 2>/dev/null
ncu -i $D/full_c4.ncu-rep --page raw --csv > $D/raw.csv 2>/dev/null
ls -la $D
