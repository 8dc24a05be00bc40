#!/bin/bash
D=gpurun_out/r2m; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
for i in 1 2; do timeout 300 python tools/time_sketch.py --config C4 --iters 10 >> $D/time_sketch.jsonl 2>&1; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sketch_sparse_tc" -c 1 -o $D/full_sk python tools/time_sketch.py --config C4 --m 16777216 --iters 1 > $D/ncu.log 2>&1
ncu -i $D/full_sk.ncu-rep --page source --csv --print-source sass > $D/src.csv 2>/dev/null
ncu -i $D/full_sk.ncu-rep --page raw --csv > $D/raw.csv 2>/dev/null
ncu -i $D/full_sk.ncu-rep --page details --csv > $D/details.csv 2>/dev/null
