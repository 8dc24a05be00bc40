#!/bin/bash
D=gpurun_out/r3d; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
nvidia-smi -q -d CLOCK,POWER,PERFORMANCE > $D/smi_q.txt 2>&1
timeout 300 python tools/series_time.py --what sketch --iters 60 > $D/series_sketch.json 2>&1
timeout 300 python tools/series_time.py --what solve --iters 60 > $D/series_solve.json 2>&1
timeout 300 python tools/series_time.py --what factor --iters 40 > $D/series_factor.json 2>&1
