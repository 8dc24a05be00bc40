#!/bin/bash
D=gpurun_out/r2h; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
RCHOLQR_DEBUG=1 CUDA_LAUNCH_BLOCKING=1 timeout 300 python .scratch/diag.py > $D/diag.txt 2>&1
RCHOLQR_DEBUG=1 timeout 600 compute-sanitizer --print-limit 20 python .scratch/diag.py > $D/sanitizer.txt 2>&1
