#!/bin/bash
D=gpurun_out/r3h; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 300 python tools/ab_time.py --config C4 --what factor,factor_cm --iters 20 --warm 5 --tag cm >> $D/time.jsonl 2>&1
RCHOLQR_COLMAJOR_ADAPTER=1 timeout 300 python tools/ab_time.py --config C4 --what factor_cm --iters 20 --warm 5 --tag adapter >> $D/time.jsonl 2>&1
timeout 300 python tools/ab_time.py --config C2 --what factor,factor_cm --iters 50 --warm 10 --tag cm >> $D/time.jsonl 2>&1
RCHOLQR_COLMAJOR_ADAPTER=1 timeout 300 python tools/ab_time.py --config C2 --what factor_cm --iters 50 --warm 10 --tag adapter >> $D/time.jsonl 2>&1
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $D/gpu_tests.txt 2>&1
echo "pytest rc=$?" >> $D/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $D/smoke.txt 2>&1
