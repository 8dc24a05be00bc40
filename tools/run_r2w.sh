#!/bin/bash
D=gpurun_out/r2w; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_rr.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "rr or sketch_parity or presplit or gauss" > $D/tests.txt 2>&1
echo "pytest rc=$?" >> $D/tests.txt
timeout 600 python bench.py --config C2 --algo rcholqr_rr --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $D/bench_rr_c2.json 2> $D/bench_rr_c2.err
