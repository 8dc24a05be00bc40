#!/bin/bash
# final check of the round: the GPU suite + smoke, the default bench line, the SRHT lines (outputs: gpurun_out/final/)
D=gpurun_out/final; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=12 > $D/gpu_tests.txt 2>&1
echo "pytest rc=$?" >> $D/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $D/smoke.txt 2>&1
timeout 600 python bench.py > $D/bench_default.json 2> $D/bench_default.err
timeout 600 python bench.py --config C3 --sketch srht --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $D/bench_c3_srht.json 2> $D/bench_c3_srht.err
timeout 900 python bench.py --config C5 --sketch srht --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $D/bench_c5_srht.json 2> $D/bench_c5_srht.err
timeout 300 python bench.py --algo rcholqr_rr --config C2 --steps 10 --warmup 3 --cpu-seconds 5 > $D/bench_rr_c2.json 2> $D/bench_rr_c2.err
