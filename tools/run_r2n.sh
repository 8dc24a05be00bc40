#!/bin/bash
D=gpurun_out/r2n; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "tri_solve or factor_parity or C2_full or C4" > $D/tests.txt 2>&1
echo "pytest rc=$?" >> $D/tests.txt
for i in 1 2; do timeout 300 python tools/time_solve.py --config C4 --iters 10 >> $D/time_solve.jsonl 2>&1; done
timeout 300 python tools/time_solve.py --config C2 --iters 20 >> $D/time_solve.jsonl 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $D/bench_c4.json 2> $D/bench_c4.err
timeout 600 python bench.py --config C2 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $D/bench_c2.json 2> $D/bench_c2.err
