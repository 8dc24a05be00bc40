#!/bin/bash
D=gpurun_out/r3a; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "tri_solve or solve" > $D/tests.txt 2>&1
echo "pytest rc=$?" >> $D/tests.txt
for i in 1 2; do timeout 300 python tools/time_solve.py --config C4 --iters 10 >> $D/time.jsonl 2>&1; done
for i in 1 2; do timeout 300 python tools/time_solve.py --config C2 --iters 50 >> $D/time.jsonl 2>&1; done
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $D/bench_c4.json 2> $D/bench_c4.err
