#!/bin/bash
D=gpurun_out/r2v; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "sketch_parity or gauss or presplit or factor_parity" > $D/tests.txt 2>&1
echo "pytest rc=$?" >> $D/tests.txt
for c in C2 C2 C3 C5; do timeout 300 python tools/time_sketch.py --config $c --iters 5 --m $([ $c = C2 ] && echo 1048576 || echo 4194304) >> $D/time_sketch.jsonl 2>&1; done
timeout 600 python bench.py --config C2 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $D/bench_c2.json 2> $D/bench_c2.err
