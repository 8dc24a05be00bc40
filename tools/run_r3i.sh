#!/bin/bash
D=gpurun_out/r3i; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_graph.py -q -p no:cacheprovider > $D/tests.txt 2>&1
echo "pytest rc=$?" >> $D/tests.txt
timeout 300 python bench.py --config C1 --steps 200 --warmup 10 --graph on > $D/bench_c1_graph.json 2> $D/bench_c1_graph.err
timeout 300 python bench.py --config C1 --steps 200 --warmup 10 --graph off --no-e2e --no-cpu-baseline > $D/bench_c1_nograph.json 2> $D/bench_c1_nograph.err
