#!/bin/bash
D=gpurun_out/r3j; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_graph.py tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "graph or sketch or factor_parity or partition" > $D/tests.txt 2>&1
echo "pytest rc=$?" >> $D/tests.txt
timeout 300 python bench.py --config C1 --steps 200 --warmup 10 --graph on --no-e2e --no-cpu-baseline > $D/bench_c1_graph.json 2> $D/bench_c1_graph.err
RCHOLQR_GAUSS_DMMA=1 timeout 300 python bench.py --config C1 --steps 200 --warmup 10 --graph on --no-e2e --no-cpu-baseline > $D/bench_c1_graph_dmma.json 2> $D/bench_c1_graph_dmma.err
