#!/bin/bash
D=gpurun_out/r3k; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_graph.py tests/test_gpu_parity.py tests/test_gpu_rr.py -q -p no:cacheprovider -x -k "graph or sketch_parity or factor_parity or rr_parity" > $D/tests.txt 2>&1
echo "pytest rc=$?" >> $D/tests.txt
timeout 300 python bench.py --config C1 --steps 200 --warmup 10 > $D/bench_c1.json 2> $D/bench_c1.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $D/smoke.txt 2>&1
