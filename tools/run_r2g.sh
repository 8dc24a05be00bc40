#!/bin/bash
# round-2 re-entry baseline: build, full GPU suite, smoke, default bench line (C4), C2 line, reference arm
D=gpurun_out/r2g; mkdir -p $D
nproc > $D/host.txt; lscpu | head -20 >> $D/host.txt
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
RCHOLQR_DEBUG=1 timeout 300 python .scratch/diag.py > $D/diag.txt 2>&1
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $D/gpu_tests.txt 2>&1
echo "pytest rc=$?" >> $D/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1; echo "smoke rc=$?" >> $D/smoke.txt
timeout 900 python bench.py --steps 10 --warmup 3 > $D/bench_c4.json 2> $D/bench_c4.err
timeout 600 python bench.py --config C2 --steps 20 --warmup 5 > $D/bench_c2.json 2> $D/bench_c2.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > $D/ref.json 2> $D/ref.err
ls -la $D
