#!/bin/bash
# the whole GPU suite + smoke on one B200 (run under gpurun); outputs in gpurun_out/tests/
D=gpurun_out/tests; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=12 > $D/gpu_tests.txt 2>&1
echo "pytest rc=$?" >> $D/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $D/smoke.txt 2>&1
