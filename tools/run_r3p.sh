#!/bin/bash
D=gpurun_out/r3p; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_srht_fwht.py -q -p no:cacheprovider --durations=8 -k "reduced or 120000" > $D/tests.txt 2>&1
echo "pytest rc=$?" >> $D/tests.txt
