#!/bin/bash
D=gpurun_out/dur; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=60 > $D/gpu_tests.txt 2>&1
echo "pytest rc=$?" >> $D/gpu_tests.txt
