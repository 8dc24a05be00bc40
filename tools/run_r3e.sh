#!/bin/bash
D=gpurun_out/r3e; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_colmajor.py -q -p no:cacheprovider > $D/tests.txt 2>&1
echo "pytest rc=$?" >> $D/tests.txt
