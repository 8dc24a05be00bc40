#!/bin/bash
# SRHT suites + the transform-vs-dense sketch timings of profiles/srht_fwht_vs_dense_r2.jsonl (run under gpurun)
D=gpurun_out/srht; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_srht_fwht.py tests/test_gpu_srht.py -q -p no:cacheprovider > $D/tests.txt 2>&1
echo "pytest rc=$?" >> $D/tests.txt
for cfg in C4 C2 C3 C5; do
  it=20; [ $cfg = C3 ] && it=3
  RCHOLQR_SRHT_FWHT=1 timeout 300 python tools/ab_time.py --config $cfg --sketch srht --what sketch --iters $it --warm 3 --tag fwht >> $D/time.jsonl 2>&1
  RCHOLQR_SRHT_DENSE=1 timeout 300 python tools/ab_time.py --config $cfg --sketch srht --what sketch --iters $it --warm 3 --tag dense >> $D/time.jsonl 2>&1
done
