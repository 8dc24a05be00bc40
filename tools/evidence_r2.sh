# Round-2 evidence on one B200 (run under gpurun from the repo root); outputs under gpurun_out/ev2/.
set -x
D=gpurun_out/ev2; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $D/smi.txt
# bench lines: the default (C4, strong-scaled metric config), the reference arm, C1 (CUDA graph), C2, C3, C5
timeout 600 python bench.py --steps 20 --warmup 5 > $D/bench_c4.json 2> $D/bench_c4.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $D/bench_ref.json 2> $D/bench_ref.err
timeout 300 python bench.py --config C1 --steps 200 --warmup 10 > $D/bench_c1.json 2> $D/bench_c1.err
timeout 300 python bench.py --config C1 --steps 200 --warmup 10 --graph off --no-e2e --no-cpu-baseline > $D/bench_c1_nograph.json 2> $D/bench_c1_nograph.err
timeout 400 python bench.py --config C2 --steps 50 --warmup 5 > $D/bench_c2.json 2> $D/bench_c2.err
timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --cpu-seconds 10 > $D/bench_c3.json 2> $D/bench_c3.err
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --cpu-seconds 10 --no-e2e > $D/bench_c5.json 2> $D/bench_c5.err
timeout 300 python bench.py --algo rcholqr_rr --config C2 --steps 10 --warmup 3 --cpu-seconds 5 > $D/bench_rr_c2.json 2> $D/bench_rr_c2.err
# SRHT by the fast Walsh-Hadamard transform on the C3 / C5 shapes (not BASELINE lines)
timeout 600 python bench.py --config C3 --sketch srht --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $D/bench_c3_srht.json 2> $D/bench_c3_srht.err
timeout 900 python bench.py --config C5 --sketch srht --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $D/bench_c5_srht.json 2> $D/bench_c5_srht.err
# column-major X and Q through the native kernels vs the adapter (C4)
timeout 300 python tools/ab_time.py --config C4 --what factor,factor_cm --iters 20 --warm 5 --tag native > $D/colmajor_c4.jsonl 2>&1
RCHOLQR_COLMAJOR_ADAPTER=1 timeout 300 python tools/ab_time.py --config C4 --what factor_cm --iters 20 --warm 5 --tag adapter >> $D/colmajor_c4.jsonl 2>&1
# launch list (cold, serialised per-launch times: shares, not absolutes) of the default bench command
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_c4.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $D/ncu_launch.log 2>&1
# full captures of one factorization's heavy kernels at the bench sizes
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"sketch_sparse_tc|solve_tc_kernel|householder" -c 3 -o $D/full_c4 python tools/prof_factor.py --config C4 --iters 1 > $D/ncu_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sketch_gauss_tcp|xdig_split|householder|solve_tc|tri_|reduce" -c 8 -o $D/full_c2 python tools/prof_factor.py --config C2 --iters 1 > $D/ncu_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"srht_fwht" -c 1 -o $D/full_c3_srht python tools/prof_factor.py --config C3 --sketch srht --m 4194304 --iters 1 > $D/ncu_c3_srht.log 2>&1
ncu -i $D/full_c4.ncu-rep --page raw --csv > $D/full_c4_raw.csv 2>/dev/null
ncu -i $D/full_c4.ncu-rep --page source --csv --print-source sass > $D/full_c4_src.csv 2>/dev/null
ncu -i $D/full_c2.ncu-rep --page raw --csv > $D/full_c2_raw.csv 2>/dev/null
ncu -i $D/full_c3_srht.ncu-rep --page raw --csv > $D/full_c3_srht_raw.csv 2>/dev/null
ncu -i $D/full_c3_srht.ncu-rep --page source --csv --print-source sass > $D/full_c3_srht_src.csv 2>/dev/null
# the GPU suite + smoke
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > $D/gpu_tests.txt 2>&1
echo "pytest rc=$?" >> $D/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $D/smoke.txt 2>&1
ls -la $D
