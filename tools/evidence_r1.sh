# Round-1 evidence on one B200 (run under gpurun from the repo root); outputs under gpurun_out/ev/.
set -x
mkdir -p gpurun_out/ev
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/ev/smi.txt
# bench lines: the north-star default (C2), the reference arm, the other BASELINE configs, the §8(f) modes
timeout 400 python bench.py > gpurun_out/ev/bench_c2.json 2> gpurun_out/ev/bench_c2.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev/bench_ref.json 2> gpurun_out/ev/bench_ref.err
timeout 400 python bench.py --config C4 --steps 10 --warmup 3 --cpu-seconds 10 > gpurun_out/ev/bench_c4.json 2> gpurun_out/ev/bench_c4.err
timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --cpu-seconds 10 > gpurun_out/ev/bench_c3.json 2> gpurun_out/ev/bench_c3.err
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --cpu-seconds 10 --no-e2e > gpurun_out/ev/bench_c5.json 2> gpurun_out/ev/bench_c5.err
timeout 300 python bench.py --algo rcholqr2 --steps 10 --warmup 3 --cpu-seconds 5 > gpurun_out/ev/bench_rcqr2_c2.json 2> gpurun_out/ev/bench_rcqr2_c2.err
timeout 400 python bench.py --algo rcholqr2 --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ev/bench_rcqr2_c4.json 2> gpurun_out/ev/bench_rcqr2_c4.err
timeout 300 python bench.py --algo rcholqr_reduced --steps 10 --warmup 3 --cpu-seconds 5 > gpurun_out/ev/bench_reduced_c2.json 2> gpurun_out/ev/bench_reduced_c2.err
timeout 300 python bench.py --algo rcholqr_rr --steps 10 --warmup 3 --cpu-seconds 5 > gpurun_out/ev/bench_rr_c2.json 2> gpurun_out/ev/bench_rr_c2.err
timeout 300 python bench.py --algo rcholqr_rr2 --steps 10 --warmup 3 --cpu-seconds 5 > gpurun_out/ev/bench_rr2_c2.json 2> gpurun_out/ev/bench_rr2_c2.err
timeout 600 python bench.py --algo rcholqr_rr --config C3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ev/bench_rr_c3.json 2> gpurun_out/ev/bench_rr_c3.err
timeout 300 python bench.py --config C4 --sketch rademacher --steps 10 --warmup 3 --cpu-seconds 5 > gpurun_out/ev/bench_c4_rademacher.json 2> gpurun_out/ev/bench_c4_rademacher.err
timeout 300 python bench.py --config C4 --sketch srht --steps 10 --warmup 3 --cpu-seconds 5 > gpurun_out/ev/bench_c4_srht.json 2> gpurun_out/ev/bench_c4_srht.err
timeout 300 python bench.py --sketch srht --steps 10 --warmup 3 --cpu-seconds 5 > gpurun_out/ev/bench_c2_srht.json 2> gpurun_out/ev/bench_c2_srht.err
# launch list (cold, serialised per-launch times: shares, not absolutes) of the default bench command
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev/launches_c2.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ev/ncu_launch.log 2>&1
# full captures of one factorization's kernels (C2, C4) and the Alg. 7 / Alg. 3 small kernels
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sketch_gauss_tcp|xdig_split|householder|solve|trsm|tri_|reduce" -c 8 -o gpurun_out/ev/full_c2 python tools/prof_factor.py --config C2 --iters 1 > gpurun_out/ev/ncu_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sketch_sparse_tc|solve_tc" -c 3 -o gpurun_out/ev/full_c4 python tools/prof_factor.py --config C4 --iters 1 > gpurun_out/ev/ncu_c4.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"qrcp|rank_kernel|colsq|gather_x" -c 4 -o gpurun_out/ev/full_rr_c2 python tools/prof_rr.py --config C2 --reps 1 > gpurun_out/ev/ncu_rr.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"sketch_gauss_tcp|xdig_split|trsm_mstream|householder|qr_panel" -c 6 -o gpurun_out/ev/full_c3 python tools/prof_factor.py --config C3 --iters 1 --m 4194304 > gpurun_out/ev/ncu_c3.log 2>&1
ls -la gpurun_out/ev
