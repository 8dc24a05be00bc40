# Round-1 follow-up evidence after the n <= 128 digit-solve default (fp32 C2 paths); outputs under gpurun_out/ev/.
set -x
mkdir -p gpurun_out/ev
timeout 400 python bench.py > gpurun_out/ev/bench_c2.json 2> gpurun_out/ev/bench_c2.err
timeout 300 python bench.py --algo rcholqr2 --steps 10 --warmup 3 --cpu-seconds 5 > gpurun_out/ev/bench_rcqr2_c2.json 2> gpurun_out/ev/bench_rcqr2_c2.err
timeout 300 python bench.py --algo rcholqr_reduced --steps 10 --warmup 3 --cpu-seconds 5 > gpurun_out/ev/bench_reduced_c2.json 2> gpurun_out/ev/bench_reduced_c2.err
timeout 300 python bench.py --algo rcholqr_rr --steps 10 --warmup 3 --cpu-seconds 5 > gpurun_out/ev/bench_rr_c2.json 2> gpurun_out/ev/bench_rr_c2.err
timeout 300 python bench.py --algo rcholqr_rr2 --steps 10 --warmup 3 --cpu-seconds 5 > gpurun_out/ev/bench_rr2_c2.json 2> gpurun_out/ev/bench_rr2_c2.err
timeout 300 python bench.py --sketch srht --steps 10 --warmup 3 --cpu-seconds 5 > gpurun_out/ev/bench_c2_srht.json 2> gpurun_out/ev/bench_c2_srht.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev/launches_c2.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ev/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"solve_tc|tri_inverse" -c 3 -o gpurun_out/ev/full_c2_solve python tools/prof_factor.py --config C2 --iters 1 > gpurun_out/ev/ncu_c2s.log 2>&1
ls -la gpurun_out/ev
