set -x
mkdir -p gpurun_out/ev
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/ev/smi.txt
timeout 400 python bench.py > gpurun_out/ev/bench_c2.json 2> gpurun_out/ev/bench_c2.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev/bench_ref.json 2> gpurun_out/ev/bench_ref.err
timeout 400 python bench.py --config C4 --steps 10 --warmup 3 --cpu-seconds 10 > gpurun_out/ev/bench_c4.json 2> gpurun_out/ev/bench_c4.err
timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --cpu-seconds 10 > gpurun_out/ev/bench_c3.json 2> gpurun_out/ev/bench_c3.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev/launches_c2.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ev/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sketch_gauss_tc|householder|solve|trsm|tri_|reduce" -c 8 -o gpurun_out/ev/full_c2 python tools/prof_factor.py --config C2 --iters 1 > gpurun_out/ev/ncu_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sketch_sparse_tc|solve_tc" -c 3 -o gpurun_out/ev/full_c4 python tools/prof_factor.py --config C4 --iters 1 > gpurun_out/ev/ncu_c4.log 2>&1
ls -la gpurun_out/ev
