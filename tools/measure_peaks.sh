#!/bin/bash
# Measured unit peaks of this pool's B200 (run under gpurun): FP64 DFMA / DMMA, FFMA, IMMA (mma.sync),
# tcgen05 kind::i8 / kind::f16 (tc_rate.cu, chip-level rate from device events + the implied SM clock),
# written to gpurun_out/peaks_r2.jsonl (copy to profiles/ and commit; bench.py reads profiles/peaks_r2.jsonl).
set -e
cd "$(dirname "$0")/micro"
ARCH="-gencode arch=compute_100a,code=sm_100a"
nvcc -O3 -std=c++17 $ARCH -o peaks peaks.cu
nvcc -O3 -std=c++17 $ARCH -o tc_rate tc_rate.cu
out=../../gpurun_out/peaks_r2.jsonl
mkdir -p ../../gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv,noheader > ../../gpurun_out/peaks_r2_clocks.txt || true
./peaks > "$out"
./tc_rate >> "$out"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv,noheader >> ../../gpurun_out/peaks_r2_clocks.txt || true
cat "$out"
