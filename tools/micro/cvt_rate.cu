// Throughput of the conversion / fp64 / integer instructions a digit-GEMM epilogue can use
// (per SM per clock, all 148 SMs, 8 independent chains per thread).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(int iters, float* outf, double* outd, long long seed) {
  long long a[8];
  float f[8];
  double d[8];
  for (int c = 0; c < 8; ++c) { a[c] = seed + threadIdx.x * 8 + c; f[c] = 0.f; d[c] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (OP == 0) { f[c] += __ll2float_rn(a[c]); a[c] += 3; }                     // I2F.F32.S64 (+FADD, IADD64)
      if (OP == 1) { d[c] += __ll2double_rn(a[c]); a[c] += 3; }                    // I2F.F64.S64
      if (OP == 2) { d[c] += __int2double_rn((int)a[c]); a[c] += 3; }              // I2F.F64.S32
      if (OP == 3) { f[c] += __double2float_rn(d[c]); d[c] += 1.0; }              // F2F.F32.F64
      if (OP == 4) { d[c] = fma(d[c], 1.0000001, 0.5); }                           // DFMA
      if (OP == 5) { a[c] = a[c] * 3 + (a[c] >> 7); }                              // int64 mul-add-shift
      if (OP == 6) { f[c] += __int2float_rn((int)a[c]); a[c] += 3; }               // I2F.F32.S32
    }
  }
  float s = 0.f; double t = 0.0;
  for (int c = 0; c < 8; ++c) { s += f[c]; t += d[c] + (double)a[c]; }
  if (s == 1.2345f) outf[0] = s;
  if (t == 1.2345) outd[0] = t;
}

template <int OP>
void run(const char* name) {
  float* f; double* d;
  cudaMalloc(&f, 4); cudaMalloc(&d, 8);
  const int iters = 4096, threads = 512, blocks = 148 * 2;
  k<OP><<<blocks, threads>>>(iters, f, d, 1);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<OP><<<blocks, threads>>>(iters, f, d, 1);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double ops = (double)iters * 8 * threads * blocks;
  printf("{\"op\":\"%s\",\"ops_per_clk_per_sm_at_max_clock\":%.1f,\"gops\":%.1f}\n", name,
         ops / (ms * 1e-3) / (clk * 1e3) / 148, ops / (ms * 1e-3) / 1e9);
  cudaFree(f); cudaFree(d);
}

int main() {
  run<0>("i2f.f32.s64+fadd+iadd64"); run<1>("i2f.f64.s64+dadd+iadd64"); run<2>("i2f.f64.s32+dadd+iadd");
  run<3>("f2f.f32.f64+fadd+dadd"); run<4>("dfma"); run<5>("int64 imad+shf+iadd"); run<6>("i2f.f32.s32+fadd+iadd");
  return 0;
}
