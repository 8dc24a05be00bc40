// DMMA issue-rate probe: TF/s vs warps per SMSP and independent accumulator chains per warp.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k1684(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 1.0 - threadIdx.x * 1e-4;
  double c[CH][4];
#pragma unroll
  for (int i = 0; i < CH; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0; for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}
// same but with an LDS feeding b each iteration (like the real kernel)
template <int CH>
__global__ void k1684_lds(double* out, int iters) {
  __shared__ double sb[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sb[i] = i * 1e-3;
  __syncthreads();
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1;
  double c[CH][4];
#pragma unroll
  for (int i = 0; i < CH; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      double b = sb[(threadIdx.x + i * 33 + it) & 1023];
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
    }
  }
  double s = 0; for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}
template <typename F>
float timeit(F f) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  f(); cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) { cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
  return best;
}
template <int CH>
void run(double* d, int sms) {
  for (int wps : {1, 2, 3, 4}) {
    int tpb = 32 * 4 * wps; int iters = 2048 / CH * 4;
    float ms = timeit([&] { k1684<CH><<<sms, tpb>>>(d, iters); });
    double fl = 2.0 * 16 * 8 * 4 * CH * (double)iters * sms * (tpb / 32);
    float ms2 = timeit([&] { k1684_lds<CH><<<sms, tpb>>>(d, iters); });
    printf("{\"chains\":%d,\"warps_per_smsp\":%d,\"tflops\":%.2f,\"tflops_lds\":%.2f}\n", CH, wps, fl / ms / 1e9, fl / ms2 / 1e9);
  }
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d; cudaMalloc(&d, 64);
  run<1>(d, sms); run<2>(d, sms); run<4>(d, sms); run<8>(d, sms); run<12>(d, sms);
  return 0;
}
