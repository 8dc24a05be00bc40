// Micro-benchmarks for the FP64 roofline denominators on B200 (sm_100a):
// DFMA (CUDA-core fp64), DMMA (mma.sync f64 shapes), FFMA. Not part of the product path.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

template<int CH>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CH];
  #pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0; for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}
template<int CH>
__global__ void ffma_kernel(float* out, int iters, float a, float b) {
  float acc[CH];
  #pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-3f + c;
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fmaf(acc[c], a, b);
  }
  float s = 0; for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 12345.678f) out[0] = s;
}
// m8n8k4 f64: A 1 reg, B 1 reg, C/D 2 regs
template<int CH>
__global__ void dmma884_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[CH][2];
  #pragma unroll
  for (int i = 0; i < CH; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}
// m16n8k4 f64: A 2 regs, B 1 reg, C 4 regs
template<int CH>
__global__ void dmma1684_kernel(double* out, int iters) {
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
// m16n8k16 f64: A 8 regs, B 4 regs, C 4 regs
template<int CH>
__global__ void dmma16816_kernel(double* out, int iters) {
  double a[8], b[4];
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3 + j;
  for (int j = 0; j < 4; ++j) b[j] = 1.0 - threadIdx.x * 1e-4 * j;
  double c[CH][4];
  #pragma unroll
  for (int i = 0; i < CH; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0; for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}
// int8 legacy mma.sync m16n8k32 s8 -> s32 (IMMA)
template<int CH>
__global__ void imma_kernel(int* out, int iters) {
  unsigned a[4], b[2];
  for (int j = 0; j < 4; ++j) a[j] = 0x01010101u * (threadIdx.x + j);
  for (int j = 0; j < 2; ++j) b[j] = 0x01010101u * (threadIdx.x ^ j);
  int c[CH][4];
  #pragma unroll
  for (int i = 0; i < CH; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(c[i][0]), "+r"(c[i][1]), "+r"(c[i][2]), "+r"(c[i][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  int s = 0; for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345) out[0] = s;
}
__global__ void copy_kernel(const double4* __restrict__ a, double4* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) b[i] = a[i];
}

template<typename F>
float timeit(F f, int reps) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  f(); cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"gpu\":\"%s\",\"sms\":%d,\"clock_khz\":%d,\"smem_optin\":%zu,\"l2\":%d}\n", p.name, sms, clk, p.sharedMemPerBlockOptin, p.l2CacheSize);
  double* dout; float* fout; int* iout; CK(cudaMalloc(&dout, 64)); fout = (float*)dout; iout = (int*)dout;
  const int iters = 4096;
  for (int tpb : {256, 512, 1024}) {
    int blocks = sms * (2048 / tpb);
    float ms = timeit([&]{ dfma_kernel<8><<<blocks, tpb>>>(dout, iters, 1.0000001, 1e-9); }, 5);
    double fl = 2.0 * 8 * iters * (double)blocks * tpb;
    printf("{\"kernel\":\"dfma\",\"tpb\":%d,\"tflops\":%.2f}\n", tpb, fl / ms / 1e9);
    ms = timeit([&]{ ffma_kernel<8><<<blocks, tpb>>>(fout, iters, 1.0000001f, 1e-9f); }, 5);
    printf("{\"kernel\":\"ffma\",\"tpb\":%d,\"tflops\":%.2f}\n", tpb, fl / ms / 1e9);
  }
  for (int tpb : {128, 256, 512}) {
    int blocks = sms * 4;
    float ms = timeit([&]{ dmma884_kernel<4><<<blocks, tpb>>>(dout, iters); }, 5);
    double fl = 2.0 * 8 * 8 * 4 * 4 * iters * (double)blocks * (tpb / 32);
    printf("{\"kernel\":\"dmma_m8n8k4\",\"tpb\":%d,\"tflops\":%.2f}\n", tpb, fl / ms / 1e9);
    ms = timeit([&]{ dmma1684_kernel<4><<<blocks, tpb>>>(dout, iters); }, 5);
    fl = 2.0 * 16 * 8 * 4 * 4 * iters * (double)blocks * (tpb / 32);
    printf("{\"kernel\":\"dmma_m16n8k4\",\"tpb\":%d,\"tflops\":%.2f}\n", tpb, fl / ms / 1e9);
    ms = timeit([&]{ dmma16816_kernel<4><<<blocks, tpb>>>(dout, iters / 4); }, 5);
    fl = 2.0 * 16 * 8 * 16 * 4 * (iters / 4) * (double)blocks * (tpb / 32);
    printf("{\"kernel\":\"dmma_m16n8k16\",\"tpb\":%d,\"tflops\":%.2f}\n", tpb, fl / ms / 1e9);
    ms = timeit([&]{ imma_kernel<4><<<blocks, tpb>>>(iout, iters); }, 5);
    fl = 2.0 * 16 * 8 * 32 * 4 * iters * (double)blocks * (tpb / 32);
    printf("{\"kernel\":\"imma_m16n8k32\",\"tpb\":%d,\"tops\":%.2f}\n", tpb, fl / ms / 1e9);
  }
  size_t n = (size_t)1 << 28;  // 2 GiB per buffer in double4 units /4 -> 8 GiB? keep 2 GiB: n double4 = 32 B each
  n = ((size_t)2 << 30) / 32;
  double4 *a, *b; CK(cudaMalloc(&a, n * 32)); CK(cudaMalloc(&b, n * 32));
  cudaMemset(a, 0, n * 32);
  float ms = timeit([&]{ copy_kernel<<<sms * 8, 256>>>(a, b, n); }, 10);
  printf("{\"kernel\":\"copy\",\"gbs\":%.1f}\n", 2.0 * n * 32 / ms / 1e6);
  CK(cudaGetLastError());
  return 0;
}
