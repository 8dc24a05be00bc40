// tcgen05.mma issue-rate probe on sm_100a: cycles per MMA (M = 128, SS operands, SWIZZLE_NONE
// K-major) for kind::i8 and kind::f16 at several N, with a commit + mbarrier wait every G MMAs.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
// kind::i8: c_format s32 (2); kind::f16: c_format f32 (1), a/b bf16 (1)
__host__ __device__ constexpr uint32_t idesc(int kind, int M, int N) {
  return kind == 0 ? ((2u << 4) | (1u << 7) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24))
                   : ((1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24));
}

template <int KIND, int N>
__global__ void rate(int iters, int G, long long* out, int sbo_b, int nreg, int shift) {
  constexpr int M = 128;
  __shared__ __align__(1024) uint8_t As[M * 32 * 2];
  __shared__ __align__(1024) uint8_t Bs[256 * 32 * 2 + 4096];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (int)sizeof(As); i += blockDim.x) As[i] = 0;
  for (int i = tid; i < (int)sizeof(Bs); i += blockDim.x) Bs[i] = 0;
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t id = idesc(KIND, M, N);
    const uint64_t da = make_desc(smem_u32(As), (M / 8) * 128, 128);
    const uint64_t db = make_desc(smem_u32(Bs), (N / 8) * sbo_b, sbo_b);
    uint32_t phase = 0;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int g = 0; g < G; ++g) {
        const uint32_t acc = 1;
        if (KIND == 0)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(tmem + (g & (nreg - 1)) * shift), "l"(da), "l"(db), "r"(id), "r"(acc));
        else
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(tmem + (g & (nreg - 1)) * shift), "l"(da), "l"(db), "r"(id), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&mbar)));
      uint32_t done = 0;
      while (!done)
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(done) : "r"(smem_u32(&mbar)), "r"(phase));
      phase ^= 1;
    }
    out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

template <int KIND, int N>
void run(int G, int sbo_b = 128, int nreg = 4, int shift = N) {
  long long* out;
  cudaMallocManaged(&out, 148 * sizeof(long long));
  const int iters = 2000;
  rate<KIND, N><<<148, 128>>>(iters, G, out, sbo_b, nreg, shift);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  rate<KIND, N><<<148, 128>>>(iters, G, out, sbo_b, nreg, shift);
  cudaEventRecord(e1);
  cudaError_t e = cudaDeviceSynchronize();
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return; }
  double s = 0;
  for (int i = 0; i < 148; ++i) s += out[i];
  s /= 148;
  const double per = s / ((double)iters * G);
  const double macs = 128.0 * N * (KIND == 0 ? 32 : 16);
  // chip-level rate from device events (all 148 SMs issue concurrently) and the SM clock it implies
  const double tops = 2.0 * macs * iters * G * 148 / (ms * 1e-3) / 1e12;
  const double mhz = s / (ms * 1e-3) / 1e6;
  printf("{\"nreg\":%d,\"shift\":%d,\"sbo_b\":%d,\"kind\":\"%s\",\"N\":%d,\"G\":%d,\"cyc_per_mma\":%.1f,\"mac_per_cyc\":%.0f,"
         "\"tops_chip\":%.1f,\"sm_mhz\":%.0f}\n", nreg, shift, sbo_b, KIND == 0 ? "i8" : "f16", N, G, per, macs / per, tops, mhz);
  cudaFree(out);
}

int main() {
  // independent D regions vs one shared accumulator vs overlapping (level-stacked) regions
  run<0, 224>(48, 128, 2, 224); run<0, 224>(48, 128, 1, 0); run<0, 224>(48, 128, 8, 32);
  run<0, 128>(48, 128, 4, 128); run<0, 128>(48, 128, 1, 0); run<0, 128>(48, 128, 4, 32);
  run<0, 64>(48, 128, 4, 64); run<0, 64>(48, 128, 1, 0);
  run<0, 256>(48, 128, 2, 256); run<0, 256>(48, 128, 1, 0);
  return 0;
}
