// tcgen05 kind::i8 issue patterns of the digit solve (sm_100a): per k-step, six MMAs with distinct
// A tiles (128 x 32 B), one shared stacked B (N = (7 - a) * 32 rows), D at column a * 32.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t idesc(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
               ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}
// mode 0: solve pattern (distinct A tiles, N = (7-a)*32, overlapping D)
// mode 1: same A tile for all six, same N/D pattern
// mode 2: distinct A tiles, N = 224 for all, D = a * 32 (overlapping)
// mode 3: distinct A, N = 224, D disjoint (a % 2) * 224
extern __shared__ __align__(1024) uint8_t dsm[];
__global__ void pat(int iters, int mode, long long* out) {
  uint8_t* As = dsm;                 // 6 tiles x 8 KB (K = 64)
  uint8_t* Bs = dsm + 6 * 8192;      // 224 rows x 64 B
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 6 * 8192 + 224 * 64; i += blockDim.x) dsm[i] = (uint8_t)(i * 7);
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
    uint32_t phase = 0;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int ks = 0; ks < 2; ++ks) {
#pragma unroll
        for (int a = 0; a < 6; ++a) {
          const int ta = mode == 1 ? 0 : a;
          const uint64_t da = make_desc(smem_u32(As + ta * 8192) + ks * 4096, 2048, 128);
          const uint64_t db = make_desc(smem_u32(Bs) + ks * 2 * 224 * 16, 224 * 16, 128);
          const int N = (mode >= 2) ? 224 : (7 - a) * 32;
          const uint32_t dcol = mode == 3 ? (a & 1) * 224 : a * 32;
          mma(tmem + dcol, da, db, idesc(128, N), 1u);
        }
      }
      if ((it & 15) == 15 || it == iters - 1) {
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&mbar)));
        uint32_t done = 0;
        while (!done)
          asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                       : "=r"(done) : "r"(smem_u32(&mbar)), "r"(phase));
        phase ^= 1;
      }
    }
    out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}
int main() {
  long long* out;
  cudaMallocManaged(&out, 148 * 8);
  const int smem = 6 * 8192 + 224 * 64;
  cudaFuncSetAttribute(pat, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 512;
  for (int mode = 0; mode < 4; ++mode) {
    pat<<<148, 128, smem>>>(iters, mode, out);
    cudaDeviceSynchronize();
    pat<<<148, 128, smem>>>(iters, mode, out);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    double s = 0; for (int i = 0; i < 148; ++i) s += out[i]; s /= 148;
    printf("{\"mode\":%d,\"cycles_per_kstep_group\":%.1f,\"cycles_per_mma\":%.1f}\n", mode, s / (iters * 2.0), s / (iters * 12.0));
  }
  return 0;
}
