// tcgen05.mma kind::i8 (M = 128, N = 256, K = 32, the same A and B every time, K-major SWIZZLE_NONE) issued in
// groups of G MMAs, one tcgen05.commit per group, waiting on the commit of the group `inflight` groups back:
// does the commit frequency limit MMA throughput?  Prints cycles per MMA (floor ~134 measured by tc_rate.cu).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);

// pattern 0: the same A and B (K-major) every MMA; 1: the sparse sketch's stage pattern (A = 128 x 64 K-major,
// B = 64 x 512 MN-major; per stage ks = 0, 1 x halves h = 0, 1, accumulator h); 2: as 1 with a K-major B
__global__ void rate(int total, int G, int inflight, int accmode, int pattern, long long* out) {
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint8_t* As = dsm;               // 8 KB
  uint8_t* Bs = dsm + 8192;        // 32 KB
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar[8];
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 8192 + 32768; i += blockDim.x) dsm[i] = (uint8_t)(i * 7);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (tid == 0) {
    for (int b = 0; b < 8; ++b) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar[b])));
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
    const uint64_t da = make_desc(smem_u32(As), 16 * 128, 128);
    const uint64_t db = make_desc(smem_u32(Bs), 32 * 128, 128);
    uint32_t phase[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const int groups = total / G;
    const long long t0 = clock64();
    for (int c = 0; c < groups; ++c) {
      const int slot = c % inflight;
      if (c >= inflight) {
        uint32_t done = 0;
        while (!done)
          asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                       : "=r"(done) : "r"(smem_u32(&mbar[slot])), "r"(phase[slot]));
        phase[slot] ^= 1;
      }
      for (int g = 0; g < G; ++g) {
        const uint32_t acc = accmode ? ((c > 0 || g > 1) ? 1u : 0u) : 1u;
        uint64_t a = da, b = db;
        uint32_t id = IDESC;
        if (pattern > 0) {
          const int h = g & 1, ks = (g >> 1) & 1;
          a = make_desc(smem_u32(As) + ks * 2 * 16 * 128, 16 * 128, 128);
          if (pattern == 1) { b = make_desc(smem_u32(Bs) + h * 16 * 128 + ks * 4 * 4096, 4096, 128); id |= 1u << 16; }
          else b = make_desc(smem_u32(Bs) + h * 32 * 128 + ks * 2 * 64 * 128, 64 * 128, 128);
        }
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(tmem + (g & 1) * 256), "l"(a), "l"(b), "r"(id), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&mbar[slot])));
    }
    for (int c = groups; c < groups + inflight; ++c) {
      const int slot = c % inflight;
      if (c < inflight) continue;
      uint32_t done = 0;
      while (!done)
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(done) : "r"(smem_u32(&mbar[slot])), "r"(phase[slot]));
      phase[slot] ^= 1;
    }
    out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

int main() {
  long long* out;
  cudaMallocManaged(&out, 148 * sizeof(long long));
  const int total = 19200;
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 + 32768);
  const int accmode = 1;
  for (int pattern = 0; pattern < 3; ++pattern)
    for (int G : {4, 8, 16, 48})
      for (int inflight : {3}) {
        rate<<<148, 128, 8192 + 32768>>>(total, G, inflight, accmode, pattern, out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        double mx = 0;
        for (int b = 0; b < 148; ++b) mx = out[b] > mx ? out[b] : mx;
        printf("{\"pattern\":%d,\"mma_per_commit\":%d,\"inflight\":%d,\"cycles_per_mma\":%.1f}\n", pattern, G, inflight,
               mx / total);
      }
  return 0;
}
