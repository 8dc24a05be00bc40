// tcgen05.mma kind::i8 throughput with an MN-major vs a K-major B operand (sm_100a), in the sparse sketch's
// stage pattern: per stage 2 k-steps x 2 MMAs of M = 128, N = 256, K = 32 reading a 32 KB B tile and an 8 KB A
// tile, one commit per stage, `inflight` stages issued before waiting on the oldest.  Prints cycles per MMA
// (floor 128 = M N / 256 per the B300 notes) for each layout.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout = 0) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, bool b_mn) {
  return (2u << 4) | (1u << 7) | ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

constexpr int M = 128, NT = 512, NH = 256, K = 64;

// mode 0: MN-major B (SBO = 128 between 16-byte MN groups, LBO = 4096 between 8-row K groups)
// mode 1: K-major B (N rows of 16-byte K chunks: SBO = 128 between 8-row groups, LBO = N/8*128 between K chunks)
// mode 2: MN-major B with N = 128 MMAs (4 per k-step)
// mode 3: A and B K-major SWIZZLE_128B (rows of 128 K bytes, 8-row atoms of 1 KB; k-step = +32 B start)
// mode 4: A K-major SWIZZLE_128B, B MN-major SWIZZLE_128B (atoms of 8 K rows x 128 MN bytes)
// mode 5: A K-major SWIZZLE_NONE, B K-major SWIZZLE_128B
// mode 6: as mode 1 but every MMA reads the SAME A and B (operand reuse); 7: same A, B varies; 8: A varies, same B
__global__ void rate(int stages, int inflight, int mode, int fill, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* As = sm;                 // 8 KB
  uint8_t* Bs = sm + 16384;         // up to 64 KB (K-major SW128: 512 rows x 128 B)
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar[8];
  const int tid = threadIdx.x, warp = tid >> 5;
  // fill 0: A, B pseudo-random; 1: A, B zero; 2: A sparse (one +-1 in 16, like the sketch's E), B random;
  // 3: A random, B zero
  for (int i = tid; i < 16384 + 65536; i += blockDim.x) {
    const uint32_t h = (uint32_t)i * 2654435761u;
    uint8_t v = (uint8_t)(h >> 13);
    if (fill == 1) v = 0;
    if (fill == 2 && i < 16384) v = ((h >> 7) & 15) == 0 ? (((h >> 20) & 1) ? 0xFF : 0x01) : 0;
    if (fill == 3 && i >= 16384) v = 0;
    sm[i] = v;
  }
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
    const uint32_t sa = smem_u32(As), sb = smem_u32(Bs);
    uint32_t phase[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const long long t0 = clock64();
    for (int c = 0; c < stages; ++c) {
      const int slot = c % inflight;
      if (c >= inflight) {
        uint32_t done = 0;
        while (!done)
          asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                       : "=r"(done) : "r"(smem_u32(&mbar[slot])), "r"(phase[slot]));
        phase[slot] ^= 1;
      }
      for (int ks0 = 0; ks0 < K / 32; ++ks0) {
        const int ks = (mode == 6 || mode == 7) ? 0 : ks0;
        const uint64_t da = (mode == 3 || mode == 4) ? make_desc(sa + ks * 32, 16, 1024, 2)
                                                     : make_desc(sa + ks * 2 * (M / 8) * 128, (M / 8) * 128, 128);
        const uint32_t acc = (c > 0 || ks0 > 0) ? 1u : 0u;
        const int nm = mode == 2 ? 4 : 2, nn = mode == 2 ? 128 : NH;
        for (int h0 = 0; h0 < nm; ++h0) {
          uint64_t db;
          const int h = (mode == 6 || mode == 8) ? 0 : h0;
          const int kb = mode == 8 ? 0 : ks;
          if (mode >= 6) db = make_desc(sb + h * (NH / 8) * 128 + kb * 2 * (NT / 8) * 128, (NT / 8) * 128, 128);
          else if (mode == 1) db = make_desc(sb + h * (NH / 8) * 128 + ks * 2 * (NT / 8) * 128, (NT / 8) * 128, 128);
          else if (mode == 3 || mode == 5) db = make_desc(sb + h * (NH / 8) * 1024 + ks * 32, 16, 1024, 2);
          else if (mode == 4) db = make_desc(sb + h * 2 * 1024 + ks * 4 * 4096, 1024, 4096, 2);
          else db = make_desc(sb + h * (nn / 16) * 128 + ks * 4 * 4096, 4096, 128);
          const uint32_t id = idesc_i8(M, nn, mode == 0 || mode == 2 || mode == 4);
          (void)kb;
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(tmem + h0 * nn), "l"(da), "l"(db), "r"(id), "r"(acc));
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&mbar[slot])));
    }
    for (int c = stages; c < stages + inflight; ++c) {   // drain
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
  const size_t smem = 16384 + 65536;
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const char* names[9] = {"MN-major N=256", "K-major N=256", "MN-major N=128", "A,B K-major SW128 N=256",
                          "A K SW128, B MN SW128 N=256", "A K none, B K SW128 N=256", "K-major, same A and B",
                          "K-major, same A, B varies", "K-major, A varies, same B"};
  const char* fills[4] = {"random", "zero", "A sparse +-1, B random", "A random, B zero"};
  for (int rep = 0; rep < 2; ++rep)
  for (int fill = 0; fill < 1; ++fill)
  for (int mode = 0; mode < 9; ++mode)
    for (int inflight : {3}) {
      const int stages = 4000;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      rate<<<148, 128, smem>>>(stages, inflight, mode, fill, out);
      cudaEventRecord(e1);
      cudaError_t e = cudaDeviceSynchronize();
      float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      double mx = 0;
      for (int b = 0; b < 148; ++b) mx = out[b] > mx ? out[b] : mx;
      const double macs = 148.0 * stages * M * 512 * K;
      printf("{\"layout\":\"%s\",\"cycles_per_mma\":%.1f,\"ms\":%.3f,\"tmac_s\":%.1f,\"mhz\":%.0f}\n",
             names[mode], mx / stages / (mode == 2 ? 8 : 4), ms, macs / ms / 1e9, mx / ms / 1e3);
    }
  return 0;
}
