// Probe of tcgen05 kind::i8 with an MN-major B operand (sm_100a): D[128 x 512] (s32, TMEM) = A[128 x K] B[K x 512]
// with A K-major (canonical no-swizzle core matrices) and B MN-major SWIZZLE_NONE:
//   element (n, k) at (n % 16) + (k % 8) * 16 + (n / 16) * SBO + (k / 8) * LBO      (SBO: MN-group stride,
//   LBO: K-group stride; CUTLASS cute/atom/mma_traits_sm100.hpp "make_umma_desc<Major::MN>", INTERLEAVE)
// The 512 columns are two MMAs of N = 256 (start address offset by 16 MN groups), K = 64 as two k-steps.
// This is the operand layout of the sparse sketch that feeds the 8 bytes of each element's magic double
// straight to the MMA (sketch_tc.cu).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t make_idesc_i8(int M, int N, bool a_signed, bool b_signed, bool b_mn) {
  return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | ((b_signed ? 1u : 0u) << 10) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

constexpr int M = 128, K = 64, NT = 512, NH = 256;

__global__ void probe(const int8_t* A, const int8_t* B, int32_t* D, int a_signed, int b_signed, int sbo, int lbo) {
  extern __shared__ __align__(1024) int8_t sm[];
  int8_t* As = sm;                      // 8 KB
  int8_t* Bs = sm + M * K;              // up to 64 KB
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int c = tid; c < M * K; c += blockDim.x) {
    const int r = c / K, k = c % K;
    As[(k / 16) * (M / 8) * 128 + (r / 8) * 128 + (r % 8) * 16 + (k % 16)] = A[c];
  }
  for (int c = tid; c < NT * K; c += blockDim.x) {       // B given as [k][n]
    const int k = c / NT, n = c % NT;
    Bs[(n % 16) + (k % 8) * 16 + (n / 16) * sbo + (k / 8) * lbo] = B[c];
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = make_idesc_i8(M, NH, a_signed, b_signed, true);
    for (int h = 0; h < NT / NH; ++h)
      for (int ks = 0; ks < K / 32; ++ks) {
        const uint64_t da = make_desc(smem_u32(As) + ks * 2 * (M / 8) * 128, (M / 8) * 128, 128);
        const uint64_t db = make_desc(smem_u32(Bs) + h * (NH / 16) * sbo + ks * 4 * lbo, lbo, sbo);
        const uint32_t acc = ks > 0;
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(tmem + h * NH), "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&mbar)));
  }
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  for (int c0 = 0; c0 < NT; c0 += 16) {
    uint32_t v[16];
    const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n");
    for (int j = 0; j < 16; ++j) D[(32 * warp + lane) * NT + c0 + j] = (int32_t)v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
}

int check(int sbo, int lbo) {
  int8_t *A, *B; int32_t* D;
  cudaMallocManaged(&A, M * K); cudaMallocManaged(&B, NT * K); cudaMallocManaged(&D, M * NT * 4);
  const size_t smem = M * K + (size_t)(NT / 16 - 1) * sbo + (size_t)(K / 8 - 1) * lbo + 128 + 16;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int bad = 0;
  for (int mode = 0; mode < 4; ++mode) {
    const int as = mode & 1, bs = (mode >> 1) & 1;
    for (int i = 0; i < M * K; ++i) A[i] = (int8_t)(as ? (rand() % 256 - 128) : (rand() % 256));
    for (int i = 0; i < NT * K; ++i) B[i] = (int8_t)(bs ? (rand() % 256 - 128) : (rand() % 256));
    probe<<<1, 128, smem>>>(A, B, D, as, bs, sbo, lbo);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
    int nb = 0;
    for (int r = 0; r < M; ++r)
      for (int c = 0; c < NT; ++c) {
        long s = 0;
        for (int k = 0; k < K; ++k) {
          const long a = as ? (long)(int8_t)A[r * K + k] : (long)(uint8_t)A[r * K + k];
          const long b = bs ? (long)(int8_t)B[k * NT + c] : (long)(uint8_t)B[k * NT + c];
          s += a * b;
        }
        if (s != D[r * NT + c]) ++nb;
      }
    bad += nb;
  }
  printf("{\"b_major\":\"MN\",\"sbo\":%d,\"lbo\":%d,\"mismatches\":%d}\n", sbo, lbo, bad);
  cudaFree(A); cudaFree(B); cudaFree(D);
  return bad;
}

int main() {
  int bad = 0;
  bad += check(128, (NT / 16) * 128);      // MN groups packed, K groups after all MN groups (the sketch's layout)
  bad += check(8 * 128, 128);              // K groups packed inside an MN group
  bad += check(144, (NT / 16) * 144);      // padded MN-group stride
  printf(bad ? "FAIL\n" : "PASS\n");
  return bad ? 1 : 0;
}
