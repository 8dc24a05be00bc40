// Probe of tcgen05.mma kind::i8 with the A operand in TENSOR MEMORY (sm_100a): D[128 x N] (s32) = A[128 x K] B[N x K]^T
// with A written by tcgen05.st (lane = row m; 32-bit column c of a k-step holds K bytes 4c .. 4c + 3, little endian)
// and B K-major in shared memory (canonical no-swizzle core matrices).  K = 64 as two MMAs; N in {16, 64, 112}.
// The solve's digit planes would live in TMEM this way (no shared-memory staging of the A operand).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t make_idesc_i8(int M, int N, bool a_signed, bool b_signed) {
  return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | ((b_signed ? 1u : 0u) << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

template <int N>
__global__ void probe(const int8_t* A, const int8_t* B, int32_t* D, int acol, int dcol) {
  constexpr int M = 128, K = 64;
  __shared__ __align__(1024) int8_t Bs[N * K];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int c = tid; c < N * K; c += blockDim.x) {
    const int r = c / K, k = c % K;
    Bs[((k / 16) * (N / 8) + r / 8) * 128 + (r % 8) * 16 + (k % 16)] = B[c];
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
  {  // row m = 32 warp + lane: K bytes packed into 16 columns (two k-steps of 8 columns)
    const int m = 32 * warp + lane;
    uint32_t v[16];
    for (int c = 0; c < 16; ++c)
      v[c] = (uint32_t)(uint8_t)A[m * K + 4 * c] | ((uint32_t)(uint8_t)A[m * K + 4 * c + 1] << 8) |
             ((uint32_t)(uint8_t)A[m * K + 4 * c + 2] << 16) | ((uint32_t)(uint8_t)A[m * K + 4 * c + 3] << 24);
    const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16) + acol;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n"
                 ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                   "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  if (tid == 0) {
    const uint32_t idesc = make_idesc_i8(M, N, true, true);
    for (int ks = 0; ks < K / 32; ++ks) {
      const uint64_t db = make_desc(smem_u32(Bs) + ks * 2 * (N / 8) * 128, (N / 8) * 128, 128);
      const uint32_t acc = ks > 0;
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                   "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n"
                   ::"r"(tmem + dcol), "r"(tmem + acol + ks * 8), "l"(db), "r"(idesc), "r"(acc));
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
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t v[8];
    const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16) + dcol + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n");
    for (int j = 0; j < 8; ++j) D[(32 * warp + lane) * N + c0 + j] = (int32_t)v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
}

template <int N>
int check(int acol, int dcol) {
  constexpr int M = 128, K = 64;
  int8_t *A, *B; int32_t* D;
  cudaMallocManaged(&A, M * K); cudaMallocManaged(&B, N * K); cudaMallocManaged(&D, M * N * 4);
  for (int i = 0; i < M * K; ++i) A[i] = (int8_t)(rand() % 256 - 128);
  for (int i = 0; i < N * K; ++i) B[i] = (int8_t)(rand() % 256 - 128);
  probe<N><<<1, 128>>>(A, B, D, acol, dcol);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
  int nb = 0;
  for (int r = 0; r < M; ++r)
    for (int c = 0; c < N; ++c) {
      long s = 0;
      for (int k = 0; k < K; ++k) s += (long)A[r * K + k] * (long)B[c * K + k];
      if (s != D[r * N + c]) ++nb;
    }
  printf("{\"a_in_tmem\":true,\"N\":%d,\"acol\":%d,\"dcol\":%d,\"mismatches\":%d}\n", N, acol, dcol, nb);
  cudaFree(A); cudaFree(B); cudaFree(D);
  return nb;
}

int main() {
  int bad = 0;
  bad += check<64>(256, 0);
  bad += check<16>(400, 32);
  bad += check<112>(392, 224);
  printf(bad ? "FAIL\n" : "PASS\n");
  return bad ? 1 : 0;
}
