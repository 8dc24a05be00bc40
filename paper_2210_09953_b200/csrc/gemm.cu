// gemm.cu -- fp64 DMMA tiled GEMM used by the blocked tall solve for n > 128 (DESIGN.md "Tall
// solve"): C = C0 + A B with A (m x K), B (K x N), all fp64 row-major, optional "B upper triangular"
// k-step skipping.  Each column block J of the solve is two launches:
//   T_J = X_J + Q_{<J} (-R_{<J,J})      (K = J*b)          then      Q_J = T_J Winv_JJ   (K = b)
// i.e. the paper's forward substitution blocked by b columns.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdlib>
#include "internal.cuh"

namespace rcq {

constexpr int GK = 16;   // K rows per pipeline chunk

template <int WM, int WN, int MW, int NW>
struct GemmCfg {
  static constexpr int TM = 16 * MW * WM;
  static constexpr int NT = 8 * NW * WN;
  static constexpr int THREADS = 32 * WM * WN;
  static constexpr int AS_LD = GK + 4;
  static constexpr int BS_LD = NT + 4;
  static constexpr size_t SMEM = sizeof(double) * (2 * (size_t)TM * AS_LD + 2 * (size_t)GK * BS_LD);
  static constexpr int AREG = (TM * GK + THREADS - 1) / THREADS;
  static constexpr int BREG = (GK * NT + THREADS - 1) / THREADS;
};

template <int WM, int WN, int MW, int NW>
__global__ void __launch_bounds__(32 * WM * WN, 1)
gemm_f64_kernel(const double* __restrict__ A, int64_t lda, const double* __restrict__ B, int64_t ldb,
                const double* __restrict__ C0, int64_t ldc0, double* __restrict__ C, int64_t ldc, int64_t m,
                int N, int K, int tri_b, int tiles_n, const int* status) {
  using G = GemmCfg<WM, WN, MW, NW>;
  if (*status) return;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + 2 * G::TM * G::AS_LD;
  const int tn = blockIdx.x % tiles_n;
  const int64_t row0 = (int64_t)(blockIdx.x / tiles_n) * G::TM;
  const int n0 = tn * G::NT;
  const int kend = tri_b ? min(K, n0 + G::NT) : K;
  const int nchunks = (kend + GK - 1) / GK;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  const int wm = warp % WM, wn = warp / WM;
  double acc[MW][NW][4];
#pragma unroll
  for (int a = 0; a < MW; ++a)
#pragma unroll
    for (int b = 0; b < NW; ++b) {
      const int64_t r = row0 + (wm * MW + a) * 16 + g;
      const int c = n0 + (wn * NW + b) * 8 + 2 * t4;
      acc[a][b][0] = (C0 && r < m && c < N) ? C0[r * ldc0 + c] : 0.0;
      acc[a][b][1] = (C0 && r < m && c + 1 < N) ? C0[r * ldc0 + c + 1] : 0.0;
      acc[a][b][2] = (C0 && r + 8 < m && c < N) ? C0[(r + 8) * ldc0 + c] : 0.0;
      acc[a][b][3] = (C0 && r + 8 < m && c + 1 < N) ? C0[(r + 8) * ldc0 + c + 1] : 0.0;
    }
  double ar[G::AREG], br[G::BREG];
  auto load = [&](int k0) {
#pragma unroll
    for (int u = 0; u < G::AREG; ++u) {
      const int c = tid + u * G::THREADS;
      const int ii = c / GK, kk = c % GK;
      ar[u] = (c < G::TM * GK && row0 + ii < m && k0 + kk < K) ? A[(row0 + ii) * lda + k0 + kk] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < G::BREG; ++u) {
      const int c = tid + u * G::THREADS;
      const int kk = c / G::NT, jj = c % G::NT;
      br[u] = (c < GK * G::NT && k0 + kk < K && n0 + jj < N) ? __ldg(B + (size_t)(k0 + kk) * ldb + n0 + jj) : 0.0;
    }
  };
  auto store = [&](int buf) {
    double* Ab = As + buf * G::TM * G::AS_LD;
    double* Bb = Bs + buf * GK * G::BS_LD;
#pragma unroll
    for (int u = 0; u < G::AREG; ++u) {
      const int c = tid + u * G::THREADS;
      if (c < G::TM * GK) Ab[(c / GK) * G::AS_LD + (c % GK)] = ar[u];
    }
#pragma unroll
    for (int u = 0; u < G::BREG; ++u) {
      const int c = tid + u * G::THREADS;
      if (c < GK * G::NT) Bb[(c / G::NT) * G::BS_LD + (c % G::NT)] = br[u];
    }
  };
  if (nchunks > 0) { load(0); store(0); }
  __syncthreads();
  for (int ch = 0; ch < nchunks; ++ch) {
    const int buf = ch & 1;
    const bool more = ch + 1 < nchunks;
    if (more) load((ch + 1) * GK);
    const double* Ab = As + buf * G::TM * G::AS_LD;
    const double* Bb = Bs + buf * GK * G::BS_LD;
#pragma unroll
    for (int ks = 0; ks < GK / 4; ++ks) {
      const int kg = ch * GK + 4 * ks;
      double a0[MW], a1[MW];
#pragma unroll
      for (int a = 0; a < MW; ++a) {
        const int r = (wm * MW + a) * 16 + g;
        a0[a] = Ab[r * G::AS_LD + 4 * ks + t4];
        a1[a] = Ab[(r + 8) * G::AS_LD + 4 * ks + t4];
      }
#pragma unroll
      for (int b = 0; b < NW; ++b) {
        if (!tri_b || kg <= n0 + (wn * NW + b) * 8 + 7) {
          const double bv = Bb[(4 * ks + t4) * G::BS_LD + (wn * NW + b) * 8 + g];
#pragma unroll
          for (int a = 0; a < MW; ++a) dmma_16x8x4(acc[a][b], a0[a], a1[a], bv);
        }
      }
    }
    if (more) store(buf ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < MW; ++a)
#pragma unroll
    for (int b = 0; b < NW; ++b) {
      const int64_t r = row0 + (wm * MW + a) * 16 + g;
      const int c = n0 + (wn * NW + b) * 8 + 2 * t4;
      if (r < m) {
        if (c < N) C[r * ldc + c] = acc[a][b][0];
        if (c + 1 < N) C[r * ldc + c + 1] = acc[a][b][1];
      }
      if (r + 8 < m) {
        if (c < N) C[(r + 8) * ldc + c] = acc[a][b][2];
        if (c + 1 < N) C[(r + 8) * ldc + c + 1] = acc[a][b][3];
      }
    }
}

// The same GEMM with a GC_STAGES-deep cp.async ring instead of register staging: every thread keeps
// its copies of the next GC_STAGES - 1 chunks in flight while the warps run the DMMAs of the current
// one (8-byte copies, so any leading dimension works; zero-filled outside A / B).
constexpr int GC_STAGES = 3;

template <int WM, int WN, int MW, int NW>
__global__ void __launch_bounds__(32 * WM * WN)
gemm_f64_cp_kernel(const double* __restrict__ A, int64_t lda, const double* __restrict__ B, int64_t ldb,
                   const double* __restrict__ C0, int64_t ldc0, double* __restrict__ C, int64_t ldc, int64_t m,
                   int N, int K, int tri_b, int tiles_n, const int* status) {
  using G = GemmCfg<WM, WN, MW, NW>;
  if (*status) return;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;                                            // [GC_STAGES][TM][AS_LD]
  double* Bs = smem + GC_STAGES * G::TM * G::AS_LD;             // [GC_STAGES][GK][BS_LD]
  const int tn = blockIdx.x % tiles_n;
  const int64_t row0 = (int64_t)(blockIdx.x / tiles_n) * G::TM;
  const int n0 = tn * G::NT;
  const int kend = tri_b ? min(K, n0 + G::NT) : K;
  const int nchunks = (kend + GK - 1) / GK;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  const int wm = warp % WM, wn = warp / WM;
  double acc[MW][NW][4];
#pragma unroll
  for (int a = 0; a < MW; ++a)
#pragma unroll
    for (int b = 0; b < NW; ++b) {
      const int64_t r = row0 + (wm * MW + a) * 16 + g;
      const int c = n0 + (wn * NW + b) * 8 + 2 * t4;
      acc[a][b][0] = (C0 && r < m && c < N) ? C0[r * ldc0 + c] : 0.0;
      acc[a][b][1] = (C0 && r < m && c + 1 < N) ? C0[r * ldc0 + c + 1] : 0.0;
      acc[a][b][2] = (C0 && r + 8 < m && c < N) ? C0[(r + 8) * ldc0 + c] : 0.0;
      acc[a][b][3] = (C0 && r + 8 < m && c + 1 < N) ? C0[(r + 8) * ldc0 + c + 1] : 0.0;
    }
  auto issue = [&](int ch) {
    const int k0 = ch * GK, slot = ch % GC_STAGES;
    double* Ab = As + slot * G::TM * G::AS_LD;
    double* Bb = Bs + slot * GK * G::BS_LD;
    for (int c = tid; c < G::TM * GK; c += G::THREADS) {
      const int ii = c / GK, kk = c % GK;
      const bool ok = row0 + ii < m && k0 + kk < K;
      const unsigned sa = (unsigned)__cvta_generic_to_shared(Ab + ii * G::AS_LD + kk);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa),
                   "l"(ok ? A + (row0 + ii) * lda + k0 + kk : A), "r"(ok ? 8 : 0));
    }
    for (int c = tid; c < GK * G::NT; c += G::THREADS) {
      const int kk = c / G::NT, jj = c % G::NT;
      const bool ok = k0 + kk < K && n0 + jj < N;
      const unsigned sa = (unsigned)__cvta_generic_to_shared(Bb + kk * G::BS_LD + jj);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa),
                   "l"(ok ? B + (size_t)(k0 + kk) * ldb + n0 + jj : B), "r"(ok ? 8 : 0));
    }
  };
#pragma unroll
  for (int p = 0; p < GC_STAGES - 1; ++p) {
    if (p < nchunks) issue(p);
    asm volatile("cp.async.commit_group;\n" ::);
  }
  for (int ch = 0; ch < nchunks; ++ch) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(GC_STAGES - 2) : "memory");
    __syncthreads();                                            // chunk ch visible; chunk ch-1's slot free
    if (ch + GC_STAGES - 1 < nchunks) issue(ch + GC_STAGES - 1);
    asm volatile("cp.async.commit_group;\n" ::);
    const int slot = ch % GC_STAGES;
    const double* Ab = As + slot * G::TM * G::AS_LD;
    const double* Bb = Bs + slot * GK * G::BS_LD;
#pragma unroll
    for (int ks = 0; ks < GK / 4; ++ks) {
      const int kg = ch * GK + 4 * ks;
      double a0[MW], a1[MW];
#pragma unroll
      for (int a = 0; a < MW; ++a) {
        const int r = (wm * MW + a) * 16 + g;
        a0[a] = Ab[r * G::AS_LD + 4 * ks + t4];
        a1[a] = Ab[(r + 8) * G::AS_LD + 4 * ks + t4];
      }
#pragma unroll
      for (int b = 0; b < NW; ++b) {
        if (!tri_b || kg <= n0 + (wn * NW + b) * 8 + 7) {
          const double bv = Bb[(4 * ks + t4) * G::BS_LD + (wn * NW + b) * 8 + g];
#pragma unroll
          for (int a = 0; a < MW; ++a) dmma_16x8x4(acc[a][b], a0[a], a1[a], bv);
        }
      }
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
#pragma unroll
  for (int a = 0; a < MW; ++a)
#pragma unroll
    for (int b = 0; b < NW; ++b) {
      const int64_t r = row0 + (wm * MW + a) * 16 + g;
      const int c = n0 + (wn * NW + b) * 8 + 2 * t4;
      if (r < m) {
        if (c < N) C[r * ldc + c] = acc[a][b][0];
        if (c + 1 < N) C[r * ldc + c + 1] = acc[a][b][1];
      }
      if (r + 8 < m) {
        if (c < N) C[(r + 8) * ldc + c] = acc[a][b][2];
        if (c + 1 < N) C[(r + 8) * ldc + c + 1] = acc[a][b][3];
      }
    }
}

template <int WM, int WN, int MW, int NW>
static cudaError_t launch_gcp(const double* A, int64_t lda, const double* B, int64_t ldb, const double* C0,
                              int64_t ldc0, double* C, int64_t ldc, int64_t m, int N, int K, bool tri_b,
                              const int* status, cudaStream_t st) {
  using GC = GemmCfg<WM, WN, MW, NW>;
  const size_t smem = sizeof(double) * GC_STAGES * ((size_t)GC::TM * GC::AS_LD + (size_t)GK * GC::BS_LD);
  auto kern = gemm_f64_cp_kernel<WM, WN, MW, NW>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int tiles_n = (N + GC::NT - 1) / GC::NT;
  const int64_t tiles_m = (m + GC::TM - 1) / GC::TM;
  if (tiles_m == 0 || tiles_n == 0) return cudaSuccess;
  kern<<<(unsigned)(tiles_m * tiles_n), GC::THREADS, smem, st>>>(A, lda, B, ldb, C0, ldc0, C, ldc, m, N, K,
                                                                 tri_b ? 1 : 0, tiles_n, status);
  return cudaGetLastError();
}

// 128 x 64 output tiles, 8 warps (4 x 2), each 2 m16 strips x 4 n8 tiles; or (RCHOLQR_GEMM_WIDE, N > 64)
// 128 x 128 tiles, 8 warps (2 x 4), each 4 m16 strips x 4 n8 tiles.
template <int WM, int WN, int MW, int NW>
static cudaError_t launch_g64(const double* A, int64_t lda, const double* B, int64_t ldb, const double* C0,
                              int64_t ldc0, double* C, int64_t ldc, int64_t m, int N, int K, bool tri_b,
                              const int* status, cudaStream_t st) {
  using GC = GemmCfg<WM, WN, MW, NW>;
  auto kern = gemm_f64_kernel<WM, WN, MW, NW>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GC::SMEM);
  if (e != cudaSuccess) return e;
  const int tiles_n = (N + GC::NT - 1) / GC::NT;
  const int64_t tiles_m = (m + GC::TM - 1) / GC::TM;
  if (tiles_m == 0 || tiles_n == 0) return cudaSuccess;
  kern<<<(unsigned)(tiles_m * tiles_n), GC::THREADS, GC::SMEM, st>>>(A, lda, B, ldb, C0, ldc0, C, ldc, m, N, K,
                                                                     tri_b ? 1 : 0, tiles_n, status);
  return cudaGetLastError();
}
using GemmC = GemmCfg<4, 2, 2, 4>;

cudaError_t launch_gemm_f64(const double* A, int64_t lda, const double* B, int64_t ldb, const double* C0,
                            int64_t ldc0, double* C, int64_t ldc, int64_t m, int N, int K, bool tri_b,
                            const int* status, cudaStream_t st) {
  // long K (the tall solve's T_J = X_J + Q_{<J} (-R_{<J,J}) and Q_J = T_J Winv_JJ): the cp.async ring;
  // short K (the blocked QR's rank-32 updates): the register-staged kernel, whose prologue is cheaper
  static const bool wide = getenv("RCHOLQR_GEMM_WIDE") != nullptr;                 // experiments
  static const bool no_cp = getenv("RCHOLQR_GEMM_NO_CP") != nullptr;               // experiments
  if (wide && N > 64) return launch_g64<2, 4, 4, 4>(A, lda, B, ldb, C0, ldc0, C, ldc, m, N, K, tri_b, status, st);
  if (!no_cp && K >= 128 && N >= 64) return launch_gcp<4, 2, 2, 4>(A, lda, B, ldb, C0, ldc0, C, ldc, m, N, K, tri_b, status, st);
  // narrow products (the blocked QR's N = 32 panel updates): 128 x 32 tiles, 8 warps of 16 x 32
  static const bool no_narrow = getenv("RCHOLQR_GEMM_NO_NARROW") != nullptr;      // experiments
  if (!no_narrow && N <= 32) return launch_g64<8, 1, 1, 4>(A, lda, B, ldb, C0, ldc0, C, ldc, m, N, K, tri_b, status, st);
  auto kern = gemm_f64_kernel<4, 2, 2, 4>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GemmC::SMEM);
  if (e != cudaSuccess) return e;
  const int tiles_n = (N + GemmC::NT - 1) / GemmC::NT;
  const int64_t tiles_m = (m + GemmC::TM - 1) / GemmC::TM;
  if (tiles_m == 0 || tiles_n == 0) return cudaSuccess;
  kern<<<(unsigned)(tiles_m * tiles_n), GemmC::THREADS, GemmC::SMEM, st>>>(A, lda, B, ldb, C0, ldc0, C, ldc, m, N, K,
                                                                         tri_b ? 1 : 0, tiles_n, status);
  return cudaGetLastError();
}

}  // namespace rcq
