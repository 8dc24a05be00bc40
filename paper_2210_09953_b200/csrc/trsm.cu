// trsm.cu -- step 3 of RCholeskyQR: Q = X R^{-1}, the method's dominant operation
// ("mainly determined by the computation of X R^{-1} ... m n^2 flops").
//
// tri prep: W = R^{-1} row by row, w_i R = e_i solved by forward substitution (the same row-wise
//           recurrence the paper applies to every row of X), one warp per row of W.
// tall solve: Q = X W as an FP64 tensor-core (DMMA m16n8k4) tiled GEMM that reads X a second time
//           and writes Q once ("multiplies by R^{-1} tile by tile", north star).  W is upper
//           triangular, so output column block [n0, n0+NT) only needs K rows [0, n0+NT) and each
//           8-column MMA tile skips the k-steps below its diagonal (mn^2 flops, not 2mn^2).
//           X is widened to fp64 on the way into shared memory; Q is rounded once to X's dtype.
#include <cuda_runtime.h>
#include <algorithm>
#include "internal.cuh"

namespace rcq {

// --------------------------------------------------------------------------------------------
__global__ void check_diag_kernel(const double* __restrict__ R, int n, int* status) {
  int bad = 0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const double d = R[(size_t)j * n + j];
    if (d == 0.0 || !isfinite(d)) bad = 1;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(status, kStSingular);
}

// W (n x n row-major, upper triangular): row i satisfies w_i R = e_i.
constexpr int INV_WARPS = 4;
__global__ void __launch_bounds__(32 * INV_WARPS)
tri_inverse_kernel(const double* __restrict__ R, int n, double* __restrict__ W, const int* status) {
  extern __shared__ __align__(16) double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x * INV_WARPS + warp;
  if (i >= n || *status) return;
  double* w = smem + (size_t)warp * n;
  for (int j = lane; j < n; j += 32) w[j] = 0.0;
  __syncwarp();
  if (lane == 0) w[i] = 1.0 / R[(size_t)i * n + i];
  __syncwarp();
  for (int j = i + 1; j < n; ++j) {
    double s = 0.0;
    for (int l = i + lane; l < j; l += 32) s += w[l] * R[(size_t)l * n + j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) w[j] = -s / R[(size_t)j * n + j];
    __syncwarp();
  }
  for (int j = lane; j < n; j += 32) W[(size_t)i * n + j] = w[j];
}

// --------------------------------------------------------------------------------------------
constexpr int KCT = 16;  // K rows of W per pipeline chunk

template <int WM, int WN, int MW, int NW>
struct TCfg {
  static constexpr int TM = 16 * MW * WM;
  static constexpr int NT = 8 * NW * WN;
  static constexpr int THREADS = 32 * WM * WN;
  static constexpr int XS_LD = KCT + 4;   // 20 doubles: A-fragment (X) loads conflict-free
  static constexpr int WS_LD = NT + 4;    // B-fragment (W) loads conflict-free
  static constexpr size_t SMEM = sizeof(double) * (2 * (size_t)TM * XS_LD + 2 * (size_t)KCT * WS_LD);
  static constexpr int XREG = (TM * KCT + THREADS - 1) / THREADS;
  static constexpr int WREG = (KCT * NT + THREADS - 1) / THREADS;
};

template <typename TX> __device__ __forceinline__ TX to_out(double v);
template <> __device__ __forceinline__ double to_out<double>(double v) { return v; }
template <> __device__ __forceinline__ float to_out<float>(double v) { return __double2float_rn(v); }

// Warp (wm, wn) owns m16 strips wm*MW .. wm*MW+MW-1 and the interleaved n8 tiles wn + WN*u
// (interleaving balances the triangular work across the warps of a CTA).
template <typename TX, int WM, int WN, int MW, int NW>
__global__ void __launch_bounds__(32 * WM * WN, 1)
trsm_kernel(const TX* __restrict__ X, int64_t m, int n, int64_t ldx, const double* __restrict__ W,
            TX* __restrict__ Q, int64_t ldq, int tiles_n, const int* status) {
  using C = TCfg<WM, WN, MW, NW>;
  if (*status) return;  // singular / non-finite: Q is left unwritten
  extern __shared__ __align__(16) double smem[];
  double* Xs = smem;                               // [2][TM][XS_LD]
  double* Ws = smem + 2 * C::TM * C::XS_LD;        // [2][KCT][WS_LD]
  const int tn = blockIdx.x % tiles_n;
  const int64_t row0 = (int64_t)(blockIdx.x / tiles_n) * C::TM;
  const int n0 = tn * C::NT;
  const int kend = min(n, n0 + C::NT);
  const int nchunks = (kend + KCT - 1) / KCT;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  const int wm = warp % WM, wn = warp / WM;

  double acc[MW][NW][4];
#pragma unroll
  for (int a = 0; a < MW; ++a)
#pragma unroll
    for (int b = 0; b < NW; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][b][c] = 0.0;

  TX xr[C::XREG];
  double wr[C::WREG];
  auto load = [&](int k0) {
#pragma unroll
    for (int u = 0; u < C::XREG; ++u) {
      const int c = tid + u * C::THREADS;
      const int ii = c / KCT, kk = c % KCT;
      TX v = TX(0);
      if (c < C::TM * KCT && row0 + ii < m && k0 + kk < n) v = __ldcs(X + (row0 + ii) * ldx + k0 + kk);
      xr[u] = v;
    }
#pragma unroll
    for (int u = 0; u < C::WREG; ++u) {
      const int c = tid + u * C::THREADS;
      const int kk = c / C::NT, jj = c % C::NT;
      double v = 0.0;
      if (c < KCT * C::NT && k0 + kk < n && n0 + jj < n) v = __ldg(W + (size_t)(k0 + kk) * n + n0 + jj);
      wr[u] = v;
    }
  };
  auto store = [&](int buf) {
    double* Xb = Xs + buf * C::TM * C::XS_LD;
    double* Wb = Ws + buf * KCT * C::WS_LD;
#pragma unroll
    for (int u = 0; u < C::XREG; ++u) {
      const int c = tid + u * C::THREADS;
      if (c < C::TM * KCT) Xb[(c / KCT) * C::XS_LD + (c % KCT)] = (double)xr[u];
    }
#pragma unroll
    for (int u = 0; u < C::WREG; ++u) {
      const int c = tid + u * C::THREADS;
      if (c < KCT * C::NT) Wb[(c / C::NT) * C::WS_LD + (c % C::NT)] = wr[u];
    }
  };

  // last K index each of this warp's n8 tiles needs (global column index of its last column)
  int chi[NW];
#pragma unroll
  for (int u = 0; u < NW; ++u) chi[u] = n0 + (wn + WN * u) * 8 + 7;

  load(0);
  store(0);
  __syncthreads();
  for (int ch = 0; ch < nchunks; ++ch) {
    const int buf = ch & 1;
    const bool more = ch + 1 < nchunks;
    if (more) load((ch + 1) * KCT);
    const double* Xb = Xs + buf * C::TM * C::XS_LD;
    const double* Wb = Ws + buf * KCT * C::WS_LD;
#pragma unroll
    for (int ks = 0; ks < KCT / 4; ++ks) {
      const int kg = ch * KCT + 4 * ks;  // global K index of this k-step
      double a0[MW], a1[MW];
#pragma unroll
      for (int mw = 0; mw < MW; ++mw) {
        const int r = (wm * MW + mw) * 16 + g;
        a0[mw] = Xb[r * C::XS_LD + 4 * ks + t4];
        a1[mw] = Xb[(r + 8) * C::XS_LD + 4 * ks + t4];
      }
#pragma unroll
      for (int u = 0; u < NW; ++u) {
        if (kg <= chi[u]) {  // warp-uniform: skip MMAs entirely below the diagonal of W
          const double b = Wb[(4 * ks + t4) * C::WS_LD + (wn + WN * u) * 8 + g];
#pragma unroll
          for (int mw = 0; mw < MW; ++mw) dmma_16x8x4(acc[mw][u], a0[mw], a1[mw], b);
        }
      }
    }
    if (more) store(buf ^ 1);
    __syncthreads();
  }

#pragma unroll
  for (int mw = 0; mw < MW; ++mw)
#pragma unroll
    for (int u = 0; u < NW; ++u) {
      const int64_t r = row0 + (wm * MW + mw) * 16 + g;
      const int c = n0 + (wn + WN * u) * 8 + 2 * t4;
      if (r < m) {
        if (c < n) Q[r * ldq + c] = to_out<TX>(acc[mw][u][0]);
        if (c + 1 < n) Q[r * ldq + c + 1] = to_out<TX>(acc[mw][u][1]);
      }
      if (r + 8 < m) {
        if (c < n) Q[(r + 8) * ldq + c] = to_out<TX>(acc[mw][u][2]);
        if (c + 1 < n) Q[(r + 8) * ldq + c + 1] = to_out<TX>(acc[mw][u][3]);
      }
    }
}

// --------------------------------------------------------------------------------------------
template <int WM, int WN, int MW, int NW>
static TrsmLaunch fill_t(int kind, int n) {
  using C = TCfg<WM, WN, MW, NW>;
  TrsmLaunch L{};
  L.kind = kind; L.TM = C::TM; L.NT = C::NT; L.threads = C::THREADS; L.smem = C::SMEM;
  L.tiles_n = (n + C::NT - 1) / C::NT;
  return L;
}

TrsmLaunch plan_trsm(int n, int dtype, size_t smem_optin) {
  (void)dtype; (void)smem_optin;
  if (n <= 24) return fill_t<4, 1, 1, 3>(kTrsm64x24, n);
  if (n <= 64) return fill_t<4, 2, 2, 4>(kTrsm128x64, n);
  if (n <= 112) return fill_t<4, 2, 2, 7>(kTrsm128x112, n);
  return fill_t<4, 4, 2, 4>(kTrsm128x128, n);
}

template <typename TX, int WM, int WN, int MW, int NW>
static cudaError_t launch_t(const TrsmLaunch& L, const void* X, int64_t m, int n, int64_t ldx, const double* W,
                            void* Q, int64_t ldq, const int* status, cudaStream_t st) {
  auto kern = trsm_kernel<TX, WM, WN, MW, NW>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem);
  if (e != cudaSuccess) return e;
  const int64_t tiles_m = (m + L.TM - 1) / L.TM;
  if (tiles_m == 0) return cudaSuccess;
  kern<<<(unsigned)(tiles_m * L.tiles_n), L.threads, L.smem, st>>>((const TX*)X, m, n, ldx, W, (TX*)Q, ldq,
                                                                   L.tiles_n, status);
  return cudaGetLastError();
}

template <typename TX>
static cudaError_t launch_trsm_typed(const TrsmLaunch& L, const void* X, int64_t m, int n, int64_t ldx,
                                     const double* W, void* Q, int64_t ldq, const int* status, cudaStream_t st) {
  switch (L.kind) {
    case kTrsm64x24: return launch_t<TX, 4, 1, 1, 3>(L, X, m, n, ldx, W, Q, ldq, status, st);
    case kTrsm128x64: return launch_t<TX, 4, 2, 2, 4>(L, X, m, n, ldx, W, Q, ldq, status, st);
    case kTrsm128x112: return launch_t<TX, 4, 2, 2, 7>(L, X, m, n, ldx, W, Q, ldq, status, st);
    default: return launch_t<TX, 4, 4, 2, 4>(L, X, m, n, ldx, W, Q, ldq, status, st);
  }
}

cudaError_t launch_trsm(const TrsmLaunch& L, const void* X, int dtype, int64_t m, int n, int64_t ldx,
                        const double* W, void* Q, int64_t ldq, const int* status, cudaStream_t st) {
  return dtype == RCHOLQR_F64 ? launch_trsm_typed<double>(L, X, m, n, ldx, W, Q, ldq, status, st)
                              : launch_trsm_typed<float>(L, X, m, n, ldx, W, Q, ldq, status, st);
}

cudaError_t launch_tri_inverse(const double* R, int n, double* W, int* status, cudaStream_t st) {
  const size_t smem = sizeof(double) * (size_t)n * INV_WARPS;
  cudaError_t e = cudaFuncSetAttribute(tri_inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  tri_inverse_kernel<<<(n + INV_WARPS - 1) / INV_WARPS, 32 * INV_WARPS, smem, st>>>(R, n, W, status);
  return cudaGetLastError();
}

cudaError_t launch_check_diag(const double* R, int n, int* status, cudaStream_t st) {
  check_diag_kernel<<<1, 256, 0, st>>>(R, n, status);
  return cudaGetLastError();
}

}  // namespace rcq
