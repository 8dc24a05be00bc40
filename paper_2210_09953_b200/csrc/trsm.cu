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
#include <cstdlib>
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

// Same W for n <= 128 (the tcgen05 digit solve's prep): R staged once per CTA in shared memory and
// the substitution done right-looking -- lane c keeps the residual s_c of w_i R = e_i for columns
// c = lane + 32 q; at step j the owner lane's s_j is final, w_ij = s_j / R_jj is broadcast and every
// lane updates s_c -= w_ij R_jc (c > j).  One shuffle + one division per step instead of a global
// load chain and a 5-step shuffle reduction; the diagonal reciprocals are taken once, so a step is
// a shuffle, a multiply and the lane's FMAs (0.074 ms -> a few us at n = 100).
constexpr int INVS_WARPS = 8;
__global__ void __launch_bounds__(32 * INVS_WARPS)
tri_inverse_small_kernel(const double* __restrict__ R, int n, double* __restrict__ W, const int* status) {
  if (*status) return;
  extern __shared__ __align__(16) double rsm[];        // R, n x n; then 1 / R_jj
  double* dinv = rsm + (size_t)n * n;
  const int nn = n * n;
  for (int t0 = 0; t0 < nn; t0 += 8 * (int)blockDim.x) {                 // 8 loads in flight per thread
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int t = t0 + u * (int)blockDim.x + (int)threadIdx.x;
      v[u] = t < nn ? R[t] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int t = t0 + u * (int)blockDim.x + (int)threadIdx.x;
      if (t < nn) rsm[t] = v[u];
    }
  }
  for (int t = threadIdx.x; t < n; t += blockDim.x) dinv[t] = 1.0 / R[(size_t)t * n + t];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x * INVS_WARPS + warp;
  if (i >= n) return;
  double s[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) s[q] = (lane + 32 * q == i) ? 1.0 : 0.0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    for (int jj = 0; jj < 32; ++jj) {
      const int j = 32 * q + jj;
      if (j >= n) break;
      if (j < i) continue;                               // w_ij = 0 below the diagonal
      const double z = __shfl_sync(0xffffffffu, s[q], jj) * dinv[j];   // w_ij (reciprocal: W is fp64 to ~1 ulp)
      if (lane == jj) s[q] = z;
#pragma unroll
      for (int q2 = q; q2 < 4; ++q2) {
        const int c = lane + 32 * q2;
        if (c > j && c < n) s[q2] = fma(-z, rsm[(size_t)j * n + c], s[q2]);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (lane + 32 * q < n) W[(size_t)i * n + lane + 32 * q] = s[q];
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
  if (n <= 128 && !getenv("RCHOLQR_TRI_INVERSE_OLD")) {
    const size_t sm = sizeof(double) * (size_t)n * (n + 1);
    cudaError_t e = cudaFuncSetAttribute(tri_inverse_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    tri_inverse_small_kernel<<<(n + INVS_WARPS - 1) / INVS_WARPS, 32 * INVS_WARPS, sm, st>>>(R, n, W, status);
    return cudaGetLastError();
  }
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

// ============================================================================================
// Blocked forward substitution (the default tall solve).  Columns are processed in blocks J of
// width 32 (last block ragged, multiple of 8):
//     T_J = X_J - Q_{<J} R_{<J,J}          (DMMA, K = 32 J)
//     Q_J = T_J  Winv_JJ                   (DMMA, K = 32, Winv_JJ = R_JJ^{-1} by row substitution)
// i.e. the paper's row-wise forward substitution with only the 32x32 diagonal
// blocks inverted, which keeps the row-wise backward stability of substitution (an explicit full
// R^{-1} lost 4x in ||I - (Theta Q)^T Theta Q|| at n=1024, kappa=1e12 -- DESIGN.md "Tall solve").
// M (npad x npad) packs both operands: M[L,J] = -R_{L,J} (L < J), M[J,J] = Winv_JJ, 0 below.
constexpr int TB = 32;           // diagonal block width



// X fragment loads of the warp-pair kernel below (the X values of block J+1 are prefetched into
// registers while block J is solved).
template <typename TX>
__device__ __forceinline__ void load_x_frag(const TX* __restrict__ X, int64_t m, int n, int64_t ldx, int64_t r0, int c,
                                            int g, TX (&v)[4]) {
  const int64_t ra = r0 + g, rb = r0 + g + 8;
  v[0] = (ra < m && c < n) ? __ldcs(X + ra * ldx + c) : TX(0);
  v[1] = (ra < m && c + 1 < n) ? __ldcs(X + ra * ldx + c + 1) : TX(0);
  v[2] = (rb < m && c < n) ? __ldcs(X + rb * ldx + c) : TX(0);
  v[3] = (rb < m && c + 1 < n) ? __ldcs(X + rb * ldx + c + 1) : TX(0);
}


// Warp-pair variant: two warps share one 16-row tile (each owns half of the 8-column MMA tiles of a
// block), so 16 warps run with the same shared-memory slabs as 8 -- twice the warps per SMSP to
// hide DMMA/shared-memory latency.  The pair synchronises with a 64-thread named barrier.
__device__ __forceinline__ void pair_sync(int id) { asm volatile("bar.sync %0, 64;\n" ::"r"(id) : "memory"); }

template <typename TX, int PAIRS>
__global__ void __launch_bounds__(64 * PAIRS, 1)
trsm_pair_kernel(const TX* __restrict__ X, int64_t m, int n, int NPAD, int64_t ldx, const double* __restrict__ Mg,
                 TX* __restrict__ Q, int64_t ldq, const int* status) {
  if (*status) return;
  extern __shared__ __align__(16) double smem_w[];
  const int LD = NPAD + 4;
  double* Ms = smem_w;                            // [NPAD][LD]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  const int pair = warp >> 1, h = warp & 1;
  double* Aw = smem_w + (size_t)NPAD * LD + (size_t)pair * 16 * LD;   // the pair's [16][LD] slab
  for (int c = threadIdx.x; c < NPAD * NPAD; c += 64 * PAIRS) Ms[(c / NPAD) * LD + (c % NPAD)] = Mg[c];
  __syncthreads();
  const int NBLK = (NPAD + TB - 1) / TB;
  const int64_t ntiles = (m + 15) / 16;
  const int64_t gp = (int64_t)blockIdx.x * PAIRS + pair, np = (int64_t)gridDim.x * PAIRS;
  constexpr int HU = TB / 16;                     // 8-column MMA tiles per warp per block (2)
  TX xn[HU][4];
  auto prefetch = [&](int64_t tile, int J) {
#pragma unroll
    for (int v = 0; v < HU; ++v)
      load_x_frag(X, m, n, ldx, tile * 16, J * TB + 8 * (HU * h + v) + 2 * t4, g, xn[v]);
  };
  if (gp < ntiles) prefetch(gp, 0);
  const double* arow = Aw + g * LD + t4;
  for (int64_t tile = gp; tile < ntiles; tile += np) {
    const int64_t r0 = tile * 16;
    for (int J = 0; J < NBLK; ++J) {
      const int c0 = J * TB;
      const int nt8 = min(TB, NPAD - c0) / 8;
      double acc[HU][4];
#pragma unroll
      for (int v = 0; v < HU; ++v)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[v][e] = (double)xn[v][e];
      if (J + 1 < NBLK) prefetch(tile, J + 1);
      else if (tile + np < ntiles) prefetch(tile + np, 0);
      const int u0 = HU * h;                      // this warp's first 8-column tile of the block
      const bool full = nt8 == TB / 8;
      // phase 1: T_J = X_J + Q_{<J} (-R_{<J,J}) for this warp's tiles
      if (full) {
#pragma unroll 4
        for (int ks = 0; ks < c0 / 4; ++ks) {
          const double a0 = arow[4 * ks], a1 = arow[8 * LD + 4 * ks];
          const double* mrow = Ms + (4 * ks + t4) * LD + c0 + 8 * u0 + g;
          const double b0 = mrow[0], b1 = mrow[8];
          dmma_16x8x4(acc[0], a0, a1, b0);
          dmma_16x8x4(acc[1], a0, a1, b1);
        }
      } else {
        for (int ks = 0; ks < c0 / 4; ++ks) {
          const double a0 = arow[4 * ks], a1 = arow[8 * LD + 4 * ks];
          const double* mrow = Ms + (4 * ks + t4) * LD + c0 + g;
#pragma unroll
          for (int v = 0; v < HU; ++v)
            if (u0 + v < nt8) dmma_16x8x4(acc[v], a0, a1, mrow[8 * (u0 + v)]);
        }
      }
#pragma unroll
      for (int v = 0; v < HU; ++v) {
        if (u0 + v < nt8) {
          double* tp = Aw + g * LD + c0 + 8 * (u0 + v) + 2 * t4;
          tp[0] = acc[v][0]; tp[1] = acc[v][1]; tp[8 * LD] = acc[v][2]; tp[8 * LD + 1] = acc[v][3];
        }
      }
      pair_sync(1 + pair);                        // all of T_J visible to both warps
      // phase 2: Q_J = T_J Winv_JJ (upper triangular: skip k-steps past each 8-column tile)
#pragma unroll
      for (int v = 0; v < HU; ++v)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[v][e] = 0.0;
#pragma unroll
      for (int ks = 0; ks < TB / 4; ++ks) {
        if (4 * ks < 8 * nt8 && 4 * ks <= 8 * (u0 + HU - 1) + 7) {
          const double a0 = arow[c0 + 4 * ks], a1 = arow[8 * LD + c0 + 4 * ks];
          const double* mrow = Ms + (c0 + 4 * ks + t4) * LD + c0 + g;
#pragma unroll
          for (int v = 0; v < HU; ++v) {
            const int u = u0 + v;
            if (u < nt8 && 4 * ks <= 8 * u + 7) dmma_16x8x4(acc[v], a0, a1, mrow[8 * u]);
          }
        }
      }
      pair_sync(1 + pair);                        // both warps done reading T_J
#pragma unroll
      for (int v = 0; v < HU; ++v) {
        const int u = u0 + v;
        if (u < nt8) {
          const int col = c0 + 8 * u + 2 * t4;
          double* tp = Aw + g * LD + col;
          tp[0] = acc[v][0]; tp[1] = acc[v][1]; tp[8 * LD] = acc[v][2]; tp[8 * LD + 1] = acc[v][3];
          const int64_t ra = r0 + g, rb = r0 + g + 8;
          if (ra < m) {
            if (col < n) Q[ra * ldq + col] = to_out<TX>(acc[v][0]);
            if (col + 1 < n) Q[ra * ldq + col + 1] = to_out<TX>(acc[v][1]);
          }
          if (rb < m) {
            if (col < n) Q[rb * ldq + col] = to_out<TX>(acc[v][2]);
            if (col + 1 < n) Q[rb * ldq + col + 1] = to_out<TX>(acc[v][3]);
          }
        }
      }
      pair_sync(1 + pair);                        // Q_J history visible before the next block
    }
  }
}

// 128 < n <= 256: the warp-pair blocked substitution with M STREAMED instead of resident (npad^2
// doubles no longer fit next to the Q slabs).  All pairs of the CTA advance through the column blocks J
// together; before each J the CTA stages M(0 : c0 + TB, c0 : c0 + TB) -- the only part of M block J
// reads -- from L2 into one [NPAD][TB + 4] buffer.  That costs (c0 + TB) TB doubles per J per CTA,
// ~5% of the block's DMMA time.  The fp64 Q history (NPAD columns) stays in the pair's [16][LD] slab.
constexpr int MS_PAIRS = 4;
constexpr int MS_MLD = TB + 4;                    // = 4 (mod 16) doubles: fragment loads conflict-free

static size_t mstream_smem(int npad) {
  return sizeof(double) * ((size_t)npad * MS_MLD + (size_t)MS_PAIRS * 16 * (npad + 4));
}

template <typename TX>
__global__ void __launch_bounds__(64 * MS_PAIRS, 1)
trsm_mstream_kernel(const TX* __restrict__ X, int64_t m, int n, int NPAD, int64_t ldx, const double* __restrict__ Mg,
                    TX* __restrict__ Q, int64_t ldq, const int* status) {
  if (*status) return;
  extern __shared__ __align__(16) double smem_w[];
  const int LD = NPAD + 4;
  double* Mb = smem_w;                                              // [NPAD][MS_MLD]: column block J of M
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  const int pair = warp >> 1, h = warp & 1;
  double* Aw = smem_w + (size_t)NPAD * MS_MLD + (size_t)pair * 16 * LD;   // the pair's [16][LD] slab
  const int NBLK = (NPAD + TB - 1) / TB;
  const int64_t ntiles = (m + 15) / 16;
  constexpr int HU = TB / 16;
  TX xn[HU][4];
  auto prefetch = [&](int64_t tile, int J) {
#pragma unroll
    for (int v = 0; v < HU; ++v)
      load_x_frag(X, m, n, ldx, tile * 16, J * TB + 8 * (HU * h + v) + 2 * t4, g, xn[v]);
  };
  const int64_t step = (int64_t)gridDim.x * MS_PAIRS;
  const int64_t first = (int64_t)blockIdx.x * MS_PAIRS + pair;
  if (first < ntiles) prefetch(first, 0);
  const double* arow = Aw + g * LD + t4;
  for (int64_t base = (int64_t)blockIdx.x * MS_PAIRS; base < ntiles; base += step) {
    const int64_t tile = base + pair;
    const bool active = tile < ntiles;
    const int64_t r0 = tile * 16;
    for (int J = 0; J < NBLK; ++J) {
      const int c0 = J * TB;
      const int nt8 = min(TB, NPAD - c0) / 8;
      const int rows = min(NPAD, c0 + TB);
      __syncthreads();                                              // everyone done with block J-1's Mb
      for (int c = threadIdx.x; c < rows * (TB / 2); c += 64 * MS_PAIRS) {   // 16-byte cp.async, all in flight
        const int rr = c / (TB / 2), cc = 2 * (c % (TB / 2));
        const bool ok = c0 + cc < NPAD;
        const unsigned sa = (unsigned)__cvta_generic_to_shared(Mb + rr * MS_MLD + cc);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa),
                     "l"(ok ? Mg + (size_t)rr * NPAD + c0 + cc : Mg), "r"(ok ? 16 : 0));
      }
      asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
      __syncthreads();
      if (!active) continue;
      double acc[HU][4];
#pragma unroll
      for (int v = 0; v < HU; ++v)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[v][e] = (double)xn[v][e];
      if (J + 1 < NBLK) prefetch(tile, J + 1);
      else if (tile + step < ntiles) prefetch(tile + step, 0);
      const int u0 = HU * h;
      const bool full = nt8 == TB / 8;
      // phase 1: T_J = X_J + Q_{<J} (-R_{<J,J})
      if (full) {
#pragma unroll 4
        for (int ks = 0; ks < c0 / 4; ++ks) {
          const double a0 = arow[4 * ks], a1 = arow[8 * LD + 4 * ks];
          const double* mrow = Mb + (4 * ks + t4) * MS_MLD + 8 * u0 + g;
          dmma_16x8x4(acc[0], a0, a1, mrow[0]);
          dmma_16x8x4(acc[1], a0, a1, mrow[8]);
        }
      } else {
        for (int ks = 0; ks < c0 / 4; ++ks) {
          const double a0 = arow[4 * ks], a1 = arow[8 * LD + 4 * ks];
          const double* mrow = Mb + (4 * ks + t4) * MS_MLD + g;
#pragma unroll
          for (int v = 0; v < HU; ++v)
            if (u0 + v < nt8) dmma_16x8x4(acc[v], a0, a1, mrow[8 * (u0 + v)]);
        }
      }
#pragma unroll
      for (int v = 0; v < HU; ++v) {
        if (u0 + v < nt8) {
          double* tp = Aw + g * LD + c0 + 8 * (u0 + v) + 2 * t4;
          tp[0] = acc[v][0]; tp[1] = acc[v][1]; tp[8 * LD] = acc[v][2]; tp[8 * LD + 1] = acc[v][3];
        }
      }
      pair_sync(1 + pair);
      // phase 2: Q_J = T_J Winv_JJ
#pragma unroll
      for (int v = 0; v < HU; ++v)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[v][e] = 0.0;
#pragma unroll
      for (int ks = 0; ks < TB / 4; ++ks) {
        if (4 * ks < 8 * nt8 && 4 * ks <= 8 * (u0 + HU - 1) + 7) {
          const double a0 = arow[c0 + 4 * ks], a1 = arow[8 * LD + c0 + 4 * ks];
          const double* mrow = Mb + (c0 + 4 * ks + t4) * MS_MLD + g;
#pragma unroll
          for (int v = 0; v < HU; ++v) {
            const int u = u0 + v;
            if (u < nt8 && 4 * ks <= 8 * u + 7) dmma_16x8x4(acc[v], a0, a1, mrow[8 * u]);
          }
        }
      }
      pair_sync(1 + pair);
#pragma unroll
      for (int v = 0; v < HU; ++v) {
        const int u = u0 + v;
        if (u < nt8) {
          const int col = c0 + 8 * u + 2 * t4;
          double* tp = Aw + g * LD + col;
          tp[0] = acc[v][0]; tp[1] = acc[v][1]; tp[8 * LD] = acc[v][2]; tp[8 * LD + 1] = acc[v][3];
          const int64_t ra = r0 + g, rb = r0 + g + 8;
          if (ra < m) {
            if (col < n) Q[ra * ldq + col] = to_out<TX>(acc[v][0]);
            if (col + 1 < n) Q[ra * ldq + col + 1] = to_out<TX>(acc[v][1]);
          }
          if (rb < m) {
            if (col < n) Q[rb * ldq + col] = to_out<TX>(acc[v][2]);
            if (col + 1 < n) Q[rb * ldq + col + 1] = to_out<TX>(acc[v][3]);
          }
        }
      }
      pair_sync(1 + pair);
    }
  }
}

bool trsm_mstream_applicable(int n, size_t smem_optin) {
  if (n <= 128 || n > 256 || getenv("RCHOLQR_NO_MSTREAM")) return false;
  return mstream_smem((n + 7) / 8 * 8) <= smem_optin;
}

cudaError_t launch_trsm_mstream(const void* X, int dtype, int64_t m, int n, int64_t ldx, const double* M, void* Q,
                                int64_t ldq, const int* status, int sms, cudaStream_t st) {
  const int npad = (n + 7) / 8 * 8;
  const size_t smem = mstream_smem(npad);
  const int64_t ntiles = (m + 15) / 16;
  const int grid = (int)std::min<int64_t>((ntiles + MS_PAIRS - 1) / MS_PAIRS, sms);
  if (grid == 0) return cudaSuccess;
  cudaError_t e;
  if (dtype == RCHOLQR_F64) {
    e = cudaFuncSetAttribute(trsm_mstream_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    trsm_mstream_kernel<double><<<grid, 64 * MS_PAIRS, smem, st>>>((const double*)X, m, n, npad, ldx, M, (double*)Q,
                                                                  ldq, status);
  } else {
    e = cudaFuncSetAttribute(trsm_mstream_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    trsm_mstream_kernel<float><<<grid, 64 * MS_PAIRS, smem, st>>>((const float*)X, m, n, npad, ldx, M, (float*)Q,
                                                                 ldq, status);
  }
  return cudaGetLastError();
}

// M = [-R_{<J,J}; Winv_JJ] packed (npad x npad, zero padded), diagonal blocks of width tb
// (32 for the resident solves, 64/128 for the streamed one; tb <= 128).  One warp per row i of M:
// the row of Winv_JJ solves w R_JJ = e_i by forward substitution, lane l holding w[Jb + l + 32 t].
__global__ void tri_prep_blocked_kernel(const double* __restrict__ R, int n, int npad, int tb, double* __restrict__ M,
                                        const int* status) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int i = warp;
  if (i >= npad || *status) return;
  const int Jb = (i / tb) * tb;                     // first column of i's diagonal block
  const int be = min(Jb + tb, n);                   // end of the block (within n)
  double w[4] = {0.0, 0.0, 0.0, 0.0};               // w[t] = Winv row entry at column Jb + lane + 32 t
  if (i < n) {
    if (lane == (i - Jb) % 32) {
      const double v = 1.0 / R[(size_t)i * n + i];
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (t == (i - Jb) / 32) w[t] = v;
    }
    for (int j = i + 1; j < be; ++j) {
      double s = 0.0;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int l = Jb + lane + 32 * t;
        if (l >= i && l < j) s += w[t] * R[(size_t)l * n + j];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == (j - Jb) % 32) {
        const double v = -s / R[(size_t)j * n + j];
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (t == (j - Jb) / 32) w[t] = v;
      }
    }
  }
  for (int base = 0; base < npad; base += 32) {   // uniform trip count: shuffles are convergent
    const int c = base + lane;
    const int tsel = (base - Jb) >= 0 ? (base - Jb) / 32 : 0;   // same for all lanes of this chunk
    double wc = 0.0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const double vv = __shfl_sync(0xffffffffu, w[t], lane);
      if (t == tsel) wc = vv;
    }
    double v = 0.0;
    if (i < n && c < n) {
      if (c >= Jb + tb) v = -R[(size_t)i * n + c];
      else if (c >= Jb) v = wc;
    }
    if (c < npad) M[(size_t)i * npad + c] = v;
  }
}

// ---------------------------------------------------------------------------------------------
static size_t warp_smem(int npad, int warps) { return sizeof(double) * (size_t)(npad + 4) * (npad + 16 * warps); }

// Warp pairs per CTA of the blocked substitution for n <= 128 (fp64 X, or fp32 X off the tcgen05 path):
// 8 when their Q-history slabs and M fit in shared memory (n <= 112), else 4 (n <= 128).
int trsm_pair_count(int n, size_t smem_optin) {
  const int npad = (n + 7) / 8 * 8;
  if (n > 128) return 0;
  if (warp_smem(npad, 8) <= smem_optin) return 8;
  if (warp_smem(npad, 4) <= smem_optin) return 4;
  return 0;
}

template <typename TX, int PAIRS>
static cudaError_t launch_p(const void* X, int64_t m, int n, int64_t ldx, const double* M, void* Q, int64_t ldq,
                            const int* status, int sms, cudaStream_t st) {
  const int npad = (n + 7) / 8 * 8;
  const size_t smem = warp_smem(npad, PAIRS);
  auto kern = trsm_pair_kernel<TX, PAIRS>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t ntiles = (m + 15) / 16;
  const int grid = (int)std::min<int64_t>((ntiles + PAIRS - 1) / PAIRS, sms);
  if (grid == 0) return cudaSuccess;
  kern<<<grid, 64 * PAIRS, smem, st>>>((const TX*)X, m, n, npad, ldx, M, (TX*)Q, ldq, status);
  return cudaGetLastError();
}

cudaError_t launch_trsm_pairs(int pairs, const void* X, int dtype, int64_t m, int n, int64_t ldx, const double* M,
                              void* Q, int64_t ldq, const int* status, int sms, cudaStream_t st) {
  if (dtype == RCHOLQR_F64)
    return pairs == 8 ? launch_p<double, 8>(X, m, n, ldx, M, Q, ldq, status, sms, st)
                      : launch_p<double, 4>(X, m, n, ldx, M, Q, ldq, status, sms, st);
  return pairs == 8 ? launch_p<float, 8>(X, m, n, ldx, M, Q, ldq, status, sms, st)
                    : launch_p<float, 4>(X, m, n, ldx, M, Q, ldq, status, sms, st);
}

cudaError_t launch_tri_prep_blocked(const double* R, int n, double* M, int* status, cudaStream_t st, int tb,
                                    int npad) {
  if (npad <= 0) npad = (n + 7) / 8 * 8;
  const int warps_per_block = 4;
  tri_prep_blocked_kernel<<<(npad + warps_per_block - 1) / warps_per_block, 32 * warps_per_block, 0, st>>>(
      R, n, npad, tb, M, status);
  return cudaGetLastError();
}

}  // namespace rcq
