// sketch.cu -- step 1 of RCholeskyQR: P = Theta X, fp64 accumulation.
//
// Gaussian Theta: a GEMM with M = k (Theta rows), N = n, K = m (rows of X).  Each CTA owns a
// KT x NT tile of P and a contiguous range of X rows ("split"); per 32-row chunk it
//   * generates the KT x 32 Theta tile in registers (Philox4x32-10 + Box-Muller, theta.cuh) and
//     parks it in shared memory as fp64 (exact: Theta's draws are fp32),
//   * stages the 32 x NT X tile (coalesced loads, fp32 -> fp64 exact widening),
//   * runs DMMA m16n8k4 (FP64 tensor core) with register-resident accumulators,
// double-buffered so the next chunk's generation and loads overlap this chunk's MMAs.  X is read
// from HBM once per (tile_k) -- exactly once when one tile covers P (C1, C2).  Per-CTA partials
// go to a workspace and are summed in a fixed order (deterministic, bitwise reproducible), then
// scaled once by fl(1/sqrt(k)) (reading A4).
//
// Sparse-sign Theta: per X row, nnz_per_col (row, sign) pairs; each warp owns one block of
// k/nnz rows of a shared-memory P tile, so the scatter-add is conflict- and atomic-free.
#include <cuda_runtime.h>
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <type_traits>
#include "internal.cuh"
#include "theta.cuh"

namespace rcq {

constexpr int KC = 32;  // X rows per pipeline chunk

template <int WM, int WN, int MW, int NW>
struct GCfg {
  static constexpr int KT = 16 * MW * WM;
  static constexpr int NT = 8 * NW * WN;
  static constexpr int THREADS = 32 * WM * WN;
  static constexpr int TS_LD = KC + 4;  // 36 doubles = 72 words: A-fragment loads conflict-free
  static constexpr int XS_LD = NT + 4;  // NT+4 = 4 or 12 (mod 16): B-fragment loads conflict-free
  static constexpr size_t SMEM = sizeof(double) * (2 * (size_t)KT * TS_LD + 2 * (size_t)KC * XS_LD);
  static constexpr int XREG = (KC * NT + THREADS - 1) / THREADS;
};

template <typename TX, int WM, int WN, int MW, int NW>
__global__ void __launch_bounds__(32 * WM * WN, 1)
sketch_gauss_kernel(const TX* __restrict__ X, int64_t m, int n, int64_t ldx, int64_t row_offset, int k,
                    uint64_t seed, int tiles_k, int tiles_n, int64_t rows_per_split,
                    double* __restrict__ part) {
  using C = GCfg<WM, WN, MW, NW>;
  extern __shared__ __align__(16) double smem[];
  double* Ts = smem;                              // [2][KT][TS_LD]  Theta tile (row r, X-row i)
  double* Xs = smem + 2 * C::KT * C::TS_LD;       // [2][KC][XS_LD]  X tile (X-row i, column j)

  const int tiles = tiles_k * tiles_n;
  const int tile = blockIdx.x % tiles, split = blockIdx.x / tiles;
  const int tk = tile % tiles_k, tn = tile / tiles_k;
  const int r0 = tk * C::KT, n0 = tn * C::NT;
  const int64_t i_begin = (int64_t)split * rows_per_split;
  const int64_t i_end = min(m, i_begin + rows_per_split);
  const int nchunks = i_end > i_begin ? (int)((i_end - i_begin + KC - 1) / KC) : 0;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  const int wm = warp % WM, wn = warp / WM;

  double acc[MW][NW][4];
#pragma unroll
  for (int a = 0; a < MW; ++a)
#pragma unroll
    for (int b = 0; b < NW; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][b][c] = 0.0;

  // Theta tile for X rows i0 .. i0+KC-1: one Philox call -> 4 consecutive Theta rows.
  auto gen_theta = [&](int buf, int64_t i0) {
    double* T = Ts + buf * C::KT * C::TS_LD;
    for (int c = tid; c < (C::KT / 4) * KC; c += C::THREADS) {
      const int qq = c / KC, ii = c % KC;
      const int rb = r0 + 4 * qq;
      float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
      if (i0 + ii < i_end && rb < k) z = gauss4(seed, (uint64_t)(row_offset + i0 + ii), (uint32_t)(rb >> 2));
      double* Tc = T + (4 * qq) * C::TS_LD + ii;
      Tc[0 * C::TS_LD] = (rb + 0 < k) ? (double)z.x : 0.0;
      Tc[1 * C::TS_LD] = (rb + 1 < k) ? (double)z.y : 0.0;
      Tc[2 * C::TS_LD] = (rb + 2 < k) ? (double)z.z : 0.0;
      Tc[3 * C::TS_LD] = (rb + 3 < k) ? (double)z.w : 0.0;
    }
  };
  TX xr[C::XREG];
  auto load_x = [&](int64_t i0) {
#pragma unroll
    for (int u = 0; u < C::XREG; ++u) {
      const int c = tid + u * C::THREADS;
      const int ii = c / C::NT, jj = c % C::NT;
      TX v = TX(0);
      if (c < KC * C::NT && i0 + ii < i_end && n0 + jj < n) v = __ldcs(X + (i0 + ii) * ldx + n0 + jj);
      xr[u] = v;
    }
  };
  auto store_x = [&](int buf) {
    double* Xb = Xs + buf * KC * C::XS_LD;
#pragma unroll
    for (int u = 0; u < C::XREG; ++u) {
      const int c = tid + u * C::THREADS;
      if (c < KC * C::NT) Xb[(c / C::NT) * C::XS_LD + (c % C::NT)] = (double)xr[u];
    }
  };

  if (nchunks > 0) {
    load_x(i_begin);
    gen_theta(0, i_begin);
    store_x(0);
  }
  __syncthreads();
  for (int ch = 0; ch < nchunks; ++ch) {
    const int buf = ch & 1;
    const bool more = ch + 1 < nchunks;
    const int64_t inext = i_begin + (int64_t)(ch + 1) * KC;
    if (more) load_x(inext);
    if (more) gen_theta(buf ^ 1, inext);
    const double* T = Ts + buf * C::KT * C::TS_LD;
    const double* Xb = Xs + buf * KC * C::XS_LD;
#pragma unroll
    for (int ks = 0; ks < KC / 4; ++ks) {
      double a0[MW], a1[MW];
#pragma unroll
      for (int mw = 0; mw < MW; ++mw) {
        const int row = (wm * MW + mw) * 16 + g;
        a0[mw] = T[row * C::TS_LD + 4 * ks + t4];
        a1[mw] = T[(row + 8) * C::TS_LD + 4 * ks + t4];
      }
#pragma unroll
      for (int nw = 0; nw < NW; ++nw) {
        const double b = Xb[(4 * ks + t4) * C::XS_LD + (wn * NW + nw) * 8 + g];
#pragma unroll
        for (int mw = 0; mw < MW; ++mw) dmma_16x8x4(acc[mw][nw], a0[mw], a1[mw], b);
      }
    }
    if (more) store_x(buf ^ 1);
    __syncthreads();
  }

  double* Pp = part + (size_t)split * (size_t)k * n;
#pragma unroll
  for (int mw = 0; mw < MW; ++mw)
#pragma unroll
    for (int nw = 0; nw < NW; ++nw) {
      const int row = r0 + (wm * MW + mw) * 16 + g;
      const int col = n0 + (wn * NW + nw) * 8 + 2 * t4;
      if (row < k) {
        if (col < n) Pp[(size_t)row * n + col] = acc[mw][nw][0];
        if (col + 1 < n) Pp[(size_t)row * n + col + 1] = acc[mw][nw][1];
      }
      if (row + 8 < k) {
        if (col < n) Pp[(size_t)(row + 8) * n + col] = acc[mw][nw][2];
        if (col + 1 < n) Pp[(size_t)(row + 8) * n + col + 1] = acc[mw][nw][3];
      }
    }
}

// ---------------------------------------------------------------------------------------------
// Sparse-sign sketch.  CTA = (column tile, split of rows).  smem: Ps[k][NTS] fp64 accumulators,
// Xs[KCS][NTS] fp64, sel[KCS][zeta] packed (row | sign << 31).
constexpr int KCS = 64;
constexpr int SPARSE_THREADS = 256;

template <typename TX>
__global__ void __launch_bounds__(SPARSE_THREADS)
sketch_sparse_kernel(const TX* __restrict__ X, int64_t m, int n, int64_t ldx, int64_t row_offset, int k,
                     int zeta, uint64_t seed, int tiles_n, int nts, int64_t rows_per_split,
                     double* __restrict__ part) {
  extern __shared__ __align__(16) double smem[];
  double* Ps = smem;                              // [k][nts]
  double* Xs = Ps + (size_t)k * nts;              // [KCS][nts]
  int* sel = reinterpret_cast<int*>(Xs + (size_t)KCS * nts);  // [KCS][zeta]
  const int tn = blockIdx.x % tiles_n, split = blockIdx.x / tiles_n;
  const int n0 = tn * nts;
  const int ncols = min(nts, n - n0);
  const int64_t i_begin = (int64_t)split * rows_per_split;
  const int64_t i_end = min(m, i_begin + rows_per_split);
  const int beta = k / zeta;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nwarps = SPARSE_THREADS / 32;
  for (int t = tid; t < k * nts; t += SPARSE_THREADS) Ps[t] = 0.0;
  for (int64_t i0 = i_begin; i0 < i_end; i0 += KCS) {
    const int rows = (int)min((int64_t)KCS, i_end - i0);
    __syncthreads();  // previous chunk fully consumed
    for (int c = tid; c < rows * ncols; c += SPARSE_THREADS) {
      const int ii = c / ncols, jj = c % ncols;
      Xs[ii * nts + jj] = (double)__ldcs(X + (i0 + ii) * ldx + n0 + jj);
    }
    for (int c = tid; c < rows * ((zeta + 7) / 8); c += SPARSE_THREADS) {
      const int ii = c / ((zeta + 7) / 8), q = c % ((zeta + 7) / 8);
      const uint4 w = philox_at(seed, (uint64_t)(row_offset + i0 + ii), (uint32_t)q, kDomainSparse);
      for (int tt = 0; tt < 8 && 8 * q + tt < zeta; ++tt) {
        const int t = 8 * q + tt;
        const uint32_t h = sparse_halfword(w, t);
        sel[ii * zeta + t] = sparse_row(h, t, beta) | ((h >> 15) ? (int)0x80000000u : 0);
      }
    }
    __syncthreads();
    for (int t = warp; t < zeta; t += nwarps) {   // warp owns Theta block t: rows t*beta .. +beta
      for (int ii = 0; ii < rows; ++ii) {
        const int s = sel[ii * zeta + t];
        double* prow = Ps + (size_t)(s & 0x7fffffff) * nts;
        const double* xrow = Xs + ii * nts;
        if (s < 0) {
          for (int j = lane; j < ncols; j += 32) prow[j] -= xrow[j];
        } else {
          for (int j = lane; j < ncols; j += 32) prow[j] += xrow[j];
        }
      }
    }
  }
  __syncthreads();
  double* Pp = part + (size_t)split * (size_t)k * n;
  for (int c = tid; c < k * ncols; c += SPARSE_THREADS) {
    const int r = c / ncols, j = c % ncols;
    Pp[(size_t)r * n + n0 + j] = Ps[r * nts + j];
  }
}

// Fixed-order sum of the per-split partials, one scaling, non-finite detection.
__global__ void sketch_reduce_kernel(const double* __restrict__ part, int splits, int64_t kn, double scale,
                                     double* __restrict__ P, int* status) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < kn;
       idx += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int sp = 0; sp < splits; ++sp) s += part[(size_t)sp * kn + idx];
    s *= scale;
    P[idx] = s;
    if (!isfinite(s)) atomicOr(status, kStNonfinite);
  }
}

// ---------------------------------------------------------------------------------------------
// Test export of Theta.
__global__ void theta_gauss_export_kernel(uint64_t seed, int k, int64_t row_offset, int64_t m, float* Z) {
  const int nq = (k + 3) / 4;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < m * nq; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = c % m;
    const int q = (int)(c / m);
    const float4 z = gauss4(seed, (uint64_t)(row_offset + i), (uint32_t)q);
    const float zz[4] = {z.x, z.y, z.z, z.w};
    for (int u = 0; u < 4 && 4 * q + u < k; ++u) Z[(int64_t)(4 * q + u) * m + i] = zz[u];
  }
}
__global__ void theta_sparse_export_kernel(uint64_t seed, int k, int zeta, int64_t row_offset, int64_t m,
                                           int32_t* rows, int8_t* signs) {
  const int beta = k / zeta;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    uint4 w = make_uint4(0, 0, 0, 0);
    for (int t = 0; t < zeta; ++t) {
      if ((t & 7) == 0) w = philox_at(seed, (uint64_t)(row_offset + i), (uint32_t)(t >> 3), kDomainSparse);
      const uint32_t h = sparse_halfword(w, t);
      if (rows) rows[i * zeta + t] = sparse_row(h, t, beta);
      if (signs) signs[i * zeta + t] = (h >> 15) ? (int8_t)-1 : (int8_t)1;
    }
  }
}

// ---------------------------------------------------------------------------------------------
// Host side.
template <int WM, int WN, int MW, int NW>
static void fill_gauss(SketchLaunch& L, int kind, int k, int n) {
  using C = GCfg<WM, WN, MW, NW>;
  L.kind = kind; L.KT = C::KT; L.NT = C::NT; L.threads = C::THREADS; L.smem = C::SMEM;
  L.tiles_k = (k + C::KT - 1) / C::KT;
  L.tiles_n = (n + C::NT - 1) / C::NT;
}

// Choose the number of row splits so tiles*splits fills whole waves of one CTA per SM.
static int choose_splits(int tiles, int sms) {
  int best = 1;
  double best_cost = 1e30;
  for (int s = 1; s <= 4 * sms; ++s) {
    const long ctas = (long)tiles * s;
    const long waves = (ctas + sms - 1) / sms;
    const double eff = (double)ctas / (double)(waves * sms);
    if (waves > 64) break;
    const double cost = (1.0 / eff) * (1.0 + 0.002 * s);  // mild preference for fewer partials
    if (cost < best_cost - 1e-12) { best_cost = cost; best = s; }
  }
  return best;
}

SketchLaunch plan_sketch(int k, int n, int dtype, int sketch, int zeta, int sms, size_t smem_optin) {
  SketchLaunch L{};
  (void)dtype;
  if (sketch == RCHOLQR_SPARSE_SIGN) {
    L.kind = kSketchSparse;
    L.threads = SPARSE_THREADS;
    L.KT = k;
    // columns per CTA so that Ps + Xs + sel fit comfortably (<= ~110 KB -> 2 CTAs / SM)
    size_t budget = std::min<size_t>(110 * 1024, smem_optin);
    int nts = n;
    while (nts > 8 && sizeof(double) * ((size_t)k * nts + (size_t)KCS * nts) + sizeof(int) * KCS * zeta > budget)
      nts = (nts + 1) / 2;
    L.NT = nts;
    L.tiles_k = 1;
    L.tiles_n = (n + nts - 1) / nts;
    L.smem = sizeof(double) * ((size_t)k * nts + (size_t)KCS * nts) + sizeof(int) * KCS * zeta;
    L.splits = choose_splits(L.tiles_n, 2 * sms);
    return L;
  }
  // Gaussian: pick the tile minimising padded work (tiles * KT * NT), ties -> larger tile.
  constexpr int NC = 5;
  SketchLaunch cand[NC];
  fill_gauss<4, 1, 1, 4>(cand[0], kSketchG64x32, k, n);
  fill_gauss<8, 1, 1, 8>(cand[1], kSketchG128x64, k, n);
  fill_gauss<7, 1, 1, 13>(cand[2], kSketchG112x104, k, n);
  fill_gauss<13, 1, 1, 7>(cand[3], kSketchG208x56, k, n);
  fill_gauss<4, 4, 2, 4>(cand[4], kSketchG128x128, k, n);
  int best = NC - 1;
  double best_cost = 1e300;
  const char* force = getenv("RCHOLQR_SKETCH_KIND");  // experiments only
  for (int c = 0; c < NC; ++c) {
    if (force && atoi(force) != cand[c].kind) continue;
    if (cand[c].smem > smem_optin) continue;
    // padded MMA work + a per-tile Theta regeneration/X re-read penalty
    const double padded = (double)cand[c].tiles_k * cand[c].KT * cand[c].tiles_n * cand[c].NT;
    const double cost = padded * (1.0 + 0.05 * (cand[c].tiles_n - 1) + 0.02 * (cand[c].tiles_k - 1)) /
                        (cand[c].threads >= 256 ? 1.0 : 1.15);
    if (cost < best_cost) { best_cost = cost; best = c; }
  }
  L = cand[best];
  L.splits = choose_splits(L.tiles_k * L.tiles_n, sms);
  return L;
}

template <typename TX, int WM, int WN, int MW, int NW>
static cudaError_t launch_g(const SketchLaunch& L, const void* X, int64_t m, int n, int64_t ldx, int64_t ro,
                            int k, uint64_t seed, int64_t rps, double* part, cudaStream_t st) {
  auto kern = sketch_gauss_kernel<TX, WM, WN, MW, NW>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem);
  if (e != cudaSuccess) return e;
  kern<<<L.tiles_k * L.tiles_n * L.splits, L.threads, L.smem, st>>>((const TX*)X, m, n, ldx, ro, k, seed,
                                                                    L.tiles_k, L.tiles_n, rps, part);
  return cudaGetLastError();
}

template <typename TX>
static cudaError_t launch_gauss_typed(const SketchLaunch& L, const void* X, int64_t m, int n, int64_t ldx,
                                      int64_t ro, int k, uint64_t seed, int64_t rps, double* part,
                                      cudaStream_t st) {
  switch (L.kind) {
    case kSketchG64x32: return launch_g<TX, 4, 1, 1, 4>(L, X, m, n, ldx, ro, k, seed, rps, part, st);
    case kSketchG128x64: return launch_g<TX, 8, 1, 1, 8>(L, X, m, n, ldx, ro, k, seed, rps, part, st);
    case kSketchG112x104: return launch_g<TX, 7, 1, 1, 13>(L, X, m, n, ldx, ro, k, seed, rps, part, st);
    case kSketchG208x56: return launch_g<TX, 13, 1, 1, 7>(L, X, m, n, ldx, ro, k, seed, rps, part, st);
    default: return launch_g<TX, 4, 4, 2, 4>(L, X, m, n, ldx, ro, k, seed, rps, part, st);
  }
}

cudaError_t launch_sketch(const SketchLaunch& L, const void* X, int dtype, int64_t m, int n, int64_t ldx,
                          int64_t row_offset, int k, int zeta, uint64_t seed, double* part, double* P,
                          int* status, cudaStream_t st, cudaEvent_t ev_mid) {
  cudaError_t e;
  const int64_t per = (m + L.splits - 1) / L.splits;
  double scale;
  if (L.kind == kSketchSparse) {
    const int64_t rps = std::max<int64_t>(KCS, ((per + KCS - 1) / KCS) * KCS);
    auto launch = [&](auto* tag) -> cudaError_t {
      using TX = std::remove_pointer_t<decltype(tag)>;
      auto kern = sketch_sparse_kernel<TX>;
      cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem);
      if (e2 != cudaSuccess) return e2;
      kern<<<L.tiles_n * L.splits, SPARSE_THREADS, L.smem, st>>>((const TX*)X, m, n, ldx, row_offset, k, zeta,
                                                                 seed, L.tiles_n, L.NT, rps, part);
      return cudaGetLastError();
    };
    e = dtype == RCHOLQR_F64 ? launch((double*)nullptr) : launch((float*)nullptr);
    scale = 1.0 / std::sqrt((double)zeta);
  } else {
    const int64_t rps = std::max<int64_t>(KC, ((per + KC - 1) / KC) * KC);
    e = dtype == RCHOLQR_F64 ? launch_gauss_typed<double>(L, X, m, n, ldx, row_offset, k, seed, rps, part, st)
                             : launch_gauss_typed<float>(L, X, m, n, ldx, row_offset, k, seed, rps, part, st);
    scale = 1.0 / std::sqrt((double)k);
  }
  if (e != cudaSuccess) return e;
  if (ev_mid) cudaEventRecord(ev_mid, st);
  const int64_t kn = (int64_t)k * n;
  const int threads = 256;
  const int blocks = (int)std::min<int64_t>((kn + threads - 1) / threads, 4096);
  sketch_reduce_kernel<<<blocks, threads, 0, st>>>(part, L.splits, kn, scale, P, status);
  return cudaGetLastError();
}

cudaError_t launch_theta_export(uint64_t seed, int k, int sketch, int zeta, int64_t row_offset, int64_t m,
                                float* Z, int32_t* rows, int8_t* signs, cudaStream_t st) {
  if (m == 0) return cudaSuccess;
  if (sketch == RCHOLQR_GAUSSIAN) {
    if (!Z) return cudaSuccess;
    const int64_t work = m * ((k + 3) / 4);
    const int blocks = (int)std::min<int64_t>((work + 255) / 256, 65535);
    theta_gauss_export_kernel<<<blocks, 256, 0, st>>>(seed, k, row_offset, m, Z);
  } else {
    const int blocks = (int)std::min<int64_t>((m + 255) / 256, 65535);
    theta_sparse_export_kernel<<<blocks, 256, 0, st>>>(seed, k, zeta, row_offset, m, rows, signs);
  }
  return cudaGetLastError();
}

}  // namespace rcq
