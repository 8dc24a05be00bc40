// sketch.cu -- step 1 of RCholeskyQR: P = Theta X, fp64 accumulation.
//
// Gaussian Theta: a GEMM with M = k (Theta rows), N = n, K = m (rows of X).  Each CTA owns a
// KT x NT tile of P and a contiguous range of X rows ("split"), and is warp-specialised:
//   * 8 producer warps, per 32-row stage, generate the KT x 32 Theta tile in registers
//     (Philox4x32-10 + Box-Muller, theta.cuh), park it in shared memory as fp64 (exact: the draws
//     are fp32) and stage the 32 x NT X tile (coalesced loads, exact fp32 -> fp64 widening);
//   * 8 MMA warps consume the stages with DMMA m16n8k4 (the FP64 tensor core) into register
//     accumulators, the CTA's m16n8 output tiles split evenly so every SMSP's DMMA pipe is loaded
//     alike; a 3-stage ring (named-barrier FULL/EMPTY handshake) overlaps generation with MMA.
// X is read from HBM once per tile_k (C2: twice from L2-adjacent CTAs).  Per-CTA partials
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

constexpr int KC = 32;             // X rows per pipeline stage
constexpr int SK_MMA_WARPS = 16;   // 4 per SMSP; output tiles split so every SMSP's DMMA pipe is loaded alike
constexpr int SK_PROD_WARPS = 4;   // Theta generation + X prefetch (1 per SMSP, 2 Philox chains each)
constexpr int SK_THREADS = 32 * (SK_MMA_WARPS + SK_PROD_WARPS);
constexpr size_t SK_SMEM_BUDGET = 200 * 1024;

__device__ __forceinline__ void cp_async_zfill4(void* s, const void* g, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"((unsigned)__cvta_generic_to_shared(s)), "l"(g),
               "r"(valid ? 4 : 0));
}
__device__ __forceinline__ void cp_async_zfill8(void* s, const void* g, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"((unsigned)__cvta_generic_to_shared(s)), "l"(g),
               "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_async_commit_grp() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// Per-MMA-warp work: a contiguous run of n8 tiles inside ONE m16 strip (so the A fragment is
// shared by all of the warp's MMAs), chosen on the host so the four SMSPs (warps w = s mod 4)
// carry the same number of m16n8 tiles to within one piece (plan_warps()).
struct WarpPlan {
  int8_t strip[SK_MMA_WARPS], t0[SK_MMA_WARPS], cnt[SK_MMA_WARPS];
};

// Tile of P per CTA: MS m16 strips (Theta rows) x NS n8 tiles (X columns).
template <typename TX, int MS, int NS>
struct GCfg {
  static constexpr int KT = 16 * MS;
  static constexpr int NT = 8 * NS;
  static constexpr int UNITS = MS * NS;                                   // m16n8 output tiles
  static constexpr int UMAX = (UNITS + SK_MMA_WARPS - 1) / SK_MMA_WARPS + 1;   // per MMA warp (plan slack)
  static constexpr int TS_LD = KC + 4;  // fp64 Theta: 36 doubles, A-fragment loads conflict-free
  // X stage keeps X's own dtype (cp.async): B-fragment loads (4 rows x 8 cols) conflict-free when the
  // row stride is 8 or 24 words (mod 32) for fp32, 4 or 12 doubles (mod 16) for fp64.
  static constexpr int XS_LD = sizeof(TX) == 4 ? NT + ((40 - NT % 32) % 32 == 32 ? 0 : (40 - NT % 32) % 32)
                                               : NT + 4;
  static constexpr size_t T_BYTES = sizeof(double) * (size_t)KT * TS_LD;
  static constexpr size_t X_BYTES = (sizeof(TX) * (size_t)KC * XS_LD + 15) / 16 * 16;
  static constexpr size_t STAGE = T_BYTES + X_BYTES;
  static constexpr int STAGES = (int)(SK_SMEM_BUDGET / STAGE) < 6 ? (int)(SK_SMEM_BUDGET / STAGE) : 6;  // barrier ids <= 13
  static constexpr size_t SMEM = STAGE * STAGES;
  static_assert(STAGES >= 2, "sketch tile too large for the stage ring");
};

__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

// Warp-specialised Gaussian sketch.  Producer warps fill a STAGES-deep ring of (Theta tile fp64,
// X tile in X's dtype) stages: the X tile of chunk c+1 is requested with cp.async (no register
// staging) before Theta of chunk c is generated, so HBM latency hides behind the generator.  MMA
// warps consume the stages with DMMA into register accumulators.  FULL(s) / EMPTY(s) are named
// barriers (ids 1..2*STAGES).  The CTA's m16n8 output tiles are split contiguously over the 16 MMA
// warps, so each SMSP (warps w, w+4, w+8, w+12) carries the same DMMA load to within one tile.
template <typename TX, int MS, int NS>
__global__ void __launch_bounds__(SK_THREADS, 1)
sketch_gauss_kernel(const TX* __restrict__ X, int64_t m, int n, int64_t ldx, int64_t row_offset, int k,
                    uint64_t seed, int tiles_k, int tiles_n, int64_t rows_per_split,
                    double* __restrict__ part, double* __restrict__ partc, const WarpPlan plan, int seg_chunks,
                    const int* __restrict__ guard, int rad, const uint64_t* __restrict__ srht_s) {
  // guard != null: recompute only if the tensor-core sketch (sketch_gtc.cu) flagged a headroom overflow
  if (guard && *guard == 0) return;
  using C = GCfg<TX, MS, NS>;
  constexpr int S = C::STAGES;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto Tst = [&](int s) { return reinterpret_cast<double*>(smem_raw + (size_t)s * C::STAGE); };
  auto Xst = [&](int s) { return reinterpret_cast<TX*>(smem_raw + (size_t)s * C::STAGE + C::T_BYTES); };

  const int tiles = tiles_k * tiles_n;
  const int tile = blockIdx.x % tiles, split = blockIdx.x / tiles;
  const int tk = tile % tiles_k, tn = tile / tiles_k;
  const int r0 = tk * C::KT, n0 = tn * C::NT;
  const int64_t i_begin = (int64_t)split * rows_per_split;
  const int64_t i_end = min(m, i_begin + rows_per_split);
  const int nchunks = i_end > i_begin ? (int)((i_end - i_begin + KC - 1) / KC) : 0;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (warp >= SK_MMA_WARPS) {
    // ------------------------------------------------------------------ producers
    const int ptid = tid - 32 * SK_MMA_WARPS;
    constexpr int PT = 32 * SK_PROD_WARPS;
    auto issue_x = [&](int ch) {   // cp.async the X tile of chunk ch into its stage (zero-filled tails)
      const int64_t i0 = i_begin + (int64_t)ch * KC;
      TX* Xb = Xst(ch % S);
      for (int c = ptid; c < KC * C::NT; c += PT) {
        const int ii = c / C::NT, jj = c % C::NT;
        const bool ok = i0 + ii < i_end && n0 + jj < n;
        const TX* src = ok ? X + (i0 + ii) * ldx + n0 + jj : X;
        if (sizeof(TX) == 4) cp_async_zfill4(Xb + ii * C::XS_LD + jj, src, ok);
        else cp_async_zfill8(Xb + ii * C::XS_LD + jj, src, ok);
      }
      cp_async_commit_grp();
    };
    if (nchunks > 0) issue_x(0);
    for (int ch = 0; ch < nchunks; ++ch) {
      const int s = ch % S;
      // stage of chunk ch+1 must be free before its X is requested
      if (ch + 1 < nchunks) {
        if (ch + 1 >= S) named_sync(1 + S + (ch + 1) % S, SK_THREADS);   // EMPTY(stage of ch+1)
        issue_x(ch + 1);
      } else {
        cp_async_commit_grp();   // keep one group per iteration so wait_group(1) stays uniform
      }
      const int64_t i0 = i_begin + (int64_t)ch * KC;
      double* T = Tst(s);
      constexpr int NGEN = (C::KT / 4) * KC;
      for (int c = ptid; c < NGEN; c += 2 * PT) {
#pragma unroll
        for (int v = 0; v < 2; ++v) {          // two independent Philox/Box-Muller chains (ILP 2)
          const int cc = c + v * PT;
          if (cc < NGEN) {
            const int qq = cc / KC, ii = cc % KC;
            const int rb = r0 + 4 * qq;
            float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
            if (i0 + ii < i_end && rb < k)
              z = rad == 2 ? srht4(srht_s, k, seed, (uint64_t)(row_offset + i0 + ii), (uint32_t)rb)
                  : rad ? rademacher4(seed, (uint64_t)(row_offset + i0 + ii), (uint32_t)rb)
                        : gauss4_x2(seed, (uint64_t)(row_offset + i0 + ii), (uint32_t)(rb >> 2));
            double* Tc = T + (4 * qq) * C::TS_LD + ii;
            Tc[0 * C::TS_LD] = (rb + 0 < k) ? (double)z.x : 0.0;
            Tc[1 * C::TS_LD] = (rb + 1 < k) ? (double)z.y : 0.0;
            Tc[2 * C::TS_LD] = (rb + 2 < k) ? (double)z.z : 0.0;
            Tc[3 * C::TS_LD] = (rb + 3 < k) ? (double)z.w : 0.0;
          }
        }
      }
      cp_async_wait_1();                        // this thread's copies for chunk ch have landed
      named_arrive(1 + s, SK_THREADS);          // FULL(s): Theta + X of chunk ch visible to MMA warps
    }
    cp_async_wait_0();
    return;
  }

  // -------------------------------------------------------------------- MMA warps
  const int g = lane >> 2, t4 = lane & 3;
  const int wstrip = plan.strip[warp], wt0 = plan.t0[warp], nun = plan.cnt[warp];
  double acc[C::UMAX][4];
#pragma unroll
  for (int u = 0; u < C::UMAX; ++u)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[u][e] = 0.0;
  const int arow = wstrip * 16 + g;
  const int bcol0 = wt0 * 8 + g;

  // Compensated two-level accumulation (the paper's "random projections in higher precision",
  // PAPER.md:83, 406, 423): the DMMA chain covers SEG chunks only, then is folded with TwoSum into
  // this CTA's private (sum, compensation) partial in global memory.
  double* __restrict__ Pp = part + (size_t)split * (size_t)k * n;
  double* __restrict__ Pc = partc + (size_t)split * (size_t)k * n;
  bool first_flush = true;
  const int frow = r0 + wstrip * 16 + g;
  const bool rok0 = frow < k, rok1 = frow + 8 < k;
  // per unit: issue the 8 loads first (no store in between), then the TwoSums, then the stores
  auto flush = [&]() {
#pragma unroll
    for (int u = 0; u < C::UMAX; ++u) {
      if (u < nun) {
        const int col = n0 + (wt0 + u) * 8 + 2 * t4;
        const size_t i0 = (size_t)frow * n + col, i1 = i0 + (size_t)8 * n;
        const bool c0 = col < n, c1 = col + 1 < n;
        const bool ok[4] = {rok0 && c0, rok0 && c1, rok1 && c0, rok1 && c1};
        const size_t ix[4] = {i0, i0 + 1, i1, i1 + 1};
        double so[4], co[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          so[e] = (ok[e] && !first_flush) ? __ldcg(Pp + ix[e]) : 0.0;
          co[e] = (ok[e] && !first_flush) ? __ldcg(Pc + ix[e]) : 0.0;
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const double av = acc[u][e];
          const double snew = so[e] + av;                              // TwoSum(so, av)
          const double bb = snew - so[e];
          co[e] += (so[e] - (snew - bb)) + (av - bb);
          so[e] = snew;
          acc[u][e] = 0.0;
        }
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (ok[e]) { __stcg(Pp + ix[e], so[e]); __stcg(Pc + ix[e], co[e]); }
      }
    }
    first_flush = false;
  };
  // fp64 X (working precision u = 2^-53) needs the sketch at u_f << u: compensated folds every SEG
  // chunks.  fp32 X (u = 2^-24): a plain fp64 DMMA chain is already u_f ~ 1e-13 << u, so one fold.
  constexpr bool kComp = sizeof(TX) == 8;
  const int SEG = seg_chunks;   // chunks per DMMA accumulation chain (default 16 = 512 rows)

  for (int ch = 0; ch < nchunks; ++ch) {
    const int s = ch % S;
    named_sync(1 + s, SK_THREADS);                                         // FULL(s)
    const double* Tk = Tst(s) + arow * C::TS_LD + t4;
    const TX* Xk = Xst(s) + t4 * C::XS_LD + bcol0;
#pragma unroll 2
    for (int ks = 0; ks < KC / 4; ++ks) {
      const double a0 = Tk[4 * ks], a1 = Tk[8 * C::TS_LD + 4 * ks];
      const TX* xrow = Xk + 4 * ks * C::XS_LD;
      TX braw[C::UMAX];
#pragma unroll
      for (int u = 0; u < C::UMAX; ++u) braw[u] = (u < nun) ? xrow[8 * u] : TX(0);
#pragma unroll
      for (int u = 0; u < C::UMAX; ++u)
        if (u < nun) dmma_16x8x4(acc[u], a0, a1, (double)braw[u]);
    }
    if (ch + S < nchunks) named_arrive(1 + S + s, SK_THREADS);            // EMPTY(s)
    if constexpr (kComp) {
      if ((ch + 1) % SEG == 0) flush();
    }
  }
  if (first_flush || !kComp || nchunks % SEG != 0) flush();   // tail segment (or the only one)
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
                     double* __restrict__ part, const int* __restrict__ guard) {
  // guard != null: recompute only if the tensor-core sketch (sketch_tc.cu) flagged a headroom overflow
  if (guard && *guard == 0) return;
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

// Register-resident sparse-sign sketch (zeta <= 8, beta = k/zeta <= 16, n <= 64): warp t owns Theta
// block t, i.e. the beta x n tile P[t*beta .. t*beta+beta-1, :] in registers (lane L: columns
// L, L+32).  For every X row the block's target row h is warp-uniform, so a uniform switch adds
// the (sign-flipped) row into acc[h] -- no shared-memory read-modify-write chain.  X chunks are
// widened to fp64 once in shared memory (shared by the zeta warps); the next chunk is prefetched
// into registers while the current one is consumed.
constexpr int SPR_KC = 32;       // rows per chunk (= warp size: one ballot per target row)
constexpr int SPR_STAGES = 4;    // cp.async ring depth (raw X chunks in flight per CTA)
constexpr int SPR_THREADS = 256;
template <typename TX, int BETA, int CPL>
__global__ void __launch_bounds__(SPR_THREADS)
sketch_sparse_reg_kernel(const TX* __restrict__ X, int64_t m, int n, int64_t ldx, int64_t row_offset, int k,
                         int zeta, uint64_t seed, int64_t rows_per_split, double* __restrict__ part,
                         const int* __restrict__ guard) {
  // guard != null: recompute only if the tensor-core sketch (sketch_tc.cu) flagged a headroom overflow
  if (guard && *guard == 0) return;
  constexpr int NC = 32 * CPL;
  extern __shared__ __align__(16) unsigned char spr_smem[];
  double (*Xs)[NC] = reinterpret_cast<double (*)[NC]>(spr_smem);                        // [KC][NC] fp64
  TX (*Xraw)[SPR_KC][NC] = reinterpret_cast<TX (*)[SPR_KC][NC]>(spr_smem + sizeof(double) * SPR_KC * NC);
  uint8_t (*sel)[SPR_KC][8] = reinterpret_cast<uint8_t (*)[SPR_KC][8]>(
      spr_smem + sizeof(double) * SPR_KC * NC + sizeof(TX) * SPR_STAGES * SPR_KC * NC);
  const int split = blockIdx.x;
  const int64_t i_begin = (int64_t)split * rows_per_split;
  const int64_t i_end = min(m, i_begin + rows_per_split);
  const int nchunks = i_end > i_begin ? (int)((i_end - i_begin + SPR_KC - 1) / SPR_KC) : 0;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double acc[BETA][CPL];
#pragma unroll
  for (int r = 0; r < BETA; ++r)
#pragma unroll
    for (int c = 0; c < CPL; ++c) acc[r][c] = 0.0;
  auto issue = [&](int ch) {      // cp.async chunk ch (zero-filled tails) + its row selections
    const int st = ch % SPR_STAGES;
    const int64_t i0 = i_begin + (int64_t)ch * SPR_KC;
    const int rows_here = (int)min((int64_t)SPR_KC, i_end - i0);
    const TX* xbase = X + i0 * ldx;
#pragma unroll
    for (int u = 0; u < SPR_KC * NC / SPR_THREADS; ++u) {
      const int cidx = tid + u * SPR_THREADS;
      const int ii = cidx / NC, jj = cidx % NC;              // NC is a power of two
      const bool ok = ii < rows_here && jj < n;
      const TX* src = ok ? xbase + (int64_t)ii * ldx + jj : X;
      if (sizeof(TX) == 4) cp_async_zfill4(&Xraw[st][ii][jj], src, ok);
      else cp_async_zfill8(&Xraw[st][ii][jj], src, ok);
    }
    cp_async_commit_grp();
    if (tid < SPR_KC) {
      uint32_t w0 = 0xFFFFFFFFu, w1 = 0xFFFFFFFFu;   // 0xFF = "no row" (tail)
      if (i0 + tid < i_end) {
        const uint4 w = philox_at(seed, (uint64_t)(row_offset + i0 + tid), 0u, kDomainSparse);
        const int beta = k / zeta;
        w0 = w1 = 0u;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          uint32_t code = 0xFFu;
          if (t < zeta) {
            const uint32_t hw = sparse_halfword(w, t);
            code = (uint32_t)(sparse_row(hw, t, beta) - t * beta) | ((hw >> 15) << 4);
          }
          if (t < 4) w0 |= code << (8 * t); else w1 |= code << (8 * (t - 4));
        }
      }
      *reinterpret_cast<uint32_t*>(&sel[st][tid][0]) = w0;
      *reinterpret_cast<uint32_t*>(&sel[st][tid][4]) = w1;
    }
  };
#pragma unroll 1
  for (int c = 0; c < SPR_STAGES - 1; ++c) {
    if (c < nchunks) issue(c);
    else cp_async_commit_grp();
  }
  for (int ch = 0; ch < nchunks; ++ch) {
    const int st = ch % SPR_STAGES;
    asm volatile("cp.async.wait_group %0;\n" ::"n"(SPR_STAGES - 2) : "memory");
    __syncthreads();   // chunk ch landed for everyone; Xs free (previous chunk consumed)
#pragma unroll
    for (int u = 0; u < SPR_KC * NC / SPR_THREADS; ++u) {
      const int cidx = tid + u * SPR_THREADS;
      Xs[cidx / NC][cidx % NC] = (double)Xraw[st][cidx / NC][cidx % NC];
    }
    __syncthreads();
    if (ch + SPR_STAGES - 1 < nchunks) issue(ch + SPR_STAGES - 1);
    else cp_async_commit_grp();
    if (warp < zeta) {
      // bucket the chunk's 32 rows by target row h (lane = row): one ballot per h, then the rows of
      // bucket h are added into the statically indexed acc[h] (no indirect branch)
      const uint32_t mycode = sel[st][lane][warp];
      const uint32_t negmask = __ballot_sync(0xffffffffu, (mycode & 16u) != 0);
#pragma unroll
      for (int r = 0; r < BETA; ++r) {
        uint32_t mask = __ballot_sync(0xffffffffu, (mycode & 0xEFu) == (uint32_t)r);
        while (mask) {
          const int ii = __ffs(mask) - 1;
          mask &= mask - 1;
          const double sg = ((negmask >> ii) & 1u) ? -1.0 : 1.0;
#pragma unroll
          for (int c = 0; c < CPL; ++c) acc[r][c] = fma(Xs[ii][lane + 32 * c], sg, acc[r][c]);
        }
      }
    }
  }
  cp_async_wait_0();
  if (warp < zeta) {
    const int beta = k / zeta;
    double* Pp = part + (size_t)split * (size_t)k * n;
#pragma unroll
    for (int r = 0; r < BETA; ++r)
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int col = lane + 32 * c;
        if (r < beta && col < n) Pp[(size_t)(warp * beta + r) * n + col] = acc[r][c];
      }
  }
}

// Fixed-order compensated sum of the per-split partials, one scaling, non-finite detection.
// Entries idx < kn_first are scaled by `scale`, the rest by `scale2` (the (k + l)-row sketch of Alg. 5:
// Theta rows by 1/sqrt(k), extractor rows by 1/sqrt(l)).
// Each warp sums 4 consecutive entries: lane = 4 * sl + il takes splits sl, sl + 8, ... of entry idx0 + il
// (a split's 4 entries are one 32-byte sector), then the 8 split lanes combine by an xor butterfly of TwoSums
// (a fixed tree: deterministic, and every lane ends with the same value).  The serial loop over all
// splits this replaces was a chain of dependent-latency loads (C1: 29 us for 800 entries).
__global__ void sketch_reduce_kernel(const double* __restrict__ part, const double* __restrict__ partc, int splits,
                                     int64_t kn, double scale, int64_t kn_first, double scale2,
                                     double* __restrict__ P, int* status, const int* flag, int* flag_seen) {
  // record (for rcholqr_last_path) that a tensor-core sketch raised its overflow flag and the guarded
  // CUDA-core kernel recomputed the partials
  if (flag && flag_seen && blockIdx.x == 0 && threadIdx.x == 0 && *flag) atomicOr(flag_seen, 1);
  const int lane = threadIdx.x & 31, il = lane & 3, sl = lane >> 2;
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t idx0 = warp0 * 4; idx0 < kn; idx0 += nwarps * 4) {
    const int64_t idx = idx0 + il;
    double s = 0.0, c = 0.0;                    // compensated (TwoSum) sum over this lane's splits
    if (idx < kn) {
#pragma unroll 4
      for (int sp = sl; sp < splits; sp += 8) {
        const double v = part[(size_t)sp * kn + idx];
        const double t = s + v;
        const double bb = t - s;
        c += (s - (t - bb)) + (v - bb);
        s = t;
        if (partc) c += partc[(size_t)sp * kn + idx];
      }
    }
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      const double s2 = __shfl_xor_sync(0xffffffffu, s, off), c2 = __shfl_xor_sync(0xffffffffu, c, off);
      const double t = s + s2;
      const double bb = t - s;
      c = (c + c2) + ((s - (t - bb)) + (s2 - bb));
      s = t;
    }
    if (sl == 0 && idx < kn) {
      s = (s + c) * (idx < kn_first ? scale : scale2);
      P[idx] = s;
      if (!isfinite(s)) atomicOr(status, kStNonfinite);
    }
  }
}

// ---------------------------------------------------------------------------------------------
// Test export of Theta.
__global__ void theta_rademacher_export_kernel(uint64_t seed, int k, int64_t row_offset, int64_t m, float* Z) {
  const int nq = (k + 3) / 4;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < m * nq; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = c % m;
    const int q = (int)(c / m);
    const float4 z = rademacher4(seed, (uint64_t)(row_offset + i), (uint32_t)(4 * q));
    const float v[4] = {z.x, z.y, z.z, z.w};
    for (int t = 0; t < 4 && 4 * q + t < k; ++t) Z[(int64_t)(4 * q + t) * m + i] = v[t];
  }
}

__global__ void theta_srht_export_kernel(const uint64_t* s, uint64_t seed, int k, int64_t row_offset, int64_t m,
                                         float* Z) {
  const int nq = (k + 3) / 4;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < m * nq; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = c % m;
    const int q = (int)(c / m);
    const float4 z = srht4(s, k, seed, (uint64_t)(row_offset + i), (uint32_t)(4 * q));
    const float v[4] = {z.x, z.y, z.z, z.w};
    for (int t = 0; t < 4 && 4 * q + t < k; ++t) Z[(int64_t)(4 * q + t) * m + i] = v[t];
  }
}

__global__ void theta_gauss_export_kernel(uint64_t seed, int k, int64_t row_offset, int64_t m, float* Z) {
  const int nq = (k + 3) / 4;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < m * nq; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = c % m;
    const int q = (int)(c / m);
    const float4 z = gauss4_x2(seed, (uint64_t)(row_offset + i), (uint32_t)q);
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
template <int MS, int NS>
static void fill_gauss(SketchLaunch& L, int kind, int k, int n, int dtype) {
  L.kind = kind; L.KT = 16 * MS; L.NT = 8 * NS; L.threads = SK_THREADS;
  L.smem = dtype == RCHOLQR_F64 ? GCfg<double, MS, NS>::SMEM : GCfg<float, MS, NS>::SMEM;
  L.tiles_k = (k + L.KT - 1) / L.KT;
  L.tiles_n = (n + L.NT - 1) / L.NT;
}

// Chunks of KC rows per DMMA accumulation chain before a compensated fold (DESIGN.md "Sketch
// accuracy"); RCHOLQR_SEG overrides it for experiments.
static int seg_chunks() {
  static int v = [] {
    const char* e = getenv("RCHOLQR_SEG");
    const int x = e ? atoi(e) : 16;
    return x > 0 ? x : 16;
  }();
  return v;
}

// Split the MS x NS m16n8 tiles into <= SK_MMA_WARPS single-strip pieces and deal them to the four
// SMSPs (warp w runs on SMSP w % 4) longest-first, so the per-SMSP DMMA loads are balanced.
static WarpPlan plan_warps(int MS, int NS) {
  WarpPlan P{};
  int pieces_per_strip[64];
  for (int s = 0; s < MS; ++s) pieces_per_strip[s] = 1;
  int npieces = MS;
  // repeatedly split the strip whose pieces are largest while warps remain
  while (true) {
    int best = -1, bestsz = 0;
    for (int s = 0; s < MS; ++s) {
      const int sz = (NS + pieces_per_strip[s] - 1) / pieces_per_strip[s];
      if (sz > bestsz && pieces_per_strip[s] < NS) { bestsz = sz; best = s; }
    }
    if (best < 0 || npieces + 1 > SK_MMA_WARPS) break;
    pieces_per_strip[best]++;
    npieces++;
  }
  struct Piece { int strip, t0, cnt; };
  Piece pc[SK_MMA_WARPS];
  int np = 0;
  for (int s = 0; s < MS; ++s) {
    const int p = pieces_per_strip[s];
    int t = 0;
    for (int q = 0; q < p; ++q) {
      const int c = NS / p + (q < NS % p ? 1 : 0);
      pc[np++] = {s, t, c};
      t += c;
    }
  }
  // longest-first onto the least-loaded SMSP that still has a free warp slot
  for (int i = 0; i < np; ++i)
    for (int j = i + 1; j < np; ++j)
      if (pc[j].cnt > pc[i].cnt) { Piece tmp = pc[i]; pc[i] = pc[j]; pc[j] = tmp; }
  int load[4] = {0, 0, 0, 0}, used[4] = {0, 0, 0, 0};
  for (int w = 0; w < SK_MMA_WARPS; ++w) { P.strip[w] = 0; P.t0[w] = 0; P.cnt[w] = 0; }
  for (int i = 0; i < np; ++i) {
    int best = -1;
    for (int sm = 0; sm < 4; ++sm)
      if (used[sm] < SK_MMA_WARPS / 4 && (best < 0 || load[sm] < load[best])) best = sm;
    const int w = best + 4 * used[best];
    used[best]++;
    load[best] += pc[i].cnt;
    P.strip[w] = (int8_t)pc[i].strip; P.t0[w] = (int8_t)pc[i].t0; P.cnt[w] = (int8_t)pc[i].cnt;
  }
  return P;
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
  if (sketch == RCHOLQR_SPARSE_SIGN) {
    if (zeta <= 8 && k / zeta <= 16 && n <= 64 && !getenv("RCHOLQR_SPARSE_SMEM")) {
      L.kind = kSketchSparseReg;
      L.threads = SPR_THREADS;
      L.KT = k; L.NT = n; L.tiles_k = 1; L.tiles_n = 1; L.smem = 0;
      L.splits = choose_splits(1, 2 * sms);
    } else {
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
    }
    // tcgen05 int8 path (sketch_tc.cu, any n by 64-column tiles) with the kernel above as its guarded fallback
    if (sparse_tc_applicable(k, n, zeta) && !getenv("RCHOLQR_SPARSE_CUDA_CORE")) {
      L.sp_tc = 1;
      L.splits = sms;
    }
    return L;
  }
  // Gaussian: pick the tile minimising padded work (tiles * KT * NT), ties -> larger tile.
  constexpr int NC = 4;
  SketchLaunch cand[NC];
  fill_gauss<3, 3>(cand[0], kSketchG48x24, k, n, dtype);
  fill_gauss<8, 8>(cand[1], kSketchG128x64, k, n, dtype);
  fill_gauss<7, 13>(cand[2], kSketchG112x104, k, n, dtype);
  fill_gauss<4, 8>(cand[3], kSketchG64x64, k, n, dtype);
  int best = NC - 1;
  double best_cost = 1e300;
  const char* force = getenv("RCHOLQR_SKETCH_KIND");  // experiments only
  for (int c = 0; c < NC; ++c) {
    if (force && atoi(force) != cand[c].kind) continue;
    if (cand[c].smem > smem_optin) continue;
    // padded MMA work + a per-tile Theta regeneration / X re-read penalty
    const double padded = (double)cand[c].tiles_k * cand[c].KT * cand[c].tiles_n * cand[c].NT;
    const double cost = padded * (1.0 + 0.05 * (cand[c].tiles_n - 1) + 0.02 * (cand[c].tiles_k - 1));
    if (cost < best_cost) { best_cost = cost; best = c; }
  }
  L = cand[best];
  L.splits = choose_splits(L.tiles_k * L.tiles_n, sms);
  L.tc = 0;
  if (sketch == RCHOLQR_RADEMACHER || sketch == RCHOLQR_SRHT) {   // DMMA kernel drawing +-1, dense tcgen05 in front
    L.rad = sketch == RCHOLQR_SRHT ? 2 : 1;
    if (L.rad == 2 && srht_fwht_applicable(k)) {           // blocked fast Walsh-Hadamard transform (srht_fwht.cu)
      L.fwht = 1;
      L.fwht_splits = srht_fwht_splits(n, sms);
    }
    if (sparse_tc_applicable(k, n, 1) && !getenv("RCHOLQR_RADEMACHER_DMMA")) {
      L.rad_tc = 1;
      L.rad_splits = sms;
    }
    return L;
  }
  // tcgen05 int8 digit sketch (sketch_gtc.cu), the DMMA kernel above as its guarded fallback
  if (!getenv("RCHOLQR_GAUSS_DMMA")) {
    const int kt = gauss_tc_kt(dtype);
    L.tc = 1;
    L.tc_tiles_k = (k + kt - 1) / kt;
    L.tc_tiles_n = (n + 127) / 128;
    L.tc_splits = choose_splits(L.tc_tiles_k * L.tc_tiles_n, sms);
  }
  return L;
}

template <typename TX, int MS, int NS>
static cudaError_t launch_g(const SketchLaunch& L, const void* X, int64_t m, int n, int64_t ldx, int64_t ro,
                            int k, uint64_t seed, int64_t rps, double* part, double* partc, cudaStream_t st,
                            const int* guard) {
  auto kern = sketch_gauss_kernel<TX, MS, NS>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem);
  if (e != cudaSuccess) return e;
  static_assert(sizeof(WarpPlan) == 3 * SK_MMA_WARPS, "plan layout");
  const WarpPlan plan = plan_warps(MS, NS);
  for (int w = 0; w < SK_MMA_WARPS; ++w)
    if (plan.cnt[w] > GCfg<TX, MS, NS>::UMAX) return cudaErrorInvalidConfiguration;
  kern<<<L.tiles_k * L.tiles_n * L.splits, SK_THREADS, L.smem, st>>>((const TX*)X, m, n, ldx, ro, k, seed,
                                                                     L.tiles_k, L.tiles_n, rps, part, partc, plan,
                                                                     seg_chunks(), guard, L.rad, L.srht_s);
  return cudaGetLastError();
}

template <typename TX>
static cudaError_t launch_gauss_typed(const SketchLaunch& L, const void* X, int64_t m, int n, int64_t ldx,
                                      int64_t ro, int k, uint64_t seed, int64_t rps, double* part, double* partc,
                                      cudaStream_t st, const int* guard) {
  switch (L.kind) {
    case kSketchG48x24: return launch_g<TX, 3, 3>(L, X, m, n, ldx, ro, k, seed, rps, part, partc, st, guard);
    case kSketchG128x64: return launch_g<TX, 8, 8>(L, X, m, n, ldx, ro, k, seed, rps, part, partc, st, guard);
    case kSketchG112x104: return launch_g<TX, 7, 13>(L, X, m, n, ldx, ro, k, seed, rps, part, partc, st, guard);
    default: return launch_g<TX, 4, 8>(L, X, m, n, ldx, ro, k, seed, rps, part, partc, st, guard);
  }
}

double gauss_tc_min_work() {
  const char* e = getenv("RCHOLQR_GAUSS_TC_MIN_WORK");     // tests: 0 sends the tiniest shapes through tcgen05 too
  return e ? atof(e) : 2.0e7;
}

cudaError_t launch_sketch(const SketchLaunch& L, const void* X, int dtype, int64_t m, int n, int64_t ldx,
                          int64_t row_offset, int k, int zeta, uint64_t seed, double* part, double* partc, double* P,
                          int* status, int* flag, void* xdig, size_t xdig_bytes, cudaStream_t st, cudaEvent_t ev_mid,
                          int k_first, unsigned* path, int* flag_seen, double* cs_part, double* cs_out, bool* cs_done,
                          bool colmajor) {
  // colmajor: X column-major (ldx >= m is the column pitch).  Only the tcgen05 kernels read that layout (sparse /
  // dense-E kernel, pre-split Gaussian); the guarded CUDA-core / DMMA fallbacks are not launched, so a raised
  // overflow flag (reported through flag_seen) means the caller must redo the call through the layout adapter.
  // cudaErrorNotSupported: no native kernel for this plan / alignment.
  if (cs_done) *cs_done = false;
  cudaError_t e;
  unsigned pb = 0;
  const int64_t per = (m + L.splits - 1) / L.splits;
  double scale;
  int reduce_splits = L.splits;
  if (L.kind == kSketchSparseReg || L.kind == kSketchSparse) {
    static_assert(KCS % SPR_KC == 0, "row chunks");
    const int64_t rps = std::max<int64_t>(KCS, ((per + KCS - 1) / KCS) * KCS);   // whole chunks of both kernels
    const int beta = k / zeta;
    // tensor-core path first; the CUDA-core kernel below then runs only if it raised the overflow
    // flag.  int32 accumulators are exact while rows_per_split * 255 < 2^31.
    const int* guard = nullptr;
    if (L.sp_tc && rps <= kSparseTcMaxRows && sparse_tc_aligned(X, dtype, m, ldx)) {
      e = cudaMemsetAsync(flag, 0, sizeof(int), st);
      if (e != cudaSuccess) return e;
      e = launch_sparse_tc(X, dtype, m, n, ldx, row_offset, k, zeta, seed, L.splits, rps, part, flag, st, nullptr,
                           cs_out ? cs_part : nullptr, colmajor);
      if (e == cudaSuccess) {
        guard = flag; pb |= kPathSketchTC;
        if (cs_out) {                                      // D of Alg. 7 came with this pass
          e = launch_colsum_reduce(cs_part, L.splits, n, cs_out, status, st);
          if (e != cudaSuccess) return e;
          if (cs_done) *cs_done = true;
        }
      } else if (e != cudaErrorNotSupported) return e;
    }
    if (colmajor && !guard) return cudaErrorNotSupported;
    if (!guard) pb |= kPathSketchCudaCore;
    auto launch = [&](auto* tag) -> cudaError_t {
      using TX = std::remove_pointer_t<decltype(tag)>;
      if (L.kind == kSketchSparse) {
        auto kern = sketch_sparse_kernel<TX>;
        cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem);
        if (e2 != cudaSuccess) return e2;
        kern<<<L.tiles_n * L.splits, SPARSE_THREADS, L.smem, st>>>((const TX*)X, m, n, ldx, row_offset, k, zeta,
                                                                   seed, L.tiles_n, L.NT, rps, part, guard);
        return cudaGetLastError();
      }
      auto go = [&](auto kern, int cpl) -> cudaError_t {
        const size_t sm = (sizeof(double) + sizeof(TX) * SPR_STAGES) * SPR_KC * 32 * cpl + SPR_STAGES * SPR_KC * 8;
        cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e2 != cudaSuccess) return e2;
        kern<<<L.splits, SPR_THREADS, sm, st>>>((const TX*)X, m, n, ldx, row_offset, k, zeta, seed, rps, part,
                                                guard);
        return cudaSuccess;
      };
      cudaError_t e2;
      if (beta <= 8) e2 = n <= 32 ? go(sketch_sparse_reg_kernel<TX, 8, 1>, 1) : go(sketch_sparse_reg_kernel<TX, 8, 2>, 2);
      else e2 = n <= 32 ? go(sketch_sparse_reg_kernel<TX, 16, 1>, 1) : go(sketch_sparse_reg_kernel<TX, 16, 2>, 2);
      if (e2 != cudaSuccess) return e2;
      return cudaGetLastError();
    };
    e = colmajor ? cudaSuccess : (dtype == RCHOLQR_F64 ? launch((double*)nullptr) : launch((float*)nullptr));
    scale = 1.0 / std::sqrt((double)zeta);
  } else if (L.fwht && !colmajor &&
             (e = launch_srht_fwht(X, dtype, m, n, ldx, row_offset, k, seed, L.srht_s, L.fwht_splits, part, partc,
                                   &reduce_splits, st)) != cudaErrorNotSupported) {
    // SRHT by the blocked fast Walsh-Hadamard transform (srht_fwht.cu): fp64 butterflies with
    // compensated block sums, no digit scales and so no overflow guard / fallback
    if (e != cudaSuccess) return e;
    pb |= kPathSketchFwht;
    scale = 1.0 / std::sqrt((double)k);
  } else {
    int splits = L.splits;
    const int* guard = nullptr;
    // launch-bound problems (C1: 2kmn = 1.6e7 flops) take the single DMMA kernel: the pre-split tcgen05 path's three
    // launches cost more than they save there (C1 sketch: 17 vs 41 us)
    const bool tc = L.tc && gauss_tc_aligned(X, dtype, n, ldx) && 2.0 * k * (double)m * n >= gauss_tc_min_work();
    // (SRHT: the tcgen05 E tile splits the global row as (multiple of 32) + lane, so row_offset % 32 == 0)
    if (L.rad_tc && sparse_tc_aligned(X, dtype, m, ldx) && (L.rad != 2 || row_offset % 32 == 0)) {
      // dense +-1 E tile on the sparse sketch's tcgen05 kernel (zeta = 0); it writes no compensation
      // partials, so they are zeroed for the fixed-order reduction; the DMMA kernel below reruns
      // (guarded) on a headroom overflow
      splits = L.rad_splits;
      const int64_t tper = (m + splits - 1) / splits;
      const int64_t trps = std::max<int64_t>(SPR_KC, ((tper + SPR_KC - 1) / SPR_KC) * SPR_KC);
      if (trps <= kSparseTcMaxRows) {
        e = cudaMemsetAsync(flag, 0, sizeof(int), st);
        if (e == cudaSuccess) e = cudaMemsetAsync(partc, 0, sizeof(double) * (size_t)splits * k * n, st);
        if (e == cudaSuccess)
          e = launch_sparse_tc(X, dtype, m, n, ldx, row_offset, k, L.rad == 2 ? -1 : 0, seed, splits, trps, part,
                               flag, st, L.srht_s, nullptr, colmajor);
        if (e != cudaSuccess) return e;
        guard = flag;
        pb |= kPathSketchTC;
      } else {
        splits = L.splits;
      }
    } else if (tc) {
      splits = L.tc_splits;
      const int64_t tper = (m + splits - 1) / splits;
      const int64_t trps = std::max<int64_t>(KC, ((tper + KC - 1) / KC) * KC);
      e = cudaMemsetAsync(flag, 0, sizeof(int), st);
      if (e != cudaSuccess) return e;
      e = cudaErrorNotSupported;
      if (xdig && !getenv("RCHOLQR_GAUSS_NO_PRESPLIT")) {   // pre-split digits (row chunks that fit the workspace)
        e = launch_gauss_tcp(X, dtype, m, n, ldx, row_offset, k, seed, L.tc_tiles_k, L.tc_tiles_n, splits, part,
                             partc, flag, xdig, xdig_bytes, st, cs_out ? cs_part : nullptr, colmajor);
        if (e == cudaSuccess) {
          pb |= kPathSketchPresplit;
          if (cs_out) {                                    // D of Alg. 7 came with this pass
            e = launch_colsum_reduce(cs_part, kXdigSplitBlocks, n, cs_out, status, st);
            if (e != cudaSuccess) return e;
            if (cs_done) *cs_done = true;
          }
        }
      }
      if (e == cudaErrorNotSupported && !colmajor)
        e = launch_gauss_tc(X, dtype, m, n, ldx, row_offset, k, seed, L.tc_tiles_k, L.tc_tiles_n, splits, trps, part,
                            partc, flag, st);
      if (e == cudaSuccess) { guard = flag; pb |= kPathSketchTC; }   // else: the DMMA kernel computes the sketch
      else if (e != cudaErrorNotSupported) return e;
    }
    if (colmajor && !guard) return cudaErrorNotSupported;
    // DMMA kernel: the path itself, or the overflow fallback of the tensor-core kernel (same splits)
    SketchLaunch Lg = L;
    Lg.splits = splits;
    const int64_t gper = (m + splits - 1) / splits;
    const int64_t rps = std::max<int64_t>(KC, ((gper + KC - 1) / KC) * KC);
    e = colmajor ? cudaSuccess
        : dtype == RCHOLQR_F64
            ? launch_gauss_typed<double>(Lg, X, m, n, ldx, row_offset, k, seed, rps, part, partc, st, guard)
            : launch_gauss_typed<float>(Lg, X, m, n, ldx, row_offset, k, seed, rps, part, partc, st, guard);
    scale = 1.0 / std::sqrt((double)k);
    reduce_splits = splits;
    if (!guard) pb |= kPathSketchCudaCore;
  }
  if (e != cudaSuccess) return e;
  if (ev_mid) cudaEventRecord(ev_mid, st);
  const int64_t kn = (int64_t)k * n;
  const int threads = 256;                                   // 8 warps x 4 entries per block pass
  const int blocks = (int)std::min<int64_t>((kn + 31) / 32, 4096);
  const bool sparse = L.kind == kSketchSparse || L.kind == kSketchSparseReg;
  // Gaussian rows >= k_first (Alg. 5's extractor rows) take 1/sqrt(k - k_first) instead of 1/sqrt(k)
  double scale2 = scale;
  if (!sparse && k_first > 0 && k_first < k) {
    scale = 1.0 / std::sqrt((double)k_first);
    scale2 = 1.0 / std::sqrt((double)(k - k_first));
  }
  sketch_reduce_kernel<<<blocks, threads, 0, st>>>(part, sparse ? nullptr : partc, reduce_splits, kn, scale,
                                                   (int64_t)std::min(std::max(k_first, 0), k) * n, scale2, P, status,
                                                   (pb & kPathSketchTC) ? flag : nullptr, flag_seen);
  if (path) *path |= pb;
  return cudaGetLastError();
}

// fixed-order compensated sum of per-split partials (also the Gram reduction of rcqr2.cu)
cudaError_t launch_reduce(const double* part, int splits, int64_t kn, double scale, double* P, int* status,
                          cudaStream_t st) {
  const int threads = 256;
  const int blocks = (int)std::min<int64_t>((kn + 31) / 32, 4096);
  sketch_reduce_kernel<<<blocks, threads, 0, st>>>(part, nullptr, splits, kn, scale, kn, scale, P, status, nullptr,
                                                   nullptr);
  return cudaGetLastError();
}

cudaError_t launch_theta_export(uint64_t seed, int k, int sketch, int zeta, int64_t row_offset, int64_t m,
                                float* Z, int32_t* rows, int8_t* signs, cudaStream_t st, const uint64_t* srht_s) {
  if (m == 0) return cudaSuccess;
  if (sketch == RCHOLQR_GAUSSIAN || sketch == RCHOLQR_RADEMACHER || sketch == RCHOLQR_SRHT) {
    if (!Z) return cudaSuccess;
    const int64_t work = m * ((k + 3) / 4);
    const int blocks = (int)std::min<int64_t>((work + 255) / 256, 65535);
    if (sketch == RCHOLQR_SRHT) theta_srht_export_kernel<<<blocks, 256, 0, st>>>(srht_s, seed, k, row_offset, m, Z);
    else if (sketch == RCHOLQR_RADEMACHER) theta_rademacher_export_kernel<<<blocks, 256, 0, st>>>(seed, k, row_offset, m, Z);
    else theta_gauss_export_kernel<<<blocks, 256, 0, st>>>(seed, k, row_offset, m, Z);
  } else {
    const int blocks = (int)std::min<int64_t>((m + 255) / 256, 65535);
    theta_sparse_export_kernel<<<blocks, 256, 0, st>>>(seed, k, zeta, row_offset, m, rows, signs);
  }
  return cudaGetLastError();
}

}  // namespace rcq
