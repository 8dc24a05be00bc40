// sketch_tc.cu -- sparse-sign (and dense +-1) sketch on the 5th-generation tensor core (tcgen05.mma kind::i8).
//
// P = E X / sqrt(zeta) (Alg. 2 step 1 with the sparse-sign Theta of reading A3; the dense
// Rademacher / SRHT Theta of readings A22 / A23 use the same kernel with a dense E tile).  E (k x m) has entries
// in {-1, 0, +1}: EXACT in int8.  X is written exactly as a fixed-point integer against a per-(CTA, column)
// power-of-two scale 2^e_j, F(x) = round(x 2^(FB - e_j)), and the int8 MMA sums E times the base-256 digits of F
// exactly in int32 TMEM (rows * 255 < 2^31: kSparseTcMaxRows) -- the "random projection in higher precision" of
// PAPER.md:83, 423; the only approximation is the rounding of x at 2^(e_j - FB) (relative 2^-44 / 2^-60 of the
// column scale).
//
// Operand layout (round 2).  B is built from each X element's magic-constant double W(x), MN-major (the 8 bytes
// of an element contiguous along N), straight out of ONE DFMA -- no digit planes, no byte transposes (round 1
// wrote six K-major digit planes with 8 PRMTs per 4 values and was bound by that work):
//   * fp32 X: W = RN(x 2^(47-e) + 2^47 + 1.5 2^52), one DFMA on x 2^-128 built from the float's bits; its low
//     48 bits are the unsigned base-256 digits of F + 2^47.  Row i of B = [the low words of the tile's 64
//     columns | their digits 4, 5 (16-bit halves) | 16 ones]: the two constant exponent bytes are not fed to the
//     tensor core.  TMEM column 4 j + b holds digit b (< 4) of column j, column 256 + 2 j + b' digit 4 + b', and
//     the ones block S_r = sum_i E_ri, which removes the 2^47 bias exactly.  The high word is 0x4338xxxx iff
//     F + 2^47 fits in 48 bits: one LOP3 per element accumulates the overflow / Inf / NaN test.
//   * fp64 X: (hi, lo) = F + C by two magic-constant floors, F = floor(x 2^(63-e)); all 8 bytes as signed
//     digits (bytes XOR 0x80 except the top one), byte b of weight 256^b at TMEM column 8 j + b.
// P_rj = 2^(e_j - FB) sum_b acc_b 256^b.  One stage (64 X rows, 64 columns) is two k-steps x two MMAs of
// M = 128, K = 32 (N = 256 + 144 for fp32, 256 + 256 for fp64); the tensor core reads B MN-major (idesc bit 16;
// probe tools/micro/tc_i8_mn_test.cu).  Columns beyond 64 are further CTAs (column tiles: X is read through a
// 2D TMA box of 64 columns x 64 rows, zero-filled outside X).
//
// e_j = (exponent of the column maximum over the CTA's FIRST stage) + 4 bits of headroom.  If a later element
// does not fit (|x| >= 2^e_j, or Inf/NaN) the kernel raises an overflow flag and a CUDA-core kernel recomputes
// the whole sketch (sketch.cu), so the result never depends on that heuristic.
//
// Roles (1 CTA per SM, 22 warps): warp 0 lane 0 issues tcgen05.mma; warp 1 lane 0 loads the raw X ring by 2D TMA
// (and prefetches STC_PF stages ahead into L2); warps 2..17 write the B bytes (two groups of 8 taking alternate
// stages); warps 18..21 build the E tile from Philox (theta.cuh; two groups of 2).  At the end warps 0..3 drain
// TMEM (tcgen05.ld, lane = Theta row) and write the fp64 partial sums.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>
#include <algorithm>
#include <type_traits>
#include "internal.cuh"
#include "tcgen05.cuh"
#include "theta.cuh"

namespace rcq {

constexpr int STC_M = 128;        // Theta rows per CTA (MMA M = TMEM lanes)
constexpr int STC_N = 64;         // X columns per CTA
constexpr int STC_KC = 64;        // X rows per stage (2 MMA k-steps of 32)
constexpr int STC_PF = 8;         // stages prefetched into L2 ahead of the raw ring
constexpr int STC_DWARPS = 8;     // B-byte warps per stage group
constexpr int STC_DGROUPS = 2;    // B-byte groups (warps 2..9, 10..17) alternating stages, like the E groups
constexpr int STC_EWARPS = 4;     // E-tile warps (18..21): two groups alternating stages, one X row per lane
constexpr int STC_THREADS = 32 * (2 + STC_DGROUPS * STC_DWARPS + STC_EWARPS);
constexpr int STC_E_BYTES = STC_M * STC_KC;              // E tile (int8, K-major)
static_assert(16 * STC_EWARPS == STC_KC, "one X row per E-warp lane, two warp groups");

#ifndef RCQ_STC_F2F
#define RCQ_STC_F2F 1             // fp32 X -> double by F2F.F64.F32 (0: built from the float's bits, x 2^-128)
#endif
template <typename TX> struct Fmt;
// B row layout (bytes along N) and the two MMAs per k-step (N0 + N1 columns):
//   fp32: [lo words of the 64 columns (256 B) | hi halves (128 B) | 16 ones]: N = 256 + 144.  The two constant
//         exponent bytes of each magic double are NOT fed to the tensor core (22% fewer MACs than 8 bytes per
//         element); the ones block gives S_r = sum_i E_ri for the 2^47 bias.
//   fp64: the 8 signed digit bytes of each element: N = 256 + 256.
template <> struct Fmt<float> {
  static constexpr int FB = 47;
  static constexpr int RAW = 5, DIG = 4;   // raw X ring / operand ring depths (DIG = 4: slot pairs, see below)
  static constexpr bool SIGNED = false;
  static constexpr int N0 = 256, N1 = 144;
};
template <> struct Fmt<double> {
  static constexpr int FB = 63;
  static constexpr int RAW = 2, DIG = 4;
  static constexpr bool SIGNED = true;
  static constexpr int N0 = 256, N1 = 256;
};

static_assert(Fmt<float>::DIG == 4 && Fmt<double>::DIG == 4, "slot pairs: stages c, c+1 share one release");

template <typename TX>
struct StcCfg {
  using Fm = Fmt<TX>;
  static constexpr int BN = Fm::N0 + Fm::N1;                  // B columns
  static constexpr int LBO = (BN / 16) * 128;                 // B: byte stride between 8-row K groups
  static constexpr int B_BYTES = STC_KC * BN;
  static constexpr int DIG_STAGE = STC_E_BYTES + B_BYTES;
  static constexpr int RAW_STAGE = STC_KC * STC_N * (int)sizeof(TX);
  static constexpr int CE = 16 / (int)sizeof(TX);            // elements per 16-byte raw chunk (4 / 2)
  static constexpr int CHUNKS = STC_N / CE;                   // raw chunks per row (16 / 32)
  static constexpr int CB = CHUNKS / 8;                       // blocks of 8 chunks (2 / 4)
  static constexpr int TASKS = STC_KC * CHUNKS / (32 * STC_DWARPS);   // chunks per thread per stage (4 / 8)
  static constexpr size_t SMEM = (size_t)Fm::DIG * DIG_STAGE + (size_t)Fm::RAW * RAW_STAGE + 1024;
  static_assert(SMEM <= 232448, "shared memory");
  static_assert(TASKS * (4 / CB) == 8 || CB == 4, "task mapping covers the 8 row blocks");
};

// Per-(CTA, column) scale: e = (exponent bound of the first stage's max |x|) + 4 bits of headroom.
struct ColParam {
  double s;          // fp32: 2^(47 - e) (RCQ_STC_F2F = 0: 2^(175 - e), applied to x 2^-128); fp64: 2^(31 - e)
  uint32_t lim;      // fp64: |x| high word must be < lim (high word of 2^e)
  bool bad;          // scale outside the exact construction range: fall back
  int e;
};

__device__ __forceinline__ uint32_t hi_abs(float x) { return __float_as_uint(x) & 0x7FFFFFFFu; }
__device__ __forceinline__ uint32_t hi_abs(double x) { return (uint32_t)__double2hiint(x) & 0x7FFFFFFFu; }

template <typename TX>
__device__ __forceinline__ ColParam col_param(uint32_t maxbits) {
  ColParam p{};
  int emax;                                                 // max |x| < 2^emax
  if constexpr (sizeof(TX) == 4) {
    emax = maxbits < 0x00800000u ? -126 : (int)(maxbits >> 23) - 126;
    if (maxbits == 0u) emax = -44;       // all-zero first stage: later |x| >= 2^-40 overflows -> fallback
    p.e = emax + 4;
    p.s = ldexp(1.0, (RCQ_STC_F2F ? 0 : 128) + Fmt<float>::FB - p.e);
    p.bad = p.e < -70;                   // subnormal inputs could then round to nonzero digits
  } else {
    emax = maxbits < 0x00100000u ? -1022 : (int)(maxbits >> 20) - 1022;
    p.e = emax + 4;
    const int be = p.e + 1023;
    p.lim = be >= 2047 ? 0x7FF00000u : (be <= 0 ? 0u : (uint32_t)be << 20);
    p.s = ldexp(1.0, 31 - p.e);
    p.bad = p.e < -900 || p.e > 900;
    if (maxbits == 0u) p.lim = 1u;       // all-zero first stage: any nonzero falls back
  }
  return p;
}

// fp32: the magic double t = RN(x 2^(47-e) + 1.5 2^52 + 2^47) as (lo, hi) words: lo, hi bytes 0, 1 = the
// unsigned digits of F + 2^47, hi bytes 2, 3 = 0x38, 0x43 unless F overflowed.  x 2^-128 is built exactly from
// the float's bits (normal x; one shift, one LOP3), so the scaling is one DFMA.
__device__ __forceinline__ uint2 magic_word(float x, double s) {
#if RCQ_STC_F2F
  // one exact F2F.F64.F32 on the conversion pipe instead of three integer-pipe instructions (s = 2^(47-e))
  const double tf = fma((double)x, s, kMagic + 140737488355328.0);
  return make_uint2((uint32_t)__double2loint(tf), (uint32_t)__double2hiint(tf));
#endif
  const uint32_t u = __float_as_uint(x);
  uint32_t h;                                                                      // x 2^-128: one LOP3
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(h) : "r"((uint32_t)((int32_t)u >> 3)), "r"(0x8FFFFFFFu), "r"(0x30000000u));
  const double t = fma(__hiloint2double((int)h, (int)(u << 29)), s, kMagic + 140737488355328.0);
  return make_uint2((uint32_t)__double2loint(t), (uint32_t)__double2hiint(t));
}
// fp64: F + C (C = 0x80 in bytes 0..6) by two magic-constant floors, returned as the signed digits (bytes XOR
// 0x80 but the top one): byte b has weight 256^b
__device__ __forceinline__ uint2 magic_word(double x, double s) {
  const double t1 = __fma_rd(x, s, kMagic + (double)0x808080u);
  const double H = t1 - (kMagic + (double)0x808080u);       // floor(x 2^(31-e)), exact
  const double r = fma(x, s, -H);                          // in [0, 1), exact
  const double t2 = __fma_rd(r, 4294967296.0, kMagic + (double)0x80808080u);
  const uint32_t lo = (uint32_t)__double2loint(t2);
  const uint32_t hi = (uint32_t)__double2loint(t1) + ((uint32_t)__double2hiint(t2) & 1u);   // carry of L + C_lo
  return make_uint2(lo ^ 0x80808080u, hi ^ 0x00808080u);
}

// CM: X column-major (element (i, j) at X[j * ldx + i]): the tensor map's contiguous dimension is
// the row, a raw stage is [64 columns][64 rows], and the B-byte warps take their elements with conflict-free
// scalar LDS (thread -> fixed chunk, 8-row blocks rotated per lane octet); E, B, the MMAs and TMEM are the same.
template <typename TX, bool CM>
__global__ void __launch_bounds__(STC_THREADS, 1)
sketch_sparse_tc_kernel(const __grid_constant__ CUtensorMap xmap, int64_t m, int n, int64_t row_offset, int k,
                        int zeta, uint64_t seed, int tiles_k, int tiles_n, int64_t rows_per_split,
                        double* __restrict__ part, int* overflow, int dbg_in, const uint64_t* __restrict__ srht_s,
                        double* __restrict__ cs_part) {
  const int dbg = kAblation ? dbg_in : 0;   // ablation switches (see internal.cuh)
  using C = StcCfg<TX>;
  using F = Fmt<TX>;
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* dig_base = sm;                                                 // [DIG][E | B]
  TX* raw_base = reinterpret_cast<TX*>(sm + (size_t)F::DIG * C::DIG_STAGE);    // [RAW][KC][64]
  uint64_t* dfull = reinterpret_cast<uint64_t*>(sm + (size_t)F::DIG * C::DIG_STAGE + (size_t)F::RAW * C::RAW_STAGE);
  uint64_t* dempty = dfull + F::DIG;      // [2]: one per PAIR of operand slots
  uint64_t* rfull = dempty + 2;
  uint64_t* rempty = rfull + F::RAW;
  uint64_t* done = rempty + F::RAW;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  uint32_t* col_max = tmem_slot + 1;                                            // [STC_N] high |x| bits
  int* col_exp = reinterpret_cast<int*>(col_max + STC_N);                      // [STC_N]

  const int tk = blockIdx.x % tiles_k, tn = (blockIdx.x / tiles_k) % tiles_n, split = blockIdx.x / (tiles_k * tiles_n);
  const int r0 = tk * STC_M, n0 = tn * STC_N;
  const int64_t i_begin = (int64_t)split * rows_per_split;
  const int64_t i_end = min(m, i_begin + rows_per_split);
  const int nstages = i_end > i_begin ? (int)((i_end - i_begin + STC_KC - 1) / STC_KC) : 0;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int beta = zeta > 0 ? k / zeta : 1;            // zeta <= 0: dense Rademacher / SRHT E (no blocks)

  if (tid == 0) {
    for (int s = 0; s < F::DIG; ++s) {
      tc::mbar_init(&dfull[s], STC_DWARPS + STC_EWARPS / 2);
      if (s < 2) tc::mbar_init(&dempty[s], 1);
    }
    for (int s = 0; s < F::RAW; ++s) { tc::mbar_init(&rfull[s], 1); tc::mbar_init(&rempty[s], STC_DWARPS); }
    tc::mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (tid < STC_N) { col_max[tid] = 0u; col_exp[tid] = 0; }
  if constexpr (sizeof(TX) == 4) {   // the constant ones block (MN group 24) of every operand slot
    for (int u = tid; u < F::DIG * STC_KC; u += STC_THREADS) {
      const int sl = u / STC_KC, i = u % STC_KC;
      *reinterpret_cast<uint4*>(dig_base + (size_t)sl * C::DIG_STAGE + STC_E_BYTES + (i & 7) * 16 + 24 * 128 + (i >> 3) * C::LBO) =
          make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(tc::smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------------------------------------------------------- MMA issuer (lane 0)
    constexpr uint32_t id0 = tc::idesc_i8(STC_M, F::N0, true, F::SIGNED) | (1u << 16);   // B MN-major
    constexpr uint32_t id1 = tc::idesc_i8(STC_M, F::N1, true, F::SIGNED) | (1u << 16);
    for (int c = 0; c < nstages; ++c) {
      const int s = c % F::DIG;
      tc::mbar_wait(&dfull[s], (uint32_t)((c / F::DIG) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      if (lane == 0) {
        const uint32_t sa = tc::smem_u32(dig_base + (size_t)s * C::DIG_STAGE);
        if (!(dbg & 1)) {
#pragma unroll
          for (int ks = 0; ks < STC_KC / 32; ++ks) {
            const uint64_t da = tc::desc(sa + ks * 2 * (STC_M / 8) * 128, (STC_M / 8) * 128, 128);
            const uint32_t accum = (c > 0 || ks > 0) ? 1u : 0u;
            const uint32_t sb = sa + STC_E_BYTES + ks * 4 * C::LBO;
            tc::mma_i8(tmem, da, tc::desc(sb, C::LBO, 128), id0, accum);
            tc::mma_i8(tmem + F::N0, da, tc::desc(sb + (F::N0 / 16) * 128, C::LBO, 128), id1, accum);
          }
        }
        // one tcgen05.commit per TWO stages (8 MMAs): a commit costs the tensor pipe ~100-400 cycles, so at
        // 4 MMAs per commit the pipe ran at ~45% (tools/micro/tc_commit_rate.cu); it releases the slot pair
        if ((c & 1) || c == nstages - 1) tc::commit(&dempty[(c >> 1) & 1]);
        if (c == nstages - 1) tc::commit(done);
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- X loader (2D TMA, lane 0)
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(&xmap) : "memory");
      for (int c = 1; c < STC_PF && c < nstages; ++c) {
        const int pr = (int)(i_begin + (int64_t)c * STC_KC);
        if (CM) tc::tma_prefetch_2d(&xmap, pr, n0); else tc::tma_prefetch_2d(&xmap, n0, pr);
      }
    }
    for (int c = 0; c < nstages; ++c) {
      const int s = c % F::RAW;
      if (c >= F::RAW) tc::mbar_wait(&rempty[s], (uint32_t)(((c / F::RAW) - 1) & 1));
      if (lane == 0) {
        if (c + STC_PF < nstages) {
          const int pr = (int)(i_begin + (int64_t)(c + STC_PF) * STC_KC);
          if (CM) tc::tma_prefetch_2d(&xmap, pr, n0); else tc::tma_prefetch_2d(&xmap, n0, pr);
        }
        tc::mbar_arrive_tx(&rfull[s], (uint32_t)C::RAW_STAGE);
        const int lr = (int)(i_begin + (int64_t)c * STC_KC);
        if (CM) tc::tma_load_2d(raw_base + (size_t)s * STC_KC * STC_N, &xmap, lr, n0, &rfull[s]);
        else tc::tma_load_2d(raw_base + (size_t)s * STC_KC * STC_N, &xmap, n0, lr, &rfull[s]);
      }
      __syncwarp();
    }
  } else if (warp < 2 + STC_DGROUPS * STC_DWARPS) {
    // ---------------------------------------------------------------- B bytes
    // Thread -> (fixed 16-byte raw chunk c of a row, rows 8 rb + q): lane = 8 p + q, chunk
    // c = 8 cb + ((q + p + rot) & 7).  Every 8-lane phase of an LDS.128 then reads 8 distinct bank groups
    // (c mod 8) and every phase of the STS.128 into B writes 8 distinct ones (row mod 8).
    const int dgrp = (warp - 2) / STC_DWARPS;            // stages c = dgrp (mod 2)
    const int w = (warp - 2) % STC_DWARPS, p = lane >> 3, q = lane & 7;
    const int wi = w & 3, rot = 4 * (w >> 2);
    const int cb = wi % C::CB, rbase = (wi / C::CB) * C::TASKS;
    // column-major: lane octet o = p takes 8 consecutive rows of one chunk; fp32: chunks 2 w + (o & 1), 8-row
    // blocks (2 t + (o >> 1) + 2 (o & 1)) mod 8; fp64: chunks 4 w + o, blocks (t + o) mod 8 -- the four octets of an
    // LDS read four distinct bank groups, the STS.128 of an octet is 128 contiguous bytes and the two octets of
    // an STS.64 phase write different 8-byte halves
    const int ch = !CM ? 8 * cb + ((q + p + rot) & 7)     // this thread's raw chunk (columns ch * CE .. + CE - 1)
                       : (sizeof(TX) == 4 ? 2 * w + (p & 1) : 4 * w + p);
    auto row_of = [&](int t) {                           // row (within the stage) of the thread's task t
      if constexpr (!CM) return 8 * (rbase + t) + q;
      else if constexpr (sizeof(TX) == 4) return 8 * ((2 * t + (p >> 1) + 2 * (p & 1)) & 7) + q;
      else return 8 * ((t + p) & 7) + q;
    };
    double sc[C::CE];
    uint32_t lim[C::CE];
    bool bad = false;
    if (nstages > 0) {                                   // column scales from the first stage (both groups)
      tc::mbar_wait(&rfull[0], 0u);
      const int rows0 = (int)min((int64_t)STC_KC, i_end - i_begin);
      const int dt = tid - 64, j = dt & (STC_N - 1);
      uint32_t mx = 0u;
      for (int r = dt >> 6; r < rows0; r += 32 * STC_DGROUPS * STC_DWARPS / STC_N)
        mx = max(mx, hi_abs(raw_base[CM ? j * STC_KC + r : r * STC_N + j]));
      atomicMax(&col_max[j], mx);
      tc::named_bar(1, 32 * STC_DGROUPS * STC_DWARPS);
#pragma unroll
      for (int e = 0; e < C::CE; ++e) {
        const ColParam cp = col_param<TX>(col_max[ch * C::CE + e]);
        sc[e] = cp.s; lim[e] = cp.lim;
        bad |= cp.bad && n0 + ch * C::CE + e < n;
      }
      if (dgrp == 0 && dt < STC_N) col_exp[dt] = col_param<TX>(col_max[dt]).e;
    }
    uint32_t acc = 0u;                                   // overflow detection
    // cs_part != null (Alg. 7): column sums of squares of X in this same pass over X
    double cs[C::CE];
#pragma unroll
    for (int e = 0; e < C::CE; ++e) cs[e] = 0.0;
    for (int c = dgrp; c < nstages; c += STC_DGROUPS) {
      const int s = c % F::DIG, sr = c % F::RAW;
      const int64_t i0 = i_begin + (int64_t)c * STC_KC;
      const int rows = (int)min((int64_t)STC_KC, i_end - i0);
      const TX* raw = raw_base + (size_t)sr * STC_KC * STC_N;
      if (c >= F::DIG) tc::mbar_wait(&dempty[(c >> 1) & 1], (uint32_t)(((c >> 2) - 1) & 1));   // slot pair free
      tc::mbar_wait(&rfull[sr], (uint32_t)((c / F::RAW) & 1));
      unsigned char* bt = dig_base + (size_t)s * C::DIG_STAGE + STC_E_BYTES;
      if (!(dbg & 2)) {
        // all of the thread's raw chunks first: the compiler cannot hoist an LDS above the STS of the previous
        // chunk (both shared memory), so a per-chunk loop paid one LDS latency per chunk
        TX xv[C::TASKS][C::CE];
#pragma unroll
        for (int t = 0; t < C::TASKS; ++t) {
          const int i = row_of(t);
          if constexpr (CM) {
#pragma unroll
            for (int e = 0; e < C::CE; ++e) xv[t][e] = raw[(ch * C::CE + e) * STC_KC + i];
          } else if constexpr (sizeof(TX) == 4) {
            const float4 f = *reinterpret_cast<const float4*>(raw + i * STC_N + ch * 4);
            xv[t][0] = f.x; xv[t][1] = f.y; xv[t][2] = f.z; xv[t][3] = f.w;
          } else {
            const double2 f = *reinterpret_cast<const double2*>(raw + i * STC_N + ch * 2);
            xv[t][0] = f.x; xv[t][1] = f.y;
          }
        }
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&rempty[sr]);     // raw slot consumed: the loader may refill it
        if (rows < STC_KC) {                             // rows of the next split (or past m): E is zero there
#pragma unroll
          for (int t = 0; t < C::TASKS; ++t)
            if (row_of(t) >= rows) {
#pragma unroll
              for (int e = 0; e < C::CE; ++e) xv[t][e] = (TX)0;
            }
        }
#pragma unroll
        for (int t = 0; t < C::TASKS; ++t) {
          const int i = row_of(t);
          uint2 wv[C::CE];
#pragma unroll
          for (int e = 0; e < C::CE; ++e) {
            if (cs_part) cs[e] = fma((double)xv[t][e], (double)xv[t][e], cs[e]);
            wv[e] = magic_word(xv[t][e], sc[e]);
            if constexpr (sizeof(TX) == 4) acc |= wv[e].y ^ 0x43380000u;
            else acc |= hi_abs(xv[t][e]) >= lim[e] ? 1u : 0u;
          }
          unsigned char* brow = bt + (i & 7) * 16 + (i >> 3) * C::LBO;   // row i, MN group 0
          if constexpr (sizeof(TX) == 4) {
            // lo words of columns 4 ch .. + 3 -> MN group ch; their hi halves (digits 4, 5) -> 8 bytes of group
            // 16 + ch / 2
            *reinterpret_cast<uint4*>(brow + ch * 128) = make_uint4(wv[0].x, wv[1].x, wv[2].x, wv[3].x);
            *reinterpret_cast<uint2*>(brow + (16 + (ch >> 1)) * 128 + (ch & 1) * 8) =
                make_uint2(__byte_perm(wv[0].y, wv[1].y, 0x5410), __byte_perm(wv[2].y, wv[3].y, 0x5410));
          } else {
            // element pair (2 ch, 2 ch + 1): the 8 digit bytes of each -> MN group ch
            *reinterpret_cast<uint4*>(brow + ch * 128) = make_uint4(wv[0].x, wv[0].y, wv[1].x, wv[1].y);
          }
        }
      } else {
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&rempty[sr]);
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // generic smem writes -> tensor core
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&dfull[s]);
    }
    bool ovf;
    if constexpr (sizeof(TX) == 4) ovf = (acc >> 16) != 0u;
    else ovf = acc != 0u;
    if (nstages > 0 && (ovf || bad)) atomicOr(overflow, 1);        // headroom exceeded / Inf / NaN
    if (cs_part) {
      // per-thread sums -> per-CTA column sums in a fixed order (thread index), through the raw ring (all B
      // warps are past their last raw read once the named barrier below completes)
      constexpr int NB = 32 * STC_DGROUPS * STC_DWARPS;
      const int bt = tid - 64;
      tc::named_bar(1, NB);
      double* scr = reinterpret_cast<double*>(raw_base);              // [NB][CE]
      int* sch = reinterpret_cast<int*>(scr + NB * C::CE);             // [NB] chunk of each thread
#pragma unroll
      for (int e = 0; e < C::CE; ++e) scr[bt * C::CE + e] = cs[e];
      sch[bt] = ch;
      tc::named_bar(1, NB);
      if (bt < STC_N && tk == 0 && n0 + bt < n) {
        double sum = 0.0;
        for (int t2 = 0; t2 < NB; ++t2)
          if (sch[t2] == bt / C::CE) sum += scr[t2 * C::CE + bt % C::CE];
        cs_part[(size_t)split * n + n0 + bt] = sum;
      }
    }
  } else {
    // ---------------------------------------------------------------- E tile (Philox, theta.cuh)
    // Two groups of two warps take alternate stages (group g: stages c = g mod 2), each lane one X
    // row; the Philox draw of a row is computed before its slot is awaited, so the generator
    // latency overlaps the MMAs still reading that slot.
    const int ew = warp - 2 - STC_DGROUPS * STC_DWARPS;
    const int grp = ew >> 1, half = ew & 1;               // rows half*32 + lane of stages c = grp (mod 2)
    const int ii = half * 32 + lane;
    const int zoff = half * 2 * STC_M * 16;               // k-blocks 2half, 2half+1 of the E tile
    const bool full_tile = (zeta == 8 && k <= STC_M);     // common case: 8 nonzeros, one Theta row tile
    const bool dense = zeta <= 0;                         // Rademacher (0, reading A22) / SRHT (-1, A23): all +-1
    const bool srht = zeta < 0;
    for (int c = grp; c < nstages; c += 2) {
      const int s = c % F::DIG;
      const int64_t i0 = i_begin + (int64_t)c * STC_KC;
      const int rows = (int)min((int64_t)STC_KC, i_end - i0);
      const uint64_t gi = (uint64_t)(row_offset + i0 + ii);
      const uint4 w = philox_at(seed, gi, srht ? 0u : (dense ? (uint32_t)tk : 0u),
                                srht ? kDomainSrhtD : (dense ? kDomainRademacher : kDomainSparse));
      if (c >= F::DIG) tc::mbar_wait(&dempty[(c >> 1) & 1], (uint32_t)(((c >> 2) - 1) & 1));   // slot pair free
      unsigned char* st = dig_base + (size_t)s * C::DIG_STAGE;
      if (dense) {
        // Transpose the warp's 32 X rows x 128 sign bits with ballots: mask (Theta row r) holds bit L =
        // sign of X row half*32 + L; lane r & 31 keeps the masks of rows r = lane + 32 q.  Each mask is
        // expanded to two 16-byte K-runs (k-blocks 2 half, 2 half + 1) of +-1 bytes (0 beyond `rows`).
        const uint32_t valid = __ballot_sync(0xffffffffu, ii < rows);
        uint32_t mine[4];
        if (srht) {
          // lane L takes Theta rows r = r0 + L + 32 q.  The warp's global rows are B + lane' with
          // B = gi - lane a multiple of 32 (row_offset % 32 == 0), so popcount(s & (B + lane')) splits
          // as popcount(s & B) + popcount(s & lane'): the mask over lane' is the Walsh mask of s & 31,
          // flipped when popcount(s & B) is odd, XOR the ballot of the d_i signs.
          const uint32_t dmask = __ballot_sync(0xffffffffu, w.x & 1u);
          const uint64_t B = gi - (uint64_t)lane;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int r = r0 + lane + 32 * q;
            const uint64_t sr = r < k ? srht_s[r] : 0ull;
            const uint32_t t = (uint32_t)sr & 31u;
            uint32_t wm = 0u;
            wm ^= (t & 1u) ? 0xAAAAAAAAu : 0u;
            wm ^= (t & 2u) ? 0xCCCCCCCCu : 0u;
            wm ^= (t & 4u) ? 0xF0F0F0F0u : 0u;
            wm ^= (t & 8u) ? 0xFF00FF00u : 0u;
            wm ^= (t & 16u) ? 0xFFFF0000u : 0u;
            mine[q] = wm ^ ((__popcll(sr & B) & 1) ? 0xFFFFFFFFu : 0u) ^ dmask;
          }
        } else {
          // 32 x 32 bit-matrix transpose per word (row = lane's X row, column = Theta row 32 q + b): a
          // butterfly of 5 shuffle levels; at level j, lanes with bit j clear keep their bit positions
          // with bit j clear and take the partner's into the others, and vice versa.
          const uint32_t wd[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint32_t x = wd[q];
#pragma unroll
            for (int j = 16; j >= 1; j >>= 1) {
              const uint32_t m = j == 16 ? 0x0000FFFFu : j == 8 ? 0x00FF00FFu : j == 4 ? 0x0F0F0F0Fu
                                 : j == 2 ? 0x33333333u : 0x55555555u;   // bit positions with bit j clear
              const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
              x = (lane & j) ? ((x & ~m) | ((y & ~m) >> j)) : ((x & m) | ((y & m) << j));
            }
            mine[q] = x;                          // bit L = sign bit of X row L for Theta row 32 q + lane
          }
        }
        if (!(dbg & 4)) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int r = 32 * q + lane;
#pragma unroll
            for (int hb = 0; hb < 2; ++hb) {
              uint32_t out[4];
#pragma unroll
              for (int nb = 0; nb < 4; ++nb) {
                const uint32_t sh = 16 * hb + 4 * nb;
                const uint32_t sg = (((mine[q] >> sh) & 0xFu) * 0x00204081u) & 0x01010101u;
                const uint32_t vb = (((valid >> sh) & 0xFu) * 0x00204081u) & 0x01010101u;
                out[nb] = (0x01010101u + sg * 0xFEu) & (vb * 0xFFu);
              }
              *reinterpret_cast<uint4*>(st + (2 * half + hb) * STC_M * 16 + r * 16) =
                  make_uint4(out[0], out[1], out[2], out[3]);
            }
          }
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&dfull[s]);
        continue;
      }
      uint4* zb = reinterpret_cast<uint4*>(st + zoff);
#pragma unroll
      for (int u = 0; u < 2 * STC_M * 16 / 16 / 32; ++u) zb[u * 32 + lane] = make_uint4(0, 0, 0, 0);
      __syncwarp();
      if (ii < rows && !(dbg & 4)) {
        unsigned char* eb = st + (ii >> 4) * STC_M * 16 + (ii & 15);
        if (full_tile) {
          const uint32_t wd[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const uint32_t hh = (t & 1) ? (wd[t >> 1] >> 16) : (wd[t >> 1] & 0xFFFFu);
            const int r = t * beta + (int)(((hh & 0x7FFFu) * (uint32_t)beta) >> 15);
            eb[r * 16] = (unsigned char)((hh >> 15) ? 0xFF : 0x01);
          }
        } else {
          uint4 ww = w;
          for (int t = 0; t < zeta; ++t) {
            if (t > 0 && (t & 7) == 0) ww = philox_at(seed, gi, (uint32_t)(t >> 3), kDomainSparse);
            const uint32_t hh = sparse_halfword(ww, t);
            const int r = sparse_row(hh, t, beta) - r0;
            if (r >= 0 && r < STC_M) eb[r * 16] = (unsigned char)((hh >> 15) ? 0xFF : 0x01);
          }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&dfull[s]);
    }
  }

  // -------------------------------------------------------------------- epilogue (warps 0..3)
  if (warp < 4) {
    double* Pp = part + (size_t)split * (size_t)k * n;
    const int row = r0 + warp * 32 + lane;             // TMEM lane = Theta row
    const uint32_t lbase = tmem + ((uint32_t)(warp * 32) << 16);
    const int ncols = min(STC_N, n - n0);
    if (nstages > 0) {
      tc::mbar_wait(done, 0u);
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      if constexpr (!F::SIGNED) {
        // fp32: F + 2^47 = sum_b lo_b 256^b + hi_0 256^4 + hi_1 256^5; the bias 2^47 S_r = 128 S_r at 256^5
        uint32_t o[8];
        tc::ld8(lbase + 384, o);                         // ones block: S_r
        tc::wait_ld();
        const int32_t bias = 128 * (int32_t)o[0];
#pragma unroll 1
        for (int j0 = 0; j0 < STC_N; j0 += 4) {
          uint32_t lo[16], hi[8];                        // columns j0 .. j0 + 3
          tc::ld16(lbase + 4 * j0, lo);
          tc::ld8(lbase + F::N0 + 2 * j0, hi);
          tc::wait_ld();
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int j = j0 + u;
            double v = (double)((int32_t)hi[2 * u + 1] - bias);
            v = fma(v, 256.0, (double)(int32_t)hi[2 * u]);
#pragma unroll
            for (int t = 3; t >= 0; --t) v = fma(v, 256.0, (double)(int32_t)lo[4 * u + t]);
            if (row < k && j < ncols) Pp[(size_t)row * n + n0 + j] = ldexp(v, col_exp[j] - F::FB);
          }
        }
      } else {
#pragma unroll 1
        for (int j0 = 0; j0 < STC_N; j0 += 2) {
          uint32_t a[16];                                // the 8 digit accumulators of columns j0, j0 + 1
          tc::ld16(lbase + 8 * j0, a);
          tc::wait_ld();
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int j = j0 + u;
            double v = (double)(int32_t)a[8 * u + 7];
#pragma unroll
            for (int t = 6; t >= 0; --t) v = fma(v, 256.0, (double)(int32_t)a[8 * u + t]);
            if (row < k && j < ncols) Pp[(size_t)row * n + n0 + j] = ldexp(v, col_exp[j] - F::FB);
          }
        }
      }
    } else if (row < k) {
      for (int j = 0; j < ncols; ++j) Pp[(size_t)row * n + n0 + j] = 0.0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

// tcgen05 path: any n (64-column tiles), k <= 4 * 128 Theta rows
static_assert(sizeof(double) * 32 * STC_DGROUPS * STC_DWARPS * 4 + sizeof(int) * 32 * STC_DGROUPS * STC_DWARPS <=
              (size_t)Fmt<double>::RAW * STC_KC * STC_N * sizeof(double), "column-sum scratch fits the raw ring");
bool sparse_tc_applicable(int k, int n, int zeta) { return n >= 1 && zeta >= 1 && k % zeta == 0 && k <= 4 * STC_M; }

using EncodeTiledFnS = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <typename TX>
static cudaError_t launch_stc(const TX* X, int64_t m, int n, int64_t ldx, int64_t ro, int k, int zeta, uint64_t seed,
                              int tiles_k, int splits, int64_t rps, double* part, int* overflow, cudaStream_t st,
                              const uint64_t* srht_s, double* cs_part, bool colmajor) {
  static EncodeTiledFnS enc = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFnS>(p);
  }();
  if (!enc) return cudaErrorNotSupported;
  CUtensorMap map;
  // row-major: dims (columns, rows), box (64 columns, 64 rows); column-major: dims (rows, columns), box (64 rows, 64 columns)
  const cuuint64_t dims[2] = {(cuuint64_t)(colmajor ? m : n), (cuuint64_t)(colmajor ? n : m)};
  const cuuint64_t strides[1] = {(cuuint64_t)ldx * sizeof(TX)};
  const cuuint32_t box[2] = {(cuuint32_t)(colmajor ? STC_KC : STC_N), (cuuint32_t)(colmajor ? STC_N : STC_KC)}, estr[2] = {1, 1};
  if (enc(&map, sizeof(TX) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
          const_cast<TX*>(X), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorNotSupported;
  auto kern = colmajor ? sketch_sparse_tc_kernel<TX, true> : sketch_sparse_tc_kernel<TX, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)StcCfg<TX>::SMEM);
  if (e != cudaSuccess) return e;
  static const int dbg = !kAblation ? 0 : getenv("RCHOLQR_STC_DEBUG") ? atoi(getenv("RCHOLQR_STC_DEBUG")) : 0;   // ablations only
  const int tiles_n = (n + STC_N - 1) / STC_N;
  kern<<<tiles_k * tiles_n * splits, STC_THREADS, StcCfg<TX>::SMEM, st>>>(map, m, n, ro, k, zeta, seed, tiles_k, tiles_n,
                                                                           rps, part, overflow, dbg, srht_s, cs_part);
  return cudaGetLastError();
}

cudaError_t launch_sparse_tc(const void* X, int dtype, int64_t m, int n, int64_t ldx, int64_t row_offset, int k,
                             int zeta, uint64_t seed, int splits, int64_t rows_per_split, double* part, int* overflow,
                             cudaStream_t st, const uint64_t* srht_s, double* cs_part, bool colmajor) {
  const int tiles_k = (k + STC_M - 1) / STC_M;
  if (dtype == RCHOLQR_F64)
    return launch_stc((const double*)X, m, n, ldx, row_offset, k, zeta, seed, tiles_k, splits, rows_per_split, part,
                      overflow, st, srht_s, cs_part, colmajor);
  return launch_stc((const float*)X, m, n, ldx, row_offset, k, zeta, seed, tiles_k, splits, rows_per_split, part,
                    overflow, st, srht_s, cs_part, colmajor);
}

// 2D TMA of X: 16-byte aligned base and row pitch, row coordinates < 2^31
bool sparse_tc_aligned(const void* X, int dtype, int64_t m, int64_t ldx) {
  const size_t es = dtype == RCHOLQR_F64 ? 8 : 4;
  return ((uintptr_t)X % 16) == 0 && ((size_t)ldx * es) % 16 == 0 && m < ((int64_t)1 << 31);
}

#ifdef RCHOLQR_ABLATION
RCQ_TRACE_READER(trace_read_sketch)
#endif

}  // namespace rcq
