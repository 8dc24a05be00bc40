// sketch_tc.cu -- sparse-sign sketch on the 5th-generation tensor core (tcgen05.mma kind::i8).
//
// P = E X / sqrt(zeta) (Alg. 2 step 1 with the sparse-sign Theta of reading A3):
// E (k x m) has entries in {-1, 0, +1}, i.e. it is EXACT in int8.  X is written exactly as a
// fixed-point integer against a per-(CTA, column) power-of-two scale 2^e_j,
//     F(x) = trunc(x 2^(FB - e_j)),  FB = 7 + 8 (D-1),  |F| < 2^FB,
// and F is split into D two's-complement bytes (d_0 signed, d_1.. unsigned):
//     F = d_0 2^(8(D-1)) + d_1 2^(8(D-2)) + ... + d_{D-1}.
// D = 6 (fp32 X, FB = 47) or 8 (fp64 X, FB = 63).  Each digit plane is one int8 GEMM into its own
// int32 TMEM accumulator, which is exact while rows * 255 < 2^31 (kSparseTcMaxRows), so the only
// approximation is the truncation of x below 2^(e_j - FB): relative 2^-43 (fp32) / 2^-59 (fp64)
// of the column scale -- the "random projection in higher precision" of PAPER.md:83, 423.
// e_j = (exponent of the column maximum over the CTA's FIRST stage) + 4 bits of headroom.  If a
// later element of the CTA does not fit (|x| >= 2^e_j, or Inf/NaN) the kernel raises an overflow
// flag and the register sparse kernel (sketch.cu) recomputes the whole sketch, so the result never
// depends on that heuristic.
//
// Roles (1 CTA per SM, 22 warps): warp 0 lane 0 issues tcgen05.mma and commits to mbarriers;
// warp 1 lane 0 streams X rows into a raw shared-memory ring with cp.async.bulk (mbarrier
// complete_tx); warps 2..21 build each stage's operands -- the D digit planes (two groups of 8 warps
// taking alternate stages) and the E tile from Philox (theta.cuh; two groups of 2 warps) -- in the
// canonical K-major SWIZZLE_NONE core-matrix layout.  At the end warps 0..3 drain TMEM (tcgen05.ld,
// lane = Theta row) and write the fp64 partial sums.  (Round 1 had one digit group of 8 warps: the
// digit warps were latency-bound at 44% issue with 3.5 warps per scheduler; C4 sketch 5.45 ms.)
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>
#include <type_traits>
#include "internal.cuh"
#include "tcgen05.cuh"
#include "theta.cuh"

namespace rcq {


constexpr int STC_M = 128;        // Theta rows per CTA (MMA M = TMEM lanes)
constexpr int STC_N = 64;         // X columns per CTA (MMA N)
constexpr int STC_KC = 64;        // X rows per stage (2 MMA k-steps of 32)
constexpr int STC_PF = 8;         // stages prefetched into L2 ahead of the raw ring (contiguous X)
constexpr int STC_DWARPS = 8;     // digit-plane warps per stage group: one (column, 16-row group) task per thread
constexpr int STC_DGROUPS = 2;    // digit groups (warps 2..9, 10..17) alternating stages, like the E groups
constexpr int STC_EWARPS = 4;     // E-tile warps (18..21): two groups alternating stages, one X row per lane
constexpr int STC_THREADS = 32 * (2 + STC_DGROUPS * STC_DWARPS + STC_EWARPS);
static_assert(32 * STC_DWARPS == STC_N * (STC_KC / 16), "one digit task per thread");
static_assert(16 * STC_EWARPS == STC_KC, "one X row per E-warp lane, two warp groups");

// Digit split of one element.  F(x) = round(x 2^(FB-e)) is
// written in base 256 with D digits, each digit plane one int8 operand; several planes are stacked
// along N so one MMA covers them (N = 192..256).
//   fp32 X (D = 6, FB = 47, the C4 hot path): x 2^-128 is built exactly from the float's bits (one
//     shift, one LOP3: exponent 0x300 | exp_f), and ONE round-to-nearest DFMA by 2^(175-e) onto
//     1.5 2^52 + 2^47 leaves F + 2^47 in the low 48 mantissa bits: six UNSIGNED digits, hi word
//     bytes 1,0 = d0,d1, lo word bytes 3..0 = d2..d5.  The bias 2^47 = 128 * 256^5 is removed
//     exactly in the epilogue with S_r = sum_i E_ri, which a constant ones-block in the first
//     MMA group accumulates (acc_0 - 128 S).  The high word is 0x4338xxxx iff F + 2^47 fits in
//     48 bits, so OR/AND accumulators of it detect overflow, Inf and NaN.
//   fp64 X (D = 8, FB = 63): H = floor(x 2^(31-e)) + C_hi, L = floor(frac 2^32) + C_lo by magic-
//     constant floors; SIGNED digits via the offset C (0x80 in all bytes but the top one; digit
//     bytes XOR 0x80), carry of L into H -> hi word bytes 3..0 = d0..d3, lo = d4..d7.
// All steps are exact (power-of-two scalings, magic-constant roundings of integers < 2^51).
template <typename TX> struct Fmt;
template <> struct Fmt<float> {
  static constexpr int D = 6, FB = 47;
  static constexpr int RAW = 4, DIG = 4;   // raw X ring / operand ring depths
  static constexpr int ONES = 16;          // ones-block rows in group 0 (bias correction)
  static constexpr bool SIGNED = false;
};
template <> struct Fmt<double> {
  static constexpr int D = 8, FB = 63;
  static constexpr int RAW = 3, DIG = 3;
  static constexpr int ONES = 0;
  static constexpr bool SIGNED = true;
};

template <typename TX>
struct StcCfg {
  using Fm = Fmt<TX>;
  static constexpr int D = Fm::D;
  static constexpr int PG = D / 2;                                  // digit planes per MMA group
  static constexpr int N0 = Fm::ONES + PG * STC_N;                  // group 0: [ones | planes 0..PG-1]
  static constexpr int N1 = (D - PG) * STC_N;                       // group 1: planes PG..D-1
  static constexpr int TBASE1 = 256;                                // TMEM column of group 1
  static constexpr int E_BYTES = STC_M * STC_KC;                    // E tile (int8)
  static constexpr int G0_BYTES = N0 * STC_KC, G1_BYTES = N1 * STC_KC;
  static constexpr int DIG_STAGE = E_BYTES + G0_BYTES + G1_BYTES;
  static constexpr int RAW_STAGE = STC_KC * STC_N * (int)sizeof(TX);
  static constexpr size_t SMEM = (size_t)Fm::DIG * DIG_STAGE + (size_t)Fm::RAW * RAW_STAGE + 1024;
  static_assert(N0 <= 256 && N0 % 16 == 0 && N1 <= 256 && N1 % 16 == 0, "MMA N");
  static_assert(N0 <= TBASE1 && TBASE1 + N1 <= 512, "TMEM columns");
  // plane t: group, row inside the group's B tile, TMEM column
  static __device__ __forceinline__ int grp(int t) { return t < PG ? 0 : 1; }
  static __device__ __forceinline__ int brow(int t) { return t < PG ? Fm::ONES + t * STC_N : (t - PG) * STC_N; }
  static __device__ __forceinline__ int tcol(int t) { return t < PG ? Fm::ONES + t * STC_N : TBASE1 + (t - PG) * STC_N; }
};

// Per-(CTA, column) scale: e = (exponent bound of the first stage's max |x|) + 4 bits of headroom.
struct ColParam {
  double s;          // fp32: 2^(175 - e) (applied to x 2^-128); fp64: 2^(31 - e)
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
    p.s = ldexp(1.0, 128 + Fmt<float>::FB - p.e);
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

// fp32: (hi, lo) words of t = RN(x 2^(47-e) + 1.5 2^52 + 2^47)
__device__ __forceinline__ void split_words(float x, const ColParam& p, uint32_t& hi, uint32_t& lo) {
  const uint32_t u = __float_as_uint(x);
  const uint32_t h = ((uint32_t)((int32_t)u >> 3) & 0x8FFFFFFFu) | 0x30000000u;   // x 2^-128 (normal x)
  const double y = __hiloint2double((int)h, (int)(u << 29));
  const double t = fma(y, p.s, kMagic + 140737488355328.0);                       // + 2^47
  hi = (uint32_t)__double2hiint(t);
  lo = (uint32_t)__double2loint(t);
}
// fp64: (hi, lo) words holding F(x) + C (signed digits, see above)
__device__ __forceinline__ void split_words(double x, const ColParam& p, uint32_t& hi, uint32_t& lo) {
  const double t1 = __fma_rd(x, p.s, kMagic + (double)0x808080u);
  const double H = t1 - (kMagic + (double)0x808080u);       // floor(x 2^(31-e)), exact
  const double r = fma(x, p.s, -H);                          // in [0, 1), exact
  const double t2 = __fma_rd(r, 4294967296.0, kMagic + (double)0x80808080u);
  lo = (uint32_t)__double2loint(t2);
  hi = (uint32_t)__double2loint(t1) + ((uint32_t)__double2hiint(t2) & 1u);   // carry of L + C_lo
}

template <typename TX>
__global__ void __launch_bounds__(STC_THREADS, 1)
sketch_sparse_tc_kernel(const TX* __restrict__ X, int64_t m, int n, int64_t ldx, int64_t row_offset, int k, int zeta,
                        uint64_t seed, int tiles_k, int64_t rows_per_split, double* __restrict__ part, int* overflow, int dbg_in,
                        const uint64_t* __restrict__ srht_s) {
  const int dbg = kAblation ? dbg_in : 0;   // ablation switches (see internal.cuh)
  using C = StcCfg<TX>;
  using F = Fmt<TX>;
  constexpr int D = C::D;
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* dig_base = sm;                                                 // [DIG][DIG_STAGE]
  TX* raw_base = reinterpret_cast<TX*>(sm + (size_t)F::DIG * C::DIG_STAGE);    // [RAW][KC][n]
  uint64_t* dfull = reinterpret_cast<uint64_t*>(sm + (size_t)F::DIG * C::DIG_STAGE + (size_t)F::RAW * C::RAW_STAGE);
  uint64_t* dempty = dfull + F::DIG;
  uint64_t* rfull = dempty + F::DIG;
  uint64_t* rempty = rfull + F::RAW;
  uint64_t* done = rempty + F::RAW;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  uint32_t* col_max = tmem_slot + 1;                                            // [STC_N] high |x| bits
  int* col_exp = reinterpret_cast<int*>(col_max + STC_N);                      // [STC_N]

  const int tk = blockIdx.x % tiles_k, split = blockIdx.x / tiles_k;
  const int r0 = tk * STC_M;
  const int64_t i_begin = (int64_t)split * rows_per_split;
  const int64_t i_end = min(m, i_begin + rows_per_split);
  const int nstages = i_end > i_begin ? (int)((i_end - i_begin + STC_KC - 1) / STC_KC) : 0;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int beta = zeta > 0 ? k / zeta : 1;            // zeta = 0: dense Rademacher E (no blocks)

  if (tid == 0) {
    for (int s = 0; s < F::DIG; ++s) {
      tc::mbar_init(&dfull[s], STC_DWARPS + STC_EWARPS / 2);
      tc::mbar_init(&dempty[s], 1);
    }
    for (int s = 0; s < F::RAW; ++s) { tc::mbar_init(&rfull[s], 1); tc::mbar_init(&rempty[s], STC_DWARPS); }
    tc::mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (tid < STC_N) { col_max[tid] = 0u; col_exp[tid] = 0; }
  if constexpr (F::ONES > 0) {   // constant ones-block (rows 0..15 of group 0) in every operand slot
    for (int u = tid; u < F::DIG * F::ONES * STC_KC / 16; u += STC_THREADS) {
      const int s = u / (F::ONES * STC_KC / 16), v = u % (F::ONES * STC_KC / 16);
      const int r = v % F::ONES, kb = v / F::ONES;
      *reinterpret_cast<uint4*>(dig_base + (size_t)s * C::DIG_STAGE + C::E_BYTES + cm_off(r, kb * 16, C::N0)) =
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
    constexpr uint32_t id0 = tc::idesc_i8(STC_M, C::N0, true, F::SIGNED);   // E (s8) x digit group
    constexpr uint32_t id1 = tc::idesc_i8(STC_M, C::N1, true, F::SIGNED);
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
            const uint32_t sb0 = sa + C::E_BYTES + ks * 2 * (C::N0 / 8) * 128;
            const uint32_t sb1 = sa + C::E_BYTES + C::G0_BYTES + ks * 2 * (C::N1 / 8) * 128;
            tc::mma_i8(tmem, da, tc::desc(sb0, (C::N0 / 8) * 128, 128), id0, accum);
            tc::mma_i8(tmem + C::TBASE1, da, tc::desc(sb1, (C::N1 / 8) * 128, 128), id1, accum);
          }
        }
        tc::commit(&dempty[s]);          // stage reusable once these MMAs have consumed it
        if (c == nstages - 1) tc::commit(done);
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- X loader (bulk copies, lane 0)
    const bool contiguous = ldx == n;
    const uint32_t row_bytes = (uint32_t)(n * sizeof(TX));
    // contiguous X: stages up to STC_PF ahead are prefetched into L2 (no shared memory), so that more
    // HBM bytes are in flight per SM than the raw ring holds; the ring's bulk copies then hit L2
    auto prefetch = [&](int c) {
      const int64_t i0 = i_begin + (int64_t)c * STC_KC;
      const int rows = (int)min((int64_t)STC_KC, i_end - i0);
      tc::bulk_prefetch_l2(X + i0 * ldx, row_bytes * rows);
    };
    if (contiguous && lane == 0)
      for (int c = 1; c < STC_PF && c < nstages; ++c) prefetch(c);
    for (int c = 0; c < nstages; ++c) {
      const int s = c % F::RAW;
      if (c >= F::RAW) tc::mbar_wait(&rempty[s], (uint32_t)(((c / F::RAW) - 1) & 1));
      if (lane == 0) {
        if (contiguous && c + STC_PF < nstages) prefetch(c + STC_PF);
        const int64_t i0 = i_begin + (int64_t)c * STC_KC;
        const int rows = (int)min((int64_t)STC_KC, i_end - i0);
        TX* dst = raw_base + (size_t)s * STC_KC * n;
        tc::mbar_arrive_tx(&rfull[s], row_bytes * rows);
        if (contiguous) {
          tc::bulk_g2s(dst, X + i0 * ldx, row_bytes * rows, &rfull[s]);
        } else {
          for (int ii = 0; ii < rows; ++ii) tc::bulk_g2s(dst + (size_t)ii * n, X + (i0 + ii) * ldx, row_bytes, &rfull[s]);
        }
      }
      __syncwarp();
    }
  } else if (warp < 2 + STC_DGROUPS * STC_DWARPS) {
    // ---------------------------------------------------------------- digit planes
    const int dgrp = (warp - 2) / STC_DWARPS;            // stages c = dgrp (mod 2)
    const int dt = tid - 64 - dgrp * 32 * STC_DWARPS;
    const int j = dt % STC_N, kg = dt / STC_N;           // fixed task: column j, rows kg*16 .. +15
    ColParam cp{};
    if (nstages > 0) {                                   // column scales from the first stage (both groups)
      tc::mbar_wait(&rfull[0], 0u);
      const int rows0 = (int)min((int64_t)STC_KC, i_end - i_begin);
      const TX* raw = raw_base;
      for (int u = tid - 64; u < rows0 * n; u += 32 * STC_DGROUPS * STC_DWARPS) atomicMax(&col_max[u % n], hi_abs(raw[u]));
      tc::named_bar(1, 32 * STC_DGROUPS * STC_DWARPS);
      cp = col_param<TX>(col_max[j < n ? j : 0]);
      if (dgrp == 0 && kg == 0 && j < n) col_exp[j] = cp.e;
    }
    int dst_off[D];
#pragma unroll
    for (int t = 0; t < D; ++t)
      dst_off[t] = C::E_BYTES + C::grp(t) * C::G0_BYTES + cm_off(C::brow(t) + j, kg * 16, C::grp(t) ? C::N1 : C::N0);
    uint32_t acc_or = 0u, acc_and = 0xFFFFFFFFu, amax = 0u;   // overflow detection
    for (int c = dgrp; c < nstages; c += STC_DGROUPS) {
      const int s = c % F::DIG, sr = c % F::RAW;
      const int64_t i0 = i_begin + (int64_t)c * STC_KC;
      const int rows = (int)min((int64_t)STC_KC, i_end - i0);
      const TX* raw = raw_base + (size_t)sr * STC_KC * n;
      if (c >= F::DIG) tc::mbar_wait(&dempty[s], (uint32_t)(((c / F::DIG) - 1) & 1));
      tc::mbar_wait(&rfull[sr], (uint32_t)((c / F::RAW) & 1));
      unsigned char* st = dig_base + (size_t)s * C::DIG_STAGE;
      auto build = [&](auto full) {
        constexpr bool FULL = decltype(full)::value;
        uint32_t W[D][4];
        const TX* src = FULL ? raw + (kg * 16) * STC_N + j : raw + (kg * 16) * n + j;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t hw[4], lw[4];
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const int ii = q * 4 + kk;
            TX x;
            if constexpr (FULL) x = src[ii * STC_N];
            else x = (kg * 16 + ii < rows && j < n) ? src[ii * n] : (TX)0;
            split_words(x, cp, hw[kk], lw[kk]);
            if constexpr (sizeof(TX) == 4) { acc_or |= hw[kk]; acc_and &= hw[kk]; }
            else amax = max(amax, hi_abs(x));
          }
          uint32_t H[4], L[4];
          transpose4(hw[0], hw[1], hw[2], hw[3], H);
          transpose4(lw[0], lw[1], lw[2], lw[3], L);
          if constexpr (D == 6) {      // unsigned digits of F + 2^47
            W[0][q] = H[1]; W[1][q] = H[0];
            W[2][q] = L[3]; W[3][q] = L[2]; W[4][q] = L[1]; W[5][q] = L[0];
          } else {                     // signed digits of F + C
            W[0][q] = H[3]; W[1][q] = H[2] ^ 0x80808080u; W[2][q] = H[1] ^ 0x80808080u;
            W[3][q] = H[0] ^ 0x80808080u;
            W[4][q] = L[3] ^ 0x80808080u; W[5][q] = L[2] ^ 0x80808080u;
            W[6][q] = L[1] ^ 0x80808080u; W[7][q] = L[0] ^ 0x80808080u;
          }
        }
#pragma unroll
        for (int t = 0; t < D; ++t)
          *reinterpret_cast<uint4*>(st + dst_off[t]) = make_uint4(W[t][0], W[t][1], W[t][2], W[t][3]);
      };
      if (!(dbg & 2)) {
        if (rows == STC_KC && n == STC_N) build(std::true_type{});
        else build(std::false_type{});
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // generic smem writes -> tensor core
      __syncwarp();
      if (lane == 0) { tc::mbar_arrive(&dfull[s]); tc::mbar_arrive(&rempty[sr]); }
    }
    bool ovf;
    if constexpr (sizeof(TX) == 4) ovf = (acc_or >> 16) != 0x4338u || (acc_and >> 16) != 0x4338u;
    else ovf = amax >= cp.lim;
    if (nstages > 0 && (ovf || cp.bad)) atomicOr(overflow, 1);        // headroom exceeded / Inf / NaN
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
      if (c >= F::DIG) tc::mbar_wait(&dempty[s], (uint32_t)(((c / F::DIG) - 1) & 1));
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
    if (nstages > 0) {
      tc::mbar_wait(done, 0u);
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      int32_t bias = 0;                                  // 128 S_r (fp32 digits are of F + 2^47)
      if constexpr (F::ONES > 0) {
        uint32_t a[16];
        tc::ld16(lbase, a);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n");
        bias = 128 * (int32_t)a[0];
      }
#pragma unroll 1
      for (int c0 = 0; c0 < STC_N; c0 += 16) {
        double v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = 0.0;
#pragma unroll
        for (int t = D - 1; t >= 0; --t) {             // least significant plane first
          uint32_t a[16];
          tc::ld16(lbase + C::tcol(t) + c0, a);
          asm volatile("tcgen05.wait::ld.sync.aligned;\n");
          const double w = (double)(1ull << (8 * (D - 1 - t)));
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = fma((double)((int32_t)a[j] - (t == 0 ? bias : 0)), w, v[j]);
        }
        if (row < k) {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (c0 + j < n) Pp[(size_t)row * n + c0 + j] = ldexp(v[j], col_exp[c0 + j] - F::FB);
        }
      }
    } else if (row < k) {
      for (int j = 0; j < n; ++j) Pp[(size_t)row * n + j] = 0.0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

bool sparse_tc_applicable(int k, int n, int zeta) { return n <= STC_N && zeta >= 1 && k % zeta == 0 && k <= 4 * STC_M; }

template <typename TX>
static cudaError_t launch_stc(const TX* X, int64_t m, int n, int64_t ldx, int64_t ro, int k, int zeta, uint64_t seed,
                              int tiles_k, int splits, int64_t rps, double* part, int* overflow, cudaStream_t st,
                              const uint64_t* srht_s) {
  auto kern = sketch_sparse_tc_kernel<TX>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)StcCfg<TX>::SMEM);
  if (e != cudaSuccess) return e;
  static const int dbg = !kAblation ? 0 : getenv("RCHOLQR_STC_DEBUG") ? atoi(getenv("RCHOLQR_STC_DEBUG")) : 0;   // ablations only
  kern<<<tiles_k * splits, STC_THREADS, StcCfg<TX>::SMEM, st>>>(X, m, n, ldx, ro, k, zeta, seed, tiles_k, rps, part,
                                                                 overflow, dbg, srht_s);
  return cudaGetLastError();
}

cudaError_t launch_sparse_tc(const void* X, int dtype, int64_t m, int n, int64_t ldx, int64_t row_offset, int k,
                             int zeta, uint64_t seed, int splits, int64_t rows_per_split, double* part, int* overflow,
                             cudaStream_t st, const uint64_t* srht_s) {
  const int tiles_k = (k + STC_M - 1) / STC_M;
  if (dtype == RCHOLQR_F64)
    return launch_stc((const double*)X, m, n, ldx, row_offset, k, zeta, seed, tiles_k, splits, rows_per_split, part,
                      overflow, st, srht_s);
  return launch_stc((const float*)X, m, n, ldx, row_offset, k, zeta, seed, tiles_k, splits, rows_per_split, part,
                    overflow, st, srht_s);
}

bool sparse_tc_aligned(const void* X, int dtype, int n, int64_t ldx) {
  const size_t es = dtype == RCHOLQR_F64 ? 8 : 4;   // cp.async.bulk: 16-byte aligned addresses and sizes
  return ((uintptr_t)X % 16) == 0 && ((size_t)n * es) % 16 == 0 && ((size_t)ldx * es) % 16 == 0;
}

}  // namespace rcq
