// sketch_gtc.cu -- Gaussian sketch P = Theta X on the 5th-generation tensor core (tcgen05 kind::i8),
// exact up to a truncation far below fp64 rounding of P (Alg. 2 step 1; the
// "random projection in higher precision" of PAPER.md:83, 423).
//
// Both factors are written EXACTLY as signed base-256 digit strings (DESIGN.md "tcgen05 Gaussian
// sketch"):
//   * Theta: the normative fp32 draws z (theta.cuh, bit-identical to the oracle's) satisfy
//     |z| <= 5.65 (Box-Muller radius with 23-bit uniforms), so F_z = round(z 2^44) fits in 47 bits
//     and equals z 2^44 EXACTLY for |z| >= 2^-20 (otherwise the error is < 2^-45): 6 digits.
//   * X: F_x = round(x 2^(FB - e_j)) against a per-(CTA, column) power-of-two scale 2^e_j (first
//     stage's column maximum + 4 bits of headroom): 6 digits (fp32, FB = 47) or 8 (fp64, FB = 63).
// Signed digits come from one magic-constant DFMA: the bytes of F + C (C = 0x80 in every byte but
// the top one) are the digits + 128, i.e. XOR 0x80.
//
// Orientation: the MMA's M dimension is 128 X COLUMNS (A = one X digit plane, K = 32 X rows) and
// its N dimension stacks the 6 Theta digit planes of KT Theta rows (N = 6 KT), so the expensive
// normative Theta draws (~65 instructions each) are generated once per X-column tile and only the
// cheap X digits are re-split per Theta-row tile.  The MMA for X digit b writes TMEM columns
// [b KT, (b + 6) KT): Theta digit a lands on level L = a + b.  The LEV = DX + 5 levels occupy
// LEV * KT <= 512 columns.  Every GT_DRAIN stages (and at the end) four drain warps read the
// levels (lane = X column), combine them in fp64 (sum_L acc_L 256^(LEV-1-L) 2^(-44 + e_j - FB)),
// add them with TwoSum into the CTA's (part, partc) slab and zero TMEM -- int32 never overflows:
// per level and stage |sum| <= 6 * 32 * 2^14, and GT_DRAIN * that < 2^31.
//
// Roles (1 CTA per SM, 16 warps): warp 0 lane 0 issues tcgen05.mma; warp 1 lane 0 streams X tiles
// (one 2D TMA box of 32 rows x 128 columns per stage, zero-filled outside X); warps 2..7 generate
// Theta (Philox + Box-Muller) and its digit tiles in two groups of three warps that alternate
// stages; warps 8..15 split X into digit planes (warps 8..11 also drain TMEM).
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <type_traits>
#include "internal.cuh"
#include "tcgen05.cuh"
#include "theta.cuh"

namespace rcq {

constexpr int GT_M = 128;          // X columns per CTA (MMA M = TMEM lanes)
constexpr int GT_KC = 32;          // X rows per stage (one MMA k-step)
constexpr int GT_DZ = 6;           // Theta digits
constexpr int GT_TWARPS = 6;       // Theta warps 2..7 (two groups of three, alternating stages)
constexpr int GT_XWARPS = 8;       // X-digit warps 8..15 (8..11 also drain TMEM: one per lane quadrant)
constexpr int GT_THREADS = 32 * (2 + GT_TWARPS + GT_XWARPS);
constexpr int GT_DRAIN = 512;      // stages between exact TMEM drains (even: group 0 drains)
constexpr int GT_BSBO = 144;       // 8-row group stride of the Theta digit stack (padded: STS.32 conflicts <= 2)
constexpr int GT_RAWLD = 128;      // raw X stage row stride (elements)
static_assert(GT_DRAIN * 6 * GT_KC * 16384.0 < 2147483648.0, "int32 level accumulators must not overflow");
static_assert(32 * GT_XWARPS == 2 * 128, "one X task (column, 16-row group) per X thread");

template <typename TX> struct GtFmt;
template <> struct GtFmt<float> {
  static constexpr int DX = 6, FB = 47, KT = 40, DIG = 4, RAW = 4;
};
template <> struct GtFmt<double> {
  static constexpr int DX = 8, FB = 63, KT = 32, DIG = 3, RAW = 3;
};

template <typename TX, int KT_ = GtFmt<TX>::KT>
struct GtCfg {
  using Fm = GtFmt<TX>;
  static constexpr int DX = Fm::DX, KT = KT_;
  static constexpr int NB = GT_DZ * KT;                               // stacked Theta digit planes (MMA N)
  static constexpr int LEV = DX + GT_DZ - 1;                          // digit-product levels
  static constexpr int A_TILE = GT_M * GT_KC;                         // one X digit plane (128 x 32 B)
  static constexpr int B_LBO = (NB / 8) * GT_BSBO;                    // stride of the two 16-byte K chunks
  static constexpr int B_BYTES = 2 * B_LBO;
  static constexpr int DIG_STAGE = DX * A_TILE + B_BYTES;
  static constexpr int RAW_STAGE = GT_KC * GT_RAWLD * (int)sizeof(TX);
  static constexpr int TASKS_Z = (KT / 4) * (GT_KC / 4);              // Theta tasks per stage (quad x 4 rows)
  static constexpr size_t SMEM = (size_t)Fm::DIG * DIG_STAGE + (size_t)Fm::RAW * RAW_STAGE + 2048;   // + barriers, scales
  static_assert(KT % 8 == 0, "TMEM / core-matrix shape");
};

// offset of Theta-digit byte (row R of the stack, k) in the padded B tile
template <typename TX, int KT_ = GtFmt<TX>::KT>
__device__ __forceinline__ int b_off(int R, int k) {
  return (k >> 4) * GtCfg<TX, KT_>::B_LBO + (R >> 3) * GT_BSBO + (R & 7) * 16 + (k & 15);
}

struct GtCol {
  double s;        // fp32: 2^(175 - e) applied to x 2^-128; fp64: 2^(31 - e)
  uint32_t lim;    // |x| high bits must stay below (bits of 2^e)
  int e;
  bool bad;
};

__device__ __forceinline__ uint32_t gt_habs(float x) { return __float_as_uint(x) & 0x7FFFFFFFu; }
__device__ __forceinline__ uint32_t gt_habs(double x) { return (uint32_t)__double2hiint(x) & 0x7FFFFFFFu; }

template <typename TX>
__device__ __forceinline__ GtCol gt_col(uint32_t maxbits) {
  GtCol p{};
  int emax;
  if constexpr (sizeof(TX) == 4) {
    emax = maxbits == 0u ? -44 : (maxbits < 0x00800000u ? -126 : (int)(maxbits >> 23) - 126);
    p.e = emax + 4;
    const int be = p.e + 127;
    p.lim = be >= 255 ? 0x7F800000u : (be <= 0 ? 0u : (uint32_t)be << 23);
    p.s = ldexp(1.0, 128 + GtFmt<float>::FB - p.e);
    p.bad = p.e < -70;
  } else {
    emax = maxbits == 0u ? -44 : (maxbits < 0x00100000u ? -1022 : (int)(maxbits >> 20) - 1022);
    p.e = emax + 4;
    const int be = p.e + 1023;
    p.lim = be >= 2047 ? 0x7FF00000u : (be <= 0 ? 0u : (uint32_t)be << 20);
    p.s = ldexp(1.0, 31 - p.e);
    p.bad = p.e < -900 || p.e > 900;
  }
  return p;
}

// (hi, lo) words of F + C for an fp32 value (x 2^-128 built from the bits, one RN DFMA).
__device__ __forceinline__ void gt_split(float x, double s, uint32_t& hi, uint32_t& lo) {
  const uint32_t u = __float_as_uint(x);
  const uint32_t h = ((uint32_t)((int32_t)u >> 3) & 0x8FFFFFFFu) | 0x30000000u;
  const double y = __hiloint2double((int)h, (int)(u << 29));
  const double t = fma(y, s, kMagic + (double)0x8080808080ull);
  hi = (uint32_t)__double2hiint(t);
  lo = (uint32_t)__double2loint(t);
}
// fp64 value: H = floor(x s) + C_hi, L = floor(frac 2^32) + C_lo, carry of L into H.
__device__ __forceinline__ void gt_split(double x, double s, uint32_t& hi, uint32_t& lo) {
  const double t1 = __fma_rd(x, s, kMagic + (double)0x808080u);
  const double H = t1 - (kMagic + (double)0x808080u);
  const double r = fma(x, s, -H);
  const double t2 = __fma_rd(r, 4294967296.0, kMagic + (double)0x80808080u);
  lo = (uint32_t)__double2loint(t2);
  hi = (uint32_t)__double2loint(t1) + ((uint32_t)__double2hiint(t2) & 1u);
}

// Digit words (a = 0 most significant) of four values whose (hi, lo) words are given: D = 6 uses
// hi bytes 1,0 and lo bytes 3..0; D = 8 uses hi bytes 3..0 and lo bytes 3..0; XOR 0x80 except d0.
template <int D>
__device__ __forceinline__ void gt_digits(const uint32_t (&hw)[4], const uint32_t (&lw)[4], uint32_t (&W)[D]) {
  uint32_t H[4], L[4];
  transpose4(hw[0], hw[1], hw[2], hw[3], H);
  transpose4(lw[0], lw[1], lw[2], lw[3], L);
  if constexpr (D == 6) {
    W[0] = H[1]; W[1] = H[0] ^ 0x80808080u;
    W[2] = L[3] ^ 0x80808080u; W[3] = L[2] ^ 0x80808080u; W[4] = L[1] ^ 0x80808080u; W[5] = L[0] ^ 0x80808080u;
  } else {
    W[0] = H[3]; W[1] = H[2] ^ 0x80808080u; W[2] = H[1] ^ 0x80808080u; W[3] = H[0] ^ 0x80808080u;
    W[4] = L[3] ^ 0x80808080u; W[5] = L[2] ^ 0x80808080u; W[6] = L[1] ^ 0x80808080u; W[7] = L[0] ^ 0x80808080u;
  }
}

template <typename TX>
__global__ void __launch_bounds__(GT_THREADS, 1)
sketch_gauss_tc_kernel(const __grid_constant__ CUtensorMap xmap, int64_t m, int n, int64_t row_offset, int k,
                       uint64_t seed, int tiles_k, int tiles_n, int64_t rows_per_split, double* __restrict__ part,
                       double* __restrict__ partc, int* overflow, int dbg_in) {
  const int dbg = kAblation ? dbg_in : 0;   // ablation switches (see internal.cuh)
  using C = GtCfg<TX>;
  static_assert(C::NB <= 256 && C::NB % 16 == 0 && C::LEV * C::KT <= 512, "MMA / TMEM shape");
  static_assert(C::TASKS_Z <= 32 * GT_TWARPS / 2, "one Theta task per group thread");
  using F = GtFmt<TX>;
  constexpr int DX = C::DX, KT = C::KT, LEV = C::LEV;
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* dig_base = sm;
  TX* raw_base = reinterpret_cast<TX*>(sm + (size_t)F::DIG * C::DIG_STAGE);
  uint64_t* dfull = reinterpret_cast<uint64_t*>(sm + (size_t)F::DIG * C::DIG_STAGE + (size_t)F::RAW * C::RAW_STAGE);
  uint64_t* dempty = dfull + F::DIG;
  uint64_t* rfull = dempty + F::DIG;
  uint64_t* rempty = rfull + F::RAW;
  uint64_t* drainbar = rempty + F::RAW;     // MMAs of a drain window complete (tcgen05.commit)
  uint64_t* drained = drainbar + 1;         // drain warps done reading / zeroing TMEM
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(drained + 1);
  uint32_t* col_max = tmem_slot + 1;                                  // [GT_M]
  int* col_exp = reinterpret_cast<int*>(col_max + GT_M);             // [GT_M]

  const int tiles = tiles_k * tiles_n;
  const int tile = blockIdx.x % tiles, split = blockIdx.x / tiles;
  const int tk = tile % tiles_k, tn = tile / tiles_k;
  const int r0 = tk * KT, n0 = tn * GT_M;
  const int ncols = min(GT_M, n - n0), nrows = min(KT, k - r0);
  const int64_t i_begin = (int64_t)split * rows_per_split;
  const int64_t i_end = min(m, i_begin + rows_per_split);
  const int nstages = i_end > i_begin ? (int)((i_end - i_begin + GT_KC - 1) / GT_KC) : 0;
  const int ndrains = (nstages + GT_DRAIN - 1) / GT_DRAIN;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    for (int s = 0; s < F::DIG; ++s) {
      tc::mbar_init(&dfull[s], GT_TWARPS / 2 + GT_XWARPS);   // the Theta group owning the stage + X warps
      tc::mbar_init(&dempty[s], 1);
    }
    for (int s = 0; s < F::RAW; ++s) { tc::mbar_init(&rfull[s], 1); tc::mbar_init(&rempty[s], GT_XWARPS); }
    tc::mbar_init(drainbar, 1);
    tc::mbar_init(drained, 4);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (tid < GT_M) { col_max[tid] = 0u; col_exp[tid] = 0; }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(tc::smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = *tmem_slot;
  if (warp < 4) {                        // zero the level accumulators (lane quadrant = warp)
    const uint32_t lb = tmem + ((uint32_t)(warp * 32) << 16);
    for (int c8 = 0; c8 < LEV * KT / 8; ++c8) tc::st8_zero(lb + c8 * 8);
    tc::wait_st();
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");

  if (warp == 0) {
    // ---------------------------------------------------------------- MMA issuer (lane 0)
    constexpr uint32_t idesc = tc::idesc_i8(GT_M, C::NB, true, true);
    for (int c = 0; c < nstages; ++c) {
      const int s = c % F::DIG;
      if (c > 0 && c % GT_DRAIN == 0) tc::mbar_wait(drained, (uint32_t)((c / GT_DRAIN - 1) & 1));
      tc::mbar_wait(&dfull[s], (uint32_t)((c / F::DIG) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      if (lane == 0) {
        const uint32_t sa = tc::smem_u32(dig_base + (size_t)s * C::DIG_STAGE);
        const uint64_t db = tc::desc(sa + DX * C::A_TILE, C::B_LBO, GT_BSBO);
        if (!(dbg & 1)) {
#pragma unroll
          for (int b = 0; b < DX; ++b)
            tc::mma_i8(tmem + b * KT, tc::desc(sa + b * C::A_TILE, (GT_M / 8) * 128, 128), db, idesc, 1u);
        }
        tc::commit(&dempty[s]);
        if ((c + 1) % GT_DRAIN == 0 || c == nstages - 1) tc::commit(drainbar);
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- X loader (lane 0): one 2D TMA box
    // (GT_KC rows x 128 columns, zero-filled outside X) per stage
    if (lane == 0) asm volatile("prefetch.tensormap [%0];\n" ::"l"(&xmap) : "memory");
    for (int c = 0; c < nstages; ++c) {
      const int s = c % F::RAW;
      if (c >= F::RAW) tc::mbar_wait(&rempty[s], (uint32_t)(((c / F::RAW) - 1) & 1));
      if (lane == 0) {
        if (dbg & 8) tc::mbar_arrive(&rfull[s]);
        else {
          tc::mbar_arrive_tx(&rfull[s], (uint32_t)C::RAW_STAGE);
          tc::tma_load_2d(raw_base + (size_t)s * GT_KC * GT_RAWLD, &xmap, n0, (int)(i_begin + (int64_t)c * GT_KC),
                          &rfull[s]);
        }
      }
      __syncwarp();
    }
  } else if (warp < 2 + GT_TWARPS) {
    // ---------------------------------------------------------------- Theta digits
    const int tw = warp - 2, grp = tw / (GT_TWARPS / 2);       // group grp takes stages c = grp (mod 2)
    const int t = (tw % (GT_TWARPS / 2)) * 32 + lane;          // task: Theta quad q, X-row quad kq
    const bool active = t < C::TASKS_Z;
    const int q = t % (KT / 4), kq = t / (KT / 4);
    const uint32_t qg = (uint32_t)((r0 >> 2) + q);
    int boff[4];
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) boff[rr] = b_off<TX>(4 * q + rr, 4 * kq);
    for (int c = grp; c < nstages; c += 2) {
      const int s = c % F::DIG;
      uint32_t W[4][GT_DZ];
      const bool act = active && !(dbg & 4);
      if (act) {
        const uint64_t gi = (uint64_t)(row_offset + i_begin + (int64_t)c * GT_KC + 4 * kq);
        float z[4][4];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const float4 g = gauss4_x2(seed, gi + kk, qg);
          z[kk][0] = g.x; z[kk][1] = g.y; z[kk][2] = g.z; z[kk][3] = g.w;
        }
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
          uint32_t hw[4], lw[4];
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) gt_split(z[kk][rr], 0x1p172, hw[kk], lw[kk]);   // F_z = round(z 2^44)
          gt_digits<GT_DZ>(hw, lw, W[rr]);
        }
      }
      if (c >= F::DIG) tc::mbar_wait(&dempty[s], (uint32_t)(((c / F::DIG) - 1) & 1));
      if (act) {
        unsigned char* st = dig_base + (size_t)s * C::DIG_STAGE + DX * C::A_TILE;
#pragma unroll
        for (int rr = 0; rr < 4; ++rr)
#pragma unroll
          for (int a = 0; a < GT_DZ; ++a)
            *reinterpret_cast<uint32_t*>(st + boff[rr] + (a * KT >> 3) * GT_BSBO) = W[rr][a];
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&dfull[s]);
    }
  } else {
    // ---------------------------------------------------------------- X digit planes (A operand)
    const int xt = tid - 32 * (2 + GT_TWARPS);
    const int j = xt & (GT_M - 1), kg = xt >> 7;               // column j, rows kg*16 .. +15
    const bool drainer = warp < 2 + GT_TWARPS + 4;
    const int dq = warp & 3;                                   // TMEM lane quadrant of a drain warp
    auto drain = [&](int d) {
      tc::mbar_wait(drainbar, (uint32_t)(d & 1));
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      const int jj = dq * 32 + lane;                           // X column of this TMEM lane
      const uint32_t lb = tmem + ((uint32_t)(dq * 32) << 16);
      double* Ps = part + (size_t)split * (size_t)k * n;
      double* Pc = partc + (size_t)split * (size_t)k * n;
      const int ej = col_exp[jj];
#pragma unroll 1
      for (int r8 = 0; r8 < KT / 8; ++r8) {
        double v[8];
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) v[rr] = 0.0;
#pragma unroll
        for (int L = LEV - 1; L >= 0; --L) {
          uint32_t a8[8];
          tc::ld8(lb + L * KT + r8 * 8, a8);
          tc::wait_ld();
          const double w = ldexp(1.0, 8 * (LEV - 1 - L));
#pragma unroll
          for (int rr = 0; rr < 8; ++rr) v[rr] = fma((double)(int32_t)a8[rr], w, v[rr]);
        }
        if (jj < ncols) {
#pragma unroll
          for (int rr = 0; rr < 8; ++rr) {
            const int r = r8 * 8 + rr;
            if (r < nrows) {
              const double val = ldexp(v[rr], ej - 44 - F::FB);
              const size_t o = (size_t)(r0 + r) * n + n0 + jj;
              if (d == 0) { Ps[o] = val; Pc[o] = 0.0; }
              else {                                   // TwoSum into the running (sum, compensation)
                const double a0 = Ps[o], sum = a0 + val, bb = sum - a0;
                Pc[o] += (a0 - (sum - bb)) + (val - bb);
                Ps[o] = sum;
              }
            }
          }
        }
      }
      if (d + 1 < ndrains) {
        for (int c8 = 0; c8 < LEV * KT / 8; ++c8) tc::st8_zero(lb + c8 * 8);
        tc::wait_st();
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n");
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(drained);
    };
    GtCol cp{};
    if (nstages > 0) {
      tc::mbar_wait(&rfull[0], 0u);
      const int rows0 = (int)min((int64_t)GT_KC, i_end - i_begin);
      if (kg == 0) {
        uint32_t mx = 0u;
        for (int ii = 0; ii < rows0; ++ii) mx = max(mx, gt_habs(raw_base[ii * GT_RAWLD + j]));
        col_max[j] = j < ncols ? mx : 0u;
      }
      tc::named_bar(1, 32 * GT_XWARPS);
      cp = gt_col<TX>(col_max[j]);
      if (kg == 0) col_exp[j] = cp.e;
    }
    uint32_t amax = 0u;
    for (int c = 0; c < nstages; ++c) {
      const int s = c % F::DIG, sr = c % F::RAW;
      const int64_t i0 = i_begin + (int64_t)c * GT_KC;
      const int rows = (int)min((int64_t)GT_KC, i_end - i0);
      const TX* raw = raw_base + (size_t)sr * GT_KC * GT_RAWLD;
      if (drainer && c > 0 && c % GT_DRAIN == 0) drain(c / GT_DRAIN - 1);
      if (c >= F::DIG) tc::mbar_wait(&dempty[s], (uint32_t)(((c / F::DIG) - 1) & 1));
      tc::mbar_wait(&rfull[sr], (uint32_t)((c / F::RAW) & 1));
      unsigned char* st = dig_base + (size_t)s * C::DIG_STAGE;
      if (j < ncols && !(dbg & 2)) {
        auto build = [&](auto full) {
          constexpr bool FULL = decltype(full)::value;
          {
            uint32_t Wd[DX][4];
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
              uint32_t hw[4], lw[4];
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) {
                const int ii = kg * 16 + qq * 4 + kk;
                TX x = raw[ii * GT_RAWLD + j];
                if constexpr (!FULL) x = ii < rows ? x : (TX)0;
                amax = max(amax, gt_habs(x));
                gt_split(x, cp.s, hw[kk], lw[kk]);
              }
              uint32_t W[DX];
              gt_digits<DX>(hw, lw, W);
#pragma unroll
              for (int b = 0; b < DX; ++b) Wd[b][qq] = W[b];
            }
#pragma unroll
            for (int b = 0; b < DX; ++b)
              *reinterpret_cast<uint4*>(st + b * C::A_TILE + cm_off(j, kg * 16, GT_M)) =
                  make_uint4(Wd[b][0], Wd[b][1], Wd[b][2], Wd[b][3]);
          }
        };
        if (rows == GT_KC) build(std::true_type{});
        else build(std::false_type{});
      } else if (c < F::DIG) {       // padding columns: zero digit rows once per slot (never rewritten)
#pragma unroll
        for (int b = 0; b < DX; ++b)
          *reinterpret_cast<uint4*>(st + b * C::A_TILE + cm_off(j, kg * 16, GT_M)) = make_uint4(0, 0, 0, 0);
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) { tc::mbar_arrive(&dfull[s]); tc::mbar_arrive(&rempty[sr]); }
    }
    if (nstages > 0 && j < ncols && (amax >= cp.lim || cp.bad)) atomicOr(overflow, 1);
    if (drainer) {
      if (ndrains > 0) drain(ndrains - 1);
      else {
        const int jj = dq * 32 + lane;
        if (jj < ncols)
          for (int r = 0; r < nrows; ++r) {
            part[(size_t)split * k * n + (size_t)(r0 + r) * n + n0 + jj] = 0.0;
            partc[(size_t)split * k * n + (size_t)(r0 + r) * n + n0 + jj] = 0.0;
          }
      }
    }
  }

  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

// =============================================================================================
// Pre-split variant (fp32/fp64 X when the digit buffer fits): X is split into its digit planes ONCE
// by xdig_split_kernel, in exactly the shared-memory tile layout of the sketch (one contiguous
// DX x 4 KB block per (split, 32-row stage, 128-column tile)), so the sketch kernel receives each
// stage with a single bulk copy and all of its producer warps generate Theta.  Column scales are
// per (split, column), from the split's first 32 rows (the same heuristic and overflow guard).
// Two differences from the in-kernel variant above: (1) only the digit-product levels L < LK are
// computed (GpLevels: X digit b multiplies a prefix of the Theta digit stack; the dropped levels are
// below the fp64 rounding of P, A17), so TMEM holds LK * KT columns; (2) fp64 tiles take
// KT = 48 Theta rows (96 Theta tasks per stage fill a 3-warp group), an N = 288 prefix being issued as
// two MMAs (N = 256 + 32).  RCHOLQR_GTP_DEBUG=1 (ablation) copies 16 B per stage instead of the digits.
constexpr int GP_TWARPS = 12;                     // Theta warps 2..13: four groups of three
constexpr int GP_THREADS = 32 * (2 + GP_TWARPS);
constexpr int GP_GROUPS = 4;
static_assert(GT_DRAIN % GP_GROUPS == 0, "drain stages belong to group 0");

// Levels the pre-split kernel keeps: L <= LK - 1.  A dropped level L >= LK holds at most 4 digit products
// of weight 256^(LEV-1-L), i.e. <= 2^-53 (fp32 X, LK = 8) / 2^-61 (fp64 X, LK = 9) of a typical
// |F_z F_x| term -- at or below the fp64 rounding of P (reading A17) -- so X digit b multiplies only
// the Theta digits a < LK - b, a PREFIX of the stacked B tile (its MMA N shrinks accordingly).
template <typename TX> struct GpLevels;
template <> struct GpLevels<float> { static constexpr int LK = 8, KT = 40; };    // 80 Theta tasks: 10 quads x 8
template <> struct GpLevels<double> { static constexpr int LK = 9, KT = 48; };   // 96 tasks fill a 3-warp group
//   (fp64 can take KT = 48 because only LK levels live in TMEM: max_b (b KT + N_b) = 432 <= 512 columns;
//    a B stack of 6 KT = 288 rows is issued as two MMAs of N = 256 and 32)
__host__ __device__ constexpr int gp_nd(int b, int lk) { return (lk - b) < GT_DZ ? (lk - b) : GT_DZ; }
__host__ __device__ constexpr int gp_n(int b, int lk, int kt) { return (gp_nd(b, lk) * kt + 15) / 16 * 16; }

template <typename TX>
struct GpCfg {
  using G = GtCfg<TX, GpLevels<TX>::KT>;
  static constexpr int A_BYTES = G::DX * 4096;                        // DX planes of 128 x 32 B
  static constexpr int DIG_STAGE = A_BYTES + G::B_BYTES;
  static constexpr int STAGES = (232448 - 2048) / DIG_STAGE < 6 ? (232448 - 2048) / DIG_STAGE : 6;
  static constexpr size_t SMEM = (size_t)STAGES * DIG_STAGE + 2048;
  static_assert(SMEM <= 232448 && STAGES >= 3, "shared memory");
};

// per (split, column): max |x| high bits over the split's first 32 rows (tile-padded columns)
template <typename TX>
__global__ void xdig_maxbits_kernel(const TX* __restrict__ X, int64_t m, int n, int64_t sr, int64_t sc,
                                    int64_t rows_per_split, int npad, uint32_t* __restrict__ maxbits) {
  // element (i, j) at X[i sr + j sc]: (ldx, 1) row-major, (1, ldx) column-major
  const int split = blockIdx.x;
  const int64_t i0 = (int64_t)split * rows_per_split;
  const int rows = (int)max((int64_t)0, min((int64_t)GT_KC, min(m, i0 + rows_per_split) - i0));
  for (int j = threadIdx.x; j < npad; j += blockDim.x) {
    uint32_t mx = 0u;
    if (j < n)
      for (int ii = 0; ii < rows; ++ii) mx = max(mx, gt_habs(X[(i0 + ii) * sr + j * sc]));
    maxbits[(size_t)split * npad + j] = mx;
  }
}

// unit u = ((split * stages + stage) * tiles_n + tn): DX digit planes of 128 columns x 32 rows
template <typename TX>
__global__ void __launch_bounds__(256)
xdig_split_kernel(const TX* __restrict__ X, int64_t m, int n, int64_t sr, int64_t sc, int64_t rows_per_split, int stages,
                  int tiles_n, int64_t units, const uint32_t* __restrict__ maxbits, unsigned char* __restrict__ dig,
                  int* overflow, double* __restrict__ cs_part) {
  constexpr int DX = GtFmt<TX>::DX;
  const int j = threadIdx.x & (GT_M - 1), kg = threadIdx.x >> 7;
  const int npad = tiles_n * GT_M;
  uint32_t amax = 0u;
  bool bad = false;
  // cs_part != null (Alg. 7, "computing this matrix along with P <- Theta X in step 1 during the
  // same pass"): the column sums of squares of X in the pass that already reads every element.  gridDim.x is a
  // multiple of tiles_n, so a block's column tile tn = blockIdx.x % tiles_n is fixed.
  double cs = 0.0;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    const int tn = (int)(u % tiles_n);
    const int64_t st_g = u / tiles_n;
    const int split = (int)(st_g / stages), stage = (int)(st_g % stages);
    const int64_t i_begin = (int64_t)split * rows_per_split, i_end = min(m, i_begin + rows_per_split);
    const int64_t i0 = i_begin + (int64_t)stage * GT_KC;
    const int col = tn * GT_M + j;
    const GtCol cp = gt_col<TX>(maxbits[(size_t)split * npad + col]);
    uint32_t Wd[DX][4];
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) {
      uint32_t hw[4], lw[4];
      // column-major X (sr == 1): the thread's 4 consecutive rows of its column are one 16 / 32-byte
      // vector when aligned (i0 is a multiple of 32 rows, so the base and sc decide)
      TX xq[4];
      const int64_t iq = i0 + kg * 16 + qq * 4;
      const bool vec = sr == 1 && col < n && iq + 4 <= i_end && ((uintptr_t)(X + iq + (int64_t)col * sc) % 16) == 0;
      if (vec) {
        if constexpr (sizeof(TX) == 4) {
          const float4 f = __ldg(reinterpret_cast<const float4*>(X + iq + (int64_t)col * sc));
          xq[0] = f.x; xq[1] = f.y; xq[2] = f.z; xq[3] = f.w;
        } else {
          const double2 f0 = __ldg(reinterpret_cast<const double2*>(X + iq + (int64_t)col * sc));
          const double2 f1 = __ldg(reinterpret_cast<const double2*>(X + iq + (int64_t)col * sc) + 1);
          xq[0] = f0.x; xq[1] = f0.y; xq[2] = f1.x; xq[3] = f1.y;
        }
      } else {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) xq[kk] = (col < n && iq + kk < i_end) ? X[(iq + kk) * sr + (int64_t)col * sc] : (TX)0;
      }
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const TX x = xq[kk];
        if (col < n) { amax = max(amax, gt_habs(x) >= cp.lim ? 0xFFFFFFFFu : 0u); bad |= cp.bad; }
        if (cs_part) cs = fma((double)x, (double)x, cs);
        gt_split(x, cp.s, hw[kk], lw[kk]);
      }
      uint32_t W[DX];
      gt_digits<DX>(hw, lw, W);
#pragma unroll
      for (int b = 0; b < DX; ++b) Wd[b][qq] = W[b];
    }
    unsigned char* blk = dig + (size_t)u * (DX * 4096);
#pragma unroll
    for (int b = 0; b < DX; ++b)
      *reinterpret_cast<uint4*>(blk + b * 4096 + cm_off(j, kg * 16, GT_M)) = make_uint4(Wd[b][0], Wd[b][1], Wd[b][2], Wd[b][3]);
  }
  if (amax || bad) atomicOr(overflow, 1);
  if (cs_part) {                                       // the two row halves of each column, fixed order
    __shared__ double csh[GT_M];
    if (kg == 1) csh[j] = cs;
    __syncthreads();
    const int col = (int)(blockIdx.x % tiles_n) * GT_M + j;
    if (kg == 0 && col < n) cs_part[(size_t)blockIdx.x * n + col] += cs + csh[j];
  }
}

template <typename TX>
__global__ void __launch_bounds__(GP_THREADS, 1)
sketch_gauss_tcp_kernel(const unsigned char* __restrict__ dig, const uint32_t* __restrict__ maxbits, int64_t m, int n,
                        int64_t row_offset, int k, uint64_t seed, int tiles_k, int tiles_n, int64_t rows_per_split,
                        int stages_per_split, double* __restrict__ part, double* __restrict__ partc, int accumulate,
                        int dbg_in) {
  const int dbg = kAblation ? dbg_in : 0;   // ablation switches (see internal.cuh)
  using C = typename GpCfg<TX>::G;
  using P = GpCfg<TX>;
  using F = GtFmt<TX>;
  constexpr int DX = C::DX, KT = C::KT, LEV = C::LEV, S = P::STAGES;
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* dfull = reinterpret_cast<uint64_t*>(sm + (size_t)S * P::DIG_STAGE);
  uint64_t* dempty = dfull + S;
  uint64_t* drainbar = dempty + S;
  uint64_t* drained = drainbar + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(drained + 1);

  const int tiles = tiles_k * tiles_n;
  const int tile = blockIdx.x % tiles, split = blockIdx.x / tiles;
  const int tk = tile % tiles_k, tn = tile / tiles_k;
  const int r0 = tk * KT, n0 = tn * GT_M;
  const int ncols = min(GT_M, n - n0), nrows = min(KT, k - r0);
  const int64_t i_begin = (int64_t)split * rows_per_split;
  const int64_t i_end = min(m, i_begin + rows_per_split);
  const int nstages = i_end > i_begin ? (int)((i_end - i_begin + GT_KC - 1) / GT_KC) : 0;
  const int ndrains = (nstages + GT_DRAIN - 1) / GT_DRAIN;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      tc::mbar_init(&dfull[s], GP_TWARPS / GP_GROUPS + 1);   // the stage's Theta group + the loader (tx)
      tc::mbar_init(&dempty[s], 1);
    }
    tc::mbar_init(drainbar, 1);
    tc::mbar_init(drained, 4);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(tc::smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = *tmem_slot;
  if (warp < 4) {
    const uint32_t lb = tmem + ((uint32_t)(warp * 32) << 16);
    for (int c8 = 0; c8 < GpLevels<TX>::LK * KT / 8; ++c8) tc::st8_zero(lb + c8 * 8);
    tc::wait_st();
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");

  if (warp == 0) {
    // ---------------------------------------------------------------- MMA issuer (lane 0)
    constexpr int LK = GpLevels<TX>::LK;
    static_assert(gp_n(0, LK, KT) == C::NB && LK > DX - 1, "level truncation shape");
    static_assert((DX - 1) * KT + gp_n(DX - 1, LK, KT) <= 512 && LK * KT <= 512, "TMEM columns");
    for (int c = 0; c < nstages; ++c) {
      const int s = c % S;
      if (c > 0 && c % GT_DRAIN == 0) tc::mbar_wait(drained, (uint32_t)((c / GT_DRAIN - 1) & 1));
      tc::mbar_wait(&dfull[s], (uint32_t)((c / S) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      if (lane == 0) {
        const uint32_t sa = tc::smem_u32(sm + (size_t)s * P::DIG_STAGE);
        const uint64_t db = tc::desc(sa + P::A_BYTES, C::B_LBO, GT_BSBO);
#pragma unroll
        for (int b = 0; b < DX; ++b) {   // X digit b x Theta digits a < LK - b (levels b .. LK - 1)
          constexpr int NMAX = 256;      // MMA N limit: a longer prefix is issued as two MMAs
          const int nb = gp_n(b, LK, KT);
          const uint64_t da = tc::desc(sa + b * 4096, (GT_M / 8) * 128, 128);
          tc::mma_i8(tmem + b * KT, da, db, tc::idesc_i8(GT_M, nb < NMAX ? nb : NMAX, true, true), 1u);
          if (nb > NMAX)
            tc::mma_i8(tmem + b * KT + NMAX, da, tc::desc(sa + P::A_BYTES + (NMAX / 8) * GT_BSBO, C::B_LBO, GT_BSBO),
                       tc::idesc_i8(GT_M, nb - NMAX, true, true), 1u);
        }
        tc::commit(&dempty[s]);
        if ((c + 1) % GT_DRAIN == 0 || c == nstages - 1) tc::commit(drainbar);
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- digit loader (lane 0)
    for (int c = 0; c < nstages; ++c) {
      const int s = c % S;
      if (c >= S) tc::mbar_wait(&dempty[s], (uint32_t)(((c / S) - 1) & 1));
      if (lane == 0) {
        const size_t u = ((size_t)split * stages_per_split + c) * tiles_n + tn;
        const uint32_t bytes = (dbg & 1) ? 16u : (uint32_t)P::A_BYTES;   // ablation: no digit traffic
        tc::mbar_arrive_tx(&dfull[s], bytes);
        tc::bulk_g2s(sm + (size_t)s * P::DIG_STAGE, dig + u * P::A_BYTES, bytes, &dfull[s]);
      }
      __syncwarp();
    }
  } else {
    // ---------------------------------------------------------------- Theta digits (+ drains: warps 2..5)
    const int tw = warp - 2, grp = tw / (GP_TWARPS / GP_GROUPS);
    const int t = (tw % (GP_TWARPS / GP_GROUPS)) * 32 + lane;
    const bool active = t < C::TASKS_Z;
    const int q = t % (KT / 4), kq = t / (KT / 4);
    const uint32_t qg = (uint32_t)((r0 >> 2) + q);
    const bool drainer = warp < 6;
    const int dq = warp & 3;
    auto drain = [&](int d) {
      tc::mbar_wait(drainbar, (uint32_t)(d & 1));
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      const int jj = dq * 32 + lane;
      const uint32_t lb = tmem + ((uint32_t)(dq * 32) << 16);
      double* Ps = part + (size_t)split * (size_t)k * n;
      double* Pc = partc + (size_t)split * (size_t)k * n;
      const int ej = gt_col<TX>(maxbits[(size_t)split * tiles_n * GT_M + n0 + jj]).e;
#pragma unroll 1
      for (int r8 = 0; r8 < KT / 8; ++r8) {
        double v[8];
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) v[rr] = 0.0;
#pragma unroll
        for (int L = GpLevels<TX>::LK - 1; L >= 0; --L) {      // levels >= LK are not computed
          uint32_t a8[8];
          tc::ld8(lb + L * KT + r8 * 8, a8);
          tc::wait_ld();
          const double w = ldexp(1.0, 8 * (LEV - 1 - L));
#pragma unroll
          for (int rr = 0; rr < 8; ++rr) v[rr] = fma((double)(int32_t)a8[rr], w, v[rr]);
        }
        if (jj < ncols) {
#pragma unroll
          for (int rr = 0; rr < 8; ++rr) {
            const int r = r8 * 8 + rr;
            if (r < nrows) {
              const double val = ldexp(v[rr], ej - 44 - F::FB);
              const size_t o = (size_t)(r0 + r) * n + n0 + jj;
              if (d == 0 && !accumulate) { Ps[o] = val; Pc[o] = 0.0; }
              else {                                   // TwoSum into the running (sum, compensation)
                const double a0 = Ps[o], sum = a0 + val, bb = sum - a0;
                Pc[o] += (a0 - (sum - bb)) + (val - bb);
                Ps[o] = sum;
              }
            }
          }
        }
      }
      if (d + 1 < ndrains) {
        for (int c8 = 0; c8 < GpLevels<TX>::LK * KT / 8; ++c8) tc::st8_zero(lb + c8 * 8);
        tc::wait_st();
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n");
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(drained);
    };
    int boff[4];
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) boff[rr] = b_off<TX, KT>(4 * q + rr, 4 * kq);
    int next_drain = 1;                                   // drain d is due before stage (d + 1) * GT_DRAIN
    for (int c = grp; c < nstages; c += GP_GROUPS) {
      const int s = c % S;
      if (drainer)
        while (next_drain * GT_DRAIN <= c) { drain(next_drain - 1); ++next_drain; }
      uint32_t W[4][GT_DZ];
      if (active) {
        const uint64_t gi = (uint64_t)(row_offset + i_begin + (int64_t)c * GT_KC + 4 * kq);
        float z[4][4];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const float4 g = gauss4_x2(seed, gi + kk, qg);
          z[kk][0] = g.x; z[kk][1] = g.y; z[kk][2] = g.z; z[kk][3] = g.w;
        }
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
          uint32_t hw[4], lw[4];
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) gt_split(z[kk][rr], 0x1p172, hw[kk], lw[kk]);
          gt_digits<GT_DZ>(hw, lw, W[rr]);
        }
      }
      if (c >= S) tc::mbar_wait(&dempty[s], (uint32_t)(((c / S) - 1) & 1));
      if (active) {
        unsigned char* st = sm + (size_t)s * P::DIG_STAGE + P::A_BYTES;
#pragma unroll
        for (int rr = 0; rr < 4; ++rr)
#pragma unroll
          for (int a = 0; a < GT_DZ; ++a)
            *reinterpret_cast<uint32_t*>(st + boff[rr] + (a * KT >> 3) * GT_BSBO) = W[rr][a];
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&dfull[s]);
    }
    if (drainer) {
      while (next_drain <= ndrains) { drain(next_drain - 1); ++next_drain; }
      if (ndrains == 0 && !accumulate) {
        const int jj = dq * 32 + lane;
        if (jj < ncols)
          for (int r = 0; r < nrows; ++r) {
            part[(size_t)split * k * n + (size_t)(r0 + r) * n + n0 + jj] = 0.0;
            partc[(size_t)split * k * n + (size_t)(r0 + r) * n + n0 + jj] = 0.0;
          }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

// bytes of the pre-split digit workspace (digit blocks + per-(split, column) maxima)
size_t gauss_tcp_workspace(int64_t m, int n, int dtype, int splits) {
  const int dx = dtype == RCHOLQR_F64 ? GtFmt<double>::DX : GtFmt<float>::DX;
  const int tiles_n = (n + GT_M - 1) / GT_M;
  const int64_t per = (m + splits - 1) / splits;
  const int64_t rps = std::max<int64_t>(GT_KC, ((per + GT_KC - 1) / GT_KC) * GT_KC);
  const int64_t stages = rps / GT_KC;
  return (size_t)splits * stages * tiles_n * dx * 4096 + (size_t)splits * tiles_n * GT_M * 4;
}

// column j of out = sum over the kXdigSplitBlocks partial rows: one warp per column, lanes take rows lane, lane + 32,
// ... in order, then a fixed shuffle tree (deterministic; the 1184-long column sums of a 256-thread reduce were
// ~0.1 ms of serial adds)
__global__ void __launch_bounds__(32) colsum_reduce_kernel(const double* __restrict__ part, int rows, int n,
                                                             double* __restrict__ out, int* status) {
  const int j = blockIdx.x, lane = threadIdx.x;
  double s = 0.0;
  for (int r = lane; r < rows; r += 32) s += part[(size_t)r * n + j];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    out[j] = s;
    if (!isfinite(s)) atomicOr(status, kStNonfinite);
  }
}
cudaError_t launch_colsum_reduce(const double* part, int rows, int n, double* out, int* status, cudaStream_t st) {
  colsum_reduce_kernel<<<n, 32, 0, st>>>(part, rows, n, out, status);
  return cudaGetLastError();
}

// split grid: at most kXdigSplitBlocks CTAs, a multiple of tiles_n (each CTA keeps one column tile)
static int xdig_split_grid(int64_t units, int tiles_n) {
  const int64_t g = std::min<int64_t>(units, kXdigSplitBlocks);
  return (int)std::max<int64_t>(tiles_n, g / tiles_n * tiles_n);
}

template <typename TX>
static cudaError_t launch_gtcp(const TX* X, int64_t m, int n, int64_t ldx, int64_t ro, int k, uint64_t seed,
                               int tiles_k, int tiles_n, int splits, int64_t rps, double* part, double* partc,
                               int* overflow, void* ws, int accumulate, double* cs_part, cudaStream_t st, bool colmajor) {
  constexpr int DX = GtFmt<TX>::DX;
  const int64_t sr = colmajor ? 1 : ldx, sc = colmajor ? ldx : 1;   // element (i, j) at X[i sr + j sc]
  const int stages = (int)(rps / GT_KC);
  const int64_t units = (int64_t)splits * stages * tiles_n;
  unsigned char* dig = reinterpret_cast<unsigned char*>(ws);
  uint32_t* maxbits = reinterpret_cast<uint32_t*>(dig + (size_t)units * DX * 4096);
  xdig_maxbits_kernel<TX><<<splits, 256, 0, st>>>(X, m, n, sr, sc, rps, tiles_n * GT_M, maxbits);
  xdig_split_kernel<TX><<<xdig_split_grid(units, tiles_n), 256, 0, st>>>(X, m, n, sr, sc, rps, stages, tiles_n, units,
                                                                          maxbits, dig, overflow, cs_part);
  auto kern = sketch_gauss_tcp_kernel<TX>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GpCfg<TX>::SMEM);
  if (e != cudaSuccess) return e;
  static const int dbg = !kAblation ? 0 : getenv("RCHOLQR_GTP_DEBUG") ? atoi(getenv("RCHOLQR_GTP_DEBUG")) : 0;   // ablations only
  kern<<<tiles_k * tiles_n * splits, GP_THREADS, GpCfg<TX>::SMEM, st>>>(dig, maxbits, m, n, ro, k, seed, tiles_k,
                                                                         tiles_n, rps, stages, part, partc, accumulate,
                                                                         dbg);
  return cudaGetLastError();
}

// Rows are processed in chunks whose digit workspace fits ws_bytes; every chunk after the first adds
// into the per-split partials (TwoSum), so the result is the sketch of all m rows.
cudaError_t launch_gauss_tcp(const void* X, int dtype, int64_t m, int n, int64_t ldx, int64_t row_offset, int k,
                             uint64_t seed, int tiles_k, int tiles_n, int splits, double* part, double* partc,
                             int* overflow, void* ws, size_t ws_bytes, cudaStream_t st, double* cs_part, bool colmajor) {
  const size_t es = dtype == RCHOLQR_F64 ? 8 : 4;
  int64_t chunk = m;
  while (chunk > GT_KC && gauss_tcp_workspace(chunk, n, dtype, splits) > ws_bytes) chunk = (chunk + 1) / 2;
  if (gauss_tcp_workspace(chunk, n, dtype, splits) > ws_bytes) return cudaErrorNotSupported;
  if (cs_part) {                                       // every chunk's split kernel adds into these partials
    cudaError_t e = cudaMemsetAsync(cs_part, 0, sizeof(double) * kXdigSplitBlocks * n, st);
    if (e != cudaSuccess) return e;
  }
  for (int64_t c0 = 0; c0 < m; c0 += chunk) {
    const int64_t mc = std::min(chunk, m - c0);
    const int64_t per = (mc + splits - 1) / splits;
    const int64_t rps = std::max<int64_t>(GT_KC, ((per + GT_KC - 1) / GT_KC) * GT_KC);
    const char* Xc = reinterpret_cast<const char*>(X) + (size_t)c0 * (colmajor ? 1 : ldx) * es;   // row c0
    cudaError_t e = dtype == RCHOLQR_F64
                        ? launch_gtcp((const double*)Xc, mc, n, ldx, row_offset + c0, k, seed, tiles_k, tiles_n, splits,
                                      rps, part, partc, overflow, ws, c0 > 0, cs_part, st, colmajor)
                        : launch_gtcp((const float*)Xc, mc, n, ldx, row_offset + c0, k, seed, tiles_k, tiles_n, splits,
                                      rps, part, partc, overflow, ws, c0 > 0, cs_part, st, colmajor);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// chunk rows the plan sizes its workspace for (at most kXdigCapBytes)
size_t gauss_tcp_chunk_workspace(int64_t m, int n, int dtype, int splits) {
  size_t cap = kXdigCapBytes;
  if (const char* e = getenv("RCHOLQR_XDIG_CAP_MB")) cap = (size_t)atoll(e) << 20;   // tests: force chunking
  int64_t chunk = m;
  while (chunk > GT_KC && gauss_tcp_workspace(chunk, n, dtype, splits) > cap) chunk = (chunk + 1) / 2;
  return gauss_tcp_workspace(chunk, n, dtype, splits);
}

int gauss_tc_kt(int dtype) { return dtype == RCHOLQR_F64 ? GpLevels<double>::KT : GpLevels<float>::KT; }

bool gauss_tc_aligned(const void* X, int dtype, int n, int64_t ldx) {
  // TMA: 16-byte aligned base and row pitch
  const size_t es = dtype == RCHOLQR_F64 ? 8 : 4;
  (void)n;
  return ((uintptr_t)X % 16) == 0 && ((size_t)ldx * es) % 16 == 0;
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

template <typename TX>
static cudaError_t launch_gtc(const TX* X, int64_t m, int n, int64_t ldx, int64_t ro, int k, uint64_t seed,
                              int tiles_k, int tiles_n, int splits, int64_t rps, double* part, double* partc,
                              int* overflow, cudaStream_t st) {
  tiles_k = (k + GtFmt<TX>::KT - 1) / GtFmt<TX>::KT;   // this variant's own Theta tile (the plan's is the pre-split's)
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return cudaErrorNotSupported;
  CUtensorMap map;
  const cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)m};
  const cuuint64_t strides[1] = {(cuuint64_t)ldx * sizeof(TX)};
  const cuuint32_t box[2] = {GT_M, GT_KC}, estr[2] = {1, 1};
  if (enc(&map, sizeof(TX) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
          const_cast<TX*>(X), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  auto kern = sketch_gauss_tc_kernel<TX>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GtCfg<TX>::SMEM);
  if (e != cudaSuccess) return e;
  static const int dbg = !kAblation ? 0 : getenv("RCHOLQR_GTC_DEBUG") ? atoi(getenv("RCHOLQR_GTC_DEBUG")) : 0;   // ablations only
  kern<<<tiles_k * tiles_n * splits, GT_THREADS, GtCfg<TX>::SMEM, st>>>(map, m, n, ro, k, seed, tiles_k, tiles_n, rps,
                                                                         part, partc, overflow, dbg);
  return cudaGetLastError();
}

cudaError_t launch_gauss_tc(const void* X, int dtype, int64_t m, int n, int64_t ldx, int64_t row_offset, int k,
                            uint64_t seed, int tiles_k, int tiles_n, int splits, int64_t rows_per_split,
                            double* part, double* partc, int* overflow, cudaStream_t st) {
  if (m > INT32_MAX) return cudaErrorNotSupported;   // TMA coordinates are int32
  if (dtype == RCHOLQR_F64)
    return launch_gtc((const double*)X, m, n, ldx, row_offset, k, seed, tiles_k, tiles_n, splits, rows_per_split,
                      part, partc, overflow, st);
  return launch_gtc((const float*)X, m, n, ldx, row_offset, k, seed, tiles_k, tiles_n, splits, rows_per_split, part,
                    partc, overflow, st);
}

}  // namespace rcq
