// solve_tc.cu -- tall solve Q = X R^{-1} (Alg. 2 step 3) for fp32 X with n <= 128 on the
// 5th-generation tensor core (tcgen05 kind::i8), the B200 form of the paper's dominant step
// ("mainly determined by the computation of X R^{-1} ... m n^2 flops").
//
// For fp32 X the solve is computed as Q = X W with W = fl64(R^{-1}) (tri_inverse_kernel, fp64) and
// the product evaluated EXACTLY in integer digits (reading A16: the forward error of
// X W vs row-wise substitution is <= kappa u_64 << u_32, far below the single rounding of Q to
// fp32 that both carry):
//   * X row i:    F_x = round(x 2^(46 - e_i)), e_i = exponent bound of the row's max |x|,
//                 6 signed base-256 digits (d_0 most significant);
//   * W column j: F_w = round(w 2^(54 - e_j)), 7 signed digits (prepared once per solve);
//   * Q_ij = 2^(e_i - 46 + e_j - 54) sum_L acc_L 256^(11 - L), acc_L = sum_{a + b = L} xd_a . wd_b,
//     levels L <= 6 kept.
// Accuracy: the solve amplifies a relative perturbation of x_i or of W by up to kappa(R) sqrt(n),
// so both are carried to ~2^-46 of their row / column scale and the dropped levels are < 2^-56
// of |x_i| |w_j| n: all far below the 2^-24 of the final rounding of Q to fp32 for kappa <= 1e6.
// Each int8 MMA has M = 128 X rows and N = (7 - a) * 32 stacked W digit planes of one 32-column
// group, writing levels a..6 at once into int32 TMEM (accumulate flag off for the first MMA of a
// tile initialises every level).  TMEM holds two 224-column level buffers, so the drain warps
// (fp64 combine, fp32 Q stores) of one group overlap the MMAs of the next.
//
// W = R^{-1} is upper triangular, so column group g only needs rows l < 32 (g + 1): its digit
// tile and its MMAs stop there (K_g = 32 (g + 1)).
//
// Roles (persistent CTAs; 20 warps for n <= 64, 18 above): warp 0 lane 0 issues tcgen05.mma; warp 1
// lane 0 stages the W digits (cp.async.bulk) and, for n <= 64, the X tiles (one 2D TMA box of 128
// rows x K+4 columns per tile, two-stage ring); the next RW = 8 warps drain TMEM -- two sets (set d
// drains level buffer d, one lane quadrant per warp, 32 columns) -- and write Q
// through shared memory with TMA stores; the last warps (10 for n <= 64, 8 above) split X into digit planes (for 64 < n <= 128 they read X with plain loads into registers
// and write the digits as two K-halves into a ring of three half slots: there is no room for a raw
// ring or a second full digit stage).
#include <cuda_runtime.h>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <type_traits>
#include "internal.cuh"
#include "tcgen05.cuh"

namespace rcq {

constexpr int QT_M = 128;       // X rows per tile (MMA M = TMEM lanes)
constexpr int QT_G = 32;        // output columns per TMEM level group
constexpr int QT_DA = 6;        // X digits
constexpr int QT_DB = 7;        // W digits
constexpr int QT_LEV = 7;       // levels kept (a + b <= 6)
constexpr int QT_NB = QT_DB * QT_G;             // stacked W digit rows of one group (224)
constexpr int QT_DWARPS = 8;    // digit warps of the K-half producers (64 < n <= 128)
constexpr int QT_RWARPS = 8;    // drain warps 2..9: two sets of four (one per TMEM level buffer)
constexpr int QT_KMAX_ALL = 128;
constexpr int QT_PF = 4;        // X tiles prefetched into L2 ahead of the raw ring (n <= 64)
static_assert(2 * QT_LEV * QT_G <= 512, "two TMEM level buffers");

// byte offset of column group g's W digit tile (triangular: K_h = 32 (h + 1) rows of W per group)
__host__ __device__ constexpr int qt_woff(int g) { return QT_NB * 32 * g * (g + 1) / 2; }

#ifndef RCQ_SOLVE_RW
#define RCQ_SOLVE_RW 8
#endif
#ifndef RCQ_SOLVE_DW
#define RCQ_SOLVE_DW 10
#endif
// kernel-experiment switches (ablation library only; the defaults are the production kernel)
#ifndef RCQ_SOLVE_F2F
#define RCQ_SOLVE_F2F 1      // X -> double by F2F.F64.F32 (0: three integer-pipe instructions)
#endif
#ifndef RCQ_SOLVE_ROT
#define RCQ_SOLVE_ROT 1      // rotate the first digit warp with the tile
#endif
template <int KMAX>
struct QCfg {
  static constexpr bool TMA_RAW = KMAX <= 64;     // raw X ring via TMA (else plain loads)
  static constexpr int DIG = KMAX <= 64 ? 2 : 1;
  static constexpr int RAW = TMA_RAW ? 2 : 0;
  static constexpr int A_TILE = QT_M * KMAX;      // one X digit plane (128 x KMAX B)
  static constexpr int RS = KMAX + 4;             // raw X row pitch (floats): K + 4 -> conflict-free LDS.128
  static constexpr int RAW_STAGE = QT_M * RS * 4;
  static constexpr int W_BYTES = qt_woff(KMAX / 32);
  // 64 < n <= 128: the X digits of a tile are kept as two K-halves (columns 0..63, 64..127) in a
  // ring of three half slots, so the first half of tile t + 1 is written while the MMAs of tile t
  // still read both halves of tile t; Q is stored from registers (no staging tile: no room)
  static constexpr bool HALF = !TMA_RAW;
  static constexpr int NSLOT = HALF ? 3 : DIG;
  static constexpr int H_TILE = QT_M * 64;        // one digit plane of one K-half
  static constexpr int SLOT_BYTES = HALF ? QT_DA * H_TILE : QT_DA * A_TILE;
  // n <= 64: 8 drain warps (one per lane quadrant per TMEM buffer, 32 columns each) and 10 digit warps.
  // Measured splits (C4, ms): 16 drain / 6 digit 8.5 (spills at 80 registers), 8 / 6 8.1, 8 / 14 8.1
  // (spills), 8 / 10 7.6 (96 registers, no spill): the digit production is the critical path
  // (tools/trace_solve.py: ~3.2 K of a ~3.7 K-cycle tile), not the TMEM read concurrency.
  // 64 < n <= 128: 8 drain warps and 8 K-half digit producers (their row mapping assumes 8)
  static constexpr int RW = TMA_RAW ? RCQ_SOLVE_RW : QT_RWARPS;
  static constexpr int DW = TMA_RAW ? RCQ_SOLVE_DW : QT_DWARPS;
  static constexpr int THREADS = 32 * (2 + RW + DW);
  static constexpr int DCOLS = QT_G * 8 / RW;     // columns of a group per drain warp (16 or 32)
  static constexpr int QS = HALF ? QT_RWARPS * 32 * 8 * 4 : RW * 32 * DCOLS * 4;   // HALF: 32 x 8 tile per drain warp
  // row-scale ring depth (tiles): 8 for the raw-ring kernel (column-major X: the loader warp writes the scales of
  // tile t as soon as its raw stage lands, up to 5 tiles ahead of the last drain that reads the ring), else 4
  static constexpr int RXD = TMA_RAW ? 8 : 4;
  static constexpr size_t SMEM =
      (size_t)W_BYTES + (size_t)NSLOT * SLOT_BYTES + (size_t)RAW * RAW_STAGE + QS + 2048 + (size_t)RXD * QT_M * 4;
  static_assert(SMEM <= 232448, "shared memory");
};

// ---------------------------------------------------------------------------------------------
// W digit prep: column scales e_j and the signed digit planes, laid out per group g as the B
// operand tile [6 * 32 rows (row = b * 32 + jj) x K bytes], K-major SWIZZLE_NONE core matrices.
__global__ void __launch_bounds__(QT_KMAX_ALL)
solve_tc_prep_kernel(const double* __restrict__ W, int n, int kpad, int8_t* __restrict__ wdig,
                     int* __restrict__ wexp, const int* status) {
  // one CTA per column j, one thread per row l of W (the serial per-column loops of a single CTA
  // cost ~0.1 ms at n = 100: two dependent global-load chains of n steps)
  if (*status) return;
  __shared__ double wmax[QT_KMAX_ALL / 32];
  const int j = blockIdx.x, l = threadIdx.x, g = j / QT_G, jj = j % QT_G;
  const int kg = min(QT_G * (g + 1), kpad);          // rows l < kg of W (upper triangular)
  const double w = (j < n && l < n) ? W[(size_t)l * n + j] : 0.0;
  double mx = fabs(w);
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((l & 31) == 0) wmax[l >> 5] = mx;
  __syncthreads();
  mx = 0.0;
  for (int q = 0; q < (int)(blockDim.x >> 5); ++q) mx = fmax(mx, wmax[q]);
  int e = 0;
  if (mx > 0.0) { frexp(mx, &e); }                     // mx < 2^e
  if (l == 0) wexp[j] = e;
  if (l >= kg) return;
  long long F = llrint(ldexp(w, 54 - e));               // |F| <= 2^54
  int d[QT_DB];
  for (int b = QT_DB - 1; b >= 1; --b) {               // balanced base-256 digits, exact
    const long long r = ((F + 128) & 255) - 128;
    d[b] = (int)r;
    F = (F - r) >> 8;
  }
  d[0] = (int)F;                                       // |d0| <= 65
  int8_t* tile = wdig + qt_woff(g);
  for (int b = 0; b < QT_DB; ++b) tile[(l >> 4) * QT_NB * 16 + (b * QT_G + jj) * 16 + (l & 15)] = (int8_t)d[b];
}

// ---------------------------------------------------------------------------------------------
// Epilogue arithmetic.  The levels are exact int32 (|acc_L| < 2^23: <= 6 pairs x 64 terms x 2^14, and
// |acc_0|, |acc_1| < 2^18, 2^21 from the small leading digits), and
//     Q_ij = 2^(e_i - 46 + e_j - 54) sum_L acc_L 256^(11 - L) = v 2^(e_i + e_j - 60),
//     v    = sum_L acc_L 256^(6 - L)  (up to ~2^66: not an int64).
// The epilogue forms T = acc_0 2^40 + acc_1 2^32 + acc_2 2^24 + acc_3 2^16 + acc_4 2^8 + acc_5 +
// floor(acc_6 / 2^8) EXACTLY in int64 (|T| < 2^60; T 2^8 differs from v by acc_6 mod 2^8 < 2^8, i.e.
// 2^-37 of a typical |v| -- far below the fp32 rounding of Q, the same order as the dropped levels),
// converts it once with round-to-nearest (I2F.F32.S64) and scales by 2^(e_i + e_j - 52) with one FMUL
// whose factor is built from the two exponents by one integer add: Q_ij = RN(T) 2^(e_i + e_j - 52).
// Round 1 combined the levels in fp64 (four magic-constant conversions, three DFMAs and two DMULs per
// output); this form needs ~10 integer-pipe instructions, one conversion and one FMUL.
template <bool K64>
__device__ __forceinline__ long long qt_combine(uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t a4,
                                                uint32_t a5, uint32_t a6) {
  // adjacent levels pair exactly in int32: |acc_0 256 + acc_1| < 2^28, |acc_2 256 + acc_3| < 2^31 for K <= 128,
  // and for K <= 64 also |acc_4 256 + acc_5 + (acc_6 >> 8)| < 2^31 (the digit bounds above); then
  // T = p0 2^32 + p1 2^16 + p2 is one IMAD.WIDE and one add into the high word
  const int p0 = (int)a0 * 256 + (int)a1;
  const int p1 = (int)a2 * 256 + (int)a3;
  if constexpr (K64) {
    // p0 2^32 + p2 as one register pair: low word p2 (as unsigned), high word p0 - [p2 < 0]; then one IMAD.WIDE
    const int p2 = (int)a4 * 256 + (int)a5 + ((int)a6 >> 8);
    long long c;
    asm("mov.b64 %0, {%1, %2};" : "=l"(c) : "r"(p2), "r"(p0 + (p2 >> 31)));
    return (long long)p1 * 65536 + c;
  } else {
    const long long t = (long long)p1 * 65536 + (long long)(int)a4 * 256 + (long long)((int)a5 + ((int)a6 >> 8));
    return t + ((long long)p0 << 32);
  }
}
// column scales of 8 consecutive outputs: fast route 2^(e_j - min e_j) as floats, exact route e_j
template <bool FAST>
__device__ __forceinline__ void qt_col_scales(const int* cexp, const float* csf, int j0, int (&cb)[8], float (&sc)[8]) {
  if constexpr (FAST) {
    const float4 s0 = *reinterpret_cast<const float4*>(csf + j0), s1 = *reinterpret_cast<const float4*>(csf + j0 + 4);
    sc[0] = s0.x; sc[1] = s0.y; sc[2] = s0.z; sc[3] = s0.w; sc[4] = s1.x; sc[5] = s1.y; sc[6] = s1.z; sc[7] = s1.w;
#pragma unroll
    for (int c = 0; c < 8; ++c) cb[c] = 0;
  } else {
    const int4 c0 = *reinterpret_cast<const int4*>(cexp + j0), c1 = *reinterpret_cast<const int4*>(cexp + j0 + 4);
    cb[0] = c0.x; cb[1] = c0.y; cb[2] = c0.z; cb[3] = c0.w; cb[4] = c1.x; cb[5] = c1.y; cb[6] = c1.z; cb[7] = c1.w;
#pragma unroll
    for (int c = 0; c < 8; ++c) sc[c] = 0.0f;
  }
}
// fast route (warp-uniform): every 2^(e_i + e_j - 52) of the warp's rows is a normal fp32, built as the bits
// (e_i + 75) << 23 plus e_j << 23; else this exact fp64 route (any exponent range)
__device__ __noinline__ float qt_scale_slow(long long t, int ei, int ej) { return (float)ldexp((double)t, ei + ej - 52); }

// CM: X and Q column-major (element (i, j) at [j * ld + i]), else row-major.  The tensor maps
// then have the row as their contiguous dimension: a raw X stage is [column][128 rows], a Q staging tile
// [column][32 rows]; the digit tiles, the MMAs and TMEM are the same.
template <int KMAX, bool CM>
__global__ void __launch_bounds__(QCfg<KMAX>::THREADS, 1)
solve_tc_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap qmap,
                const int8_t* __restrict__ wdig, const int* __restrict__ wexp, const float* __restrict__ X,
                int64_t ldx, int64_t m, int n, int kpad, float* __restrict__ Q, int64_t ldq, int* status,
                int dbg_in) {
  const int dbg = kAblation ? dbg_in : 0;   // ablation switches (see internal.cuh)
  using Cf = QCfg<KMAX>;
  constexpr int QT_DIG = Cf::DIG, QT_RAW = Cf::RAW > 0 ? Cf::RAW : 1, QT_A_TILE = Cf::A_TILE;
  constexpr int NSLOT = Cf::NSLOT, SLOT = Cf::SLOT_BYTES, H_TILE = Cf::H_TILE;
  constexpr int QT_RS_MAX = Cf::RS, QT_RAW_STAGE = Cf::RAW_STAGE;
  if (*status) return;                                 // singular R: Q is not written
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* wsm = sm;                                                   // W digits, all groups
  unsigned char* abase = sm + Cf::W_BYTES;                                    // [NSLOT][DA][A_TILE or H_TILE]
  float* raw_base = reinterpret_cast<float*>(abase + (size_t)NSLOT * SLOT);  // [RAW][128][RS]
  unsigned char* qstage = reinterpret_cast<unsigned char*>(raw_base) + (size_t)Cf::RAW * QT_RAW_STAGE;   // [8][32 rows][128 B]
  uint64_t* bars = reinterpret_cast<uint64_t*>(qstage + Cf::QS);
  uint64_t* dfull = bars;                   // [NSLOT] X digits of a tile (or K-half) ready
  uint64_t* dempty = dfull + NSLOT;         // [NSLOT] MMAs reading the slot complete (tcgen05.commit)
  uint64_t* rfull = dempty + NSLOT;         // [RAW]
  uint64_t* rempty = rfull + QT_RAW;        // [RAW]
  uint64_t* tready = rempty + QT_RAW;       // [2] level buffer written (commit)
  uint64_t* tfree = tready + 2;             // [2] level buffer drained
  uint64_t* wbar = tfree + 2;               // W digits staged
  uint64_t* sfull = wbar + 1;               // [RAW] column-major: raw stage landed AND its row scales written
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sfull + QT_RAW);
  // row scales: a ring of 4 tiles, so the digit slot can be refilled while the drain of the tile
  // before still reads its scales (a slot is free once the MMAs of tile t complete, and those
  // follow every drain of tile t - 2; see the TMEM buffer waits below)
  // 16-byte aligned (the drain reads the column exponents cexp with LDS.128); offset from sm, so the compiler
  // keeps these accesses in the shared window (LDS/STS, not generic LD/ST)
  const size_t rexp_off = ((size_t)(reinterpret_cast<unsigned char*>(tmem_slot + 4) - sm) + 15) & ~(size_t)15;
  int* rexp = reinterpret_cast<int*>(sm + rexp_off);                          // [RXD][128]
  constexpr int RXD = Cf::RXD;
  int* cexp = rexp + RXD * QT_M;                                                // [KMAX] e_j (W column exponents)
  int* crange = cexp + QT_KMAX_ALL;                                           // [2] min, max e_j
  float* csf = reinterpret_cast<float*>(crange + 4);                          // [KMAX] 2^(e_j - min e_j) (fast scaling route)

  const int groups = (n + QT_G - 1) / QT_G;
  const int64_t ntiles = (m + QT_M - 1) / QT_M;
  const int my_tiles = blockIdx.x < ntiles ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int lg_n = kpad / 16;                                                 // 16-column groups per row

  if (tid == 0) {
    for (int s = 0; s < NSLOT; ++s) { tc::mbar_init(&dfull[s], Cf::DW); tc::mbar_init(&dempty[s], 1); }
    for (int s = 0; s < QT_RAW; ++s) { tc::mbar_init(&rfull[s], 1); tc::mbar_init(&rempty[s], Cf::DW); tc::mbar_init(&sfull[s], 1); }
    for (int b = 0; b < 2; ++b) { tc::mbar_init(&tready[b], 1); tc::mbar_init(&tfree[b], Cf::RW / 2); }
    tc::mbar_init(wbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (tid < 2) crange[tid] = tid == 0 ? INT32_MAX : INT32_MIN;
  __syncthreads();
  if (tid < groups * QT_G) {
    const int ej = wexp[tid];
    cexp[tid] = ej;
    if (tid < n) { atomicMin(&crange[0], ej); atomicMax(&crange[1], ej); }
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(tc::smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = *tmem_slot;
  if (tid < groups * QT_G) csf[tid] = __int_as_float(min(max(cexp[tid] - crange[0], 0), 127) + 127 << 23);
  __syncthreads();

  if (warp == 0) {
    // ---------------------------------------------------------------- MMA issuer (lane 0)
    tc::mbar_wait(wbar, 0u);
    for (int tt = 0; tt < my_tiles; ++tt) {
      // full-tile slot s (n <= 64), or the two K-half slots s, s1 (uses 2 tt and 2 tt + 1 of the ring)
      const int s = Cf::HALF ? (2 * tt) % NSLOT : tt % NSLOT, s1 = (2 * tt + 1) % NSLOT;
      if (lane == 0) trace(0, tt, 0);
      tc::mbar_wait(&dfull[s], (uint32_t)(((Cf::HALF ? 2 * tt : tt) / NSLOT) & 1));
      if (lane == 0) trace(0, tt, 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      bool have1 = !Cf::HALF;
      for (int g = 0; g < groups; ++g) {
        const int use = tt * groups + g, buf = use & 1, u = use >> 1;
        if (u > 0) tc::mbar_wait(&tfree[buf], (uint32_t)((u - 1) & 1));
        if (lane == 0 && g < 2) trace(0, tt, 2 + 2 * g);
        const int ksteps = min(g + 1, kpad / 32);             // W rows l < 32 (g + 1): upper triangular
        if (!have1 && ksteps > 2) {                           // second K-half needed from here on
          tc::mbar_wait(&dfull[s1], (uint32_t)(((2 * tt + 1) / NSLOT) & 1));
          have1 = true;
        }
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        if (lane == 0 && !(dbg & 1)) {
          const uint32_t sb = tc::smem_u32(wsm + qt_woff(g));
          for (int ks = 0; ks < ksteps; ++ks) {
            const uint32_t sa = Cf::HALF ? tc::smem_u32(abase + (size_t)(ks < 2 ? s : s1) * SLOT) + (ks & 1) * 2 * (QT_M * 16)
                                         : tc::smem_u32(abase + (size_t)s * SLOT) + ks * 2 * (QT_M * 16);
            constexpr int PLANE = Cf::HALF ? H_TILE : QT_A_TILE;
#pragma unroll
            for (int a = 0; a < QT_DA; ++a) {
              const uint64_t da = tc::desc(sa + a * PLANE, QT_M * 16, 128);
              const uint64_t db = tc::desc(sb + ks * 2 * (QT_NB * 16), QT_NB * 16, 128);
              const uint32_t idesc = tc::idesc_i8(QT_M, (QT_DB - a) * QT_G, true, true);
              tc::mma_i8(tmem + buf * (QT_LEV * QT_G) + a * QT_G, da, db, idesc, (ks > 0 || a > 0) ? 1u : 0u);
            }
          }
        }
        if (lane == 0) { tc::commit(&tready[buf]); if (g < 2) trace(0, tt, 3 + 2 * g); }
        __syncwarp();
      }
      if (lane == 0) {                                    // digit slot(s) free once these MMAs complete
        tc::commit(&dempty[s]);
        if (Cf::HALF) tc::commit(&dempty[s1]);
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- loader (lane 0)
    if (lane == 0) {
      if (Cf::TMA_RAW) asm volatile("prefetch.tensormap [%0];\n" ::"l"(&xmap) : "memory");
      const uint32_t wbytes = (uint32_t)qt_woff(groups);
      tc::mbar_arrive_tx(wbar, wbytes);
      tc::bulk_g2s(wsm, wdig, wbytes, wbar);
    }
    __syncwarp();
    // the raw ring holds two tiles; tiles up to QT_PF ahead are prefetched into L2 so that enough HBM
    // bytes are in flight per SM (~QT_PF x 34 KB) -- the ring loads then hit L2
    // raw-stage coordinates: (column 0, row r) row-major, (row r, column 0) column-major
    auto pf_tile = [&](int64_t row) { if (CM) tc::tma_prefetch_2d(&xmap, (int)row, 0); else tc::tma_prefetch_2d(&xmap, 0, (int)row); };
    // column-major: this warp also computes the row scales e_i of a landed stage (lane = row; the stage is
    // [column][128 rows], so a row's columns are 512 B apart and a 16-column digit task cannot see the whole
    // row) and publishes stage + scales on sfull; row-major: the digit warps do it with a shuffle max
    auto row_scales = [&](int t2) {
      const int s2 = t2 % QT_RAW;
      tc::mbar_wait(&rfull[s2], (uint32_t)((t2 / QT_RAW) & 1));
      const float* raw = raw_base + (size_t)s2 * QT_M * QT_RS_MAX;
#pragma unroll 1
      for (int rb = 0; rb < QT_M / 32; ++rb) {
        float mf = 0.0f;
#pragma unroll 8
        for (int c = 0; c < kpad; c += 2)
          asm("max.NaN.f32 %0, %0, %1, %2;" : "+f"(mf) : "f"(fabsf(raw[c * QT_M + rb * 32 + lane])),
              "f"(fabsf(raw[(c + 1) * QT_M + rb * 32 + lane])));
        const uint32_t mx = __float_as_uint(mf);
        if (mx >= 0x7F800000u) atomicOr(status, kStNonfinite);
        rexp[(t2 % RXD) * QT_M + rb * 32 + lane] = mx == 0u ? 0 : (mx < 0x00800000u ? -126 : (int)(mx >> 23) - 126);
      }
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&sfull[s2]);           // release: the scales above are visible to the waiters
    };
    if (Cf::TMA_RAW && lane == 0)
      for (int tp = 1; tp < QT_PF && tp < my_tiles; ++tp) pf_tile((blockIdx.x + (int64_t)tp * gridDim.x) * QT_M);
    for (int tt = 0; tt < (Cf::TMA_RAW ? my_tiles : 0); ++tt) {
      const int s = tt % QT_RAW;
      if (lane == 0) trace(1, tt, 0);
      // scales of the stage before (landed while the digit warps worked on tile tt - 2), so the digits of tile
      // tt - 1 can start the moment those warps are free; only then wait for the slot of tile tt
      if (CM && tt > 0) row_scales(tt - 1);
      if (tt >= QT_RAW) tc::mbar_wait(&rempty[s], (uint32_t)(((tt / QT_RAW) - 1) & 1));
      if (lane == 0) {
        trace(1, tt, 1);
        if (tt + QT_PF < my_tiles) pf_tile((blockIdx.x + (int64_t)(tt + QT_PF) * gridDim.x) * QT_M);
        const int64_t row0 = (blockIdx.x + (int64_t)tt * gridDim.x) * QT_M;
        if (dbg & 8) tc::mbar_arrive(&rfull[s]);
        else if (CM) {
          tc::mbar_arrive_tx(&rfull[s], (uint32_t)(QT_M * kpad * 4));
          tc::tma_load_2d(raw_base + (size_t)s * QT_M * QT_RS_MAX, &xmap, (int)row0, 0, &rfull[s]);
        } else {
          tc::mbar_arrive_tx(&rfull[s], (uint32_t)(QT_M * (kpad + 4) * 4));
          tc::tma_load_2d(raw_base + (size_t)s * QT_M * QT_RS_MAX, &xmap, 0, (int)row0, &rfull[s]);
        }
      }
      __syncwarp();
    }
    if (CM && Cf::TMA_RAW && my_tiles > 0) row_scales(my_tiles - 1);
  } else if (warp < 2 + Cf::RW) {
    // ---------------------------------------------------------------- drain (set = buffer, lane quadrant)
    // set = buffer (warps 2..5, 6..9, then again for the second column half when RW = 16)
    const int dset = ((warp - 2) >> 2) & 1, dq = warp & 3, row_l = dq * 32 + lane;
    const int dc0 = ((warp - 2) >> 3) * Cf::DCOLS;     // first column of the group this warp drains
    const uint32_t lb = tmem + ((uint32_t)(dq * 32) << 16);
    // Column-major Q: a TMA store clips its contiguous (row) dimension in 16-byte units, not by element (measured:
    // tools/micro/tma_clip_test.cu), so the Q tensor map ends at row m & ~3 and the last m % 4 rows are written by
    // these plain stores -- the pitch padding of Q is never touched.
    auto cm_tail = [&](const float (&o)[8], int col0, int64_t row) {
      if (CM && row >= (m & ~(int64_t)3) && row < m) {
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (col0 + c < n) Q[(size_t)(col0 + c) * ldq + row] = o[c];
      }
    };
    for (int tt = 0; tt < my_tiles; ++tt) {
      for (int g = 0; g < groups; ++g) {
        const int use = tt * groups + g, buf = use & 1, u = use >> 1;
        if (buf != dset) continue;
        const int trole = (warp == 2 || warp == 6) ? 2 + dset : -1;
        if (lane == 0 && trole >= 0) trace(trole, tt, 0);
        tc::mbar_wait(&tready[buf], (uint32_t)(u & 1));
        if (lane == 0 && trole >= 0) trace(trole, tt, 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        // the seven exact int32 levels of an output combine into one int64 (qt_combine); the warp
        // takes the fp32 scaling route unless some 2^(e_i + e_j - 52) of its rows leaves the normal range
        static_assert(QT_LEV == 7, "qt_combine assumes 7 levels");
        if constexpr (Cf::HALF) {
          // 8 columns at a time: all 7 level loads in flight before one wait; each 32-row x 8-column
          // fp32 chunk is staged in a 1 KB tile (all the room the K-half ring leaves) and written
          // by a 2D TMA store; the TMEM buffer is released right after the last chunk's loads
          const int ei = rexp[(tt % RXD) * QT_M + row_l];
          const float rs = __int_as_float((ei + crange[0] + 75) << 23);   // 2^(e_i + min e_j - 52), used if fast
          const bool fast = __all_sync(0xffffffffu, ei + crange[0] + 75 >= 1 && ei + crange[1] + 75 <= 254 &&
                                                        crange[1] - crange[0] <= 127);
          const uint32_t lv = lb + buf * (QT_LEV * QT_G);
          unsigned char* qs = qstage + (warp - 2) * (32 * 8 * 4);
          auto drain = [&](auto fast_tag) {
            constexpr bool FAST = decltype(fast_tag)::value;
#pragma unroll
            for (int h = 0; h < QT_G / 8; ++h) {
              uint32_t lvl[QT_LEV][8];
#pragma unroll
              for (int L = 0; L < QT_LEV; ++L) tc::ld8(lv + L * QT_G + h * 8, lvl[L]);
              int cb[8];
              float sc[8];
              qt_col_scales<FAST>(cexp, csf, g * QT_G + h * 8, cb, sc);
              tc::wait_ld();
              if (h == QT_G / 8 - 1) {
                asm volatile("tcgen05.fence::before_thread_sync;\n");
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&tfree[buf]);
              }
              float o[8];
#pragma unroll
              for (int c = 0; c < 8; ++c) {
                const long long t = qt_combine<KMAX <= 64>(lvl[0][c], lvl[1][c], lvl[2][c], lvl[3][c], lvl[4][c], lvl[5][c], lvl[6][c]);
                if constexpr (FAST) o[c] = __ll2float_rn(t) * (rs * sc[c]);   // exact power-of-two factor (normal: fast)
                else o[c] = qt_scale_slow(t, ei, cb[c]);
              }
              if (lane == 0) tc::bulk_wait_read0();          // previous chunk's store has read the tile
              __syncwarp();
              // 32-byte rows, TMA SWIZZLE_32B (16-byte chunk c of row r at c ^ ((r >> 2) & 1)): conflict-free STS.128
              if constexpr (CM) {                            // [8 columns][32 rows]: conflict-free STS.32
#pragma unroll
                for (int c = 0; c < 8; ++c) reinterpret_cast<float*>(qs)[c * 32 + lane] = o[c];
                cm_tail(o, g * QT_G + h * 8, (blockIdx.x + (int64_t)tt * gridDim.x) * QT_M + row_l);
              } else {
                const int sw = (lane >> 2) & 1;
                *reinterpret_cast<float4*>(qs + lane * 32 + (sw << 4)) = make_float4(o[0], o[1], o[2], o[3]);
                *reinterpret_cast<float4*>(qs + lane * 32 + ((sw ^ 1) << 4)) = make_float4(o[4], o[5], o[6], o[7]);
              }
              asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
              __syncwarp();
              if (lane == 0) {                               // TMA clips rows >= m and columns >= n
                const int qrow = (int)((blockIdx.x + (int64_t)tt * gridDim.x) * QT_M + dq * 32);
                if (CM) tc::tma_store_2d(&qmap, qs, qrow, g * QT_G + h * 8);
                else tc::tma_store_2d(&qmap, qs, g * QT_G + h * 8, qrow);
                tc::bulk_commit();
              }
            }
          };
          if (fast) drain(std::true_type{});
          else drain(std::false_type{});
        } else {
        constexpr int DC = Cf::DCOLS;
        const uint32_t lv = lb + buf * (QT_LEV * QT_G) + dc0;
        // row scale read before the buffer is released: the rexp ring slot is reused only after
        // later MMAs, which wait on this release
        const int ei = rexp[(tt % RXD) * QT_M + row_l];
        const float rs = __int_as_float((ei + crange[0] + 75) << 23);     // 2^(e_i + min e_j - 52), used if fast
        const bool fast = __all_sync(0xffffffffu, ei + crange[0] + 75 >= 1 && ei + crange[1] + 75 <= 254 &&
                                                      crange[1] - crange[0] <= 127);
        // this warp's 32 rows x DC columns (fp32) are staged in shared memory (16-column rows: plain
        // 64-byte rows; 32-column rows: 128-byte swizzle, chunk c of row r at c ^ (r & 7) -- conflict-free
        // STS.128) as they are computed, then one 2D TMA store writes them (rows >= m, columns >= n clipped)
        unsigned char* qs = qstage + (warp - 2) * (32 * DC * 4);
        if (lane == 0) tc::bulk_wait_read0();                // the previous store has read the tile
        __syncwarp();
        // the fast / exact-range choice is warp-uniform, so it is taken once per drained group
        auto drain = [&](auto fast_tag) {
          constexpr bool FAST = decltype(fast_tag)::value;
#pragma unroll
          for (int h = 0; h < DC / 8; ++h) {
            uint32_t lvl[QT_LEV][8];                         // all seven levels in flight before one wait
#pragma unroll
            for (int L = 0; L < QT_LEV; ++L) tc::ld8(lv + L * QT_G + h * 8, lvl[L]);
            int cb[8];
            float sc[8];
            qt_col_scales<FAST>(cexp, csf, g * QT_G + dc0 + h * 8, cb, sc);
            tc::wait_ld();
            if (h == DC / 8 - 1) {                           // TMEM buffer free; the stores below need no TMEM
              asm volatile("tcgen05.fence::before_thread_sync;\n");
              __syncwarp();
              if (lane == 0) { tc::mbar_arrive(&tfree[buf]); if (trole >= 0) trace(trole, tt, 2); }
            }
            float o[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const long long t = qt_combine<KMAX <= 64>(lvl[0][c], lvl[1][c], lvl[2][c], lvl[3][c], lvl[4][c], lvl[5][c], lvl[6][c]);
              if constexpr (FAST) o[c] = __ll2float_rn(t) * (rs * sc[c]);   // exact power-of-two factor (normal: fast)
              else o[c] = qt_scale_slow(t, ei, cb[c]);
            }
            if constexpr (CM) {                              // [DC columns][32 rows]: conflict-free STS.32
#pragma unroll
              for (int c = 0; c < 8; ++c) reinterpret_cast<float*>(qs)[(h * 8 + c) * 32 + lane] = o[c];
              cm_tail(o, g * QT_G + dc0 + h * 8, (blockIdx.x + (int64_t)tt * gridDim.x) * QT_M + row_l);
            } else {
#pragma unroll
              for (int c = 0; c < 8; c += 4) {
                const int ch = h * 2 + (c >> 2);                // 16-byte chunk of the row
                // 128-byte rows (DC = 32): TMA SWIZZLE_128B, chunk ch at ch ^ (r & 7); 64-byte rows (DC = 16): SWIZZLE_64B,
                // chunk ch at ch ^ ((r >> 1) & 3) -- each 8-lane phase of the STS.128 hits 8 distinct bank groups
                const int off = DC == 32 ? lane * 128 + ((ch ^ (lane & 7)) << 4) : lane * 64 + ((ch ^ ((lane >> 1) & 3)) << 4);
                *reinterpret_cast<float4*>(qs + off) = make_float4(o[c], o[c + 1], o[c + 2], o[c + 3]);
              }
            }
          }
        };
        if (dbg & 4) {                                     // ablation: no TMEM loads, combine or Q stores
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&tfree[buf]);
        } else if (fast) drain(std::true_type{});
        else drain(std::false_type{});
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        if (lane == 0 && !(dbg & 4)) {
          const int qrow = (int)((blockIdx.x + (int64_t)tt * gridDim.x) * QT_M + dq * 32);
          if (CM) tc::tma_store_2d(&qmap, qs, qrow, g * QT_G + dc0);
          else tc::tma_store_2d(&qmap, qs, g * QT_G + dc0, qrow);
          tc::bulk_commit();
          if (trole >= 0) trace(trole, tt, 3);
        }
        }   // TMA_RAW drain
      }
    }
  } else {
    // ---------------------------------------------------------------- X digit planes
    // lane -> (column group lg, row): consecutive lanes take consecutive rows of one column group,
    // so with the (K + 4)-float pitch every 8-lane phase of an LDS.128 hits 8 distinct 16-byte
    // bank groups, and the digit STS.128 of a phase are contiguous.  The column groups per row are
    // rounded up to a power of two (lg_map) for the shuffle max; groups >= lg_n read zeros.
    // Plain-load producers (64 < n <= 128) issue the loads of all their tasks of a tile before
    // waiting for the digit slot, so the HBM latency overlaps the MMAs of the tile before.
    const int dt = tid - 32 * (2 + Cf::RW);
    const int lg_map = lg_n <= 2 ? lg_n : (lg_n <= 4 ? 4 : 8), rpw = 32 / lg_map;
    const int lsh = 31 - __clz(rpw);
    const int ntask = (dbg & 2) ? 0 : QT_M * lg_map;
    auto task_pos = [&](int task, int& lg, int& i) {
      const int w = task >> 5, l = task & 31;
      lg = l >> lsh; i = (w << lsh) + (l & (rpw - 1));           // rpw = 2^lsh
    };
    // the six signed base-256 digits of round(x 2^(46 - e)), packed 4 columns per word, for 16 x
    auto digit_words = [&](const float* x, int e, uint32_t (&W)[QT_DA][4]) {
      // 2^(46 - e) built from its exponent field (e in [-126, 128]: always a normal double)
      const double sx = __hiloint2double((1023 + 46 - e + (RCQ_SOLVE_F2F ? 0 : 128)) << 20, 0);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          // one exact F2F.F64.F32 (conversion pipe) instead of three integer-pipe instructions building the double
#if RCQ_SOLVE_F2F
          const double t = fma((double)x[q * 4 + kk], sx, kMagic + (double)0x8080808080ull);
#else
          const uint32_t ub = __float_as_uint(x[q * 4 + kk]);
          uint32_t h;                                                                        // x 2^-128: one LOP3
          asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(h) : "r"((uint32_t)((int32_t)ub >> 3)), "r"(0x8FFFFFFFu), "r"(0x30000000u));
          const double t = fma(__hiloint2double((int)h, (int)(ub << 29)), sx, kMagic + (double)0x8080808080ull);
#endif
          hw[kk] = (uint32_t)__double2hiint(t);                                              // F + C, 48 bits
          lw[kk] = (uint32_t)__double2loint(t);
        }
        uint32_t H[4], L[4];
        transpose4(hw[0], hw[1], hw[2], hw[3], H);
        transpose4(lw[0], lw[1], lw[2], lw[3], L);
        W[0][q] = H[1]; W[1][q] = H[0] ^ 0x80808080u;
        W[2][q] = L[3] ^ 0x80808080u; W[3][q] = L[2] ^ 0x80808080u;
        W[4][q] = L[1] ^ 0x80808080u; W[5][q] = L[0] ^ 0x80808080u;
      }
    };
    auto digits = [&](int task, int tt, unsigned char* at, const float* x) {
      int lg, i;
      task_pos(task, lg, i);
      float mf = 0.0f;                                     // max |x|, NaN-propagating: 8 FMNMX3.NAN with |.| operands
#pragma unroll
      for (int c = 0; c < 16; c += 2)
        asm("max.NaN.f32 %0, %0, %1, %2;" : "+f"(mf) : "f"(fabsf(x[c])), "f"(fabsf(x[c + 1])));
      uint32_t mx = __float_as_uint(mf);                   // NaN -> 0x7FFFFFFF
      for (int o = rpw; o < 32; o <<= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      // e_i: smallest e with max |x| < 2^e.  Inside rcholqr_factor the sketch has already rejected
      // NaN/Inf; a direct tri_solve call reports them here (Q is then not meaningful)
      if (mx >= 0x7F800000u) atomicOr(status, kStNonfinite);
      const int e = mx == 0u ? 0 : (mx < 0x00800000u ? -126 : (int)(mx >> 23) - 126);
      if (lg == 0) rexp[(tt % RXD) * QT_M + i] = e;
      uint32_t W[QT_DA][4];
      digit_words(x, e, W);
#pragma unroll
      for (int a = 0; a < QT_DA; ++a)
        *reinterpret_cast<uint4*>(at + a * QT_A_TILE + lg * (QT_M * 16) + i * 16) =
            make_uint4(W[a][0], W[a][1], W[a][2], W[a][3]);
    };
    // column-major raw stage [column][128 rows]: warp-task w = (32-row block, 16-column group), lane = row, so
    // the 16 LDS.32 of a task and its digit STS.128 are conflict-free; the row scale comes from the loader warp
    auto digits_cm = [&](int w, int tt, unsigned char* at, const float* raw) {
      const int lg = w % lg_n, i = (w / lg_n) * 32 + lane;
      float x[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) x[c] = raw[(lg * 16 + c) * QT_M + i];
      const int e = rexp[(tt % RXD) * QT_M + i];
      uint32_t W[QT_DA][4];
      digit_words(x, e, W);
#pragma unroll
      for (int a = 0; a < QT_DA; ++a)
        *reinterpret_cast<uint4*>(at + a * QT_A_TILE + lg * (QT_M * 16) + i * 16) =
            make_uint4(W[a][0], W[a][1], W[a][2], W[a][3]);
    };
    float xh0[2][16], xh1[2][16];                          // HALF producers: [task][16] per K-half
    for (int tt = 0; tt < my_tiles; ++tt) {
      const int s = tt % QT_DIG, sr = tt % QT_RAW;
      unsigned char* at = abase + (size_t)s * QT_DA * QT_A_TILE;
      if constexpr (Cf::TMA_RAW) {
        if (dt == 0) trace(4, tt, 0);
        if (tt >= QT_DIG) tc::mbar_wait(&dempty[s], (uint32_t)(((tt / QT_DIG) - 1) & 1));
        if (dt == 0) trace(4, tt, 1);
        tc::mbar_wait(CM ? &sfull[sr] : &rfull[sr], (uint32_t)((tt / QT_RAW) & 1));
        if (dt == 0) trace(4, tt, 2);
        const float* raw = raw_base + (size_t)sr * QT_M * QT_RS_MAX;
        const int rs = kpad + 4;                                         // raw row pitch
        // the tile's NW = 4 lg_map warp-tasks (32 lanes x 16 columns each) are dealt round-robin to the DW
        // digit warps starting at a warp that rotates with the tile: NW is not a multiple of DW (16 over 10),
        // so a fixed start would leave the same warps with the extra task on every tile (the digit stages
        // let a lightly loaded warp run ahead into the next tile, which evens the load out)
        const int nw = ntask >> 5, dw = dt >> 5;
        const int off = RCQ_SOLVE_ROT ? (int)(((unsigned)tt * (unsigned)(nw % Cf::DW)) % Cf::DW) : 0;
        for (int w = (dw + Cf::DW - off) % Cf::DW; w < nw; w += Cf::DW) {
          if constexpr (CM) { digits_cm(w, tt, at, raw); continue; }
          const int task = w * 32 + lane;
          int lg, i;
          task_pos(task, lg, i);
          float x[16];
#pragma unroll
          for (int c = 0; c < 16; c += 4) {
            const float4 f = *reinterpret_cast<const float4*>(raw + i * rs + lg * 16 + c);
            x[c] = f.x; x[c + 1] = f.y; x[c + 2] = f.z; x[c + 3] = f.w;
          }
          digits(task, tt, at, x);
        }
      } else {
        // K-half producers: lane -> (row i = 8 w + (lane & 7), 16-column group lg' = lane >> 3 of
        // each half); each task holds its row's columns 16 lg' .. + 15 of both halves, so the row
        // exponent (max over the row: lanes xor 8, 16) is known before either half is written.
        // Software-pipelined: the loads of a half of tile t + 1 are issued as soon as the digits of
        // that half of tile t are written, so HBM latency overlaps the waits for free half slots.
        const int dw = warp - (2 + Cf::RW), lgp = lane >> 3;
        auto load_half = [&](int t2, int h, float (&xo)[2][16]) {
          const int64_t r0 = (blockIdx.x + (int64_t)t2 * gridDim.x) * QT_M;
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            const int64_t row = r0 + (dw + QT_DWARPS * b) * 8 + (lane & 7);
            const int c0 = 64 * h + 16 * lgp;
            const float* xr = X + row * ldx + c0;
            if constexpr (CM) {                              // column-major: element (row, c0 + c) at X[(c0 + c) ldx + row]
#pragma unroll
              for (int c = 0; c < 16; ++c) xo[b][c] = (row < m && c0 + c < n) ? __ldg(X + (int64_t)(c0 + c) * ldx + row) : 0.0f;
            } else if (row < m && c0 + 16 <= n) {
#pragma unroll
              for (int c = 0; c < 16; c += 4) {
                const float4 f = __ldg(reinterpret_cast<const float4*>(xr + c));
                xo[b][c] = f.x; xo[b][c + 1] = f.y; xo[b][c + 2] = f.z; xo[b][c + 3] = f.w;
              }
            } else {
#pragma unroll
              for (int c = 0; c < 16; ++c) xo[b][c] = (row < m && c0 + c < n) ? xr[c] : 0.0f;
            }
          }
        };
        if (tt == 0) { load_half(0, 0, xh0); load_half(0, 1, xh1); }
        int ee[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int u = 2 * tt + h, sh = u % NSLOT;
          if (u >= NSLOT) tc::mbar_wait(&dempty[sh], (uint32_t)(((u / NSLOT) - 1) & 1));
          float (&xc)[2][16] = h == 0 ? xh0 : xh1;
          if (h == 0) {
#pragma unroll
            for (int b = 0; b < 2; ++b) {
              float mf = 0.0f;                             // NaN-propagating max |x| (FMNMX3.NAN)
#pragma unroll
              for (int c = 0; c < 16; ++c)
                asm("max.NaN.f32 %0, %0, %1, %2;" : "+f"(mf) : "f"(fabsf(xh0[b][c])), "f"(fabsf(xh1[b][c])));
              uint32_t mx = __float_as_uint(mf);
              mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
              mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
              if (mx >= 0x7F800000u) atomicOr(status, kStNonfinite);   // tri_solve on NaN/Inf X
              ee[b] = mx == 0u ? 0 : (mx < 0x00800000u ? -126 : (int)(mx >> 23) - 126);
              if (lgp == 0) rexp[(tt % RXD) * QT_M + (dw + QT_DWARPS * b) * 8 + (lane & 7)] = ee[b];
            }
          }
          unsigned char* ah = abase + (size_t)sh * SLOT;
          if (!(dbg & 2)) {
#pragma unroll
            for (int b = 0; b < 2; ++b) {
              uint32_t W[QT_DA][4];
              digit_words(xc[b], ee[b], W);
              const int i = (dw + QT_DWARPS * b) * 8 + (lane & 7);
#pragma unroll
              for (int a = 0; a < QT_DA; ++a)
                *reinterpret_cast<uint4*>(ah + a * H_TILE + lgp * (QT_M * 16) + i * 16) =
                    make_uint4(W[a][0], W[a][1], W[a][2], W[a][3]);
            }
          }
          if (tt + 1 < my_tiles) load_half(tt + 1, h, xc);      // next tile's half, in flight early
          if (h == 0) {                                  // the second half is published below
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&dfull[sh]);
          }
        }
      }
      const int sdone = Cf::HALF ? (2 * tt + 1) % NSLOT : s;
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) { tc::mbar_arrive(&dfull[sdone]); if (Cf::TMA_RAW) tc::mbar_arrive(&rempty[sr]); }
      if (dt == 0) trace(4, tt, 3);
    }
  }
  if (warp >= 2 && warp < 2 + Cf::RW && lane == 0) tc::bulk_wait0();   // Q stores complete before exit
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

// fp32 X, n <= 128 (RCHOLQR_SOLVE_DMMA=1 selects the DMMA substitution instead).  At C2 (n = 100)
// the digit solve with its prep takes 0.54 ms against the DMMA kernel's 0.70 ms.
bool solve_tc_applicable(int dtype, int n) {
  if (dtype != RCHOLQR_F32 || n < 1 || getenv("RCHOLQR_SOLVE_DMMA")) return false;
  return n <= QT_KMAX_ALL;
}

bool solve_tc_supported(const void* X, int64_t m, int64_t ldx, const void* Q, int64_t ldq) {
  return m <= INT32_MAX && ((uintptr_t)X % 16) == 0 && ((size_t)ldx * 4) % 16 == 0 &&   // TMA base / pitch
         ((uintptr_t)Q % 16) == 0 && ((size_t)ldq * 4) % 16 == 0;
}

size_t solve_tc_workspace() { return (size_t)qt_woff(QT_KMAX_ALL / QT_G) + sizeof(int) * QT_KMAX_ALL; }

using EncodeTiledFn2 = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// W = R^{-1} already in Winv (n x n fp64).  ws: workspace of solve_tc_workspace(n) bytes.
// colmajor: X and Q column-major with leading dimensions ldx, ldq >= m (native kernels, no transposes).
cudaError_t launch_solve_tc(const double* Winv, int n, const float* X, int64_t m, int64_t ldx, float* Q, int64_t ldq,
                            void* ws, int* status, int sms, cudaStream_t st, bool colmajor) {
  if (m == 0) return cudaSuccess;
  if (!solve_tc_supported(X, m, ldx, Q, ldq)) return cudaErrorNotSupported;
  static EncodeTiledFn2 enc = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn2>(p);
  }();
  if (!enc) return cudaErrorNotSupported;
  const int kpad = (n + 31) / 32 * 32;
  const int groups = (n + QT_G - 1) / QT_G;
  int8_t* wdig = reinterpret_cast<int8_t*>(ws);
  int* wexp = reinterpret_cast<int*>(wdig + qt_woff(QT_KMAX_ALL / QT_G));
  solve_tc_prep_kernel<<<groups * QT_G, kpad, 0, st>>>(Winv, n, kpad, wdig, wexp, status);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  CUtensorMap map;
  // row-major: dims (columns, rows), box (K + 4 zero-padded columns, 128 rows); column-major: dims (rows, columns),
  // box (128 rows, K columns)
  const cuuint64_t dims[2] = {(cuuint64_t)(colmajor ? m : n), (cuuint64_t)(colmajor ? n : m)};
  const cuuint64_t strides[1] = {(cuuint64_t)ldx * 4};
  const cuuint32_t estr[2] = {1, 1};
  const cuuint32_t box[2] = {colmajor ? (cuuint32_t)QT_M : (cuuint32_t)std::min(kpad, 64) + 4,
                             colmajor ? (cuuint32_t)std::min(kpad, 64) : (cuuint32_t)QT_M};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(X), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  CUtensorMap qmapd;
  // column-major: rows m & ~3 .. m - 1 are written by plain stores (cm_tail), see there
  if (colmajor && m < 4) return cudaErrorNotSupported;
  const cuuint64_t qdims[2] = {(cuuint64_t)(colmajor ? (m & ~(int64_t)3) : n), (cuuint64_t)(colmajor ? n : m)};
  const cuuint64_t qstrides[1] = {(cuuint64_t)ldq * 4};
  const bool half = kpad > 64;                       // QCfg<128>::HALF: 8-column store boxes
  const int dcols = QCfg<64>::DCOLS;                 // n <= 64: columns per drain warp
  const cuuint32_t qcols = half ? 8u : (cuuint32_t)dcols;
  const cuuint32_t qbox[2] = {colmajor ? 32u : qcols, colmajor ? qcols : 32u};   // column-major: [columns][32 rows], no swizzle
  if (enc(&qmapd, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, Q, qdims, qstrides, qbox, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
          colmajor ? CU_TENSOR_MAP_SWIZZLE_NONE
                   : (half ? CU_TENSOR_MAP_SWIZZLE_32B : (dcols == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B)),
          CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  const int64_t ntiles = (m + QT_M - 1) / QT_M;
  const int grid = (int)std::min<int64_t>(ntiles, sms);
  static const int dbg = !kAblation ? 0 : getenv("RCHOLQR_QTC_DEBUG") ? atoi(getenv("RCHOLQR_QTC_DEBUG")) : 0;   // ablations only
  auto go = [&](auto kern, size_t smem, int threads) -> cudaError_t {
    cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e2 != cudaSuccess) return e2;
    kern<<<grid, threads, smem, st>>>(map, qmapd, wdig, wexp, X, ldx, m, n, kpad, Q, ldq, status, dbg);
    return cudaGetLastError();
  };
  if (colmajor)
    return kpad <= 64 ? go(solve_tc_kernel<64, true>, QCfg<64>::SMEM, QCfg<64>::THREADS)
                      : go(solve_tc_kernel<128, true>, QCfg<128>::SMEM, QCfg<128>::THREADS);
  return kpad <= 64 ? go(solve_tc_kernel<64, false>, QCfg<64>::SMEM, QCfg<64>::THREADS)
                    : go(solve_tc_kernel<128, false>, QCfg<128>::SMEM, QCfg<128>::THREADS);
}

#ifdef RCHOLQR_ABLATION
RCQ_TRACE_READER(trace_read_solve)
#endif

}  // namespace rcq
