// srht_fwht.cu -- the SRHT sketch P = Theta X by a blocked FAST Walsh-Hadamard transform: the m n log2 m cost the
// paper prices the SRHT at ("the SRHT ... takes only mn log2 m flops"), instead of the
// 2 k m n of a dense +-1 product.
//
// Theta (reading A23): Theta_ri = (-1)^popcount(s_r & i) d_i / sqrt(k), i the GLOBAL row of X, s_r the k
// sampled 48-bit Hadamard rows, d_i = +-1 from bit 0 of Philox(i, 0, domain 6).  Split i = 1024 h + l and
// s_r = 1024 sh_r + sl_r.  Then popcount(s_r & i) = popcount(sh_r & h) + popcount(sl_r & l), so
//     P_rc sqrt(k) = sum_h (-1)^popcount(sh_r & h)  Y_h[sl_r][c],
//     Y_h[t][c]    = sum_{l < 1024} (-1)^popcount(t & l) d_{1024 h + l} X[1024 h + l][c]
// i.e. Y_h is the 1024-point Walsh-Hadamard transform of the sign-flipped row block h (rows outside this rank's
// X are zero), evaluated at t, and each block adds ONE gathered, signed row of Y_h to every row of P.
// Cost per element of X: log2(1024) = 10 adds for the transform + k / 1024 for the gather, against 2 k for the
// dense product (k = 512: 10.5 vs 1024).  Blocks are aligned to global multiples of 1024 rows, so any row
// partition (any row_offset) gives the same block transforms and the ranks' partial sketches just add.
//
// One CTA (256 threads) owns 8 columns and a contiguous range of blocks (grid = column tiles x row splits):
//   * 32 TMA boxes (32 rows x 8 columns; out-of-range rows and columns arrive as zeros, also for the negative
//     start row of a rank's first, partial block) fill a stage of a 2 (fp64) / 3 (fp32) deep ring, refilled as soon
//     as pass 1 has read it;
//   * pass 1: thread (c, L) holds rows 32 q + L, q = 0..31, of column c in registers, applies d and the
//     radix-32 butterfly over q (row bits 5..9);  pass 2: thread (c, H) holds rows 32 H + q and transforms row
//     bits 0..4.  Both passes read and write shared memory without bank conflicts (per 32-row group the row
//     index is XOR-swizzled by the group's parity); everything is fp64;
//   * gather: thread (c, r mod 32) adds +-Y[sl_r][c] into its register accumulators for rows r = (t / 8) + 32 u
//     with a TwoSum compensation (the same "minor operations in higher precision" as the DMMA sketch);
//   * at the end the CTA writes its k x 8 partial and compensation; sketch_reduce_kernel sums the splits.
#include <cuda.h>
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include "internal.cuh"
#include "tcgen05.cuh"
#include "theta.cuh"

namespace rcq {

constexpr int FW_B = 1024;             // rows per transform block
constexpr int FW_CT = 8;               // columns per CTA
constexpr int FW_T = 32 * FW_CT;       // threads
constexpr int FW_GS = 32 * FW_CT + 16; // doubles per 32-row group of the fp64 buffers (2176 B: 128-byte multiple)
constexpr int FW_KMAX = 1024;

template <typename TX>
struct FwCfg {
  static constexpr bool F64 = sizeof(TX) == 8;
  static constexpr int GS_IN = 32 * FW_CT;                              // elements per 32-row group of a stage (one TMA box)
  static constexpr int STAGE_BYTES = 32 * GS_IN * (int)sizeof(TX);      // fp64 65536, fp32 32768
  static constexpr int NST = F64 ? 2 : 3;                               // a stage is refilled right after pass 1 has read it
  static constexpr int Y_BYTES = 32 * FW_GS * 8;                        // the fp64 work buffer of the block being transformed
  static constexpr size_t SMEM = (size_t)NST * STAGE_BYTES + Y_BYTES + FW_KMAX * 8 + 32 * 4 + NST * 8 + 256;
  static_assert(SMEM <= 232448, "shared memory");
};

__device__ __forceinline__ void fwht32(double (&v)[32]) {
#pragma unroll
  for (int h = 1; h < 32; h <<= 1)
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (!(i & h)) {
        const double a = v[i], b = v[i | h];
        v[i] = a + b;
        v[i | h] = a - b;
      }
}

// physical offset (doubles) of row t (0..1023) of the transformed block, column 0
__device__ __forceinline__ int fw_phys(int t) { return (t >> 5) * FW_GS + (((t & 31) ^ ((t >> 5) & 1)) << 3); }

template <typename TX, int KU>
__global__ void __launch_bounds__(FW_T, 1)
srht_fwht_kernel(const __grid_constant__ CUtensorMap xmap, const uint64_t* __restrict__ srows, int k, int k_total,
                 int r0, int n, uint64_t seed, int64_t row_offset, int64_t hb0, int64_t nblk, int64_t blocks_per_split,
                 double* __restrict__ part, double* __restrict__ partc) {
  // this launch computes sketch rows r0 .. r0 + k - 1 (k <= 1024) of the k_total rows
  using Cf = FwCfg<TX>;
  extern __shared__ __align__(1024) unsigned char sm[];
  TX* stage = reinterpret_cast<TX*>(sm);                                                 // [NST][32][GS_IN]
  double* y = reinterpret_cast<double*>(sm + (size_t)Cf::NST * Cf::STAGE_BYTES);
  uint64_t* s_sm = reinterpret_cast<uint64_t*>(sm + (size_t)Cf::NST * Cf::STAGE_BYTES + Cf::Y_BYTES);   // [FW_KMAX]
  uint32_t* dbits = reinterpret_cast<uint32_t*>(s_sm + FW_KMAX);                          // [32] bit q of word g: d of row 32 q + g
  uint64_t* full = reinterpret_cast<uint64_t*>(dbits + 32);                              // [NST]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int c = tid & (FW_CT - 1), g = tid >> 3;          // column of the tile; L (pass 1), H (pass 2), r mod 32 (gather)
  const int col0 = blockIdx.x * FW_CT;
  const int64_t b_begin = blockIdx.y * blocks_per_split;
  const int64_t b_end = min(nblk, b_begin + blocks_per_split);
  const int nb = b_end > b_begin ? (int)(b_end - b_begin) : 0;

  // per sketch row: (sh_r << 16) | (offset of Y[sl_r] in 8-double units)
  for (int r = tid; r < k; r += FW_T) {
    const uint64_t sr = srows[r0 + r];
    s_sm[r] = ((sr >> 10) << 16) | (uint64_t)(fw_phys((int)(sr & (FW_B - 1))) >> 3);
  }
  if (tid == 0) {
    for (int s = 0; s < Cf::NST; ++s) tc::mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // stage loads by warp 0: lane j brings rows 32 j .. 32 j + 31 of the block (one box)
  auto load_block = [&](int b) {
    const int s = b % Cf::NST;
    const int64_t lrow0 = (hb0 + b_begin + b) * FW_B - row_offset;       // local row of the block's first row (may be < 0)
    if (lane == 0) tc::mbar_arrive_tx(&full[s], (uint32_t)(32 * 32 * FW_CT * sizeof(TX)));
    __syncwarp();
    tc::tma_load_2d(stage + (size_t)s * 32 * Cf::GS_IN + (size_t)lane * Cf::GS_IN, &xmap, col0, (int)(lrow0 + 32 * lane),
                    &full[s]);
  };
  if (warp == 0)
    for (int b = 0; b < Cf::NST && b < nb; ++b) load_block(b);

  // fp64 X: TwoSum-compensated block sums (the DMMA sketch's "higher precision", reading A15); fp32 X: a plain
  // fp64 chain already has u_f ~ 1e-13 << u_32 (same reading), so no compensation registers or adds
  constexpr int KC_ = Cf::F64 ? KU : 1;
  double acc[KU], accc[KC_];
#pragma unroll
  for (int u = 0; u < KU; ++u) acc[u] = 0.0;
#pragma unroll
  for (int u = 0; u < KC_; ++u) accc[u] = 0.0;

  for (int b = 0; b < nb; ++b) {
    const int s = b % Cf::NST;
    const int64_t hb = hb0 + b_begin + b;                                 // global block index h
    // d_i of the block's 1024 rows: lane q of warp w takes rows 32 q + g for g = w + 8 a, so the warp's ballot is
    // the sign word of pass-1 thread row g (bit q = d of row 32 q + g)
#pragma unroll
    for (int a = 0; a < FW_B / FW_T; ++a) {
      const int gg = warp + 8 * a;
      const uint32_t neg = philox_at(seed, (uint64_t)(hb * FW_B + 32 * lane + gg), 0u, kDomainSrhtD).x & 1u;
      const uint32_t w = __ballot_sync(0xffffffffu, neg);
      if (lane == 0) dbits[gg] = w;
    }
    tc::mbar_wait(&full[s], (uint32_t)((b / Cf::NST) & 1));
    __syncthreads();                                                      // dbits visible; previous gather done with ybuf
    double v[32];
    {
      const TX* in = stage + (size_t)s * 32 * Cf::GS_IN + tid;            // element (row 32 q + g, column c) at q GS_IN + 8 g + c
      const uint32_t dw = dbits[g];
#pragma unroll
      for (int q = 0; q < 32; ++q) {                                      // x d: the sign bit of the double flipped
        const double x = (double)in[q * Cf::GS_IN];
        v[q] = __hiloint2double(__double2hiint(x) ^ (int)((dw << (31 - q)) & 0x80000000u), __double2loint(x));
      }
    }
    fwht32(v);                                                            // row bits 5..9
#pragma unroll
    for (int q = 0; q < 32; ++q) y[q * FW_GS + ((g ^ (q & 1)) << 3) + c] = v[q];   // row 32 q + g, swizzled
    __syncthreads();
    if (warp == 0 && b + Cf::NST < nb) load_block(b + Cf::NST);           // every thread has read the stage: refill it
#pragma unroll
    for (int q = 0; q < 32; ++q) v[q] = y[g * FW_GS + ((q ^ (g & 1)) << 3) + c];  // row 32 g + q
    fwht32(v);                                                            // row bits 0..4
#pragma unroll
    for (int q = 0; q < 32; ++q) y[g * FW_GS + ((q ^ (g & 1)) << 3) + c] = v[q];
    __syncthreads();
    // gather: P_r += (-1)^popcount(sh_r & h) Y[sl_r]
#pragma unroll
    for (int u = 0; u < KU; ++u) {
      const int r = g + 32 * u;
      if (r < k) {
        const uint64_t sr = s_sm[r];
        double yv = y[(((int)sr & 0xFFFF) << 3) + c];
        if (__popcll((sr >> 16) & (uint64_t)hb) & 1) yv = -yv;
        if constexpr (Cf::F64) {
          const double t = acc[u] + yv;
          const double bb = t - acc[u];
          accc[u] += (acc[u] - (t - bb)) + (yv - bb);
          acc[u] = t;
        } else {
          acc[u] += yv;
        }
      }
    }
  }
  const size_t kn = (size_t)k_total * n;
#pragma unroll
  for (int u = 0; u < KU; ++u) {
    const int r = g + 32 * u;
    if (r < k && col0 + c < n) {
      part[blockIdx.y * kn + (size_t)(r0 + r) * n + col0 + c] = acc[u];
      partc[blockIdx.y * kn + (size_t)(r0 + r) * n + col0 + c] = Cf::F64 ? accc[u % KC_] : 0.0;
    }
  }
}

// Measured on B200 (tools/ab_time.py --sketch srht, ms per sketch; dense = the +-1 E tile on tcgen05):
//   C4 shape (fp32, n = 64, k = 128): transform 9.1, dense 4.9      C2 shape (fp32, n = 100, k = 200): 0.32 vs 0.41
//   C3 shape (fp64, n = 256, k = 512): 13.9 vs 26.4                 C5 shape (fp64, n = 1024, k = 2048): 43.3 vs 1070
// The transform's cost does not grow with k (10 + k / 1024 adds per element), the dense product's does, so the
// transform serves k > 128 (more than one Theta tile of the dense kernel); RCHOLQR_SRHT_FWHT=1 / RCHOLQR_SRHT_DENSE=1
// force one or the other.  k > 1024 runs one launch per 1024 sketch rows (the accumulators live in registers).
bool srht_fwht_applicable(int k) {
  if (getenv("RCHOLQR_SRHT_DENSE")) return false;
  return k >= 1 && (k > 128 || getenv("RCHOLQR_SRHT_FWHT"));
}

int srht_fwht_splits(int n, int sms) { return std::max(1, 2 * sms / ((n + FW_CT - 1) / FW_CT)); }

using EncodeTiledFn3 = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// part / partc: [splits_max][k][n]; *splits_used receives the number of row splits written (the caller reduces
// exactly those).  cudaErrorNotSupported: X not TMA-addressable (base or row pitch not 16-byte aligned) or too tall.
cudaError_t launch_srht_fwht(const void* X, int dtype, int64_t m, int n, int64_t ldx, int64_t row_offset, int k,
                             uint64_t seed, const uint64_t* srht_s, int splits_max, double* part, double* partc,
                             int* splits_used, cudaStream_t st) {
  const size_t es = dtype == RCHOLQR_F64 ? 8 : 4;
  if (m <= 0 || m > (int64_t)INT32_MAX - 2 * FW_B || ((uintptr_t)X % 16) != 0 || ((size_t)ldx * es) % 16 != 0)
    return cudaErrorNotSupported;
  static EncodeTiledFn3 enc = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn3>(p);
  }();
  if (!enc) return cudaErrorNotSupported;
  CUtensorMap map;
  const cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)m};
  const cuuint64_t strides[1] = {(cuuint64_t)ldx * es};
  const cuuint32_t box[2] = {(cuuint32_t)FW_CT, 32u}, estr[2] = {1, 1};
  if (enc(&map, dtype == RCHOLQR_F64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
          const_cast<void*>(X), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorNotSupported;
  const int64_t hb0 = row_offset / FW_B;                                  // first global block touching this rank's rows
  const int64_t nblk = (row_offset + m - 1) / FW_B - hb0 + 1;
  const int splits = (int)std::min<int64_t>(std::max(1, splits_max), nblk);
  const int64_t bps = (nblk + splits - 1) / splits;
  const dim3 grid((unsigned)((n + FW_CT - 1) / FW_CT), (unsigned)splits);
  int r0 = 0, kc = 0;
  auto go = [&](auto kern, size_t smem) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, FW_T, smem, st>>>(map, srht_s, kc, k, r0, n, seed, row_offset, hb0, nblk, bps, part, partc);
    return cudaGetLastError();
  };
  auto pick = [&](auto* tag) -> cudaError_t {
    using TX = std::remove_pointer_t<decltype(tag)>;
    const size_t smem = FwCfg<TX>::SMEM;
    if (kc <= 128) return go(srht_fwht_kernel<TX, 4>, smem);
    if (kc <= 256) return go(srht_fwht_kernel<TX, 8>, smem);
    if (kc <= 512) return go(srht_fwht_kernel<TX, 16>, smem);
    return go(srht_fwht_kernel<TX, 32>, smem);
  };
  *splits_used = splits;
  for (r0 = 0; r0 < k; r0 += FW_KMAX) {                                   // one launch per 1024 sketch rows
    kc = std::min(FW_KMAX, k - r0);
    const cudaError_t e = dtype == RCHOLQR_F64 ? pick((double*)nullptr) : pick((float*)nullptr);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace rcq
