// internal.cuh -- plan layout and launch interfaces shared by the library's translation units.
#pragma once
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>
#include "rcholqr.h"

namespace rcq {

// Ablation switches of the tensor-core kernels (role work switched off, RCHOLQR_*_DEBUG): compiled in only
// with -DRCHOLQR_ABLATION (tools/ experiments); production builds fold them to 0 and drop the branches.
#ifdef RCHOLQR_ABLATION
constexpr bool kAblation = true;
#else
constexpr bool kAblation = false;
#endif

// Per-role event timeline of CTA 0 (clock64), ablation builds only: trace(role, tile, event) for the first
// kTraceTiles tiles; read back with rcholqr_trace_read (tools/trace_*.py).  Compiled out of production.
constexpr int kTraceRoles = 8, kTraceTiles = 64, kTraceEvents = 8;
#ifdef RCHOLQR_ABLATION
// one buffer per translation unit (no relocatable device code); each traced TU defines a reader below
static __device__ long long g_trace[kTraceRoles * kTraceTiles * kTraceEvents];
#define RCQ_TRACE_READER(name)                                                                                \
  int name(void* host) {                                                                                        \
    static long long zero[kTraceRoles * kTraceTiles * kTraceEvents];                                            \
    if (cudaDeviceSynchronize() != cudaSuccess || cudaMemcpyFromSymbol(host, g_trace, sizeof(zero)) != cudaSuccess) \
      return -2;                                                                                                \
    return cudaMemcpyToSymbol(g_trace, zero, sizeof(zero)) == cudaSuccess ? 0 : -3;                             \
  }
int trace_read_solve(void* host);
int trace_read_sketch(void* host);
#endif
__device__ __forceinline__ void trace(int role, int tile, int ev) {
#ifdef RCHOLQR_ABLATION
  if (blockIdx.x == 0 && tile < kTraceTiles) g_trace[(role * kTraceTiles + tile) * kTraceEvents + ev] = clock64();
#else
  (void)role; (void)tile; (void)ev;
#endif
}

// Status bits written by kernels into the plan's device status word (0 = OK).
enum : int { kStNonfinite = 1, kStSingular = 2 };
// Which kernels served the last call (rcholqr_last_path; the bits are RCHOLQR_PATH_* of rcholqr.h).
enum : unsigned { kPathSketchTC = RCHOLQR_PATH_SKETCH_TC, kPathSketchPresplit = RCHOLQR_PATH_SKETCH_PRESPLIT,
                  kPathSketchCudaCore = RCHOLQR_PATH_SKETCH_CUDA_CORE, kPathSketchFallback = RCHOLQR_PATH_SKETCH_FALLBACK,
                  kPathSolveTC = RCHOLQR_PATH_SOLVE_TC, kPathSolveDmma = RCHOLQR_PATH_SOLVE_DMMA,
                  kPathColmajorNative = RCHOLQR_PATH_COLMAJOR_NATIVE, kPathSketchFwht = RCHOLQR_PATH_SKETCH_FWHT };

// One FP64 tensor-core MMA: D(16x8) += A(16x4) B(4x8)  (DMMA on sm_100a; tcgen05 has no f64 kind).
// Fragments (PTX ISA, mma.m16n8k4 .f64): g = lane/4, t = lane%4;
//   A: a0 = A[g][t], a1 = A[g+8][t];  B: b0 = B[t][g];  D: d0,d1 = D[g][2t..2t+1], d2,d3 = D[g+8][..].
__device__ __forceinline__ void dmma_16x8x4(double (&d)[4], double a0, double a1, double b) {
  asm("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a0), "d"(a1), "d"(b));
}

// ---- launch configurations chosen at plan creation ----
enum SketchKind : int { kSketchG48x24 = 0, kSketchG128x64 = 1, kSketchG112x104 = 2, kSketchG64x64 = 3,
                        kSketchSparse = 10, kSketchSparseReg = 11 };
// tcgen05 int8 sparse sketch (sketch_tc.cu): exact int32 accumulation bound on rows per CTA
constexpr int64_t kSparseTcMaxRows = 8 * 1024 * 1024;
bool sparse_tc_applicable(int k, int n, int zeta);
bool sparse_tc_aligned(const void* X, int dtype, int64_t m, int64_t ldx);
cudaError_t launch_sparse_tc(const void* X, int dtype, int64_t m, int n, int64_t ldx, int64_t row_offset, int k,
                             int zeta, uint64_t seed, int splits, int64_t rows_per_split, double* part, int* overflow,
                             cudaStream_t st, const uint64_t* srht_s = nullptr, double* cs_part = nullptr,
                             bool colmajor = false);
enum TrsmKind : int { kTrsm64x24 = 0, kTrsm128x64 = 1, kTrsm128x112 = 2, kTrsm128x128 = 3 };
enum QrKind : int { kQrSmem = 0, kQrGlobal = 1, kQrBlocked = 2 };

struct SketchLaunch {
  int kind;
  int KT, NT, threads;   // tile of P per CTA (sparse: NT = columns per CTA, KT = k)
  int tiles_k, tiles_n, splits;
  size_t smem;
  // Gaussian: tcgen05 digit sketch (sketch_gtc.cu) in front of the DMMA kernel described above
  int tc = 0, tc_tiles_k = 0, tc_tiles_n = 0, tc_splits = 0;
  // Rademacher Theta (reading A22): the DMMA kernel above draws +-1 instead of N(0,1); rad_tc: the
  // tcgen05 int8 kernel of sketch_tc.cu with a dense E tile in front of it (n <= 64, k <= 512)
  int rad = 0, rad_tc = 0, rad_splits = 0;   // rad: 1 = Rademacher, 2 = SRHT (reading A23)
  // sparse-sign: the tcgen05 kernel of sketch_tc.cu in front of the CUDA-core kind above (its guarded fallback)
  int sp_tc = 0;
  const uint64_t* srht_s = nullptr;          // SRHT: the k sampled Hadamard rows (plan-owned device array)
  // SRHT by the blocked fast Walsh-Hadamard transform (srht_fwht.cu; k <= 1024), in front of the dense kernels
  int fwht = 0, fwht_splits = 0;
  int max_splits() const {
    int s = tc && tc_splits > splits ? tc_splits : splits;
    s = rad_tc && rad_splits > s ? rad_splits : s;
    return fwht && fwht_splits > s ? fwht_splits : s;
  }
};
int gauss_tc_kt(int dtype);   // Theta rows per tcgen05 Gaussian-sketch tile (X columns per tile: 128)
bool gauss_tc_aligned(const void* X, int dtype, int n, int64_t ldx);
cudaError_t launch_gauss_tc(const void* X, int dtype, int64_t m, int n, int64_t ldx, int64_t row_offset, int k,
                            uint64_t seed, int tiles_k, int tiles_n, int splits, int64_t rows_per_split,
                            double* part, double* partc, int* overflow, cudaStream_t st);
// pre-split variant: X digit planes written once to a workspace of gauss_tcp_workspace() bytes
size_t gauss_tcp_workspace(int64_t m, int n, int dtype, int splits);
size_t gauss_tcp_chunk_workspace(int64_t m, int n, int dtype, int splits);   // capped at kXdigCapBytes
// cs_part (optional, kXdigSplitBlocks x n doubles): per-CTA column sums of squares of X from the
// digit-split pass (Alg. 7's D), reduced by the caller with launch_reduce(.., kXdigSplitBlocks, ..)
constexpr int kXdigSplitBlocks = 148 * 8;
cudaError_t launch_colsum_reduce(const double* part, int rows, int n, double* out, int* status, cudaStream_t st);
cudaError_t launch_gauss_tcp(const void* X, int dtype, int64_t m, int n, int64_t ldx, int64_t row_offset, int k,
                             uint64_t seed, int tiles_k, int tiles_n, int splits, double* part, double* partc,
                             int* overflow, void* ws, size_t ws_bytes, cudaStream_t st, double* cs_part = nullptr,
                             bool colmajor = false);
constexpr size_t kXdigCapBytes = (size_t)4 << 30;   // largest pre-split digit workspace a plan allocates
struct TrsmLaunch {
  int kind;
  int TM, NT, threads, tiles_n;
  size_t smem;
};

// Host-side launchers (defined in sketch.cu / qr.cu / trsm.cu).
SketchLaunch plan_sketch(int k, int n, int dtype, int sketch, int zeta, int sms, size_t smem_optin);
bool srht_fwht_applicable(int k);
int srht_fwht_splits(int n, int sms);
cudaError_t launch_srht_fwht(const void* X, int dtype, int64_t m, int n, int64_t ldx, int64_t row_offset, int k,
                             uint64_t seed, const uint64_t* srht_s, int splits_max, double* part, double* partc,
                             int* splits_used, cudaStream_t st);
double gauss_tc_min_work();   // 2kmn below which the Gaussian sketch takes the single DMMA kernel (launch-bound sizes)
cudaError_t launch_sketch(const SketchLaunch& L, const void* X, int dtype, int64_t m, int n, int64_t ldx,
                          int64_t row_offset, int k, int zeta, uint64_t seed, double* part, double* partc, double* P,
                          int* status, int* flag, void* xdig, size_t xdig_bytes, cudaStream_t st, cudaEvent_t ev_mid,
                          int k_first = 0, unsigned* path = nullptr, int* flag_seen = nullptr,
                          double* cs_part = nullptr, double* cs_out = nullptr, bool* cs_done = nullptr,
                          bool colmajor = false);
TrsmLaunch plan_trsm(int n, int dtype, size_t smem_optin);
cudaError_t launch_tri_inverse(const double* R, int n, double* W, int* status, cudaStream_t st);
cudaError_t launch_trsm(const TrsmLaunch& L, const void* X, int dtype, int64_t m, int n, int64_t ldx,
                        const double* W, void* Q, int64_t ldq, const int* status, cudaStream_t st);
int plan_qr(int k, int n, size_t smem_optin);
cudaError_t launch_qr(int kind, const double* P, int k, int n, double* R, double* Awork, double* diag,
                      double* tau, double* qr_ws, int* status, cudaStream_t st);
// blocked Householder (qr_blocked.cu) for sketches the single-CTA kernels do not fit
size_t qr_blocked_workspace(int k, int n);
cudaError_t launch_qr_blocked(const double* P, int k, int n, double* R, double* A, double* diag, double* tau,
                              double* ws, int* status, cudaStream_t st);
cudaError_t launch_form_s(const double* Awork, const double* tau, const double* diag, int k, int n,
                          double* S, const int* status, cudaStream_t st);
cudaError_t launch_theta_export(uint64_t seed, int k, int sketch, int zeta, int64_t row_offset, int64_t m,
                                float* Z, int32_t* rows, int8_t* signs, cudaStream_t st,
                                const uint64_t* srht_s = nullptr);
cudaError_t launch_check_diag(const double* R, int n, int* status, cudaStream_t st);
// blocked substitution (default tall solve for n <= 128): M = [-R_{<J,J}; Winv_JJ] packed
int trsm_pair_count(int n, size_t smem_optin);                 // warp pairs per CTA; 0 = not applicable
cudaError_t launch_trsm_pairs(int pairs, const void* X, int dtype, int64_t m, int n, int64_t ldx, const double* M,
                              void* Q, int64_t ldq, const int* status, int sms, cudaStream_t st);
// 128 < n <= 256: warp-pair blocked substitution with M streamed per column block (trsm.cu)
bool trsm_mstream_applicable(int n, size_t smem_optin);
cudaError_t launch_trsm_mstream(const void* X, int dtype, int64_t m, int n, int64_t ldx, const double* M, void* Q,
                                int64_t ldq, const int* status, int sms, cudaStream_t st);
cudaError_t launch_tri_prep_blocked(const double* R, int n, double* M, int* status, cudaStream_t st, int tb = 32,
                                    int npad = 0);
// fp64 DMMA GEMM C = C0 + A B (gemm.cu), used by the streamed blocked solve (n > 128, fp64 X)
cudaError_t launch_gemm_f64(const double* A, int64_t lda, const double* B, int64_t ldb, const double* C0,
                            int64_t ldc0, double* C, int64_t ldc, int64_t m, int N, int K, bool tri_b,
                            const int* status, cudaStream_t st);
// tcgen05 int8 digit solve for fp32 X, n <= 64 (solve_tc.cu): Q = X fl64(R^{-1})
bool solve_tc_applicable(int dtype, int n);
bool solve_tc_supported(const void* X, int64_t m, int64_t ldx, const void* Q, int64_t ldq);
size_t solve_tc_workspace();
cudaError_t launch_solve_tc(const double* Winv, int n, const float* X, int64_t m, int64_t ldx, float* Q, int64_t ldq,
                            void* ws, int* status, int sms, cudaStream_t st, bool colmajor = false);
// RCholeskyQR2 (rcqr2.cu): Gram A = Q^T Q, Cholesky R', R' R
cudaError_t launch_reduce(const double* part, int splits, int64_t kn, double scale, double* P, int* status,
                          cudaStream_t st);
int gram_splits(int n, int sms);
cudaError_t launch_gram(const void* Q, int dtype, int64_t m, int n, int64_t ldq, int splits, double* part, double* A,
                        int* status, cudaStream_t st);
cudaError_t launch_cholesky(const double* A, int n, double* W, double* Rp, int* status, cudaStream_t st);
cudaError_t launch_trmm_upper(const double* U, const double* V, int n, double* out, const int* status,
                              cudaStream_t st);
cudaError_t launch_trmm_trap(const double* U, int r, const double* V, int n, double* out, const int* status,
                             cudaStream_t st);
// reduced RCholeskyQR (reduced.cu): Z = Y R^{-1} for the small l x n extract Y, row-wise substitution
cudaError_t launch_rowsub(const double* Y, int64_t l, int n, const double* R, double* Z, const int* status,
                          cudaStream_t st);
// rank-revealing RCholeskyQR (rrqr.cu)
int colsq_splits(int n, int sms);
cudaError_t launch_colsq(const void* X, int dtype, int64_t m, int n, int64_t ldx, int splits, double* part,
                         double* out, int* status, cudaStream_t st);
cudaError_t launch_rr_normalize(const double* buf, int k, int n, double* Pn, double* d, cudaStream_t st);
cudaError_t launch_qrcp(const double* Pn, int k, int n, double* A, int* perm, cudaStream_t st);
cudaError_t launch_rr_gather(const double* Pn, int k, int n, const int* perm, double* Pg, cudaStream_t st);
cudaError_t launch_rank(const double* R, int n, double tau, int rank_fixed, int* rank, double* sigma, cudaStream_t st);
cudaError_t launch_strong(const double* R, int n, int r, double* W, double* out_v, int* out_i, cudaStream_t st);
cudaError_t launch_rr_finalize(const double* Rf, int n, int r, const double* d, const int* perm, double* Rout,
                               double* R11, cudaStream_t st);
cudaError_t launch_gather_x(const void* X, int dtype, int64_t m, int64_t ldx, const int* perm, int r, void* Xr,
                            int sms, cudaStream_t st);
// out (cols x rows, ld ldo) = in^T (rows x cols, ld ldi), element size es (reduced.cu)
cudaError_t launch_transpose(const void* in, int64_t rows, int64_t cols, int64_t ldi, void* out, int64_t ldo,
                             size_t es, cudaStream_t st);

}  // namespace rcq
