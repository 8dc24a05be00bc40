/*
 * rcholqr.h -- C ABI of the B200 (sm_100a) direct randomized Cholesky QR library.
 *
 * Method: RCholeskyQR, Algorithm 2 of O. Balabanov, "Randomized Cholesky QR factorizations",
 * arXiv 2210.09953:
 *     1. P <- Theta X  sketch, fp64 accumulation
 *     2. [R, S] <- QR(P)  fp64 Householder
 *     3. Q <- X R^{-1}  tall triangular solve
 * Multi-GPU ("only one global synchronization", reduction operator = addition):
 * X is row-partitioned, each rank sketches its rows with Theta keyed by the GLOBAL row index,
 * one in-place NCCL all-reduce (sum) of the k x n sketch, R computed redundantly on every rank,
 * Q solved locally.
 *
 * Conventions (all entry points):
 *   - C linkage, no exceptions cross the boundary; every call returns an rcholqr_status.
 *   - Matrices are ROW-MAJOR with an explicit leading dimension (elements, >= number of columns).
 *     X and Q: m_local x n in the plan's dtype; P, S: k x n fp64; R: n x n fp64 upper triangular
 *     (zeros below the diagonal), diag(R) >= 0 (reading A5).
 *   - Pointers passed to rcholqr_factor / _sketch / _small_qr / _tri_solve / _theta_export are
 *     CUDA DEVICE pointers on the plan's device, owned by the caller; the library never frees
 *     them.  rcholqr_factor_host takes HOST pointers (pinned memory recommended) and performs the
 *     host<->device copies itself.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  Work is
 *     stream-ordered; functions documented "synchronous" block the host until the stream has
 *     drained and return a definitive numerical status.
 *   - Q must not alias X.  S may be NULL (not requested).
 *   - A plan is not thread-safe; distinct plans are independent.
 *
 * Theta (readings A1-A4): Philox4x32-10, key = (lo32(seed),
 * hi32(seed)), counter = (lo32(i), hi32(i), q, domain), i = global X row.  Gaussian: entries
 * z/sqrt(k), z from a fixed fp32 Box-Muller transform ("i.i.d. Gaussian ...
 * scaled by sqrt(1/k)").  Sparse-sign: nnz_per_col nonzeros +-1/sqrt(nnz_per_col) per column,
 * one per block of k/nnz_per_col rows (BASELINE.json config 4; OSNAP block construction).
 * Rademacher (reading A22): +-1/sqrt(k), sign = bit (r mod 32) of word ((r mod 128)/32) of the
 * Philox call (i, r/128, domain 5).  SRHT (reading A23): sqrt(m'/k) R H D with m' = 2^48, i.e.
 * (-1)^popcount(s_r & i) d_i / sqrt(k); d_i from Philox(i, 0, domain 6), the k distinct rows s_r from
 * Philox(r, attempt, domain 7) (computed on the host when the plan is created).
 */
#ifndef RCHOLQR_H
#define RCHOLQR_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RCHOLQR_VERSION 100  /* 1.0.0 */

typedef struct rcholqr_plan_s* rcholqr_plan;

typedef enum { RCHOLQR_F64 = 0, RCHOLQR_F32 = 1 } rcholqr_dtype;          /* dtype of X and Q */
typedef enum {
  RCHOLQR_GAUSSIAN = 0, RCHOLQR_SPARSE_SIGN = 1, RCHOLQR_RADEMACHER = 2, RCHOLQR_SRHT = 3
} rcholqr_sketch_kind;

typedef enum {
  RCHOLQR_OK = 0,
  RCHOLQR_E_INVALID = 1,   /* null pointer, bad enum, ld < n, Q aliases X, m_local < 0        */
  RCHOLQR_E_SHAPE = 2,     /* n < 1, k < n, sparse: nnz < 1 or k % nnz != 0                    */
  RCHOLQR_E_NONFINITE = 3, /* the (reduced) sketch P contains NaN/Inf (non-finite X / overflow) */
  RCHOLQR_E_SINGULAR = 4,  /* some R_jj == 0 or non-finite: X not numerically full rank
                              (eq:condstab); Q is left unwritten              */
  RCHOLQR_E_CUDA = 5,      /* a CUDA runtime call or kernel launch failed                       */
  RCHOLQR_E_NCCL = 6,      /* NCCL unavailable or a collective failed                           */
  RCHOLQR_E_NOMEM = 7      /* device or host allocation failed                                   */
} rcholqr_status;

typedef struct {
  int32_t n;            /* columns of X (>= 1)                                                  */
  int32_t k;            /* sketch rows (>= n); k = 2n is the paper's choice  */
  int32_t dtype;        /* rcholqr_dtype of X and Q                                             */
  int32_t sketch;       /* rcholqr_sketch_kind                                                    */
  int32_t nnz_per_col;  /* sparse-sign nonzeros per column of Theta (ignored otherwise)        */
  int32_t device;       /* CUDA device ordinal the plan lives on                                */
  uint64_t seed;        /* Theta seed                                                            */
  void* nccl_comm;      /* communicator from rcholqr_comm_create, or NULL for a single GPU.
                           Referenced, not owned.                                                */
} rcholqr_desc;

/* Create a plan: validates the descriptor, allocates the workspace (per-CTA sketch partials,
 * P, R^{-1}, QR scratch, status word) on desc->device.  *out is NULL on failure. */
rcholqr_status rcholqr_create(const rcholqr_desc* desc, rcholqr_plan* out);

/* Free the plan and its workspace (NULL is a no-op). */
rcholqr_status rcholqr_destroy(rcholqr_plan plan);

/* Whole Algorithm 2 on this rank's row block, SYNCHRONOUS.
 *   X        [device] m_local x n, leading dim ldx, rows row_offset .. row_offset+m_local-1 of
 *            the global X (row_offset keys Theta; 0 on a single GPU).  m_local may be 0.
 *   Q        [device] m_local x n output, leading dim ldq, X's dtype (computed in fp64, rounded
 *            once -- reading A7).  Not written if the status is E_SINGULAR / E_NONFINITE.
 *   R        [device] n x n fp64 output (identical bits on every rank).
 *   S        [device] k x n fp64 output or NULL (Alg. 2's orthonormal sketch of Q).
 * With a communicator every rank must call this (collective). */
rcholqr_status rcholqr_factor(rcholqr_plan plan, const void* X, int64_t m_local, int64_t row_offset,
                              int64_t ldx, void* Q, int64_t ldq, double* R, double* S, void* stream);

/* Same as rcholqr_factor but ASYNCHRONOUS: only argument/launch errors are reported; the
 * numerical status (E_NONFINITE / E_SINGULAR) is fetched later with rcholqr_query_status. */
rcholqr_status rcholqr_factor_async(rcholqr_plan plan, const void* X, int64_t m_local,
                                    int64_t row_offset, int64_t ldx, void* Q, int64_t ldq,
                                    double* R, double* S, void* stream);

/* Synchronize `stream` and return the numerical status of the last factor/sketch/QR call. */
rcholqr_status rcholqr_query_status(rcholqr_plan plan, void* stream);

/* End-to-end call with HOST buffers (X_host read, Q_host/R_host/S_host written): copies X to a
 * plan-owned device buffer, factors, copies Q, R (and S) back.  SYNCHRONOUS. */
rcholqr_status rcholqr_factor_host(rcholqr_plan plan, const void* X_host, int64_t m_local,
                                   int64_t row_offset, int64_t ldx, void* Q_host, int64_t ldq,
                                   double* R_host, double* S_host, void* stream);

/* rcholqr_factor_async replayed from a CUDA GRAPH: for launch-bound problems (BASELINE config C1, 10^4 x 20:
 * every kernel of the chain runs a few microseconds, so the ~8 launches are the cost; PAPER.md:163 expects
 * the small QR and the other small steps to "not have much impact").  The first call with a given argument
 * tuple (X, m_local, row_offset, ldx, Q, ldq, R, S) runs the chain directly and captures it; every later call
 * with the SAME tuple replays the captured graph with one launch on `stream`.  A different tuple re-captures
 * (one graph is cached per plan), and so does a call made after another entry point regrew the plan's
 * workspaces.  The buffers' CONTENTS may change between calls, their addresses may not.
 * Plans with an NCCL communicator, and plans with event timing enabled, launch directly (same results).
 * ASYNCHRONOUS like rcholqr_factor_async: numerical status through rcholqr_query_status. */
rcholqr_status rcholqr_factor_graph(rcholqr_plan plan, const void* X, int64_t m_local, int64_t row_offset,
                                    int64_t ldx, void* Q, int64_t ldq, double* R, double* S, void* stream);

/* Alg. 2 for COLUMN-MAJOR X and Q (element (i, j) at X[j * ldx + i], ldx >= m_local; the storage the
 * paper notes favours sketching).
 * NATIVE kernels (no transposes; the same two reads of X and one write of Q as the row-major path) serve
 * fp32 X with n <= 128 when X, Q and their column pitches are 16-byte aligned: the tcgen05 sketch kernels
 * (sparse-sign, Rademacher, SRHT, pre-split Gaussian) and the tcgen05 digit solve take column-major tiles
 * through their TMA tensor maps; rcholqr_last_path then reports RCHOLQR_PATH_COLMAJOR_NATIVE.  R, S and Q
 * are bitwise those of the row-major path on the transposed input.
 * Otherwise (fp64 X, n > 128, misaligned buffers, or a sketch kernel's headroom-overflow flag) a layout
 * ADAPTER runs: X is transposed on the GPU into a plan-owned row-major buffer, factored by the row-major
 * path and Q transposed back -- two extra passes over m_local x n.
 *   X [device] n columns of m_local rows, leading dim ldx;  Q [device] likewise, leading dim ldq;
 *   R, S, row_offset, stream: as for rcholqr_factor.  Q must not overlap X.  SYNCHRONOUS. */
rcholqr_status rcholqr_factor_colmajor(rcholqr_plan plan, const void* X, int64_t m_local, int64_t row_offset,
                                       int64_t ldx, void* Q, int64_t ldq, double* R, double* S, void* stream);

/* RCholeskyQR2 (Alg. 3, alg:RCQR2): RCholeskyQR (Alg. 2) followed by one
 * CholeskyQR pass, A = Q1^T Q1 (all-reduced over the communicator), R' = chol(A), R = R' R1,
 * Q = Q1 R'^{-1} -- an orthonormal Q factor (to O(n u)) and the QR factor R of X.
 *   X, m_local, row_offset, ldx, Q, ldq, stream: as for rcholqr_factor.
 *   R        [device] n x n fp64 output: R' R1 (upper triangular, positive diagonal).
 *   Rprime   [device] n x n fp64 output or NULL: R' (A = R'^T R').
 *   implicit 0: Q receives the explicit orthonormal factor Q1 R'^{-1} (a plan-owned m_local x n
 *              buffer holds Q1); nonzero: Q receives Q1 and Rprime (then required) R' -- the
 *              implicit form of PAPER.md:206 (products with Q as (Y Q1) R'^{-1}, Q1 (R'^{-1} Y)).
 * Status: as rcholqr_factor; E_SINGULAR also if A is not numerically positive definite.
 * SYNCHRONOUS.  With a communicator every rank must call this (collective; two all-reduces). */
rcholqr_status rcholqr_factor2(rcholqr_plan plan, const void* X, int64_t m_local, int64_t row_offset,
                               int64_t ldx, void* Q, int64_t ldq, double* R, double* Rprime, int32_t implicit,
                               void* stream);

/* Reduced RCholeskyQR (Alg. 5, alg:oneRCQR): the extract Z = L Q of the Q factor
 * without forming Q -- P = Theta X and Y = L X in step 1, [S, R] = QR(P), Z = Y R^{-1}.
 * L (l x m) is a Gaussian extractor from the normative Gaussian stream (reading A20):
 * L_ji = z(seed, global row i, l0 + j) / sqrt(l), l0 = k for a Gaussian plan (then [Theta; L] is
 * one (k + l)-row sketch and X is read ONCE), l0 = 0 for a sparse-sign plan (a second pass).
 *   X, m_local, row_offset, ldx, stream: as for rcholqr_factor.
 *   l  rows of L (>= 1; (k + l) n <= 2^28).
 *   Z  [device] l x n fp64 row-major output (required).
 *   R  [device] n x n fp64 output or NULL;  S [device] k x n fp64 or NULL (Alg. 5's S);
 *   Y  [device] l x n fp64 or NULL: the extract L X (after the all-reduce).
 * Status: E_INVALID (arguments), E_SHAPE, E_NONFINITE (P or Y), E_SINGULAR (Z not written).
 * Memory: the plan grows an (k + l) x n sketch workspace on the first call with a new l.
 * SYNCHRONOUS.  With a communicator every rank must call this (one all-reduce of [P; Y]); Z is
 * computed redundantly and is identical on every rank. */
rcholqr_status rcholqr_factor_reduced(rcholqr_plan plan, const void* X, int64_t m_local, int64_t row_offset,
                                      int64_t ldx, int32_t l, double* Z, double* R, double* S, double* Y,
                                      void* stream);

/* Rank-revealing RCholeskyQR (Alg. 7, alg:RRRCholeskyQR; reading A21):
 * X Pi ~= Q R with Q (m x r) well conditioned and R (r x n) upper trapezoidal, for numerically
 * rank-deficient X.  P = Theta X and D = diag(||X(:, j)||) in step 1 (one all-reduce of both),
 * P <- P D^{-1}, strong RRQR of P (column pivoting + Gu-Eisenstat swaps with parameter f),
 * r = min r with ||R(r+1:n, r+1:n)||_F <= tau ||R||_2, Q = (X Pi(:, 1:r)) R(1:r, 1:r)^{-1},
 * R <- R(1:r, :) Pi^T D Pi.
 *   X, m_local, row_offset, ldx, stream: as for rcholqr_factor.
 *   tau         truncation tolerance (>= 0; the paper uses ~1e-15 in fp64, ~1e-7 in fp32).
 *   f           strong-RRQR parameter (> 1; the paper's 1.5).
 *   rank_fixed  0: r from tau; > 0: r = min(rank_fixed, n) (fixed-rank strong RRQR).
 *   Q     [device] m_local x n buffer (ldq >= n); columns 0..r-1 receive Q (X's dtype), the rest untouched.
 *   R     [device] n x n fp64 (row-major, ld n): rows 0..r-1 = R(1:r, :) in permuted column order, rows
 *         r..n-1 zero.
 *   perm  [device] n int32: Pi as perm[j] = original column in position j.
 *   D     [device] n fp64 column norms or NULL;  S [device] k x n fp64 or NULL (columns 0..r-1 = S).
 *   rank_out, swaps_out [host] int32: r and the number of Gu-Eisenstat swaps (swaps_out may be NULL).
 * Status: E_INVALID (arguments, f <= 1, tau < 0), E_SHAPE (n > 1024), E_NONFINITE, E_SINGULAR if r = 0 (X = 0).
 * Memory: the plan allocates an O(k n) workspace on first use and an m_local x r gather buffer.
 * SYNCHRONOUS (the rank and each swap decision are read on the host).  With a communicator every
 * rank must call this (one all-reduce); Pi, r and R are identical on every rank. */
rcholqr_status rcholqr_factor_rr(rcholqr_plan plan, const void* X, int64_t m_local, int64_t row_offset,
                                 int64_t ldx, double tau, double f, int32_t rank_fixed, void* Q, int64_t ldq,
                                 double* R, int32_t* perm, double* D, double* S, int32_t* rank_out,
                                 int32_t* swaps_out, void* stream);

/* RRRCholeskyQR2 (RRRCholeskyQR "augmented with the classical CholeskyQR in exactly the same
 * way as done in RCholeskyQR2"): rcholqr_factor_rr gives (Q1, R1, Pi, r); then A = Q1^T Q1 (r x r,
 * all-reduced), R' = chol(A), R = R' R1, Q = Q1 R'^{-1} -- an ORTHONORMAL m x r Q with X Pi ~= Q R.
 *   Arguments as rcholqr_factor_rr (tau, f, rank_fixed, perm, D, rank_out, swaps_out); Rprime [device]
 *   r x r (ld r, n x n buffer) or NULL: R'.  R: rows 0..r-1 = R' R1 (permuted column order), the rest 0.
 * Status: as rcholqr_factor_rr; E_SINGULAR also if Q1^T Q1 is not numerically positive definite.
 * Memory: a plan-owned m_local x n buffer for Q1.  SYNCHRONOUS; collective with a communicator. */
rcholqr_status rcholqr_factor_rr2(rcholqr_plan plan, const void* X, int64_t m_local, int64_t row_offset,
                                  int64_t ldx, double tau, double f, int32_t rank_fixed, void* Q, int64_t ldq,
                                  double* R, double* Rprime, int32_t* perm, double* D, int32_t* rank_out,
                                  int32_t* swaps_out, void* stream);

/* ---- step-level entry points (same kernels as rcholqr_factor; used by the parity tests) ---- */

/* Step 1 (+ the all-reduce when the plan has a communicator): P = Theta X, k x n fp64 row-major
 * [device].  SYNCHRONOUS; returns E_NONFINITE if P has NaN/Inf. */
rcholqr_status rcholqr_sketch(rcholqr_plan plan, const void* X, int64_t m_local, int64_t row_offset,
                              int64_t ldx, double* P, void* stream);

/* Step 2: Householder QR of the k x n fp64 matrix P [device] -> R [device] (n x n), S [device]
 * (k x n) or NULL.  SYNCHRONOUS; returns E_SINGULAR on a zero/non-finite pivot (R still written). */
rcholqr_status rcholqr_small_qr(rcholqr_plan plan, const double* P, double* R, double* S,
                                void* stream);

/* Step 3: Q = X R^{-1} [device] for a given upper-triangular R [device].  SYNCHRONOUS. */
rcholqr_status rcholqr_tri_solve(rcholqr_plan plan, const void* X, int64_t m_local, int64_t ldx,
                                 const double* R, void* Q, int64_t ldq, void* stream);

/* Test export of Theta for global rows row_offset .. row_offset+m-1 [device buffers]:
 *   Gaussian:    Z (k x m fp32, row-major) = the unscaled N(0,1) draws z_ri (Theta = z/sqrt(k)).
 *   Sparse-sign: rows (m x nnz int32) and signs (m x nnz int8). Unused outputs may be NULL.
 * SYNCHRONOUS. */
rcholqr_status rcholqr_theta_export(uint64_t seed, int32_t k, int32_t sketch, int32_t nnz_per_col,
                                    int64_t row_offset, int64_t m, float* Z, int32_t* rows,
                                    int8_t* signs, void* stream);

/* ---- multi-GPU: library-owned NCCL communicator (NCCL is loaded on first use) ---- */

/* Write a 128-byte ncclUniqueId (call on rank 0, broadcast it with torch.distributed). */
rcholqr_status rcholqr_comm_unique_id(uint8_t id_out[128]);
/* ncclCommInitRank on `device`; *comm receives an opaque ncclComm_t. Collective over nranks. */
rcholqr_status rcholqr_comm_create(const uint8_t id[128], int32_t nranks, int32_t rank,
                                   int32_t device, void** comm);
rcholqr_status rcholqr_comm_destroy(void* comm);

/* ---- introspection ---- */
const char* rcholqr_strerror(rcholqr_status s);
int32_t rcholqr_version(void);
/* Number of kernels rcholqr_factor_async launches per call for this plan and m_local. */
int32_t rcholqr_launches_per_factor(rcholqr_plan plan, int64_t m_local);
/* Per-step device times (ms) of the last factor call when timing is enabled:
 * out[0] sketch, out[1] partial reduce, out[2] all-reduce, out[3] small QR, out[4] tri prep,
 * out[5] tall solve.  Enable with rcholqr_set_timing(plan, 1) (adds events, no host syncs). */
rcholqr_status rcholqr_set_timing(rcholqr_plan plan, int32_t enable);
rcholqr_status rcholqr_last_timings(rcholqr_plan plan, float out_ms[6]);

/* Which kernels served the last sketch / factor / solve call on this plan (a bit set; the parity
 * tests assert with it that the tcgen05 kernels, not the guarded CUDA-core fallbacks, computed a
 * result).  Bits accumulate over the steps of one call and are cleared when the next call starts:
 *   SKETCH_TC        a tcgen05 sketch kernel ran (Gaussian digit, sparse-sign or dense +-1 E tile)
 *   SKETCH_PRESPLIT  the Gaussian sketch took X from pre-split digit planes (xdig_split_kernel)
 *   SKETCH_CUDA_CORE the sketch was computed by a CUDA-core / DMMA kernel alone (no tcgen05 kernel)
 *   SKETCH_FALLBACK  a tcgen05 sketch raised its headroom-overflow flag and the guarded DMMA /
 *                    CUDA-core kernel recomputed the partials (PAPER.md:423's u_f is kept either way)
 *   SOLVE_TC         the tall solve ran on tcgen05 (fp32 X, n <= 128; solve_tc.cu)
 *   SOLVE_DMMA       the tall solve ran on a blocked fp64 DMMA substitution kernel
 *   COLSQ_FUSED      (rcholqr_factor_rr / _rr2) D = diag ||X(:,j)|| came out of the sketch's own pass over X
 *                    (the pre-split Gaussian digit split), no separate column-norm pass
 *   COLMAJOR_NATIVE  (rcholqr_factor_colmajor) the native column-major kernels served the call (no transposes)
 *   SKETCH_FWHT      the SRHT sketch ran as a blocked fast Walsh-Hadamard transform (m n log2 m,
 *                    here 10 + k/1024 adds per element of X) instead of a dense +-1 product
 * *out receives the bits.  SYNCHRONIZES on `stream` (reads the device overflow word).  Errors:
 * E_INVALID for a NULL plan or out. */
#define RCHOLQR_PATH_SKETCH_TC 1u
#define RCHOLQR_PATH_SKETCH_PRESPLIT 2u
#define RCHOLQR_PATH_SKETCH_CUDA_CORE 4u
#define RCHOLQR_PATH_SKETCH_FALLBACK 8u
#define RCHOLQR_PATH_SOLVE_TC 16u
#define RCHOLQR_PATH_SOLVE_DMMA 32u
#define RCHOLQR_PATH_COLSQ_FUSED 64u
#define RCHOLQR_PATH_COLMAJOR_NATIVE 128u /* rcholqr_factor_colmajor: native column-major kernels, no layout adapter */
#define RCHOLQR_PATH_SKETCH_FWHT 256u /* SRHT sketch computed by the blocked fast Walsh-Hadamard transform (m n log2 1024) */
rcholqr_status rcholqr_last_path(rcholqr_plan plan, uint32_t* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RCHOLQR_H */
