// qr_blocked.cu -- step 2 of RCholeskyQR (Householder per PAPER.md:163, 424) for sketches
// too large for the single-CTA kernels (C3: 512 x 256, C5: 2048 x 1024): right-looking blocked
// Householder in compact-WY form (Q_panel = H_j0 ... H_j0+nb-1 = I - V T V^T).  Same reflectors,
// pivots and output conventions as qr.cu (column-major reflectors with v0 on the diagonal in the
// workspace, raw R_jj and v0 in diag[], beta in tau[]), so form_s_kernel and the status rules are
// shared; only the order of the floating-point operations differs (blocked trailing updates).
//
// Per panel of nb <= 32 columns starting at j0:
//   qr_panel_kernel (1 CTA, warp w owns panel column j0 + w): the unblocked loop of qr.cu on rows
//     j0..k-1 (look-ahead norm, one barrier per column), then V with explicit zeros above the
//     diagonal in two layouts (Vt: K x nb row-major, Vr: nb x K row-major, K = k - j0), G = V^T V
//     and the WY factor T (T_jj = beta_j, T_{<j,j} = -beta_j T_{<j,<j} G_{<j,j}), stored negated.
//   three fp64 DMMA GEMMs (gemm.cu) update the trailing columns A_t (column-major = row-major A_t^T):
//     W1t = A_t^T Vt   (nt x nb),   W2t = W1t (-T)   (nt x nb),   A_t^T += W2t Vr,
//   i.e. A_t <- (I - V T^T V^T) A_t = Q_panel^T A_t.
#include <cuda_runtime.h>
#include <algorithm>
#include <cooperative_groups.h>
#include <cstdlib>
#include "internal.cuh"

namespace rcq {

constexpr int QB_NB = 32;          // panel width (one warp per panel column)
constexpr int QB_THREADS = 1024;

__device__ __forceinline__ double qb_warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// P (k x n row-major) -> A (column-major, lda = k); non-finite entries raise kStNonfinite.
__global__ void qr_copy_kernel(const double* __restrict__ P, int k, int n, double* __restrict__ A, int* status) {
  int bad = 0;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < (int64_t)k * n;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(c / n), j = (int)(c % n);
    const double v = P[c];
    if (!isfinite(v)) bad = 1;
    A[(size_t)j * k + i] = v;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(status, kStNonfinite);
}

__global__ void __launch_bounds__(QB_THREADS, 1)
qr_panel_kernel(double* __restrict__ A, int k, int n, int j0, int nb, double* __restrict__ diag,
                double* __restrict__ tau, double* __restrict__ Vt, double* __restrict__ Vr,
                double* __restrict__ Tneg, const int* status) {
  if (*status) return;
  __shared__ double sh_norm2[2];
  __shared__ double sh_beta[QB_NB];
  __shared__ double sh_G[QB_NB][QB_NB + 1];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int K = k - j0;
  if (warp == 0) {   // ||A[j0:, j0]||^2
    const double* a = A + (size_t)j0 * k;
    double ss = 0.0;
    for (int i = j0 + lane; i < k; i += 32) ss += a[i] * a[i];
    ss = qb_warp_sum(ss);
    if (lane == 0) sh_norm2[0] = ss;
  }
  __syncthreads();
  for (int p = 0; p < nb; ++p) {
    const int j = j0 + p;
    const double* a = A + (size_t)j * k;
    const double alpha = sqrt(sh_norm2[p & 1]);
    const double x0 = a[j];
    const double sgn = x0 >= 0.0 ? 1.0 : -1.0;
    const double v0 = x0 + sgn * alpha;
    const double beta = alpha == 0.0 ? 0.0 : 1.0 / (alpha * fabs(v0));
    if (tid == 0) {
      tau[j] = beta;
      diag[j] = alpha == 0.0 ? 0.0 : -sgn * alpha;
      diag[n + j] = v0;
      sh_beta[p] = beta;
    }
    if (warp > p && warp < nb) {                 // panel column j0 + warp
      double* c = A + (size_t)(j0 + warp) * k;
      if (beta != 0.0) {
        double w = (lane == 0) ? v0 * c[j] : 0.0;
        for (int i = j + 1 + lane; i < k; i += 32) w += a[i] * c[i];
        w = qb_warp_sum(w) * beta;
        if (lane == 0) c[j] -= v0 * w;
        for (int i = j + 1 + lane; i < k; i += 32) c[i] -= a[i] * w;
      }
      if (warp == p + 1) {                       // look-ahead norm of the next pivot column
        __syncwarp();
        double ss = 0.0;
        for (int i = j + 1 + lane; i < k; i += 32) ss += c[i] * c[i];
        ss = qb_warp_sum(ss);
        if (lane == 0) sh_norm2[(p + 1) & 1] = ss;
      }
    }
    __syncthreads();
  }
  // V (rows j0..k-1) with v0 on the diagonal and zeros above it, in both layouts
  for (int c = tid; c < K * nb; c += QB_THREADS) {
    const int i = c / nb, a = c % nb;               // Vt row-major [K][nb]
    const int row = j0 + i, col = j0 + a;
    const double v = row < col ? 0.0 : (row == col ? diag[n + col] : A[(size_t)col * k + row]);
    Vt[c] = v;
    Vr[(size_t)a * K + i] = v;
  }
  __syncthreads();
  for (int a = 0; a < nb; ++a)                      // the workspace keeps v0 on the diagonal (qr.cu layout)
    if (tid == 0) A[(size_t)(j0 + a) * k + j0 + a] = diag[n + j0 + a];
  // G = V^T V (upper part), warp w computes column w
  if (warp < nb) {
    const double* vw = Vr + (size_t)warp * K;
    for (int a = 0; a <= warp; ++a) {
      const double* va = Vr + (size_t)a * K;
      double s = 0.0;
      for (int i = a + lane; i < K; i += 32) s += va[i] * vw[i];   // va is zero above row a
      s = qb_warp_sum(s);
      if (lane == 0) sh_G[a][warp] = s;
    }
  }
  __syncthreads();
  // T (upper triangular): T_jj = beta_j, T(0:j, j) = -beta_j T(0:j, 0:j) G(0:j, j); stored as -T
  if (warp == 0) {
    __shared__ double Tsh[QB_NB][QB_NB + 1];
    for (int j = 0; j < nb; ++j) {
      // lane i < j: y_i = sum_{q=i}^{j-1} T[i][q] G[q][j]
      double y = 0.0;
      if (lane < j)
        for (int q = lane; q < j; ++q) y += Tsh[lane][q] * sh_G[q][j];
      __syncwarp();
      if (lane < j) Tsh[lane][j] = -sh_beta[j] * y;
      if (lane == j) Tsh[j][j] = sh_beta[j];
      if (lane > j) Tsh[lane][j] = 0.0;
      __syncwarp();
    }
    for (int c = lane; c < nb * nb; c += 32) Tneg[c] = -Tsh[c / nb][c % nb];
  }
}

// ---------------------------------------------------------------------------------------------
// The same panel factorization on a thread-block CLUSTER (K = k - j0 <= QC_ROWS * QC_MAXCL rows): CTA c
// owns rows j0 + c QC_ROWS .. + QC_ROWS - 1, one row per thread, the row's nb panel values in REGISTERS.
// Per column p: the partial column norm (rows >= j) and the nb - p - 1 partial dot products of each CTA
// are exchanged through distributed shared memory around cluster barriers and summed in a fixed CTA
// order (every CTA computes bit-identical alpha, beta, w_q).  The pivot row j0 + p always lies in CTA 0
// (p < nb <= QC_ROWS).  Outputs exactly as qr_panel_kernel: the updated panel in A (v0 on the diagonal),
// diag / tau, Vt / Vr, and -T from G = V^T V (partial G per CTA from a shared V tile, summed in CTA 0).
constexpr int QC_ROWS = 256;
constexpr int QC_MAXCL = 8;

// warp all-reduce of 32 per-lane vectors by a transpose-reduce butterfly: on return lane L holds the
// warp sum of component L (31 shuffles instead of 32 x 5)
__device__ __forceinline__ double qc_transpose_reduce(double (&v)[32], int lane) {
#pragma unroll
  for (int j = 16; j >= 1; j >>= 1) {
    const bool lo = !(lane & j);
#pragma unroll
    for (int i = 0; i < j; ++i) {
      const double send = lo ? v[i + j] : v[i];
      const double keep = lo ? v[i] : v[i + j];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, j);
    }
  }
  return v[0];
}

__global__ void __launch_bounds__(QC_ROWS, 1)
qr_panel_cluster_kernel(double* __restrict__ A, int k, int n, int j0, int nb, double* __restrict__ diag,
                        double* __restrict__ tau, double* __restrict__ Vt, double* __restrict__ Vr,
                        double* __restrict__ Tneg, const int* status) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = (int)cluster.block_rank(), csize = (int)cluster.num_blocks();
  if (*status) return;                                     // uniform over the cluster
  __shared__ double sh_norm[2];                            // this CTA's partial norm^2, by step parity
  __shared__ double sh_x0[2];                              // CTA 0: the next pivot entry
  __shared__ double sh_dot[2][QB_NB];                      // this CTA's partial dots, by step parity
  __shared__ double sh_wred[QC_ROWS / 32][QB_NB];          // per-warp partials
  __shared__ double sh_nred[QC_ROWS / 32];
  __shared__ double sh_G[QB_NB][QB_NB + 1];                // partial G (upper), then (CTA 0) the sum
  __shared__ double sh_beta[QB_NB], sh_v0[QB_NB];
  __shared__ double sh_w[QB_NB], sh_gath[2];              // gathered (cluster-summed) dots / norm^2, x0
  extern __shared__ double qc_dyn[];
  double (*Vs)[QB_NB + 1] = reinterpret_cast<double (*)[QB_NB + 1]>(qc_dyn);   // [QC_ROWS][QB_NB + 1]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int K = k - j0;
  const int lr = tid, gi = j0 + crank * QC_ROWS + lr;      // this thread's global row
  const bool live = gi < k;
  double x[QB_NB];
#pragma unroll
  for (int q = 0; q < QB_NB; ++q) x[q] = (live && q < nb) ? A[(size_t)(j0 + q) * k + gi] : 0.0;
  auto block_sum = [&](double v) {                         // CTA sum (all threads get it)
    v = qb_warp_sum(v);
    if (lane == 0) sh_nred[warp] = v;
    __syncthreads();
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < QC_ROWS / 32; ++w) t += sh_nred[w];
    __syncthreads();
    return t;
  };
  {   // partial ||A[j0:, j0]||^2 and the first pivot entry
    const double t = block_sum(x[0] * x[0]);
    if (tid == 0) sh_norm[0] = t;
    if (crank == 0 && tid == 0) sh_x0[0] = x[0];
  }
  for (int p = 0; p < nb; ++p) {
    const int j = j0 + p, par = p & 1;
    cluster.sync();                                        // exchange 1: norm partials and x0 of step p
    if (tid == 0) {                                        // one gather per CTA, fixed CTA order
      double t = 0.0;
      for (int c = 0; c < csize; ++c) t += *cluster.map_shared_rank(&sh_norm[par], c);
      sh_gath[0] = t;
      sh_gath[1] = *cluster.map_shared_rank(&sh_x0[par], 0);
    }
    __syncthreads();
    const double norm2 = sh_gath[0], x0 = sh_gath[1];
    const double alpha = sqrt(norm2);
    const double sgn = x0 >= 0.0 ? 1.0 : -1.0;
    const double v0 = x0 + sgn * alpha;
    const double beta = alpha == 0.0 ? 0.0 : 1.0 / (alpha * fabs(v0));
    if (crank == 0 && tid == 0) {
      tau[j] = beta;
      diag[j] = alpha == 0.0 ? 0.0 : -sgn * alpha;
      diag[n + j] = v0;
    }
    if (tid == 0) { sh_beta[p] = beta; sh_v0[p] = v0; }
    // this thread's reflector entry: v0 on row j, the column below it, 0 above
    double vt = 0.0;
#pragma unroll
    for (int q = 0; q < QB_NB; ++q)
      if (q == p) vt = (live && gi > j) ? x[q] : (gi == j ? v0 : 0.0);
    // partial dots of the trailing panel columns q > p
    double prod[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) prod[q] = (q > p && q < nb) ? vt * x[q < QB_NB ? q : 0] : 0.0;
    const double wsum = qc_transpose_reduce(prod, lane);   // lane q: warp partial of column q
    sh_wred[warp][lane] = wsum;
    __syncthreads();
    if (warp == 0) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < QC_ROWS / 32; ++w) t += sh_wred[w][lane];
      sh_dot[par][lane] = t;
    }
    cluster.sync();                                        // exchange 2: dot partials of step p
    if (warp == 0) {                                       // lane q gathers column q, fixed CTA order
      double t = 0.0;
      if (lane > p && lane < nb)
        for (int c = 0; c < csize; ++c) t += cluster.map_shared_rank(&sh_dot[par][0], c)[lane];
      sh_w[lane] = t * beta;
    }
    __syncthreads();
    if (beta != 0.0) {
#pragma unroll
      for (int q = 0; q < QB_NB; ++q)
        if (q > p && q < nb && live && gi >= j) x[q] -= vt * sh_w[q];   // row j: v0 * w
    }
    // look-ahead: partial norm^2 of column p + 1 over rows >= j + 1, and its pivot entry
    if (p + 1 < nb) {
      double xn = 0.0;
#pragma unroll
      for (int q = 0; q < QB_NB; ++q)
        if (q == p + 1) xn = x[q];
      const double t = block_sum((live && gi > j) ? xn * xn : 0.0);
      if (tid == 0) sh_norm[par ^ 1] = t;
      if (crank == 0 && lr == p + 1) sh_x0[par ^ 1] = xn;
    }
  }
  // write back the panel (v0 on the diagonal), V in both layouts, the partial G from the V tile
#pragma unroll
  for (int q = 0; q < QB_NB; ++q) {
    if (q >= nb) break;
    const int col = j0 + q;
    double v;
    if (!live) v = 0.0;
    else if (gi < col) v = 0.0;
    else if (gi == col) v = sh_v0[q];
    else v = x[q];
    Vs[lr][q] = v;
    if (live) {
      A[(size_t)col * k + gi] = gi == col ? sh_v0[q] : x[q];
      Vt[(size_t)(gi - j0) * nb + q] = v;
      Vr[(size_t)q * K + (gi - j0)] = v;
    }
  }
  __syncthreads();
  for (int e = tid; e < nb * nb; e += QC_ROWS) {           // partial G(a, b), a <= b
    const int a = e / nb, b = e % nb;
    if (a > b) continue;
    double t = 0.0;
    for (int r = 0; r < QC_ROWS; ++r) t += Vs[r][a] * Vs[r][b];
    sh_G[a][b] = t;
  }
  cluster.sync();
  if (crank == 0) {
    for (int e = tid; e < nb * nb; e += QC_ROWS) {
      const int a = e / nb, b = e % nb;
      if (a > b) continue;
      double t = 0.0;
      for (int c = 0; c < csize; ++c) t += cluster.map_shared_rank(&sh_G[0][0], c)[a * (QB_NB + 1) + b];
      Tneg[a * nb + b] = t;                                // scratch: the summed G (upper), read below
    }
  }
  cluster.sync();                                          // remote reads of sh_G finished
  if (crank == 0) {
    __threadfence_block();
    if (warp == 0) {
      __shared__ double Tsh[QB_NB][QB_NB + 1];
      for (int jj = 0; jj < nb; ++jj) {
        double y = 0.0;
        if (lane < jj)
          for (int q = lane; q < jj; ++q) y += Tsh[lane][q] * Tneg[q * nb + jj];
        __syncwarp();
        if (lane < jj) Tsh[lane][jj] = -sh_beta[jj] * y;
        if (lane == jj) Tsh[jj][jj] = sh_beta[jj];
        if (lane > jj) Tsh[lane][jj] = 0.0;
        __syncwarp();
      }
      __syncwarp();
      for (int c = lane; c < nb * nb; c += 32) Tneg[c] = -Tsh[c / nb][c % nb];
    }
  }
}

// R (row-major, zeros below the diagonal, rows with a negative pivot negated) + singular flag.
__global__ void qr_finalize_kernel(const double* __restrict__ A, int k, int n, const double* __restrict__ diag,
                                   double* __restrict__ R, int* status) {
  if (*status & kStNonfinite) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n * n; c += gridDim.x * blockDim.x) R[c] = 0.0;
    return;
  }
  int bad = 0;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n * n; c += gridDim.x * blockDim.x) {
    const int j = c / n, l = c % n;
    const double d = diag[j];
    const double sg = d < 0.0 ? -1.0 : 1.0;
    double v = 0.0;
    if (l == j) { v = d; if (d == 0.0 || !isfinite(d)) bad = 1; }
    else if (l > j) v = A[(size_t)l * k + j];
    R[c] = sg * v;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(status, kStSingular);
}

size_t qr_blocked_workspace(int k, int n) {
  // Vt + Vr (k x 32 each), W1t + W2t (n x 32 each), Tneg (32 x 32)
  return sizeof(double) * ((size_t)2 * k * QB_NB + (size_t)2 * n * QB_NB + QB_NB * QB_NB);
}

cudaError_t launch_qr_blocked(const double* P, int k, int n, double* R, double* A, double* diag, double* tau,
                              double* ws, int* status, cudaStream_t st) {
  double* Vt = ws;
  double* Vr = Vt + (size_t)k * QB_NB;
  double* W1t = Vr + (size_t)k * QB_NB;
  double* W2t = W1t + (size_t)n * QB_NB;
  double* Tneg = W2t + (size_t)n * QB_NB;
  qr_copy_kernel<<<148, 256, 0, st>>>(P, k, n, A, status);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  for (int j0 = 0; j0 < n; j0 += QB_NB) {
    const int nb = std::min(QB_NB, n - j0);
    const int K = k - j0;
    static const bool old_panel = getenv("RCHOLQR_QR_PANEL_OLD") != nullptr;   // experiments
    const int cl = (K + QC_ROWS - 1) / QC_ROWS;
    bool done = false;
    if (!old_panel && cl >= 3 && cl <= QC_MAXCL) {      // panel held on-chip by a cluster of cl CTAs (K > 512)
      constexpr size_t qc_smem = sizeof(double) * QC_ROWS * (QB_NB + 1);
      static const bool attr_ok = cudaFuncSetAttribute(qr_panel_cluster_kernel,
                                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                       (int)qc_smem) == cudaSuccess;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cl);
      cfg.blockDim = dim3(QC_ROWS);
      cfg.dynamicSmemBytes = qc_smem;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = cl;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      done = attr_ok && cudaLaunchKernelEx(&cfg, qr_panel_cluster_kernel, A, k, n, j0, nb, diag, tau, Vt, Vr, Tneg,
                                (const int*)status) == cudaSuccess;
      if (!done) cudaGetLastError();                       // no cluster launch: the single-CTA kernel
    }
    if (!done) qr_panel_kernel<<<1, QB_THREADS, 0, st>>>(A, k, n, j0, nb, diag, tau, Vt, Vr, Tneg, status);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    const int nt = n - j0 - nb;
    if (nt <= 0) continue;
    double* At = A + (size_t)(j0 + nb) * k + j0;     // row l of A_t^T = column j0+nb+l from row j0
    // W1t = A_t^T Vt  (nt x nb, K = k - j0)
    if ((e = launch_gemm_f64(At, k, Vt, nb, nullptr, 0, W1t, nb, nt, nb, K, false, status, st)) != cudaSuccess) return e;
    // W2t = W1t (-T)
    if ((e = launch_gemm_f64(W1t, nb, Tneg, nb, nullptr, 0, W2t, nb, nt, nb, nb, false, status, st)) != cudaSuccess)
      return e;
    // A_t^T += W2t Vr
    if ((e = launch_gemm_f64(W2t, nb, Vr, K, At, k, At, k, nt, K, nb, false, status, st)) != cudaSuccess) return e;
  }
  qr_finalize_kernel<<<std::max(1, std::min(148, (n * n + 255) / 256)), 256, 0, st>>>(A, k, n, diag, R, status);
  return cudaGetLastError();
}

}  // namespace rcq
