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
    qr_panel_kernel<<<1, QB_THREADS, 0, st>>>(A, k, n, j0, nb, diag, tau, Vt, Vr, Tneg, status);
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
