// qr.cu -- step 2 of RCholeskyQR: [R, S] = QR(P) by Householder reflections
// ("more stable methods in step 2 such as Householder QR").
//
// One CTA (1024 threads) factors the k x n fp64 sketch.  The working copy A lives column-major in
// shared memory when it fits (k*n*8 <= ~200 KB: configs C1, C2, C4) and in a global workspace
// (L2-resident) otherwise.  For column j (one CTA barrier per column):
//   every warp: alpha = ||A[j:,j]||, v = A[j:,j] + sign(a_jj) alpha e_j, beta = 1/(alpha |v_0|),
//               R_jj = -sign(a_jj) alpha   (from the look-ahead norm of the previous step)
//   all warps:  each trailing column l > j (dealt cyclically) gets
//               A[j:,l] -= v * beta * (v^T A[j:,l])   (warp-shuffle dot product); the owner of
//               column j+1 then computes ||A[j+1:,j+1]||^2 for the next step.
// Then diag(R) >= 0 by negating rows (reading A5) and a zero/non-finite pivot raises the
// singular flag (reading A6).  The reflectors (v, beta) stay in the workspace so that S (Alg. 2's
// orthonormal sketch) can be formed on request: S = H_0 ... H_{n-1} [I_n; 0], one warp
// per column of S.
#include <cuda_runtime.h>
#include <algorithm>
#include "internal.cuh"

namespace rcq {

constexpr int QR_THREADS = 1024;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// A: column-major working copy with leading dimension lda (= k).  One barrier per column:
// every warp derives (alpha_j, v0, beta) redundantly from ||A[j:,j]||^2, which the owner of
// column j (columns are dealt cyclically to warps) computed at the end of step j-1 right after
// updating that column ("look-ahead"); the reflector's head v0 is kept in diag_v[] instead of
// being written into A[j][j], so no warp races the others for it.
template <bool use_smem>   // compile-time, so A's accesses are LDS/STS (not generic LD/ST)
__global__ void __launch_bounds__(QR_THREADS, 1)
householder_kernel(const double* __restrict__ P, int k, int n, double* __restrict__ R,
                   double* __restrict__ Aglob, double* __restrict__ diag_out, double* __restrict__ tau_out,
                   int* status) {
  extern __shared__ __align__(16) double smem[];
  __shared__ int sh_flag;
  __shared__ double sh_norm2[2];     // ping-pong: ||A[j:,j]||^2 for the current / next column
  double* A = use_smem ? smem : Aglob;
  const int lda = k;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nwarps = QR_THREADS / 32;
  if (tid == 0) sh_flag = 0;
  __syncthreads();
  for (int64_t c = tid; c < (int64_t)k * n; c += QR_THREADS) {   // row-major P -> column-major A
    const int i = (int)(c / n), j = (int)(c % n);
    const double v = P[c];
    if (!isfinite(v)) sh_flag = 1;
    A[(size_t)j * lda + i] = v;
  }
  __syncthreads();
  if (sh_flag) {  // non-finite sketch: report, leave R as zeros
    for (int c = tid; c < n * n; c += QR_THREADS) R[c] = 0.0;
    if (tid == 0) atomicOr(status, kStNonfinite);
    return;
  }
  if (warp == 0) {   // ||A[:,0]||^2
    double ss = 0.0;
    for (int i = lane; i < k; i += 32) ss += A[i] * A[i];
    ss = warp_sum(ss);
    if (lane == 0) sh_norm2[0] = ss;
  }
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    const double* a = A + (size_t)j * lda;
    const double alpha = sqrt(sh_norm2[j & 1]);
    const double x0 = a[j];
    const double sgn = x0 >= 0.0 ? 1.0 : -1.0;
    const double v0 = x0 + sgn * alpha;
    const double beta = alpha == 0.0 ? 0.0 : 1.0 / (alpha * fabs(v0));
    if (tid == 0) {
      tau_out[j] = beta;
      diag_out[j] = alpha == 0.0 ? 0.0 : -sgn * alpha;
      diag_out[n + j] = v0;           // reflector head (v = [v0; A[j+1:, j]])
    }
    // trailing columns l > j, dealt cyclically: warp w owns l = w, w + nwarps, ...
    int l = j + 1 + ((warp - (j + 1)) % nwarps + nwarps) % nwarps;
    for (; l < n; l += nwarps) {
      double* c = A + (size_t)l * lda;
      if (beta != 0.0) {
        double w = (lane == 0) ? v0 * c[j] : 0.0;
        for (int i = j + 1 + lane; i < k; i += 32) w += a[i] * c[i];
        w = warp_sum(w) * beta;
        if (lane == 0) c[j] -= v0 * w;
        for (int i = j + 1 + lane; i < k; i += 32) c[i] -= a[i] * w;
      }
      if (l == j + 1) {              // look-ahead: norm of the next pivot column below row j+1
        __syncwarp();
        double ss = 0.0;
        for (int i = j + 1 + lane; i < k; i += 32) ss += c[i] * c[i];
        ss = warp_sum(ss);
        if (lane == 0) sh_norm2[(j + 1) & 1] = ss;
      }
    }
    __syncthreads();
  }
  // R (row-major, zeros below the diagonal), rows with negative pivot negated.
  for (int c = tid; c < n * n; c += QR_THREADS) {
    const int j = c / n, l = c % n;
    const double d = diag_out[j];
    const double sg = d < 0.0 ? -1.0 : 1.0;
    double v = 0.0;
    if (l == j) v = d;
    else if (l > j) v = A[(size_t)l * lda + j];
    R[c] = sg * v;
  }
  // keep the reflectors (column-major, head v0 on the diagonal) for S formation
  for (int64_t c = tid; c < (int64_t)k * n; c += QR_THREADS) {
    const int j = (int)(c / lda), i = (int)(c % lda);
    if (i == j) Aglob[c] = diag_out[n + j];
    else if (use_smem) Aglob[c] = A[c];
  }
  if (tid < 32) {
    int bad = 0;
    for (int j = lane; j < n; j += 32) {
      const double d = diag_out[j];
      if (d == 0.0 || !isfinite(d)) bad = 1;
    }
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0 && bad) atomicOr(status, kStSingular);
  }
}

// S = H_0 ... H_{n-1} [I_n; 0], then column l negated where diag_l < 0.  One warp per column;
// the column lives in a shared-memory buffer of k doubles per warp.
constexpr int FS_WARPS = 4;
__global__ void __launch_bounds__(32 * FS_WARPS)
form_s_kernel(const double* __restrict__ A, const double* __restrict__ tau, const double* __restrict__ diag,
              int k, int n, double* __restrict__ S, const int* status) {
  extern __shared__ __align__(16) double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int l = blockIdx.x * FS_WARPS + warp;
  if (l >= n || (*status & kStNonfinite)) return;
  double* s = smem + (size_t)warp * k;
  for (int i = lane; i < k; i += 32) s[i] = (i == l) ? 1.0 : 0.0;
  __syncwarp();
  for (int j = l; j >= 0; --j) {
    const double b = tau[j];
    if (b == 0.0) continue;
    const double* v = A + (size_t)j * k;
    double w = 0.0;
    for (int i = j + lane; i < k; i += 32) w += v[i] * s[i];
    w = warp_sum(w) * b;
    for (int i = j + lane; i < k; i += 32) s[i] -= v[i] * w;
    __syncwarp();
  }
  const double sg = diag[l] < 0.0 ? -1.0 : 1.0;
  for (int i = lane; i < k; i += 32) S[(size_t)i * n + l] = sg * s[i];
}

int plan_qr(int k, int n, size_t smem_optin) {
  const size_t need = sizeof(double) * (size_t)k * n;
  return need + 1024 <= std::min<size_t>(smem_optin, 220 * 1024) ? kQrSmem : kQrGlobal;
}

cudaError_t launch_qr(int kind, const double* P, int k, int n, double* R, double* Awork, double* diag,
                      double* tau, int* status, cudaStream_t st) {
  if (kind == kQrSmem) {
    const size_t smem = sizeof(double) * (size_t)k * n;
    cudaError_t e = cudaFuncSetAttribute(householder_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    householder_kernel<true><<<1, QR_THREADS, smem, st>>>(P, k, n, R, Awork, diag, tau, status);
  } else {
    householder_kernel<false><<<1, QR_THREADS, 0, st>>>(P, k, n, R, Awork, diag, tau, status);
  }
  return cudaGetLastError();
}

cudaError_t launch_form_s(const double* Awork, const double* tau, const double* diag, int k, int n, double* S,
                          const int* status, cudaStream_t st) {
  const size_t smem = sizeof(double) * (size_t)k * FS_WARPS;
  cudaError_t e = cudaFuncSetAttribute(form_s_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  form_s_kernel<<<(n + FS_WARPS - 1) / FS_WARPS, 32 * FS_WARPS, smem, st>>>(Awork, tau, diag, k, n, S, status);
  return cudaGetLastError();
}

}  // namespace rcq
