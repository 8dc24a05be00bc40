// rcqr2.cu -- the extra CholeskyQR pass of RCholeskyQR2 (Alg. 3):
//   2. A <- Q^T Q          gram_kernel (fp64 DMMA, per-CTA row splits) + sketch_reduce_kernel
//   3. R' <- chol(A)       cholesky_kernel (one CTA, right-looking, A = R'^T R')
//      R <- R' R           trmm_upper_kernel
//   4. Q <- Q R'^{-1}      the tall solve of step 3 of Alg. 2 with R' (api.cu)
// The Gram is a symmetric rank-m update: each CTA owns a 64 x 64 tile of the upper triangle and a
// range of rows ("split"), stages 32 x 64 column blocks of Q in shared memory as fp64 (fp32 Q is
// widened exactly) and accumulates with DMMA m16n8k4; it writes its tile and the transposed tile,
// so the fixed-order compensated reduction over splits (sketch.cu) yields the full symmetric A.
#include <cuda_runtime.h>
#include <algorithm>
#include "internal.cuh"

namespace rcq {

constexpr int GR_T = 64;       // A tile (rows i, cols j)
constexpr int GR_KC = 32;      // Q rows per chunk
constexpr int GR_LD = GR_T + 4;
constexpr int GR_THREADS = 128;

template <typename TX>
__global__ void __launch_bounds__(GR_THREADS)
gram_kernel(const TX* __restrict__ Q, int64_t m, int n, int64_t ldq, int tb, int ntiles, int64_t rows_per_split,
            double* __restrict__ part, const int* status) {
  if (*status) return;
  __shared__ double Qi[GR_KC][GR_LD], Qj[GR_KC][GR_LD];
  // upper-triangle tile (ti <= tj) of linear index t
  int t = blockIdx.x % ntiles, ti = 0;
  const int split = blockIdx.x / ntiles;
  while (t >= tb - ti) { t -= tb - ti; ++ti; }
  const int tj = ti + t;
  const int i0 = ti * GR_T, j0 = tj * GR_T;
  const int64_t r_begin = (int64_t)split * rows_per_split, r_end = min(m, r_begin + rows_per_split);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  const int wi = warp & 1, wj = warp >> 1;            // warp tile 32 x 32 = 2 m16 x 4 n8
  double acc[2][4][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[a][b][e] = 0.0;
  for (int64_t r0 = r_begin; r0 < r_end; r0 += GR_KC) {
    __syncthreads();
    for (int c = tid; c < GR_KC * GR_T; c += GR_THREADS) {
      const int rr = c / GR_T, cc = c % GR_T;
      const int64_t r = r0 + rr;
      Qi[rr][cc] = (r < r_end && i0 + cc < n) ? (double)Q[r * ldq + i0 + cc] : 0.0;
      Qj[rr][cc] = (r < r_end && j0 + cc < n) ? (double)Q[r * ldq + j0 + cc] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < GR_KC / 4; ++ks) {
      const int k = 4 * ks + t4;
      double a0[2], a1[2];
#pragma unroll
      for (int a = 0; a < 2; ++a) {                   // A[i][k] = Q[k][i]
        a0[a] = Qi[k][wi * 32 + a * 16 + g];
        a1[a] = Qi[k][wi * 32 + a * 16 + g + 8];
      }
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const double bv = Qj[k][wj * 32 + b * 8 + g];   // B[k][j] = Q[k][j]
#pragma unroll
        for (int a = 0; a < 2; ++a) dmma_16x8x4(acc[a][b], a0[a], a1[a], bv);
      }
    }
  }
  double* P = part + (size_t)split * n * n;
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = i0 + wi * 32 + a * 16 + g + (e >= 2 ? 8 : 0);
        const int j = j0 + wj * 32 + b * 8 + 2 * t4 + (e & 1);
        if (i < n && j < n) {
          P[(size_t)i * n + j] = acc[a][b][e];
          if (ti != tj) P[(size_t)j * n + i] = acc[a][b][e];
        }
      }
}

// ---------------------------------------------------------------------------------------------
// n <= 128: one CTA per row split computes EVERY upper 32 x 32 sub-tile of the Gram from one shared
// row chunk (KC rows x NPAD columns, cp.async, GS_STAGES-deep ring, zero-filled outside Q), one
// warp per sub-tile (2 m16 x 4 n8 DMMA accumulators), so Q1 is read once and each staged element
// feeds every sub-tile it belongs to.
constexpr int GS_KC = 32;
constexpr int GS_STAGES = 3;

__device__ __forceinline__ void gs_cp4(void* s, const void* g, bool v) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(g), "r"(v ? 4 : 0));
}
__device__ __forceinline__ void gs_cp8(void* s, const void* g, bool v) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(g), "r"(v ? 8 : 0));
}

template <typename TX>
__global__ void gram_small_kernel(const TX* __restrict__ Q, int64_t m, int n, int64_t ldq, int nb,
                                  int64_t rows_per_split, double* __restrict__ part, const int* status) {
  if (*status) return;
  extern __shared__ __align__(16) unsigned char gs_sm[];
  const int npad = nb * 32, LD = npad + 4;
  TX* S = reinterpret_cast<TX*>(gs_sm);                 // [GS_STAGES][GS_KC][LD]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  // warp -> upper sub-tile (bi <= bj) in row-major order of the upper triangle
  int bi = 0, t = warp;
  while (t >= nb - bi) { t -= nb - bi; ++bi; }
  const int bj = bi + t;
  const int64_t r_begin = (int64_t)blockIdx.x * rows_per_split, r_end = min(m, r_begin + rows_per_split);
  const int nchunks = r_end > r_begin ? (int)((r_end - r_begin + GS_KC - 1) / GS_KC) : 0;
  const int nthr = blockDim.x;
  auto issue = [&](int ch) {
    TX* dst = S + (size_t)(ch % GS_STAGES) * GS_KC * LD;
    const int64_t r0 = r_begin + (int64_t)ch * GS_KC;
    for (int c = threadIdx.x; c < GS_KC * npad; c += nthr) {
      const int rr = c / npad, cc = c % npad;
      const bool ok = r0 + rr < r_end && cc < n;
      const TX* src = ok ? Q + (r0 + rr) * ldq + cc : Q;
      if (sizeof(TX) == 4) gs_cp4(dst + rr * LD + cc, src, ok);
      else gs_cp8(dst + rr * LD + cc, src, ok);
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  double acc[2][4][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[a][b][e] = 0.0;
  for (int ch = 0; ch < GS_STAGES - 1; ++ch) {
    if (ch < nchunks) issue(ch);
    else asm volatile("cp.async.commit_group;\n" ::);
  }
  const int i0 = bi * 32, j0 = bj * 32;
  for (int ch = 0; ch < nchunks; ++ch) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(GS_STAGES - 2) : "memory");
    __syncthreads();                                    // chunk ch visible; chunk ch-1's slot free
    if (ch + GS_STAGES - 1 < nchunks) issue(ch + GS_STAGES - 1);
    else asm volatile("cp.async.commit_group;\n" ::);
    const TX* C = S + (size_t)(ch % GS_STAGES) * GS_KC * LD;
#pragma unroll
    for (int ks = 0; ks < GS_KC / 4; ++ks) {
      const TX* row = C + (4 * ks + t4) * LD;
      double a0[2], a1[2], bv[4];
#pragma unroll
      for (int a = 0; a < 2; ++a) {                    // A[i][k] = Q[k][i]
        a0[a] = (double)row[i0 + a * 16 + g];
        a1[a] = (double)row[i0 + a * 16 + g + 8];
      }
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = (double)row[j0 + b * 8 + g];   // B[k][j] = Q[k][j]
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int a = 0; a < 2; ++a) dmma_16x8x4(acc[a][b], a0[a], a1[a], bv[b]);
    }
  }
  double* P = part + (size_t)blockIdx.x * n * n;
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = i0 + a * 16 + g + (e >= 2 ? 8 : 0);
        const int j = j0 + b * 8 + 2 * t4 + (e & 1);
        if (i < n && j < n && (bi != bj || i <= j)) {
          P[(size_t)i * n + j] = acc[a][b][e];
          P[(size_t)j * n + i] = acc[a][b][e];
        }
      }
}

// R' (upper, row-major) with A = R'^T R'; reads the upper triangle of A.  One CTA; A is copied to
// the work buffer W (n x n), updated in place (right-looking), R' written as rows are finished.
__global__ void __launch_bounds__(1024)
cholesky_kernel(const double* __restrict__ A, int n, double* __restrict__ Wg, double* __restrict__ Rp, int* status,
                int stage) {
  if (*status) return;
  extern __shared__ double ch_s[];
  __shared__ int bad;
  __shared__ double sh_r;
  double* W = stage ? ch_s : Wg;                      // the working copy in shared memory when it fits
  const int tid = threadIdx.x;
  if (tid == 0) bad = 0;
  for (int c = tid; c < n * n; c += blockDim.x) { W[c] = A[c]; Rp[c] = 0.0; }
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    if (tid == 0) {
      const double d = W[(size_t)j * n + j];
      if (!(d > 0.0) || !isfinite(d)) bad = 1;
      sh_r = sqrt(d);
      Rp[(size_t)j * n + j] = sh_r;
    }
    __syncthreads();
    if (bad) break;
    const double r = sh_r;
    for (int l = j + 1 + tid; l < n; l += blockDim.x) Rp[(size_t)j * n + l] = W[(size_t)j * n + l] / r;
    __syncthreads();
    // trailing update of the upper triangle: W[i][l] -= R'[j][i] R'[j][l], j < i <= l (warp per row)
    const int warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
    for (int i = j + 1 + warp; i < n; i += nw) {
      const double ri = Rp[(size_t)j * n + i];
      for (int l = i + lane; l < n; l += 32) W[(size_t)i * n + l] -= ri * Rp[(size_t)j * n + l];
    }
    __syncthreads();
  }
  if (tid == 0 && bad) atomicOr(status, kStSingular);
}

// out = U V for upper triangular U, V (row-major n x n): out_ij = sum_{l=i..j} u_il v_lj.
__global__ void trmm_upper_kernel(const double* __restrict__ U, const double* __restrict__ V, int n,
                                  double* __restrict__ out, const int* status) {
  if (*status) return;
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= (int64_t)n * n) return;
  const int i = (int)(c / n), j = (int)(c % n);
  double s = 0.0;
  for (int l = i; l <= j; ++l) s += U[(size_t)i * n + l] * V[(size_t)l * n + j];
  out[c] = j >= i ? s : 0.0;
}

int gram_splits(int n, int sms) {
  if (n <= 128) return 4 * sms;                       // gram_small_kernel: one CTA per split
  const int tb = (n + GR_T - 1) / GR_T, ntiles = tb * (tb + 1) / 2;
  return std::max(1, (2 * sms + ntiles - 1) / ntiles);
}

cudaError_t launch_gram(const void* Q, int dtype, int64_t m, int n, int64_t ldq, int splits, double* part, double* A,
                        int* status, cudaStream_t st) {
  const int tb = (n + GR_T - 1) / GR_T, ntiles = tb * (tb + 1) / 2;
  const int64_t per = (m + splits - 1) / splits;
  const int64_t rps = std::max<int64_t>(GR_KC, (per + GR_KC - 1) / GR_KC * GR_KC);
  if (n <= 128) {
    const int nb = (n + 31) / 32, nt = nb * (nb + 1) / 2;
    const size_t es = dtype == RCHOLQR_F64 ? 8 : 4;
    const size_t smem = (size_t)GS_STAGES * GS_KC * (nb * 32 + 4) * es;
    cudaError_t e2;
    if (dtype == RCHOLQR_F64) {
      e2 = cudaFuncSetAttribute(gram_small_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e2 == cudaSuccess)
        gram_small_kernel<double><<<splits, 32 * nt, smem, st>>>((const double*)Q, m, n, ldq, nb, rps, part, status);
    } else {
      e2 = cudaFuncSetAttribute(gram_small_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e2 == cudaSuccess)
        gram_small_kernel<float><<<splits, 32 * nt, smem, st>>>((const float*)Q, m, n, ldq, nb, rps, part, status);
    }
    if (e2 != cudaSuccess) return e2;
    e2 = cudaGetLastError();
    if (e2 != cudaSuccess) return e2;
    return launch_reduce(part, splits, (int64_t)n * n, 1.0, A, status, st);
  }
  if (dtype == RCHOLQR_F64)
    gram_kernel<double><<<ntiles * splits, GR_THREADS, 0, st>>>((const double*)Q, m, n, ldq, tb, ntiles, rps, part,
                                                                 status);
  else
    gram_kernel<float><<<ntiles * splits, GR_THREADS, 0, st>>>((const float*)Q, m, n, ldq, tb, ntiles, rps, part,
                                                                status);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_reduce(part, splits, (int64_t)n * n, 1.0, A, status, st);
}

cudaError_t launch_cholesky(const double* A, int n, double* W, double* Rp, int* status, cudaStream_t st) {
  const size_t need = sizeof(double) * (size_t)n * n;
  const int stage = need <= 200 * 1024;
  cudaError_t e = cudaFuncSetAttribute(cholesky_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       stage ? (int)need : 0);
  if (e != cudaSuccess) return e;
  cholesky_kernel<<<1, 1024, stage ? need : 0, st>>>(A, n, W, Rp, status, stage);
  return cudaGetLastError();
}

// out (n x n, rows >= r zero) = U V for U r x r upper (ld r) and V r x n upper trapezoidal (ld n):
// RRRCholeskyQR2's R = R' R1.
__global__ void trmm_trap_kernel(const double* __restrict__ U, int r, const double* __restrict__ V, int n,
                                 double* __restrict__ out, const int* status) {
  if (*status) return;
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= (int64_t)n * n) return;
  const int i = (int)(c / n), j = (int)(c % n);
  double s = 0.0;
  if (i < r && j >= i)
    for (int l = i; l <= min(j, r - 1); ++l) s += U[(size_t)i * r + l] * V[(size_t)l * n + j];
  out[c] = s;
}

cudaError_t launch_trmm_trap(const double* U, int r, const double* V, int n, double* out, const int* status,
                             cudaStream_t st) {
  const int64_t nn = (int64_t)n * n;
  trmm_trap_kernel<<<(unsigned)((nn + 255) / 256), 256, 0, st>>>(U, r, V, n, out, status);
  return cudaGetLastError();
}

cudaError_t launch_trmm_upper(const double* U, const double* V, int n, double* out, const int* status,
                              cudaStream_t st) {
  const int64_t nn = (int64_t)n * n;
  trmm_upper_kernel<<<(unsigned)((nn + 255) / 256), 256, 0, st>>>(U, V, n, out, status);
  return cudaGetLastError();
}

}  // namespace rcq
