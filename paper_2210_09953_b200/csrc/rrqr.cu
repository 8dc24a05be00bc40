// rrqr.cu -- device kernels of the rank-revealing RCholeskyQR (Alg. 7; DESIGN.md
// reading A21).  The tall steps are one extra pass each: the column norms D of X (next
// to the sketch of Alg. 2's kernels) and the gather of the r selected columns for step 4's solve.
// Everything between is the small k x n / n x n work of steps 2-3 ("negligible"),
// run by single-CTA kernels in fp64:
//   colsq_kernel         per-split column sums of squares (only when the sketch pass could not carry D)
//   rr_normalize_kernel  d_j = sqrt(sum), P <- P D^{-1} (zero columns stay zero)
//   qrcp_kernel          Businger-Golub column pivoting: the permutation only (norms recomputed)
//   rr_gather_kernel     P(:, perm) for the unpivoted Householder of qr.cu / qr_blocked.cu
//   rank_kernel          ||R||_2 by 64 power iterations, r = min r: ||R(r:, r:)||_F <= tau ||R||_2
//   strong_kernel        max rho_ij^2 of the Gu-Eisenstat test at rank r and its (i, j)
//   rr_finalize_kernel   R(1:r, :) Pi^T D Pi and its compact leading r x r block
//   gather_x_kernel      X(:, perm(1:r)) for the tall solve
#include <cuda_runtime.h>
#include <algorithm>
#include <cmath>
#include <cstdint>
#include "internal.cuh"

namespace rcq {

constexpr int CS_ROWS = 8;   // colsq: 32 columns x 8 row lanes per CTA

template <typename TX>
__global__ void __launch_bounds__(32 * CS_ROWS)
colsq_kernel(const TX* __restrict__ X, int64_t m, int n, int64_t ldx, int64_t rows_per_split,
             double* __restrict__ part) {
  __shared__ double red[CS_ROWS][33];
  const int c = blockIdx.y * 32 + threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_split, r1 = min(m, r0 + rows_per_split);
  double s = 0.0;
  if (c < n)
    for (int64_t r = r0 + threadIdx.y; r < r1; r += CS_ROWS) {
      const double x = (double)X[r * ldx + c];
      s = fma(x, x, s);
    }
  red[threadIdx.y][threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.y == 0 && c < n) {
    double t = 0.0;
#pragma unroll
    for (int y = 0; y < CS_ROWS; ++y) t += red[y][threadIdx.x];
    part[(size_t)blockIdx.x * n + c] = t;
  }
}

// buf: (k + 1) x n, rows 0..k-1 = P, row k = column sums of squares (both all-reduced)
__global__ void rr_normalize_kernel(const double* __restrict__ buf, int k, int n, double* __restrict__ Pn,
                                    double* __restrict__ d) {
  const int64_t kn = (int64_t)k * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < kn + n; t += (int64_t)gridDim.x * blockDim.x) {
    if (t < kn) {
      const int j = (int)(t % n);
      const double dj = sqrt(buf[kn + j]);
      Pn[t] = dj > 0.0 ? buf[t] / dj : 0.0;
    } else {
      d[t - kn] = sqrt(buf[t]);
    }
  }
}

__device__ __forceinline__ double rr_warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// (value, index) argmax with ties to the smaller index, over the block; result in *bv / *bi.
__device__ void rr_block_argmax(double v, int idx, double* sv, int* si, double* bv, int* bi) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
  }
  if (lane == 0) { sv[warp] = v; si[warp] = idx; }
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    v = lane < nw ? sv[lane] : -INFINITY;
    idx = lane < nw ? si[lane] : INT32_MAX;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, o);
      const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
      if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
    }
    if (lane == 0) { *bv = v; *bi = idx; }
  }
  __syncthreads();
}

// block sum (every thread gets the result); red: 32 doubles of shared scratch
__device__ double rr_block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = rr_warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = lane < nw ? red[lane] : 0.0;
  return rr_warp_sum(t);
}

// Column pivoting on the k x n row-major Pn (A: k x n column-major workspace, in shared memory when
// `stage` -- the loops below are L2-latency bound otherwise); writes perm only.  The trailing column
// norms are DOWNDATED after each step (nrm2_l -= A(j, l)^2, as LAPACK's dgeqp3 / dlaqp2) and recomputed
// exactly when cancellation makes the downdate unreliable (remaining < 1e-4 of the last exact value) --
// the pivots equal the oracle's recomputed-norm choices except at rounding-level ties.
__global__ void __launch_bounds__(1024) qrcp_kernel(const double* __restrict__ Pn, int k, int n, double* __restrict__ Ag,
                                                    int* __restrict__ perm, int stage) {
  extern __shared__ double qp_s[];
  __shared__ double sv[32], s_bv;
  __shared__ int si[32], s_bi;
  __shared__ double nrm[1024], nref[1024];          // current (downdated) and last exact squared norms (n <= 1024)
  double* A = stage ? qp_s : Ag;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int64_t t = tid; t < (int64_t)k * n; t += blockDim.x) {
    const int i = (int)(t / n), j = (int)(t % n);
    A[(size_t)j * k + i] = Pn[t];
  }
  for (int j = tid; j < n; j += blockDim.x) perm[j] = j;
  __syncthreads();
  auto exact_norm = [&](int l, int j0) {            // warp-wide sum of squares of column l, rows j0..k-1
    const double* c = A + (size_t)l * k;
    double ss = 0.0;
    for (int i = j0 + lane; i < k; i += 32) ss = fma(c[i], c[i], ss);
    return rr_warp_sum(ss);
  };
  for (int l = warp; l < n; l += nw) {
    const double v = exact_norm(l, 0);
    if (lane == 0) { nrm[l] = v; nref[l] = v; }
  }
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    // argmax of the trailing norms (first index on ties)
    double best = -1.0;
    int bidx = n;
    for (int l = j + tid; l < n; l += blockDim.x)
      if (nrm[l] > best) { best = nrm[l]; bidx = l; }
    rr_block_argmax(best, bidx, sv, si, &s_bv, &s_bi);
    const int p = s_bi;
    if (p >= n) break;                         // no comparable norm (non-finite P: the status word reports it)
    if (p != j) {
      for (int i = tid; i < k; i += blockDim.x) {
        const double t = A[(size_t)j * k + i];
        A[(size_t)j * k + i] = A[(size_t)p * k + i];
        A[(size_t)p * k + i] = t;
      }
      if (tid == 0) {
        const int t = perm[j]; perm[j] = perm[p]; perm[p] = t;
        const double a = nrm[j]; nrm[j] = nrm[p]; nrm[p] = a;
        const double b = nref[j]; nref[j] = nref[p]; nref[p] = b;
      }
    }
    __syncthreads();
    // the pivot column's norm exactly (its reflector needs it)
    if (warp == 0) {
      const double v = exact_norm(j, j);
      if (lane == 0) s_bv = v;
    }
    __syncthreads();
    const double alpha = sqrt(s_bv);
    if (!(alpha > 0.0)) break;                 // the trailing columns are all zero
    const double* a = A + (size_t)j * k;
    const double aj = a[j];
    const double v0 = aj + (aj >= 0.0 ? alpha : -alpha);
    const double scale = 1.0 / (alpha * fabs(v0));
    for (int l0 = j + 1 + warp; l0 < n; l0 += 4 * nw) {
      double dot[4] = {0.0, 0.0, 0.0, 0.0}, cj[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int q = 0; q < 4; ++q)               // read by every lane before lane 0 rewrites it
        if (l0 + q * nw < n) cj[q] = A[(size_t)(l0 + q * nw) * k + j];
      for (int i = j + 1 + lane; i < k; i += 32) {
        const double ai = a[i];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (l0 + q * nw < n) dot[q] = fma(ai, A[(size_t)(l0 + q * nw) * k + i], dot[q]);
      }
      double t[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) t[q] = (rr_warp_sum(dot[q]) + v0 * cj[q]) * scale;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int l = l0 + q * nw;
        if (l < n) {
          const double rjl = cj[q] - t[q] * v0;           // the new A(j, l) = R(j, l)
          if (lane == 0) {
            A[(size_t)l * k + j] = rjl;
            const double left = nrm[l] - rjl * rjl;       // downdate
            nrm[l] = left;
          }
        }
      }
      for (int i = j + 1 + lane; i < k; i += 32) {
        const double ai = a[i];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (l0 + q * nw < n) A[(size_t)(l0 + q * nw) * k + i] -= t[q] * ai;
      }
      __syncwarp();                                       // lane 0's downdates and every lane's axpys visible
#pragma unroll
      for (int q = 0; q < 4; ++q) {                       // cancellation: recompute rows j+1.. exactly
        const int l = l0 + q * nw;
        if (l < n) {
          const bool redo = !(nrm[l] > 1e-4 * nref[l]);
          if (redo) {
            const double v = exact_norm(l, j + 1);
            if (lane == 0) { nrm[l] = v; nref[l] = v; }
          }
        }
      }
    }
    __syncthreads();
  }
}

__global__ void rr_gather_kernel(const double* __restrict__ Pn, int k, int n, const int* __restrict__ perm,
                                 double* __restrict__ Pg) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)k * n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / n;
    const int j = (int)(t % n);
    Pg[t] = Pn[i * n + perm[j]];
  }
}

// ||R||_2 (64 power iterations, as the oracle) and the rank rule; warp-per-row mat-vecs and block sums.
// R is staged in shared memory when it fits (stage != 0), else read from L2.
__global__ void __launch_bounds__(1024) rank_kernel(const double* __restrict__ Rg, int n, double tau, int* rank,
                                                    double* sigma_out, int rank_fixed, int stage) {
  extern __shared__ double rk_s[];
  double* x = rk_s;
  double* y = rk_s + n;
  __shared__ double red[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const double* R = Rg;
  const double* Rt = nullptr;                       // R^T (staged): conflict-free R^T y
  if (stage) {
    double* Rs = rk_s + 2 * n;
    double* Rts = Rs + (size_t)n * n;
    for (int t = tid; t < n * n; t += blockDim.x) {
      const double v = Rg[t];
      Rs[t] = v;
      Rts[(size_t)(t % n) * n + t / n] = v;
    }
    R = Rs;
    Rt = Rts;
  }
  for (int j = tid; j < n; j += blockDim.x) x[j] = 1.0 / sqrt((double)n);
  __syncthreads();
  double sigma = 0.0;
  for (int it = 0; it <= 64; ++it) {
    for (int i = warp; i < n; i += nw) {          // y = R x
      double s = 0.0;
      for (int j = i + lane; j < n; j += 32) s = fma(R[(size_t)i * n + j], x[j], s);
      s = rr_warp_sum(s);
      if (lane == 0) y[i] = s;
    }
    __syncthreads();
    double part = 0.0;
    for (int i = tid; i < n; i += blockDim.x) part = fma(y[i], y[i], part);
    sigma = sqrt(rr_block_sum(part, red));
    if (it == 64 || sigma == 0.0) break;
    for (int j = warp; j < n; j += nw) {          // x = R^T y
      double s = 0.0;
      if (Rt)
        for (int i = lane; i <= j; i += 32) s = fma(Rt[(size_t)j * n + i], y[i], s);
      else
        for (int i = lane; i <= j; i += 32) s = fma(R[(size_t)i * n + j], y[i], s);
      s = rr_warp_sum(s);
      if (lane == 0) x[j] = s;
    }
    __syncthreads();
    part = 0.0;
    for (int j = tid; j < n; j += blockDim.x) part = fma(x[j], x[j], part);
    const double nx = sqrt(rr_block_sum(part, red));
    if (nx == 0.0) break;
    for (int j = tid; j < n; j += blockDim.x) x[j] /= nx;
    __syncthreads();
  }
  // row sums of squares of the trailing triangle, then the suffix rule (sequential, as the oracle)
  for (int j = warp; j < n; j += nw) {
    double row = 0.0;
    for (int l = j + lane; l < n; l += 32) row = fma(R[(size_t)j * n + l], R[(size_t)j * n + l], row);
    row = rr_warp_sum(row);
    if (lane == 0) y[j] = row;
  }
  __syncthreads();
  if (tid == 0) {
    int r = n;
    if (rank_fixed > 0) {
      r = min(rank_fixed, n);
    } else {
      const double thr = tau * sigma;
      double t2 = 0.0;
      for (int j = n - 1; j >= 0; --j) {
        t2 += y[j];
        if (sqrt(t2) <= thr) r = j;
        else break;
      }
    }
    *rank = r;
    *sigma_out = sigma;
  }
}

// Gu-Eisenstat test at rank r: out_v = max rho^2, out_i = flat index i (n - r) + j (first in (i, j) order).
__global__ void __launch_bounds__(1024) strong_kernel(const double* __restrict__ R, int n, int r,
                                                      double* __restrict__ W, double* out_v, int* out_i) {
  extern __shared__ double st_s[];
  double* iw2 = st_s;          // 1 / omega_i^2, i < r
  double* g2 = st_s + r;       // gamma_j^2, j < n - r
  __shared__ double sv[32];
  __shared__ int si[32];
  const int tid = threadIdx.x, nt = n - r;
  for (int j = tid; j < r; j += blockDim.x)     // W = R11^{-1}, column j by back substitution
    for (int i = j; i >= 0; --i) {
      double s = i == j ? 1.0 : 0.0;
      for (int l = i + 1; l <= j; ++l) s -= R[(size_t)i * n + l] * W[(size_t)l * r + j];
      W[(size_t)i * r + j] = s / R[(size_t)i * n + i];
    }
  __syncthreads();
  for (int i = tid; i < r; i += blockDim.x) {
    double s = 0.0;
    for (int l = i; l < r; ++l) s += W[(size_t)i * r + l] * W[(size_t)i * r + l];
    iw2[i] = s;
  }
  for (int j = tid; j < nt; j += blockDim.x) {
    double s = 0.0;
    for (int l = r; l <= r + j; ++l) s += R[(size_t)l * n + r + j] * R[(size_t)l * n + r + j];
    g2[j] = s;
  }
  __syncthreads();
  double best = -1.0;
  int bidx = INT32_MAX;
  for (int64_t t = tid; t < (int64_t)r * nt; t += blockDim.x) {
    const int i = (int)(t / nt), j = (int)(t % nt);
    double a = 0.0;
    for (int l = i; l < r; ++l) a += W[(size_t)i * r + l] * R[(size_t)l * n + r + j];
    const double rho2 = a * a + g2[j] * iw2[i];
    if (rho2 > best) { best = rho2; bidx = (int)t; }
  }
  __shared__ double s_bv;
  __shared__ int s_bi;
  rr_block_argmax(best, bidx, sv, si, &s_bv, &s_bi);
  if (tid == 0) { *out_v = s_bv; *out_i = s_bi; }
}

__global__ void rr_finalize_kernel(const double* __restrict__ Rf, int n, int r, const double* __restrict__ d,
                                   const int* __restrict__ perm, double* __restrict__ Rout, double* __restrict__ R11) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)n * n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(t / n), l = (int)(t % n);
    const double v = i < r ? Rf[t] * d[perm[l]] : 0.0;
    Rout[t] = v;
    if (i < r && l < r) R11[(size_t)i * r + l] = v;
  }
}

template <typename TX>
__global__ void gather_x_kernel(const TX* __restrict__ X, int64_t m, int64_t ldx, const int* __restrict__ perm, int r,
                                TX* __restrict__ Xr) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m * r; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / r;
    const int j = (int)(t % r);
    Xr[t] = X[i * ldx + perm[j]];
  }
}

// ---------------------------------------------------------------------------------------------
int colsq_splits(int n, int sms) {
  const int cb = (n + 31) / 32;
  return std::max(1, (4 * sms + cb - 1) / cb);
}

cudaError_t launch_colsq(const void* X, int dtype, int64_t m, int n, int64_t ldx, int splits, double* part,
                         double* out, int* status, cudaStream_t st) {
  const int64_t rps = (m + splits - 1) / splits;
  const dim3 grid(splits, (n + 31) / 32), block(32, CS_ROWS);
  if (dtype == RCHOLQR_F64) colsq_kernel<double><<<grid, block, 0, st>>>((const double*)X, m, n, ldx, rps, part);
  else colsq_kernel<float><<<grid, block, 0, st>>>((const float*)X, m, n, ldx, rps, part);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_reduce(part, splits, n, 1.0, out, status, st);
}

static unsigned ew_blocks(int64_t work) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, 4096)); }

cudaError_t launch_rr_normalize(const double* buf, int k, int n, double* Pn, double* d, cudaStream_t st) {
  rr_normalize_kernel<<<ew_blocks((int64_t)(k + 1) * n), 256, 0, st>>>(buf, k, n, Pn, d);
  return cudaGetLastError();
}

cudaError_t launch_qrcp(const double* Pn, int k, int n, double* A, int* perm, cudaStream_t st) {
  const size_t need = sizeof(double) * (size_t)k * n;
  const int stage = need <= 200 * 1024;
  cudaError_t e = cudaFuncSetAttribute(qrcp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       stage ? (int)need : 0);
  if (e != cudaSuccess) return e;
  qrcp_kernel<<<1, 1024, stage ? need : 0, st>>>(Pn, k, n, A, perm, stage);
  return cudaGetLastError();
}

cudaError_t launch_rr_gather(const double* Pn, int k, int n, const int* perm, double* Pg, cudaStream_t st) {
  rr_gather_kernel<<<ew_blocks((int64_t)k * n), 256, 0, st>>>(Pn, k, n, perm, Pg);
  return cudaGetLastError();
}

cudaError_t launch_rank(const double* R, int n, double tau, int rank_fixed, int* rank, double* sigma, cudaStream_t st) {
  const size_t base = sizeof(double) * 2 * (size_t)n, staged = base + sizeof(double) * 2 * (size_t)n * n;
  const int stage = staged <= 200 * 1024;
  const size_t smem = stage ? staged : base;
  cudaError_t e = cudaFuncSetAttribute(rank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  rank_kernel<<<1, 1024, smem, st>>>(R, n, tau, rank, sigma, rank_fixed, stage);
  return cudaGetLastError();
}

cudaError_t launch_strong(const double* R, int n, int r, double* W, double* out_v, int* out_i, cudaStream_t st) {
  const size_t smem = sizeof(double) * (size_t)n;
  cudaError_t e = cudaFuncSetAttribute(strong_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  strong_kernel<<<1, 1024, smem, st>>>(R, n, r, W, out_v, out_i);
  return cudaGetLastError();
}

cudaError_t launch_rr_finalize(const double* Rf, int n, int r, const double* d, const int* perm, double* Rout,
                               double* R11, cudaStream_t st) {
  rr_finalize_kernel<<<ew_blocks((int64_t)n * n), 256, 0, st>>>(Rf, n, r, d, perm, Rout, R11);
  return cudaGetLastError();
}

cudaError_t launch_gather_x(const void* X, int dtype, int64_t m, int64_t ldx, const int* perm, int r, void* Xr,
                            int sms, cudaStream_t st) {
  if (m <= 0 || r <= 0) return cudaSuccess;
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((m * r + 255) / 256, 8 * sms));
  if (dtype == RCHOLQR_F64)
    gather_x_kernel<double><<<blocks, 256, 0, st>>>((const double*)X, m, ldx, perm, r, (double*)Xr);
  else
    gather_x_kernel<float><<<blocks, 256, 0, st>>>((const float*)X, m, ldx, perm, r, (float*)Xr);
  return cudaGetLastError();
}

}  // namespace rcq
