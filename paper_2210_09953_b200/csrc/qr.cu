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
#include <cstdlib>
#include <utility>
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

// (beta, v0, raw R_jj) of a pivot column from ||A[j:,j]||^2 and A[j][j].
__device__ __forceinline__ void pivot_params(double ss, double x0, double* par) {
  const double alpha = sqrt(ss);
  const double sgn = x0 >= 0.0 ? 1.0 : -1.0;
  const double v0 = x0 + sgn * alpha;
  par[0] = alpha == 0.0 ? 0.0 : 1.0 / (alpha * fabs(v0));   // beta
  par[1] = v0;
  par[2] = alpha == 0.0 ? 0.0 : -sgn * alpha;               // raw R_jj
}

// Register-resident variant (k <= 32*RPL, n <= 16*CPW; configs C1, C2, C4): 16 warps own the
// columns cyclically (column l -> warp l % 16, slot l / 16) and lane L holds rows L, L+32, ... of
// every owned column in registers.  Per column j only the Householder vector v_j (k doubles) goes
// through shared memory: the owner of column j+1 updates that column first, computes its norm,
// publishes (beta, v0, R_jj) and v_{j+1}, then all warps update their other columns two at a time
// (two dot products and reductions in flight).  One barrier per column; rows above the pivot need no
// predicate because v_j is zero there.

// Pivot column j sits in slot C (compile time) of warp j % 16: norm below row j, pivot parameters,
// v_j into shared memory (and the reflector into the global workspace for S).
template <int CPW, int RPL, int C, int NW>
__device__ __forceinline__ void qr_publish(const double (&col)[CPW][RPL], int j, int k, int n, int lane,
                                           double (*vbuf)[32 * RPL], double (*sh_par)[3], double* Aglob,
                                           double* diag_out, double* tau_out) {
  double ss = 0.0, x0 = 0.0;
#pragma unroll
  for (int r = 0; r < RPL; ++r) {
    const int i = r * 32 + lane;
    const double v = col[C][r];
    ss = fma(i >= j ? v : 0.0, v, ss);
    x0 = (i == j) ? v : x0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
    x0 += __shfl_xor_sync(0xffffffffu, x0, o);
  }
  double par[3];
  pivot_params(ss, x0, par);
  if (lane == 0) {
    sh_par[j & 1][0] = par[0]; sh_par[j & 1][1] = par[1]; sh_par[j & 1][2] = par[2];
    tau_out[j] = par[0]; diag_out[j] = par[2]; diag_out[n + j] = par[1];
  }
#pragma unroll
  for (int r = 0; r < RPL; ++r) {
    const int i = r * 32 + lane;
    const double v = i < j ? 0.0 : (i == j ? par[1] : col[C][r]);
    vbuf[j & 1][i] = v;
    if (i < k) Aglob[(size_t)j * k + i] = v;            // reflector (head v0 on the diagonal)
  }
}

// A[:, slot C] -= v (beta v^T A[:, slot C]) for this warp's column in slot C (v = vbuf, zero above j).
template <int CPW, int RPL, int C>
__device__ __forceinline__ void qr_update1(double (&col)[CPW][RPL], const double* vr, double beta) {
  double w = 0.0;
#pragma unroll
  for (int r = 0; r < RPL; ++r) w = fma(vr[32 * r], col[C][r], w);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
  w *= beta;
#pragma unroll
  for (int r = 0; r < RPL; ++r) col[C][r] = fma(-vr[32 * r], w, col[C][r]);
}

// Register-resident variant (k <= 32*RPL, n <= 16*CPW; configs C1, C2, C4): 16 warps own the
// columns cyclically (column l -> warp l % 16, slot l / 16) and lane L holds rows L, L+32, ... of
// every owned column in registers.  Per column j only the Householder vector v_j (k doubles) goes
// through shared memory: the owner of column j+1 updates that column first and publishes pivot
// j+1, then every warp updates its remaining live columns with all dot products and reductions in
// flight together.  One barrier per column.  The column loop is unrolled over slots so every slot
// index is a compile-time constant (no dynamic register-array indexing).
template <int CPW, int RPL, int NW>
__global__ void __launch_bounds__(32 * NW, 1)
householder_reg_kernel(const double* __restrict__ P, int k, int n, double* __restrict__ R,
                       double* __restrict__ Aglob, double* __restrict__ diag_out, double* __restrict__ tau_out,
                       int* status) {
  __shared__ double vbuf[2][32 * RPL];
  __shared__ double sh_par[2][3];
  __shared__ int sh_flag;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) sh_flag = 0;
  __syncthreads();
  double col[CPW][RPL];
  int bad = 0;
#pragma unroll
  for (int c = 0; c < CPW; ++c) {
    const int l = warp + NW * c;
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int i = r * 32 + lane;
      double v = 0.0;
      if (l < n && i < k) v = P[(size_t)i * n + l];
      if (!isfinite(v)) bad = 1;
      col[c][r] = v;
    }
  }
  if (__syncthreads_or(bad)) {
    for (int c = tid; c < n * n; c += 32 * NW) R[c] = 0.0;
    if (tid == 0) atomicOr(status, kStNonfinite);
    return;
  }
  if (warp == 0) qr_publish<CPW, RPL, 0, NW>(col, 0, k, n, lane, vbuf, sh_par, Aglob, diag_out, tau_out);
  __syncthreads();
  auto step = [&](auto CC, int jj) {            // column j = 16*C + jj (owner: warp jj, slot C)
    constexpr int C = decltype(CC)::value;
    const int j = NW * C + jj;
    if (j >= n) return;
    const double beta = sh_par[j & 1][0];
    const double* vr = vbuf[j & 1] + lane;
    const int jn = j + 1;
    // owner of column j+1: warp jj+1 slot C, or warp 0 slot C+1 when jj == 15
    if (jn < n) {
      if (jj + 1 < NW) {
        if (warp == jj + 1) {
          if (beta != 0.0) qr_update1<CPW, RPL, C>(col, vr, beta);
          qr_publish<CPW, RPL, C, NW>(col, jn, k, n, lane, vbuf, sh_par, Aglob, diag_out, tau_out);
        }
      } else if constexpr (C + 1 < CPW) {
        if (warp == 0) {
          if (beta != 0.0) qr_update1<CPW, RPL, C + 1>(col, vr, beta);
          qr_publish<CPW, RPL, C + 1, NW>(col, jn, k, n, lane, vbuf, sh_par, Aglob, diag_out, tau_out);
        }
      }
    }
    // every other live owned column l > j+1: all dots, one interleaved reduction, all axpys
    if (beta != 0.0) {
      double w[CPW];
#pragma unroll
      for (int c = 0; c < CPW; ++c) w[c] = 0.0;
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        const double v = vr[32 * r];
#pragma unroll
        for (int c = C; c < CPW; ++c) w[c] = fma(v, col[c][r], w[c]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int c = C; c < CPW; ++c) w[c] += __shfl_xor_sync(0xffffffffu, w[c], o);
#pragma unroll
      for (int c = C; c < CPW; ++c) {
        const int l = warp + NW * c;
        w[c] = (l > jn && l < n) ? w[c] * beta : 0.0;
      }
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        const double v = vr[32 * r];
#pragma unroll
        for (int c = C; c < CPW; ++c) col[c][r] = fma(-v, w[c], col[c][r]);
      }
    }
    // row j of R (raw; signs fixed at the end): A[j][l] for the owned columns l > j
    if (lane == (j & 31)) {
#pragma unroll
      for (int c = C; c < CPW; ++c) {
        const int l = warp + NW * c;
        if (l > j && l < n) {
#pragma unroll
          for (int r = 0; r < RPL; ++r)
            if (r == (j >> 5)) R[(size_t)j * n + l] = col[c][r];
        }
      }
    }
    __syncthreads();
  };
  [&]<int... Cs>(std::integer_sequence<int, Cs...>) {
    (([&] {
       for (int jj = 0; jj < NW; ++jj) step(std::integral_constant<int, Cs>{}, jj);
     }()), ...);
  }(std::make_integer_sequence<int, CPW>{});
  for (int c = tid; c < n * n; c += 32 * NW) {
    const int j = c / n, l = c % n;
    const double d = diag_out[j];
    const double sg = d < 0.0 ? -1.0 : 1.0;
    if (l < j) R[c] = 0.0;
    else if (l == j) R[c] = sg * d;
    else R[c] = sg * R[c];
  }
  if (tid < 32) {
    int b2 = 0;
    for (int j = lane; j < n; j += 32) {
      const double d = diag_out[j];
      if (d == 0.0 || !isfinite(d)) b2 = 1;
    }
    b2 = __any_sync(0xffffffffu, b2);
    if (lane == 0 && b2) atomicOr(status, kStSingular);
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
  if (getenv("RCHOLQR_QR_BLOCKED")) return kQrBlocked;   // experiments: blocked QR at any size
  if (need + 1024 <= std::min<size_t>(smem_optin, 220 * 1024)) return kQrSmem;
  return getenv("RCHOLQR_QR_UNBLOCKED") ? kQrGlobal : kQrBlocked;
}

cudaError_t launch_qr(int kind, const double* P, int k, int n, double* R, double* Awork, double* diag,
                      double* tau, double* qr_ws, int* status, cudaStream_t st) {
  if (kind == kQrBlocked && qr_ws) return launch_qr_blocked(P, k, n, R, Awork, diag, tau, qr_ws, status, st);
  if (k <= 32 * 4 && n <= 16 * 4) {
    householder_reg_kernel<4, 4, 16><<<1, 32 * 16, 0, st>>>(P, k, n, R, Awork, diag, tau, status);
  } else if (k <= 32 * 7 && n <= 16 * 7) {
    householder_reg_kernel<7, 7, 16><<<1, 32 * 16, 0, st>>>(P, k, n, R, Awork, diag, tau, status);
  } else if (kind == kQrSmem) {
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
