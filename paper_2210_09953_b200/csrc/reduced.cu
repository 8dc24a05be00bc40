// reduced.cu -- step 3 of the reduced RCholeskyQR (Alg. 5): Z = Y R^{-1} for the
// small l x n extract Y = L X.  Z is l x n, tiny next to X, so this is a latency-bound
// "low-dimensional operation": one warp per row of Y, forward substitution in the
// right-looking (axpy) order -- after z_j = s_j / R_jj every lane updates its residuals
// s_c -= z_j R_jc, c > j -- so each s_c subtracts z_0 R_0c, z_1 R_1c, ... in ascending order,
// with separately rounded products and differences (no FMA contraction), like the oracle's
// row-wise substitution.  Steps 1 and 2 (the one-pass (k + l)-row sketch, the QR) are the
// Alg. 2 kernels (api.cu).
#include <cuda_runtime.h>
#include <algorithm>
#include "internal.cuh"

namespace rcq {

constexpr int RS_WARPS = 8;

__global__ void __launch_bounds__(32 * RS_WARPS)
rowsub_kernel(const double* __restrict__ Y, int64_t l, int n, const double* __restrict__ R, double* __restrict__ Z,
              const int* status) {
  if (*status) return;
  extern __shared__ double rs_s[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * RS_WARPS + warp;
  if (row >= l) return;
  double* s = rs_s + (size_t)warp * n;
  for (int c = lane; c < n; c += 32) s[c] = Y[row * n + c];
  __syncwarp();
  for (int j = 0; j < n; ++j) {
    const double zj = __ddiv_rn(s[j], R[(size_t)j * n + j]);
    for (int c = j + 1 + lane; c < n; c += 32) s[c] = __dsub_rn(s[c], __dmul_rn(zj, R[(size_t)j * n + c]));
    if (lane == 0) Z[row * n + j] = zj;
    __syncwarp();
  }
}

cudaError_t launch_rowsub(const double* Y, int64_t l, int n, const double* R, double* Z, const int* status,
                          cudaStream_t st) {
  if (l <= 0) return cudaSuccess;
  const size_t smem = sizeof(double) * (size_t)n * RS_WARPS;
  cudaError_t e = cudaFuncSetAttribute(rowsub_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const unsigned blocks = (unsigned)((l + RS_WARPS - 1) / RS_WARPS);
  rowsub_kernel<<<blocks, 32 * RS_WARPS, smem, st>>>(Y, l, n, R, Z, status);
  return cudaGetLastError();
}

}  // namespace rcq
