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

// ---------------------------------------------------------------------------------------------
// Column-major layout adapter (rcholqr_factor_colmajor): out(r, c) = in(c, r) through 32 x 33 shared
// tiles -- coalesced reads of the source's rows and writes of the destination's rows.
template <typename T>
__global__ void transpose_kernel(const T* __restrict__ in, int64_t rows, int64_t cols, int64_t ldi, T* __restrict__ out,
                                 int64_t ldo) {
  __shared__ T tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;   // tile of `in` (rows x cols)
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t r = r0 + y, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[y][threadIdx.x] = in[r * ldi + c];
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t c = c0 + y, r = r0 + threadIdx.x;                               // out is cols x rows
    if (r < rows && c < cols) out[c * ldo + r] = tile[threadIdx.x][y];
  }
}

cudaError_t launch_transpose(const void* in, int64_t rows, int64_t cols, int64_t ldi, void* out, int64_t ldo,
                             size_t es, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  const dim3 block(32, 8), grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
  if (grid.y > 65535u) {                                         // very tall: chunk the rows
    const int64_t chunk = (int64_t)65535 * 32;
    for (int64_t r = 0; r < rows; r += chunk) {
      const int64_t rr = std::min(chunk, rows - r);
      cudaError_t e = launch_transpose((const char*)in + (size_t)r * ldi * es, rr, cols, ldi,
                                       (char*)out + (size_t)r * es, ldo, es, st);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  if (es == 8) transpose_kernel<double><<<grid, block, 0, st>>>((const double*)in, rows, cols, ldi, (double*)out, ldo);
  else transpose_kernel<float><<<grid, block, 0, st>>>((const float*)in, rows, cols, ldi, (float*)out, ldo);
  return cudaGetLastError();
}

}  // namespace rcq
