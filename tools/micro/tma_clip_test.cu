// Probe: does a 2D TMA tile clip the INNER dimension at element granularity when globalDim[0] * 4 is not a
// multiple of 16 bytes?  fp32 tensor, dims (m, n) with m = 103, pitch 104 floats.  A box of 32 x 4 at inner
// coordinate 96 covers rows 96..127: rows 103.. are out of bounds.
//   load : the padding element (row 103) holds 1e30 in global memory; in-bounds fill must be 0 if clipping is by element
//   store: shared tile = 5.0 everywhere; the padding element must keep its old value if clipping is by element
// Used by the native column-major kernels (solve_tc.cu, sketch_tc.cu), whose contiguous dimension is the ragged m.
#include <cstdint>
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap map, float* out, int c0) {
  __shared__ __align__(128) float tile[4 * 32];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&bar)), "r"(4 * 32 * 4) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
                 ::"r"(smem_u32(tile)), "l"(&map), "r"(c0), "r"(0), "r"(smem_u32(&bar)) : "memory");
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(smem_u32(&bar)) : "memory");
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 128; i += blockDim.x) out[i] = tile[i];
  __syncthreads();
  for (int i = threadIdx.x; i < 128; i += blockDim.x) tile[i] = 5.0f;
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];\n"
                 ::"l"(&map), "r"(smem_u32(tile)), "r"(c0), "r"(0) : "memory");
    asm volatile("cp.async.bulk.commit_group;\ncp.async.bulk.wait_group 0;\n" ::: "memory");
  }
}

int main() {
  using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  Fn enc = (Fn)p;
  for (int m : {103, 102, 101, 100}) {
    const int ld = 104, n = 4;
    float h[ld * n];
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < ld; ++i) h[j * ld + i] = i < m ? 1.0f : 1e30f;
    float *d, *o;
    cudaMalloc(&d, sizeof(h));
    cudaMalloc(&o, 128 * 4);
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    CUtensorMap map;
    const cuuint64_t dims[2] = {(cuuint64_t)m, (cuuint64_t)n}, str[1] = {ld * 4};
    const cuuint32_t box[2] = {32, 4}, es[2] = {1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("{\"m\": %d, \"encode\": %d}\n", m, (int)r); continue; }
    probe<<<1, 128>>>(map, o, 96);
    cudaError_t e = cudaDeviceSynchronize();
    float ho[128], hq[ld * n];
    cudaMemcpy(ho, o, sizeof(ho), cudaMemcpyDeviceToHost);
    cudaMemcpy(hq, d, sizeof(hq), cudaMemcpyDeviceToHost);
    int load_bad = 0, store_bad = 0, store_ok = 0;
    for (int j = 0; j < n; ++j)
      for (int i = 96; i < 128; ++i) {
        const float v = ho[j * 32 + (i - 96)];
        if (i < m ? v != 1.0f : v != 0.0f) ++load_bad;
      }
    for (int j = 0; j < n; ++j)
      for (int i = 96; i < ld; ++i) {
        if (i < m) store_ok += hq[j * ld + i] == 5.0f;
        else store_bad += hq[j * ld + i] != 1e30f;
      }
    printf("{\"m\": %d, \"cuda\": \"%s\", \"load_elements_wrong\": %d, \"store_inbounds_written\": %d, \"store_padding_overwritten\": %d, "
           "\"first_oob_loaded\": %g, \"first_pad_after_store\": %g}\n",
           m, cudaGetErrorString(e), load_bad, store_ok, store_bad, ho[m - 96], hq[m]);
    cudaFree(d); cudaFree(o);
  }
  return 0;
}
