#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  float* p; cudaMalloc(&p, 128 * 16 * 16 * 32 * 4);
  CUtensorMap m; cuuint32_t es[4] = {1, 1, 1, 1};
  // image {C=32, W=16, H=16, N=128}
  cuuint64_t d[4] = {32, 16, 16, 128}; cuuint64_t st[3] = {128, 16 * 128, 256 * 128};
  cuuint32_t b1[4] = {32, 20, 24, 1}, b2[4] = {32, 16, 16, 1}, b3[4] = {32, 16, 24, 1};
  printf("box>W: %d\n", (int)enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, p, d, st, b1, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  printf("box=dims: %d\n", (int)enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, p, d, st, b2, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  printf("box>H: %d\n", (int)enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, p, d, st, b3, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  // filter {C=32, Co=32, T=25} strides {25*32*4, 32*4}
  cuuint64_t wd[3] = {32, 32, 25}; cuuint64_t ws[2] = {25 * 32 * 4, 32 * 4};
  cuuint32_t wb[3] = {32, 32, 25};
  printf("W box: %d\n", (int)enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, p, wd, ws, wb, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  cuuint64_t ws2[2] = {32 * 4, 25 * 32 * 4}; cuuint64_t wd2[3] = {32, 25, 32};
  printf("W box natural order: %d\n", (int)enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, p, wd2, ws2, wb, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  return 0;
}
