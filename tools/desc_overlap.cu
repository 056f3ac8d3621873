// Probe (not part of the library): a K-major SWIZZLE_NONE tcgen05 operand whose
// core matrices overlap.  X[p][4] (16 B per pixel, contiguous); descriptor with
// SBO = 128 B (8 rows) and LBO = 16 B (next 4 K elements = next pixel) should
// read A[m][k] = X[m + d + k/4][k % 4] (two 4-channel filter taps per K = 8).
// B = W[t][n][4] staged tap-major: LBO = NB*16 (next tap), SBO = 128.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//        -I paper_1603_07846_b200/csrc tools/desc_overlap.cu -o tools/desc_overlap
#include <cmath>
#include <cstdio>
#include <vector>

#include "sg_common.cuh"

using namespace sg;

constexpr int P = 200, NB = 32;

__global__ void probe(const float* X, const float* W, float* out, int d) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  const uint32_t bbase = base + 4096;
  const int tid = threadIdx.x;
  for (int i = tid; i < P * 4; i += blockDim.x) asm volatile("st.shared.f32 [%0], %1;" ::"r"(base + i * 4), "f"(X[i]));
  for (int i = tid; i < 2 * NB * 4; i += blockDim.x)
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(bbase + i * 4), "f"(W[i]));
  fence_proxy_async_smem();
  if (tid < 32) tmem_alloc<32>(smem_u32(&slot));
  if (tid == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (tid == 0) {
    constexpr uint32_t idesc = idesc_tf32(128, NB, 0, 0);
    const uint64_t ad = umma_desc_noswz(base + d * 16, 16, 128);
    const uint64_t bd = umma_desc_noswz(bbase, NB * 16, 128);
    mma_tf32(tmem, ad, bd, idesc, 0u);
    mma_commit(smem_u32(&bar));
  }
  __syncwarp();
  mbar_wait(smem_u32(&bar), 0);
  tc_fence_after();
  const int warp = tid >> 5, lane = tid & 31;
  if (warp < 4) {
    float v[16];
    for (int c0 = 0; c0 < NB; c0 += 16) {
      tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
      for (int i = 0; i < 16; ++i) out[(warp * 32 + lane) * NB + c0 + i] = v[i];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) {
    tc_fence_after();
    tmem_dealloc<32>(tmem);
  }
}

int main() {
  std::vector<float> X(P * 4), W(2 * NB * 4), O(128 * NB);
  for (int i = 0; i < P * 4; ++i) X[i] = (float)((i * 7 + 3) % 13 - 6);
  for (int i = 0; i < 2 * NB * 4; ++i) W[i] = (float)((i * 5 + 1) % 11 - 5);
  float *dX, *dW, *dO;
  cudaMalloc(&dX, X.size() * 4);
  cudaMalloc(&dW, W.size() * 4);
  cudaMalloc(&dO, O.size() * 4);
  cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dW, W.data(), W.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 1024);
  for (int d = 0; d < 6; ++d) {
    cudaMemset(dO, 0, O.size() * 4);
    probe<<<1, 128, 32 * 1024>>>(dX, dW, dO, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
    double err = 0, ref = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < NB; ++n) {
        double acc = 0;
        for (int k = 0; k < 8; ++k) acc += (double)X[(m + d + k / 4) * 4 + k % 4] * W[((k / 4) * NB + n) * 4 + k % 4];
        err += (O[m * NB + n] - acc) * (O[m * NB + n] - acc);
        ref += acc * acc;
      }
    printf("d=%d: %s rel=%.2e\n", d, e ? cudaGetErrorString(e) : "ok", std::sqrt(err / ref));
  }
  return 0;
}
