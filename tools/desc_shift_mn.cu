// Probe (not part of the library): MN-major tf32 operands (SWIZZLE_128B_BASE32B)
// starting at an arbitrary 128-byte k-line, with the four 32-wide MN atoms of
// an M = 128 tile at a uniform k-line stride (LBO = dstep * 128 bytes, the atoms
// may overlap).  Smem holds X[k-line][32 floats] (k-line kr at kr*128, 32-byte
// granule g at (g ^ (kr & 3)) << 5), B = Y[k-line][32] in the same layout.
// D[a*32 + c][n] = sum_{k<32} X[d + a*dstep + k][c] * Y[k][n].
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//        -I paper_1603_07846_b200/csrc tools/desc_shift_mn.cu -o tools/desc_shift_mn
#include <cmath>
#include <cstdio>
#include <vector>

#include "sg_common.cuh"

using namespace sg;

constexpr int ROWS = 256, NB = 32, KB = 32;

__device__ __forceinline__ uint32_t mn_addr(uint32_t base, int kr, int c) {
  return base + kr * 128 + ((((c >> 3) ^ (kr & 3))) << 5) + (c & 7) * 4;
}

__global__ void probe(const float* X, const float* Y, float* out, int d, int dstep) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  const uint32_t bbase = base + ROWS * 128;
  const int tid = threadIdx.x;
  for (int i = tid; i < ROWS * 32; i += blockDim.x)
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(mn_addr(base, i >> 5, i & 31)), "f"(X[i]));
  for (int i = tid; i < KB * 32; i += blockDim.x)
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(mn_addr(bbase, i >> 5, i & 31)), "f"(Y[i]));
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
    constexpr uint32_t idesc = idesc_tf32(128, NB, 1, 1);
    for (int kk = 0; kk < KB / 8; ++kk) {
      const uint64_t ad = umma_desc_mn_sw128_32b(base + (d + kk * 8) * 128, dstep * 128, 512);
      const uint64_t bd = umma_desc_mn_sw128_32b(bbase + kk * 8 * 128, 4096, 512);
      mma_tf32(tmem, ad, bd, idesc, kk ? 1u : 0u);
    }
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
  std::vector<float> X(ROWS * 32), Y(KB * 32), O(128 * NB);
  for (int i = 0; i < ROWS * 32; ++i) X[i] = (float)((i * 7 + 3) % 13 - 6);
  for (int i = 0; i < KB * 32; ++i) Y[i] = (float)((i * 5 + 1) % 11 - 5);
  float *dX, *dY, *dO;
  cudaMalloc(&dX, X.size() * 4);
  cudaMalloc(&dY, Y.size() * 4);
  cudaMalloc(&dO, O.size() * 4);
  cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dY, Y.data(), Y.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int dsteps[] = {1, 5, 20, 32};
  for (int dstep : dsteps)
    for (int d = 0; d < 10; ++d) {
      cudaMemset(dO, 0, O.size() * 4);
      probe<<<1, 128, 64 * 1024>>>(dX, dY, dO, d, dstep);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
      double err = 0, ref = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < NB; ++n) {
          const int a = m >> 5, c = m & 31;
          double acc = 0;
          for (int k = 0; k < KB; ++k) acc += (double)X[(d + a * dstep + k) * 32 + c] * Y[k * 32 + n];
          err += (O[m * NB + n] - acc) * (O[m * NB + n] - acc);
          ref += acc * acc;
        }
      printf("dstep=%2d d=%d: %s rel=%.2e\n", dstep, d, e ? cudaGetErrorString(e) : "ok", std::sqrt(err / ref));
    }
  return 0;
}
