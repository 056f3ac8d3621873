// Probe (not part of the library): SWIZZLE_32B variant.  Can a tcgen05.mma K-major SWIZZLE_32B A
// operand start at an arbitrary 128-byte row inside the swizzle pattern?  The
// smem tile holds X[row][32 floats] in the TMA SWIZZLE_128B layout (16-byte
// chunk c of row r at r*128 + ((c ^ (r & 7)) << 4), 1024-byte aligned base).
// For row shifts d = 0..15 the MMA reads A rows d .. d+127 with the descriptor
// start moved by d*128 bytes and the 3-bit base-offset field set to each of
// {0, d & 7}; the result is compared with the CPU product.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//        -I paper_1603_07846_b200/csrc tools/desc_shift.cu -o tools/desc_shift
#include <cmath>
#include <cstdio>
#include <vector>

#include "sg_common.cuh"

using namespace sg;

constexpr int ROWS = 160, NB = 32;  // rows of 8 floats (32 B)

__global__ void probe(const float* X, const float* W, float* out, int d, int bo_mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  const uint32_t bbase = base + ROWS * 32 + 1024 - (ROWS * 32) % 1024;  // B: NB rows x 32 B
  const int tid = threadIdx.x;
  for (int i = tid; i < ROWS * 2; i += blockDim.x) {
    const int r = i >> 1, c = i & 1;
    const float4 v = reinterpret_cast<const float4*>(X)[r * 2 + c];
    const uint32_t a = base + r * 32 + ((c ^ ((r >> 2) & 1)) << 4);
    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w));
  }
  for (int i = tid; i < NB * 2; i += blockDim.x) {
    const int r = i >> 1, c = i & 1;
    const float4 v = reinterpret_cast<const float4*>(W)[r * 2 + c];
    const uint32_t a = bbase + r * 32 + ((c ^ ((r >> 2) & 1)) << 4);
    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w));
  }
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
    {
      // layout type 6 = SWIZZLE_32B; SBO = 8 rows x 32 B = 256 B
      uint64_t ad = umma_desc_sw128(base + d * 32, 16, 256);
      ad = (ad & ~((uint64_t)7 << 61)) | ((uint64_t)6 << 61);
      const uint64_t bo = bo_mode == 0 ? 0 : bo_mode == 1 ? (uint64_t)(d & 7) : (uint64_t)((8 - (d & 7)) & 7);
      ad |= bo << 49;
      uint64_t bd = umma_desc_sw128(bbase, 16, 256);
      bd = (bd & ~((uint64_t)7 << 61)) | ((uint64_t)6 << 61);
      mma_tf32(tmem, ad, bd, idesc, 0u);
    }
    mma_commit(smem_u32(&bar));
  }
  __syncwarp();
  mbar_wait(smem_u32(&bar), 0);
  tc_fence_after();
  // 4 warps x 32 lanes = 128 rows, 32 columns
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
  std::vector<float> X(ROWS * 8), W(NB * 8), O(128 * NB);
  for (int i = 0; i < ROWS * 8; ++i) X[i] = (float)((i * 7 + 3) % 13 - 6);
  for (int i = 0; i < NB * 8; ++i) W[i] = (float)((i * 5 + 1) % 11 - 5);
  float *dX, *dW, *dO;
  cudaMalloc(&dX, X.size() * 4);
  cudaMalloc(&dW, W.size() * 4);
  cudaMalloc(&dO, O.size() * 4);
  cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dW, W.data(), W.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int d = 0; d < 16; ++d) {
    printf("d=%2d:", d);
    for (int mode = 0; mode < 3; ++mode) {
      cudaMemset(dO, 0, O.size() * 4);
      probe<<<1, 128, 64 * 1024>>>(dX, dW, dO, d, mode);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
      double err = 0, ref = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < NB; ++n) {
          double acc = 0;
          for (int k = 0; k < 8; ++k) acc += (double)X[(d + m) * 8 + k] * W[n * 8 + k];
          err += (O[m * NB + n] - acc) * (O[m * NB + n] - acc);
          ref += acc * acc;
        }
      printf("  bo=%s %s rel=%.2e", mode == 0 ? "0   " : mode == 1 ? "d&7 " : "-d&7", e ? cudaGetErrorString(e) : "ok",
             std::sqrt(err / ref));
    }
    printf("\n");
  }
  return 0;
}
