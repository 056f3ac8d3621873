// Microbenchmark (not part of the library): cycles per tcgen05.mma kind::tf32
// (M = 128, K = 8) by operand layout (K-major SWIZZLE_128B / MN-major
// SWIZZLE_128B_BASE32B) and commit cadence, one issuing thread.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//        -I paper_1603_07846_b200/csrc tools/mma_layout_rate.cu -o tools/mma_layout_rate
#include <cstdio>

#include "sg_common.cuh"

using namespace sg;

__device__ __forceinline__ void mma_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t acc) {
  asm volatile(
      "{\n .reg .pred e, p;\n elect.sync _|e, 0xffffffff;\n setp.ne.b32 p, %4, 0;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit_elect(uint32_t bar) {
  asm volatile(
      "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(bar)
      : "memory");
}

template <int N>
__global__ void rate_warp(long long* out, int iters, int amn, int bmn, int commit_every) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar, bar2;
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x)
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(base + i * 4), "f"(0.001f * (i & 255)));
  fence_proxy_async_smem();
  if (threadIdx.x < 32) tmem_alloc<256>(smem_u32(&slot));
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    mbar_init(smem_u32(&bar2), 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x < 32) {
    const uint32_t A = base, B = base + 65536;
    constexpr int KL = 32;
    const uint32_t idesc = idesc_tf32(128, N, amn, bmn);
    auto adesc = [&](int kk) {
      return amn ? umma_desc_mn_sw128_32b(A + kk * 8 * 128, KL * 128, 512) : umma_desc_sw128(A + kk * 32, 16, 1024);
    };
    auto bdesc = [&](int kk) {
      return bmn ? umma_desc_mn_sw128_32b(B + kk * 8 * 128, KL * 128, 512) : umma_desc_sw128(B + kk * 32, 16, 1024);
    };
    for (int i = 0; i < 8; ++i) mma_elect(tmem, adesc(i & 3), bdesc(i & 3), idesc, 1);
    commit_elect(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      mma_elect(tmem, adesc(i & 3), bdesc(i & 3), idesc, 1);
      if (commit_every && (i & (commit_every - 1)) == commit_every - 1) commit_elect(smem_u32(&bar2));
    }
    commit_elect(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 1);
    if (threadIdx.x == 0) out[0] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}

template <int N>
__global__ void rate(long long* out, int iters, int amn, int bmn, int commit_every) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar, bar2;
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x)
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(base + i * 4), "f"(0.001f * (i & 255)));
  fence_proxy_async_smem();
  if (threadIdx.x < 32) tmem_alloc<256>(smem_u32(&slot));
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    mbar_init(smem_u32(&bar2), 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    // A: 128 rows x 32 k-lines (4 KB per 8 k) ; B at +64 KB
    const uint32_t A = base, B = base + 65536;
    constexpr int KL = 32;  // k-lines per stage
    const uint32_t idesc = idesc_tf32(128, N, amn, bmn);
    auto adesc = [&](int kk) {
      return amn ? umma_desc_mn_sw128_32b(A + kk * 8 * 128, KL * 128, 512) : umma_desc_sw128(A + kk * 32, 16, 1024);
    };
    auto bdesc = [&](int kk) {
      return bmn ? umma_desc_mn_sw128_32b(B + kk * 8 * 128, KL * 128, 512) : umma_desc_sw128(B + kk * 32, 16, 1024);
    };
    for (int i = 0; i < 8; ++i) mma_tf32(tmem, adesc(i & 3), bdesc(i & 3), idesc, 1);
    mma_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      mma_tf32(tmem, adesc(i & 3), bdesc(i & 3), idesc, 1);
      if (commit_every && i % commit_every == commit_every - 1) mma_commit(smem_u32(&bar2));
    }
    mma_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 1);
    out[0] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}

template <int N>
void run(long long* d) {
  const int iters = 4096;
  cudaFuncSetAttribute(rate<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int amn = 0; amn < 2; ++amn)
    for (int bmn = amn; bmn < amn + 1; ++bmn)
      for (int ce : {0, 4, 16, 4096}) {
        rate<N><<<1, 128, 200 * 1024>>>(d, iters, amn, bmn, ce);
        long long h = 0;
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("N=%3d A %s B %s commit every %2d: %6.1f cycles / MMA\n", N, amn ? "MN" : "K ", bmn ? "MN" : "K ", ce,
               (double)h / iters);
        cudaFuncSetAttribute(rate_warp<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        rate_warp<N><<<1, 128, 200 * 1024>>>(d, iters, amn, bmn, ce);
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("   whole-warp + elect.sync:      %6.1f cycles / MMA\n", (double)h / iters);
      }
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  run<32>(d);
  run<64>(d);
  run<128>(d);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
