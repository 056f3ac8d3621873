// Microbenchmark (not part of the library): cycles per tcgen05.mma kind::tf32
// (M = 128, K = 8, cta_group::1) as a function of N, operands K-major
// SWIZZLE_128B in shared memory (contents irrelevant), one issuing thread.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//        -I paper_1603_07846_b200/csrc tools/mma_rate.cu -o tools/mma_rate
#include <cstdio>

#include "sg_common.cuh"

using namespace sg;

template <int N>
__global__ void mma_rate(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  if (threadIdx.x < 32) tmem_alloc<256>(smem_u32(&slot));
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint64_t ad = umma_desc_sw128(base, 16, 1024);
    const uint64_t bd = umma_desc_sw128(base + 16384, 16, 1024);
    constexpr uint32_t idesc = idesc_tf32(128, N, 0, 0);
    // warm-up
    for (int i = 0; i < 8; ++i) mma_tf32(tmem, ad, bd, idesc, 1);
    mma_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) mma_tf32(tmem, ad + (i & 3) * 2, bd + (i & 3) * 2, idesc, 1);
    mma_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 1);
    long long t1 = clock64();
    out[0] = t1 - t0;
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
  cudaFuncSetAttribute(mma_rate<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  mma_rate<N><<<1, 128, 64 * 1024>>>(d, iters);
  long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double cyc = (double)h / iters;
  printf("N=%3d: %6.1f cycles per 128x%dx8 MMA  -> %7.0f MAC/clk/SM\n", N, cyc, N, 128.0 * N * 8 / cyc);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  run<16>(d);
  run<32>(d);
  run<64>(d);
  run<128>(d);
  run<256>(d);
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
