// Microbenchmark (not part of the library): cycles per tcgen05.mma kind::tf32
// (M = 128, K = 8, cta_group::1) as a function of N, operands K-major
// SWIZZLE_128B in shared memory (contents irrelevant), one issuing thread.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//        -I paper_1603_07846_b200/csrc tools/mma_rate.cu -o tools/mma_rate
#include <cstdio>

#include "sg_common.cuh"

using namespace sg;

template <int N>
__global__ void mma_rate(long long* out, int iters, int mode, int fill, int nowarm) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar, bar2;
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
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
  if (fill) {  // pseudo-random finite operands in the whole operand region
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) {
      const uint32_t h = (uint32_t)i * 2654435761u;
      const float v = (float)((h >> 8) & 0xffff) / 65536.f - 0.5f;
      asm volatile("st.shared.f32 [%0], %1;" ::"r"(base + i * 4), "f"(v));
    }
    fence_proxy_async_smem();
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const uint64_t ad = umma_desc_sw128(base, 16, 1024);
    const uint64_t bd = umma_desc_sw128(base + 65536, 16, 1024);  // 25 taps x 4 KB fit below 200 KB
    constexpr uint32_t idesc = idesc_tf32(128, N, 0, 0);
    // warm-up (cfg 1 skips it)
    if (!nowarm) for (int i = 0; i < 8; ++i) mma_tf32(tmem, ad, bd, idesc, 1);
    mma_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
    long long t0 = clock64();
    if (mode == 0) {
      for (int i = 0; i < iters; ++i) mma_tf32(tmem, ad + (i & 3) * 2, bd + (i & 3) * 2, idesc, 1);
    } else if (mode == 1) {  // A start shifted by 3 rows (not 8-row aligned)
      for (int i = 0; i < iters; ++i) mma_tf32(tmem, ad + 24 + (i & 3) * 2, bd + (i & 3) * 2, idesc, 1);
    } else if (mode == 3) {  // accumulator switches between 3 TMEM column blocks every 4 MMAs
      for (int i = 0; i < iters; ++i)
        mma_tf32(tmem + ((i >> 2) % 3) * N, ad + (i & 3) * 2, bd + (i & 3) * 2, idesc, 1);
    } else if (mode == 4) {  // conv-like: group g of 4 MMAs reads A rows shifted by 20*g + g%5
      for (int i = 0; i < iters; ++i) {
        const int g = (i >> 2) % 25;
        mma_tf32(tmem + ((i >> 2) % 3) * N, ad + (uint64_t)(((g / 5) * 20 + g % 5) * 8) + (i & 3) * 2,
                 bd + (i & 3) * 2, idesc, 1);
      }
    } else if (mode == 5) {  // mode 4 + a tcgen05.commit after every 12 MMAs (one conv tap)
      for (int i = 0; i < iters; ++i) {
        const int g = (i >> 2) % 25;
        mma_tf32(tmem + ((i >> 2) % 3) * N, ad + (uint64_t)(((g / 5) * 20 + g % 5) * 8) + (i & 3) * 2,
                 bd + (i & 3) * 2, idesc, 1);
        if (i % 12 == 11) mma_commit(smem_u32(&bar2));
      }
    } else if (mode == 6) {  // mode 4 + fence.proxy.async + tcgen05 fence every 12 MMAs
      for (int i = 0; i < iters; ++i) {
        const int g = (i >> 2) % 25;
        mma_tf32(tmem + ((i >> 2) % 3) * N, ad + (uint64_t)(((g / 5) * 20 + g % 5) * 8) + (i & 3) * 2,
                 bd + (i & 3) * 2, idesc, 1);
        if (i % 12 == 11) {
          fence_proxy_async_smem();
          tc_fence_after();
        }
      }
    } else if (mode == 7) {  // exact conv_img issue loop: 25 taps x 3 tiles x 4 kk, lo/hi descriptors
      const uint32_t a_lo0 = (uint32_t)ad, a_hi = (uint32_t)(ad >> 32);
      const uint32_t b_lo0 = (uint32_t)bd, b_hi = (uint32_t)(bd >> 32);
      for (int rep = 0; rep < iters / 300; ++rep)
        for (int t = 0; t < 25; ++t) {
          const int r = t / 5, sc = t - r * 5;
          const uint32_t a_t = a_lo0 + (uint32_t)(r * 20 + sc) * 8;
          const uint32_t b_t = b_lo0 + (uint32_t)(t * 4096) / 16 * (fill > 1 ? 1 : 0);
          for (int i = 0; i < 3; ++i) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_tf32_lh(tmem + i * N, a_t + i * 1024 + kk * 2, a_hi, b_t + kk * 2, b_hi, idesc, 1);
          }
        }
    } else {  // A walks over 3 different 128-row tiles (no operand reuse between MMAs)
      for (int i = 0; i < iters; ++i)
        mma_tf32(tmem, ad + ((i % 3) * 128 * 128 >> 4) * 0 + (i & 3) * 2 + ((i >> 2) % 3) * (16384 >> 4), bd + (i & 3) * 2, idesc, 1);
    }
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
  const int iters = 4200;
  cudaFuncSetAttribute(mma_rate<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(mma_rate<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int mode = 7; mode < 8; ++mode)
  for (int cfg = 0; cfg < 3; ++cfg) {
    const int fill = 2;
    const int thr = 192, sm = 200 * 1024;
    const int it = cfg == 2 ? iters : 300;  // cfg 0/1: one conv pass of 300 MMAs (1: no warm-up)
    mma_rate<N><<<1, thr, sm>>>(d, it, mode, fill, cfg == 1);
    long long h = 0;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double cyc = (double)h / (cfg == 2 ? iters : 300);
    printf("cfg=%d N=%3d mode %d: %6.1f cycles per 128x%dx8 MMA  -> %7.0f MAC/clk/SM\n", cfg, N, mode, cyc, N, 128.0 * N * 8 / cyc);
  }
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
