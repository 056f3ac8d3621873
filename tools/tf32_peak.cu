// Measured TF32 tensor-core ceiling of this B200 (not part of the library):
// every SM issues back-to-back tcgen05.mma kind::tf32 (cta_group::1, M = 128,
// N = 256, K = 8) on operands resident in shared memory -- no global traffic,
// so the rate is the tensor pipe's at the clocks the chip holds under load.
// Timed with CUDA events over several durations; prints one JSON line.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//        -I paper_1603_07846_b200/csrc tools/tf32_peak.cu -o tools/tf32_peak -lnvidia-ml
#include <cstdio>
#include <vector>

#include "sg_common.cuh"

using namespace sg;

__global__ void __launch_bounds__(128, 1) peak(int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x)
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(base + i * 4), "f"(1e-3f * (i & 63)));
  fence_proxy_async_smem();
  const int warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);
  if (warp == 0) tmem_alloc<512>(smem_u32(&slot));
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 0) {
    constexpr uint32_t idesc = idesc_tf32(128, 256, 0, 0);
    const uint64_t ad = umma_desc_sw128(base, 16, 1024), bd = umma_desc_sw128(base + 16384, 16, 1024);
    for (int i = 0; i < iters; ++i)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) mma_tf32_warp(tmem + (i & 1) * 256, ad + kk * 2, bd + kk * 2, idesc, 1u);
    mma_commit_warp(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(peak, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  peak<<<sms, 128, 64 * 1024>>>(2000);  // warm-up
  cudaDeviceSynchronize();
  double best = 0, sustained = 0;
  for (int iters : {20000, 20000, 20000, 200000}) {
    cudaEventRecord(e0);
    peak<<<sms, 128, 64 * 1024>>>(iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 128 * 256 * 8 * 4.0 * iters * sms;
    const double tf = flops / (ms * 1e-3) / 1e12;
    if (iters == 200000) sustained = tf; else if (tf > best) best = tf;
    fprintf(stderr, "iters %d: %.3f ms, %.1f TFLOP/s\n", iters, ms, tf);
  }
  printf("{\"tf32_tflops\": %.1f, \"tf32_tflops_sustained\": %.1f, \"sms\": %d, \"shape\": \"tcgen05.mma kind::tf32 "
         "cta_group::1 128x256x8, smem-resident operands, every SM\", \"error\": \"%s\"}\n",
         best, sustained, sms, cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
