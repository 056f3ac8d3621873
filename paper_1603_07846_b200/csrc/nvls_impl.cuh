// C5 server-group exchange through NVSwitch multicast (NVLS; SURVEY §8(f)
// NEXT-1 (i); §5.2.1 AllReduce framework P:419-422, Updater P:282-284,
// "broadcast back" P:586).  The Param buffer (grad_full | w_full) is allocated
// by ncclMemAlloc and registered as a symmetric NCCL window; NCCL's device API
// (ncclDevCommCreate with lsaMultimem) hands each kernel a multicast view of it.
// One kernel per step:
//   LSA barrier (every rank's gradient complete)
//   -> multimem.ld_reduce.add over rank r's shard: the SUM of the K gradients
//      is computed by the switch (the summation order is the switch's, not the
//      oracle's ascending rank order: parity within fp32 rounding)
//   -> the Updater on the shard (master = the rank's slice of w_full)
//   -> multimem.st of the new weights: the switch writes them into every rank
//   -> LSA barrier (every rank's stores landed).
// Per rank and shard element: one multicast load and one multicast store over
// NVLink, instead of K-1 peer loads and K-1 peer stores.
// (Included at the end of runtime.cu: it needs sg_cluster and lr_at.)
#pragma once
#include <nccl_device.h>

namespace sg_nvls {

constexpr int kNvlsBlocks = 592;  // CTAs of the exchange kernel (4 per SM; one LSA barrier each)
constexpr int kNvlsUnroll = 4;    // float4 per thread per round: all multicast loads in flight first

__device__ __forceinline__ float4 mm_ld_reduce_add(const float* p) {
  float4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ void mm_st(float* p, float4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}

__global__ void __launch_bounds__(256) nvls_sync_kernel(ncclWindow_t win, ncclDevComm dc, float* __restrict__ v,
                                                        long long n, long long shard, int rank, const float* lr_dev,
                                                        float mu, float wd, float s) {
  ncclCoopCta coop;
  ncclLsaBarrierSession<ncclCoopCta> bar(coop, dc, ncclTeamTagLsa{}, blockIdx.x, /*multimem=*/true);
  bar.sync(coop, cuda::memory_order_acq_rel);  // every rank's gradient is complete
  const float* gmc = static_cast<const float*>(ncclGetLsaMultimemPointer(win, 0, dc));
  float* wmc = static_cast<float*>(ncclGetLsaMultimemPointer(win, (size_t)n * sizeof(float), dc));
  float* wl = static_cast<float*>(ncclGetLocalPointer(win, (size_t)n * sizeof(float)));
  const float lr = lr_dev[0];
  const long long base = (long long)rank * shard, n4 = shard >> 2;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < n4; i0 += kNvlsUnroll * stride) {
    float4 g[kNvlsUnroll];
#pragma unroll
    for (int u = 0; u < kNvlsUnroll; ++u)
      if (i0 + u * stride < n4) g[u] = mm_ld_reduce_add(gmc + base + 4 * (i0 + u * stride));
#pragma unroll
    for (int u = 0; u < kNvlsUnroll; ++u) {
      const long long i = i0 + u * stride;
      if (i >= n4) break;
      float4 w = reinterpret_cast<const float4*>(wl + base)[i];
      float4 h = reinterpret_cast<float4*>(v)[i];
      sg::sgd1(w.x, g[u].x, h.x, lr, mu, wd, s);
      sg::sgd1(w.y, g[u].y, h.y, lr, mu, wd, s);
      sg::sgd1(w.z, g[u].z, h.z, lr, mu, wd, s);
      sg::sgd1(w.w, g[u].w, h.w, lr, mu, wd, s);
      reinterpret_cast<float4*>(v)[i] = h;
      mm_st(wmc + base + 4 * i, w);
    }
  }
  bar.sync(coop, cuda::memory_order_acq_rel);  // every rank's stores landed
}

}  // namespace sg_nvls

struct sg_nvls_sync {
  sg_cluster* c = nullptr;
  int64_t n = 0;
  float* buf = nullptr;  // [grad_full (n) | w_full (n)], ncclMemAlloc, symmetric window
  float* v = nullptr;    // history shard
  float* lr = nullptr;
  ncclWindow_t win = nullptr;
  ncclDevComm dc{};
  bool dc_made = false;
};

extern "C" {

SG_API sg_status sg_nvls_sync_create(sg_cluster* c, int64_t n, sg_nvls_sync** out, float** grad_full_dev,
                                     float** w_full_dev, float** v_shard_dev) {
  SG_CHECK(c && out && grad_full_dev && w_full_dev && v_shard_dev, SG_ERR_INVALID_ARG,
           "sg_nvls_sync_create: null argument");
  SG_CHECK(n > 0 && n % (32LL * c->world) == 0, SG_ERR_PARTITION, "partition error: n=%lld not a multiple of 32*K=%d",
           (long long)n, 32 * c->world);
  SG_CUDA(cudaSetDevice(c->device));
  sg_nvls_sync* p = new sg_nvls_sync();
  p->c = c;
  p->n = n;
  const size_t bytes = ((size_t)2 * n * sizeof(float) + 4095) / 4096 * 4096;
  auto fail = [&](sg_status st, const char* what, const char* why) {
    if (p->dc_made) ncclDevCommDestroy(c->comm_par, &p->dc);
    if (p->win) ncclCommWindowDeregister(c->comm_par, p->win);
    if (p->buf) ncclMemFree(p->buf);
    cudaFree(p->v);
    cudaFree(p->lr);
    delete p;
    SG_FAIL(st, "sg_nvls_sync_create: %s: %s", what, why);
  };
  // every step below is collective: a failure is returned by every rank alike
  ncclResult_t r = ncclMemAlloc(reinterpret_cast<void**>(&p->buf), bytes);
  if (r != ncclSuccess) return fail(SG_ERR_OOM, "ncclMemAlloc", ncclGetErrorString(r));
  cudaError_t e = cudaMemset(p->buf, 0, bytes);
  if (e == cudaSuccess) e = cudaMalloc(&p->v, n / c->world * sizeof(float));
  if (e == cudaSuccess) e = cudaMemset(p->v, 0, n / c->world * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&p->lr, sizeof(float));
  if (e != cudaSuccess) return fail(SG_ERR_OOM, "allocation", cudaGetErrorString(e));
  r = ncclCommWindowRegister(c->comm_par, p->buf, bytes, &p->win, NCCL_WIN_COLL_SYMMETRIC);
  if (r != ncclSuccess) return fail(SG_ERR_UNSUPPORTED, "window registration", ncclGetErrorString(r));
  ncclDevCommRequirements req{};
  req.lsaMultimem = true;
  req.lsaBarrierCount = sg_nvls::kNvlsBlocks;
  r = ncclDevCommCreate(c->comm_par, &req, &p->dc);
  if (r != ncclSuccess) return fail(SG_ERR_UNSUPPORTED, "ncclDevCommCreate (NVLS multimem)", ncclGetErrorString(r));
  p->dc_made = true;
  *grad_full_dev = p->buf;
  *w_full_dev = p->buf + n;
  *v_shard_dev = p->v;
  *out = p;
  return SG_OK;
}

SG_API sg_status sg_nvls_sync_step(sg_nvls_sync* p, const sg_updater_cfg* cfg, int64_t step, void* stream) {
  SG_CHECK(p && cfg, SG_ERR_INVALID_ARG, "sg_nvls_sync_step: null argument");
  sg_cluster* c = p->c;
  SG_CUDA(cudaSetDevice(c->device));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const float s = cfg->grad_scale > 0 ? cfg->grad_scale : 1.f / c->world;
  SG_CUDA(sg::fill_scalar(p->lr, lr_at(*cfg, step), st));
  const int64_t shard = p->n / c->world;
  sg_nvls::nvls_sync_kernel<<<sg_nvls::kNvlsBlocks, 256, 0, st>>>(p->win, p->dc, p->v, p->n, shard, c->rank, p->lr, cfg->momentum,
                                                cfg->weight_decay, s);
  ++sg::g_kernel_launches;
  SG_CUDA(cudaGetLastError());
  return SG_OK;
}

SG_API sg_status sg_nvls_sync_destroy(sg_nvls_sync* p) {
  if (!p) return SG_OK;
  sg_cluster* c = p->c;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  if (p->dc_made) ncclDevCommDestroy(c->comm_par, &p->dc);
  if (p->win) ncclCommWindowDeregister(c->comm_par, p->win);
  if (p->buf) ncclMemFree(p->buf);
  cudaFree(p->v);
  cudaFree(p->lr);
  delete p;
  return SG_OK;
}

}  // extern "C"
