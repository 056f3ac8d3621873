// Fused peer-memory exchange of the training step; see exchange.h.
#include <cstring>

#include "exchange.h"
#include "ops.h"
#include "sg_common.cuh"

namespace sg {

namespace {

constexpr int kPxMaxPeers = 8;
constexpr int kPxUnroll = 2;  // float4 per thread per round (U = 4 needs 255 registers with 8 peer slots)

struct PxPeers {
  const float* g[kPxMaxPeers];  // rank k's gradient bucket
  float* w[kPxMaxPeers];        // rank k's working-copy bucket
};

struct PxFlags {
  unsigned* f[kPxMaxPeers];  // rank k's flag array [nstore][2 phases][kPxMaxPeers]
};

__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Cross-rank flag barrier of bucket sid, phase ph: lane j < world of the calling
// warp signals rank j (slot [sid][ph][rank] of rank j's flags; only when
// `signal`) and waits for slot [sid][ph][j] of its own flags to reach `target`.
// Bounded spin: a peer that never arrives sets the error flag (device and
// mapped host memory) and the wait gives up.
__device__ __forceinline__ void px_warp_barrier(const PxFlags& fl, int sid, int ph, int rank, int world,
                                                unsigned target, bool signal, int* err, int* err_host) {
  const int j = threadIdx.x & 31;
  const int slot = (sid * 2 + ph) * kPxMaxPeers;
  if (signal && j < world) st_release_sys(fl.f[j] + slot + rank, target);
  if (j < world) {
    const unsigned* mine = fl.f[rank] + slot + j;
    long long spins = 0;
    while (ld_acquire_sys(mine) < target) {
      if (*(volatile int*)err) break;
      if (++spins > (1LL << 26)) {
        atomicExch(err, 1);
        *(volatile int*)err_host = 1;  // mapped host memory: visible to sg_net_sync without a copy
        break;
      }
      __nanosleep(64);
    }
  }
  __syncwarp();
}

// The whole exchange of bucket sid in ONE kernel (rank r owns shard r):
//   entry barrier (every rank's gradient of the bucket complete: CTA 0 signals,
//   every CTA waits) -> ascending-rank sum of the K gradients of the shard,
//   Updater on the fp32 master shard, TF32 working copy stored into every rank
//   -> each CTA fences its stores system-wide and arrives on a counter; the last
//   CTA runs the trailing barrier (every rank's stores into this rank landed, no
//   peer reads this rank's gradient any more) and advances the bucket's epoch.
// The epoch lives in device memory, so the launch is CUDA-graph replayable.
template <int TYPE>
__global__ void __launch_bounds__(256) px_exchange_kernel(PxPeers p, PxFlags fl, float* __restrict__ m,
                                                          float* __restrict__ v, long long shard, long long rn_end,
                                                          int sid, int rank, int world, const float* lr_dev,
                                                          float lr_scale, float mu, float wd, float s, float eps,
                                                          unsigned* epoch, unsigned* counter, int* err, int* err_host,
                                                          int agg_out) {
  pdl_entry();
  __shared__ int last;
  if (*(volatile const int*)err) return;  // an earlier exchange failed: no waiting, no work
  const unsigned e0 = epoch[sid];
  if (threadIdx.x < 32) {
    if (blockIdx.x == 0) __threadfence_system();  // this rank's gradient before the signal
    px_warp_barrier(fl, sid, 0, rank, world, e0 + 1, blockIdx.x == 0, err, err_host);
  }
  __syncthreads();
  if (!*(volatile const int*)err) {
    const float lr = lr_dev[0] * lr_scale;
    const long long base = (long long)rank * shard;
    const long long n4 = shard >> 2;
    float4* m4 = reinterpret_cast<float4*>(m);
    float4* v4 = reinterpret_cast<float4*>(v);
    // kPxUnroll float4 per thread per grid-stride round: every load (local and
    // remote) of the round in flight before the arithmetic
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < n4; i0 += kPxUnroll * stride) {
      float4 gk[kPxUnroll][kPxMaxPeers];
#pragma unroll
      for (int u = 0; u < kPxUnroll; ++u) {
        const long long i = i0 + u * stride;
#pragma unroll
        for (int k = 0; k < kPxMaxPeers; ++k)
          if (k < world && i < n4) gk[u][k] = reinterpret_cast<const float4*>(p.g[k] + base)[i];
      }
#pragma unroll
      for (int u = 0; u < kPxUnroll; ++u) {
        const long long i = i0 + u * stride;
        if (i >= n4) break;
        float4 g = gk[u][0];
#pragma unroll
        for (int k = 1; k < kPxMaxPeers; ++k)
          if (k < world) {
            g.x = __fadd_rn(g.x, gk[u][k].x);
            g.y = __fadd_rn(g.y, gk[u][k].y);
            g.z = __fadd_rn(g.z, gk[u][k].z);
            g.w = __fadd_rn(g.w, gk[u][k].w);
          }
        float4 ww = m4[i], vv = v4[i];
        float* wp = &ww.x;
        float* vp = &vv.x;
        const float* gp = &g.x;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float gq = __fmaf_rn(wd, wp[e], __fmul_rn(s, gp[e]));
          if (TYPE == 0) {
            vp[e] = __fmaf_rn(mu, vp[e], -__fmul_rn(lr, gq));
            wp[e] = __fadd_rn(wp[e], vp[e]);
          } else {
            vp[e] = __fmaf_rn(gq, gq, vp[e]);
            wp[e] = __fsub_rn(wp[e], __fdiv_rn(__fmul_rn(lr, gq), __fadd_rn(__fsqrt_rn(vp[e]), eps)));
          }
        }
        m4[i] = ww;
        v4[i] = vv;
        const long long el = base + 4 * i;
        float4 wk = ww;
        if (el < rn_end) wk.x = tf32_rna(wk.x);
        if (el + 1 < rn_end) wk.y = tf32_rna(wk.y);
        if (el + 2 < rn_end) wk.z = tf32_rna(wk.z);
        if (el + 3 < rn_end) wk.w = tf32_rna(wk.w);
#pragma unroll
        for (int k = 0; k < kPxMaxPeers; ++k)
          if (k < world) reinterpret_cast<float4*>(p.w[k] + base)[i] = wk;
        // the aggregated gradient of this shard (only this rank reads this region of its own bucket)
        if (agg_out) reinterpret_cast<float4*>(const_cast<float*>(p.g[rank]) + base)[i] = g;
      }
    }
  }
  // completion: this CTA's stores (local and remote) before its arrival
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter + sid, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last || threadIdx.x >= 32) return;
  __threadfence_system();
  px_warp_barrier(fl, sid, 1, rank, world, e0 + 2, true, err, err_host);
  if (threadIdx.x == 0) {
    counter[sid] = 0;
    epoch[sid] = e0 + 2;
  }
}

}  // namespace

struct PeerExchange {
  int rank = 0, world = 1, device = 0;
  std::vector<PxStore> stores;
  std::vector<PxPeers> peers;  // per store
  PxFlags flags{};
  unsigned* flags_own = nullptr;
  unsigned* epoch = nullptr;
  unsigned* counter = nullptr;  // per bucket: CTAs of the running exchange kernel that finished
  int* err_dev = nullptr;     // device memory, read by every exchange kernel
  int* err_host = nullptr;    // mapped pinned copy (written on failure only)
  int* err_host_dev = nullptr;
  std::vector<void*> opened;  // peer allocations opened through IPC
  int sms = 148;
};

sg_status px_create(ncclComm_t comm, int rank, int world, int device, const std::vector<PxStore>& stores,
                    PeerExchange** out) {
  SG_CHECK(world >= 1 && world <= kPxMaxPeers, SG_ERR_UNSUPPORTED, "peer exchange: at most %d ranks (got %d)",
           kPxMaxPeers, world);
  for (const PxStore& s : stores)
    SG_CHECK(s.padded % (32LL * world) == 0, SG_ERR_PARTITION, "peer exchange: bucket of %lld not a multiple of 32K",
             (long long)s.padded);
  SG_CUDA(cudaSetDevice(device));
  PeerExchange* px = new PeerExchange();
  px->rank = rank;
  px->world = world;
  px->device = device;
  px->stores = stores;
  cudaDeviceGetAttribute(&px->sms, cudaDevAttrMultiProcessorCount, device);
  const size_t nflags = (size_t)std::max<size_t>(stores.size(), 1) * 2 * kPxMaxPeers;
  bool ok = true;
  std::string why;
  auto check = [&](cudaError_t e, const char* what) {
    if (ok && e != cudaSuccess) {
      ok = false;
      why = std::string(what) + ": " + cudaGetErrorString(e);
    }
  };
  check(cudaMalloc(&px->flags_own, nflags * sizeof(unsigned)), "flags");
  if (ok) check(cudaMemset(px->flags_own, 0, nflags * sizeof(unsigned)), "flags");
  if (ok) check(cudaMalloc(&px->epoch, std::max<size_t>(stores.size(), 1) * sizeof(unsigned)), "epoch");
  if (ok) check(cudaMemset(px->epoch, 0, std::max<size_t>(stores.size(), 1) * sizeof(unsigned)), "epoch");
  if (ok) check(cudaMalloc(&px->counter, std::max<size_t>(stores.size(), 1) * sizeof(unsigned)), "counter");
  if (ok) check(cudaMemset(px->counter, 0, std::max<size_t>(stores.size(), 1) * sizeof(unsigned)), "counter");
  if (ok) check(cudaMalloc(&px->err_dev, sizeof(int)), "error flag");
  if (ok) check(cudaMemset(px->err_dev, 0, sizeof(int)), "error flag");
  if (ok) check(cudaHostAlloc(&px->err_host, sizeof(int), cudaHostAllocMapped), "error flag");
  if (ok) {
    *px->err_host = 0;
    check(cudaHostGetDevicePointer(&px->err_host_dev, px->err_host, 0), "error flag");
  }
  px->peers.assign(stores.size(), PxPeers{});
  for (size_t i = 0; i < stores.size(); ++i) {
    px->peers[i].g[rank] = stores[i].g;
    px->peers[i].w[rank] = stores[i].w;
  }
  px->flags.f[rank] = px->flags_own;
  if (world > 1) {
    // every rank contributes {status, handles of (flags, g_i, w_i ...)}; the
    // exchange always runs so that a local failure fails every rank together
    const size_t nh = 1 + 2 * stores.size();
    struct Rec {
      int32_t ok;
      cudaIpcMemHandle_t h;
    };
    std::vector<Rec> mine(nh), all(nh * world);
    memset(mine.data(), 0, nh * sizeof(Rec));
    if (ok) check(cudaIpcGetMemHandle(&mine[0].h, px->flags_own), "IPC handle");
    for (size_t i = 0; ok && i < stores.size(); ++i) {
      check(cudaIpcGetMemHandle(&mine[1 + 2 * i].h, stores[i].g), "IPC handle");
      if (ok) check(cudaIpcGetMemHandle(&mine[2 + 2 * i].h, stores[i].w), "IPC handle");
    }
    mine[0].ok = ok ? 1 : 0;
    char* dbuf = nullptr;
    const size_t bytes = nh * sizeof(Rec);
    cudaError_t e = cudaMalloc(&dbuf, bytes * (world + 1));
    ncclResult_t r = ncclSuccess;
    if (e != cudaSuccess) {  // cannot take part in the exchange at all
      px_destroy(px, nullptr);
      SG_FAIL(SG_ERR_OOM, "peer exchange setup: %s", cudaGetErrorString(e));
    }
    e = cudaMemcpy(dbuf, mine.data(), bytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      mine[0].ok = 0;
      ok = false;
      why = std::string("handle upload: ") + cudaGetErrorString(e);
    }
    // (the gather runs even after a local failure: the peers are waiting in the
    // same collective and learn the failure from the status word)
    r = ncclAllGather(dbuf, dbuf + bytes, bytes, ncclChar, comm, 0);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e == cudaSuccess && r == ncclSuccess) e = cudaMemcpy(all.data(), dbuf + bytes, bytes * world, cudaMemcpyDeviceToHost);
    cudaFree(dbuf);
    if (r != ncclSuccess) {
      ok = false;
      why = std::string("handle exchange: ") + ncclGetErrorString(r);
    }
    check(e, "handle exchange");
    for (int k = 0; ok && k < world; ++k)
      if (!all[k * nh].ok) {
        ok = false;
        why = "rank " + std::to_string(k) + " failed to set up its buffers";
      }
    for (int k = 0; ok && k < world; ++k) {
      if (k == rank) continue;
      for (size_t j = 0; ok && j < nh; ++j) {
        void* q = nullptr;
        check(cudaIpcOpenMemHandle(&q, all[k * nh + j].h, cudaIpcMemLazyEnablePeerAccess), "IPC open");
        if (!ok) break;
        px->opened.push_back(q);
        if (j == 0)
          px->flags.f[k] = static_cast<unsigned*>(q);
        else if (j % 2 == 1)
          px->peers[(j - 1) / 2].g[k] = static_cast<const float*>(q);
        else
          px->peers[(j - 1) / 2].w[k] = static_cast<float*>(q);
      }
    }
    // second collective decision: every rank opened every peer's buffers
    int32_t* d = nullptr;
    int32_t flag = ok ? 1 : 0;
    if (cudaMalloc(&d, sizeof(int32_t)) == cudaSuccess) {
      cudaMemcpy(d, &flag, sizeof(flag), cudaMemcpyHostToDevice);
      ncclAllReduce(d, d, 1, ncclInt32, ncclMin, comm, 0);
      cudaDeviceSynchronize();
      cudaMemcpy(&flag, d, sizeof(flag), cudaMemcpyDeviceToHost);
      cudaFree(d);
    } else {
      flag = 0;
    }
    if (ok && !flag) {
      ok = false;
      why = "a peer failed to open the IPC buffers";
    }
  }
  if (!ok) {
    px_destroy(px, nullptr);
    SG_FAIL(SG_ERR_CUDA, "peer exchange setup failed: %s", why.c_str());
  }
  *out = px;
  return SG_OK;
}

void px_destroy(PeerExchange* px, ncclComm_t comm) {
  if (!px) return;
  cudaSetDevice(px->device);
  cudaDeviceSynchronize();
  if (comm && px->world > 1) {  // nobody may still access our buffers when they are unmapped / freed
    float* one = nullptr;
    if (cudaMalloc(&one, sizeof(float)) == cudaSuccess) {
      ncclAllReduce(one, one, 1, ncclFloat, ncclSum, comm, 0);
      cudaDeviceSynchronize();
      cudaFree(one);
    }
  }
  for (void* q : px->opened) cudaIpcCloseMemHandle(q);
  cudaFree(px->flags_own);
  cudaFree(px->epoch);
  cudaFree(px->counter);
  cudaFree(px->err_dev);
  if (px->err_host) cudaFreeHost(px->err_host);
  delete px;
}

int px_failed(const PeerExchange* px) { return px && px->err_host ? *(volatile int*)px->err_host : 0; }

cudaError_t px_update(PeerExchange* px, int sid, const float* lr_dev, float lr_scale, float mu, float wd, float s,
                      int type, float eps, cudaStream_t st) {
  const PxStore& S = px->stores[sid];
  const long long shard = S.padded / px->world;
  const long long n4 = shard / 4;
  const int blocks = (int)std::max<long long>(1, std::min<long long>((n4 + 255) / 256, 4LL * px->sms));
  auto k = type == 1 ? px_exchange_kernel<1> : px_exchange_kernel<0>;
  return launch_k(k, blocks, 256, 0, st, px->peers[sid], px->flags, S.m, S.v, shard, (long long)S.rn_end, sid,
                  px->rank, px->world, lr_dev, lr_scale, mu, wd, s, eps, px->epoch, px->counter, px->err_dev,
                  px->err_host_dev, S.agg_out);
}

}  // namespace sg
