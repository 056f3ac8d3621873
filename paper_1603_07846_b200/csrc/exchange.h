// Fused worker -> server -> worker exchange of the training step over NVLink
// peer memory (§5.2.1 AllReduce framework
// P:419-422, per-layer Update of Alg. 1, parameters "broadcast back"
// P:586, Updater P:282-284): per sharded Param bucket, instead of
// reduce-scatter -> Updater -> all-gather, ONE kernel:
//   entry barrier (every rank's gradient of the bucket is complete; CTA 0
//   signals, every CTA waits)
//   -> rank r loads shard r of every rank's gradient straight from the peers'
//      HBM, sums them in ascending rank order (the oracle's order), applies the
//      Updater to its fp32 master shard + history, writes the TF32 working copy
//      of the shard into EVERY rank's weight bucket (P2P stores) and the
//      aggregated gradient into its own bucket (sg_param_get_grad)
//   -> the last CTA to finish (arrival counter) runs the trailing barrier
//      (every rank's stores have landed; no rank will overwrite a gradient a
//      peer still reads).
// Barrier flags live in IPC-shared device memory; the epoch of every bucket is
// kept in device memory and advanced by the kernel itself, so the launch is
// CUDA-graph replayable.  A peer that never
// arrives: bounded spin, then an error flag in mapped host memory; every later
// exchange kernel skips its work, the error is reported by sg_net_sync.
#pragma once
#include <nccl.h>

#include <cstdint>
#include <vector>

#include "abi_common.h"

namespace sg {

struct PxStore {
  float* g;        // this rank's gradient bucket [padded] (IPC shared)
  float* w;        // this rank's working-copy bucket [padded] (IPC shared; peers store into it)
  float* m;        // fp32 master shard [padded / K]
  float* v;        // history shard [padded / K] (momentum or AdaGrad accumulator)
  int64_t padded;  // bucket elements, a multiple of 32 K
  int64_t rn_end;  // elements [0, rn_end) are the weight matrix (TF32-rounded working copy)
  int agg_out = 1; // write the aggregated gradient of the shard back into g (0: g is only read)
};

struct PeerExchange;

// COLLECTIVE over `comm` (world > 1: CUDA IPC handles exchanged over NCCL; a
// failure on any rank fails every rank).  world == 1 runs the same kernels
// with this rank as its only peer.
sg_status px_create(ncclComm_t comm, int rank, int world, int device, const std::vector<PxStore>& stores,
                    PeerExchange** out);
// COLLECTIVE; synchronises the device first.
void px_destroy(PeerExchange* px, ncclComm_t comm);
// Enqueue the exchange of bucket `sid` on `st` (one kernel launch).
// type 0: SGD momentum (mu), 1: AdaGrad (eps); lr = lr_dev[0] * lr_scale.
cudaError_t px_update(PeerExchange* px, int sid, const float* lr_dev, float lr_scale, float mu, float wd, float s,
                      int type, float eps, cudaStream_t st);
// Nonzero once a barrier timed out (reads mapped host memory; no sync).
int px_failed(const PeerExchange* px);

}  // namespace sg
