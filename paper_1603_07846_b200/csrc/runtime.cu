// Runtime: cluster topology, NeuralNet on the device, BPTrainOneBatch
// (Alg. 1), server-group Updater over sharded Params (P:282-284,
// P:419-422) and the connection layers' collectives over NCCL.
//
// Streams: every net owns a compute stream (forward / backward / connection
// collectives on the activation communicator) and a parameter stream (per-layer
// Update = reduce-scatter -> sharded Updater -> all-gather on the parameter
// communicator), joined by events: Update(layer) overlaps the backward of the
// layers below it, Collect(layer) waits for its Update (Alg. 1 line "Collect").
// sg_train_one_batch can be captured once into a CUDA graph and replayed.
#include <nccl.h>

#include <cmath>
#include <cstring>
#include <vector>

#include "abi_common.h"
#include "exchange.h"
#include "elt_common.cuh"
#include "ops.h"
#include "plan.h"

namespace sg {
size_t colsum_ws_floats(int M, int N);
}

#define SG_NCCL(expr)                                                                                 \
  do {                                                                                                \
    ncclResult_t _r = (expr);                                                                         \
    if (_r != ncclSuccess) SG_FAIL(SG_ERR_NCCL, "NCCL error %s at %s:%d (%s)", ncclGetErrorString(_r), \
                                   __FILE__, __LINE__, #expr);                                        \
  } while (0)

#define SG_LCH(expr)                                                                               \
  do {                                                                                             \
    cudaError_t _e = (expr);                                                                       \
    if (_e != cudaSuccess) SG_FAIL(SG_ERR_CUDA, "%s: %s (%s)", L.name.c_str(), cudaGetErrorString(_e), #expr); \
  } while (0)

struct sg_cluster {
  int rank = 0, world = 1, device = 0;
  bool force = false;             // exercise_collectives at world 1 (partitioned plans, 1-rank NCCL)
  ncclComm_t comm_act = nullptr;  // activations / connection layers (compute stream)
  ncclComm_t comm_par = nullptr;  // parameter sync (parameter stream)
};

struct sg_updater {
  sg_updater_cfg cfg;
  float s;
  float eps;  // AdaGrad
};

struct sg_net {
  sg_cluster* cl = nullptr;
  sg_plan plan;
  cudaStream_t cs = nullptr, ps = nullptr;
  std::vector<float*> data, grad, scale;
  // strided first-layer conv by space-to-depth (conv_s2d.cu): image, filter, filter gradient
  std::vector<float*> s2d_x, s2d_w, s2d_dw;
  bool s2d_wgrad = true;
  int s2d_of_input = -1;  // conv whose space-to-depth image the input layer writes (or -1)
  std::vector<uint8_t*> mask;
  // per store: working copy of the weights (full; what the GEMMs read: TF32-RN
  // weights, fp32 biases), gradients (full), fp32 master weights and history
  // (the rank's shard when the store is sharded, else full)
  std::vector<float*> sw, sgr, sm, sv;
  float* row_loss = nullptr;
  float* loss_int = nullptr;
  float* lr_dev = nullptr;
  float lr_last = -1.f;  // value in lr_dev (the device write is skipped while unchanged)
  int* err = nullptr;
  int32_t* labels = nullptr;
  float* x_stage = nullptr;
  // pipelined host path (sg_train_one_batch_host_async): a second input slot,
  // label slots, a copy stream, and per-slot events (copied / free again)
  float* x_stage2 = nullptr;
  int32_t* lab_stage[2] = {nullptr, nullptr};
  cudaStream_t hs = nullptr;
  cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_free[2] = {nullptr, nullptr};
  int stage_k = 0;
  bool stage_used[2] = {false, false};
  float* x_exact = nullptr;  // unrounded copy of the input blob (a Euclidean loss's target when the input is rounded)
  const float* x_src = nullptr;
  sg::Workspace ws;
  // weight / bias gradients run on the parameter stream, off the critical path
  // of the data-gradient chain (they are needed only by the layer's Update);
  // their kernels use a workspace of their own
  bool wgrad_side = true;
  sg::Workspace ws2;
  std::vector<cudaEvent_t> ev_grad, ev_upd, ev_dy, ev_wg;
  // Updates (and their collectives / peer exchange) run on a stream of their own
  // when the weight gradients use the parameter stream, so an exchange waiting
  // for the peers never holds up the next layer's weight gradient
  cudaStream_t us = nullptr;
  cudaEvent_t ev_join_u = nullptr;
  std::vector<char> wg_on_ps;      // layer i's weight gradient of this step ran on the parameter stream
  // first layer at K = 1: its Update applied by the weight-gradient reduction
  // (the step's last operation); update() then only records the event
  std::vector<char> upd_in_bwd;
  std::vector<cudaStream_t> upd_bwd_stream;
  bool fuse_update = true;
  bool ps_used = false, us_used = false;  // streams forked in this step (joined at its end)
  std::vector<char> upd_pending, fwd_done, bwd_done;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr, ev_fork = nullptr, ev_join = nullptr;
  bool input_set = false;
  // graph
  bool graph_on = false;
  // conv / inner-product -> ReLU fusion: the producer's epilogue applies the
  // ReLU and writes the ReLU layer's blob (its own data blob aliases it)
  bool fuse = true;
  std::vector<float*> data_own;
  std::vector<int> relu_of;     // producer i -> fused ReLU layer (or -1)
  std::vector<char> fused_away; // ReLU layer whose forward is done by its producer
  std::vector<int> relu_after;  // pool i -> ReLU layer whose forward the pool kernel also writes (or -1)
  std::vector<int> relu_into;   // consumer c -> ReLU layer whose backward c's kernel also does (or -1)
  std::vector<char> bwd_fused_away;  // ReLU layer whose backward is done by its consumer
  std::vector<int> lrn_after;   // pool i -> LRN layer computed by the pool's forward kernel (or -1)
  std::vector<int> pool_into;   // first-layer conv i -> max pool whose backward its weight-gradient kernel does (or -1)
  std::vector<char> pool_bwd_fused;  // max pool whose backward is done by its source conv's kernel
  std::vector<char> lrn_fused;  // LRN layer whose forward is done by the pool before it
  cudaGraphExec_t gexec = nullptr;
  // the captured step bakes the Updater's hyper-parameters in by value: the
  // graph is reused only for an updater with identical values
  sg_updater graph_upd{};
  long long graph_launches = 0;
  long long last_launches = 0;
  // per-operation event timing (sg_net_profile)
  bool prof = false, prof_concurrent = false, capturing = false;
  std::vector<cudaEvent_t> pev;  // 2 per slot, 4 slots per layer
  std::vector<char> pused;
  std::vector<double> pacc;
  std::vector<long long> pcnt;
  std::vector<void*> allocs;
  // fused peer-memory exchange of the sharded buckets (sg_net_set_exchange), else NCCL
  sg::PeerExchange* px = nullptr;
  std::vector<int> px_sid;  // store -> exchange bucket (or -1)
  // Update(layer) overlaps the backward of the layers below (default); off: the
  // compute stream waits for every Update right away ("Sync Copy")
  bool overlap = true;
};

namespace sg {
namespace {

const Plan& PL(const sg_net* n) { return n->plan.p; }

sg_status dalloc(sg_net* n, size_t bytes, void** out) {
  if (bytes == 0) bytes = 16;
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) SG_FAIL(SG_ERR_OOM, "device allocation of %zu bytes failed: %s", bytes, cudaGetErrorString(e));
  e = cudaMemset(p, 0, bytes);
  if (e != cudaSuccess) SG_FAIL(SG_ERR_CUDA, "memset: %s", cudaGetErrorString(e));
  n->allocs.push_back(p);
  *out = p;
  return SG_OK;
}
template <class T>
sg_status dalloc_t(sg_net* n, size_t count, T** out) {
  void* p;
  SG_TRY(dalloc(n, count * sizeof(T), &p));
  *out = static_cast<T*>(p);
  return SG_OK;
}

// TF32 round to nearest, ties away from zero (= tf32_rna in sg_common.cuh)
float tf32_rna_host(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u = (u + 0x1000u) & 0xFFFFE000u;
  memcpy(&x, &u, 4);
  return x;
}

float lr_at(const sg_updater_cfg& c, int64_t step) {
  if (c.lr_policy == 1 && c.step_size > 0) return (float)(c.base_lr * std::pow((double)c.gamma, (double)(step / c.step_size)));
  return c.base_lr;
}

// ---- views of blobs ----
View2D feat_view(const LayerPlan& L, float* p, int64_t logical_cols) {
  View2D v;
  v.p = p;
  v.ld = L.ld;
  v.bs = L.rows * L.ld;
  v.rows = (int)L.rows;
  v.cols = (int)logical_cols;
  v.cb = L.nblocks > 1 ? (int)L.ld : (int)logical_cols;
  return v;
}
// real-column view (losses): blocked with the real block width
View2D real_view(const LayerPlan& L, float* p) {
  View2D v;
  v.p = p;
  v.ld = L.ld;
  v.bs = L.rows * L.ld;
  v.rows = (int)L.rows;
  v.cols = (int)(L.nblocks > 1 ? L.feat : L.cols);
  v.cb = L.nblocks > 1 ? (int)L.blk_cols : v.cols;
  return v;
}

ConvShape conv_shape(const LayerPlan& L, const LayerPlan& S) {
  return ConvShape{(int)L.rows, S.h, S.w, S.c, L.c, L.kernel, L.kernel, L.stride, L.pad, L.h, L.w};
}
PoolShape pool_shape(const LayerPlan& L, const LayerPlan& S) {
  return PoolShape{(int)L.rows, S.h, S.w, S.c, L.kernel, L.stride, L.pad, L.h, L.w};
}

// ---- per-operation event timing ----
void prof_mark(sg_net* n, int slot, int end, cudaStream_t st) {
  if (!n->prof) return;
  cudaEvent_t e = n->pev[2 * slot + end];
  if (n->capturing)
    cudaEventRecordWithFlags(e, st, cudaEventRecordExternal);
  else
    cudaEventRecord(e, st);
  n->pused[slot] = 1;
}

// Epilogue flags of a conv / inner-product layer: the fused ReLU, and TF32
// rounding when the blob it writes (its own, or the fused ReLU's) is a GEMM
// operand (reading A19).
int epi_flags(const sg_net* n, int i) {
  const Plan& P = PL(n);
  const int j = n->relu_of[i];
  const bool rn = (j >= 0 ? P.layers[j] : P.layers[i]).rn_data;
  return (j >= 0 ? EPI_RELU : 0) | (rn ? EPI_RN : 0);
}

// ---- ComputeFeature ----
sg_status forward_impl(sg_net* n, int i);
sg_status forward(sg_net* n, int i) {
  prof_mark(n, 4 * i, 0, n->cs);
  SG_TRY(forward_impl(n, i));
  prof_mark(n, 4 * i, 1, n->cs);
  return SG_OK;
}
sg_status forward_impl(sg_net* n, int i) {
  const Plan& P = PL(n);
  const LayerPlan& L = P.layers[i];
  cudaStream_t st = n->cs;
  const int K = P.world;
  float* W = L.pW >= 0 ? n->sw[L.store] + P.params[L.pW].store_off : nullptr;
  float* b = L.pb >= 0 ? n->sw[L.store] + P.params[L.pb].store_off : nullptr;
  const LayerPlan* S = L.src >= 0 ? &P.layers[L.src] : nullptr;
  switch (L.kind) {
    case SG_INPUT:
      SG_CHECK(n->x_src, SG_ERR_SEQUENCE, "sequence error: no input set (sg_net_set_input)");
      if (L.image && n->s2d_of_input >= 0) {
        const int c = n->s2d_of_input;
        SG_LCH(pad_channels_s2d(n->x_src, L.c_real, n->data[i], n->s2d_x[c], conv_shape(P.layers[c], L), st,
                                L.rn_data));
      } else if (L.image) {
        SG_LCH(pad_channels(n->x_src, n->data[i], L.rows * L.h * L.w, L.c_real, L.c, st, L.rn_data));
      }
      else
        SG_LCH(copy2d(n->x_src, L.feat, n->data[i], L.ld, (int)L.rows, (int)L.feat, st, L.rn_data));
      if (n->x_exact) SG_LCH(copy2d(n->x_src, L.feat, n->x_exact, L.ld, (int)L.rows, (int)L.feat, st, 0));
      break;
    case SG_CONV:
      if (n->s2d_x[i]) {  // stride-st first layer as a stride-1 conv of the space-to-depth image
        if (n->s2d_of_input != i) SG_LCH(conv_s2d_input(conv_shape(L, *S), n->data[L.src], n->s2d_x[i], st));
        SG_LCH(conv_fwd_s2d(conv_shape(L, *S), n->s2d_x[i], W, n->s2d_w[i], b, n->data[i], epi_flags(n, i), n->ws, st));
      } else {
        SG_LCH(conv_fwd(conv_shape(L, *S), n->data[L.src], W, b, n->data[i], epi_flags(n, i), n->ws, st));
      }
      break;
    case SG_POOL_MAX:
    case SG_POOL_AVG: {
      float* relu_out = n->relu_after[i] >= 0 ? n->data[n->relu_after[i]] : nullptr;
      const int k = n->lrn_after[i];
      const int rn = (L.rn_data ? RN_OUT : 0) | (n->relu_after[i] >= 0 && P.layers[n->relu_after[i]].rn_data ? RN_AUX : 0);
      if (k >= 0) {  // pooling [-> ReLU] -> LRN in one kernel
        const LayerPlan& Lk = P.layers[k];
        SG_LCH(pool_lrn_fwd(pool_shape(L, *S), L.kind == SG_POOL_MAX, n->data[L.src], n->data[i],
                            L.kind == SG_POOL_MAX ? n->mask[i] : nullptr, relu_out,
                            LrnShape{Lk.rows * Lk.h * Lk.w, Lk.c, Lk.lrn_size, Lk.alpha, Lk.beta, Lk.k}, n->data[k],
                            n->scale[k], st, Lk.rn_data));
      } else if (L.kind == SG_POOL_MAX) {
        SG_LCH(maxpool_fwd(pool_shape(L, *S), n->data[L.src], n->data[i], n->mask[i], st, relu_out, rn));
      } else {
        SG_LCH(avgpool_fwd(pool_shape(L, *S), n->data[L.src], n->data[i], st, relu_out, rn));
      }
      break;
    }
    case SG_LRN:
      if (!n->lrn_fused[i])
        SG_LCH(lrn_fwd(LrnShape{L.rows * L.h * L.w, L.c, L.lrn_size, L.alpha, L.beta, L.k}, n->data[L.src],
                       n->data[i], n->scale[i], st, L.rn_data));
      break;
    case SG_RELU:
      if (!n->fused_away[i]) SG_LCH(relu_fwd(n->data[L.src], n->data[i], L.blob_floats(), st, L.rn_data));
      break;
    case SG_SIGMOID:
      SG_LCH(sigmoid_fwd(n->data[L.src], n->data[i], L.blob_floats(), st, L.rn_data));
      break;
    case SG_INNER_PRODUCT:
      SG_LCH(ip_fwd(feat_view(*S, n->data[L.src], L.kin), W, (int)L.kin, (int)L.nout, b,
                    plain(n->data[i], (int)L.rows, (int)L.nout, L.ld), epi_flags(n, i), n->ws, st));
      break;
    case SG_CONCAT:
      SG_NCCL(ncclAllGather(n->data[L.src], n->data[i], (size_t)(S->rows * S->ld), ncclFloat, n->cl->comm_act, st));
      break;
    case SG_SLICE: {
      const size_t cnt = (size_t)(L.rows * S->ld);
      SG_NCCL(ncclGroupStart());
      for (int j = 0; j < K; ++j) {
        SG_NCCL(ncclSend(n->data[L.src] + j * cnt, cnt, ncclFloat, j, n->cl->comm_act, st));
        SG_NCCL(ncclRecv(n->data[i] + j * cnt, cnt, ncclFloat, j, n->cl->comm_act, st));
      }
      SG_NCCL(ncclGroupEnd());
      break;
    }
    case SG_SOFTMAX_CE:
      SG_LCH(softmax_ce(real_view(*S, n->data[L.src]), n->labels, n->row_loss, real_view(*S, n->grad[L.src]),
                        (float)(1.0 / (double)P.loss_rows), n->err, st, S->rn_grad));
      break;
    case SG_EUCLIDEAN: {
      const LayerPlan& in = P.layers[0];
      View2D u = real_view(*S, n->data[L.src]);
      View2D v = plain((n->x_exact ? n->x_exact : n->data[0]) + S->col_off, (int)S->rows, (int)S->cols, in.ld);
      SG_LCH(euclidean(u, v, n->row_loss, real_view(*S, n->grad[L.src]), (float)(1.0 / (double)P.loss_rows), st,
                       S->rn_grad));
      break;
    }
  }
  return SG_OK;
}

// ---- ComputeGradient ----
sg_status backward(sg_net* n, int i, const sg_updater* u = nullptr) {
  const Plan& P = PL(n);
  const LayerPlan& L = P.layers[i];
  cudaStream_t st = n->cs;
  const int K = P.world;
  if (L.kind == SG_INPUT || L.kind == SG_SOFTMAX_CE || L.kind == SG_EUCLIDEAN) return SG_OK;
  const LayerPlan& S = P.layers[L.src];
  const bool need_dx = S.kind != SG_INPUT;
  float* W = L.pW >= 0 ? n->sw[L.store] + P.params[L.pW].store_off : nullptr;
  float* dW = L.pW >= 0 ? n->sgr[L.store] + P.params[L.pW].store_off : nullptr;
  float* db = L.pb >= 0 ? n->sgr[L.store] + P.params[L.pb].store_off : nullptr;
  const int s1 = 4 * i + 1, s2 = 4 * i + 2;
  const int rn_dx = S.rn_grad ? RN_OUT : 0;  // this layer's dx is a GEMM operand (reading A19)
  // weight gradient stream: the parameter stream (after dy is ready) or in line;
  // in line while profiling, so every slot times its kernels alone
  const bool side = n->wgrad_side && (!n->prof || n->prof_concurrent) && (L.kind == SG_CONV || L.kind == SG_INNER_PRODUCT);
  cudaStream_t wst = side ? n->ps : st;
  const Workspace wws = side ? n->ws2 : n->ws;
  n->wg_on_ps[i] = side;
  if (side) {
    n->ps_used = true;
    SG_CUDA(cudaEventRecord(n->ev_dy[i], st));  // dy of this layer is complete
    SG_CUDA(cudaStreamWaitEvent(n->ps, n->ev_dy[i], 0));
  }
  prof_mark(n, s1, 0, wst);
  switch (L.kind) {
    case SG_CONV:
      if (n->pool_into[i] >= 0) {  // fused: the max pool's backward builds this layer's dy (a13 + a15)
        const int c = n->pool_into[i];
        // K = 1 and no data gradient: the reduction also applies the Updater
        const bool fu_on = u && n->fuse_update && K == 1 && !need_dx && L.store >= 0 && L.pW >= 0 && L.pb >= 0 &&
                           !P.stores[L.store].sharded;
        FusedUpdate fu{};
        if (fu_on) {
          const int64_t ow = P.params[L.pW].store_off, ob = P.params[L.pb].store_off;
          fu = FusedUpdate{n->sm[L.store] + ow, n->sv[L.store] + ow, n->sw[L.store] + ow, n->sm[L.store] + ob,
                           n->sv[L.store] + ob, n->sw[L.store] + ob, n->lr_dev, L.lr_scale, u->cfg.momentum,
                           u->cfg.weight_decay * L.wd_scale, u->s, u->eps, u->cfg.type == SG_UPD_ADAGRAD ? 1 : 0};
          n->upd_in_bwd[i] = 1;
          n->upd_bwd_stream[i] = wst;
        }
        SG_LCH(conv_img4_pool_bwd(conv_shape(L, S), pool_shape(P.layers[c], L), n->data[L.src], n->grad[c],
                                  n->mask[c], n->grad[i], L.rn_grad, dW, db, wws, wst, fu_on ? &fu : nullptr));
      } else if (n->s2d_x[i] && n->s2d_wgrad) {
        SG_LCH(conv_wgrad_s2d(conv_shape(L, S), n->s2d_x[i], n->grad[i], n->s2d_dw[i], dW, db, wws, wst));
      } else {
        SG_LCH(conv_wgrad(conv_shape(L, S), n->data[L.src], n->grad[i], dW, db, wws, wst));
      }
      prof_mark(n, s1, 1, wst);
      if (need_dx) {
        prof_mark(n, s2, 0, st);
        SG_LCH(conv_dgrad(conv_shape(L, S), n->grad[i], W, n->grad[L.src], n->ws, st, S.rn_grad ? EPI_RN : 0));
        prof_mark(n, s2, 1, st);
      }
      return SG_OK;
    case SG_POOL_MAX:
    case SG_POOL_AVG:
    case SG_LRN: {
      // fused backward of the ReLU feeding this layer: also dx_relu = dx * [relu_y > 0]
      const int j = n->relu_into[i];
      const float* ry = j >= 0 ? n->data[j] : nullptr;
      float* dxr = j >= 0 ? n->grad[P.layers[j].src] : nullptr;
      if (!need_dx || n->pool_bwd_fused[i]) break;
      const int rn = rn_dx | (j >= 0 && P.layers[P.layers[j].src].rn_grad ? RN_AUX : 0);
      if (L.kind == SG_POOL_MAX)
        SG_LCH(maxpool_bwd(pool_shape(L, S), n->grad[i], n->mask[i], n->grad[L.src], st, ry, dxr, rn));
      else if (L.kind == SG_POOL_AVG)
        SG_LCH(avgpool_bwd(pool_shape(L, S), n->grad[i], n->grad[L.src], st, ry, dxr, rn));
      else
        SG_LCH(lrn_bwd(LrnShape{L.rows * L.h * L.w, L.c, L.lrn_size, L.alpha, L.beta, L.k}, n->data[L.src],
                       n->data[i], n->scale[i], n->grad[i], n->grad[L.src], st, ry, dxr, rn));
      break;
    }
    case SG_RELU:
      if (need_dx && !n->bwd_fused_away[i])
        SG_LCH(relu_bwd(n->data[i], n->grad[i], n->grad[L.src], L.blob_floats(), st, rn_dx));
      break;
    case SG_SIGMOID:
      if (need_dx) SG_LCH(sigmoid_bwd(n->data[i], n->grad[i], n->grad[L.src], L.blob_floats(), st, rn_dx));
      break;
    case SG_INNER_PRODUCT: {
      View2D dy = plain(n->grad[i], (int)L.rows, (int)L.nout, L.ld);
      SG_LCH(ip_wgrad(feat_view(S, n->data[L.src], L.kin), dy, (int)L.kin, (int)L.nout, dW, db, wws, wst));
      prof_mark(n, s1, 1, wst);
      if (need_dx) {
        prof_mark(n, s2, 0, st);
        SG_LCH(ip_dgrad(dy, W, (int)L.kin, (int)L.nout, feat_view(S, n->grad[L.src], L.kin), n->ws, st,
                        S.rn_grad ? EPI_RN : 0));
        prof_mark(n, s2, 1, st);
      }
      return SG_OK;
    }
    case SG_CONCAT:
      SG_NCCL(ncclReduceScatter(n->grad[i], n->grad[L.src], (size_t)(S.rows * S.ld), ncclFloat, ncclSum,
                                n->cl->comm_act, st));
      // the sum of the ranks' partial input gradients is a GEMM operand of the source (reading A19)
      if (S.rn_grad) SG_LCH(round_tf32(n->grad[L.src], S.blob_floats(), st));
      break;
    case SG_SLICE: {
      const size_t cnt = (size_t)(L.rows * S.ld);
      SG_NCCL(ncclGroupStart());
      for (int j = 0; j < K; ++j) {
        SG_NCCL(ncclSend(n->grad[i] + j * cnt, cnt, ncclFloat, j, n->cl->comm_act, st));
        SG_NCCL(ncclRecv(n->grad[L.src] + j * cnt, cnt, ncclFloat, j, n->cl->comm_act, st));
      }
      SG_NCCL(ncclGroupEnd());
      break;
    }
  }
  prof_mark(n, s1, 1, st);
  return SG_OK;
}

// ---- Update(layer.params()): worker group -> server group -> workers ----
sg_status update(sg_net* n, sg_updater* u, int i) {
  const Plan& P = PL(n);
  const LayerPlan& L = P.layers[i];
  if (L.store < 0) return SG_OK;
  const StorePlan& S = P.stores[L.store];
  if (n->upd_in_bwd[i]) {  // applied by the weight-gradient reduction (backward)
    n->upd_in_bwd[i] = 0;
    SG_CUDA(cudaEventRecord(n->ev_upd[i], n->upd_bwd_stream[i]));
    n->upd_pending[i] = 1;
    if (!n->overlap) SG_CUDA(cudaStreamWaitEvent(n->cs, n->ev_upd[i], 0));
    return SG_OK;
  }
  // the layer's backward (the data gradient reads the working copy the Updater
  // rewrites) is complete; a side-stream weight gradient precedes in stream order
  SG_CUDA(cudaEventRecord(n->ev_grad[i], n->cs));
  cudaStream_t us = n->us ? n->us : n->ps;
  (n->us ? n->us_used : n->ps_used) = true;
  SG_CUDA(cudaStreamWaitEvent(us, n->ev_grad[i], 0));
  if (n->us && n->wg_on_ps[i]) {  // the layer's weight gradient (parameter stream) is complete
    SG_CUDA(cudaEventRecord(n->ev_wg[i], n->ps));
    SG_CUDA(cudaStreamWaitEvent(us, n->ev_wg[i], 0));
  }
  prof_mark(n, 4 * i + 3, 0, us);
  const float mu = u->cfg.momentum, wd = u->cfg.weight_decay * L.wd_scale;
  // elements [0, rn_end) of the store are the weight matrix (TF32-RN working copy); the bias follows
  const int64_t rn_end = P.params[L.pW].isize;
  if (S.sharded && n->px && n->px_sid[L.store] >= 0) {
    // the same exchange in one fused kernel over NVLink peer memory (exchange.h)
    SG_LCH(px_update(n->px, n->px_sid[L.store], n->lr_dev, L.lr_scale, mu, wd, u->s, u->cfg.type, u->eps, us));
  } else if (S.sharded) {
    // worker group -> server group: reduce-scatter (sum) of the gradient bucket;
    // the server owning shard `rank` updates its fp32 master and writes the
    // working copy of the shard, which the all-gather distributes (Collect)
    const int64_t shard = S.padded / P.world;
    float* g = n->sgr[L.store];
    float* w = n->sw[L.store];
    SG_NCCL(ncclReduceScatter(g, g + P.rank * shard, (size_t)shard, ncclFloat, ncclSum, n->cl->comm_par, us));
    if (u->cfg.type == SG_UPD_ADAGRAD)
      SG_LCH(adagrad_dev(n->sm[L.store], g + P.rank * shard, n->sv[L.store], shard, n->lr_dev, L.lr_scale, wd, u->s,
                         u->eps, us, w + P.rank * shard, rn_end - P.rank * shard));
    else
      SG_LCH(sgd_momentum_dev(n->sm[L.store], g + P.rank * shard, n->sv[L.store], shard, n->lr_dev, L.lr_scale, mu,
                              wd, u->s, us, w + P.rank * shard, rn_end - P.rank * shard));
    SG_NCCL(ncclAllGather(w + P.rank * shard, w, (size_t)shard, ncclFloat, n->cl->comm_par, us));
  } else if (u->cfg.type == SG_UPD_ADAGRAD) {
    SG_LCH(adagrad_dev(n->sm[L.store], n->sgr[L.store], n->sv[L.store], S.padded, n->lr_dev, L.lr_scale, wd, u->s,
                       u->eps, us, n->sw[L.store], rn_end));
  } else {
    SG_LCH(sgd_momentum_dev(n->sm[L.store], n->sgr[L.store], n->sv[L.store], S.padded, n->lr_dev, L.lr_scale, mu, wd,
                            u->s, us, n->sw[L.store], rn_end));
  }
  prof_mark(n, 4 * i + 3, 1, us);
  SG_CUDA(cudaEventRecord(n->ev_upd[i], us));
  n->upd_pending[i] = 1;
  if (!n->overlap) SG_CUDA(cudaStreamWaitEvent(n->cs, n->ev_upd[i], 0));
  return SG_OK;
}

sg_status collect(sg_net* n, int i) {
  if (n->upd_pending[i]) {
    SG_CUDA(cudaStreamWaitEvent(n->cs, n->ev_upd[i], 0));
    n->upd_pending[i] = 0;
  }
  return SG_OK;
}

sg_status loss_reduce(sg_net* n) {
  const Plan& P = PL(n);
  cudaError_t e = sum_scaled(n->row_loss, (int)P.loss_rows, (float)(1.0 / P.batch), n->loss_int, n->err, n->cs);
  SG_CHECK(e == cudaSuccess, SG_ERR_CUDA, "loss reduction: %s", cudaGetErrorString(e));
  if (P.dist) SG_NCCL(ncclAllReduce(n->loss_int, n->loss_int, 1, ncclFloat, ncclSum, n->cl->comm_act, n->cs));
  return SG_OK;
}

sg_status set_input(sg_net* n, const float* x, const int32_t* labels) {
  const Plan& P = PL(n);
  SG_CHECK(x, SG_ERR_INVALID_ARG, "set_input: null input");
  n->x_src = x;
  if (P.layers[P.loss].kind == SG_SOFTMAX_CE) {
    SG_CHECK(labels, SG_ERR_INVALID_ARG, "set_input: labels required for a softmax loss");
    SG_CUDA(cudaMemcpyAsync(n->labels, labels, P.loss_rows * sizeof(int32_t), cudaMemcpyDeviceToDevice, n->cs));
  }
  n->input_set = true;
  std::fill(n->fwd_done.begin(), n->fwd_done.end(), 0);
  std::fill(n->bwd_done.begin(), n->bwd_done.end(), 0);
  return SG_OK;
}

// The whole Alg. 1 step on the compute stream (input already set).
sg_status step_body(sg_net* n, sg_updater* u) {
  const Plan& P = PL(n);
  const int nl = (int)P.layers.size();
  n->ps_used = n->us_used = false;  // set by the backward / Update calls below
  for (int i = 0; i < nl; ++i) {
    SG_TRY(collect(n, i));
    // the input layer reads the caller's x pointer, which changes per call: the
    // graph path runs it eagerly before the replay instead of capturing it
    if (i == 0 && n->capturing) continue;
    SG_TRY(forward(n, i));
  }
  for (int i = nl - 1; i >= 0; --i) {
    SG_TRY(backward(n, i, u));
    SG_TRY(update(n, u, i));
  }
  SG_TRY(loss_reduce(n));
  // join the parameter / update streams (weight gradients, all Updates of this
  // step) back into the compute stream
  if (n->ps_used) {
    SG_CUDA(cudaEventRecord(n->ev_join, n->ps));
    SG_CUDA(cudaStreamWaitEvent(n->cs, n->ev_join, 0));
  }
  if (n->us_used) {
    SG_CUDA(cudaEventRecord(n->ev_join_u, n->us));
    SG_CUDA(cudaStreamWaitEvent(n->cs, n->ev_join_u, 0));
  }
  n->ps_used = n->us_used = false;
  std::fill(n->upd_pending.begin(), n->upd_pending.end(), 0);
  return SG_OK;
}

sg_status enter(sg_net* n, void* stream) {
  SG_CUDA(cudaSetDevice(n->cl->device));
  SG_CUDA(cudaEventRecord(n->ev_in, reinterpret_cast<cudaStream_t>(stream)));
  SG_CUDA(cudaStreamWaitEvent(n->cs, n->ev_in, 0));
  return SG_OK;
}
sg_status leave(sg_net* n, void* stream) {
  SG_CUDA(cudaEventRecord(n->ev_out, n->cs));
  SG_CUDA(cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(stream), n->ev_out, 0));
  return SG_OK;
}

// ---- user layout <-> internal layout of one Param (host arrays) ----
void to_internal(const Plan& P, const ParamPlan& q, const float* user, std::vector<float>& out) {
  const LayerPlan& L = P.layers[q.layer];
  const LayerPlan& S = P.layers[L.src];
  out.assign(q.isize, 0.f);
  if (L.kind == SG_CONV) {
    if (q.is_bias) {
      for (int64_t j = 0; j < q.isize; ++j) out[j] = user[j];
      return;
    }
    const int RS = L.kernel * L.kernel;
    for (int co = 0; co < L.c; ++co)
      for (int rs = 0; rs < RS; ++rs)
        for (int c = 0; c < S.c_real; ++c)
          out[((int64_t)co * RS + rs) * S.c + c] = user[((int64_t)co * RS + rs) * S.c_real + c];
    return;
  }
  const int64_t dh = q.cols;
  if (q.is_bias) {
    for (int64_t j = 0; j < L.cols; ++j) out[j] = user[L.col_off + j];
    return;
  }
  for (int64_t i = 0; i < L.kin; ++i) {
    int64_t r = i;
    if (L.rmap_pad > 0) {
      const int64_t blk = i / L.rmap_pad, jj = i % L.rmap_pad;
      if (jj >= L.rmap_real) continue;
      r = blk * L.rmap_real + jj;
    }
    const float* src = user + r * dh + L.col_off;
    float* dst = out.data() + i * L.nout;
    for (int64_t j = 0; j < L.cols; ++j) dst[j] = src[j];
  }
}

// internal local block of rank `rk` -> user layout (only the entries that rank owns)
void from_internal(const Plan& P, const ParamPlan& q, const float* in, int rk, float* user) {
  const LayerPlan& L = P.layers[q.layer];
  const LayerPlan& S = P.layers[L.src];
  if (L.kind == SG_CONV) {
    if (q.is_bias) {
      for (int64_t j = 0; j < q.cols; ++j) user[j] = in[j];
      return;
    }
    const int RS = L.kernel * L.kernel;
    for (int co = 0; co < L.c; ++co)
      for (int rs = 0; rs < RS; ++rs)
        for (int c = 0; c < S.c_real; ++c)
          user[((int64_t)co * RS + rs) * S.c_real + c] = in[((int64_t)co * RS + rs) * S.c + c];
    return;
  }
  const int64_t dh = q.cols;
  const int64_t col_off = (q.split_dim == 1) ? rk * L.cols : 0;
  if (q.is_bias) {
    for (int64_t j = 0; j < L.cols; ++j) user[col_off + j] = in[j];
    return;
  }
  for (int64_t i = 0; i < L.kin; ++i) {
    int64_t r = i;
    if (L.rmap_pad > 0) {
      const int64_t blk = i / L.rmap_pad, jj = i % L.rmap_pad;
      if (jj >= L.rmap_real) continue;
      r = blk * L.rmap_real + jj;
    }
    for (int64_t j = 0; j < L.cols; ++j) user[r * dh + col_off + j] = in[i * L.nout + j];
  }
}

// Gathers a Param-shaped quantity (which: 0 master value, 1 grad, 2 history,
// 3 working copy) into the user layout.
sg_status param_export(sg_net* n, int p, int which, float* user) {
  const Plan& P = PL(n);
  SG_CHECK(p >= 0 && p < (int)P.params.size(), SG_ERR_INVALID_ARG, "param index %d out of range", p);
  SG_CHECK(user, SG_ERR_INVALID_ARG, "null host buffer");
  const ParamPlan& q = P.params[p];
  const StorePlan& S = P.stores[q.store];
  SG_CUDA(cudaSetDevice(n->cl->device));
  SG_CUDA(cudaStreamSynchronize(n->ps));
  if (n->us) SG_CUDA(cudaStreamSynchronize(n->us));
  SG_CUDA(cudaStreamSynchronize(n->cs));
  const int K = P.world;
  if (which == 3) {  // working copy: full on every rank (dim-0) or the rank's columns (dim-1)
    std::vector<float> h((size_t)q.isize * (q.split_dim == 1 ? K : 1));
    if (q.split_dim == 1) {
      float* tmp;
      SG_CUDA(cudaMalloc(&tmp, h.size() * sizeof(float)));
      ncclResult_t r = ncclAllGather(n->sw[q.store] + q.store_off, tmp, (size_t)q.isize, ncclFloat, n->cl->comm_act,
                                     n->cs);
      cudaError_t e = cudaStreamSynchronize(n->cs);
      if (e == cudaSuccess) e = cudaMemcpy(h.data(), tmp, h.size() * sizeof(float), cudaMemcpyDeviceToHost);
      cudaFree(tmp);
      SG_CHECK(r == ncclSuccess, SG_ERR_NCCL, "param export: %s", ncclGetErrorString(r));
      SG_CHECK(e == cudaSuccess, SG_ERR_CUDA, "param export: %s", cudaGetErrorString(e));
      for (int rk = 0; rk < K; ++rk) from_internal(P, q, h.data() + (size_t)rk * q.isize, rk, user);
    } else {
      SG_CUDA(cudaMemcpy(h.data(), n->sw[q.store] + q.store_off, h.size() * sizeof(float), cudaMemcpyDeviceToHost));
      from_internal(P, q, h.data(), P.rank, user);
    }
    return SG_OK;
  }
  if (q.split_dim == 1) {
    const float* src = (which == 0 ? n->sm : which == 1 ? n->sgr : n->sv)[q.store] + q.store_off;
    float* tmp;
    SG_CUDA(cudaMalloc(&tmp, (size_t)q.isize * K * sizeof(float)));
    ncclResult_t r = ncclAllGather(src, tmp, (size_t)q.isize, ncclFloat, n->cl->comm_act, n->cs);
    std::vector<float> h((size_t)q.isize * K);
    cudaError_t e = cudaStreamSynchronize(n->cs);
    if (e == cudaSuccess) e = cudaMemcpy(h.data(), tmp, h.size() * sizeof(float), cudaMemcpyDeviceToHost);
    cudaFree(tmp);
    SG_CHECK(r == ncclSuccess, SG_ERR_NCCL, "param export: %s", ncclGetErrorString(r));
    SG_CHECK(e == cudaSuccess, SG_ERR_CUDA, "param export: %s", cudaGetErrorString(e));
    for (int rk = 0; rk < K; ++rk) from_internal(P, q, h.data() + (size_t)rk * q.isize, rk, user);
    return SG_OK;
  }
  // replicated (dim-0) Param: master value, aggregated gradient and history are
  // sharded over the server group when the store is
  std::vector<float> h((size_t)S.padded);
  if (!S.sharded) {
    const float* src = (which == 0 ? n->sm : which == 1 ? n->sgr : n->sv)[q.store];
    SG_CUDA(cudaMemcpy(h.data(), src, (size_t)S.padded * sizeof(float), cudaMemcpyDeviceToHost));
  } else {
    const int64_t shard = S.padded / K;
    const float* src = which == 1 ? n->sgr[q.store] + P.rank * shard : which == 0 ? n->sm[q.store] : n->sv[q.store];
    float* tmp;
    SG_CUDA(cudaMalloc(&tmp, (size_t)S.padded * sizeof(float)));
    ncclResult_t r = ncclAllGather(src, tmp, (size_t)shard, ncclFloat, n->cl->comm_act, n->cs);
    cudaError_t e = cudaStreamSynchronize(n->cs);
    if (e == cudaSuccess) e = cudaMemcpy(h.data(), tmp, h.size() * sizeof(float), cudaMemcpyDeviceToHost);
    cudaFree(tmp);
    SG_CHECK(r == ncclSuccess, SG_ERR_NCCL, "param export: %s", ncclGetErrorString(r));
    SG_CHECK(e == cudaSuccess, SG_ERR_CUDA, "param export: %s", cudaGetErrorString(e));
  }
  from_internal(P, q, h.data() + q.store_off, P.rank, user);
  return SG_OK;
}

void apply_fusion(sg_net* n) {
  const Plan& P = PL(n);
  const int nl = (int)P.layers.size();
  n->data = n->data_own;
  n->relu_of.assign(nl, -1);
  n->fused_away.assign(nl, 0);
  n->relu_after.assign(nl, -1);
  n->relu_into.assign(nl, -1);
  n->bwd_fused_away.assign(nl, 0);
  n->lrn_after.assign(nl, -1);
  n->lrn_fused.assign(nl, 0);
  n->pool_into.assign(nl, -1);
  n->pool_bwd_fused.assign(nl, 0);
  if (!n->fuse) return;
  std::vector<int> consumers(nl, 0), consumer(nl, -1);
  for (int c = 0; c < nl; ++c)
    if (P.layers[c].src >= 0) {
      ++consumers[P.layers[c].src];
      consumer[P.layers[c].src] = c;
    }
  for (int j = 0; j < nl; ++j) {
    const LayerPlan& R = P.layers[j];
    if (R.kind != SG_RELU || R.src < 0) continue;
    const LayerPlan& S = P.layers[R.src];
    // forward: a pooling layer also writes the ReLU of its output
    if ((S.kind == SG_POOL_MAX || S.kind == SG_POOL_AVG) && S.blob_floats() == R.blob_floats() && S.ld == R.ld &&
        S.nblocks == R.nblocks) {
      n->relu_after[R.src] = j;
      n->fused_away[j] = 1;
    }
    // backward: the ReLU's single consumer (LRN / pooling) also applies the ReLU mask
    const int c = consumer[j];
    if (consumers[j] == 1 && S.kind != SG_INPUT &&
        (P.layers[c].kind == SG_LRN || P.layers[c].kind == SG_POOL_MAX || P.layers[c].kind == SG_POOL_AVG)) {
      n->relu_into[c] = j;
      n->bwd_fused_away[j] = 1;
    }
  }
  for (int j = 0; j < nl; ++j) {
    const LayerPlan& R = P.layers[j];
    if (R.kind != SG_RELU || R.src < 0) continue;
    const int i = R.src;
    const LayerPlan& L = P.layers[i];
    if (L.kind != SG_CONV && L.kind != SG_INNER_PRODUCT) continue;
    if (L.blob_floats() != R.blob_floats() || L.ld != R.ld || L.nblocks != R.nblocks) continue;
    n->relu_of[i] = j;
    n->fused_away[j] = 1;
    n->data[i] = n->data[j];
  }
  // pooling [-> ReLU] -> LRN: one kernel (the pool feeds only the ReLU / LRN)
  for (int k = 0; k < nl; ++k) {
    const LayerPlan& Lk = P.layers[k];
    if (Lk.kind != SG_LRN || Lk.src < 0) continue;
    int pool = Lk.src;
    if (P.layers[pool].kind == SG_RELU) {
      const int j = pool;
      pool = P.layers[j].src;
      if (pool < 0 || n->relu_after[pool] != j || consumers[j] != 1) continue;
    }
    const LayerPlan& Lp = P.layers[pool];
    if ((Lp.kind != SG_POOL_MAX && Lp.kind != SG_POOL_AVG) || consumers[pool] != 1) continue;
    const LrnShape ls{Lk.rows * Lk.h * Lk.w, Lk.c, Lk.lrn_size, Lk.alpha, Lk.beta, Lk.k};
    if (!pool_lrn_fusable(pool_shape(Lp, P.layers[Lp.src]), ls)) continue;
    n->lrn_after[pool] = k;
    n->lrn_fused[k] = 1;
  }
  // first-layer convolution -> max pool: the pool's backward runs inside the
  // convolution's weight-gradient kernel (conv_img4_pool_bwd)
  for (int i = 0; i < nl; ++i) {
    const LayerPlan& L = P.layers[i];
    if (L.kind != SG_CONV || L.src < 0 || P.layers[L.src].kind != SG_INPUT || consumers[i] != 1) continue;
    const int c = consumer[i];
    const LayerPlan& Lc = P.layers[c];
    if (Lc.kind != SG_POOL_MAX || n->relu_into[c] >= 0) continue;
    if (!conv_img4_pool_bwd_ok(conv_shape(L, P.layers[L.src]), pool_shape(Lc, L))) continue;
    n->pool_into[i] = c;
    n->pool_bwd_fused[c] = 1;
  }
}

sg_status destroy_net(sg_net* n) {
  if (!n) return SG_OK;
  cudaSetDevice(n->cl ? n->cl->device : 0);
  if (n->cs) cudaStreamSynchronize(n->cs);
  if (n->ps) cudaStreamSynchronize(n->ps);
  if (n->us) cudaStreamSynchronize(n->us);
  if (n->gexec) cudaGraphExecDestroy(n->gexec);
  if (n->px) px_destroy(n->px, n->cl ? n->cl->comm_par : nullptr);
  for (void* p : n->allocs) cudaFree(p);
  for (auto e : n->ev_grad) cudaEventDestroy(e);
  for (auto e : n->ev_upd) cudaEventDestroy(e);
  for (auto e : n->ev_dy) cudaEventDestroy(e);
  for (auto e : n->ev_wg) cudaEventDestroy(e);
  for (auto e : {n->ev_in, n->ev_out, n->ev_fork, n->ev_join, n->ev_join_u})
    if (e) cudaEventDestroy(e);
  for (auto e : n->pev) cudaEventDestroy(e);
  if (n->cs) cudaStreamDestroy(n->cs);
  if (n->ps) cudaStreamDestroy(n->ps);
  if (n->us) cudaStreamDestroy(n->us);
  if (n->hs) cudaStreamDestroy(n->hs);
  for (int k = 0; k < 2; ++k) {
    if (n->ev_copied[k]) cudaEventDestroy(n->ev_copied[k]);
    if (n->ev_free[k]) cudaEventDestroy(n->ev_free[k]);
  }
  delete n;
  return SG_OK;
}

sg_status create_net(sg_cluster* c, const sg_net_cfg* cfg, sg_net* n) {
  SG_TRY(build_plan(cfg, c->rank, c->world, &n->plan.p, c->force));
  const Plan& P = n->plan.p;
  SG_CUDA(cudaSetDevice(c->device));
  SG_CUDA(cudaStreamCreateWithFlags(&n->cs, cudaStreamNonBlocking));
  SG_CUDA(cudaStreamCreateWithFlags(&n->ps, cudaStreamNonBlocking));
  for (cudaEvent_t* e : {&n->ev_in, &n->ev_out, &n->ev_fork, &n->ev_join})
    SG_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  const int nl = (int)P.layers.size();
  n->data.assign(nl, nullptr);
  n->grad.assign(nl, nullptr);
  n->scale.assign(nl, nullptr);
  n->s2d_x.assign(nl, nullptr);
  n->s2d_w.assign(nl, nullptr);
  n->s2d_dw.assign(nl, nullptr);
  n->mask.assign(nl, nullptr);
  n->ev_grad.resize(nl);
  n->ev_upd.resize(nl);
  n->ev_dy.resize(nl);
  n->ev_wg.resize(nl);
  n->wg_on_ps.assign(nl, 0);
  n->upd_in_bwd.assign(nl, 0);
  n->upd_bwd_stream.assign(nl, nullptr);
  {
    const char* env = getenv("SG_FUSE_UPDATE");
    n->fuse_update = env ? atoi(env) != 0 : true;
  }
  n->upd_pending.assign(nl, 0);
  n->fwd_done.assign(nl, 0);
  n->bwd_done.assign(nl, 0);
  for (int i = 0; i < nl; ++i) {
    SG_CUDA(cudaEventCreateWithFlags(&n->ev_grad[i], cudaEventDisableTiming));
    SG_CUDA(cudaEventCreateWithFlags(&n->ev_upd[i], cudaEventDisableTiming));
    SG_CUDA(cudaEventCreateWithFlags(&n->ev_dy[i], cudaEventDisableTiming));
    SG_CUDA(cudaEventCreateWithFlags(&n->ev_wg[i], cudaEventDisableTiming));
  }
  size_t ws = 1 << 16;
  auto need = [&](size_t f) {
    if (f > ws) ws = f;
  };
  for (int i = 0; i < nl; ++i) {
    const LayerPlan& L = P.layers[i];
    if (L.kind == SG_SOFTMAX_CE || L.kind == SG_EUCLIDEAN) continue;
    SG_TRY(dalloc_t(n, (size_t)L.blob_floats(), &n->data[i]));
    if (L.kind != SG_INPUT) SG_TRY(dalloc_t(n, (size_t)L.blob_floats(), &n->grad[i]));
    if (L.kind == SG_POOL_MAX) SG_TRY(dalloc_t(n, (size_t)L.blob_floats(), &n->mask[i]));
    if (L.kind == SG_LRN) SG_TRY(dalloc_t(n, (size_t)L.blob_floats(), &n->scale[i]));
    if (L.kind == SG_CONV) {
      const LayerPlan& S = P.layers[L.src];
      const int Kg = L.kernel * L.kernel * S.c;
      need(gemm_ws_floats((int)(L.rows * L.h * L.w), L.c, Kg));
      need(gemm_ws_floats(Kg, L.c, (int)(L.rows * L.h * L.w)));
      need(gemm_ws_floats((int)(L.rows * S.h * S.w), S.c, L.kernel * L.kernel * L.c));
      need(colsum_ws_floats((int)(L.rows * L.h * L.w), L.c));
      need(conv_img_wgrad_ws_floats(conv_shape(L, S)));
      need(conv_img4_wgrad_ws_floats(conv_shape(L, S)));
      const ConvShape cs = conv_shape(L, S);
      if (conv_s2d_ok(cs) && !conv_img_fwd_ok(cs)) {
        const ConvShape t = conv_s2d_shape(cs);
        const int Kt = t.R * t.S * t.C;
        SG_TRY(dalloc_t(n, conv_s2d_x_floats(cs), &n->s2d_x[i]));
        SG_TRY(dalloc_t(n, conv_s2d_w_floats(cs), &n->s2d_w[i]));
        SG_TRY(dalloc_t(n, conv_s2d_w_floats(cs), &n->s2d_dw[i]));
        // the input layer writes the image directly (channel padding to 4 and one consumer)
        if (S.kind == SG_INPUT && S.image && S.c == 4 && S.c_real <= 4 && n->s2d_of_input < 0) {
          int consumers = 0;
          for (int j = 0; j < nl; ++j) consumers += P.layers[j].src == L.src;
          if (consumers == 1) n->s2d_of_input = i;
        }
        need(gemm_ws_floats((int)(L.rows * L.h * L.w), L.c, Kt));
        need(gemm_ws_floats(Kt + 1, L.c, (int)(L.rows * L.h * L.w)));
        need(conv_img_wgrad_ws_floats(t));
      }
    }
    if (L.kind == SG_INNER_PRODUCT) {
      need(gemm_ws_floats((int)L.rows, (int)L.nout, (int)L.kin));
      need(gemm_ws_floats((int)L.kin, (int)L.nout, (int)L.rows));
      need(gemm_ws_floats((int)L.rows, (int)L.kin, (int)L.nout));
      need(colsum_ws_floats((int)L.rows, (int)L.nout));
    }
  }
  // the input blob's source (input layer pad) is the user's x; gradients of the
  // input layer are never formed.  The loss layer writes dz into its source's grad.
  SG_TRY(dalloc_t(n, ws, &n->ws.ptr));
  n->ws.floats = ws;
  {
    const char* env = getenv("SG_S2D_WGRAD");
    n->s2d_wgrad = env ? atoi(env) != 0 : true;
  }
  {
    const char* env = getenv("SG_WGRAD_SIDE");
    n->wgrad_side = env ? atoi(env) != 0 : true;
  }
  if (n->wgrad_side) {
    SG_TRY(dalloc_t(n, ws, &n->ws2.ptr));
    n->ws2.floats = ws;
    const char* env = getenv("SG_UPDATE_STREAM");
    if (!env || atoi(env) != 0) {
      SG_CUDA(cudaStreamCreateWithFlags(&n->us, cudaStreamNonBlocking));
      SG_CUDA(cudaEventCreateWithFlags(&n->ev_join_u, cudaEventDisableTiming));
    }
  }
  SG_TRY(dalloc_t(n, (size_t)std::max<int64_t>(P.loss_rows, 1), &n->row_loss));
  n->data[P.loss] = n->row_loss;
  SG_TRY(dalloc_t(n, 4, &n->loss_int));
  SG_TRY(dalloc_t(n, 4, &n->lr_dev));
  SG_TRY(dalloc_t(n, 4, &n->err));
  SG_TRY(dalloc_t(n, (size_t)std::max<int64_t>(P.loss_rows, 1), &n->labels));
  {
    const LayerPlan& in = P.layers[0];
    SG_TRY(dalloc_t(n, (size_t)(in.rows * in.feat), &n->x_stage));
    // the pipelined host path's second input slot, label slots, copy stream, events
    SG_TRY(dalloc_t(n, (size_t)(in.rows * in.feat), &n->x_stage2));
    SG_CUDA(cudaStreamCreateWithFlags(&n->hs, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k) {
      SG_CUDA(cudaEventCreateWithFlags(&n->ev_copied[k], cudaEventDisableTiming));
      SG_CUDA(cudaEventCreateWithFlags(&n->ev_free[k], cudaEventDisableTiming));
      SG_TRY(dalloc_t(n, (size_t)std::max<int64_t>(P.loss_rows, 1), &n->lab_stage[k]));
    }
  }
  if (P.layers[P.loss].kind == SG_EUCLIDEAN && P.layers[0].rn_data)
    SG_TRY(dalloc_t(n, (size_t)P.layers[0].blob_floats(), &n->x_exact));
  for (const StorePlan& S : P.stores) {
    float *w, *g, *m, *v;
    const size_t own = (size_t)(S.sharded ? S.padded / P.world : S.padded);
    SG_TRY(dalloc_t(n, (size_t)S.padded, &w));
    SG_TRY(dalloc_t(n, (size_t)S.padded, &g));
    SG_TRY(dalloc_t(n, own, &m));
    SG_TRY(dalloc_t(n, own, &v));
    n->sw.push_back(w);
    n->sgr.push_back(g);
    n->sm.push_back(m);
    n->sv.push_back(v);
  }
  n->data_own = n->data;
  apply_fusion(n);
  SG_CUDA(cudaDeviceSynchronize());
  return SG_OK;
}

}  // namespace
}  // namespace sg

using namespace sg;

extern "C" {

// ------------------------------------------------------------------ cluster --
SG_API sg_status sg_get_unique_id(uint8_t out[128]) {
  SG_CHECK(out, SG_ERR_INVALID_ARG, "null output");
  ncclUniqueId id;
  SG_NCCL(ncclGetUniqueId(&id));
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  memcpy(out, &id, 128);
  return SG_OK;
}

SG_API sg_status sg_cluster_create(const sg_cluster_cfg* cfg, sg_cluster** out) {
  SG_CHECK(cfg && out, SG_ERR_INVALID_ARG, "sg_cluster_create: null argument");
  SG_CHECK(cfg->world_size >= 1 && cfg->rank >= 0 && cfg->rank < cfg->world_size, SG_ERR_INVALID_ARG,
           "cluster: rank %d world %d", cfg->rank, cfg->world_size);
  SG_CHECK(cfg->nworker_groups == 1 && cfg->nserver_groups == 1, SG_ERR_UNSUPPORTED,
           "unsupported: %d worker groups / %d server groups (asynchronous frameworks are out of scope; "
           "synchronous training uses 1 worker group and 1 server group, P:411-422)",
           cfg->nworker_groups, cfg->nserver_groups);
  SG_CHECK(cfg->workers_per_group == cfg->world_size && cfg->servers_per_group == cfg->world_size,
           SG_ERR_UNSUPPORTED, "unsupported: %d workers / %d servers per group on %d ranks (AllReduce framework binds "
           "one worker and one server per rank, P:419-422)",
           cfg->workers_per_group, cfg->servers_per_group, cfg->world_size);
  SG_CUDA(cudaSetDevice(cfg->device));
  sg_cluster* c = new sg_cluster();
  c->rank = cfg->rank;
  c->world = cfg->world_size;
  c->device = cfg->device;
  c->force = c->world == 1 && cfg->exercise_collectives != 0;
  if (c->world > 1 || c->force) {
    ncclUniqueId id;
    memcpy(&id, cfg->nccl_id, 128);
    ncclResult_t r = ncclCommInitRank(&c->comm_act, c->world, id, c->rank);
    if (r == ncclSuccess) r = ncclCommSplit(c->comm_act, 0, c->rank, &c->comm_par, nullptr);
    if (r != ncclSuccess) {
      delete c;
      SG_FAIL(SG_ERR_NCCL, "NCCL communicator creation failed: %s", ncclGetErrorString(r));
    }
    // Establish every connection now (one of each collective kind on both
    // communicators, serialised), so no lazy connection setup can happen while
    // kernels of the other communicator are in flight during a step.
    float* buf = nullptr;
    const size_t cnt = 1024;
    cudaError_t ce = cudaMalloc(&buf, 2 * cnt * c->world * sizeof(float));
    if (ce != cudaSuccess) {
      delete c;
      SG_FAIL(SG_ERR_OOM, "cluster warm-up buffer: %s", cudaGetErrorString(ce));
    }
    cudaMemset(buf, 0, 2 * cnt * c->world * sizeof(float));
    for (ncclComm_t comm : {c->comm_act, c->comm_par}) {
      if (r == ncclSuccess) r = ncclAllReduce(buf, buf, cnt, ncclFloat, ncclSum, comm, 0);
      if (r == ncclSuccess) r = ncclAllGather(buf, buf + cnt * c->world, cnt, ncclFloat, comm, 0);
      if (r == ncclSuccess) r = ncclReduceScatter(buf + cnt * c->world, buf, cnt, ncclFloat, ncclSum, comm, 0);
      if (r == ncclSuccess) {
        r = ncclGroupStart();
        for (int j = 0; j < c->world && r == ncclSuccess; ++j) {
          r = ncclSend(buf + j * cnt, cnt, ncclFloat, j, comm, 0);
          if (r == ncclSuccess) r = ncclRecv(buf + cnt * c->world + j * cnt, cnt, ncclFloat, j, comm, 0);
        }
        ncclResult_t r2 = ncclGroupEnd();
        if (r == ncclSuccess) r = r2;
      }
      if (cudaDeviceSynchronize() != cudaSuccess && r == ncclSuccess) r = ncclUnhandledCudaError;
    }
    cudaFree(buf);
    if (r != ncclSuccess) {
      SG_FAIL(SG_ERR_NCCL, "NCCL warm-up failed: %s", ncclGetErrorString(r));
    }
  }
  *out = c;
  return SG_OK;
}

SG_API sg_status sg_cluster_framework(const sg_cluster* c, const char** name) {
  SG_CHECK(c && name, SG_ERR_INVALID_ARG, "null argument");
  *name = "AllReduce";
  return SG_OK;
}

SG_API sg_status sg_cluster_destroy(sg_cluster* c) {
  if (!c) return SG_OK;
  if (c->comm_par) ncclCommDestroy(c->comm_par);
  if (c->comm_act) ncclCommDestroy(c->comm_act);
  delete c;
  return SG_OK;
}

// ---------------------------------------------------------------------- net --
SG_API sg_status sg_net_create(sg_cluster* c, const sg_net_cfg* cfg, sg_net** out) {
  SG_CHECK(c && cfg && out, SG_ERR_INVALID_ARG, "sg_net_create: null argument");
  sg_net* n = new sg_net();
  n->cl = c;
  sg_status st = create_net(c, cfg, n);
  if (st != SG_OK) {
    std::string msg = get_error();
    destroy_net(n);
    set_error("%s", msg.c_str());
    return st;
  }
  *out = n;
  return SG_OK;
}

SG_API sg_status sg_net_destroy(sg_net* n) { return destroy_net(n); }

SG_API sg_status sg_net_plan(const sg_net* n, const sg_plan** out) {
  SG_CHECK(n && out, SG_ERR_INVALID_ARG, "null argument");
  *out = &n->plan;
  return SG_OK;
}

SG_API sg_status sg_param_set_value(sg_net* n, int32_t p, const float* user) {
  SG_CHECK(n && user, SG_ERR_INVALID_ARG, "null argument");
  const Plan& P = PL(n);
  SG_CHECK(p >= 0 && p < (int)P.params.size(), SG_ERR_INVALID_ARG, "param index %d out of range", p);
  const ParamPlan& q = P.params[p];
  const StorePlan& S = P.stores[q.store];
  std::vector<float> h;
  to_internal(P, q, user, h);
  SG_CUDA(cudaSetDevice(n->cl->device));
  SG_CUDA(cudaStreamSynchronize(n->ps));
  if (n->us) SG_CUDA(cudaStreamSynchronize(n->us));
  SG_CUDA(cudaStreamSynchronize(n->cs));
  // fp32 master: the whole Param, or its part inside this rank's shard
  const int64_t shard = S.sharded ? S.padded / P.world : S.padded;
  const int64_t lo = S.sharded ? (int64_t)P.rank * shard : 0;
  const int64_t b0 = std::max<int64_t>(q.store_off, lo), b1 = std::min<int64_t>(q.store_off + q.isize, lo + shard);
  if (b1 > b0)
    SG_CUDA(cudaMemcpy(n->sm[q.store] + (b0 - lo), h.data() + (b0 - q.store_off), (size_t)(b1 - b0) * sizeof(float),
                       cudaMemcpyHostToDevice));
  // working copy: weights TF32-RN (reading A19), biases exact
  if (!q.is_bias)
    for (float& x : h) x = tf32_rna_host(x);
  SG_CUDA(cudaMemcpy(n->sw[q.store] + q.store_off, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice));
  return SG_OK;
}
SG_API sg_status sg_param_get_value(sg_net* n, int32_t p, float* user) {
  SG_CHECK(n, SG_ERR_INVALID_ARG, "null net");
  return param_export(n, p, 0, user);
}
SG_API sg_status sg_param_get_grad(sg_net* n, int32_t p, float* user) {
  SG_CHECK(n, SG_ERR_INVALID_ARG, "null net");
  return param_export(n, p, 1, user);
}
SG_API sg_status sg_param_get_history(sg_net* n, int32_t p, float* user) {
  SG_CHECK(n, SG_ERR_INVALID_ARG, "null net");
  return param_export(n, p, 2, user);
}
SG_API sg_status sg_param_get_working(sg_net* n, int32_t p, float* user) {
  SG_CHECK(n, SG_ERR_INVALID_ARG, "null net");
  return param_export(n, p, 3, user);
}

SG_API sg_status sg_updater_create(sg_net* n, const sg_updater_cfg* cfg, sg_updater** out) {
  SG_CHECK(n && cfg && out, SG_ERR_INVALID_ARG, "null argument");
  SG_CHECK(cfg->base_lr >= 0.f && cfg->momentum >= 0.f && cfg->momentum < 1.f && cfg->weight_decay >= 0.f,
           SG_ERR_CONFIG, "updater: base_lr=%g momentum=%g weight_decay=%g", (double)cfg->base_lr,
           (double)cfg->momentum, (double)cfg->weight_decay);
  SG_CHECK(cfg->lr_policy == 0 || (cfg->lr_policy == 1 && cfg->step_size > 0), SG_ERR_CONFIG,
           "updater: lr_policy=%d step_size=%d", cfg->lr_policy, cfg->step_size);
  SG_CHECK(cfg->type == SG_UPD_SGD_MOMENTUM || (cfg->type == SG_UPD_ADAGRAD && cfg->momentum == 0.f), SG_ERR_CONFIG,
           "updater: type=%d momentum=%g (AdaGrad takes no momentum)", cfg->type, (double)cfg->momentum);
  sg_updater* u = new sg_updater();
  memset(u, 0, sizeof(*u));  // compared bytewise by the graph cache
  u->cfg = *cfg;
  u->s = cfg->grad_scale > 0.f ? cfg->grad_scale : PL(n).grad_scale;
  u->eps = cfg->eps > 0.f ? cfg->eps : 1e-8f;
  *out = u;
  return SG_OK;
}
SG_API sg_status sg_updater_destroy(sg_updater* u) {
  delete u;
  return SG_OK;
}

SG_API sg_status sg_net_set_input(sg_net* n, const float* x, const int32_t* labels, void* stream) {
  SG_CHECK(n, SG_ERR_INVALID_ARG, "null net");
  SG_TRY(enter(n, stream));
  SG_TRY(set_input(n, x, labels));
  return leave(n, stream);
}

SG_API sg_status sg_net_collect(sg_net* n, int32_t layer, void* stream) {
  SG_CHECK(n && layer >= 0 && layer < (int)PL(n).layers.size(), SG_ERR_INVALID_ARG, "bad layer %d", layer);
  SG_TRY(enter(n, stream));
  SG_TRY(collect(n, layer));
  return leave(n, stream);
}

SG_API sg_status sg_layer_compute_feature(sg_net* n, int32_t layer, void* stream) {
  SG_CHECK(n && layer >= 0 && layer < (int)PL(n).layers.size(), SG_ERR_INVALID_ARG, "bad layer %d", layer);
  const Plan& P = PL(n);
  SG_CHECK(n->input_set, SG_ERR_SEQUENCE, "sequence error: ComputeFeature(%s) before sg_net_set_input",
           P.layers[layer].name.c_str());
  const int src = P.layers[layer].src;
  SG_CHECK(src < 0 || n->fwd_done[src], SG_ERR_SEQUENCE,
           "sequence error: ComputeFeature(%s) before ComputeFeature of its source %s", P.layers[layer].name.c_str(),
           P.layers[src].name.c_str());
  SG_TRY(enter(n, stream));
  long long l0 = g_kernel_launches;
  SG_TRY(forward(n, layer));
  n->last_launches = g_kernel_launches - l0;
  n->fwd_done[layer] = 1;
  return leave(n, stream);
}

SG_API sg_status sg_layer_compute_gradient(sg_net* n, int32_t layer, void* stream) {
  SG_CHECK(n && layer >= 0 && layer < (int)PL(n).layers.size(), SG_ERR_INVALID_ARG, "bad layer %d", layer);
  const Plan& P = PL(n);
  SG_CHECK(n->fwd_done[P.loss], SG_ERR_SEQUENCE,
           "sequence error: ComputeGradient(%s) before the forward pass reached the loss",
           P.layers[layer].name.c_str());
  for (int j = layer + 1; j < (int)P.layers.size(); ++j)
    if (P.layers[j].src == layer)
      SG_CHECK(n->bwd_done[j] || P.layers[j].kind == SG_SOFTMAX_CE || P.layers[j].kind == SG_EUCLIDEAN,
               SG_ERR_SEQUENCE, "sequence error: ComputeGradient(%s) before ComputeGradient of its consumer %s",
               P.layers[layer].name.c_str(), P.layers[j].name.c_str());
  SG_TRY(enter(n, stream));
  SG_TRY(backward(n, layer));
  n->bwd_done[layer] = 1;
  return leave(n, stream);
}

SG_API sg_status sg_net_update(sg_net* n, sg_updater* u, int32_t layer, int64_t step, void* stream) {
  SG_CHECK(n && u && layer >= 0 && layer < (int)PL(n).layers.size(), SG_ERR_INVALID_ARG, "bad argument");
  SG_CHECK(n->bwd_done[layer] || PL(n).layers[layer].store < 0, SG_ERR_PROTOCOL,
           "protocol error: Update(%s) before its ComputeGradient in this step", PL(n).layers[layer].name.c_str());
  SG_TRY(enter(n, stream));
  if (lr_at(u->cfg, step) != n->lr_last) {
    n->lr_last = lr_at(u->cfg, step);
    cudaError_t e = fill_scalar(n->lr_dev, n->lr_last, n->cs);
    SG_CHECK(e == cudaSuccess, SG_ERR_CUDA, "update: %s", cudaGetErrorString(e));
  }
  SG_TRY(update(n, u, layer));
  return leave(n, stream);
}

SG_API sg_status sg_net_loss(sg_net* n, float* loss_dev, void* stream) {
  SG_CHECK(n && loss_dev, SG_ERR_INVALID_ARG, "null argument");
  SG_TRY(enter(n, stream));
  SG_TRY(loss_reduce(n));
  SG_CUDA(cudaMemcpyAsync(loss_dev, n->loss_int, sizeof(float), cudaMemcpyDeviceToDevice, n->cs));
  return leave(n, stream);
}

SG_API sg_status sg_train_one_batch(sg_net* n, sg_updater* u, int64_t step, const float* x, const int32_t* labels,
                                    float* loss_dev, void* stream) {
  SG_CHECK(n && u && x, SG_ERR_INVALID_ARG, "sg_train_one_batch: null argument");
  const Plan& P = PL(n);
  SG_TRY(enter(n, stream));
  long long l0 = g_kernel_launches;
  if (lr_at(u->cfg, step) != n->lr_last) {  // fixed / step schedules change it rarely
    n->lr_last = lr_at(u->cfg, step);
    cudaError_t e = fill_scalar(n->lr_dev, n->lr_last, n->cs);
    SG_CHECK(e == cudaSuccess, SG_ERR_CUDA, "train: %s", cudaGetErrorString(e));
  }
  if (n->graph_on) {
    SG_TRY(set_input(n, x, labels));
    SG_TRY(forward(n, 0));  // input layer on the caller's buffer, then the captured rest of the step
    if (!n->gexec || memcmp(&n->graph_upd, u, sizeof(sg_updater)) != 0) {
      if (n->gexec) cudaGraphExecDestroy(n->gexec), n->gexec = nullptr;
      cudaGraph_t g;
      long long c0 = g_kernel_launches;
      SG_CUDA(cudaStreamBeginCapture(n->cs, cudaStreamCaptureModeThreadLocal));
      n->capturing = true;
      sg_status st = step_body(n, u);
      n->capturing = false;
      cudaError_t ce = cudaStreamEndCapture(n->cs, &g);
      SG_TRY(st);
      SG_CHECK(ce == cudaSuccess, SG_ERR_CUDA, "graph capture failed: %s", cudaGetErrorString(ce));
      ce = cudaGraphInstantiate(&n->gexec, g, 0);
      cudaGraphDestroy(g);
      SG_CHECK(ce == cudaSuccess, SG_ERR_CUDA, "graph instantiation failed: %s", cudaGetErrorString(ce));
      n->graph_launches = g_kernel_launches - c0;
      n->graph_upd = *u;
    }
    SG_CUDA(cudaGraphLaunch(n->gexec, n->cs));
    n->last_launches = (g_kernel_launches - l0) + n->graph_launches;
  } else {
    SG_TRY(set_input(n, x, labels));
    SG_TRY(step_body(n, u));
    n->last_launches = g_kernel_launches - l0;
  }
  if (loss_dev) SG_CUDA(cudaMemcpyAsync(loss_dev, n->loss_int, sizeof(float), cudaMemcpyDeviceToDevice, n->cs));
  n->input_set = false;
  return leave(n, stream);
}

SG_API sg_status sg_train_one_batch_host(sg_net* n, sg_updater* u, int64_t step, const float* x_host,
                                         const int32_t* labels_host, float* loss_host, void* stream) {
  SG_CHECK(n && u && x_host && loss_host, SG_ERR_INVALID_ARG, "sg_train_one_batch_host: null argument");
  const Plan& P = PL(n);
  const LayerPlan& in = P.layers[0];
  SG_CUDA(cudaSetDevice(n->cl->device));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // host -> device staging of this step's inputs (part of the measured end-to-end path)
  SG_CUDA(cudaMemcpyAsync(n->x_stage, x_host, (size_t)(in.rows * in.feat) * sizeof(float), cudaMemcpyHostToDevice,
                          st));
  const int32_t* ldev = nullptr;
  if (labels_host && P.layers[P.loss].kind == SG_SOFTMAX_CE) {
    SG_CUDA(cudaMemcpyAsync(n->labels, labels_host, (size_t)P.loss_rows * sizeof(int32_t), cudaMemcpyHostToDevice,
                            st));
    ldev = n->labels;
  }
  SG_TRY(sg_train_one_batch(n, u, step, n->x_stage, ldev, n->loss_int, stream));
  SG_CUDA(cudaMemcpyAsync(loss_host, n->loss_int, sizeof(float), cudaMemcpyDeviceToHost, st));
  SG_CUDA(cudaStreamSynchronize(st));
  return SG_OK;
}

SG_API sg_status sg_train_one_batch_host_async(sg_net* n, sg_updater* u, int64_t step, const float* x_host,
                                               const int32_t* labels_host, float* loss_host, void* stream) {
  SG_CHECK(n && u && x_host && loss_host, SG_ERR_INVALID_ARG, "sg_train_one_batch_host_async: null argument");
  const Plan& P = PL(n);
  const LayerPlan& in = P.layers[0];
  SG_CUDA(cudaSetDevice(n->cl->device));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int k = n->stage_k;
  n->stage_k ^= 1;
  float* xs = k ? n->x_stage2 : n->x_stage;
  // the step that last read slot k is done; then this step's inputs, on the copy
  // stream (overlapping the previous step's compute)
  if (n->stage_used[k]) SG_CUDA(cudaStreamWaitEvent(n->hs, n->ev_free[k], 0));
  SG_CUDA(cudaMemcpyAsync(xs, x_host, (size_t)(in.rows * in.feat) * sizeof(float), cudaMemcpyHostToDevice, n->hs));
  const int32_t* ldev = nullptr;
  if (labels_host && P.layers[P.loss].kind == SG_SOFTMAX_CE) {
    SG_CUDA(cudaMemcpyAsync(n->lab_stage[k], labels_host, (size_t)P.loss_rows * sizeof(int32_t),
                            cudaMemcpyHostToDevice, n->hs));
    ldev = n->lab_stage[k];
  }
  SG_CUDA(cudaEventRecord(n->ev_copied[k], n->hs));
  SG_CUDA(cudaStreamWaitEvent(st, n->ev_copied[k], 0));
  SG_TRY(sg_train_one_batch(n, u, step, xs, ldev, n->loss_int, stream));
  SG_CUDA(cudaEventRecord(n->ev_free[k], st));
  n->stage_used[k] = true;
  SG_CUDA(cudaMemcpyAsync(loss_host, n->loss_int, sizeof(float), cudaMemcpyDeviceToHost, st));
  return SG_OK;
}

SG_API sg_status sg_net_sync(sg_net* n) {
  SG_CHECK(n, SG_ERR_INVALID_ARG, "null net");
  SG_CUDA(cudaSetDevice(n->cl->device));
  SG_CUDA(cudaStreamSynchronize(n->ps));
  if (n->us) SG_CUDA(cudaStreamSynchronize(n->us));
  if (n->hs) SG_CUDA(cudaStreamSynchronize(n->hs));
  SG_CUDA(cudaStreamSynchronize(n->cs));
  int flags = 0;
  SG_CUDA(cudaMemcpy(&flags, n->err, sizeof(int), cudaMemcpyDeviceToHost));
  if (flags) SG_CUDA(cudaMemset(n->err, 0, sizeof(int)));
  SG_CHECK(!(flags & 1), SG_ERR_LABEL, "label error: a label is outside [0, %d)", PL(n).num_classes);
  SG_CHECK(!(flags & 2), SG_ERR_DIVERGED, "diverged: non-finite loss");
  SG_CHECK(!px_failed(n->px), SG_ERR_CUDA,
           "peer exchange: a barrier timed out (a rank did not arrive); the exchange is disabled for this net");
  return SG_OK;
}

SG_API sg_status sg_net_enable_graph(sg_net* n, int32_t enable) {
  SG_CHECK(n, SG_ERR_INVALID_ARG, "null net");
  n->graph_on = enable != 0;
  if (!n->graph_on && n->gexec) {
    cudaStreamSynchronize(n->cs);
    cudaGraphExecDestroy(n->gexec);
    n->gexec = nullptr;
  }
  return SG_OK;
}

SG_API sg_status sg_net_profile(sg_net* n, int32_t enable) {
  SG_CHECK(n, SG_ERR_INVALID_ARG, "null net");
  SG_CUDA(cudaSetDevice(n->cl->device));
  const int slots = 4 * (int)PL(n).layers.size();
  if (enable && n->pev.empty()) {
    n->pev.resize(2 * slots);
    for (auto& e : n->pev) SG_CUDA(cudaEventCreate(&e));
    n->pused.assign(slots, 0);
    n->pacc.assign(slots, 0.0);
    n->pcnt.assign(slots, 0);
  }
  n->prof = enable != 0;
  n->prof_concurrent = enable == 2;
  if (n->gexec) {  // re-capture with / without the timing events
    SG_CUDA(cudaStreamSynchronize(n->cs));
    cudaGraphExecDestroy(n->gexec);
    n->gexec = nullptr;
  }
  return SG_OK;
}

SG_API sg_status sg_net_op_times(sg_net* n, double* ms, int64_t* counts, int32_t cap, int32_t* nslots,
                                 int32_t reset) {
  SG_CHECK(n && nslots, SG_ERR_INVALID_ARG, "null argument");
  const int slots = 4 * (int)PL(n).layers.size();
  *nslots = slots;
  if (n->pev.empty()) return SG_OK;
  SG_CUDA(cudaSetDevice(n->cl->device));
  SG_CUDA(cudaStreamSynchronize(n->ps));
  if (n->us) SG_CUDA(cudaStreamSynchronize(n->us));
  SG_CUDA(cudaStreamSynchronize(n->cs));
  for (int s = 0; s < slots; ++s) {
    if (!n->pused[s]) continue;
    float t = 0.f;
    if (cudaEventElapsedTime(&t, n->pev[2 * s], n->pev[2 * s + 1]) == cudaSuccess) {
      n->pacc[s] += t;
      n->pcnt[s] += 1;
    } else {
      cudaGetLastError();
    }
  }
  for (int s = 0; s < slots && s < cap; ++s) {
    if (ms) ms[s] = n->pacc[s];
    if (counts) counts[s] = n->pcnt[s];
  }
  if (reset) {
    std::fill(n->pacc.begin(), n->pacc.end(), 0.0);
    std::fill(n->pcnt.begin(), n->pcnt.end(), 0);
  }
  return SG_OK;
}

SG_API sg_status sg_net_op_timeline(sg_net* n, double* t_start, double* t_end, int32_t cap, int32_t* nslots) {
  SG_CHECK(n && nslots && t_start && t_end, SG_ERR_INVALID_ARG, "null argument");
  const int slots = 4 * (int)PL(n).layers.size();
  *nslots = slots;
  SG_CHECK(!n->pev.empty(), SG_ERR_INVALID_ARG, "profiling never enabled");
  SG_CUDA(cudaSetDevice(n->cl->device));
  SG_CUDA(cudaStreamSynchronize(n->ps));
  if (n->us) SG_CUDA(cudaStreamSynchronize(n->us));
  SG_CUDA(cudaStreamSynchronize(n->cs));
  int first = -1;
  for (int s = 0; s < slots && first < 0; ++s)
    if (n->pused[s]) first = s;
  for (int s = 0; s < slots && s < cap; ++s) {
    t_start[s] = t_end[s] = -1.0;
    float a = 0.f, b = 0.f;
    if (first < 0 || !n->pused[s]) continue;
    if (cudaEventElapsedTime(&a, n->pev[2 * first], n->pev[2 * s]) == cudaSuccess &&
        cudaEventElapsedTime(&b, n->pev[2 * first], n->pev[2 * s + 1]) == cudaSuccess) {
      t_start[s] = a;
      t_end[s] = b;
    } else {
      cudaGetLastError();
    }
  }
  return SG_OK;
}

SG_API sg_status sg_net_set_overlap(sg_net* n, int32_t enable) {
  SG_CHECK(n, SG_ERR_INVALID_ARG, "null net");
  SG_CUDA(cudaSetDevice(n->cl->device));
  SG_CUDA(cudaStreamSynchronize(n->cs));
  n->overlap = enable != 0;
  if (n->gexec) {
    cudaGraphExecDestroy(n->gexec);
    n->gexec = nullptr;
  }
  return SG_OK;
}

SG_API sg_status sg_net_set_exchange(sg_net* n, int32_t mode) {
  SG_CHECK(n && (mode == 0 || mode == 1), SG_ERR_INVALID_ARG, "sg_net_set_exchange: bad argument");
  const Plan& P = PL(n);
  SG_CUDA(cudaSetDevice(n->cl->device));
  SG_CUDA(cudaStreamSynchronize(n->ps));
  if (n->us) SG_CUDA(cudaStreamSynchronize(n->us));
  SG_CUDA(cudaStreamSynchronize(n->cs));
  if (n->gexec) {  // the captured step encodes the exchange path
    cudaGraphExecDestroy(n->gexec);
    n->gexec = nullptr;
  }
  if (n->px) {
    px_destroy(n->px, n->cl->comm_par);
    n->px = nullptr;
  }
  n->px_sid.assign(P.stores.size(), -1);
  if (mode == 0) return SG_OK;
  SG_CHECK(P.dist && n->cl->comm_par, SG_ERR_CONFIG,
           "config error: the peer-memory exchange needs a partitioned net (world > 1 or exercise_collectives)");
  std::vector<PxStore> stores;
  for (size_t s = 0; s < P.stores.size(); ++s) {
    const StorePlan& S = P.stores[s];
    if (!S.sharded) continue;
    n->px_sid[s] = (int)stores.size();
    stores.push_back(PxStore{n->sgr[s], n->sw[s], n->sm[s], n->sv[s], S.padded, P.params[P.layers[S.layer].pW].isize});
  }
  sg_status st = px_create(n->cl->comm_par, P.rank, P.world, n->cl->device, stores, &n->px);
  if (st != SG_OK) {
    n->px = nullptr;
    n->px_sid.assign(P.stores.size(), -1);
  }
  return st;
}

SG_API sg_status sg_net_set_fusion(sg_net* n, int32_t enable) {
  SG_CHECK(n, SG_ERR_INVALID_ARG, "null net");
  SG_CUDA(cudaSetDevice(n->cl->device));
  SG_CUDA(cudaStreamSynchronize(n->cs));
  n->fuse = enable != 0;
  apply_fusion(n);
  if (n->gexec) {
    cudaGraphExecDestroy(n->gexec);
    n->gexec = nullptr;
  }
  return SG_OK;
}

SG_API sg_status sg_net_last_launch_count(const sg_net* n, int64_t* launches) {
  SG_CHECK(n && launches, SG_ERR_INVALID_ARG, "null argument");
  *launches = n->last_launches;
  return SG_OK;
}

SG_API sg_status sg_blob_size(sg_net* n, int32_t layer, int32_t which, size_t* bytes) {
  SG_CHECK(n && bytes && layer >= 0 && layer < (int)PL(n).layers.size() && which >= 0 && which <= 2,
           SG_ERR_INVALID_ARG, "bad blob request layer=%d which=%d", layer, which);
  const Plan& P = PL(n);
  const LayerPlan& L = P.layers[layer];
  *bytes = 0;
  if (which == 0) {
    *bytes = (L.kind == SG_SOFTMAX_CE || L.kind == SG_EUCLIDEAN) ? (size_t)P.loss_rows * 4 : L.blob_floats() * 4;
  } else if (which == 1) {
    if (L.src >= 0 && P.layers[L.src].kind != SG_INPUT) *bytes = P.layers[L.src].blob_floats() * 4;
  } else if (L.kind == SG_POOL_MAX) {
    *bytes = L.blob_floats() * 4;
  }
  return SG_OK;
}

SG_API sg_status sg_blob_get(sg_net* n, int32_t layer, int32_t which, void* dst, size_t bytes, void* stream) {
  size_t need;
  SG_TRY(sg_blob_size(n, layer, which, &need));
  SG_CHECK(need > 0 && dst && bytes >= need, SG_ERR_INVALID_ARG, "blob %d/%d: %zu bytes needed, %zu given", layer,
           which, need, bytes);
  const Plan& P = PL(n);
  const LayerPlan& L = P.layers[layer];
  SG_TRY(enter(n, stream));
  if (which == 0) {
    SG_CUDA(cudaMemcpyAsync(dst, n->data[layer], need, cudaMemcpyDeviceToDevice, n->cs));
  } else if (which == 1) {
    SG_CUDA(cudaMemcpyAsync(dst, n->grad[L.src], need, cudaMemcpyDeviceToDevice, n->cs));
  } else {
    cudaError_t e = pool_argmax_expand(pool_shape(L, P.layers[L.src]), n->mask[layer], (int32_t*)dst, n->cs);
    SG_CHECK(e == cudaSuccess, SG_ERR_CUDA, "argmax export: %s", cudaGetErrorString(e));
  }
  return leave(n, stream);
}

SG_API sg_status sg_blob_set(sg_net* n, int32_t layer, int32_t which, const void* src, size_t bytes, void* stream) {
  size_t need;
  SG_TRY(sg_blob_size(n, layer, which, &need));
  SG_CHECK(which <= 1 && need > 0 && src && bytes == need, SG_ERR_INVALID_ARG,
           "blob set %d/%d: %zu bytes expected, %zu given", layer, which, need, bytes);
  const LayerPlan& L = PL(n).layers[layer];
  SG_TRY(enter(n, stream));
  SG_CUDA(cudaMemcpyAsync(which == 0 ? n->data[layer] : n->grad[L.src], src, need, cudaMemcpyDeviceToDevice, n->cs));
  return leave(n, stream);
}

// ------------------------------------------------------ C5 server sync sweep --
SG_API sg_status sg_server_sync(sg_cluster* c, const sg_updater_cfg* cfg, int64_t step, float* grad, float* w,
                                float* v_shard, int64_t n, void* stream) {
  SG_CHECK(c && cfg && grad && w && v_shard, SG_ERR_INVALID_ARG, "sg_server_sync: null argument");
  SG_CHECK(n > 0 && n % (32LL * c->world) == 0, SG_ERR_PARTITION, "partition error: n=%lld not a multiple of 32*K=%d",
           (long long)n, 32 * c->world);
  SG_CUDA(cudaSetDevice(c->device));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int64_t shard = n / c->world;
  const float s = cfg->grad_scale > 0 ? cfg->grad_scale : 1.f / c->world;
  if (c->world > 1)
    SG_NCCL(ncclReduceScatter(grad, grad + c->rank * shard, (size_t)shard, ncclFloat, ncclSum, c->comm_par, st));
  cudaError_t e = sgd_momentum(w + c->rank * shard, grad + c->rank * shard, v_shard, shard, lr_at(*cfg, step),
                               cfg->momentum, cfg->weight_decay, s, st);
  SG_CHECK(e == cudaSuccess, SG_ERR_CUDA, "server sync update: %s", cudaGetErrorString(e));
  if (c->world > 1) SG_NCCL(ncclAllGather(w + c->rank * shard, w, (size_t)shard, ncclFloat, c->comm_par, st));
  return SG_OK;
}

}  // extern "C"

// ------------------------------------- C5 fused server sync over peer memory --
// The worker-group -> server-group exchange of one flat Param (P:419-422,
// P:527) as ONE kernel over NVLink peer memory instead of
// reduce-scatter -> Updater -> all-gather: the step's fused exchange
// (exchange.h / exchange.cu: entry barrier, ascending-rank sum of the shard's
// gradients read straight out of the peers' HBM, SGD-momentum Updater on the
// rank's shard of w_full, the new weights stored into every rank's w_full,
// trailing barrier by the last CTA; a barrier timeout sets an error flag that
// every later exchange kernel checks and skips its work on).  Here the master
// shard IS the rank's slice of w_full and nothing is TF32-rounded (rn_end 0).
struct sg_peer_sync {
  sg_cluster* c = nullptr;
  int64_t n = 0;
  float *grad = nullptr, *w = nullptr, *v = nullptr, *lr = nullptr;
  sg::PeerExchange* px = nullptr;
};

extern "C" {

SG_API sg_status sg_peer_sync_create(sg_cluster* c, int64_t n, sg_peer_sync** out, float** grad_full_dev,
                                     float** w_full_dev, float** v_shard_dev) {
  SG_CHECK(c && out && grad_full_dev && w_full_dev && v_shard_dev, SG_ERR_INVALID_ARG, "sg_peer_sync_create: null argument");
  SG_CHECK(c->world <= 8, SG_ERR_UNSUPPORTED, "sg_peer_sync: at most 8 ranks (got %d)", c->world);
  SG_CHECK(n > 0 && n % (32LL * c->world) == 0, SG_ERR_PARTITION, "partition error: n=%lld not a multiple of 32*K=%d",
           (long long)n, 32 * c->world);
  SG_CUDA(cudaSetDevice(c->device));
  sg_peer_sync* p = new sg_peer_sync();
  p->c = c;
  p->n = n;
  const int64_t shard = n / c->world;
  cudaError_t e = cudaMalloc(&p->grad, n * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&p->w, n * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&p->v, shard * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&p->lr, sizeof(float));
  if (e == cudaSuccess) e = cudaMemset(p->v, 0, shard * sizeof(float));
  // px_create is collective and runs even after a local allocation failure: the
  // missing buffers fail its IPC step, and its status word makes every rank fail
  sg::PxStore st{e == cudaSuccess ? p->grad : nullptr, e == cudaSuccess ? p->w : nullptr,
                 e == cudaSuccess ? p->w + c->rank * shard : nullptr, p->v, n, 0};
  st.agg_out = 0;  // grad_full is read, not modified
  const sg_status ps = sg::px_create(c->comm_par, c->rank, c->world, c->device, {st}, &p->px);
  if (ps != SG_OK || e != cudaSuccess) {
    cudaFree(p->grad); cudaFree(p->w); cudaFree(p->v); cudaFree(p->lr);
    delete p;
    if (e != cudaSuccess) SG_FAIL(SG_ERR_OOM, "sg_peer_sync_create: %s", cudaGetErrorString(e));
    return ps;
  }
  *grad_full_dev = p->grad;
  *w_full_dev = p->w;
  *v_shard_dev = p->v;
  *out = p;
  return SG_OK;
}

SG_API sg_status sg_peer_sync_step(sg_peer_sync* p, const sg_updater_cfg* cfg, int64_t step, void* stream) {
  SG_CHECK(p && cfg, SG_ERR_INVALID_ARG, "sg_peer_sync_step: null argument");
  sg_cluster* c = p->c;
  SG_CUDA(cudaSetDevice(c->device));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const float s = cfg->grad_scale > 0 ? cfg->grad_scale : 1.f / c->world;
  SG_CUDA(sg::fill_scalar(p->lr, lr_at(*cfg, step), st));
  SG_CUDA(sg::px_update(p->px, 0, p->lr, 1.f, cfg->momentum, cfg->weight_decay, s, 0, 0.f, st));
  return SG_OK;
}

SG_API sg_status sg_peer_sync_destroy(sg_peer_sync* p) {
  if (!p) return SG_OK;
  sg_cluster* c = p->c;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  const int err = sg::px_failed(p->px);
  sg::px_destroy(p->px, c->world > 1 ? c->comm_par : nullptr);
  cudaFree(p->grad); cudaFree(p->w); cudaFree(p->v); cudaFree(p->lr);
  delete p;
  SG_CHECK(err == 0, SG_ERR_CUDA, "sg_peer_sync: a peer barrier timed out (a rank did not arrive)");
  return SG_OK;
}

}  // extern "C"

#include "nvls_impl.cuh"
