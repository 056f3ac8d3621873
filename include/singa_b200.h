/*
 * singa_b200.h — C ABI of the B200-native SINGA TrainOneBatch path.
 *
 * The calls follow the paper's own abstractions (arXiv 1603.07846, PAPER.md):
 *   NeuralNet / Layer ComputeFeature, ComputeGradient ........ §4.1.1-4.1.2
 *   BPTrainOneBatch (Collect, ComputeFeature; ComputeGradient, Update)  Alg. 1
 *   Updater (server-side parameter update protocol) .......... §4.1.4
 *   Cluster topology: 1 worker group x K workers, 1 server group x K co-located
 *     servers = the AllReduce framework ...................... §5.1-5.2.1
 *   partition_dim 0 (batch, data parallel) / 1 (feature, model parallel) per
 *     layer, connection layers inserted automatically ........ §5.3
 *
 * Conventions (all functions):
 *   - Every function returns sg_status: SG_OK (0) or a negative error code; no
 *     C++ exception crosses the boundary.  sg_last_error() returns a
 *     thread-local message naming the layer and shapes involved.
 *   - "dev" pointers are CUDA device pointers on the calling rank's device;
 *     "host" pointers are host memory (pageable or pinned).
 *   - stream arguments are cudaStream_t passed as void*; NULL = legacy stream.
 *     Device work is stream-ordered and asynchronous: the return code covers
 *     validation and launch errors; device-side conditions (bad label,
 *     non-finite loss) surface at sg_net_sync().
 *   - Calls marked COLLECTIVE must be made by every rank, in the same order.
 *   - Layouts: images NHWC fp32; conv weights [Cout][R][S][Cin]; inner-product
 *     weights [d_v][d_h] (y = xW + b); biases [n]; labels int32.
 *   - Ownership: the caller owns every buffer it passes and the streams; the
 *     library owns everything it allocates (params, blobs, workspaces, the NCCL
 *     communicator) and frees it in the matching *_destroy.
 *   - A handle is used by one host thread at a time.
 */
#ifndef SINGA_B200_H
#define SINGA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SG_ABI_VERSION 2
#define SG_API __attribute__((visibility("default")))

typedef int32_t sg_status;
enum {
  SG_OK = 0,
  SG_ERR_INVALID_ARG = -1, /* null handle/pointer, bad enum value, index out of range */
  SG_ERR_DIMENSION = -2,   /* shape mismatch (e.g. conv Cin not a multiple of 4 at the op level) */
  SG_ERR_PARTITION = -3,   /* parts > extent; b % K != 0 for a dim-0 loss; K does not divide a dim-1 width */
  SG_ERR_CONFIG = -4,      /* unknown kind, bad hyper-parameter, loss not last, dim-1 conv/pool/LRN */
  SG_ERR_SEQUENCE = -5,    /* ComputeGradient before ComputeFeature, no input set */
  SG_ERR_PROTOCOL = -6,    /* Update before ComputeGradient of that layer in this step */
  SG_ERR_DIVERGED = -7,    /* non-finite loss (reported by sg_net_sync) */
  SG_ERR_LABEL = -8,       /* label outside [0, num_classes) (reported by sg_net_sync) */
  SG_ERR_CUDA = -9,
  SG_ERR_NCCL = -10,
  SG_ERR_OOM = -11,
  SG_ERR_UNSUPPORTED = -12 /* >1 worker/server group (asynchronous frameworks), servers != workers */
};

SG_API const char* sg_last_error(void);
SG_API int32_t sg_abi_version(void);

/* ======================================================================
 * Partition map (host only; P:479-484 slice by row / by column).
 * Remainder-first: len_i = floor(E/K) + [i < E mod K], off_i = sum_{j<i} len_j
 * (reading A12).  SG_ERR_PARTITION if parts > extent,
 * SG_ERR_INVALID_ARG if parts < 1, idx outside [0, parts) or a null output.
 * ====================================================================== */
SG_API sg_status sg_partition_range(int64_t extent, int32_t parts, int32_t idx, int64_t* off, int64_t* len);

/* ======================================================================
 * Layer-isolated operations (ComputeFeature / ComputeGradient of one layer on
 * caller buffers).  Device pointers, stream-ordered; scratch space for
 * split-K partials is owned by the library (per device, grown on demand:
 * these calls are NOT CUDA-graph capturable, the net path is).
 * ====================================================================== */

/* Plain TF32 tensor-core GEMM (test entry of the implicit-GEMM engine):
 * C[M][N] = op(A) op(B); A is [M][K] (ta=0) or [K][M] (ta=1); B is [K][N]
 * (tb=0) or [N][K] (tb=1); all row-major fp32, fp32 accumulate. */
SG_API sg_status sg_op_gemm(const float* A_dev, int32_t ta, const float* B_dev, int32_t tb, float* C_dev, int32_t M,
                            int32_t N, int32_t K, void* stream);

/* Convolution (reading A4: cross-correlation, zero padding,
 * Ho = floor((H + 2p - R)/s) + 1).  x [N][H][W][C] with C % 4 == 0
 * (SG_ERR_DIMENSION otherwise), W [Co][R][S][C], b [Co], y [N][Ho][Wo][Co]. */
typedef struct {
  int32_t N, H, W, C, Co, R, S, stride, pad;
} sg_conv_desc;
SG_API sg_status sg_conv_out_shape(const sg_conv_desc* d, int32_t* Ho, int32_t* Wo);
SG_API sg_status sg_op_conv_forward(const sg_conv_desc* d, const float* x_dev, const float* W_dev, const float* b_dev,
                                    float* y_dev, void* stream);
/* dW = sum dy (x) x-window, db = sum dy, dx (skipped when dx_dev == NULL). */
SG_API sg_status sg_op_conv_backward(const sg_conv_desc* d, const float* x_dev, const float* W_dev,
                                     const float* dy_dev, float* dx_dev, float* dW_dev, float* db_dev, void* stream);

/* Inner product ("rotates (multiply W), shifts (plus b)"):
 * y[rows][dh] = x[rows][dv] W[dv][dh] + b ; dW = x^T dy ; db = colsum dy ;
 * dx = dy W^T (skipped when dx_dev == NULL). */
SG_API sg_status sg_op_ip_forward(const float* x_dev, const float* W_dev, const float* b_dev, float* y_dev,
                                  int32_t rows, int32_t dv, int32_t dh, void* stream);
SG_API sg_status sg_op_ip_backward(const float* x_dev, const float* W_dev, const float* dy_dev, float* dx_dev,
                                   float* dW_dev, float* db_dev, int32_t rows, int32_t dv, int32_t dh, void* stream);

/* Pooling (P:553, P:658-659 Caffe pooling; reading A5: ceil-mode output
 * size, avg divisor = window size before clipping, max = first maximum in
 * row-major window scan).  mode 0 = max, 1 = avg.  mask_dev (max only) receives
 * the uint8 offset (dh*kernel + dw) of the argmax inside its window, consumed by
 * the backward; sg_op_pool_argmax expands it to int32 flat h*W + w. */
typedef struct {
  int32_t N, H, W, C, kernel, stride, pad, mode;
} sg_pool_desc;
SG_API sg_status sg_pool_out_shape(const sg_pool_desc* d, int32_t* Ho, int32_t* Wo);
SG_API sg_status sg_op_pool_forward(const sg_pool_desc* d, const float* x_dev, float* y_dev, uint8_t* mask_dev,
                                    void* stream);
SG_API sg_status sg_op_pool_backward(const sg_pool_desc* d, const float* dy_dev, const uint8_t* mask_dev,
                                     float* dx_dev, void* stream);
SG_API sg_status sg_op_pool_argmax(const sg_pool_desc* d, const uint8_t* mask_dev, int32_t* argmax_dev, void* stream);

/* LRN across channels (reading A6): scale = k + alpha/n sum_{window} x^2,
 * y = x scale^-beta.  x, y, scale: [pixels][C]. */
typedef struct {
  int64_t pixels;
  int32_t C, size;
  float alpha, beta, k;
} sg_lrn_desc;
SG_API sg_status sg_op_lrn_forward(const sg_lrn_desc* d, const float* x_dev, float* y_dev, float* scale_dev,
                                   void* stream);
SG_API sg_status sg_op_lrn_backward(const sg_lrn_desc* d, const float* x_dev, const float* y_dev,
                                    const float* scale_dev, const float* dy_dev, float* dx_dev, void* stream);

/* Elementwise neurons: kind SG_RELU or SG_SIGMOID (see sg_kind). ReLU'(0) = 0. */
SG_API sg_status sg_op_neuron_forward(int32_t kind, const float* x_dev, float* y_dev, int64_t n, void* stream);
SG_API sg_status sg_op_neuron_backward(int32_t kind, const float* y_dev, const float* dy_dev, float* dx_dev,
                                       int64_t n, void* stream);

/* Softmax cross-entropy (readings A2, A7):
 * row_loss[i] = LSE(z_i) - z_{i,y_i}; dz = (softmax(z) - onehot(y)) / n_loc.
 * err_dev (int32, may be NULL) is set to nonzero for a label outside [0, C). */
SG_API sg_status sg_op_softmax_ce(const float* z_dev, const int32_t* labels_dev, int32_t rows, int32_t C,
                                  int32_t n_loc, float* row_loss_dev, float* dz_dev, int32_t* err_dev, void* stream);
/* Euclidean loss: row_loss[i] = 0.5 ||u_i - v_i||^2, du = (u - v) / n_loc. */
SG_API sg_status sg_op_euclidean(const float* u_dev, const float* v_dev, int32_t rows, int32_t d, int32_t n_loc,
                                 float* row_loss_dev, float* du_dev, void* stream);

/* Updater (P:282-284 + north star; reading A1):
 * g' = s g + wd w ; v = mu v - lr g' ; w = w + v   (fp32, fixed FMA order). */
SG_API sg_status sg_op_sgd_momentum(float* w_dev, const float* g_dev, float* v_dev, int64_t n, float lr, float mu,
                                    float wd, float s, void* stream);
/* AdaGrad Updater ("such as AdaGrad"; reading A26):
 * g' = s g + wd w ; h = h + g'^2 ; w = w - lr g' / (sqrt(h) + eps)  (fp32, fixed order). */
SG_API sg_status sg_op_adagrad(float* w_dev, const float* g_dev, float* h_dev, int64_t n, float lr, float wd, float s,
                               float eps, void* stream);

/* ======================================================================
 * Cluster topology (AllReduce framework P:419-422).
 * ====================================================================== */
typedef struct sg_cluster sg_cluster;
typedef struct {
  int32_t rank, world_size, device;
  int32_t nworker_groups, workers_per_group; /* must be 1, world_size */
  int32_t nserver_groups, servers_per_group; /* must be 1, world_size (servers co-located) */
  uint8_t nccl_id[128];                      /* from sg_get_unique_id on rank 0, broadcast by the caller */
  /* Test switch (0 = off): at world_size 1, still create a one-rank NCCL
   * communicator and plan every net as partitioned — connection layers
   * (Concat / Slice) inserted, dim-0 gradient buckets sharded (reduce-scatter
   * -> Updater on the shard -> all-gather), dim-1 inner products column-split —
   * so the whole collective data plane runs (and is checked against the oracle)
   * on a single GPU.  Ignored (always on) for world_size > 1. */
  int32_t exercise_collectives;
} sg_cluster_cfg;
/* rank 0 only; the caller broadcasts the 128 bytes to all ranks (process boundary). */
SG_API sg_status sg_get_unique_id(uint8_t out[128]);
/* COLLECTIVE. Sets the CUDA device, creates the NCCL communicator (skipped at world_size 1).
 * Asynchronous topologies (several worker / server groups) -> SG_ERR_UNSUPPORTED. */
SG_API sg_status sg_cluster_create(const sg_cluster_cfg* cfg, sg_cluster** out);
SG_API sg_status sg_cluster_framework(const sg_cluster* c, const char** name); /* "AllReduce" */
SG_API sg_status sg_cluster_destroy(sg_cluster* c);

/* ======================================================================
 * NeuralNet configuration (layers record their source layers; here
 * a single-path chain, the source of layer i is layer i-1 and of layer 0 the
 * input; P:479-493 partition_dim per layer).
 * ====================================================================== */
typedef enum {
  SG_CONV = 1,
  SG_POOL_MAX = 2,
  SG_POOL_AVG = 3,
  SG_RELU = 4,
  SG_SIGMOID = 5,
  SG_LRN = 6,
  SG_INNER_PRODUCT = 7,
  SG_SOFTMAX_CE = 8,
  SG_EUCLIDEAN = 9,
  /* connection layers, inserted by the planner only (Table II) */
  SG_INPUT = 20,
  SG_CONCAT = 21, /* all-gather: rows (dim0 -> dim1) or features (dim1 -> dim1 IP) */
  SG_SLICE = 22   /* all-to-all: feature-split rows -> row-split rows (dim1 -> dim0 loss) */
} sg_kind;

typedef struct {
  const char* name;
  int32_t kind;           /* sg_kind, user kinds only */
  int32_t partition_dim;  /* -1 inherit from source, 0 batch, 1 feature */
  int32_t num_output;     /* conv Cout / inner-product d_h */
  int32_t kernel, stride, pad;
  int32_t lrn_size;
  float lrn_alpha, lrn_beta, lrn_k;
  float lr_scale, wd_scale; /* per-Param multipliers (0 -> 1) */
} sg_layer_cfg;

typedef struct {
  int32_t nlayers;
  const sg_layer_cfg* layers;
  int32_t batch;               /* global mini-batch b, "summed over all workers" */
  int32_t in_c, in_h, in_w;    /* image input; in_h = in_w = 0 for a vector of in_c features */
  int32_t num_classes;         /* softmax classes (0 for a Euclidean net) */
} sg_net_cfg;

/* ---- Host-only planning (no device needed): partitioning, connection-layer
 * insertion, shape inference, Param table, server shard map.  Every map is
 * compared bit-exactly with the oracle's. ---- */
typedef struct sg_plan sg_plan;
SG_API sg_status sg_plan_create(const sg_net_cfg* cfg, int32_t rank, int32_t world, sg_plan** out);
SG_API sg_status sg_plan_destroy(sg_plan* p);

typedef struct {
  char name[64];
  int32_t kind, partition_dim, is_connection, src;
  /* global and local (this rank's) blob shapes: {rows, h, w, c} or {rows, features, 1, 1};
   * local_offset = where the local block starts in the global blob. */
  int64_t global_shape[4], local_shape[4], local_offset[4];
  /* element stride between consecutive feature rows of the local blob (vector
   * blobs are padded to a multiple of 4 floats; = h*w*c for images).  A
   * feature-gathered (Concat dim 1) or all-to-all (Slice) blob is stored as K
   * rank blocks [K][rows][ld]; nblocks = K then (else 1). */
  int64_t ld;
  int32_t nblocks;
  /* Reading A19: 1 when the layer's output blob (tf32_data) / the
   * gradient w.r.t. its output (tf32_grad) is read as a tensor-core operand; its
   * producing kernel then stores it rounded to TF32 (round to nearest, ties
   * away from zero: 13 low mantissa bits zero).  Parameters: the Updater keeps
   * an fp32 master copy and writes a TF32-rounded working copy of every weight
   * matrix (biases stay fp32); sg_param_get_value returns the master. */
  int32_t tf32_data, tf32_grad;
} sg_layer_info;
SG_API sg_status sg_plan_num_layers(const sg_plan* p, int32_t* n);
SG_API sg_status sg_plan_layer_info(const sg_plan* p, int32_t i, sg_layer_info* out); /* execution order */

typedef struct {
  char name[64];           /* "<layer>/W" or "<layer>/b" */
  int32_t layer;           /* index into the layer list (execution order) */
  int32_t split_dim;       /* -1: replicated (dim-0 layer, server-sharded); 1: columns split (dim-1 layer) */
  int64_t rows, cols;      /* global, user layout: conv W rows=Cout cols=R*S*Cin ; IP W rows=d_v cols=d_h ; bias rows=1 */
  int64_t local_col_off, local_cols;
  int32_t bucket;          /* gradient bucket (dim-0 layer) or -1 */
  int64_t bucket_off;      /* element offset of this Param in its bucket (internal elements) */
  int64_t internal_size;   /* elements of the local internal layout (first-conv channels padded
                              to 4, inner-product output columns padded to a multiple of 4) */
} sg_param_info;
SG_API sg_status sg_plan_num_params(const sg_plan* p, int32_t* n);
SG_API sg_status sg_plan_param_info(const sg_plan* p, int32_t i, sg_param_info* out);

/* Server shard map (reading A13): per dim-0 layer a bucket
 * concat(W, b) zero-padded to E' = ceil(E / 32K) * 32K; rank k owns
 * [k E'/K, (k+1) E'/K).  One entry per (param, owner) slice. */
typedef struct {
  int32_t param, bucket, owner_rank;
  int64_t param_off, bucket_off, len;
} sg_shard_range;
SG_API sg_status sg_plan_num_buckets(const sg_plan* p, int32_t* n, int64_t* padded_sizes /* cap n or NULL */);
SG_API sg_status sg_plan_shard_map(const sg_plan* p, sg_shard_range* out, int32_t cap, int32_t* n);

/* ---- Partitioning cost model (§5.4.1) ----
 * Elements transferred per worker per iteration by one layer with p Params,
 * per-sample visible / hidden feature lengths d_v / d_h, effective mini-batch
 * b (summed over workers) and K workers: data parallelism p; model parallelism
 * partitioned on hidden b*d_v, on visible b*d_h; no partitioning
 * b*(K-1)*d_v/K (integer division); 0 for every strategy at K = 1.
 * SG_ERR_INVALID_ARG for negative sizes, b < 1, K < 1 or an unknown strategy. */
enum { SG_STRAT_DATA = 0, SG_STRAT_MODEL_HIDDEN = 1, SG_STRAT_MODEL_VISIBLE = 2, SG_STRAT_NONE = 3 };
SG_API sg_status sg_layer_cost(int64_t p, int64_t d_v, int64_t d_h, int64_t b, int32_t K, int32_t strategy,
                               int64_t* cost);
/* Minimum-total-cost partition_dim per user layer for K workers at the
 * config's global batch: exhaustive search over data / model parallelism of
 * every conv / inner-product layer (model = the cheaper of the hidden /
 * visible variants); pooling and LRN data parallel, element-wise layers inherit
 * their source, a softmax loss is dim 0; ties toward data parallelism.
 * dims[nlayers] receives 0 / 1 (directly usable as sg_layer_cfg.partition_dim),
 * strategy[nlayers] / cost[nlayers] (may be NULL) the per-layer choice and
 * cost, *total the plan's cost.  SG_ERR_CONFIG beyond 24 parameterised layers. */
SG_API sg_status sg_recommend_plan(const sg_net_cfg* cfg, int32_t K, int32_t* dims, int32_t* strategy, int64_t* cost,
                                   int64_t* total);

/* ---- The net on the device ---- */
typedef struct sg_net sg_net;
/* COLLECTIVE (world > 1).  Plans (as sg_plan_create with the cluster's rank /
 * world), allocates every blob / Param / workspace on the cluster's device,
 * initialises Params to 0 (set them with sg_param_set_value). */
SG_API sg_status sg_net_create(sg_cluster* c, const sg_net_cfg* cfg, sg_net** out);
SG_API sg_status sg_net_destroy(sg_net* n);
SG_API sg_status sg_net_plan(const sg_net* n, const sg_plan** out); /* borrowed, valid until destroy */

/* Param values in GLOBAL user layout on the host.  set: every rank passes the
 * full value, the rank keeps its part (synchronous).  get: COLLECTIVE for
 * world > 1, returns the full value.  get_grad: COLLECTIVE, the aggregated
 * (sum over workers, unscaled) gradient of the last step. */
SG_API sg_status sg_param_set_value(sg_net* n, int32_t p, const float* global_host);
SG_API sg_status sg_param_get_value(sg_net* n, int32_t p, float* global_host);
SG_API sg_status sg_param_get_grad(sg_net* n, int32_t p, float* global_host);
SG_API sg_status sg_param_get_history(sg_net* n, int32_t p, float* global_host); /* momentum v, COLLECTIVE */
/* The working copy the GEMMs read (reading A19): the master weight matrix
 * rounded to TF32 (round to nearest, ties away from zero), biases equal to the
 * master.  COLLECTIVE for world > 1 (dim-1 Params are gathered). */
SG_API sg_status sg_param_get_working(sg_net* n, int32_t p, float* global_host);

/* ---- Updater ---- */
typedef struct sg_updater sg_updater;
typedef struct {
  float base_lr, momentum, weight_decay;
  float grad_scale;   /* <= 0: library default s = n_loc / b (1/K for a dim-0 loss, 1 for a dim-1 loss) */
  int32_t lr_policy;  /* 0 fixed, 1 step: lr = base_lr * gamma^floor(step / step_size) */
  float gamma;
  int32_t step_size;
  /* updating protocol: SG_UPD_SGD_MOMENTUM (default, uses momentum) or
   * SG_UPD_ADAGRAD (the history buffer holds the squared-gradient accumulator h,
   * momentum must be 0; eps <= 0 means 1e-8).  SG_ERR_CONFIG for other values. */
  int32_t type;
  float eps;
} sg_updater_cfg;
enum { SG_UPD_SGD_MOMENTUM = 0, SG_UPD_ADAGRAD = 1 };
SG_API sg_status sg_updater_create(sg_net* n, const sg_updater_cfg* cfg, sg_updater** out);
SG_API sg_status sg_updater_destroy(sg_updater* u);

/* ---- BPTrainOneBatch (Alg. 1) ----
 * x_dev: this rank's input rows (rows = local_shape[0] of the input layer:
 * b/K for a dim-0 first layer, b for a dim-1 first layer), NHWC with the
 * configured in_c channels (3 for images) or [rows][in_c].  labels_dev: this
 * rank's labels for the loss layer's rows (b/K for a dim-0 softmax loss);
 * NULL for a Euclidean net.  loss_dev: device float, receives the global mean
 * loss L = (1/b) sum_i l_i.  COLLECTIVE for world > 1. */
SG_API sg_status sg_train_one_batch(sg_net* n, sg_updater* u, int64_t step, const float* x_dev,
                                    const int32_t* labels_dev, float* loss_dev, void* stream);
/* End-to-end variant from HOST buffers: copies the inputs host->device, runs the
 * step, copies the loss back and synchronises the stream (so *loss_host is valid
 * on return).  Use pinned buffers for asynchronous copies. COLLECTIVE. */
SG_API sg_status sg_train_one_batch_host(sg_net* n, sg_updater* u, int64_t step, const float* x_host,
                                         const int32_t* labels_host, float* loss_host, void* stream);
/* Pipelined variant (a training loop's data path): enqueues the host->device
 * copy of this step's inputs on an internal copy stream (two device input
 * slots, so it overlaps the previous step's compute), the step on `stream`, and
 * the device->host copy of the loss into *loss_host, and returns without
 * waiting.  x_host / labels_host (pinned) must stay unchanged, and *loss_host
 * is valid, only after the stream has been synchronised (or sg_net_sync).
 * COLLECTIVE. */
SG_API sg_status sg_train_one_batch_host_async(sg_net* n, sg_updater* u, int64_t step, const float* x_host,
                                               const int32_t* labels_host, float* loss_host, void* stream);

/* Alg. 1 driven layer by layer (same work as sg_train_one_batch):
 *   sg_net_set_input; for i: sg_net_collect(i), sg_layer_compute_feature(i);
 *   for i reversed: sg_layer_compute_gradient(i), sg_net_update(i). */
SG_API sg_status sg_net_set_input(sg_net* n, const float* x_dev, const int32_t* labels_dev, void* stream);
SG_API sg_status sg_net_collect(sg_net* n, int32_t layer, void* stream);
SG_API sg_status sg_layer_compute_feature(sg_net* n, int32_t layer, void* stream);
SG_API sg_status sg_layer_compute_gradient(sg_net* n, int32_t layer, void* stream);
SG_API sg_status sg_net_update(sg_net* n, sg_updater* u, int32_t layer, int64_t step, void* stream);
SG_API sg_status sg_net_loss(sg_net* n, float* loss_dev, void* stream);
/* Drain all streams; returns SG_ERR_LABEL / SG_ERR_DIVERGED raised by device kernels since the last sync. */
SG_API sg_status sg_net_sync(sg_net* n);
/* Capture the whole sg_train_one_batch step in a CUDA graph (NCCL included) and replay it. */
SG_API sg_status sg_net_enable_graph(sg_net* n, int32_t enable);
/* Layer fusion (default on; results bit-identical either way; call between steps):
 *  - a ReLU after a convolution / inner product runs in the GEMM epilogue; the
 *    producer's data blob then holds the post-ReLU values (it aliases the ReLU
 *    layer's blob);
 *  - a ReLU after a pooling layer is written by the pooling kernel, and
 *    pooling [-> ReLU] -> LRN runs as one kernel;
 *  - a ReLU's backward is done by the backward kernel of its single consumer
 *    (LRN or pooling);
 *  - a first-layer 4-channel stride-1 convolution feeding a max pool computes
 *    the pool's backward (its dy) inside its weight-gradient kernel.
 * Every layer's data / grad blob is still written (sg_blob_get sees them). */
SG_API sg_status sg_net_set_fusion(sg_net* n, int32_t enable);
/* Gradient exchange of the sharded (dim-0) Param buckets (COLLECTIVE; call
 * between steps): mode 0 = NCCL reduce-scatter -> Updater on the shard ->
 * all-gather (default); mode 1 = one fused kernel per bucket over NVLink peer
 * memory (CUDA IPC): ascending-rank gradient sum, Updater, the TF32 working
 * copy stored into every rank, bracketed by two flag barriers whose epochs live
 * in device memory (graph replayable).  Needs a partitioned net (world > 1 or
 * exercise_collectives), at most 8 ranks.  A barrier that times out makes every
 * later exchange skip its work and sg_net_sync return SG_ERR_CUDA.  With mode 1
 * on, sg_net_destroy is COLLECTIVE. */
SG_API sg_status sg_net_set_exchange(sg_net* n, int32_t mode);
/* Overlap of communication and computation (§5.4.2, P:557-587;
 * default on): Update(layer) runs on the parameter stream concurrently with the
 * backward of the layers below it.  Off: the compute stream waits for each
 * Update before continuing (the paper's "Sync Copy" baseline). */
SG_API sg_status sg_net_set_overlap(sg_net* n, int32_t enable);
/* Kernel launches issued by the last sg_train_one_batch (graph replay counts the captured kernels). */
SG_API sg_status sg_net_last_launch_count(const sg_net* n, int64_t* launches);
/* Per-operation device timing (CUDA events around every layer operation, also
 * inside captured graphs).  enable != 0 arms it (a graph is re-captured).
 * sg_net_op_times: after the stream has drained, accumulates the last step's
 * event intervals and returns the running sums in ms, 4 slots per layer:
 * [4*i + 0] ComputeFeature, [4*i + 1] ComputeGradient (weight gradient for
 * conv / inner product), [4*i + 2] data gradient (conv / inner product),
 * [4*i + 3] Update (parameter stream).  counts[] (may be NULL) = intervals
 * summed per slot; reset != 0 clears the sums after reading.  enable == 1
 * serialises the weight gradients onto the compute stream so every slot times
 * its kernels alone; enable == 2 keeps the step's stream concurrency.
 * sg_net_op_timeline: the last step's slot intervals as start / end times in
 * ms relative to the start of the first used slot (-1 for unused slots). */
SG_API sg_status sg_net_profile(sg_net* n, int32_t enable);
SG_API sg_status sg_net_op_times(sg_net* n, double* ms, int64_t* counts, int32_t cap, int32_t* nslots,
                                 int32_t reset);
SG_API sg_status sg_net_op_timeline(sg_net* n, double* t_start, double* t_end, int32_t cap, int32_t* nslots);

/* ---- Blob access for layer-isolated parity (this rank's local blob) ----
 * which: 0 data (layer output), 1 grad (gradient w.r.t. the layer's SOURCE
 * data, i.e. the layer's dx), 2 argmax (max pool, int32 flat h*W + w).
 * Layout: as sg_layer_info.local_shape; the internal input blob of an image
 * net has channels padded to a multiple of 4 (pad channel = 0). */
SG_API sg_status sg_blob_size(sg_net* n, int32_t layer, int32_t which, size_t* bytes);
SG_API sg_status sg_blob_get(sg_net* n, int32_t layer, int32_t which, void* dst_dev, size_t bytes, void* stream);
SG_API sg_status sg_blob_set(sg_net* n, int32_t layer, int32_t which, const void* src_dev, size_t bytes,
                             void* stream);

/* ======================================================================
 * Server-group synchronisation of one flat Param (C5 sweep):
 * reduce-scatter(sum) grad_full -> Updater on this rank's shard of w_full
 * (with v_shard) -> all-gather w_full.  n must be a multiple of 32 * world.
 * grad_full is overwritten.  COLLECTIVE.
 * ====================================================================== */
SG_API sg_status sg_server_sync(sg_cluster* c, const sg_updater_cfg* cfg, int64_t step, float* grad_full_dev,
                                float* w_full_dev, float* v_shard_dev, int64_t n, void* stream);

/* ======================================================================
 * Fused server sync over NVLink peer memory (C5; the a16 -> a17 -> a18 chain,
 * P:419-422 "AllReduce" framework, "broadcast back"
 * Updater) in ONE kernel instead of reduce-scatter -> Updater -> all-gather:
 * rank r loads every rank's gradient for its shard [r*n/K, (r+1)*n/K) from
 * the peers' HBM, sums them in ascending rank order, applies the Updater
 * (s = grad_scale, else 1/K) and stores the new weights into every rank's
 * weight buffer (the step's fused exchange, exchange.h: entry barrier in the
 * kernel, trailing barrier by its last CTA).
 *
 * sg_peer_sync_create: COLLECTIVE (all ranks of the cluster).  Allocates the
 *   library-owned device buffers grad_full[n], w_full[n] and v_shard[n/K]
 *   (the caller writes its gradient into grad_full and the initial weights
 *   into w_full — identical on every rank — before the first step; the
 *   pointers stay valid until destroy) and exchanges CUDA IPC handles over the
 *   parameter communicator.  n must be a multiple of 32*K (SG_ERR_PARTITION);
 *   K <= 8 (SG_ERR_UNSUPPORTED); allocation failure -> SG_ERR_OOM; IPC
 *   failure -> SG_ERR_CUDA.  A failure on any rank fails every rank (status
 *   word in the handle exchange, then an all-reduced decision).
 * sg_peer_sync_step: COLLECTIVE, asynchronous on `stream` (the learning-rate
 *   write and ONE exchange kernel).  grad_full is read, not modified.  After
 *   the step every rank's w_full holds the same updated weights.  A peer that
 *   never arrives makes the barrier give up after a bounded spin and sets an
 *   error flag: that step and every later one skip their work (no unsynchronised
 *   reads or stores); sg_peer_sync_destroy reports it.
 * sg_peer_sync_destroy: COLLECTIVE; synchronises, frees the buffers; returns
 *   SG_ERR_CUDA if any barrier timed out.
 * ====================================================================== */
typedef struct sg_peer_sync sg_peer_sync;
SG_API sg_status sg_peer_sync_create(sg_cluster* c, int64_t n, sg_peer_sync** out, float** grad_full_dev,
                                     float** w_full_dev, float** v_shard_dev);
SG_API sg_status sg_peer_sync_step(sg_peer_sync* p, const sg_updater_cfg* cfg, int64_t step, void* stream);
SG_API sg_status sg_peer_sync_destroy(sg_peer_sync* p);

/* The same exchange through NVSwitch multicast (NVLS): grad_full | w_full in one
 * ncclMemAlloc'd, symmetrically registered NCCL window; ONE kernel per step:
 * LSA barrier -> multimem.ld_reduce.add of rank r's shard (the switch sums the
 * K gradients; the summation order is the switch's) -> Updater -> multimem.st
 * of the new weights into every rank -> LSA barrier.  Same arguments and
 * contract as sg_peer_sync_*; SG_ERR_UNSUPPORTED when the communicator has no
 * multicast (no NVSwitch / NVLS).  All three calls are COLLECTIVE. */
typedef struct sg_nvls_sync sg_nvls_sync;
SG_API sg_status sg_nvls_sync_create(sg_cluster* c, int64_t n, sg_nvls_sync** out, float** grad_full_dev,
                                     float** w_full_dev, float** v_shard_dev);
SG_API sg_status sg_nvls_sync_step(sg_nvls_sync* p, const sg_updater_cfg* cfg, int64_t step, void* stream);
SG_API sg_status sg_nvls_sync_destroy(sg_nvls_sync* p);

#ifdef __cplusplus
}
#endif
#endif /* SINGA_B200_H */
