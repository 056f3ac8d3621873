// Host-side NeuralNet planner: resolves partition_dim per layer,
// inserts connection layers where the partitioning changes (Table
// II), infers shapes, lays out Params (internal padded layouts) and the
// server-group shard map (reading A13).  No device code.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "singa_b200.h"

namespace sg {

enum BlobState { ST_ROWS = 0, ST_COLS = 1, ST_FULL = 2 };

struct LayerPlan {
  std::string name;
  int kind = 0, pdim = 0, conn = 0, src = -1, user = -1;
  // hyper-parameters
  int num_output = 0, kernel = 0, stride = 1, pad = 0, lrn_size = 0;
  float alpha = 0, beta = 0, k = 0, lr_scale = 1, wd_scale = 1;
  // output blob
  bool image = false;
  int h = 1, w = 1, c = 1;         // image per-sample shape (c = stored channels)
  int c_real = 1;                  // channels without padding (input layer pads 3 -> 4)
  int64_t feat = 0;                // per-sample real features (global)
  int state = ST_ROWS;
  int64_t rows = 0, row_off = 0;   // local rows and their global offset
  int64_t cols = 0, col_off = 0;   // local real features and their global offset
  int64_t ld = 0;                  // row stride of one block (elements)
  int nblocks = 1;                 // K for [K][rows][ld] blobs (Concat dim 1, Slice)
  int64_t blk_cols = 0;            // real columns per block (blocked blobs)
  // inner product GEMM geometry (local): y[rows][nout] = x[rows][kin] W[kin][nout]
  int64_t kin = 0, nout = 0;
  int64_t rmap_real = 0, rmap_pad = 0;  // logical input row i -> (i/pad)*real + i%pad (if pad > 0)
  int pW = -1, pb = -1, store = -1;
  // Reading A19: the layer's output blob (rn_data) / the gradient w.r.t. its
  // output (rn_grad) is read as a tensor-core operand, so its producer stores
  // it rounded to TF32 (round to nearest).
  bool rn_data = false, rn_grad = false;
  int64_t blob_floats() const { return (int64_t)nblocks * rows * ld; }
};

struct ParamPlan {
  std::string name;
  int layer = -1, split_dim = -1, is_bias = 0;
  int64_t rows = 0, cols = 0;              // user global layout
  int64_t local_col_off = 0, local_cols = 0;
  int bucket = -1;                         // dim-0 bucket id (shard map) or -1
  int store = -1;                          // storage bucket (every param-owning layer)
  int64_t store_off = 0;                   // element offset inside the storage bucket
  int64_t isize = 0;                       // internal (local) element count
};

struct StorePlan {
  int layer = -1;
  int64_t size = 0;     // sum of internal param sizes
  int64_t padded = 0;   // padded to 32*K when sharded
  bool sharded = false; // dim-0 layer with K > 1: RS -> shard update -> AG
  int bucket = -1;
};

struct Plan {
  int rank = 0, world = 1, batch = 0, num_classes = 0;
  // partitioned data plane: world > 1, or forced at world 1 (sg_cluster_cfg
  // exercise_collectives: connection layers and sharded buckets on one rank)
  bool dist = false;
  std::vector<LayerPlan> layers;  // execution order; layers[0] = input
  std::vector<ParamPlan> params;
  std::vector<StorePlan> stores;
  std::vector<int> buckets;       // bucket id -> store index
  int loss = -1;                  // index of the loss layer
  int64_t loss_rows = 0;          // n_loc of the loss instance on this rank
  float grad_scale = 1.f;         // default s = n_loc / b
};

// Builds the plan; on failure returns the sg_status and sets the error message.
// force_dist: plan as partitioned even at world 1 (test switch, see Plan::dist).
sg_status build_plan(const sg_net_cfg* cfg, int rank, int world, Plan* out, bool force_dist = false);

}  // namespace sg

struct sg_plan {
  sg::Plan p;
};
