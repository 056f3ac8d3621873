// NeuralNet planner (host only): partition dims, connection layers, shapes,
// Param layouts and the server shard map.  See plan.h.
//
// PAPER.md §5.3: partition_dim 0 slices a layer's feature matrix by
// row (data parallelism), 1 by column (model parallelism); connection layers
// are inserted between differently-partitioned layers.  Here (K > 1, or a forced partitioned plan at K = 1):
//   Concat(rows)  row-split -> replicated    ncclAllGather   (fwd) / ReduceScatter (bwd)
//   Concat(cols)  column-split -> replicated  ncclAllGather   (fwd) / ReduceScatter (bwd)
//   Slice         column-split -> row-split   all-to-all      (fwd) / all-to-all    (bwd)
// The remainder-first partition map is used for rows and columns;
// training requires b % K == 0 for row-split layers and K | d_h for dim-1
// inner-product layers (SG_ERR_PARTITION otherwise; reading A2).
#include <cstring>
#include <map>

#include "abi_common.h"
#include "plan.h"

namespace sg {

namespace {

int64_t round4(int64_t x) { return (x + 3) / 4 * 4; }

const char* kind_name(int k) {
  switch (k) {
    case SG_CONV: return "conv";
    case SG_POOL_MAX: return "pool_max";
    case SG_POOL_AVG: return "pool_avg";
    case SG_RELU: return "relu";
    case SG_SIGMOID: return "sigmoid";
    case SG_LRN: return "lrn";
    case SG_INNER_PRODUCT: return "inner_product";
    case SG_SOFTMAX_CE: return "softmax_ce";
    case SG_EUCLIDEAN: return "euclidean";
    case SG_INPUT: return "input";
    case SG_CONCAT: return "concat";
    case SG_SLICE: return "slice";
  }
  return "?";
}

// Appends a connection layer converting the last layer's state to `target`.
sg_status add_connection(Plan& P, int target) {
  const int K = P.world;
  LayerPlan src = P.layers.back();
  const int si = (int)P.layers.size() - 1;
  LayerPlan c;
  c.src = si;
  c.conn = 1;
  c.image = false;
  c.feat = src.feat;
  if (src.state == ST_ROWS && target == ST_FULL) {
    c.kind = SG_CONCAT;
    c.name = src.name + ".concat_rows";
    c.pdim = 1;
    c.state = ST_FULL;
    c.rows = (int64_t)P.batch;
    c.row_off = 0;
    c.cols = src.feat;
    c.col_off = 0;
    c.ld = src.ld;
    if (src.image) c.ld = src.ld;  // NHWC image flattened: ld = h*w*c
    c.nblocks = 1;
    c.blk_cols = c.cols;
  } else if (src.state == ST_COLS && target == ST_FULL) {
    c.kind = SG_CONCAT;
    c.name = src.name + ".concat_cols";
    c.pdim = 1;
    c.state = ST_FULL;
    c.rows = src.rows;
    c.row_off = 0;
    c.cols = src.feat;
    c.col_off = 0;
    c.ld = src.ld;
    c.nblocks = K;
    c.blk_cols = src.cols;
  } else if (src.state == ST_COLS && target == ST_ROWS) {
    c.kind = SG_SLICE;
    c.name = src.name + ".slice";
    c.pdim = 0;
    c.state = ST_ROWS;
    if (P.batch % K) SG_FAIL(SG_ERR_PARTITION, "partition error: batch %d not divisible by K=%d at %s", P.batch, K,
                             c.name.c_str());
    c.rows = P.batch / K;
    c.row_off = (int64_t)P.rank * c.rows;
    c.cols = src.feat;
    c.col_off = 0;
    c.ld = src.ld;
    c.nblocks = K;
    c.blk_cols = src.cols;
  } else {
    SG_FAIL(SG_ERR_CONFIG, "config error: no connection layer converts %s (state %d) to state %d",
            src.name.c_str(), src.state, target);
  }
  P.layers.push_back(c);
  return SG_OK;
}

}  // namespace

sg_status build_plan(const sg_net_cfg* cfg, int rank, int world, Plan* out, bool force_dist) {
  SG_CHECK(cfg && out, SG_ERR_INVALID_ARG, "plan: null argument");
  SG_CHECK(world >= 1 && rank >= 0 && rank < world, SG_ERR_INVALID_ARG, "plan: rank %d world %d", rank, world);
  SG_CHECK(cfg->nlayers >= 1 && cfg->layers, SG_ERR_CONFIG, "config error: empty net");
  SG_CHECK(cfg->batch >= 1, SG_ERR_CONFIG, "config error: batch %d", cfg->batch);
  SG_CHECK(cfg->in_c >= 1 && cfg->in_h >= 0 && cfg->in_w >= 0 && (cfg->in_h > 0) == (cfg->in_w > 0), SG_ERR_CONFIG,
           "config error: input c=%d h=%d w=%d", cfg->in_c, cfg->in_h, cfg->in_w);
  Plan P;
  P.rank = rank;
  P.world = world;
  P.batch = cfg->batch;
  P.num_classes = cfg->num_classes;
  P.dist = world > 1 || force_dist;
  const int K = world;
  const bool dist = P.dist;

  // resolve partition dims (inherit from the source layer; first defaults to 0)
  std::vector<int> dims(cfg->nlayers);
  int cur = 0;
  std::map<std::string, int> names;
  for (int i = 0; i < cfg->nlayers; ++i) {
    const sg_layer_cfg& l = cfg->layers[i];
    SG_CHECK(l.name && l.name[0] && strlen(l.name) < 48, SG_ERR_CONFIG, "config error: layer %d has no/too long name", i);
    SG_CHECK(!names.count(l.name), SG_ERR_CONFIG, "config error: duplicate layer name %s", l.name);
    names[l.name] = i;
    SG_CHECK(l.partition_dim >= -1 && l.partition_dim <= 1, SG_ERR_CONFIG, "config error: %s partition_dim %d",
             l.name, l.partition_dim);
    if (l.partition_dim >= 0) cur = l.partition_dim;
    dims[i] = dist ? cur : 0;
  }

  // input layer
  {
    LayerPlan in;
    in.name = "input";
    in.kind = SG_INPUT;
    in.src = -1;
    if (cfg->in_h > 0) {
      in.image = true;
      in.h = cfg->in_h;
      in.w = cfg->in_w;
      in.c_real = cfg->in_c;
      in.c = (int)round4(cfg->in_c);
      in.feat = (int64_t)in.h * in.w * in.c_real;
      in.ld = (int64_t)in.h * in.w * in.c;
    } else {
      in.feat = cfg->in_c;
      in.ld = round4(cfg->in_c);
    }
    in.cols = in.feat;
    in.blk_cols = in.feat;
    in.pdim = dims[0];
    if (dims[0] == 0) {
      if (P.batch % K) SG_FAIL(SG_ERR_PARTITION, "partition error: batch %d not divisible by K=%d", P.batch, K);
      in.state = ST_ROWS;
      in.rows = P.batch / K;
      in.row_off = (int64_t)rank * in.rows;
    } else {
      in.state = ST_FULL;
      in.rows = P.batch;
    }
    P.layers.push_back(in);
  }

  for (int i = 0; i < cfg->nlayers; ++i) {
    const sg_layer_cfg& u = cfg->layers[i];
    const int d = dims[i];
    const int kind = u.kind;
    const bool is_loss = kind == SG_SOFTMAX_CE || kind == SG_EUCLIDEAN;
    SG_CHECK(kind >= SG_CONV && kind <= SG_EUCLIDEAN, SG_ERR_CONFIG, "config error: layer %s has unknown kind %d",
             u.name, kind);
    SG_CHECK(!is_loss || i == cfg->nlayers - 1, SG_ERR_CONFIG, "config error: loss layer %s is not the last layer",
             u.name);
    SG_CHECK(is_loss || i != cfg->nlayers - 1, SG_ERR_CONFIG, "config error: the last layer (%s) must be a loss",
             u.name);
    // bring the source into the state this layer needs (partitioned plans only)
    if (dist) {
      int st = P.layers.back().state;
      int need = -1;
      switch (kind) {
        case SG_CONV: case SG_POOL_MAX: case SG_POOL_AVG: case SG_LRN:
          SG_CHECK(d == 0, SG_ERR_CONFIG, "config error: %s (%s) supports partition_dim 0 only", u.name,
                   kind_name(kind));
          need = ST_ROWS;
          break;
        case SG_RELU: case SG_SIGMOID:
          need = d == 0 ? ST_ROWS : ST_COLS;
          break;
        case SG_INNER_PRODUCT:
          need = d == 0 ? ST_ROWS : ST_FULL;
          break;
        case SG_SOFTMAX_CE:
          SG_CHECK(d == 0, SG_ERR_CONFIG,
                   "config error: %s: a softmax loss needs whole rows; partition_dim 1 is invalid (SPEC S:224)", u.name);
          need = ST_ROWS;
          break;
        case SG_EUCLIDEAN:
          need = d == 0 ? ST_ROWS : ST_COLS;
          break;
      }
      if (st != need) {
        if (need == ST_ROWS && st == ST_COLS) {
          SG_TRY(add_connection(P, ST_ROWS));
        } else if (need == ST_FULL && (st == ST_ROWS || st == ST_COLS)) {
          SG_TRY(add_connection(P, ST_FULL));
        } else {
          SG_FAIL(SG_ERR_CONFIG, "config error: %s (%s, partition_dim %d) cannot consume %s's partitioning", u.name,
                  kind_name(kind), d, P.layers.back().name.c_str());
        }
      }
    }
    const int si = (int)P.layers.size() - 1;
    const LayerPlan& s = P.layers[si];
    LayerPlan L;
    L.name = u.name;
    L.kind = kind;
    L.pdim = d;
    L.src = si;
    L.user = i;
    L.num_output = u.num_output;
    L.kernel = u.kernel;
    L.stride = u.stride;
    L.pad = u.pad;
    L.lrn_size = u.lrn_size;
    L.alpha = u.lrn_alpha;
    L.beta = u.lrn_beta;
    L.k = u.lrn_k;
    L.lr_scale = u.lr_scale > 0 ? u.lr_scale : 1.f;
    L.wd_scale = u.wd_scale > 0 ? u.wd_scale : 1.f;
    L.rows = s.rows;
    L.row_off = s.row_off;
    L.state = s.state;
    L.nblocks = 1;
    switch (kind) {
      case SG_CONV: {
        SG_CHECK(s.image, SG_ERR_CONFIG, "config error: conv %s needs an image source", u.name);
        SG_CHECK(u.num_output > 0 && u.kernel > 0 && u.stride > 0 && u.pad >= 0, SG_ERR_CONFIG,
                 "config error: conv %s num_output=%d kernel=%d stride=%d pad=%d", u.name, u.num_output, u.kernel,
                 u.stride, u.pad);
        SG_CHECK(u.num_output % 4 == 0, SG_ERR_CONFIG, "config error: conv %s num_output %d not a multiple of 4",
                 u.name, u.num_output);
        int Ho = (s.h + 2 * u.pad - u.kernel) / u.stride + 1, Wo = (s.w + 2 * u.pad - u.kernel) / u.stride + 1;
        SG_CHECK(Ho > 0 && Wo > 0 && s.h + 2 * u.pad >= u.kernel, SG_ERR_DIMENSION,
                 "dimension error: conv %s kernel %d on %dx%d input (pad %d)", u.name, u.kernel, s.h, s.w, u.pad);
        L.image = true;
        L.h = Ho;
        L.w = Wo;
        L.c = L.c_real = u.num_output;
        L.feat = (int64_t)Ho * Wo * L.c;
        L.ld = L.feat;
        break;
      }
      case SG_POOL_MAX: case SG_POOL_AVG: {
        SG_CHECK(s.image, SG_ERR_CONFIG, "config error: pooling %s needs an image source", u.name);
        SG_CHECK(u.kernel > 0 && u.kernel <= 16 && u.stride > 0 && u.pad >= 0 && u.pad < u.kernel, SG_ERR_CONFIG,
                 "config error: pooling %s kernel=%d stride=%d pad=%d", u.name, u.kernel, u.stride, u.pad);
        SG_CHECK(s.c % 4 == 0 && s.c == s.c_real, SG_ERR_CONFIG, "config error: pooling %s on %d channels", u.name,
                 s.c);
        SG_CHECK(s.h + 2 * u.pad >= u.kernel && s.w + 2 * u.pad >= u.kernel, SG_ERR_DIMENSION,
                 "dimension error: pooling %s window %d on %dx%d", u.name, u.kernel, s.h, s.w);
        auto osz = [&](int h) {
          int ho = (h + 2 * u.pad - u.kernel + u.stride - 1) / u.stride + 1;
          if (u.pad > 0 && (ho - 1) * u.stride >= h + u.pad) --ho;
          return ho;
        };
        L.image = true;
        L.h = osz(s.h);
        L.w = osz(s.w);
        L.c = L.c_real = s.c;
        L.feat = (int64_t)L.h * L.w * L.c;
        L.ld = L.feat;
        break;
      }
      case SG_LRN:
        SG_CHECK(s.image && s.c == s.c_real, SG_ERR_CONFIG, "config error: LRN %s needs an image source", u.name);
        SG_CHECK(u.lrn_size > 0 && u.lrn_size % 2 == 1 && u.lrn_k > 0.f, SG_ERR_CONFIG,
                 "config error: LRN %s size=%d k=%g (odd size, k > 0)", u.name, u.lrn_size, (double)u.lrn_k);
        L.image = true;
        L.h = s.h;
        L.w = s.w;
        L.c = L.c_real = s.c;
        L.feat = s.feat;
        L.ld = s.ld;
        break;
      case SG_RELU: case SG_SIGMOID:
        SG_CHECK(s.kind != SG_INPUT || !s.image || s.c == s.c_real, SG_ERR_CONFIG,
                 "config error: %s directly on a padded image input", u.name);
        L.image = s.image;
        L.h = s.h;
        L.w = s.w;
        L.c = s.c;
        L.c_real = s.c_real;
        L.feat = s.feat;
        L.cols = s.cols;
        L.col_off = s.col_off;
        L.ld = s.ld;
        L.nblocks = s.nblocks;
        L.blk_cols = s.blk_cols;
        break;
      case SG_INNER_PRODUCT: {
        SG_CHECK(u.num_output > 0, SG_ERR_CONFIG, "config error: inner product %s num_output %d", u.name,
                 u.num_output);
        SG_CHECK(!(s.image && s.c != s.c_real), SG_ERR_CONFIG,
                 "config error: inner product %s directly on a channel-padded image input", u.name);
        SG_CHECK(s.kind != SG_SLICE || s.blk_cols % 4 == 0, SG_ERR_CONFIG,
                 "config error: inner product %s after a slice with %lld columns per block", u.name,
                 (long long)s.blk_cols);
        const int64_t dh = u.num_output;
        L.image = false;
        L.feat = dh;
        if (s.nblocks > 1) {  // feature-gathered input: logical padded columns, W rows remapped
          L.kin = (int64_t)s.nblocks * s.ld;
          L.rmap_real = s.blk_cols;
          L.rmap_pad = s.ld;
        } else {
          L.kin = s.feat;
        }
        if (d == 1 && dist) {
          if (dh % K) SG_FAIL(SG_ERR_PARTITION, "partition error: %s d_h=%lld not divisible by K=%d", u.name,
                              (long long)dh, K);
          L.state = ST_COLS;
          L.rows = s.rows;
          L.row_off = 0;
          L.cols = dh / K;
          L.col_off = (int64_t)rank * L.cols;
        } else {
          L.cols = dh;
          L.col_off = 0;
        }
        L.nout = round4(L.cols);
        L.ld = L.nout;
        L.blk_cols = L.cols;
        break;
      }
      case SG_SOFTMAX_CE: {
        SG_CHECK(cfg->num_classes > 0 && s.feat == cfg->num_classes, SG_ERR_DIMENSION,
                 "dimension error: softmax %s on %lld features, num_classes=%d", u.name, (long long)s.feat,
                 cfg->num_classes);
        L.image = false;
        L.feat = 1;
        L.cols = 1;
        L.ld = 1;
        break;
      }
      case SG_EUCLIDEAN: {
        const LayerPlan& in = P.layers[0];
        SG_CHECK(!in.image && s.feat == in.feat, SG_ERR_DIMENSION,
                 "dimension error: Euclidean %s compares %lld features with the %lld-feature input", u.name,
                 (long long)s.feat, (long long)in.feat);
        SG_CHECK(d == 0 || in.state == ST_FULL || !dist, SG_ERR_CONFIG,
                 "config error: a partition_dim 1 Euclidean loss (%s) needs a replicated input", u.name);
        SG_CHECK(d == 1 || !dist || in.state == ST_ROWS, SG_ERR_CONFIG,
                 "config error: a partition_dim 0 Euclidean loss (%s) needs a row-split input", u.name);
        L.image = false;
        L.feat = 1;
        L.cols = 1;
        L.ld = 1;
        break;
      }
    }
    if (L.kind != SG_INNER_PRODUCT && L.kind != SG_RELU && L.kind != SG_SIGMOID) {
      L.cols = L.feat;
      L.col_off = 0;
      L.blk_cols = L.feat;
    }
    if (L.kind == SG_SOFTMAX_CE || L.kind == SG_EUCLIDEAN) {
      L.cols = L.feat = L.ld = 1;
    }
    P.layers.push_back(L);
  }

  // loss instance and default gradient scale s = n_loc / b (reading A2)
  P.loss = (int)P.layers.size() - 1;
  {
    const LayerPlan& Ls = P.layers[P.loss];
    const LayerPlan& src = P.layers[Ls.src];
    if (Ls.kind == SG_SOFTMAX_CE || Ls.pdim == 0) {
      if (P.batch % K) SG_FAIL(SG_ERR_PARTITION, "partition error: batch %d not divisible by K=%d", P.batch, K);
      P.loss_rows = src.rows;
      P.grad_scale = (float)((double)src.rows / (double)P.batch);
    } else {
      P.loss_rows = P.batch;
      P.grad_scale = 1.f;
    }
  }

  // Params, storage buckets and dim-0 gradient buckets
  int nbucket = 0;
  for (int li = 0; li < (int)P.layers.size(); ++li) {
    LayerPlan& L = P.layers[li];
    if (L.kind != SG_CONV && L.kind != SG_INNER_PRODUCT) continue;
    const LayerPlan& s = P.layers[L.src];
    ParamPlan W, b;
    W.name = L.name + "/W";
    b.name = L.name + "/b";
    W.layer = b.layer = li;
    b.is_bias = 1;
    const bool split = (L.kind == SG_INNER_PRODUCT && L.pdim == 1 && dist);
    W.split_dim = b.split_dim = split ? 1 : -1;
    if (L.kind == SG_CONV) {
      W.rows = L.c;
      W.cols = (int64_t)L.kernel * L.kernel * s.c_real;
      W.local_cols = W.cols;
      W.isize = (int64_t)L.c * L.kernel * L.kernel * s.c;
      b.rows = 1;
      b.cols = L.c;
      b.local_cols = L.c;
      b.isize = L.c;
    } else {
      const int64_t dv = (s.nblocks > 1) ? s.feat : s.feat;
      W.rows = dv;
      W.cols = L.feat;
      W.local_col_off = L.col_off;
      W.local_cols = L.cols;
      W.isize = L.kin * L.nout;
      b.rows = 1;
      b.cols = L.feat;
      b.local_col_off = L.col_off;
      b.local_cols = L.cols;
      b.isize = L.nout;
    }
    StorePlan S;
    S.layer = li;
    S.size = W.isize + b.isize;
    S.sharded = !split && dist;
    const int64_t unit = 32LL * K;
    S.padded = (S.size + unit - 1) / unit * unit;
    if (!split) {
      S.bucket = nbucket++;
      W.bucket = b.bucket = S.bucket;
    }
    L.store = (int)P.stores.size();
    W.store = b.store = L.store;
    W.store_off = 0;
    b.store_off = W.isize;
    L.pW = (int)P.params.size();
    P.params.push_back(W);
    L.pb = (int)P.params.size();
    P.params.push_back(b);
    P.stores.push_back(S);
    if (S.bucket >= 0) P.buckets.push_back(L.store);
  }

  // Tensor-core operands (reading A19): the input of every conv / inner
  // product and the gradient w.r.t. its output.  An all-gather (Concat
  // forward) moves its source's values unchanged, so the source's producer
  // rounds; the loss gradient reaches a dim-1 producer through the Slice's
  // all-to-all unchanged, so the loss kernel rounds.  (A Concat's backward is
  // a reduce-scatter sum: the runtime rounds its result in place.)
  const int nl = (int)P.layers.size();
  for (LayerPlan& L : P.layers)
    if (L.kind == SG_CONV || L.kind == SG_INNER_PRODUCT) {
      P.layers[L.src].rn_data = true;
      L.rn_grad = true;
    }
  for (int i = nl - 1; i >= 0; --i) {
    LayerPlan& L = P.layers[i];
    if (L.kind == SG_CONCAT && L.rn_data) P.layers[L.src].rn_data = true;
    if (L.kind == SG_SLICE && P.layers[L.src].rn_grad) L.rn_grad = true;
  }
  *out = std::move(P);
  return SG_OK;
}

}  // namespace sg

using namespace sg;

extern "C" {

// ------------------------------------------------------------ cost model --
// PAPER.md §5.4.1: elements transferred per worker per iteration.
SG_API sg_status sg_layer_cost(int64_t p, int64_t d_v, int64_t d_h, int64_t b, int32_t K, int32_t strategy,
                               int64_t* cost) {
  SG_CHECK(cost, SG_ERR_INVALID_ARG, "sg_layer_cost: null output");
  SG_CHECK(p >= 0 && d_v >= 0 && d_h >= 0 && b >= 1 && K >= 1, SG_ERR_INVALID_ARG,
           "validation error: layer cost p=%lld d_v=%lld d_h=%lld b=%lld K=%d", (long long)p, (long long)d_v,
           (long long)d_h, (long long)b, K);
  SG_CHECK(strategy >= SG_STRAT_DATA && strategy <= SG_STRAT_NONE, SG_ERR_INVALID_ARG, "unknown strategy %d",
           strategy);
  if (K == 1) {
    *cost = 0;
  } else if (strategy == SG_STRAT_DATA) {
    *cost = p;                                   // replicated Params exchanged
  } else if (strategy == SG_STRAT_MODEL_HIDDEN) {
    *cost = b * d_v;                             // whole visible features gathered
  } else if (strategy == SG_STRAT_MODEL_VISIBLE) {
    *cost = b * d_h;                             // partial hidden features combined
  } else {
    *cost = b * (K - 1) * d_v / K;               // no partitioning
  }
  return SG_OK;
}

// Exhaustive search over data / model parallelism of every parameterised layer
// (S:564-571): pooling / LRN layers data parallel, element-wise layers
// and the loss inherit their source's partitioning (a softmax loss: whole rows,
// dim 0); ties toward data parallelism (lexicographically smallest dims).
SG_API sg_status sg_recommend_plan(const sg_net_cfg* cfg, int32_t K, int32_t* dims, int32_t* strategy,
                                   int64_t* cost, int64_t* total) {
  SG_CHECK(cfg && dims && total && K >= 1, SG_ERR_INVALID_ARG, "sg_recommend_plan: bad argument");
  Plan P;
  SG_TRY(build_plan(cfg, 0, 1, &P));
  const int nu = cfg->nlayers;
  std::vector<int64_t> pz(nu, 0), dv(nu, 0), dh(nu, 0);
  std::vector<int> kind(nu, 0), choose;
  for (const LayerPlan& L : P.layers) {
    if (L.user < 0) continue;
    kind[L.user] = L.kind;
    dv[L.user] = P.layers[L.src].feat;
    dh[L.user] = L.feat;
  }
  for (const ParamPlan& q : P.params) pz[P.layers[q.layer].user] += q.rows * q.cols;
  for (int i = 0; i < nu; ++i)
    if (kind[i] == SG_CONV || kind[i] == SG_INNER_PRODUCT) choose.push_back(i);
  SG_CHECK(choose.size() <= 24, SG_ERR_CONFIG, "config error: %zu parameterised layers (exhaustive search <= 24)",
           choose.size());
  const int64_t b = cfg->batch;
  int64_t best = -1;
  std::vector<int> bd(nu), bs(nu), cd(nu), cs(nu);
  std::vector<int64_t> bc(nu), cc(nu);
  const int64_t combos = 1LL << choose.size();
  for (int64_t m = 0; m < combos; ++m) {
    // bit (L-1-j) of m = strategy of the j-th parameterised layer: ascending m is lexicographic order
    int cur = 0;
    int64_t tot = 0;
    size_t j = 0;
    for (int i = 0; i < nu; ++i) {
      int64_t c = 0;
      int st = SG_STRAT_DATA;
      if (j < choose.size() && choose[j] == i) {
        cur = (int)((m >> (choose.size() - 1 - j)) & 1);
        ++j;
        if (cur == 0) {
          SG_TRY(sg_layer_cost(pz[i], dv[i], dh[i], b, K, SG_STRAT_DATA, &c));
        } else {
          int64_t ch, cv;
          SG_TRY(sg_layer_cost(pz[i], dv[i], dh[i], b, K, SG_STRAT_MODEL_HIDDEN, &ch));
          SG_TRY(sg_layer_cost(pz[i], dv[i], dh[i], b, K, SG_STRAT_MODEL_VISIBLE, &cv));
          c = ch <= cv ? ch : cv;
          st = ch <= cv ? SG_STRAT_MODEL_HIDDEN : SG_STRAT_MODEL_VISIBLE;
        }
      } else {
        if (kind[i] == SG_POOL_MAX || kind[i] == SG_POOL_AVG || kind[i] == SG_LRN || kind[i] == SG_SOFTMAX_CE) cur = 0;
        st = cur == 0 ? SG_STRAT_DATA : SG_STRAT_MODEL_HIDDEN;
      }
      cd[i] = cur;
      cs[i] = st;
      cc[i] = c;
      tot += c;
    }
    if (best < 0 || tot < best) {
      best = tot;
      bd = cd;
      bs = cs;
      bc = cc;
    }
  }
  for (int i = 0; i < nu; ++i) {
    dims[i] = bd[i];
    if (strategy) strategy[i] = bs[i];
    if (cost) cost[i] = bc[i];
  }
  *total = best;
  return SG_OK;
}

SG_API sg_status sg_plan_create(const sg_net_cfg* cfg, int32_t rank, int32_t world, sg_plan** out) {
  SG_CHECK(out, SG_ERR_INVALID_ARG, "sg_plan_create: null output");
  sg_plan* p = new sg_plan();
  sg_status st = build_plan(cfg, rank, world, &p->p);
  if (st != SG_OK) {
    delete p;
    return st;
  }
  *out = p;
  return SG_OK;
}

SG_API sg_status sg_plan_destroy(sg_plan* p) {
  delete p;
  return SG_OK;
}

SG_API sg_status sg_plan_num_layers(const sg_plan* p, int32_t* n) {
  SG_CHECK(p && n, SG_ERR_INVALID_ARG, "null argument");
  *n = (int32_t)p->p.layers.size();
  return SG_OK;
}

SG_API sg_status sg_plan_layer_info(const sg_plan* p, int32_t i, sg_layer_info* o) {
  SG_CHECK(p && o, SG_ERR_INVALID_ARG, "null argument");
  SG_CHECK(i >= 0 && i < (int)p->p.layers.size(), SG_ERR_INVALID_ARG, "layer index %d out of range", i);
  const LayerPlan& L = p->p.layers[i];
  memset(o, 0, sizeof(*o));
  strncpy(o->name, L.name.c_str(), sizeof(o->name) - 1);
  o->kind = L.kind;
  o->partition_dim = L.pdim;
  o->is_connection = L.conn;
  o->src = L.src;
  if (L.image) {
    int64_t gs[4] = {p->p.batch, L.h, L.w, L.c};
    int64_t ls[4] = {L.rows, L.h, L.w, L.c};
    for (int k = 0; k < 4; ++k) o->global_shape[k] = gs[k], o->local_shape[k] = ls[k];
  } else {
    o->global_shape[0] = p->p.batch;
    o->global_shape[1] = L.feat;
    o->global_shape[2] = o->global_shape[3] = 1;
    o->local_shape[0] = L.rows;
    o->local_shape[1] = L.cols;
    o->local_shape[2] = o->local_shape[3] = 1;
    o->local_offset[1] = L.col_off;
  }
  o->local_offset[0] = L.row_off;
  o->ld = L.ld;
  o->nblocks = L.nblocks;
  o->tf32_data = L.rn_data ? 1 : 0;
  o->tf32_grad = L.rn_grad ? 1 : 0;
  return SG_OK;
}

SG_API sg_status sg_plan_num_params(const sg_plan* p, int32_t* n) {
  SG_CHECK(p && n, SG_ERR_INVALID_ARG, "null argument");
  *n = (int32_t)p->p.params.size();
  return SG_OK;
}

SG_API sg_status sg_plan_param_info(const sg_plan* p, int32_t i, sg_param_info* o) {
  SG_CHECK(p && o, SG_ERR_INVALID_ARG, "null argument");
  SG_CHECK(i >= 0 && i < (int)p->p.params.size(), SG_ERR_INVALID_ARG, "param index %d out of range", i);
  const ParamPlan& q = p->p.params[i];
  memset(o, 0, sizeof(*o));
  strncpy(o->name, q.name.c_str(), sizeof(o->name) - 1);
  o->layer = q.layer;
  o->split_dim = q.split_dim;
  o->rows = q.rows;
  o->cols = q.cols;
  o->local_col_off = q.local_col_off;
  o->local_cols = q.local_cols;
  o->bucket = q.bucket;
  o->bucket_off = q.store_off;
  o->internal_size = q.isize;
  return SG_OK;
}

SG_API sg_status sg_plan_num_buckets(const sg_plan* p, int32_t* n, int64_t* sizes) {
  SG_CHECK(p && n, SG_ERR_INVALID_ARG, "null argument");
  *n = (int32_t)p->p.buckets.size();
  if (sizes)
    for (size_t b = 0; b < p->p.buckets.size(); ++b) sizes[b] = p->p.stores[p->p.buckets[b]].padded;
  return SG_OK;
}

SG_API sg_status sg_plan_shard_map(const sg_plan* p, sg_shard_range* out, int32_t cap, int32_t* n) {
  SG_CHECK(p && n, SG_ERR_INVALID_ARG, "null argument");
  const Plan& P = p->p;
  int cnt = 0;
  for (size_t b = 0; b < P.buckets.size(); ++b) {
    const StorePlan& S = P.stores[P.buckets[b]];
    const int64_t shard = S.padded / P.world;
    for (int pi = 0; pi < (int)P.params.size(); ++pi) {
      const ParamPlan& q = P.params[pi];
      if (q.store != P.buckets[b]) continue;
      int64_t off = 0;
      while (off < q.isize) {
        const int64_t pos = q.store_off + off;
        const int owner = (int)(pos / shard);
        const int64_t len = std::min(q.isize - off, (owner + 1) * shard - pos);
        if (out && cnt < cap) out[cnt] = sg_shard_range{pi, (int32_t)b, owner, off, pos, len};
        ++cnt;
        off += len;
      }
    }
  }
  *n = cnt;
  SG_CHECK(!out || cnt <= cap, SG_ERR_INVALID_ARG, "shard map needs %d entries, cap %d", cnt, cap);
  return SG_OK;
}

}  // extern "C"
