"""Partitioning cost model and plan recommender (oracle).  Test infrastructure only.

PAPER.md §5.4.1, per layer and per worker, counted in transferred
elements (SPEC S:552-575 design decision: no bandwidth / latency modelling):

* data parallelism (partition_dim 0): the worker exchanges its gradients /
  parameters: cost = p, the size of the replicated Params ("the
  communication overhead per worker is p");
* model parallelism, partition on hidden (Fig. fc-hid): every worker needs
  the whole visible feature matrix: cost = b*d_v (own part b*d_v/K sent,
  b*(K-1)*d_v/K received);
* model parallelism, partition on visible (Fig. fc-vis): cost = b*d_h
  (partial hidden features of all workers are combined -- reading A15: summed);
* no partitioning: one worker computes the layer for all rows:
  cost = b*(K-1)*d_v/K;
* K = 1: no communication, cost 0 for every strategy.

The model-parallel cost of a layer is min(b*d_v, b*d_h), reporting the variant
that achieves it (hidden on a tie).  b is the effective mini-batch summed over
all workers.

recommend_plan: exhaustive search over the strategy of every layer
WITH parameters (conv / inner product: data or model); pooling and LRN layers
are data parallel ("it is cheaper to apply data parallelism");
element-wise layers (ReLU, sigmoid) and the loss inherit their source's
partitioning ("consistent with their source layers"); the minimum total
cost wins, ties broken toward data parallelism (the plan with the
lexicographically smallest list of dims).  Written as a plain enumeration of
all 2^L assignments (L = parameterised layers) -- the search the paper
describes, without pruning.

Pins (tests/test_oracle_cost.py): S:558 / S:685 exact integers (p = 177e6,
d_v = d_h = 4096, K = 8, per-worker batch 128 -> 177e6 vs 4,194,304); K = 1 -> 0;
decision boundary p > b*d_v; monotonicity in b; the AlexNet plan of P:554
(data below the first FC layer, model at and above it); all-zero-parameter nets
-> all data parallel; cost <= every all-data / all-model plan.
"""

import itertools

DATA, MODEL_HIDDEN, MODEL_VISIBLE, NONE = "data", "model_hidden", "model_visible", "none"


def layer_cost(p, d_v, d_h, b, K, strategy):
    """Elements transferred per worker per iteration for one layer."""
    for v in (p, d_v, d_h, b, K):
        if v < 0:
            raise ValueError("validation error: negative cost-model input")
    if K < 1 or b < 1:
        raise ValueError("validation error: K >= 1 and b >= 1 required")
    if K == 1:
        return 0
    if strategy == DATA:
        return p
    if strategy == MODEL_HIDDEN:
        return b * d_v
    if strategy == MODEL_VISIBLE:
        return b * d_h
    if strategy == NONE:
        return b * (K - 1) * d_v // K
    raise ValueError(f"unknown strategy {strategy!r}")


def model_cost(d_v, d_h, b, K):
    """min(b*d_v, b*d_h) and the variant achieving it (hidden on a tie)."""
    h = layer_cost(0, d_v, d_h, b, K, MODEL_HIDDEN)
    v = layer_cost(0, d_v, d_h, b, K, MODEL_VISIBLE)
    return (h, MODEL_HIDDEN) if h <= v else (v, MODEL_VISIBLE)


def profiles(net):
    """Per user layer: (name, kind, p, d_v, d_h) with per-sample feature lengths."""
    from . import net as ON
    info, params = ON.setup(net)
    psize = {}
    for name, shape, _, _, _, layer in params:
        n = 1
        for s in shape:
            n *= s
        psize[layer] = psize.get(layer, 0) + n
    out = []
    for li in info:
        dv = 1
        for s in li["in_shape"]:
            dv *= s
        dh = 1
        for s in li["out_shape"]:
            dh *= s
        out.append((li["name"], li["kind"], psize.get(li["name"], 0), dv, dh))
    return out


def recommend_plan(net, b, K):
    """Returns (dims per user layer, total cost, per-layer [(name, strategy, cost)])."""
    prof = profiles(net)
    if not prof:
        raise ValueError("validation error: empty profile list")
    choose = [i for i, (_, kind, _, _, _) in enumerate(prof) if kind in ("conv", "ip")]
    best = None
    for combo in itertools.product((0, 1), repeat=len(choose)):   # 0 data, 1 model; lexicographic order
        dims, total, rows = [], 0, []
        pick = dict(zip(choose, combo))
        cur = 0
        for i, (name, kind, p, dv, dh) in enumerate(prof):
            if i in pick:
                cur = pick[i]
            elif kind in ("pool_max", "pool_avg", "lrn"):
                cur = 0
            elif kind == "softmax_ce":
                cur = 0                    # a softmax loss needs whole rows
            # relu / sigmoid / euclidean inherit cur
            if i in pick and cur == 1:
                c, strat = model_cost(dv, dh, b, K)
            elif i in pick:
                c, strat = layer_cost(p, dv, dh, b, K, DATA), DATA
            else:
                c, strat = 0, DATA if cur == 0 else MODEL_HIDDEN
            dims.append(cur)
            total += c
            rows.append((name, strat, c))
        if best is None or total < best[1]:
            best = (dims, total, rows)
    return best
