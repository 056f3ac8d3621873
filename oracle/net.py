"""NeuralNet, BPTrainOneBatch and synchronous worker/server aggregation (oracle).

Test infrastructure only.  Follows PAPER.md in the paper's order:

* NeuralNet = single-path layer chain, each layer's source is the previous one
  (§4.1.1); per-layer ``partition_dim`` (§5.3), inherited
  from the source layer when unset ("consistent with source layers").
* BPTrainOneBatch (Alg. 1): forward over layers (Collect then
  ComputeFeature), backward over reverse(layers) (ComputeGradient then Update).
* Synchronous training within one worker group of K workers, gradients summed
  by the server group (AllReduce framework, §5.2.1): every worker
  runs Alg. 1 on its b/K rows (§5.3 partition on dim 0), the server sums the
  K gradients in ascending worker order and applies the Updater with
  s = n_loc/b (reading A2 / S:439).
* Hybrid partitioning: ``train_one_batch_partitioned``
  executes the dim-0 / dim-1 data flow literally (row blocks per worker below
  the first dim-1 layer, column slices of W and of the features above it,
  partial sums for the input gradient) — the transparency check of S:251-252.

Pins: tests/test_oracle_net.py (end-to-end finite differences on tiny nets,
K-invariance K in {1,2,4,8}, hybrid transparency, paper's AlexNet parameter /
computation shares P:531, P:546 and the 177-million count P:550).
The multi-step whole-network trajectory has no printed value in the paper:
beyond composition it is "parity unpinned".
"""

import numpy as np

from . import layers as L
from . import partition as P
from . import updater as U

PARAM_KINDS = ("conv", "ip")


def resolve_dims(net):
    dims = []
    cur = 0
    for l in net["layers"]:
        cur = l.get("partition_dim", cur)
        dims.append(cur)
    return dims


def setup(net):
    """Shape inference (SPEC S:113-118 setup): per-sample output shape of each
    layer and the Param table [(name, shape, fan_in, fan_out, is_bias, layer)]."""
    inp = net["input"]
    shape = (inp["h"], inp["w"], inp["c"]) if "d" not in inp else (inp["d"],)
    info, params = [], []
    for l in net["layers"]:
        k = l["kind"]
        ins = shape
        if k == "conv":
            H, W, C = ins
            R = l["kernel"]
            Ho = L.conv_out_size(H, R, l["stride"], l["pad"])
            Wo = L.conv_out_size(W, R, l["stride"], l["pad"])
            Co = l["num_output"]
            shape = (Ho, Wo, Co)
            params.append((l["name"] + "/W", (Co, R, R, C), C * R * R, Co * R * R, False, l["name"]))
            params.append((l["name"] + "/b", (Co,), 0, 0, True, l["name"]))
        elif k in ("pool_max", "pool_avg"):
            H, W, C = ins
            shape = (L.pool_out_size(H, l["kernel"], l["stride"], l["pad"]),
                     L.pool_out_size(W, l["kernel"], l["stride"], l["pad"]), C)
        elif k == "ip":
            dv = int(np.prod(ins))
            dh = l["num_output"]
            shape = (dh,)
            params.append((l["name"] + "/W", (dv, dh), dv, dh, False, l["name"]))
            params.append((l["name"] + "/b", (dh,), 0, 0, True, l["name"]))
        elif k in ("relu", "sigmoid", "lrn", "softmax_ce", "euclidean"):
            pass
        else:
            raise ValueError(f"config error: unknown layer kind {k!r} ({l['name']})")
        info.append({"name": l["name"], "kind": k, "in_shape": ins, "out_shape": shape})
    return info, params


def param_specs(net):
    """(name, shape, fan_in, fan_out, is_bias) for workloads.generate.init_params."""
    return [p[:5] for p in setup(net)[1]]


# ----------------------------------------------------------------------------
# One worker's forward / backward over its rows (Alg. 1 loops).
# ----------------------------------------------------------------------------
def forward(net, params, x, labels, n_loc):
    """Forward pass; returns (blobs, per-row losses).  blobs[i] = dict(data=..,
    aux=..) for layer i.  ``x`` float64 [rows][H][W][C] or [rows][d]."""
    info, _ = setup(net)
    blobs = []
    cur = x
    src_data = x
    rows = x.shape[0]
    for l, li in zip(net["layers"], info):
        k = l["kind"]
        rec = {}
        if k == "conv":
            out = L.conv_forward(cur, params[l["name"] + "/W"], params[l["name"] + "/b"], l["stride"], l["pad"])
        elif k == "pool_max":
            out, rec["argmax"] = L.maxpool_forward(cur, l["kernel"], l["stride"], l["pad"])
        elif k == "pool_avg":
            out = L.avgpool_forward(cur, l["kernel"], l["stride"], l["pad"])
        elif k == "lrn":
            out, rec["scale"] = L.lrn_forward(cur, l["size"], l["alpha"], l["beta"], l["k"])
        elif k == "relu":
            out = L.relu_forward(cur)
        elif k == "sigmoid":
            out = L.sigmoid_forward(cur)
        elif k == "ip":
            out = L.ip_forward(cur.reshape(rows, -1), params[l["name"] + "/W"], params[l["name"] + "/b"])
        elif k == "softmax_ce":
            loss, dz = L.softmax_ce(cur.reshape(rows, -1), labels, n_loc)
            rec["grad_in"] = dz
            out = loss
        elif k == "euclidean":
            loss, du = L.euclidean(cur.reshape(rows, -1), src_data.reshape(rows, -1), n_loc)
            rec["grad_in"] = du
            out = loss
        rec["data"] = out
        blobs.append(rec)
        cur = out
    return blobs, blobs[-1]["data"]


def backward(net, params, x, blobs):
    """Reverse pass; returns (grads dict, per-layer input gradients).
    dgrads[i] = gradient w.r.t. layer i's SOURCE data (layer i's dx)."""
    rows = x.shape[0]
    grads = {}
    dgrads = [None] * len(net["layers"])
    dy = None
    for i in range(len(net["layers"]) - 1, -1, -1):
        l = net["layers"][i]
        k = l["kind"]
        src = blobs[i - 1]["data"] if i > 0 else x
        y = blobs[i]["data"]
        need_dx = i > 0   # first layer: input has no gradient (reading A24)
        if k in ("softmax_ce", "euclidean"):
            dx = blobs[i]["grad_in"].reshape(src.shape)
        elif k == "conv":
            dx, dW, db = L.conv_backward(src, params[l["name"] + "/W"], dy, l["stride"], l["pad"], need_dx)
            grads[l["name"] + "/W"], grads[l["name"] + "/b"] = dW, db
        elif k == "pool_max":
            dx = L.maxpool_backward(src.shape, blobs[i]["argmax"], dy)
        elif k == "pool_avg":
            dx = L.avgpool_backward(src.shape, dy, l["kernel"], l["stride"], l["pad"])
        elif k == "lrn":
            dx = L.lrn_backward(src, y, blobs[i]["scale"], dy, l["size"], l["alpha"], l["beta"])
        elif k == "relu":
            dx = L.relu_backward(y, dy)
        elif k == "sigmoid":
            dx = L.sigmoid_backward(y, dy)
        elif k == "ip":
            dxf, dW, db = L.ip_backward(src.reshape(rows, -1), params[l["name"] + "/W"], dy, need_dx)
            grads[l["name"] + "/W"], grads[l["name"] + "/b"] = dW, db
            dx = dxf.reshape(src.shape) if need_dx else None
        dgrads[i] = dx
        dy = dx
    return grads, dgrads


def loss_instances(net, b, K):
    """Reading A2: a dim-0 loss runs as K instances over b/K rows (b % K == 0
    required), a dim-1 loss as one instance over all b rows."""
    dims = resolve_dims(net)
    if dims[-1] == 0:
        if b % K:
            raise ValueError(f"partition error: batch {b} not divisible by K={K}")
        return [P.partition_range(b, K, k) for k in range(K)]
    return [(0, b)]


def train_one_batch(net, params, vel, x, labels, step, K, upd, return_blobs=False):
    """One synchronous BP step (Alg. 1 per worker; server sum + Updater).

    params / vel: dict name -> float array (global layouts).  Returns dict with
    new params/vel, loss L = (1/b) sum_i l_i, raw aggregated grads (sum over
    workers, ascending k), per-worker blobs/dgrads when requested.
    """
    x = np.asarray(x, np.float64)
    b = x.shape[0]
    p64 = {k: np.asarray(v, np.float64) for k, v in params.items()}
    inst = loss_instances(net, b, K)
    agg = {k: np.zeros_like(v) for k, v in p64.items()}
    total = 0.0
    per_worker = []
    for off, ln in inst:
        xb = x[off:off + ln]
        blobs, losses = forward(net, p64, xb, labels[off:off + ln], ln)
        g, dg = backward(net, p64, xb, blobs)
        for k in agg:
            agg[k] = agg[k] + g[k]
        total += float(np.sum(losses))
        if return_blobs:
            per_worker.append({"rows": (off, ln), "blobs": blobs, "dgrads": dg, "grads": g})
    n_loc = inst[0][1]
    s = n_loc / b
    _, pinfo = setup(net)
    lscale = {l["name"]: (l.get("lr_scale", 1.0), l.get("wd_scale", 1.0)) for l in net["layers"]}
    new_p, new_v = {}, {}
    for name, *_rest in pinfo:
        ls, ws = lscale[_rest[-1]]
        new_p[name], new_v[name] = U.update(p64[name], vel[name], agg[name], upd, step, s, ls, ws)
    out = {"params": new_p, "vel": new_v, "loss": total / b, "grads": agg, "grad_scale": s}
    if return_blobs:
        out["workers"] = per_worker
    return out


# ----------------------------------------------------------------------------
# Hybrid partitioning executed literally (S:251-252 transparency).
# ----------------------------------------------------------------------------
def train_one_batch_partitioned(net, params, vel, x, labels, step, K, upd):
    """Same step, but with the §5.3 data flow: layers with partition_dim 0 run
    per worker on row blocks; layers with partition_dim 1 run per worker on
    column slices (W[:, cols_k], b[cols_k] for IP; feature columns for
    elementwise layers), with Concat at dim0->dim1 (all rows gathered), Concat
    along features before every dim-1 IP, Slice(0) at dim1->dim0.
    Backward mirrors it: IP input gradients are partial sums over the K column
    slices, added in ascending k.  Only chain nets whose dim-1 layers are IP /
    relu / sigmoid followed by a loss are supported (all configs)."""
    x = np.asarray(x, np.float64)
    b = x.shape[0]
    p = {k: np.asarray(v, np.float64) for k, v in params.items()}
    dims = resolve_dims(net)
    layers = net["layers"]
    nl = len(layers)
    info, pinfo = setup(net)
    inst = loss_instances(net, b, K)
    rowsplit = [P.partition_range(b, K, k) for k in range(K)]
    # state: either ("rows", [blk_k]) or ("cols", [blk_k], widths)
    state = ("rows", [x[o:o + n] for o, n in rowsplit])
    fwd = []
    labels = np.asarray(labels)
    for i, l in enumerate(layers):
        k = l["kind"]
        d = dims[i]
        if k in ("softmax_ce", "euclidean"):
            break
        if d == 0:
            assert state[0] == "rows", "dim-1 -> dim-0 conv side not supported"
            outs, recs = [], []
            for kk, xb in enumerate(state[1]):
                bl, _ = forward_single(l, p, xb)
                outs.append(bl["data"])
                recs.append(bl)
            fwd.append(("rows", recs, state))
            state = ("rows", outs)
        else:
            if k == "ip":
                # Concat: gather full input (rows, then features) on every worker.
                full = P.concat_blobs([blk.reshape(blk.shape[0], -1) for blk in state[1]],
                                      0 if state[0] == "rows" else 1)
                W, bb = p[l["name"] + "/W"], p[l["name"] + "/b"]
                outs = []
                for kk in range(K):
                    o, n = P.partition_range(W.shape[1], K, kk)
                    outs.append(full @ W[:, o:o + n] + bb[None, o:o + n])
                fwd.append(("ip", full, state))
                state = ("cols", outs)
            elif k in ("relu", "sigmoid"):
                assert state[0] == "cols"
                f = L.relu_forward if k == "relu" else L.sigmoid_forward
                outs = [f(blk) for blk in state[1]]
                fwd.append(("elt", outs, state))
                state = ("cols", outs)
            else:
                raise ValueError("unsupported dim-1 layer kind " + k)
    # Loss layer: reassemble rows per loss instance (Slice(0) / A2A).
    feat = P.concat_blobs(state[1], 1) if state[0] == "cols" else P.concat_blobs(
        [blk.reshape(blk.shape[0], -1) for blk in state[1]], 0)
    lk = layers[-1]["kind"]
    total = 0.0
    dfeat = np.zeros_like(feat)
    for o, n in inst:
        if lk == "softmax_ce":
            ls, dz = L.softmax_ce(feat[o:o + n], labels[o:o + n], n)
        else:
            ls, dz = L.euclidean(feat[o:o + n], x[o:o + n].reshape(n, -1), n)
        total += float(np.sum(ls))
        dfeat[o:o + n] = dz
    # back to the last state's partitioning
    if state[0] == "cols":
        widths = [blk.shape[1] for blk in state[1]]
        offs = np.cumsum([0] + widths)
        dstate = [dfeat[:, offs[kk]:offs[kk + 1]] for kk in range(K)]
    else:
        dstate = [dfeat[o:o + n].reshape(state[1][kk].shape) for kk, (o, n) in enumerate(rowsplit)]
    grads = {}
    for i in range(len(fwd) - 1, -1, -1):
        l = layers[i]
        tag, saved, prev_state = fwd[i]
        need_dx = i > 0
        if tag == "elt":
            outs = saved
            f = L.relu_backward if l["kind"] == "relu" else L.sigmoid_backward
            dstate = [f(outs[kk], dstate[kk]) for kk in range(K)]
        elif tag == "ip":
            full = saved
            W = p[l["name"] + "/W"]
            dW = np.zeros_like(W)
            db = np.zeros(W.shape[1])
            dfull = np.zeros_like(full)
            for kk in range(K):
                o, n = P.partition_range(W.shape[1], K, kk)
                dW[:, o:o + n] = full.T @ dstate[kk]
                db[o:o + n] = dstate[kk].sum(axis=0)
                dfull = dfull + dstate[kk] @ W[:, o:o + n].T    # partial sums, ascending k
            grads[l["name"] + "/W"], grads[l["name"] + "/b"] = dW, db
            # Slice back to the previous layer's partitioning.
            if prev_state[0] == "rows":
                dstate = [dfull[o:o + n].reshape(prev_state[1][kk].shape) for kk, (o, n) in enumerate(rowsplit)]
            else:
                widths = [blk.shape[1] for blk in prev_state[1]]
                offs = np.cumsum([0] + widths)
                dstate = [dfull[:, offs[kk]:offs[kk + 1]] for kk in range(K)]
        else:
            recs = saved
            new = []
            gsum = None
            for kk in range(K):
                xb = prev_state[1][kk]
                dx, g = backward_single(l, p, xb, recs[kk], dstate[kk], need_dx)
                new.append(dx)
                if g:
                    gsum = g if gsum is None else {n: gsum[n] + g[n] for n in g}
            if gsum:
                grads.update(gsum)
            dstate = new
    n_loc = inst[0][1]
    s = n_loc / b
    lscale = {l["name"]: (l.get("lr_scale", 1.0), l.get("wd_scale", 1.0)) for l in net["layers"]}
    new_p, new_v = {}, {}
    for name, *_r in pinfo:
        ls, ws = lscale[_r[-1]]
        new_p[name], new_v[name] = U.update(p[name], vel[name], grads[name], upd, step, s, ls, ws)
    return {"params": new_p, "vel": new_v, "loss": total / b, "grads": grads}


def forward_single(l, p, x):
    k = l["kind"]
    rec = {}
    if k == "conv":
        rec["data"] = L.conv_forward(x, p[l["name"] + "/W"], p[l["name"] + "/b"], l["stride"], l["pad"])
    elif k == "pool_max":
        rec["data"], rec["argmax"] = L.maxpool_forward(x, l["kernel"], l["stride"], l["pad"])
    elif k == "pool_avg":
        rec["data"] = L.avgpool_forward(x, l["kernel"], l["stride"], l["pad"])
    elif k == "lrn":
        rec["data"], rec["scale"] = L.lrn_forward(x, l["size"], l["alpha"], l["beta"], l["k"])
    elif k == "relu":
        rec["data"] = L.relu_forward(x)
    elif k == "sigmoid":
        rec["data"] = L.sigmoid_forward(x)
    elif k == "ip":
        rec["data"] = L.ip_forward(x.reshape(x.shape[0], -1), p[l["name"] + "/W"], p[l["name"] + "/b"])
    else:
        raise ValueError(k)
    return rec, None


def backward_single(l, p, x, rec, dy, need_dx):
    k = l["kind"]
    g = {}
    if k == "conv":
        dx, dW, db = L.conv_backward(x, p[l["name"] + "/W"], dy, l["stride"], l["pad"], need_dx)
        g = {l["name"] + "/W": dW, l["name"] + "/b": db}
    elif k == "pool_max":
        dx = L.maxpool_backward(x.shape, rec["argmax"], dy)
    elif k == "pool_avg":
        dx = L.avgpool_backward(x.shape, dy, l["kernel"], l["stride"], l["pad"])
    elif k == "lrn":
        dx = L.lrn_backward(x, rec["data"], rec["scale"], dy, l["size"], l["alpha"], l["beta"])
    elif k == "relu":
        dx = L.relu_backward(rec["data"], dy)
    elif k == "sigmoid":
        dx = L.sigmoid_backward(rec["data"], dy)
    elif k == "ip":
        dxf, dW, db = L.ip_backward(x.reshape(x.shape[0], -1), p[l["name"] + "/W"], dy, need_dx)
        g = {l["name"] + "/W": dW, l["name"] + "/b": db}
        dx = dxf.reshape(x.shape) if need_dx else None
    return dx, g


# ----------------------------------------------------------------------------
# Work accounting (for the P:531 / P:546 / P:550 pins and DESIGN.md rooflines).
# ----------------------------------------------------------------------------
def work(net):
    """Per-image forward MACs and parameter counts per layer."""
    info, pinfo = setup(net)
    out = []
    for l, li in zip(net["layers"], info):
        if l["kind"] == "conv":
            Ho, Wo, Co = li["out_shape"]
            Ci = li["in_shape"][2]
            macs = Ho * Wo * Co * l["kernel"] * l["kernel"] * Ci
            params = Co * l["kernel"] * l["kernel"] * Ci + Co
        elif l["kind"] == "ip":
            dv = int(np.prod(li["in_shape"]))
            macs = dv * l["num_output"]
            params = dv * l["num_output"] + l["num_output"]
        else:
            continue
        out.append({"name": l["name"], "kind": l["kind"], "fwd_macs": macs, "params": params})
    return out
