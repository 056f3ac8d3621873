"""Layer-isolated parity of a whole net on the GPU (reading A10).

After one sg_train_one_batch step, every layer's GPU outputs -- y, the input
gradient dx, dW, db, the argmax -- are compared with the float64 oracle layer
(oracle/layers.py) fed the GPU's OWN input blobs and output gradient
(sg_blob_get), so TF32 contractions are judged one GEMM at a time:

* conv / inner product: normwise < 2e-3 (TF32, readings A9 / A19);
* pooling, LRN, ReLU, sigmoid, losses (fp32 SIMT): normwise < 1e-5;
* max-pool argmax and label indexing: bit-exact (A11);
* blobs the plan marks as tensor-core operands (layer_info tf32_data /
  tf32_grad, reading A19) must be stored TF32-rounded (tests/gpu_util.check_blob);
* connection layers (Concat / Slice) at world size 1 move their
  source unchanged;
* weights: the layer's operand is the working copy the library held before the
  step, checked bit-exactly to be TF32-RN(master) (weights) / the master
  (biases), so the contraction itself is judged on its own operands;
* Updater: new fp32 master params from the GPU's own aggregated gradient
  within 1e-6, and the new working copy = TF32-RN(master) / master, bit-exact.

``fused``: the runtime's layer fusion is on (a ReLU after a conv / inner
product runs in the GEMM epilogue, so the producer's blob holds the post-ReLU
values -- it aliases the ReLU's blob).  ``sub``: row indices used for the
per-sample outputs (forward blobs, dx, argmax) at full batch sizes; weight and
bias gradients always use the whole batch (they sum over it).
"""

import numpy as np
import torch

from oracle import layers as OL
from oracle import updater as OU
from tests.gpu_util import FP32_TOL, TF32_TOL, check_blob, f64, normwise, rna_tf32
from workloads import configs


def blob(n, i, which=0, dtype=torch.float32):
    from paper_1603_07846_b200 import _lib as L
    nb = n.blob_size(i, which)
    t = torch.empty(nb // 4, dtype=dtype, device="cuda")
    L.sg_blob_get(n.h, i, which, t.data_ptr(), nb, None)
    torch.cuda.synchronize()
    return t.cpu().numpy()


def local_blob(n, i, which=0):
    """Blob i (which 0 data / 1 dx) as float64 in the oracle's per-sample layout (padding stripped)."""
    li = n.layer_info[i]
    if which == 1:
        li = n.layer_info[li["src"]]
    raw = blob(n, i, which)
    rows = li["local_shape"][0]
    if li["kind"] == "input" or (li["local_shape"][2] > 1 or li["local_shape"][3] > 1):
        _, h, w, c = li["local_shape"]
        return f64(raw.reshape(rows, h, w, c))
    cols = li["local_shape"][1]
    if li["nblocks"] > 1:
        # rank-blocked [K][rows][ld] (feature all-gather / all-to-all): block j
        # holds columns [j*blk, (j+1)*blk) of the logical rows x cols blob
        K = li["nblocks"]
        blk = cols // K
        a = raw.reshape(K, rows, li["ld"])[:, :, :blk]
        return f64(np.concatenate(list(a), axis=1))
    return f64(raw.reshape(rows, li["ld"])[:, :cols])


def operands(p0, work0):
    """The weights the step's GEMMs read: the working copy the library held
    before the step, which must be TF32-RN(master) for weight matrices and the
    master itself for biases, bit-exactly (reading A19)."""
    for k, v in p0.items():
        want = v if k.endswith("/b") else rna_tf32(v)
        assert np.array_equal(work0[k], want), (k, "working copy before the step")
    return {k: f64(v) for k, v in work0.items()}


def check_layers(n, net, b, x, lab, p0, work0, grads, newp, work, upd, fused=False, sub=None, hist=None):
    """Returns [(layer, quantity, error)]; raises AssertionError on a miss.
    p0 / work0: master and working copy before the step; newp / work after it."""
    infos = n.layer_info
    p = operands(p0, work0)          # the layer's own weight operands (layer-isolated)
    pm = {k: f64(v) for k, v in p0.items()}
    rows = np.arange(b) if sub is None else np.asarray(sub)
    report = []

    def rec(name, what, e):
        report.append((name, what, float(e)))

    consumers = {i: [j for j, lj in enumerate(infos) if lj["src"] == i] for i in range(len(infos))}
    gpu_in = None
    for i, li in enumerate(infos):
        k = li["kind"]
        lname = li["name"]
        if k == "input":
            # the input layer stores the batch rounded to TF32 when a GEMM reads it (reading A19)
            g = local_blob(n, 0)
            if g.ndim == 4:
                g = g[..., :x.shape[-1]]          # strip the zero pad channel (reading A25)
            r32 = np.asarray(x, np.float32).reshape(g.shape)
            assert np.array_equal(g, f64(rna_tf32(r32) if li["tf32_data"] else r32)), "input"
            gpu_in = g
            continue
        src = li["src"]
        xin = gpu_in if infos[src]["kind"] == "input" else local_blob(n, src)
        cons = consumers[i]   # dy = the consumer's dx (with a fused ReLU: the ReLU's, already masked)
        is_loss = k in ("softmax_ce", "euclidean")
        dy = local_blob(n, cons[0], 1) if cons and not is_loss else None
        has_dx = infos[src]["kind"] != "input"
        dx = local_blob(n, i, 1) if has_dx else None
        rn_y, rn_dx = li["tf32_data"], infos[src]["tf32_grad"]
        lc = next((l for l in net["layers"] if l["name"] == lname), None)
        # fused ReLU epilogue: this layer's blob is the ReLU's
        relu_fused = fused and k in ("conv", "ip") and len(cons) == 1 and infos[cons[0]]["kind"] == "relu"
        if relu_fused:
            rn_y = infos[cons[0]]["tf32_data"]
        act = OL.relu_forward if relu_fused else (lambda v: v)
        if k == "conv":
            y = local_blob(n, i)
            ref = act(OL.conv_forward(xin[rows], p[lname + "/W"], p[lname + "/b"], lc["stride"], lc["pad"]))
            rec(lname, "y", check_blob(y[rows], ref, TF32_TOL, rn_y, lname + ".y"))
            _, rdW, rdb = OL.conv_backward(xin, p[lname + "/W"], dy, lc["stride"], lc["pad"], need_dx=False)
            e = normwise(grads[lname + "/W"], rdW)
            assert e < TF32_TOL, (lname, "dW", e)
            rec(lname, "dW", e)
            e = normwise(grads[lname + "/b"], rdb)   # fused ones-row of the TF32 wgrad GEMM
            assert e < TF32_TOL, (lname, "db", e)
            rec(lname, "db", e)
            if has_dx:
                rdx, _, _ = OL.conv_backward(xin[rows], p[lname + "/W"], dy[rows], lc["stride"], lc["pad"])
                rec(lname, "dx", check_blob(dx[rows], rdx, TF32_TOL, rn_dx, lname + ".dx"))
        elif k == "ip":
            y = local_blob(n, i)
            xf = xin.reshape(xin.shape[0], -1)
            ref = act(OL.ip_forward(xf[rows], p[lname + "/W"], p[lname + "/b"]))
            rec(lname, "y", check_blob(y[rows], ref, TF32_TOL, rn_y, lname + ".y"))
            dyf = dy.reshape(dy.shape[0], -1)
            _, rdW, rdb = OL.ip_backward(xf, p[lname + "/W"], dyf, need_dx=False)
            e = normwise(grads[lname + "/W"], rdW)
            assert e < TF32_TOL, (lname, "dW", e)
            rec(lname, "dW", e)
            e = normwise(grads[lname + "/b"], rdb)
            assert e < TF32_TOL, (lname, "db", e)
            rec(lname, "db", e)
            if has_dx:
                rdx, _, _ = OL.ip_backward(xf[rows], p[lname + "/W"], dyf[rows])
                rec(lname, "dx", check_blob(dx.reshape(dx.shape[0], -1)[rows], rdx, TF32_TOL, rn_dx, lname + ".dx"))
        elif k == "pool_max":
            y = local_blob(n, i)
            ry, ridx = OL.maxpool_forward(xin[rows], lc["kernel"], lc["stride"], lc["pad"])
            r32 = ry.astype(np.float32)
            assert np.array_equal(y[rows], f64(rna_tf32(r32) if rn_y else r32)), lname   # max is exact
            am = blob(n, i, 2, torch.int32).reshape((y.shape[0],) + ridx.shape[1:])
            assert np.array_equal(am[rows], ridx), (lname, "argmax")                     # bit-exact (A11)
            rec(lname, "y", 0.0)
            if has_dx:
                rdx = OL.maxpool_backward(xin[rows].shape, ridx, dy[rows])
                rec(lname, "dx", check_blob(dx[rows], rdx, FP32_TOL, rn_dx, lname + ".dx"))
        elif k == "pool_avg":
            y = local_blob(n, i)
            ref = OL.avgpool_forward(xin[rows], lc["kernel"], lc["stride"], lc["pad"])
            rec(lname, "y", check_blob(y[rows], ref, FP32_TOL, rn_y, lname + ".y"))
            if has_dx:
                rdx = OL.avgpool_backward(xin[rows].shape, dy[rows], lc["kernel"], lc["stride"], lc["pad"])
                rec(lname, "dx", check_blob(dx[rows], rdx, FP32_TOL, rn_dx, lname + ".dx"))
        elif k == "lrn":
            y = local_blob(n, i)
            ry, rsc = OL.lrn_forward(xin[rows], lc["size"], lc["alpha"], lc["beta"], lc["k"])
            rec(lname, "y", check_blob(y[rows], ry, FP32_TOL, rn_y, lname + ".y"))
            if has_dx:
                rdx = OL.lrn_backward(xin[rows], y[rows], rsc, dy[rows], lc["size"], lc["alpha"], lc["beta"])
                rec(lname, "dx", check_blob(dx[rows], rdx, 2 * FP32_TOL, rn_dx, lname + ".dx"))
        elif k in ("relu", "sigmoid"):
            y = local_blob(n, i)
            f, bw = (OL.relu_forward, OL.relu_backward) if k == "relu" else (OL.sigmoid_forward, OL.sigmoid_backward)
            rec(lname, "y", check_blob(y[rows], f(xin[rows]), FP32_TOL, rn_y, lname + ".y"))
            if has_dx:
                rec(lname, "dx", check_blob(dx[rows], bw(y[rows], dy[rows]), FP32_TOL, rn_dx, lname + ".dx"))
        elif k in ("concat", "slice"):
            # connection layers at world size 1: the all-gather / all-to-all moves
            # the source blob unchanged; the reduce-scatter / all-to-all returns
            # the gradient unchanged (rounded when it is a GEMM operand of the source)
            y = local_blob(n, i)
            assert np.array_equal(y, xin.reshape(y.shape)), lname
            if has_dx:
                g = dy.reshape(dx.shape)
                if k == "concat" and rn_dx:
                    g = f64(rna_tf32(g))
                assert np.array_equal(dx, g), lname
            rec(lname, "identity", 0.0)
        elif k == "softmax_ce":
            z = xin.reshape(xin.shape[0], -1)
            rl, rdz = OL.softmax_ce(z, lab, b)
            e = normwise(blob(n, i, 0)[:b], rl)
            assert e < FP32_TOL, (lname, "row loss", e)
            rec(lname, "loss", e)
            rec(lname, "dz", check_blob(dx.reshape(b, -1), rdz, FP32_TOL, rn_dx, "dz"))
            assert np.array_equal(np.argmin(dx.reshape(b, -1), axis=1), lab), "label invariant"   # A11
        elif k == "euclidean":
            u = xin.reshape(xin.shape[0], -1)
            rl, rdu = OL.euclidean(u, f64(x).reshape(b, -1), b)
            e = normwise(blob(n, i, 0)[:b], rl)
            assert e < FP32_TOL, (lname, "row loss", e)
            rec(lname, "loss", e)
            rec(lname, "du", check_blob(dx.reshape(b, -1), rdu, FP32_TOL, rn_dx, "du"))
    # Updater (layer-isolated): fp32 master from the GPU's own aggregated
    # gradient; working copy = TF32-RN(master) for weights, master for biases
    for name in p0:
        w1, h1 = OU.update(pm[name], np.zeros_like(pm[name]), f64(grads[name]), upd, 0, 1.0)
        e = normwise(newp[name], w1)
        assert e < 1e-6, (name, e)
        if hist is not None and np.any(h1):   # history after the first step: -lr g' (momentum) / g'^2 (AdaGrad)
            assert normwise(hist[name], h1) < 1e-6, (name, "history")
        want = newp[name] if name.endswith("/b") else rna_tf32(newp[name])
        assert np.array_equal(work[name], want), (name, "working copy")
        rec(name, "update", e)
    return report


# ---------------------------------------------------------------------------
# K ranks (torchrun, one GPU each): the same layer-isolated checks on every
# rank's LOCAL blobs, with the cross-rank quantities assembled over the gloo
# process group:
#   * dim-0 layers (rows b/K): y / dx / argmax from the rank's own rows; the
#     aggregated weight / bias gradient (sum over workers) against the
#     sum over ranks of each rank's float64 oracle contribution;
#   * dim-1 inner products (columns d_h/K): y and dW / db on the
#     rank's columns from the gathered input; dx = the rank's partial sum;
#   * connection layers: Concat = the gathered sources exactly,
#     its backward = the fp64 sum of the ranks' partial gradients (TF32-RN when
#     the source is a GEMM operand); Slice = the all-to-all exactly both ways.
# ---------------------------------------------------------------------------
def check_layers_dist(n, net, b, x, lab, p0, work0, grads, newp, upd, rank, world, fused=False):
    import torch.distributed as dist

    def gather(a):
        out = [None] * world
        dist.all_gather_object(out, a)
        return out

    def allsum(a):
        t = torch.from_numpy(np.ascontiguousarray(a, np.float64))
        dist.all_reduce(t)
        return t.numpy()

    infos = n.layer_info
    p = operands(p0, work0)
    pm = {k: f64(v) for k, v in p0.items()}
    report = []

    def rec(name, what, e):
        report.append((name, what, float(e)))

    consumers = {i: [j for j, lj in enumerate(infos) if lj["src"] == i] for i in range(len(infos))}
    gpu_in = None
    for i, li in enumerate(infos):
        k = li["kind"]
        lname = li["name"]
        r0, nr = li["local_offset"][0], li["local_shape"][0]
        if k == "input":
            g = local_blob(n, 0)
            if g.ndim == 4:
                g = g[..., :x.shape[-1]]
            r32 = np.asarray(x, np.float32)[r0:r0 + nr].reshape(g.shape)
            assert np.array_equal(g, f64(rna_tf32(r32) if li["tf32_data"] else r32)), "input"
            gpu_in = g
            continue
        src = li["src"]
        S = infos[src]
        xin = gpu_in if S["kind"] == "input" else local_blob(n, src)
        cons = consumers[i]
        is_loss = k in ("softmax_ce", "euclidean")
        dy = local_blob(n, cons[0], 1) if cons and not is_loss else None
        has_dx = S["kind"] != "input"
        dx = local_blob(n, i, 1) if has_dx else None
        rn_y, rn_dx = li["tf32_data"], S["tf32_grad"]
        lc = next((l for l in net["layers"] if l["name"] == lname), None)
        relu_fused = fused and k in ("conv", "ip") and len(cons) == 1 and infos[cons[0]]["kind"] == "relu"
        if relu_fused:
            rn_y = infos[cons[0]]["tf32_data"]
        act = OL.relu_forward if relu_fused else (lambda v: v)
        if k == "conv":        # dim 0
            y = local_blob(n, i)
            ref = act(OL.conv_forward(xin, p[lname + "/W"], p[lname + "/b"], lc["stride"], lc["pad"]))
            rec(lname, "y", check_blob(y, ref, TF32_TOL, rn_y, lname + ".y"))
            rdx, rdW, rdb = OL.conv_backward(xin, p[lname + "/W"], dy, lc["stride"], lc["pad"], need_dx=has_dx)
            for q, r in (("W", allsum(rdW)), ("b", allsum(rdb))):
                e = normwise(grads[lname + "/" + q], r)
                assert e < TF32_TOL, (lname, "d" + q, e)
                rec(lname, "d" + q, e)
            if has_dx:
                rec(lname, "dx", check_blob(dx, rdx, TF32_TOL, rn_dx, lname + ".dx"))
        elif k == "ip":
            y = local_blob(n, i)
            xf = xin.reshape(xin.shape[0], -1)
            c0, nc = li["local_offset"][1], li["local_shape"][1]
            W, bb = p[lname + "/W"], p[lname + "/b"]
            split = li["partition_dim"] == 1
            Wl, bl = (W[:, c0:c0 + nc], bb[c0:c0 + nc]) if split else (W, bb)
            rec(lname, "y", check_blob(y, act(OL.ip_forward(xf, Wl, bl)), TF32_TOL, rn_y, lname + ".y"))
            dyf = dy.reshape(dy.shape[0], -1)
            rdx, rdW, rdb = OL.ip_backward(xf, Wl, dyf, need_dx=has_dx)
            gW, gb = grads[lname + "/W"], grads[lname + "/b"]
            if split:    # owner-local gradient of the rank's columns
                gW, gb = gW[:, c0:c0 + nc], gb[c0:c0 + nc]
            else:        # dim-0: aggregated over the workers
                rdW, rdb = allsum(rdW), allsum(rdb)
            for q, g, r in (("dW", gW, rdW), ("db", gb, rdb)):
                e = normwise(g, r)
                assert e < TF32_TOL, (lname, q, e)
                rec(lname, q, e)
            if has_dx:   # dim 1: the rank's partial sum over its columns (reduced by the Concat's backward)
                rn = rn_dx and not split
                rec(lname, "dx", check_blob(dx.reshape(dx.shape[0], -1), rdx, TF32_TOL, rn, lname + ".dx"))
        elif k == "pool_max":
            y = local_blob(n, i)
            ry, ridx = OL.maxpool_forward(xin, lc["kernel"], lc["stride"], lc["pad"])
            r32 = ry.astype(np.float32)
            assert np.array_equal(y, f64(rna_tf32(r32) if rn_y else r32)), lname
            am = blob(n, i, 2, torch.int32).reshape(ridx.shape)
            assert np.array_equal(am, ridx), (lname, "argmax")
            rec(lname, "y", 0.0)
            if has_dx:
                rec(lname, "dx", check_blob(dx, OL.maxpool_backward(xin.shape, ridx, dy), FP32_TOL, rn_dx, lname))
        elif k == "pool_avg":
            y = local_blob(n, i)
            rec(lname, "y", check_blob(y, OL.avgpool_forward(xin, lc["kernel"], lc["stride"], lc["pad"]), FP32_TOL,
                                       rn_y, lname + ".y"))
            if has_dx:
                rdx = OL.avgpool_backward(xin.shape, dy, lc["kernel"], lc["stride"], lc["pad"])
                rec(lname, "dx", check_blob(dx, rdx, FP32_TOL, rn_dx, lname + ".dx"))
        elif k == "lrn":
            y = local_blob(n, i)
            ry, rsc = OL.lrn_forward(xin, lc["size"], lc["alpha"], lc["beta"], lc["k"])
            rec(lname, "y", check_blob(y, ry, FP32_TOL, rn_y, lname + ".y"))
            if has_dx:
                rdx = OL.lrn_backward(xin, y, rsc, dy, lc["size"], lc["alpha"], lc["beta"])
                rec(lname, "dx", check_blob(dx, rdx, 2 * FP32_TOL, rn_dx, lname + ".dx"))
        elif k in ("relu", "sigmoid"):
            y = local_blob(n, i)
            f, bw = (OL.relu_forward, OL.relu_backward) if k == "relu" else (OL.sigmoid_forward, OL.sigmoid_backward)
            rec(lname, "y", check_blob(y, f(xin), FP32_TOL, rn_y, lname + ".y"))
            if has_dx:
                rec(lname, "dx", check_blob(dx, bw(y, dy), FP32_TOL, rn_dx, lname + ".dx"))
        elif k == "concat":
            y = local_blob(n, i)
            srcs = gather(xin.reshape(xin.shape[0], -1))
            full = np.concatenate(srcs, axis=0 if S["partition_dim"] == 0 else 1)   # rows or feature blocks
            assert np.array_equal(y.reshape(full.shape), full), lname
            if has_dx:
                parts = gather(dy.reshape(dy.shape[0], -1))
                tot = np.sum(np.stack(parts), axis=0)
                if S["partition_dim"] == 0:
                    mine = tot[S["local_offset"][0]:S["local_offset"][0] + S["local_shape"][0]]
                else:
                    c0 = S["local_offset"][1]
                    mine = tot[:, c0:c0 + S["local_shape"][1]]
                rec(lname, "dx", check_blob(dx.reshape(mine.shape), mine, FP32_TOL, rn_dx, lname + ".dx"))
        elif k == "slice":
            # forward: my rows of every rank's column block; backward: my columns of every rank's rows
            y = local_blob(n, i)
            srcs = gather(xin)
            full = np.concatenate(srcs, axis=1)
            assert np.array_equal(y, full[r0:r0 + nr]), lname
            if has_dx:
                parts = gather((r0, dy))
                full_dy = np.zeros((b, dy.shape[1]))
                for (o, d) in parts:
                    full_dy[o:o + d.shape[0]] = d
                c0, nc = S["local_offset"][1], S["local_shape"][1]
                assert np.array_equal(dx, full_dy[:, c0:c0 + nc]), lname + ".dx"
            rec(lname, "identity", 0.0)
        elif k == "softmax_ce":
            z = xin.reshape(xin.shape[0], -1)
            rl, rdz = OL.softmax_ce(z, lab[r0:r0 + nr], nr)
            e = normwise(blob(n, i, 0)[:nr], rl)
            assert e < FP32_TOL, (lname, "row loss", e)
            rec(lname, "dz", check_blob(dx.reshape(nr, -1), rdz, FP32_TOL, rn_dx, "dz"))
            assert np.array_equal(np.argmin(dx.reshape(nr, -1), axis=1), lab[r0:r0 + nr]), "label invariant"
        elif k == "euclidean":
            u = xin.reshape(xin.shape[0], -1)
            c0, nc = S["local_offset"][1], S["local_shape"][1]
            v = f64(x).reshape(b, -1)
            v = v[:, c0:c0 + nc] if S["partition_dim"] == 1 else v[r0:r0 + nr]
            rl, rdu = OL.euclidean(u, v, b if S["partition_dim"] == 1 else nr)
            e = normwise(blob(n, i, 0)[:u.shape[0]], rl)
            assert e < FP32_TOL, (lname, "row loss", e)
            rec(lname, "du", check_blob(dx.reshape(u.shape), rdu, FP32_TOL, rn_dx, "du"))
    # Updater: every rank's exported master values = the oracle Updater applied
    # to the exported aggregated gradient with the default scale s = n_loc / b
    loss_dim = infos[-1]["partition_dim"]
    s = 1.0 / world if loss_dim == 0 else 1.0
    for name in p0:
        w1, _ = OU.update(pm[name], np.zeros_like(pm[name]), f64(grads[name]), upd, 0, s)
        e = normwise(newp[name], w1)
        assert e < 1e-6, (name, e)
        rec(name, "update", e)
    return report
