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
* Updater: new fp32 master params from the GPU's own aggregated gradient
  within 1e-6, and the working copy = TF32-RN(master) (weights) / master
  (biases), bit-exact.

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
    return f64(raw.reshape(rows, li["ld"])[:, :cols])


def check_layers(n, net, b, x, lab, p0, grads, newp, work, upd, fused=False, sub=None):
    """Returns [(layer, quantity, error)]; raises AssertionError on a miss."""
    infos = n.layer_info
    p = {k: f64(v) for k, v in p0.items()}
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
        w1, _ = OU.sgd_momentum(p[name], np.zeros_like(p[name]), f64(grads[name]), upd, 0, 1.0)
        e = normwise(newp[name], w1)
        assert e < 1e-6, (name, e)
        want = newp[name] if name.endswith("/b") else rna_tf32(newp[name])
        assert np.array_equal(work[name], want), (name, "working copy")
        rec(name, "update", e)
    return report
