"""Whole-net GPU parity through the C ABI (sg_net_* / sg_train_one_batch) vs
the float64 oracle, on seeded synthetic inputs (workloads/generate.py).

* layer-isolated (reading A10): every layer's GPU outputs (y, dx, dW, db) vs
  the oracle layer fed the GPU's own fp32 input blobs and dy; TF32 contractions
  within 2e-3 normwise (A9), fp32 SIMT within 1e-5, max-pool argmax bit-exact;
* whole step: loss and aggregated gradients of a sigmoid MLP (no ReLU /
  max-pool decision flips) within 2e-3;
* free-running loss curves within 1% (A20);
* invariants: lr = 0 keeps params bit-exact; graph replay == eager, bit-exact;
  bad label -> SG_ERR_LABEL.
"""

import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import layers as OL  # noqa: E402
from oracle import net as ON  # noqa: E402
from oracle import updater as OU  # noqa: E402
from tests.gpu_util import FP32_TOL, TF32_TOL, f64, normwise  # noqa: E402
from workloads import configs, generate  # noqa: E402

if torch.cuda.is_available():
    from paper_1603_07846_b200 import _lib as L  # noqa: E402
    from paper_1603_07846_b200 import net as PN  # noqa: E402


def build(net, b, upd=None, params=None, graph=False):
    cl = PN.Cluster(0, 1, 0)
    n = PN.Net(cl, net, b)
    n.set_updater(upd or configs.UPDATERS.get(net["name"], configs.UPDATERS["mlp"]))
    if params is None:
        params = generate.init_params(ON.param_specs(net))
    n.set_params(params)
    if graph:
        n.enable_graph(True)
    return cl, n, params


def shapes_of(params):
    return {k: v.shape for k, v in params.items()}


class Run:
    def __init__(self, net, b, upd=None, graph=False):
        self.net, self.b = net, b
        self.cl, self.n, self.p0 = build(net, b, upd, graph=graph)
        self.loss = torch.zeros(1, device="cuda")

    def step(self, t, x, lab):
        xd = torch.from_numpy(x).cuda()
        ld = torch.from_numpy(lab).cuda() if self.net["num_classes"] else None
        self.n.train_one_batch(t, xd.data_ptr(), ld.data_ptr() if ld is not None else None, self.loss.data_ptr())
        self.n.sync()
        self._keep = (xd, ld)
        return float(self.loss.item())

    def blob(self, i, which=0, dtype=torch.float32):
        nb = self.n.blob_size(i, which)
        t = torch.empty(nb // 4, dtype=dtype, device="cuda")
        L.sg_blob_get(self.n.h, i, which, t.data_ptr(), nb, None)
        torch.cuda.synchronize()
        return t.cpu().numpy()

    def close(self):
        self.n.close()
        self.cl.close()


def local_blob(run, i, which=0):
    """Blob i as a float64 array in the oracle's per-sample layout (padding stripped)."""
    li = run.n.layer_info[i]
    if which == 1:
        li = run.n.layer_info[li["src"]]
    raw = run.blob(i, which)
    rows = li["local_shape"][0]
    if li["kind"] == "input" or (li["local_shape"][2] > 1 or li["local_shape"][3] > 1):
        _, h, w, c = li["local_shape"]
        a = raw.reshape(rows, h, w, c)
        return f64(a)
    cols = li["local_shape"][1]
    return f64(raw.reshape(rows, li["ld"])[:, :cols])


def run_layer_isolated(net, b, steps=1):
    run = Run(net, b)
    run.n.set_fusion(False)   # every layer's own output blob is materialised
    try:
        x, lab = generate.batch(net, b, 0)
        run.step(0, x, lab)
        grads = run.n.get_grads(shapes_of(run.p0))
        newp = run.n.get_params(shapes_of(run.p0))
        infos = run.n.layer_info
        p = {k: f64(v) for k, v in run.p0.items()}
        x_in = f64(x)
        checked = []
        for i, li in enumerate(infos):
            k = li["kind"]
            if k == "input":
                continue
            src = li["src"]
            xin = x_in if infos[src]["kind"] == "input" else local_blob(run, src)
            consumers = [j for j, lj in enumerate(infos) if lj["src"] == i]
            dy = local_blob(run, consumers[0], 1) if consumers and k not in ("softmax_ce", "euclidean") else None
            dx = local_blob(run, i, 1) if infos[src]["kind"] != "input" else None
            lname = li["name"]
            lc = next(l for l in net["layers"] if l["name"] == lname)
            if k == "conv":
                y = local_blob(run, i)
                assert normwise(y, OL.conv_forward(xin, p[lname + "/W"], p[lname + "/b"], lc["stride"], lc["pad"])) < TF32_TOL
                rdx, rdW, rdb = OL.conv_backward(xin, p[lname + "/W"], dy, lc["stride"], lc["pad"])
                assert normwise(grads[lname + "/W"], rdW) < TF32_TOL
                assert normwise(grads[lname + "/b"], rdb) < TF32_TOL   # fused ones-row of the TF32 wgrad GEMM
                if dx is not None:
                    assert normwise(dx, rdx) < TF32_TOL
            elif k == "ip":
                y = local_blob(run, i)
                xf = xin.reshape(xin.shape[0], -1)
                assert normwise(y, OL.ip_forward(xf, p[lname + "/W"], p[lname + "/b"])) < TF32_TOL
                rdx, rdW, rdb = OL.ip_backward(xf, p[lname + "/W"], dy)
                assert normwise(grads[lname + "/W"], rdW) < TF32_TOL
                assert normwise(grads[lname + "/b"], rdb) < TF32_TOL   # fused ones-row of the TF32 wgrad GEMM
                if dx is not None:
                    assert normwise(dx.reshape(dx.shape[0], -1), rdx) < TF32_TOL
            elif k == "pool_max":
                y = local_blob(run, i)
                ry, ridx = OL.maxpool_forward(xin, lc["kernel"], lc["stride"], lc["pad"])
                assert np.array_equal(y, ry.astype(np.float32).astype(np.float64))
                am = run.blob(i, 2, torch.int32).reshape(ridx.shape)
                assert np.array_equal(am, ridx)                        # bit-exact argmax
                assert normwise(dx, OL.maxpool_backward(xin.shape, ridx, dy)) < FP32_TOL
            elif k == "pool_avg":
                y = local_blob(run, i)
                assert normwise(y, OL.avgpool_forward(xin, lc["kernel"], lc["stride"], lc["pad"])) < FP32_TOL
                assert normwise(dx, OL.avgpool_backward(xin.shape, dy, lc["kernel"], lc["stride"], lc["pad"])) < FP32_TOL
            elif k == "lrn":
                y = local_blob(run, i)
                ry, rsc = OL.lrn_forward(xin, lc["size"], lc["alpha"], lc["beta"], lc["k"])
                assert normwise(y, ry) < FP32_TOL
                assert normwise(dx, OL.lrn_backward(xin, y, rsc, dy, lc["size"], lc["alpha"], lc["beta"])) < 2 * FP32_TOL
            elif k in ("relu", "sigmoid"):
                y = local_blob(run, i)
                f, bw = (OL.relu_forward, OL.relu_backward) if k == "relu" else (OL.sigmoid_forward, OL.sigmoid_backward)
                assert normwise(y, f(xin)) < FP32_TOL
                if dx is not None:
                    assert normwise(dx, bw(y, dy)) < FP32_TOL
            elif k == "softmax_ce":
                z = xin.reshape(xin.shape[0], -1)
                rl, rdz = OL.softmax_ce(z, lab, b)
                assert normwise(run.blob(i, 0)[:b], rl) < FP32_TOL
                assert normwise(dx.reshape(b, -1), rdz) < FP32_TOL
                assert np.array_equal(np.argmin(dx.reshape(b, -1), axis=1), lab)
            elif k == "euclidean":
                u = xin.reshape(xin.shape[0], -1)
                rl, rdu = OL.euclidean(u, x_in.reshape(b, -1), b)
                assert normwise(run.blob(i, 0)[:b], rl) < FP32_TOL
                assert normwise(dx.reshape(b, -1), rdu) < FP32_TOL
            checked.append(k)
        # Updater, layer-isolated: new params from the GPU's own aggregated gradients
        upd = configs.UPDATERS[net["name"]]
        for name in run.p0:
            w1, _ = OU.sgd_momentum(p[name], np.zeros_like(p[name]), f64(grads[name]), upd, 0, 1.0)
            assert normwise(newp[name], w1) < 1e-6, name
        return checked
    finally:
        run.close()


def test_layer_isolated_cifar():
    net = configs.get("cifar10")
    checked = run_layer_isolated(net, 16)
    assert set(checked) == {"conv", "pool_max", "relu", "lrn", "pool_avg", "ip", "softmax_ce"}


def test_layer_isolated_mlp():
    assert set(run_layer_isolated(configs.get("mlp"), 64)) == {"ip", "sigmoid", "softmax_ce"}


def test_layer_isolated_ae():
    assert set(run_layer_isolated(configs.get("ae"), 32)) == {"ip", "sigmoid", "euclidean"}


def test_layer_isolated_tiny_conv_ragged():
    net = configs.get("tiny_conv")
    run_layer_isolated(net, 6)


def test_alexnet_layer_isolated_small_batch():
    net = configs.alexnet(hybrid=False)
    run_layer_isolated(net, 2)


def test_mlp_whole_step_and_loss_curve():
    """Sigmoid MLP: no decision flips, so chained gradients meet 2e-3; 100-step
    free-running loss within 1% (A20)."""
    net = configs.get("mlp")
    b = 64
    upd = configs.UPDATERS["mlp"]
    run = Run(net, b)
    try:
        p = {k: f64(v) for k, v in run.p0.items()}
        v = {k: np.zeros_like(a) for k, a in p.items()}
        for t in range(100):
            x, lab = generate.batch(net, b, t)
            gl = run.step(t, x, lab)
            out = ON.train_one_batch(net, p, v, x, lab, t, 1, upd)
            if t == 0:
                g = run.n.get_grads(shapes_of(run.p0))
                for k in g:
                    assert normwise(g[k], out["grads"][k]) < TF32_TOL, k
            assert abs(gl - out["loss"]) <= 0.01 * out["loss"], (t, gl, out["loss"])
            p, v = out["params"], out["vel"]
        gp = run.n.get_params(shapes_of(run.p0))
        for k in gp:
            assert normwise(gp[k], p[k]) < 1e-2, k
    finally:
        run.close()


@pytest.mark.parametrize("name,b,steps", [("cifar10", 128, 20), ("ae", 64, 20)])
def test_loss_curve_within_1pct(name, b, steps):
    net = configs.get(name)
    upd = configs.UPDATERS[name]
    run = Run(net, b)
    try:
        p = {k: f64(v) for k, v in run.p0.items()}
        v = {k: np.zeros_like(a) for k, a in p.items()}
        for t in range(steps):
            x, lab = generate.batch(net, b, t)
            gl = run.step(t, x, lab)
            out = ON.train_one_batch(net, p, v, x, lab, t, 1, upd)
            assert abs(gl - out["loss"]) <= 0.01 * out["loss"], (t, gl, out["loss"])
            p, v = out["params"], out["vel"]
    finally:
        run.close()


def test_graph_replay_bit_exact_and_host_entry():
    net = configs.get("cifar10")
    b = 32
    runs = [Run(net, b), Run(net, b, graph=True)]
    try:
        losses = [[], []]
        for t in range(4):
            x, lab = generate.batch(net, b, t)
            for r, ls in zip(runs, losses):
                ls.append(r.step(t, x, lab))
        assert losses[0] == losses[1]
        pe = runs[0].n.get_params(shapes_of(runs[0].p0))
        pg = runs[1].n.get_params(shapes_of(runs[1].p0))
        for k in pe:
            assert np.array_equal(pe[k], pg[k]), k
        assert runs[1].n.launches() > 10
        # host-buffer entry point gives the same loss as the device entry point
        x, lab = generate.batch(net, b, 4)
        lh = runs[1].n.train_one_batch_host(4, x, lab)
        ld = runs[0].step(4, x, lab)
        assert lh == ld
    finally:
        for r in runs:
            r.close()


def test_zero_lr_keeps_params_and_label_error():
    net = configs.get("cifar10")
    b = 16
    upd = dict(configs.UPDATERS["cifar10"], base_lr=0.0)
    run = Run(net, b, upd=upd)
    try:
        for t in range(3):
            x, lab = generate.batch(net, b, t)
            run.step(t, x, lab)
        got = run.n.get_params(shapes_of(run.p0))
        for k in got:
            assert np.array_equal(got[k], run.p0[k]), k
        x, lab = generate.batch(net, b, 9)
        lab[3] = 10
        xd, ld = torch.from_numpy(x).cuda(), torch.from_numpy(lab).cuda()
        run.n.train_one_batch(9, xd.data_ptr(), ld.data_ptr(), run.loss.data_ptr())
        with pytest.raises(L.SingaError) as e:
            run.n.sync()
        assert e.value.name == "SG_ERR_LABEL"
    finally:
        run.close()


def test_alg1_layer_by_layer_api_matches_train_one_batch():
    net = configs.get("mlp")
    b = 64
    a, c = Run(net, b), Run(net, b)
    try:
        x, lab = generate.batch(net, b, 0)
        la = a.step(0, x, lab)
        xd, ld = torch.from_numpy(x).cuda(), torch.from_numpy(lab).cuda()
        h, u = c.n.h, c.n.upd
        nl = len(c.n.layer_info)
        with pytest.raises(L.SingaError) as e:       # ComputeGradient before ComputeFeature
            L.sg_layer_compute_gradient(h, nl - 2, None)
        assert e.value.name == "SG_ERR_SEQUENCE"
        L.sg_net_set_input(h, xd.data_ptr(), ld.data_ptr(), None)
        for i in range(nl):
            L.sg_net_collect(h, i, None)
            L.sg_layer_compute_feature(h, i, None)
        with pytest.raises(L.SingaError) as e:       # Update before ComputeGradient
            L.sg_net_update(h, u, 1, 0, None)
        assert e.value.name == "SG_ERR_PROTOCOL"
        for i in reversed(range(nl)):
            L.sg_layer_compute_gradient(h, i, None)
            L.sg_net_update(h, u, i, 0, None)
        L.sg_net_loss(h, c.loss.data_ptr(), None)
        c.n.sync()
        assert float(c.loss.item()) == la
        pa, pc = a.n.get_params(shapes_of(a.p0)), c.n.get_params(shapes_of(c.p0))
        for k in pa:
            assert np.array_equal(pa[k], pc[k])
    finally:
        a.close()
        c.close()


def test_relu_fusion_bit_exact():
    net = configs.alexnet(hybrid=False)
    b = 2
    runs = [Run(net, b), Run(net, b)]
    runs[1].n.set_fusion(False)
    try:
        for t in range(2):
            x, lab = generate.batch(net, b, t)
            assert runs[0].step(t, x, lab) == runs[1].step(t, x, lab)
        pa, pb = runs[0].n.get_params(shapes_of(runs[0].p0)), runs[1].n.get_params(shapes_of(runs[1].p0))
        for k in pa:
            assert np.array_equal(pa[k], pb[k]), k
    finally:
        for r in runs:
            r.close()
