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
from tests import layer_check as LC  # noqa: E402
from tests.gpu_util import TF32_TOL, f64, normwise  # noqa: E402
from workloads import configs, generate  # noqa: E402

if torch.cuda.is_available():
    from paper_1603_07846_b200 import _lib as L  # noqa: E402
    from paper_1603_07846_b200 import net as PN  # noqa: E402


def build(net, b, upd=None, params=None, graph=False, cluster=None):
    cl = cluster or PN.Cluster(0, 1, 0)
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
    def __init__(self, net, b, upd=None, graph=False, cluster=None):
        self.net, self.b = net, b
        self.cl, self.n, self.p0 = build(net, b, upd, graph=graph, cluster=cluster)
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


def run_layer_isolated(net, b, cluster=None, fused=False, graph=False, sub=None, upd=None):
    """One step, then every layer layer-isolated against the oracle
    (tests/layer_check.py).  Returns the set of layer kinds checked."""
    upd = upd or configs.UPDATERS.get(net["name"]) or configs.UPDATERS[net["name"].split("_")[0]]
    run = Run(net, b, upd=upd, cluster=cluster, graph=graph)
    run.n.set_fusion(fused)
    try:
        x, lab = generate.batch(net, b, 0)
        sh = shapes_of(run.p0)
        work0 = run.n.get_working(sh)
        run.step(0, x, lab)
        LC.check_layers(run.n, net, b, x, lab, run.p0, work0, run.n.get_grads(sh), run.n.get_params(sh),
                        run.n.get_working(sh), upd, fused=fused, sub=sub, hist=run.n.get_history(sh))
        return {li["kind"] for li in run.n.layer_info if li["kind"] != "input"}
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


@pytest.mark.parametrize("name,b", [("cifar10", 16), ("tiny_conv", 6), ("mlp", 64)])
def test_layer_isolated_fused_graph(name, b):
    """The bench configuration (layer fusion + CUDA-graph replay) layer-isolated."""
    run_layer_isolated(configs.get(name), b, fused=True, graph=True)


def test_alexnet_layer_isolated_small_batch():
    net = configs.alexnet(hybrid=False)
    run_layer_isolated(net, 2)


# Rows a7 / a11 / a16 / a18 / a19 of SURVEY §8(a) on ONE GPU: the cluster's
# exercise_collectives switch plans the net as partitioned at world size 1 (a
# one-rank NCCL communicator), so the connection layers' all-gather /
# reduce-scatter / all-to-all, the worker->server reduce-scatter,
# the Updater on the server shard and the parameter all-gather (P:419-422,
# P:527) and the loss all-reduce all run, layer-isolated against the
# oracle; K = 2 / 4 are tests/test_gpu_dist.py.
def hybrid_alexnet():
    return configs.alexnet(hybrid=True)


@pytest.mark.parametrize("name,b,expect", [
    ("cifar10", 16, set()),                  # dim-0 only: sharded buckets, loss all-reduce
    ("alexnet_hybrid", 2, {"concat", "slice"}),  # pool5 -> concat(rows) -> fc6 (dim 1) -> ... -> slice -> loss
    ("ae", 32, {"concat"}),                  # all dim 1: concat(cols) between every FC, dim-1 Euclidean
    ("mlp", 64, set()),
])
def test_layer_isolated_exercised_collectives(name, b, expect):
    net = hybrid_alexnet() if name == "alexnet_hybrid" else configs.get(name)
    cl = PN.Cluster(0, 1, 0, exercise_collectives=True)
    checked = run_layer_isolated(net, b, cluster=cl)
    assert expect <= set(checked), checked


@pytest.mark.parametrize("name,b", [("cifar10", 32), ("alexnet_hybrid", 2), ("ae", 64)])
def test_exercised_collectives_bit_identical_to_plain(name, b):
    """At world size 1 the partitioned data plane is an identity (one-rank
    collectives), so three free-running steps (graph replay) must give the
    SAME bits as the unpartitioned plan: losses, master params, history."""
    net = hybrid_alexnet() if name == "alexnet_hybrid" else configs.get(name)
    upd = configs.UPDATERS[name.split("_")[0]]
    runs = [Run(net, b, upd=upd, graph=True),
            Run(net, b, upd=upd, graph=True, cluster=PN.Cluster(0, 1, 0, exercise_collectives=True)),
            Run(net, b, upd=upd, graph=True, cluster=PN.Cluster(0, 1, 0, exercise_collectives=True))]
    runs[2].n.set_exchange("p2p")     # the fused peer-memory exchange (NEXT-1) with this rank as its only peer
    try:
        assert any(l["is_connection"] for l in runs[1].n.layer_info) or name == "cifar10"
        for t in range(3):
            x, lab = generate.batch(net, b, t)
            la, lb, lc = (r.step(t, x, lab) for r in runs)
            assert la == lb == lc, (t, la, lb, lc)
        sh = shapes_of(runs[0].p0)
        for get in ("get_params", "get_history", "get_working", "get_grads"):
            pa = getattr(runs[0].n, get)(sh)
            for r in runs[1:]:
                pb = getattr(r.n, get)(sh)
                for k in pa:
                    assert np.array_equal(pa[k], pb[k]), (get, k)
    finally:
        for r in runs:
            r.close()


def test_diverged_is_reported():
    """A non-finite loss raises SG_ERR_DIVERGED at sg_net_sync (SPEC S:288 /
    S:341 via SURVEY §8(a) a19): an infinite output bias makes every logit row
    contain inf, so LSE - z_y is nan."""
    net = configs.get("cifar10")
    b = 16
    run = Run(net, b)
    try:
        x, lab = generate.batch(net, b, 0)
        run.step(0, x, lab)
        pi = run.n.param_index()["ip1/b"]
        bias = np.zeros(10, np.float32)
        bias[3] = np.inf
        L.sg_param_set_value(run.n.h, pi, bias.ctypes.data_as(C.c_void_p))
        xd, ld = torch.from_numpy(x).cuda(), torch.from_numpy(lab).cuda()
        run.n.train_one_batch(1, xd.data_ptr(), ld.data_ptr(), run.loss.data_ptr())
        with pytest.raises(L.SingaError) as e:
            run.n.sync()
        assert e.value.name == "SG_ERR_DIVERGED" and e.value.code == -7
        assert not np.isfinite(float(run.loss.item()))
        run.n.sync()                       # the flag is cleared once reported
    finally:
        run.close()


ADAGRAD = {"base_lr": 0.01, "momentum": 0.0, "weight_decay": 5e-4, "lr_policy": "fixed", "type": "adagrad",
           "eps": 1e-8}


@pytest.mark.parametrize("name,b,lr", [("mlp", 64, 0.01), ("cifar10", 32, 0.001)])
def test_adagrad_layer_isolated_and_loss_curve(name, b, lr):
    """AdaGrad Updater (reading A26) in the training step: layer-isolated
    Updater parity (master and TF32 working copy) and a 20-step free-running loss
    within 1% of the oracle (A20).  AdaGrad's first steps move every weight by
    ~lr regardless of its gradient, so the ReLU / max-pool net runs at lr 1e-3
    (the A20 small-step regime; at 1e-2 decision flips drift the trajectory)."""
    net = configs.get(name)
    upd = dict(ADAGRAD, base_lr=lr)
    run_layer_isolated(net, b, upd=upd, fused=True, graph=True)
    run = Run(net, b, upd=upd, graph=True)
    try:
        p = {k: f64(v) for k, v in run.p0.items()}
        h = {k: np.zeros_like(a) for k, a in p.items()}
        for t in range(20):
            x, lab = generate.batch(net, b, t)
            gl = run.step(t, x, lab)
            out = ON.train_one_batch(net, p, h, x, lab, t, 1, upd)
            assert abs(gl - out["loss"]) <= 0.01 * out["loss"], (t, gl, out["loss"])
            p, h = out["params"], out["vel"]
        hist = run.n.get_history(shapes_of(run.p0))
        for k in hist:          # the accumulator is a sum of squares (its per-step value: layer-isolated above)
            assert np.all(hist[k] >= 0), k
    finally:
        run.close()


def test_adagrad_rejects_momentum():
    net = configs.get("mlp")
    cl = PN.Cluster(0, 1, 0)
    n = PN.Net(cl, net, 64)
    try:
        with pytest.raises(L.SingaError) as e:
            n.set_updater(dict(ADAGRAD, momentum=0.9))
        assert e.value.name == "SG_ERR_CONFIG"
    finally:
        n.close()
        cl.close()


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


@pytest.mark.parametrize("name,b,steps", [("cifar10", 128, 100), ("ae", 256, 100), ("alexnet", 64, 20)])
def test_loss_curve_within_1pct(name, b, steps):
    """Free-running loss, GPU vs oracle, within 1% at every step (reading A20;
    SURVEY §8(c).5 item 3: C2 and C4a over 100 steps, C3 at b = 64 over 20),
    each step on a fresh batch of the non-repeating synthetic pool."""
    net = configs.alexnet(hybrid=False) if name == "alexnet" else configs.get(name)
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


def test_pipelined_host_entry_matches_sync():
    """sg_train_one_batch_host_async (two input slots, copies on their own stream)
    gives bit-identical losses and parameters to the synchronous host entry."""
    import torch
    net = configs.get("cifar10")
    b = 32
    runs = [Run(net, b, graph=True), Run(net, b, graph=True)]
    try:
        steps = 6
        xs = [torch.from_numpy(np.ascontiguousarray(generate.batch(net, b, t)[0])).pin_memory() for t in range(steps)]
        ls = [torch.from_numpy(np.ascontiguousarray(generate.batch(net, b, t)[1])).pin_memory() for t in range(steps)]
        loss_h = torch.zeros(steps, dtype=torch.float32).pin_memory()
        sync_losses = []
        for t in range(steps):
            lh = C.c_float()
            L.sg_train_one_batch_host(runs[0].n.h, runs[0].n.upd, t, C.c_void_p(xs[t].data_ptr()),
                                      C.c_void_p(ls[t].data_ptr()), C.byref(lh), None)
            sync_losses.append(lh.value)
        for t in range(steps):
            L.sg_train_one_batch_host_async(runs[1].n.h, runs[1].n.upd, t, C.c_void_p(xs[t].data_ptr()),
                                            C.c_void_p(ls[t].data_ptr()), C.c_void_p(loss_h[t:].data_ptr()), None)
        runs[1].n.sync()
        torch.cuda.synchronize()
        assert [float(v) for v in loss_h] == sync_losses
        pa = runs[0].n.get_params(shapes_of(runs[0].p0))
        pb = runs[1].n.get_params(shapes_of(runs[1].p0))
        for k in pa:
            assert np.array_equal(pa[k], pb[k]), k
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


@pytest.mark.parametrize("name,b", [("alexnet", 2), ("cifar10", 16)])
def test_relu_fusion_bit_exact(name, b):
    """Layer fusion (fused ReLU epilogues, pool [-> ReLU] -> LRN, ReLU backward in
    the consumer, the first conv's weight gradient with the max pool's backward)
    gives the same bits as the unfused layer-by-layer kernels."""
    net = configs.alexnet(hybrid=False) if name == "alexnet" else configs.get(name)
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
