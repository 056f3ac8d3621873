"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (CUDA-graph replay, layer fusion on), layer-isolated (reading A10) for
EVERY layer of the net (tests/layer_check.py):

* CIFAR-10 ConvNet, batch 128 (BASELINE configs[1], the bench workload): all
  rows of every blob; conv1 forward / weight + bias gradient, conv2 / conv3
  forward / data / weight gradients, every pooling (argmax bit-exact), LRN and
  ReLU forward + backward, ip1, the softmax gradient and label invariant, the
  Updater and the TF32 working copy; plus the loss of the full oracle step
  within 1% (A20).
* AlexNet-shaped, batch 256 on one GPU (configs[2]): every layer likewise,
  conv1-conv5 and fc6-fc8 in all three directions.  Weight / bias gradients
  use the whole batch (they sum over it); the per-sample outputs (forward
  blobs, dx, argmax) are checked on 8 images spread over the batch (first,
  middle, last rows: every M tile edge of the GEMMs is a multiple of 128
  pixels, so these rows sit in different tiles and split-K groups).
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import net as ON  # noqa: E402
from tests import layer_check as LC  # noqa: E402
from tests.gpu_util import f64  # noqa: E402
from workloads import configs, generate  # noqa: E402

if torch.cuda.is_available():
    from paper_1603_07846_b200 import net as PN  # noqa: E402


class Full:
    def __init__(self, net, b, cluster=None):
        self.net, self.b = net, b
        self.cl = cluster or PN.Cluster(0, 1, 0)
        self.n = PN.Net(self.cl, net, b)
        self.upd = configs.UPDATERS[net["name"].split("_")[0]]
        self.n.set_updater(self.upd)
        self.p0 = generate.init_params(ON.param_specs(net))
        self.n.set_params(self.p0)
        self.n.enable_graph(True)
        self.loss = torch.zeros(1, device="cuda")

    def step(self, t):
        self.work0 = self.n.get_working({k: v.shape for k, v in self.p0.items()})
        x, lab = generate.batch(self.net, self.b, t)
        xd, ld = torch.from_numpy(x).cuda(), torch.from_numpy(lab).cuda()
        self.n.train_one_batch(t, xd.data_ptr(), ld.data_ptr(), self.loss.data_ptr())
        self.n.sync()
        return x, lab, float(self.loss.item())

    def check(self, x, lab, sub=None):
        sh = {k: v.shape for k, v in self.p0.items()}
        return LC.check_layers(self.n, self.net, self.b, x, lab, self.p0, self.work0, self.n.get_grads(sh),
                               self.n.get_params(sh),
                               self.n.get_working(sh), self.upd, fused=True, sub=sub)

    def close(self):
        self.n.close()
        self.cl.close()


def summary(rep):
    worst = {}
    for name, what, e in rep:
        worst[what] = max(worst.get(what, 0.0), e)
    return worst


def test_cifar_full_batch_every_layer():
    net = configs.get("cifar10")
    b = 128
    f = Full(net, b)
    try:
        x, lab, loss = f.step(0)
        rep = f.check(x, lab)
        layers = {r[0] for r in rep}
        assert {"conv1", "conv2", "conv3", "pool1", "pool2", "pool3", "norm1", "norm2", "norm3", "relu1", "relu2",
                "relu3", "ip1", "loss"} <= layers
        for q in ("dW", "db", "dx", "y"):
            assert any(r[1] == q and r[0].startswith("conv") for r in rep), q
        ref = ON.train_one_batch(net, {k: f64(v) for k, v in f.p0.items()},
                                 {k: np.zeros(v.shape) for k, v in f.p0.items()}, x, lab, 0, 1, f.upd)
        assert abs(loss - ref["loss"]) <= 0.01 * ref["loss"]
        print("cifar b=128 worst per quantity:", summary(rep))
    finally:
        f.close()


def test_alexnet_full_batch_every_layer():
    net = configs.alexnet(hybrid=False)
    b = 256
    f = Full(net, b)
    try:
        x, lab, loss = f.step(0)
        sub = [0, 1, 63, 127, 128, 200, 254, 255]
        rep = f.check(x, lab, sub=sub)
        for lname in ("conv1", "conv2", "conv3", "conv4", "conv5", "fc6", "fc7", "fc8"):
            got = {r[1] for r in rep if r[0] == lname}
            want = {"y", "dW", "db"} | ({"dx"} if lname != "conv1" else set())
            assert want <= got, (lname, got)
        print("alexnet b=256 worst per quantity:", summary(rep))
    finally:
        f.close()


def test_alexnet_full_batch_loss():
    net = configs.alexnet(hybrid=False)
    b = 256
    f = Full(net, b)
    try:
        x, lab, loss = f.step(0)
        p = {k: f64(v) for k, v in f.p0.items()}
        ref = ON.train_one_batch(net, p, {k: np.zeros(v.shape) for k, v in p.items()}, x, lab, 0, 1, f.upd)
        assert abs(loss - ref["loss"]) <= 0.01 * ref["loss"]
    finally:
        f.close()
