"""Parity at BASELINE.json's full sizes in the launch configuration bench.py
times (CUDA-graph replay, ReLU fusion on):

* CIFAR-10 ConvNet, batch 128: every layer layer-isolated (reading A10) against
  the float64 oracle, argmax bit-exact, loss within 1% of the full oracle step;
* AlexNet-shaped, batch 256 on one GPU: sampled outputs the oracle computes one
  image / one row at a time (conv1 + ReLU for images 0 and 255, pool1 argmax
  bit-exact for those images, fc8 logits and the fc8 weight gradient from the
  GPU's own fc7 blob and loss gradient) and the loss of the full oracle step.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import layers as OL  # noqa: E402
from oracle import net as ON  # noqa: E402
from tests.gpu_util import FP32_TOL, TF32_TOL, f64, normwise  # noqa: E402
from workloads import configs, generate  # noqa: E402

if torch.cuda.is_available():
    from paper_1603_07846_b200 import _lib as L  # noqa: E402
    from paper_1603_07846_b200 import net as PN  # noqa: E402


class Full:
    def __init__(self, net, b):
        self.net, self.b = net, b
        self.cl = PN.Cluster(0, 1, 0)
        self.n = PN.Net(self.cl, net, b)
        self.n.set_updater(configs.UPDATERS[net["name"].split("_")[0]])
        self.p0 = generate.init_params(ON.param_specs(net))
        self.n.set_params(self.p0)
        self.n.enable_graph(True)
        self.loss = torch.zeros(1, device="cuda")
        self.info = self.n.layer_info

    def step(self, t):
        x, lab = generate.batch(self.net, self.b, t)
        xd, ld = torch.from_numpy(x).cuda(), torch.from_numpy(lab).cuda()
        self.n.train_one_batch(t, xd.data_ptr(), ld.data_ptr(), self.loss.data_ptr())
        self.n.sync()
        return x, lab, float(self.loss.item())

    def blob(self, i, which=0, dtype=torch.float32):
        nb = self.n.blob_size(i, which)
        t = torch.empty(nb // 4, dtype=dtype, device="cuda")
        L.sg_blob_get(self.n.h, i, which, t.data_ptr(), nb, None)
        torch.cuda.synchronize()
        return t.cpu().numpy()

    def image(self, i, which=0):
        li = self.info[i if which == 0 else self.info[i]["src"]]
        return f64(self.blob(i, which).reshape(li["local_shape"]))

    def vec(self, i, which=0):
        li = self.info[i if which == 0 else self.info[i]["src"]]
        rows, cols = li["local_shape"][:2]
        return f64(self.blob(i, which).reshape(rows, li["ld"])[:, :cols])

    def idx(self, name):
        return self.n.layer_index(name)

    def close(self):
        self.n.close()
        self.cl.close()


def test_cifar_full_batch_graph_fused():
    net = configs.get("cifar10")
    b = 128
    f = Full(net, b)
    try:
        x, lab, loss = f.step(0)
        ref = ON.train_one_batch(net, {k: f64(v) for k, v in f.p0.items()},
                                 {k: np.zeros(v.shape) for k, v in f.p0.items()}, x, lab, 0, 1,
                                 configs.UPDATERS["cifar10"])
        assert abs(loss - ref["loss"]) <= 0.01 * ref["loss"]
        p = {k: f64(v) for k, v in f.p0.items()}
        grads = f.n.get_grads({k: v.shape for k, v in f.p0.items()})
        # conv2 (fused with relu2): relu(conv(x)) from the GPU's own norm1 blob
        xin = f.image(f.idx("norm1"))
        y = f.image(f.idx("conv2"))
        assert normwise(y, OL.relu_forward(OL.conv_forward(xin, p["conv2/W"], p["conv2/b"], 1, 2))) < TF32_TOL
        # conv2 weight / bias gradient from the GPU's relu2 input gradient
        dy = f.image(f.idx("relu2"), 1)
        _, rdW, rdb = OL.conv_backward(xin, p["conv2/W"], dy, 1, 2, need_dx=False)
        assert normwise(grads["conv2/W"], rdW) < TF32_TOL and normwise(grads["conv2/b"], rdb) < TF32_TOL
        # pool1 argmax bit-exact on the GPU's own conv1 output
        c1 = f.image(f.idx("conv1"))
        _, ridx = OL.maxpool_forward(c1, 3, 2, 0)
        am = f.blob(f.idx("pool1"), 2, torch.int32).reshape(ridx.shape)
        assert np.array_equal(am, ridx)
        # LRN and avg pool layer-isolated
        r3 = f.image(f.idx("relu3"))
        p3 = f.image(f.idx("pool3"))
        assert normwise(p3, OL.avgpool_forward(r3, 3, 2, 0)) < FP32_TOL
        n3 = f.image(f.idx("norm3"))
        assert normwise(n3, OL.lrn_forward(p3, 3, 5e-5, 0.75, 1.0)[0]) < FP32_TOL
        # softmax gradient and the label invariant
        z = f.vec(f.idx("ip1"))
        _, rdz = OL.softmax_ce(z, lab, b)
        dz = f.vec(f.idx("loss"), 1)
        assert normwise(dz, rdz) < FP32_TOL and np.array_equal(np.argmin(dz, axis=1), lab)
    finally:
        f.close()


def test_alexnet_full_batch_sampled():
    net = configs.alexnet(hybrid=False)
    b = 256
    f = Full(net, b)
    try:
        x, lab, loss = f.step(0)
        p = {k: f64(v) for k, v in f.p0.items()}
        conv1 = f.image(f.idx("conv1"))      # post-ReLU (fused)
        for i in (0, b - 1):
            ref = OL.relu_forward(OL.conv_forward(f64(x[i:i + 1]), p["conv1/W"], p["conv1/b"], 4, 2))
            assert normwise(conv1[i:i + 1], ref) < TF32_TOL
            _, ridx = OL.maxpool_forward(conv1[i:i + 1], 3, 2, 0)
            am = f.blob(f.idx("pool1"), 2, torch.int32).reshape((b,) + ridx.shape[1:])
            assert np.array_equal(am[i:i + 1], ridx)
        fc7 = f.vec(f.idx("fc7"))            # post-ReLU (fused), fc8 input
        fc8 = f.vec(f.idx("fc8"))
        rows = np.array([0, 1, 100, 255])
        assert normwise(fc8[rows], OL.ip_forward(fc7[rows], p["fc8/W"], p["fc8/b"])) < TF32_TOL
        dz = f.vec(f.idx("loss"), 1)
        grads = f.n.get_grads({k: v.shape for k, v in f.p0.items()})
        assert normwise(grads["fc8/W"], fc7.T @ dz) < TF32_TOL
        assert np.array_equal(np.argmin(dz, axis=1), lab)
        ref = ON.train_one_batch(net, p, {k: np.zeros(v.shape) for k, v in p.items()}, x, lab, 0, 1,
                                 configs.UPDATERS["alexnet"])
        assert abs(loss - ref["loss"]) <= 0.01 * ref["loss"]
    finally:
        f.close()
