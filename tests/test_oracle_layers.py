"""Pins for oracle/layers.py against things other than itself.

* pure-Python brute force on tiny shapes, written from the
  sums' definitions index by index;
* central finite differences, h = 1e-5, rel < 1e-6;
* closed forms and SPEC examples (tests/golden/spec_examples.json);
* torch CPU float64 library routines (conv2d, max_pool2d / avg_pool2d with
  ceil_mode — Caffe's geometry —, local_response_norm) as independent
  implementations.
"""

import itertools
import json
import math
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import layers as L

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
RNG = np.random.default_rng(1234)


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def fd_grad(f, x, h=1e-5, idx=None):
    """Central differences of scalar f w.r.t. x at the given flat indices."""
    g = np.zeros(x.size)
    flat = x.reshape(-1)
    idx = range(x.size) if idx is None else idx
    for i in idx:
        old = flat[i]
        flat[i] = old + h
        fp = f()
        flat[i] = old - h
        fm = f()
        flat[i] = old
        g[i] = (fp - fm) / (2 * h)
    return g.reshape(x.shape)


# ---------------------------------------------------------------- conv -------
def brute_conv(x, W, b, st, p):
    N, H, Wd, C = x.shape
    Co, R, S, _ = W.shape
    Ho, Wo = (H + 2 * p - R) // st + 1, (Wd + 2 * p - S) // st + 1
    y = np.zeros((N, Ho, Wo, Co))
    dWfn = None
    for n in range(N):
        for oh in range(Ho):
            for ow in range(Wo):
                for co in range(Co):
                    acc = b[co]
                    for r in range(R):
                        for s in range(S):
                            h, w = oh * st - p + r, ow * st - p + s
                            if 0 <= h < H and 0 <= w < Wd:
                                for c in range(C):
                                    acc += W[co, r, s, c] * x[n, h, w, c]
                    y[n, oh, ow, co] = acc
    return y


def brute_conv_bwd(x, W, dy, st, p):
    N, H, Wd, C = x.shape
    Co, R, S, _ = W.shape
    Ho, Wo = dy.shape[1:3]
    dx = np.zeros_like(x)
    dW = np.zeros_like(W)
    for n, oh, ow, co, r, s, c in itertools.product(range(N), range(Ho), range(Wo), range(Co),
                                                    range(R), range(S), range(C)):
        h, w = oh * st - p + r, ow * st - p + s
        if 0 <= h < H and 0 <= w < Wd:
            dW[co, r, s, c] += dy[n, oh, ow, co] * x[n, h, w, c]
            dx[n, h, w, c] += dy[n, oh, ow, co] * W[co, r, s, c]
    return dx, dW, dy.sum(axis=(0, 1, 2))


CONV_CASES = [  # (N, H, W, C, Co, R, stride, pad)
    (2, 5, 5, 3, 2, 1, 1, 0),
    (1, 7, 6, 2, 3, 3, 1, 1),
    (2, 9, 9, 4, 2, 3, 2, 1),
    (1, 9, 9, 3, 2, 5, 1, 2),
    (1, 9, 9, 2, 2, 5, 2, 2),
    (1, 13, 13, 2, 2, 11, 4, 2),
]


@pytest.mark.parametrize("case", CONV_CASES)
def test_conv_matches_brute_force(case):
    N, H, Wd, C, Co, R, st, p = case
    x = RNG.standard_normal((N, H, Wd, C))
    W = RNG.standard_normal((Co, R, R, C))
    b = RNG.standard_normal(Co)
    y = L.conv_forward(x, W, b, st, p)
    assert np.max(np.abs(y - brute_conv(x, W, b, st, p))) < 1e-12
    dy = RNG.standard_normal(y.shape)
    dx, dW, db = L.conv_backward(x, W, dy, st, p)
    bdx, bdW, bdb = brute_conv_bwd(x, W, dy, st, p)
    assert np.max(np.abs(dx - bdx)) < 1e-12
    assert np.max(np.abs(dW - bdW)) < 1e-12
    assert np.max(np.abs(db - bdb)) < 1e-12


def test_conv_1x1_is_matmul():
    x = RNG.standard_normal((3, 4, 5, 6))
    W = RNG.standard_normal((7, 1, 1, 6))
    b = RNG.standard_normal(7)
    y = L.conv_forward(x, W, b, 1, 0)
    ref = x.reshape(-1, 6) @ W.reshape(7, 6).T + b
    assert np.max(np.abs(y.reshape(-1, 7) - ref)) < 1e-12


@pytest.mark.parametrize("case", [(4, 32, 32, 3, 8, 5, 1, 2), (2, 35, 35, 3, 4, 11, 4, 2), (2, 13, 13, 16, 8, 3, 1, 1)])
def test_conv_vs_torch(case):
    N, H, Wd, C, Co, R, st, p = case
    x = RNG.standard_normal((N, H, Wd, C))
    W = RNG.standard_normal((Co, R, R, C))
    b = RNG.standard_normal(Co)
    xt = torch.tensor(x.transpose(0, 3, 1, 2), requires_grad=True)
    Wt = torch.tensor(W.transpose(0, 3, 1, 2), requires_grad=True)
    bt = torch.tensor(b, requires_grad=True)
    yt = F.conv2d(xt, Wt, bt, stride=st, padding=p)
    y = L.conv_forward(x, W, b, st, p)
    assert rel(y, yt.detach().numpy().transpose(0, 2, 3, 1)) < 1e-13
    dy = RNG.standard_normal(y.shape)
    yt.backward(torch.tensor(dy.transpose(0, 3, 1, 2)))
    dx, dW, db = L.conv_backward(x, W, dy, st, p)
    assert rel(dx, xt.grad.numpy().transpose(0, 2, 3, 1)) < 1e-13
    assert rel(dW, Wt.grad.numpy().transpose(0, 2, 3, 1)) < 1e-13
    assert rel(db, bt.grad.numpy()) < 1e-13


def test_conv_finite_difference():
    x = RNG.standard_normal((2, 5, 5, 2))
    W = RNG.standard_normal((3, 3, 3, 2))
    b = RNG.standard_normal(3)
    c = RNG.standard_normal((2, 3, 3, 3))  # L = sum(c * y)
    f = lambda: float(np.sum(c * L.conv_forward(x, W, b, 2, 1)))
    dx, dW, db = L.conv_backward(x, W, c, 2, 1)
    assert rel(dW, fd_grad(f, W)) < 1e-6
    assert rel(db, fd_grad(f, b)) < 1e-6
    assert rel(dx, fd_grad(f, x)) < 1e-6


# ---------------------------------------------------------------- pool -------
def brute_pool(x, k, s, mode):
    """Caffe pooling loops (p = 0): ceil-mode output, clip windows to the image."""
    N, H, W, C = x.shape
    Ho = int(math.ceil((H - k) / s)) + 1
    Wo = int(math.ceil((W - k) / s)) + 1
    y = np.zeros((N, Ho, Wo, C))
    idx = np.zeros((N, Ho, Wo, C), dtype=np.int64)
    for n, oh, ow, c in itertools.product(range(N), range(Ho), range(Wo), range(C)):
        hs, ws = oh * s, ow * s
        he, we = min(hs + k, H), min(ws + k, W)
        if mode == "max":
            best, bi = -np.inf, -1
            for h in range(hs, he):
                for w in range(ws, we):
                    if x[n, h, w, c] > best:
                        best, bi = x[n, h, w, c], h * W + w
            y[n, oh, ow, c], idx[n, oh, ow, c] = best, bi
        else:
            tot = 0.0
            for h in range(hs, he):
                for w in range(ws, we):
                    tot += x[n, h, w, c]
            y[n, oh, ow, c] = tot / ((he - hs) * (we - ws))
    return y, idx


@pytest.mark.parametrize("H", [8, 9, 7, 13])
def test_pool_brute_force(H):
    x = RNG.standard_normal((2, H, H, 3))
    y, idx = L.maxpool_forward(x, 3, 2, 0)
    by, bidx = brute_pool(x, 3, 2, "max")
    assert np.array_equal(idx, bidx) and np.array_equal(y, by)
    ya = L.avgpool_forward(x, 3, 2, 0)
    bya, _ = brute_pool(x, 3, 2, "avg")
    assert np.max(np.abs(ya - bya)) < 1e-13


@pytest.mark.parametrize("H", [32, 16, 8, 55, 27, 13])
def test_pool_vs_torch_ceil_mode(H):
    x = RNG.standard_normal((2, H, H, 4))
    xt = torch.tensor(x.transpose(0, 3, 1, 2))
    yt, it = F.max_pool2d(xt, 3, 2, 0, ceil_mode=True, return_indices=True)
    y, idx = L.maxpool_forward(x, 3, 2, 0)
    assert y.shape[1] == yt.shape[2]
    assert np.array_equal(idx, it.numpy().transpose(0, 2, 3, 1))
    assert np.array_equal(y, yt.numpy().transpose(0, 2, 3, 1))
    ya = L.avgpool_forward(x, 3, 2, 0)
    yat = F.avg_pool2d(xt, 3, 2, 0, ceil_mode=True, count_include_pad=True)
    assert rel(ya, yat.numpy().transpose(0, 2, 3, 1)) < 1e-14
    # backward
    dy = RNG.standard_normal(y.shape)
    xg = torch.tensor(x.transpose(0, 3, 1, 2), requires_grad=True)
    F.max_pool2d(xg, 3, 2, 0, ceil_mode=True).backward(torch.tensor(dy.transpose(0, 3, 1, 2)))
    assert rel(L.maxpool_backward(x.shape, idx, dy), xg.grad.numpy().transpose(0, 2, 3, 1)) < 1e-14
    xg.grad = None
    F.avg_pool2d(xg, 3, 2, 0, ceil_mode=True, count_include_pad=True).backward(torch.tensor(dy.transpose(0, 3, 1, 2)))
    assert rel(L.avgpool_backward(x.shape, dy, 3, 2, 0), xg.grad.numpy().transpose(0, 2, 3, 1)) < 1e-14


def test_pool_sizes_caffe():
    # Caffe ceil mode: 32->16->8->4 (CIFAR), 55->27->13->6 (AlexNet)
    for h, ho in [(32, 16), (16, 8), (8, 4), (55, 27), (27, 13), (13, 6)]:
        assert L.pool_out_size(h, 3, 2, 0) == ho
    # pad > 0 last-window rule: window must start inside image + pad
    assert L.pool_out_size(5, 2, 2, 1) == 3


def test_pool_identity_k1():
    x = RNG.standard_normal((2, 4, 5, 3))
    y, idx = L.maxpool_forward(x, 1, 1, 0)
    assert np.array_equal(y, x)
    assert np.array_equal(idx[0, :, :, 0], np.arange(20).reshape(4, 5))
    assert np.array_equal(L.avgpool_forward(x, 1, 1, 0), x)


def test_maxpool_first_max_tie_break():
    x = np.zeros((1, 3, 3, 1))
    _, idx = L.maxpool_forward(x, 3, 2, 0)
    assert idx[0, 0, 0, 0] == 0
    x[0, :, :, 0] = [[0, 5, 5], [5, 0, 0], [0, 0, 5]]
    _, idx = L.maxpool_forward(x, 3, 2, 0)
    assert idx[0, 0, 0, 0] == 1


def test_pool_finite_difference():
    x = RNG.standard_normal((1, 7, 7, 2))
    c = RNG.standard_normal((1, 3, 3, 2))
    f = lambda: float(np.sum(c * L.avgpool_forward(x, 3, 2, 0)))
    assert rel(L.avgpool_backward(x.shape, c, 3, 2, 0), fd_grad(f, x)) < 1e-6
    fm = lambda: float(np.sum(c * L.maxpool_forward(x, 3, 2, 0)[0]))
    _, idx = L.maxpool_forward(x, 3, 2, 0)
    assert rel(L.maxpool_backward(x.shape, idx, c), fd_grad(fm, x)) < 1e-6


# ---------------------------------------------------------------- LRN --------
def brute_lrn(x, n, alpha, beta, k):
    y = np.zeros_like(x)
    C = x.shape[-1]
    for pos in itertools.product(*[range(s) for s in x.shape[:-1]]):
        for c in range(C):
            acc = 0.0
            for cc in range(c - n // 2, c + n // 2 + 1):
                if 0 <= cc < C:
                    acc += x[pos + (cc,)] ** 2
            y[pos + (c,)] = x[pos + (c,)] / (k + alpha / n * acc) ** beta
    return y


def test_lrn_brute_and_torch():
    x = RNG.standard_normal((2, 3, 3, 7))
    y, scale = L.lrn_forward(x, 3, 0.3, 0.75, 1.0)
    assert np.max(np.abs(y - brute_lrn(x, 3, 0.3, 0.75, 1.0))) < 1e-14
    for n in (3, 5):
        y, _ = L.lrn_forward(x, n, 5e-2, 0.75, 2.0)
        yt = F.local_response_norm(torch.tensor(x.transpose(0, 3, 1, 2)), n, 5e-2, 0.75, 2.0)
        assert rel(y, yt.numpy().transpose(0, 2, 3, 1)) < 1e-14


def test_lrn_closed_forms():
    x = RNG.standard_normal((2, 2, 2, 5))
    y, _ = L.lrn_forward(x, 3, 0.0, 0.75, 2.0)         # alpha = 0 -> y = x k^-beta
    assert np.max(np.abs(y - x * 2.0 ** -0.75)) < 1e-15
    x = np.zeros((1, 1, 1, 6))
    x[0, 0, 0, 2] = 1.7                               # single channel -> x / (k + a x^2/n)^b
    y, _ = L.lrn_forward(x, 3, 0.4, 0.75, 1.0)
    assert abs(y[0, 0, 0, 2] - 1.7 / (1 + 0.4 * 1.7 ** 2 / 3) ** 0.75) < 1e-15
    assert np.count_nonzero(y) == 1


def test_lrn_finite_difference():
    x = RNG.standard_normal((2, 2, 2, 6))
    c = RNG.standard_normal(x.shape)
    f = lambda: float(np.sum(c * L.lrn_forward(x, 3, 0.5, 0.75, 1.0)[0]))
    y, sc = L.lrn_forward(x, 3, 0.5, 0.75, 1.0)
    assert rel(L.lrn_backward(x, y, sc, c, 3, 0.5, 0.75), fd_grad(f, x)) < 1e-6


# ------------------------------------------------------- neurons / IP --------
def test_sigmoid_spec_values():
    g = GOLD["sigmoid_zero"]
    assert L.sigmoid_forward(np.array([g["x"]]))[0] == g["y"]
    g = GOLD["sigmoid_grad"]
    assert L.sigmoid_backward(np.array([g["y"]]), np.array([g["dy"]]))[0] == g["dx"]
    x = np.array([-800.0, -30.0, 0.0, 30.0, 800.0])   # stable branch: no overflow/NaN
    y = L.sigmoid_forward(x)
    assert np.all(np.isfinite(y)) and y[0] == 0.0 and y[-1] == 1.0
    assert abs(y[1] - 1 / (1 + math.exp(30))) < 1e-25


def test_sigmoid_relu_fd():
    x = RNG.standard_normal(20)
    c = RNG.standard_normal(20)
    f = lambda: float(np.sum(c * L.sigmoid_forward(x)))
    assert rel(L.sigmoid_backward(L.sigmoid_forward(x), c), fd_grad(f, x)) < 1e-6
    fr = lambda: float(np.sum(c * L.relu_forward(x)))
    assert rel(L.relu_backward(L.relu_forward(x), c), fd_grad(fr, x)) < 1e-6
    assert L.relu_backward(np.array([0.0]), np.array([1.0]))[0] == 0.0   # reading A8


def test_ip_spec_and_fd():
    g = GOLD["ip_hand"]
    y = L.ip_forward(np.array(g["x"]), np.array(g["W"]), np.array(g["b"]))
    assert np.array_equal(y, np.array(g["y"]))
    gm = GOLD["gemm_hand"]
    assert np.array_equal(L.ip_forward(np.array(gm["A"]), np.array(gm["B"]), np.zeros(1)), np.array(gm["C"]))
    x = RNG.standard_normal((4, 3))
    W = RNG.standard_normal((3, 2))
    b = RNG.standard_normal(2)
    c = RNG.standard_normal((4, 2))
    f = lambda: float(np.sum(c * L.ip_forward(x, W, b)))
    dx, dW, db = L.ip_backward(x, W, c)
    assert rel(dW, fd_grad(f, W)) < 1e-6 and rel(db, fd_grad(f, b)) < 1e-6 and rel(dx, fd_grad(f, x)) < 1e-6


# ------------------------------------------------------------- losses --------
def test_softmax_ce_spec():
    g = GOLD["softmax_ce_grad"]
    loss, dz = L.softmax_ce(np.array(g["z"]), np.array(g["label"]), 1)
    assert np.max(np.abs(dz - np.array(g["dx"]))) < 1e-15
    assert abs(loss[0] - math.log(3)) < 1e-15
    for C in (10, 1000):   # equal logits -> L = ln C exactly
        loss, _ = L.softmax_ce(np.full((3, C), 0.25), np.array([0, 1, 2]), 3)
        assert np.max(np.abs(loss - math.log(C))) < 1e-13
    with pytest.raises(ValueError):
        L.softmax_ce(np.zeros((1, 3)), np.array([3]), 1)


def test_softmax_ce_fd_and_argmin():
    z = RNG.standard_normal((5, 7)) * 3
    lab = RNG.integers(0, 7, 5)
    f = lambda: float(np.sum(L.softmax_ce(z, lab, 5)[0])) / 5
    _, dz = L.softmax_ce(z, lab, 5)
    assert rel(dz, fd_grad(f, z)) < 1e-6
    assert np.array_equal(np.argmin(dz, axis=1), lab)       # reading A11 invariant
    # vs torch cross_entropy (mean reduction)
    zt = torch.tensor(z, requires_grad=True)
    lt = F.cross_entropy(zt, torch.tensor(lab))
    lt.backward()
    assert abs(lt.item() - np.mean(L.softmax_ce(z, lab, 5)[0])) < 1e-14
    assert rel(dz, zt.grad.numpy()) < 1e-14


def test_euclidean():
    u = RNG.standard_normal((4, 6))
    loss, du = L.euclidean(u, u.copy(), 4)
    assert np.all(loss == 0) and np.all(du == 0)
    v = RNG.standard_normal((4, 6))
    f = lambda: float(np.sum(L.euclidean(u, v, 4)[0])) / 4
    _, du = L.euclidean(u, v, 4)
    assert rel(du, fd_grad(f, u)) < 1e-6
    assert abs(np.sum(L.euclidean(u, v, 4)[0]) / 4 - np.sum((u - v) ** 2) / 8) < 1e-14
