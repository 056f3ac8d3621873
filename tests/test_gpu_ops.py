"""Layer-isolated GPU parity through the C ABI (sg_op_*) vs the float64 oracle.

Each CUDA layer is fed fp32 inputs; the oracle gets the same values widened to
float64 (reading A10: layer-isolated comparison).  Tolerances: TF32
tensor-core contractions within 2e-3 normwise (reading A9), fp32 SIMT kernels
within 1e-5, argmax / labels bit-exact.
"""

import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import layers as L  # noqa: E402
from oracle import updater as U  # noqa: E402
from tests.gpu_util import TF32_TOL, FP32_TOL, dev, empty, f64, host, normwise, ptr  # noqa: E402

lib = pytest.importorskip("paper_1603_07846_b200._lib") if torch.cuda.is_available() else None
RNG = np.random.default_rng(2024)


def r32(*shape, scale=1.0):
    return (RNG.standard_normal(shape) * scale).astype(np.float32)


# ------------------------------------------------------------------ GEMM ----
@pytest.mark.parametrize("M,N,K", [(128, 32, 32), (200, 96, 100), (256, 300, 520), (64, 256, 784),
                                   (1000, 64, 36), (96, 512, 4096)])
@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_gemm(M, N, K, ta, tb):
    A = r32(K, M) if ta else r32(M, K)
    B = r32(N, K) if tb else r32(K, N)
    Cd = empty((M, N))
    lib.sg_op_gemm(ptr(dev(A)), ta, ptr(dev(B)), tb, ptr(Cd), M, N, K, None)
    ref = (f64(A).T if ta else f64(A)) @ (f64(B).T if tb else f64(B))
    assert normwise(host(Cd), ref) < TF32_TOL


# ------------------------------------------------------------------ conv ----
CONV = [  # N, H, W, C, Co, R, stride, pad
    (4, 32, 32, 4, 32, 5, 1, 2),      # CIFAR conv1 (C padded to 4): direct CUDA-core path
    (3, 12, 10, 4, 8, 3, 1, 1),       # direct path, ragged Wo (10 = 2 x 4 + 2)
    (150, 8, 8, 4, 32, 5, 1, 2),      # 4-channel resident-image weight gradient: 150 samples on 148 CTAs
    (5, 7, 9, 4, 32, 3, 1, 1),        # ... ragged last 32-pixel stage (63 pixels)
    (4, 16, 16, 32, 32, 5, 1, 2),     # CIFAR conv2
    (8, 8, 8, 32, 64, 5, 1, 2),       # CIFAR conv3
    (3, 10, 7, 32, 32, 3, 1, 1),      # resident-image path, non-square, 3x3
    (2, 11, 11, 64, 32, 3, 1, 0),     # resident-image path, 2 K blocks, no padding
    (2, 24, 24, 32, 32, 3, 1, 1),     # resident-image weight gradient: column tap groups only
    (2, 16, 16, 32, 64, 5, 1, 2),     # resident-image weight gradient, Co = 64
    (2, 35, 35, 4, 64, 11, 4, 2),     # AlexNet conv1 geometry
    (2, 27, 27, 64, 192, 5, 1, 2),    # AlexNet conv2 (TMA wgrad, C = 64)
    (2, 13, 13, 192, 384, 3, 1, 1),   # AlexNet conv3
    (27, 27, 27, 64, 192, 5, 1, 2),   # 192-wide tiles (>= 148 M tiles): im2col forward, TMA weight gradient
    (26, 27, 27, 192, 32, 3, 1, 1),   # 192-wide tiles: TMA data gradient (N = C = 192)
    (52, 27, 27, 64, 64, 3, 1, 1),    # 256-row work items (N = 64, >= 148 of them): forward and data gradient
    (3, 9, 7, 8, 12, 3, 2, 1),        # ragged, strided dgrad
]


@pytest.mark.parametrize("case", CONV)
def test_conv(case):
    N, H, W, Ci, Co, R, st, p = case
    x = r32(N, H, W, Ci)
    Wt = r32(Co, R, R, Ci, scale=0.1)
    b = r32(Co)
    d = lib.ConvDesc(N, H, W, Ci, Co, R, R, st, p)
    Ho, Wo = C.c_int32(), C.c_int32()
    lib.sg_conv_out_shape(C.byref(d), C.byref(Ho), C.byref(Wo))
    y = empty((N, Ho.value, Wo.value, Co))
    xd, Wd = dev(x), dev(Wt)
    lib.sg_op_conv_forward(C.byref(d), ptr(xd), ptr(Wd), ptr(dev(b)), ptr(y), None)
    yref = L.conv_forward(f64(x), f64(Wt), f64(b), st, p)
    assert normwise(host(y), yref) < TF32_TOL
    dy = r32(*yref.shape)
    dx, dW, db = empty(x.shape), empty(Wt.shape), empty((Co,))
    lib.sg_op_conv_backward(C.byref(d), ptr(xd), ptr(Wd), ptr(dev(dy)), ptr(dx), ptr(dW), ptr(db), None)
    rdx, rdW, rdb = L.conv_backward(f64(x), f64(Wt), f64(dy), st, p)
    assert normwise(host(dW), rdW) < TF32_TOL
    assert normwise(host(db), rdb) < TF32_TOL   # fused ones-row of the TF32 wgrad GEMM
    assert normwise(host(dx), rdx) < TF32_TOL


def test_conv_implicit_gemm_path():
    """With the resident-image convolution disabled (SG_IMG_CONV=0, read once per
    process) the implicit-GEMM path passes the same conv parity cases."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_gpu_ops.py", "-m", "gpu", "-q", "-x",
                        "-k", "test_conv and not rejects and not implicit", "-p", "no:cacheprovider"],
                       cwd=root, env=dict(os.environ, SG_IMG_CONV="0"), capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_conv_rejects_unpadded_channels():
    d = lib.ConvDesc(1, 8, 8, 3, 8, 3, 3, 1, 1)
    with pytest.raises(lib.SingaError) as e:
        lib.sg_op_conv_forward(C.byref(d), None, None, None, None, None)
    assert e.value.name in ("SG_ERR_DIMENSION", "SG_ERR_INVALID_ARG")


# ------------------------------------------------------------------- IP -----
@pytest.mark.parametrize("rows,dv,dh", [(64, 784, 256), (64, 256, 12), (128, 1024, 12), (256, 9216, 512),
                                        (8, 4, 4)])
def test_ip(rows, dv, dh):
    x, W, b = r32(rows, dv), r32(dv, dh, scale=0.05), r32(dh)
    y = empty((rows, dh))
    xd, Wd = dev(x), dev(W)
    lib.sg_op_ip_forward(ptr(xd), ptr(Wd), ptr(dev(b)), ptr(y), rows, dv, dh, None)
    assert normwise(host(y), L.ip_forward(f64(x), f64(W), f64(b))) < TF32_TOL
    dy = r32(rows, dh)
    dx, dW, db = empty((rows, dv)), empty((dv, dh)), empty((dh,))
    lib.sg_op_ip_backward(ptr(xd), ptr(Wd), ptr(dev(dy)), ptr(dx), ptr(dW), ptr(db), rows, dv, dh, None)
    rdx, rdW, rdb = L.ip_backward(f64(x), f64(W), f64(dy))
    assert normwise(host(dx), rdx) < TF32_TOL
    assert normwise(host(dW), rdW) < TF32_TOL
    assert normwise(host(db), rdb) < TF32_TOL   # fused ones-row of the TF32 wgrad GEMM


# ------------------------------------------------------------------ pool ----
@pytest.mark.parametrize("N,H,Cc", [(4, 32, 32), (2, 16, 32), (2, 8, 64), (2, 55, 64), (2, 13, 256), (1, 7, 4)])
@pytest.mark.parametrize("mode", [0, 1])
def test_pool(N, H, Cc, mode):
    x = r32(N, H, H, Cc)
    d = lib.PoolDesc(N, H, H, Cc, 3, 2, 0, mode)
    Ho, Wo = C_int_pair(d)
    y = empty((N, Ho, Wo, Cc))
    mask = torch.zeros((N, Ho, Wo, Cc), dtype=torch.uint8, device="cuda")
    xd = dev(x)
    lib.sg_op_pool_forward(C.byref(d), ptr(xd), ptr(y), ptr(mask), None)
    dy = r32(N, Ho, Wo, Cc)
    dx = empty(x.shape)
    lib.sg_op_pool_backward(C.byref(d), ptr(dev(dy)), ptr(mask), ptr(dx), None)
    if mode == 0:
        ry, ridx = L.maxpool_forward(f64(x), 3, 2, 0)
        assert np.array_equal(host(y), ry.astype(np.float32))           # max is exact
        am = torch.zeros((N, Ho, Wo, Cc), dtype=torch.int32, device="cuda")
        lib.sg_op_pool_argmax(C.byref(d), ptr(mask), ptr(am), None)
        assert np.array_equal(host(am), ridx)                             # bit-exact argmax
        assert normwise(host(dx), L.maxpool_backward(x.shape, ridx, f64(dy))) < FP32_TOL
    else:
        assert normwise(host(y), L.avgpool_forward(f64(x), 3, 2, 0)) < FP32_TOL
        assert normwise(host(dx), L.avgpool_backward(x.shape, f64(dy), 3, 2, 0)) < FP32_TOL


def C_int_pair(d):
    Ho, Wo = C.c_int32(), C.c_int32()
    lib.sg_pool_out_shape(C.byref(d), C.byref(Ho), C.byref(Wo))
    return Ho.value, Wo.value


def test_maxpool_ties_first_max():
    x = np.zeros((1, 3, 3, 4), np.float32)
    x[0, :, :, 1] = [[0, 5, 5], [5, 0, 0], [0, 0, 5]]
    d = lib.PoolDesc(1, 3, 3, 4, 3, 2, 0, 0)
    y = empty((1, 1, 1, 4))
    mask = torch.zeros((1, 1, 1, 4), dtype=torch.uint8, device="cuda")
    lib.sg_op_pool_forward(C.byref(d), ptr(dev(x)), ptr(y), ptr(mask), None)
    am = torch.zeros((1, 1, 1, 4), dtype=torch.int32, device="cuda")
    lib.sg_op_pool_argmax(C.byref(d), ptr(mask), ptr(am), None)
    assert host(am).reshape(-1).tolist() == [0, 1, 0, 0]


# ------------------------------------------------------------------- LRN ----
@pytest.mark.parametrize("pixels,Cc,n,alpha", [(128 * 256, 32, 3, 5e-5), (300, 64, 5, 0.1), (17, 8, 3, 1.0),
                                               (31, 4, 3, 1.0), (64, 128, 9, 0.2),      # shuffle path edges
                                               (50, 12, 3, 0.5), (40, 256, 5, 0.1)])   # element-wise path
def test_lrn(pixels, Cc, n, alpha):
    x = r32(pixels, Cc)
    d = lib.LrnDesc(pixels, Cc, n, alpha, 0.75, 1.0)
    y, sc, dx = empty(x.shape), empty(x.shape), empty(x.shape)
    xd = dev(x)
    lib.sg_op_lrn_forward(C.byref(d), ptr(xd), ptr(y), ptr(sc), None)
    ry, rsc = L.lrn_forward(f64(x), n, alpha, 0.75, 1.0)
    assert normwise(host(y), ry) < FP32_TOL
    dy = r32(pixels, Cc)
    lib.sg_op_lrn_backward(C.byref(d), ptr(xd), ptr(y), ptr(sc), ptr(dev(dy)), ptr(dx), None)
    # oracle fed the GPU's own forward blobs (layer-isolated)
    gy, gsc = f64(host(y)), f64(host(sc))
    assert normwise(host(dx), L.lrn_backward(f64(x), gy, gsc, f64(dy), n, alpha, 0.75)) < FP32_TOL


# ------------------------------------------------------- neurons / losses ---
@pytest.mark.parametrize("n", [1, 7, 4096, 100003])
def test_neurons(n):
    x = r32(n, scale=3.0)
    x[0] = 0.0
    dy = r32(n)
    for kind, f, b in [(4, L.relu_forward, L.relu_backward), (5, L.sigmoid_forward, L.sigmoid_backward)]:
        y, dx = empty((n,)), empty((n,))
        lib.sg_op_neuron_forward(kind, ptr(dev(x)), ptr(y), n, None)
        assert normwise(host(y), f(f64(x))) < FP32_TOL
        gy = host(y)
        lib.sg_op_neuron_backward(kind, ptr(dev(gy)), ptr(dev(dy)), ptr(dx), n, None)
        assert normwise(host(dx), b(f64(gy), f64(dy))) < FP32_TOL


@pytest.mark.parametrize("rows,Cc", [(128, 10), (32, 1000), (3, 3), (257, 125)])
def test_softmax_ce(rows, Cc):
    z = r32(rows, Cc, scale=2.0)
    lab = RNG.integers(0, Cc, rows).astype(np.int32)
    loss, dz = empty((rows,)), empty((rows, Cc))
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    lib.sg_op_softmax_ce(ptr(dev(z)), ptr(dev(lab)), rows, Cc, rows, ptr(loss), ptr(dz), ptr(err), None)
    rl, rdz = L.softmax_ce(f64(z), lab, rows)
    assert normwise(host(loss), rl) < FP32_TOL
    assert normwise(host(dz), rdz) < FP32_TOL
    assert np.array_equal(np.argmin(host(dz), axis=1), lab)   # label-indexing invariant (A11)
    assert host(err)[0] == 0
    lab[0] = Cc
    lib.sg_op_softmax_ce(ptr(dev(z)), ptr(dev(lab)), rows, Cc, rows, ptr(loss), ptr(dz), ptr(err), None)
    assert host(err)[0] != 0


def test_softmax_spec_example():
    z = np.zeros((1, 3), np.float32)
    loss, dz = empty((1,)), empty((1, 3))
    lib.sg_op_softmax_ce(ptr(dev(z)), ptr(dev(np.zeros(1, np.int32))), 1, 3, 1, ptr(loss), ptr(dz), None, None)
    assert np.allclose(host(dz), [[-2 / 3, 1 / 3, 1 / 3]], atol=1e-7)


@pytest.mark.parametrize("rows,d", [(256, 784), (5, 3)])
def test_euclidean(rows, d):
    u, v = r32(rows, d), r32(rows, d)
    loss, du = empty((rows,)), empty((rows, d))
    lib.sg_op_euclidean(ptr(dev(u)), ptr(dev(v)), rows, d, rows, ptr(loss), ptr(du), None)
    rl, rdu = L.euclidean(f64(u), f64(v), rows)
    assert normwise(host(loss), rl) < FP32_TOL and normwise(host(du), rdu) < FP32_TOL


# --------------------------------------------------------------- Updater ----
def test_updater_vs_oracle_and_sharding():
    n = 1 << 20 | 3
    w, g = r32(n, scale=0.05), r32(n, scale=0.01)
    v = np.zeros(n, np.float32)
    cfg = {"base_lr": 0.01, "momentum": 0.9, "weight_decay": 5e-4, "lr_policy": "fixed"}
    wd_, gd, vd = dev(w), dev(g), dev(v)
    rw, rv = f64(w), f64(v)
    for t in range(5):
        lib.sg_op_sgd_momentum(ptr(wd_), ptr(gd), ptr(vd), n, 0.01, 0.9, 5e-4, 0.5, None)
        rw, rv = U.sgd_momentum(rw, rv, f64(g), cfg, t, 0.5)
    assert normwise(host(wd_), rw) < 1e-6 and normwise(host(vd), rv) < 1e-6
    # sharded == unsharded, bit-exact (elementwise update)
    w2, v2 = dev(w), dev(v)
    half = (n // 2) & ~3
    for t in range(5):
        for off, ln in [(0, half), (half, n - half)]:
            lib.sg_op_sgd_momentum(ptr(w2) + 4 * off, ptr(gd) + 4 * off, ptr(v2) + 4 * off, ln, 0.01, 0.9, 5e-4,
                                   0.5, None)
    assert np.array_equal(host(w2), host(wd_)) and np.array_equal(host(v2), host(vd))
    # SPEC S:409 hand value and lr = 0 constancy
    a, gg, vv = dev(np.array([1.0, 1, 1, 1], np.float32)), dev(np.full(4, 0.5, np.float32)), dev(np.zeros(4, np.float32))
    lib.sg_op_sgd_momentum(ptr(a), ptr(gg), ptr(vv), 4, 0.1, 0.0, 0.0, 1.0, None)
    assert np.allclose(host(a), 0.95, atol=1e-7)
    w3 = dev(w)
    lib.sg_op_sgd_momentum(ptr(w3), ptr(gd), ptr(dev(v)), n, 0.0, 0.9, 5e-4, 1.0, None)
    assert np.array_equal(host(w3), w)


def test_adagrad_vs_oracle():
    """AdaGrad Updater (reading A26) vs the float64 oracle
    over 5 steps; S:418 first step -alpha*sign(g); zero gradient leaves w, h."""
    n = (1 << 18) + 5
    w, g = r32(n, scale=0.05), r32(n, scale=0.01)
    cfg = {"base_lr": 0.01, "momentum": 0.0, "weight_decay": 5e-4, "lr_policy": "fixed", "type": "adagrad",
           "eps": 1e-8}
    wd_, gd, hd = dev(w), dev(g), dev(np.zeros(n, np.float32))
    rw, rh = f64(w), np.zeros(n)
    for t in range(5):
        lib.sg_op_adagrad(ptr(wd_), ptr(gd), ptr(hd), n, 0.01, 5e-4, 0.5, 1e-8, None)
        rw, rh = U.adagrad(rw, rh, f64(g), cfg, t, 0.5)
    assert normwise(host(wd_), rw) < 1e-6 and normwise(host(hd), rh) < 1e-6
    a, gg, hh = dev(np.zeros(4, np.float32)), dev(np.array([0.37, -2.5, 1e-3, 4.0], np.float32)), dev(np.zeros(4, np.float32))
    lib.sg_op_adagrad(ptr(a), ptr(gg), ptr(hh), 4, 0.1, 0.0, 1.0, 1e-8, None)
    assert np.allclose(host(a), -0.1 * np.sign([0.37, -2.5, 1e-3, 4.0]), atol=1e-6)
    w0, h0 = dev(w), dev(np.abs(w))
    lib.sg_op_adagrad(ptr(w0), ptr(dev(np.zeros(n, np.float32))), ptr(h0), n, 0.1, 0.0, 1.0, 1e-8, None)
    assert np.array_equal(host(w0), w) and np.array_equal(host(h0), np.abs(w))


def test_peer_sync_single_rank_vs_oracle_and_errors():
    """sg_peer_sync_* at K = 1 (no peers, no barriers): the fused exchange kernel
    is the Updater on the whole Param, s = grad_scale; bit-identical
    to sg_op_sgd_momentum (same FMA order) and within 1e-6 of the oracle.
    n not a multiple of 32 -> SG_ERR_PARTITION (header contract)."""
    from paper_1603_07846_b200 import net as PN
    cl = PN.Cluster(0, 1, 0)
    n = 32 * 4099
    w, g = r32(n, scale=0.05), r32(n, scale=0.01)
    cfgd = {"base_lr": 0.01, "momentum": 0.9, "weight_decay": 5e-4, "lr_policy": "fixed"}
    cfg = PN.updater_cfg(cfgd, grad_scale=0.5)
    h, gp, wp, vp = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
    lib.sg_peer_sync_create(cl.h, n, C.byref(h), C.byref(gp), C.byref(wp), C.byref(vp))

    class _A:
        def __init__(self, p):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (p, False), "version": 2}
    gd, wd_ = torch.as_tensor(_A(gp.value), device="cuda"), torch.as_tensor(_A(wp.value), device="cuda")
    gd.copy_(torch.from_numpy(g))
    wd_.copy_(torch.from_numpy(w))
    w2, v2, g2 = dev(w), dev(np.zeros(n, np.float32)), dev(g)
    rw, rv = f64(w), np.zeros(n)
    for t in range(3):
        lib.sg_peer_sync_step(h, C.byref(cfg), t, None)
        lib.sg_op_sgd_momentum(ptr(w2), ptr(g2), ptr(v2), n, 0.01, 0.9, 5e-4, 0.5, None)
        rw, rv = U.sgd_momentum(rw, rv, f64(g), cfgd, t, 0.5)
    torch.cuda.synchronize()
    got = wd_.cpu().numpy().copy()
    assert np.array_equal(got, host(w2))
    assert normwise(got, rw) < 1e-6
    lib.sg_peer_sync_destroy(h)
    with pytest.raises(lib.SingaError):
        lib.sg_peer_sync_create(cl.h, n + 1, C.byref(h), C.byref(gp), C.byref(wp), C.byref(vp))
    cl.close()
