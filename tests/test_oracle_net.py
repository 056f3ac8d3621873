"""Pins for oracle/net.py: end-to-end finite differences, K-invariance
(S:434), hybrid-partition transparency, the paper's AlexNet
parameter / computation shares and the fc6 size."""

import copy
import json
import os

import numpy as np
import pytest

from oracle import net as N
from workloads import configs, generate

PV = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))
UPD = {"base_lr": 0.05, "momentum": 0.9, "weight_decay": 1e-3, "lr_policy": "fixed"}

TINY_MLP = {"name": "tiny_mlp", "input": {"d": 6}, "num_classes": 3, "layers": [
    {"name": "ip1", "kind": "ip", "num_output": 5, "partition_dim": 0},
    {"name": "sig1", "kind": "sigmoid"},
    {"name": "ip2", "kind": "ip", "num_output": 4},
    {"name": "relu2", "kind": "relu"},
    {"name": "ip3", "kind": "ip", "num_output": 3},
    {"name": "loss", "kind": "softmax_ce"}]}

TINY_AE = {"name": "tiny_ae", "input": {"d": 8}, "num_classes": 0, "layers": [
    {"name": "ip1", "kind": "ip", "num_output": 6, "partition_dim": 1},
    {"name": "sig1", "kind": "sigmoid"},
    {"name": "ip2", "kind": "ip", "num_output": 2},
    {"name": "ip3", "kind": "ip", "num_output": 8},
    {"name": "loss", "kind": "euclidean"}]}

TINY_HYBRID = {"name": "tiny_hybrid", "input": {"c": 3, "h": 9, "w": 9}, "num_classes": 4, "layers": [
    {"name": "conv1", "kind": "conv", "num_output": 4, "kernel": 3, "stride": 2, "pad": 1, "partition_dim": 0},
    {"name": "relu1", "kind": "relu"},
    {"name": "pool1", "kind": "pool_max", "kernel": 3, "stride": 2, "pad": 0},
    {"name": "fc1", "kind": "ip", "num_output": 8, "partition_dim": 1},
    {"name": "relu2", "kind": "relu"},
    {"name": "fc2", "kind": "ip", "num_output": 4},
    {"name": "loss", "kind": "softmax_ce", "partition_dim": 0}]}


def make(net, b, t=0):
    params = generate.init_params(N.param_specs(net))
    rng = np.random.default_rng(5)
    # non-zero biases so that bias paths are exercised
    for k in params:
        if k.endswith("/b"):
            params[k] = rng.standard_normal(params[k].shape).astype(np.float32) * 0.1
    x, lab = generate.batch(net, b, t)
    return params, x, lab


def loss_of(net, params, x, lab):
    p64 = {k: np.asarray(v, np.float64) for k, v in params.items()}
    b = x.shape[0]
    _, losses = N.forward(net, p64, np.asarray(x, np.float64), lab, b)
    return float(np.sum(losses)) / b


@pytest.mark.parametrize("netname", ["tiny_mlp", "tiny_ae", "tiny_conv", "tiny_hybrid"])
def test_end_to_end_finite_difference(netname):
    net = {"tiny_mlp": TINY_MLP, "tiny_ae": TINY_AE, "tiny_conv": configs.TINY_CONV,
           "tiny_hybrid": TINY_HYBRID}[netname]
    b = 4
    params, x, lab = make(net, b)
    vel = {k: np.zeros_like(v, np.float64) for k, v in params.items()}
    out = N.train_one_batch(net, params, vel, x, lab, 0, 1, UPD)
    p64 = {k: np.asarray(v, np.float64) for k, v in params.items()}
    rng = np.random.default_rng(9)
    for name, g in out["grads"].items():
        flat = p64[name].reshape(-1)
        idx = rng.choice(flat.size, size=min(flat.size, 12), replace=False)
        for i in idx:
            old = flat[i]
            flat[i] = old + 1e-5
            fp = loss_of(net, p64, x, lab)
            flat[i] = old - 1e-5
            fm = loss_of(net, p64, x, lab)
            flat[i] = old
            fd = (fp - fm) / 2e-5
            an = out["grad_scale"] * g.reshape(-1)[i]
            assert abs(fd - an) <= 1e-6 * max(abs(fd), 1e-4), (name, i, fd, an)


@pytest.mark.parametrize("netname", ["tiny_mlp", "tiny_conv"])
def test_k_invariance(netname):
    net = {"tiny_mlp": TINY_MLP, "tiny_conv": configs.TINY_CONV}[netname]
    b = 16
    params, x, lab = make(net, b)
    vel = {k: np.zeros_like(v, np.float64) for k, v in params.items()}
    ref = None
    for K in (1, 2, 4, 8):
        p, v = dict(params), dict(vel)
        losses = []
        for t in range(3):
            xb, lb = generate.batch(net, b, t)
            out = N.train_one_batch(net, p, v, xb, lb, t, K, UPD)
            p, v = out["params"], out["vel"]
            losses.append(out["loss"])
        if ref is None:
            ref = (p, losses)
        else:
            for k in p:
                assert np.max(np.abs(p[k] - ref[0][k])) < 1e-12
            assert np.max(np.abs(np.array(losses) - ref[1])) < 1e-12


def test_k_requires_divisible_batch():
    params, x, lab = make(TINY_MLP, 6)
    vel = {k: np.zeros_like(v, np.float64) for k, v in params.items()}
    with pytest.raises(ValueError):
        N.train_one_batch(TINY_MLP, params, vel, x, lab, 0, 4, UPD)


@pytest.mark.parametrize("netname,K", [("tiny_hybrid", 2), ("tiny_hybrid", 4), ("tiny_ae", 2), ("tiny_mlp_dim1", 2)])
def test_hybrid_partition_transparency(netname, K):
    if netname == "tiny_mlp_dim1":
        net = configs.with_partition(TINY_MLP, {"ip1": 1, "loss": 0})
        net["layers"][0]["partition_dim"] = 0
        net = configs.with_partition(net, {"ip2": 1})
    else:
        net = {"tiny_hybrid": TINY_HYBRID, "tiny_ae": TINY_AE}[netname]
    b = 8
    params, x, lab = make(net, b)
    vel = {k: np.zeros_like(v, np.float64) for k, v in params.items()}
    ref = N.train_one_batch(net, params, vel, x, lab, 0, K, UPD)
    part = N.train_one_batch_partitioned(net, params, vel, x, lab, 0, K, UPD)
    assert abs(ref["loss"] - part["loss"]) < 1e-12
    for k in ref["params"]:
        assert np.max(np.abs(ref["grads"][k] - part["grads"][k])) < 1e-12, k
        assert np.max(np.abs(ref["params"][k] - part["params"][k])) < 1e-12, k


def test_alexnet_shares_match_paper():
    w = N.work(configs.alexnet())
    conv = [r for r in w if r["kind"] == "conv"]
    fc = [r for r in w if r["kind"] == "ip"]
    P = sum(r["params"] for r in w)
    F = sum(r["fwd_macs"] for r in w)
    cp = sum(r["params"] for r in conv) / P
    cf = sum(r["fwd_macs"] for r in conv) / F
    pv = PV["alexnet_conv_param_share"]
    assert abs(cp - pv["param_share_approx"]) < pv["param_share_tolerance"]
    assert pv["compute_share_range"][0] <= cf <= pv["compute_share_range"][1]
    pv = PV["alexnet_fc_share"]
    assert abs(sum(r["params"] for r in fc) / P - pv["param_share_approx"]) < pv["param_share_tolerance"]
    assert pv["compute_share_range"][0] <= 1 - cf <= pv["compute_share_range"][1]
    assert P == 61100840          # SURVEY §8.0 C3 parameter count


def test_fc6_177_million():
    pv = PV["fc6_params"]
    w = {r["name"]: r for r in N.work(configs.alexnet(pool5=False))}
    fc6 = w["fc6"]["params"] - pv["d_h"]           # weights only
    assert fc6 == 13 * 13 * 256 * 4096
    assert abs(fc6 - pv["approx"]) / pv["approx"] < pv["rel_tolerance"]
    # cost model: model-parallel cost b*d_v with b = K*128, d_v = 4096
    assert 8 * 128 * 4096 == PV["cost_model"]["model_parallel_cost"]
    assert fc6 > PV["cost_model"]["model_parallel_cost"]


def test_config_shapes():
    info, params = N.setup(configs.CIFAR10)
    assert [i["out_shape"] for i in info if i["kind"] == "pool_max" or i["kind"] == "pool_avg"] == \
        [(16, 16, 32), (8, 8, 32), (4, 4, 64)]
    assert sum(int(np.prod(p[1])) for p in params) == 89578
    _, params = N.setup(configs.MLP)
    assert sum(int(np.prod(p[1])) for p in params) == 203530
    _, params = N.setup(configs.AE)
    assert sum(int(np.prod(p[1])) for p in params) == 2823286
    _, params = N.setup(configs.AE_WIDE)
    assert sum(int(np.prod(p[1])) for p in params) == 92636800


@pytest.mark.parametrize("updater", ["sgd_momentum", "adagrad"])
def test_partition_transparency_with_multipliers_and_adagrad(updater):
    """The partitioned data flow applies the per-layer lr / wd multipliers (reading
    A23) and the configured Updater exactly like the unpartitioned step; a layer
    with lr_scale 0 keeps its Params."""
    net = copy.deepcopy(TINY_HYBRID)
    net["layers"][0]["lr_scale"] = 0.0
    for l in net["layers"]:
        if l["kind"] == "ip":
            l["lr_scale"], l["wd_scale"] = 2.0, 0.5
            break
    upd = dict(UPD, type=updater, eps=1e-8)
    b, K = 8, 2
    params, x, lab = make(net, b)
    vel = {k: np.zeros_like(v, np.float64) for k, v in params.items()}
    ref = N.train_one_batch(net, params, vel, x, lab, 0, K, upd)
    part = N.train_one_batch_partitioned(net, params, vel, x, lab, 0, K, upd)
    first = net["layers"][0]["name"]
    for k in ref["params"]:
        assert np.max(np.abs(ref["params"][k] - part["params"][k])) < 1e-12, k
        assert np.max(np.abs(ref["vel"][k] - part["vel"][k])) < 1e-12, k
        if k.startswith(first + "/"):
            assert np.array_equal(ref["params"][k], np.asarray(params[k], np.float64)), k
