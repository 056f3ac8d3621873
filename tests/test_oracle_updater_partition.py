"""Pins for oracle/updater.py and oracle/partition.py (SPEC values, closed forms)."""

import json
import os

import numpy as np
import pytest

from oracle import partition as P
from oracle import updater as U

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def cfg(lr, mu=0.0, wd=0.0, **kw):
    d = {"base_lr": lr, "momentum": mu, "weight_decay": wd, "lr_policy": "fixed"}
    d.update(kw)
    return d


def test_sgd_spec_values():
    g = GOLD["sgd_hand"]
    w, v = U.sgd_momentum(np.array([g["w"]]), np.zeros(1), np.array([g["g"]]), cfg(g["lr"]), 0, 1.0)
    assert abs(w[0] - g["w_new"]) < 1e-15
    g = GOLD["sgd_zero_grad"]
    w, v = U.sgd_momentum(np.array([g["w"]]), np.zeros(1), np.array([g["g"]]), cfg(g["lr"]), 0, 1.0)
    assert w[0] == g["w_new"]


def test_weight_decay_reduces_to_spec_form():
    # mu = 0: value <- value - alpha (grad + wd value)
    w0, g0 = 0.8, 0.3
    w, _ = U.sgd_momentum(np.array([w0]), np.zeros(1), np.array([g0]), cfg(0.1, wd=0.01), 0, 1.0)
    assert abs(w[0] - (w0 - 0.1 * (g0 + 0.01 * w0))) < 1e-16


def test_lr_step_schedule():
    g = GOLD["lr_step"]
    c = cfg(0.4, lr_policy="step", gamma=g["gamma"], step_size=g["step_size"])
    assert U.learning_rate(c, g["iteration"]) == pytest.approx(g["ratio"] * 0.4, abs=0)


def test_momentum_closed_form():
    # constant g, wd = 0, fixed eta: w_t = w0 - eta g [t/(1-mu) - mu(1-mu^t)/(1-mu)^2]
    eta, mu, gg, w0 = 0.1, 0.9, 0.5, 1.0
    w, v = np.array([w0]), np.zeros(1)
    c = cfg(eta, mu)
    for t in range(1, 38):
        w, v = U.sgd_momentum(w, v, np.array([gg]), c, t, 1.0)
        closed = w0 - eta * gg * (t / (1 - mu) - mu * (1 - mu ** t) / (1 - mu) ** 2)
        assert abs(w[0] - closed) < 1e-12


def test_zero_lr_constant():
    w0 = np.random.default_rng(0).standard_normal(100)
    w, v = w0.copy(), np.zeros(100)
    for t in range(5):
        w, v = U.sgd_momentum(w, v, np.ones(100), cfg(0.0, 0.9, 0.01), t, 0.5)
    assert np.array_equal(w, w0)


def test_grad_scale():
    w, _ = U.sgd_momentum(np.zeros(1), np.zeros(1), np.array([4.0]), cfg(1.0), 0, 0.25)
    assert w[0] == -1.0


def test_lr_wd_multipliers():
    """Per-Param multipliers (reading A23): lr_scale = the base rate scaled, wd_scale =
    the decay scaled, exactly (same arithmetic order)."""
    rng = np.random.default_rng(3)
    w0, g0 = rng.standard_normal(50), rng.standard_normal(50)
    v0 = rng.standard_normal(50) * 0.1
    a = U.sgd_momentum(w0, v0, g0, cfg(0.05, 0.9, 0.01), 0, 0.5, lr_scale=2.0, wd_scale=0.5)
    b = U.sgd_momentum(w0, v0, g0, cfg(0.1, 0.9, 0.005), 0, 0.5)
    assert np.allclose(a[0], b[0], rtol=0, atol=1e-15) and np.allclose(a[1], b[1], rtol=0, atol=1e-15)
    w, v = U.sgd_momentum(w0, np.zeros(50), g0, cfg(0.05, 0.9, 0.01), 0, 1.0, lr_scale=0.0)
    assert np.array_equal(w, w0)                       # lr_scale 0 freezes the Param


def test_adagrad_first_step_is_sign():
    """first update with gradient g, alpha 0.1, eps 1e-8 -> step -0.1 g / (|g| + eps) ~ -0.1 sign(g)."""
    g = np.array([0.37, -2.5, 1e-3])
    w, h = U.adagrad(np.zeros(3), np.zeros(3), g, cfg(0.1, eps=1e-8), 0, 1.0)
    assert np.allclose(w, -0.1 * g / (np.abs(g) + 1e-8), rtol=0, atol=1e-17)
    assert np.allclose(w, -0.1 * np.sign(g), atol=1e-6) and np.array_equal(h, g * g)


def test_adagrad_constant_gradient_closed_form():
    """constant gradient 1.0 -> cumulative displacement -alpha * sum_{i<=t} 1/(sqrt(i) + eps)."""
    w, h = np.zeros(1), np.zeros(1)
    alpha, eps = 0.05, 1e-8
    for t in range(1, 60):
        w, h = U.adagrad(w, h, np.ones(1), cfg(alpha, eps=eps), t, 1.0)
        closed = -alpha * sum(1.0 / (np.sqrt(i) + eps) for i in range(1, t + 1))
        assert abs(w[0] - closed) < 1e-13 and h[0] == t


def test_adagrad_zero_gradient_unchanged():
    """gradient 0 everywhere (no decay) -> value and accumulator unchanged."""
    w0, h0 = np.random.default_rng(1).standard_normal(20), np.abs(np.random.default_rng(2).standard_normal(20))
    w, h = U.adagrad(w0, h0, np.zeros(20), cfg(0.3, eps=1e-8), 0, 1.0)
    assert np.array_equal(w, w0) and np.array_equal(h, h0)


# ------------------------------------------------------------ partition -----
@pytest.mark.parametrize("key", ["slice_rows", "slice_cols", "slice_remainder"])
def test_partition_spec(key):
    g = GOLD[key]
    lens = [P.partition_range(g["extent"], g["parts"], i)[1] for i in range(g["parts"])]
    assert lens == g["lens"]
    if "offs" in g:
        assert [P.partition_range(g["extent"], g["parts"], i)[0] for i in range(g["parts"])] == g["offs"]


def test_partition_exhaustive():
    for E in range(1, 70):
        for K in range(1, min(E, 9) + 1):
            rs = [P.partition_range(E, K, i) for i in range(K)]
            assert rs[0][0] == 0 and sum(r[1] for r in rs) == E
            assert all(rs[i][0] + rs[i][1] == rs[i + 1][0] for i in range(K - 1))
            assert max(r[1] for r in rs) - min(r[1] for r in rs) <= 1
            assert [r[1] for r in rs] == sorted([r[1] for r in rs], reverse=True)
    with pytest.raises(ValueError):
        P.partition_range(3, 4, 0)


def test_slice_concat_round_trip():
    a = np.random.default_rng(3).standard_normal((7, 5))
    for d in (0, 1):
        for k in (1, 2, 3):
            assert np.array_equal(P.concat_blobs(P.slice_blob(a, d, k), d), a)
    W = np.zeros((784, 50))
    parts = P.slice_blob(W, 1, 2)
    assert [p.shape for p in parts] == [(784, 25), (784, 25)]


def test_bucket_shard_map():
    for sizes in ([2400, 32], [75 * 32, 32, 800 * 32, 32], [1], [31, 1, 64]):
        for K in range(1, 9):
            padded, m = P.bucket_shard_map(sizes, K)
            assert padded % (32 * K) == 0 and padded >= sum(sizes) and padded - sum(sizes) < 32 * K
            # every element of every param covered exactly once, in order
            cover = {p: 0 for p in range(len(sizes))}
            boff = 0
            for (p, owner, poff, bo, ln) in m:
                assert poff == cover[p] and bo == boff
                assert owner == bo // (padded // K) == (bo + ln - 1) // (padded // K)
                cover[p] += ln
                boff += ln
            assert all(cover[p] == sizes[p] for p in cover)
            # each param split into at most K slices
            for p in range(len(sizes)):
                assert sum(1 for r in m if r[0] == p) <= K
