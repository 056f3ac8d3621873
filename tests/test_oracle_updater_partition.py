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
