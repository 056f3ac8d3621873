"""CPU tests of the C ABI library (no GPU): it loads, exports every symbol the
header declares, and its host-side planner (partition maps, shapes, connection
layers, Param table, server shard map) agrees BIT-EXACTLY with the oracle's
independent implementation."""

import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle import net as ON
from oracle import partition as OP
from workloads import configs

L = pytest.importorskip("paper_1603_07846_b200._lib")
from paper_1603_07846_b200 import net as PN  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "singa_b200.h")).read()
    names = re.findall(r"SG_API\s+[\w\s\*]*?\b(sg_\w+)\s*\(", hdr)
    assert len(names) >= 50
    for n in names:
        assert hasattr(L.lib, n), n
    assert L.sg_abi_version() == 2


def test_partition_range_matches_oracle():
    off, ln = C.c_int64(), C.c_int64()
    for E in range(1, 80):
        for K in range(1, min(E, 9) + 1):
            for i in range(K):
                L.sg_partition_range(E, K, i, C.byref(off), C.byref(ln))
                assert (off.value, ln.value) == OP.partition_range(E, K, i)
    with pytest.raises(L.SingaError) as e:
        L.sg_partition_range(3, 4, 0, C.byref(off), C.byref(ln))
    assert e.value.name == "SG_ERR_PARTITION"
    with pytest.raises(L.SingaError) as e:
        L.sg_partition_range(3, 2, 2, C.byref(off), C.byref(ln))
    assert e.value.name == "SG_ERR_INVALID_ARG"


def user_layers(plan):
    return [l for l in plan.layers() if not l["is_connection"] and l["kind"] != "input"]


@pytest.mark.parametrize("name", ["mlp", "cifar10", "alexnet", "ae", "ae_wide", "tiny_conv"])
def test_plan_shapes_and_params_match_oracle(name):
    net = configs.get(name)
    b = configs.BATCH[name]
    plan = PN.Plan(net, b)
    info, params = ON.setup(net)
    ul = user_layers(plan)
    assert [l["name"] for l in ul] == [l["name"] for l in net["layers"]]
    for l, o in zip(ul, info):
        if l["kind"] in ("softmax_ce", "euclidean"):
            continue
        shp = o["out_shape"]
        if len(shp) == 3:
            assert l["global_shape"] == (b,) + tuple(shp), l["name"]
        else:
            assert l["global_shape"][:2] == (b, shp[0]), l["name"]
    pp = plan.params()
    assert [p["name"] for p in pp] == [p[0] for p in params]
    for p, o in zip(pp, params):
        shp = o[1]
        if len(shp) == 4:      # conv W [Co][R][S][C] reported as rows=Co, cols=R*S*C
            assert (p["rows"], p["cols"]) == (shp[0], shp[1] * shp[2] * shp[3])
        elif len(shp) == 2:
            assert (p["rows"], p["cols"]) == shp
        else:
            assert (p["rows"], p["cols"]) == (1, shp[0])
        assert p["split_dim"] == -1 and p["local_cols"] == p["cols"]


@pytest.mark.parametrize("K", [2, 4, 8])
def test_alexnet_hybrid_plan(K):
    net = configs.alexnet(hybrid=True)
    b = 256
    for rank in range(K):
        plan = PN.Plan(net, b, rank, K)
        ls = plan.layers()
        names = [l["name"] for l in ls]
        # connection layers exactly at the partitioning changes
        conn = [l["name"] for l in ls if l["is_connection"]]
        assert conn == ["pool5.concat_rows", "relu6.concat_cols", "relu7.concat_cols", "fc8.slice"]
        assert names.index("pool5.concat_rows") == names.index("fc6") - 1
        roff, rlen = OP.partition_range(b, K, rank)
        for l in ls:
            if l["name"].startswith(("conv", "relu1", "relu2", "relu3", "relu4", "relu5", "pool")) and \
                    not l["is_connection"]:
                assert (l["local_offset"][0], l["local_shape"][0]) == (roff, rlen), l["name"]
        for fc, dh in (("fc6", 4096), ("fc7", 4096), ("fc8", 1000)):
            l = ls[names.index(fc)]
            coff, clen = OP.partition_range(dh, K, rank)
            assert l["local_shape"][:2] == (b, clen) and l["local_offset"][1] == coff
            assert l["ld"] % 4 == 0 and l["ld"] >= clen
        sl = ls[names.index("fc8.slice")]
        assert sl["local_shape"][:2] == (rlen, 1000) and sl["nblocks"] == K
        pp = {p["name"]: p for p in plan.params()}
        for fc in ("fc6", "fc7", "fc8"):
            assert pp[fc + "/W"]["split_dim"] == 1 and pp[fc + "/W"]["bucket"] == -1
        assert pp["conv1/W"]["split_dim"] == -1 and pp["conv1/W"]["bucket"] == 0


@pytest.mark.parametrize("name,K", [("cifar10", 1), ("cifar10", 2), ("cifar10", 3), ("cifar10", 8),
                                    ("alexnet", 4), ("mlp", 1), ("tiny_conv", 2)])
def test_shard_map_matches_oracle(name, K):
    net = configs.get(name)
    b = 24 if name == "tiny_conv" else configs.BATCH[name]
    if b % K:
        b = K * 16
    plan = PN.Plan(net, b, 0, K)
    pp = plan.params()
    sizes = plan.buckets()
    got = plan.shard_map()
    expect = []
    for bk in range(len(sizes)):
        members = [(i, p) for i, p in enumerate(pp) if p["bucket"] == bk]
        padded, m = OP.bucket_shard_map([p["internal_size"] for _, p in members], K)
        assert padded == sizes[bk]
        for (pi, owner, poff, boff, ln) in m:
            expect.append((members[pi][0], bk, owner, poff, boff, ln))
    assert got == expect
    # internal sizes: user sizes except the documented paddings (reading: first-conv
    # channels 3 -> 4, inner-product output columns to a multiple of 4)
    for p in pp:
        user = p["rows"] * p["local_cols"]
        assert p["internal_size"] >= user


@pytest.mark.parametrize("mutate,code", [
    (lambda n: n["layers"][-1].__setitem__("partition_dim", 1), "SG_ERR_CONFIG"),           # softmax dim 1
    (lambda n: n["layers"][0].__setitem__("partition_dim", 1), "SG_ERR_CONFIG"),            # conv dim 1
    (lambda n: n["layers"].insert(3, {"name": "lossx", "kind": "softmax_ce"}), "SG_ERR_CONFIG"),
    (lambda n: n["layers"].pop(), "SG_ERR_CONFIG"),                                          # no loss
    (lambda n: n["layers"][1].__setitem__("kernel", 40), "SG_ERR_CONFIG"),
])
def test_plan_errors(mutate, code):
    net = configs.get("cifar10")
    mutate(net)
    with pytest.raises(L.SingaError) as e:
        PN.Plan(net, 128, 0, 2)
    assert e.value.name == code


def test_partition_errors():
    with pytest.raises(L.SingaError) as e:
        PN.Plan(configs.get("cifar10"), 130, 0, 4)        # b % K != 0 (reading A2)
    assert e.value.name == "SG_ERR_PARTITION"
    net = configs.autoencoder([784, 1002, 784], "odd")
    with pytest.raises(L.SingaError) as e:
        PN.Plan(net, 8, 0, 4)                             # K does not divide d_h
    assert e.value.name == "SG_ERR_PARTITION"
    PN.Plan(net, 8, 0, 2)


def test_async_topology_unsupported():
    cfg = L.ClusterCfg()
    cfg.rank, cfg.world_size, cfg.device = 0, 2, 0
    cfg.nworker_groups, cfg.workers_per_group, cfg.nserver_groups, cfg.servers_per_group = 2, 1, 1, 2
    h = C.c_void_p()
    with pytest.raises(L.SingaError) as e:
        L.sg_cluster_create(C.byref(cfg), C.byref(h))
    assert e.value.name == "SG_ERR_UNSUPPORTED"


def test_ae_feature_partition_plan():
    net = configs.get("ae_wide")
    for K in (2, 4, 8):
        for rank in range(K):
            plan = PN.Plan(net, 256, rank, K)
            ls = plan.layers()
            assert ls[0]["kind"] == "input" and ls[0]["local_shape"][:2] == (256, 784)   # replicated input
            for l in ls:
                if l["kind"] == "ip":
                    dh = l["global_shape"][1]
                    assert (l["local_offset"][1], l["local_shape"][1]) == OP.partition_range(dh, K, rank)
            assert sum(1 for l in ls if l["is_connection"]) == 7       # Concat(dim 1) before ip2..ip8


@pytest.mark.parametrize("name,K,params", [("cifar10", 2, 89_578),
                                           ("alexnet", 2, 23_296 + 307_392 + 663_936 + 884_992 + 590_080),
                                           ("ae_wide", 2, 0)])
def test_bench_grad_sync_bytes(name, K, params):
    """bench.py's grad_sync object counts the fp32 bytes of every dim-0 layer's
    bucket (a16 / a18); dim-1 FC slices (AlexNet fc6-fc8, the all-FC
    auto-encoder) update owner-locally and move no Param bytes."""
    import bench
    net = configs.alexnet(hybrid=True) if name == "alexnet" else configs.get(name)
    plan = PN.Plan(net, 256, 0, K)
    got = bench.grad_sync_bytes(net, plan.layers(), K)
    assert sum(got.values()) == 4 * params
    assert bench.grad_sync_bytes(net, plan.layers(), 1) == {}


@pytest.mark.parametrize("name,K,data,grad", [
    ("cifar10", 1, {"input", "norm1", "norm2", "norm3"}, {"conv1", "conv2", "conv3", "ip1"}),
    ("mlp", 1, {"input", "sig1"}, {"ip1", "ip2"}),
    ("alexnet", 2,
     {"input", "pool1", "pool2", "relu3", "relu4", "pool5", "pool5.concat_rows", "relu6", "relu6.concat_cols",
      "relu7", "relu7.concat_cols"},
     {"conv1", "conv2", "conv3", "conv4", "conv5", "fc6", "fc7", "fc8", "fc8.slice"}),
])
def test_tf32_operand_flags(name, K, data, grad):
    """Reading A19: a blob is stored TF32-rounded exactly when a tensor-core GEMM
    reads it -- the input of every conv / inner product (through an all-gather
    Concat, which moves values unchanged), and the gradient w.r.t. a conv / IP
    output (through the loss Slice's all-to-all)."""
    net = configs.get(name) if name != "alexnet" else configs.alexnet(hybrid=True)
    plan = PN.Plan(net, configs.BATCH[name], rank=0, world=K)
    ls = plan.layers()
    assert {l["name"] for l in ls if l["tf32_data"]} == data
    assert {l["name"] for l in ls if l["tf32_grad"]} == grad
