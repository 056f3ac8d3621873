"""World-size-2 (and 4) CPU tests of the multi-rank host logic over gloo.

Each rank builds its own plan through the C ABI (sg_plan_create(rank, K): no
device needed) and the ranks exchange what they planned: the shard maps must be
identical, row blocks of dim-0 layers and column blocks of dim-1 layers must
tile the global extents exactly once, every Param element must have exactly one
owner; plus the bench's max-over-ranks timing reduction.
"""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import partition as OP
from workloads import configs


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1603_07846_b200 import net as PN
        out = {}
        for name, b in (("cifar10", 128), ("alexnet", 256), ("ae_wide", 256), ("mlp", 64)):
            plan = PN.Plan(configs.get(name), b, rank, world)
            out[name] = {"layers": plan.layers(), "params": plan.params(), "shards": plan.shard_map(),
                         "buckets": plan.buckets()}
        gathered = [None] * world
        dist.all_gather_object(gathered, out)
        # max-over-ranks timing (bench.py): each rank reports its own time
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            q.put(("ok", gathered, float(t.item())))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put(("err", repr(e), 0.0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_multi_rank_plans_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    status, gathered, tmax = q.get(timeout=300)
    for p in procs:
        p.join(60)
    assert status == "ok", gathered
    assert tmax == float(world)
    for name in gathered[0]:
        plans = [g[name] for g in gathered]
        # shard maps and bucket sizes are global facts: identical on every rank
        assert all(p["shards"] == plans[0]["shards"] for p in plans)
        assert all(p["buckets"] == plans[0]["buckets"] for p in plans)
        # each bucket element owned exactly once, shards equal-sized
        for bk, size in enumerate(plans[0]["buckets"]):
            rs = sorted((r[4], r[5], r[2]) for r in plans[0]["shards"] if r[1] == bk)
            pos = 0
            for off, ln, owner in rs:
                assert off == pos and owner == off // (size // world)
                pos += ln
        # layer partitions tile the global extents
        nl = len(plans[0]["layers"])
        assert all(len(p["layers"]) == nl for p in plans)
        for i in range(nl):
            ls = [p["layers"][i] for p in plans]
            l0 = ls[0]
            if l0["kind"] in ("softmax_ce", "euclidean"):
                continue
            if l0["partition_dim"] == 0 and l0["local_shape"][0] < l0["global_shape"][0]:
                blocks = sorted((l["local_offset"][0], l["local_shape"][0]) for l in ls)
                assert blocks == [OP.partition_range(l0["global_shape"][0], world, k) for k in range(world)]
            if l0["kind"] == "ip" and l0["partition_dim"] == 1:
                blocks = sorted((l["local_offset"][1], l["local_shape"][1]) for l in ls)
                assert blocks == [OP.partition_range(l0["global_shape"][1], world, k) for k in range(world)]
        # split Params: column slices tile the user columns
        for j, p0 in enumerate(plans[0]["params"]):
            if p0["split_dim"] == 1:
                cols = sorted((p["params"][j]["local_col_off"], p["params"][j]["local_cols"]) for p in plans)
                assert cols == [OP.partition_range(p0["cols"], world, k) for k in range(world)]
