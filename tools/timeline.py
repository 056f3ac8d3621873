"""Per-operation timeline of one graph-replayed training step (tools only).

Usage: python tools/timeline.py [config] [batch]
       torchrun --nproc-per-node K tools/timeline.py [config] [batch]   (rank 0 prints; fused exchange)
Prints every layer operation's start / end (us, relative to the step's first
operation) with the stream concurrency of the real step (sg_net_profile(2)), and
the same operations' solo durations (sg_net_profile(1), serialised).
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1603_07846_b200 import _lib as L  # noqa: E402
from paper_1603_07846_b200 import net as PN  # noqa: E402
from workloads import configs, generate  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cifar10"
rank, world, local = bench.env_rank()
torch.cuda.set_device(local)
nccl_id = None
if world > 1:
    import torch.distributed as dist
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    obj = [PN.Cluster.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    nccl_id = obj[0]
net_cfg = configs.get(cfg)
b = int(sys.argv[2]) if len(sys.argv) > 2 else bench.PER_GPU_BATCH[cfg] * world
n = PN.Net(PN.Cluster(rank, world, local, nccl_id), net_cfg, b)
n.set_updater(configs.UPDATERS[cfg])
n.set_params(bench.init_params(PN, n, net_cfg))
if world > 1:
    n.set_exchange("p2p")
info0 = n.layer_info[0]
x, lab = generate.batch(net_cfg, b, 0)
r0, rows = info0["local_offset"][0], info0["local_shape"][0]
x = torch.from_numpy(np.ascontiguousarray(x[r0:r0 + rows])).cuda()
ll = n.layer_info[-1]
lo, lr = n.layer_info[ll["src"]]["local_offset"][0], ll["local_shape"][0]
lab = torch.from_numpy(np.ascontiguousarray(lab[lo:lo + lr])).cuda()
loss = torch.zeros(1, device="cuda")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
info = n.layer_info
names = {}
for i, li in enumerate(info):
    for k, s in enumerate(("fwd", "wgrad", "dgrad", "update")):
        names[4 * i + k] = f'{li["name"]}.{s}'
ns = C.c_int32()
nslots = 4 * len(info)


def run(mode, reps=20):
    L.sg_net_profile(n.h, mode)
    n.enable_graph(True)
    ts = np.zeros(nslots)
    te = np.zeros(nslots)
    a = (C.c_double * nslots)()
    e = (C.c_double * nslots)()
    for t in range(reps + 3):
        flush.zero_()
        n.train_one_batch(t, x.data_ptr(), lab.data_ptr() if net_cfg["num_classes"] else None, loss.data_ptr(), sp)
        L.sg_net_op_timeline(n.h, a, e, nslots, C.byref(ns))
        if t >= 3:
            ts += np.array(a[:nslots])
            te += np.array(e[:nslots])
    L.sg_net_profile(n.h, 0)
    n.enable_graph(False)
    return ts / reps, te / reps


cs, ce = run(2)
ss, se = run(1)
if rank != 0:
    sys.exit(0)
order = sorted([s for s in range(nslots) if cs[s] >= 0], key=lambda s: cs[s])
print(f"{'op':<16}{'start':>8}{'end':>8}{'dur':>8}{'solo':>8}   (us; concurrent step vs serialised)")
for s in order:
    print(f"{names[s]:<16}{cs[s]*1e3:8.1f}{ce[s]*1e3:8.1f}{(ce[s]-cs[s])*1e3:8.1f}{(se[s]-ss[s])*1e3:8.1f}")
print(f"step span {max(ce[s] for s in order)*1e3:.1f} us; serialised sum {sum(se[s]-ss[s] for s in order)*1e3:.1f} us")
