"""Per-operation timeline of one graph-replayed training step (1 GPU, tools only).

Usage: python tools/timeline.py [config] [batch]
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
torch.cuda.set_device(0)
net_cfg = configs.get(cfg)
b = int(sys.argv[2]) if len(sys.argv) > 2 else bench.PER_GPU_BATCH[cfg]
n = PN.Net(PN.Cluster(0, 1, 0, None), net_cfg, b)
n.set_updater(configs.UPDATERS[cfg])
n.set_params(bench.init_params(PN, n, net_cfg))
x, lab = generate.batch(net_cfg, b, 0)
x = torch.from_numpy(np.ascontiguousarray(x)).cuda()
lab = torch.from_numpy(np.ascontiguousarray(lab)).cuda()
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
order = sorted([s for s in range(nslots) if cs[s] >= 0], key=lambda s: cs[s])
print(f"{'op':<16}{'start':>8}{'end':>8}{'dur':>8}{'solo':>8}   (us; concurrent step vs serialised)")
for s in order:
    print(f"{names[s]:<16}{cs[s]*1e3:8.1f}{ce[s]*1e3:8.1f}{(ce[s]-cs[s])*1e3:8.1f}{(se[s]-ss[s])*1e3:8.1f}")
print(f"step span {max(ce[s] for s in order)*1e3:.1f} us; serialised sum {sum(se[s]-ss[s] for s in order)*1e3:.1f} us")
