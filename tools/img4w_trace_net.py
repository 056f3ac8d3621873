"""CTA-0 timeline of the fused pool-backward + conv1 weight-gradient kernel inside
the CIFAR-10 step (trace build variant).
Usage: SG_LIB=build/trace/libsinga_b200.so python tools/img4w_trace_net.py"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import net as ON  # noqa: E402
from paper_1603_07846_b200 import _lib as L  # noqa: E402
from paper_1603_07846_b200 import net as PN  # noqa: E402
from workloads import configs, generate  # noqa: E402

net = configs.get("cifar10")
b = 128
cl = PN.Cluster(0, 1, 0)
n = PN.Net(cl, net, b)
n.set_updater(configs.UPDATERS["cifar10"])
n.set_params(generate.init_params(ON.param_specs(net)))
n.enable_graph(True)
x, lab = generate.batch(net, b, 0)
xd, ld = torch.from_numpy(x).cuda(), torch.from_numpy(lab).cuda()
loss = torch.zeros(1, device="cuda")
for t in range(5):
    n.train_one_batch(t, xd.data_ptr(), ld.data_ptr(), loss.data_ptr())
torch.cuda.synchronize()
buf = (C.c_longlong * (6 * 64))()
assert L.lib.sg_debug_img_trace(buf) == 0
t = np.frombuffer(buf, dtype=np.int64).reshape(6, 64).astype(np.float64)
t0 = t[5, 0]
for r, name in enumerate(["pool/dy/img", "A built", "mma issued", "epilogue"]):
    if r == 0:
        print("row0 raw", [int(x - t0) if x > 0 else 0 for x in t[0][:12]])
    v = t[r][t[r] > 0] - t0
    print(f"{name:12s} " + " ".join(f"{x:6.0f}" for x in v[:34]), flush=True)
