"""CTA-0 timeline of the 4-channel first-layer forward kernel (trace build variant).
Usage: python -m paper_1603_07846_b200.build --variant trace -D SG_GEMM_TRACE
       SG_LIB=build/trace/libsinga_b200.so python tools/img4f_trace.py [N]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1603_07846_b200 import _lib as L  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 128
d = L.ConvDesc(N, 32, 32, 4, 32, 5, 5, 1, 2)
x = torch.randn(N, 32, 32, 4, device="cuda")
Wt = torch.randn(32, 5, 5, 4, device="cuda") * 0.05
b = torch.randn(32, device="cuda")
y = torch.empty(N, 32, 32, 32, device="cuda")
for _ in range(4):
    assert L.sg_op_conv_forward(C.byref(d), x.data_ptr(), Wt.data_ptr(), b.data_ptr(), y.data_ptr(), None) == 0
torch.cuda.synchronize()
buf = (C.c_longlong * (6 * 64))()
assert L.lib.sg_debug_img_trace(buf) == 0
t = np.frombuffer(buf, dtype=np.int64).reshape(6, 64).astype(np.float64)
t0 = t[5, 0]
for r, name in [(3, "image ready"), (2, "mma issued"), (4, "epilogue"), (0, "done")]:
    v = t[r][t[r] > 0] - t0
    print(f"{name:12s} " + " ".join(f"{x:6.0f}" for x in v[:8]))
