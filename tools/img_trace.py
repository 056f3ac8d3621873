"""CTA-0 timeline of the resident-image convolution (trace build variant).
Usage: SG_LIB=build/trace/libsinga_b200.so img_trace.py N H C Co R p [fwd|dgrad]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1603_07846_b200 import _lib as L  # noqa: E402

N, H, Ci, Co, R, p = (int(v) for v in sys.argv[1:7])
which = sys.argv[7] if len(sys.argv) > 7 else "fwd"
d = L.ConvDesc(N, H, H, Ci, Co, R, R, 1, p)
Ho, Wo = C.c_int32(), C.c_int32()
L.sg_conv_out_shape(C.byref(d), C.byref(Ho), C.byref(Wo))
x = torch.randn(N, H, H, Ci, device="cuda")
Wt = torch.randn(Co, R, R, Ci, device="cuda") * 0.05
b = torch.zeros(Co, device="cuda")
y = torch.empty(N, Ho.value, Wo.value, Co, device="cuda")
dy, dx, dW, db = torch.randn_like(y), torch.empty_like(x), torch.empty_like(Wt), torch.empty_like(b)
if which == "fwd":
    fn = lambda: L.sg_op_conv_forward(C.byref(d), x.data_ptr(), Wt.data_ptr(), b.data_ptr(), y.data_ptr(), None)  # noqa
else:
    fn = lambda: L.sg_op_conv_backward(C.byref(d), x.data_ptr(), Wt.data_ptr(), dy.data_ptr(), dx.data_ptr(),  # noqa
                                       dW.data_ptr(), db.data_ptr(), None)
for _ in range(4):
    fn()
torch.cuda.synchronize()
buf = (C.c_longlong * (6 * 64))()
assert L.lib.sg_debug_img_trace(buf) == 0
t = np.frombuffer(buf, dtype=np.int64).reshape(6, 64).astype(np.float64)
t0 = t[5, 0]
for r, name in enumerate(["end", "tap ready", "mma issued", "image ready", "done"]):
    v = t[r][t[r] > 0] - t0
    print(f"{name:13s} " + " ".join(f"{x:6.0f}" for x in v[:26]))
