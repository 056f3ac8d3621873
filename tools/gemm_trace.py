"""CTA-0 timeline of one GEMM-engine launch (needs the trace variant:
python -m paper_1603_07846_b200.build --variant trace -D SG_GEMM_TRACE; run with
SG_LIB=build/trace/libsinga_b200.so).  Usage: gemm_trace.py conv N H C Co R st p [fwd|wgrad|dgrad]
                                      or gemm_trace.py gemm M N K"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1603_07846_b200 import _lib as L  # noqa: E402


def run(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    fn()
    torch.cuda.synchronize()
    buf = (C.c_longlong * (7 * 256))()
    assert L.lib.sg_debug_gemm_trace(buf) == 0
    t = np.frombuffer(buf, dtype=np.int64).reshape(7, 256).astype(np.float64)
    t0 = t[6, 0]
    names = ["prod start", "prod end", "mma ready", "mma issued", "epi ready", "epi done"]
    for r in range(6):
        v = t[r][t[r] > 0] - t0
        print(f"{names[r]:11s} n={len(v):3d} " + " ".join(f"{x:7.0f}" for x in v[:40]))


def main():
    kind = sys.argv[1]
    if kind == "gemm":
        M, N, K = (int(v) for v in sys.argv[2:5])
        A, B, Cm = torch.randn(M, K, device="cuda"), torch.randn(K, N, device="cuda"), torch.empty(M, N, device="cuda")
        run(lambda: L.sg_op_gemm(A.data_ptr(), 0, B.data_ptr(), 0, Cm.data_ptr(), M, N, K, None))
        return
    N, H, Ci, Co, R, st, p = (int(v) for v in sys.argv[2:9])
    which = sys.argv[9] if len(sys.argv) > 9 else "fwd"
    d = L.ConvDesc(N, H, H, Ci, Co, R, R, st, p)
    Ho, Wo = C.c_int32(), C.c_int32()
    L.sg_conv_out_shape(C.byref(d), C.byref(Ho), C.byref(Wo))
    x = torch.randn(N, H, H, Ci, device="cuda")
    Wt = torch.randn(Co, R, R, Ci, device="cuda") * 0.05
    b = torch.zeros(Co, device="cuda")
    y = torch.empty(N, Ho.value, Wo.value, Co, device="cuda")
    dy = torch.randn_like(y)
    dW, db = torch.empty_like(Wt), torch.empty_like(b)
    if which == "fwd":
        run(lambda: L.sg_op_conv_forward(C.byref(d), x.data_ptr(), Wt.data_ptr(), b.data_ptr(), y.data_ptr(), None))
    elif which == "dgrad":  # the data gradient is the last GEMM launched
        dx = torch.empty_like(x)
        run(lambda: L.sg_op_conv_backward(C.byref(d), x.data_ptr(), Wt.data_ptr(), dy.data_ptr(), dx.data_ptr(),
                                          dW.data_ptr(), db.data_ptr(), None))
    else:
        run(lambda: L.sg_op_conv_backward(C.byref(d), x.data_ptr(), Wt.data_ptr(), dy.data_ptr(), None, dW.data_ptr(),
                                          db.data_ptr(), None))


if __name__ == "__main__":
    main()
