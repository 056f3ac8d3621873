"""Time one convolution shape through the C ABI at several batch sizes (CUDA events)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1603_07846_b200 import _lib as L  # noqa: E402
from tools.gemm_bench import timeit  # noqa: E402


def main():
    H, Ci, Co, R, st, p = (int(v) for v in (sys.argv[1:7] if len(sys.argv) > 6 else (32, 4, 32, 5, 1, 2)))
    for N in (8, 32, 128, 512):
        d = L.ConvDesc(N, H, H, Ci, Co, R, R, st, p)
        Ho, Wo = C.c_int32(), C.c_int32()
        L.sg_conv_out_shape(C.byref(d), C.byref(Ho), C.byref(Wo))
        x = torch.randn(N, H, H, Ci, device="cuda")
        Wt = torch.randn(Co, R, R, Ci, device="cuda") * 0.05
        b = torch.zeros(Co, device="cuda")
        y = torch.empty(N, Ho.value, Wo.value, Co, device="cuda")
        dy = torch.randn_like(y)
        dW, db = torch.empty_like(Wt), torch.empty_like(b)
        tf = timeit(lambda: L.sg_op_conv_forward(C.byref(d), x.data_ptr(), Wt.data_ptr(), b.data_ptr(), y.data_ptr(), None), 20, False)
        tw = timeit(lambda: L.sg_op_conv_backward(C.byref(d), x.data_ptr(), Wt.data_ptr(), dy.data_ptr(), None,
                                                  dW.data_ptr(), db.data_ptr(), None), 20, False)
        print(f"N={N:4d} fwd {tf * 1e3:8.1f} us  wgrad {tw * 1e3:8.1f} us", flush=True)


if __name__ == "__main__":
    main()
