"""Micro-benchmark of the tcgen05 GEMM engine through the C ABI (CUDA events,
warm L2 unless --flush): conv fwd / wgrad / dgrad and IP shapes of the configs."""
import argparse
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1603_07846_b200 import _lib as L  # noqa: E402

TF32_PEAK = 1651.4 * 1.1 / 2.25


def timeit(fn, reps, flush):
    buf = torch.empty(64 * 1024 * 1024, device="cuda") if flush else None
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if flush:
            buf.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        ts.append((a, b))
    torch.cuda.synchronize()
    v = sorted(x.elapsed_time(y) for x, y in ts)
    return v[len(v) // 2]


def conv_cases(flush):
    cases = [("cifar conv1", 128, 32, 32, 4, 32, 5, 1, 2, 3), ("cifar conv2", 128, 16, 16, 32, 32, 5, 1, 2, 32),
             ("cifar conv3", 128, 8, 8, 32, 64, 5, 1, 2, 32), ("alex conv2", 256, 27, 27, 64, 192, 5, 1, 2, 64),
             ("alex conv3", 256, 13, 13, 192, 384, 3, 1, 1, 192), ("alex conv1", 256, 224, 224, 4, 64, 11, 4, 2, 3)]
    for name, N, H, W, Ci, Co, R, st, p, creal in cases:
        d = L.ConvDesc(N, H, W, Ci, Co, R, R, st, p)
        Ho, Wo = C.c_int32(), C.c_int32()
        L.sg_conv_out_shape(C.byref(d), C.byref(Ho), C.byref(Wo))
        x = torch.randn(N, H, W, Ci, device="cuda")
        Wt = torch.randn(Co, R, R, Ci, device="cuda") * 0.05
        b = torch.zeros(Co, device="cuda")
        y = torch.empty(N, Ho.value, Wo.value, Co, device="cuda")
        dy = torch.randn_like(y)
        dx, dW, db = torch.empty_like(x), torch.empty_like(Wt), torch.empty_like(b)
        fl = 2.0 * N * Ho.value * Wo.value * Co * R * R * creal
        tf = timeit(lambda: L.sg_op_conv_forward(C.byref(d), x.data_ptr(), Wt.data_ptr(), b.data_ptr(), y.data_ptr(), None), 20, flush)
        tw = timeit(lambda: L.sg_op_conv_backward(C.byref(d), x.data_ptr(), Wt.data_ptr(), dy.data_ptr(), None,
                                                  dW.data_ptr(), db.data_ptr(), None), 20, flush)
        td = timeit(lambda: L.sg_op_conv_backward(C.byref(d), x.data_ptr(), Wt.data_ptr(), dy.data_ptr(), dx.data_ptr(),
                                                  dW.data_ptr(), db.data_ptr(), None), 20, flush) - tw
        print(f"{name:12s} fwd {tf * 1e3:8.1f} us {fl / tf / 1e9:7.1f} TF/s ({fl / tf / 1e9 / TF32_PEAK:5.1%})   "
              f"wgrad {tw * 1e3:8.1f} us {fl / tw / 1e9:7.1f} TF/s   dgrad {td * 1e3:8.1f} us {fl / td / 1e9:7.1f} TF/s",
              flush=True)


def gemm_cases(flush):
    for (M, N, K) in [(256, 8000, 4000), (256, 4096, 9216), (4096, 4096, 4096), (8192, 8192, 8192)]:
        A = torch.randn(M, K, device="cuda")
        B = torch.randn(K, N, device="cuda")
        Cm = torch.empty(M, N, device="cuda")
        t = timeit(lambda: L.sg_op_gemm(A.data_ptr(), 0, B.data_ptr(), 0, Cm.data_ptr(), M, N, K, None), 10, flush)
        fl = 2.0 * M * N * K
        ref = timeit(lambda: torch.matmul(A, B, out=Cm), 10, flush)
        print(f"gemm {M}x{N}x{K}: {t * 1e3:8.1f} us {fl / t / 1e9:7.1f} TF/s ({fl / t / 1e9 / TF32_PEAK:5.1%}); "
              f"torch fp32(tf32={torch.backends.cuda.matmul.allow_tf32}) {ref * 1e3:8.1f} us", flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--flush", action="store_true")
    ap.add_argument("--gemm", default="")
    a = ap.parse_args()
    torch.backends.cuda.matmul.allow_tf32 = True
    if a.gemm:
        M, N, K, tb = (int(v) for v in a.gemm.split(","))
        A, B, Cm = torch.randn(M, K, device="cuda"), torch.randn(N, K, device="cuda") if tb else torch.randn(K, N, device="cuda"), torch.empty(M, N, device="cuda")
        t = timeit(lambda: L.sg_op_gemm(A.data_ptr(), 0, B.data_ptr(), tb, Cm.data_ptr(), M, N, K, None), 10, a.flush)
        print(f"gemm {M}x{N}x{K} tb={tb}: {t * 1e3:.1f} us {2.0 * M * N * K / t / 1e9:.1f} TF/s")
        sys.exit(0)
    gemm_cases(a.flush)
    conv_cases(a.flush)
