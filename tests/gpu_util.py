"""Helpers shared by the -m gpu tests (device buffers via torch, norms)."""

import numpy as np
import torch

# Reading A9: per-tensor normwise relative error for TF32
# tensor-core results (north star: "within 2e-3 relative").
TF32_TOL = 2e-3
# fp32 SIMT kernels vs the float64 oracle (rounding only).
FP32_TOL = 1e-5


# Device tensors created by dev()/empty() stay referenced until the end of the
# test (tests/conftest.py clears this list): a raw pointer handed to the C ABI
# must not outlive its tensor.
KEEP = []


def dev(a, dtype=None):
    a = np.ascontiguousarray(a)
    if dtype is None:
        dtype = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float32,
                 np.dtype(np.int32): torch.int32, np.dtype(np.int64): torch.int32,
                 np.dtype(np.uint8): torch.uint8}[a.dtype]
    if a.dtype == np.float64:
        a = a.astype(np.float32)
    t = torch.from_numpy(a).to(device="cuda", dtype=dtype).contiguous()
    KEEP.append(t)
    return t


def empty(shape, dtype=torch.float32):
    t = torch.full(tuple(shape), float("nan") if dtype.is_floating_point else 0, dtype=dtype, device="cuda")
    KEEP.append(t)
    return t


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def ptr(t):
    return None if t is None else t.data_ptr()


def normwise(got, ref):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    assert got.shape == ref.shape, (got.shape, ref.shape)
    assert np.all(np.isfinite(got)), "non-finite values in GPU output"
    den = np.linalg.norm(ref)
    return np.linalg.norm(got - ref) / (den if den > 0 else 1.0)


def f64(a):
    return np.asarray(a, np.float64)
