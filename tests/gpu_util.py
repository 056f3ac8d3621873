"""Helpers shared by the -m gpu tests (device buffers via torch, norms)."""

import numpy as np
import torch

# Reading A9: per-tensor normwise relative error for TF32
# tensor-core results (north star: "within 2e-3 relative").
TF32_TOL = 2e-3
# fp32 SIMT kernels vs the float64 oracle (rounding only).
FP32_TOL = 1e-5
# Reading A19: a blob read as a tensor-core operand is stored rounded to TF32
# (10 explicit mantissa bits, round to nearest): |rna(v) - v| <= 2^-11 |v|
# elementwise, hence normwise too.
RN_BOUND = 2.0 ** -11


def rna_tf32(a):
    """TF32 round to nearest, ties away from zero, of fp32 values (numpy bit ops;
    the definition, written independently of the CUDA path)."""
    a = np.ascontiguousarray(np.asarray(a, np.float32))
    u = a.view(np.uint32).astype(np.uint64)
    return ((u + 0x1000) & 0xFFFFE000).astype(np.uint32).view(np.float32)


def tf32_representable(a):
    u = np.ascontiguousarray(np.asarray(a, np.float32)).view(np.uint32)
    return bool(np.all((u & 0x1FFF) == 0))


def check_blob(got, ref, tol, rounded, what=""):
    """GPU blob vs the float64 oracle.  Not rounded: normwise < tol.  Rounded
    (the layer_info tf32_data / tf32_grad flag): every value TF32-representable,
    normwise < tol + RN_BOUND, and -- for SIMT kernels (tol <= 1e-4) -- equal to
    rna(fp32(oracle)) for all but the values whose fp32 result and the oracle
    straddle a TF32 rounding boundary (< 1%; truncation would miss ~half)."""
    e = normwise(got, ref)
    if not rounded:
        assert e < tol, (what, e)
        return e
    assert tf32_representable(np.asarray(got, np.float32)), (what, "not TF32-rounded")
    assert e < tol + RN_BOUND, (what, e)
    if tol <= 1e-4:
        g32 = np.asarray(got, np.float32)
        miss = np.mean(g32 != rna_tf32(np.asarray(ref, np.float64).astype(np.float32)))
        assert miss < 0.01, (what, "RN mismatch fraction", miss)
    return e


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
