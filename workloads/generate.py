"""Seeded synthetic inputs shared by the oracle and the CUDA path.

Holds none of the method's arithmetic: only random draws with the shapes and
value distributions of the paper's workloads (DESIGN.md
"Input recipe").  Everything is produced as float32 (int32 labels) on the host;
the oracle widens to float64 exactly.
"""

import zlib

import numpy as np

from . import configs


def _rng(*key):
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(k) & 0xFFFFFFFF for k in key])))


def param_seed(name, job_seed=configs.JOB_SEED):
    """seed = jobSeed XOR crc32(paramName) (SPEC S:163 reading A3)."""
    return (job_seed ^ zlib.crc32(name.encode())) & 0xFFFFFFFF


def glorot(name, shape, fan_in, fan_out, job_seed=configs.JOB_SEED):
    """Glorot-uniform U[-sqrt(6/(fan_in+fan_out)), +...] on the GLOBAL tensor,
    seeded per Param so the draw is partition-invariant."""
    lim = np.sqrt(6.0 / (fan_in + fan_out))
    g = _rng(param_seed(name, job_seed))
    return g.uniform(-lim, lim, size=shape).astype(np.float32)


def init_params(param_specs, job_seed=configs.JOB_SEED):
    """param_specs: iterable of (name, shape, fan_in, fan_out, is_bias)."""
    out = {}
    for name, shape, fan_in, fan_out, is_bias in param_specs:
        if is_bias:
            out[name] = np.zeros(shape, np.float32)
        else:
            out[name] = glorot(name, shape, fan_in, fan_out, job_seed)
    return out


_TEMPLATES = {}


def _templates(cfg_name, num_classes, shape, kind):
    key = (cfg_name, num_classes, shape, kind)
    if key not in _TEMPLATES:
        g = _rng(configs.JOB_SEED, 7, zlib.crc32(cfg_name.encode()))
        if kind == "uniform":
            _TEMPLATES[key] = g.random((num_classes,) + shape, dtype=np.float32)
        else:
            _TEMPLATES[key] = g.standard_normal((num_classes,) + shape, dtype=np.float32)
    return _TEMPLATES[key]


def batch(net, b, t, job_seed=configs.JOB_SEED):
    """Global mini-batch ``t`` (rows [t*b, (t+1)*b) of an endless seeded pool).

    Returns (x, labels): x float32 [b][H][W][C] (NHWC, C = 3 unpadded) or
    [b][d]; labels int32 [b] (all zeros for a net without classes).
    """
    name = net["name"]
    inp = net["input"]
    nc = max(net["num_classes"], 1)
    g = _rng(job_seed, 11, zlib.crc32(name.encode()), b, t)
    labels = g.integers(0, nc, size=b, dtype=np.int32) if net["num_classes"] else np.zeros(b, np.int32)
    if "d" in inp:
        d = inp["d"]
        T = _templates(name, nc, (d,), "uniform")
        x = np.clip(0.1 * T[labels] + g.random((b, d), dtype=np.float32), 0.0, 1.0).astype(np.float32)
    else:
        h, w, c = inp["h"], inp["w"], inp["c"]
        if h <= 64:
            T = _templates(name, nc, (h, w, c), "normal")
            x = g.standard_normal((b, h, w, c), dtype=np.float32) + np.float32(0.05) * T[labels]
        else:
            # 7x7 class templates nearest-upsampled (avoids a 600 MB template bank).
            T = _templates(name, nc, (7, 7, c), "normal")
            up = h // 7
            Tl = T[labels].repeat(up, axis=1).repeat(up, axis=2)
            Tl = np.pad(Tl, ((0, 0), (0, h - Tl.shape[1]), (0, w - Tl.shape[2]), (0, 0)))
            x = g.standard_normal((b, h, w, c), dtype=np.float32) + np.float32(0.05) * Tl
        x = x.astype(np.float32)
    return x, labels


def server_sync_inputs(n, world, rank, job_seed=configs.JOB_SEED):
    """C5 Updater sweep: per-rank gradient N(0, 1e-2^2), shared w ~ U(-0.05, 0.05), v = 0."""
    g = _rng(job_seed, 13, n, rank)
    grad = (g.standard_normal(n, dtype=np.float32) * np.float32(1e-2)).astype(np.float32)
    gw = _rng(job_seed, 17, n)
    w = gw.uniform(-0.05, 0.05, size=n).astype(np.float32)
    return grad, w
