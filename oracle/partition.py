"""Partition maps (oracle).  Test infrastructure only.

PAPER.md §5.3: a layer is partitioned on dimension 0 (rows = feature
vectors of a mini-batch, "slices the feature matrix by row") or dimension 1
("by column").  The paper does not fix how uneven extents split
fixes remainder-first (larger slices at lower indices) — DESIGN.md reading A12.

Pins: tests/test_oracle_partition.py (SPEC S:46-47 and S:227-228 examples,
round trip S:72, exhaustive coverage).
"""

import numpy as np


def partition_range(extent, parts, idx):
    """Remainder-first: len_i = floor(E/K) + [i < E mod K]; off_i = sum_{j<i} len_j (A12)."""
    if parts < 1 or idx < 0 or idx >= parts:
        raise ValueError("bad partition arguments")
    if parts > extent:
        raise ValueError(f"partition error: {parts} parts > extent {extent}")
    base, rem = divmod(extent, parts)
    off = 0
    for j in range(idx):
        off += base + (1 if j < rem else 0)
    return off, base + (1 if idx < rem else 0)


def slice_blob(a, dim, parts):
    """SPEC S:40-47 slice(A, dim, parts)."""
    out = []
    for i in range(parts):
        off, ln = partition_range(a.shape[dim], parts, i)
        out.append(a[off:off + ln] if dim == 0 else a[:, off:off + ln])
    return out


def concat_blobs(parts, dim):
    """SPEC S:49-55 concat(parts, dim): inverse of slice."""
    return np.concatenate(parts, axis=dim)


def bucket_shard_map(param_sizes, world):
    """Server shard map for one dim-0 layer bucket (reading A13).

    The bucket is concat(params in order), zero-padded to E' = ceil(E/(32K))*32K;
    rank k owns [k*E'/K, (k+1)*E'/K).  Returns (E', [(param, owner, param_off,
    bucket_off, len), ...]) in ascending bucket order.
    """
    total = sum(param_sizes)
    unit = 32 * world
    padded = -(-total // unit) * unit
    shard = padded // world
    out = []
    boff = 0
    for p, sz in enumerate(param_sizes):
        poff = 0
        while poff < sz:
            owner = (boff + poff) // shard
            end_owner = (owner + 1) * shard
            ln = min(sz - poff, end_owner - (boff + poff))
            out.append((p, owner, poff, boff + poff, ln))
            poff += ln
        boff += sz
    return padded, out
