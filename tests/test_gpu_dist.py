"""Multi-GPU parity (K = 2 / 4 ranks over NCCL): data-parallel K-invariance,
hybrid partitioning (dim-0 conv, dim-1 FC, dim-0 loss), feature-partitioned
auto-encoder, AlexNet hybrid, and the server-group sync — each rank one
process (torchrun), rank 0 checks against the float64 oracle at the same K.
Skipped when fewer than 2 GPUs are visible."""

import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0


def run_cases(k, cases, port):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={k}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "tests", "dist_worker.py")] + cases
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=420, cwd=ROOT)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-6000:]


@pytest.mark.skipif(NGPU < 2, reason="needs 2 GPUs")
def test_two_ranks():
    run_cases(2, ["server_sync", "peer_sync", "nvls_sync", "k_invariance", "hybrid", "autoencoder", "isolated", "alexnet", "p2p_step"],
              29611)


@pytest.mark.skipif(NGPU < 4, reason="needs 4 GPUs")
def test_four_ranks():
    run_cases(4, ["server_sync", "peer_sync", "nvls_sync", "k_invariance", "hybrid", "isolated", "alexnet", "p2p_step"], 29613)
