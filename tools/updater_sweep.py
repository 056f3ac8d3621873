"""C5 server-group Updater sweep (BASELINE configs[4]).

One flat fp32 Param of P elements per rank; each step is the paper's
worker-group -> server-group exchange through the
C ABI call ``sg_server_sync``: reduce-scatter(sum) of the full gradient,
the fused SGD-momentum Updater (a17) on the rank's P/K shard, and
all-gather of the updated weights.

    python -m torch.distributed.run --nnodes=1 --nproc-per-node K \
        --master-addr 127.0.0.1 --master-port 29511 tools/updater_sweep.py [--iters 20]
    python tools/updater_sweep.py            # K = 1: the Updater kernel alone

Timing: CUDA events on the stream the call is launched on, W = 3 untimed
warm-up calls, then ``iters`` calls; barrier + synchronize on both sides;
max over ranks.  Per P, one JSON line on rank 0:
  t_us          time of one sg_server_sync
  algbw_gbs     4P / t (gradient bytes per rank per second)
  busbw_gbs     nccl-tests convention for RS + AG: 2 (K-1)/K * 4P / t
  upd_hbm_gbs   (K = 1 only) 20 B per element / t against MEASURED_PEAKS hbm_gbs
At K > 1 the line also carries ``torch_nccl_t_us``: the same exchange through
stock ``torch.distributed`` reduce_scatter_tensor / all_gather_into_tensor with
the update as torch elementwise ops (context, not the product path), and
``fused_p2p_t_us``: the fused peer-memory path ``sg_peer_sync_step`` (one
kernel reading every rank's gradient shard over NVLink and storing the new
weights into every rank, between two flag barriers).
P >= 16M exceed the 126 MB L2 per step (grad + w + v); the smaller sizes may be
partly L2-resident between iterations (stated in the line as "l2_resident").
"""

import argparse
import ctypes as C
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1603_07846_b200 import _lib as L  # noqa: E402
from paper_1603_07846_b200 import net as PN  # noqa: E402

SIZES_M = [1, 2, 4, 8, 16, 32, 61.10084]   # 61,100,840 = the AlexNet-shaped net's Params (C3)


def dev_view(ptr, n):
    """A torch view of a library-owned device buffer (no copy)."""
    class _A:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 2}
    return torch.as_tensor(_A(), device="cuda")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [PN.Cluster.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        cl = PN.Cluster(rank, world, local, obj[0])
    else:
        cl = PN.Cluster(0, 1, local)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    cfg = PN.updater_cfg({"base_lr": 0.01, "momentum": 0.9, "weight_decay": 5e-4})
    stream = torch.cuda.Stream()
    g = torch.Generator(device="cuda").manual_seed(1234 + rank)
    for pm in SIZES_M:
        q = 32 * world
        n = (int(pm * 1e6) + q - 1) // q * q
        w = torch.randn(n, device="cuda", generator=g) * 0.01
        if world > 1:
            dist.barrier()
        grad0 = torch.randn(n, device="cuda", generator=g)
        grad = grad0.clone()
        v = torch.zeros(n // world, device="cuda")
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            for t in range(args.warmup):
                L.sg_server_sync(cl.h, C.byref(cfg), t, grad.data_ptr(), w.data_ptr(), v.data_ptr(), n,
                                 C.c_void_p(stream.cuda_stream))
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            ev0.record(stream)
            for t in range(args.iters):
                # grad is overwritten by the reduce-scatter; its values do not change the cost
                L.sg_server_sync(cl.h, C.byref(cfg), args.warmup + t, grad.data_ptr(), w.data_ptr(), v.data_ptr(),
                                 n, C.c_void_p(stream.cuda_stream))
            ev1.record(stream)
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1) / args.iters
        # context only: the same exchange as stock torch.distributed collectives plus
        # the update as torch elementwise ops (5 kernels) on the shard
        tms = None
        if world > 1:
            shard = n // world
            ws = w[rank * shard:(rank + 1) * shard]
            gs = torch.empty(shard, device="cuda")
            with torch.cuda.stream(stream):
                for t in range(args.warmup + args.iters):
                    if t == args.warmup:
                        torch.cuda.synchronize()
                        dist.barrier()
                        ev0.record(stream)
                    dist.reduce_scatter_tensor(gs, grad)
                    gs.mul_(1.0 / world).add_(ws, alpha=5e-4)
                    v.mul_(0.9).sub_(gs, alpha=0.01)
                    ws.add_(v)
                    dist.all_gather_into_tensor(w, ws)   # in place, as sg_server_sync
                ev1.record(stream)
            torch.cuda.synchronize()
            tms = ev0.elapsed_time(ev1) / args.iters
            tt = torch.tensor([ms, tms], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms, tms = float(tt[0].item()), float(tt[1].item())
            dist.barrier()
        # the fused peer-memory path (sg_peer_sync_*: one kernel, P2P loads / stores)
        # and the NVSwitch multicast path (sg_nvls_sync_*), when available
        def fused(api):
            h, gp, wp, vp = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
            try:
                getattr(L, f"sg_{api}_sync_create")(cl.h, n, C.byref(h), C.byref(gp), C.byref(wp), C.byref(vp))
            except L.SingaError:
                return None
            dev_view(gp.value, n).copy_(grad0)
            dev_view(wp.value, n).fill_(0.01)
            torch.cuda.synchronize()
            dist.barrier()
            step_fn = getattr(L, f"sg_{api}_sync_step")
            with torch.cuda.stream(stream):
                for t in range(args.warmup + args.iters):
                    if t == args.warmup:
                        torch.cuda.synchronize()
                        dist.barrier()
                        ev0.record(stream)
                    step_fn(h, C.byref(cfg), t, C.c_void_p(stream.cuda_stream))
                ev1.record(stream)
            torch.cuda.synchronize()
            r = ev0.elapsed_time(ev1) / args.iters
            getattr(L, f"sg_{api}_sync_destroy")(h)
            tt = torch.tensor([r], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            return float(tt[0].item())

        fms = nms = None
        if world > 1:
            nms = fused("nvls")
        if False:
            h, gp, wp, vp = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
            L.sg_peer_sync_create(cl.h, n, C.byref(h), C.byref(gp), C.byref(wp), C.byref(vp))
            dev_view(gp.value, n).copy_(grad0)
            dev_view(wp.value, n).fill_(0.01)
            torch.cuda.synchronize()
            dist.barrier()
            with torch.cuda.stream(stream):
                for t in range(args.warmup + args.iters):
                    if t == args.warmup:
                        torch.cuda.synchronize()
                        dist.barrier()
                        ev0.record(stream)
                    L.sg_peer_sync_step(h, C.byref(cfg), t, C.c_void_p(stream.cuda_stream))
                ev1.record(stream)
            torch.cuda.synchronize()
            fms = ev0.elapsed_time(ev1) / args.iters
            L.sg_peer_sync_destroy(h)
            tt = torch.tensor([fms], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            fms = float(tt[0].item())
        if world > 1:
            fms = fused("peer")
        t_s = ms * 1e-3
        line = {"workload": "updater_sweep", "params": n, "n_gpus": world, "iters": args.iters,
                "warmup": args.warmup, "t_us": round(ms * 1e3, 2),
                "algbw_gbs": round(4 * n / t_s / 1e9, 1),
                "l2_resident": 12 * n < 126e6}
        if world > 1:
            line["busbw_gbs"] = round(2 * (world - 1) / world * 4 * n / t_s / 1e9, 1)
            line["nvlink_peak_gbs"] = 900.0
            line["torch_nccl_t_us"] = round(tms * 1e3, 2)
            line["fused_p2p_t_us"] = round(fms * 1e3, 2)
            line["fused_p2p_busbw_gbs"] = round(2 * (world - 1) / world * 4 * n / (fms * 1e-3) / 1e9, 1)
            line["nvls_t_us"] = round(nms * 1e3, 2) if nms is not None else None
        else:
            a = 20 * n / t_s / 1e9
            line["upd_hbm_gbs"] = round(a, 1)
            line["hbm_peak_gbs"] = peaks["hbm_gbs"]
            line["frac"] = round(a / peaks["hbm_gbs"], 3)
        if rank == 0:
            print(json.dumps(line), flush=True)
        del w, grad, grad0, v
        torch.cuda.empty_cache()
    cl.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
