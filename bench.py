#!/usr/bin/env python
"""Benchmark: synchronous BP TrainOneBatch of the SINGA path on B200.

One JSON line on rank 0 (contract in the task statement; workload and roofline
conventions in DESIGN.md "Measurement"):

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cifar10|alexnet|mlp|ae_wide]
    torchrun --nproc-per-node N bench.py --gpus N ...        (N > 1, one rank per GPU)
    python bench.py --impl reference ...                      (the float64 CPU oracle arm)

* value: training images/s of the whole job, device time (CUDA events on the
  launching stream) of exactly K steps, max over ranks, inputs resident in HBM,
  L2 flushed (256 MB write) before every timed step (flush excluded);
* e2e: the same metric through the pipelined host entry
  sg_train_one_batch_host_async from pinned host buffers (every step's H2D
  input copy and D2H loss read inside the timed region; the next step's copy
  overlaps the current step); e2e.sync_api_value: the synchronous
  sg_train_one_batch_host (copy in, step, loss out, wait, every call);
* roofline: the dominant operation of the step, from a second, profiled pass of
  the same graph with CUDA events around every layer operation;
* cpu_baseline: the oracle (oracle/, float64 numpy) timed on this host's cores on
  a bounded sample of the same workload (rank 0, N = 1 only).
"""

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import configs, generate  # noqa: E402

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
TF32_OVER_BF16 = 1.1 / 2.25      # guide's nominal dense ratio (tf32 1.1 PF vs bf16 2.25 PF)
PER_GPU_BATCH = {"cifar10": 128, "mlp": 64, "alexnet": 256, "alexnet_dp": 256, "ae_wide": 256, "ae": 256}
SCALING = {"cifar10": "weak", "mlp": "weak", "alexnet": "strong", "alexnet_dp": "strong", "ae_wide": "strong",
           "ae": "strong"}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        src = "measured"
    else:
        d, src = dict(PEAKS_FALLBACK), "fallback"
    # TF32 tensor-pipe ceiling measured on a B200 of this pool (tools/tf32_peak.cu:
    # every SM issuing 128x256x8 kind::tf32 MMAs from shared memory)
    t = os.path.join(ROOT, "profiles", "r02_tf32_peak.json")
    if os.path.exists(t):
        d = dict(d, tf32_tflops=json.load(open(t))["tf32_tflops"])
    return d, src


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


# ----------------------------------------------------------------------------
# Algorithmic work per operation (reporting only).
# ----------------------------------------------------------------------------
def op_work(net_cfg, infos, world):
    """slot -> (name, flops, bytes) for every layer operation (4 slots per layer)."""
    out = {}
    ucfg = {l["name"]: l for l in net_cfg["layers"]}
    in_c = net_cfg["input"].get("c", 0)
    for i, li in enumerate(infos):
        k = li["kind"]
        if k == "input" or li["is_connection"]:
            continue
        src = infos[li["src"]]
        rows = li["local_shape"][0]
        cfg = ucfg[li["name"]]
        if k == "conv":
            _, Ho, Wo, Co = li["local_shape"]
            _, H, W, Cs = src["local_shape"]
            Ci = in_c if src["kind"] == "input" else Cs
            R = cfg["kernel"]
            fl = 2.0 * rows * Ho * Wo * Co * R * R * Ci
            x, y, w = rows * H * W * Ci * 4, rows * Ho * Wo * Co * 4, (Co * R * R * Ci + Co) * 4
            out[4 * i] = (li["name"] + ".fwd", fl, x + y + w)
            out[4 * i + 1] = (li["name"] + ".wgrad", fl, x + y + w)
            if src["kind"] != "input":
                out[4 * i + 2] = (li["name"] + ".dgrad", fl, x + y + w)
            out[4 * i + 3] = (li["name"] + ".update", 0.0, 20.0 * (Co * R * R * Ci + Co) / world)
        elif k == "ip":
            dh = li["local_shape"][1]
            dv = int(np.prod(src["global_shape"][1:])) if src["kind"] != "input" else net_cfg["input"].get("d", 0)
            if src["kind"] == "input" and "d" not in net_cfg["input"]:
                dv = int(np.prod(src["global_shape"][1:]))
            fl = 2.0 * rows * dv * dh
            b = (rows * dv + dv * dh + rows * dh) * 4
            out[4 * i] = (li["name"] + ".fwd", fl, b)
            out[4 * i + 1] = (li["name"] + ".wgrad", fl, b)
            if src["kind"] != "input":
                out[4 * i + 2] = (li["name"] + ".dgrad", fl, b)
            sharded = li["partition_dim"] == 0
            out[4 * i + 3] = (li["name"] + ".update", 0.0, 20.0 * (dv * dh + dh) / (world if sharded else 1))
        else:
            n_out = rows * int(np.prod(li["local_shape"][1:]))
            n_in = rows * int(np.prod(src["local_shape"][1:]))
            if k in ("relu", "sigmoid"):
                out[4 * i] = (li["name"] + ".fwd", 0.0, 8.0 * n_out)
                out[4 * i + 1] = (li["name"] + ".bwd", 0.0, 12.0 * n_out)
            elif k == "pool_max":
                out[4 * i] = (li["name"] + ".fwd", 0.0, 4.0 * (n_in + n_out) + n_out)
                out[4 * i + 1] = (li["name"] + ".bwd", 0.0, 4.0 * (n_in + n_out) + n_out)
            elif k == "pool_avg":
                out[4 * i] = (li["name"] + ".fwd", 0.0, 4.0 * (n_in + n_out))
                out[4 * i + 1] = (li["name"] + ".bwd", 0.0, 4.0 * (n_in + n_out))
            elif k == "lrn":
                out[4 * i] = (li["name"] + ".fwd", 0.0, 12.0 * n_out)
                out[4 * i + 1] = (li["name"] + ".bwd", 0.0, 20.0 * n_out)
            elif k in ("softmax_ce", "euclidean"):
                feats = int(np.prod(src["global_shape"][1:]))
                out[4 * i] = (li["name"] + ".fwd", 0.0, 8.0 * rows * feats)
    return out


# ----------------------------------------------------------------------------
class ClockLog:
    """nvidia-smi sampling of SM clocks and throttle reasons during a region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(gpu_index), "--query-gpu=" + self.FIELDS,
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = [l.split(", ") for l in open(self.f.name).read().strip().splitlines() if l.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, r[3:7]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}



def grad_sync_bytes(net_cfg, infos, world):
    """'<layer>.update' -> fp32 gradient bytes the layer's bucket moves per step at N > 1
    (dim-0 layers only: reduce-scatter of the full gradient + all-gather of the weights, a16/a18).
    Dim-1 FC slices update owner-locally and move no Param bytes."""
    out = {}
    if world < 2:
        return out
    w_of = {}
    for name, fl, by in op_work(net_cfg, infos, world).values():
        if name.endswith(".update"):
            w_of[name[:-7]] = by / 20.0
    for li in infos:
        if li["kind"] == "conv" or (li["kind"] == "ip" and li["partition_dim"] == 0):
            out[li["name"] + ".update"] = 4.0 * w_of[li["name"]] * world
    return out

def init_params(PN, n, net_cfg):
    ucfg = {l["name"]: l for l in net_cfg["layers"]}
    out = {}
    for p in n.param_info:
        name = p["name"]
        layer = name.split("/")[0]
        if name.endswith("/b"):
            out[name] = np.zeros(p["cols"], np.float32)
            continue
        if ucfg[layer]["kind"] == "conv":
            R = ucfg[layer]["kernel"]
            Ci = p["cols"] // (R * R)
            shape = (p["rows"], R, R, Ci)
            fan_in, fan_out = Ci * R * R, p["rows"] * R * R
        else:
            shape = (p["rows"], p["cols"])
            fan_in, fan_out = p["rows"], p["cols"]
        out[name] = generate.glorot(name, shape, fan_in, fan_out)
    return out


def cpu_oracle_rate(net_cfg, b, budget_s, steps=None):
    """Oracle images/s on a bounded sample of the workload (this host's cores)."""
    from oracle import net as ON   # the oracle: only here (cpu_baseline) and in --impl reference
    upd = configs.UPDATERS[net_cfg["name"]]
    params = generate.init_params(ON.param_specs(net_cfg))
    p = {k: v.astype(np.float64) for k, v in params.items()}
    v = {k: np.zeros_like(a) for k, a in p.items()}
    done, t0 = 0, time.perf_counter()
    times = []
    while True:
        x, lab = generate.batch(net_cfg, b, done)
        s = time.perf_counter()
        out = ON.train_one_batch(net_cfg, p, v, x, lab, done, 1, upd)
        times.append(time.perf_counter() - s)
        p, v = out["params"], out["vel"]
        done += 1
        if steps is not None and done >= steps:
            break
        if steps is None and (time.perf_counter() - t0 > budget_s or done >= 50):
            break
    return b * done / sum(times), done, times


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max((i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"), default=1)
    except Exception:
        return len(os.sched_getaffinity(0))


def run_reference(args, rank, world):
    """--impl reference: the float64 CPU oracle as the reference arm."""
    if rank != 0:
        return
    net_cfg = configs.get(args.config)
    b = PER_GPU_BATCH[args.config] if SCALING[args.config] == "weak" else configs.BATCH[args.config]
    if args.config == "alexnet":
        b = 8    # bounded sample (an oracle AlexNet step at b=256 takes minutes)
    for t in range(args.warmup):
        cpu_oracle_rate(net_cfg, b, 0, steps=1)
    rate, done, times = cpu_oracle_rate(net_cfg, b, 0, steps=args.steps)
    cores = blas_threads()
    sample = f"{args.config} b={b}, {done} oracle steps (float64 numpy), {len(os.sched_getaffinity(0))} host cores visible"
    line = {"metric": "training images/sec", "value": rate, "unit": "images/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
            "higher_is_better": True, "scaling": SCALING[args.config], "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": args.config, "batch": b, "sample": "bounded"},
            "cpu_baseline": {"value": rate, "unit": "images/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": rate, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", default="cifar10", choices=sorted(PER_GPU_BATCH))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-steps", type=int, default=50)
    ap.add_argument("--batch", type=int, default=0, help="global batch override (ablations)")
    ap.add_argument("--no-overlap", action="store_true", help="Update waits on the compute stream (P:770-774)")
    ap.add_argument("--exchange", default="p2p", choices=["nccl", "p2p"],
                    help="gradient exchange of the sharded buckets at N > 1: NCCL chain or fused peer-memory kernel")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank, world, local = env_rank()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    from paper_1603_07846_b200 import _lib as L
    from paper_1603_07846_b200 import net as PN

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [PN.Cluster.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    else:
        nccl_id = None
    cluster = PN.Cluster(rank, world, local, nccl_id)
    net_cfg = configs.get(args.config)
    weak = SCALING[args.config] == "weak"
    b = args.batch or PER_GPU_BATCH[args.config] * (world if weak else 1)
    n = PN.Net(cluster, net_cfg, b)
    n.set_updater(configs.UPDATERS[args.config])
    n.set_params(init_params(PN, n, net_cfg))
    if world > 1 and args.exchange != "nccl":
        n.set_exchange(args.exchange)
    if args.no_overlap:
        L.sg_net_set_overlap(n.h, 0)
    info = n.layer_info
    rows_in = info[0]["local_shape"][0]
    row_off = info[0]["local_offset"][0]
    loss_layer = info[-1]
    lab_rows = loss_layer["local_shape"][0]
    lab_off = info[loss_layer["src"]]["local_offset"][0]

    npool = 4 if args.config == "alexnet" else 8
    xs, ls, xs_h, ls_h = [], [], [], []
    for t in range(npool):
        x, lab = generate.batch(net_cfg, b, t)
        x = np.ascontiguousarray(x[row_off:row_off + rows_in])
        lab = np.ascontiguousarray(lab[lab_off:lab_off + lab_rows])
        xs.append(torch.from_numpy(x).cuda())
        ls.append(torch.from_numpy(lab).cuda())
        xs_h.append(torch.from_numpy(x).pin_memory())
        ls_h.append(torch.from_numpy(lab).pin_memory())
    has_labels = net_cfg["num_classes"] > 0
    loss = torch.zeros(1, device="cuda")
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")   # 256 MB > 126 MB L2
    stream = torch.cuda.current_stream()
    sp = C.c_void_p(stream.cuda_stream)
    if not args.no_graph:
        n.enable_graph(True)

    def step(t):
        j = t % npool
        n.train_one_batch(t, xs[j].data_ptr(), ls[j].data_ptr() if has_labels else None, loss.data_ptr(), sp)

    for t in range(args.warmup):
        step(t)
    n.sync()
    torch.cuda.synchronize()

    # ---------------- timed region: exactly K steps ----------------
    clock = ClockLog(local)
    # let nvidia-smi finish its (driver-locking) start-up before the timed
    # region: a rank whose host stalls while enqueueing the first steps leaves
    # the other ranks' device-side barriers spinning (seen once per scaling run)
    time.sleep(1.0)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = []
    for t in range(args.steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step(args.warmup + t)
        e1.record(stream)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clock.stop()
    launches = n.launches()
    n.sync()
    step_ms = [a.elapsed_time(b_) for a, b_ in evs]
    total_ms = sum(step_ms)
    srt = sorted(step_ms)
    print(f"[rank {rank}] step ms min {srt[0]:.4f} median {srt[len(srt) // 2]:.4f} max {srt[-1]:.4f} "
          f"(argmax {step_ms.index(srt[-1])})", file=sys.stderr)
    if world > 1:
        t_ = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t_, op=dist.ReduceOp.MAX)
        total_ms = float(t_.item())
    imgs = b * args.steps
    value = imgs / (total_ms / 1e3)
    final_loss = float(loss.item())

    # ---------------- profiled pass: per-operation device times ----------------
    n.enable_graph(False)
    L.sg_net_profile(n.h, 1)
    if not args.no_graph:
        n.enable_graph(True)
    nslots = len(info) * 4
    ms = (C.c_double * nslots)()
    cnt = (C.c_int64 * nslots)()
    ns = C.c_int32()
    for t in range(3):
        step(t)
    L.sg_net_op_times(n.h, ms, cnt, nslots, C.byref(ns), 1)
    prof_steps = max(1, min(args.profile_steps, args.steps))
    for t in range(prof_steps):
        flush.zero_()
        step(t)
        L.sg_net_op_times(n.h, ms, cnt, nslots, C.byref(ns), 0)
    L.sg_net_profile(n.h, 0)
    work = op_work(net_cfg, info, world)
    peaks, peaks_src = load_peaks()
    hbm_peak = peaks.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"])
    tf32_peak = peaks.get("tf32_tflops") or peaks.get("bf16_tflops", PEAKS_FALLBACK["bf16_tflops"]) * TF32_OVER_BF16
    tf32_src = "measured tf32 (profiles/r02_tf32_peak.json)" if peaks.get("tf32_tflops") else \
        "bf16 x 1.1/2.25 nominal ratio"
    ops = []
    for s in range(nslots):
        if cnt[s] > 0 and s in work:
            name, fl, by = work[s]
            avg = ms[s] / cnt[s]
            ops.append({"op": name, "ms": avg, "flops": fl, "bytes": by})
    ops.sort(key=lambda o: -o["ms"])
    prof_total = sum(o["ms"] for o in ops)
    # at N > 1 a layer's update slot times the reduce-scatter -> Updater -> all-gather
    # chain on the parameter stream (mostly NCCL waiting); the roofline names the
    # dominant compute operation instead
    cand = [o for o in ops if world == 1 or not o["op"].endswith(".update")]
    dom = cand[0] if cand else None
    roof = None
    if dom:
        t_s = dom["ms"] / 1e3
        f_frac = (dom["flops"] / t_s / 1e12) / tf32_peak if dom["flops"] else 0.0
        b_frac = (dom["bytes"] / t_s / 1e9) / hbm_peak
        if dom["flops"] and dom["flops"] / tf32_peak / 1e12 >= dom["bytes"] / hbm_peak / 1e9:
            roof = {"bound": "tensor", "achieved": dom["flops"] / t_s / 1e12, "peak": tf32_peak, "unit": "TFLOP/s",
                    "frac": f_frac}
        else:
            roof = {"bound": "hbm", "achieved": dom["bytes"] / t_s / 1e9, "peak": hbm_peak, "unit": "GB/s",
                    "frac": b_frac}
        roof.update({"kernel": dom["op"], "kernel_ms": dom["ms"], "share_of_step": dom["ms"] / (total_ms / args.steps),
                     "peak_source": f"{peaks_src} ({tf32_src if roof['bound'] == 'tensor' else 'hbm copy'})",
                     "traffic": None})
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            roof["traffic"] = json.load(open(tp)).get(f"{args.config}:{dom['op']}")

    # gradient synchronisation over NVLink (a16 -> a17 -> a18): each dim-0 layer's
    # update slot times its reduce-scatter -> Updater -> all-gather chain on the
    # parameter stream (it overlaps the backward of the layers below)
    grad_sync = None
    gsb = grad_sync_bytes(net_cfg, info, world)
    if gsb:
        upd = [o for o in ops if o["op"] in gsb]
        t_upd = sum(o["ms"] for o in upd) / 1e3
        nbytes = sum(gsb.values())
        grad_sync = {"bytes_per_step": int(nbytes), "layers": len(gsb), "chain_ms": t_upd * 1e3,
                     "algbw_gbs": nbytes / t_upd / 1e9 if t_upd > 0 else None,
                     "busbw_gbs": 2.0 * (world - 1) / world * nbytes / t_upd / 1e9 if t_upd > 0 else None,
                     "peak_gbs": 900.0, "peak_source": "NVLink 5 per direction per GPU (nominal)",
                     "note": "chain time includes the Updater and NCCL launch/wait; busbw = 2(K-1)/K x bytes / chain time"}

    # ---------------- end-to-end through the public host-buffer entry ----------------
    # (a) synchronous host API: copy in, step, loss out, wait -- every call;
    # (b) the pipelined host API (sg_train_one_batch_host_async): the same copies
    #     and loss read-back per step, the next step's input copy overlapping the
    #     current step's compute, one wait at the end.  (b) is the reported value.
    e2e_steps = min(args.steps, 100)
    loss_h = torch.zeros(e2e_steps, dtype=torch.float32).pin_memory()

    def e2e_run(async_api):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for t in range(e2e_steps):
            j = t % npool
            xp = C.c_void_p(xs_h[j].data_ptr())
            lp = C.c_void_p(ls_h[j].data_ptr()) if has_labels else None
            if async_api:
                L.sg_train_one_batch_host_async(n.h, n.upd, t, xp, lp, C.c_void_p(loss_h[t:].data_ptr()), sp)
            else:
                lh = C.c_float()
                L.sg_train_one_batch_host(n.h, n.upd, t, xp, lp, C.byref(lh), sp)
        if async_api:
            n.sync()
            torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
        if world > 1:
            t_ = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
            dist.all_reduce(t_, op=dist.ReduceOp.MAX)
            e2e_s = float(t_.item())
        return b * e2e_steps / e2e_s

    e2e_sync = e2e_run(False)
    e2e_pipe = e2e_run(True)
    if not np.isfinite(loss_h.numpy()).all():
        raise RuntimeError("non-finite loss read back by the pipelined host path")
    e2e = {"value": e2e_pipe, "unit": "images/s",
           "api": "sg_train_one_batch_host_async (pinned host inputs copied in and loss read back every step; "
                  "the next step's copy overlaps the current step)",
           "sync_api_value": e2e_sync,
           "h2d_bytes_per_step": int(xs_h[0].numel() * 4 + (ls_h[0].numel() * 4 if has_labels else 0)),
           "d2h_bytes_per_step": 4}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, done, _ = cpu_oracle_rate(net_cfg, PER_GPU_BATCH[args.config] if args.config != "alexnet" else 4, 12.0)
        cpu = {"value": rate, "unit": "images/s", "cores": blas_threads(), "kind": "oracle",
               "sample": f"{args.config} b={PER_GPU_BATCH[args.config] if args.config != 'alexnet' else 4}, "
                         f"{done} float64 oracle steps on {len(os.sched_getaffinity(0))} visible host cores"}

    if rank == 0:
        line = {"metric": "training images/sec", "value": value, "unit": "images/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
                "higher_is_better": True, "scaling": SCALING[args.config], "vs_baseline": None, "dtype": "tf32",
                "data": "synthetic",
                "config": {"workload": args.config, "global_batch": b, "per_gpu_batch": b // world if weak else None,
                           "parallelism": f"dp{world}" if args.config in ("cifar10", "mlp", "alexnet_dp") else f"hybrid{world}",
                           "l2": "flushed (256 MB write) before every timed step",
                           "graph": not args.no_graph, "final_loss": final_loss,
                           "exchange": args.exchange if world > 1 else None, "overlap": not args.no_overlap},
                "roofline": roof, "grad_sync": grad_sync, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches * args.steps),
                "clocks": clocks,
                "ops": [{k: (round(v, 5) if isinstance(v, float) else v) for k, v in o.items()} for o in ops[:12]],
                "ops_total_ms": prof_total}
        print(json.dumps(line), flush=True)
    n.close()
    cluster.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
