"""Write the round's profile evidence into profiles/ (run here after the GPU calls):
bench lines, the ncu launch list aggregated per kernel (and the raw CSV), the key
`ncu --set full` metrics of the captured kernels, and profiles/traffic.json
(dram bytes per launch, read by bench.py for roofline.traffic)."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from launches import load, short  # noqa: E402

KEYS = ["gpu__time_duration.sum", "launch__grid_size", "launch__registers_per_thread",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active"]


def ncu_rows(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    return [(dict(zip(h, r)), dict(zip(h, u))) for r in rows[2:]]


def to_bytes(v, unit):
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main(tag, cfg, rep, launches, bench, op_of_kernel):
    out = [f"# Round 1 profile evidence: {cfg} ({tag})", "",
           "Produced by tools/profile_round.sh on a B200 and tools/write_profiles.py here.", ""]
    b = json.loads(open(bench).read().strip().splitlines()[-1])
    json.dump(b, open(os.path.join(ROOT, "profiles", f"r01_{cfg}_bench.json"), "w"), indent=1)
    out += [f"bench: {b['value']:.0f} {b['unit']}, {b['ms_per_step'] * 1e3:.1f} us/step, roofline {b['roofline']['kernel']} "
            f"frac {b['roofline']['frac']:.4f} ({b['roofline']['bound']}), e2e {b['e2e']['value']:.0f}", ""]
    # launch list
    agg = {}
    for r in load(launches):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = short(r["Kernel Name"])
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += float(r["Metric Value"]) / 1e3
    tot = sum(v[1] for v in agg.values())
    out += ["## Launch list (ncu gpu__time_duration.sum, --clock-control none; cold, serialised)", "",
            "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{k}` | {n} | {t:.1f} | {100 * t / tot:.1f}% |")
    out.append("")
    subprocess.run(["cp", launches, os.path.join(ROOT, "profiles", f"r01_{cfg}_launches.csv")])
    # full-set metrics
    traffic_path = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    out += ["## ncu --set full (one steady-state launch each)", ""]
    for d, u in ncu_rows(rep):
        name = d.get("Kernel Name", "?")
        out.append(f"### `{name[:100]}`")
        for k in KEYS:
            if k in d:
                out.append(f"- {k}: {d[k]} {u.get(k, '')}")
        for frag, op in op_of_kernel.items():
            if frag in name:
                traffic[f"{cfg}:{op}"] = to_bytes(d["dram__bytes_read.sum"], u["dram__bytes_read.sum"]) + \
                    to_bytes(d["dram__bytes_write.sum"], u["dram__bytes_write.sum"])
        out.append("")
    json.dump(traffic, open(traffic_path, "w"), indent=1, sort_keys=True)
    open(os.path.join(ROOT, "profiles", f"r01_{cfg}_summary.md"), "w").write("\n".join(out) + "\n")
    print("\n".join(out[:8]))


if __name__ == "__main__":
    # usage: write_profiles.py TAG CONFIG  'kernel-fragment=op,...'
    tag, cfg = sys.argv[1], sys.argv[2]
    ops = dict(kv.split("=") for kv in sys.argv[3].split(",")) if len(sys.argv) > 3 else {}
    main(tag, cfg, f"gpurun_out/{tag}_full.ncu-rep", f"gpurun_out/{tag}_launches.csv", f"gpurun_out/{tag}_bench.json", ops)
