"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel."""
import collections
import csv
import re
import sys


def load(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    return list(csv.DictReader(lines[start:]))


def short(n):
    n = re.sub(r"\(.*", "", n).replace("void ", "").replace("sg::", "").replace("(anonymous namespace)::", "")
    m = re.match(r"gemm_tc_kernel<(\d+), (\d+), (\w+), (\w+)>", n)
    if m:
        return f"gemm_tc<BN={m.group(1)},{m.group(3)},{m.group(4)}>"
    return n[:80]


def main(path, per=1):
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in load(path):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = short(r["Kernel Name"])
        agg[k][0] += 1
        agg[k][1] += float(r["Metric Value"]) / 1e3
    tot = sum(v[1] for v in agg.values())
    print(f"{'us':>10} {'share':>6} {'launches':>8}  kernel")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{v[1] / per:10.1f} {100 * v[1] / tot:5.1f}% {v[0]:8d}  {k}")
    print(f"total {tot / per:.1f} us")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)
