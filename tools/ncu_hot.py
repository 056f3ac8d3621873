"""Top SASS instructions by warp-stall samples from an ncu report (source page)."""
import csv
import io
import os
import subprocess
import sys


def main(path, kregex=None, top=30):
    cmd = ["ncu", "-i", os.path.abspath(path), "--page", "source", "--csv", "--print-source", "sass"]
    if kregex:
        cmd += ["--kernel-name-base", "demangled", "-k", "regex:" + kregex]
    out = subprocess.run(cmd, capture_output=True, text=True, cwd="/tmp").stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = next(r for r in rows if "Source" in r and "Address" in r)
    iS, iE = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")

    def f(x):
        try:
            return float(x)
        except ValueError:
            return None
    seen, d = set(), []
    for r in rows:
        if len(r) > iS and f(r[iS]) is not None and r[0] not in seen:
            seen.add(r[0])
            d.append(r)
    tot = sum(f(r[iS]) for r in d) or 1
    print(f"{path}: {tot:.0f} samples, {len(d)} instructions")
    for i in sorted(sorted(range(len(d)), key=lambda i: -f(d[i][iS]))[:top]):
        r = d[i]
        print(f"{i:6d} {100 * f(r[iS]) / tot:5.1f}% {r[iE]:>9s}  {r[1][:110]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None, int(sys.argv[3]) if len(sys.argv) > 3 else 30)
