"""SASS instruction-class count of the shipped library (tools only).
Usage: python tools/sass_classes.py [lib] > profiles/r02_sass_classes.md
Counts, per kernel, the static tcgen05 / TMA / async-copy instructions that prove
the path: UTCHMMA (tcgen05.mma), UTCBAR (tcgen05.commit), LDTM (tcgen05.ld),
UTMALDG / UTMASTG (TMA tensor load / store), UBLKCP (bulk copy), LDGSTS
(cp.async), ELECT (elect.sync), HMMA (legacy mma.sync: must be 0)."""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_1603_07846_b200", "libsinga_b200.so")
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
KEYS = ["UTCHMMA", "UTCBAR", "LDTM", "UTMALDG", "UTMASTG", "UBLKCP", "LDGSTS", "ELECT", "HMMA"]
funcs = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = collections.Counter()
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
    if m and cur:
        funcs[cur][m.group(2).split(".")[0]] += 1
names = subprocess.run(["c++filt"], input="\n".join(funcs), capture_output=True, text=True).stdout.splitlines()
tot = collections.Counter()
for c in funcs.values():
    tot.update({k: c[k] for k in KEYS})
print(f"# SASS instruction classes of `{os.path.relpath(lib, ROOT)}` (sm_100a)\n")
print(f"{len(funcs)} kernels.  Totals: " + ", ".join(f"{k} {tot[k]}" for k in KEYS) + "\n")
print("| kernel | " + " | ".join(KEYS) + " |")
print("|---|" + "---|" * len(KEYS))
for (f, c), n in zip(funcs.items(), names):
    if not any(c[k] for k in ("UTCHMMA", "UTMALDG", "UBLKCP", "LDGSTS")):
        continue
    n = re.sub(r"\(anonymous namespace\)::|sg::", "", n.split("(sg::")[0])[:90]
    print(f"| `{n}` | " + " | ".join(str(c[k]) for k in KEYS) + " |")
