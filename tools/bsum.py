"""Print a compact summary of bench.py JSON lines (tools only)."""
import json
import sys

for f in sys.argv[1:]:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    r = d.get("roofline") or {}
    print(f, round(d["value"]), f'{d["ms_per_step"]*1000:.1f} us/step', r.get("kernel"), round(r.get("frac", 0), 3),
          "e2e", round(d["e2e"]["value"]), "launches/step", d["gpu_launches"] // d["steps"])
    for o in d["ops"][:14]:
        print(f'    {o["op"]:<16} {o["ms"]*1000:7.1f} us')
    print("    ops_total", round(d["ops_total_ms"] * 1000, 1), "us")
