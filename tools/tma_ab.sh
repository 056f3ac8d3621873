#!/bin/bash
# A/B of the TMA operand paths per operation (SG_TMA_OPS bits, see ops_gemm.cu)
for ops in 0x1f 0x1b 0x1e 0x1d 0x17; do
  for cfg in "$@"; do
    SG_TMA_OPS=$((ops)) timeout 300 python bench.py --config $cfg --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
    python - "$ops" "$cfg" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
ops = {o["op"]: o["ms"] for o in d["ops"]}
w = {k: round(v * 1e3, 1) for k, v in ops.items() if k.startswith("conv") and not k.endswith("update")}
print(sys.argv[1], sys.argv[2], "%.0f img/s" % d["value"], w)
PY
  done
done
