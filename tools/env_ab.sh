#!/bin/bash
# A/B of an environment toggle on the bench configs:  bash tools/env_ab.sh VAR "v1 v2" cfg...
VAR=$1; VALS=$2; shift 2
for v in $VALS; do
  tag=$(echo "$v" | tr "/." "__")
  for cfg in "$@"; do
    env $VAR=$v timeout 300 python bench.py --config $cfg --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/ab_${tag}_${cfg}.json 2>gpurun_out/ab.err || tail -5 gpurun_out/ab.err
    python - "$VAR=$v" "$cfg" "gpurun_out/ab_${tag}_${cfg}.json" <<'PY'
import json, sys
d = json.loads(open(sys.argv[3]).read().strip().splitlines()[-1])
top = ", ".join("%s %.1f" % (o["op"], o["ms"] * 1e3) for o in d["ops"][:6])
print(sys.argv[1], sys.argv[2], "%.0f img/s  %.3f ms/step  e2e %.0f | %s" % (d["value"], d["ms_per_step"], d["e2e"]["value"], top))
PY
  done
done
