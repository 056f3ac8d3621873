#!/bin/bash
# A/B of programmatic dependent launch (SG_PDL) on the bench configs
for pdl in 0 1; do
  for cfg in "$@"; do
    SG_PDL=$pdl timeout 300 python bench.py --config $cfg --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/pdl_${pdl}_${cfg}.json 2>gpurun_out/pdl.err || tail -5 gpurun_out/pdl.err
    python -c "
import json
d=json.loads(open('gpurun_out/pdl_${pdl}_${cfg}.json').read().strip().splitlines()[-1])
print('pdl=$pdl $cfg %.0f img/s  %.3f ms/step  e2e %.0f' % (d['value'], d['ms_per_step'], d['e2e']['value']))"
  done
done
