#!/bin/bash
# bench lines for several configs / GPU counts (run on the GPU box)
TAG=$1; shift
NG=$(nvidia-smi -L | wc -l)
mkdir -p gpurun_out
for spec in "$@"; do
  cfg=${spec%:*}; n=${spec#*:}
  [ "$n" -gt "$NG" ] && continue
  if [ "$n" = 1 ]; then
    timeout 900 python bench.py --config $cfg --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/${TAG}_${cfg}_n1.json 2> gpurun_out/${TAG}_${cfg}_n1.err
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29620 \
      bench.py --gpus $n --config $cfg --steps 100 --warmup 10 > gpurun_out/${TAG}_${cfg}_n$n.json 2> gpurun_out/${TAG}_${cfg}_n$n.err
  fi
  echo "$cfg n=$n rc=$?"; python -c "
import json,sys
try:
  d=json.loads(open('gpurun_out/${TAG}_${cfg}_n$n.json').read().strip().splitlines()[-1])
  r=d['roofline']; print(' value %.0f img/s  ms/step %.3f  e2e %.0f  top %s %.3f ms frac %.4f'%(d['value'],d['ms_per_step'],d['e2e']['value'],r['kernel'],r['kernel_ms'],r['frac']))
except Exception as e: print(' parse error', e); print(open('gpurun_out/${TAG}_${cfg}_n$n.err').read()[-1500:])
"
done
