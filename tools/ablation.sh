#!/bin/bash
# §5.4 ablations (run on a 4-GPU box):
#  E9 analogue: AlexNet hybrid (dim-0 conv, dim-1 FC) vs pure data
#     parallelism at K = 2 / 4 over the global batch b in {64, 128, 256, 512};
#  E8 analogue: overlap of Update with the backward on / off.
mkdir -p gpurun_out
for N in 2 4; do
  for B in 64 128 256 512; do
    for CFG in alexnet alexnet_dp; do
      timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
        --master-port $((29600 + N)) bench.py --gpus $N --config $CFG --batch $B --steps 20 --warmup 5 \
        --no-cpu-baseline --profile-steps 5 > gpurun_out/abl_${CFG}_n${N}_b${B}.json 2> gpurun_out/abl_${CFG}_n${N}_b${B}.err \
        || echo "fail $CFG $N $B"
    done
  done
  for CFG in cifar10 alexnet; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29700 + N)) bench.py --gpus $N --config $CFG --steps 30 --warmup 5 --no-cpu-baseline \
      --profile-steps 5 --no-overlap > gpurun_out/abl_${CFG}_n${N}_nooverlap.json 2> gpurun_out/abl_${CFG}_n${N}_nooverlap.err \
      || echo "fail nooverlap $CFG $N"
  done
done
echo done
