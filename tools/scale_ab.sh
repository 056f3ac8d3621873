#!/bin/bash
# Multi-GPU bench lines, NCCL chain vs fused peer-memory exchange (run on a box with >= N GPUs):
#   bash tools/scale_ab.sh <tag> <N...>
TAG=$1; shift
mkdir -p gpurun_out
for N in "$@"; do
  for CFG in cifar10 alexnet; do
    for EX in nccl p2p; do
      timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
        --master-port $((29500 + N)) bench.py --gpus $N --config $CFG --exchange $EX --steps 50 --warmup 10 \
        > gpurun_out/${TAG}_${CFG}_n${N}_${EX}.json 2> gpurun_out/${TAG}_${CFG}_n${N}_${EX}.err || echo "fail $CFG $N $EX"
    done
  done
done
echo done
