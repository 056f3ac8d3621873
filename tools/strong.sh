#!/bin/bash
# A21: CIFAR-10 global batch fixed at 128 (strong scaling) next to the per-GPU-128 weak series
mkdir -p gpurun_out
python bench.py --steps 50 --warmup 10 --no-cpu-baseline --batch 128 > gpurun_out/${1}_cifar_strong_n1.json 2>/dev/null
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29800 + N)) \
    bench.py --gpus $N --steps 50 --warmup 10 --no-cpu-baseline --batch 128 > gpurun_out/${1}_cifar_strong_n${N}.json 2>/dev/null
done
echo done
