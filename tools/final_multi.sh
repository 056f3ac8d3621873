#!/bin/bash
# Final multi-GPU evidence (4 GPUs): full pytest -m gpu (incl. K=2/4 dist), weak / strong scaling lines.
mkdir -p gpurun_out
timeout 1400 python -m pytest tests -m gpu -q -rf --timeout 900 -p no:cacheprovider -s > gpurun_out/t12.log 2>&1
tail -3 gpurun_out/t12.log
bash tools/scale_ab.sh sc7 2 4
bash tools/strong.sh st7
python bench.py --steps 50 --warmup 10 --no-cpu-baseline > gpurun_out/sc7_cifar10_n1.json 2>/dev/null
python bench.py --config alexnet --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/sc7_alexnet_n1.json 2>/dev/null
echo done
