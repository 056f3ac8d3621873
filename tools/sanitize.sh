#!/bin/bash
# compute-sanitizer (memcheck / racecheck / synccheck) over every tcgen05 / TMA /
# mbarrier kernel family of the library at tiny shapes (run on the GPU box):
#   bash tools/sanitize.sh  -> gpurun_out/sanitize_<tool>.log
mkdir -p gpurun_out
SEL="not implicit and not peer_sync"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 99 \
    python -m pytest tests/test_gpu_ops.py -q -p no:cacheprovider -k "$SEL" > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit $?" | tee -a gpurun_out/sanitize_$tool.log
done
# the whole CIFAR-10 step (fused conv1 backward, resident-image kernels, graph replay) at batch 2
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 99 \
    python -m pytest tests/test_gpu_net.py -q -p no:cacheprovider -k "test_layer_isolated_tiny_conv_ragged or test_layer_isolated_fused_graph or test_layer_isolated_exercised_collectives" \
    > gpurun_out/sanitize_net_$tool.log 2>&1
  echo "$tool exit $?" | tee -a gpurun_out/sanitize_net_$tool.log
done
