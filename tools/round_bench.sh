#!/bin/bash
# Round bench evidence (1 GPU): default bench line (with cpu_baseline), other workloads,
# launch list and ncu --set full of the dominant CIFAR kernel.
mkdir -p gpurun_out
python bench.py > gpurun_out/r02_cifar10_bench.json 2> gpurun_out/r02_cifar10_bench.err
for c in alexnet mlp ae ae_wide; do
  python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r02_${c}_bench.json 2>/dev/null
done
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02_cifar10_reference_arm.json 2>/dev/null
ARGS="--steps 3 --warmup 3 --no-cpu-baseline --profile-steps 1"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_cifar10_launches.csv \
  python bench.py $ARGS > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:conv_img_wgrad_kernel|conv_img4_wgrad_kernel|conv_img4_fwd|pool_lrn_fwd_kernel<1>" -s 8 -c 4 \
  -o gpurun_out/r02_cifar10_full python bench.py $ARGS --no-graph > /dev/null 2>&1
echo done
