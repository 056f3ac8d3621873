#!/bin/bash
# Round bench evidence (1 GPU): default bench line (with cpu_baseline), other workloads,
# the reference arm, the CIFAR-10 launch list and ncu --set full captures of the
# dominant CIFAR-10 and AlexNet kernels (exported to CSV / text on the box; the
# .ncu-rep files stay there).
mkdir -p gpurun_out
python bench.py > gpurun_out/r02_cifar10_bench.json 2> gpurun_out/r02_cifar10_bench.err
for c in alexnet alexnet_dp mlp ae ae_wide; do
  python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r02_${c}_bench.json 2>/dev/null
done
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02_cifar10_reference_arm.json 2>/dev/null
ARGS="--steps 3 --warmup 3 --no-cpu-baseline --profile-steps 1"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_cifar10_launches.csv \
  python bench.py $ARGS > /dev/null 2>&1
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size
mkdir -p /tmp/ncu
ncu --set full --clock-control none --import-source on \
  -k "regex:conv_img_wgrad_kernel|conv_img4_wgrad_kernel|conv_img4_fwd|conv_img_kernel|pool_lrn_fwd" -s 12 -c 6 \
  -o /tmp/ncu/cifar python bench.py $ARGS --no-graph > /dev/null 2>&1
ncu -i /tmp/ncu/cifar.ncu-rep --page raw --csv --metrics $M > gpurun_out/r02_cifar10_full_raw.csv 2>&1
ncu -i /tmp/ncu/cifar.ncu-rep --page details > gpurun_out/r02_cifar10_full_details.txt 2>&1
ncu --set full --clock-control none -k "regex:gemm_tc_kernel" -s 69 -c 23 \
  -o /tmp/ncu/alex python bench.py --config alexnet $ARGS --no-graph > /dev/null 2>&1
ncu -i /tmp/ncu/alex.ncu-rep --page raw --csv --metrics $M > gpurun_out/r02_alexnet_full_raw.csv 2>&1
echo done
