#!/bin/bash
# AlexNet GEMM / conv kernels of one training step: tensor pipe, L2 and DRAM counters (ncu, 1 GPU).
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sectors.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,sm__inst_executed_pipe_uniform.sum \
  --clock-control none -k "regex:gemm_tc_kernel|conv_img" -s 100 -c 60 --csv --log-file gpurun_out/alex_ncu.csv \
  python bench.py --config alexnet --no-graph --steps 3 --warmup 3 --no-cpu-baseline --profile-steps 1 > gpurun_out/alex_ncu.log 2>&1
echo rc=$?
