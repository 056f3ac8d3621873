#!/bin/bash
# Usage (on the GPU box): bash tools/ncu_round.sh <tag> [kernel-regex] [bench args...]
# 1) plain run, 2) launch list (gpu__time_duration per launch), 3) --set full on the top kernel.
set -u
TAG=$1; KRE=${2:-gemm_tc_kernel}; shift 2 || true
ARGS="--steps 3 --warmup 3 --no-cpu-baseline --profile-steps 1 $*"
mkdir -p gpurun_out
python bench.py $ARGS > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err || { echo "plain run failed"; tail gpurun_out/${TAG}_plain.err; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py $ARGS > gpurun_out/${TAG}_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$KRE" -s ${NCU_SKIP:-5} -c 1 \
    -o gpurun_out/${TAG}_full python bench.py $ARGS > gpurun_out/${TAG}_ncu2.log 2>&1
echo done
