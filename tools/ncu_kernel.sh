#!/bin/bash
# Usage: bash tools/ncu_kernel.sh <tag> <demangled-name-regex> <skip> [bench args]
TAG=$1; KRE=$2; SKIP=$3; shift 3
ARGS="--steps 2 --warmup 3 --no-cpu-baseline --profile-steps 1 --no-graph $*"
mkdir -p gpurun_out
python bench.py $ARGS > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err || { echo plain run failed; tail gpurun_out/${TAG}_plain.err; exit 1; }
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$KRE" -s $SKIP -c 1 \
    -o gpurun_out/${TAG} python bench.py $ARGS > gpurun_out/${TAG}_ncu.log 2>&1
tail -2 gpurun_out/${TAG}_ncu.log
