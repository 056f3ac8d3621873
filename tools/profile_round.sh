#!/bin/bash
# Round profile evidence (run on the GPU box):  bash tools/profile_round.sh <tag> <config> <kernel-regex>
#  1) default-style bench line (with cpu_baseline) -> gpurun_out/<tag>_bench.json
#  2) ncu launch list of the same command (gpu__time_duration per launch)
#  3) ncu --set full on the kernels matching <kernel-regex> (one launch each, steady state)
set -u
TAG=$1; CFG=$2; KRE=$3
mkdir -p gpurun_out
timeout 900 python bench.py --config $CFG > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err || { echo "bench failed"; tail gpurun_out/${TAG}_bench.err; exit 1; }
ARGS="--config $CFG --steps 3 --warmup 3 --no-cpu-baseline --profile-steps 1"
timeout 900 python bench.py $ARGS > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err || { echo "plain run failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py $ARGS > gpurun_out/${TAG}_ncu1.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$KRE" -s ${NCU_SKIP:-8} -c ${NCU_COUNT:-2} \
    -o gpurun_out/${TAG}_full python bench.py $ARGS > gpurun_out/${TAG}_ncu2.log 2>&1
tail -1 gpurun_out/${TAG}_ncu2.log
echo done
