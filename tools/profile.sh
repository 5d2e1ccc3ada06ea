#!/bin/bash
# Profiling recipe (run under gpurun on one B200; /opt/skills/guides/B200_PROFILING.md).
#   tools/profile.sh <config> <tag> [kernel-regex]
# 1. plain run (must exit 0), 2. per-launch device times, 3. --set full on the
# listing kernels. Outputs under gpurun_out/.
set -u
CFG=${1:-rmat20}; TAG=${2:-r01}; KRE=${3:-k_list}
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_$TAG.json 2> gpurun_out/plain_$TAG.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$KRE -c ${4:-6} \
    -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "profile rc=$?"
