#!/bin/bash
# Per-launch device times of one bench step (tools/launchlist.sh <config> <tag>)
CFG=${1:-c4}; TAG=${2:-x}; EXTRA=${3:-}
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline $EXTRA"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_$TAG.json 2> gpurun_out/plain_$TAG.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "launchlist rc=$?"
