#!/bin/bash
# Launch list (every kernel, device time) of a short bench run.
# usage: bash tools/ncu_launches.sh <tag> [bench args...]
TAG=${1:-r01}; shift
ARGS=${@:---steps 3 --warmup 1 --no-e2e --no-cpu-baseline --no-registry-rate}
mkdir -p gpurun_out
python bench.py $ARGS > gpurun_out/plain_launch_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py $ARGS > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "ncu rc=$?"
