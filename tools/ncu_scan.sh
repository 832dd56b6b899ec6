#!/bin/bash
# One `ncu --set full` capture of the shadow-scan kernel on the C2 bench step
# (run on the GPU box via gpurun; the plain run must exit 0 first).
# usage: bash tools/ncu_scan.sh <tag> [kernel-regex] [bench args...]
TAG=${1:-scan}; KRE=${2:-k_check_scan}; shift 2
ARGS=${@:---steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-registry-rate}
mkdir -p gpurun_out
python bench.py $ARGS > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$KRE -s 1 -c 1 \
    -o gpurun_out/prof_$TAG python bench.py $ARGS > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?"
