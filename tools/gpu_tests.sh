#!/bin/bash
# GPU tests only: selected (-k) first, then the full -m gpu suite; logs in gpurun_out/
TAG=${1:-x}
K=${2:-}
mkdir -p gpurun_out
(nproc; free -g; lscpu | head -20) > gpurun_out/host_$TAG.txt 2>&1
python paper_1310_0901_b200/build.py > gpurun_out/build_$TAG.log 2>&1
if [ -n "$K" ]; then
  timeout 1200 python -m pytest tests/ -q -m gpu -k "$K" > gpurun_out/pytest_sel_$TAG.log 2>&1
  echo "sel rc=$?" >> gpurun_out/pytest_sel_$TAG.log
fi
timeout 1800 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
