#!/bin/bash
# one GPU session: selected tests first, then the whole -m gpu suite, then the default bench
# usage: tools/gpu_round.sh TAG [pytest -k expression for the first pass]
TAG=${1:-x}
K=${2:-}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$TAG.txt 2>&1
python -c "from paper_1310_0901_b200 import build; build.build()" > gpurun_out/build_$TAG.log 2>&1
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests/ -q -m gpu -k "$K" -x > gpurun_out/pytest_sel_$TAG.log 2>&1
  echo "sel rc=$?" >> gpurun_out/pytest_sel_$TAG.log
fi
timeout 1500 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
