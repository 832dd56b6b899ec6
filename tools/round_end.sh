#!/bin/bash
# full GPU test suite, the default bench line, launch list and one ncu capture of the scan
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
bash tools/ncu_launches.sh $TAG --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --no-registry-rate
bash tools/ncu_scan.sh $TAG k_check_scan
