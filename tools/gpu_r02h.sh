#!/bin/bash
mkdir -p gpurun_out
T=r02h
python paper_1310_0901_b200/build.py > gpurun_out/build_$T.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
B="--no-cpu-baseline --no-per-config --no-registry-rate --no-e2e"
timeout 300 python bench.py --shadow 2bit --steps 20 --warmup 3 $B > gpurun_out/c2x_$T.json 2>> gpurun_out/sweep_$T.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:"k_front|k_check|k_finish|k_leak|k_apply" -c 300 --csv --log-file gpurun_out/launches_c5_$T.csv python bench.py --config c5_sharded --steps 1 --warmup 1 $B > /dev/null 2>&1
timeout 2700 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu_$T.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$T.log
