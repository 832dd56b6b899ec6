#!/bin/bash
# new small pass / apply-after / sharded library path: tests, benches, C5 launch list
mkdir -p gpurun_out
T=r02d
python paper_1310_0901_b200/build.py > gpurun_out/build_$T.log 2>&1
timeout 600 python -m pytest tests/ -q -m gpu -x -k "sharded or r10 or toy or listing or tiny_traces" > gpurun_out/pytest_sel_$T.log 2>&1
echo "sel rc=$?" >> gpurun_out/pytest_sel_$T.log
timeout 300 python bench.py --config c5_sharded --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-registry-rate > gpurun_out/bench_c5_$T.json 2> gpurun_out/bench_c5_$T.err
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/bench_c2_$T.json 2> gpurun_out/bench_c2_$T.err
timeout 400 python bench.py --sharded --steps 10 --warmup 3 > gpurun_out/bench_sharded1_$T.json 2> gpurun_out/bench_sharded1_$T.err
timeout 400 python bench.py --loopback 4 --steps 10 --warmup 3 > gpurun_out/bench_loop4_$T.json 2> gpurun_out/bench_loop4_$T.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5_$T.csv python bench.py --config c5_sharded --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-registry-rate > gpurun_out/ncu_c5_$T.log 2>&1
timeout 2400 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu_$T.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$T.log
