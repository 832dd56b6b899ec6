#!/bin/bash
# CG_APPLY_LAST: ping-pong parity, fused-path suites, C5 at one batch, k_front capture
mkdir -p gpurun_out
T=r02m
python paper_1310_0901_b200/build.py --force > gpurun_out/build_$T.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_medium.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -m gpu -x > gpurun_out/pytest_$T.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$T.log
B="--no-cpu-baseline --no-registry-rate --no-e2e"
timeout 600 python bench.py --steps 10 --warmup 3 $B --no-interleaved > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
K='regex:k_front|k_check|k_finish|k_leak|k_apply|k_prop|k_wave'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name "$K" -c 100 --csv --log-file gpurun_out/launches_c5_$T.csv python bench.py --config c5_sharded --steps 1 --warmup 1 $B --no-per-config > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:k_front --launch-skip 1 -c 1 -o gpurun_out/front_c5_$T python bench.py --config c5_sharded --steps 1 --warmup 1 $B --no-per-config > /dev/null 2>&1
