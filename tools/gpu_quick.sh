#!/bin/bash
# quick: build, a test selection, C2 / C5 / C2-2bit bench lines
mkdir -p gpurun_out
T=${1:-q}
python paper_1310_0901_b200/build.py > gpurun_out/build_$T.log 2>&1
timeout 900 python -m pytest tests/ -q -m gpu -x -k "${2:-tiny_traces or test_gpu_parity or medium_fused or c5_scaled}" > gpurun_out/pytest_sel_$T.log 2>&1
echo "sel rc=$?" >> gpurun_out/pytest_sel_$T.log
B="--no-cpu-baseline --no-per-config --no-registry-rate --no-e2e"
timeout 300 python bench.py --steps 20 --warmup 3 $B > gpurun_out/c2_$T.json 2>> gpurun_out/sweep_$T.err
timeout 300 python bench.py --config c5_sharded --steps 10 --warmup 3 $B > gpurun_out/c5_$T.json 2>> gpurun_out/sweep_$T.err
timeout 300 python bench.py --shadow 2bit --steps 20 --warmup 3 $B > gpurun_out/c2x_$T.json 2>> gpurun_out/sweep_$T.err
