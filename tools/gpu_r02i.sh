#!/bin/bash
mkdir -p gpurun_out
T=r02i
python paper_1310_0901_b200/build.py > gpurun_out/build_$T.log 2>&1
timeout 900 python -m pytest tests/ -q -m gpu -x -k "tiny_traces or test_gpu_parity or r10 or medium or c5_scaled or next1" > gpurun_out/pytest_sel_$T.log 2>&1
echo "sel rc=$?" >> gpurun_out/pytest_sel_$T.log
B="--no-cpu-baseline --no-per-config --no-registry-rate --no-e2e"
timeout 300 python bench.py --steps 20 --warmup 3 $B > gpurun_out/c2_$T.json 2>> gpurun_out/sweep_$T.err
timeout 300 python bench.py --config c5_sharded --steps 10 --warmup 3 $B > gpurun_out/c5_$T.json 2>> gpurun_out/sweep_$T.err
timeout 300 python bench.py --shadow 2bit --steps 20 --warmup 3 $B > gpurun_out/c2x_$T.json 2>> gpurun_out/sweep_$T.err
timeout 300 python bench.py --config c4_pitched --steps 5 --warmup 3 $B > gpurun_out/c4_$T.json 2>> gpurun_out/sweep_$T.err
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:k_front --launch-skip 8 -c 1 -o gpurun_out/front_c5_$T python bench.py --config c5_sharded --steps 2 --warmup 1 $B > gpurun_out/ncu_front_c5_$T.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:k_check_small --launch-skip 9 -c 1 -o gpurun_out/small_c5_$T python bench.py --config c5_sharded --steps 2 --warmup 1 $B > gpurun_out/ncu_small_c5_$T.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:k_check_scan --launch-skip 2 -c 1 -o gpurun_out/scan_c4_$T python bench.py --config c4_pitched --steps 1 --warmup 1 $B > gpurun_out/ncu_scan_c4_$T.log 2>&1
