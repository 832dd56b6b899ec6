#!/bin/bash
mkdir -p gpurun_out
T=r02g
python paper_1310_0901_b200/build.py > gpurun_out/build_$T.log 2>&1
timeout 900 python -m pytest tests/ -q -m gpu -x -k "tiny_traces or test_gpu_parity or r10 or next4 or medium or c5_scaled" > gpurun_out/pytest_sel_$T.log 2>&1
echo "sel rc=$?" >> gpurun_out/pytest_sel_$T.log
B="--no-cpu-baseline --no-per-config --no-registry-rate --no-e2e"
for SB in 0 4096; do
  CG_SMALL_BYTES=$SB timeout 300 python bench.py --steps 20 --warmup 3 $B > gpurun_out/c2_sb${SB}_$T.json 2>> gpurun_out/sweep_$T.err
  CG_SMALL_BYTES=$SB timeout 300 python bench.py --config c5_sharded --steps 10 --warmup 3 $B > gpurun_out/c5_sb${SB}_$T.json 2>> gpurun_out/sweep_$T.err
  CG_SMALL_BYTES=$SB timeout 300 python bench.py --shadow 2bit --steps 20 --warmup 3 $B > gpurun_out/c2x_sb${SB}_$T.json 2>> gpurun_out/sweep_$T.err
done
CG_LOOKUP64=0 CG_SMALL_BYTES=4096 timeout 300 python bench.py --config c5_sharded --steps 10 --warmup 3 $B > gpurun_out/c5_lk0_$T.json 2>> gpurun_out/sweep_$T.err
CG_SMALL_BYTES=4096 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:"k_front|k_check|k_finish|k_leak|k_apply" -c 300 --csv --log-file gpurun_out/launches_c5_sb4096_$T.csv python bench.py --config c5_sharded --steps 1 --warmup 1 $B > /dev/null 2>&1
CG_SMALL_BYTES=4096 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:k_check_small --launch-skip 3 -c 1 -o gpurun_out/small_c5_$T python bench.py --config c5_sharded --steps 1 --warmup 1 $B > gpurun_out/ncu_small_c5_$T.log 2>&1
