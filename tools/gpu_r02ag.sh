#!/bin/bash
# captures of the C5 path's prep (separate kernel above 4M descriptors) and k_finish
mkdir -p gpurun_out
T=r02ag
python paper_1310_0901_b200/build.py --force > gpurun_out/build_$T.log 2>&1
B="--no-cpu-baseline --no-registry-rate --no-e2e --no-per-config"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:k_check_prep --launch-skip 2 -c 1 -o gpurun_out/prep_c5_$T python bench.py --config c5_sharded --steps 2 --warmup 1 $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:k_finish --launch-skip 2 -c 1 -o gpurun_out/finish_c5_$T python bench.py --config c5_sharded --steps 2 --warmup 1 $B > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name 'regex:k_front|k_check|k_finish|k_leak|k_scan|k_plan' -c 40 --csv --log-file gpurun_out/launches_c5_$T.csv python bench.py --config c5_sharded --steps 2 --warmup 1 $B > /dev/null 2>&1
