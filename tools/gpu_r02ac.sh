#!/bin/bash
# final evidence: full GPU suite, default bench line, reference arm, per-format lines, launch lists, ncu captures
mkdir -p gpurun_out
T=r02ac
python paper_1310_0901_b200/build.py --force > gpurun_out/build_$T.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref_$T.json 2> gpurun_out/ref_$T.err
B="--no-cpu-baseline --no-per-config --no-registry-rate --no-e2e"
timeout 400 python bench.py --sharded --steps 10 --warmup 3 > gpurun_out/sharded1_$T.json 2> gpurun_out/sharded1_$T.err
timeout 400 python bench.py --loopback 8 --steps 5 --warmup 3 $B > gpurun_out/loop8_$T.json 2> gpurun_out/loop8_$T.err
timeout 300 python bench.py --shadow 2bit --steps 20 --warmup 3 $B > gpurun_out/c2x_$T.json 2>> gpurun_out/sweep_$T.err
timeout 300 python bench.py --shadow sparse --steps 20 --warmup 3 $B > gpurun_out/c2s_$T.json 2>> gpurun_out/sweep_$T.err
timeout 300 python bench.py --track --steps 10 --warmup 3 $B > gpurun_out/c2t_$T.json 2>> gpurun_out/sweep_$T.err
K='regex:k_front|k_check|k_finish|k_leak|k_apply|k_prop|k_wave'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name "$K" -c 300 --csv --log-file gpurun_out/launches_c5_$T.csv python bench.py --config c5_sharded --steps 2 --warmup 1 $B > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name "$K" -c 60 --csv --log-file gpurun_out/launches_c2_$T.csv python bench.py --steps 2 --warmup 1 $B > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name "$K" -c 60 --csv --log-file gpurun_out/launches_c4_$T.csv python bench.py --config c4_pitched --steps 1 --warmup 1 $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:k_check_scan --launch-skip 1 -c 1 -o gpurun_out/scan_c2_$T python bench.py --steps 2 --warmup 1 $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:k_check_small --launch-skip 2 -c 1 -o gpurun_out/small_c5_$T python bench.py --config c5_sharded --steps 2 --warmup 1 $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:k_front --launch-skip 2 -c 1 -o gpurun_out/front_c5_$T python bench.py --config c5_sharded --steps 2 --warmup 1 $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:k_check_scan --launch-skip 1 -c 1 -o gpurun_out/scan_c4_$T python bench.py --config c4_pitched --steps 1 --warmup 1 $B > /dev/null 2>&1
timeout 2700 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu_$T.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1
