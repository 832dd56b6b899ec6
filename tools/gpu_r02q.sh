#!/bin/bash
# flattened small pass: verify build on C5 (staged vs global), then the normal build: parity, diag, benches
mkdir -p gpurun_out
T=r02q
CG_NVCC_EXTRA="-DCG_SMALL_VERIFY=1" python paper_1310_0901_b200/build.py --force > gpurun_out/build_v_$T.log 2>&1
timeout 1500 python tests/diag_c5.py 1 > gpurun_out/diag_v_$T.txt 2>&1
python paper_1310_0901_b200/build.py --force > gpurun_out/build_$T.log 2>&1
timeout 900 env CG_SMALL_MODE=1 python -m pytest tests/test_gpu_parity.py tests/test_gpu_medium.py tests/test_gpu_next4.py -q -m gpu -x > gpurun_out/pytest_small_$T.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_small_$T.log
B="--no-cpu-baseline --no-registry-rate --no-e2e --no-per-config"
run() { tag=$1; shift; echo "== $tag" >> gpurun_out/sweep_$T.txt; timeout 300 env "$@" >> gpurun_out/sweep_$T.txt 2>> gpurun_out/sweep_$T.err; }
run c5 python bench.py --config c5_sharded --steps 10 --warmup 3 $B
run c2 python bench.py --steps 20 --warmup 3 $B
run c2x_small CG_SMALL_MODE=1 python bench.py --shadow 2bit --steps 20 --warmup 3 $B
run c2_small CG_SMALL_MODE=1 python bench.py --steps 20 --warmup 3 $B
K='regex:k_front|k_check|k_finish|k_leak|k_apply|k_prop|k_wave'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name "$K" -c 100 --csv --log-file gpurun_out/launches_c5_$T.csv python bench.py --config c5_sharded --steps 2 --warmup 1 $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:k_check_small --launch-skip 2 -c 1 -o gpurun_out/small_c5_$T python bench.py --config c5_sharded --steps 2 --warmup 1 $B > /dev/null 2>&1
