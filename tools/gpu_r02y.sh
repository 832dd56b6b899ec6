#!/bin/bash
# 2-bit small-pass limit sweep; C5 prep / plan split (non-cooperative front)
mkdir -p gpurun_out
T=r02y
python paper_1310_0901_b200/build.py --force > gpurun_out/build_$T.log 2>&1
B="--no-cpu-baseline --no-registry-rate --no-e2e --no-per-config"
run() { tag=$1; shift; echo "== $tag" >> gpurun_out/sweep_$T.txt; timeout 300 env "$@" >> gpurun_out/sweep_$T.txt 2>> gpurun_out/sweep_$T.err; }
run c2x python bench.py --shadow 2bit --steps 20 --warmup 3 $B
run c2x_8k CG_SMALL_BYTES=8192 CG_SMALL_STAT=8192 python bench.py --shadow 2bit --steps 20 --warmup 3 $B
run c2x_16k CG_SMALL_BYTES=16384 CG_SMALL_STAT=16384 python bench.py --shadow 2bit --steps 20 --warmup 3 $B
run c2s_16k CG_SMALL_BYTES=16384 CG_SMALL_STAT=16384 python bench.py --shadow sparse --steps 20 --warmup 3 $B
run c2s_8k CG_SMALL_BYTES=8192 CG_SMALL_STAT=8192 python bench.py --shadow sparse --steps 20 --warmup 3 $B
run c5x python bench.py --config c5_sharded --shadow 2bit --steps 10 --warmup 3 $B
run c5_nocoop CG_FRONT_COOP=0 python bench.py --config c5_sharded --steps 10 --warmup 3 $B
timeout 600 env CG_FRONT_COOP=0 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name 'regex:k_check|k_scan|k_plan|k_finish|k_leak' -c 40 --csv --log-file gpurun_out/launches_c5_split_$T.csv python bench.py --config c5_sharded --steps 2 --warmup 1 $B > /dev/null 2>&1
