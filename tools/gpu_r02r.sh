#!/bin/bash
# small pass: 4-warp CTAs with 10 KB stages; correctness at C5 full size (normal build), 2-bit limits, stage sweep
mkdir -p gpurun_out
T=r02r
python paper_1310_0901_b200/build.py --force > gpurun_out/build_$T.log 2>&1
timeout 1500 python tests/diag_c5.py 1 > gpurun_out/diag_$T.txt 2>&1
timeout 900 env CG_SMALL_MODE=1 python -m pytest tests/test_gpu_parity.py tests/test_gpu_medium.py tests/test_gpu_next4.py -q -m gpu -x > gpurun_out/pytest_small_$T.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_small_$T.log
B="--no-cpu-baseline --no-registry-rate --no-e2e --no-per-config"
run() { tag=$1; shift; echo "== $tag" >> gpurun_out/sweep_$T.txt; timeout 300 env "$@" >> gpurun_out/sweep_$T.txt 2>> gpurun_out/sweep_$T.err; }
run c5 python bench.py --config c5_sharded --steps 10 --warmup 3 $B
run c2x python bench.py --shadow 2bit --steps 20 --warmup 3 $B
run c2x_16k_adapt CG_SMALL_BYTES=16384 CG_SMALL_STAT=16384 python bench.py --shadow 2bit --steps 20 --warmup 3 $B
run c2x_16k_on CG_SMALL_MODE=1 CG_SMALL_BYTES=16384 python bench.py --shadow 2bit --steps 20 --warmup 3 $B
run c2x_4k_on CG_SMALL_MODE=1 python bench.py --shadow 2bit --steps 20 --warmup 3 $B
run c2_4k_on CG_SMALL_MODE=1 python bench.py --steps 20 --warmup 3 $B
run c2s_16k_on CG_SMALL_MODE=1 CG_SMALL_BYTES=16384 python bench.py --shadow sparse --steps 20 --warmup 3 $B
CG_NVCC_EXTRA="-DCG_SMALL_THREADS=256 -DCG_SMALL_STAGE=4864 -DCG_SMALL_MINB=4" python paper_1310_0901_b200/build.py --force > gpurun_out/build2_$T.log 2>&1
run c5_256_4864 python bench.py --config c5_sharded --steps 10 --warmup 3 $B
CG_NVCC_EXTRA="-DCG_SMALL_THREADS=64 -DCG_SMALL_STAGE=20480 -DCG_SMALL_MINB=5" python paper_1310_0901_b200/build.py --force > gpurun_out/build3_$T.log 2>&1
run c5_64_20480 python bench.py --config c5_sharded --steps 10 --warmup 3 $B
CG_NVCC_EXTRA="-DCG_SMALL_THREADS=128 -DCG_SMALL_STAGE=7168 -DCG_SMALL_MINB=6" python paper_1310_0901_b200/build.py --force > gpurun_out/build4_$T.log 2>&1
run c5_128_7168 python bench.py --config c5_sharded --steps 10 --warmup 3 $B
python paper_1310_0901_b200/build.py --force > /dev/null 2>&1
