#!/bin/bash
# apply pieces: bulk zero-page stores vs 16-byte stores of all lanes
mkdir -p gpurun_out
T=r02ad
B="--no-cpu-baseline --no-registry-rate --no-e2e --no-per-config"
run() { tag=$1; shift; echo "== $tag" >> gpurun_out/sweep_$T.txt; timeout 300 env "$@" >> gpurun_out/sweep_$T.txt 2>> gpurun_out/sweep_$T.err; }
python paper_1310_0901_b200/build.py --force > gpurun_out/build_$T.log 2>&1
run c4_bulk python bench.py --config c4_pitched --steps 4 --warmup 3 $B
run c2u_bulk python bench.py --unfused --steps 20 --warmup 3 $B
run c5_bulk python bench.py --config c5_sharded --steps 10 --warmup 3 $B
CG_NVCC_EXTRA="-DCG_APPLY_BULK=0" python paper_1310_0901_b200/build.py --force > gpurun_out/build2_$T.log 2>&1
run c4_stg python bench.py --config c4_pitched --steps 4 --warmup 3 $B
run c2u_stg python bench.py --unfused --steps 20 --warmup 3 $B
run c5_stg python bench.py --config c5_sharded --steps 10 --warmup 3 $B
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_medium.py -q -m gpu -x -k "unfused or pitched or medium" > gpurun_out/pytest_$T.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$T.log
python paper_1310_0901_b200/build.py --force > /dev/null 2>&1
