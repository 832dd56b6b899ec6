#!/bin/bash
# separate prep + plan kernels above 4M descriptors; the single fused C5 batch at full size vs the oracle
mkdir -p gpurun_out
T=r02z
python paper_1310_0901_b200/build.py --force > gpurun_out/build_$T.log 2>&1
B="--no-cpu-baseline --no-registry-rate --no-e2e --no-per-config"
run() { tag=$1; shift; echo "== $tag" >> gpurun_out/sweep_$T.txt; timeout 300 env "$@" >> gpurun_out/sweep_$T.txt 2>> gpurun_out/sweep_$T.err; }
run c5 python bench.py --config c5_sharded --steps 10 --warmup 3 $B
run c2 python bench.py --steps 20 --warmup 3 $B
run c2_nocoop CG_FRONT_COOP=0 python bench.py --steps 20 --warmup 3 $B
timeout 1800 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_medium.py -q -m gpu -x -k "c5_full_fused or front_split or pingpong" > gpurun_out/pytest_$T.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$T.log
