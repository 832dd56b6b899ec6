#!/bin/bash
# ring consume: edge units masked in the fast loop (no warp-wide edge passes)
mkdir -p gpurun_out
T=r02ab
python paper_1310_0901_b200/build.py --force > gpurun_out/build_$T.log 2>&1
B="--no-cpu-baseline --no-registry-rate --no-e2e --no-per-config"
run() { tag=$1; shift; echo "== $tag" >> gpurun_out/sweep_$T.txt; timeout 300 env "$@" >> gpurun_out/sweep_$T.txt 2>> gpurun_out/sweep_$T.err; }
run c2 python bench.py --steps 20 --warmup 3 $B
run c4 python bench.py --config c4_pitched --steps 4 --warmup 3 $B
run c5 python bench.py --config c5_sharded --steps 10 --warmup 3 $B
run c3 python bench.py --config c3_single --steps 20 --warmup 3 $B
run c2_unfused python bench.py --unfused --steps 20 --warmup 3 $B
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_medium.py tests/test_gpu_r10.py tests/test_gpu_sharded.py tests/test_gpu_fullsize.py -q -m gpu -x -k "not c5_full" > gpurun_out/pytest_$T.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$T.log
