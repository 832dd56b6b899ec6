#!/bin/bash
# k_check_small variants on C5 (min blocks per SM x tiny-loop unroll)
mkdir -p gpurun_out
T=r02k
B="--no-cpu-baseline --no-per-config --no-registry-rate --no-e2e"
for V in "1 4" "4 4" "1 8" "3 8" "4 2"; do
  set -- $V
  CG_NVCC_EXTRA="-DCG_SMALL_MINB=$1 -DCG_TINY_UNROLL=$2" python paper_1310_0901_b200/build.py --force > gpurun_out/build_${T}_$1_$2.log 2>&1
  timeout 300 python bench.py --config c5_sharded --steps 10 --warmup 3 $B > gpurun_out/c5_${T}_$1_$2.json 2>> gpurun_out/ab_$T.err
done
python paper_1310_0901_b200/build.py --force > /dev/null 2>&1
