#!/bin/bash
# occupancy sweep: prep CTAs per SM, small-pass CTA shapes (C5)
mkdir -p gpurun_out
T=r02ae
B="--no-cpu-baseline --no-registry-rate --no-e2e --no-per-config"
run() { tag=$1; shift; echo "== $tag" >> gpurun_out/sweep_$T.txt; timeout 300 env "$@" >> gpurun_out/sweep_$T.txt 2>> gpurun_out/sweep_$T.err; }
for v in "-DCG_FRONT_MINB=5" "-DCG_SMALL_STAGE=3840" "-DCG_SMALL_STAGE=4352" ""; do
  CG_NVCC_EXTRA="$v" python paper_1310_0901_b200/build.py --force > gpurun_out/build_$T.log 2>&1 || echo "build failed $v" >> gpurun_out/sweep_$T.txt
  run "c5 [$v]" python bench.py --config c5_sharded --steps 10 --warmup 3 $B
  run "c2 [$v]" python bench.py --steps 20 --warmup 3 $B
done
