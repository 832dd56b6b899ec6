#!/bin/bash
# diagnose the C5 full-size mismatch (small pass on / off), then the staged-store prep A/B
mkdir -p gpurun_out
T=r02p
python paper_1310_0901_b200/build.py --force > gpurun_out/build_$T.log 2>&1
timeout 1500 python tests/diag_c5.py 1 2 > gpurun_out/diag_$T.txt 2>&1
B="--no-cpu-baseline --no-registry-rate --no-e2e --no-per-config"
run() { tag=$1; shift; echo "== $tag" >> gpurun_out/sweep_$T.txt; timeout 300 env "$@" >> gpurun_out/sweep_$T.txt 2>> gpurun_out/sweep_$T.err; }
run c5 python bench.py --config c5_sharded --steps 10 --warmup 3 $B
run c2 python bench.py --steps 20 --warmup 3 $B
CG_NVCC_EXTRA="-DCG_PREP_STAGED_STORES=0" python paper_1310_0901_b200/build.py --force > gpurun_out/build2_$T.log 2>&1
run c5_nostage python bench.py --config c5_sharded --steps 10 --warmup 3 $B
run c2_nostage python bench.py --steps 20 --warmup 3 $B
