#!/bin/bash
# prep lookups in lockstep (table_lookup2) A/B
mkdir -p gpurun_out
T=r02x
B="--no-cpu-baseline --no-registry-rate --no-e2e --no-per-config"
run() { tag=$1; shift; echo "== $tag" >> gpurun_out/sweep_$T.txt; timeout 300 env "$@" >> gpurun_out/sweep_$T.txt 2>> gpurun_out/sweep_$T.err; }
for v in "0 4" "1 3" "1 4" "0 3"; do
  set -- $v
  CG_NVCC_EXTRA="-DCG_LOOKUP2=$1 -DCG_FRONT_MINB=$2" python paper_1310_0901_b200/build.py --force > gpurun_out/build_${T}_$1$2.log 2>&1
  run c5_l$1_m$2 python bench.py --config c5_sharded --steps 10 --warmup 3 $B
  run c2_l$1_m$2 python bench.py --steps 20 --warmup 3 $B
done
python paper_1310_0901_b200/build.py --force > gpurun_out/build_$T.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_medium.py tests/test_gpu_next3.py tests/test_gpu_next1.py -q -m gpu -x > gpurun_out/pytest_$T.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$T.log
timeout 1500 python tests/diag_c5.py 1 > gpurun_out/diag_$T.txt 2>&1
