#!/bin/bash
# bench every configuration once (not the default bench line; for profiles/)
mkdir -p gpurun_out
for c in c2_small c3_single c4_pitched; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-registry-rate > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err
  echo "$c rc=$?"
done
timeout 1200 python bench.py --config c5_sharded --steps 5 --warmup 2 --no-cpu-baseline --no-registry-rate --no-e2e > gpurun_out/cfg_c5_sharded.json 2> gpurun_out/cfg_c5_sharded.err
echo "c5 rc=$?"
# NEXT rows on the C2 batch
timeout 600 python bench.py --shadow 2bit --no-cpu-baseline --no-registry-rate > gpurun_out/cfg_c2_2bit.json 2> gpurun_out/cfg_c2_2bit.err
timeout 600 python bench.py --shadow sparse --no-cpu-baseline --no-registry-rate > gpurun_out/cfg_c2_sparse.json 2> gpurun_out/cfg_c2_sparse.err
timeout 600 python bench.py --conc 8 --no-cpu-baseline --no-registry-rate > gpurun_out/cfg_c2_next2.json 2> gpurun_out/cfg_c2_next2.err
echo "next rows done"
