#!/bin/bash
# bench every configuration once (not the default bench line; for profiles/)
mkdir -p gpurun_out
for c in c2_small c3_single c4_pitched; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-registry-rate > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err
  echo "$c rc=$?"
done
timeout 1200 python bench.py --config c5_sharded --steps 5 --warmup 2 --no-cpu-baseline --no-registry-rate --no-e2e > gpurun_out/cfg_c5_sharded.json 2> gpurun_out/cfg_c5_sharded.err
echo "c5 rc=$?"
