#!/bin/bash
# End-of-round evidence on one B200: the default bench line, the reference arm,
# every config and NEXT row, launch lists and ncu captures of the two dominant kernels.
set -x
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
timeout 600 python bench.py --track > gpurun_out/final_track.json 2> gpurun_out/final_track.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err
bash tools/bench_configs.sh
bash tools/ncu_launches.sh final --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --no-registry-rate
bash tools/ncu_scan.sh final k_check_scan
bash tools/ncu_launches.sh final_track --track --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-registry-rate
bash tools/ncu_scan.sh final_waves k_prop_waves --track --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-registry-rate
ls gpurun_out
