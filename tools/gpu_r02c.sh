#!/bin/bash
# full GPU suite (incl. full-size C4/C5 parity), then the default bench line (per_config) and the reference arm
mkdir -p gpurun_out
python paper_1310_0901_b200/build.py > gpurun_out/build_r02c.log 2>&1
timeout 2400 python -m pytest tests/ -q -m gpu -x --durations=15 > gpurun_out/pytest_gpu_r02c.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r02c.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_r02c.json 2> gpurun_out/bench_r02c.err
echo "bench rc=$?" >> gpurun_out/bench_r02c.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_r02c.json 2> gpurun_out/ref_r02c.err
