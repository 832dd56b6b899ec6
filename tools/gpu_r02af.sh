#!/bin/bash
# final-commit validation: full GPU suite, smoke, default bench line
mkdir -p gpurun_out
T=r02af
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$T.log 2>&1
timeout 2700 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu_$T.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
