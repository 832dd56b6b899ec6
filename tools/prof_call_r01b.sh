set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu_r01b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r01b.log
timeout 600 python bench.py > gpurun_out/bench_r01b.json 2> gpurun_out/bench_r01b.err
timeout 600 python bench.py --track > gpurun_out/bench_track_r01b.json 2> gpurun_out/bench_track_r01b.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r01b.json 2> gpurun_out/bench_ref_r01b.err
bash tools/ncu_launches.sh r01b --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --no-registry-rate
bash tools/ncu_scan.sh r01b k_check_scan
bash tools/ncu_launches.sh r01b_track --track --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-registry-rate
bash tools/ncu_scan.sh r01b_waves k_prop_waves --track --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-registry-rate
ls gpurun_out
