#!/bin/bash
# e2e (cg_check_host) pipeline sweep: chunk count x geometric sizes
mkdir -p gpurun_out
for g in 1; do for c in 2 3 4 5; do
  CG_HOST_CHUNKS=$c CG_HOST_GEOMETRIC=$g timeout 300 python bench.py --steps 12 --warmup 3 --no-cpu-baseline --no-registry-rate \
    > gpurun_out/e2e_c${c}_g${g}.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/e2e_c${c}_g${g}.json')); print('chunks $c geo $g', round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3))" >> gpurun_out/e2e_sweep.txt
done; done
python - >> gpurun_out/e2e_sweep.txt <<'PY'
import torch
h = torch.empty(40_000_000, dtype=torch.uint8).pin_memory(); d = torch.empty_like(h, device="cuda")
for _ in range(3): d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); [d.copy_(h, non_blocking=True) for _ in range(10)]; e1.record(); torch.cuda.synchronize()
print("H2D 40 MB pinned: %.3f ms, %.1f GB/s" % (e0.elapsed_time(e1) / 10, 40e6 / (e0.elapsed_time(e1) / 10 * 1e-3) / 1e9))
PY
