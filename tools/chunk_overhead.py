"""How much does splitting one C2 batch into k cg_check_apply calls cost
(device-resident descriptors, no uploads)?  Prints ms per full batch."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_1310_0901_b200 as cg
import tracegen as tg

tr = tg.c2_small()
chk, descs, _, nreg = bench.setup_checker(cg, tr, 0, host_staging=False)
n = len(descs)
dd = cg.to_device_descs(descs)
out = torch.empty(n * 64, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
for k in (1, 2, 3, 4, 5, 8):
    b = [n * i // k for i in range(k + 1)]
    def step():
        for i in range(k):
            cg.cg_check_apply(chk.ctx, dd.data_ptr() + b[i] * 96, b[i + 1] - b[i], out.data_ptr() + b[i] * 64,
                              s.cuda_stream)
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(10):
        step()
    e1.record(s)
    torch.cuda.synchronize()
    print("calls %d: %.3f ms per batch" % (k, e0.elapsed_time(e1) / 10))

for k in (1, 8):
    b = [n * i // k for i in range(k + 1)]
    chk.profile_begin()
    for _ in range(5):
        for i in range(k):
            cg.cg_check_apply(chk.ctx, dd.data_ptr() + b[i] * 96, b[i + 1] - b[i], out.data_ptr() + b[i] * 64,
                              s.cuda_stream)
    torch.cuda.synchronize()
    st = chk.profile_end()
    print("calls %d:" % k, {a: round(v[0] / 5, 3) for a, v in st.items() if v[1]})
