"""NEXT-1: device time of every propagation wave of the C2 batch (diagnostic)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_1310_0901_b200 as cg
import tracegen as tg

tr = tg.c2_small()
chk, descs, _, nreg = bench.setup_checker(cg, tr, 0, host_staging=False, track=True)
dd = cg.to_device_descs(descs)
dv = chk.check_copies(dd)
lev, nl = cg.plan_waves(descs)
W = cg.Waves(descs, 0)
waves = [(torch.from_numpy(w.astype(np.int32)).cuda(), mb) for w, mb in cg.wave_indices(lev, nl, descs)]
s = torch.cuda.current_stream()
for rep in range(2):
    chk.check_copies(dd, dv)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(waves) + 1)]
    ev[0].record(s)
    for k, (w, mb) in enumerate(waves):
        chk.apply_copies(dd, dv, index=w, max_bytes=mb)
        ev[k + 1].record(s)
    chk.apply_flush()
    torch.cuda.synchronize()
t = [ev[k].elapsed_time(ev[k + 1]) for k in range(len(waves))]
nb = descs["width"].astype(np.float64) * descs["height"]
for k in list(range(8)) + list(range(8, len(waves), 16)):
    w = waves[k][0].cpu().numpy()
    print(f"wave {k:3d}: {len(w):7d} copies {nb[w].sum() / 1e6:9.1f} MB  {t[k] * 1e3:8.1f} us")
print("total %.3f ms over %d waves" % (sum(t), len(t)))
for rep in range(2):
    chk.check_copies(dd, dv)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    chk.apply_waves(dd, dv, W)
    e1.record(s)
    torch.cuda.synchronize()
print("one cg_apply_copies_waves call: %.3f ms" % e0.elapsed_time(e1))
