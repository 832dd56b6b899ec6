"""NEXT-1 diagnostic: raw V-bit move throughput of cg_apply_copies_waves on the
C2 batch with synthetic level assignments (timing only -- the orders are not
R-28's, so the resulting V-bits are not checked): one wave, and the real
plan's wave sizes.  Run with CG_WAVE_KERNEL=0 / 1 to compare the paths."""
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

nb = descs["width"].astype(np.float64) * descs["height"]
ok = nb.sum()
s = torch.cuda.current_stream()


def waves_from(lev):
    W = cg.Waves.__new__(cg.Waves)
    nl = int(lev.max()) + 1
    order = np.argsort(lev, kind="stable").astype(np.uint32)
    W.start = np.searchsorted(lev[order], np.arange(nl + 1)).astype(np.uint64)
    W.max_bytes = np.full(nl, int(nb.max()), np.uint64)
    W.index = torch.from_numpy(order.astype(np.int32)).cuda()
    W.n_waves = nl
    return W


def timeit(W, reps=3):
    best = 1e9
    for _ in range(reps):
        chk.check_copies(dd, dv)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        chk.apply_waves(dd, dv, W)
        e1.record(s)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


lev_real, nl = cg.plan_waves(descs)
rng = np.random.default_rng(1)
cases = {
    "one wave": np.zeros(len(descs), np.uint32),
    "real plan": lev_real.astype(np.uint32),
    "128 equal waves": rng.integers(0, 128, len(descs)).astype(np.uint32),
}
print("CG_WAVE_KERNEL=%s  copies %d  payload %.2f GB" % (os.environ.get("CG_WAVE_KERNEL", "1"), len(descs), ok / 1e9))
only = os.environ.get("WAVE_CASE")
for name, lev in cases.items():
    if only and name != only:
        continue
    t = timeit(waves_from(lev))
    print(f"{name:16s}: {t:8.3f} ms  payload {ok / t / 1e6:7.1f} GB/s  (x2 read+write {2 * ok / t / 1e6:7.1f})")
# fixed cost per wave: 128 waves of one small copy each
small = np.flatnonzero(nb <= 256)[:128]
W = cg.Waves.__new__(cg.Waves)
W.start = np.arange(129, dtype=np.uint64)
W.max_bytes = np.full(128, 256, np.uint64)
W.index = torch.from_numpy(small.astype(np.int32)).cuda()
W.n_waves = 128
t = timeit(W)
print(f"128 waves x 1 small copy: {t * 1e3:8.1f} us = {t * 1e3 / 128:6.2f} us per wave")
