"""Test infrastructure, run by hand on a GPU box (not collected by pytest):
C5 at full size on the GPU (per R-20 epoch, as tests/test_gpu_fullsize.py
_full_replay) against the T-thread oracle; prints the mismatching verdict
rows and their descriptors for each small-pass mode in argv (CG_SMALL_MODE
values)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))   # repo root
import oracle  # noqa: E402
import tracegen as tg  # noqa: E402


def gpu_verdicts(cg, tr, mode):
    import torch
    os.environ["CG_SMALL_MODE"] = mode
    ev = tr.events
    is_copy = ev["op"] == tg.OP_COPY
    copies = ev[is_copy]
    nreg = int(np.count_nonzero(ev["op"] == tg.OP_REG))
    chk = cg.Checker(tr.host_base, tr.host_size, max_descs=max(len(copies), 1024), max_allocs=max(nreg, 1024))
    cg.replay_events(chk, ev[~is_copy], tr.blob)
    descs = tg.events_to_descs(copies)
    dd = cg.to_device_descs(descs)
    dv = torch.empty(len(descs) * 64, dtype=torch.uint8, device=dd.device)
    cuts = [0] + [int(c) for c in cg.plan_batches(descs)]
    for a, b in zip(cuts[:-1], cuts[1:]):
        if b <= a:
            continue
        x, y = dd[a * 96:b * 96], dv[a * 64:b * 64]
        if cg.batch_disjoint(descs[a:b]):
            chk.check_apply(x, y)
        else:
            chk.check_copies(x, y)
            chk.apply_dtoh(x, y)
    torch.cuda.synchronize()
    gv = cg.verdicts_to_numpy(dv)
    chk.close()
    return gv, descs, cuts


def main():
    from paper_1310_0901_b200 import build
    build.build()
    import paper_1310_0901_b200 as cg
    tr = tg.c5_sharded()
    o = oracle.Oracle(tr.host_base, tr.host_size)
    ov, _ = o.replay_parallel(tr.events, tr.blob, threads=0)
    for mode in sys.argv[1:] or ["0"]:
        gv, descs, cuts = gpu_verdicts(cg, tr, mode)
        bad = np.zeros(len(gv), bool)
        for f in ov.dtype.names:
            bad |= gv[f] != ov[f]
        idx = np.flatnonzero(bad)
        print(f"mode {mode}: {len(idx)} mismatching verdicts; epochs {len(cuts) - 1}", flush=True)
        for i in idx[:12]:
            ep = int(np.searchsorted(cuts, i, side="right")) - 1
            d = descs[i]
            print(f"  [{i}] epoch {ep} [{cuts[ep]},{cuts[ep + 1]}) kind {int(d['kind'])} w {int(d['width'])} "
                  f"dst {int(d['dst']):#x} src {int(d['src']):#x}")
            print("     gpu", {f: int(gv[f][i]) for f in gv.dtype.names})
            print("     orc", {f: int(ov[f][i]) for f in ov.dtype.names})


if __name__ == "__main__":
    main()
