"""Replay a recorded call stream through the C ABI (the way the paper's
wrappers see a program: "Anytime a program handles memory on the device
or transfers data ... the respective Cudagrind wrapper will be called").

``events`` is any numpy structured array with the fields
``op, kind, seq, width, height, dst, dst_x, dst_y, dst_pitch, src, src_x,
src_y, src_pitch`` (op: 1 host mark, 2 set V-bytes, 3 register, 4 free,
5 copy, 6 register array [dst = handle, width, height, dst_x = depth,
dst_y = format, dst_pitch = channels], 7 free array [dst = handle]).  Host shadow updates are applied in order; between two of them, all
registry events are submitted first (the table is lifetime-stamped, so a copy
sees exactly the allocations live at its seq) and the copies are checked in the
hazard-free batches cg_plan_batches cuts (check, then DtoH apply, per batch).
"""
from __future__ import annotations

import numpy as np

OP_MARK, OP_SETV, OP_REG, OP_FREE, OP_COPY, OP_REGA, OP_FREEA, OP_SYNC = 1, 2, 3, 4, 5, 6, 7, 8
_REGISTRY = (OP_REG, OP_FREE, OP_COPY, OP_REGA, OP_FREEA, OP_SYNC)
_DESC_FIELDS = ("kind", "seq", "width", "height", "dst", "dst_x", "dst_y", "dst_pitch",
                "src", "src_x", "src_y", "src_pitch")


def events_to_descs(ev: np.ndarray) -> np.ndarray:
    from . import DESC_DTYPE
    d = np.zeros(len(ev), DESC_DTYPE)
    for f in _DESC_FIELDS:
        d[f] = ev[f]
    return d


def replay_events(chk, events: np.ndarray, blob=None, stream=None, fuse: bool = True, conc=None, threads=None):
    """Returns (verdicts of the COPY events in order, status per event).
    With fuse, batches that cg_batch_disjoint accepts use cg_check_apply.
    conc (a ConcChecker) adds NEXT-2: SYNC events go to cg_conc_sync and every
    checked batch to cg_conc_check with the copies' threads (threads[i] = the
    issuing thread of event i, default all 0)."""
    import torch
    from . import MARK_DTYPE, REG_EVENT_DTYPE, VERDICT_DTYPE, to_device_descs, verdicts_to_numpy

    ops = np.asarray(events["op"])
    n = len(events)
    status = np.zeros(n, np.uint32)
    is_copy = ops == OP_COPY
    copy_rank = np.cumsum(is_copy) - 1
    verdicts = np.zeros(int(is_copy.sum()), VERDICT_DTYPE)
    regs_since = 0
    i = 0
    while i < n:
        op = ops[i]
        if op == OP_MARK:
            j = i
            while j < n and ops[j] == OP_MARK:
                j += 1
            m = np.zeros(j - i, MARK_DTYPE)
            m["addr"] = events["dst"][i:j]
            m["len"] = events["width"][i:j]
            m["state"] = events["kind"][i:j]
            st = np.zeros(j - i, np.uint32)
            chk.host_mark_batch(m, status_out=st, stream=stream)
            status[i:j] = st
            i = j
        elif op == OP_SETV:
            off, ln = int(events["src"][i]), int(events["width"][i])
            status[i] = chk.host_set_vbits(int(events["dst"][i]), bytes(blob[off:off + ln]), stream=stream)
            i += 1
        else:
            j = i
            while j < n and ops[j] in _REGISTRY:
                j += 1
            if j == i:   # an unknown op: invalid call, like the oracle's replay
                status[i] = 1
                i += 1
                continue
            # every later copy has seq >= this block's first seq: tombstones freed
            # before it are invisible to them (cg_registry_compact), so drop
            # them before the table (live + tombstones) can fill up
            n_reg = int(np.count_nonzero((ops[i:j] == OP_REG) | (ops[i:j] == OP_REGA)))
            regs_since += n_reg
            if regs_since > getattr(chk, "max_allocs", 1 << 62) // 2:
                chk.registry_compact(int(events["seq"][i]))
                regs_since = n_reg
            k = i
            while k < j:
                if ops[k] in (OP_REG, OP_FREE):   # a run of registry events: one cg_registry_batch
                    r = k
                    while r < j and ops[r] in (OP_REG, OP_FREE):
                        r += 1
                    re = np.zeros(r - k, REG_EVENT_DTYPE)
                    re["op"] = np.where(ops[k:r] == OP_REG, 1, 2)
                    re["seq"], re["addr"], re["size"] = events["seq"][k:r], events["dst"][k:r], events["width"][k:r]
                    st = np.zeros(r - k, np.uint32)
                    chk.registry_batch(re, st)
                    status[k:r] = st
                    k = r
                    continue
                if ops[k] == OP_REGA:
                    e = events[k]
                    status[k] = chk.register_array(int(e["dst"]), int(e["width"]), int(e["height"]), int(e["dst_x"]),
                                                   int(e["dst_y"]), int(e["dst_pitch"]), int(e["seq"]))
                elif ops[k] == OP_FREEA:
                    status[k] = chk.free_array(int(events["dst"][k]), int(events["seq"][k]))
                elif ops[k] == OP_SYNC and conc is not None:
                    conc.sync(int(threads[k]) if threads is not None else 0, int(events["seq"][k]))
                k += 1
            idx = np.flatnonzero(is_copy[i:j]) + i
            if len(idx):
                descs = events_to_descs(events[idx])
                pkg = __import__(__package__)
                tracking = getattr(chk, "tracking", False)
                # R-20 epochs for the check; with tracking, each epoch's V-bit
                # propagation runs in the waves of cg_plan_waves (R-28); fused
                # (cg_check_apply): the batches of cg_plan_batches_fused, which
                # also sets CG_CHECK_AFTER / CG_APPLY_AFTER / CG_APPLY_LAST
                fused_plan = fuse and fuse != "disjoint" and not tracking
                descs = np.ascontiguousarray(descs)
                parts = []   # (s0, s1): batches of at most max_descs copies
                cuts = [0] + [int(c) for c in (pkg.plan_batches_fused(descs) if fused_plan
                                                else pkg.plan_batches(descs))]
                for a, b in zip(cuts[:-1], cuts[1:]):
                    for s0 in range(a, b, chk.max_descs):
                        s1 = min(b, s0 + chk.max_descs)
                        if fused_plan and s1 - s0 < b - a:   # a piece of a fused batch: its own plan
                            part = np.ascontiguousarray(descs[s0:s1])
                            sub = [0] + [int(c) for c in pkg.plan_batches_fused(part)]
                            descs[s0:s1] = part
                            parts += [(s0 + c0, s0 + c1) for c0, c1 in zip(sub[:-1], sub[1:])]
                        else:
                            parts.append((s0, s1))
                for s0, s1 in parts:
                        dd = to_device_descs(descs[s0:s1], chk.device)
                        if tracking:    # NEXT-1: check, then move V-bits wave by wave
                            dv = chk.check_copies(dd, stream=stream)
                            waves = pkg.Waves(descs[s0:s1], chk.device)
                            if waves.n_waves <= 1:
                                chk.apply_copies(dd, dv, stream=stream)
                            else:
                                chk.apply_waves(dd, dv, waves, stream=stream)
                        elif fused_plan:
                            dv = chk.check_apply(dd, stream=stream)
                        elif fuse and pkg.batch_disjoint(descs[s0:s1]):
                            dv = chk.check_apply(dd, stream=stream)
                        else:
                            dv = chk.check_copies(dd, stream=stream)
                            chk.apply_dtoh(dd, dv, stream=stream)
                        if conc is not None:
                            th = np.zeros(s1 - s0, np.int32) if threads is None else \
                                np.asarray(threads[idx[s0:s1]]).astype(np.int32)
                            conc.check(dd, torch.from_numpy(th).to(dd.device), dv, stream=stream)
                        v = verdicts_to_numpy(dv)
                        verdicts[copy_rank[idx[s0:s1]]] = v
                        status[idx[s0:s1]] = v["status"]
            i = j
    torch.cuda.synchronize(chk.device)
    return verdicts, status
