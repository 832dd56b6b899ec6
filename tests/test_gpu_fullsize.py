"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (the whole batch in one cg_check_copies + one cg_apply_dtoh).

The oracle recomputes a sample of descriptors one by one: it replays every
setup event (host marks, V-bytes, registry) and only the sampled copies.  In
C2 and C4 the copies are independent (private host ranges in C2; in C4 DtoH
targets are never HtoD sources and DtoH checks read only A bits), so the
sampled verdicts equal the full replay's.  Everything else is checked with
properties that hold at any size: C2's dirty set equals its injected set, C3's
count / first offset are the generator's closed form, and the final shadow
equals the setup state with exactly the non-injected DtoH ranges defined.
"""
import numpy as np
import pytest

import oracle
import tracegen as tg

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def cg():
    import torch
    assert torch.cuda.is_available()
    from paper_1310_0901_b200 import build
    build.build()
    import paper_1310_0901_b200 as m
    return m


def gpu_batch(cg, tr, fused=False, **kw):
    """Setup events through the ABI, then the whole copy batch in one call
    (cg_check_copies + cg_apply_dtoh, or the bench's fused cg_check_apply)."""
    import torch
    from paper_1310_0901_b200.replay import events_to_descs
    ev = tr.events
    copies = ev[ev["op"] == tg.OP_COPY]
    nreg = int(np.count_nonzero(ev["op"] == tg.OP_REG))
    chk = cg.Checker(tr.host_base, tr.host_size, max_descs=max(len(copies), 1024), max_allocs=max(nreg, 1024), **kw)
    _, st = cg.replay_events(chk, ev[ev["op"] != tg.OP_COPY], tr.blob)
    assert not st.any(), "every setup call of the generated trace is valid"
    descs = events_to_descs(copies)
    dd = cg.to_device_descs(descs)
    if fused:
        dv = chk.check_apply(dd)
    else:
        dv = chk.check_copies(dd)
        chk.apply_dtoh(dd, dv)
    torch.cuda.synchronize()
    return chk, descs, cg.verdicts_to_numpy(dv)


def sampled_oracle(tr, idx):
    """Oracle verdicts of the copies idx (indices into the copy list)."""
    ev = tr.events
    is_copy = ev["op"] == tg.OP_COPY
    keep = ~is_copy
    pos = np.flatnonzero(is_copy)[idx]
    keep[pos] = True
    o = oracle.Oracle(tr.host_base, tr.host_size)
    v, _ = o.replay(ev[keep], tr.blob)
    return o, v


def compare(gv, ov, idx):
    for f in ov.dtype.names:
        a, b = gv[f][idx], ov[f]
        bad = np.flatnonzero(a != b)
        assert len(bad) == 0, (f, idx[bad[:5]], a[bad[:5]], b[bad[:5]])


def test_c2_full(cg):
    tr = tg.c2_small()
    chk, descs, gv = gpu_batch(cg, tr)
    rng = np.random.default_rng(1)
    inj = tr.meta["inject"]
    # every injected copy plus 10k random ones, plus the first and last
    idx = np.unique(np.concatenate([np.flatnonzero(inj), rng.choice(len(descs), 10000, replace=False),
                                    [0, len(descs) - 1]]))
    o, ov = sampled_oracle(tr, idx)
    compare(gv, ov, idx)
    # property at full size: the dirty set is exactly the injected set
    assert np.array_equal(gv["flags"] != 0, inj != 0)
    # final shadow: setup state + the non-injected DtoH ranges defined
    A, V = chk.shadow()
    assert np.array_equal(A, o.A)
    expect = o.V.copy()
    for i in np.flatnonzero((descs["kind"] == tg.DTOH) & (inj == 0)):
        a = int(descs["dst"][i]) - tr.host_base
        expect[a:a + int(descs["width"][i])] = 0
    assert np.array_equal(V, expect)
    chk.close()


@pytest.mark.parametrize("dtoh", [False, True])
def test_c3_full(cg, dtoh):
    tr = tg.c3_single(dtoh=dtoh)
    chk, descs, gv = gpu_batch(cg, tr)
    o, ov = sampled_oracle(tr, np.array([0]))
    compare(gv, ov, np.array([0]))
    if not dtoh:
        offs = tr.meta["hole_offsets"]
        assert gv[0]["undef_count"] == len(offs) == 8192            # closed form
        assert gv[0]["first_undef"] == offs[0]
    else:
        A, V = chk.shadow()
        assert not V[4096:4096 + tr.meta["size"]].any()
        assert np.array_equal(V, o.V)
    chk.close()


def test_c4_full_sampled(cg):
    tr = tg.c4_pitched()
    chk, descs, gv = gpu_batch(cg, tr)
    rng = np.random.default_rng(2)
    inj = tr.meta["inject"]
    idx = np.unique(np.concatenate([rng.choice(np.flatnonzero(inj), 200, replace=False),
                                    rng.choice(len(descs), 800, replace=False)]))
    o, ov = sampled_oracle(tr, idx)
    compare(gv, ov, idx)
    assert np.all(gv["flags"][inj == 0] == 0)
    A, _ = chk.shadow()
    assert np.array_equal(A, o.A)
    chk.close()


@pytest.mark.parametrize("fmt", [0, 1, 2])
def test_c2_full_fused_formats(cg, fmt):
    """the bench's launch configuration (one fused cg_check_apply over the 1M
    batch) in every host shadow format (NEXT-4: 2-bit, sparse map)"""
    tr = tg.c2_small()
    chk, descs, gv = gpu_batch(cg, tr, fused=True, shadow_format=fmt)
    rng = np.random.default_rng(2 + fmt)
    inj = tr.meta["inject"]
    idx = np.unique(np.concatenate([np.flatnonzero(inj), rng.choice(len(descs), 5000, replace=False)]))
    o, ov = sampled_oracle(tr, idx)
    compare(gv, ov, idx)
    assert np.array_equal(gv["flags"] != 0, inj != 0)
    # the fused apply defined exactly the non-injected DtoH ranges: sample some
    dtoh = np.flatnonzero((descs["kind"] == 2) & (inj == 0))
    for i in rng.choice(dtoh, 50, replace=False):
        a, v = chk.shadow_read(int(descs["dst"][i]), int(descs["width"][i]))
        assert a.all() and not v.any(), i


def test_c2_full_tracking(cg):
    """NEXT-1 at full C2 size, as `bench.py --track` runs it: R-20 epochs for the
    check, each epoch's V-bit propagation in its 128 dependency waves through
    one cooperative k_prop_waves launch (R-28).  The oracle replays the whole
    trace sequentially in tracking mode: every verdict, the whole host shadow
    and the device V-bits of 3000 sampled live allocations must agree."""
    tr = tg.c2_small()
    ev = tr.events
    o, ov, os_, oleaks = oracle.replay_trace(tr, track_device=True)
    regs = ev[ev["op"] == tg.OP_REG]
    pool = int(regs["width"].astype(np.int64).sum()) + 256 * len(regs) + (1 << 20)
    copies = ev[ev["op"] == tg.OP_COPY]
    chk = cg.Checker(tr.host_base, tr.host_size, max_descs=len(copies), max_allocs=max(len(regs), 1024),
                     dev_vsize=pool)
    gv, gs = cg.replay_events(chk, ev, tr.blob)
    for f in ov.dtype.names:
        bad = np.flatnonzero(gv[f] != ov[f])
        assert len(bad) == 0, (f, bad[:5])
    assert np.array_equal(gs, os_)
    A, V = chk.shadow()
    assert np.array_equal(A, o.A) and np.array_equal(V, o.V)
    rng = np.random.default_rng(7)
    for r in oleaks[rng.choice(len(oleaks), size=min(3000, len(oleaks)), replace=False)]:
        b, n = int(r["base"]), int(r["size"])
        assert np.array_equal(chk.device_vbits(b, n), o.device_vbits(b, n)), hex(b)
    chk.close()


def _compare_shadow_chunks(chk, o, base, size, chunk=1 << 30):
    """the whole final host shadow, GPU against oracle, chunk by chunk"""
    Abits = o.A
    for q in range(0, size, chunk):
        n = min(chunk, size - q)
        a, v = chk.shadow_read(base + q, n)
        assert np.array_equal(v, o.V[q:q + n]), ("V", q)
        oa = np.unpackbits(Abits[q // 8:(q + n) // 8], bitorder="little")
        assert np.array_equal(a, oa), ("A", q)


def _full_replay(cg, tr, fused=True, T=0, fused_plan=False):
    """The GPU checks the trace the way bench.py does (setup events, then the
    copies in the R-20 epochs cg_plan_batches cuts, fused where the epoch is
    apply-disjoint; registry events are lifetime-stamped, so they all go first);
    the oracle replays the whole trace in order on T host threads
    (or_replay_parallel, equal to the 1-thread replay: tests/test_oracle_parallel.py)."""
    import torch
    ev = tr.events
    is_copy = ev["op"] == tg.OP_COPY
    copies = ev[is_copy]
    nreg = int(np.count_nonzero(ev["op"] == tg.OP_REG))
    chk = cg.Checker(tr.host_base, tr.host_size, max_descs=max(len(copies), 1024), max_allocs=max(nreg, 1024))
    _, st = cg.replay_events(chk, ev[~is_copy], tr.blob)
    descs = tg.events_to_descs(copies)
    dd = cg.to_device_descs(descs)
    dv = torch.empty(len(descs) * 64, dtype=torch.uint8, device=dd.device)
    if fused_plan:   # the bench's batches: cg_plan_batches_fused marks the descriptors in place
        descs = np.ascontiguousarray(descs)
        cuts = [0] + [int(c) for c in cg.plan_batches_fused(descs)]
        dd = cg.to_device_descs(descs)
    else:
        cuts = [0] + [int(c) for c in cg.plan_batches(descs)]
    for a, b in zip(cuts[:-1], cuts[1:]):
        if b <= a:
            continue
        x, y = dd[a * 96:b * 96], dv[a * 64:b * 64]
        if fused_plan:
            chk.check_apply(x, y)
        elif fused and cg.batch_disjoint(descs[a:b]):
            chk.check_apply(x, y)
        else:
            chk.check_copies(x, y)
            chk.apply_dtoh(x, y)
    torch.cuda.synchronize()
    gv = cg.verdicts_to_numpy(dv)
    o = oracle.Oracle(tr.host_base, tr.host_size)
    ov, os_ = o.replay_parallel(ev, tr.blob, threads=T)
    for f in ov.dtype.names:
        bad = np.flatnonzero(gv[f] != ov[f])
        assert len(bad) == 0, (tr.name, f, len(bad), bad[:5], gv[f][bad[:5]], ov[f][bad[:5]])
    # registry statuses of the setup events
    assert np.array_equal(st, os_[~is_copy])
    gl, ol = chk.leak_report(), o.leaks()
    assert np.array_equal(gl["base"], ol["base"]) and np.array_equal(gl["size"], ol["size"])
    assert np.array_equal(gl["alloc_seq"], ol["seq"])
    _compare_shadow_chunks(chk, o, tr.host_base, tr.host_size)
    chk.close()
    return gv, ov


def test_c4_full(cg):
    """C4 at full size: all 100k verdicts (273 GB of host bytes checked), the
    final A and V shadow (8 GiB window) bit for bit against the T-thread oracle"""
    tr = tg.c4_pitched()
    gv, _ = _full_replay(cg, tr)
    inj = tr.meta["inject"]
    assert np.all(gv["flags"][inj == 0] == 0) and np.all(gv["flags"][inj != 0] != 0)


def test_c5_full_fused(cg):
    """C5 at full size the way bench.py times it: cg_plan_batches_fused makes
    ONE batch of the 10M descriptors (the ping-pongs become CG_CHECK_AFTER /
    CG_APPLY_AFTER / CG_APPLY_LAST), checked by one cg_check_apply (separate
    prep and plan kernels above 4M descriptors, the small pass, the ring, the
    late pass and the last applies in k_finish): every verdict, the leak list
    and the whole final shadow against the sequential T-thread oracle."""
    import psutil
    if psutil.virtual_memory().available < (100 << 30):
        pytest.skip("needs ~100 GiB of host memory for the oracle's 64 GiB window")
    tr = tg.c5_sharded()
    gv, _ = _full_replay(cg, tr, fused_plan=True)
    assert int(np.count_nonzero(gv["flags"])) > 0


def test_c5_full(cg):
    """C5 at full size on one GPU: 10M descriptors in 11 R-20 epochs against a
    ~150k-entry lifetime-stamped table with alloc / free bursts, the 64 GiB
    window (V 64 GiB + A 8 GiB), leak report: every verdict, every registry
    status, the leak list and the whole final shadow against the T-thread
    oracle (~72 GiB of host memory)."""
    import os
    import psutil
    if psutil.virtual_memory().available < (100 << 30):
        pytest.skip("needs ~100 GiB of host memory for the oracle's 64 GiB window")
    tr = tg.c5_sharded()
    gv, _ = _full_replay(cg, tr)
    assert int(np.count_nonzero(gv["flags"])) > 0
