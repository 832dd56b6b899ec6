"""NEXT-2 on the GPU: cg_conc_check (merge-sort tree + cover-list segment
tree over each batch, last-access map between batches) bit-exact against the
oracle's stamp-list scan on the same seeded multi-threaded traces."""
import numpy as np
import pytest

import oracle
import tracegen as tg

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cg():
    import torch
    assert torch.cuda.is_available()
    from paper_1310_0901_b200 import build
    build.build()
    import paper_1310_0901_b200 as m
    return m


def run(cg, tr, mode="fused", max_descs=None, max_stamps=1 << 16):
    track = mode == "track"
    o, ov, os_, oleaks = oracle.replay_trace(tr, track_device=track, concurrency=True)
    ev = tr.events
    kw = {}
    if track:
        regs = ev[ev["op"] == tg.OP_REG]
        kw["dev_vsize"] = int(sum(int(x) + 256 for x in regs["width"])) + (1 << 20)
    md = max_descs or max(tr.n_copies, 64)
    chk = cg.Checker(tr.host_base, tr.host_size, max_descs=md, max_allocs=max(len(ev), 64), **kw)
    conc = cg.ConcChecker(md, max_stamps)
    gv, gs = cg.replay_events(chk, ev, tr.blob, fuse=(mode == "fused"), conc=conc, threads=tr.threads)
    for f in ov.dtype.names:
        bad = np.flatnonzero(gv[f] != ov[f])
        assert len(bad) == 0, (mode, f, bad[:5], gv[f][bad[:5]], ov[f][bad[:5]])
    assert np.array_equal(gs, os_)
    A, V = chk.shadow()
    assert np.array_equal(A, o.A) and np.array_equal(V, o.V)
    st = conc.stamps()
    conc.close()
    chk.close()
    return gv, st


@pytest.mark.parametrize("mode", ["fused", "unfused", "track"])
@pytest.mark.parametrize("seed", range(30))
def test_random_tiny_threads(cg, seed, mode):
    tr = tg.random_tiny(seed + 40000, threads=int(2 + seed % 3), arrays=seed % 2 == 1)
    gv, _ = run(cg, tr, mode)
    assert tr.n_copies == len(gv)


@pytest.mark.parametrize("seed", range(20))
def test_history_across_small_batches(cg, seed):
    """batches of 1..16 copies: most overlaps are resolved through the last-access map"""
    tr = tg.random_tiny(seed + 41000, threads=3)
    run(cg, tr, "fused", max_descs=int(1 + seed % 16))


def test_spec_examples(cg):
    import sys, os
    sys.path.insert(0, os.path.dirname(__file__))
    from test_oracle_next2 import _trace
    for sched, want in [([(1, "W"), (2, "R")], [0, 1]), ([(1, "W"), (1, "S"), (2, "W")], [0, 0]),
                        ([(1, "R"), (2, "R")], [0, 0]), ([(1, "W"), (2, "S"), (2, "R")], [0, 1])]:
        for md in (1, 8):
            gv, _ = run(cg, _trace(sched), max_descs=md)
            assert [int(f >> 9) & 1 for f in gv["flags"]] == want, (sched, md)


def test_single_thread_never_flags_and_map_is_compact(cg):
    """one thread, no hazards; the last-access map never holds more ranges
    than there are distinct stamped ranges"""
    tr = tg.c2_small(n_copies=20000, n_allocs=2000)
    gv, (nh, nd) = run(cg, tr, max_stamps=1 << 17)
    assert not (gv["flags"] & (1 << 9)).any()
    assert 0 < nh <= 20000 and 0 < nd <= 40000


@pytest.mark.parametrize("nt", [2, 8])
def test_c2_scaled_threads(cg, nt):
    tr = tg.with_threads(tg.c2_small(n_copies=20000, n_allocs=2000), nt, sync_frac=0.002)
    gv, _ = run(cg, tr, max_stamps=1 << 17)
    assert (gv["flags"] & (1 << 9)).any()


def test_c2_scaled_threads_batches(cg):
    tr = tg.with_threads(tg.c2_small(n_copies=20000, n_allocs=2000), 4, sync_frac=0.01, seed=5)
    run(cg, tr, max_descs=3000, max_stamps=1 << 17)


def test_c4_pitched_threads(cg):
    tr = tg.with_threads(tg.c4_pitched(n_copies=600, n_bufs=2, rows=64, inject_frac=0.05), 3, sync_frac=0.02)
    run(cg, tr, max_stamps=1 << 16)


def test_map_capacity_error(cg):
    tr = tg.with_threads(tg.c2_small(n_copies=2000, n_allocs=500), 2)
    ev = tr.events
    chk = cg.Checker(tr.host_base, tr.host_size, max_descs=4096, max_allocs=4096)
    conc = cg.ConcChecker(4096, 64)
    with pytest.raises(cg.CgError) as e:
        cg.replay_events(chk, ev, tr.blob, conc=conc, threads=tr.threads)
    assert e.value.status == cg.CG_ERR_OUT_OF_MEMORY
    conc.close()
    chk.close()


@pytest.mark.parametrize("uie", [False, True])
def test_error_summary_counts(cg, uie):
    """NEXT-4 cg_summarize: one diagnostic per set flag; HOST_UNDEFINED (unless
    undef_is_error) and CONCURRENT are the Warnings"""
    import torch
    tr = tg.with_threads(tg.c2_small(n_copies=20000, n_allocs=2000), 4)
    o, ov, _, _ = oracle.replay_trace(tr, undef_is_error=uie, concurrency=True)
    d = torch.from_numpy(ov.view(np.uint8).copy()).cuda()
    e, w = cg.summarize(d, undef_is_error=uie)
    f = ov["flags"].astype(np.uint64)
    bits = np.array([[(int(x) >> b) & 1 for b in range(10)] for x in f])
    warn = [5, 9] if not uie else [9]
    assert w == int(bits[:, warn].sum()) and e == int(bits.sum()) - w
    assert w > 0 and e > 0


def test_batch_order_contract(cg):
    """cg_conc_check rejects a batch whose seqs do not increase, or that does
    not come after the previous batch, and then changes nothing"""
    import torch
    from paper_1310_0901_b200.replay import events_to_descs
    tr = tg.with_threads(tg.c2_small(n_copies=2000, n_allocs=500), 2)
    ev = tr.events
    chk = cg.Checker(tr.host_base, tr.host_size, max_descs=4096, max_allocs=4096)
    cg.replay_events(chk, ev[ev["op"] != tg.OP_COPY], tr.blob)
    copies = ev[ev["op"] == tg.OP_COPY]
    descs = events_to_descs(copies)
    th = torch.from_numpy(tr.threads[ev["op"] == tg.OP_COPY].astype(np.int32)).cuda()
    conc = cg.ConcChecker(4096, 1 << 16)
    dd = cg.to_device_descs(descs[:1000])
    dv = chk.check_copies(dd)
    conc.check(dd, th[:1000], dv)
    before = conc.stamps()
    for bad in (descs[:1000], descs[1000:2000][::-1].copy()):   # repeated / descending seqs
        d2 = cg.to_device_descs(bad)
        v2 = chk.check_copies(d2)
        with pytest.raises(cg.CgError):
            conc.check(d2, th[:1000], v2)
        assert conc.stamps() == before
    d3 = cg.to_device_descs(descs[1000:2000])
    conc.check(d3, th[1000:2000], chk.check_copies(d3))       # the next batch in order is fine
    conc.close()
    chk.close()
