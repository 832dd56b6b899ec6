"""NEXT-2 pins ("certain concurrent accesses when several
threads are used"; SPEC check_concurrent S:258-266 with the rule of S:285).
The oracle scans its stamp list for the newest overlapping stamp; it is pinned
by SPEC's three examples, by invariants, and against tests/flatmodel.py, which
keeps a per-byte last-access map instead (an independent formulation)."""
import itertools

import numpy as np
import pytest

import oracle
import tracegen as tg
from flatmodel import FlatModel

H0 = 0x10000
F_CONC = oracle.F_CONCURRENT


def _trace(schedule, nbytes=256):
    """schedule: (thread, op) with op in {'W' host->device write, 'R' device->host read,
    'S' sync}; all on the same device range (and distinct host ranges)."""
    tb = tg.TraceBuilder("sched", H0, 1 << 16)
    tb.mark(H0, 1 << 16, tg.DEFINED)
    d = tb.malloc(nbytes)
    for k, (t, op) in enumerate(schedule):
        tb.thread = t
        if op == "S":
            tb.sync()
        elif op == "W":
            tb.copy1d(tg.HTOD, d, H0 + 1024 * k, nbytes)
        else:
            tb.copy1d(tg.DTOH, H0 + 1024 * k, d, nbytes)
    return tb.build()


def _flags(tr):
    o, v, s, _ = oracle.replay_trace(tr, concurrency=True)
    assert not s.any()
    return [bool(f & F_CONC) for f in v["flags"]]


def test_spec_examples():
    # S:264 write by thread 1 then read by thread 2, no sync between -> ConcurrentHazard
    assert _flags(_trace([(1, "W"), (2, "R")])) == [False, True]
    # S:265 write by thread 1, sync, write by thread 2 -> no diagnostic
    assert _flags(_trace([(1, "W"), (1, "S"), (2, "W")])) == [False, False]
    # S:266 two reads, different threads, no sync -> no diagnostic
    assert _flags(_trace([(1, "R"), (2, "R")])) == [False, False]


def test_hazard_is_a_warning():
    """S:279 severity rule: ConcurrentHazard never makes the call fail."""
    o, v, s, _ = oracle.replay_trace(_trace([(1, "W"), (2, "W")]), concurrency=True)
    assert v[1]["flags"] == F_CONC and v[1]["status"] == 0 and not s.any()


def test_only_the_newest_stamp_decides():
    # thread 2 reads after thread 1 wrote and thread 1 itself read again: the
    # newest overlapping stamp is thread 1's read, so thread 2's read is clean
    assert _flags(_trace([(1, "W"), (1, "R"), (2, "R")])) == [False, False, False]
    # a sync by the *other* thread does not order thread 1's write
    assert _flags(_trace([(1, "W"), (2, "S"), (2, "R")])) == [False, True]


@pytest.mark.parametrize("n", [2, 3])
def test_exhaustive_two_thread_schedules(n):
    """every 2-thread schedule of n events from {W, R, S} agrees with
    the flat model's per-byte last-access view; single-thread and read-only
    schedules never race."""
    for sched in itertools.product([(1, "W"), (1, "R"), (1, "S"), (2, "W"), (2, "R"), (2, "S")], repeat=n):
        tr = _trace(list(sched))
        got = _flags(tr)
        fm = FlatModel(tr.host_base, tr.host_size, conc=True)
        fv, _ = fm.replay(tr.events, tr.blob, tr.threads)
        assert got == [bool(v["flags"] & 512) for v in fv], sched
        acc = [x for x in sched if x[1] != "S"]
        if len({t for t, _ in acc}) <= 1 or all(op == "R" for _, op in acc):
            assert not any(got), sched


def test_failed_copies_record_nothing():
    """R-34: a copy with an Error is checked but not performed, so it leaves no stamp."""
    tb = tg.TraceBuilder("fail", H0, 1 << 16)
    tb.mark(H0, 1 << 16, tg.DEFINED)
    d = tb.malloc(256)
    tb.thread = 1
    tb.copy1d(tg.HTOD, d, H0, 512)          # DstTooSmall: not performed
    tb.thread = 2
    tb.copy1d(tg.DTOH, H0 + 4096, d, 256)   # nothing recorded on d before
    tb.copy1d(tg.HTOD, d, H0, 256)          # thread 2 again
    tb.thread = 1
    tb.copy1d(tg.HTOD, d, H0 + 8192, 256)   # thread 1 after thread 2's write -> hazard
    o, v, s, _ = oracle.replay_trace(tb.build(), concurrency=True)
    assert [bool(f & F_CONC) for f in v["flags"]] == [False, False, False, True]
    assert v[0]["status"] == 1


def test_disjoint_ranges_never_race():
    tb = tg.TraceBuilder("disj", H0, 1 << 16)
    tb.mark(H0, 1 << 16, tg.DEFINED)
    d = tb.malloc(4096)
    for k in range(16):
        tb.thread = k % 4
        tb.copy1d(tg.HTOD, d + 256 * k, H0 + 256 * k, 256)   # adjacent, not overlapping
    o, v, s, _ = oracle.replay_trace(tb.build(), concurrency=True)
    assert not (v["flags"] & F_CONC).any()


def test_single_thread_traces_unchanged():
    """concurrency mode changes nothing for a single-threaded program"""
    for seed in range(10):
        tr = tg.random_tiny(seed)
        a = oracle.replay_trace(tr, concurrency=True)
        b = oracle.replay_trace(tr)
        assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])


@pytest.mark.parametrize("seed", range(60))
def test_flat_model_equivalence_threads(seed):
    tr = tg.random_tiny(seed + 40000, threads=int(2 + seed % 3), arrays=seed % 2 == 1)
    o, v, s, _ = oracle.replay_trace(tr, concurrency=True)
    fm = FlatModel(tr.host_base, tr.host_size, conc=True)
    fv, fs = fm.replay(tr.events, tr.blob, tr.threads)
    assert list(s) == fs
    for i, (a, b) in enumerate(zip(v, fv)):
        assert {k: int(a[k]) for k in v.dtype.names} == b, i
    assert np.array_equal(o.V, fm.v)


def test_random_traces_have_hazards():
    n = sum(int((oracle.replay_trace(tg.random_tiny(s, threads=3), concurrency=True)[1]["flags"] & F_CONC).any())
            for s in range(20))
    assert n >= 15
