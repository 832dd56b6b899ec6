"""Brute force and invariants pinning the oracle on tiny inputs (CPU only).

* exhaustive over every (kind, start, len) in a 64-byte host window with
  fixed random A/V (numpy one-liners: np.flatnonzero / np.count_nonzero);
* every device query against 4 allocations (``bisect`` over sorted bases);
* 2D special cases that reduce to 1D (pitch = W, X = 0; H = 1);
* SPEC S:546 flat-model equivalence on random <=200-event traces
  (tests/flatmodel.py, an independent numpy/bisect implementation);
* SPEC invariants S:41, and the adapted round trip.
"""
import bisect

import numpy as np
import pytest

import oracle
import tracegen as tg
from flatmodel import FlatModel
from oracle import NONE, Oracle


def _copy(kind, dst, src, n, seq, **kw):
    e = np.zeros(1, tg.EVENT_DTYPE)[0]
    e["op"] = tg.OP_COPY; e["kind"] = kind; e["seq"] = seq
    e["width"] = n; e["height"] = 1; e["dst"] = dst; e["src"] = src
    e["dst_pitch"] = n; e["src_pitch"] = n
    for k, v in kw.items():
        e[k] = v
    return e


def test_exhaustive_host_window_64():
    H0 = 0x10000
    rng = np.random.default_rng(7)
    abits = rng.random(4096) < 0.8
    vbytes = np.where(rng.random(4096) < 0.3, rng.integers(1, 256, 4096), 0).astype(np.uint8)
    o = Oracle(H0, 4096)
    # materialise the random A/V through the public calls
    for i in range(64):
        if abits[i]:
            o.mark(H0 + i, 1, tg.DEFINED)
            if vbytes[i]:
                o.set_vbits(H0 + i, bytes([vbytes[i]]))
    dev = 0x1000000
    o.register(dev, 1 << 20, 1)
    seq = 2
    for kind in (tg.HTOD, tg.DTOH):
        for start in range(H0 - 4, H0 + 68):
            for n in range(0, 73):
                if kind == tg.HTOD:
                    e = _copy(kind, dev, start, n, seq)
                else:
                    e = _copy(kind, start, dev, n, seq)
                seq += 1
                # brute force
                xs = np.arange(start, start + n)
                inwin = (xs >= H0) & (xs < H0 + 64)
                a = np.zeros(n, bool)
                a[inwin] = abits[xs[inwin] - H0]
                bad = np.flatnonzero(~a)
                exp_unaddr = int(bad[0]) if len(bad) else NONE
                if kind == tg.HTOD:
                    vv = np.zeros(n, np.uint8)
                    vv[inwin] = np.where(abits[xs[inwin] - H0], vbytes[xs[inwin] - H0], 0xFF)
                    und = a & (vv != 0)
                    u = np.flatnonzero(und)
                    exp_first, exp_cnt = (int(u[0]) if len(u) else NONE), int(np.count_nonzero(und))
                else:
                    exp_first, exp_cnt = NONE, 0
                v = o.check_copy(e)
                if kind == tg.DTOH and v["status"] == 0 and n:
                    # restore V (the DtoH applied); the brute force is per-call
                    for i in range(64):
                        if abits[i]:
                            o.set_vbits(H0 + i, bytes([vbytes[i]]))
                assert (int(v["first_unaddr"]), int(v["first_undef"]), int(v["undef_count"])) == \
                    (exp_unaddr, exp_first, exp_cnt), (kind, start, n)


def test_every_device_query_against_4_allocations():
    rng = np.random.default_rng(11)
    o = Oracle(0x10000, 4096)
    bases, sizes = [], []
    cur = 0x2000
    for k in range(4):
        sz = int(rng.integers(1, 200))
        bases.append(cur); sizes.append(sz)
        o.register(cur, sz, k + 1)
        cur += sz + (0 if k == 1 else int(rng.integers(1, 40)))   # allocations 1,2 adjacent
    seq = 10
    for start in range(0x2000 - 8, cur + 8):
        for n in (0, 1, 7, 64, 300):
            v = o.check_copy(_copy(tg.DTOD, start, bases[0], n, seq))
            seq += 1
            i = bisect.bisect_right(bases, start) - 1
            if i < 0 or start >= bases[i] + sizes[i]:
                assert v["flags"] & 1 and v["dst_found"] == 0, start
            else:
                avail = bases[i] + sizes[i] - start
                if avail < n:
                    assert v["flags"] & 2 and (v["dst_expected"], v["dst_found"]) == (n, avail)
                else:
                    assert not v["flags"] & 3


def test_2d_reduces_to_1d():
    """2D with pitch = W and X = 0 equals 1D of W*H; H = 1 equals 1D."""
    rng = np.random.default_rng(3)
    H0 = 0x10000
    o = Oracle(H0, 1 << 16)
    o.mark(H0, 1 << 16, tg.DEFINED)
    for _ in range(200):
        a = H0 + int(rng.integers(0, 1 << 16)); n = int(rng.integers(0, 300))
        st = int(rng.integers(0, 3))
        if a + n <= H0 + (1 << 16):
            o.mark(a, n, st)
    o.register(0x1000000, 1 << 20, 1)
    seq = 2
    for _ in range(400):
        w = int(rng.integers(0, 300)); h = int(rng.integers(0, 40))
        hs = H0 + int(rng.integers(0, 1 << 16)) - 100
        kind = int(rng.choice([tg.HTOD, tg.DTOH]))
        if kind == tg.HTOD:
            e2 = _copy(kind, 0x1000000, hs, w, seq, height=h, dst_pitch=w, src_pitch=w)
            e1 = _copy(kind, 0x1000000, hs, w * h, seq + 1)
        else:
            e2 = _copy(kind, hs, 0x1000000, w, seq, height=h, dst_pitch=w, src_pitch=w)
            e1 = _copy(kind, hs, 0x1000000, w * h, seq + 1)
        seq += 2
        if kind == tg.DTOH:
            # evaluate both on the same state: check without apply via a fresh copy
            snapV = o.V.copy()
        v2 = o.check_copy(e2)
        if kind == tg.DTOH:
            o.V[:] = snapV
        v1 = o.check_copy(e1)
        if kind == tg.DTOH:
            o.V[:] = snapV
        for f in ("first_unaddr", "first_undef", "undef_count", "flags", "status"):
            assert v1[f] == v2[f], (f, w, h)
        # H = 1 2D (with an arbitrary pitch >= W) equals 1D
        p = w + int(rng.integers(0, 50))
        if kind == tg.HTOD:
            e3 = _copy(kind, 0x1000000, hs, w, seq, dst_pitch=p, src_pitch=p)
            e4 = _copy(kind, 0x1000000, hs, w, seq + 1)
        else:
            e3 = _copy(kind, hs, 0x1000000, w, seq, dst_pitch=p, src_pitch=p)
            e4 = _copy(kind, hs, 0x1000000, w, seq + 1)
        seq += 2
        snapV = o.V.copy()
        v3 = o.check_copy(e3); o.V[:] = snapV
        v4 = o.check_copy(e4); o.V[:] = snapV
        for f in ("first_unaddr", "first_undef", "undef_count", "flags", "status"):
            assert v3[f] == v4[f]


@pytest.mark.parametrize("seed", range(60))
def test_flat_model_equivalence(seed):
    """random <=200-event traces in a 64 KiB window; zero mismatches."""
    tr = tg.random_tiny(seed)
    o, v, s, leaks = oracle.replay_trace(tr)
    fm = FlatModel(tr.host_base, tr.host_size)
    fv, fs = fm.replay(tr.events, tr.blob)
    assert list(s) == fs
    assert len(v) == len(fv)
    for i, (a, b) in enumerate(zip(v, fv)):
        assert {k: int(a[k]) for k in v.dtype.names} == b, i
    assert np.array_equal(o.V, fm.v)
    assert np.array_equal(o.A, fm.packed_a())
    assert [(int(l["base"]), int(l["size"]), int(l["seq"])) for l in leaks] == fm.leaks()


@pytest.mark.parametrize("seed", range(20))
def test_no_mutation_on_error(seed):
    """injecting one guaranteed-Error call at a random position
    leaves all other verdicts and the final state unchanged."""
    tr = tg.random_tiny(seed + 1000)
    rng = np.random.default_rng(seed)
    _, v0, s0, l0 = oracle.replay_trace(tr)
    o0 = oracle.replay_trace(tr)[0]
    pos = int(rng.integers(0, len(tr.events) + 1))
    bad = np.zeros(1, tg.EVENT_DTYPE)
    # a DtoH from an address that is never allocated: an Error, so no apply
    bad[0] = _copy(tg.DTOH, tr.host_base + 64, 0x7000_0000_0000, 512, 0)
    ev = np.concatenate([tr.events[:pos], bad, tr.events[pos:]])
    ev["seq"] = np.arange(1, len(ev) + 1)
    o1 = Oracle(tr.host_base, tr.host_size)
    v1, s1 = o1.replay(ev, tr.blob)
    k = int(np.count_nonzero(tr.events["op"][:pos] == tg.OP_COPY))
    assert v1[k]["status"] == 1
    others = np.delete(v1, k)
    assert np.array_equal(others, v0)
    assert np.array_equal(o1.V, o0.V) and np.array_equal(o1.A, o0.A)


def test_invariants_on_fuzz():
    for seed in range(40):
        tr = tg.random_tiny(seed + 500)
        o, v, s, leaks = oracle.replay_trace(tr)
        # S:41 fully_defined <=> count == 0 <=> first absent
        assert np.all((v["undef_count"] == 0) == (v["first_undef"] == NONE))
        # S:366 status = InvalidValue iff >= 1 Error flag
        err = v["flags"] & ~np.uint32(oracle.F_HOST_UNDEFINED)
        assert np.all((v["status"] == 1) == (err != 0))
        # R-4: HOST_UNDEFINED flag only when the range is fully addressable
        hu = (v["flags"] & oracle.F_HOST_UNDEFINED) != 0
        assert np.all(v["first_unaddr"][hu] == NONE)
        # R-19: expected/found only for TooSmall
        assert np.all((v["dst_found"] != 0) <= ((v["flags"] & oracle.F_DST_TOO_SMALL) != 0))
        # S:419 determinism
        _, v2, s2, _ = oracle.replay_trace(tr)
        assert np.array_equal(v, v2) and np.array_equal(s, s2)


def test_fully_defined_input_gives_no_reports_and_dtoh_defines():
    """BASELINE north_star pins: fully defined input -> zero reports;
    DtoH makes the range defined (adapted round trip)."""
    rng = np.random.default_rng(5)
    H0 = 0x100000
    tb = tg.TraceBuilder("rt", H0, 1 << 20)
    d = tb.malloc(1 << 16)
    src = H0 + 4096
    tb.mark(src, 5000, tg.DEFINED)
    pattern = rng.integers(0, 256, 5000, dtype=np.uint8)
    tb.copy1d(tg.HTOD, d, src, 5000)                      # fully defined: clean
    tb.setv(src, pattern.tobytes())                        # any host pattern
    tb.copy1d(tg.HTOD, d, src, 5000)                       # now undefined bytes reported
    dst = H0 + 65536
    tb.mark(dst, 5000, tg.UNDEFINED)                       # fresh range
    tb.copy1d(tg.DTOH, dst, d, 5000)                       # error-free DtoH
    tb.copy1d(tg.HTOD, d, dst, 5000)                       # the range is now defined
    o, v, s, _ = oracle.replay_trace(tb.build())
    assert v[0]["flags"] == 0
    assert v[1]["undef_count"] == int(np.count_nonzero(pattern))
    assert v[2]["flags"] == 0 and v[3]["flags"] == 0
    assert not o.V[65536:65536 + 5000].any()
