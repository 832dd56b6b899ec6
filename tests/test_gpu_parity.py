"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bit-exact on every verdict field, every call status, the leak list and the
final host shadow (A and V arrays).  Small cases replay whole traces on both
sides; the full-size configurations are run on the GPU in the launch
configuration bench.py times and compared on a sample of descriptors the
oracle recomputes (exact for C2/C4 because their copies are independent --
private host ranges, one hazard-free batch) and through properties that hold
at any size (C2 dirty set = injected set, C3 closed form).
"""
import numpy as np
import pytest

import oracle
import tracegen as tg

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cg():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1310_0901_b200 import build
    build.build()
    import paper_1310_0901_b200 as m
    return m


def new_checker(cg, tr, **kw):
    kw.setdefault("max_descs", max(tr.n_copies, 1024))
    kw.setdefault("max_allocs", max(int(np.count_nonzero(tr.events["op"] == tg.OP_REG)), 1024))
    return cg.Checker(tr.host_base, tr.host_size, **kw)


def assert_verdicts_equal(gv, ov, where=""):
    assert len(gv) == len(ov)
    for f in ov.dtype.names:
        a, b = np.asarray(gv[f]), np.asarray(ov[f])
        bad = np.flatnonzero(a != b)
        assert len(bad) == 0, f"{where} field {f}: {len(bad)} mismatches, first at {bad[:5]}: gpu {a[bad[:5]]} oracle {b[bad[:5]]}"


def run_parity(cg, tr, undef_is_error=False, fuse=True, **kw):
    o, ov, os_, oleaks = oracle.replay_trace(tr, undef_is_error=undef_is_error)
    chk = new_checker(cg, tr, undef_is_error=undef_is_error, **kw)
    gv, gs = cg.replay_events(chk, tr.events, tr.blob, fuse=fuse)
    assert_verdicts_equal(gv, ov, tr.name)
    assert np.array_equal(gs, os_), np.flatnonzero(gs != os_)[:10]
    gl = chk.leak_report()
    assert np.array_equal(gl["base"], oleaks["base"]) and np.array_equal(gl["size"], oleaks["size"])
    assert np.array_equal(gl["alloc_seq"], oleaks["seq"])
    A, V = chk.shadow()
    assert np.array_equal(A, o.A), "final A differs"
    assert np.array_equal(V, o.V), "final V differs"
    chk.close()
    return gv


def test_toy_trace(cg):
    v = run_parity(cg, tg.toy())
    assert v[1]["first_undef"] == 100 and v[1]["undef_count"] == 33


def test_listing2_golden(cg):
    v = run_parity(cg, tg.listing2())
    assert (v[2]["src_expected"], v[2]["src_found"]) == (8000000, 4000000)


@pytest.mark.parametrize("seed", range(120))
def test_random_tiny_traces(cg, seed):
    run_parity(cg, tg.random_tiny(seed))


@pytest.mark.parametrize("seed", range(40))
def test_random_tiny_unfused(cg, seed):
    """check and apply as two calls (cg_check_copies + cg_apply_dtoh)"""
    run_parity(cg, tg.random_tiny(seed + 3000), fuse=False)


@pytest.mark.parametrize("seed", range(8))
def test_random_tiny_undef_is_error(cg, seed):
    run_parity(cg, tg.random_tiny(seed + 7000), undef_is_error=True)


@pytest.mark.parametrize("seed", range(6))
def test_random_larger_windows(cg, seed):
    """bigger windows and copies: several chunks per descriptor, ragged tails"""
    tr = tg.random_tiny(seed + 9000, n_events=400, window=4 << 20, host_base=0x4000000)
    run_parity(cg, tr)


def test_small_max_descs_splits_batches(cg):
    run_parity(cg, tg.random_tiny(4242, n_events=300), max_descs=7)


@pytest.mark.parametrize("fuse", [True, False])
def test_c2_scaled(cg, fuse):
    tr = tg.c2_small(n_copies=60000, n_allocs=6000)
    v = run_parity(cg, tr, fuse=fuse)
    assert np.array_equal(v["flags"] != 0, tr.meta["inject"] != 0)


def test_c3_scaled(cg):
    tr = tg.c3_single(size=256 << 20)
    v = run_parity(cg, tr)
    assert v[0]["undef_count"] == len(tr.meta["hole_offsets"])
    assert v[0]["first_undef"] == tr.meta["hole_offsets"][0]


@pytest.mark.parametrize("fuse", [True, False])
def test_c3_dtoh_scaled(cg, fuse):
    run_parity(cg, tg.c3_single(size=128 << 20, dtoh=True), fuse=fuse)


def test_c4_scaled(cg):
    tr = tg.c4_pitched(n_copies=4000, n_bufs=4, rows=256, inject_frac=0.03)
    run_parity(cg, tr)


def test_mark_batch_larger_than_max_descs(cg):
    """2048 consecutive host marks through a context with max_descs = 1000"""
    tr = tg.c4_pitched(n_copies=900, n_bufs=4, rows=256, inject_frac=0.03)
    run_parity(cg, tr, max_descs=1000)


# ---------------------------------------------------------------------------
# edge cases of the ABI
# ---------------------------------------------------------------------------
def test_empty_and_oversized_batches(cg):
    import torch
    tr = tg.toy()
    chk = new_checker(cg, tr, max_descs=16)
    d = torch.empty(0, dtype=torch.uint8, device="cuda")
    assert cg.cg_check_copies(chk.ctx, d.data_ptr(), 0, d.data_ptr(), None) == 0
    big = cg.to_device_descs(np.zeros(17, cg.DESC_DTYPE))
    out = torch.empty(17 * 64, dtype=torch.uint8, device="cuda")
    assert cg.cg_check_copies(chk.ctx, big.data_ptr(), 17, out.data_ptr(), None) == cg.CG_ERR_INVALID_VALUE
    assert cg.cg_check_copies(chk.ctx, None, 1, out.data_ptr(), None) == cg.CG_ERR_INVALID_VALUE
    chk.close()


def test_registry_errors_match_spec(cg):
    tr = tg.toy()
    chk = new_checker(cg, tr, max_allocs=2)
    assert chk.register_alloc(0x1000, 16, 1) == 0
    assert chk.register_alloc(0x1000, 16, 2) == cg.CG_ERR_INVALID_VALUE          # S:146 overlap
    assert chk.register_alloc(0x2000, 0, 3) == cg.CG_ERR_INVALID_VALUE           # S:330 size 0
    assert chk.register_alloc(0, 16, 4) == cg.CG_ERR_INVALID_VALUE               # base 0
    assert chk.register_alloc(0x3000, 16, 4) == 0
    assert chk.register_alloc(0x4000, 16, 5) == cg.CG_ERR_OUT_OF_MEMORY           # table full
    assert chk.free(0x1008, 6) == cg.CG_ERR_INVALID_VALUE                         # S:339 offset free
    assert chk.free(0x1000, 7) == 0
    assert chk.free(0x1000, 8) == cg.CG_ERR_INVALID_VALUE                         # S:340 double free
    assert chk.free(0x3000, 7) == cg.CG_ERR_INVALID_VALUE                         # seq not increasing
    leaks = chk.leak_report()
    assert list(leaks["base"]) == [0x3000]
    assert cg.cg_registry_compact(chk.ctx, 10) == 0
    assert chk.register_alloc(0x4000, 16, 11) == 0                                # tombstone dropped
    chk.close()


def test_marks_and_setv_errors(cg):
    tr = tg.toy()
    chk = new_checker(cg, tr)
    H0, S = tr.host_base, tr.host_size
    m = np.zeros(4, cg.MARK_DTYPE)
    m[0] = (H0, 64, cg.CG_DEFINED, 0)
    m[1] = (H0 + S - 8, 16, cg.CG_DEFINED, 0)       # leaves the window: skipped
    m[2] = (H0 + 128, 64, 7, 0)                     # bad state: skipped
    m[3] = (H0 + 32, 64, cg.CG_UNDEFINED, 0)        # overlaps m[0]: applied after it
    st = np.zeros(4, np.uint32)
    assert chk.host_mark_batch(m, status_out=st) == cg.CG_ERR_INVALID_VALUE
    assert list(st) == [0, 1, 1, 0]
    assert chk.host_set_vbits(H0 + 200, b"\x01") == cg.CG_ERR_INVALID_VALUE   # unaddressable
    assert chk.host_set_vbits(H0 + 40, b"\x01\x02") == 0
    A, V = chk.shadow()
    o = oracle.Oracle(H0, S)
    o.mark(H0, 64, tg.DEFINED); o.mark(H0 + 32, 64, tg.UNDEFINED); o.set_vbits(H0 + 40, b"\x01\x02")
    assert np.array_equal(A, o.A) and np.array_equal(V, o.V)
    chk.close()


def test_check_copies_host_matches_device_path(cg):
    tr = tg.c2_small(n_copies=20000, n_allocs=2000)
    o, ov, _, _ = oracle.replay_trace(tr)
    chk = new_checker(cg, tr, host_staging=True)
    from paper_1310_0901_b200.replay import events_to_descs
    ev = tr.events
    marks = ev[ev["op"] == tg.OP_MARK]
    m = np.zeros(len(marks), cg.MARK_DTYPE)
    m["addr"], m["len"], m["state"] = marks["dst"], marks["width"], marks["kind"]
    assert chk.host_mark_batch(m) == 0
    for e in ev[ev["op"] == tg.OP_SETV]:
        assert chk.host_set_vbits(int(e["dst"]), bytes(tr.blob[int(e["src"]):int(e["src"]) + int(e["width"])])) == 0
    for e in ev[(ev["op"] == tg.OP_REG) | (ev["op"] == tg.OP_FREE)]:
        if e["op"] == tg.OP_REG:
            assert chk.register_alloc(int(e["dst"]), int(e["width"]), int(e["seq"])) == 0
        else:
            assert chk.free(int(e["dst"]), int(e["seq"])) == 0
    gv = chk.check_copies_host(events_to_descs(ev[ev["op"] == tg.OP_COPY]), apply=True)
    assert_verdicts_equal(gv, ov, "host path")
    A, V = chk.shadow()
    assert np.array_equal(V, o.V) and np.array_equal(A, o.A)
    chk.close()


def test_leak_sweep_device(cg):
    import torch
    tr = tg.c2_small(n_copies=5000, n_allocs=3000)
    o, _, _, oleaks = oracle.replay_trace(tr)
    chk = new_checker(cg, tr)
    cg.replay_events(chk, tr.events, tr.blob)
    out = torch.zeros(len(oleaks) * 24, dtype=torch.uint8, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    chk.leak_sweep(out, len(oleaks), cnt)
    torch.cuda.synchronize()
    rec = out.cpu().numpy().view(cg.ALLOC_RECORD_DTYPE)
    assert int(cnt.item()) == len(oleaks)
    assert np.array_equal(rec["base"], oleaks["base"]) and np.array_equal(rec["alloc_seq"], oleaks["seq"])
    chk.close()


@pytest.mark.parametrize("coop", ["1", "0"])
@pytest.mark.parametrize("cap_frac", [1.0, 0.37])
def test_leak_sweep_device_large_capped(cg, monkeypatch, coop, cap_frac):
    """a8 on a 100k-entry table (many grid slices), the cooperative one-launch
    sweep (CG_LEAK_COOP=1) and the 5-launch one: the count is the full k, the
    first min(cap, k) records in base order equal the oracle's."""
    import torch
    monkeypatch.setenv("CG_LEAK_COOP", coop)
    tr = tg.c2_small(n_copies=2000, n_allocs=100000)
    o, _, _, oleaks = oracle.replay_trace(tr)
    chk = new_checker(cg, tr)
    cg.replay_events(chk, tr.events, tr.blob)
    k = len(oleaks)
    cap = max(1, int(k * cap_frac))
    out = torch.full((k * 24,), 0xAB, dtype=torch.uint8, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    chk.leak_sweep(out, cap, cnt)
    torch.cuda.synchronize()
    rec = out.cpu().numpy().view(cg.ALLOC_RECORD_DTYPE)
    assert int(cnt.item()) == k
    assert np.array_equal(rec["base"][:cap], oleaks["base"][:cap])
    assert np.array_equal(rec["alloc_seq"][:cap], oleaks["seq"][:cap])
    assert np.all(out.cpu().numpy()[cap * 24:] == 0xAB)   # nothing written past cap
    chk.close()


@pytest.mark.parametrize("fmt", ["1d", "2d"])
def test_check_host_compact_chunked(cg, fmt):
    """cg_check_host: 600k host descriptors (4 pipelined chunks), dirty-only
    result; the dense verdicts it implies equal the oracle's."""
    from paper_1310_0901_b200.replay import events_to_descs
    tr = tg.c2_small(n_copies=600000, n_allocs=2000)
    o, ov, _, _ = oracle.replay_trace(tr)
    chk = new_checker(cg, tr, host_staging=True)
    ev = tr.events
    _, st = cg.replay_events(chk, ev[ev["op"] != tg.OP_COPY], tr.blob)
    assert not st.any()
    descs = events_to_descs(ev[ev["op"] == tg.OP_COPY])
    if fmt == "1d":
        d1 = np.zeros(len(descs), cg.COPY1D_DTYPE)
        for f in ("kind", "seq", "dst", "src"):
            d1[f] = descs[f]
        d1["bytes"] = descs["width"]
        nd, idx, dirty = chk.check_host(d1, apply=2)
    else:
        nd, idx, dirty = chk.check_host(descs, apply=2)
    dense = np.zeros(len(descs), cg.VERDICT_DTYPE)
    dense["first_unaddr"] = cg.CG_NONE
    dense["first_undef"] = cg.CG_NONE
    dense[idx.astype(np.int64)] = dirty
    assert nd == int(np.count_nonzero(ov["flags"]))
    assert_verdicts_equal(dense, ov, "check_host")
    A, V = chk.shadow()
    assert np.array_equal(V, o.V) and np.array_equal(A, o.A)
    chk.close()


@pytest.mark.parametrize("parts", [2, 5])
def test_check_host_submit_pipelined(cg, parts):
    """cg_check_host_submit / _wait: the batch cut into consecutive parts,
    part k+1 submitted to the other staging slot before part k is waited
    for; the dense verdicts and the final shadow equal the oracle's
    sequential replay.  Misuse of a slot is an invalid call."""
    from paper_1310_0901_b200.replay import events_to_descs
    tr = tg.c2_small(n_copies=300000, n_allocs=2000)
    o, ov, _, _ = oracle.replay_trace(tr)
    chk = new_checker(cg, tr, host_staging=True)
    ev = tr.events
    _, st = cg.replay_events(chk, ev[ev["op"] != tg.OP_COPY], tr.blob)
    assert not st.any()
    descs = events_to_descs(ev[ev["op"] == tg.OP_COPY])
    d1 = np.zeros(len(descs), cg.COPY1D_DTYPE)
    for f in ("kind", "seq", "dst", "src"):
        d1[f] = descs[f]
    d1["bytes"] = descs["width"]
    cuts = np.linspace(0, len(d1), parts + 1).astype(np.int64)
    pieces = [d1[a:b] for a, b in zip(cuts[:-1], cuts[1:])]
    dense = np.zeros(len(descs), cg.VERDICT_DTYPE)
    dense["first_unaddr"] = cg.CG_NONE
    dense["first_undef"] = cg.CG_NONE
    total = 0
    chk.check_host_submit(pieces[0], 0, apply=2)
    with pytest.raises(cg.CgError):
        chk.check_host_submit(pieces[0], 0, apply=2)   # slot 0 is busy
    with pytest.raises(cg.CgError):
        chk.check_host_wait(1, 16)                     # nothing submitted to slot 1
    for k in range(parts):
        if k + 1 < parts:
            chk.check_host_submit(pieces[k + 1], (k + 1) % 2, apply=2)
        nd, idx, dirty = chk.check_host_wait(k % 2, len(pieces[k]))
        dense[idx.astype(np.int64) + cuts[k]] = dirty
        total += nd
    with pytest.raises(cg.CgError):
        chk.check_host_submit(pieces[0], 2, apply=2)   # no slot 2
    assert total == int(np.count_nonzero(ov["flags"]))
    assert_verdicts_equal(dense, ov, "check_host_submit")
    A, V = chk.shadow()
    assert np.array_equal(V, o.V) and np.array_equal(A, o.A)
    chk.close()


def test_unknown_op_status(cg):
    """an unknown event op is an invalid call on both sides (oracle status 1)"""
    tr = tg.random_tiny(5)
    ev = tr.events.copy()
    ev[3]["op"] = 42
    tr2 = tg.Trace(tr.name, ev, tr.blob, tr.host_base, tr.host_size, tr.meta)
    run_parity(cg, tr2)
