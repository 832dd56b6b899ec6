"""Pins for the CPU oracle against things other than itself (CPU only).

Each test names the passage it pins.  Kinds of pin used (task ③):
  * values the paper prints for its worked example  (Listing 2 -> Listing 5)
  * SPEC.md's per-operation examples
  * hand-computed golden verdicts of the toy trace  (tests/golden/toy_a1.tsv)
  * closed forms of the synthetic configs           (C3: count = #holes, first = first hole)
"""
import os

import numpy as np
import pytest

import oracle
import tracegen as tg
from oracle import (F_BAD_KIND, F_BAD_PITCH, F_DST_NOT_ALLOCATED, F_DST_TOO_SMALL,
                    F_HOST_UNADDRESSABLE, F_HOST_UNDEFINED, F_INVALID_RANGE,
                    F_SRC_NOT_ALLOCATED, F_SRC_TOO_SMALL, NONE, Oracle)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def ev_copy(kind, dst, src, n, seq):
    e = np.zeros(1, tg.EVENT_DTYPE)[0]
    e["op"] = tg.OP_COPY; e["kind"] = kind; e["seq"] = seq
    e["width"] = n; e["height"] = 1; e["dst"] = dst; e["src"] = src
    e["dst_pitch"] = n; e["src_pitch"] = n
    return e


def ev_copy2d(kind, w, h, dst, dx, dy, dp, src, sx, sy, sp, seq):
    e = np.zeros(1, tg.EVENT_DTYPE)[0]
    e["op"] = tg.OP_COPY; e["kind"] = kind; e["seq"] = seq; e["width"] = w; e["height"] = h
    e["dst"], e["dst_x"], e["dst_y"], e["dst_pitch"] = dst, dx, dy, dp
    e["src"], e["src_x"], e["src_y"], e["src_pitch"] = src, sx, sy, sp
    return e


# --------------------------------------------------------------------------
# The paper's worked example (P:129-146 -> P:233-235)
# --------------------------------------------------------------------------
def test_listing5_golden():
    lines = [l for l in open(os.path.join(GOLDEN, "listing5.txt")) if not l.startswith("#")]
    assert "device->host" in lines[0] and "too small" in lines[0]
    words = lines[1].split()
    expected, found = int(words[1]), int(words[-1].rstrip("."))
    tr = tg.listing2()
    o, v, s, leaks = oracle.replay_trace(tr)
    assert len(v) == 3
    assert v[0]["flags"] == 0 and v[1]["flags"] == 0          # HtoD fills of a, b are clean
    bad = v[2]
    assert bad["flags"] == F_SRC_TOO_SMALL                      # "device->host", src side
    assert (bad["src_expected"], bad["src_found"]) == (expected, found) == (8000000, 4000000)
    assert bad["status"] == 1                                   # "invalid argument"
    assert int(np.count_nonzero(s)) == 1                        # exactly one Error
    # no apply on error (the copy fails): c_host stays undefined
    c_host = tr.meta["c_host"] - tr.host_base
    assert np.all(o.V[c_host:c_host + 8000000] == 0xFF)
    assert len(leaks) == 3                                      # c, a, b never freed


def _parse_golden_toy():
    rows, leaks = {}, []
    for line in open(os.path.join(GOLDEN, "toy_a1.tsv")):
        if line.startswith("#") or not line.strip():
            continue
        f = line.split()
        if f[0] == "LEAK":
            leaks.append((int(f[1], 16), int(f[2])))
            continue
        rows[f[0]] = [NONE if x == "NONE" else int(x) for x in f[1:]]
    return rows, leaks


def test_toy_trace_golden():
    rows, gleaks = _parse_golden_toy()
    tr = tg.toy()
    o, v, s, leaks = oracle.replay_trace(tr)
    names = list(v.dtype.names)
    for i in range(10):
        assert [int(v[i][n]) for n in names] == rows[f"C{i + 1}"], f"C{i + 1}"
    assert [(int(l["base"]), int(l["size"])) for l in leaks] == gleaks
    # final host state: h0..h3 fully defined (Appendix A.1 totals)
    for h, n in zip(tr.meta["h"], [256, 1024, 4096, 4096]):
        assert np.all(o.V[h - tr.host_base:h - tr.host_base + n] == 0)


# --------------------------------------------------------------------------
# SPEC shadow_memory examples
# --------------------------------------------------------------------------
def test_spec_mark_and_check_examples():
    o = Oracle(0x1000 * 16, 1 << 16)
    H = 0x10000
    # S:51 mark 8 bytes addressable, undefined -> 8 addressable bytes, 64 undefined V-bits
    assert o.mark(H, 8, tg.UNDEFINED) == 0
    assert np.all(np.unpackbits(o.A[0:1], bitorder="little") == 1)
    assert np.all(o.V[0:8] == 0xFF)
    # S:52 zero length leaves the map unchanged
    before = (o.A.copy(), o.V.copy())
    assert o.mark(H + 100, 0, tg.DEFINED) == 0
    assert np.array_equal(before[0], o.A) and np.array_equal(before[1], o.V)
    # S:60 mark, unmark, query -> unaddressable
    o.mark(H + 64, 8, tg.DEFINED); o.mark(H + 64, 8, tg.NOACCESS)
    assert o.A[8] == 0
    # S:70 range extending 1 byte past an interval -> offset = interval_len
    seq = 10
    o.mark(H + 256, 100, tg.DEFINED)
    o.register(0x100000, 1 << 12, seq); seq += 1
    v = o.check_copy(ev_copy(tg.HTOD, 0x100000, H + 256, 101, seq)); seq += 1
    assert v["first_unaddr"] == 100 and v["flags"] & F_HOST_UNADDRESSABLE and v["status"] == 1
    # S:69 fully tracked range -> absent
    v = o.check_copy(ev_copy(tg.HTOD, 0x100000, H + 256, 100, seq)); seq += 1
    assert v["first_unaddr"] == NONE and v["flags"] == 0
    # S:79 8-byte range with only byte 3 undefined -> first 3, count 1
    o.mark(H + 512, 8, tg.DEFINED)
    o.set_vbits(H + 512 + 3, b"\x01")
    v = o.check_copy(ev_copy(tg.HTOD, 0x100000, H + 512, 8, seq)); seq += 1
    assert (v["first_undef"], v["undef_count"]) == (3, 1)
    assert v["flags"] == F_HOST_UNDEFINED and v["status"] == 0      # Warning
    # S:78 freshly marked-defined range -> fully defined (count 0 <=> first absent)
    v = o.check_copy(ev_copy(tg.HTOD, 0x100000, H + 256, 100, seq)); seq += 1
    assert v["undef_count"] == 0 and v["first_undef"] == NONE
    # S:75 a byte with any undefined bit counts: only the top bit undefined
    o.set_vbits(H + 512 + 3, b"\x80")
    v = o.check_copy(ev_copy(tg.HTOD, 0x100000, H + 512, 8, seq)); seq += 1
    assert (v["first_undef"], v["undef_count"]) == (3, 1)
    # S:74 set_vbits on unaddressable bytes is refused, nothing changes
    Vb = o.V.copy()
    assert o.set_vbits(H + 1000, b"\x00") == 1
    assert np.array_equal(Vb, o.V)
    # out-of-window mark refused (R-15)
    assert o.mark(H - 1, 4, tg.DEFINED) == 1


def test_undef_is_error_promotes_warning():
    """a CLI flag promotes HostUndefined to an Error."""
    for flag, status in ((False, 0), (True, 1)):
        o = Oracle(0x10000, 1 << 16, undef_is_error=flag)
        o.mark(0x10000, 16, tg.UNDEFINED)
        o.register(0x200000, 64, 1)
        v = o.check_copy(ev_copy(tg.HTOD, 0x200000, 0x10000, 16, 2))
        assert v["flags"] == F_HOST_UNDEFINED and v["status"] == status


# --------------------------------------------------------------------------
# SPEC device_registry / driver examples
# --------------------------------------------------------------------------
def test_spec_registry_examples():
    o = Oracle(0x10000, 1 << 16)
    o.mark(0x10000, 1 << 16, tg.DEFINED)
    # S:145 register 4,000,000 then coverage(base, 4,000,000) -> Covered
    assert o.register(0x10000000, 4000000, 1) == 0
    v = o.check_copy(ev_copy(tg.DTOD, 0x10000000, 0x10000000, 4000000, 2))
    assert v["flags"] == 0
    # S:163 query len 8,000,000 at base -> Truncated, available 4000000
    v = o.check_copy(ev_copy(tg.DTOD, 0x10000000, 0x10000000, 8000000, 3))
    assert v["flags"] == F_DST_TOO_SMALL | F_SRC_TOO_SMALL
    assert (v["dst_expected"], v["dst_found"]) == (8000000, 4000000)
    # S:164 one past end -> NotAllocated
    v = o.check_copy(ev_copy(tg.DTOD, 0x10000000 + 4000000, 0x10000000, 1, 4))
    assert v["flags"] == F_DST_NOT_ALLOCATED and v["dst_expected"] == 0   # R-19
    # S:146 register same base again -> OverlapWithLive
    assert o.register(0x10000000, 16, 5) == 1
    # S:141 size 0 / base 0 rejected (S:330 alloc 0 -> InvalidValue)
    assert o.register(0x20000000, 0, 6) == 1
    assert o.register(0, 16, 7) == 1
    # S:155 offset free rejected, S:340 double free
    assert o.free(0x10000000 + 8, 8) == 1
    assert o.free(0x10000000, 9) == 0
    assert o.free(0x10000000, 10) == 1
    # S:154 register, unregister, coverage -> NotAllocated
    v = o.check_copy(ev_copy(tg.DTOD, 0x10000000, 0x10000000, 1, 11))
    assert v["flags"] == F_DST_NOT_ALLOCATED | F_SRC_NOT_ALLOCATED
    # S:187 unregister(register(x)) restores the registry exactly
    assert len(o.leaks()) == 0
    # S:180 3 registers, 1 unregister -> 2 records, ordered by base
    o.register(0x30000000, 16, 12); o.register(0x20000000, 16, 13); o.register(0x40000000, 16, 14)
    o.free(0x30000000, 15)
    l = o.leaks()
    assert [int(x) for x in l["base"]] == [0x20000000, 0x40000000]
    assert [int(x) for x in l["seq"]] == [13, 14]
    # S:181 empty -> empty
    assert len(Oracle(0x10000, 4096).leaks()) == 0


def test_spec_checker_examples():
    H = 0x100000
    o = Oracle(H, 16 << 20)
    # S:228 8 MB defined host src, 8 MB dst region -> no diagnostics
    o.mark(H, 8 << 20, tg.DEFINED)
    o.register(0x10000000, 8 << 20, 1)
    v = o.check_copy(ev_copy(tg.HTOD, 0x10000000, H, 8 << 20, 2))
    assert v["flags"] == 0 and v["status"] == 0
    # S:229 host src with 1 undefined byte -> one Warning, count 1
    o.set_vbits(H + 12345, b"\xff")
    v = o.check_copy(ev_copy(tg.HTOD, 0x10000000, H, 8 << 20, 3))
    assert v["flags"] == F_HOST_UNDEFINED and v["undef_count"] == 1 and v["status"] == 0
    # S:238 / S:353 len 0 with valid pointers -> no diagnostics
    v = o.check_copy(ev_copy(tg.DTOH, H, 0x10000000, 0, 4))
    assert v["flags"] == 0
    v = o.check_copy(ev_copy(tg.HTOD, 0x10000000, H, 0, 5))
    assert v["flags"] == 0
    # S:247 src covers, dst short by 1 byte -> DstTooSmall with found = len-1
    o.register(0x20000000, 999, 6)
    v = o.check_copy(ev_copy(tg.DTOD, 0x20000000, 0x10000000, 1000, 7))
    assert v["flags"] == F_DST_TOO_SMALL and (v["dst_expected"], v["dst_found"]) == (1000, 999)
    # S:273 2 live regions at end -> 2 leaks; S:274 all freed -> empty
    assert len(o.leaks()) == 2
    o.free(0x10000000, 8); o.free(0x20000000, 9)
    assert len(o.leaks()) == 0


def test_listing2_variant_double_alloc_clean():
    """Fixing the bug of Listing 2 (sizeof(double) for c) removes the
    only diagnostic -- the 'sibling trace' of S:548."""
    tb = tg.TraceBuilder("fixed", 1 << 20, 32 << 20)
    c = tb.malloc(8000000)
    ch = 1 << 20
    tb.mark(ch, 8000000, tg.UNDEFINED)
    tb.copy1d(tg.DTOH, ch, c, 8000000)
    o, v, s, _ = oracle.replay_trace(tb.build())
    assert v[0]["flags"] == 0 and v[0]["status"] == 0
    assert np.all(o.V[:8000000] == 0)                 # DtoH marks defined (BASELINE (3))


def test_bad_kind_and_invalid_range():
    o = Oracle(0x10000, 1 << 16)
    e = ev_copy(7, 0x10000, 0x10000, 4, 1)
    v = o.check_copy(e)
    assert v["flags"] == F_BAD_KIND and v["status"] == 1
    e = ev_copy2d(tg.HTOD, 4, 2, 0x1000, 0, 1 << 62, 8, 0x10000, 0, 0, 8, 2)
    v = o.check_copy(e)
    assert v["flags"] & F_INVALID_RANGE and not v["flags"] & F_DST_NOT_ALLOCATED
    # pitch rule (R-12): pitch < W + X is BAD_PITCH, an Error, other checks still run
    e = ev_copy2d(tg.HTOD, 8, 2, 0x1000, 1, 0, 8, 0x10000, 0, 0, 8, 3)
    v = o.check_copy(e)
    assert v["flags"] & F_BAD_PITCH and v["flags"] & F_DST_NOT_ALLOCATED
    assert v["flags"] & F_HOST_UNADDRESSABLE and v["first_unaddr"] == 0


# --------------------------------------------------------------------------
# Closed forms of the synthetic configurations
# --------------------------------------------------------------------------
def test_c3_closed_form_scaled():
    """C3: one HtoD buffer with one undefined byte per stride; the count equals
    the number of holes and the first offset is the first hole's offset --
    both known without scanning."""
    tr = tg.c3_single(size=32 << 20, stride=1 << 16)
    o, v, s, leaks = oracle.replay_trace(tr)
    offs = tr.meta["hole_offsets"]
    assert v[0]["undef_count"] == len(offs) == 512
    assert v[0]["first_undef"] == offs[0]
    assert v[0]["first_unaddr"] == NONE and v[0]["flags"] == F_HOST_UNDEFINED
    assert len(leaks) == 1 and leaks[0]["size"] == 32 << 20


def test_c3_dtoh_variant_applies():
    tr = tg.c3_single(size=8 << 20, dtoh=True)
    o, v, s, _ = oracle.replay_trace(tr)
    assert v[0]["flags"] == 0
    assert not o.V[4096:4096 + (8 << 20)].any()
    assert np.all(o.V[:4096] == 0xFF) and np.all(o.V[4096 + (8 << 20):] == 0xFF)


def test_c2_dirty_set_equals_injected_set():
    """C2 gives every copy a private host range, so exactly the injected copies
    are dirty and each carries the flag of its injection class."""
    tr = tg.c2_small(n_copies=30000, n_allocs=3000)
    o, v, s, leaks = oracle.replay_trace(tr)
    inj = tr.meta["inject"]
    dirty = v["flags"] != 0
    assert np.array_equal(dirty, inj != 0)
    f = v["flags"]
    assert np.all(f[inj == tg.INJ_DST_NA] == F_DST_NOT_ALLOCATED)
    assert np.all(f[inj == tg.INJ_SRC_NA] == F_SRC_NOT_ALLOCATED)
    assert np.all(f[inj == tg.INJ_DTOD_BAD_SRC] == F_SRC_NOT_ALLOCATED)
    ts = f[inj == tg.INJ_TOO_SMALL]
    assert np.all((ts == F_DST_TOO_SMALL) | (ts == F_SRC_TOO_SMALL))
    assert np.all(f[inj == tg.INJ_HOST_UNADDR] == F_HOST_UNADDRESSABLE)
    assert np.all(f[inj == tg.INJ_HOST_UNDEF] == F_HOST_UNDEFINED)
    # HostUnaddressable: the first bad byte is exactly at the buffer end
    lens = tr.events[tr.copy_index]["width"]
    hu = np.flatnonzero(inj == tg.INJ_HOST_UNADDR)
    assert np.all(v["first_unaddr"][hu] < lens[hu])
    # registry: n_allocs registered, n_freed freed, the rest leak
    assert len(leaks) == tr.meta["n_allocs"] - tr.meta["n_freed"]
    assert int(np.count_nonzero(s)) == int(np.count_nonzero(v["status"]))


def test_c4_injection_classes():
    tr = tg.c4_pitched(n_copies=3000, n_bufs=2, rows=128, inject_frac=0.05)
    o, v, s, _ = oracle.replay_trace(tr)
    inj = tr.meta["inject"]
    f = v["flags"]
    assert np.all(f[inj == 0] == 0)
    assert np.all(f[inj == 1] == F_HOST_UNADDRESSABLE)            # column overrun into padding
    assert np.all(f[inj == 2] & F_BAD_PITCH)                      # X+W > pitch
    assert np.all((f[inj == 3] == F_DST_TOO_SMALL) | (f[inj == 3] == F_SRC_TOO_SMALL))


# --------------------------------------------------------------------------
# R-10: no size cap -- INVALID_RANGE only on 64-bit overflow ("arithmetic
# overflow of start+len -> InvalidRange"); bytes outside the
# window are unaddressable (R-15), so check_addressable's "lowest
# offending byte offset" of a copy running past the window end is the
# offset of the window end.  Every expected value below is derived by hand.
# --------------------------------------------------------------------------
def test_huge_copies_hand_derived():
    tr = tg.huge_copies()
    o, v, s, leaks = oracle.replay_trace(tr)
    H0, S = tr.host_base, tr.host_size                  # 1 MiB, 4 MiB
    start = tr.meta["start"]                            # H0 + 4096
    to_end = H0 + S - start                             # 4 MiB - 4096 = 4190208 bytes left in the window
    assert to_end == 4190208
    # the five undefined bytes sit at start + d, d in HUGE_D (all < to_end)
    assert all(d < to_end for d in tg.HUGE_D)
    names = list(tr.meta["copies"])
    V = {k: v[i] for i, k in enumerate(names)}
    for k in names:                                     # no copy is an INVALID_RANGE except the overflow one
        assert bool(V[k]["flags"] & F_INVALID_RANGE) == (k == "overflow"), k
    # 1D, W*H = 2^38+1 and 2^40: every byte from start to the window end is
    # addressable, the first one past it is not -> first_unaddr = to_end;
    # the 5 undefined bytes are all before it (R-4: raw count reported, but
    # HOST_UNDEFINED only when first_unaddr is NONE)
    for k in ("1d_2^38+1", "1d_2^40"):
        assert V[k]["first_unaddr"] == 4190208
        assert (V[k]["first_undef"], V[k]["undef_count"]) == (100, 5)
        assert V[k]["flags"] == F_HOST_UNADDRESSABLE and V[k]["status"] == 1
    # 2D, W = 525313, H = 523265 (W*H = 2^38+1), pitch 528384: row r covers
    # start + [528384 r, 528384 r + 525313).  Row 7 starts at 3698688 < 4190208
    # and ends at 4224001 > 4190208, rows 0..6 end before the window end; so the
    # first unaddressable logical offset is 7*525313 + (4190208 - 3698688) =
    # 3677191 + 491520 = 4168711.  Undefined bytes: d=100 (row 0, o=100),
    # d=525318 (between rows 0 and 1: pitch padding, not a logical byte),
    # d=1056778 (row 2 col 10, o=1050636), d=2000000 (row 3 col 414848,
    # o=1990787), d=3698788 (row 7 col 100, o=3677291) -> 4 bytes, first 100.
    assert V["2d_2^38+1"]["first_unaddr"] == 7 * 525313 + (4190208 - 7 * 528384) == 4168711
    assert (V["2d_2^38+1"]["first_undef"], V["2d_2^38+1"]["undef_count"]) == (100, 4)
    # 2D, W = H = 2^20, pitch 2^20 + 2^16 = 1114112: row 3 starts at 3342336
    # and ends at 4390912 > 4190208 (row 2 ends at 3276800), so first_unaddr =
    # 3*2^20 + (4190208 - 3342336) = 3145728 + 847872 = 3993600.  Undefined:
    # d=100 (row 0), d=525318 (row 0), d=1056778 (padding [1048576, 1114112)),
    # d=2000000 (row 1), d=3698788 (row 3 col 356452, before the window end).
    assert V["2d_2^40"]["first_unaddr"] == 3 * (1 << 20) + (4190208 - 3 * 1114112) == 3993600
    assert (V["2d_2^40"]["first_undef"], V["2d_2^40"]["undef_count"]) == (100, 4)
    # host start 4 KiB before the window: offset 0 is unaddressable; the raw
    # undefined count covers the whole window: offsets shift by 8192
    assert V["1d_before"]["first_unaddr"] == 0
    assert (V["1d_before"]["first_undef"], V["1d_before"]["undef_count"]) == (100 + 8192, 5)
    # DtoH: A-bits only (R-6); the error means no apply (R-7): V keeps the 5 undefined bytes
    assert V["dtoh_1d_2^40"]["first_unaddr"] == 4190208 and V["dtoh_2d_2^40"]["first_unaddr"] == 3993600
    for k in ("dtoh_1d_2^40", "dtoh_2d_2^40"):
        assert V[k]["first_undef"] == NONE and V[k]["undef_count"] == 0 and V[k]["status"] == 1
    assert int(np.count_nonzero(o.V)) == 5
    # W*H = 2^65 does not fit 64 bits (the spans do: pitch 0) -> INVALID_RANGE,
    # BAD_PITCH (0 < W); the host side is not scanned
    assert V["overflow"]["flags"] == F_INVALID_RANGE | F_BAD_PITCH
    assert V["overflow"]["first_unaddr"] == NONE and V["overflow"]["undef_count"] == 0


@pytest.mark.parametrize("seed", range(4))
def test_overlapping_rows_multiplicity(seed):
    """BAD_PITCH rows that overlap (pitch < W, R-12): the oracle loops over the
    W*H logical bytes row by row.  An independent derivation over PHYSICAL
    bytes u = x - start: u lies in rows r_lo(u)..r_hi(u), r_lo = 0 if u < W
    else (u - W) // pitch + 1, r_hi = min(H - 1, u // pitch); its first logical
    offset is u + r_lo (W - pitch), which grows with u, so first_unaddr /
    first_undef are those of the first bad physical byte and undef_count is
    the sum of the row counts of the undefined physical bytes.  pitch 0: every
    row is the same W bytes -> count = H * (undefined bytes of the row)."""
    W, pitch, H = [(4096, 64, 20000), (1000, 999, 3000), (64, 1, 50000), (4096, 0, 5000)][seed]
    tr = tg.overlap_rows(seed, W=W, pitch=pitch, H=H)
    o, v, s, _ = oracle.replay_trace(tr)
    start, h0 = tr.meta["start"], tr.host_base
    span = (H - 1) * pitch + W
    A = np.unpackbits(o.A, bitorder="little").astype(bool)
    ok = A[start - h0:start - h0 + span]
    und = ok & (o.V[start - h0:start - h0 + span] != 0)
    u = np.arange(span, dtype=np.int64)
    if pitch:
        r_lo = np.where(u < W, 0, (u - W) // pitch + 1)
        r_hi = np.minimum(H - 1, u // pitch)
    else:
        r_lo, r_hi = np.zeros(span, np.int64), np.full(span, H - 1)
    first_o = u + r_lo * (W - pitch)
    assert np.all(np.diff(first_o) > 0)
    exp_cnt = int(np.sum((r_hi - r_lo + 1)[und]))
    exp_fd = int(first_o[und][0]) if und.any() else NONE
    exp_fu = int(first_o[~ok][0]) if (~ok).any() else NONE
    assert (v[0]["first_unaddr"], v[0]["first_undef"], v[0]["undef_count"]) == (exp_fu, exp_fd, exp_cnt)
    assert v[0]["flags"] & F_BAD_PITCH and v[0]["status"] == 1
    # pitch 0: H copies of row 0 = the first W physical bytes
    row = ok[:W] & (o.V[start - h0:start - h0 + W] != 0)
    assert v[1]["undef_count"] == H * int(np.count_nonzero(row))
