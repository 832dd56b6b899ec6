"""C-ABI checks that need no GPU: the library loads, exports every symbol
include/cg.h declares, the ctypes/numpy layouts match the header, and the
host-side epoch planner (cg_plan_batches) cuts exactly at DtoH->HtoD hazards."""
import ctypes
import os
import re

import numpy as np
import pytest

import tracegen as tg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cg.h")


@pytest.fixture(scope="module")
def cg():
    from paper_1310_0901_b200 import build
    build.build()
    import paper_1310_0901_b200 as m
    return m


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cg_[a-z_0-9]+)\s*\(", src)))


def test_every_declared_symbol_is_exported(cg):
    names = declared_functions()
    assert len(names) >= 17
    lib = ctypes.CDLL(cg.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(cg.EXPORTED)


def test_struct_sizes_match_header(cg):
    assert ctypes.sizeof(cg.cg_config) == 112
    assert cg.DESC_DTYPE.itemsize == 96 and cg.VERDICT_DTYPE.itemsize == 64
    # the header states the same sizes in its comments
    src = open(HEADER).read()
    assert "96 bytes" in src and "64 bytes" in src and "24 bytes" in src


def test_workspace_size_validation(cg):
    c = cg.cg_config(host_base=1 << 20, host_size=1 << 20, max_descs=1000, max_allocs=100)
    assert cg.cg_workspace_size(ctypes.byref(c)) > 0
    bad = cg.cg_config(host_base=(1 << 20) + 1, host_size=1 << 20, max_descs=1000, max_allocs=100)
    assert cg.cg_workspace_size(ctypes.byref(bad)) == 0
    bad = cg.cg_config(host_base=1 << 20, host_size=1 << 20, shard_base=1 << 21, shard_size=4096,
                       max_descs=1000, max_allocs=100)
    assert cg.cg_workspace_size(ctypes.byref(bad)) == 0


READS_HOST, WRITES_HOST = (1, 4), (2, 5)   # HtoD / HtoA read the host, DtoH / AtoH write it


def _hazard_free(descs, a, b):
    """brute force: no host read in [a,b) overlaps the host bytes of an earlier host write in [a,b)"""
    def host(d):
        if d["kind"] not in (1, 2, 4, 5) or d["width"] == 0 or d["height"] == 0:
            return None
        p = "src" if d["kind"] in READS_HOST else "dst"
        s = int(d[p]) + int(d[p + "_y"]) * int(d[p + "_pitch"]) + int(d[p + "_x"])
        e = s + (int(d["height"]) - 1) * int(d[p + "_pitch"]) + int(d["width"])
        return None if e > (1 << 64) - 1 else (s, e)
    seen = []
    for i in range(a, b):
        r = host(descs[i])
        if r is None:
            continue
        if descs[i]["kind"] in WRITES_HOST:
            seen.append(r)
        elif any(r[0] < e and s < r[1] for s, e in seen):
            return False
    return True


@pytest.mark.parametrize("arrays", [False, True])
@pytest.mark.parametrize("seed", range(30))
def test_plan_batches_cuts_only_at_hazards(cg, seed, arrays):
    from paper_1310_0901_b200.replay import events_to_descs
    tr = tg.random_tiny(seed, arrays=arrays)
    ev = tr.events[tr.events["op"] == tg.OP_COPY]
    descs = events_to_descs(ev)
    cuts = [0] + [int(c) for c in cg.plan_batches(descs)]
    assert cuts[-1] == len(descs)
    for a, b in zip(cuts[:-1], cuts[1:]):
        assert b > a
        assert _hazard_free(descs, a, b)           # every batch is hazard-free
        if b < len(descs):                          # and each cut is necessary (greedy)
            assert not _hazard_free(descs, a, b + 1)


def test_plan_batches_toy(cg):
    """Appendix A.1: the toy trace's copies form the epochs {C1-C4}, {C5-C7}, {C8-C10}."""
    from paper_1310_0901_b200.replay import events_to_descs
    tr = tg.toy()
    descs = events_to_descs(tr.events[tr.events["op"] == tg.OP_COPY])
    assert [int(c) for c in cg.plan_batches(descs)] == [4, 7, 10]


def test_plan_batches_c2_single_epoch(cg):
    from paper_1310_0901_b200.replay import events_to_descs
    tr = tg.c2_small(n_copies=20000, n_allocs=2000)
    descs = events_to_descs(tr.events[tr.events["op"] == tg.OP_COPY])
    assert [int(c) for c in cg.plan_batches(descs)] == [len(descs)]


def _disjoint_brute(descs):
    def host(d):
        if d["kind"] not in (1, 2, 4, 5) or d["width"] == 0 or d["height"] == 0:
            return None
        p = "src" if d["kind"] in READS_HOST else "dst"
        s = int(d[p]) + int(d[p + "_y"]) * int(d[p + "_pitch"]) + int(d[p + "_x"])
        e = s + (int(d["height"]) - 1) * int(d[p + "_pitch"]) + int(d["width"])
        return None if e > (1 << 64) - 1 else (s, e, int(d["kind"]) in READS_HOST)
    r = [h for h in map(host, descs) if h]
    for a in r:
        for b in r:
            if a[2] and not b[2] and a[0] < b[1] and b[0] < a[1]:
                return False
    return True


@pytest.mark.parametrize("arrays", [False, True])
@pytest.mark.parametrize("seed", range(40))
def test_batch_disjoint_matches_brute_force(cg, seed, arrays):
    from paper_1310_0901_b200.replay import events_to_descs
    tr = tg.random_tiny(seed, arrays=arrays)
    descs = events_to_descs(tr.events[tr.events["op"] == tg.OP_COPY])
    rng = np.random.default_rng(seed)
    for _ in range(10):
        a = int(rng.integers(0, len(descs)))
        b = int(rng.integers(a, len(descs) + 1))
        assert cg.batch_disjoint(descs[a:b]) == _disjoint_brute(descs[a:b])


def test_batch_disjoint_configs(cg):
    from paper_1310_0901_b200.replay import events_to_descs
    for tr in (tg.c2_small(n_copies=20000, n_allocs=2000), tg.c4_pitched(n_copies=2000, n_bufs=2, rows=64)):
        assert cg.batch_disjoint(events_to_descs(tr.events[tr.events["op"] == tg.OP_COPY]))


def test_listing5_text_from_verdict(cg):
    """NEXT-4: the TooSmall verdict of the paper's worked example renders the
    first two lines of Listing 5 byte for byte (tests/golden)."""
    lines = [l for l in open(os.path.join(ROOT, "tests", "golden", "listing5.txt")) if not l.startswith("#")]
    v = np.zeros(1, cg.VERDICT_DTYPE)[0]
    v["first_unaddr"] = v["first_undef"] = cg.CG_NONE
    v["src_expected"], v["src_found"], v["flags"], v["status"] = 8000000, 4000000, cg.CG_F_SRC_TOO_SMALL, 1
    assert cg.format_verdict(v, cg.CG_DTOH) == "".join(lines)
    assert cg.format_verdict(np.zeros(1, cg.VERDICT_DTYPE)[0], cg.CG_HTOD) == ""
    rec = np.zeros(1, cg.ALLOC_RECORD_DTYPE)[0]
    rec["size"] = 4096
    assert cg.format_leak(rec) == "Warning: Device memory leak of 4096 bytes.\n"


def test_format_is_injective_on_fuzzed_verdicts(cg):
    """formatting is injective over (flags, expected, found, offsets)."""
    rng = np.random.default_rng(0)
    seen = {}
    for _ in range(3000):
        v = np.zeros(1, cg.VERDICT_DTYPE)[0]
        v["flags"] = int(rng.integers(1, 1 << 9))
        for f in ("first_unaddr", "first_undef", "undef_count", "dst_expected", "dst_found", "src_expected", "src_found"):
            v[f] = int(rng.integers(0, 1 << 40))
        k = int(rng.integers(1, 4))
        key = cg.format_verdict(v, k)
        rel = tuple(int(v[f]) for f in v.dtype.names if f != "status") + (k,)
        # only fields a set flag reports are part of the identity
        fl = int(v["flags"])
        ident = (k, fl,
                 int(v["dst_expected"]) if fl & 2 else None, int(v["dst_found"]) if fl & 2 else None,
                 int(v["src_expected"]) if fl & 8 else None, int(v["src_found"]) if fl & 8 else None,
                 int(v["first_unaddr"]) if fl & 16 else None,
                 (int(v["undef_count"]), int(v["first_undef"])) if fl & 32 else None)
        if key in seen:
            assert seen[key] == ident
        seen[key] = ident


def _sets(d):
    """(space, lo, hi) reads and writes of one descriptor for propagation"""
    def rng(p):
        if d["width"] == 0 or d["height"] == 0:
            return None
        s = int(d[p]) + int(d[p + "_y"]) * int(d[p + "_pitch"]) + int(d[p + "_x"])
        e = s + (int(d["height"]) - 1) * int(d[p + "_pitch"]) + int(d["width"])
        return None if e > (1 << 64) - 1 else (s, e)
    def arr(p):   # an array side (R-29): bytes [offset, offset + W*H) of that array's own space (R-30)
        if d["width"] == 0 or d["height"] == 0:
            return None
        s = int(d[p + "_x"])
        e = s + int(d["width"]) * int(d["height"])
        return None if e > (1 << 64) - 1 else (s, e)
    k = int(d["kind"])
    if k not in (1, 2, 3, 4, 5):
        return [], []
    r = rng("src") if k != 5 else arr("src")
    w = rng("dst") if k != 4 else arr("dst")
    rs = ("a", int(d["src"])) if k == 5 else "h" if k in READS_HOST else "d"
    ws = ("a", int(d["dst"])) if k == 4 else "h" if k in WRITES_HOST else "d"
    return ([(rs,) + r] if r else []), ([(ws,) + w] if w else [])


def _prop_ok(descs, a, b):
    R, W = [], []
    for i in range(a, b):
        r, w = _sets(descs[i])
        for x in r:
            if any(x[0] == y[0] and x[1] < y[2] and y[1] < x[2] for y in W):
                return False
        for x in w:
            if any(x[0] == y[0] and x[1] < y[2] and y[1] < x[2] for y in R + W):
                return False
        R += r
        W += w
    return True


@pytest.mark.parametrize("arrays", [False, True])
@pytest.mark.parametrize("seed", range(30))
def test_plan_batches_propagate(cg, seed, arrays):
    from paper_1310_0901_b200.replay import events_to_descs
    tr = tg.random_tiny(seed + 20000, arrays=arrays)
    descs = events_to_descs(tr.events[tr.events["op"] == tg.OP_COPY])
    cuts = [0] + [int(c) for c in cg.plan_batches(descs, propagate=True)]
    assert cuts[-1] == len(descs)
    for a, b in zip(cuts[:-1], cuts[1:]):
        assert _prop_ok(descs, a, b)
        if b < len(descs):
            assert not _prop_ok(descs, a, b + 1)


def test_array_bytes_matches_oracle(cg):
    """NEXT-3: cg_array_bytes against the oracle's or_array_bytes
    over random descriptors, including zero extents, bad formats / channel
    counts and products that overflow 64 bits."""
    import oracle
    rng = np.random.default_rng(3)
    o = oracle.Oracle(1 << 20, 1 << 12)
    for _ in range(5000):
        big = rng.random() < 0.1
        w, h, d = (int(rng.integers(0, 1 << 40 if big else 300)) for _ in range(3))
        f, c = int(rng.integers(0, 10)), int(rng.integers(0, 6))
        assert cg.cg_array_bytes(w, h, d, f, c) == o.array_bytes(w, h, d, f, c), (w, h, d, f, c)
    assert cg.cg_array_bytes(64, 8, 0, 3, 2) == 1024


def test_array_format_text(cg):
    """NEXT-4 wording for array transfers: the noun and direction change, the Listing-5 shape stays."""
    v = np.zeros(1, cg.VERDICT_DTYPE)[0]
    v["first_unaddr"] = v["first_undef"] = cg.CG_NONE
    v["dst_expected"], v["dst_found"], v["flags"], v["status"] = 100, 24, cg.CG_F_DST_TOO_SMALL, 1
    assert cg.format_verdict(v, cg.CG_HTOA) == ("Error: Allocated device array too small for host->array copy.\n"
                                                "Expected 100 allocated bytes but only found 24.\n")
    v["flags"] = cg.CG_F_SRC_NOT_ALLOCATED
    assert cg.format_verdict(v, cg.CG_ATOH) == "Error: Source device array of array->host copy is not allocated.\n"


def test_error_summary_line(cg):
    """1 error, 0 suppressions -> "ERROR SUMMARY: 1 errors, 0 warnings (0 suppressed)" """
    assert cg.format_summary(1, 0, 0) == "ERROR SUMMARY: 1 errors, 0 warnings (0 suppressed)\n"
    assert cg.format_summary(12, 345, 6) == "ERROR SUMMARY: 12 errors, 345 warnings (6 suppressed)\n"


def test_replay_unknown_op_is_an_invalid_call():
    """an event with an unknown op is an invalid call (status 1) in the oracle;
    the GPU replays must agree without a GPU call (checked on the host path)"""
    import oracle
    tr = tg.random_tiny(5)
    ev = tr.events.copy()
    ev[3]["op"] = 42
    o = oracle.Oracle(tr.host_base, tr.host_size)
    _, st = o.replay(ev, tr.blob)
    assert st[3] == 1


def test_header_is_plain_c(tmp_path):
    """include/cg.h is a C header: a C11 translation unit that includes it and
    takes the address of every declared function compiles with gcc"""
    import subprocess
    names = declared_functions()
    src = tmp_path / "use.c"
    src.write_text('#include "cg.h"\n#include <stddef.h>\ntypedef void (*fn)(void);\nfn table[] = {\n' +
                   ",\n".join(f"  (fn)&{n}" for n in names) + "\n};\nint main(void) { return table[0] == NULL; }\n")
    r = subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", "-pedantic", "-fsyntax-only",
                        "-I", os.path.join(ROOT, "include"), str(src)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.parametrize("arrays", [False, True])
@pytest.mark.parametrize("seed", range(30))
def test_plan_waves_brute_force(cg, seed, arrays):
    """cg_plan_waves: level(i) = 1 + the highest level of an earlier copy whose
    V-bit reads / writes conflict with copy i's (RAW, WAR, WAW), 0 if none --
    recomputed here by brute force over all earlier pairs"""
    from paper_1310_0901_b200.replay import events_to_descs
    tr = tg.random_tiny(seed + 50000, arrays=arrays)
    descs = events_to_descs(tr.events[tr.events["op"] == tg.OP_COPY])
    lev, nl = cg.plan_waves(descs)
    sets = [_sets(d) for d in descs]

    def ov(x, y):
        return x[0] == y[0] and x[1] < y[2] and y[1] < x[2]
    want = []
    for i, (ri, wi) in enumerate(sets):
        lv = 0
        for j in range(i):
            rj, wj = sets[j]
            if any(ov(a, b) for a in ri for b in wj) or any(ov(a, b) for a in wi for b in rj + wj):
                lv = max(lv, want[j] + 1)
        want.append(lv)
    assert list(lev) == want
    assert nl == (max(want) + 1 if want else 0)


@pytest.mark.parametrize("seed", range(20))
def test_plan_apply_after(cg, seed):
    """cg_plan_apply_after marks exactly the DtoH / AtoH descriptors whose host
    bounding range overlaps the host range of some HtoD / HtoA of the batch"""
    tr = tg.random_tiny(seed + 21000, arrays=seed % 2 == 0)
    descs = np.ascontiguousarray(tg.events_to_descs(tr.events[tr.events["op"] == tg.OP_COPY]))
    descs["reserved"] = np.where(np.arange(len(descs)) % 3 == 0, cg.CG_APPLY_AFTER, 0)   # stale bits get cleared

    def hrange(d, p):
        if d["width"] == 0 or d["height"] == 0:
            return None
        s = int(d[p]) + int(d[p + "_y"]) * int(d[p + "_pitch"]) + int(d[p + "_x"])
        e = s + (int(d["height"]) - 1) * int(d[p + "_pitch"]) + int(d["width"])
        return None if e > (1 << 64) - 1 else (s, e)
    reads = [hrange(d, "src") for d in descs if int(d["kind"]) in (1, 4)]
    reads = [r for r in reads if r]
    expect = []
    for d in descs:
        w = hrange(d, "dst") if int(d["kind"]) in (2, 5) else None
        expect.append(bool(w) and any(a < w[1] and w[0] < b for a, b in reads))
    k = cg.plan_apply_after(descs)
    got = (descs["reserved"] & cg.CG_APPLY_AFTER) != 0
    assert list(got) == expect and k == sum(expect)


@pytest.mark.parametrize("seed", range(20))
def test_plan_batches_fused(cg, seed):
    """cg_plan_batches_fused: inside every batch, an HtoD whose host range
    overlaps an earlier DtoH of the batch carries CG_CHECK_AFTER, a DtoH
    overlapping an earlier CG_CHECK_AFTER HtoD carries CG_APPLY_LAST, no HtoD
    overlaps an earlier CG_APPLY_LAST DtoH of its batch, CG_APPLY_AFTER is
    cg_plan_apply_after of the batch on the other DtoH copies, and every cut is
    forced (an HtoD reading a CG_APPLY_LAST range, or a late HtoD > 1 MiB)"""
    if seed % 4 == 3:
        tr = tg.pingpong_trace(seed)
    else:
        tr = tg.random_tiny(seed + 22000) if seed % 2 else tg.random_medium(seed, n_copies=80)
    descs = np.ascontiguousarray(tg.events_to_descs(tr.events[tr.events["op"] == tg.OP_COPY]))
    cuts = [0] + [int(c) for c in cg.plan_batches_fused(descs)]
    assert cuts[-1] == len(descs)

    def hrange(d):
        k = int(d["kind"])
        if k not in (1, 2, 4, 5) or d["width"] == 0 or d["height"] == 0:
            return None
        p = "src" if k in (1, 4) else "dst"
        s = int(d[p]) + int(d[p + "_y"]) * int(d[p + "_pitch"]) + int(d[p + "_x"])
        e = s + (int(d["height"]) - 1) * int(d[p + "_pitch"]) + int(d["width"])
        return None if e > (1 << 64) - 1 else (s, e)

    def hits(r, rs):
        return any(x < r[1] and r[0] < y for x, y in rs)
    prev = None   # (writes, last) of the batch before
    for a, b in zip(cuts[:-1], cuts[1:]):
        if prev is not None:   # the cut is forced by descriptor a
            r = hrange(descs[a])
            assert r is not None and int(descs[a]["kind"]) in (1, 4)
            assert hits(r, prev[1]) or (hits(r, prev[0]) and r[1] - r[0] > (1 << 20))
        writes, late, last = [], [], []
        for d in descs[a:b]:
            r = hrange(d)
            k = int(d["kind"])
            if r is None:
                assert not d["reserved"] & (cg.CG_CHECK_AFTER | cg.CG_APPLY_LAST)
                continue
            if k in (1, 4):
                assert not hits(r, last)
                dep = hits(r, writes)
                assert bool(d["reserved"] & cg.CG_CHECK_AFTER) == dep
                assert not d["reserved"] & cg.CG_APPLY_LAST
                if dep:
                    late.append(r)
            else:
                is_last = hits(r, late)
                assert bool(d["reserved"] & cg.CG_APPLY_LAST) == is_last
                assert not d["reserved"] & cg.CG_CHECK_AFTER
                if is_last:
                    last.append(r)
                    assert not d["reserved"] & cg.CG_APPLY_AFTER
                writes.append(r)
        prev = (writes, last)
        part = np.ascontiguousarray(descs[a:b]).copy()
        part["reserved"] &= ~np.uint32(cg.CG_APPLY_AFTER)
        cg.plan_apply_after(part)
        expect = np.where(descs["reserved"][a:b] & cg.CG_APPLY_LAST, 0, part["reserved"] & cg.CG_APPLY_AFTER)
        assert np.array_equal(expect, descs["reserved"][a:b] & cg.CG_APPLY_AFTER)
