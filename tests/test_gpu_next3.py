"""NEXT-3 on the GPU: device arrays (HtoA / AtoH transfers, register / free
array, array leak report) bit-exact against the oracle on the same seeded
traces -- in the fused, unfused and device-V-bit-tracking replays."""
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


def run(cg, tr, mode):
    track = mode == "track"
    o, ov, os_, oleaks = oracle.replay_trace(tr, track_device=track)
    ev = tr.events
    regs = ev[ev["op"] == tg.OP_REG]
    kw = {}
    if track:
        rega = ev[ev["op"] == tg.OP_REGA]
        arr = sum(o.array_bytes(int(e["width"]), int(e["height"]), int(e["dst_x"]), int(e["dst_y"]),
                                int(e["dst_pitch"])) + 16 for e in rega)
        kw["dev_vsize"] = int(sum(int(x) + 256 for x in regs["width"])) + arr + (1 << 20)
    chk = cg.Checker(tr.host_base, tr.host_size, max_descs=max(tr.n_copies, 64),
                     max_allocs=max(len(ev), 64), **kw)
    gv, gs = cg.replay_events(chk, ev, tr.blob, fuse=(mode == "fused"))
    for f in ov.dtype.names:
        bad = np.flatnonzero(gv[f] != ov[f])
        assert len(bad) == 0, (mode, f, bad[:5], gv[f][bad[:5]], ov[f][bad[:5]])
    bad = np.flatnonzero(gs != os_)
    assert len(bad) == 0, (mode, bad[:5], ev["op"][bad[:5]], gs[bad[:5]], os_[bad[:5]])
    gl = chk.leak_report()
    assert np.array_equal(gl["base"], oleaks["base"]) and np.array_equal(gl["size"], oleaks["size"])
    ga, oa = chk.array_report(), o.array_leaks()
    assert np.array_equal(ga["base"], oa["base"]) and np.array_equal(ga["size"], oa["size"])
    assert np.array_equal(ga["alloc_seq"], oa["seq"])
    A, V = chk.shadow()
    assert np.array_equal(A, o.A) and np.array_equal(V, o.V)
    if track:   # R-30 / S:252: every live array's own V-bits
        for a in oa:
            h, n = int(a["base"]), int(a["size"])
            assert np.array_equal(chk.array_vbits(h, 0, n), o.array_vbits(h, 0, n)), h
    chk.close()
    return gv


@pytest.mark.parametrize("mode", ["fused", "unfused", "track"])
@pytest.mark.parametrize("seed", range(40))
def test_random_tiny_arrays(cg, seed, mode):
    tr = tg.random_tiny(seed + 30000, arrays=True)
    ops = tr.events["op"]
    assert (ops == tg.OP_REGA).any()
    run(cg, tr, mode)


def _one_array_trace():
    H0 = 1 << 20
    tb = tg.TraceBuilder("arr", H0, 1 << 16)
    tb.mark(H0, 4096, tg.DEFINED)
    tb.mark(H0 + 4096, 4096, tg.UNDEFINED)
    h = 0xA000
    tb.register_array(h, 64, 8, 0, 3, 2)       # 64*8 * 1 B * 2 ch = 1024 B
    tb.copy_htoa(h, 0, H0, 1024)               # OK
    tb.copy_htoa(h, 1000, H0, 100)             # TooSmall: expected 100, found 24
    tb.copy_htoa(h, 5000, H0, 10)              # TooSmall: found 0 (offset past the end)
    tb.copy_atoh(H0 + 4096, h, 0, 512)         # OK: host becomes defined
    tb.copy_htoa(h + 1, 0, H0, 8)              # NotAllocated (unknown handle)
    tb.copy_htoa(h, 0, H0 + 4000, 200)         # host: 96 defined + 104 now-defined -> OK
    tb.copy_htoa(h, 0, H0 + 8192 - 16, 32)     # host partly unaddressable
    tb.free_array(h)
    tb.copy_atoh(H0, h, 0, 8)                  # NotAllocated (freed)
    tb.register_array(h, 16, 0, 0, 7, 4)       # handle reuse: 16 * 4 B * 4 ch = 256 B
    tb.copy_atoh(H0, h, 0, 256)                # OK against the new lifetime
    tb.copy_atoh(H0, h, 0, 257)                # TooSmall
    return tb.build()


@pytest.mark.parametrize("mode", ["fused", "unfused", "track"])
def test_array_edge_cases(cg, mode):
    tr = _one_array_trace()
    gv = run(cg, tr, mode)
    F = cg
    expect = [0, F.CG_F_DST_TOO_SMALL, F.CG_F_DST_TOO_SMALL, 0, F.CG_F_DST_NOT_ALLOCATED, 0,
              F.CG_F_HOST_UNADDRESSABLE, F.CG_F_SRC_NOT_ALLOCATED, 0, F.CG_F_SRC_TOO_SMALL]
    assert [int(x) for x in gv["flags"]] == expect
    assert (int(gv[1]["dst_expected"]), int(gv[1]["dst_found"])) == (100, 24)
    assert (int(gv[2]["dst_expected"]), int(gv[2]["dst_found"])) == (10, 0)


def test_array_registry_errors(cg):
    chk = cg.Checker(1 << 20, 1 << 16, max_descs=64, max_allocs=4)
    assert chk.register_array(7, 0, 1, 1, 0, 1, 1) == cg.CG_ERR_INVALID_VALUE     # zero extent
    assert chk.register_array(7, 4, 1, 1, 9, 1, 2) == cg.CG_ERR_INVALID_VALUE     # unknown format
    assert chk.register_array(7, 4, 1, 1, 0, 3, 3) == cg.CG_ERR_INVALID_VALUE     # 3 channels
    assert chk.register_array(7, 4, 1, 1, 0, 1, 3) == cg.CG_OK
    assert chk.register_array(7, 4, 1, 1, 0, 1, 4) == cg.CG_ERR_INVALID_VALUE     # DuplicateHandle
    assert chk.register_array(8, 4, 1, 1, 0, 1, 3) == cg.CG_ERR_INVALID_VALUE     # seq not increasing
    assert chk.free_array(9, 5) == cg.CG_ERR_INVALID_VALUE                        # UnknownHandle
    assert chk.free_array(7, 5) == cg.CG_OK
    assert chk.free_array(7, 6) == cg.CG_ERR_INVALID_VALUE                        # double free
    for k in range(3):
        assert chk.register_array(100 + k, 1, 1, 1, 0, 1, 10 + k) == cg.CG_OK
    assert chk.register_array(200, 1, 1, 1, 0, 1, 20) == cg.CG_ERR_OUT_OF_MEMORY  # 4 entries incl. tombstone
    assert cg.cg_registry_compact(chk.ctx, 6) == cg.CG_OK
    assert chk.register_array(200, 1, 1, 1, 0, 1, 21) == cg.CG_OK
    rep = chk.array_report()
    assert [int(x) for x in rep["base"]] == [100, 101, 102, 200]
    chk.close()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("seed", range(6))
def test_random_tiny_arrays_sharded(cg, world, seed):
    """array transfers through host-range shards (their host side is sharded
    like HtoD / DtoH; the array side is looked up by the owner shard only)"""
    from test_gpu_sharded import run_sharded
    run_sharded(cg, tg.random_tiny(seed + 31000, arrays=True), world, fuse=bool(seed % 2))
