"""NEXT-3 pins (Fig. 2 caption P:88 "list of linear memory or
device arrays")."""
import numpy as np
import pytest

import oracle
import tracegen as tg
from flatmodel import FlatModel
from oracle import Oracle


def test_array_descriptor_bytes():
    o = Oracle(0x10000, 4096)
    assert o.array_bytes(1024, 0, 0, 6, 1) == 2048            # f16, 1D
    assert o.array_bytes(1024, 0, 0, 7, 1) == 4096            # width 1024, f32, 1 channel -> 4096
    assert o.array_bytes(16, 8, 2, 1, 4) == 16 * 8 * 2 * 2 * 4
    assert o.array_bytes(0, 1, 1, 0, 1) == 0                  # zero extent
    assert o.array_bytes(4, 1, 1, 0, 3) == 0                  # channels in {1,2,4}
    assert o.array_bytes(4, 1, 1, 8, 1) == 0                  # unknown format


def test_spec_array_transfer_examples():
    H = 0x10000
    o = Oracle(H, 1 << 16)
    o.mark(H, 8192, tg.DEFINED)
    assert o.register_array(7, 4096, 1) == 0
    e = np.zeros(1, tg.EVENT_DTYPE)[0]
    e["op"], e["kind"], e["seq"], e["width"], e["height"] = tg.OP_COPY, tg.HTOA, 2, 4096, 1
    e["dst"], e["dst_x"], e["src"], e["src_pitch"] = 7, 0, H, 4096
    v = o.check_copy(e)
    assert v["flags"] == 0                                    # total 4096, offset 0, len 4096
    e["seq"], e["dst_x"], e["width"], e["src_pitch"] = 3, 4000, 200, 200
    v = o.check_copy(e)
    assert v["flags"] == oracle.F_DST_TOO_SMALL               # offset 4000, len 200
    assert (v["dst_expected"], v["dst_found"]) == (200, 96)
    assert o.register_array(7, 16, 4) == 1                    # DuplicateHandle
    assert o.free_array(8, 5) == 1                            # UnknownHandle
    assert o.free_array(7, 6) == 0
    e["seq"] = 7
    v = o.check_copy(e)
    assert v["flags"] == oracle.F_DST_NOT_ALLOCATED           # lookup after unregister -> absent


@pytest.mark.parametrize("seed", range(40))
def test_flat_model_equivalence_arrays(seed):
    tr = tg.random_tiny(seed + 30000, arrays=True)
    o, v, s, leaks = oracle.replay_trace(tr)
    fm = FlatModel(tr.host_base, tr.host_size)
    fv, fs = fm.replay(tr.events, tr.blob)
    assert list(s) == fs
    for i, (a, b) in enumerate(zip(v, fv)):
        assert {k: int(a[k]) for k in v.dtype.names} == b, i
    assert np.array_equal(o.V, fm.v)
    al = o.array_leaks()
    assert sorted(fm.arrays.items()) == [(int(x["base"]), int(x["size"])) for x in al]


def test_array_vbits_per_array_shadow_round_trip():
    """S:252 "array V-bits tracked in a per-array shadow" (R-30) with device
    V-bit tracking: a fresh array is undefined (as fresh device memory,
    S:326); an error-free HtoA copies host V-bits into the array, AtoH copies
    them back (the chained-copy acceptance of S:547 through an array); an
    erroring copy moves nothing."""
    H = 0x100000
    o = Oracle(H, 1 << 16, track_device=True)
    rng = np.random.default_rng(5)
    pat = rng.integers(0, 256, 1024, dtype=np.uint8)
    o.mark(H, 1 << 16, tg.DEFINED)
    assert o.set_vbits(H, pat.tobytes()) == 0
    assert o.register_array(9, 4096, 1) == 0
    assert np.all(o.array_vbits(9, 0, 4096) == 0xFF)          # fresh = undefined

    def copy(kind, seq, width, host, off):
        e = np.zeros(1, tg.EVENT_DTYPE)[0]
        e["op"], e["kind"], e["seq"], e["width"], e["height"] = tg.OP_COPY, kind, seq, width, 1
        if kind == tg.HTOA:
            e["dst"], e["dst_x"], e["src"], e["src_pitch"] = 9, off, host, width
        else:
            e["src"], e["src_x"], e["dst"], e["dst_pitch"] = 9, off, host, width
        return o.check_copy(e)

    v = copy(tg.HTOA, 2, 1024, H, 100)
    assert v["flags"] == oracle.F_HOST_UNDEFINED and v["status"] == 0   # a Warning: the copy happens
    assert np.array_equal(o.array_vbits(9, 100, 1024), pat)
    assert np.all(o.array_vbits(9, 0, 100) == 0xFF)
    v = copy(tg.ATOH, 3, 1024, H + 8192, 100)                  # array -> another host buffer
    assert v["flags"] == 0
    assert np.array_equal(o.V[8192:8192 + 1024], pat)          # the pattern survives H -> A -> H
    v = copy(tg.ATOH, 4, 512, H + 16384, 3500)                 # from never-written array bytes
    assert v["flags"] == 0 and np.all(o.V[16384:16384 + 512] == 0xFF)
    v = copy(tg.ATOH, 5, 512, H + 20000, 3800)                 # offset 3800 + 512 > 4096: TooSmall, nothing moves
    assert v["flags"] == oracle.F_SRC_TOO_SMALL and np.all(o.V[20000:20512] == 0)


@pytest.mark.parametrize("seed", range(30))
def test_flat_model_equivalence_arrays_tracking(seed):
    tr = tg.random_tiny(seed + 31000, arrays=True)
    o, v, s, leaks = oracle.replay_trace(tr, track_device=True)
    fm = FlatModel(tr.host_base, tr.host_size, track=True)
    fv, fs = fm.replay(tr.events, tr.blob)
    assert list(s) == fs
    for i, (a, b) in enumerate(zip(v, fv)):
        assert {k: int(a[k]) for k in v.dtype.names} == b, i
    assert np.array_equal(o.V, fm.v)
    for h, av in fm.av.items():
        assert np.array_equal(o.array_vbits(h, 0, len(av)), av), h
