"""R-10 on the GPU: copies of any size (INVALID_RANGE only on 64-bit overflow,
S:49) and BAD_PITCH rows that overlap (R-12).  The kernels clip every host
side to the shard analytically (bytes outside the window are unaddressable,
R-15) and send overlapping rows -- and, in the sparse map, sides longer than
2^36 bytes -- to the deferred pass.  Every case is bit-exact against the CPU
oracle (verdicts, statuses, leaks, final host shadow), in every shadow format,
fused and unfused, sharded; the cases the oracle cannot finish (2^40 logical
bytes on overlapping rows) against closed forms."""
import numpy as np
import pytest

import oracle
import tracegen as tg
from test_gpu_parity import run_parity
from test_gpu_sharded import run_sharded

pytestmark = pytest.mark.gpu
FORMATS = {"bytes": {}, "2bit": dict(shadow_format=1), "sparse": dict(shadow_format=2, sparse_capacity=8 << 20)}


@pytest.fixture(scope="module")
def cg():
    import torch
    assert torch.cuda.is_available()
    from paper_1310_0901_b200 import build
    build.build()
    import paper_1310_0901_b200 as m
    return m


@pytest.mark.parametrize("fmt", list(FORMATS))
@pytest.mark.parametrize("fuse", [True, False])
def test_huge_copies(cg, fmt, fuse):
    v = run_parity(cg, tg.huge_copies(), fuse=fuse, **FORMATS[fmt])
    # the hand-derived values of tests/test_oracle_pins.py::test_huge_copies_hand_derived
    assert list(v["first_unaddr"][:5]) == [4190208, 4190208, 4168711, 3993600, 0]
    assert list(v["undef_count"][:5]) == [5, 5, 4, 4, 5]
    assert v[7]["flags"] == oracle.F_INVALID_RANGE | oracle.F_BAD_PITCH


@pytest.mark.parametrize("world", [2, 4])
def test_huge_copies_sharded(cg, world):
    run_sharded(cg, tg.huge_copies(), world, fuse=world == 2)


@pytest.mark.parametrize("fmt", list(FORMATS))
@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("dtoh", [False, True])
def test_overlapping_rows(cg, fmt, seed, dtoh):
    W, pitch, H = [(4096, 64, 20000), (1000, 999, 3000), (64, 1, 50000), (4096, 0, 5000)][seed]
    run_parity(cg, tg.overlap_rows(seed, W=W, pitch=pitch, H=H, dtoh=dtoh), fuse=bool(seed % 2), **FORMATS[fmt])


@pytest.mark.parametrize("world", [2, 4])
def test_overlapping_rows_sharded(cg, world):
    run_sharded(cg, tg.overlap_rows(7, W=8192, pitch=100, H=30000), world)


@pytest.mark.parametrize("fmt", list(FORMATS))
def test_overlapping_rows_2_40_closed_form(cg, fmt):
    """pitch 0, W = 4096, H = 2^28: 2^40 logical bytes on one physical row.
    Every row is the same 4096 bytes, so undef_count = H * (undefined bytes of
    the row), first_undef = the first undefined byte's column (row 0), and a
    row inside the window has no unaddressable byte (flags: BAD_PITCH,
    HOST_UNDEFINED).  The same with pitch 1: byte u lies in rows
    max(0, u-W+1) .. min(H-1, u), so count = sum over undefined u of that."""
    H0, S = 1 << 20, 1 << 20
    start = H0 + 8192
    tb = tg.TraceBuilder("ov40", H0, S)
    tb.mark(H0, S, tg.DEFINED)
    und = [5, 777, 4095]
    for u in und:
        tb.setv(start + u, b"\x10")
    dev = tb.malloc(1 << 41)                     # the device side is contiguous: 2^40 bytes
    tb.copy2d(tg.HTOD, 4096, 1 << 28, dev, 0, 0, 4096, start, 0, 0, 0)
    tb.copy2d(tg.HTOD, 4096, 1 << 28, dev, 0, 0, 4096, start, 0, 0, 1)
    tr = tb.build()
    kw = dict(FORMATS[fmt])
    chk = cg.Checker(tr.host_base, tr.host_size, max_descs=1024, max_allocs=1024, **kw)
    gv, gs = cg.replay_events(chk, tr.events, tr.blob)
    chk.close()
    H = 1 << 28
    assert gv[0]["undef_count"] == H * len(und) and gv[0]["first_undef"] == 5
    assert gv[0]["first_unaddr"] == oracle.NONE
    assert gv[0]["flags"] == oracle.F_BAD_PITCH | oracle.F_HOST_UNDEFINED
    # pitch 1: span = H - 1 + 4096 bytes from start run past the 1 MiB window end
    span = H - 1 + 4096
    to_end = H0 + S - start
    assert span > to_end
    # the first byte past the window: u = to_end, in rows u-4095 .. u -> first offset
    # u + (u - 4095) * (4096 - 1)
    u = to_end
    assert gv[1]["first_unaddr"] == u + (u - 4095) * 4095
    assert gv[1]["undef_count"] == sum(min(H - 1, x) - max(0, x - 4095) + 1 for x in und)
    assert gv[1]["first_undef"] == 5


def test_sparse_huge_gap(cg):
    """sparse map, a 2^40-byte HtoD starting in a marked region: the region is
    followed by unmarked chunks (no secondary: NOACCESS) and, 2^39 bytes later,
    by a second marked region -- first_unaddr is the region end, the undefined
    bytes of both regions count (R-4 raw count)."""
    base = 0x7000_0000_0000
    R = 3 * 65536
    chk = cg.Checker(0, 1 << 16, max_descs=64, max_allocs=64, shadow_format=2, sparse_capacity=8 * 65536)
    assert chk.host_mark(base, R, cg.CG_DEFINED) == 0
    assert chk.host_mark(base + (1 << 39), R, cg.CG_DEFINED) == 0
    assert chk.host_set_vbits(base + 1000, b"\x01") == 0
    assert chk.host_set_vbits(base + (1 << 39) + 7, b"\x80\x80") == 0
    dev = 1 << 44
    assert chk.register_alloc(dev, 1 << 41, 1) == 0
    d = np.zeros(2, cg.DESC_DTYPE)
    for i, (start, n) in enumerate([(base + 100, 1 << 40), (base + 100, (1 << 39) + R - 100)]):
        d[i]["kind"], d[i]["seq"], d[i]["width"], d[i]["height"] = tg.HTOD, 2 + i, n, 1
        d[i]["dst"], d[i]["dst_pitch"], d[i]["src"], d[i]["src_pitch"] = dev, n, start, n
    gv = cg.verdicts_to_numpy(chk.check_copies(cg.to_device_descs(d)))
    chk.close()
    for i in range(2):
        assert gv[i]["first_unaddr"] == R - 100
        assert gv[i]["undef_count"] == 3 and gv[i]["first_undef"] == 900
        assert gv[i]["flags"] == oracle.F_HOST_UNADDRESSABLE
