"""NEXT-4 compressed host shadow on the GPU (CG_SHADOW_2BIT, R-36):
the same checks over 2-bit states -- every verdict, status, leak and the
decoded final host shadow bit-exact against the oracle, in the fused and
unfused paths, sharded, and with the paper-shaped configurations."""
import numpy as np
import pytest

import oracle
import tracegen as tg
from test_gpu_parity import run_parity, new_checker

pytestmark = pytest.mark.gpu
TWO = dict(shadow_format=1)


@pytest.fixture(scope="module")
def cg():
    import torch
    assert torch.cuda.is_available()
    from paper_1310_0901_b200 import build
    build.build()
    import paper_1310_0901_b200 as m
    return m


def test_toy_and_listing2(cg):
    v = run_parity(cg, tg.toy(), **TWO)
    assert v[1]["first_undef"] == 100 and v[1]["undef_count"] == 33
    v = run_parity(cg, tg.listing2(), **TWO)
    assert (v[2]["src_expected"], v[2]["src_found"]) == (8000000, 4000000)


@pytest.mark.parametrize("seed", range(80))
def test_random_tiny(cg, seed):
    run_parity(cg, tg.random_tiny(seed, arrays=seed % 3 == 0), **TWO)


@pytest.mark.parametrize("seed", range(30))
def test_random_tiny_unfused(cg, seed):
    run_parity(cg, tg.random_tiny(seed + 3000), fuse=False, **TWO)


@pytest.mark.parametrize("seed", range(6))
def test_random_tiny_undef_is_error(cg, seed):
    run_parity(cg, tg.random_tiny(seed + 7000), undef_is_error=True, **TWO)


@pytest.mark.parametrize("seed", range(6))
def test_random_larger_windows(cg, seed):
    tr = tg.random_tiny(seed + 9000, n_events=400, window=4 << 20, host_base=0x4000000)
    run_parity(cg, tr, **TWO)


def test_small_batches(cg):
    run_parity(cg, tg.random_tiny(4242, n_events=300), max_descs=7, **TWO)


@pytest.mark.parametrize("fuse", [True, False])
def test_c2_scaled(cg, fuse):
    tr = tg.c2_small(n_copies=60000, n_allocs=6000)
    v = run_parity(cg, tr, fuse=fuse, **TWO)
    assert np.array_equal(v["flags"] != 0, tr.meta["inject"] != 0)


def test_c3_scaled(cg):
    tr = tg.c3_single(size=256 << 20)
    v = run_parity(cg, tr, **TWO)
    assert v[0]["undef_count"] == len(tr.meta["hole_offsets"])


@pytest.mark.parametrize("fuse", [True, False])
def test_c3_dtoh_scaled(cg, fuse):
    run_parity(cg, tg.c3_single(size=128 << 20, dtoh=True), fuse=fuse, **TWO)


def test_c4_scaled(cg):
    run_parity(cg, tg.c4_pitched(n_copies=4000, n_bufs=4, rows=256, inject_frac=0.03), **TWO)


def test_partial_vbytes_round_trip(cg):
    """set_vbits keeps exact partial V-bytes (host table) while the device
    state only says 'undefined'; a mark or a DtoH apply replaces them"""
    H0, S = 1 << 20, 1 << 16
    chk = cg.Checker(H0, S, max_descs=64, max_allocs=64, **TWO)
    o = oracle.Oracle(H0, S)
    rng = np.random.default_rng(1)
    for x, n, st in [(H0, 4096, cg.CG_DEFINED), (H0 + 100, 37, cg.CG_UNDEFINED), (H0 + 9000, 5000, cg.CG_DEFINED)]:
        assert chk.host_mark(x, n, st) == 0
        o.mark(x, n, st)
    for x in (H0 + 3, H0 + 130, H0 + 9001, H0 + 13950):
        vb = rng.integers(0, 256, int(rng.integers(1, 40)), dtype=np.uint8).tobytes()
        assert chk.host_set_vbits(x, vb) == 0
        assert o.set_vbits(x, vb) == 0
    assert chk.host_mark(H0 + 9000, 16, cg.CG_UNDEFINED) == 0
    o.mark(H0 + 9000, 16, cg.CG_UNDEFINED)
    A, V = chk.shadow()
    assert np.array_equal(A, o.A) and np.array_equal(V, o.V)
    a, v = chk.shadow_read(H0 + 120, 50)
    assert np.array_equal(v, o.V[120:170])
    assert chk.host_set_vbits(H0 + 60000, b"\x01") == cg.CG_ERR_INVALID_VALUE   # unaddressable
    chk.close()


def test_shadow_read_bytes_format(cg):
    """cg_host_shadow_read in the bytes format equals the raw shadow tensors"""
    tr = tg.random_tiny(77)
    chk = new_checker(cg, tr)
    cg.replay_events(chk, tr.events, tr.blob)
    A, V = chk.shadow()
    a, v = chk.shadow_read(tr.host_base, tr.host_size)
    assert np.array_equal(np.packbits(a, bitorder="little"), A) and np.array_equal(v, V)
    a, v = chk.shadow_read(tr.host_base + 13, 1000)
    assert np.array_equal(v, V[13:1013])
    chk.close()


def test_tracking_rejected(cg):
    with pytest.raises(cg.CgError):
        cg.Checker(1 << 20, 1 << 16, max_descs=64, max_allocs=64, dev_vsize=1 << 20, **TWO)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("seed", range(6))
def test_random_tiny_sharded(cg, world, seed):
    from test_gpu_sharded import run_sharded
    run_sharded(cg, tg.random_tiny(seed + 11000), world, fuse=bool(seed % 2), **TWO)


def test_c3_straddler_sharded(cg):
    from test_gpu_sharded import run_sharded
    tr = tg.c3_single(size=64 << 20, stride=1 << 16)
    v = run_sharded(cg, tr, 4, **TWO)
    assert v[0]["undef_count"] == len(tr.meta["hole_offsets"])


def test_c5_scaled_sharded(cg):
    from test_gpu_sharded import run_sharded
    run_sharded(cg, tg.c5_sharded(scale=0.01), 8, **TWO)


# ---------------------------------------------------------------------------
# the sparse two-level map (CG_SHADOW_SPARSE): the whole 64-bit host space
# ---------------------------------------------------------------------------
SPARSE = dict(shadow_format=2)


def test_sparse_toy_and_listing2(cg):
    run_parity(cg, tg.toy(), **SPARSE)
    v = run_parity(cg, tg.listing2(), **SPARSE)
    assert (v[2]["src_expected"], v[2]["src_found"]) == (8000000, 4000000)


@pytest.mark.parametrize("seed", range(40))
def test_sparse_random_tiny(cg, seed):
    run_parity(cg, tg.random_tiny(seed + 500, arrays=seed % 3 == 0), fuse=bool(seed % 2), **SPARSE)


@pytest.mark.parametrize("fuse", [True, False])
def test_sparse_c2_scaled(cg, fuse):
    tr = tg.c2_small(n_copies=30000, n_allocs=3000)
    v = run_parity(cg, tr, fuse=fuse, **SPARSE)
    assert np.array_equal(v["flags"] != 0, tr.meta["inject"] != 0)


def test_sparse_c4_scaled(cg):
    run_parity(cg, tg.c4_pitched(n_copies=2000, n_bufs=4, rows=128, inject_frac=0.03), **SPARSE)


@pytest.mark.parametrize("seed", range(6))
def test_sparse_relocated_regions(cg, seed):
    """relocation invariance: host regions scattered over the 64-bit space
    (the GPU's sparse map) give the verdicts the oracle computes with the
    regions packed into one dense window; each region's final shadow matches"""
    dense, sparse, bases, R = tg.sparse_regions(seed)
    o, ov, os_, _ = oracle.replay_trace(dense)
    chk = cg.Checker(sparse.host_base, R, max_descs=max(sparse.n_copies, 64), max_allocs=4096,
                     sparse_capacity=len(bases) * (R + 65536), **SPARSE)
    gv, gs = cg.replay_events(chk, sparse.events, sparse.blob, fuse=bool(seed % 2))
    for f in ov.dtype.names:
        bad = np.flatnonzero(gv[f] != ov[f])
        assert len(bad) == 0, (f, bad[:5], gv[f][bad[:5]], ov[f][bad[:5]])
    assert np.array_equal(gs, os_)
    for k, b in enumerate(bases):
        a, v = chk.shadow_read(b, R)
        lo = k * R
        assert np.array_equal(v, o.V[lo:lo + R]), k
        A = np.unpackbits(o.A, bitorder="little")[lo:lo + R]
        assert np.array_equal(a, A), k
    a, v = chk.shadow_read(1 << 40, 4096)                          # never marked: NOACCESS
    assert not a.any() and (v == 0xFF).all()
    chk.close()


def test_sparse_capacity(cg):
    chk = cg.Checker(0, 1 << 16, max_descs=64, max_allocs=64, sparse_capacity=2 * 65536, **SPARSE)
    assert chk.host_mark(0x7F00_0000_0000, 65536 + 10, cg.CG_DEFINED) == 0       # two chunks
    st = np.zeros(1, np.uint32)
    m = np.zeros(1, cg.MARK_DTYPE)
    m[0] = (0x5500_0000_0000, 16, cg.CG_UNDEFINED, 0)
    assert chk.host_mark_batch(m, status_out=st) == cg.CG_ERR_OUT_OF_MEMORY
    assert st[0] == cg.CG_ERR_OUT_OF_MEMORY
    assert chk.host_mark(0x5500_0000_0000, 16, cg.CG_NOACCESS) == 0              # needs no secondary
    assert chk.host_query_addressable(0x7F00_0000_0000, 65536 + 10)
    assert not chk.host_query_addressable(0x7F00_0000_0000, 65536 + 11)
    chk.close()
