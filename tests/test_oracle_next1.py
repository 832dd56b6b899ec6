"""NEXT-1 pins (SPEC copy_vbits S:81-89, S:92, S:101, S:547,
S:279): with device V-bits tracked, error-free copies move V-bits
bit-exactly between host and device shadows."""
import numpy as np
import pytest

import oracle
import tracegen as tg
from flatmodel import FlatModel
from oracle import Oracle


def _copy(kind, dst, src, n, seq, **kw):
    e = np.zeros(1, tg.EVENT_DTYPE)[0]
    e["op"] = tg.OP_COPY; e["kind"] = kind; e["seq"] = seq
    e["width"] = n; e["height"] = 1; e["dst"] = dst; e["src"] = src
    e["dst_pitch"] = n; e["src_pitch"] = n
    for k, v in kw.items():
        e[k] = v
    return e


H0 = 0x100000


def fresh(n_alloc=4, size=1 << 14):
    o = Oracle(H0, 1 << 20, track_device=True)
    devs = []
    for i in range(n_alloc):
        base = 0x1000000 + i * 0x10000
        assert o.register(base, size, i + 1) == 0
        devs.append(base)
    return o, devs


def test_fresh_device_memory_is_undefined():
    o, d = fresh()
    assert np.all(o.device_vbits(d[0], 1 << 14) == 0xFF)


def test_copy_from_defined_source_defines_destination():
    o, d = fresh()
    o.mark(H0, 4096, tg.DEFINED)
    v = o.check_copy(_copy(tg.HTOD, d[0], H0, 4096, 10))
    assert v["flags"] == 0
    assert not o.device_vbits(d[0], 4096).any()
    assert np.all(o.device_vbits(d[0] + 4096, 100) == 0xFF)


def test_zero_length_changes_nothing():
    o, d = fresh()
    o.mark(H0, 64, tg.DEFINED)
    before = o.device_vbits(d[0], 64).copy()
    o.check_copy(_copy(tg.HTOD, d[0], H0, 0, 10))
    assert np.array_equal(before, o.device_vbits(d[0], 64))


@pytest.mark.parametrize("seed", range(200))
def test_round_trip_htod_dtod_dtoh(seed):
    """S:547 / S:89: for any host V pattern P, HtoD -> DtoD -> DtoH into a fresh
    addressable host range reproduces P bit-exactly (also conservation S:92)."""
    rng = np.random.default_rng(seed)
    o, d = fresh()
    n = int(rng.integers(1, 5000))
    pat = rng.integers(0, 256, n, dtype=np.uint8)
    pat[rng.random(n) < 0.5] = 0
    o.mark(H0, n, tg.DEFINED)
    o.set_vbits(H0, pat.tobytes())
    o.mark(H0 + 0x20000, n, tg.UNDEFINED)
    off1, off2 = int(rng.integers(0, 100)), int(rng.integers(0, 100))
    v1 = o.check_copy(_copy(tg.HTOD, d[0] + off1, H0, n, 10))
    assert np.unpackbits(o.device_vbits(d[0] + off1, n)).sum() == np.unpackbits(pat).sum()
    v2 = o.check_copy(_copy(tg.DTOD, d[1] + off2, d[0] + off1, n, 11))
    v3 = o.check_copy(_copy(tg.DTOH, H0 + 0x20000, d[1] + off2, n, 12))
    assert v1["status"] == v2["status"] == v3["status"] == 0
    assert np.array_equal(o.V[0x20000:0x20000 + n], pat)


@pytest.mark.parametrize("shift", [-300, -17, -1, 1, 5, 129, 2000])
def test_self_overlapping_dtod_is_memmove(shift):
    """a self-overlapping DtoD behaves as if staged through a
    scratch buffer (brute force: numpy copy then assign)."""
    rng = np.random.default_rng(abs(shift))
    o, d = fresh()
    pat = rng.integers(0, 256, 1 << 14, dtype=np.uint8)
    o.mark(H0, 1 << 14, tg.DEFINED)
    o.set_vbits(H0, pat.tobytes())
    o.check_copy(_copy(tg.HTOD, d[0], H0, 1 << 14, 10))
    n, s0 = 5000, 4000
    expect = pat.copy()
    expect[s0 + shift:s0 + shift + n] = pat[s0:s0 + n].copy()
    v = o.check_copy(_copy(tg.DTOD, d[0] + s0 + shift, d[0] + s0, n, 11))
    assert v["status"] == 0
    assert np.array_equal(o.device_vbits(d[0], 1 << 14), expect)


def test_error_leaves_device_bits_unchanged():
    o, d = fresh(size=1024)
    o.mark(H0, 4096, tg.DEFINED)
    before = o.device_vbits(d[0], 1024).copy()
    v = o.check_copy(_copy(tg.HTOD, d[0], H0, 2048, 10))          # DstTooSmall: an Error
    assert v["status"] == 1
    assert np.array_equal(before, o.device_vbits(d[0], 1024))


def test_free_then_reuse_is_fresh():
    o, d = fresh(n_alloc=1)
    o.mark(H0, 64, tg.DEFINED)
    o.check_copy(_copy(tg.HTOD, d[0], H0, 64, 10))
    assert o.free(d[0], 11) == 0
    assert o.register(d[0], 1 << 14, 12) == 0
    assert np.all(o.device_vbits(d[0], 64) == 0xFF)


@pytest.mark.parametrize("seed", range(40))
def test_flat_model_equivalence_tracking(seed):
    """S:546 with V-bit propagation: oracle == independent numpy model."""
    tr = tg.random_tiny(seed + 20000)
    o, v, s, leaks = oracle.replay_trace(tr, track_device=True)
    fm = FlatModel(tr.host_base, tr.host_size, track=True)
    fv, fs = fm.replay(tr.events, tr.blob)
    assert list(s) == fs
    for i, (a, b) in enumerate(zip(v, fv)):
        assert {k: int(a[k]) for k in v.dtype.names} == b, i
    assert np.array_equal(o.V, fm.v)
    for base, arr in fm.dv.items():
        assert np.array_equal(o.device_vbits(base, len(arr)), arr), hex(base)
