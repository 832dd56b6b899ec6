"""NEXT-1 on the GPU: device V-bit tracking (SPEC copy_vbits) bit-exact against
the oracle's tracking mode -- verdicts, statuses, leaks, host A/V and the
device V-bits of every allocation live at the end."""
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


def run_tracking(cg, tr, **kw):
    o, ov, os_, oleaks = oracle.replay_trace(tr, track_device=True)
    ev = tr.events
    regs = ev[ev["op"] == tg.OP_REG]
    pool = int(sum(int(x) + 256 for x in regs["width"])) + (1 << 20)
    chk = cg.Checker(tr.host_base, tr.host_size, max_descs=max(tr.n_copies, 1024),
                     max_allocs=max(len(regs), 1024), dev_vsize=pool, **kw)
    gv, gs = cg.replay_events(chk, ev, tr.blob)
    for f in ov.dtype.names:
        bad = np.flatnonzero(gv[f] != ov[f])
        assert len(bad) == 0, (f, bad[:5], gv[f][bad[:5]], ov[f][bad[:5]])
    assert np.array_equal(gs, os_)
    gl = chk.leak_report()
    assert np.array_equal(gl["base"], oleaks["base"]) and np.array_equal(gl["size"], oleaks["size"])
    A, V = chk.shadow()
    assert np.array_equal(A, o.A) and np.array_equal(V, o.V)
    for r in oleaks:
        b, n = int(r["base"]), int(r["size"])
        assert np.array_equal(chk.device_vbits(b, n), o.device_vbits(b, n)), hex(b)
    chk.close()
    return gv


@pytest.mark.parametrize("seed", range(60))
def test_random_tiny_tracking(cg, seed):
    run_tracking(cg, tg.random_tiny(seed + 20000))


def test_c2_scaled_tracking(cg):
    run_tracking(cg, tg.c2_small(n_copies=20000, n_allocs=2000))


def test_c4_scaled_tracking(cg):
    run_tracking(cg, tg.c4_pitched(n_copies=600, n_bufs=2, rows=64, inject_frac=0.05))


@pytest.mark.parametrize("seed", range(20))
def test_round_trip(cg, seed):
    """any host pattern, HtoD -> DtoD -> DtoH into a fresh range, comes back bit-exact."""
    rng = np.random.default_rng(seed)
    H0 = 1 << 20
    tb = tg.TraceBuilder("rt", H0, 1 << 20)
    n = int(rng.integers(1, 60000))
    d0, d1 = tb.malloc(n + 200), tb.malloc(n + 200)
    pat = rng.integers(0, 256, n, dtype=np.uint8)
    pat[rng.random(n) < 0.6] = 0
    tb.mark(H0, n, tg.DEFINED)
    tb.setv(H0, pat.tobytes())
    tb.mark(H0 + (1 << 19), n, tg.UNDEFINED)
    a, b = int(rng.integers(0, 100)), int(rng.integers(0, 100))
    tb.copy1d(tg.HTOD, d0 + a, H0, n)
    tb.copy1d(tg.DTOD, d1 + b, d0 + a, n)
    tb.copy1d(tg.DTOH, H0 + (1 << 19), d1 + b, n)
    tr = tb.build()
    run_tracking(cg, tr)
    o = oracle.replay_trace(tr, track_device=True)[0]
    assert np.array_equal(o.V[1 << 19:(1 << 19) + n], pat)


@pytest.mark.parametrize("shape", ["1d", "2d_equal", "2d_unequal"])
@pytest.mark.parametrize("shift", [-4100, -33, 7, 5000])
def test_self_overlapping_dtod(cg, shape, shift):
    """memmove semantics for a DtoD overlapping itself"""
    rng = np.random.default_rng(abs(shift))
    H0 = 1 << 20
    tb = tg.TraceBuilder("mm", H0, 1 << 18)
    d = tb.malloc(1 << 17)
    pat = rng.integers(0, 256, 1 << 16, dtype=np.uint8)
    tb.mark(H0, 1 << 16, tg.DEFINED)
    tb.setv(H0, pat.tobytes())
    tb.copy1d(tg.HTOD, d + 20000, H0, 1 << 16)
    s0 = 30000
    if shape == "1d":
        tb.copy1d(tg.DTOD, d + s0 + shift, d + s0, 20000)
    elif shape == "2d_equal":
        tb.copy2d(tg.DTOD, 300, 40, d + s0 + shift, 0, 0, 700, d + s0, 0, 0, 700)
    else:
        tb.copy2d(tg.DTOD, 300, 40, d + s0 + shift, 0, 0, 650, d + s0, 0, 0, 700)
    run_tracking(cg, tb.build())


@pytest.mark.parametrize("seed", range(3))
def test_round_trip_large_waves(cg, seed):
    """HtoD -> DtoD -> DtoH chains of 2-3 MiB copies: three waves whose copies
    exceed the warp-per-copy limit, so each wave takes the planned path"""
    rng = np.random.default_rng(seed + 100)
    H0 = 1 << 24
    tb = tg.TraceBuilder("rtl", H0, 16 << 20)
    n = int(rng.integers(2 << 20, 3 << 20))
    d0, d1 = tb.malloc(n + 256), tb.malloc(n + 256)
    pat = rng.integers(0, 256, n, dtype=np.uint8)
    pat[rng.random(n) < 0.7] = 0
    tb.mark(H0, n, tg.DEFINED)
    tb.setv(H0, pat.tobytes())
    tb.mark(H0 + (8 << 20), n, tg.UNDEFINED)
    tb.copy1d(tg.HTOD, d0, H0, n)
    tb.copy1d(tg.DTOD, d1 + 16, d0, n)
    tb.copy1d(tg.DTOH, H0 + (8 << 20), d1 + 16, n)
    tr = tb.build()
    run_tracking(cg, tr)
    o = oracle.replay_trace(tr, track_device=True)[0]
    assert np.array_equal(o.V[8 << 20:(8 << 20) + n], pat)


@pytest.mark.parametrize("wave_kernel", ["0", "1"])
def test_c2_scaled_tracking_both_wave_paths(cg, monkeypatch, wave_kernel):
    """cg_apply_copies_waves in one cooperative launch (default) and wave by
    wave (CG_WAVE_KERNEL=0) give the same, oracle-exact device V-bits"""
    monkeypatch.setenv("CG_WAVE_KERNEL", wave_kernel)
    run_tracking(cg, tg.c2_small(n_copies=30000, n_allocs=1500))


@pytest.mark.parametrize("seed", range(4))
def test_deep_chains_tracking(cg, seed):
    """many dependency waves: copies ping-pong over few host buffers and
    allocations, so most copies conflict with an earlier one (R-28)"""
    rng = np.random.default_rng(seed + 500)
    H0 = 1 << 20
    tb = tg.TraceBuilder("chain", H0, 1 << 20)
    devs = [tb.malloc(1 << 14) for _ in range(4)]
    tb.mark(H0, 1 << 16, tg.DEFINED)
    pat = rng.integers(0, 256, 1 << 16, dtype=np.uint8)
    pat[rng.random(1 << 16) < 0.5] = 0
    tb.setv(H0, pat.tobytes())
    tb.mark(H0 + (1 << 17), 1 << 16, tg.UNDEFINED)
    for _ in range(400):
        n = int(rng.integers(1, 9000))
        k = int(rng.integers(0, 3))
        if k == 0:
            tb.copy1d(tg.HTOD, devs[rng.integers(4)] + int(rng.integers(0, (1 << 14) - n)),
                      H0 + int(rng.integers(0, (1 << 16) - n)), n)
        elif k == 1:
            tb.copy1d(tg.DTOD, devs[rng.integers(4)] + int(rng.integers(0, (1 << 14) - n)),
                      devs[rng.integers(4)] + int(rng.integers(0, (1 << 14) - n)), n)
        else:
            tb.copy1d(tg.DTOH, H0 + (1 << 17) + int(rng.integers(0, (1 << 16) - n)),
                      devs[rng.integers(4)] + int(rng.integers(0, (1 << 14) - n)), n)
    run_tracking(cg, tb.build())


@pytest.mark.parametrize("shift", [-5000, 3333])
@pytest.mark.parametrize("wave_kernel", ["0", "1"])
def test_self_overlapping_2d_beyond_staging(cg, monkeypatch, shift, wave_kernel):
    """S:84 / S:101 memmove semantics for a 32 MiB self-overlapping 2D DtoD with
    unequal pitches -- four times the 8 MiB staging area: it is staged through
    a buffer of its own size after the rest of its wave, and the next wave (a
    DtoH of the moved bytes) sees the moved V-bits"""
    monkeypatch.setenv("CG_WAVE_KERNEL", wave_kernel)
    rng = np.random.default_rng(abs(shift))
    H0 = 1 << 24
    W, H = 8192, 4096                       # 32 MiB
    sp, dp = 8192 + 512, 8192 + 128         # unequal pitches: the rows interleave
    tb = tg.TraceBuilder("mm32", H0, 96 << 20)
    d = tb.malloc((H + 2) * sp + (1 << 16))
    n = (H - 1) * sp + W
    pat = rng.integers(0, 256, n, dtype=np.uint8)
    pat[rng.random(n) < 0.6] = 0
    tb.mark(H0, n, tg.DEFINED)
    tb.setv(H0, pat.tobytes())
    s0 = 40000
    tb.copy1d(tg.HTOD, d + s0, H0, n)
    tb.copy2d(tg.DTOD, W, H, d + s0 + shift, 0, 0, dp, d + s0, 0, 0, sp)
    tb.mark(H0 + (40 << 20), W * H, tg.UNDEFINED)
    tb.copy2d(tg.DTOH, W, H, H0 + (40 << 20), 0, 0, W, d + s0 + shift, 0, 0, dp)
    tr = tb.build()
    run_tracking(cg, tr)
    o = oracle.replay_trace(tr, track_device=True)[0]
    # the DtoH brought the rows of the moved V-bits back: row r of the result = row r of the source pattern
    got = o.V[40 << 20:(40 << 20) + W * H].reshape(H, W)
    exp = np.stack([pat[r * sp:r * sp + W] for r in range(H)])
    assert np.array_equal(got, exp)
