"""Random medium traces on the GPU (tracegen.random_medium): copies up to
8 MiB, unaligned, 2D with hundreds of rows, straddling the window edges, with
violations planted at +-1 of the scan's 4 KiB tile, 32 KiB block / chunk and
128 KiB split boundaries (absolute and per copy).  These reach the split
(k_finalize_split / k_finish) path and the tile-edge code that the tiny traces
cannot.  Bit-exact against the oracle: verdicts, statuses, leaks, final
shadow."""
import numpy as np
import pytest

import tracegen as tg
from test_gpu_parity import run_parity
from test_gpu_sharded import run_sharded

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cg():
    import torch
    assert torch.cuda.is_available()
    from paper_1310_0901_b200 import build
    build.build()
    import paper_1310_0901_b200 as m
    return m


@pytest.mark.parametrize("seed", range(50))
def test_medium_fused(cg, seed):
    run_parity(cg, tg.random_medium(seed), fuse=True)


@pytest.mark.parametrize("seed", range(50))
def test_medium_unfused(cg, seed):
    run_parity(cg, tg.random_medium(seed + 100), fuse=False)


@pytest.mark.parametrize("seed", range(16))
def test_medium_2bit(cg, seed):
    run_parity(cg, tg.random_medium(seed + 200), fuse=bool(seed % 2), shadow_format=1)


@pytest.mark.parametrize("seed", range(8))
def test_medium_sparse(cg, seed):
    run_parity(cg, tg.random_medium(seed + 300), fuse=bool(seed % 2), shadow_format=2,
               sparse_capacity=(64 << 20) + (1 << 20))


@pytest.mark.parametrize("seed", range(8))
def test_medium_small_batches(cg, seed):
    """max_descs 7: batches are cut far more often than the epochs require"""
    run_parity(cg, tg.random_medium(seed + 400, n_copies=60), max_descs=7)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("seed", range(4))
def test_medium_sharded(cg, world, seed):
    run_sharded(cg, tg.random_medium(seed + 500, n_copies=60), world, fuse=bool(seed % 2))


@pytest.mark.parametrize("seed", range(24))
def test_pingpong_fused(cg, seed):
    """DtoH -> HtoD ping-pongs: CG_CHECK_AFTER HtoDs, CG_APPLY_AFTER and
    CG_APPLY_LAST DtoHs (some failing) in the same fused batch; bytes, 2-bit
    and sparse formats"""
    fmt = (0, 0, 1, 2)[seed % 4]
    kw = dict(sparse_capacity=(8 << 20) + (1 << 20)) if fmt == 2 else {}
    run_parity(cg, tg.pingpong_trace(seed), fuse=True, shadow_format=fmt, **kw)


@pytest.mark.parametrize("seed", range(4))
def test_pingpong_small_batches(cg, seed):
    """the same with max_descs 5: the replay splits fused batches into pieces"""
    run_parity(cg, tg.pingpong_trace(seed + 100, n_copies=80), fuse=True, max_descs=5)


@pytest.mark.parametrize("seed", range(6))
def test_medium_front_split(cg, seed, monkeypatch):
    """the prep and the plan as separate kernels (CG_FRONT_COOP=0, the path of
    batches above 4M descriptors)"""
    monkeypatch.setenv("CG_FRONT_COOP", "0")
    run_parity(cg, tg.random_medium(seed + 600), fuse=bool(seed % 2))
    run_parity(cg, tg.pingpong_trace(seed + 600), fuse=True)
