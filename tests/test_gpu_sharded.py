"""Sharded checking on one GPU (loopback): G contexts, each holding one shard
of the host window, run the per-rank kernels; the straddler all-reduces and
the verdict gather are done across the G device tensors.  Results must equal
the unsharded sequential oracle bit for bit (verdicts, statuses, leaks, and
the concatenated shard shadows), for G = 2, 4, 8 -- shard invariance."""
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


def run_sharded(cg, tr, world, fuse=True, **kw):
    """G shards of one window in this process (the library's loopback
    cg_comm): per-rank lists from cg_shard_lists, cg_check_sharded (check,
    straddler exchange, gather, root merge kernel into the dense array)"""
    from paper_1310_0901_b200.sharded import ShardGroup, replay_sharded
    o, ov, os_, oleaks = oracle.replay_trace(tr)
    nreg = max(int(np.count_nonzero(tr.events["op"] == tg.OP_REG)), 1024)
    n = max(tr.n_copies, 1024)
    grp = ShardGroup(tr.host_base, tr.host_size, world, backend="loopback", max_descs=n, max_allocs=nreg,
                     max_straddlers=n, cap=n, **kw)
    gv, gs = replay_sharded(grp, tr.events, tr.blob, fuse=fuse)
    for f in ov.dtype.names:
        bad = np.flatnonzero(gv[f] != ov[f])
        assert len(bad) == 0, (world, f, bad[:5], gv[f][bad[:5]], ov[f][bad[:5]])
    assert np.array_equal(gs, os_), np.flatnonzero(gs != os_)[:10]
    for c in grp.chks:
        l = c.leak_report()
        assert np.array_equal(l["base"], oleaks["base"]) and np.array_equal(l["size"], oleaks["size"])
    shards = [c.shadow() for c in grp.chks]
    A = np.concatenate([s[0] for s in shards])
    V = np.concatenate([s[1] for s in shards])
    assert np.array_equal(A, o.A) and np.array_equal(V, o.V)
    grp.close()
    return gv


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("seed", range(12))
def test_random_tiny_sharded(cg, world, seed):
    run_sharded(cg, tg.random_tiny(seed + 11000), world, fuse=bool(seed % 2))


@pytest.mark.parametrize("world", [2, 4])
def test_c2_sharded(cg, world):
    tr = tg.c2_small(n_copies=30000, n_allocs=3000)
    run_sharded(cg, tr, world)


def test_c3_single_descriptor_straddles_all_shards(cg):
    tr = tg.c3_single(size=64 << 20, stride=1 << 16)
    v = run_sharded(cg, tr, 4)
    assert v[0]["undef_count"] == len(tr.meta["hole_offsets"])


@pytest.mark.parametrize("dtoh", [False, True])
def test_c3_dtoh_straddler_apply(cg, dtoh):
    run_sharded(cg, tg.c3_single(size=32 << 20, dtoh=dtoh), 4)


def test_c4_sharded(cg):
    tr = tg.c4_pitched(n_copies=1500, n_bufs=4, rows=128, inject_frac=0.05)
    run_sharded(cg, tr, 2)


@pytest.mark.parametrize("world", [1, 8])
def test_c5_scaled_sharded(cg, world):
    """C5 at 1% scale: 100k copies, interleaved alloc/free bursts, ping-pong
    epochs, large copies straddling shard boundaries, final leak report."""
    tr = tg.c5_sharded(scale=0.01)
    run_sharded(cg, tr, world, fuse=True)


def test_nccl_path_single_rank(cg):
    """The library's NCCL backend end to end on a 1-rank process group (the
    NCCL id handed over with torch.distributed): check, (empty) straddler
    exchange, gather, root merge -- equal to the oracle and to the loopback
    backend with one shard."""
    import os
    import torch
    import torch.distributed as dist
    from paper_1310_0901_b200.sharded import ShardGroup, replay_sharded
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29531")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        tr = tg.c2_small(n_copies=20000, n_allocs=2000)
        o, ov, _, _ = oracle.replay_trace(tr)
        grp = ShardGroup(tr.host_base, tr.host_size, 1, backend="nccl", rank=0, max_descs=20000, max_allocs=4096,
                         max_straddlers=1024, cap=20000)
        v, _ = replay_sharded(grp, tr.events, tr.blob)
        for f in ov.dtype.names:
            assert np.array_equal(v[f], ov[f]), f
        grp.close()
        v1 = run_sharded(cg, tr, 1)
        assert np.array_equal(v1, v)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_cap_overflow_reported(cg, world):
    """a cap smaller than a rank's dirty count: the root's list is marked
    incomplete (cg_comm_overflow), the ranks' own verdicts stay exact"""
    from paper_1310_0901_b200.sharded import ShardGroup
    tr = tg.c2_small(n_copies=20000, n_allocs=2000, inject_frac=0.05)
    grp = ShardGroup(tr.host_base, tr.host_size, world, backend="loopback", max_descs=20000, max_allocs=4096,
                     max_straddlers=1024, cap=8)
    ev = tr.events
    for c in grp.chks:
        cg.replay_events(c, ev[ev["op"] != tg.OP_COPY], tr.blob)
    b = grp.batch(tg.events_to_descs(ev[ev["op"] == tg.OP_COPY]))
    grp.check(b)
    import torch
    torch.cuda.synchronize()
    assert grp.overflow()
    assert not grp.overflow()          # the query resets it
    grp.close()
