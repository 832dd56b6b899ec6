"""Multi-GPU host logic on CPU: the shard plan against brute force, and the
N>1 communication path (three all-reduces with the u64->i64 order map, the
padded all_gather of compacted verdicts, root assembly) on world_size-2 gloo
process groups with 127.0.0.1 rendezvous."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import tracegen as tg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def cg():
    from paper_1310_0901_b200 import build
    build.build()
    import paper_1310_0901_b200 as m
    return m


def _host_range(d):
    if d["kind"] not in (1, 2) or d["width"] == 0 or d["height"] == 0:
        return None
    p = "src" if d["kind"] == 1 else "dst"
    s = int(d[p]) + int(d[p + "_y"]) * int(d[p + "_pitch"]) + int(d[p + "_x"])
    e = s + (int(d["height"]) - 1) * int(d[p + "_pitch"]) + int(d["width"])
    return None if e > (1 << 64) - 1 else (s, e)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_shard_plan_brute_force(cg, world):
    from paper_1310_0901_b200.replay import events_to_descs
    for seed in range(10):
        tr = tg.random_tiny(seed + 100 * world)
        descs = events_to_descs(tr.events[tr.events["op"] == tg.OP_COPY])
        owner, first, last = cg.shard_plan(descs, tr.host_base, tr.host_size, world)
        S = tr.host_size // world
        for i, d in enumerate(descs):
            r = _host_range(d)
            if r is None:
                assert owner[i] == i % world and first[i] == last[i] == owner[i]
                continue
            lo, hi = r
            s0 = min(max(lo, tr.host_base), tr.host_base + tr.host_size - 1)
            assert owner[i] == (s0 - tr.host_base) // S
            shards = {(x - tr.host_base) // S for x in range(max(lo, tr.host_base), min(hi, tr.host_base + tr.host_size))}
            shards.add(int(owner[i]))
            assert (first[i], last[i]) == (min(shards), max(shards))


def test_batch_plan_partition(cg):
    from paper_1310_0901_b200.replay import events_to_descs
    from paper_1310_0901_b200.sharded import BatchPlan
    tr = tg.c4_pitched(n_copies=3000, n_bufs=4, rows=128)
    descs = events_to_descs(tr.events[tr.events["op"] == tg.OP_COPY])
    plan = BatchPlan(descs, tr.host_base, tr.host_size, 4)
    # every descriptor is owned by exactly one rank or is a straddler on all
    seen = np.zeros(len(descs), int)
    for r in range(4):
        d, idx, n_mine, m = plan.local(r)
        assert m == len(plan.strad_idx)
        seen[idx[:n_mine]] += 1
        assert np.all(d["reserved"][:n_mine] == 0)
        assert np.all(d["reserved"][n_mine:] & cg.CG_SHARD_RAW)
        own = plan.owner[plan.strad_idx] == r
        assert np.array_equal((d["reserved"][n_mine:] & cg.CG_SHARD_NOT_OWNER) == 0, own)
    seen[plan.strad_idx] += 1
    assert np.all(seen == 1)
    assert len(plan.strad_idx) > 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys
    sys.path.insert(0, ROOT)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1310_0901_b200 import VERDICT_DTYPE, CG_NONE
        from paper_1310_0901_b200.sharded import TorchComm, _u64_min_fix
        comm = TorchComm()
        m = 5
        rng = np.random.default_rng(rank)
        # raw partials: first offsets (u64, NONE = 2^64-1), sums, flags
        firsts = rng.integers(0, 1 << 62, 2 * m).astype(np.uint64)
        firsts[rank::2] = np.uint64(CG_NONE)
        firsts[0] = np.uint64((1 << 63) + rank)        # above 2^63: needs the order map
        mins = torch.from_numpy(firsts.view(np.int64).copy())
        sums = torch.from_numpy(rng.integers(0, 1000, 5 * m).astype(np.int64))
        # validation flags are common to all shards; device flags come from the owner (rank 0)
        common = np.array([64, 64, 0, 2, 4], np.int32)
        dev = np.array([1, 0, 0, 1, 1], np.int32) if rank == 0 else 0
        maxs = torch.from_numpy(common | dev)
        all_f = [None] * world
        mins = _u64_min_fix(mins)
        comm.allreduce3(mins, sums, maxs)
        mins = _u64_min_fix(mins)
        # compacted verdict gather
        n_dirty = rank + 1
        dirty = np.zeros(n_dirty, VERDICT_DTYPE)
        dirty["flags"] = rank + 1
        dirty["first_unaddr"] = np.arange(n_dirty) + 10 * rank
        idx = torch.arange(n_dirty, dtype=torch.int64) * 2 + rank
        cnt = torch.tensor([n_dirty], dtype=torch.int32)
        g = comm.gather_dirty(cnt, idx, torch.from_numpy(dirty.view(np.uint8).copy()))
        q.put((rank, mins.numpy().view(np.uint64).tolist(), sums.tolist(), maxs.tolist(),
               [(c, i[:c].tolist(), d[:c]["first_unaddr"].tolist(), d[:c]["flags"].tolist()) for c, i, d in g],
               firsts.tolist(), rng.bit_generator.state is not None))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_exchange():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict()
    for _ in range(world):
        r = q.get(timeout=180)
        res[r[0]] = r
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    # recompute the expected merge from the inputs each rank reported
    f0, f1 = np.array(res[0][5], np.uint64), np.array(res[1][5], np.uint64)
    exp_min = np.minimum(f0, f1)
    for r in range(world):
        assert np.array_equal(np.array(res[r][1], np.uint64), exp_min)
        assert res[r][3] == [65, 64, 0, 3, 5]          # MAX == OR for common | owner-only flags
        gathered = res[r][4]
        assert [g[0] for g in gathered] == [1, 2]
        assert gathered[1][1] == [1, 3] and gathered[1][3] == [2, 2]
    assert res[0][2] == res[1][2]


def _packed_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys
    sys.path.insert(0, ROOT)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1310_0901_b200 import VERDICT_DTYPE
        from paper_1310_0901_b200.sharded import PackedDirtyGather
        g = PackedDirtyGather(dist, 5, torch.device("cpu"))
        c = 2 + rank
        # what cg_compact_dirty would write into the send buffer
        g.send[:4] = torch.from_numpy(np.array([c], np.int32).view(np.uint8))
        idx = np.arange(c, dtype=np.int64) * 3 + rank
        g.send[16:16 + 8 * c] = torch.from_numpy(idx.view(np.uint8))
        dv = np.zeros(c, VERDICT_DTYPE)
        dv["flags"] = 100 + rank
        dv["first_unaddr"] = idx * 7
        off = 16 + 8 * g.mx
        g.send[off:off + 64 * c] = torch.from_numpy(dv.view(np.uint8))
        g.gather()
        q.put((rank, [(cc, i.tolist(), d["flags"].tolist(), d["first_unaddr"].tolist()) for cc, i, d in g.unpack()]))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_packed_gather():
    """the bench's one-collective exchange of compacted verdicts on world_size 2"""
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_packed_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        for src in range(world):
            c, idx, flags, fu = res[r][src]
            assert c == 2 + src
            assert idx == [3 * k + src for k in range(c)]
            assert flags == [100 + src] * c and fu == [7 * x for x in idx]
