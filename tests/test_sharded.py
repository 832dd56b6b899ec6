"""Multi-GPU host logic on CPU: the shard plan against brute force, the
per-rank lists of cg_shard_lists (a partition: every descriptor owned by one
rank or a straddler everywhere, same straddler order on every rank, mode and
apply-after bits), and the N>1 host path on world_size-2 gloo process groups
with 127.0.0.1 rendezvous: every rank plans its own list independently, the
NCCL unique id travels from rank 0 over torch.distributed as ShardGroup hands
it over, and the lists the ranks built agree with each other.  The
collectives themselves run inside the library (cg_check_sharded, NCCL) and
are covered on the GPU (loopback backend, 1-rank NCCL)."""
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


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_shard_lists_partition(cg, world):
    from paper_1310_0901_b200.sharded import shard_lists
    for tr in (tg.c4_pitched(n_copies=3000, n_bufs=4, rows=128), tg.random_tiny(77 + world),
               tg.random_medium(3, n_copies=60)):
        descs = tg.events_to_descs(tr.events[tr.events["op"] == tg.OP_COPY])
        owner, first, last = cg.shard_plan(descs, tr.host_base, tr.host_size, world)
        strad = np.flatnonzero(first < last)
        seen = np.zeros(len(descs), int)
        for r in range(world):
            d, gidx, n_own, m = shard_lists(descs, tr.host_base, tr.host_size, world, r)
            assert m == len(strad) and np.array_equal(gidx[n_own:], strad)
            mine = gidx[:n_own].astype(np.int64)
            assert np.all(owner[mine] == r) and np.all(first[mine] == last[mine])
            seen[mine] += 1
            raw = d["reserved"][n_own:]
            assert np.all(raw & cg.CG_SHARD_RAW)
            assert np.array_equal((raw & cg.CG_SHARD_NOT_OWNER) == 0, owner[strad] == r)
            assert np.all((d["reserved"][:n_own] & (cg.CG_SHARD_RAW | cg.CG_SHARD_NOT_OWNER)) == 0)
            # CG_APPLY_AFTER exactly as cg_plan_apply_after sets it on the owned part of the list
            own = np.ascontiguousarray(d[:n_own]).copy()
            own["reserved"] = 0
            plain = np.ascontiguousarray(d).copy()
            plain["reserved"] &= ~np.uint32(cg.CG_APPLY_AFTER)
            cg.plan_apply_after(plain)
            assert np.array_equal(plain["reserved"][:n_own], d["reserved"][:n_own])
            for f in ("kind", "seq", "width", "height", "dst", "src", "dst_pitch", "src_pitch"):
                assert np.array_equal(d[f], descs[f][gidx.astype(np.int64)])
        seen[strad] += 1
        assert np.all(seen == 1)


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
        import tracegen as tgw
        from paper_1310_0901_b200.sharded import shard_lists
        tr = tgw.c5_sharded(scale=0.002, shards=world)
        descs = tgw.events_to_descs(tr.events[tr.events["op"] == tgw.OP_COPY])
        d, gidx, n_own, m = shard_lists(descs, tr.host_base, tr.host_size, world, rank)
        # the id hand-over ShardGroup does for the NCCL backend (rank 0's bytes to all)
        nid = torch.arange(128, dtype=torch.uint8) if rank == 0 else torch.zeros(128, dtype=torch.uint8)
        dist.broadcast(nid, 0)
        # every rank's view of the straddlers, gathered for comparison
        sg = torch.from_numpy(gidx[n_own:].astype(np.int64))
        lens = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(lens, torch.tensor([len(sg)]))
        outs = [torch.zeros(int(l.item()), dtype=torch.int64) for l in lens]
        dist.all_gather(outs, sg)
        q.put((rank, nid.tolist(), n_own, m, [o.tolist() for o in outs], gidx[:n_own].tolist(), len(descs)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_host_path():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=300)
        res[r[0]] = r
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        assert res[r][1] == list(range(128))                      # rank 0's NCCL id reached every rank
        assert res[r][4][0] == res[r][4][1]                        # same straddlers, same order
    n = res[0][6]
    owned = sorted(res[0][5] + res[1][5])
    strad = res[0][4][0]
    assert sorted(owned + strad) == list(range(n))               # a partition of the batch
    assert res[0][3] == res[1][3] == len(strad) and len(strad) > 0
