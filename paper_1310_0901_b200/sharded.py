"""Host-address-range sharding across GPUs (BASELINE north_star:
"The shadow address space and copy batch are partitioned across the 8 B200s
by host-address range, with an NCCL gather over NVLink only for the
per-descriptor verdicts").

Argument marshalling only: the planning (cg_shard_lists), the check, the
straddler exchange, the gather and the root merge all run in the library
(cg_comm / cg_check_sharded, csrc/cg_shard.cu); torch provides the device
buffers, the process group that hands the NCCL id to every rank, and the
streams.

Rank r stores the shadow of shard r = [H0 + r*S/G, H0 + (r+1)*S/G) of the
global window and replays every setup event (only its shard part is stored;
the allocation table is replicated).  Two backends: NCCL (one rank per
process, torchrun) and loopback (all G shards in this process on one GPU --
the single-GPU test and measurement of the same code path).
"""
from __future__ import annotations

import ctypes
from typing import List, Optional

import numpy as np

from . import (CG_COMM_LOOPBACK, CG_COMM_NCCL, CG_NCCL_ID_BYTES, CG_NONE, DESC_DTYPE, MARK_DTYPE, VERDICT_DTYPE,
               Checker, CgError, _lib, _stream_ptr, plan_batches)


def shard_lists(descs: np.ndarray, host_base: int, host_size: int, world: int, rank: int):
    """cg_shard_lists: (rank's list with mode bits, global indices, n_own, m)"""
    d = np.ascontiguousarray(descs, dtype=DESC_DTYPE)
    n = len(d)
    out = np.zeros(max(n, 1), DESC_DTYPE)
    gidx = np.zeros(max(n, 1), np.uint64)
    n_own, m = ctypes.c_uint64(0), ctypes.c_uint64(0)
    st = _lib.cg_shard_lists(d.ctypes.data if n else None, n, host_base, host_size, world, rank, out.ctypes.data,
                             gidx.ctypes.data, ctypes.byref(n_own), ctypes.byref(m))
    if st:
        raise CgError(st, "cg_shard_lists")
    k = n_own.value + m.value
    return out[:k], gidx[:k], n_own.value, m.value


class ShardBatch:
    """One batch uploaded for every local rank (device lists, global indices,
    verdict arrays) plus the root's outputs."""

    def __init__(self, group: "ShardGroup", descs: np.ndarray, dense: bool = True):
        torch = group.torch
        self.n = len(descs)
        self.lists = []
        self.keep = []
        for r in group.local_ranks:
            d, gidx, n_own, m = shard_lists(descs, group.host_base, group.host_size, group.world, r)
            dev = torch.device("cuda", group.device)
            dd = torch.from_numpy(d.view(np.uint8).copy()).to(dev) if len(d) else torch.empty(96, dtype=torch.uint8, device=dev)
            dg = torch.from_numpy(gidx.view(np.int64).copy()).to(dev) if len(d) else torch.empty(1, dtype=torch.int64, device=dev)
            dv = torch.empty(max(len(d), 1) * VERDICT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
            self.keep.append((dd, dg, dv))
            self.lists.append((n_own, m))
        self.m = self.lists[0][1]
        B = _ShardBatchC * len(self.lists)
        self.c = B()
        for k, ((n_own, m), (dd, dg, dv)) in enumerate(zip(self.lists, self.keep)):
            self.c[k] = _ShardBatchC(dd.data_ptr(), n_own, m, dg.data_ptr(), dv.data_ptr())
        dev = torch.device("cuda", group.device)
        cap_all = group.world * group.cap
        self.root_idx = torch.empty(cap_all, dtype=torch.int64, device=dev)
        self.root_dirty = torch.empty(cap_all * VERDICT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        self.root_count = torch.zeros(1, dtype=torch.int64, device=dev)
        self.dense = torch.empty(max(self.n, 1) * VERDICT_DTYPE.itemsize, dtype=torch.uint8, device=dev) \
            if dense else None


class _ShardBatchC(ctypes.Structure):
    _fields_ = [("d_descs", ctypes.c_void_p), ("n_own", ctypes.c_uint64), ("m", ctypes.c_uint64),
                ("d_gidx", ctypes.c_void_p), ("d_out", ctypes.c_void_p)]


class ShardGroup:
    """G shards of [host_base, host_base + host_size) with a cg_comm.  backend
    "loopback": all G contexts here (one GPU); "nccl": this process's rank
    (torch.distributed must be initialised; the NCCL id is broadcast over it)."""

    def __init__(self, host_base: int, host_size: int, world: int, *, backend: str = "loopback", rank: int = 0,
                 device: int = 0, max_straddlers: int = 1 << 16, cap: int = 1 << 16, **kw):
        import torch
        if host_size % world or (host_size // world) % 4096:
            raise CgError(1, "shards must be multiples of 4096 bytes")
        if world > 8:
            raise CgError(1, "at most 8 shards")
        self.torch = torch
        self.host_base, self.host_size, self.world, self.device = host_base, host_size, world, device
        self.cap = cap
        self.backend = backend
        shard = host_size // world
        self.local_ranks = list(range(world)) if backend == "loopback" else [rank]
        self.rank = rank
        self.chks = [Checker(host_base, host_size, shard_base=host_base + r * shard, shard_size=shard, device=device,
                             **kw) for r in self.local_ranks]
        comm = ctypes.c_void_p()
        if backend == "loopback":
            arr = (ctypes.c_void_p * world)(*[c.ctx.value for c in self.chks])
            st = _lib.cg_comm_create_loopback(arr, world, max_straddlers, cap, ctypes.byref(comm))
        else:
            import torch.distributed as dist
            nid = torch.zeros(CG_NCCL_ID_BYTES, dtype=torch.uint8)
            if rank == 0:
                buf = (ctypes.c_uint8 * CG_NCCL_ID_BYTES)()
                st = _lib.cg_comm_nccl_id(buf)
                if st:
                    raise CgError(st, "cg_comm_nccl_id")
                nid = torch.from_numpy(np.frombuffer(bytes(buf), np.uint8).copy())
            if dist.get_backend() == "nccl":
                nid = nid.to(torch.device("cuda", device))
            dist.broadcast(nid, 0)
            idb = (ctypes.c_uint8 * CG_NCCL_ID_BYTES)(*nid.cpu().numpy().tolist())
            st = _lib.cg_comm_create_nccl(self.chks[0].ctx, world, rank, idb, max_straddlers, cap, ctypes.byref(comm))
        if st:
            raise CgError(st, "cg_comm_create")
        self.comm = comm

    @property
    def is_root(self) -> bool:
        return self.backend == "loopback" or self.rank == 0

    def close(self):
        if getattr(self, "comm", None):
            _lib.cg_comm_destroy(self.comm)
            self.comm = None
        for c in self.chks:
            c.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def kernel_launches(self) -> int:
        return int(_lib.cg_comm_kernel_launches(self.comm)) + sum(c.kernel_launches for c in self.chks)

    def batch(self, descs: np.ndarray, dense: bool = True) -> ShardBatch:
        return ShardBatch(self, descs, dense)

    def check(self, b: ShardBatch, stream=None):
        """cg_check_sharded: every local rank's part, asynchronous"""
        dense = b.dense.data_ptr() if b.dense is not None else None
        st = _lib.cg_check_sharded(self.comm, b.c, b.root_idx.data_ptr(), b.root_dirty.data_ptr(),
                                   b.root_count.data_ptr(), dense, b.n, _stream_ptr(stream))
        if st:
            raise CgError(st, "cg_check_sharded: " + _lib.cg_comm_last_error(self.comm).decode())

    def overflow(self) -> bool:
        o = ctypes.c_uint32(0)
        st = _lib.cg_comm_overflow(self.comm, ctypes.byref(o))
        if st:
            raise CgError(st, "cg_comm_overflow")
        return bool(o.value)

    def dense(self, b: ShardBatch) -> np.ndarray:
        """the root's dense verdicts of the last check of b (synchronises)"""
        self.torch.cuda.synchronize(self.device)
        assert not self.overflow(), "a rank had more dirty verdicts than cap"
        return b.dense.cpu().numpy().view(VERDICT_DTYPE)[:b.n]

    # ---- setup calls go to every local rank --------------------------------
    def all(self, fn):
        return [fn(c) for c in self.chks]


def replay_sharded(group: ShardGroup, events: np.ndarray, blob=None, fuse: bool = True):
    """Replay a call stream over the shards of a group: setup calls go to every
    local shard, copies are checked with cg_check_sharded in the hazard-free
    batches cg_plan_batches cuts.  Returns (verdicts of the copies, status per
    event) on the root (NCCL: every rank returns its statuses, the verdicts are
    the root's).  fuse is accepted for symmetry: the sharded check is always
    the fused one (CG_APPLY_AFTER planned per rank list)."""
    from .replay import OP_COPY, OP_FREE, OP_FREEA, OP_MARK, OP_REG, OP_REGA, OP_SETV, OP_SYNC, events_to_descs
    ops = np.asarray(events["op"])
    n = len(events)
    status = np.zeros(n, np.uint32)
    is_copy = ops == OP_COPY
    copy_rank = np.cumsum(is_copy) - 1
    verdicts = np.zeros(int(is_copy.sum()), VERDICT_DTYPE)
    i = 0
    while i < n:
        op = ops[i]
        if op == OP_MARK:
            j = i
            while j < n and ops[j] == OP_MARK:
                j += 1
            m = np.zeros(j - i, MARK_DTYPE)
            m["addr"], m["len"], m["state"] = events["dst"][i:j], events["width"][i:j], events["kind"][i:j]
            sts = []
            for c in group.chks:
                s_ = np.zeros(j - i, np.uint32)
                c.host_mark_batch(m, status_out=s_)
                sts.append(s_)
            status[i:j] = sts[0]
            i = j
        elif op == OP_SETV:
            off, ln = int(events["src"][i]), int(events["width"][i])
            addr = int(events["dst"][i])
            # all-or-nothing across shards: every shard must hold only addressable bytes of it
            ok = all(c.host_query_addressable(addr, ln) for c in group.chks)
            if group.backend == "nccl":
                t = group.torch.tensor([0 if ok else 1], dtype=group.torch.int32,
                                       device=group.torch.device("cuda", group.device))
                import torch.distributed as dist
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                ok = int(t.item()) == 0
            status[i] = max(c.host_set_vbits(addr, bytes(blob[off:off + ln])) for c in group.chks) if ok else 1
            i += 1
        else:
            j = i
            while j < n and ops[j] in (OP_REG, OP_FREE, OP_COPY, OP_REGA, OP_FREEA, OP_SYNC):   # SYNC: NEXT-2 only
                j += 1
            if j == i:   # an unknown op: invalid call, like the oracle's replay
                status[i] = 1
                i += 1
                continue
            for k in range(i, j):
                e = events[k]
                if ops[k] == OP_REG:
                    status[k] = group.all(lambda c: c.register_alloc(int(e["dst"]), int(e["width"]), int(e["seq"])))[0]
                elif ops[k] == OP_FREE:
                    status[k] = group.all(lambda c: c.free(int(e["dst"]), int(e["seq"])))[0]
                elif ops[k] == OP_REGA:   # NEXT-3 arrays are replicated like allocations
                    status[k] = group.all(lambda c: c.register_array(int(e["dst"]), int(e["width"]), int(e["height"]),
                                                                     int(e["dst_x"]), int(e["dst_y"]),
                                                                     int(e["dst_pitch"]), int(e["seq"])))[0]
                elif ops[k] == OP_FREEA:
                    status[k] = group.all(lambda c: c.free_array(int(e["dst"]), int(e["seq"])))[0]
            idx = np.flatnonzero(is_copy[i:j]) + i
            if len(idx):
                descs = events_to_descs(events[idx])
                cuts = [0] + [int(c) for c in plan_batches(descs)]
                for a, b in zip(cuts[:-1], cuts[1:]):
                    if b <= a:
                        continue
                    batch = group.batch(descs[a:b])
                    group.check(batch)
                    if group.is_root:
                        v = group.dense(batch)
                        verdicts[copy_rank[idx[a:b]]] = v
                        status[idx[a:b]] = v["status"]
            i = j
    group.torch.cuda.synchronize(group.device)
    return verdicts, status
