"""B200-native batched Cudagrind transfer checker (arXiv 1310.0901).

Thin Python binding over the C-ABI library ``libcgcheck.so`` (include/cg.h).
Functions keep the C names (``cg_check_copies`` ...) and only marshal
arguments; every step of the check runs in the library's sm_100a kernels.
PyTorch provides device memory (the shadow store and workspace are torch
tensors) and streams.

There is no CPU fallback: importing this package without the built library
raises.  Build it with ``python -m paper_1310_0901_b200.build`` (or
``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcgcheck.so")

# ---- ABI constants (include/cg.h) -----------------------------------------
CG_OK, CG_ERR_INVALID_VALUE, CG_ERR_INVALID_CONTEXT, CG_ERR_OUT_OF_MEMORY = 0, 1, 2, 3
CG_ERR_NOT_INITIALIZED, CG_ERR_CUDA, CG_ERR_NCCL = 4, 5, 6
CG_HTOD, CG_DTOH, CG_DTOD, CG_HTOA, CG_ATOH = 1, 2, 3, 4, 5
CG_NOACCESS, CG_UNDEFINED, CG_DEFINED = 0, 1, 2
CG_NONE = (1 << 64) - 1
CG_F_DST_NOT_ALLOCATED = 1 << 0
CG_F_DST_TOO_SMALL = 1 << 1
CG_F_SRC_NOT_ALLOCATED = 1 << 2
CG_F_SRC_TOO_SMALL = 1 << 3
CG_F_HOST_UNADDRESSABLE = 1 << 4
CG_F_HOST_UNDEFINED = 1 << 5
CG_F_BAD_PITCH = 1 << 6
CG_F_INVALID_RANGE = 1 << 7
CG_F_BAD_KIND = 1 << 8
CG_F_CONCURRENT = 1 << 9

DESC_DTYPE = np.dtype([
    ("kind", "<u4"), ("reserved", "<u4"), ("seq", "<u8"), ("width", "<u8"), ("height", "<u8"),
    ("dst", "<u8"), ("dst_x", "<u8"), ("dst_y", "<u8"), ("dst_pitch", "<u8"),
    ("src", "<u8"), ("src_x", "<u8"), ("src_y", "<u8"), ("src_pitch", "<u8"),
])
VERDICT_DTYPE = np.dtype([
    ("first_unaddr", "<u8"), ("first_undef", "<u8"), ("undef_count", "<u8"),
    ("dst_expected", "<u8"), ("dst_found", "<u8"), ("src_expected", "<u8"), ("src_found", "<u8"),
    ("flags", "<u4"), ("status", "<u4"),
])
ALLOC_RECORD_DTYPE = np.dtype([("base", "<u8"), ("size", "<u8"), ("alloc_seq", "<u8")])
MARK_DTYPE = np.dtype([("addr", "<u8"), ("len", "<u8"), ("state", "<u4"), ("reserved", "<u4")])
assert DESC_DTYPE.itemsize == 96 and VERDICT_DTYPE.itemsize == 64
assert ALLOC_RECORD_DTYPE.itemsize == 24 and MARK_DTYPE.itemsize == 24


class cg_config(ctypes.Structure):
    _fields_ = [
        ("host_base", ctypes.c_uint64), ("host_size", ctypes.c_uint64),
        ("shard_base", ctypes.c_uint64), ("shard_size", ctypes.c_uint64),
        ("max_descs", ctypes.c_uint64), ("max_allocs", ctypes.c_uint64),
        ("undef_is_error", ctypes.c_uint32), ("host_staging", ctypes.c_uint32),
        ("device", ctypes.c_int32), ("shadow_format", ctypes.c_int32),
        ("v_buf", ctypes.c_void_p), ("a_buf", ctypes.c_void_p), ("workspace", ctypes.c_void_p),
        ("workspace_size", ctypes.c_uint64),
        ("dev_vbuf", ctypes.c_void_p), ("dev_vsize", ctypes.c_uint64),
    ]


class CgError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"cg status {status}: {msg}")
        self.status = status


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_1310_0901_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P, U64, U32, I = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int
    sig = {
        "cg_workspace_size": (U64, [P]),
        "cg_ctx_create": (I, [P, P]),
        "cg_ctx_destroy": (I, [P]),
        "cg_last_error": (ctypes.c_char_p, [P]),
        "cg_host_mark": (I, [P, U64, U64, U32, P]),
        "cg_host_mark_batch": (I, [P, P, U64, P, P]),
        "cg_host_set_vbits": (I, [P, U64, U64, P, P]),
        "cg_register_alloc": (I, [P, U64, U64, U64]),
        "cg_free": (I, [P, U64, U64]),
        "cg_registry_compact": (I, [P, U64]),
        "cg_check_copies": (I, [P, P, U64, P, P]),
        "cg_apply_dtoh": (I, [P, P, P, U64, P]),
        "cg_check_copies_host": (I, [P, P, U64, P, I, P]),
        "cg_check_apply": (I, [P, P, U64, P, P]),
        "cg_straddler_pack": (I, [P, P, U64, P, P, P, P]),
        "cg_straddler_finalize": (I, [P, P, P, P, U64, P, P]),
        "cg_compact_dirty": (I, [P, P, U64, P, P, P, P]),
        "cg_host_query_addressable": (I, [P, U64, U64, P, P]),
        "cg_expand_copy1d": (I, [P, P, U64, P, P]),
        "cg_check_host": (I, [P, P, U32, U64, I, P, P, U64, P, P]),
        "cg_check_host_submit": (I, [P, P, U32, U64, I, U32, P]),
        "cg_check_host_wait": (I, [P, U32, P, P, U64, P]),
        "cg_format_verdict": (U64, [P, U32, P, U64]),
        "cg_apply_copies": (I, [P, P, P, U64, P]),
        "cg_device_vbits": (I, [P, U64, U64, P]),
        "cg_array_vbits": (I, [P, U64, U64, U64, P]),
        "cg_plan_batches_propagate": (I, [P, U64, P, P]),
        "cg_format_leak": (U64, [P, P, U64]),
        "cg_shard_plan": (I, [P, U64, U64, U64, U32, P, P, P]),
        "cg_batch_disjoint": (I, [P, U64, P]),
        "cg_plan_apply_after": (I, [P, U64, P]),
        "cg_leak_sweep": (I, [P, P, U64, P, P]),
        "cg_leak_report": (I, [P, P, U64, P]),
        "cg_plan_batches": (I, [P, U64, P, P]),
        "cg_plan_batches_fused": (I, [P, U64, P, P]),
        "cg_kernel_launches": (U64, [P]),
        "cg_profile_begin": (I, [P]),
        "cg_profile_end": (I, [P, P, P]),
        "cg_array_bytes": (U64, [U64, U64, U64, U32, U32]),
        "cg_register_array": (I, [P, U64, U64, U64, U64, U32, U32, U64]),
        "cg_free_array": (I, [P, U64, U64]),
        "cg_array_report": (I, [P, P, U64, P]),
        "cg_host_shadow_read": (I, [P, U64, U64, P, P, P]),
        "cg_apply_copies_subset": (I, [P, P, P, U64, P, U64, U64, P]),
        "cg_plan_waves": (I, [P, U64, P, P]),
        "cg_apply_flush": (I, [P, P]),
        "cg_apply_copies_waves": (I, [P, P, P, U64, P, P, P, U32, P]),
        "cg_summarize": (I, [P, U64, U32, P, P]),
        "cg_format_summary": (U64, [U64, U64, U64, P, U64]),
        "cg_conc_create": (I, [I, U64, U64, P]),
        "cg_conc_destroy": (I, [P]),
        "cg_conc_last_error": (ctypes.c_char_p, [P]),
        "cg_conc_sync": (I, [P, U32, U64]),
        "cg_conc_check": (I, [P, P, P, U64, P, P]),
        "cg_conc_stamps": (I, [P, P, P]),
        "cg_conc_kernel_launches": (U64, [P]),
        "cg_ctx_device": (I, [P]),
        "cg_comm_nccl_id": (I, [P]),
        "cg_comm_create_nccl": (I, [P, U32, U32, P, U64, U64, P]),
        "cg_comm_create_loopback": (I, [P, U32, U64, U64, P]),
        "cg_comm_destroy": (I, [P]),
        "cg_comm_last_error": (ctypes.c_char_p, [P]),
        "cg_comm_kernel_launches": (U64, [P]),
        "cg_comm_overflow": (I, [P, P]),
        "cg_check_sharded": (I, [P, P, P, P, P, P, U64, P]),
        "cg_shard_lists": (I, [P, U64, U64, U64, U32, U32, P, P, P, P]),
        "cg_registry_batch": (I, [P, P, U64, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_lib = _load()
EXPORTED = ("cg_workspace_size", "cg_ctx_create", "cg_ctx_destroy", "cg_last_error", "cg_host_mark",
            "cg_host_mark_batch", "cg_host_set_vbits", "cg_register_alloc", "cg_free", "cg_registry_compact",
            "cg_check_copies", "cg_apply_dtoh", "cg_check_copies_host", "cg_leak_sweep", "cg_leak_report",
            "cg_plan_batches", "cg_kernel_launches", "cg_profile_begin", "cg_profile_end", "cg_check_apply",
            "cg_batch_disjoint", "cg_plan_apply_after", "cg_straddler_pack", "cg_straddler_finalize", "cg_compact_dirty", "cg_shard_plan",
            "cg_host_query_addressable", "cg_expand_copy1d", "cg_check_host", "cg_check_host_submit", "cg_check_host_wait", "cg_format_verdict",
            "cg_format_leak", "cg_apply_copies", "cg_device_vbits", "cg_array_vbits", "cg_plan_batches_propagate",
            "cg_host_shadow_read", "cg_apply_copies_subset", "cg_plan_waves", "cg_apply_flush", "cg_apply_copies_waves", "cg_summarize", "cg_format_summary", "cg_array_bytes", "cg_register_array", "cg_free_array", "cg_array_report", "cg_conc_create",
            "cg_conc_destroy", "cg_conc_last_error", "cg_conc_sync", "cg_conc_check", "cg_conc_stamps",
            "cg_conc_kernel_launches", "cg_ctx_device", "cg_comm_nccl_id", "cg_comm_create_nccl",
            "cg_comm_create_loopback", "cg_comm_destroy", "cg_comm_last_error", "cg_comm_kernel_launches",
            "cg_comm_overflow", "cg_check_sharded", "cg_shard_lists", "cg_registry_batch",
            "cg_plan_batches_fused")

# ---- same-name thin wrappers of every exported function (status codes returned unchanged) ----
globals().update({_n: getattr(_lib, _n) for _n in EXPORTED})

# ---- constants of include/cg.h and the numpy views of its records ----
CG_SHADOW_BYTES, CG_SHADOW_2BIT, CG_SHADOW_SPARSE = 0, 1, 2
CG_FMT_2D, CG_FMT_1D = 0, 1
COPY1D_DTYPE = np.dtype([("kind", "<u4"), ("reserved", "<u4"), ("seq", "<u8"), ("dst", "<u8"), ("src", "<u8"),
                         ("bytes", "<u8")])
CG_SHARD_NOT_OWNER, CG_SHARD_RAW, CG_APPLY_AFTER, CG_CHECK_AFTER, CG_APPLY_LAST = 1, 2, 4, 8, 16
CG_COMM_NCCL, CG_COMM_LOOPBACK = 0, 1
CG_NCCL_ID_BYTES = 128
CG_REG_ALLOC, CG_REG_FREE = 1, 2
REG_EVENT_DTYPE = np.dtype([("op", "<u4"), ("reserved", "<u4"), ("seq", "<u8"), ("addr", "<u8"), ("size", "<u8")])
STAGES = ("check_prep", "check_plan", "check_scan", "check_finalize", "apply_prep", "apply_plan", "apply",
          "leak_sweep")


class Waves:
    """NEXT-1 propagation waves of one checked batch, uploaded once: the
    concatenated device index lists plus host offsets / largest copy per wave
    (for cg_apply_copies_waves)."""

    def __init__(self, descs: np.ndarray, device: int = 0):
        import torch
        lev, nl = plan_waves(descs)
        order = np.argsort(lev, kind="stable").astype(np.uint32)
        self.start = np.searchsorted(lev[order], np.arange(nl + 1)).astype(np.uint64)
        nb = descs["width"].astype(np.uint64) * descs["height"].astype(np.uint64)
        self.max_bytes = np.array([int(nb[order[self.start[w]:self.start[w + 1]]].max())
                                   if self.start[w + 1] > self.start[w] else 0 for w in range(nl)], np.uint64)
        self.index = torch.from_numpy(order.astype(np.int32)).to(torch.device("cuda", device))
        self.n_waves = nl


def summarize(d_verdicts, undef_is_error: bool = False, stream=None):
    """NEXT-4: (errors, warnings) of the verdicts in a CUDA uint8 tensor"""
    import torch
    n = d_verdicts.numel() // VERDICT_DTYPE.itemsize
    out = torch.zeros(2, dtype=torch.int64, device=d_verdicts.device)
    st = _lib.cg_summarize(d_verdicts.data_ptr(), n, int(undef_is_error), out.data_ptr(), _stream_ptr(stream))
    if st:
        raise CgError(st, "cg_summarize")
    e, w = out.cpu().tolist()
    return int(e), int(w)


def format_summary(errors: int, warnings: int, suppressed: int = 0) -> str:
    k = _lib.cg_format_summary(errors, warnings, suppressed, None, 0)
    buf = ctypes.create_string_buffer(k + 1)
    _lib.cg_format_summary(errors, warnings, suppressed, buf, k + 1)
    return buf.value.decode()


def format_verdict(v, kind: int) -> str:
    """Diagnostic text of one verdict (cg_format_verdict; Listing 5 style)."""
    a = np.ascontiguousarray(np.asarray(v, dtype=VERDICT_DTYPE).reshape(1))
    need = _lib.cg_format_verdict(a.ctypes.data, int(kind), None, 0)
    buf = ctypes.create_string_buffer(need + 1)
    _lib.cg_format_verdict(a.ctypes.data, int(kind), buf, need + 1)
    return buf.value.decode()


def format_leak(rec) -> str:
    a = np.ascontiguousarray(np.asarray(rec, dtype=ALLOC_RECORD_DTYPE).reshape(1))
    buf = ctypes.create_string_buffer(128)
    _lib.cg_format_leak(a.ctypes.data, buf, 128)
    return buf.value.decode()


def plan_batches(descs: np.ndarray, propagate: bool = False) -> np.ndarray:
    """Batch end indices (cg_plan_batches, or cg_plan_batches_propagate for
    device V-bit tracking) for a host DESC_DTYPE array."""
    d = np.ascontiguousarray(descs, dtype=DESC_DTYPE)
    cuts = np.zeros(max(len(d), 1), np.uint64)
    nc = ctypes.c_uint64(0)
    fn = _lib.cg_plan_batches_propagate if propagate else _lib.cg_plan_batches
    st = fn(d.ctypes.data if len(d) else None, len(d), cuts.ctypes.data, ctypes.byref(nc))
    if st:
        raise CgError(st, "cg_plan_batches")
    return cuts[: nc.value]


def plan_waves(descs: np.ndarray):
    """cg_plan_waves: (level per descriptor, number of levels) for NEXT-1
    propagation of a batch whose copies touch each other's bytes."""
    d = np.ascontiguousarray(descs, dtype=DESC_DTYPE)
    lev = np.zeros(max(len(d), 1), np.uint32)
    nl = ctypes.c_uint32(0)
    st = _lib.cg_plan_waves(d.ctypes.data if len(d) else None, len(d), lev.ctypes.data, ctypes.byref(nl))
    if st:
        raise CgError(st, "cg_plan_waves")
    return lev[:len(d)], int(nl.value)


def wave_indices(levels: np.ndarray, n_levels: int, descs: Optional[np.ndarray] = None):
    """per level, the (uint32) indices of its descriptors in batch order; with
    descs, (indices, largest width*height) pairs for cg_apply_copies_subset"""
    order = np.argsort(levels, kind="stable").astype(np.uint32)
    bounds = np.searchsorted(levels[order], np.arange(n_levels + 1))
    waves = [order[bounds[w]:bounds[w + 1]] for w in range(n_levels)]
    if descs is None:
        return waves
    nb = descs["width"].astype(np.uint64) * descs["height"].astype(np.uint64)
    return [(w, int(nb[w].max()) if len(w) else 0) for w in waves]


def batch_disjoint(descs: np.ndarray) -> bool:
    """cg_batch_disjoint: no HtoD host range overlaps any DtoH host range."""
    d = np.ascontiguousarray(descs, dtype=DESC_DTYPE)
    out = ctypes.c_int(0)
    st = _lib.cg_batch_disjoint(d.ctypes.data if len(d) else None, len(d), ctypes.byref(out))
    if st:
        raise CgError(st, "cg_batch_disjoint")
    return bool(out.value)


def plan_batches_fused(descs: np.ndarray) -> np.ndarray:
    """cg_plan_batches_fused: batch end indices for cg_check_apply, setting
    CG_CHECK_AFTER / CG_APPLY_AFTER / CG_APPLY_LAST in place (descs: contiguous DESC_DTYPE)"""
    assert descs.dtype == DESC_DTYPE and descs.flags["C_CONTIGUOUS"]
    cuts = np.zeros(max(len(descs), 1), np.uint64)
    nc = ctypes.c_uint64(0)
    st = _lib.cg_plan_batches_fused(descs.ctypes.data if len(descs) else None, len(descs), cuts.ctypes.data,
                                    ctypes.byref(nc))
    if st:
        raise CgError(st, "cg_plan_batches_fused")
    return cuts[: nc.value]


def plan_apply_after(descs: np.ndarray) -> int:
    """cg_plan_apply_after: sets CG_APPLY_AFTER (in place) on the DtoH
    descriptors whose host range overlaps an HtoD host range of the batch, so
    that cg_check_apply is exact on any R-20 epoch; returns how many."""
    assert descs.dtype == DESC_DTYPE and descs.flags["C_CONTIGUOUS"]
    out = ctypes.c_uint64(0)
    st = _lib.cg_plan_apply_after(descs.ctypes.data if len(descs) else None, len(descs), ctypes.byref(out))
    if st:
        raise CgError(st, "cg_plan_apply_after")
    return int(out.value)


def shard_plan(descs: np.ndarray, host_base: int, host_size: int, world: int):
    """cg_shard_plan: (owner, first shard, last shard) per descriptor."""
    d = np.ascontiguousarray(descs, dtype=DESC_DTYPE)
    owner, first, last = (np.zeros(len(d), np.uint32) for _ in range(3))
    st = _lib.cg_shard_plan(d.ctypes.data if len(d) else None, len(d), host_base, host_size, world,
                            owner.ctypes.data, first.ctypes.data, last.ctypes.data)
    if st:
        raise CgError(st, "cg_shard_plan")
    return owner, first, last


def _stream_ptr(stream) -> Optional[int]:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


class Checker:
    """One context (one GPU, one shard of the host window).

    Device memory -- the V/A shadow store and the workspace -- are torch
    tensors owned by this object; the library only borrows them.
    """

    def __init__(self, host_base: int, host_size: int, *, max_descs: int = 1 << 20,
                 max_allocs: int = 1 << 18, undef_is_error: bool = False, device: int = 0,
                 shard_base: int = 0, shard_size: int = 0, host_staging: bool = False, dev_vsize: int = 0,
                 shadow_format: int = 0, sparse_capacity: int = 0):
        """shadow_format CG_SHADOW_SPARSE: the library map covers the whole
        64-bit host space with room for sparse_capacity host bytes (default:
        host_size + 128 KiB, rounded to 64 KiB); host_base / host_size then
        only name the window shadow() reads back."""
        import torch
        self.torch = torch
        self.device = device
        dev = torch.device("cuda", device)
        ss = shard_size or host_size
        self.sparse = shadow_format == CG_SHADOW_SPARSE
        self.view = (host_base, host_size)
        if self.sparse:
            cap = sparse_capacity or host_size + (128 << 10)
            cap = (cap + 65535) // 65536 * 65536
            host_base, host_size, shard_base, shard_size = 0, cap, 0, 0
        self.cfg = cg_config(host_base=host_base, host_size=host_size, shard_base=shard_base,
                             shard_size=shard_size, max_descs=max_descs, max_allocs=max_allocs,
                             undef_is_error=int(undef_is_error), host_staging=int(host_staging),
                             device=device, shadow_format=shadow_format)
        self.two_bit = shadow_format in (CG_SHADOW_2BIT, CG_SHADOW_SPARSE)
        self.shard_base = shard_base if shard_size else host_base
        self.shard_size = ss
        if self.sparse:
            self.shard_base, self.shard_size = self.view
        self.tracking = dev_vsize > 0
        if self.tracking:   # NEXT-1 device V-bit pool
            dev_vsize = (dev_vsize + 15) // 16 * 16
            self.dev_v = torch.empty(dev_vsize, dtype=torch.uint8, device=dev)
            self.cfg.dev_vbuf = self.dev_v.data_ptr()
            self.cfg.dev_vsize = dev_vsize
        ws = _lib.cg_workspace_size(ctypes.byref(self.cfg))
        if ws == 0:
            raise CgError(CG_ERR_INVALID_VALUE, "invalid configuration")
        if self.sparse:    # NEXT-4: secondaries of 16 KiB states, the first one distinguished
            self.V = torch.empty((host_size // 65536 + 1) * 16384, dtype=torch.uint8, device=dev)
            self.A = None
        elif self.two_bit:   # NEXT-4: 2-bit states, shard/4 bytes; no A bitmap
            self.V = torch.empty(ss // 4, dtype=torch.uint8, device=dev)
            self.A = None
        else:
            self.V = torch.empty(ss, dtype=torch.uint8, device=dev)
            self.A = torch.empty(ss // 8, dtype=torch.uint8, device=dev)
        self.workspace = torch.empty(ws, dtype=torch.uint8, device=dev)
        self.cfg.v_buf = self.V.data_ptr()
        self.cfg.a_buf = self.A.data_ptr() if self.A is not None else None
        self.cfg.workspace = self.workspace.data_ptr()
        self.cfg.workspace_size = ws
        ctx = ctypes.c_void_p()
        st = _lib.cg_ctx_create(ctypes.byref(self.cfg), ctypes.byref(ctx))
        if st:
            raise CgError(st, "cg_ctx_create failed")
        self.ctx = ctx
        self.max_descs = max_descs
        self.max_allocs = max_allocs

    def close(self):
        if getattr(self, "ctx", None):
            _lib.cg_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _ok(self, st: int, what: str):
        if st:
            raise CgError(st, f"{what}: {_lib.cg_last_error(self.ctx).decode()}")

    @property
    def kernel_launches(self) -> int:
        return int(_lib.cg_kernel_launches(self.ctx))

    # ---- host shadow plumbing ---------------------------------------------
    def host_mark(self, addr: int, length: int, state: int, stream=None) -> int:
        return _lib.cg_host_mark(self.ctx, addr, length, state, _stream_ptr(stream))

    def host_mark_batch(self, marks: np.ndarray, status_out: Optional[np.ndarray] = None, stream=None) -> int:
        m = np.ascontiguousarray(marks, dtype=MARK_DTYPE)
        if status_out is not None:
            assert status_out.dtype == np.uint32 and status_out.flags.c_contiguous and len(status_out) >= len(m)
        return _lib.cg_host_mark_batch(self.ctx, m.ctypes.data if len(m) else None, len(m),
                                       status_out.ctypes.data if status_out is not None else None,
                                       _stream_ptr(stream))

    def host_set_vbits(self, addr: int, vbytes: bytes, stream=None) -> int:
        b = np.ascontiguousarray(np.frombuffer(bytes(vbytes), np.uint8))
        return _lib.cg_host_set_vbits(self.ctx, addr, len(b), b.ctypes.data if len(b) else None,
                                      _stream_ptr(stream))

    def host_query_addressable(self, addr: int, length: int, stream=None) -> bool:
        out = ctypes.c_uint32(0)
        self._ok(_lib.cg_host_query_addressable(self.ctx, addr, length, ctypes.byref(out), _stream_ptr(stream)),
                 "cg_host_query_addressable")
        return bool(out.value)

    # ---- registry ------------------------------------------------------------
    def register_alloc(self, base: int, size: int, seq: int) -> int:
        return _lib.cg_register_alloc(self.ctx, base, size, seq)

    def registry_batch(self, events: np.ndarray, status_out: Optional[np.ndarray] = None) -> int:
        """cg_registry_batch over REG_EVENT_DTYPE records"""
        e = np.ascontiguousarray(events, dtype=REG_EVENT_DTYPE)
        st = status_out if status_out is not None else None
        return _lib.cg_registry_batch(self.ctx, e.ctypes.data if len(e) else None, len(e),
                                      st.ctypes.data if st is not None else None)

    def registry_compact(self, before_seq: int) -> int:
        """cg_registry_compact: drop tombstones no descriptor with seq >= before_seq can see"""
        return _lib.cg_registry_compact(self.ctx, before_seq)

    def free(self, ptr: int, seq: int) -> int:
        return _lib.cg_free(self.ctx, ptr, seq)

    def register_array(self, handle: int, width: int, height: int, depth: int, fmt: int, channels: int,
                       seq: int) -> int:
        """NEXT-3 cg_register_array (cuArrayCreate / cuArray3DCreate)."""
        return _lib.cg_register_array(self.ctx, handle, width, height, depth, fmt, channels, seq)

    def free_array(self, handle: int, seq: int) -> int:
        return _lib.cg_free_array(self.ctx, handle, seq)

    def array_report(self) -> np.ndarray:
        """live arrays {handle, total bytes, alloc_seq}, ascending handle"""
        n = ctypes.c_uint64(0)
        self._ok(_lib.cg_array_report(self.ctx, None, 0, ctypes.byref(n)), "cg_array_report")
        out = np.zeros(n.value, ALLOC_RECORD_DTYPE)
        if n.value:
            self._ok(_lib.cg_array_report(self.ctx, out.ctypes.data, n.value, ctypes.byref(n)), "cg_array_report")
        return out

    # ---- the hot path --------------------------------------------------------
    def check_copies(self, d_descs, d_out=None, stream=None):
        """d_descs: a CUDA uint8 tensor holding n DESC_DTYPE records."""
        torch = self.torch
        n = d_descs.numel() // DESC_DTYPE.itemsize
        if d_out is None:
            d_out = torch.empty(n * VERDICT_DTYPE.itemsize, dtype=torch.uint8, device=d_descs.device)
        self._ok(_lib.cg_check_copies(self.ctx, d_descs.data_ptr(), n, d_out.data_ptr(), _stream_ptr(stream)),
                 "cg_check_copies")
        return d_out

    def apply_copies(self, d_descs, d_verdicts, index=None, max_bytes: int = 0, stream=None):
        """cg_apply_copies: the a6 step (V-bit propagation with tracking);
        with index (a CUDA uint32/int32 tensor of descriptor indices) only that
        subset (cg_apply_copies_subset, one wave of cg_plan_waves)."""
        n = d_descs.numel() // DESC_DTYPE.itemsize
        if index is None:
            self._ok(_lib.cg_apply_copies(self.ctx, d_descs.data_ptr(), d_verdicts.data_ptr(), n,
                                          _stream_ptr(stream)), "cg_apply_copies")
        else:
            self._ok(_lib.cg_apply_copies_subset(self.ctx, d_descs.data_ptr(), d_verdicts.data_ptr(), n,
                                                 index.data_ptr(), index.numel(), max_bytes, _stream_ptr(stream)),
                     "cg_apply_copies_subset")

    def apply_waves(self, d_descs, d_verdicts, waves: "Waves", stream=None):
        """cg_apply_copies_waves: every wave of the batch, in order, one call"""
        n = d_descs.numel() // DESC_DTYPE.itemsize
        self._ok(_lib.cg_apply_copies_waves(self.ctx, d_descs.data_ptr(), d_verdicts.data_ptr(), n,
                                            waves.index.data_ptr(), waves.start.ctypes.data,
                                            waves.max_bytes.ctypes.data, waves.n_waves, _stream_ptr(stream)),
                 "cg_apply_copies_waves")

    def apply_flush(self, stream=None):
        """cg_apply_flush: sync, report a staging overflow of the subset calls"""
        self._ok(_lib.cg_apply_flush(self.ctx, _stream_ptr(stream)), "cg_apply_flush")

    def device_vbits(self, addr: int, length: int) -> np.ndarray:
        out = np.zeros(max(length, 1), np.uint8)
        self.torch.cuda.synchronize(self.device)
        self._ok(_lib.cg_device_vbits(self.ctx, addr, length, out.ctypes.data), "cg_device_vbits")
        return out[:length]

    def array_vbits(self, handle: int, offset: int, length: int) -> np.ndarray:
        out = np.zeros(max(length, 1), np.uint8)
        self.torch.cuda.synchronize(self.device)
        self._ok(_lib.cg_array_vbits(self.ctx, handle, offset, length, out.ctypes.data), "cg_array_vbits")
        return out[:length]

    def check_apply(self, d_descs, d_out=None, stream=None):
        """cg_check_apply (fused check + DtoH apply; needs a disjoint batch)."""
        torch = self.torch
        n = d_descs.numel() // DESC_DTYPE.itemsize
        if d_out is None:
            d_out = torch.empty(n * VERDICT_DTYPE.itemsize, dtype=torch.uint8, device=d_descs.device)
        self._ok(_lib.cg_check_apply(self.ctx, d_descs.data_ptr(), n, d_out.data_ptr(), _stream_ptr(stream)),
                 "cg_check_apply")
        return d_out

    def apply_dtoh(self, d_descs, d_verdicts, stream=None):
        n = d_descs.numel() // DESC_DTYPE.itemsize
        self._ok(_lib.cg_apply_dtoh(self.ctx, d_descs.data_ptr(), d_verdicts.data_ptr(), n, _stream_ptr(stream)),
                 "cg_apply_dtoh")

    def check_copies_host(self, descs: np.ndarray, out: Optional[np.ndarray] = None, apply: int = 1,
                          stream=None) -> np.ndarray:
        """apply: 0 check only, 1 check + apply, 2 fused cg_check_apply."""
        d = np.ascontiguousarray(descs, dtype=DESC_DTYPE)
        if out is None:
            out = np.empty(len(d), VERDICT_DTYPE)
        self._ok(_lib.cg_check_copies_host(self.ctx, d.ctypes.data, len(d), out.ctypes.data, int(apply),
                                           _stream_ptr(stream)), "cg_check_copies_host")
        return out

    def check_host(self, descs: np.ndarray, apply: int = 1, cap: Optional[int] = None, stream=None):
        """cg_check_host: host descriptors (DESC_DTYPE or COPY1D_DTYPE) in,
        dirty verdicts out.  Returns (n_dirty, idx, dirty verdicts)."""
        fmt = CG_FMT_1D if descs.dtype == COPY1D_DTYPE else CG_FMT_2D
        n = len(descs)
        cap = n if cap is None else cap
        idx = np.empty(max(cap, 1), np.uint64)
        dirty = np.empty(max(cap, 1), VERDICT_DTYPE)
        nd = ctypes.c_uint64(0)
        self._ok(_lib.cg_check_host(self.ctx, descs.ctypes.data, fmt, n, int(apply), idx.ctypes.data,
                                    dirty.ctypes.data, cap, ctypes.byref(nd), _stream_ptr(stream)), "cg_check_host")
        m = min(nd.value, cap)
        return nd.value, idx[:m], dirty[:m]

    def check_host_submit(self, descs: np.ndarray, slot: int, apply: int = 1, stream=None):
        """cg_check_host_submit: enqueue a host batch into staging slot 0/1
        (descs must stay alive and unchanged until check_host_wait(slot))"""
        fmt = CG_FMT_1D if descs.dtype == COPY1D_DTYPE else CG_FMT_2D
        self._ok(_lib.cg_check_host_submit(self.ctx, descs.ctypes.data, fmt, len(descs), int(apply), int(slot),
                                           _stream_ptr(stream)), "cg_check_host_submit")

    def check_host_wait(self, slot: int, cap: int):
        """cg_check_host_wait: (n_dirty, idx, dirty verdicts) of the slot's batch"""
        idx = np.empty(max(cap, 1), np.uint64)
        dirty = np.empty(max(cap, 1), VERDICT_DTYPE)
        nd = ctypes.c_uint64(0)
        self._ok(_lib.cg_check_host_wait(self.ctx, int(slot), idx.ctypes.data, dirty.ctypes.data, cap,
                                         ctypes.byref(nd)), "cg_check_host_wait")
        m = min(nd.value, cap)
        return nd.value, idx[:m], dirty[:m]

    def leak_sweep(self, d_out, cap: int, d_count, stream=None):
        self._ok(_lib.cg_leak_sweep(self.ctx, d_out.data_ptr(), cap, d_count.data_ptr(), _stream_ptr(stream)),
                 "cg_leak_sweep")

    def leak_report(self) -> np.ndarray:
        n = ctypes.c_uint64(0)
        self._ok(_lib.cg_leak_report(self.ctx, None, 0, ctypes.byref(n)), "cg_leak_report")
        out = np.zeros(n.value, ALLOC_RECORD_DTYPE)
        if n.value:
            self._ok(_lib.cg_leak_report(self.ctx, out.ctypes.data, n.value, ctypes.byref(n)), "cg_leak_report")
        return out

    # ---- instrumentation -----------------------------------------------------
    def profile_begin(self):
        self._ok(_lib.cg_profile_begin(self.ctx), "cg_profile_begin")

    def profile_end(self) -> dict:
        ms = np.zeros(len(STAGES), np.float64)
        n = np.zeros(len(STAGES), np.uint64)
        self._ok(_lib.cg_profile_end(self.ctx, ms.ctypes.data, n.ctypes.data), "cg_profile_end")
        return {s: (float(ms[i]), int(n[i])) for i, s in enumerate(STAGES)}

    # ---- state download (tests) ---------------------------------------------
    def shadow(self):
        """(packed A bits, V bytes) of the whole shard in the bytes-format layout"""
        self.torch.cuda.synchronize(self.device)
        if not self.two_bit:
            return self.A.cpu().numpy(), self.V.cpu().numpy()
        a, v = self.shadow_read(self.shard_base, self.shard_size)
        return np.packbits(a, bitorder="little"), v

    def shadow_read(self, addr: int, length: int, stream=None):
        """cg_host_shadow_read: (addressable 0/1 per byte, V byte per byte)"""
        a = np.zeros(max(length, 1), np.uint8)
        v = np.zeros(max(length, 1), np.uint8)
        self._ok(_lib.cg_host_shadow_read(self.ctx, addr, length, a.ctypes.data, v.ctypes.data, _stream_ptr(stream)),
                 "cg_host_shadow_read")
        return a[:length], v[:length]


class ConcChecker:
    """NEXT-2 concurrency checker (cg_conc_*): owns its device memory."""

    def __init__(self, max_n: int, max_stamps: int, device: int = 0):
        import torch
        self.torch = torch
        self.device = device
        self.max_n = max_n
        h = ctypes.c_void_p()
        st = _lib.cg_conc_create(device, max_n, max_stamps, ctypes.byref(h))
        if st:
            raise CgError(st, "cg_conc_create")
        self.h = h

    def close(self):
        if self.h:
            _lib.cg_conc_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _ok(self, st: int, what: str):
        if st:
            raise CgError(st, f"{what}: {_lib.cg_conc_last_error(self.h).decode()}")

    def sync(self, thread: int, seq: int):
        self._ok(_lib.cg_conc_sync(self.h, thread, seq), "cg_conc_sync")

    def check(self, d_descs, d_threads, d_verdicts, stream=None):
        """d_descs: CUDA uint8 tensor of DESC_DTYPE records; d_threads: CUDA int32/uint32 tensor (one per copy)."""
        n = d_descs.numel() // DESC_DTYPE.itemsize
        assert d_threads.numel() == n
        self._ok(_lib.cg_conc_check(self.h, d_descs.data_ptr(), d_threads.data_ptr(), n, d_verdicts.data_ptr(),
                                    _stream_ptr(stream)), "cg_conc_check")

    def stamps(self):
        a, b = ctypes.c_uint64(0), ctypes.c_uint64(0)
        self._ok(_lib.cg_conc_stamps(self.h, ctypes.byref(a), ctypes.byref(b)), "cg_conc_stamps")
        return a.value, b.value

    @property
    def kernel_launches(self) -> int:
        return int(_lib.cg_conc_kernel_launches(self.h))


def to_device_descs(descs: np.ndarray, device: int = 0):
    import torch
    d = np.ascontiguousarray(descs, dtype=DESC_DTYPE)
    return torch.from_numpy(d.view(np.uint8).copy()).to(torch.device("cuda", device))


def verdicts_to_numpy(d_verdicts) -> np.ndarray:
    return d_verdicts.cpu().numpy().view(VERDICT_DTYPE)


from .replay import replay_events  # noqa: E402,F401
