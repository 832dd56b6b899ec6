"""CPU oracle for the batched transfer checker -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product package
(``paper_1310_0901_b200``) never imports it and shares no code with it.

The arithmetic lives in ``cg_oracle.c`` (plain sequential C, byte loops, a
linear allocation list).  This file only loads it and marshals numpy arrays.

Parity status: every function is pinned by tests/test_oracle_*.py (see
DESIGN.md §3 "Pins").  Readings R-4, R-6, R-11, R-12 are pinned only by the
DESIGN.md ledger (the paper has no statement to check them against).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "cg_oracle.c")
_LIB = os.path.join(_HERE, "libcgoracle.so")

VERDICT_DTYPE = np.dtype([
    ("first_unaddr", "<u8"), ("first_undef", "<u8"), ("undef_count", "<u8"),
    ("dst_expected", "<u8"), ("dst_found", "<u8"),
    ("src_expected", "<u8"), ("src_found", "<u8"),
    ("flags", "<u4"), ("status", "<u4"),
])
ALLOC_DTYPE = np.dtype([("base", "<u8"), ("size", "<u8"), ("seq", "<u8")])
NONE = (1 << 64) - 1

# flag bits restated from the ledger (R-14); not imported from the CUDA path
F_DST_NOT_ALLOCATED = 1 << 0
F_DST_TOO_SMALL = 1 << 1
F_SRC_NOT_ALLOCATED = 1 << 2
F_SRC_TOO_SMALL = 1 << 3
F_HOST_UNADDRESSABLE = 1 << 4
F_HOST_UNDEFINED = 1 << 5
F_BAD_PITCH = 1 << 6
F_INVALID_RANGE = 1 << 7
F_BAD_KIND = 1 << 8
F_CONCURRENT = 1 << 9


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc (building the checker is not using it)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-pthread", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P, U64, U32, I = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int
        lib.or_create.restype = P; lib.or_create.argtypes = [U64, U64, I]
        lib.or_destroy.argtypes = [P]
        lib.or_A.restype = P; lib.or_A.argtypes = [P]
        lib.or_V.restype = P; lib.or_V.argtypes = [P]
        lib.or_mark.restype = I; lib.or_mark.argtypes = [P, U64, U64, U32]
        lib.or_set_vbits.restype = I; lib.or_set_vbits.argtypes = [P, U64, U64, P]
        lib.or_register.restype = I; lib.or_register.argtypes = [P, U64, U64, U64]
        lib.or_free.restype = I; lib.or_free.argtypes = [P, U64, U64]
        lib.or_check_copy.argtypes = [P, P, P]
        lib.or_leaks.restype = U64; lib.or_leaks.argtypes = [P, P, U64]
        lib.or_replay.restype = U64; lib.or_replay.argtypes = [P, P, U64, P, P, P]
        lib.or_track_device.argtypes = [P, I]
        lib.or_array_bytes.restype = U64; lib.or_array_bytes.argtypes = [U64, U64, U64, U64, U64]
        lib.or_register_array.restype = I; lib.or_register_array.argtypes = [P, U64, U64, U64]
        lib.or_free_array.restype = I; lib.or_free_array.argtypes = [P, U64, U64]
        lib.or_array_leaks.restype = U64; lib.or_array_leaks.argtypes = [P, P, U64]
        lib.or_device_vbits.restype = I; lib.or_device_vbits.argtypes = [P, U64, U64, P]
        lib.or_array_vbits.restype = I; lib.or_array_vbits.argtypes = [P, U64, U64, U64, P]
        lib.or_track_concurrency.argtypes = [P, I]
        lib.or_sync.argtypes = [P, U32, U64]
        lib.or_check_copy_mt.argtypes = [P, P, U32, P]
        lib.or_replay_mt.restype = U64; lib.or_replay_mt.argtypes = [P, P, U64, P, P, P, P]
        lib.or_replay_parallel.restype = U64; lib.or_replay_parallel.argtypes = [P, P, U64, P, I, P, P]
        _lib = lib
    return _lib


class Oracle:
    """Sequential replay state: host window shadow + device allocation list."""

    def __init__(self, host_base: int, host_size: int, undef_is_error: bool = False, track_device: bool = False,
                 concurrency: bool = False):
        self.lib = _load()
        self.h0, self.s = host_base, host_size
        self.st = self.lib.or_create(host_base, host_size, int(undef_is_error))
        if not self.st:
            raise MemoryError("oracle state allocation failed")
        if track_device:
            self.lib.or_track_device(self.st, 1)
        if concurrency:
            self.lib.or_track_concurrency(self.st, 1)

    def close(self):
        if self.st:
            self.lib.or_destroy(self.st)
            self.st = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- views of the shadow state -----------------------------------------
    @property
    def A(self) -> np.ndarray:
        buf = (ctypes.c_uint8 * (self.s // 8)).from_address(self.lib.or_A(self.st))
        return np.frombuffer(buf, np.uint8)

    @property
    def V(self) -> np.ndarray:
        buf = (ctypes.c_uint8 * self.s).from_address(self.lib.or_V(self.st))
        return np.frombuffer(buf, np.uint8)

    # -- single calls --------------------------------------------------------
    def mark(self, addr, length, state) -> int:
        return self.lib.or_mark(self.st, addr, length, state)

    def set_vbits(self, addr, vbytes) -> int:
        b = np.ascontiguousarray(np.frombuffer(bytes(vbytes), np.uint8))
        return self.lib.or_set_vbits(self.st, addr, len(b), b.ctypes.data)

    def register(self, base, size, seq) -> int:
        return self.lib.or_register(self.st, base, size, seq)

    def free(self, ptr, seq) -> int:
        return self.lib.or_free(self.st, ptr, seq)

    def check_copy(self, event: np.ndarray, thread: int = 0) -> np.ndarray:
        ev = np.ascontiguousarray(np.asarray(event).reshape(1))
        out = np.zeros(1, VERDICT_DTYPE)
        self.lib.or_check_copy_mt(self.st, ev.ctypes.data, thread, out.ctypes.data)
        return out[0]

    def sync(self, thread: int, seq: int):
        """NEXT-2 ctx_synchronize of a thread"""
        self.lib.or_sync(self.st, thread, seq)

    def device_vbits(self, addr: int, length: int) -> Optional[np.ndarray]:
        out = np.zeros(max(length, 1), np.uint8)
        if self.lib.or_device_vbits(self.st, addr, length, out.ctypes.data):
            return None
        return out[:length]

    def array_vbits(self, handle: int, offset: int, length: int) -> Optional[np.ndarray]:
        """NEXT-1 x NEXT-3: V-bytes of an array's per-array shadow"""
        out = np.zeros(max(length, 1), np.uint8)
        if self.lib.or_array_vbits(self.st, handle, offset, length, out.ctypes.data):
            return None
        return out[:length]

    def array_bytes(self, width, height, depth, fmt, channels) -> int:
        return self.lib.or_array_bytes(width, height, depth, fmt, channels)

    def register_array(self, handle, total, seq) -> int:
        return self.lib.or_register_array(self.st, handle, total, seq)

    def free_array(self, handle, seq) -> int:
        return self.lib.or_free_array(self.st, handle, seq)

    def array_leaks(self) -> np.ndarray:
        n = self.lib.or_array_leaks(self.st, None, 0)
        out = np.zeros(n, ALLOC_DTYPE)
        if n:
            self.lib.or_array_leaks(self.st, out.ctypes.data, n)
        return np.sort(out, order="base")

    def leaks(self) -> np.ndarray:
        n = self.lib.or_leaks(self.st, None, 0)
        out = np.zeros(n, ALLOC_DTYPE)
        self.lib.or_leaks(self.st, out.ctypes.data if n else None, n)
        return out

    # -- whole traces --------------------------------------------------------
    def replay(self, events: np.ndarray, blob: Optional[np.ndarray] = None, threads: Optional[np.ndarray] = None):
        """Returns (verdicts per COPY event, status per event); threads[i] is
        the thread of event i (NEXT-2; None = all thread 0)."""
        ev = np.ascontiguousarray(events)
        n = len(ev)
        ncopy = int(np.count_nonzero(ev["op"] == 5))
        out_v = np.zeros(max(ncopy, 1), VERDICT_DTYPE)
        out_s = np.zeros(max(n, 1), np.uint32)
        b = np.ascontiguousarray(blob if blob is not None and len(blob) else np.zeros(1, np.uint8))
        t = None if threads is None else np.ascontiguousarray(threads, dtype=np.uint32)
        assert t is None or len(t) == n
        self.lib.or_replay_mt(self.st, ev.ctypes.data, n, b.ctypes.data, t.ctypes.data if t is not None else None,
                              out_v.ctypes.data, out_s.ctypes.data)
        return out_v[:ncopy], out_s[:n]


    def replay_parallel(self, events: np.ndarray, blob: Optional[np.ndarray] = None, threads: int = 0):
        """The same replay with the per-copy checks of each epoch on `threads`
        host threads (0: os.cpu_count()); equal to replay() by construction
        (cg_oracle.c or_replay_parallel; tests assert it)."""
        ev = np.ascontiguousarray(events)
        n = len(ev)
        ncopy = int(np.count_nonzero(ev["op"] == 5))
        out_v = np.zeros(max(ncopy, 1), VERDICT_DTYPE)
        out_s = np.zeros(max(n, 1), np.uint32)
        b = np.ascontiguousarray(blob if blob is not None and len(blob) else np.zeros(1, np.uint8))
        T = threads or os.cpu_count() or 1
        self.lib.or_replay_parallel(self.st, ev.ctypes.data, n, b.ctypes.data, T, out_v.ctypes.data,
                                    out_s.ctypes.data)
        return out_v[:ncopy], out_s[:n]


def replay_trace(trace, undef_is_error: bool = False, track_device: bool = False, concurrency: bool = False):
    """Convenience: fresh oracle, replay the whole trace, return
    (oracle, verdicts, statuses, leaks).  With concurrency, the trace's
    per-event threads (NEXT-2) are used."""
    o = Oracle(trace.host_base, trace.host_size, undef_is_error, track_device, concurrency)
    v, s = o.replay(trace.events, trace.blob, getattr(trace, "threads", None) if concurrency else None)
    return o, v, s, o.leaks()
