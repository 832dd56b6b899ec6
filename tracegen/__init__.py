"""Seeded synthetic trace generators (input data only).

This module is shared by the tests, ``bench.py`` and the oracle wrapper as the
single source of *inputs*.  It deliberately contains none of the checking
arithmetic of the method (no start-address folding, no span, no coverage, no
shadow scan, no verdict logic): it only records what a program did -- host
buffer allocations/writes, device allocations/frees and copy calls -- the way
the paper's wrappers observe them (§3: "Anytime a program
handles memory on the device or transfers data between the device and/or the
host the respective Cudagrind wrapper will be called").

Event stream format (one numpy structured record per call, ``EVENT_DTYPE``):

=========  ==========================================================
op         meaning of the fields
=========  ==========================================================
MARK       host shadow update: ``dst`` = addr,
           ``width`` = len, ``kind`` = state (NOACCESS/UNDEFINED/DEFINED)
SETV       exact V-bytes: ``dst`` = addr, ``width`` = len,
           ``src`` = offset of the bytes in the trace's ``blob``
REG        device allocation (Fig. 2 caption P:88): ``dst`` = base,
           ``width`` = size
FREE       device free: ``dst`` = ptr
COPY       one cuMemcpy{HtoD,DtoH,DtoD,2D} call: ``kind``,
           ``width`` (WidthInBytes), ``height`` (1 for 1D), and per side the
           raw CUDA_MEMCPY2D fields base / X / Y / pitch
SYNC       NEXT-2 ctx_synchronize of the event's thread
=========  ==========================================================

``seq`` is one global, strictly increasing event counter (SPEC's
``SimState.seq``).  ``Trace.threads[i]`` is the thread that issued
event i (NEXT-2; all 0 for single-threaded traces).

Device addresses come from SPEC's deterministic bump allocator (S:370:
"Device addresses come from a deterministic bump allocator starting at
0x0100_0000"), with a 256-byte alignment (an invented detail, R-17).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Optional

import numpy as np

OP_MARK, OP_SETV, OP_REG, OP_FREE, OP_COPY, OP_REGA, OP_FREEA, OP_SYNC = 1, 2, 3, 4, 5, 6, 7, 8
HTOD, DTOH, DTOD, HTOA, ATOH = 1, 2, 3, 4, 5
NOACCESS, UNDEFINED, DEFINED = 0, 1, 2

EVENT_DTYPE = np.dtype([
    ("op", "<u4"), ("kind", "<u4"), ("seq", "<u8"),
    ("width", "<u8"), ("height", "<u8"),
    ("dst", "<u8"), ("dst_x", "<u8"), ("dst_y", "<u8"), ("dst_pitch", "<u8"),
    ("src", "<u8"), ("src_x", "<u8"), ("src_y", "<u8"), ("src_pitch", "<u8"),
])
assert EVENT_DTYPE.itemsize == 96

# the copy-descriptor records the checker takes (include/cg.h cg_copy_desc, 96 B):
# the COPY events' CUDA_MEMCPY2D fields, restated here so that the oracle arm
# of bench.py never has to import the product package
DESC_DTYPE = np.dtype([
    ("kind", "<u4"), ("reserved", "<u4"), ("seq", "<u8"), ("width", "<u8"), ("height", "<u8"),
    ("dst", "<u8"), ("dst_x", "<u8"), ("dst_y", "<u8"), ("dst_pitch", "<u8"),
    ("src", "<u8"), ("src_x", "<u8"), ("src_y", "<u8"), ("src_pitch", "<u8"),
])
assert DESC_DTYPE.itemsize == 96


def events_to_descs(ev: np.ndarray) -> np.ndarray:
    """COPY events -> descriptor records (field copy)"""
    d = np.zeros(len(ev), DESC_DTYPE)
    for f in DESC_DTYPE.names:
        if f != "reserved":
            d[f] = ev[f]
    return d


DEVICE_HEAP_BASE = 0x0100_0000
DEVICE_ALIGN = 256               # invented (R-17)
KiB, MiB, GiB = 1 << 10, 1 << 20, 1 << 30


@dataclasses.dataclass
class Trace:
    """A recorded call stream plus the host shadow window it lives in."""
    name: str
    events: np.ndarray            # EVENT_DTYPE[n]
    blob: np.ndarray              # uint8 bytes referenced by SETV events
    host_base: int                # H0 (4096-aligned)
    host_size: int                # S  (multiple of 4096)
    meta: Dict = dataclasses.field(default_factory=dict)
    threads: Optional[np.ndarray] = None   # uint32[n]: issuing thread per event (NEXT-2)

    @property
    def copy_index(self) -> np.ndarray:
        return np.flatnonzero(self.events["op"] == OP_COPY)

    @property
    def n_copies(self) -> int:
        return int(np.count_nonzero(self.events["op"] == OP_COPY))


class TraceBuilder:
    """Append-only recorder. Columns are kept as Python lists of tuples for
    small traces and as bulk numpy blocks for the large configurations."""

    def __init__(self, name: str, host_base: int, host_size: int):
        assert host_base % 4096 == 0 and host_size % 4096 == 0
        self.name = name
        self.host_base = host_base
        self.host_size = host_size
        self._blocks: List[np.ndarray] = []
        self._tblocks: List[np.ndarray] = []
        self._rows: List[tuple] = []
        self._row_threads: List[int] = []
        self.thread = 0                    # NEXT-2: thread of the next recorded events
        self._blob = bytearray()
        self._seq = 0
        self.heap_cursor = DEVICE_HEAP_BASE
        self.meta: Dict = {}

    # -- raw appends ---------------------------------------------------------
    def _flush_rows(self):
        if self._rows:
            arr = np.zeros(len(self._rows), EVENT_DTYPE)
            for i, r in enumerate(self._rows):
                arr[i] = r
            self._blocks.append(arr)
            self._tblocks.append(np.array(self._row_threads, np.uint32))
            self._rows = []
            self._row_threads = []

    def _next_seq(self) -> int:
        self._seq += 1
        return self._seq

    def _row(self, op, kind=0, width=0, height=0, dst=0, dst_x=0, dst_y=0,
             dst_pitch=0, src=0, src_x=0, src_y=0, src_pitch=0) -> int:
        seq = self._next_seq()
        self._rows.append((op, kind, seq, width, height, dst, dst_x, dst_y,
                           dst_pitch, src, src_x, src_y, src_pitch))
        self._row_threads.append(self.thread)
        return seq

    def block(self, arr: np.ndarray) -> np.ndarray:
        """Append a pre-built EVENT_DTYPE block; assigns its seq numbers."""
        self._flush_rows()
        arr = arr.copy()
        arr["seq"] = np.arange(self._seq + 1, self._seq + 1 + len(arr), dtype=np.uint64)
        self._seq += len(arr)
        self._blocks.append(arr)
        self._tblocks.append(np.full(len(arr), self.thread, np.uint32))
        return arr

    # -- calls ---------------------------------------------------------------
    def mark(self, addr: int, length: int, state: int) -> int:
        return self._row(OP_MARK, kind=state, dst=addr, width=length)

    def setv(self, addr: int, vbytes: bytes) -> int:
        off = len(self._blob)
        self._blob += bytes(vbytes)
        return self._row(OP_SETV, dst=addr, width=len(vbytes), src=off)

    def register(self, base: int, size: int) -> int:
        return self._row(OP_REG, dst=base, width=size)

    def free(self, ptr: int) -> int:
        return self._row(OP_FREE, dst=ptr)

    def sync(self) -> int:
        """NEXT-2: ctx_synchronize by the current thread."""
        return self._row(OP_SYNC)

    def register_array(self, handle: int, width: int, height: int = 0, depth: int = 0, fmt: int = 0,
                       channels: int = 1) -> int:
        """cuArrayCreate (Fig. 2 caption P:88; SPEC ArrayDescriptor S:125-128):
        REGA with dst = handle, width/height, dst_x = depth, dst_y = format code,
        dst_pitch = channels."""
        return self._row(OP_REGA, dst=handle, width=width, height=height, dst_x=depth, dst_y=fmt,
                         dst_pitch=channels)

    def free_array(self, handle: int) -> int:
        return self._row(OP_FREEA, dst=handle)

    def copy_htoa(self, handle: int, offset: int, src: int, nbytes: int) -> int:
        return self._row(OP_COPY, kind=HTOA, width=nbytes, height=1, dst=handle, dst_x=offset,
                         src=src, src_pitch=nbytes)

    def copy_atoh(self, dst: int, handle: int, offset: int, nbytes: int) -> int:
        return self._row(OP_COPY, kind=ATOH, width=nbytes, height=1, dst=dst, dst_pitch=nbytes,
                         src=handle, src_x=offset)

    def malloc(self, size: int) -> int:
        """Play the driver: bump allocate, then record REG."""
        base = self.heap_cursor
        self.heap_cursor = (base + size + DEVICE_ALIGN - 1) // DEVICE_ALIGN * DEVICE_ALIGN
        self.register(base, size)
        return base

    def copy1d(self, kind: int, dst: int, src: int, nbytes: int) -> int:
        """cuMemcpyHtoD/DtoH/DtoD: a 2D copy of one row, pitch = width."""
        return self._row(OP_COPY, kind=kind, width=nbytes, height=1,
                         dst=dst, dst_pitch=nbytes, src=src, src_pitch=nbytes)

    def copy2d(self, kind: int, width: int, height: int,
               dst: int, dst_x: int, dst_y: int, dst_pitch: int,
               src: int, src_x: int, src_y: int, src_pitch: int) -> int:
        """cuMemcpy2D with raw CUDA_MEMCPY2D fields."""
        return self._row(OP_COPY, kind=kind, width=width, height=height,
                         dst=dst, dst_x=dst_x, dst_y=dst_y, dst_pitch=dst_pitch,
                         src=src, src_x=src_x, src_y=src_y, src_pitch=src_pitch)

    def build(self) -> Trace:
        self._flush_rows()
        ev = np.concatenate(self._blocks) if self._blocks else np.zeros(0, EVENT_DTYPE)
        th = np.concatenate(self._tblocks) if self._tblocks else np.zeros(0, np.uint32)
        return Trace(self.name, ev, np.frombuffer(bytes(self._blob), np.uint8).copy(),
                     self.host_base, self.host_size, self.meta, th)


def _log_uniform(rng: np.random.Generator, a: float, b: float, n: int) -> np.ndarray:
    """exp(U[ln a, ln b]) rounded down (SURVEY §8(d) recipe)."""
    return np.floor(np.exp(rng.uniform(math.log(a), math.log(b), n))).astype(np.uint64)


# ---------------------------------------------------------------------------
# Config 1: the toy trace (BASELINE.json configs[0])
# ---------------------------------------------------------------------------
def toy() -> Trace:
    H0 = 0x10000
    tb = TraceBuilder("toy", H0, 64 * KiB)
    h0, h1, h2, h3 = H0 + 0x0000, H0 + 0x0200, H0 + 0x0800, H0 + 0x2000
    # host buffers (host_alloc = UNDEFINED, host_write = DEFINED)
    tb.mark(h0, 256, UNDEFINED); tb.mark(h0, 256, DEFINED)
    tb.mark(h1, 1024, UNDEFINED); tb.mark(h1, 100, DEFINED); tb.mark(h1 + 132, 1024 - 132, DEFINED)
    tb.setv(h1 + 500, b"\x0f")
    tb.mark(h2, 4096, UNDEFINED); tb.mark(h2, 4096, DEFINED)
    tb.mark(h3, 4096, UNDEFINED)
    d0 = tb.malloc(256); d1 = tb.malloc(1024); d2 = tb.malloc(4096)
    c = {}
    c["C1"] = tb.copy1d(HTOD, d0, h0, 256)
    c["C2"] = tb.copy1d(HTOD, d1, h1, 1024)
    c["C3"] = tb.copy1d(HTOD, d2, h2, 4096)
    c["C4"] = tb.copy1d(DTOH, h3, d2, 4096)
    c["C5"] = tb.copy1d(HTOD, d2, h3, 4096)
    c["C6"] = tb.copy1d(HTOD, d0, h2, 272)
    c["C7"] = tb.copy1d(DTOH, h1, d1, 1024)
    c["C8"] = tb.copy1d(HTOD, d0, h1, 256)
    tb.free(d1)
    c["C9"] = tb.copy1d(HTOD, d1, h1, 1024)
    c["C10"] = tb.copy1d(DTOH, h0, d0, 256)
    tb.free(d0)
    tb.meta.update(dict(d=[d0, d1, d2], h=[h0, h1, h2, h3], copies=c))
    return tb.build()


# ---------------------------------------------------------------------------
# The paper's worked example: Listing 2 -> Listing 5
# ---------------------------------------------------------------------------
def listing2() -> Trace:
    size = 1000000
    H0 = 1 << 20
    tb = TraceBuilder("listing2", H0, 32 * MiB)
    c = tb.malloc(size * 4)                          # P:139 sizeof(float)
    a = tb.malloc(size * 8)
    b = tb.malloc(size * 8)
    a_h, b_h, c_host = H0, H0 + 8 * MiB + 4096, H0 + 16 * MiB + 8192
    tb.mark(a_h, size * 8, DEFINED)
    tb.mark(b_h, size * 8, DEFINED)
    tb.mark(c_host, size * 8, UNDEFINED)
    tb.copy1d(HTOD, a, a_h, size * 8)
    tb.copy1d(HTOD, b, b_h, size * 8)
    s = tb.copy1d(DTOH, c_host, c, size * 8)
    tb.meta.update(dict(c=c, a=a, b=b, c_host=c_host, faulty_seq=s))
    return tb.build()


# ---------------------------------------------------------------------------
# Random tiny traces (<=200 events in a 64 KiB window)
# ---------------------------------------------------------------------------
def random_tiny(seed: int, n_events: int = 200, window: int = 64 * KiB,
                host_base: int = 0x40000, arrays: bool = False, threads: int = 0) -> Trace:
    """Unaligned, overlapping, out-of-window, 2D, reuse-after-free: everything
    the method must handle, at sizes a brute-force checker finishes quickly.
    threads > 0 (NEXT-2): every event is issued by a random one of `threads`
    threads and SYNC events are interleaved (drawn from a second generator,
    so the call stream itself is the same as with threads = 0)."""
    rng = np.random.default_rng(seed)
    rng_t = np.random.default_rng(seed + 0x5EED) if threads else None
    tb = TraceBuilder(f"tiny{seed}", host_base, window)
    live: List[tuple] = []
    freed: List[tuple] = []
    cursor = DEVICE_HEAP_BASE

    def rand_host(maxlen=4096):
        # mostly inside the window, sometimes straddling either edge
        u = rng.random()
        if u < 0.05:
            start = host_base - int(rng.integers(1, 64))
        elif u < 0.10:
            start = host_base + window - int(rng.integers(1, 64))
        else:
            start = host_base + int(rng.integers(0, window))
        return start, int(rng.integers(0, maxlen))

    def rand_dev():
        u = rng.random()
        if live and u < 0.75:
            b, s = live[int(rng.integers(len(live)))]
            return b + int(rng.integers(0, s + 2))       # sometimes one past end
        if freed and u < 0.85:
            b, s = freed[int(rng.integers(len(freed)))]
            return b + int(rng.integers(0, s))
        return DEVICE_HEAP_BASE + int(rng.integers(0, 1 << 16))

    # a few large host buffers first, so that many copies see addressable bytes
    for _ in range(4):
        a = host_base + int(rng.integers(0, window // 2))
        l = int(rng.integers(window // 8, window // 2))
        tb.mark(a, min(l, host_base + window - a), int(rng.choice([UNDEFINED, DEFINED], p=[0.3, 0.7])))
    handles: List[tuple] = []      # (handle, nominal bytes) of created arrays
    for _ in range(n_events - 4):
        if rng_t is not None:
            tb.thread = int(rng_t.integers(threads))
            if rng_t.random() < 0.08:
                tb.sync()
        u = rng.random()
        if arrays and u < 0.22:         # NEXT-3: device arrays and their transfers
            v = rng.random()
            if v < 0.25 or not handles:
                h = int(rng.choice([0x1000 + len(handles), int(rng.integers(1, 8))]))
                w = int(rng.integers(0, 400)); fmt = int(rng.integers(0, 9)); ch = int(rng.choice([1, 2, 3, 4]))
                tb.register_array(h, w, int(rng.integers(0, 3)), int(rng.integers(0, 2)), fmt, ch)
                handles.append((h, max(w, 1) * 8))
            elif v < 0.35:
                tb.free_array(int(rng.choice([hh for hh, _ in handles] + [99])))
            else:
                h, cap = handles[int(rng.integers(len(handles)))]
                off = int(rng.integers(0, cap + 16))
                a, l = rand_host(cap + 64)
                if rng.random() < 0.5:
                    tb.copy_htoa(h, off, a, l)
                else:
                    tb.copy_atoh(a, h, off, l)
            continue
        if u < 0.18:
            a, l = rand_host(6000)
            st = int(rng.integers(0, 3))
            a = max(a, host_base); l = min(l, host_base + window - a)
            tb.mark(a, l, st)
        elif u < 0.24:
            a, l = rand_host(64)
            a = max(a, host_base); l = min(l, host_base + window - a)
            tb.setv(a, rng.integers(0, 256, l, dtype=np.uint8).tobytes())
        elif u < 0.34:
            size = int(rng.integers(0, 3000))
            if freed and rng.random() < 0.3:             # address reuse
                b, s = freed[int(rng.integers(len(freed)))]
                base = b + int(rng.integers(0, 64))
            elif rng.random() < 0.05:
                base = int(rng.choice([0, cursor]))        # base 0 / duplicate
            else:
                base = cursor
                cursor = (cursor + max(size, 1) + int(rng.integers(0, 3)) * 128 + 255) // 256 * 256
            tb.register(base, size)
            # our own bookkeeping only to aim later calls; no checking here
            if size and base and not any(b < base + size and base < b + s for b, s in live):
                live.append((base, size))
        elif u < 0.42:
            if live and rng.random() < 0.8:
                i = int(rng.integers(len(live)))
                b, s = live[i]
                ptr = b if rng.random() < 0.85 else b + int(rng.integers(0, 16))
                tb.free(ptr)
                if ptr == b:
                    freed.append(live.pop(i))
            else:
                tb.free(int(rng.choice([0, DEVICE_HEAP_BASE + 8])))
        else:
            kind = int(rng.choice([HTOD, DTOH, DTOD], p=[0.45, 0.4, 0.15]))
            two_d = rng.random() < 0.35
            if kind == HTOD:
                dst = rand_dev(); src, ln = rand_host()
            elif kind == DTOH:
                dst, ln = rand_host(); src = rand_dev()
            else:
                dst = rand_dev(); src = rand_dev(); ln = int(rng.integers(0, 4096))
            if not two_d:
                if rng.random() < 0.05:
                    ln = 0
                tb.copy1d(kind, dst, src, ln)
            else:
                w = int(rng.integers(0, 200)); h = int(rng.integers(0, 24))
                def side():
                    x = int(rng.integers(0, 64)); y = int(rng.integers(0, 4))
                    pitch = w + x + int(rng.integers(0, 64))
                    if rng.random() < 0.1:
                        pitch = int(rng.integers(0, max(w + x, 1)))   # BAD_PITCH
                    return x, y, pitch
                dx, dy, dp = side(); sx, sy, sp = side()
                if rng.random() < 0.02:
                    dy = 1 << 62                                     # overflow
                tb.copy2d(kind, w, h, dst, dx, dy, dp, src, sx, sy, sp)
    return tb.build()


# ---------------------------------------------------------------------------
# Config 2: 1M small copies vs a 100k-entry table, 1% injected (configs[1])
# ---------------------------------------------------------------------------
INJ_NONE, INJ_DST_NA, INJ_SRC_NA, INJ_TOO_SMALL, INJ_HOST_UNADDR, INJ_HOST_UNDEF, INJ_DTOD_BAD_SRC = range(7)


def c2_small(seed: int = 13100902, n_copies: int = 1_000_000, n_allocs: int = 100_000,
             inject_frac: float = 0.01, redzone: int = 16, host_base: int = 1 << 32,
             host_size: Optional[int] = None) -> Trace:
    """SURVEY §8(d) C2.  Every copy gets a private host buffer (malloc-like:
    16-byte aligned, >= ``redzone`` NOACCESS bytes on both sides), so the trace
    is a single hazard-free batch and the dirty set is exactly the injected
    set.  HtoD sources are written (DEFINED); DtoH destinations are allocated
    but not written (UNDEFINED), like ``c_host`` in Listing 2."""
    assert redzone >= 16 and redzone % 16 == 0
    rng = np.random.default_rng(seed)
    H0 = host_base
    # ---- device allocations (bump allocator)
    sizes = _log_uniform(rng, 64, 64 * KiB, n_allocs)
    aligned = (sizes + DEVICE_ALIGN - 1) // DEVICE_ALIGN * DEVICE_ALIGN
    bases = (DEVICE_HEAP_BASE + np.concatenate([[0], np.cumsum(aligned)[:-1]])).astype(np.uint64)
    heap_end = int(bases[-1] + aligned[-1])
    n_freed = max(1, n_allocs // 100)
    freed_ids = rng.choice(n_allocs, n_freed, replace=False)
    usable = np.ones(n_allocs, bool); usable[freed_ids] = False
    use_ids = np.flatnonzero(usable)
    order = use_ids[np.argsort(sizes[use_ids], kind="stable")]
    sorted_sizes = sizes[order]

    def pick_alloc(lens):
        """an allocation at least as large as the copy, uniformly among those"""
        lo = np.searchsorted(sorted_sizes, lens, side="left")
        lo = np.minimum(lo, len(order) - 1)
        p = lo + np.floor(rng.random(len(lens)) * (len(order) - lo)).astype(np.int64)
        return order[np.minimum(p, len(order) - 1)]

    # ---- copies: kind mix 50/40/10, length log-uniform 64 B-64 KiB
    kinds = rng.choice(np.array([HTOD, DTOH, DTOD], np.uint32), n_copies, p=[0.5, 0.4, 0.1])
    lens = _log_uniform(rng, 64, 64 * KiB, n_copies)
    aid = pick_alloc(lens)
    lens = np.minimum(lens, sizes[aid])
    dev = bases[aid] + np.floor(rng.random(n_copies) * (sizes[aid] - lens + 1)).astype(np.uint64)
    aid2 = pick_alloc(lens)
    dev2 = bases[aid2] + np.floor(rng.random(n_copies) * (sizes[aid2] - lens + 1)).astype(np.uint64)

    # ---- injection classes (1 %), kinds made consistent with the class
    inj = np.zeros(n_copies, np.uint8)
    n_inj = int(round(n_copies * inject_frac))
    inj_idx = rng.choice(n_copies, n_inj, replace=False)
    inj[inj_idx] = np.arange(n_inj) % 6 + 1
    kinds[(inj == INJ_DST_NA) & (kinds == DTOH)] = HTOD
    kinds[(inj == INJ_SRC_NA) & (kinds == HTOD)] = DTOH
    kinds[(inj == INJ_HOST_UNADDR) & (kinds == DTOD)] = HTOD
    kinds[inj == INJ_HOST_UNDEF] = HTOD
    kinds[inj == INJ_DTOD_BAD_SRC] = DTOD

    # device pointers per side: HtoD dst=dev; DtoH src=dev; DtoD dst=dev, src=dev2
    dptr_dst = np.where(kinds == DTOH, 0, dev).astype(np.uint64)
    dptr_src = np.where(kinds == DTOH, dev, np.where(kinds == DTOD, dev2, 0)).astype(np.uint64)
    freed_bases = bases[freed_ids]

    def bad_ptr(mask):
        """alternately inside a freed allocation (use after free) or past the heap"""
        k = int(np.count_nonzero(mask))
        fb = freed_bases[rng.integers(0, len(freed_bases), k)]
        beyond = heap_end + rng.integers(0, 1 << 20, k).astype(np.uint64)
        return np.where(np.arange(k) % 2 == 0, fb, beyond).astype(np.uint64)
    m = inj == INJ_DST_NA; dptr_dst[m] = bad_ptr(m)
    m = inj == INJ_SRC_NA; dptr_src[m] = bad_ptr(m)
    m = inj == INJ_DTOD_BAD_SRC; dptr_src[m] = bad_ptr(m)
    # TooSmall: the device range starts max(len-over,1) bytes before its
    # allocation's end, over = 1..64 (the copy runs past the end)
    m = np.flatnonzero(inj == INJ_TOO_SMALL)
    over = rng.integers(1, 65, len(m)).astype(np.uint64)
    room = np.maximum(lens[m].astype(np.int64) - over.astype(np.int64), 1).astype(np.uint64)
    a_end = bases[aid[m]] + sizes[aid[m]]
    on_src = kinds[m] == DTOH
    dptr_src[m[on_src]] = (a_end - room)[on_src]
    dptr_dst[m[~on_src]] = (a_end - room)[~on_src]

    # ---- host buffers: private, 16-aligned, redzoned
    has_host = kinds != DTOD
    buf_len = np.where(has_host, lens, 0).astype(np.uint64)
    copy_len = lens.copy()
    m = inj == INJ_HOST_UNADDR       # +1..redzone bytes past the buffer end
    copy_len[m] += rng.integers(1, redzone + 1, int(np.count_nonzero(m))).astype(np.uint64)
    slot = np.where(has_host, (buf_len + 2 * redzone + 15) // 16 * 16, 0).astype(np.uint64)
    host_start = (H0 + 4096 + redzone + np.concatenate([[0], np.cumsum(slot)[:-1]])).astype(np.uint64)
    end = int(host_start[-1]) - redzone + int(slot[-1]) + 4096
    S = (end - H0 + MiB - 1) // MiB * MiB
    if host_size is not None:           # a fixed window (e.g. one shard of a sharded bench)
        assert host_size >= S, (host_size, S)
        S = host_size

    tb = TraceBuilder("c2_small", H0, S)
    hidx = np.flatnonzero(has_host)
    marks = np.zeros(len(hidx), EVENT_DTYPE)
    marks["op"] = OP_MARK
    marks["dst"] = host_start[hidx]
    marks["width"] = buf_len[hidx]
    marks["kind"] = np.where(kinds[hidx] == HTOD, DEFINED, UNDEFINED)
    tb.block(marks)
    # HostUndefined: 1..16 random bytes of the source get a random non-zero V-byte
    for i in np.flatnonzero(inj == INJ_HOST_UNDEF):
        k = min(int(rng.integers(1, 17)), int(buf_len[i]))
        for p in np.sort(rng.choice(int(buf_len[i]), k, replace=False)):
            tb.setv(int(host_start[i]) + int(p), bytes([int(rng.integers(1, 256))]))
    regs = np.zeros(n_allocs, EVENT_DTYPE)
    regs["op"] = OP_REG; regs["dst"] = bases; regs["width"] = sizes
    tb.block(regs)
    frees = np.zeros(n_freed, EVENT_DTYPE)
    frees["op"] = OP_FREE; frees["dst"] = np.sort(freed_bases)
    tb.block(frees)
    cp = np.zeros(n_copies, EVENT_DTYPE)
    cp["op"] = OP_COPY; cp["kind"] = kinds; cp["width"] = copy_len; cp["height"] = 1
    cp["dst_pitch"] = copy_len; cp["src_pitch"] = copy_len
    cp["dst"] = np.where(kinds == DTOH, host_start, dptr_dst)
    cp["src"] = np.where(kinds == HTOD, host_start, dptr_src)
    tb.block(cp)
    tb.meta.update(dict(inject=inj, kinds=kinds, n_freed=n_freed, n_allocs=n_allocs, seed=seed))
    return tb.build()


# ---------------------------------------------------------------------------
# Config 3: one 8 GiB HtoD buffer, one undefined byte per MiB (configs[2])
# ---------------------------------------------------------------------------
def c3_single(seed: int = 13100903, size: int = 8 * GiB, dtoh: bool = False,
              stride: int = MiB) -> Trace:
    rng = np.random.default_rng(seed)
    H0 = 1 << 36
    S = size + 32 * KiB          # divisible into 4096-multiple shards for G <= 8
    tb = TraceBuilder("c3_single" + ("_dtoh" if dtoh else ""), H0, S)
    hbuf = H0 + 4096
    tb.mark(hbuf, size, DEFINED if not dtoh else UNDEFINED)
    n_holes = size // stride
    offs = np.arange(n_holes, dtype=np.uint64) * stride + rng.integers(0, stride, n_holes).astype(np.uint64)
    vals = rng.integers(1, 256, n_holes).astype(np.uint8)
    if not dtoh:
        rows = np.zeros(n_holes, EVENT_DTYPE)
        rows["op"] = OP_SETV; rows["dst"] = hbuf + offs; rows["width"] = 1
        rows["src"] = np.arange(n_holes, dtype=np.uint64)
        tb._blob += vals.tobytes()
        tb.block(rows)
    d = tb.malloc(size)
    if dtoh:
        tb.copy1d(DTOH, hbuf, d, size)
    else:
        tb.copy1d(HTOD, d, hbuf, size)
    tb.meta.update(dict(hole_offsets=offs, hole_values=vals, size=size, dtoh=dtoh))
    return tb.build()


# ---------------------------------------------------------------------------
# Config 4: 100k cuMemcpy2D pitched copies (configs[3])
# ---------------------------------------------------------------------------
def c4_pitched(seed: int = 13100904, n_copies: int = 100_000, n_bufs: int = 32,
               rows: int = 4096, width: int = 16 * KiB, pitch: int = 16896,
               inject_frac: float = 0.01) -> Trace:
    """W log-uniform [1 KiB, 16 KiB], H log-uniform [1, 4096] (SURVEY's
    reading of "width 1-16 KB, height 1-4096"); host 2D buffers whose pitch
    padding is NOACCESS; injected column overruns into the padding, BAD_PITCH
    and device height overruns."""
    rng = np.random.default_rng(seed)
    H0 = 1 << 40
    guard = MiB
    buf_bytes = rows * pitch
    n_host = 2 * n_bufs
    S = (n_host * (buf_bytes + guard) + guard + (1 << 20) - 1) // (1 << 20) * (1 << 20)
    tb = TraceBuilder("c4_pitched", H0, S)
    hbase = H0 + guard + np.arange(n_host, dtype=np.uint64) * (buf_bytes + guard)
    # valid width of every row addressable; padding stays NOACCESS
    r = np.arange(rows, dtype=np.uint64)
    marks = np.zeros(n_host * rows, EVENT_DTYPE)
    marks["op"] = OP_MARK
    marks["dst"] = (hbase[:, None] + r[None, :] * pitch).ravel()
    marks["width"] = width
    marks["kind"] = np.repeat(np.where(np.arange(n_host) < n_bufs, DEFINED, UNDEFINED), rows)
    tb.block(marks)
    dbases = np.array([tb.malloc(buf_bytes) for _ in range(n_host)], dtype=np.uint64)

    kinds = np.where(rng.random(n_copies) < 0.5, HTOD, DTOH).astype(np.uint32)
    W = _log_uniform(rng, KiB, width + 1, n_copies)
    W = np.minimum(W, width)
    H = _log_uniform(rng, 1, rows + 1, n_copies)
    H = np.minimum(H, rows)
    hb = rng.integers(0, n_bufs, n_copies)
    hb = np.where(kinds == HTOD, hb, hb + n_bufs)
    db = rng.integers(0, n_host, n_copies)
    hx = np.floor(rng.random(n_copies) * (width - W + 1)).astype(np.uint64)
    hy = np.floor(rng.random(n_copies) * (rows - H + 1)).astype(np.uint64)
    dx = np.floor(rng.random(n_copies) * (width - W + 1)).astype(np.uint64)
    dy = np.floor(rng.random(n_copies) * (rows - H + 1)).astype(np.uint64)
    hpitch = np.full(n_copies, pitch, np.uint64)
    dpitch = np.full(n_copies, pitch, np.uint64)

    inj = np.zeros(n_copies, np.uint8)
    n_inj = int(round(n_copies * inject_frac))
    inj_idx = rng.choice(n_copies, n_inj, replace=False)
    cls = np.arange(n_inj) % 3 + 1           # 1 column overrun, 2 BAD_PITCH, 3 height overrun
    inj[inj_idx] = cls
    m = np.flatnonzero(inj == 1)             # X+W in (16 KiB, pitch]
    hx[m] = width - W[m] + rng.integers(1, pitch - width + 1, len(m)).astype(np.uint64)
    m = np.flatnonzero(inj == 2)             # X+W > pitch
    hx[m] = pitch - W[m] + rng.integers(1, 64, len(m)).astype(np.uint64)
    m = np.flatnonzero(inj == 3)             # device rows past the allocation (Y stays inside)
    H[m] = np.maximum(H[m], 9)
    hy[m] = np.minimum(hy[m], rows - H[m])
    dy[m] = rows - H[m] + rng.integers(1, 9, len(m)).astype(np.uint64)

    cp = np.zeros(n_copies, EVENT_DTYPE)
    cp["op"] = OP_COPY; cp["kind"] = kinds; cp["width"] = W; cp["height"] = H
    is_h2d = kinds == HTOD
    cp["src"] = np.where(is_h2d, hbase[hb], dbases[db])
    cp["src_x"] = np.where(is_h2d, hx, dx); cp["src_y"] = np.where(is_h2d, hy, dy)
    cp["src_pitch"] = np.where(is_h2d, hpitch, dpitch)
    cp["dst"] = np.where(is_h2d, dbases[db], hbase[hb])
    cp["dst_x"] = np.where(is_h2d, dx, hx); cp["dst_y"] = np.where(is_h2d, dy, hy)
    cp["dst_pitch"] = np.where(is_h2d, dpitch, hpitch)
    tb.block(cp)
    tb.meta.update(dict(inject=inj, kinds=kinds, W=W, H=H, seed=seed))
    return tb.build()


CONFIGS = {
    "toy": toy,
    "c2_small": c2_small,
    "c3_single": c3_single,
    "c4_pitched": c4_pitched,
}


# ---------------------------------------------------------------------------
# Config 5: 64 GB host shadow, 10M mixed descriptors, interleaved alloc/free,
# final leak report (configs[4]); scale < 1 shrinks every count and the window
# ---------------------------------------------------------------------------
def c5_sharded(seed: int = 13100905, scale: float = 1.0, shards: int = 8, inject_frac: float = 0.01,
               redzone: int = 16) -> Trace:
    """SURVEY §8(d) C5.  Window 64 GiB (x scale) cut into 64 KiB slots, one host
    buffer per slot (even slots: written HtoD sources; odd slots: allocated DtoH
    targets), except 128 MiB (x scale) bands centred on the `shards`-1 shard
    boundaries, which hold 100 large (1-64 MiB) straddling HtoD/DtoH buffers
    (HtoD and DtoH on disjoint halves).  Registry: 100k initial allocations;
    after every 10k descriptors 50 random live ones are freed and 50 new ones
    allocated (bump, no reuse); at the end all but a seeded 1 % are freed.
    10M copies HtoD 45 % / DtoH 45 % / DtoD 10 %, 1 % injected (incl. use after
    free), plus 10 deliberate DtoH -> HtoD ping-pongs on odd slots (the only
    batch hazards: ~11 epochs)."""
    rng = np.random.default_rng(seed)
    H0 = 1 << 44
    S = int(round((64 << 30) * scale)) // (shards * 65536) * (shards * 65536)
    slot = 65536
    n_slots = S // slot
    band = max(2 * slot, int((128 << 20) * scale) // slot * slot)
    bounds = [H0 + k * (S // shards) for k in range(1, shards)]
    slot_start = H0 + np.arange(n_slots, dtype=np.uint64) * slot
    in_band = np.zeros(n_slots, bool)
    for b in bounds:
        lo, hi = (b - band // 2 - H0) // slot, (b + band // 2 - H0) // slot
        in_band[lo:hi] = True
    free_slots = np.flatnonzero(~in_band)
    buf_len = np.minimum(_log_uniform(rng, 64, slot, n_slots), slot - 2 * redzone - 64).astype(np.uint64)
    buf_start = slot_start + redzone
    is_src = (np.arange(n_slots) % 2 == 0)

    tb = TraceBuilder("c5_sharded", H0, S)
    marks = np.zeros(len(free_slots), EVENT_DTYPE)
    marks["op"] = OP_MARK
    marks["dst"] = buf_start[free_slots]
    marks["width"] = buf_len[free_slots]
    marks["kind"] = np.where(is_src[free_slots], DEFINED, UNDEFINED)
    tb.block(marks)
    # straddling band buffers: each band = [HtoD half | DtoH half] around the boundary
    big = []      # (host start, length, kind) of a region straddling boundary b
    for k, b in enumerate(bounds):
        half = band // 2
        if k % 2 == 0:      # HtoD sources across even boundaries
            tb.mark(b - half + 4096, band - 8192, DEFINED)
            big.append((b - half + 4096, band - 8192, HTOD))
        else:               # DtoH targets across odd boundaries
            tb.mark(b - half + 4096, band - 8192, UNDEFINED)
            big.append((b - half + 4096, band - 8192, DTOH))
    # one 64 MiB device buffer per band for the large copies
    big_dev = [tb.malloc(64 << 20) for _ in bounds]

    n_copies = max(1000, int(10_000_000 * scale))
    n_init = max(1000, int(100_000 * scale))
    burst_every, burst = 10_000, 50
    sizes0 = _log_uniform(rng, 64, 64 * KiB, n_init)
    live_base: List[int] = []
    live_size: List[int] = []
    freed: List[tuple] = []
    rows = []
    for sz in sizes0:
        base = tb.heap_cursor
        tb.heap_cursor = (base + int(sz) + DEVICE_ALIGN - 1) // DEVICE_ALIGN * DEVICE_ALIGN
        live_base.append(base)
        live_size.append(int(sz))
    regs = np.zeros(n_init, EVENT_DTYPE)
    regs["op"] = OP_REG
    regs["dst"] = np.array(live_base, np.uint64)
    regs["width"] = sizes0
    tb.block(regs)
    # HostUndefined injections are prepared on even slots up front
    inj_classes = 7
    n_inj = int(round(n_copies * inject_frac))
    kinds_all = rng.choice(np.array([HTOD, DTOH, DTOD], np.uint32), n_copies, p=[0.45, 0.45, 0.10])
    inj = np.zeros(n_copies, np.uint8)
    inj_idx = rng.choice(n_copies, n_inj, replace=False)
    inj[inj_idx] = np.arange(n_inj) % 6 + 1
    kinds_all[(inj == INJ_HOST_UNDEF) | (inj == INJ_DST_NA)] = HTOD
    kinds_all[inj == INJ_SRC_NA] = DTOH
    kinds_all[inj == INJ_DTOD_BAD_SRC] = DTOD
    kinds_all[(inj == INJ_HOST_UNADDR) & (kinds_all == DTOD)] = HTOD
    src_slots = free_slots[is_src[free_slots]]
    dst_slots = free_slots[~is_src[free_slots]]
    slot_pick = np.where(kinds_all == HTOD, rng.choice(src_slots, n_copies), rng.choice(dst_slots, n_copies))
    undef_slots = np.unique(slot_pick[inj == INJ_HOST_UNDEF])
    for sl in undef_slots:
        k = int(rng.integers(1, 17))
        for p in np.sort(rng.choice(int(buf_len[sl]), min(k, int(buf_len[sl])), replace=False)):
            tb.setv(int(buf_start[sl]) + int(p), bytes([int(rng.integers(1, 256))]))
    lens = np.minimum(_log_uniform(rng, 64, 64 * KiB, n_copies), buf_len[slot_pick]).astype(np.uint64)
    pingpong = set(int(x) for x in rng.choice(np.flatnonzero(inj == 0), 10, replace=False))
    big_at = set(int(x) for x in rng.choice(n_copies, 100, replace=False))
    heap_end_probe = 1 << 50

    chunk_rows = []
    for c0 in range(0, n_copies, burst_every):
        c1 = min(n_copies, c0 + burst_every)
        if c0:
            # registry burst: free 50 random live, allocate 50 new (bump, no reuse)
            fr = rng.choice(len(live_base), burst, replace=False)
            for j in sorted(fr, reverse=True):
                tb.free(live_base[j])
                freed.append((live_base[j], live_size[j]))
                live_base.pop(j)
                live_size.pop(j)
            for sz in _log_uniform(rng, 64, 64 * KiB, burst):
                live_base.append(tb.malloc(int(sz)))
                live_size.append(int(sz))
        lb = np.array(live_base, np.uint64)
        ls = np.array(live_size, np.uint64)
        m = c1 - c0
        kinds = kinds_all[c0:c1]
        ln = lens[c0:c1].copy()
        a1 = rng.integers(0, len(lb), m)
        a2 = rng.integers(0, len(lb), m)
        ln = np.where(kinds == DTOD, np.minimum(ln, np.minimum(ls[a1], ls[a2])), np.minimum(ln, ls[a1]))
        ln = np.maximum(ln, 1)
        off1 = np.floor(rng.random(m) * (ls[a1] - ln + 1)).astype(np.uint64)
        off2 = np.floor(rng.random(m) * (ls[a2] - np.minimum(ln, ls[a2]) + 1)).astype(np.uint64)
        dev1, dev2 = lb[a1] + off1, lb[a2] + off2
        host = buf_start[slot_pick[c0:c1]]
        cls = inj[c0:c1]
        cp = np.zeros(m, EVENT_DTYPE)
        cp["op"] = OP_COPY
        cp["kind"] = kinds
        cp["height"] = 1
        dst = np.where(kinds == DTOH, host, dev1)
        src = np.where(kinds == HTOD, host, np.where(kinds == DTOH, dev1, dev2))
        width = ln.copy()
        # injections
        bad = lambda k: (np.array([f[0] for f in freed], np.uint64)[rng.integers(0, len(freed), k)]
                         if freed and rng.random() < 0.5 else heap_end_probe + rng.integers(0, 1 << 20, k).astype(np.uint64))
        mk = cls == INJ_DST_NA
        if mk.any():
            dst[mk] = bad(int(mk.sum()))
        mk = (cls == INJ_SRC_NA) | (cls == INJ_DTOD_BAD_SRC)
        if mk.any():
            src[mk] = bad(int(mk.sum()))
        mk = np.flatnonzero(cls == INJ_TOO_SMALL)
        for i in mk:
            over = int(rng.integers(1, 65))
            end = int(lb[a1[i]] + ls[a1[i]])
            room = max(int(ln[i]) - over, 1)
            if kinds[i] == DTOH:
                src[i] = end - room
            else:
                dst[i] = end - room
        mk = cls == INJ_HOST_UNADDR
        width[mk] = buf_len[slot_pick[c0:c1][mk]] + rng.integers(1, redzone + 1, int(mk.sum())).astype(np.uint64)
        cp["dst"], cp["src"], cp["width"] = dst, src, width
        cp["dst_pitch"] = width
        cp["src_pitch"] = width
        # large straddlers inside the boundary bands
        for i in range(c0, c1):
            if i in big_at and big and cls[i - c0] == 0:
                j = int(rng.integers(len(big)))
                hs, hl, kd = big[j]
                L = int(min(_log_uniform(rng, 1 << 20, 64 << 20, 1)[0], hl))
                start = hs + (hl - L) // 2          # centred on the shard boundary
                k = i - c0
                cp[k]["kind"] = kd
                if kd == DTOH:
                    cp[k]["dst"], cp[k]["src"] = start, big_dev[j]
                else:
                    cp[k]["src"], cp[k]["dst"] = start, big_dev[j]
                cp[k]["width"] = L
                cp[k]["dst_pitch"] = L
                cp[k]["src_pitch"] = L
        tb.block(cp)
        # deliberate ping-pongs: a DtoH into an odd slot, then an HtoD reading it back
        for i in range(c0, c1):
            if i in pingpong:
                sl = int(rng.choice(dst_slots))
                ln2 = int(buf_len[sl])
                d = tb.malloc(ln2)
                live_base.append(d)
                live_size.append(ln2)
                tb.copy1d(DTOH, int(buf_start[sl]), d, ln2)
                tb.copy1d(HTOD, d, int(buf_start[sl]), ln2)
    # final frees: all but 1 % leak
    keep = set(int(x) for x in rng.choice(len(live_base), max(1, len(live_base) // 100), replace=False))
    fr = np.zeros(len(live_base) - len(keep), EVENT_DTYPE)
    fr["op"] = OP_FREE
    fr["dst"] = [b for j, b in enumerate(live_base) if j not in keep]
    tb.block(fr)
    tb.meta.update(dict(inject=inj, shards=shards, bounds=bounds, n_leaks=len(keep), scale=scale))
    return tb.build()


CONFIGS["c5_sharded"] = c5_sharded


# ---------------------------------------------------------------------------
# NEXT-2: multi-threaded variants of any trace
# ---------------------------------------------------------------------------
def with_threads(tr: Trace, n_threads: int, sync_frac: float = 0.01, seed: int = 0x7C) -> Trace:
    """Every event of `tr` is issued by a uniformly random one of n_threads
    threads, and SYNC events (each by a random thread) are inserted at a
    `sync_frac` fraction of the positions; seqs are renumbered 1..n (the call
    order is unchanged, so every non-SYNC event keeps its meaning)."""
    rng = np.random.default_rng(seed)
    n = len(tr.events)
    ns = int(round(n * sync_frac))
    at = np.sort(rng.integers(0, n + 1, ns))
    syncs = np.zeros(ns, EVENT_DTYPE)
    syncs["op"] = OP_SYNC
    ev = np.insert(tr.events, at, syncs)
    ev["seq"] = np.arange(1, len(ev) + 1, dtype=np.uint64)
    th = rng.integers(0, n_threads, len(ev)).astype(np.uint32)
    return Trace(f"{tr.name}_t{n_threads}", ev, tr.blob, tr.host_base, tr.host_size, dict(tr.meta), th)


# ---------------------------------------------------------------------------
# NEXT-4: host regions scattered over the 64-bit space (sparse host map)
# ---------------------------------------------------------------------------
def sparse_regions(seed: int = 0, n_regions: int = 6, region: int = 256 * KiB, n_copies: int = 400):
    """The same program twice: `dense` keeps its n_regions host regions packed
    in one window [H0, H0 + n_regions*region) (what the dense oracle can
    represent), `sparse` places region k at bases[k], scattered over the
    64-bit address space (64 KiB aligned).  Every host range of every event
    stays inside one region, so the two programs have the same meaning: the
    verdicts (logical offsets, counts, flags) must be identical.
    Returns (dense, sparse, bases, region)."""
    rng = np.random.default_rng(seed + 0x5AA5)
    H0 = 1 << 20
    tb = TraceBuilder(f"regions{seed}", H0, n_regions * region)
    allocs = [tb.malloc(int(rng.integers(256, 64 * KiB))) for _ in range(24)]
    sizes = {}
    for k in range(n_regions):   # fragmented regions: DEFINED / UNDEFINED runs with NOACCESS gaps
        o = 0
        while o < region:
            n = int(rng.integers(64, 24 * KiB))
            n = min(n, region - o)
            st = int(rng.choice([DEFINED, UNDEFINED, NOACCESS], p=[0.6, 0.25, 0.15]))
            tb.mark(H0 + k * region + o, n, st)
            o += n
        for _ in range(4):
            a = int(rng.integers(0, region - 64))
            tb.setv(H0 + k * region + a, rng.integers(0, 256, int(rng.integers(1, 64)), dtype=np.uint8).tobytes())
    for b in allocs:
        sizes[b] = None
    for _ in range(n_copies):
        k = int(rng.integers(n_regions))
        d = allocs[int(rng.integers(len(allocs)))]
        kind = int(rng.choice([HTOD, DTOH], p=[0.55, 0.45]))
        if rng.random() < 0.3:   # 2D, host side pitched inside the region
            w = int(rng.integers(1, 512)); h = int(rng.integers(1, 32)); pitch = w + int(rng.integers(0, 256))
            span = (h - 1) * pitch + w
            a = H0 + k * region + int(rng.integers(0, region - span))
            if kind == HTOD:
                tb.copy2d(HTOD, w, h, d, 0, 0, w, a, 0, 0, pitch)
            else:
                tb.copy2d(DTOH, w, h, a, 0, 0, pitch, d, 0, 0, w)
        else:
            n = int(rng.integers(1, 32 * KiB))
            a = H0 + k * region + int(rng.integers(0, region - n))
            if kind == HTOD:
                tb.copy1d(HTOD, d, a, n)
            else:
                tb.copy1d(DTOH, a, d, n)
        if rng.random() < 0.1:
            tb.mark(H0 + k * region + int(rng.integers(0, region - 4096)), 4096,
                    int(rng.choice([DEFINED, UNDEFINED, NOACCESS])))
    dense = tb.build()
    # scattered bases: distinct 64 KiB-aligned slots far apart
    slots = rng.choice(1 << 30, n_regions, replace=False)          # 8 MiB slots over 2^53 bytes
    bases = [((1 << 32) + int(s) * (1 << 23) + int(rng.integers(0, 1 << 22))) & ~0xFFFF for s in slots]

    def move(x):
        k = (int(x) - H0) // region
        return bases[k] + (int(x) - H0 - k * region)

    ev = dense.events.copy()
    for i, e in enumerate(ev):
        op = int(e["op"])
        if op in (OP_MARK, OP_SETV):
            ev[i]["dst"] = move(e["dst"])
        elif op == OP_COPY:
            p = "src" if int(e["kind"]) == HTOD else "dst"
            ev[i][p] = move(e[p])
    sparse = Trace(dense.name + "_sparse", ev, dense.blob, bases[0] & ~0xFFFF, region, dict(dense.meta),
                   dense.threads)
    return dense, sparse, bases, region


# ---------------------------------------------------------------------------
# R-10: copies larger than any window (no size cap: INVALID_RANGE only on
# 64-bit overflow, S:49 / S:58 / S:65)
# ---------------------------------------------------------------------------
HUGE_D = (100, 525318, 1056778, 2000000, 3698788)   # undefined bytes: offsets from HUGE_START


def huge_copies() -> Trace:
    """A 4 MiB window, fully DEFINED except five undefined bytes at
    HUGE_START + d (d in HUGE_D), one 2 TiB device allocation, and copies of
    2^38 + 1 and 2^40 logical bytes (1D and pitched 2D) whose host side starts
    inside the window (or 4 KiB before it), plus one whose W*H overflows 64
    bits.  The expected verdicts are derived by hand in
    tests/test_oracle_pins.py::test_huge_copies_hand_derived."""
    H0, S = 1 << 20, 4 * MiB
    tb = TraceBuilder("huge", H0, S)
    start = H0 + 4096
    tb.mark(H0, S, DEFINED)
    for k, d in enumerate(HUGE_D):
        tb.setv(start + d, bytes([0x01 << k]))
    dev = 1 << 44
    tb.register(dev, 1 << 41)
    wa, ha, pa = 525313, 523265, 528384                 # 2^38 + 1 = 525313 * 523265, pitch > W
    wb, hb, pb = 1 << 20, 1 << 20, (1 << 20) + (1 << 16)   # 2^40
    c = {}
    c["1d_2^38+1"] = tb.copy1d(HTOD, dev, start, (1 << 38) + 1)
    c["1d_2^40"] = tb.copy1d(HTOD, dev, start, 1 << 40)
    c["2d_2^38+1"] = tb.copy2d(HTOD, wa, ha, dev, 0, 0, wa, start, 0, 0, pa)
    c["2d_2^40"] = tb.copy2d(HTOD, wb, hb, dev, 0, 0, wb, start, 0, 0, pb)
    c["1d_before"] = tb.copy1d(HTOD, dev, H0 - 4096, 1 << 40)
    c["dtoh_1d_2^40"] = tb.copy1d(DTOH, start, dev, 1 << 40)
    c["dtoh_2d_2^40"] = tb.copy2d(DTOH, wb, hb, start, 0, 0, pb, dev, 0, 0, wb)
    c["overflow"] = tb.copy2d(HTOD, 1 << 33, 1 << 32, dev, 0, 0, 0, start, 0, 0, 0)
    tb.meta.update(dict(start=start, dev=dev, copies=c))
    return tb.build()


def overlap_rows(seed: int = 0, W: int = 4096, pitch: int = 64, H: int = 20000, dtoh: bool = False) -> Trace:
    """BAD_PITCH 2D copies whose rows overlap (pitch < W): every physical byte
    belongs to several rows and is counted once per row (R-12).  A 4 MiB
    window, DEFINED with scattered undefined bytes and a NOACCESS hole placed
    by the seed; one HtoD (or DtoH) of W x H logical bytes plus one with pitch
    0 (all rows on the same bytes)."""
    rng = np.random.default_rng(seed + 0x0E1A)
    H0, S = 1 << 20, 4 * MiB
    tb = TraceBuilder(f"overlap{seed}", H0, S)
    tb.mark(H0, S, DEFINED)
    start = H0 + 4096 + int(rng.integers(0, 4096))
    span = (H - 1) * pitch + W
    for _ in range(8):
        tb.setv(start + int(rng.integers(0, span)), bytes([int(rng.integers(1, 256))]))
    if rng.random() < 0.5:                                    # a NOACCESS hole somewhere in the span
        tb.mark(start + int(rng.integers(0, span)), int(rng.integers(1, 64)), NOACCESS)
    dev = tb.malloc(1 << 30)
    if dtoh:
        tb.copy2d(DTOH, W, H, start, 0, 0, pitch, dev, 0, 0, W)
        tb.copy2d(DTOH, W, H, start, 0, 0, 0, dev, 0, 0, W)
    else:
        tb.copy2d(HTOD, W, H, dev, 0, 0, W, start, 0, 0, pitch)
        tb.copy2d(HTOD, W, H, dev, 0, 0, W, start, 0, 0, 0)
    tb.meta.update(dict(start=start, dev=dev))
    return tb.build()


# ---------------------------------------------------------------------------
# Random medium traces: the scan's work-splitting boundaries (4 KiB
# HtoD tiles, 32 KiB DtoH tiles / chunk-map units, 128 KiB split threshold)
# ---------------------------------------------------------------------------
SPLIT_BOUNDARIES = (4 * KiB, 32 * KiB, 128 * KiB)


def random_medium(seed: int, n_copies: int = 120, window: int = 64 * MiB, host_base: int = 0x4000_0000) -> Trace:
    """Copies up to 8 MiB with unaligned starts, 2D copies with hundreds of
    rows, ranges straddling either window edge, and violations planted one
    byte before / at / after multiples of 4 KiB, 32 KiB and 128 KiB -- both as
    absolute shard offsets (tile and block edges) and as logical offsets from a
    copy's start (piece and split edges).  Setup first (marks, planted bytes),
    then the copies; DtoH applies make later epochs differ."""
    rng = np.random.default_rng(seed + 0x3ED1)
    host_base += int(rng.integers(0, 16)) * 4096
    tb = TraceBuilder(f"medium{seed}", host_base, window)
    tb.mark(host_base, window, DEFINED)
    for _ in range(int(rng.integers(0, 6))):                       # UNDEFINED runs (malloc'ed, unwritten)
        a = int(rng.integers(0, window - MiB))
        tb.mark(host_base + a, int(rng.integers(1, 256 * KiB)), UNDEFINED)
    def boundary_offset(limit):
        b = int(rng.choice(SPLIT_BOUNDARIES))
        k = int(rng.integers(1, max(2, limit // b)))
        return k * b + int(rng.integers(-1, 2))
    # planted at absolute shard offsets around tile / block edges
    for _ in range(60):
        q = min(max(boundary_offset(window), 0), window - 1)
        if rng.random() < 0.7:
            tb.setv(host_base + q, bytes([int(rng.integers(1, 256))]))
        else:
            tb.mark(host_base + q, int(rng.integers(1, 3)), NOACCESS)
    allocs = [tb.malloc(32 * MiB) for _ in range(6)]
    copies = []
    for _ in range(n_copies):
        kind = int(rng.choice([HTOD, DTOH], p=[0.55, 0.45]))
        u = rng.random()
        if u < 0.25:                                               # sizes right at the boundaries
            n = max(boundary_offset(8 * MiB), 0)
        else:
            n = int(_log_uniform(rng, 1, 8 * MiB, 1)[0])
        two_d = rng.random() < 0.3
        if two_d:
            w = int(_log_uniform(rng, 1, 64 * KiB, 1)[0])
            h = int(rng.integers(2, 700))
            while w * h > 8 * MiB and h > 2:
                h //= 2
            pitch = w + int(rng.choice([0, int(rng.integers(1, 4096))]))
            x = int(rng.integers(0, 64))
            if rng.random() < 0.06:
                pitch = int(rng.integers(1, max(w + x, 2)))        # BAD_PITCH (may overlap rows)
            else:
                pitch += x
            span = (h - 1) * pitch + w + x
        else:
            w, h, pitch, x, span = n, 1, n, 0, n
        v = rng.random()
        if v < 0.06:                                               # straddles the window end
            start = host_base + window - int(rng.integers(1, max(2, span)))
        elif v < 0.1:                                              # starts below the window
            start = host_base - int(rng.integers(1, 8 * KiB))
        else:
            start = host_base + int(rng.integers(0, max(1, window - span)))
        if rng.random() < 0.35 and w * h > 2:                      # planted at a logical boundary of this copy
            o = min(max(boundary_offset(w * h), 0), w * h - 1)
            r, c = divmod(o, w)
            xaddr = start + x + r * pitch + c
            if host_base <= xaddr < host_base + window:
                if kind == HTOD and rng.random() < 0.6:
                    tb.setv(xaddr, bytes([int(rng.integers(1, 256))]))
                else:
                    tb.mark(xaddr, 1, NOACCESS)
        dev = allocs[int(rng.integers(len(allocs)))]
        doff = int(rng.integers(0, 32 * MiB))
        if rng.random() < 0.8:                                     # fits (else TooSmall)
            doff = int(rng.integers(0, max(1, 32 * MiB - w * h - 1)))
        copies.append((kind, w, h, pitch, x, start, dev + doff))
    for kind, w, h, pitch, x, start, dptr in copies:
        if h == 1 and x == 0 and pitch == w:
            if kind == HTOD:
                tb.copy1d(HTOD, dptr, start, w)
            else:
                tb.copy1d(DTOH, start, dptr, w)
        elif kind == HTOD:
            tb.copy2d(HTOD, w, h, dptr, 0, 0, w, start, x, 0, pitch)
        else:
            tb.copy2d(DTOH, w, h, start, x, 0, pitch, dptr, 0, 0, w)
    return tb.build()


def pingpong_trace(seed: int, n_copies: int = 240, n_bufs: int = 12) -> Trace:
    """DtoH -> HtoD ping-pongs on a few host buffers (the fused batch planner's
    CG_CHECK_AFTER / CG_APPLY_AFTER / CG_APPLY_LAST cases): 1D and
    2D copies over partly overlapping slices of buffers that start UNDEFINED
    (or DEFINED with planted bytes), DtoH copies that fail (device source too
    small or unallocated: nothing becomes defined) next to ones that succeed,
    and now and then a 2 MiB HtoD (too large for the late pass: a cut)."""
    rng = np.random.default_rng(seed + 0x9090)
    H0, S = 1 << 30, 8 * MiB
    tb = TraceBuilder(f"pingpong{seed}", H0, S)
    tb.mark(H0, S, UNDEFINED)
    slot = S // n_bufs // 4096 * 4096
    bufs = []
    for b in range(n_bufs):
        start = H0 + b * slot + int(rng.integers(0, 64))
        length = int(_log_uniform(rng, 64, min(slot - 128, 96 * KiB), 1)[0])
        if rng.random() < 0.4:
            tb.mark(start, length, DEFINED)
            for _ in range(int(rng.integers(0, 3))):
                tb.setv(start + int(rng.integers(0, length)), bytes([int(rng.integers(1, 256))]))
        bufs.append((start, length))
    dev = tb.malloc(4 * MiB)
    small = tb.malloc(256)
    for _ in range(n_copies):
        start, length = bufs[int(rng.integers(len(bufs)))]
        kind = int(rng.choice([HTOD, DTOH]))
        if kind == HTOD and rng.random() < 0.03:                   # too large for the late pass
            tb.copy1d(HTOD, dev, H0 + int(rng.integers(0, S - 2 * MiB)), 2 * MiB)
            continue
        a = int(rng.integers(0, length))
        n = int(rng.integers(1, length - a + 1))
        src_dev = dev
        u = rng.random()
        if kind == DTOH and u < 0.15:
            src_dev = small if n > 256 else 1 << 52                # TooSmall / not allocated: the copy fails
        if rng.random() < 0.25 and n >= 8:                          # 2D over the slice
            w = int(rng.integers(1, min(n, 4096) + 1))
            h = max(1, min(64, n // max(w, 1)))
            pitch = w + int(rng.integers(0, 64))
            while (h - 1) * pitch + w > length - a and h > 1:
                h -= 1
            if kind == HTOD:
                tb.copy2d(HTOD, w, h, dev, 0, 0, w, start + a, 0, 0, pitch)
            else:
                tb.copy2d(DTOH, w, h, start + a, 0, 0, pitch, src_dev, 0, 0, w)
        elif kind == HTOD:
            tb.copy1d(HTOD, dev, start + a, n)
        else:
            tb.copy1d(DTOH, start + a, src_dev, n)
    tb.meta.update(dict(bufs=bufs, dev=dev))
    return tb.build()
