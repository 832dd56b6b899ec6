"""An independent brute-force flat model ("an independent
brute-force checker using dense per-byte A-bit and per-bit V-bit arrays").

Used ONLY to pin the C oracle on tiny inputs.  It shares nothing with the
oracle (different language, different algorithms): the allocation list is a
``bisect``-searched sorted list, the host side is evaluated with numpy index
arithmetic (``np.add.outer`` over rows x columns), first offsets come from
``np.flatnonzero`` and counts from ``np.count_nonzero``.  Memory: dense
unpacked arrays, so keep windows small (<= a few MiB).
"""
from __future__ import annotations

import bisect

import numpy as np

NONE = (1 << 64) - 1
U64 = (1 << 64) - 1
FLAG = dict(DST_NA=1, DST_SMALL=2, SRC_NA=4, SRC_SMALL=8, HOST_UNADDR=16,
            HOST_UNDEF=32, BAD_PITCH=64, INVALID_RANGE=128, BAD_KIND=256, CONCURRENT=512)


class _PagedLast:
    """NEXT-2: per-byte "id of the last recorded access" over a sparse 64-bit
    address space (dense 4 KiB numpy pages, -1 = never accessed)."""
    PAGE = 4096

    def __init__(self):
        self.pages: dict = {}

    def _chunks(self, lo, hi):
        while lo < hi:
            pg, off = divmod(lo, self.PAGE)
            n = min(hi - lo, self.PAGE - off)
            yield pg, off, n
            lo += n

    def max_id(self, lo, hi) -> int:
        m = -1
        for pg, off, n in self._chunks(lo, hi):
            a = self.pages.get(pg)
            if a is not None:
                m = max(m, int(a[off:off + n].max()))
        return m

    def paint(self, lo, hi, ident):
        for pg, off, n in self._chunks(lo, hi):
            a = self.pages.setdefault(pg, np.full(self.PAGE, -1, np.int64))
            a[off:off + n] = ident


class FlatModel:
    def __init__(self, h0: int, s: int, undef_is_error: bool = False, track: bool = False, conc: bool = False):
        self.h0, self.s = h0, s
        self.conc = conc                          # NEXT-2 per-byte last-access model
        self.last_acc = (_PagedLast(), _PagedLast())   # host space, device space
        self.stamps: list = []                    # id -> (thread, seq, is_write)
        self.syncs: dict = {}                     # thread -> sorted sync seqs
        self.track = track
        self.dv: dict = {}                        # base -> numpy V-bytes of the allocation (NEXT-1)
        self.arrays: dict = {}                    # handle -> total bytes (NEXT-3)
        self.av: dict = {}                        # handle -> numpy V-bytes of the array (track mode)
        self.a = np.zeros(s, bool)               # unpacked A
        self.v = np.full(s, 0xFF, np.uint8)
        self.bases: list = []                     # sorted live bases
        self.info: dict = {}                      # base -> (size, seq)
        self.last = 0
        self.uie = undef_is_error

    # packed A in the on-device format (R-2) for state comparison
    def packed_a(self) -> np.ndarray:
        return np.packbits(self.a, bitorder="little")

    def _win(self, addr, n):
        return addr >= self.h0 and addr + n <= self.h0 + self.s

    def mark(self, addr, n, state):
        if state > 2:
            return 1
        if n == 0:
            return 0
        if not self._win(addr, n):
            return 1
        i = addr - self.h0
        self.a[i:i + n] = state != 0
        self.v[i:i + n] = 0 if state == 2 else 0xFF
        return 0

    def setv(self, addr, data):
        n = len(data)
        if n == 0:
            return 0
        if not self._win(addr, n):
            return 1
        i = addr - self.h0
        if not self.a[i:i + n].all():
            return 1
        self.v[i:i + n] = np.frombuffer(bytes(data), np.uint8)
        return 0

    def _containing(self, x):
        k = bisect.bisect_right(self.bases, x) - 1
        if k >= 0:
            b = self.bases[k]
            if x < b + self.info[b][0]:
                return b
        return None

    def register(self, base, size, seq):
        if seq <= self.last or size == 0 or base == 0 or base + size > U64:
            return 1
        k = bisect.bisect_left(self.bases, base)
        if k < len(self.bases) and self.bases[k] < base + size:
            return 1
        if k > 0 and self.bases[k - 1] + self.info[self.bases[k - 1]][0] > base:
            return 1
        self.bases.insert(k, base)
        self.info[base] = (size, seq)
        if self.track:
            self.dv[base] = np.full(size, 0xFF, np.uint8)
        self.last = seq
        return 0

    def free(self, ptr, seq):
        if seq <= self.last or ptr not in self.info:
            return 1
        self.bases.remove(ptr)
        del self.info[ptr]
        self.dv.pop(ptr, None)
        self.last = seq
        return 0

    @staticmethod
    def array_bytes(w, h, d, fmt, ch):
        if w == 0 or fmt > 7 or ch not in (1, 2, 4):
            return 0
        t = w * max(h, 1) * max(d, 1) * [1, 2, 4, 1, 2, 4, 2, 4][fmt] * ch
        return t if t <= U64 else 0

    def register_array(self, handle, total, seq):
        if seq <= self.last or total == 0 or handle in self.arrays:
            return 1
        self.arrays[handle] = total
        if self.track:                            # S:252 per-array shadow, fresh = undefined
            self.av[handle] = np.full(total, 0xFF, np.uint8)
        self.last = seq
        return 0

    def free_array(self, handle, seq):
        if seq <= self.last or handle not in self.arrays:
            return 1
        del self.arrays[handle]
        self.av.pop(handle, None)
        self.last = seq
        return 0

    def array_copy(self, e):
        kind, w, h = int(e["kind"]), int(e["width"]), int(e["height"])
        htoa = kind == 4
        out = dict(first_unaddr=NONE, first_undef=NONE, undef_count=0, dst_expected=0,
                   dst_found=0, src_expected=0, src_found=0, flags=0, status=0)
        hs = "src" if htoa else "dst"
        aside = "dst" if htoa else "src"
        handle, off = int(e[aside]), int(e[aside + "_x"])
        base, x, y, pitch = int(e[hs]), int(e[hs + "_x"]), int(e[hs + "_y"]), int(e[hs + "_pitch"])
        if pitch < w + x:
            out["flags"] |= FLAG["BAD_PITCH"]
        start = base + y * pitch + x
        span = 0 if (w == 0 or h == 0) else (h - 1) * pitch + w
        nb = w * h
        hok, nbok, aok = start + span <= U64, nb <= U64, off + nb <= U64   # R-10: overflow only
        if not (hok and nbok and aok):
            out["flags"] |= FLAG["INVALID_RANGE"]
        P = "DST" if htoa else "SRC"
        if aok and nbok:
            if handle not in self.arrays:
                out["flags"] |= FLAG[P + "_NA"]
            elif off + nb > self.arrays[handle]:
                out["flags"] |= FLAG[P + "_SMALL"]
                tot = self.arrays[handle]
                out[aside + "_expected"], out[aside + "_found"] = nb, (tot - off if off < tot else 0)
        if hok and nbok and w and h:
            xs = self._host_index(start, pitch, w, h)
            inwin = np.array([(self.h0 <= xx < self.h0 + self.s) for xx in xs], bool)
            idx = np.array([xx - self.h0 if iw else 0 for xx, iw in zip(xs, inwin)], np.int64)
            addr = inwin & self.a[idx]
            bad = np.flatnonzero(~addr)
            if len(bad):
                out["first_unaddr"] = int(bad[0])
            if htoa:
                und = addr & (self.v[idx] != 0)
                u = np.flatnonzero(und)
                out["undef_count"] = int(np.count_nonzero(und))
                if len(u):
                    out["first_undef"] = int(u[0])
        if out["first_unaddr"] != NONE:
            out["flags"] |= FLAG["HOST_UNADDR"]
        if out["undef_count"] and out["first_unaddr"] == NONE:
            out["flags"] |= FLAG["HOST_UNDEF"]
        err = out["flags"] & ~(0 if self.uie else FLAG["HOST_UNDEF"])
        out["status"] = 1 if err else 0
        if out["status"] == 0 and w and h:
            idx = np.array([xx - self.h0 for xx in self._host_index(start, pitch, w, h)], np.int64)
            if self.track:                        # V-bits move host <-> the array's shadow
                if htoa:
                    self.av[handle][off:off + nb] = self.v[idx]
                else:
                    self.v[idx] = self.av[handle][off:off + nb]
            elif not htoa:
                self.v[idx] = 0
        return out

    def leaks(self):
        return [(b, self.info[b][0], self.info[b][1]) for b in self.bases]

    def _host_index(self, start, pitch, w, h):
        """addresses of the logical bytes o = r*w + c, in o order"""
        r = np.arange(h, dtype=object) if h else np.zeros(0, dtype=object)
        c = np.arange(w, dtype=object) if w else np.zeros(0, dtype=object)
        return np.add.outer(np.asarray(r) * pitch + start, np.asarray(c)).ravel()

    def copy(self, e):
        kind, w, h = int(e["kind"]), int(e["width"]), int(e["height"])
        out = dict(first_unaddr=NONE, first_undef=NONE, undef_count=0, dst_expected=0,
                   dst_found=0, src_expected=0, src_found=0, flags=0, status=0)
        if kind in (4, 5):
            return self.array_copy(e)
        if kind not in (1, 2, 3):
            out["flags"] = FLAG["BAD_KIND"]; out["status"] = 1
            return out
        sides = {}
        for p in ("dst", "src"):
            base, x, y, pitch = (int(e[p]), int(e[p + "_x"]), int(e[p + "_y"]), int(e[p + "_pitch"]))
            if pitch < w + x:
                out["flags"] |= FLAG["BAD_PITCH"]
            start = base + y * pitch + x
            span = 0 if (w == 0 or h == 0) else (h - 1) * pitch + w
            sides[p] = (start, span, pitch, start + span <= U64)
        bytes_ok = w * h <= U64               # R-10: overflow only
        if not (sides["dst"][3] and sides["src"][3] and bytes_ok):
            out["flags"] |= FLAG["INVALID_RANGE"]
        dev = {1: ["dst"], 2: ["src"], 3: ["dst", "src"]}[kind]
        for p in dev:
            start, span, _, ok = sides[p]
            if not ok:
                continue
            b = self._containing(start)
            P = p.upper()
            if b is None:
                out["flags"] |= FLAG[P + "_NA"]
            else:
                avail = b + self.info[b][0] - start
                if avail < span:
                    out["flags"] |= FLAG[P + "_SMALL"]
                    out[p + "_expected"], out[p + "_found"] = span, avail
        hp = {1: "src", 2: "dst", 3: None}[kind]
        if hp is not None and sides[hp][3] and bytes_ok and w and h:
            start, _, pitch, _ = sides[hp]
            xs = self._host_index(start, pitch, w, h)
            inwin = np.array([(self.h0 <= x < self.h0 + self.s) for x in xs], bool)
            idx = np.array([x - self.h0 if iw else 0 for x, iw in zip(xs, inwin)], np.int64)
            addr = inwin & self.a[idx]
            bad = np.flatnonzero(~addr)
            if len(bad):
                out["first_unaddr"] = int(bad[0])
            if kind == 1:
                und = addr & (self.v[idx] != 0)
                u = np.flatnonzero(und)
                out["undef_count"] = int(np.count_nonzero(und))
                if len(u):
                    out["first_undef"] = int(u[0])
        if out["first_unaddr"] != NONE:
            out["flags"] |= FLAG["HOST_UNADDR"]
        if out["undef_count"] and out["first_unaddr"] == NONE:
            out["flags"] |= FLAG["HOST_UNDEF"]
        err = out["flags"] & ~(0 if self.uie else FLAG["HOST_UNDEF"])
        out["status"] = 1 if err else 0
        if kind == 2 and out["status"] == 0 and w and h and not self.track:
            start, _, pitch, _ = sides["dst"]
            xs = self._host_index(start, pitch, w, h)
            self.v[np.array([x - self.h0 for x in xs], np.int64)] = 0
        if self.track and out["status"] == 0 and w and h:
            def read(p):
                start, _, pitch, _ = sides[p]
                xs = self._host_index(start, pitch, w, h)
                if p == {1: "src", 2: "dst", 3: None}[kind]:
                    return self.v[np.array([x - self.h0 for x in xs], np.int64)].copy()
                b = self._containing(start)
                return self.dv[b][np.array([x - b for x in xs], np.int64)].copy()

            def write(p, vals):
                start, _, pitch, _ = sides[p]
                xs = self._host_index(start, pitch, w, h)
                if kind == 2:
                    self.v[np.array([x - self.h0 for x in xs], np.int64)] = vals
                else:
                    b = self._containing(start)
                    self.dv[b][np.array([x - b for x in xs], np.int64)] = vals
            write("dst", read("src"))    # read everything first: memmove semantics
        return out

    def sync(self, thread, seq):
        bisect.insort(self.syncs.setdefault(thread, []), seq)

    def concurrency(self, e, thread, out):
        """NEXT-2 per byte: the last recorded access of every byte of the new
        access's range; the newest of them decides (R-31..R-34)."""
        kind, w, h = int(e["kind"]), int(e["width"]), int(e["height"])
        acc = {1: [(0, "src", 0), (1, "dst", 1)], 2: [(1, "src", 0), (0, "dst", 1)],
               3: [(1, "src", 0), (1, "dst", 1)], 4: [(0, "src", 0)], 5: [(0, "dst", 1)]}.get(kind, [])
        rng = []
        for space, p, wr in acc:
            start = int(e[p]) + int(e[p + "_y"]) * int(e[p + "_pitch"]) + int(e[p + "_x"])
            span = 0 if (w == 0 or h == 0) else (h - 1) * int(e[p + "_pitch"]) + w
            if span == 0 or start + span > U64:
                continue
            rng.append((space, start, start + span, wr))
        seq = int(e["seq"])
        for space, lo, hi, wr in rng:
            m = self.last_acc[space].max_id(lo, hi)
            if m < 0:
                continue
            pt, ps, pw = self.stamps[m]
            s_list = self.syncs.get(pt, [])
            synced = bisect.bisect_right(s_list, ps) < bisect.bisect_left(s_list, seq)
            if pt != thread and not synced and (pw or wr):
                out["flags"] |= FLAG["CONCURRENT"]
        if out["status"] == 0:
            for space, lo, hi, wr in sorted(rng, key=lambda r: r[3]):   # reads first: a write wins a tie
                self.stamps.append((thread, seq, wr))
                self.last_acc[space].paint(lo, hi, len(self.stamps) - 1)

    def replay(self, events, blob, threads=None):
        verdicts, status = [], []
        for i, e in enumerate(events):
            op = int(e["op"])
            th = int(threads[i]) if threads is not None else 0
            if op == 8:
                self.sync(th, int(e["seq"]))
                status.append(0)
                continue
            if op == 1:
                status.append(self.mark(int(e["dst"]), int(e["width"]), int(e["kind"])))
            elif op == 2:
                off, n = int(e["src"]), int(e["width"])
                status.append(self.setv(int(e["dst"]), bytes(blob[off:off + n])))
            elif op == 3:
                status.append(self.register(int(e["dst"]), int(e["width"]), int(e["seq"])))
            elif op == 4:
                status.append(self.free(int(e["dst"]), int(e["seq"])))
            elif op == 5:
                v = self.copy(e)
                if self.conc:
                    self.concurrency(e, th, v)
                verdicts.append(v)
                status.append(v["status"])
            elif op == 6:
                tot = self.array_bytes(int(e["width"]), int(e["height"]), int(e["dst_x"]), int(e["dst_y"]),
                                       int(e["dst_pitch"]))
                status.append(self.register_array(int(e["dst"]), tot, int(e["seq"])))
            elif op == 7:
                status.append(self.free_array(int(e["dst"]), int(e["seq"])))
        return verdicts, status
