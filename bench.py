#!/usr/bin/env python
"""Benchmark of the batched transfer checker on B200 (BASELINE.json metric:
"shadow GB/s and copy-descriptors/s validated (1/2/4/8 B200, % of HBM peak)").

N=1 (default): one step = one pass of the whole hot path over
the 1M-copy / 100k-allocation configuration (BASELINE.json configs[1], C2):
cg_check_apply (a1-a6, fused) per R-20 epoch + cg_leak_sweep (a8).  The
registry (a7) is built once before timing; its host throughput is reported
separately.  Inputs are resident in HBM when the timed region starts; the
shadow read per step (~8.5 GB) is far larger than the 126 MB L2, so no flush
is needed.  The same line carries `per_config`: C3, C4 and C5 (at one GPU)
through the same measured step.

`value` = algorithmic bytes per step (shadow: HtoD 1.125 B, DtoH check 0.125 B
+ apply 1 B per host byte; descriptors: 96 B read + 64 B verdict written;
SURVEY §8(d)) / device time.  `e2e` = the same through the public host-buffer
entry point cg_check_host_submit / _wait (pinned host descriptors up, dirty
verdicts down, inside the timed region).

N>1 (torchrun): strong scaling on C5 (configs[4], "64 GB host shadow space
sharded across 8 B200"): the same trace on every rank, the window split N
ways, one cg_check_sharded per epoch (NCCL straddler exchange + verdict
gather inside the library); time = max over ranks.  --sharded runs that code
path at N=1 (one NCCL rank), --loopback G with G shards on one GPU.

--impl reference times the CPU oracle (the reference arm of this tier), on
the host's cores, on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "shadow GB/s and copy-descriptors/s validated (1/2/4/8 B200, % of HBM peak)"
UNIT = "GB/s"


def algorithmic_bytes(descs: np.ndarray, verdicts: np.ndarray | None, track: bool = False, two_bit: bool = False):
    """Shadow bytes the method must move: HtoD 1 V-byte + 1/8
    A-byte per host byte; DtoH 1/8 A-byte per host byte for the check and 1
    V-byte written per host byte by the apply when the verdict has no Error.
    With device V-bit tracking (NEXT-1) the apply instead reads and writes one
    V-byte per byte of every error-free copy (HtoD, DtoD, DtoH).  With the
    NEXT-4 2-bit shadow both checks read 0.25 B per host byte and the apply
    writes 0.25 B."""
    nb = descs["width"].astype(np.float64) * descs["height"].astype(np.float64)
    htod = descs["kind"] == 1
    dtoh = descs["kind"] == 2
    okv = np.ones(len(descs), bool) if verdicts is None else verdicts["status"] == 0
    if two_bit:
        return 0.25 * float(nb[htod | dtoh].sum()), 0.25 * float(nb[dtoh & okv].sum())
    check = float(nb[htod].sum()) * 1.125 + float(nb[dtoh].sum()) * 0.125
    if track:
        return check, 2.0 * float(nb[okv & (descs["kind"] >= 1) & (descs["kind"] <= 3)].sum())
    apply = float(nb[dtoh & okv].sum())
    return check, apply


def fused_apply_bytes(descs: np.ndarray, verdicts: np.ndarray, max_descs: int, two_bit: bool = False) -> float:
    """Bytes the fused scan writes itself in cg_check_apply: DtoH descriptors
    with status OK, contiguous and not split by the scan's grouping (weight at
    most one group, or inside one group); the rest go to the residual pass.  Replicates the
    library's plan (weight = 256 + host units; never split below Trule =
    max(128 KiB, T), T = max(32 KiB, ceil(total / max(2^20, 2 max_descs)))) for accounting only."""
    nb = descs["width"].astype(np.uint64) * descs["height"].astype(np.uint64)
    if two_bit:
        units = np.where((descs["kind"] == 1) | (descs["kind"] == 2), (nb + np.uint64(3)) // np.uint64(4), 0)
    else:
        units = np.where(descs["kind"] == 1, nb, np.where(descs["kind"] == 2, (nb + np.uint64(7)) // np.uint64(8), 0))
    w = np.uint64(256) + units.astype(np.uint64)
    P = np.concatenate([[0], np.cumsum(w, dtype=np.uint64)])
    total = int(P[-1])
    chunks = max(1 << 20, 2 * max_descs)
    T = max(32 * 1024, -(-total // chunks))
    whole = (P[1:] - P[:-1]) <= max(T, 128 * 1024)   # descriptors of at most Trule weight are never split
    contig = (descs["height"] == 1) | (descs["width"] == descs["dst_pitch"])
    ok = (descs["kind"] == 2) & (verdicts["status"] == 0) & contig & whole
    return float(nb[ok].astype(np.float64).sum()) * (0.25 if two_bit else 1.0)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """Samples SM clocks and throttle reasons with NVML during the timed region."""

    def __init__(self, device: int, period: float = 0.005):
        self.device, self.period = device, period
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            names = {
                "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
                "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
                "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
                "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
                "hw_power_brake": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
            }

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for k, bit in names.items():
                            if r & bit:
                                self.reasons.add(k)
                    except Exception:
                        pass
                    time.sleep(self.period)
            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
        except Exception as e:  # NVML missing: report nothing rather than guess
            self.error = str(e)
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


C2_SHARD = 8 << 30        # per-rank window of the weak-scaling C2 workload (7.94 GiB used)


def workload_name(config: str) -> str:
    """config.workload of both arms"""
    if config == "c2_small":
        return ("c2_small (BASELINE.json configs[1]: 1M small copies 64 B-64 KiB log-uniform "
                "vs a 100k-entry allocation table, 1% injected violations)")
    return config


_TRACES = {}


def make_workload(name: str, rank: int = 0, scale: float = 1.0):
    key = (name, rank, scale)
    if key not in _TRACES:
        _TRACES.clear()   # one trace at a time (C5's is 1.1 GB)
        _TRACES[key] = _make_workload(name, rank, scale)
    return _TRACES[key]


def _make_workload(name: str, rank: int = 0, scale: float = 1.0):
    """Rank r's workload.  Weak scaling: rank r's host buffers live in shard r
    of a global window [2^32, 2^32 + world * 8 GiB); its copies, allocations and
    verdicts are its own."""
    import tracegen as tg
    if name == "c2_small":
        n = max(1000, int(1_000_000 * scale))
        shard = C2_SHARD if scale >= 1.0 else None
        return tg.c2_small(seed=13100902 + rank, n_copies=n, n_allocs=max(1000, int(100_000 * min(scale, 1.0))),
                           host_base=(1 << 32) + rank * C2_SHARD, host_size=shard)
    if name == "c3_single":
        return tg.c3_single(seed=13100903 + rank, size=int((8 << 30) * scale) // (1 << 20) * (1 << 20))
    if name == "c4_pitched":
        return tg.c4_pitched(seed=13100904 + rank, n_copies=max(1000, int(100_000 * scale)))
    if name == "c5_sharded":
        return tg.c5_sharded(seed=13100905 + rank, scale=scale)
    raise SystemExit(f"unknown config {name}")


def setup_checker(cg, tr, device: int, host_staging: bool, rank: int = 0, world: int = 1, track: bool = False,
                  shadow_format: int = 0):
    """Replays the non-copy events (host marks, V-bytes, registry) and returns
    the checker and the copy descriptors (host array).  With world > 1 the
    context holds shard `rank` of the global window."""
    from paper_1310_0901_b200.replay import events_to_descs
    ev = tr.events
    copies = ev[ev["op"] == 5]
    nreg = int(np.count_nonzero(ev["op"] == 3))
    if world > 1:
        gbase = tr.host_base - rank * tr.host_size
        chk = cg.Checker(gbase, world * tr.host_size, shard_base=tr.host_base, shard_size=tr.host_size,
                         max_descs=max(len(copies), 1024), max_allocs=max(nreg, 1024), device=device,
                         host_staging=host_staging, shadow_format=shadow_format)
    else:
        regs = ev[ev["op"] == 3]
        pool = int(regs["width"].astype(np.int64).sum()) + 256 * len(regs) + (1 << 20) if track else 0
        chk = cg.Checker(tr.host_base, tr.host_size, max_descs=max(len(copies), 1024),
                         max_allocs=max(nreg, 1024), device=device, host_staging=host_staging, dev_vsize=pool,
                         shadow_format=shadow_format)
    setup = ev[ev["op"] != 5]
    t0 = time.perf_counter()
    cg.replay_events(chk, setup, tr.blob)
    t_setup = time.perf_counter() - t0
    return chk, events_to_descs(copies), t_setup, nreg


def registry_rate(cg, tr, device):
    """a7 host throughput: registry events per second through the C ABI, one
    call per event (cg_register_alloc / cg_free from Python) and in one
    cg_registry_batch call."""
    ev = tr.events
    regs = ev[(ev["op"] == 3) | (ev["op"] == 4)]
    out = {}
    for mode in ("per_call", "batch"):
        chk = cg.Checker(tr.host_base, 1 << 20 if tr.host_size > (1 << 20) else tr.host_size,
                         max_descs=1024, max_allocs=max(len(regs), 1024), device=device)
        t0 = time.perf_counter()
        if mode == "batch":
            re = np.zeros(len(regs), cg.REG_EVENT_DTYPE)
            re["op"] = np.where(regs["op"] == 3, cg.CG_REG_ALLOC, cg.CG_REG_FREE)
            re["seq"], re["addr"], re["size"] = regs["seq"], regs["dst"], regs["width"]
            chk.registry_batch(re)
        else:
            for e in regs:
                if e["op"] == 3:
                    chk.register_alloc(int(e["dst"]), int(e["width"]), int(e["seq"]))
                else:
                    chk.free(int(e["dst"]), int(e["seq"]))
        dt = time.perf_counter() - t0
        chk.close()
        out[mode] = len(regs) / dt if dt > 0 else None
    return out


def run_ours(args, rank, world, device, config=None, steps=None, warmup=None, e2e_on=None, extras=True):
    """One workload: setup (untimed), warm-up, `steps` timed steps, e2e; the
    JSON fields of the line.  config / steps / warmup / e2e_on override args
    (the per_config runs of the default line)."""
    import torch
    import paper_1310_0901_b200 as cg

    torch.cuda.set_device(device)
    config = config or args.config
    steps = steps or args.steps
    warmup = warmup or args.warmup
    no_e2e = args.no_e2e if e2e_on is None else not e2e_on
    tr = make_workload(config, rank, args.scale)
    two_bit = args.shadow in ("2bit", "sparse")
    chk, descs, t_setup, nreg = setup_checker(cg, tr, device, host_staging=not no_e2e, rank=rank, world=world,
                                              track=args.track,
                                              shadow_format={"bytes": 0, "2bit": 1, "sparse": 2}[args.shadow])
    n = len(descs)
    stream = torch.cuda.current_stream()
    d_out = torch.empty(n * 64, dtype=torch.uint8, device=device)
    nalloc = nreg
    d_leaks = torch.empty(max(nalloc, 1) * 24, dtype=torch.uint8, device=device)
    d_cnt = torch.zeros(1, dtype=torch.int64, device=device)

    # fused (cg_check_apply): the batches of cg_plan_batches_fused (one for
    # every config, C5's ping-pongs included), which marks
    # the DtoH copies an HtoD of their batch reads CG_APPLY_AFTER and the HtoD
    # copies that read an earlier DtoH's bytes CG_CHECK_AFTER, so that a DtoH ->
    # HtoD ping-pong no longer ends the batch (a DtoH that then writes such an
    # HtoD's bytes is applied after the late checks, CG_APPLY_LAST); unfused /
    # tracking: the R-20 epochs of cg_plan_batches (host planning, untimed)
    fused = not args.unfused and not args.track
    descs = np.ascontiguousarray(descs)
    cuts = [0] + [int(c) for c in (cg.plan_batches_fused(descs) if fused else cg.plan_batches(descs))]
    epochs = [(a, b) for a, b in zip(cuts[:-1], cuts[1:]) if b > a]
    efused = [fused for _ in epochs]
    n_after = int(np.count_nonzero(descs["reserved"] & cg.CG_APPLY_AFTER))
    n_late = int(np.count_nonzero(descs["reserved"] & cg.CG_CHECK_AFTER))
    n_last = int(np.count_nonzero(descs["reserved"] & cg.CG_APPLY_LAST))
    d_descs = cg.to_device_descs(descs, device)
    waves = []   # NEXT-1: per epoch, the device index lists of its propagation waves (cg_plan_waves)
    t_waves = 0.0
    if args.track:
        t0 = time.perf_counter()
        for a, b in epochs:
            waves.append(cg.Waves(descs[a:b], device))
        t_waves = time.perf_counter() - t0

    def check_epochs():
        for k, ((a, b), fu) in enumerate(zip(epochs, efused)):
            dd, dv = d_descs[a * 96:b * 96], d_out[a * 64:b * 64]
            if args.track:      # NEXT-1: check, then V-bit propagation wave by wave
                chk.check_copies(dd, dv, stream=stream)
                chk.apply_waves(dd, dv, waves[k], stream=stream)
            elif fu:
                chk.check_apply(dd, dv, stream=stream)
            else:
                chk.check_copies(dd, dv, stream=stream)
                chk.apply_dtoh(dd, dv, stream=stream)

    def step():
        check_epochs()
        chk.leak_sweep(d_leaks, nalloc, d_cnt, stream=stream)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    verd = cg.verdicts_to_numpy(d_out)
    check_b, apply_b = algorithmic_bytes(descs, verd, track=args.track, two_bit=two_bit)
    desc_b = float(n) * (96 + 64)   # every descriptor read, every verdict written
    bytes_per_step = check_b + apply_b + desc_b

    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    launches0 = chk.kernel_launches
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    chk.profile_begin()
    with ClockSampler(device) as clocks:
        ev0.record(stream)
        for _ in range(steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    stages = chk.profile_end()
    launches = chk.kernel_launches - launches0
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / steps

    # e2e through the public host-buffer entry point cg_check_host (pinned
    # buffers; 1D copies in the compact 40-byte form when the batch allows it;
    # dirty verdicts only come back)
    e2e = None
    if not no_e2e:
        is1d = bool(np.all(descs["height"] == 1) and np.all(descs["dst_x"] == 0) and np.all(descs["src_x"] == 0)
                    and np.all(descs["dst_y"] == 0) and np.all(descs["src_y"] == 0)
                    and np.all(descs["dst_pitch"] == descs["width"]) and np.all(descs["src_pitch"] == descs["width"]))
        if is1d:
            d1 = np.zeros(n, cg.COPY1D_DTYPE)
            for f in ("kind", "reserved", "seq", "dst", "src"):
                d1[f] = descs[f]
            d1["bytes"] = descs["width"]
            hbuf = torch.from_numpy(d1.view(np.uint8).copy()).pin_memory()
            hd = hbuf.numpy().view(cg.COPY1D_DTYPE)
        else:
            hbuf = torch.from_numpy(descs.view(np.uint8).copy()).pin_memory()
            hd = hbuf.numpy().view(cg.DESC_DTYPE)
        n_dirty_ref = int(np.count_nonzero(verd["flags"]))
        cap = max(n_dirty_ref, 1)
        h_idx = torch.empty(cap, dtype=torch.int64).pin_memory()
        h_dirty = torch.empty(cap * 64, dtype=torch.uint8).pin_memory()
        nd_box = ctypes.c_uint64(0)

        e_base = []   # per epoch: first dirty slot in the host result buffers
        fmt = cg.CG_FMT_1D if is1d else cg.CG_FMT_2D

        def e2e_run(k_steps):
            """k_steps steps through cg_check_host_submit / _wait, double
            buffered: the upload of the next (step, epoch) batch overlaps the
            check of the current one; every upload and download is inside"""
            units = [(st_, e_, a, b, fu) for st_ in range(k_steps)
                     for e_, ((a, b), fu) in enumerate(zip(epochs, efused))]
            got = [0]

            def submit(u):
                st_, e_, a, b, fu = units[u]
                if e_ == 0 and st_ > 0:   # the previous step's leak sweep, in stream order
                    chk.leak_sweep(d_leaks, nalloc, d_cnt, stream=stream)
                r = cg.cg_check_host_submit(chk.ctx, hd.ctypes.data + a * hd.dtype.itemsize, fmt, b - a,
                                            2 if fu else 1, u % 2, stream.cuda_stream)
                assert r == 0, cg.cg_last_error(chk.ctx)

            submit(0)
            for u in range(len(units)):
                if u + 1 < len(units):
                    submit(u + 1)
                else:
                    chk.leak_sweep(d_leaks, nalloc, d_cnt, stream=stream)
                if units[u][1] == 0:
                    e_base.clear()
                    got[0] = 0
                r = cg.cg_check_host_wait(chk.ctx, u % 2, h_idx.data_ptr() + got[0] * 8,
                                          h_dirty.data_ptr() + got[0] * 64, cap - got[0], ctypes.byref(nd_box))
                assert r == 0, cg.cg_last_error(chk.ctx)
                e_base.append(got[0])
                got[0] += nd_box.value
            nd_box.value = got[0]
        e2e_run(max(1, warmup // 2))
        torch.cuda.synchronize()
        k = max(3, steps // 4)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        e2e_run(k)
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms = e0.elapsed_time(e1) / k
        if world > 1:
            t = torch.tensor([e_ms], dtype=torch.float64, device=device)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            e_ms = float(t.item())
        assert nd_box.value == n_dirty_ref
        dense = verd.copy()
        dense["flags"] = 0
        gidx = h_idx.numpy()[:n_dirty_ref].copy()
        for (a, _), g0, g1 in zip(epochs, e_base, e_base[1:] + [n_dirty_ref]):
            gidx[g0:g1] += a   # epoch-relative indices -> batch indices
        dense[gidx] = h_dirty.numpy()[:n_dirty_ref * 64].view(cg.VERDICT_DTYPE)
        assert np.array_equal(dense["flags"], verd["flags"])
        e2e = {"value": world * bytes_per_step / (e_ms * 1e-3) / 1e9, "unit": UNIT,
               "ms_per_step": e_ms, "entry": "cg_check_host_submit / cg_check_host_wait (%s descriptors, "
               "dirty-only result, double-buffered across steps)" % ("1D" if is1d else "2D"),
               "h2d_bytes_per_step": int(n * hd.dtype.itemsize),
               "d2h_bytes_per_step": int(4 * len(epochs) + n_dirty_ref * 72),
               "descriptors_per_s": world * n / (e_ms * 1e-3)}

    peak, peak_kind = load_peaks()
    scan_ms, scan_n = stages["check_scan"]
    apply_ms, apply_n = stages["apply"]
    scan_avg = scan_ms / max(scan_n, 1)
    scan_bytes = check_b + sum(fused_apply_bytes(descs[a:b], verd[a:b], max(n, 1024), two_bit)
                               for (a, b), fu in zip(epochs, efused) if fu)
    launches_scan = max(scan_n / max(steps, 1), 1.0)   # one per epoch
    achieved = scan_bytes / (scan_avg * launches_scan * 1e-3) / 1e9
    traffic = None
    suffix = "" if args.shadow == "bytes" else "_" + args.shadow
    prof_json = os.path.join(ROOT, "profiles", f"ncu_{config}{suffix}_check_scan.json")
    if os.path.exists(prof_json):
        with open(prof_json) as f:
            pj = json.load(f)
        if pj.get("fused") == fused:
            traffic = pj.get("dram_bytes_per_launch")
    value = world * bytes_per_step / (ms_step * 1e-3) / 1e9
    roof = {"bound": "hbm", "kernel": "k_check_scan", "achieved": achieved, "peak": peak,
            "peak_source": peak_kind, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "algorithmic_bytes_per_launch": scan_bytes / launches_scan,
            "avg_launch_ms": scan_avg,
            "share_of_step": scan_ms / ms if ms > 0 else None}
    check_roof = None
    if args.track and apply_ms:
        # NEXT-1: the propagation (k_prop_waves, one cooperative launch per
        # epoch with waves) dominates the step: 1 B read + 1 B written per byte
        # of every error-free copy
        check_roof, launches_apply = roof, max(apply_n / max(steps, 1), 1.0)
        ach = apply_b / (apply_ms / max(steps, 1) * 1e-3) / 1e9
        wj = os.path.join(ROOT, "profiles", f"ncu_{config}_track_prop_waves.json")
        wtraffic = json.load(open(wj)).get("dram_bytes_per_launch") if os.path.exists(wj) else None
        roof = {"bound": "hbm", "kernel": "k_prop_waves", "achieved": ach, "peak": peak,
                "peak_source": peak_kind, "unit": "GB/s", "frac": ach / peak, "traffic": wtraffic,
                "algorithmic_bytes_per_launch": apply_b / launches_apply,
                "avg_launch_ms": apply_ms / max(apply_n, 1), "share_of_step": apply_ms / ms if ms > 0 else None}
    res = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
        "warmup": warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": workload_name(config),
                   "descriptors_per_step": n, "allocations": nreg, "host_window_bytes": tr.host_size,
                   "algorithmic_bytes_per_step": bytes_per_step, "check_bytes": check_b, "apply_bytes": apply_b,
                   "descriptor_bytes": desc_b,
                   "bytes_counted": "shadow: HtoD 1.125 B + DtoH 0.125 B per host byte checked, 1 B per host "
                                    "byte a DtoH apply defines; descriptors: 96 B read + 64 B verdict written "
                                    "(SURVEY §8(d))",
                   "l2": "no flush: >= 8.5 GB of shadow streamed per step vs 126 MB L2",
                   "parallelism": f"host-range shards x{world}",
                   "shadow_format": {"bytes": "V bytes + A bits", "2bit": "2-bit states (NEXT-4)",
                                     "sparse": "2-bit states in the two-level sparse map (NEXT-4)"}[args.shadow],
                   "entry": ("cg_check_copies + cg_apply_copies (NEXT-1 V-bit propagation)" if args.track else
                             "cg_check_apply (fused)" if fused else "cg_check_copies + cg_apply_dtoh"
                             if not any(efused) else "cg_check_apply / cg_check_copies + cg_apply_dtoh per epoch"),
                   "epochs": len(epochs), "apply_after_descriptors": n_after, "check_after_descriptors": n_late,
                   "apply_last_descriptors": n_last,
                   "propagation_waves": sum(w.n_waves for w in waves) if args.track else None,
                   "wave_planning_s": t_waves if args.track else None},
        "descriptors_per_s": world * n / (ms_step * 1e-3),
        "shadow_gbs": world * (check_b + apply_b) / (ms_step * 1e-3) / 1e9,
        "frac_of_hbm": value / (world * peak),
        "roofline": roof,
        "check_roofline": check_roof,
        "stages_ms_per_step": {k: v[0] / max(steps, 1) for k, v in stages.items()},
        "apply_roofline": {"achieved": (apply_b - (scan_bytes - check_b)) / (apply_ms / max(steps, 1) * 1e-3) / 1e9
                           if apply_ms else None, "unit": "GB/s", "peak": peak,
                           "note": "k_apply alone (the residual pass when fused)"},
        "gpu_launches": int(launches),
        "gpu_launches_per_step": launches / steps,
        "clocks": clocks.summary(),
        "e2e": e2e,
        "setup_s": t_setup,
    }
    if extras and rank == 0 and not args.no_registry_rate:
        res["registry_events_per_s"] = registry_rate(cg, tr, device)
    if extras and args.conc:
        res["next2"] = conc_rate(cg, descs, d_out, args, device, stream)
    chk.close()
    return res


def run_sharded_bench(args, rank, world, device, backend):
    """Strong scaling on C5 (BASELINE.json configs[4]: "64 GB host shadow space
    sharded across 8 B200, 10M mixed HtoD/DtoH/DtoD descriptors with
    interleaved alloc/free and final leak report"): the SAME trace on every
    rank, the 64 GiB window split `world` ways (shard r on rank r), the
    allocation table replicated; per step and R-20 epoch one cg_check_sharded
    (fused check + apply of the rank's list, the straddler exchange over NCCL,
    the dirty-verdict gather to the root and its merge kernel, all on the
    device), then the leak sweep.  backend "nccl": one rank per process
    (torchrun); "loopback": all shards in this process on one GPU (the same
    library path, for one-GPU measurement and testing)."""
    import torch
    import paper_1310_0901_b200 as cg
    import tracegen as tg
    from paper_1310_0901_b200.sharded import ShardGroup, replay_sharded
    torch.cuda.set_device(device)
    tr = make_workload("c5_sharded", 0, args.scale)   # one trace, the same on every rank
    ev = tr.events
    descs = tg.events_to_descs(ev[ev["op"] == 5])
    n = len(descs)
    nreg = int(np.count_nonzero(ev["op"] == 3))
    cuts = [0] + [int(c) for c in cg.plan_batches(descs)]
    epochs = [(a, b) for a, b in zip(cuts[:-1], cuts[1:]) if b > a]
    max_epoch = max(b - a for a, b in epochs)
    cap = max(4096, max_epoch // 8)
    group = ShardGroup(tr.host_base, tr.host_size, world, backend=backend, rank=rank, device=device,
                       max_descs=max_epoch, max_allocs=max(nreg, 1024), max_straddlers=max(4096, max_epoch // 64),
                       cap=cap)
    t0 = time.perf_counter()
    replay_sharded(group, ev[ev["op"] != 5], tr.blob)
    t_setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    batches = [group.batch(descs[a:b], dense=False) for a, b in epochs]
    t_plan = time.perf_counter() - t0
    stream = torch.cuda.current_stream()
    leaks = [(torch.empty(max(nreg, 1) * 24, dtype=torch.uint8, device=device),
              torch.zeros(1, dtype=torch.int64, device=device)) for _ in group.chks]
    # e2e: every step uploads each rank's lists from pinned host memory and the
    # root downloads its merged dirty lists
    pinned = [[(torch.empty_like(t, device="cpu").pin_memory(), t) for t in (bt.keep[0][0], bt.keep[0][1])]
              for bt in batches] if not args.no_e2e else None
    if pinned:
        for bp in pinned:
            for h, d in bp:
                h.copy_(d)

    def step(upload=False):
        for k, bt in enumerate(batches):
            if upload:
                for h, d in pinned[k]:
                    d.copy_(h, non_blocking=True)
            group.check(bt, stream=stream)
        for c, (dl, dc) in zip(group.chks, leaks):
            c.leak_sweep(dl, nreg, dc, stream=stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    assert not group.overflow(), "a rank had more dirty verdicts than the gather capacity"
    # the root's merged dirty lists -> algorithmic bytes (an OK DtoH is a clean one)
    dirty = np.zeros(n, bool)
    if group.is_root:
        for (a, b), bt in zip(epochs, batches):
            c = int(bt.root_count.item())
            dirty[a + bt.root_idx[:c].cpu().numpy()] = True
    n_dirty = int(dirty.sum())
    fake = np.zeros(n, [("status", "<u4")])
    fake["status"] = dirty
    check_b, apply_b = algorithmic_bytes(descs, fake)
    desc_b = float(n) * (96 + 64)
    bytes_per_step = check_b + apply_b + desc_b
    dist = None
    if backend == "nccl" and world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    l0 = group.kernel_launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(device) as clocks:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    launches = group.kernel_launches - l0
    ms = e0.elapsed_time(e1)
    if dist is not None:
        t = torch.tensor([ms], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    e2e = None
    if pinned:
        k = max(3, args.steps // 4)
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        e0.record(stream)
        for _ in range(k):
            step(upload=True)
            if group.is_root:   # the root reads its merged dirty lists (count, then the records)
                for bt in batches:
                    c = int(bt.root_count.item())
                    bt.root_idx[:c].cpu()
                    bt.root_dirty[:c * 64].cpu()
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms = e0.elapsed_time(e1) / k
        if dist is not None:
            t = torch.tensor([e_ms], dtype=torch.float64, device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        up = sum(h.numel() * h.element_size() for bp in pinned for h, _ in bp)
        e2e = {"value": bytes_per_step / (e_ms * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": e_ms,
               "entry": "ShardGroup.check = cg_check_sharded per epoch, lists uploaded from pinned host memory, "
                        "the root's merged dirty lists downloaded",
               "h2d_bytes_per_step": int(up), "d2h_bytes_per_step": int(8 * len(batches) + 72 * n_dirty),
               "wall_s": time.perf_counter() - w0}
    peak, peak_kind = load_peaks()
    value = bytes_per_step / (ms_step * 1e-3) / 1e9
    res = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world if backend == "nccl" else 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": "c5_sharded (BASELINE.json configs[4]: 64 GiB host window, 10M mixed descriptors, "
                               "alloc/free bursts, leak report)",
                   "descriptors_per_step": n, "allocations": nreg, "host_window_bytes": tr.host_size,
                   "algorithmic_bytes_per_step": bytes_per_step, "check_bytes": check_b, "apply_bytes": apply_b,
                   "descriptor_bytes": desc_b, "epochs": len(epochs),
                   "straddlers_per_step": int(sum(bt.m for bt in batches)),
                   "parallelism": f"host-range shards x{world} ({backend})",
                   "l2": "no flush: >= 1 GB of shadow streamed per rank per step vs 126 MB L2",
                   "entry": "cg_check_sharded per epoch + cg_leak_sweep", "gather_cap_per_rank": cap},
        "descriptors_per_s": n / (ms_step * 1e-3),
        "shadow_gbs": (check_b + apply_b) / (ms_step * 1e-3) / 1e9,
        "frac_of_hbm": value / ((world if backend == "nccl" else 1) * peak),
        "gpu_launches": int(launches), "gpu_launches_per_step": launches / args.steps,
        "clocks": clocks.summary(), "e2e": e2e, "setup_s": t_setup, "plan_s": t_plan,
        "dirty_verdicts": n_dirty,
    }
    group.close()
    return res


def run_interleaved(args, device):
    """C5 as a program issues it: the registry events (a7: 1000 bursts of 50
    frees + 50 allocations, then the final frees) interleaved with the copy
    checks inside the timed region -- per block: one cg_registry_batch, then
    the R-20 epochs of the block's copies (cg_check_apply; the registry goes to
    the device by difference inside the check call).  The host shadow setup
    and the 100k initial allocations are replayed untimed; a pass mutates the
    registry, so each pass runs on a fresh context (one warm-up pass, then the
    timed one)."""
    import torch
    import paper_1310_0901_b200 as cg
    import tracegen as tg
    tr = make_workload("c5_sharded", 0, args.scale)
    ev = tr.events
    ops = ev["op"]
    first_copy = int(np.flatnonzero(ops == 5)[0])
    setup, rest = ev[:first_copy], ev[first_copy:]
    rops = rest["op"]
    # blocks: [registry run][copies ...] in trace order
    blocks = []
    i = 0
    while i < len(rest):
        j = i
        while j < len(rest) and rops[j] in (3, 4):
            j += 1
        k = j
        while k < len(rest) and rops[k] == 5:
            k += 1
        regs = rest[i:j]
        re = np.zeros(len(regs), cg.REG_EVENT_DTYPE)
        re["op"] = np.where(regs["op"] == 3, cg.CG_REG_ALLOC, cg.CG_REG_FREE)
        re["seq"], re["addr"], re["size"] = regs["seq"], regs["dst"], regs["width"]
        descs = np.ascontiguousarray(tg.events_to_descs(rest[j:k]))
        cuts = [0] + [int(c) for c in cg.plan_batches_fused(descs)] if len(descs) else [0]
        eps = [(a, b) for a, b in zip(cuts[:-1], cuts[1:])]
        blocks.append((re, descs, eps))
        i = k
    n = int(np.count_nonzero(rops == 5))
    nreg_ev = int(np.count_nonzero((rops == 3) | (rops == 4)))
    nreg = int(np.count_nonzero(ops == 3))
    stream = torch.cuda.current_stream()

    def one_pass(timed):
        chk = cg.Checker(tr.host_base, tr.host_size, max_descs=max(max(len(d) for _, d, _ in blocks), 1024),
                         max_allocs=max(nreg, 1024), device=device)
        cg.replay_events(chk, setup, tr.blob)
        dd = [cg.to_device_descs(d, device) if len(d) else None for _, d, _ in blocks]
        dv = [torch.empty(max(len(d), 1) * 64, dtype=torch.uint8, device=device) for _, d, _ in blocks]
        dl = torch.empty(max(nreg, 1) * 24, dtype=torch.uint8, device=device)
        dc = torch.zeros(1, dtype=torch.int64, device=device)
        torch.cuda.synchronize()
        l0 = chk.kernel_launches
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t_reg = 0.0
        w0 = time.perf_counter()
        e0.record(stream)
        for (re, descs, eps), x, y in zip(blocks, dd, dv):
            if len(re):
                t = time.perf_counter()
                st = chk.registry_batch(re)
                t_reg += time.perf_counter() - t
                assert st == 0, cg.cg_last_error(chk.ctx)
            for a, b in eps:
                chk.check_apply(x[a * 96:b * 96], y[a * 64:b * 64], stream=stream)
        chk.leak_sweep(dl, nreg, dc, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
        ms = e0.elapsed_time(e1)
        launches = chk.kernel_launches - l0
        chk.close()
        return ms, wall, t_reg, launches

    one_pass(False)
    ms, wall, t_reg, launches = one_pass(True)
    return {"ms_per_pass": ms, "wall_s_per_pass": wall, "descriptors": n, "registry_events": nreg_ev,
            "blocks": len(blocks), "epochs": sum(len(e) for _, _, e in blocks),
            "registry_events_per_s": nreg_ev / t_reg if t_reg > 0 else None,
            "registry_host_s": t_reg, "descriptors_per_s": n / (ms * 1e-3),
            "gpu_launches_per_pass": launches,
            "entry": "per block: cg_registry_batch, then cg_check_apply per R-20 epoch (table by diff upload); "
                     "one timed pass on a fresh context after one warm-up pass"}


PER_CONFIG = ("c3_single", "c4_pitched", "c5_sharded")


def per_config(args, device):
    """The other BASELINE.json configurations, each through the same measured
    step (its own setup, 3 warm-up steps, device-timed steps, CUDA-event stage
    timing) so that every config is in the driver-observed line."""
    import gc
    import torch
    out = {}
    for cfg in PER_CONFIG:
        steps = {"c3_single": 20, "c4_pitched": 6, "c5_sharded": 10}[cfg]
        r = run_ours(args, 0, 1, device, config=cfg, steps=steps, warmup=3, e2e_on=False, extras=False)
        out[cfg] = {"value": r["value"], "unit": UNIT, "ms_per_step": r["ms_per_step"], "steps": steps, "warmup": 3,
                    "descriptors_per_s": r["descriptors_per_s"], "shadow_gbs": r["shadow_gbs"],
                    "frac_of_hbm": r["frac_of_hbm"], "roofline": {k: r["roofline"][k] for k in
                                                                  ("kernel", "achieved", "frac", "avg_launch_ms",
                                                                   "share_of_step")},
                    "stages_ms_per_step": r["stages_ms_per_step"], "epochs": r["config"]["epochs"],
                    "gpu_launches_per_step": r["gpu_launches_per_step"], "clocks": r["clocks"],
                    "config": {k: r["config"][k] for k in ("descriptors_per_step", "allocations", "host_window_bytes",
                                                           "algorithmic_bytes_per_step", "entry")}}
        gc.collect()
        torch.cuda.empty_cache()
        if cfg == "c5_sharded" and not args.no_interleaved:
            out["c5_interleaved"] = run_interleaved(args, device)
            gc.collect()
            torch.cuda.empty_cache()
    return out


def conc_rate(cg, descs, d_out, args, device, stream):
    """NEXT-2: cg_conc_check on the same batch and verdicts, issued by
    args.conc random threads; every call gets the batch with its seqs shifted
    past the previous call's (the contract), so the last-access map is carried
    from call to call as in a long program."""
    import torch
    n = len(descs)
    rng = np.random.default_rng(0x2C)
    th = torch.from_numpy(rng.integers(0, args.conc, n).astype(np.int32)).to(device)
    span = int(descs["seq"].max()) + 1
    k, w = max(3, args.steps // 4), max(3, args.warmup)
    arrs = []
    for i in range(k + w):
        d = descs.copy()
        d["seq"] += np.uint64(i * span)
        arrs.append(cg.to_device_descs(d, device))
    conc = cg.ConcChecker(n, 4 * n, device)
    for i in range(w):
        conc.check(arrs[i], th, d_out, stream=stream)
    torch.cuda.synchronize()
    l0 = conc.kernel_launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(w, w + k):
        conc.check(arrs[i], th, d_out, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / k
    v = cg.verdicts_to_numpy(d_out)
    out = {"threads": args.conc, "ms_per_call": ms, "copies_per_s": n / (ms * 1e-3),
           "hazard_copies": int(np.count_nonzero(v["flags"] & cg.CG_F_CONCURRENT)),
           "map_ranges": conc.stamps(), "gpu_launches_per_call": (conc.kernel_launches - l0) / k,
           "entry": "cg_conc_check (synchronous: 3 host reads of counts per address space)"}
    conc.close()
    return out


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class OracleArm:
    """The CPU oracle, as it stands, on a bounded sample of the workload: the
    same generator and allocation table with fewer copies.  Setup events are
    replayed once (untimed); every step replays the copy batch (timed) with the
    per-copy checks of each epoch on `threads` host threads
    (or_replay_parallel; 1 = the sequential or_replay).  A repeated replay sees
    the same verdicts (DtoH checks read only A; HtoD sources are never DtoH
    targets), so every step is the same work.  Imports only oracle/ and
    tracegen/ -- never the product package."""

    def __init__(self, config: str, threads: int = 0, n_copies: int | None = None):
        import oracle
        import tracegen as tg
        self.threads = threads or os.cpu_count() or 1
        if config == "c2_small":
            tr = tg.c2_small(n_copies=n_copies or (100_000 if self.threads > 1 else 20000), n_allocs=100_000)
        elif config == "c3_single":
            tr = tg.c3_single(size=(2 << 30) if self.threads > 1 else 256 << 20)
        elif config == "c5_sharded":
            tr = tg.c5_sharded(scale=0.01)
        else:
            tr = tg.c4_pitched(n_copies=n_copies or (4000 if self.threads > 1 else 400))
        ev = tr.events
        self.o = oracle.Oracle(tr.host_base, tr.host_size)
        self.o.replay(ev[ev["op"] != 5], tr.blob)
        self.copies = ev[ev["op"] == 5]
        self.blob = tr.blob
        self.descs = tg.events_to_descs(self.copies)
        self.nalloc = int(np.count_nonzero(ev["op"] == 3))
        self.config = config
        self.verdicts = None

    def step(self):
        t0 = time.perf_counter()
        if self.threads > 1:
            v, _ = self.o.replay_parallel(self.copies, self.blob, self.threads)
        else:
            v, _ = self.o.replay(self.copies, self.blob)
        dt = time.perf_counter() - t0
        self.verdicts = v
        cb, ab = algorithmic_bytes(self.descs, v)
        return (cb + ab + len(self.descs) * (96 + 64)), dt

    def describe(self, value, dt_total, steps):
        return {"value": value, "unit": UNIT, "cores": self.threads, "kind": "oracle", "cpu_model": cpu_model(),
                "nproc": os.cpu_count(), "descriptors_per_s": len(self.copies) * steps / dt_total,
                "sample": f"{self.config} generator, {len(self.copies)} copies against {self.nalloc} "
                          f"allocations per step x {steps} steps, "
                          + (f"{self.threads} threads (or_replay_parallel: checks of each epoch in parallel)"
                             if self.threads > 1 else "single-threaded sequential replay")
                          + " -- plain C, linear allocation list"}


def run_cpu_baseline(config: str, steps: int = 3):
    """T-thread oracle (T = the host's cores) on a bounded sample, plus the
    1-thread replay of a smaller sample; the T-thread verdicts of that smaller
    sample must equal the 1-thread ones."""
    if config not in ("c2_small", "c3_single", "c4_pitched", "c5_sharded"):
        config = "c2_small"
    arm = OracleArm(config)
    tot_b = tot_t = 0.0
    for _ in range(steps):
        b, t = arm.step()
        tot_b += b
        tot_t += t
    out = arm.describe(tot_b / tot_t / 1e9, tot_t, steps)
    one = OracleArm(config, threads=1)
    b1, t1 = one.step()
    par = OracleArm(config, threads=arm.threads, n_copies=len(one.copies))
    par.step()
    same = all(np.array_equal(one.verdicts[f], par.verdicts[f]) for f in one.verdicts.dtype.names)
    assert same, "T-thread oracle differs from the 1-thread oracle"
    out["single_thread"] = {"value": b1 / t1 / 1e9, "unit": UNIT, "cores": 1,
                            "descriptors_per_s": len(one.copies) / t1, "copies": len(one.copies),
                            "equal_to_T_thread": same}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2_small")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-registry-rate", action="store_true")
    ap.add_argument("--no-per-config", action="store_true", help="skip the C3/C4/C5 per_config runs")
    ap.add_argument("--no-interleaved", action="store_true", help="skip the interleaved C5 registry pass")
    ap.add_argument("--sharded", action="store_true",
                    help="at N=1: the multi-GPU code path (C5 through cg_check_sharded, NCCL with one rank)")
    ap.add_argument("--loopback", type=int, default=0,
                    help="C5 split into this many shards on ONE GPU through the loopback cg_comm")
    ap.add_argument("--unfused", action="store_true", help="check and apply as two calls")
    ap.add_argument("--track", action="store_true", help="NEXT-1 device V-bit tracking (apply = propagation)")
    ap.add_argument("--conc", type=int, default=0, help="NEXT-2: also time cg_conc_check with this many threads")
    ap.add_argument("--shadow", default="bytes", choices=["bytes", "2bit", "sparse"],
                    help="host shadow format: V bytes + A bits, or NEXT-4 2-bit states")
    args = ap.parse_args()
    assert args.warmup >= 1

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return
        arm = OracleArm(args.config)
        for _ in range(args.warmup):
            arm.step()
        tot_b = tot_t = 0.0
        for _ in range(args.steps):
            b, t = arm.step()
            tot_b += b
            tot_t += t
        val = tot_b / tot_t / 1e9
        loaded = [l.split()[-1] for l in open("/proc/self/maps") if l.rstrip().endswith(".so")
                  and ROOT in l]
        out = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
               "repo_libraries_loaded": sorted(set(loaded)),
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_t / args.steps * 1e3,
               "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
               "data": "synthetic", "config": {"workload": workload_name(args.config)},
               "cpu_baseline": arm.describe(val, tot_t, args.steps),
               "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(out))
        return

    import torch
    if world > 1 or args.sharded:
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29517")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
        res = run_sharded_bench(args, rank, world, local, "nccl")
        if rank == 0:
            print(json.dumps(res))
        torch.distributed.destroy_process_group()
        return
    if args.loopback > 1:
        print(json.dumps(run_sharded_bench(args, 0, args.loopback, local, "loopback")))
        return
    res = run_ours(args, rank, world, local)
    if rank == 0:
        if world == 1 and args.config == "c2_small" and not args.no_per_config and not args.track \
                and args.shadow == "bytes":
            res["per_config"] = per_config(args, local)
        if not args.no_cpu_baseline:
            res["cpu_baseline"] = run_cpu_baseline(args.config)
        print(json.dumps(res))
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
