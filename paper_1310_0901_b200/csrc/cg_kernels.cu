// sm_100a kernels of the batched Cudagrind transfer checker.
//
// Hot path of one check + apply:
//   a1+a3  k_check_prep     one thread per descriptor: CUDA_MEMCPY2D start /
//                           span / pitch / overflow validation, then a batched
//                           interval search of every device endpoint in the
//                           lifetime-stamped, base-sorted allocation table
//                           (splitters staged in shared memory; PAPER.md P:77,
//                           P:80).  Writes
//                           the device half of the verdict and the item weight.
//   a2     k_scan_* + k_plan   exclusive prefix sum of weights and the chunk ->
//                           first item map: equal-weight chunks, so a 64-byte
//                           copy and an 8 GiB copy are load-balanced alike.
//   a4     k_check_scan     persistent grid; a warp per chunk; 128-bit
//                           coalesced non-allocating loads of V (16 B/lane) and
//                           A (2 B/lane), a warp-uniform clean test and, only
//                           for dirty 16-byte groups, per-byte masks with
//                           __ffs (first violation) and __popc (count); warp
//                           shuffles reduce min/min/sum ("bitwise
//                           precision").
//   a5     inline in k_check_scan for descriptors that fit one chunk,
//          k_finalize_split for the ones split across chunks (u64 atomics only
//          for non-identity partials): flags + status.
//   a6     k_apply_prep + plan + k_apply   V := 0 over DtoH ranges with
//                           status OK (BASELINE north_star (3)).
//   a8     k_leak: one cooperative launch (per-slice live counts, grid barrier,
//          compaction in base order); CG_LEAK_COOP=0: k_live + scan +
//          k_leak_scatter (abstract P:12).
// Plumbing (setup, untimed): k_fill (fresh shadow), k_mark (S:45-62,
// S:355-363), k_setv_check.
//
// Layout: V is one byte per host byte, A one bit per host byte (LSB first),
// both indexed by (x - shard_base); H0 % 4096 == 0 so a 16-byte V group maps to
// one aligned 16-bit A half-word and a 128-byte V range to one 16-byte A vector.

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "cg_internal.h"

namespace cgk {

namespace {

constexpr int kThreads = 256;
constexpr unsigned kFull = 0xffffffffu;

// Programmatic dependent launch: every kernel waits for its stream
// predecessor's completion (griddepcontrol.wait: all its writes visible) and
// then lets its own successor launch, so launch latency and block scheduling
// of back-to-back kernels overlap the previous kernel's tail.  A no-op for
// kernels launched without the PDL attribute.
__device__ __forceinline__ void pdl_entry() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---------------------------------------------------------------------------
// small device helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ void stg_val16(uint4* p, uint32_t v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%1,%1,%1};" ::"l"(p), "r"(v));
}

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }
__device__ __forceinline__ uint64_t umax64(uint64_t a, uint64_t b) { return a > b ? a : b; }

// one bit per byte of w: bit j set iff byte j of w is nonzero
__device__ __forceinline__ uint32_t nz4(uint32_t w) {
  uint32_t t = (((w & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | w) & 0x80808080u;
  return ((t >> 7) * 0x01020408u) >> 24;
}
__device__ __forceinline__ uint32_t nz16(uint4 v) {
  return nz4(v.x) | (nz4(v.y) << 4) | (nz4(v.z) << 8) | (nz4(v.w) << 12);
}

// mask of the bits [lo, hi) of a `width`-bit group starting at gb, with lo/hi
// absolute positions; lo <= gb + width, hi >= gb (caller guarantees overlap)
__device__ __forceinline__ uint32_t range_mask(uint64_t gb, int width, uint64_t lo, uint64_t hi) {
  uint32_t full = (width == 32) ? 0xffffffffu : ((1u << width) - 1u);
  uint32_t m = full;
  if (gb < lo) {
    uint64_t sh = lo - gb;
    m = sh >= (uint64_t)width ? 0u : (m << sh) & full;
  }
  if (gb + width > hi) {
    uint64_t sh = gb + width - hi;
    m = sh >= (uint64_t)width ? 0u : m & (full >> sh);
  }
  return m;
}

__device__ __forceinline__ uint64_t warp_min(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = umin64(v, __shfl_xor_sync(kFull, v, o));
  return v;
}
__device__ __forceinline__ uint64_t warp_sum(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// ---------------------------------------------------------------------------
// a1: descriptor normalisation (CUDA_MEMCPY2D start-address rule, pitch rule,
// 64-bit overflow) -- DESIGN.md readings R-10, R-11, R-12, R-16
// ---------------------------------------------------------------------------
// fold_side (cg_internal.h): CUDA_MEMCPY2D start / span of one side

struct Norm {
  uint32_t kind, flags;
  uint32_t skind;      // scan kind: CG_HTOD-like (V + A), CG_DTOH-like (A), CG_DTOD (no host side)
  bool dok, sok;
  uint64_t ds, dspan, ss, sspan;
  bool host;           // has a host side that is scanned
  uint64_t hstart, hpitch, W, nbytes;
  bool aok;            // NEXT-3: the array side (handle, byte offset) of HtoA / AtoH
  uint64_t ahandle, aoff;
};

__device__ __forceinline__ Norm normalize(const cg_copy_desc& d) {
  Norm n;
  n.kind = d.kind;
  n.flags = 0;
  n.skind = CG_DTOD;
  n.dok = n.sok = n.aok = false;
  n.ds = n.dspan = n.ss = n.sspan = 0;
  n.host = false;
  n.hstart = n.hpitch = n.nbytes = 0;
  n.ahandle = n.aoff = 0;
  n.W = d.width;
  if (d.kind < CG_HTOD || d.kind > CG_ATOH) {
    n.flags = CG_F_BAD_KIND;
    return n;
  }
  const uint64_t W = d.width, H = d.height;
  // R-10: the logical byte count W*H -- the range of the offsets a
  // verdict reports -- must fit in 64 bits; there is no size cap
  const bool bytes_ok = __umul64hi(W, H) == 0;
  if (d.kind >= CG_HTOA) {   // NEXT-3 array transfer: pitch rule and fold on the host side only
    const bool htoa = d.kind == CG_HTOA;
    const uint64_t hx = htoa ? d.src_x : d.dst_x, hp = htoa ? d.src_pitch : d.dst_pitch;
    if (W + hx < W || hp < W + hx) n.flags |= CG_F_BAD_PITCH;
    uint64_t hs = 0, hspan = 0;
    const bool hok = htoa ? fold_side(d.src, d.src_x, d.src_y, d.src_pitch, W, H, hs, hspan)
                          : fold_side(d.dst, d.dst_x, d.dst_y, d.dst_pitch, W, H, hs, hspan);
    n.ahandle = htoa ? d.dst : d.src;
    n.aoff = htoa ? d.dst_x : d.src_x;
    n.aok = bytes_ok && n.aoff + W * H >= n.aoff;
    if (!hok || !n.aok) n.flags |= CG_F_INVALID_RANGE;
    n.skind = htoa ? CG_HTOD : CG_DTOH;
    if (htoa) { n.sok = hok; n.ss = hs; n.sspan = hspan; }
    else      { n.dok = hok; n.ds = hs; n.dspan = hspan; }
    if (hok && bytes_ok) {
      n.host = true;
      n.hstart = hs;
      n.hpitch = hp;
      n.nbytes = W * H;
    }
    return n;
  }
  // pitch rule: pitch >= WidthInBytes + XInBytes (evaluated without overflow)
  if (W + d.dst_x < W || d.dst_pitch < W + d.dst_x) n.flags |= CG_F_BAD_PITCH;
  if (W + d.src_x < W || d.src_pitch < W + d.src_x) n.flags |= CG_F_BAD_PITCH;
  n.dok = fold_side(d.dst, d.dst_x, d.dst_y, d.dst_pitch, W, H, n.ds, n.dspan);
  n.sok = fold_side(d.src, d.src_x, d.src_y, d.src_pitch, W, H, n.ss, n.sspan);
  if (!n.dok || !n.sok || !bytes_ok) n.flags |= CG_F_INVALID_RANGE;
  n.skind = d.kind;
  if (d.kind == CG_HTOD && n.sok && bytes_ok) {
    n.host = true;
    n.hstart = n.ss;
    n.hpitch = d.src_pitch;
    n.nbytes = W * H;
  } else if (d.kind == CG_DTOH && n.dok && bytes_ok) {
    n.host = true;
    n.hstart = n.ds;
    n.hpitch = d.dst_pitch;
    n.nbytes = W * H;
  }
  return n;
}

// ---------------------------------------------------------------------------
// R-10 / R-15: analytic clipping of a host side.  The side's rows are
// x_r = x0 + r*pitch (r < H), W bytes each, logical offset o = r*W + c (R-11);
// a contiguous side (H == 1 or pitch == W) is one row of N = W*H bytes.  Host
// bytes outside the window are unaddressable, so the scan only needs the bytes
// inside this GPU's shard; those outside the window only contribute the lowest
// logical offset among them (pfu), which has a closed form: o grows with the
// address along the rows (pitch >= 0), so it is the first byte at or past the
// window end, or offset 0 when the side starts below the window.
// ---------------------------------------------------------------------------
// first row r with x0 + r*pitch + W > lim (H if none); x0 + W cannot overflow
// (start + span fits in 64 bits and span >= W)
__device__ __forceinline__ uint64_t first_row_past(uint64_t x0, uint64_t W, uint64_t pitch, uint64_t H,
                                                   uint64_t lim) {
  if (x0 + W > lim) return 0;
  if (pitch == 0) return H;
  const uint64_t r = (lim - x0 - W) / pitch + 1;
  return r < H ? r : H;
}

struct HostClip {
  uint64_t olo, ohi;   // logical [olo, ohi): every shard byte of a side whose rows do not overlap (maybe empty)
  uint64_t pfu;        // lowest logical offset of a byte outside the window (kNone if none)
  bool overlap;        // BAD_PITCH rows that overlap (pitch < W): the deferred pass (multiplicity, R-12)
};

// nm.host must hold (a valid, bytes_ok host side)
__device__ __forceinline__ HostClip host_clip(const Norm& nm, uint64_t H, const ShadowView& sv) {
  HostClip c;
  c.olo = c.ohi = 0;
  c.pfu = kNone;
  const bool contig = H == 1 || nm.W == nm.hpitch;
  const uint64_t W = contig ? nm.nbytes : nm.W, Hr = contig ? 1 : H, pitch = contig ? 0 : nm.hpitch;
  c.overlap = false;
  if (nm.nbytes == 0) return c;   // W == 0 or H == 0: no host bytes
  c.overlap = !contig && pitch < W;
  const uint64_t x0 = nm.hstart;
  if (x0 < sv.wb) {
    c.pfu = 0;
  } else {
    const uint64_t r = first_row_past(x0, W, pitch, Hr, sv.we);
    if (r < Hr) {
      const uint64_t xr = x0 + r * pitch;
      c.pfu = r * W + (sv.we > xr ? sv.we - xr : 0);
    }
  }
  if (c.overlap) return c;
  const uint64_t rlo = first_row_past(x0, W, pitch, Hr, sv.sb);
  if (rlo == Hr) return c;
  const uint64_t xlo = x0 + rlo * pitch;
  if (xlo >= sv.se) return c;
  uint64_t rhi = Hr - 1;
  if (pitch) rhi = umin64(rhi, (sv.se - 1 - x0) / pitch);
  const uint64_t xhi = x0 + rhi * pitch;
  c.olo = rlo * W + (sv.sb > xlo ? sv.sb - xlo : 0);
  c.ohi = rhi * W + umin64(W, sv.se - xhi);
  return c;
}

// olo of host_clip without the rest (the scan's generator, per piece): the
// logical offset of the first shard byte; 0 unless the side starts below the shard
__device__ __forceinline__ uint64_t clip_base(uint64_t x0, uint64_t W, uint64_t pitch, bool contig, uint64_t sb) {
  if (x0 >= sb) return 0;
  if (contig) return sb - x0;
  const uint64_t r = first_row_past(x0, W, pitch, ~0ull, sb);
  const uint64_t xr = x0 + r * pitch;
  return r * W + (sb > xr ? sb - xr : 0);
}

// packed per-descriptor metadata written by k_check_prep for the scan
struct __align__(16) ScanMeta {
  uint64_t hstart, hpitch, W, info;   // info: see kInfo*
};
// info: scanned bytes (the shard clip, < 2^40) | scan kind << 40 | host << 42 |
// contiguous << 43 | raw << 44 | pfu << 45 | not the ring's (deferred pass or
// small pass) << 46 | apply after the scan (CG_APPLY_AFTER) << 47 | flags << 48
// | small pass << 58 | CG_APPLY_LAST (cg_check_apply) << 59
constexpr int kInfoKind = 40, kInfoHost = 42, kInfoContig = 43, kInfoRaw = 44, kInfoPfu = 45, kInfoDefer = 46,
              kInfoAfter = 47, kInfoFlags = 48, kInfoSmall = 58,   // flags: 10 bits (48..57)
              kInfoLast = 59;
constexpr uint64_t kInfoBytes = (1ull << 40) - 1;

// The table's lines are kept in L2 against the descriptor / verdict streams of
// the prep (which evict them otherwise: a 150k-entry table is a few MB, the
// streams hundreds of MB): its loads carry an L2 evict_last policy.
__device__ __forceinline__ uint64_t evict_last_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t ld_keep(const uint64_t* a, uint64_t pol) {
  uint64_t v;
  asm volatile("ld.global.nc.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ uint4 ld_keep4(const uint4* a, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(a), "l"(pol));
  return v;
}

// ---------------------------------------------------------------------------
// a3: batched interval search (lifetime-stamped, base-sorted table)
// ---------------------------------------------------------------------------
// Returns true and the containing allocation's end if some entry e has
// base_e <= start < end_e and aseq_e < seq < fseq_e.  At most one entry can
// match (live allocations never overlap).  Probe i = last base <= start
// (smem splitters, then a short global binary search), then walk left while
// the prefix max of ends exceeds start (one step without address reuse).
[[maybe_unused]] __device__ __forceinline__ bool table_lookup(const Table& t, const uint64_t* s_split, uint64_t start,
                                             uint64_t seq, uint64_t& end_out, uint64_t& idx_out) {
  if (t.nsplit == 0 || s_split[0] > start) return false;
  const uint64_t pol = evict_last_policy();
  uint32_t lo = 0, hi = t.nsplit;
  while (hi - lo > 1) {
    uint32_t mid = (lo + hi) >> 1;
    if (s_split[mid] <= start) lo = mid; else hi = mid;
  }
  uint64_t a = (uint64_t)lo * t.stride;
  uint64_t b = umin64(a + t.stride, t.n);
  if (t.stride == 32 || (t.stride == 64 && t.two_round64)) {
    // two independent-load rounds instead of five or six dependent ones: the
    // bucket's 8 or 16 every-4th bases (64 or 128 B), then the 4 bases of the
    // chosen quarter (32 B); each picks the last entry <= start (the first always is)
    const uint4* q = reinterpret_cast<const uint4*>(t.l2 + a / 4);
    const int nq = (int)(t.stride >> 3);   // uint4 loads of 2 every-4th bases each
    uint32_t c2 = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (k >= nq) break;
      const uint4 v = ld_keep4(q + k, pol);
      c2 += (a + 8 * k < b && (((uint64_t)v.y << 32) | v.x) <= start) +
            (a + 8 * k + 4 < b && (((uint64_t)v.w << 32) | v.z) <= start);
    }
    const uint64_t a1 = a + 4 * (c2 - 1);
    const uint4* r = reinterpret_cast<const uint4*>(t.base + a1);
    uint32_t c1 = 0;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const uint4 v = ld_keep4(r + k, pol);
      c1 += (a1 + 2 * k < b && (((uint64_t)v.y << 32) | v.x) <= start) +
            (a1 + 2 * k + 1 < b && (((uint64_t)v.w << 32) | v.z) <= start);
    }
    a = a1 + c1 - 1;
  } else {
    while (b - a > 1) {
      const uint64_t mid = (a + b) >> 1;
      if (ld_keep(t.base + mid, pol) <= start) a = mid; else b = mid;
    }
  }
  for (int64_t j = (int64_t)a; j >= 0; --j) {
    const uint4 w0 = ld_keep4(t.walk + 2 * j, pol), w1 = ld_keep4(t.walk + 2 * j + 1, pol);   // one 32-byte sector
    const uint64_t pm = ((uint64_t)w0.y << 32) | w0.x, e = ((uint64_t)w0.w << 32) | w0.z;
    const uint64_t as = ((uint64_t)w1.y << 32) | w1.x, fs = ((uint64_t)w1.w << 32) | w1.z;
    if (pm <= start) break;
    if (e > start && as < seq && seq < fs) {
      end_out = e;
      idx_out = (uint64_t)j;
      return true;
    }
  }
  return false;
}

// CG_LOOKUP2=1: the prep's two lookups (a DtoD copy) in lockstep (table_lookup2);
// measured slower on C5 (prep 1.05 -> 1.21 ms at 64 registers, 1.23 at 80) and C2
#ifndef CG_LOOKUP2
#define CG_LOOKUP2 0
#endif
#ifndef CG_FRONT_MINB
#define CG_FRONT_MINB 4   // CTAs per SM of the prep kernels (64 registers)
#endif

// table_lookup for two keys at once (a DtoD copy's destination and source):
// every phase -- the splitter search, the bucket rounds, the walk -- runs for
// both keys in lockstep, so their dependent load chains overlap.  A warp with
// one DtoD lane (C5: 97 % of the warps at 10 % DtoD) waited for two chains
// one after the other.
[[maybe_unused]] __device__ __forceinline__ void table_lookup2(const Table& t, const uint64_t* s_split, const uint64_t key[2],
                                              const bool want[2], uint64_t seq, uint64_t end_out[2],
                                              uint64_t idx_out[2], bool found[2]) {
  const uint64_t pol = evict_last_policy();
  bool act[2];
  uint64_t a[2], b[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    found[q] = false;
    end_out[q] = idx_out[q] = 0;
    act[q] = want[q] && t.nsplit != 0 && s_split[0] <= key[q];
    uint32_t lo = 0, hi = t.nsplit;
    if (act[q])
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (s_split[mid] <= key[q]) lo = mid; else hi = mid;
      }
    a[q] = (uint64_t)lo * t.stride;
    b[q] = umin64(a[q] + t.stride, t.n);
  }
  if (t.stride == 32) {   // (the opt-in stride-64 rounds take the lockstep binary search here)
    constexpr int nq = 4;   // uint4 loads of 2 every-4th bases each
    uint4 v[2][nq];
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int k = 0; k < nq; ++k)
        v[q][k] = act[q] ? ld_keep4(reinterpret_cast<const uint4*>(t.l2 + a[q] / 4) + k, pol) : make_uint4(0, 0, 0, 0);
    uint64_t a1[2];
    uint4 r[2][2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      uint32_t c2 = 0;
#pragma unroll
      for (int k = 0; k < nq; ++k) {
        c2 += (a[q] + 8 * k < b[q] && (((uint64_t)v[q][k].y << 32) | v[q][k].x) <= key[q]) +
              (a[q] + 8 * k + 4 < b[q] && (((uint64_t)v[q][k].w << 32) | v[q][k].z) <= key[q]);
      }
      a1[q] = a[q] + 4 * (c2 > 0 ? c2 - 1 : 0);
#pragma unroll
      for (int k = 0; k < 2; ++k)
        r[q][k] = act[q] ? ld_keep4(reinterpret_cast<const uint4*>(t.base + a1[q]) + k, pol) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      uint32_t c1 = 0;
#pragma unroll
      for (int k = 0; k < 2; ++k)
        c1 += (a1[q] + 2 * k < b[q] && (((uint64_t)r[q][k].y << 32) | r[q][k].x) <= key[q]) +
              (a1[q] + 2 * k + 1 < b[q] && (((uint64_t)r[q][k].w << 32) | r[q][k].z) <= key[q]);
      a[q] = a1[q] + (c1 > 0 ? c1 - 1 : 0);
    }
  } else {
    while ((act[0] && b[0] - a[0] > 1) || (act[1] && b[1] - a[1] > 1)) {
      uint64_t m[2], x[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        m[q] = (a[q] + b[q]) >> 1;
        x[q] = (act[q] && b[q] - a[q] > 1) ? ld_keep(t.base + m[q], pol) : 0;
      }
#pragma unroll
      for (int q = 0; q < 2; ++q)
        if (act[q] && b[q] - a[q] > 1) {
          if (x[q] <= key[q]) a[q] = m[q]; else b[q] = m[q];
        }
    }
  }
  int64_t j[2] = {(int64_t)a[0], (int64_t)a[1]};
  while ((act[0] && j[0] >= 0) || (act[1] && j[1] >= 0)) {   // the prefix-max walks, in lockstep
    uint4 w0[2], w1[2];
#pragma unroll
    for (int q = 0; q < 2; ++q)
      if (act[q] && j[q] >= 0) {
        w0[q] = ld_keep4(t.walk + 2 * j[q], pol);
        w1[q] = ld_keep4(t.walk + 2 * j[q] + 1, pol);   // one 32-byte sector
      }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (!(act[q] && j[q] >= 0)) continue;
      const uint64_t pm = ((uint64_t)w0[q].y << 32) | w0[q].x, e = ((uint64_t)w0[q].w << 32) | w0[q].z;
      const uint64_t as = ((uint64_t)w1[q].y << 32) | w1[q].x, fs = ((uint64_t)w1[q].w << 32) | w1[q].z;
      if (pm <= key[q]) {
        act[q] = false;
      } else if (e > key[q] && as < seq && seq < fs) {
        end_out[q] = e;
        idx_out[q] = (uint64_t)j[q];
        found[q] = true;
        act[q] = false;
      } else {
        --j[q];
      }
    }
  }
}

// NEXT-3: the array with this handle alive at seq -> its total bytes
__device__ __forceinline__ bool array_lookup(const Table& t, uint64_t handle, uint64_t seq, uint64_t& total,
                                             uint64_t& idx) {
  uint64_t lo = 0, hi = t.na;   // first entry with handle >= handle
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (__ldg(t.ahandle + mid) < handle) lo = mid + 1; else hi = mid;
  }
  for (uint64_t j = lo; j < t.na && __ldg(t.ahandle + j) == handle; ++j) {
    if (__ldg(t.aaseq + j) < seq && seq < __ldg(t.afseq + j)) {
      total = __ldg(t.atotal + j);
      idx = j;
      return true;
    }
  }
  return false;
}

// the splitters (every stride-th base) are a contiguous array uploaded with the
// table: coalesced 16-byte loads into shared memory
__device__ __forceinline__ void load_splitters(const Table& t, uint64_t* s_split) {
  const uint4* src = reinterpret_cast<const uint4*>(t.split);
  uint4* dst = reinterpret_cast<uint4*>(s_split);
  for (uint32_t k = threadIdx.x; k < (t.nsplit + 1) / 2; k += blockDim.x) dst[k] = __ldg(src + k);
  __syncthreads();
}

// Check weights (units): HtoD 1 per host byte (V-byte + 1/8 A-byte), DtoH 1 per
// 8 host bytes (A only), plus kItemCost per descriptor (its fixed work).
constexpr uint64_t kItemCost = 256;

__device__ __forceinline__ uint64_t check_host_units(uint32_t skind, uint64_t nscan, bool two_bit) {
  if (two_bit) return (nscan + 3) >> 2;   // NEXT-4: one state byte per 4 host bytes, both kinds
  return skind == CG_HTOD ? nscan : (nscan + 7) >> 3;
}

// ---------------------------------------------------------------------------
// a4: the host shadow scan -- one TMA bulk-copy ring per warp
// ---------------------------------------------------------------------------
// Work: equal-weight groups of the prefix-summed descriptor weights, handed
// out dynamically (one atomic per group).  Inside a group a warp walks its
// descriptors in order; a warp-uniform generator cuts every descriptor's host
// range into row segments (R-11), clips them to the window (bytes outside are
// unaddressable, R-15) and to this GPU's shard, and cuts the shard part into
// tiles that never cross a 4 KiB (HtoD: V bytes) or 32 KiB (DtoH: host bytes
// whose A bits fill 4 KiB) boundary.  Lane 0 stages each tile with
// cp.async.bulk (V and/or A, 128-byte aligned supersets) into the next ring
// slot and arms the slot's mbarrier with the byte count; the warp consumes the
// slots in order from shared memory while kStages-1 later tiles are in flight.
// The descriptor metadata the generator needs comes from a 32-descriptor
// register window (one coalesced load per 32 descriptors).
constexpr int kRingWarps = 4;
constexpr int kStages = 3;
constexpr uint32_t kTileV = 4096;      // HtoD: V bytes per tile
constexpr uint32_t kTileA = kTileV / 8;
// tile blocks (log2 of host bytes): HtoD 4 KiB (= kTileV V bytes), DtoH 32 KiB
// (4 KiB of A), NEXT-4 2-bit states 16 KiB for both kinds (4 KiB of states)
constexpr uint32_t kHtodShift = 12, kDtohShift = 15, k2bitShift = 14;
constexpr uint32_t kGrab = 4;          // chunks per group while the plan is far from its end
constexpr uint32_t kTileData = 1, kTileHtod = 2, kTileEnd = 4, kTileWhole = 8, kTileFuse = 16, kTileRaw = 32,
                   kTileAfter = 64,   // CG_APPLY_AFTER: a DtoH piece the residual pass applies
                   kTileLast = 128,   // CG_APPLY_LAST: ... which k_finish applies after the late checks
                   kTilePacked = 512;   // several whole rows of one 2D DtoH piece (see TileGen::packed_tile)

struct __align__(16) TileInfo {
  uint64_t ob;        // logical offset of staged host byte 0
  uint64_t pend_fu;   // END tiles: first unaddressable offset found analytically
  uint32_t d;         // descriptor
  uint32_t flags;
  uint32_t q0, q1;    // valid host bytes [q0, q1) relative to the staged base
  uint64_t qs, qe;    // kTileFuse END tiles: the piece's shard range (fused DtoH apply)
};

struct WarpRing {
  uint8_t data[kStages][kTileV + kTileA];
  TileInfo info[kStages];
  uint64_t bar[kStages];
};
constexpr size_t kScanSmem = sizeof(WarpRing) * kRingWarps;


__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

struct Partial {
  uint64_t fu, fd, cnt;   // first unaddressable, first undefined, undefined count
};

__device__ __forceinline__ void finalize_fields(uint32_t& flags, uint32_t& status, uint64_t fu, uint64_t cnt,
                                                uint32_t err_mask) {
  if (fu != kNone) flags |= CG_F_HOST_UNADDRESSABLE;
  if (cnt != 0 && fu == kNone) flags |= CG_F_HOST_UNDEFINED;
  status = (flags & err_mask) ? (uint32_t)CG_ERR_INVALID_VALUE : (uint32_t)CG_OK;
}

// HtoD tile: V bytes and their A bits, host bytes [q0, q1) of the staged tile.
// Fast path: lane j folds the 16-byte V units j, j+32, ... (contiguous 16-byte
// lanes: one LDS.128 per lane reads 512 consecutive bytes, bank-conflict free)
// into one OR, and their 16-bit A half-words into one AND (LDS.U16 of 64
// consecutive bytes); only a lane that saw an undefined or unaddressable byte
// rescans its units with per-byte masks (__ffs for the first offset, __popc
// for the count).  The partial 32-byte groups at the tile edges always take
// the masked path.
__device__ __forceinline__ void htod_unit(const uint8_t* st, uint32_t u, uint64_t ob, Partial& p) {
  const uint4 v = reinterpret_cast<const uint4*>(st)[u];
  const uint32_t a = reinterpret_cast<const unsigned short*>(st + kTileV)[u];
  const uint32_t bad = ~a & 0xFFFFu;
  const uint32_t und = nz16(v) & a;
  const uint64_t gb = ob + 16ull * u;
  if (bad) p.fu = umin64(p.fu, gb + (__ffs(bad) - 1));
  if (und) {
    p.fd = umin64(p.fd, gb + (__ffs(und) - 1));
    p.cnt += __popc(und);
  }
}

// a partial 32-byte HtoD group g with the whole warp: lane j looks at host byte 32 g + j
__device__ __forceinline__ void htod_edge(const uint8_t* st, uint32_t g, uint32_t q0, uint32_t q1, uint64_t ob,
                                          Partial& p) {
  const int lane = threadIdx.x & 31;
  const uint32_t x = (g << 5) + lane;
  const bool in = x >= q0 && x < q1;
  const uint32_t a = (st[kTileV + (x >> 3)] >> (x & 7)) & 1u;
  const uint32_t bad = __ballot_sync(kFull, in && !a);
  const uint32_t und = __ballot_sync(kFull, in && a && st[x] != 0);
  if (lane == 0) {
    const uint64_t gb = ob + ((uint64_t)g << 5);
    if (bad) p.fu = umin64(p.fu, gb + (__ffs(bad) - 1));
    if (und) {
      p.fd = umin64(p.fd, gb + (__ffs(und) - 1));
      p.cnt += __popc(und);
    }
  }
}

__device__ __forceinline__ void consume_htod(const uint8_t* st, uint32_t q0, uint32_t q1, uint64_t ob,
                                             Partial& p) {
  const int lane = threadIdx.x & 31;
  const uint32_t i0 = (q0 + 31) >> 5, i1 = q1 >> 5;   // full 32-byte groups [i0, i1) = 16-byte units [2 i0, 2 i1)
  const uint4* V4 = reinterpret_cast<const uint4*>(st);
  const unsigned short* A2 = reinterpret_cast<const unsigned short*>(st + kTileV);
  uint32_t orv = 0, anda = 0xFFFFu;
#pragma unroll 4
  for (uint32_t u = 2 * i0 + lane; u < 2 * i1; u += 32) {
    const uint4 v = V4[u];
    orv |= v.x | v.y | v.z | v.w;
    anda &= A2[u];
  }
  if (orv != 0 || anda != 0xFFFFu)
    for (uint32_t u = 2 * i0 + lane; u < 2 * i1; u += 32) htod_unit(st, u, ob, p);
  // partial edge groups, warp-parallel
  if (i0 > i1) {                                   // [q0, q1) inside one 32-byte group
    htod_edge(st, i1, q0, q1, ob, p);
  } else {
    if (q0 & 31) htod_edge(st, i0 - 1, q0, q1, ob, p);
    if (q1 & 31) htod_edge(st, i1, q0, q1, ob, p);
  }
}

// DtoH tile: A bits only; one 16-byte A vector covers 128 host bytes
__device__ __forceinline__ void dtoh_group(const uint8_t* st, uint32_t i, uint32_t q0, uint32_t q1, uint64_t ob,
                                           Partial& p) {
  const uint4 a = reinterpret_cast<const uint4*>(st)[i];
  const uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t gb = i * 128 + 32 * j;
    if (gb + 32 <= q0 || gb >= q1) continue;
    const uint32_t bad = ~w[j] & range_mask(gb, 32, q0, q1);
    if (bad) {
      p.fu = umin64(p.fu, ob + gb + (__ffs(bad) - 1));
      break;
    }
  }
}

// a partial 128-byte DtoH group g: lanes 0-3 take its four A words
__device__ __forceinline__ void dtoh_edge(const uint8_t* st, uint32_t g, uint32_t q0, uint32_t q1, uint64_t ob,
                                          Partial& p) {
  const int lane = threadIdx.x & 31;
  uint32_t bad = 0;
  if (lane < 4) {
    const uint32_t k = g * 4 + lane;
    const int base = (int)(k << 5);
    const int lo = max((int)q0 - base, 0), hi = min((int)q1 - base, 32);
    if (hi > lo) {
      const uint32_t m = (hi >= 32 ? 0xffffffffu : ((1u << hi) - 1u)) & ~((1u << lo) - 1u);
      bad = ~reinterpret_cast<const uint32_t*>(st)[k] & m;
    }
  }
  const uint32_t any = __ballot_sync(kFull, bad != 0);
  if (any) {
    const int fl = __ffs(any) - 1;
    const uint32_t b = __shfl_sync(kFull, bad, fl);
    if (lane == 0) p.fu = umin64(p.fu, ob + ((uint64_t)(g * 4 + fl) << 5) + (__ffs(b) - 1));
  }
}

__device__ __forceinline__ void consume_dtoh(const uint8_t* st, uint32_t q0, uint32_t q1, uint64_t ob,
                                             Partial& p) {
  const int lane = threadIdx.x & 31;
  const uint32_t i0 = (q0 + 127) >> 7, i1 = q1 >> 7;   // full 128-byte groups [i0, i1)
  const uint4* A16 = reinterpret_cast<const uint4*>(st);
  uint32_t anda = 0xffffffffu;
#pragma unroll 4
  for (uint32_t i = i0 + lane; i < i1; i += 32) {
    const uint4 a = A16[i];
    anda &= a.x & a.y & a.z & a.w;
  }
  if (anda != 0xffffffffu)
    for (uint32_t i = i0 + lane; i < i1; i += 32) dtoh_group(st, i, q0, q1, ob, p);
  if (i0 > i1) {
    dtoh_edge(st, i1, q0, q1, ob, p);
  } else {
    if (q0 & 127) dtoh_edge(st, i0 - 1, q0, q1, ob, p);
    if (q1 & 127) dtoh_edge(st, i1, q0, q1, ob, p);
  }
}


// ---- NEXT-4 2-bit shadow (R-36): 16 host bytes per 32-bit state word ----
// pair mask of host bytes [lo, hi) in the word whose first host byte is gb
__device__ __forceinline__ uint32_t pair_mask(uint64_t gb, uint64_t lo, uint64_t hi) {
  const uint64_t b0 = lo > gb ? umin64(lo - gb, 16) : 0;
  const uint64_t b1 = hi > gb ? umin64(hi - gb, 16) : 0;
  if (b1 <= b0) return 0u;
  const uint32_t him = b1 >= 16 ? 0xffffffffu : ((1u << (2 * b1)) - 1u);
  return him & ~((1u << (2 * b0)) - 1u);
}

// the same for a touched word k of a staged tile (k >= q0 >> 4, 16 k < q1; 32-bit arithmetic)
__device__ __forceinline__ uint32_t pair_mask32(uint32_t k, uint32_t q0, uint32_t q1) {
  const int base = (int)(k << 4);
  const int b0 = max((int)q0 - base, 0), b1 = min((int)q1 - base, 16);
  const uint32_t him = b1 >= 16 ? 0xffffffffu : ((1u << (2 * b1)) - 1u);
  return him & ~((1u << (2 * b0)) - 1u);
}

// one state word: unaddressable = state 0, undefined = bit 0 (PARTIAL / UNDEFINED, always addressable)
template <bool kHtod>
__device__ __forceinline__ void word2(uint32_t w, uint32_t m, uint64_t gb, Partial& p) {
  const uint32_t u = ~(w | (w >> 1)) & 0x55555555u & m;
  if (u) p.fu = umin64(p.fu, gb + ((__ffs(u) - 1) >> 1));
  if (kHtod) {
    const uint32_t und = w & 0x55555555u & m;
    if (und) {
      p.fd = umin64(p.fd, gb + ((__ffs(und) - 1) >> 1));
      p.cnt += __popc(und);
    }
  }
}

// a staged state tile, host bytes [q0, q1): fast fold per 64 host bytes (one
// LDS.128), per-word masks only for dirty groups and the edge words
template <bool kHtod>
__device__ __forceinline__ void consume_2bit(const uint8_t* st, uint32_t q0, uint32_t q1, uint64_t ob, Partial& p) {
  const int lane = threadIdx.x & 31;
  const uint32_t* W = reinterpret_cast<const uint32_t*>(st);
  const uint4* W4 = reinterpret_cast<const uint4*>(st);
  const uint32_t g0 = (q0 + 63) >> 6, g1 = q1 >> 6;   // full 64-byte groups [g0, g1)
  const uint32_t e0 = q0 >> 4, e1 = (q1 + 15) >> 4;   // all words touched
  if (g0 < g1) {
    uint32_t acc = 0;
#pragma unroll 4
    for (uint32_t i = g0 + lane; i < g1; i += 32) {
      const uint4 v = W4[i];
      if (kHtod) {
        acc |= (v.x ^ 0xAAAAAAAAu) | (v.y ^ 0xAAAAAAAAu) | (v.z ^ 0xAAAAAAAAu) | (v.w ^ 0xAAAAAAAAu);
      } else {
        acc |= ~((v.x | (v.x >> 1)) & (v.y | (v.y >> 1)) & (v.z | (v.z >> 1)) & (v.w | (v.w >> 1))) & 0x55555555u;
      }
    }
    if (acc)
      for (uint32_t i = g0 + lane; i < g1; i += 32)
#pragma unroll
        for (uint32_t j = 0; j < 4; ++j) word2<kHtod>(W[4 * i + j], 0xffffffffu, ob + 64ull * i + 16 * j, p);
    if (lane < 4) {
      const uint32_t k = e0 + lane;
      if (k < 4 * g0) word2<kHtod>(W[k], pair_mask32(k, q0, q1), ob + 16ull * k, p);
    } else if (lane < 8) {
      const uint32_t k = 4 * g1 + (lane - 4);
      if (k < e1) word2<kHtod>(W[k], pair_mask32(k, q0, q1), ob + 16ull * k, p);
    }
  } else {
    for (uint32_t k = e0 + lane; k < e1; k += 32) word2<kHtod>(W[k], pair_mask32(k, q0, q1), ob + 16ull * k, p);
  }
}

// states of host bytes [q0, q1) := pat (0x00000000 NOACCESS, 0xAAAAAAAA DEFINED,
// 0xFFFFFFFF UNDEFINED); a partial word is updated in ONE atomic step (CAS
// loop) because a neighbouring range of the same batch may own its other bytes
// and a concurrent scan may read it: an AND-then-OR pair would expose an
// intermediate state (PARTIAL 01 -> 00 -> DEFINED 10 passes through NOACCESS)
__device__ __forceinline__ void fill2_word(uint32_t* S, uint64_t k, uint32_t m, uint32_t pat) {
  if (m == 0xffffffffu) {
    S[k] = pat;
  } else if (m) {
    uint32_t old = *reinterpret_cast<volatile uint32_t*>(S + k), prev;
    do {
      prev = old;
      old = atomicCAS(S + k, prev, (prev & ~m) | (pat & m));
    } while (old != prev);
  }
}

__device__ __forceinline__ void warp_fill2(uint8_t* states, uint64_t q0, uint64_t q1, uint32_t pat) {
  const int lane = threadIdx.x & 31;
  uint32_t* S = reinterpret_cast<uint32_t*>(states);
  const uint64_t g0 = (q0 + 63) >> 6, g1 = q1 >> 6, e0 = q0 >> 4, e1 = (q1 + 15) >> 4;
  if (g0 < g1) {
    uint4* S4 = reinterpret_cast<uint4*>(states);
    for (uint64_t i = g0 + lane; i < g1; i += 32) stg_val16(S4 + i, pat);
    if (lane < 4) {
      const uint64_t k = e0 + lane;
      if (k < 4 * g0) fill2_word(S, k, pair_mask(16ull * k, q0, q1), pat);
    } else if (lane < 8) {
      const uint64_t k = 4 * g1 + (lane - 4);
      if (k < e1) fill2_word(S, k, pair_mask(16ull * k, q0, q1), pat);
    }
  } else {
    for (uint64_t k = e0 + lane; k < e1; k += 32) fill2_word(S, k, pair_mask(16ull * k, q0, q1), pat);
  }
}

__device__ __forceinline__ void lane_fill2(uint8_t* states, uint64_t q0, uint64_t q1, uint32_t pat) {
  uint32_t* S = reinterpret_cast<uint32_t*>(states);
  for (uint64_t k = q0 >> 4; k < (q1 + 15) >> 4; ++k) fill2_word(S, k, pair_mask(16ull * k, q0, q1), pat);
}

// NEXT-4 sparse map: the secondary holding `chunk` (0 = distinguished NOACCESS)
__device__ __forceinline__ uint32_t sparse_secondary(const ShadowView& sv, uint64_t chunk) {
  const uint64_t mask = (1ull << sv.dir_bits) - 1;
  for (uint64_t h = dir_hash(chunk, sv.dir_bits);; h = (h + 1) & mask) {
    const uint64_t k = __ldg(sv.dir_key + h);
    if (k == chunk + 1) return __ldg(sv.dir_val + h);
    if (k == 0) return 0u;
  }
}

// a states base for `chunk`: base + (q >> 2) is the state byte of host byte q of the chunk
__device__ __forceinline__ uint8_t* chunk_base(const ShadowView& sv, uint64_t chunk, uint32_t sec) {
  return reinterpret_cast<uint8_t*>(reinterpret_cast<uintptr_t>(sv.V) + (uint64_t)sec * kSecondaryBytes -
                                    ((chunk << kChunkShift) >> 2));
}

// states of shard bytes [q0, q1) := pat in either 2-bit layout (sparse: chunk
// by chunk; chunks without a secondary are NOACCESS and left alone)
template <bool kWarp, bool kMaySparse = true>
__device__ __forceinline__ void fill2_any(const ShadowView& sv, uint64_t q0, uint64_t q1, uint32_t pat) {
  if (!kMaySparse || !sv.sparse) {
    if (kWarp) warp_fill2(sv.V, q0, q1, pat);
    else lane_fill2(sv.V, q0, q1, pat);
    return;
  }
  if constexpr (kMaySparse)
  for (uint64_t q = q0; q < q1;) {
    const uint64_t c = q >> kChunkShift;
    const uint64_t n = umin64(q1 - q, (1ull << kChunkShift) - (q & ((1ull << kChunkShift) - 1)));
    const uint32_t sec = sparse_secondary(sv, c);
    if (sec) {
      if (kWarp) warp_fill2(chunk_base(sv, c, sec), q, q + n, pat);
      else lane_fill2(chunk_base(sv, c, sec), q, q + n, pat);
    }
    q += n;
  }
}

// V := 0 over shard bytes [q0, q1) with the whole warp (16-byte stores, byte
// stores at the unaligned edges)
__device__ __forceinline__ void warp_store_zero(uint8_t* V, uint64_t q0, uint64_t q1) {
  const int lane = threadIdx.x & 31;
  const uint64_t a0 = (q0 + 15) & ~15ull, a1 = q1 & ~15ull;
  if (a0 >= a1) {
    if (lane < (int)(q1 - q0)) V[q0 + lane] = 0;
    return;
  }
  if (lane < (int)(a0 - q0)) V[q0 + lane] = 0;
  if (lane < (int)(q1 - a1)) V[a1 + lane] = 0;
  uint4* V4 = reinterpret_cast<uint4*>(V);
  for (uint64_t k = (a0 >> 4) + lane; k < (a1 >> 4); k += 32) stg_val16(V4 + k, 0u);
}

// ---------------------------------------------------------------------------
// The small pass: contiguous host sides of at most sv.small_limit (<= 4 KiB)
// bytes are checked by k_check_small instead of the TMA ring: a warp takes 32
// consecutive descriptors (one coalesced meta load) and stages the shadow of
// its small sides in shared memory with one cp.async.bulk per side (two for
// an HtoD side in the bytes format: its V units and its A bytes), as many
// sides per fill as fit kSmallStage bytes, all completing on one mbarrier --
// so a whole window's loads are in flight at once without holding registers
// (the earlier lane-load version kept 64 bytes in flight per lane and spent
// ~2 us per side on dependent DRAM round trips).  Sides of at most 32 units
// (HtoD 512 B, DtoH 4 KiB, 2-bit 2 KiB) are then folded by their own lane,
// longer ones by the whole warp; a unit is 16 shadow bytes (HtoD: 16 V bytes
// and their 16 A bits; DtoH: 16 A bytes = 128 host bytes; 2-bit: 16 state
// bytes = 64 host bytes).  The fold is an OR / AND per unit; masks, __ffs and
// __popc and the warp reduction only run for a side that has a finding.
// ---------------------------------------------------------------------------
#ifndef CG_SMALL_THREADS
#define CG_SMALL_THREADS 256   // 8 warps per CTA, 4 CTAs per SM
#endif
#ifndef CG_SMALL_STAGE
#define CG_SMALL_STAGE 4864   // C5 small pass: 4864 B x 32 warps/SM 1.62 ms < 7168 B x 24 (1.68) < 10240 B x 20 (1.72) < 20480 B x 10 (2.6)
#endif
constexpr int kSmallThreads = CG_SMALL_THREADS;
// staged bytes per warp and fill (a side of <= 4 KiB needs <= 4.7 KB; a C5
// window's small sides ~14 KB: each fill is a DRAM round trip of its warp,
// but more warps per SM hide it better than fewer, larger fills)
constexpr uint32_t kSmallStage = CG_SMALL_STAGE;
// a side of 4 KiB (the limit) stages at most 257 V units + 34 A units = 4656 bytes
static_assert(kSmallStage >= 4656 && kSmallStage % 16 == 0, "the stage must hold the largest small side");
template <bool kTwoBit>
__device__ __forceinline__ uint32_t lane_span(bool htod) {
  return kTwoBit ? 64u : htod ? 16u : 128u;
}


// after a check: the small pass for the next check iff at least sv.small_share
// percent of this batch's host sides had at most sv.small_stat bytes (bytes
// format 80 %: C5 has ~94 %, C2 ~60 %, and C2 runs 1.5 % faster on the ring;
// 2-bit states 50 %: C2 runs 11 % faster on the small pass)
// (counter[9] = 1; 2 = the ring only); the statistics (counter[10..11]:
// smalls << 32 | sides) restart.  A stream of
// similar batches (a program's calls, the bench's steps) is thus served by the
// path that suits it from its second batch on; the result is the same either way.
__device__ __forceinline__ void next_small_choice(uint32_t* counter, uint32_t share) {
  unsigned long long* st = reinterpret_cast<unsigned long long*>(counter + 10);
  const uint64_t sides = st[0] & 0xFFFFFFFFull, smalls = st[0] >> 32;   // <= 2^24 each (kMaxDescs)
  counter[9] = (sides && 100 * smalls >= share * sides) ? 1u : 2u;   // at least share % of the sides small
  st[0] = 0;
}

struct SmallRound {
  uint4 x;      // HtoD: V bytes; DtoH: A bytes; 2-bit: states
  uint32_t a;   // HtoD: the A bits of the 16 V bytes
};

// fold one lane unit [gp, gp + span) of a side [q0, q1) into p (logical offset
// of shard byte q = ob + q)
template <bool kTwoBit>
__device__ __forceinline__ void small_fold(const SmallRound& u, uint64_t gp, uint64_t q0, uint64_t q1, uint64_t ob,
                                           bool htod, Partial& p) {
  if (gp >= q1) return;
  if (kTwoBit) {
    const uint32_t w[4] = {u.x.x, u.x.y, u.x.z, u.x.w};
    const bool inner = gp >= q0 && gp + 64 <= q1;
    if (inner) {   // the common case: a clean unit costs the fold only
      const uint32_t acc = htod ? ((w[0] ^ 0xAAAAAAAAu) | (w[1] ^ 0xAAAAAAAAu) | (w[2] ^ 0xAAAAAAAAu) |
                                   (w[3] ^ 0xAAAAAAAAu))
                                : (~((w[0] | (w[0] >> 1)) & (w[1] | (w[1] >> 1)) & (w[2] | (w[2] >> 1)) &
                                     (w[3] | (w[3] >> 1))) & 0x55555555u);
      if (!acc) return;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint64_t gb = gp + 16u * j;
      if (gb + 16 <= q0 || gb >= q1) continue;
      const uint32_t m = pair_mask(gb, q0, q1);
      if (htod) word2<true>(w[j], m, ob + gb, p);
      else word2<false>(w[j], m, ob + gb, p);
    }
    return;
  }
  if (htod) {
    const uint32_t m = (gp >= q0 && gp + 16 <= q1) ? 0xFFFFu : range_mask(gp, 16, q0, q1);
    if ((u.x.x | u.x.y | u.x.z | u.x.w) == 0 && (u.a & m) == m) return;   // clean
    const uint32_t bad = ~u.a & m, und = nz16(u.x) & u.a & m;
    if (bad) p.fu = umin64(p.fu, ob + gp + (__ffs(bad) - 1));
    if (und) {
      p.fd = umin64(p.fd, ob + gp + (__ffs(und) - 1));
      p.cnt += __popc(und);
    }
    return;
  }
  if (gp >= q0 && gp + 128 <= q1 && (u.x.x & u.x.y & u.x.z & u.x.w) == 0xFFFFFFFFu) return;   // clean
  const uint32_t w[4] = {u.x.x, u.x.y, u.x.z, u.x.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint64_t gb = gp + 32u * j;
    if (gb + 32 <= q0 || gb >= q1) continue;
    const uint32_t bad = ~w[j] & range_mask(gb, 32, q0, q1);
    if (bad) {
      p.fu = umin64(p.fu, ob + gb + (__ffs(bad) - 1));
      break;
    }
  }
}

// The warp's descriptors [base, base + 32) (lane k gets base + k): 16-byte
// coalesced loads through a per-warp staging area, half a window at a time
// (16 descriptors, rows padded to 112 bytes so that the LDS.128 reads of eight
// lanes hit distinct banks); a descriptor array that is not 16-byte aligned
// (the header allows 8) falls back to per-lane loads.  Lane-per-descriptor
// loads of the 96-byte records touch 24 cache lines per instruction, which
// kept the L1 of k_front 70 % busy.
constexpr int kDescRow = 7;   // uint4 per staged descriptor (6 + 1 pad)
#ifndef CG_PREP_STAGED_STORES
#define CG_PREP_STAGED_STORES 1   // verdicts and scan records leave the prep through the staging area too
#endif
__device__ __forceinline__ cg_copy_desc warp_load_desc(const cg_copy_desc* __restrict__ descs, uint64_t base,
                                                       uint64_t n, uint4* stage) {
  const int lane = threadIdx.x & 31;
  union {
    cg_copy_desc d;
    uint4 u[6];
  } r;
  r.d.kind = 0;
  if (reinterpret_cast<uintptr_t>(descs) & 15) {
    if (base + lane < n) r.d = descs[base + lane];
    return r.d;
  }
  const uint4* src = reinterpret_cast<const uint4*>(descs + base);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const uint64_t b = base + 16 * h;
    const uint32_t cnt = b < n ? (uint32_t)umin64(16, n - b) : 0u;
    for (uint32_t k = lane; k < cnt * 6; k += 32) stage[(k / 6) * kDescRow + k % 6] = __ldcs(src + 96 * h + k);
    __syncwarp();
    if ((lane >> 4) == h && (uint32_t)(lane & 15) < cnt) {
#pragma unroll
      for (int j = 0; j < 6; ++j) r.u[j] = stage[(lane & 15) * kDescRow + j];
    }
    __syncwarp();
  }
  return r.d;
}

__device__ __forceinline__ void prep_body(const cg_copy_desc* __restrict__ descs, uint64_t n, const Table& t,
                                          cg_verdict* __restrict__ out, uint64_t* __restrict__ weight,
                                          ScanMeta* __restrict__ meta, uint64_t* __restrict__ dvoff,
                                          const ShadowView& sv, uint32_t* __restrict__ counter,
                                          uint32_t* __restrict__ defer, uint64_t* s_split, uint32_t err_mask,
                                          int fuse, uint32_t* __restrict__ late) {
  // the scan's group counter and the apply count: reset here instead of by a
  // memset node, which would break the PDL chain.  The residual list (count:
  // counter[2]) and the deferred list (count, cursor: counter[4], [5]) are
  // appended to right here, so the kernels after the scan (k_finish,
  // k_finalize_split) reset them for the next check.
  if (blockIdx.x == 0 && threadIdx.x < 2) counter[threadIdx.x] = 0;
  __shared__ uint4 s_desc[kThreads / 32][16 * kDescRow];
  const bool small_on = sv.small_mode == 1 ||
                        (sv.small_mode == 0 && *reinterpret_cast<volatile const uint32_t*>(counter + 9) == 1u);
  load_splitters(t, s_split);
  const int lane = threadIdx.x & 31;
  const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < n; base += nthr) {
    const uint64_t i = base + lane;
    const bool act = i < n;
    cg_copy_desc d = warp_load_desc(descs, base, n, s_desc[threadIdx.x >> 5]);
    if (!act) d.kind = 0;
    const Norm nm = normalize(d);
    uint32_t flags = nm.flags;
    uint64_t de = 0, df = 0, se = 0, sf = 0;
    const bool owner = !(d.reserved & CG_SHARD_NOT_OWNER);   // only the owner shard looks up the device side
    uint64_t dv_dst = 0, dv_src = 0;   // NEXT-1: device V-bit offsets in the pool
    if (act && nm.kind >= CG_HTOA && owner) {  // NEXT-3: array side
      const bool htoa = nm.kind == CG_HTOA;
      uint64_t total, j;
      if (nm.aok) {
        if (!array_lookup(t, nm.ahandle, d.seq, total, j)) {
          flags |= htoa ? CG_F_DST_NOT_ALLOCATED : CG_F_SRC_NOT_ALLOCATED;
        } else {
          if (nm.aoff + d.width * d.height > total) {
            flags |= htoa ? CG_F_DST_TOO_SMALL : CG_F_SRC_TOO_SMALL;
            const uint64_t ex = d.width * d.height, fd = nm.aoff < total ? total - nm.aoff : 0;
            if (htoa) { de = ex; df = fd; } else { se = ex; sf = fd; }
          }
          // NEXT-1 x NEXT-3 (S:252 per-array shadow, R-30): the array side's V-bits in the pool
          if (t.apool) (htoa ? dv_dst : dv_src) = __ldg(t.apool + j) + nm.aoff;
        }
      }
#if CG_LOOKUP2
    } else if (act && !(flags & CG_F_BAD_KIND) && owner) {
      // dst side first in the flag order; both lookups in lockstep
      const uint64_t key[2] = {nm.ds, nm.ss};
      const bool want[2] = {(nm.kind == CG_HTOD || nm.kind == CG_DTOD) && nm.dok,
                            (nm.kind == CG_DTOH || nm.kind == CG_DTOD) && nm.sok};
      uint64_t end[2], j[2];
      bool found[2];
      table_lookup2(t, s_split, key, want, d.seq, end, j, found);
      if (want[0]) {
        if (!found[0]) {
          flags |= CG_F_DST_NOT_ALLOCATED;
        } else {
          if (end[0] - nm.ds < nm.dspan) {
            flags |= CG_F_DST_TOO_SMALL;
            de = nm.dspan;
            df = end[0] - nm.ds;
          }
          if (t.pool) dv_dst = __ldg(t.pool + j[0]) + (nm.ds - __ldg(t.base + j[0]));
        }
      }
      if (want[1]) {
        if (!found[1]) {
          flags |= CG_F_SRC_NOT_ALLOCATED;
        } else {
          if (end[1] - nm.ss < nm.sspan) {
            flags |= CG_F_SRC_TOO_SMALL;
            se = nm.sspan;
            sf = end[1] - nm.ss;
          }
          if (t.pool) dv_src = __ldg(t.pool + j[1]) + (nm.ss - __ldg(t.base + j[1]));
        }
      }
    }
#else
    } else if (act && !(flags & CG_F_BAD_KIND) && owner) {
      uint64_t end, j;
      if ((nm.kind == CG_HTOD || nm.kind == CG_DTOD) && nm.dok) {      // dst side first
        if (!table_lookup(t, s_split, nm.ds, d.seq, end, j)) {
          flags |= CG_F_DST_NOT_ALLOCATED;
        } else {
          if (end - nm.ds < nm.dspan) {
            flags |= CG_F_DST_TOO_SMALL;
            de = nm.dspan;
            df = end - nm.ds;
          }
          if (t.pool) dv_dst = __ldg(t.pool + j) + (nm.ds - __ldg(t.base + j));
        }
      }
      if ((nm.kind == CG_DTOH || nm.kind == CG_DTOD) && nm.sok) {
        if (!table_lookup(t, s_split, nm.ss, d.seq, end, j)) {
          flags |= CG_F_SRC_NOT_ALLOCATED;
        } else {
          if (end - nm.ss < nm.sspan) {
            flags |= CG_F_SRC_TOO_SMALL;
            se = nm.sspan;
            sf = end - nm.ss;
          }
          if (t.pool) dv_src = __ldg(t.pool + j) + (nm.ss - __ldg(t.base + j));
        }
      }
    }
#endif
    if (act && t.pool) {
      dvoff[2 * i] = dv_dst;
      dvoff[2 * i + 1] = dv_src;
    }
    // R-10 / R-15: the shard part of the host side, and the analytic first
    // offset outside the window (initial first_unaddr: partials min into it)
    HostClip hc{0, 0, kNone, false};
    if (act && nm.host) hc = host_clip(nm, d.height, sv);
    // CG_CHECK_AFTER (fused only): checked by k_finish after the batch's applies
    // (fuse == 2: cg_check_apply, whose k_finish runs the late pass and the
    // CG_APPLY_LAST applies after it; fuse == 1 treats CG_APPLY_LAST as CG_APPLY_AFTER)
    const bool is_late = act && fuse == 2 && nm.host && nm.skind == CG_HTOD && (d.reserved & CG_CHECK_AFTER);
    const bool is_last = act && fuse == 2 && nm.host && nm.skind == CG_DTOH && (d.reserved & CG_APPLY_LAST);
    const bool is_after = (d.reserved & (CG_APPLY_AFTER | CG_APPLY_LAST)) != 0;
    const bool deferred = act && nm.host && !is_late && (hc.overlap || (sv.sparse && hc.ohi - hc.olo > kDeferBytes));
    const uint64_t nscan = act && nm.host && !deferred && !is_late ? hc.ohi - hc.olo : 0;
    if (deferred) defer[atomicAdd(counter + 4, 1u)] = (uint32_t)i;
    if (is_late) late[atomicAdd(counter + 6, 1u)] = (uint32_t)i;
    const bool contig = d.height == 1 || d.width == nm.hpitch;
    const bool raw = d.reserved & CG_SHARD_RAW;   // partial of a straddler: no finalisation here
    // the small pass (every format; in the sparse map a side inside one 64 KiB
    // chunk): contiguous, whole, not raw -- checked by k_check_small, not by
    // the ring; its verdict is written
    // here already finalised as if the host side were clean (k_check_small
    // rewrites only the dirty ones)
    // the small pass runs when the previous check's sides were small on average
    // (counter[9] == 1, decided after each check from the statistics below:
    // many descriptors with few bytes each, C5); else (C2) the ring checks the
    // small sides too, their latency hidden behind the big tiles' streams
    const uint64_t xs = nm.hstart + (sv.sb > nm.hstart ? sv.sb - nm.hstart : 0);   // the side's first shard byte
    const bool small = nscan != 0 && nscan <= sv.small_limit && contig && !raw && small_on &&
                       (!sv.sparse || (xs >> kChunkShift) == ((xs + nscan - 1) >> kChunkShift));
    {   // the statistics of the small-pass choice: host sides, and those of at most sv.small_stat
      const uint32_t sides = __popc(__ballot_sync(kFull, nscan != 0));
      const uint32_t smalls = __popc(__ballot_sync(kFull, nscan != 0 && nscan <= sv.small_stat));
      if (lane == 0 && sides)
        atomicAdd(reinterpret_cast<unsigned long long*>(counter + 10),
                  ((unsigned long long)smalls << 32) | (unsigned long long)sides);
    }
    union {
      cg_verdict v;
      uint4 u[4];
    } V;
    union {
      ScanMeta m;
      uint4 u[2];
    } M;
    V.v.first_unaddr = hc.pfu;
    V.v.first_undef = kNone;
    V.v.undef_count = 0;
    V.v.dst_expected = de;
    V.v.dst_found = df;
    V.v.src_expected = se;
    V.v.src_found = sf;
    V.v.flags = flags;
    V.v.status = 0;
    if (small) finalize_fields(V.v.flags, V.v.status, V.v.first_unaddr, 0, err_mask);
    if (act) weight[i] = small ? 0 : kItemCost + check_host_units(nm.skind, nscan, sv.two_bit != 0);
    M.m.hstart = nm.hstart;
    M.m.hpitch = nm.hpitch;
    M.m.W = nm.W;
    M.m.info = nscan | ((uint64_t)(nm.skind & 3u) << kInfoKind) | ((uint64_t)(nscan != 0) << kInfoHost) |
               ((uint64_t)contig << kInfoContig) | ((uint64_t)raw << kInfoRaw) |
               ((uint64_t)(hc.pfu != kNone) << kInfoPfu) | ((uint64_t)(deferred || small || is_late) << kInfoDefer) |
               ((uint64_t)is_after << kInfoAfter) | ((uint64_t)flags << kInfoFlags) |
               ((uint64_t)small << kInfoSmall) | ((uint64_t)is_last << kInfoLast);
    // the 64-byte verdicts and 32-byte records of the warp's descriptors:
    // coalesced 16-byte stores through the staging area (an 8-byte store per
    // lane and field touched 32 sectors per instruction)
    uint4* stg = s_desc[threadIdx.x >> 5];
    if (CG_PREP_STAGED_STORES && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint64_t b = base + 16 * h;
        const uint32_t cnt = b < n ? (uint32_t)umin64(16, n - b) : 0u;
        if ((lane >> 4) == h && (uint32_t)(lane & 15) < cnt) {
          uint4* row = stg + (lane & 15) * kDescRow;
#pragma unroll
          for (int j = 0; j < 4; ++j) row[j] = V.u[j];
          row[4] = M.u[0];
          row[5] = M.u[1];
        }
        __syncwarp();
        uint4* ov = reinterpret_cast<uint4*>(out + b);
        uint4* om = reinterpret_cast<uint4*>(meta + b);
        for (uint32_t k = lane; k < cnt * 4; k += 32) ov[k] = stg[(k >> 2) * kDescRow + (k & 3)];
        if ((uint32_t)lane < cnt * 2) om[lane] = stg[(lane >> 1) * kDescRow + 4 + (lane & 1)];
        __syncwarp();
      }
    } else if (act) {
      out[i] = V.v;
      meta[i] = M.m;
    }
  }
}

// a DtoH side with status OK that a later pass applies: a CG_APPLY_LAST one to
// the last list (count counter[8] = resid_n[6]; k_finish applies it after the
// late checks), any other to the residual list (count counter[2] = resid_n[0])
__device__ __forceinline__ void push_apply(bool is_last, uint32_t d, uint32_t* __restrict__ resid,
                                           uint32_t* __restrict__ resid_n, uint32_t* __restrict__ last) {
  if (is_last) last[atomicAdd(resid_n + 6, 1u)] = d;
  else resid[atomicAdd(resid_n, 1u)] = d;
}

#ifndef CG_SMALL_VERIFY
#define CG_SMALL_VERIFY 0   // debug builds: every staged side re-checked from global memory
#endif
#if CG_SMALL_VERIFY
__device__ uint32_t g_small_verify;
#endif

// a staged small side (k_check_small's pass 1): its main units at stage + off
// (16 bytes each), HtoD bytes format: its A half-words from stage + aoff, the
// inclusive unit count of the fill's sides up to it, the bytes outside the
// side at the start of unit 0 (skip) and the bytes inside it in the last unit
// (keep)
struct SmallSide {
  uint32_t off, aoff, uincl, units;
  uint32_t skip, keep;
  bool htod;
};

template <bool kTwoBit>
__device__ __forceinline__ uint32_t sh_of(bool htod) {
  return kTwoBit ? 6u : htod ? 4u : 7u;
}

// bits [lo, hi) of a 32-bit group starting at bit b (lo, hi, b in bits of one unit)
__device__ __forceinline__ uint32_t bits_in(uint32_t b, uint32_t lo, uint32_t hi) {
  const uint32_t l = lo > b ? lo - b : 0u, h = hi > b ? min(hi - b, 32u) : 0u;
  if (h <= l) return 0u;
  return (h >= 32 ? 0xffffffffu : ((1u << h) - 1u)) & ~((1u << l) - 1u);
}

// unit k of a staged side clean (no unaddressable byte; HtoD: no undefined
// byte) over its host bytes [lo, hi) relative to the unit's first byte
template <bool kTwoBit>
__device__ __forceinline__ bool small_unit_clean(const uint4& v, const uint8_t* stage, const SmallSide& r, uint32_t k,
                                                 uint32_t lo, uint32_t hi) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  if (kTwoBit) {   // 16 host bytes per state word, 2 bits each
    if (lo == 0 && hi == 64)   // an inner unit (the common case): no masks
      return r.htod ? ((w[0] ^ 0xAAAAAAAAu) | (w[1] ^ 0xAAAAAAAAu) | (w[2] ^ 0xAAAAAAAAu) | (w[3] ^ 0xAAAAAAAAu)) == 0
                    : (~((w[0] | (w[0] >> 1)) & (w[1] | (w[1] >> 1)) & (w[2] | (w[2] >> 1)) & (w[3] | (w[3] >> 1))) &
                       0x55555555u) == 0;
    uint32_t bad = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t l = lo > 16u * i ? min(lo - 16u * i, 16u) : 0u;
      const uint32_t h = hi > 16u * i ? min(hi - 16u * i, 16u) : 0u;
      const uint32_t m = h <= l ? 0u : ((h >= 16 ? 0xffffffffu : ((1u << (2 * h)) - 1u)) & ~((1u << (2 * l)) - 1u));
      bad |= (r.htod ? (w[i] ^ 0xAAAAAAAAu) : (~(w[i] | (w[i] >> 1)) & 0x55555555u)) & m;
    }
    return bad == 0;
  }
  if (r.htod) {   // 16 V bytes and their 16 A bits
    const uint32_t a = *reinterpret_cast<const unsigned short*>(stage + r.aoff + 2 * k);
    if (lo == 0 && hi == 16) return a == 0xFFFFu && (w[0] | w[1] | w[2] | w[3]) == 0;   // an inner unit
    const uint32_t m = bits_in(0, lo, hi) & 0xFFFFu;
    if ((a & m) != m) return false;
    return (w[0] | w[1] | w[2] | w[3]) == 0 || (nz16(v) & m) == 0;
  }
  // DtoH: 16 A bytes = 128 host bytes
  if (lo == 0 && hi == 128) return (w[0] & w[1] & w[2] & w[3]) == 0xffffffffu;
  uint32_t bad = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) bad |= ~w[i] & bits_in(32u * i, lo, hi);
  return bad == 0;
}

// The small pass (a4-a6 for small contiguous host sides; see kSmallStage):
// a dirty verdict is rewritten, a clean one was final already (the prep
// wrote it); small DtoH sides with status OK are applied here when fused (a6)
// unless CG_APPLY_AFTER sends them to the residual pass.
#ifndef CG_SMALL_MINB
#define CG_SMALL_MINB 4   // 64 registers, 32 warps per SM
#endif
template <bool kTwoBit>
__global__ void __launch_bounds__(kSmallThreads, CG_SMALL_MINB) k_check_small(const ScanMeta* __restrict__ meta, uint64_t n,
                                                          ShadowView sv, cg_verdict* __restrict__ out,
                                                          uint32_t err_mask, int fuse, uint32_t* __restrict__ resid,
                                                          uint32_t* __restrict__ resid_n, uint32_t* __restrict__ last) {
  pdl_entry();
  if (sv.small_mode == 2 || (sv.small_mode == 0 && *reinterpret_cast<volatile const uint32_t*>(resid_n + 7) != 1u))
    return;   // counter[9]: the ring takes them all
  __shared__ __align__(128) uint8_t s_stage[kSmallThreads / 32][kSmallStage];
  __shared__ uint64_t s_bar[kSmallThreads / 32];
  __shared__ SmallSide s_side[kSmallThreads / 32][32];
  __shared__ __align__(16) uint8_t s_umap[kSmallThreads / 32][kSmallStage / 16 + 16];
  const int lane = threadIdx.x & 31;
  uint8_t* stage = s_stage[threadIdx.x >> 5];
  uint64_t* bar = &s_bar[threadIdx.x >> 5];
  SmallSide* side = s_side[threadIdx.x >> 5];
  uint8_t* umap = s_umap[threadIdx.x >> 5];
  if (lane == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint32_t parity = 0;
  const uint64_t policy = evict_first_policy();
  const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < n; base += nthr) {
    const uint64_t i = base + lane;
    uint64_t info = 0, x0 = 0;
    if (i < n) {
      const ScanMeta m = meta[i];
      info = m.info;
      x0 = m.hstart;
    }
    const bool small = (info >> kInfoSmall) & 1u;
    uint32_t todo = __ballot_sync(kFull, small);
    if (!todo) continue;
    const bool htod = ((info >> kInfoKind) & 3u) == CG_HTOD;
    uint64_t q0 = 0, q1 = 0, ob = 0;
    if (small) {   // shard bytes [x, x + nscan); logical offset of shard byte q = q + sb - x0 (R-10 clip)
      const uint64_t x = x0 + (sv.sb > x0 ? sv.sb - x0 : 0);
      q0 = x - sv.sb;
      q1 = q0 + (info & kInfoBytes);
      ob = sv.sb - x0;
    }
    Partial mine{kNone, kNone, 0};
    // staging: the side's shadow units (16 bytes each: HtoD V, DtoH A, 2-bit
    // states; lane unit gp = g0 + k span) and, HtoD bytes format, its A bytes
    const uint32_t sh = kTwoBit ? 6u : htod ? 4u : 7u;   // log2 of the host bytes per unit
    const uint64_t g0 = q0 & ~((1ull << sh) - 1);
    const uint32_t mlen = small ? (uint32_t)(((q1 - g0 + (1ull << sh) - 1) >> sh) << 4) : 0u;
    uint64_t ab = 0;
    uint32_t alen = 0;
    if (!kTwoBit && htod && small) {
      ab = (g0 >> 3) & ~15ull;
      alen = (uint32_t)((((q1 + 127) & ~127ull) >> 3) - ab);
    }
    const uint32_t need = mlen + alen;   // <= 4.7 KB for a side of <= 4 KiB
    uint32_t rem = todo;
    while (rem) {   // fills: the longest prefix of the remaining sides that fits the stage
      const bool cand = (rem >> lane) & 1u;
      const uint32_t x = cand ? need : 0u;
      uint32_t incl = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
      }
      const bool in = cand && incl <= kSmallStage;
      const uint32_t fill = __ballot_sync(kFull, in);
      const uint32_t total = __shfl_sync(kFull, incl, 31 - __clz(fill));
      const uint32_t off = incl - x;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // the last fill's generic reads first
      if (lane == 0) mbar_arrive_tx(bar, total);
      __syncwarp();
      if (in) {
        const uint8_t* src = !kTwoBit ? (htod ? sv.V + g0 : sv.A + (g0 >> 3))
                             : sv.sparse ? chunk_base(sv, g0 >> kChunkShift, sparse_secondary(sv, g0 >> kChunkShift)) + (g0 >> 2)
                                         : sv.V + (g0 >> 2);
        bulk_g2s(stage + off, src, mlen, bar, policy);
        if (alen) bulk_g2s(stage + off + mlen, sv.A + ab, alen, bar, policy);
      }
      mbar_wait(bar, parity);
      parity ^= 1u;
      // pass 1: every unit of the fill, spread evenly over the lanes (flat unit
      // f -> side j = the lane whose inclusive unit count first exceeds f):
      // only which sides have a finding
      const uint32_t units = in ? (mlen >> 4) : 0u;
      uint32_t uincl = units;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, uincl, o);
        if (lane >= o) uincl += y;
      }
      const uint32_t U = __shfl_sync(kFull, uincl, 31);
      {
        SmallSide r;
        r.off = off;
        r.aoff = off + mlen + (uint32_t)((g0 >> 3) - ab);
        r.uincl = uincl;
        r.units = units;
        r.skip = (uint32_t)(q0 - g0);
        r.keep = units ? (uint32_t)(q1 - (g0 + ((uint64_t)(units - 1) << sh))) : 0u;
        r.htod = htod;
        side[lane] = r;
      }
      // the unit -> side map of the fill (one byte per unit, side + 1): side
      // starts marked, then a prefix maximum (a block of ceil(U / 32) units
      // per lane, the carries by a warp max-scan)
      for (uint32_t w = lane; w < (U + 3) >> 2; w += 32) reinterpret_cast<uint32_t*>(umap)[w] = 0u;
      __syncwarp();
      if (units) umap[uincl - units] = (uint8_t)(lane + 1);
      __syncwarp();
      {
        const uint32_t B = (U + 31) >> 5, b0 = min(U, lane * B), b1 = min(U, b0 + B);
        uint32_t run = 0;
        for (uint32_t f = b0; f < b1; ++f) run = max(run, (uint32_t)umap[f]);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(kFull, run, o);
          if (lane >= o) run = max(run, y);
        }
        uint32_t cur = __shfl_up_sync(kFull, run, 1);
        if (lane == 0) cur = 0;
        for (uint32_t f = b0; f < b1; ++f) {
          cur = max(cur, (uint32_t)umap[f]);
          umap[f] = (uint8_t)cur;
        }
      }
      __syncwarp();
      uint32_t dirty = 0;   // lane-local: bit j = side j has a finding
      for (uint32_t f = lane; f < U; f += 32) {
        const uint32_t j = umap[f] - 1u;
        const SmallSide& r = side[j];
        const uint32_t k = f - (r.uincl - r.units);
        const uint4 v = *reinterpret_cast<const uint4*>(stage + r.off + 16 * k);
        const uint32_t lo = k == 0 ? r.skip : 0u, hi = k + 1 == r.units ? r.keep : (1u << sh_of<kTwoBit>(r.htod));
        if (!small_unit_clean<kTwoBit>(v, stage, r, k, lo, hi)) dirty |= 1u << j;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) dirty |= __shfl_xor_sync(kFull, dirty, o);
#if CG_SMALL_VERIFY
      {   // debug: every side of the fill, exactly from the stage and from global memory
        uint32_t all = fill;
        while (all) {
          const int jj = __ffs(all) - 1;
          all &= all - 1;
          const uint64_t cq0 = __shfl_sync(kFull, q0, jj), cq1 = __shfl_sync(kFull, q1, jj);
          const uint64_t cob = __shfl_sync(kFull, ob, jj), cg0 = __shfl_sync(kFull, g0, jj);
          const uint64_t cab = __shfl_sync(kFull, ab, jj);
          const uint32_t coff = __shfl_sync(kFull, off, jj), cm = __shfl_sync(kFull, mlen, jj);
          const bool ch = __shfl_sync(kFull, htod, jj);
          const uint32_t csh = kTwoBit ? 6u : ch ? 4u : 7u;
          const bool cd = __shfl_sync(kFull, dirty, 0) >> jj & 1u;
          Partial ps{kNone, kNone, 0}, pg{kNone, kNone, 0};
          uint32_t diffs = 0;
          for (uint32_t k = lane; k < (cm >> 4); k += 32) {
            const uint64_t gp = cg0 + ((uint64_t)k << csh);
            SmallRound u, g;
            u.x = *reinterpret_cast<const uint4*>(stage + coff + 16 * k);
            u.a = (!kTwoBit && ch) ? *reinterpret_cast<const unsigned short*>(stage + coff + cm + ((gp >> 3) - cab))
                                   : 0xFFFFu;
            g.x = __ldcg(reinterpret_cast<const uint4*>(kTwoBit ? sv.V + (gp >> 2) : ch ? sv.V + gp : sv.A + (gp >> 3)));
            g.a = (!kTwoBit && ch) ? __ldcg(reinterpret_cast<const unsigned short*>(sv.A + (gp >> 3))) : 0xFFFFu;
            if (u.x.x != g.x.x || u.x.y != g.x.y || u.x.z != g.x.z || u.x.w != g.x.w || u.a != g.a) ++diffs;
            small_fold<kTwoBit>(u, gp, cq0, cq1, cob, ch, ps);
            small_fold<kTwoBit>(g, gp, cq0, cq1, cob, ch, pg);
          }
          ps.fu = warp_min(ps.fu); ps.fd = warp_min(ps.fd); ps.cnt = warp_sum(ps.cnt);
          pg.fu = warp_min(pg.fu); pg.fd = warp_min(pg.fd); pg.cnt = warp_sum(pg.cnt);
          diffs = (uint32_t)warp_sum(diffs);
          const bool gd = pg.fu != kNone || pg.fd != kNone || pg.cnt != 0;
          if (lane == 0 && (diffs || gd != cd || ps.fu != pg.fu || ps.fd != pg.fd || ps.cnt != pg.cnt) &&
              atomicAdd(&g_small_verify, 1u) < 40)
            printf("VERIFY i=%llu side=%d htod=%d q0=%llu q1=%llu off=%u mlen=%u total=%u fill=%08x diffs=%u dirty=%d/%d "
                   "stage(%llx,%llx,%llu) global(%llx,%llx,%llu)\n",
                   (unsigned long long)(base + jj), jj, (int)ch, (unsigned long long)cq0, (unsigned long long)cq1,
                   coff, cm, total, fill, diffs, (int)cd, (int)gd, (unsigned long long)ps.fu,
                   (unsigned long long)ps.fd, (unsigned long long)ps.cnt, (unsigned long long)pg.fu,
                   (unsigned long long)pg.fd, (unsigned long long)pg.cnt);
        }
      }
#endif
      // pass 2: a side with a finding, exactly, by the whole warp
      while (dirty) {
        const int jj = __ffs(dirty) - 1;
        dirty &= dirty - 1;
        const uint64_t cq0 = __shfl_sync(kFull, q0, jj), cq1 = __shfl_sync(kFull, q1, jj);
        const uint64_t cob = __shfl_sync(kFull, ob, jj), cg0 = __shfl_sync(kFull, g0, jj);
        const uint64_t cab = __shfl_sync(kFull, ab, jj);
        const uint32_t coff = __shfl_sync(kFull, off, jj), cm = __shfl_sync(kFull, mlen, jj);
        const bool ch = __shfl_sync(kFull, htod, jj);
        const uint32_t csh = kTwoBit ? 6u : ch ? 4u : 7u;
        Partial p{kNone, kNone, 0};
        for (uint32_t k = lane; k < (cm >> 4); k += 32) {
          const uint64_t gp = cg0 + ((uint64_t)k << csh);
          SmallRound u;
          u.x = *reinterpret_cast<const uint4*>(stage + coff + 16 * k);
          u.a = (!kTwoBit && ch) ? *reinterpret_cast<const unsigned short*>(stage + coff + cm + ((gp >> 3) - cab))
                                 : 0xFFFFu;
          small_fold<kTwoBit>(u, gp, cq0, cq1, cob, ch, p);
        }
        p.fu = warp_min(p.fu);
        p.fd = warp_min(p.fd);
        p.cnt = warp_sum(p.cnt);
        if (lane == jj) mine = p;
      }
      rem &= ~fill;
      __syncwarp();
    }
    bool apply_me = false;
    if (small) {
      uint64_t fu = mine.fu;
      if ((info >> kInfoPfu) & 1u) fu = umin64(fu, out[i].first_unaddr);
      uint32_t flags = (uint32_t)((info >> kInfoFlags) & 0x3FFu), status;
      finalize_fields(flags, status, fu, mine.cnt, err_mask);
      if (fu != kNone || mine.fd != kNone || mine.cnt) {   // dirty: rewrite (clean verdicts are final already)
        cg_verdict* v = out + i;
        v->first_unaddr = fu;
        v->first_undef = mine.fd;
        v->undef_count = mine.cnt;
        v->flags = flags;
        v->status = status;
      }
      if (fuse && !htod && status == CG_OK) {
        if ((info >> kInfoAfter) & 1u) push_apply((info >> kInfoLast) & 1u, (uint32_t)i, resid, resid_n, last);
        else apply_me = true;
      }
    }
    // fused a6: a side of at most 512 bytes by its own lane (16-byte stores,
    // byte stores at the edges), bigger ones by the whole warp
    if (apply_me && q1 - q0 <= 512) {
      if (kTwoBit) {
        fill2_any<false>(sv, q0, q1, 0xAAAAAAAAu);
      } else {
        const uint64_t a0 = (q0 + 15) & ~15ull, a1 = q1 & ~15ull;
        if (a0 >= a1) {
          for (uint64_t q = q0; q < q1; ++q) sv.V[q] = 0;
        } else {
          for (uint64_t q = q0; q < a0; ++q) sv.V[q] = 0;
          for (uint64_t q = a0; q < a1; q += 16) stg_val16(reinterpret_cast<uint4*>(sv.V + q), 0u);
          for (uint64_t q = a1; q < q1; ++q) sv.V[q] = 0;
        }
      }
      apply_me = false;
    }
    uint32_t ap = __ballot_sync(kFull, apply_me);
    while (ap) {   // fused a6, the whole warp per side
      const int k = __ffs(ap) - 1;
      ap &= ap - 1;
      const uint64_t a = __shfl_sync(kFull, q0, k), b = __shfl_sync(kFull, q1, k);
      if (kTwoBit) fill2_any<true>(sv, a, b, 0xAAAAAAAAu);
      else warp_store_zero(sv.V, a, b);
    }
  }
}

__global__ void __launch_bounds__(kThreads, CG_FRONT_MINB) k_check_prep(const cg_copy_desc* __restrict__ descs,
                                                         uint64_t n, Table t, cg_verdict* __restrict__ out,
                                                         uint64_t* __restrict__ weight,
                                                         ScanMeta* __restrict__ meta,
                                                         uint64_t* __restrict__ dvoff, ShadowView sv,
                                                         uint32_t* __restrict__ counter,
                                                         uint32_t* __restrict__ defer, uint32_t err_mask, int fuse,
                                                         uint32_t* __restrict__ late) {
  pdl_entry();
  extern __shared__ uint64_t s_split[];
  prep_body(descs, n, t, out, weight, meta, dvoff, sv, counter, defer, s_split, err_mask, fuse, late);
}

// ---------------------------------------------------------------------------
// a2: exclusive prefix sum (3 kernels) and the chunk plan
// ---------------------------------------------------------------------------
constexpr int kScanThreads = 256;
constexpr int kScanItems = kScanTile / kScanThreads;   // 8

__device__ __forceinline__ uint64_t block_exclusive_scan(uint64_t x, uint64_t* s_warp, uint64_t& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint64_t inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint64_t y = __shfl_up_sync(kFull, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_warp[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    uint64_t w = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0;
    uint64_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint64_t y = __shfl_up_sync(kFull, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < (int)(blockDim.x >> 5)) s_warp[lane] = wi - w;
    if (lane == 31) s_warp[32] = wi;
  }
  __syncthreads();
  total = s_warp[32];
  uint64_t r = inc - x + s_warp[wid];
  __syncthreads();
  return r;
}

// n_dev != nullptr: the item count is min(n, *n_dev), known only on the device
__device__ __forceinline__ uint64_t eff_n(uint64_t n, const uint32_t* n_dev) {
  return n_dev ? umin64(n, *n_dev) : n;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(const uint64_t* __restrict__ in, uint64_t n,
                                                              uint64_t* __restrict__ bsum,
                                                              const uint32_t* __restrict__ n_dev) {
  pdl_entry();
  __shared__ uint64_t s_warp[33];
  n = eff_n(n, n_dev);
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
  if (base >= n && base > 0) return;
  uint64_t acc = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    uint64_t i = base + (uint64_t)j * kScanThreads + threadIdx.x;
    if (i < n) acc += in[i];
  }
  uint64_t total;
  block_exclusive_scan(acc, s_warp, total);
  if (threadIdx.x == 0) bsum[blockIdx.x] = total;
}

// single block: exclusive scan of bsum[0..nb) in place; bsum[nb] = out[n] = total
__global__ void __launch_bounds__(1024) k_scan_top(uint64_t* __restrict__ bsum, uint64_t n,
                                                   uint64_t* __restrict__ out, const uint32_t* __restrict__ n_dev) {
  pdl_entry();
  __shared__ uint64_t s_warp[33];
  n = eff_n(n, n_dev);
  const uint64_t nb = (n + kScanTile - 1) / kScanTile;
  uint64_t carry = 0;
  for (uint64_t base = 0; base < nb; base += blockDim.x) {
    uint64_t i = base + threadIdx.x;
    uint64_t x = i < nb ? bsum[i] : 0;
    uint64_t total;
    uint64_t ex = block_exclusive_scan(x, s_warp, total);
    if (i < nb) bsum[i] = carry + ex;
    carry += total;
  }
  if (threadIdx.x == 0) {
    bsum[nb] = carry;
    out[n] = carry;
  }
}

__global__ void __launch_bounds__(kScanThreads) k_scan_down(const uint64_t* __restrict__ in, uint64_t n,
                                                            const uint64_t* __restrict__ bsum,
                                                            uint64_t* __restrict__ out,
                                                            const uint32_t* __restrict__ n_dev) {
  pdl_entry();
  __shared__ uint64_t s_items[kScanTile];
  __shared__ uint64_t s_warp[33];
  n = eff_n(n, n_dev);
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
  if (base >= n) return;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    uint64_t i = base + (uint64_t)j * kScanThreads + threadIdx.x;
    s_items[j * kScanThreads + threadIdx.x] = i < n ? in[i] : 0;
  }
  __syncthreads();
  uint64_t loc[kScanItems];
  uint64_t acc = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    loc[j] = acc;
    acc += s_items[threadIdx.x * kScanItems + j];
  }
  uint64_t total;
  uint64_t ex = block_exclusive_scan(acc, s_warp, total) + bsum[blockIdx.x];
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) s_items[threadIdx.x * kScanItems + j] = ex + loc[j];
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    uint64_t i = base + (uint64_t)j * kScanThreads + threadIdx.x;
    if (i < n) out[i] = s_items[j * kScanThreads + threadIdx.x];
  }
}

// T: the chunk map's granularity (weight units); Trule >= T: descriptors of
// at most Trule weight are never split (owned by the group their weight
// interval starts in), heavier ones always go through the split path
constexpr uint64_t kSmallT = 128 * 1024;
struct ChunkGeom {
  uint64_t total, T, nchunks, Trule;
};

__device__ __forceinline__ ChunkGeom chunk_geom(const uint64_t* P, uint64_t n, uint64_t t_min,
                                                uint64_t max_chunks) {
  ChunkGeom g;
  g.total = P[n];
  uint64_t T = (g.total + max_chunks - 1) / max_chunks;
  g.T = umax64(T, t_min);
  g.nchunks = (g.total + g.T - 1) / g.T;
  g.Trule = umax64(g.T, kSmallT);
  return g;
}

// chunk_first[c] = the item whose weight interval [P[d], P[d+1]) contains c*T
__global__ void __launch_bounds__(kThreads) k_plan(const uint64_t* __restrict__ P, uint64_t n, uint64_t t_min,
                                                   uint64_t max_chunks, uint32_t* __restrict__ chunk_first,
                                                   const uint32_t* __restrict__ n_dev) {
  pdl_entry();
  n = eff_n(n, n_dev);
  const ChunkGeom g = chunk_geom(P, n, t_min, max_chunks);
  for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < g.nchunks;
       c += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t target = c * g.T;
    uint64_t lo = 0, hi = n;   // P[lo] <= target < P[hi]
    while (hi - lo > 1) {
      uint64_t mid = (lo + hi) >> 1;
      if (__ldg(P + mid) <= target) lo = mid; else hi = mid;
    }
    chunk_first[c] = (uint32_t)lo;
  }
}

// a1-a3 + a2 in one cooperative launch: the prep (k_check_prep), then the
// exclusive prefix sum of the weights and the chunk map with grid barriers
// between the phases (k_scan_reduce / _top / _down, k_plan): one launch and
// four barriers instead of five launches.
__global__ void __launch_bounds__(kThreads, CG_FRONT_MINB) k_front(const cg_copy_desc* __restrict__ descs, uint64_t n, Table t,
                                                    cg_verdict* __restrict__ out, uint64_t* __restrict__ weight,
                                                    ScanMeta* __restrict__ meta, uint64_t* __restrict__ dvoff,
                                                    ShadowView sv, uint32_t* __restrict__ counter,
                                                    uint32_t* __restrict__ defer, uint64_t* P,
                                                    uint64_t* __restrict__ bsum, uint64_t t_min, uint64_t max_chunks,
                                                    uint32_t* __restrict__ chunk_first, uint32_t err_mask, int fuse,
                                                    uint32_t* __restrict__ late) {
  pdl_entry();
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  extern __shared__ uint64_t s_split[];
  __shared__ uint64_t s_warp[33];
  prep_body(descs, n, t, out, weight, meta, dvoff, sv, counter, defer, s_split, err_mask, fuse, late);
  grid.sync();

  // block b owns items [b*per, (b+1)*per)
  const uint64_t per = (n + gridDim.x - 1) / gridDim.x;
  const uint64_t lo = umin64(n, (uint64_t)blockIdx.x * per), hi = umin64(n, lo + per);
  {
    uint64_t acc = 0;
    for (uint64_t k = lo + threadIdx.x; k < hi; k += blockDim.x) acc += __ldcg(weight + k);
    uint64_t total;
    block_exclusive_scan(acc, s_warp, total);
    if (threadIdx.x == 0) bsum[blockIdx.x] = total;
  }
  grid.sync();
  if (blockIdx.x == 0) {
    uint64_t carry = 0;
    for (uint64_t b0 = 0; b0 < gridDim.x; b0 += blockDim.x) {
      const uint64_t b = b0 + threadIdx.x;
      const uint64_t x = b < gridDim.x ? __ldcg(bsum + b) : 0;
      uint64_t total;
      const uint64_t ex = block_exclusive_scan(x, s_warp, total);
      if (b < gridDim.x) bsum[b] = carry + ex;
      carry += total;
    }
    if (threadIdx.x == 0) P[n] = carry;
  }
  grid.sync();
  {
    uint64_t carry = __ldcg(bsum + blockIdx.x);
    for (uint64_t k0 = lo; k0 < hi; k0 += blockDim.x) {
      const uint64_t k = k0 + threadIdx.x;
      const uint64_t x = k < hi ? __ldcg(weight + k) : 0;
      uint64_t total;
      const uint64_t ex = block_exclusive_scan(x, s_warp, total);
      if (k < hi) P[k] = carry + ex;
      carry += total;
    }
  }
  grid.sync();
  const ChunkGeom g = chunk_geom(P, n, t_min, max_chunks);
  for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < g.nchunks;
       c += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t target = c * g.T;
    uint64_t a = 0, b = n;   // P[a] <= target < P[b]
    while (b - a > 1) {
      const uint64_t mid = (a + b) >> 1;
      if (__ldcg(P + mid) <= target) a = mid; else b = mid;
    }
    chunk_first[c] = (uint32_t)a;
  }
}

// Tile generator.  All bookkeeping is lane-parallel:
//  * descriptor window: lane i owns descriptor wbase+i and, whenever the window
//    or the group changes, computes its piece (its share of the group's weight
//    interval) -- for contiguous host ranges directly as a shard byte range
//    plus the analytic first out-of-window offset -- and finalises pieces
//    without shard bytes itself (DtoD, invalid or empty host sides, ranges
//    outside the shard);
//  * segment window: lane j owns one contiguous shard range (a contiguous
//    piece, or one row of a 2D piece, R-11) and its number of block-aligned
//    tiles; a warp prefix sum numbers all tiles of the window, and every tile
//    is issued by the lane that owns it (tile parameters never leave that
//    lane's registers).
// The warp-uniform part is a cursor over tile numbers plus a small phase
// machine (group -> window -> contiguous pieces -> 2D pieces row by row).
constexpr uint32_t kPieceIn = 1, kPieceWhole = 2, kPieceHtod = 4, kPiece2D = 8, kPieceEmpty = 16;
constexpr uint32_t kSegEndLast = 1u << 8;   // the segment's last tile ends its piece
constexpr int kPhaseGroup = 0, kPhaseContig = 1, kPhase2D = 2, kPhaseWindow = 3;
constexpr uint32_t kSubNone = 0, kSubHead = 1, kSubBody = 2, kSubTail = 3;

__device__ __forceinline__ uint32_t warp_excl_scan(uint32_t x, uint32_t& total) {
  const int lane = threadIdx.x & 31;
  uint32_t inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, inc, o);
    if (lane >= o) inc += y;
  }
  total = __shfl_sync(kFull, inc, 31);
  return inc - x;
}

struct TileGen {
  // inputs
  const ScanMeta* meta;
  const uint64_t* P;
  const uint32_t* chunk_first;
  uint32_t* counter;
  cg_verdict* out;
  uint32_t err_mask;
  uint64_t n, T, nchunks, total, Trule;
  uint32_t nwarps;      // warps of the grid (group grab size policy)
  uint64_t wb, we, sb, se;
  bool fuse;            // check + apply in one pass (cg_check_apply)
  bool two_bit;         // NEXT-4 2-bit states: 16 KiB host bytes per tile for both kinds
  bool sparse;          // NEXT-4 two-level sparse map (2-bit states behind a chunk directory)
  // group
  uint64_t w0, w1;
  uint32_t g_pending;   // lane 0: first chunk of the next group
  uint32_t k_pending;   // lane 0: its chunk count
  int phase;
  // descriptor window (lane i <-> wbase + i)
  uint64_t wbase;
  uint64_t m_x0, m_pitch, m_W, m_info, m_ps, m_pe;
  uint32_t p_fl;
  uint64_t p_lo, p_hi, p_qs, p_qe, p_ob, p_fu;
  uint32_t twod;        // remaining 2D pieces of the window (lane mask)
  // segment window (lane j)
  uint64_t s_q0, s_q1, s_ob, s_pfu;
  uint32_t s_d, s_fl, s_k, s_excl;
  uint32_t K, t;
  // current 2D piece
  bool in2d;
  uint64_t x0, pitch, W, lo2, hi2, r2, fu2;
  uint32_t d2, fl2;
  // packed rows of a 2D DtoH piece: sub-phase (kSubNone: rows one by one;
  // kSubHead -> kSubBody -> kSubTail: the partial first row, the whole rows
  // [r2, pk_end) several per tile, the partial last row) and the piece's end
  uint32_t sub;
  uint64_t pk_end, t_hi;

  __device__ __forceinline__ void load_window(uint64_t base) {
    const int lane = threadIdx.x & 31;
    wbase = base;
    const uint64_t i = base + lane;
    if (i < n) {
      const ScanMeta m = meta[i];
      m_x0 = m.hstart;
      m_pitch = m.hpitch;
      m_W = m.W;
      m_info = m.info;
      m_ps = P[i];
      m_pe = P[i + 1];
    } else {
      m_info = 0;
      m_ps = m_pe = ~0ull;
    }
    // the next window is usually needed next: bring its records into L2 now
    // (no registers held), so that load does not stall the ring's owner warp
    if (i + 32 < n) {
      asm volatile("prefetch.global.L2 [%0];" ::"l"(meta + i + 32));
      if ((lane & 3) == 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(P + i + 32));
    }
  }

  __device__ __forceinline__ void compute_pieces() {
    const int lane = threadIdx.x & 31;
    p_fl = 0;
    // a descriptor of at most one group's weight is never split: it belongs
    // to the group its weight interval starts in
    const bool small = m_pe - m_ps <= Trule;
    const bool deferred = (m_info >> kInfoDefer) & 1u;   // the deferred pass checks it (k_check_scan's tail)
    if (!deferred && (small ? (m_ps >= w0 && m_ps < w1) : (m_ps < w1 && m_pe > w0))) {
      const uint64_t nbytes = m_info & kInfoBytes;
      const uint32_t kind = (uint32_t)(m_info >> kInfoKind) & 3u;
      const bool host = (m_info >> kInfoHost) & 1u, contig = (m_info >> kInfoContig) & 1u;
      const bool htod = kind == CG_HTOD;
      uint32_t f = kPieceIn | (htod ? kPieceHtod : 0u);
      if (small) f |= kPieceWhole;
      uint64_t a = small ? 0 : umax64(w0, m_ps) - m_ps, b = small ? m_pe - m_ps : umin64(w1, m_pe) - m_ps;
      a = a > kItemCost ? a - kItemCost : 0;
      b = b > kItemCost ? b - kItemCost : 0;
      uint64_t lo = a, hi = b;
      if (two_bit) {
        lo = a << 2;
        hi = umin64(b << 2, nbytes);
      } else if (!htod) {
        lo = a << 3;
        hi = umin64(b << 3, nbytes);
      }
      // a whole piece carries the side's analytic first offset outside the
      // window (R-15; the prep stored it as the initial first_unaddr); split
      // pieces min into that initial value
      p_fu = kNone;
      if (small && ((m_info >> kInfoPfu) & 1u)) p_fu = out[wbase + lane].first_unaddr;
      if (!host || lo >= hi) {
        f |= kPieceEmpty;
      } else {
        // [lo, hi) counts scanned bytes from the side's first shard byte (R-10 clip)
        const uint64_t ob = clip_base(m_x0, m_W, m_pitch, contig, sb);
        lo += ob;
        hi += ob;
      }
      if (f & kPieceEmpty) {
      } else if (!contig) {
        f |= kPiece2D;
        p_lo = lo;
        p_hi = hi;
      } else {
        const uint64_t x = m_x0 + lo, len = hi - lo;
        const uint64_t y0 = umax64(x, sb), y1 = umin64(x + len, se);
        if (y0 < y1) {
          p_qs = y0 - sb;
          p_qe = y1 - sb;
          p_ob = lo - x + sb;   // logical offset of shard byte q is p_ob + q (mod 2^64)
        } else {
          f |= kPieceEmpty;
        }
      }
      p_fl = f;
      if (f & kPieceEmpty) {
        cg_verdict* v = out + (wbase + lane);
        if ((f & kPieceWhole) && ((m_info >> kInfoRaw) & 1u)) {
          v->first_unaddr = p_fu;   // raw partial (straddler): finalised after the merge
        } else if (f & kPieceWhole) {
          uint32_t flags = (uint32_t)((m_info >> kInfoFlags) & 0x3FFu), status;
          finalize_fields(flags, status, p_fu, 0, err_mask);
          v->first_unaddr = p_fu;
          v->flags = flags;
          v->status = status;
        }
      }
    }
    const uint32_t live2d = __ballot_sync(kFull, (p_fl & (kPiece2D | kPieceEmpty)) == kPiece2D);
    twod = live2d;
    // the contiguous pieces form the first segment window
    const bool live = (p_fl & (kPieceIn | kPiece2D | kPieceEmpty)) == kPieceIn;
    set_segment(live, p_qs, p_qe, p_ob, p_fu, (uint32_t)(wbase + lane),
                (p_fl & kPieceHtod ? kTileHtod : 0u) | (p_fl & kPieceWhole ? kTileWhole : 0u) | kSegEndLast |
                    (((m_info >> kInfoRaw) & 1u) ? kTileRaw : 0u) | (((m_info >> kInfoAfter) & 1u) ? kTileAfter : 0u) |
                    (((m_info >> kInfoLast) & 1u) ? kTileLast : 0u) |
                    ((uint32_t)((m_info >> kInfoFlags) & 0x3FFu) << 16));
    phase = kPhaseContig;
  }

  __device__ __forceinline__ void set_segment(bool live, uint64_t q0, uint64_t q1, uint64_t ob, uint64_t pfu,
                                              uint32_t d, uint32_t fl) {
    s_q0 = q0;
    s_q1 = q1;
    s_ob = ob;
    s_pfu = pfu;
    s_d = d;
    s_fl = fl;
    uint32_t k = 0;
    if (live) {
      const uint64_t sh = two_bit ? k2bitShift : (fl & kTileHtod) ? kHtodShift : kDtohShift;   // log2 of the tile block
      k = (uint32_t)(((q1 - 1) >> sh) - (q0 >> sh) + 1);
    }
    s_k = k;
    s_excl = warp_excl_scan(k, K);
    t = 0;
  }

  __device__ __forceinline__ bool next_group() {
    const int lane = threadIdx.x & 31;
    const uint32_t g = __shfl_sync(kFull, g_pending, 0);
    const uint32_t k = __shfl_sync(kFull, k_pending, 0);
    if (g >= nchunks) return false;
    if (lane == 0) {   // kGrab chunks at a time while plenty are left, single chunks for the tail
      k_pending = (uint64_t)g + 16ull * kGrab * nwarps < nchunks ? kGrab : 1u;
      g_pending = atomicAdd(counter, k_pending);
    }
    w0 = (uint64_t)g * T;
    w1 = umin64((uint64_t)(g + k) * T, total);
    const uint64_t d = chunk_first[g];
    if (d < wbase || d >= wbase + 32) load_window(d);
    compute_pieces();
    return true;
  }

  // rows [r2, r2 + 32) of the current 2D piece as a segment window (the
  // piece lies in the shard clip, so every row segment is shard bytes)
  __device__ __forceinline__ void row_window() {
    const int lane = threadIdx.x & 31;
    const uint64_t r = r2 + lane;
    const uint64_t rs = r * W;                       // logical offset of the row start
    bool live = false;
    uint64_t q0 = 0, q1 = 0, ob = 0;
    if (rs < hi2) {
      const uint64_t L0 = umax64(lo2, rs), L1 = umin64(hi2, rs + W);
      const uint64_t x = x0 + r * pitch + (L0 - rs), len = L1 - L0;
      const uint64_t y0 = umax64(x, sb), y1 = umin64(x + len, se);
      if (y0 < y1) {
        live = true;
        q0 = y0 - sb;
        q1 = y1 - sb;
        ob = L0 - x + sb;
      }
    }
    set_segment(live, q0, q1, ob, kNone, d2, fl2 & kTileHtod);
    r2 += 32;
  }

  // Packed DtoH rows: a 2D DtoH piece's whole rows are staged several per tile
  // (row j of the tile at byte j * pk_rs of the slot: its A bytes from the
  // 16-byte boundary below it), instead of one tile per row segment, which
  // made narrow-row copies (C4) issue-bound.  Only for pieces whose rows lie
  // inside the stored shard, in the bytes format.  Row r starts at shard byte
  // q_r = x0 + r pitch - sb, and the logical offset of its shard byte q is
  // r W + q - q_r = ob_r + q, so ob_{r+j} = ob_r + j (W - pitch) (mod 2^64).
  __device__ __forceinline__ static uint32_t packed_rs(uint64_t W) {   // A bytes of a row at any 128-byte phase, at most
    return (uint32_t)(16 * ((W + 127) / 128 + 1));
  }

  __device__ __forceinline__ void enter_2d() {
    sub = kSubNone;
    if (two_bit || (fl2 & kTileHtod) || W == 0 || W > 16 * (kTileV + kTileA)) return;
    if (2 * packed_rs(W) > kTileV + kTileA) return;
    const uint64_t rA = (lo2 + W - 1) / W, rB = hi2 / W;   // whole rows [rA, rB)
    if (rB <= rA) return;
    const uint64_t a = x0 + rA * pitch, b = x0 + (rB - 1) * pitch + W;
    if (a < sb || b > se) return;
    pk_end = rB;
    t_hi = hi2;
    hi2 = umin64(hi2, rA * W);   // the head: [lo2, rA W)
    sub = kSubHead;
  }

  // one tile of whole rows [r2, r2 + k): every lane stages its row's A bytes
  __device__ __forceinline__ void packed_tile(WarpRing& ring, int s, const ShadowView& sv, uint64_t policy) {
    const int lane = threadIdx.x & 31;
    const uint32_t rs = packed_rs(W);
    const uint32_t k = (uint32_t)umin64(umin64(32, (kTileV + kTileA) / rs), pk_end - r2);
    const uint64_t q_first = x0 + r2 * pitch - sb;
    uint32_t len = 0;
    uint64_t qa = 0;
    if ((uint32_t)lane < k) {
      const uint64_t q = q_first + (uint64_t)lane * pitch;
      qa = q & ~127ull;
      len = (uint32_t)((((q + W + 127) & ~127ull) - qa) >> 3);
    }
    uint32_t total = len;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(kFull, total, o);
    if (lane == 0) {
      TileInfo ti;
      ti.ob = r2 * W - q_first;   // ob of row r2
      ti.pend_fu = kNone;
      ti.d = d2;
      ti.flags = kTileData | kTilePacked | (fl2 & ~(kSegEndLast | kTileWhole));
      ti.q0 = (uint32_t)W;
      ti.q1 = k | (rs << 16);
      ti.qs = q_first;
      ti.qe = pitch;
      ring.info[s] = ti;
      mbar_arrive_tx(&ring.bar[s], total);
    }
    __syncwarp();
    if (len) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      bulk_g2s(ring.data[s] + lane * rs, sv.A + qa / 8, len, &ring.bar[s], policy);
    }
    r2 += k;
  }

  // issues the next tile into ring slot s; false when the warp has no more work
  __device__ __forceinline__ bool next(WarpRing& ring, int s, const ShadowView& sv, uint64_t policy) {
    const int lane = threadIdx.x & 31;
    while (t >= K) {
      if (phase == kPhaseGroup) {
        if (!next_group()) return false;
      } else if (phase == kPhaseContig || phase == kPhase2D) {
        phase = kPhase2D;
        if (in2d) {
          if (r2 * W < hi2) {
            row_window();
          } else if (sub == kSubHead) {   // head rows done: the whole rows, packed
            sub = kSubBody;
            r2 = (lo2 + W - 1) / W;
          } else if (sub == kSubBody) {
            if (r2 < pk_end) {
              packed_tile(ring, s, sv, policy);
              return true;
            }
            sub = kSubTail;   // then the partial last row, one by one
            lo2 = pk_end * W;
            hi2 = t_hi;
            r2 = pk_end;
          } else {   // all rows done: a data-less END tile carrying the analytic offset
            in2d = false;
            if (lane == 0) {
              TileInfo ti;
              ti.ob = 0;
              ti.pend_fu = fu2;
              ti.d = d2;
              ti.flags = kTileEnd | (fl2 & ~kSegEndLast);
              ti.q0 = ti.q1 = 0;
              ring.info[s] = ti;
              mbar_arrive(&ring.bar[s]);
            }
            return true;
          }
        } else if (twod) {
          const int src = __ffs(twod) - 1;
          twod &= twod - 1;
          x0 = __shfl_sync(kFull, m_x0, src);
          pitch = __shfl_sync(kFull, m_pitch, src);
          W = __shfl_sync(kFull, m_W, src);
          lo2 = __shfl_sync(kFull, p_lo, src);
          hi2 = __shfl_sync(kFull, p_hi, src);
          const uint32_t pf = __shfl_sync(kFull, p_fl, src);
          const uint64_t info = __shfl_sync(kFull, m_info, src);
          d2 = (uint32_t)(wbase + src);
          fl2 = (pf & kPieceHtod ? kTileHtod : 0u) | (pf & kPieceWhole ? kTileWhole : 0u) |
                (((info >> kInfoRaw) & 1u) ? kTileRaw : 0u) | (((info >> kInfoLast) & 1u) ? kTileLast : 0u) |
                ((uint32_t)((info >> kInfoFlags) & 0x3FFu) << 16);
          fu2 = __shfl_sync(kFull, p_fu, src);
          enter_2d();
          r2 = lo2 / W;
          in2d = true;
        } else {
          phase = kPhaseWindow;
        }
      } else {   // kPhaseWindow: the group may continue past this window
        const bool more = __shfl_sync(kFull, m_ps, 31) < w1 && wbase + 32 < n;
        if (more) {
          load_window(wbase + 32);
          compute_pieces();
        } else {
          phase = kPhaseGroup;
        }
      }
    }
    // tile t belongs to the last lane whose tiles start at or before t
    const uint32_t own = __ballot_sync(kFull, s_k != 0 && s_excl <= t);
    const int owner = 31 - __clz(own);
    if (lane == owner) {
      const uint32_t j = t - s_excl;
      const bool htod = s_fl & kTileHtod;
      const uint32_t bsh = two_bit ? k2bitShift : htod ? kHtodShift : kDtohShift;   // log2 of the tile block
      const uint64_t base = (s_q0 >> bsh) << bsh;
      const uint64_t tq0 = j ? base + ((uint64_t)j << bsh) : s_q0;
      const uint64_t tq1 = umin64(s_q1, base + ((uint64_t)(j + 1) << bsh));
      const uint64_t qa = tq0 & (two_bit ? ~63ull : ~127ull);
      TileInfo ti;
      ti.ob = s_ob + qa;
      ti.pend_fu = s_pfu;
      ti.d = s_d;
      uint32_t f = kTileData | (s_fl & ~(kSegEndLast | kTileWhole));
      if (j + 1 == s_k && (s_fl & kSegEndLast)) {
        f |= kTileEnd | (s_fl & kTileWhole);
        if (fuse && !htod && !(s_fl & (kTileRaw | kTileAfter))) {   // a contiguous DtoH piece: the consumer may apply it
          f |= kTileFuse;
          ti.qs = s_q0;
          ti.qe = s_q1;
        }
      }
      ti.flags = f;
      ti.q0 = (uint32_t)(tq0 - qa);
      ti.q1 = (uint32_t)(tq1 - qa);
      ring.info[s] = ti;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (two_bit) {   // host bytes [qa, qa + span) <-> 16-byte aligned state bytes [qa/4, (qa + span)/4)
        const uint32_t span = (ti.q1 + 63u) & ~63u;
        const uint8_t* base = sv.V;
        if (sparse) {   // a tile never leaves its 16 KiB block, so never its chunk
          const uint64_t c = qa >> kChunkShift;
          base = chunk_base(sv, c, sparse_secondary(sv, c));
        }
        mbar_arrive_tx(&ring.bar[s], span / 4);
        bulk_g2s(ring.data[s], base + qa / 4, span / 4, &ring.bar[s], policy);
        ++t;
        return true;
      }
      const uint32_t span = (ti.q1 + 127u) & ~127u;   // staged host bytes (multiple of 128)
      if (f & kTileHtod) {
        mbar_arrive_tx(&ring.bar[s], span + span / 8);
        bulk_g2s(ring.data[s], sv.V + qa, span, &ring.bar[s], policy);
        bulk_g2s(ring.data[s] + kTileV, sv.A + qa / 8, span / 8, &ring.bar[s], policy);
      } else {
        mbar_arrive_tx(&ring.bar[s], span / 8);
        bulk_g2s(ring.data[s], sv.A + qa / 8, span / 8, &ring.bar[s], policy);
      }
    }
    ++t;
    return true;
  }
};

// ---------------------------------------------------------------------------
// The deferred pass (R-10, R-12): host sides the tile generator does not take
// -- BAD_PITCH rows that overlap (pitch < W: a physical byte lies in several
// rows and counts once per row) and, in the sparse map, sides longer than
// kDeferBytes (walked over the chunks that have a secondary; the bytes between
// them are NOACCESS).  One warp per descriptor, taken from a list by warps
// whose ring has drained, in physical address order with plain 16-byte loads.
// Along a side the logical offset grows with the address (rows move up by
// pitch >= 0), so each lane's first bad / undefined byte gives its minimum.
// Physical byte u = x - x0 of overlapping rows lies in rows r_lo..r_hi,
// r_lo = u < W ? 0 : (u - W) / pitch + 1, r_hi = min(H - 1, u / pitch), with
// first logical offset u + r_lo (W - pitch) (pitch 0: rows 0..H-1, offset u).
// Pathological inputs only: not tuned.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t even_bits(uint32_t x) {   // bit 2j -> bit j
  x &= 0x55555555u;
  x = (x | (x >> 1)) & 0x33333333u;
  x = (x | (x >> 2)) & 0x0F0F0F0Fu;
  x = (x | (x >> 4)) & 0x00FF00FFu;
  return (x | (x >> 8)) & 0x0000FFFFu;
}

// addressable / undefined masks of the 16 host bytes at shard byte q (q % 16 == 0)
__device__ __forceinline__ void host16(const ShadowView& sv, uint64_t q, uint32_t& addr, uint32_t& und) {
  if (!sv.two_bit) {
    const uint4 v = __ldcg(reinterpret_cast<const uint4*>(sv.V + q));
    addr = __ldcg(reinterpret_cast<const unsigned short*>(sv.A + (q >> 3)));
    und = nz16(v) & addr;
    return;
  }
  uint32_t w;
  if (sv.sparse) {
    const uint64_t c = q >> kChunkShift;
    w = __ldcg(reinterpret_cast<const unsigned int*>(chunk_base(sv, c, sparse_secondary(sv, c)) + (q >> 2)));
  } else {
    w = __ldcg(reinterpret_cast<const unsigned int*>(sv.V) + (q >> 4));
  }
  addr = even_bits(w | (w >> 1));   // state != 00
  und = even_bits(w);               // PARTIAL / UNDEFINED (always addressable)
}

struct DeferSide {
  uint64_t x0, W, pitch, H;   // rows; a contiguous side is one row of N bytes
  bool overlap, htod;
};

__device__ __forceinline__ uint64_t ov_rlo(const DeferSide& s, uint64_t u) {
  return (s.pitch == 0 || u < s.W) ? 0 : (u - s.W) / s.pitch + 1;
}

// physical host bytes [a, b) of the side, inside the stored shard; rowbase =
// the logical offset of a when the segment lies in one row (non-overlapping rows)
__device__ __noinline__ void defer_segment(const ShadowView& sv, const DeferSide& s, uint64_t a, uint64_t b,
                                           uint64_t rowbase, Partial& p) {
  const int lane = threadIdx.x & 31;
  const uint64_t g1 = b - sv.sb;
  constexpr int kDeep = 4;   // 16-byte groups in flight per lane (a side's loads are independent)
  for (uint64_t g0 = ((a - sv.sb) & ~15ull) + 16ull * lane; g0 < g1; g0 += 512 * kDeep) {
    uint32_t ad[kDeep], un[kDeep];
#pragma unroll
    for (int k = 0; k < kDeep; ++k) {
      ad[k] = 0xFFFFu;
      un[k] = 0;
      if (g0 + 512ull * k < g1) host16(sv, g0 + 512ull * k, ad[k], un[k]);
    }
#pragma unroll
    for (int k = 0; k < kDeep; ++k) {
      const uint64_t g = g0 + 512ull * k;
      if (g >= g1) break;
      const uint64_t xa = sv.sb + g;   // address of the group's byte 0
      uint32_t m = 0xFFFFu;
      if (xa < a) m &= 0xFFFFu << (uint32_t)(a - xa);
      if (xa + 16 > b) m &= 0xFFFFu >> (uint32_t)(xa + 16 - b);
      const uint32_t bad = ~ad[k] & m;
      uint32_t u = s.htod ? un[k] & m : 0u;
      if (!(bad | u)) continue;
      if (bad) {
        const uint64_t x = xa + (__ffs(bad) - 1);
        p.fu = umin64(p.fu, s.overlap ? (x - s.x0) + ov_rlo(s, x - s.x0) * (s.W - s.pitch) : rowbase + (x - a));
      }
      if (u) {
        const uint64_t x = xa + (__ffs(u) - 1);
        p.fd = umin64(p.fd, s.overlap ? (x - s.x0) + ov_rlo(s, x - s.x0) * (s.W - s.pitch) : rowbase + (x - a));
        if (!s.overlap) {
          p.cnt += __popc(u);
        } else {
          while (u) {   // each undefined byte counts once per row it lies in
            const uint64_t uu = xa + (__ffs(u) - 1) - s.x0;
            u &= u - 1;
            p.cnt += s.pitch == 0 ? s.H : umin64(s.H - 1, uu / s.pitch) - ov_rlo(s, uu) + 1;
          }
        }
      }
    }
  }
}

// the side's bytes in the physical range [a, e) (inside the stored shard)
__device__ __forceinline__ void defer_range(const ShadowView& sv, const DeferSide& s, uint64_t a, uint64_t e,
                                            Partial& p) {
  if (s.overlap) {
    defer_segment(sv, s, a, e, 0, p);
    return;
  }
  for (uint64_t r = first_row_past(s.x0, s.W, s.pitch, s.H, a); r < s.H; ++r) {
    const uint64_t xr = s.x0 + r * s.pitch;
    if (xr >= e) break;
    const uint64_t sa = umax64(xr, a), sb = umin64(xr + s.W, e);
    if (sa < sb) defer_segment(sv, s, sa, sb, r * s.W + (sa - xr), p);
    if (s.pitch == 0) break;
  }
}

// lowest logical offset of a side byte in the NOACCESS gap [y, a) (kNone if none)
__device__ __forceinline__ uint64_t gap_offset(const DeferSide& s, uint64_t y, uint64_t a) {
  if (y >= a) return kNone;
  if (s.overlap || s.pitch == 0) {   // the side's bytes are the contiguous [x0, x0 + span)
    const uint64_t b = umax64(y, s.x0);
    if (b >= a) return kNone;
    return s.overlap ? (b - s.x0) + ov_rlo(s, b - s.x0) * (s.W - s.pitch) : b - s.x0;
  }
  const uint64_t r = first_row_past(s.x0, s.W, s.pitch, s.H, y);
  if (r >= s.H) return kNone;
  const uint64_t xr = s.x0 + r * s.pitch, b = umax64(xr, y);
  return b < a ? r * s.W + (b - xr) : kNone;
}

__device__ __noinline__ void defer_one(const cg_copy_desc* __restrict__ descs, uint32_t d,
                                       const ScanMeta* __restrict__ meta, const ShadowView& sv,
                                       cg_verdict* __restrict__ out, uint32_t err_mask, int fuse,
                                       uint32_t* __restrict__ resid, uint32_t* __restrict__ resid_n,
                                       uint32_t* __restrict__ last) {
  const int lane = threadIdx.x & 31;
  const cg_copy_desc dd = descs[d];
  const Norm nm = normalize(dd);
  const HostClip hc = host_clip(nm, dd.height, sv);
  const bool contig = dd.height == 1 || dd.width == nm.hpitch;
  DeferSide s;
  s.x0 = nm.hstart;
  s.W = contig ? nm.nbytes : nm.W;
  s.pitch = contig ? 0 : nm.hpitch;
  s.H = contig ? 1 : dd.height;
  s.overlap = hc.overlap;
  s.htod = nm.skind == CG_HTOD;
  const uint64_t hi = s.x0 + ((s.H - 1) * s.pitch + s.W);   // end of the physical span (fits: R-10)
  Partial p{lane == 0 ? hc.pfu : kNone, kNone, 0};
  if (!sv.sparse) {   // dense: overlapping rows only; the shard part of the span
    const uint64_t a = umax64(s.x0, sv.sb), b = umin64(hi, sv.se);
    if (a < b) defer_range(sv, s, a, b, p);
  } else {            // sparse: the chunks with a secondary, ascending
    uint64_t k0 = 0, k1 = sv.n_chunks;
    while (k0 < k1) {
      const uint64_t mid = (k0 + k1) >> 1;
      if (sv.chunk_list[mid] < (s.x0 >> kChunkShift)) k0 = mid + 1; else k1 = mid;
    }
    uint64_t y = s.x0;   // side bytes below y are done
    for (uint64_t k = k0; k < sv.n_chunks; ++k) {
      const uint64_t ca = sv.chunk_list[k] << kChunkShift, clast = ca + ((1ull << kChunkShift) - 1);
      if (ca >= hi) break;
      const uint64_t a = umax64(ca, s.x0), e = umin64(clast, hi - 1) + 1;
      if (lane == 0) p.fu = umin64(p.fu, gap_offset(s, y, a));
      defer_range(sv, s, a, e, p);
      y = e;
    }
    if (lane == 0) p.fu = umin64(p.fu, gap_offset(s, y, hi));
  }
  p.fu = warp_min(p.fu);
  p.fd = warp_min(p.fd);
  p.cnt = warp_sum(p.cnt);
  if (lane == 0) {
    // the prep's device / validation flags: from the scan record, or (meta ==
    // nullptr, the late pass) from the verdict the prep wrote
    cg_verdict* v = out + d;
    const bool raw = meta ? ((meta[d].info >> kInfoRaw) & 1u) : (dd.reserved & CG_SHARD_RAW) != 0;
    const uint32_t flags0 = meta ? (uint32_t)((meta[d].info >> kInfoFlags) & 0x3FFu) : v->flags;
    v->first_unaddr = p.fu;
    v->first_undef = p.fd;
    v->undef_count = p.cnt;
    if (!raw) {   // a raw straddler partial is finalised after the merge
      uint32_t flags = flags0, status;
      finalize_fields(flags, status, p.fu, p.cnt, err_mask);
      v->flags = flags;
      v->status = status;
      if (fuse && status == CG_OK && !s.htod)   // the residual (or, CG_APPLY_LAST, the last) pass applies it
        push_apply(meta && ((meta[d].info >> kInfoLast) & 1u), d, resid, resid_n, last);
    }
  }
  __syncwarp();
}

// the late pass (CG_CHECK_AFTER, dense formats), spread over the grid: part
// `part` of `nparts` of late descriptor d's physical span (16-byte aligned
// pieces), combined into the verdict the prep wrote (first_unaddr = the
// analytic offset outside the window, first_undef none, count 0) by atomics;
// late_finalize then sets flags and status.  One warp per side took ~1 us per
// 512 bytes of it.
__device__ __noinline__ void late_part(const cg_copy_desc* __restrict__ descs, uint32_t d, uint32_t part,
                                       uint32_t nparts, const ShadowView& sv, cg_verdict* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const cg_copy_desc dd = descs[d];
  const Norm nm = normalize(dd);
  const HostClip hc = host_clip(nm, dd.height, sv);
  const bool contig = dd.height == 1 || dd.width == nm.hpitch;
  DeferSide s;
  s.x0 = nm.hstart;
  s.W = contig ? nm.nbytes : nm.W;
  s.pitch = contig ? 0 : nm.hpitch;
  s.H = contig ? 1 : dd.height;
  s.overlap = hc.overlap;
  s.htod = true;
  if (!nm.host || s.W == 0) return;
  const uint64_t hi = s.x0 + ((s.H - 1) * s.pitch + s.W);   // end of the physical span (fits: R-10)
  const uint64_t a0 = umax64(s.x0, sv.sb), b0 = umin64(hi, sv.se);
  if (a0 >= b0) return;
  const uint64_t step = (((b0 - a0) + nparts - 1) / nparts + 15) & ~15ull;
  const uint64_t a = a0 + (uint64_t)part * step, b = umin64(a + step, b0);
  if (a >= b) return;
  Partial p{kNone, kNone, 0};
  defer_range(sv, s, a, b, p);
  p.fu = warp_min(p.fu);
  p.fd = warp_min(p.fd);
  p.cnt = warp_sum(p.cnt);
  if (lane == 0) {
    cg_verdict* v = out + d;
    if (p.fu != kNone) atomicMin(reinterpret_cast<unsigned long long*>(&v->first_unaddr), p.fu);
    if (p.fd != kNone) atomicMin(reinterpret_cast<unsigned long long*>(&v->first_undef), p.fd);
    if (p.cnt) atomicAdd(reinterpret_cast<unsigned long long*>(&v->undef_count), p.cnt);
  }
}

__device__ __forceinline__ void late_finalize(cg_verdict* v, uint32_t err_mask) {
  uint32_t flags = v->flags, status;
  finalize_fields(flags, status, v->first_unaddr, v->undef_count, err_mask);
  v->flags = flags;
  v->status = status;
}

// a warp whose ring has drained takes deferred descriptors until the list is done
__device__ __noinline__ void defer_tail(const cg_copy_desc* __restrict__ descs, const uint32_t* __restrict__ defer,
                                        uint32_t* counter, const ScanMeta* __restrict__ meta, const ShadowView& sv,
                                        cg_verdict* __restrict__ out, uint32_t err_mask, int fuse,
                                        uint32_t* __restrict__ resid, uint32_t* __restrict__ resid_n,
                                        uint32_t* __restrict__ last) {
  const int lane = threadIdx.x & 31;
  const uint32_t n = *reinterpret_cast<volatile uint32_t*>(counter + 4);   // final: written by the prep
  while (true) {
    uint32_t k = 0;
    if (lane == 0) k = atomicAdd(counter + 5, 1u);
    k = __shfl_sync(kFull, k, 0);
    if (k >= n) break;
    defer_one(descs, defer[k], meta, sv, out, err_mask, fuse, resid, resid_n, last);
  }
}

// one instantiation per host shadow format (kTwoBit: NEXT-4 2-bit states)
// and apply mode (kFuse: cg_check_apply): the other paths are compiled out of
// each, which relieves instruction-cache stalls
template <bool kTwoBit, bool kFuse, bool kSparse>
__global__ void __launch_bounds__(kRingWarps * 32, 4) k_check_scan(
    const ScanMeta* __restrict__ meta, uint64_t n, const uint64_t* __restrict__ P,
    const uint32_t* __restrict__ chunk_first, uint32_t* counter, uint64_t t_min, uint64_t max_chunks,
    ShadowView sv, cg_verdict* __restrict__ out, uint32_t err_mask, int fuse, uint32_t* __restrict__ resid,
    uint32_t* __restrict__ resid_n, const cg_copy_desc* __restrict__ descs, const uint32_t* __restrict__ defer,
    uint32_t* __restrict__ last) {
  pdl_entry();
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WarpRing& ring = reinterpret_cast<WarpRing*>(smem)[wid];
  const ChunkGeom geo = chunk_geom(P, n, t_min, max_chunks);
  if (lane == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&ring.bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const uint64_t policy = evict_first_policy();

  TileGen gen;
  gen.meta = meta;
  gen.P = P;
  gen.chunk_first = chunk_first;
  gen.counter = counter;
  gen.out = out;
  gen.err_mask = err_mask;
  gen.n = n;
  gen.T = geo.T;
  gen.nchunks = geo.nchunks;
  gen.total = geo.total;
  gen.Trule = geo.Trule;
  gen.nwarps = gridDim.x * kRingWarps;
  gen.wb = sv.wb;
  gen.we = sv.we;
  gen.sb = sv.sb;
  gen.se = sv.se;
  gen.fuse = kFuse;
  (void)fuse;
  gen.two_bit = kTwoBit;
  gen.sparse = kSparse;
  gen.k_pending = kGrab;
  gen.g_pending = lane == 0 ? atomicAdd(counter, kGrab) : 0;
  gen.phase = kPhaseGroup;
  gen.wbase = ~0ull >> 1;   // no window yet
  gen.p_fl = 0;
  gen.twod = 0;
  gen.in2d = false;
  gen.sub = kSubNone;
  gen.K = gen.t = 0;

  int filled = 0;
  while (filled < kStages && gen.next(ring, filled, sv, policy)) ++filled;
  uint32_t phase = 0;   // bit s = parity to wait for on slot s
  Partial p{kNone, kNone, 0};
  for (int s = 0, left = filled; left > 0; s = (s + 1 == kStages) ? 0 : s + 1) {
    mbar_wait(&ring.bar[s], (phase >> s) & 1u);
    phase ^= 1u << s;
    const TileInfo t = ring.info[s];
    if (t.flags & kTileData) {
      if (gen.two_bit) {
        if (t.flags & kTileHtod) consume_2bit<true>(ring.data[s], t.q0, t.q1, t.ob, p);
        else consume_2bit<false>(ring.data[s], t.q0, t.q1, t.ob, p);
      } else if (t.flags & kTileHtod) {
        consume_htod(ring.data[s], t.q0, t.q1, t.ob, p);
      } else if (t.flags & kTilePacked) {   // rows j = 0..k-1 (TileGen::packed_tile)
        const uint32_t k = t.q1 & 0xFFFFu, rs = t.q1 >> 16, W = t.q0;
        for (uint32_t j = 0; j < k; ++j) {
          const uint64_t q = t.qs + (uint64_t)j * t.qe, qa = q & ~127ull;
          const uint32_t c0 = (uint32_t)(q - qa);
          consume_dtoh(ring.data[s] + j * rs, c0, c0 + W, t.ob + (uint64_t)j * (W - t.qe) + qa, p);
        }
      } else {
        consume_dtoh(ring.data[s], t.q0, t.q1, t.ob, p);
      }
    }
    if (t.flags & kTileEnd) {
      p.fu = umin64(p.fu, t.pend_fu);
      if (__any_sync(kFull, p.fu != kNone || p.fd != kNone || p.cnt != 0)) {
        p.fu = warp_min(p.fu);
        p.fd = warp_min(p.fd);
        p.cnt = warp_sum(p.cnt);
      }
      bool apply = false;
      if (lane == 0) {
        cg_verdict* v = out + t.d;
        if ((t.flags & (kTileWhole | kTileRaw)) == (kTileWhole | kTileRaw)) {
          v->first_unaddr = p.fu;   // raw partial (straddler): finalised after the merge
          v->first_undef = p.fd;
          v->undef_count = p.cnt;
        } else if (t.flags & kTileWhole) {
          uint32_t flags = t.flags >> 16, status;
          finalize_fields(flags, status, p.fu, p.cnt, err_mask);
          v->first_unaddr = p.fu;
          v->first_undef = p.fd;
          v->undef_count = p.cnt;
          v->flags = flags;
          v->status = status;
          apply = (t.flags & kTileFuse) && status == CG_OK;
          // a whole 2D DtoH piece with status OK: the residual pass applies it
          if (kFuse && !(t.flags & (kTileFuse | kTileHtod)) && status == CG_OK)
            push_apply(t.flags & kTileLast, t.d, resid, resid_n, last);
        } else {
          if (p.fu != kNone) atomicMin(reinterpret_cast<unsigned long long*>(&v->first_unaddr), p.fu);
          if (p.fd != kNone) atomicMin(reinterpret_cast<unsigned long long*>(&v->first_undef), p.fd);
          if (p.cnt) atomicAdd(reinterpret_cast<unsigned long long*>(&v->undef_count), p.cnt);
        }
      }
      p = Partial{kNone, kNone, 0};
      // fused a6: a whole contiguous DtoH piece with status OK becomes defined
      if (__shfl_sync(kFull, apply, 0)) {
        if (gen.two_bit) fill2_any<true, kSparse>(sv, t.qs, t.qe, 0xAAAAAAAAu);
        else warp_store_zero(sv.V, t.qs, t.qe);
      }
    }
    __syncwarp();
    if (!gen.next(ring, s, sv, policy)) --left;
  }
  defer_tail(descs, defer, counter, meta, sv, out, err_mask, kFuse ? 1 : 0, resid, resid_n, last);
}


// which of the descriptors d0 + u nthr (u < kSplitDeep) were split across
// groups (weight above the never-split limit, see compute_pieces): their prefix
// sums loaded together -- a plain grid-stride loop over 10M descriptors waited
// one DRAM round trip per descriptor and thread (C5: 0.13 ms of k_finish)
constexpr int kSplitDeep = 8;
__device__ __forceinline__ uint32_t split_mask(const uint64_t* __restrict__ P, uint64_t n, uint64_t d0, uint64_t nthr,
                                               uint64_t trule) {
  uint64_t a[kSplitDeep], b[kSplitDeep];
#pragma unroll
  for (int u = 0; u < kSplitDeep; ++u) {
    const uint64_t d = d0 + (uint64_t)u * nthr;
    a[u] = d < n ? __ldcg(P + d) : 0;
    b[u] = d < n ? __ldcg(P + d + 1) : 0;
  }
  uint32_t m = 0;
#pragma unroll
  for (int u = 0; u < kSplitDeep; ++u) m |= (uint32_t)(b[u] - a[u] > trule) << u;
  return m;
}

// a5 for descriptors split across groups
__global__ void __launch_bounds__(kThreads) k_finalize_split(uint64_t n, const uint64_t* __restrict__ P,
                                                             uint64_t t_min, uint64_t max_chunks,
                                                             cg_verdict* __restrict__ out, uint32_t err_mask,
                                                             const ScanMeta* __restrict__ meta, int fuse,
                                                             uint32_t* __restrict__ resid,
                                                             uint32_t* __restrict__ resid_n, uint32_t small_share) {
  pdl_entry();
  // the deferred list of the next check starts empty (its prep appends to it,
  // so it cannot reset it itself); resid_n = counter + 2
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    resid_n[2] = resid_n[3] = 0;   // counter[4], [5]: the deferred list
    next_small_choice(resid_n - 2, small_share);
  }
  if (!fuse && blockIdx.x == 0 && threadIdx.x == 0) resid_n[0] = 0;   // nothing appends to the residual list unfused
  const ChunkGeom g = chunk_geom(P, n, t_min, max_chunks);
  const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t d0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; d0 < n; d0 += kSplitDeep * nthr) {
    uint32_t split = split_mask(P, n, d0, nthr, g.Trule);
    while (split) {
      const uint64_t d = d0 + (uint64_t)(__ffs(split) - 1) * nthr;
      split &= split - 1;
      const uint64_t info = meta[d].info;
      if ((info >> kInfoRaw) & 1u) continue;   // raw partial of a straddler
      cg_verdict* v = out + d;
      uint32_t flags = v->flags, status;
      finalize_fields(flags, status, v->first_unaddr, v->undef_count, err_mask);
      v->flags = flags;
      v->status = status;
      // fused check: a split DtoH piece is applied by the residual pass
      if (fuse && status == CG_OK && ((info >> kInfoKind) & 3u) == CG_DTOH && ((info >> kInfoHost) & 1u))
        resid[atomicAdd(resid_n, 1u)] = (uint32_t)d;
    }
  }
}

// Logical host bytes [lo, hi) of a descriptor, row by row (R-11).
template <typename SegFn>
__device__ __forceinline__ void for_rows(const Norm& nm, uint64_t lo, uint64_t hi, SegFn fn) {
  const uint64_t W = nm.W;
  uint64_t r = lo / W;
  uint64_t c = lo - r * W;
  uint64_t o = lo;
  while (o < hi) {
    const uint64_t seg = umin64(W - c, hi - o);
    fn(nm.hstart + r * nm.hpitch + c, seg, o);
    o += seg;
    ++r;
    c = 0;
  }
}


// ---------------------------------------------------------------------------
// a6: DtoH apply
// ---------------------------------------------------------------------------
// The written host bytes of every DtoH descriptor with status OK become
// defined: V := 0x00.  Same equal-weight dynamic groups and lane-parallel
// descriptor window as the scan; the zeros are written by bulk asynchronous
// copies (cp.async.bulk shared -> global, <= 4 KiB each) from a zero page in
// shared memory, so one lane instruction writes 4 KiB; only the unaligned
// head/tail bytes (< 16 per segment) use byte stores.
constexpr uint64_t kApplyItemCost = 64;
constexpr int kApplyContig = 63;   // apply records: info = host bytes | contiguous << 63
constexpr uint32_t kZeroPage = 4096;

// The applicable descriptors (DtoH, status OK, host bytes) are compacted to
// the front of weight[] / meta[] (order is irrelevant: the apply is idempotent
// and commutative), so the apply walk never crosses runs of inapplicable
// descriptors; weight[] must be zero on entry.
__global__ void __launch_bounds__(kThreads) k_apply_prep(const cg_copy_desc* __restrict__ descs,
                                                         const cg_verdict* __restrict__ verd, uint64_t n,
                                                         uint64_t* __restrict__ weight, ScanMeta* __restrict__ meta,
                                                         uint32_t* __restrict__ count) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  for (uint64_t b0 = (uint64_t)blockIdx.x * blockDim.x; b0 < n; b0 += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = b0 + threadIdx.x;
    bool ok = false;
    ScanMeta m;
    uint64_t w = 0;
    if (i < n && (descs[i].kind == CG_DTOH || descs[i].kind == CG_ATOH) && verd[i].status == CG_OK) {
      const cg_copy_desc d = descs[i];
      const Norm nm = normalize(d);
      if (nm.host && nm.nbytes) {
        ok = true;
        w = kApplyItemCost + nm.nbytes;
        m.hstart = nm.hstart;
        m.hpitch = nm.hpitch;
        m.W = nm.W;
        m.info = nm.nbytes | ((uint64_t)(d.height == 1 || d.width == nm.hpitch) << kApplyContig);
      }
    }
    const uint32_t mask = __ballot_sync(kFull, ok);
    if (mask) {
      const int leader = __ffs(mask) - 1;
      uint32_t base = 0;
      if (lane == leader) base = atomicAdd(count, (uint32_t)__popc(mask));
      base = __shfl_sync(kFull, base, leader);
      if (ok) {
        const uint32_t k = base + __popc(mask & ((1u << lane) - 1u));
        weight[k] = w;
        meta[k] = m;
      }
    }
  }
}

// after cg_check_apply: the DtoH descriptors the fused scan did not apply
// itself (split across groups, or 2D) and whose verdict is OK were listed by
// the scan / k_finalize_split; compact weights and metadata for them
__global__ void __launch_bounds__(kThreads) k_apply_list_prep(const cg_copy_desc* __restrict__ descs,
                                                              const uint32_t* __restrict__ list,
                                                              const uint32_t* __restrict__ count,
                                                              uint64_t* __restrict__ weight,
                                                              ScanMeta* __restrict__ meta,
                                                              uint32_t* __restrict__ group_counter) {
  pdl_entry();
  if (blockIdx.x == 0 && threadIdx.x == 0) *group_counter = 0;   // k_apply's (no memset node)
  const uint64_t m = *count;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m; k += (uint64_t)gridDim.x * blockDim.x) {
    const cg_copy_desc d = descs[list[k]];
    const Norm nm = normalize(d);
    ScanMeta mm;
    mm.hstart = nm.hstart;
    mm.hpitch = nm.hpitch;
    mm.W = nm.W;
    mm.info = nm.nbytes | ((uint64_t)(d.height == 1 || d.width == nm.hpitch) << kApplyContig);
    meta[k] = mm;
    weight[k] = kApplyItemCost + nm.nbytes;
  }
}

__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
               "r"(bytes)
               : "memory");
}

// zero shard bytes [q0, q1) from one lane: byte stores for the unaligned
// edges, bulk stores of the zero page for the 16-byte aligned middle
__device__ __forceinline__ void lane_zero(uint8_t* V, uint64_t q0, uint64_t q1, const uint8_t* zeros) {
  const uint64_t a0 = (q0 + 15) & ~15ull, a1 = q1 & ~15ull;
  if (a0 >= a1) {
    for (uint64_t q = q0; q < q1; ++q) V[q] = 0;
    return;
  }
  for (uint64_t q = q0; q < a0; ++q) V[q] = 0;
  for (uint64_t q = a1; q < q1; ++q) V[q] = 0;
  for (uint64_t p = a0; p < a1; p += kZeroPage) bulk_s2g(V + p, zeros, (uint32_t)umin64(kZeroPage, a1 - p));
}

// zero [q0, q1) with the whole warp: lane j takes the 4 KiB pages j, j+32, ...
__device__ __forceinline__ void warp_zero(uint8_t* V, uint64_t q0, uint64_t q1, const uint8_t* zeros) {
  const int lane = threadIdx.x & 31;
  const uint64_t a0 = (q0 + 15) & ~15ull, a1 = q1 & ~15ull;
  if (a0 >= a1) {
    if (lane == 0)
      for (uint64_t q = q0; q < q1; ++q) V[q] = 0;
    return;
  }
  if (lane == 0)
    for (uint64_t q = q0; q < a0; ++q) V[q] = 0;
  if (lane == 1)
    for (uint64_t q = a1; q < q1; ++q) V[q] = 0;
  for (uint64_t p = a0 + (uint64_t)lane * kZeroPage; p < a1; p += 32ull * kZeroPage)
    bulk_s2g(V + p, zeros, (uint32_t)umin64(kZeroPage, a1 - p));
}

#ifndef CG_APPLY_BULK
#define CG_APPLY_BULK 1   // the apply's warp pieces: bulk stores from a zero page (0: 16-byte stores of all lanes)
#endif
// the apply walk over planned groups (shared by k_apply and k_finish)
template <bool kTwoBit>
__device__ __forceinline__ void apply_body(const ScanMeta* __restrict__ meta, uint64_t n,
                                           const uint64_t* __restrict__ P, const uint32_t* __restrict__ chunk_first,
                                           uint32_t* counter, uint64_t t_min, uint64_t max_chunks,
                                           const ShadowView& sv, const uint8_t* zeros) {
  const ChunkGeom geo = chunk_geom(P, n, t_min, max_chunks);
  const int lane = threadIdx.x & 31;
  uint32_t gnext = lane == 0 ? atomicAdd(counter, 1u) : 0;
  while (true) {
    const uint64_t g = __shfl_sync(kFull, gnext, 0);
    if (g >= geo.nchunks) break;
    if (lane == 0) gnext = atomicAdd(counter, 1u);
    const uint64_t w0 = g * geo.T, w1 = umin64(w0 + geo.T, geo.total);
    for (uint64_t base = chunk_first[g];; base += 32) {
      // lane-parallel: this lane's descriptor piece in the group
      const uint64_t i = base + lane;
      uint64_t ps = ~0ull, pe = ~0ull;
      if (i < n) {
        ps = P[i];
        pe = P[i + 1];
      }
      const bool in = ps < w1 && pe > w0 && pe > ps;
      bool small = false, big = false;
      uint64_t qs = 0, qe = 0, lo = 0, hi = 0;
      ScanMeta m{0, 0, 0, 0};
      if (in) {
        m = meta[i];
        uint64_t a = umax64(w0, ps) - ps, b = umin64(w1, pe) - ps;
        lo = a > kApplyItemCost ? a - kApplyItemCost : 0;
        hi = b > kApplyItemCost ? b - kApplyItemCost : 0;
        if (lo < hi) {
          if ((m.info >> kApplyContig) & 1u) {
            const uint64_t x = m.hstart + lo, y0 = umax64(x, sv.sb), y1 = umin64(x + (hi - lo), sv.se);
            if (y0 < y1) {
              qs = y0 - sv.sb;
              qe = y1 - sv.sb;
              small = qe - qs <= (kTwoBit ? 256u : 2 * kZeroPage);
              big = !small;
            }
          } else {
            big = true;   // 2D: rows, whole warp
          }
        }
      }
      if (small) {
        if (kTwoBit) fill2_any<false>(sv, qs, qe, 0xAAAAAAAAu);
        else lane_zero(sv.V, qs, qe, zeros);
      }
      uint32_t todo = __ballot_sync(kFull, big);
      while (todo) {
        const int src = __ffs(todo) - 1;
        todo &= todo - 1;
        const uint64_t s_info = __shfl_sync(kFull, m.info, src);
        if ((s_info >> kApplyContig) & 1u) {
          const uint64_t a = __shfl_sync(kFull, qs, src), b = __shfl_sync(kFull, qe, src);
          if (kTwoBit) fill2_any<true>(sv, a, b, 0xAAAAAAAAu);
          else if (CG_APPLY_BULK) warp_zero(sv.V, a, b, zeros);
          else warp_store_zero(sv.V, a, b);
        } else {
          const uint64_t x0 = __shfl_sync(kFull, m.hstart, src), pitch = __shfl_sync(kFull, m.hpitch, src);
          const uint64_t W = __shfl_sync(kFull, m.W, src);
          const uint64_t o = __shfl_sync(kFull, lo, src), h = __shfl_sync(kFull, hi, src);
          uint64_t oo = o, r = o / W, c = o - r * W;
          while (oo < h) {   // row segments (R-11), each with the whole warp
            const uint64_t len = umin64(W - c, h - oo);
            const uint64_t x = x0 + r * pitch + c;
            const uint64_t y0 = umax64(x, sv.sb), y1 = umin64(x + len, sv.se);
            if (y0 < y1) {
              if (kTwoBit) fill2_any<true>(sv, y0 - sv.sb, y1 - sv.sb, 0xAAAAAAAAu);
              else if (CG_APPLY_BULK) warp_zero(sv.V, y0 - sv.sb, y1 - sv.sb, zeros);
              else warp_store_zero(sv.V, y0 - sv.sb, y1 - sv.sb);
            }
            oo += len;
            ++r;
            c = 0;
          }
        }
      }
      // continue with the next 32 descriptors while the group does
      if (!(__shfl_sync(kFull, (uint32_t)(ps < w1), 31) && base + 32 < n)) break;
    }
  }
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ void zero_page(uint8_t* zeros) {
  for (uint32_t i = threadIdx.x; i < kZeroPage / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(zeros)[i] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
}

template <bool kTwoBit>
__global__ void __launch_bounds__(kThreads) k_apply(const ScanMeta* __restrict__ meta, uint64_t n,
                                                    const uint64_t* __restrict__ P,
                                                    const uint32_t* __restrict__ chunk_first, uint32_t* counter,
                                                    uint64_t t_min, uint64_t max_chunks, ShadowView sv,
                                                    const uint32_t* __restrict__ n_dev) {
  pdl_entry();
  n = eff_n(n, n_dev);
  __shared__ __align__(128) uint8_t zeros[kZeroPage];
  zero_page(zeros);
  apply_body<kTwoBit>(meta, n, P, chunk_first, counter, t_min, max_chunks, sv, zeros);
}

// a6 for one whole DtoH descriptor with the whole warp, row by row (R-11),
// clipped to the shard: its host bytes become defined (CG_APPLY_LAST; rare,
// so plain generic stores and no plan)
template <bool kTwoBit>
__device__ __noinline__ void apply_whole(const cg_copy_desc d, const ShadowView& sv) {
  const Norm nm = normalize(d);
  const bool contig = d.height == 1 || d.width == nm.hpitch;
  const uint64_t rows = contig ? 1 : d.height, len = contig ? nm.nbytes : nm.W;
  for (uint64_t r = 0; r < rows && len; ++r) {
    const uint64_t x = nm.hstart + r * nm.hpitch;
    if (x >= sv.se) break;   // rows ascend (pitch >= 0)
    const uint64_t y0 = umax64(x, sv.sb), y1 = umin64(x + len, sv.se);
    if (y0 >= y1) continue;
    if (kTwoBit) fill2_any<true>(sv, y0 - sv.sb, y1 - sv.sb, 0xAAAAAAAAu);
    else warp_store_zero(sv.V, y0 - sv.sb, y1 - sv.sb);
  }
}

// cg_check_apply's tail in one cooperative launch (after the fused scan):
// finalise split descriptors (k_finalize_split), then -- only if the scan or
// the finalisation left a residual DtoH list (split or 2D pieces) -- its
// records and weights, their prefix sum, the chunk plan and the apply walk,
// with grid barriers between the phases.  An empty list (C2: every DtoH piece
// was applied by the scan) costs one launch and one barrier instead of six
// launches.
template <bool kTwoBit>
__global__ void __launch_bounds__(kThreads) k_finish(
    const cg_copy_desc* __restrict__ descs, uint64_t n, uint64_t* P, uint64_t t_min, uint64_t max_chunks,
    cg_verdict* __restrict__ out, uint32_t err_mask, ScanMeta* meta, uint32_t* __restrict__ resid,
    uint32_t* counter, uint64_t* __restrict__ weight, uint64_t* __restrict__ bsum, uint32_t* __restrict__ chunk_first,
    ShadowView sv, const uint32_t* __restrict__ late_list, uint32_t* __restrict__ last_list) {
  pdl_entry();
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  __shared__ __align__(128) uint8_t zeros[kZeroPage];
  __shared__ uint64_t s_warp[33];
  uint32_t* resid_n = counter + 2;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nthr = (uint64_t)gridDim.x * blockDim.x;
  {   // a5 for split descriptors
    const ChunkGeom g = chunk_geom(P, n, t_min, max_chunks);
    for (uint64_t d0 = tid; d0 < n; d0 += kSplitDeep * nthr) {
      uint32_t split = split_mask(P, n, d0, nthr, g.Trule);
      while (split) {
        const uint64_t d = d0 + (uint64_t)(__ffs(split) - 1) * nthr;
        split &= split - 1;
        const uint64_t info = meta[d].info;
        if ((info >> kInfoRaw) & 1u) continue;     // raw partial of a straddler
        cg_verdict* v = out + d;
        uint32_t flags = v->flags, status;
        finalize_fields(flags, status, v->first_unaddr, v->undef_count, err_mask);
        v->flags = flags;
        v->status = status;
        if (status == CG_OK && ((info >> kInfoKind) & 3u) == CG_DTOH && ((info >> kInfoHost) & 1u))
          push_apply((info >> kInfoLast) & 1u, (uint32_t)d, resid, resid_n, last_list);
      }
    }
    if (tid == 0) {
      counter[0] = 0;   // the apply walk's group counter
      counter[4] = counter[5] = 0;   // the deferred list of the next check (the prep appends to it)
      next_small_choice(counter, sv.small_share);
    }
  }
  grid.sync();
  const uint64_t m = __ldcg(resid_n);
  if (m > 0) {   // uniform
  for (uint64_t k = tid; k < m; k += nthr) {   // residual records (k_apply_list_prep)
    const cg_copy_desc d = descs[resid[k]];
    const Norm nm = normalize(d);
    ScanMeta mm;
    mm.hstart = nm.hstart;
    mm.hpitch = nm.hpitch;
    mm.W = nm.W;
    mm.info = nm.nbytes | ((uint64_t)(d.height == 1 || d.width == nm.hpitch) << kApplyContig);
    meta[k] = mm;
    weight[k] = kApplyItemCost + nm.nbytes;
  }
  grid.sync();
  if (tid == 0) *resid_n = 0;   // every block has read m: the next check's residual list starts empty
  // prefix sum of weight[0..m) into P: block b owns items [b*per, (b+1)*per)
  const uint64_t per = (m + gridDim.x - 1) / gridDim.x;
  const uint64_t lo = umin64(m, (uint64_t)blockIdx.x * per), hi = umin64(m, lo + per);
  {
    uint64_t acc = 0;
    for (uint64_t k = lo + threadIdx.x; k < hi; k += blockDim.x) acc += __ldcg(weight + k);
    uint64_t total;
    block_exclusive_scan(acc, s_warp, total);
    if (threadIdx.x == 0) bsum[blockIdx.x] = total;
  }
  grid.sync();
  if (blockIdx.x == 0) {   // exclusive scan of the block sums
    uint64_t carry = 0;
    for (uint64_t b0 = 0; b0 < gridDim.x; b0 += blockDim.x) {
      const uint64_t b = b0 + threadIdx.x;
      const uint64_t x = b < gridDim.x ? __ldcg(bsum + b) : 0;
      uint64_t total;
      const uint64_t ex = block_exclusive_scan(x, s_warp, total);
      if (b < gridDim.x) bsum[b] = carry + ex;
      carry += total;
    }
    if (threadIdx.x == 0) P[m] = carry;
  }
  grid.sync();
  {
    uint64_t carry = __ldcg(bsum + blockIdx.x);
    for (uint64_t k0 = lo; k0 < hi; k0 += blockDim.x) {
      const uint64_t k = k0 + threadIdx.x;
      const uint64_t x = k < hi ? __ldcg(weight + k) : 0;
      uint64_t total;
      const uint64_t ex = block_exclusive_scan(x, s_warp, total);
      if (k < hi) P[k] = carry + ex;
      carry += total;
    }
  }
  grid.sync();
  {   // the chunk plan (k_plan)
    const ChunkGeom g = chunk_geom(P, m, t_min, max_chunks);
    for (uint64_t c = tid; c < g.nchunks; c += nthr) {
      const uint64_t target = c * g.T;
      uint64_t a = 0, b = m;   // P[a] <= target < P[b]
      while (b - a > 1) {
        const uint64_t mid = (a + b) >> 1;
        if (__ldcg(P + mid) <= target) a = mid; else b = mid;
      }
      chunk_first[c] = (uint32_t)a;
    }
  }
  zero_page(zeros);
  grid.sync();
  apply_body<kTwoBit>(meta, m, P, chunk_first, counter, t_min, max_chunks, sv, zeros);
  }
  // CG_CHECK_AFTER: the HtoD sides that read bytes an earlier DtoH of the batch
  // wrote, checked now that every apply of the batch is done (warp per side);
  // then the CG_APPLY_LAST DtoH sides, which write bytes such an HtoD reads
  const uint32_t nl = __ldcg(counter + 6), nz = __ldcg(counter + 8);   // final since the first barrier
  if (nl == 0 && nz == 0) return;   // uniform
  asm volatile("fence.proxy.async.global;" ::: "memory");   // the residual apply's bulk stores, before generic loads
  __threadfence();
  grid.sync();
  if (!sv.sparse) {   // (late side, part) items over all warps, then the finalisation
    constexpr uint32_t kLateParts = 32;
    for (uint64_t k = tid >> 5; k < (uint64_t)nl * kLateParts; k += nthr >> 5)
      late_part(descs, late_list[k / kLateParts], (uint32_t)(k % kLateParts), kLateParts, sv, out);
    __threadfence();
    grid.sync();
    for (uint64_t k = tid; k < nl; k += nthr) late_finalize(out + late_list[k], err_mask);
  } else {   // the records in meta[] were reused above: flags from the verdict
    for (uint64_t k = tid >> 5; k < nl; k += nthr >> 5)
      defer_one(descs, late_list[k], nullptr, sv, out, err_mask, 0, resid, resid_n, last_list);
  }
  if (nz) {   // uniform
    grid.sync();   // every late check has read the shadow
    for (uint64_t k = tid >> 5; k < nz; k += nthr >> 5) apply_whole<kTwoBit>(descs[last_list[k]], sv);
  }
  grid.sync();
  if (tid == 0) counter[6] = counter[7] = counter[8] = 0;   // the next check's late and last lists start empty
}

// fill shard-relative V bytes [q0, q1) with the byte value `val` (0x00/0xFF)
__device__ __forceinline__ void fill_v(const ShadowView& sv, uint64_t q0, uint64_t q1, uint32_t val) {
  const int lane = threadIdx.x & 31;
  const uint64_t k0 = q0 >> 4, k1 = (q1 + 15) >> 4;
  uint4* V4 = reinterpret_cast<uint4*>(sv.V);
  const uint32_t word = val * 0x01010101u;
  for (uint64_t k = k0 + lane; k < k1; k += 32) {
    const uint64_t qb = k << 4;
    if (qb >= q0 && qb + 16 <= q1) {
      stg_val16(V4 + k, word);
    } else {
      for (uint64_t q = umax64(qb, q0); q < umin64(qb + 16, q1); ++q) sv.V[q] = (uint8_t)val;
    }
  }
}

// ---------------------------------------------------------------------------
// NEXT-1: V-bit propagation (SPEC copy_vbits S:81-89) through error-free copies
// ---------------------------------------------------------------------------
struct __align__(16) PropMeta {
  uint64_t src, dst;        // offsets: host V (x - shard_base) or device V pool
  uint64_t spitch, dpitch;
  uint64_t W, info;         // info: nbytes | src in pool << 41 | dst in pool << 42
};
constexpr uint64_t kPropItemCost = 64;
constexpr uint64_t kStageBytes = 8ull << 20;   // staging of self-overlapping 2D DtoD

// Every descriptor with status OK and bytes to move gets a compacted PropMeta
// and weight; a DtoD whose pool source and target ranges overlap goes to the
// memmove list instead (processed by k_memmove, one CTA each).
__global__ void __launch_bounds__(kThreads) k_prop_prep(const cg_copy_desc* __restrict__ descs,
                                                        const cg_verdict* __restrict__ verd,
                                                        const uint32_t* __restrict__ index, uint64_t n,
                                                        const uint64_t* __restrict__ dvoff, uint64_t sb,
                                                        uint64_t* __restrict__ weight, PropMeta* __restrict__ pm,
                                                        uint32_t* __restrict__ count, uint32_t* __restrict__ mm,
                                                        uint32_t* __restrict__ mm_count) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  for (uint64_t b0 = (uint64_t)blockIdx.x * blockDim.x; b0 < n; b0 += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = b0 + threadIdx.x;
    const uint64_t i = k < n ? (index ? (uint64_t)index[k] : k) : ~0ull;   // a wave's subset, or all
    bool ok = false;
    PropMeta m;
    uint64_t w = 0;
    if (k < n && verd[i].status == CG_OK) {
      const cg_copy_desc d = descs[i];
      const Norm nm = normalize(d);
      const uint64_t nb = d.width * d.height;   // status OK: no INVALID_RANGE, so no overflow
      if (nb) {
        m.W = d.width;
        m.spitch = d.src_pitch;
        m.dpitch = d.dst_pitch;
        if (d.kind == CG_HTOA) {       // S:252 / R-30: host -> the array's V-bits (W*H contiguous bytes)
          m.src = nm.ss - sb;
          m.dst = dvoff[2 * i];
          m.dpitch = d.width;
          m.info = nb | (1ull << 42);
        } else if (d.kind == CG_ATOH) {   // the array's V-bits -> host
          m.src = dvoff[2 * i + 1];
          m.spitch = d.width;
          m.dst = nm.ds - sb;
          m.info = nb | (1ull << 41);
        } else if (d.kind == CG_HTOD) {
          m.src = nm.ss - sb;
          m.dst = dvoff[2 * i];
          m.info = nb | (1ull << 42);
        } else if (d.kind == CG_DTOH) {
          m.src = dvoff[2 * i + 1];
          m.dst = nm.ds - sb;
          m.info = nb | (1ull << 41);
        } else {
          m.src = dvoff[2 * i + 1];
          m.dst = dvoff[2 * i];
          m.info = nb | (3ull << 41);
        }
        ok = true;
        if (d.kind == CG_DTOD && m.src < m.dst + nm.dspan && m.dst < m.src + nm.sspan) {
          ok = false;   // overlaps itself: memmove list
          mm[atomicAdd(mm_count, 1u)] = (uint32_t)i;
        }
        w = kPropItemCost + nb;
      }
    }
    const uint32_t mask = __ballot_sync(kFull, ok);
    if (mask) {
      const int leader = __ffs(mask) - 1;
      uint32_t base = 0;
      if (lane == leader) base = atomicAdd(count, (uint32_t)__popc(mask));
      base = __shfl_sync(kFull, base, leader);
      if (ok) {
        const uint32_t k = base + __popc(mask & ((1u << lane) - 1u));
        weight[k] = w;
        pm[k] = m;
      }
    }
  }
}

// 16 bytes from an arbitrary address: the two aligned 16-byte vectors around
// it, realigned with funnel shifts (both vectors start inside the source
// range, and V / pool sizes are multiples of 16, so no read leaves its buffer)
__device__ __forceinline__ uint4 load_unaligned16(const uint8_t* p) {
  const uintptr_t a = (uintptr_t)p & ~(uintptr_t)15;
  const uint32_t m = (uint32_t)((uintptr_t)p & 15);
  const uint4 lo = *reinterpret_cast<const uint4*>(a);
  if (m == 0) return lo;
  const uint4 hi = *reinterpret_cast<const uint4*>(a + 16);
  const uint32_t q = m >> 2, r = (m & 3) * 8;
  const uint32_t w0 = q == 0 ? lo.x : q == 1 ? lo.y : q == 2 ? lo.z : lo.w;
  const uint32_t w1 = q == 0 ? lo.y : q == 1 ? lo.z : q == 2 ? lo.w : hi.x;
  const uint32_t w2 = q == 0 ? lo.z : q == 1 ? lo.w : q == 2 ? hi.x : hi.y;
  const uint32_t w3 = q == 0 ? lo.w : q == 1 ? hi.x : q == 2 ? hi.y : hi.z;
  const uint32_t w4 = q == 0 ? hi.x : q == 1 ? hi.y : q == 2 ? hi.z : hi.w;
  return make_uint4(__funnelshift_r(w0, w1, r), __funnelshift_r(w1, w2, r), __funnelshift_r(w2, w3, r),
                    __funnelshift_r(w3, w4, r));
}

// copy len bytes src -> dst with the whole warp: 16-byte stores to the aligned
// body of dst (sources realigned when the two are not equally aligned), byte
// copies for the unaligned head / tail
__device__ __forceinline__ void warp_copy(uint8_t* dst, const uint8_t* src, uint64_t len) {
  const int lane = threadIdx.x & 31;
  if (len < 64) {
    for (uint64_t k = lane; k < len; k += 32) dst[k] = src[k];
    return;
  }
  const uint64_t head = (16 - ((uintptr_t)dst & 15)) & 15;
  const uint64_t body = (len - head) & ~15ull;
  if ((uint64_t)lane < head) dst[lane] = src[lane];
  uint4* d4 = reinterpret_cast<uint4*>(dst + head);
  const uint64_t nv = body / 16;
  const bool same = (((uintptr_t)dst ^ (uintptr_t)src) & 15) == 0;
  // four vectors per lane in flight: all loads before the stores (src and dst may alias)
  uint64_t k = lane;
  for (; k + 96 < nv; k += 128) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      v[u] = same ? reinterpret_cast<const uint4*>(src + head)[k + 32 * u] : load_unaligned16(src + head + 16 * (k + 32 * u));
#pragma unroll
    for (int u = 0; u < 4; ++u) d4[k + 32 * u] = v[u];
  }
  for (; k < nv; k += 32)
    d4[k] = same ? reinterpret_cast<const uint4*>(src + head)[k] : load_unaligned16(src + head + 16 * k);
  for (uint64_t k = head + body + lane; k < len; k += 32) dst[k] = src[k];
}

__global__ void __launch_bounds__(kThreads) k_propagate(const PropMeta* __restrict__ pm, uint64_t n,
                                                        const uint64_t* __restrict__ P,
                                                        const uint32_t* __restrict__ chunk_first, uint32_t* counter,
                                                        uint64_t t_min, uint64_t max_chunks, uint8_t* V,
                                                        uint8_t* pool, const uint32_t* __restrict__ n_dev) {
  pdl_entry();
  n = eff_n(n, n_dev);
  const ChunkGeom geo = chunk_geom(P, n, t_min, max_chunks);
  const int lane = threadIdx.x & 31;
  uint32_t gnext = lane == 0 ? atomicAdd(counter, 1u) : 0;
  while (true) {
    const uint64_t g = __shfl_sync(kFull, gnext, 0);
    if (g >= geo.nchunks) break;
    if (lane == 0) gnext = atomicAdd(counter, 1u);
    const uint64_t w0 = g * geo.T, w1 = umin64(w0 + geo.T, geo.total);
    for (uint64_t d = chunk_first[g]; d < n; ++d) {
      const uint64_t pd = P[d];
      if (pd >= w1) break;
      const uint64_t pd1 = P[d + 1];
      uint64_t a = umax64(w0, pd) - pd, b = umin64(w1, pd1) - pd;
      a = a > kPropItemCost ? a - kPropItemCost : 0;
      b = b > kPropItemCost ? b - kPropItemCost : 0;
      if (a >= b) continue;
      const PropMeta m = pm[d];
      uint8_t* sbase = ((m.info >> 41) & 1u) ? pool : V;
      uint8_t* dbase = ((m.info >> 42) & 1u) ? pool : V;
      const bool zero = (m.info >> 43) & 1u;
      uint64_t r = a / m.W, c = a - r * m.W, o = a;
      while (o < b) {   // row segments (R-11); both sides advance by their own pitch
        const uint64_t len = umin64(m.W - c, b - o);
        const uint64_t q = m.dst + r * m.dpitch + c;
        if (zero) warp_store_zero(dbase, q, q + len);
        else warp_copy(dbase + q, sbase + m.src + r * m.spitch + c, len);
        o += len;
        ++r;
        c = 0;
      }
    }
  }
}

// copy len bytes with the whole CTA (the block-wide analogue of warp_copy)
__device__ __forceinline__ void block_copy(uint8_t* dst, const uint8_t* src, uint64_t len) {
  const uint32_t t = threadIdx.x, nt = blockDim.x;
  if (len < 64) {
    for (uint64_t k = t; k < len; k += nt) dst[k] = src[k];
    return;
  }
  const uint64_t head = (16 - ((uintptr_t)dst & 15)) & 15;
  const uint64_t body = (len - head) & ~15ull;
  if (t < head) dst[t] = src[t];
  uint4* d4 = reinterpret_cast<uint4*>(dst + head);
  const bool same = (((uintptr_t)dst ^ (uintptr_t)src) & 15) == 0;
  for (uint64_t k = t; k < body / 16; k += nt)
    d4[k] = same ? reinterpret_cast<const uint4*>(src + head)[k] : load_unaligned16(src + head + 16 * k);
  for (uint64_t k = head + body + t; k < len; k += nt) dst[k] = src[k];
}

__device__ __forceinline__ void block_zero(uint8_t* dst, uint64_t len) {
  for (uint64_t k = threadIdx.x; k < len; k += blockDim.x) dst[k] = 0;
}

// one wave copy's V-bit move: bases, offsets (false: nothing to move, or a
// self-overlapping DtoD, which the caller hands to the memmove list)
struct WaveCopy {
  uint8_t *sbase, *dbase;
  uint64_t src, dst, W, nb, spitch, dpitch;
  bool zero, self_overlap;
};
__device__ __forceinline__ bool wave_copy(const cg_copy_desc& d, uint32_t i, const uint64_t* dvoff, uint64_t sb,
                                          uint8_t* V, uint8_t* pool, WaveCopy& w) {
  w.W = d.width;
  w.nb = d.width * d.height;
  w.zero = w.self_overlap = false;
  w.spitch = d.src_pitch;
  w.dpitch = d.dst_pitch;
  if (w.nb == 0 || d.kind < CG_HTOD || d.kind > CG_ATOH) return false;
  const Norm nm = normalize(d);
  w.sbase = w.dbase = V;
  w.src = w.dst = 0;
  if (d.kind == CG_HTOA) {   // S:252 / R-30: host -> the array's V-bits
    w.src = nm.ss - sb;
    w.dst = dvoff[2 * i];
    w.dbase = pool;
    w.dpitch = d.width;
  } else if (d.kind == CG_ATOH) {   // the array's V-bits -> host
    w.src = dvoff[2 * i + 1];
    w.sbase = pool;
    w.spitch = d.width;
    w.dst = nm.ds - sb;
  } else if (d.kind == CG_HTOD) {
    w.src = nm.ss - sb;
    w.dst = dvoff[2 * i];
    w.dbase = pool;
  } else if (d.kind == CG_DTOH) {
    w.src = dvoff[2 * i + 1];
    w.dst = nm.ds - sb;
    w.sbase = pool;
  } else {
    w.src = dvoff[2 * i + 1];
    w.dst = dvoff[2 * i];
    w.sbase = w.dbase = pool;
    w.self_overlap = w.src < w.dst + nm.dspan && w.dst < w.src + nm.sspan;
    if (w.self_overlap) return false;
  }
  return true;
}

// one propagation wave (NEXT-1, cg_plan_waves) without a plan, three launches
// per wave.  Many copies: a warp per copy; few: CTA (x, y) moves the y-th
// 16 KiB slice of copy x.  A self-overlapping DtoD goes to the memmove list.
constexpr uint64_t kDirectSlice = 16384;
__global__ void __launch_bounds__(kThreads) k_prop_direct_warp(const cg_copy_desc* __restrict__ descs,
                                                               const cg_verdict* __restrict__ verd,
                                                               const uint32_t* __restrict__ index, uint64_t m,
                                                               const uint64_t* __restrict__ dvoff, uint64_t sb,
                                                               uint8_t* V, uint8_t* pool, uint32_t* __restrict__ mm,
                                                               uint32_t* __restrict__ mm_count) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t k = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < m; k += nw) {
    const uint32_t i = index[k];
    if (verd[i].status != CG_OK) continue;
    const cg_copy_desc d = descs[i];
    WaveCopy w;
    if (!wave_copy(d, i, dvoff, sb, V, pool, w)) {
      if (w.self_overlap && lane == 0) mm[atomicAdd(mm_count, 1u)] = i;
      continue;
    }
    for (uint64_t r = 0; r < d.height; ++r) {
      if (w.zero) warp_store_zero(w.dbase, w.dst + r * w.dpitch, w.dst + r * w.dpitch + w.W);
      else warp_copy(w.dbase + w.dst + r * w.dpitch, w.sbase + w.src + r * w.spitch, w.W);
    }
  }
}

__global__ void __launch_bounds__(kThreads) k_prop_direct(const cg_copy_desc* __restrict__ descs,
                                                          const cg_verdict* __restrict__ verd,
                                                          const uint32_t* __restrict__ index, uint64_t m,
                                                          const uint64_t* __restrict__ dvoff, uint64_t sb, uint8_t* V,
                                                          uint8_t* pool, uint32_t* __restrict__ mm,
                                                          uint32_t* __restrict__ mm_count) {
  pdl_entry();
  const uint64_t k = blockIdx.x;
  if (k >= m) return;
  const uint32_t i = index[k];
  if (verd[i].status != CG_OK) return;
  const cg_copy_desc d = descs[i];
  const uint64_t lo = (uint64_t)blockIdx.y * kDirectSlice;
  if (lo >= d.width * d.height) return;
  WaveCopy w;
  if (!wave_copy(d, i, dvoff, sb, V, pool, w)) {
    if (w.self_overlap && blockIdx.y == 0 && threadIdx.x == 0) mm[atomicAdd(mm_count, 1u)] = i;   // once
    return;
  }
  const uint64_t W = w.W, hi = umin64(w.nb, lo + kDirectSlice), src = w.src, dst = w.dst;
  uint8_t *sbase = w.sbase, *dbase = w.dbase;
  uint64_t r = lo / W, c = lo - r * W, o = lo;
  while (o < hi) {   // row segments (R-11); both sides advance by their own pitch
    const uint64_t len = umin64(W - c, hi - o);
    if (w.zero) block_zero(dbase + dst + r * w.dpitch + c, len);
    else block_copy(dbase + dst + r * w.dpitch + c, sbase + src + r * w.spitch + c, len);
    o += len;
    ++r;
    c = 0;
  }
}

// one self-overlapping DtoD with the whole CTA: equal pitches shift every byte
// by the same delta, so a directional block copy is exact memmove; unequal
// pitches stage all logical bytes first (scratch of stage_cap bytes); one
// that does not fit moves nothing here: it is flagged (*overflow) and listed
// (overflow[1] entries after overflow[2..]: the descriptor index) for the
// host's recovery pass, which stages it through a scratch of its size
__device__ __forceinline__ void block_memmove(const cg_copy_desc& d, uint32_t i, uint64_t so, uint64_t dso,
                                              uint8_t* pool, uint8_t* scratch, uint32_t* overflow,
                                              uint64_t stage_cap = kStageBytes) {
  const uint64_t W = d.width, H = d.height;
  if (d.src_pitch == d.dst_pitch || H == 1) {
    // chunks of 16 bytes per thread, each read completely before it is
    // written; moving down the chunks go in ascending order, up descending, so
    // a chunk's stores only reach source bytes already read
    const bool fwd = dso < so;
    const uint64_t CH = 16ull * blockDim.x;
    const bool vec = ((so ^ dso) & 15) == 0 && d.src_pitch % 16 == 0;   // 16-byte vectors line up
    for (uint64_t rr = 0; rr < H; ++rr) {
      const uint64_t r = fwd ? rr : H - 1 - rr;
      const uint8_t* rs = pool + so + r * d.src_pitch;
      uint8_t* rd = pool + dso + r * d.dst_pitch;
      for (uint64_t c0 = 0; c0 < W; c0 += CH) {
        const uint64_t cb = fwd ? c0 : (W > c0 + CH ? W - c0 - CH : 0);
        const uint64_t ce = fwd ? umin64(W, c0 + CH) : W - c0;
        const uint64_t c = cb + 16ull * threadIdx.x;
        const bool full = vec && c + 16 <= ce && ((uintptr_t)(rs + c) & 15) == 0;
        uint4 x = make_uint4(0, 0, 0, 0);
        uint8_t* xb = reinterpret_cast<uint8_t*>(&x);
        if (full) {
          x = __ldcg(reinterpret_cast<const uint4*>(rs + c));
        } else {
#pragma unroll
          for (int q = 0; q < 16; ++q)
            if (c + q < ce) xb[q] = __ldcg(rs + c + q);
        }
        __syncthreads();
        if (full) {
          *reinterpret_cast<uint4*>(rd + c) = x;
        } else {
#pragma unroll
          for (int q = 0; q < 16; ++q)
            if (c + q < ce) rd[c + q] = xb[q];
        }
        __syncthreads();
      }
    }
  } else if (W * H <= stage_cap) {
    for (uint64_t o = threadIdx.x; o < W * H; o += blockDim.x)
      scratch[o] = __ldcg(pool + so + (o / W) * d.src_pitch + o % W);
    __syncthreads();
    for (uint64_t o = threadIdx.x; o < W * H; o += blockDim.x)
      pool[dso + (o / W) * d.dst_pitch + o % W] = __ldcg(scratch + o);
    __syncthreads();
  } else if (threadIdx.x == 0) {
    atomicOr(overflow, 1u);
    overflow[2 + atomicAdd(overflow + 1, 1u)] = i;
  }
}

// the memmove list of one wave, one CTA per entry (equal pitches: entry k on
// block k mod grid; unequal: block 0, the scratch is shared)
__global__ void __launch_bounds__(kThreads) k_memmove(const cg_copy_desc* __restrict__ descs,
                                                      const uint64_t* __restrict__ dvoff,
                                                      const uint32_t* __restrict__ mm,
                                                      const uint32_t* __restrict__ mm_count, uint8_t* pool,
                                                      uint8_t* scratch, uint32_t* overflow, uint64_t stage_cap) {
  pdl_entry();
  const uint32_t cnt = *mm_count;
  for (uint32_t k = 0; k < cnt; ++k) {
    const uint32_t i = mm[k];
    const cg_copy_desc d = descs[i];
    const bool shared = d.src_pitch != d.dst_pitch && d.height > 1;
    if (shared ? blockIdx.x != 0 : k % gridDim.x != blockIdx.x) continue;
    block_memmove(d, i, dvoff[2 * i + 1], dvoff[2 * i], pool, scratch, overflow, stage_cap);
  }
}

// ---------------------------------------------------------------------------
// NEXT-1: all waves of a batch in one persistent cooperative launch
// ---------------------------------------------------------------------------
// cg_plan_waves orders the batch's copies into dependency waves (R-28); wave w
// is positions [wstart[w], wstart[w+1]) of the wave-ordered index.  k_wave_prep
// writes one PropMeta and weight per position (no compaction, so the wave
// bounds stay valid); one prefix sum over all positions; k_prop_waves then
// runs wave after wave with a grid barrier in between: the weight range of a
// wave is cut into equal pieces, one per warp, so a wave of 170k small copies
// and a wave of five 64 KiB copies both keep every warp streaming.  A copy
// whose weight range spans several pieces is moved by all of them, each its
// own bytes.  Self-overlapping DtoDs (memmove) go to a list worked off at the
// end of their wave, between two barriers, one CTA per entry.
constexpr uint64_t kWaveItemCost = 2048;     // per-copy latency, in bytes of bandwidth (env CG_WAVE_COST)
constexpr uint64_t kWaveMinPiece = 2048;     // smallest per-warp share of a wave (env CG_WAVE_PIECE)
constexpr uint64_t kPropMemmove = 1ull << 44;

__global__ void __launch_bounds__(kThreads) k_wave_prep(const cg_copy_desc* __restrict__ descs,
                                                        const cg_verdict* __restrict__ verd,
                                                        const uint32_t* __restrict__ index, uint64_t m,
                                                        const uint64_t* __restrict__ dvoff, uint64_t sb,
                                                        uint64_t* __restrict__ weight, PropMeta* __restrict__ pm,
                                                        uint32_t* __restrict__ mm, uint32_t* __restrict__ mm_count,
                                                        uint64_t item_cost) {
  pdl_entry();
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m; k += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = index[k];
    uint64_t w = 0;
    PropMeta pmk;
    pmk.info = 0;
    if (verd[i].status == CG_OK) {
      const cg_copy_desc d = descs[i];
      const uint64_t nb = d.width * d.height;   // status OK: no INVALID_RANGE, so no overflow
      if (nb) {
        const Norm nm = normalize(d);
        pmk.W = d.width;
        pmk.spitch = d.src_pitch;
        pmk.dpitch = d.dst_pitch;
        if (d.kind == CG_HTOA) {       // S:252 / R-30: host -> the array's V-bits (W*H contiguous bytes)
          pmk.src = nm.ss - sb;
          pmk.dst = dvoff[2 * i];
          pmk.dpitch = d.width;
          pmk.info = nb | (1ull << 42);
        } else if (d.kind == CG_ATOH) {   // the array's V-bits -> host
          pmk.src = dvoff[2 * i + 1];
          pmk.spitch = d.width;
          pmk.dst = nm.ds - sb;
          pmk.info = nb | (1ull << 41);
        } else if (d.kind == CG_HTOD) {
          pmk.src = nm.ss - sb;
          pmk.dst = dvoff[2 * i];
          pmk.info = nb | (1ull << 42);
        } else if (d.kind == CG_DTOH) {
          pmk.src = dvoff[2 * i + 1];
          pmk.dst = nm.ds - sb;
          pmk.info = nb | (1ull << 41);
        } else {
          pmk.src = dvoff[2 * i + 1];
          pmk.dst = dvoff[2 * i];
          pmk.info = nb | (3ull << 41);
        }
        w = item_cost + nb;
        if (d.kind == CG_DTOD && pmk.src < pmk.dst + nm.dspan && pmk.dst < pmk.src + nm.sspan) {
          w = 0;   // overlaps itself: the wave's memmove list
          pmk.info |= kPropMemmove;
          mm[atomicAdd(mm_count, 1u)] = (uint32_t)k;
        }
      }
    }
    weight[k] = w;
    pm[k] = pmk;
  }
}

// Per warp, a ring of kWStages tiles of up to kWTile source bytes: lane 0
// stages the 16-byte-aligned superset of a tile's source bytes with one
// cp.async.bulk (mbarrier transaction count), the warp then writes the tile's
// destination from shared memory with 16-byte stores to its aligned body
// (realigned with funnel shifts when source and destination differ mod 16) and
// byte stores for the head (lanes 0-15) and tail (lanes 16-31).  Loads are the
// latency-bound side, stores are posted: the ring keeps kWStages - 1 tiles of
// loads in flight per warp while one is written.
constexpr int kWRing = 4;                  // warps per CTA
constexpr int kWStages = 6;
constexpr uint32_t kWTile = 2048;          // source bytes per tile
constexpr uint32_t kWBuf = kWTile + 128;   // staged span <= kWTile + 15, rounded up to 16

struct __align__(16) WTile {
  uint64_t D;     // destination of the tile's first byte (generic address)
  uint32_t L;     // bytes
  uint32_t so;    // offset of the first source byte in the staged buffer; bit 31: zero tile (no staging)
};
struct WaveRing {
  uint8_t data[kWStages][kWBuf];
  WTile info[kWStages];
  uint64_t bar[kWStages];
};
constexpr size_t kWaveSmem = sizeof(WaveRing) * kWRing;

__device__ __forceinline__ void bulk_g2s_nohint(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// the tile generator of one warp (warp-uniform state; the 32-copy metadata
// window is lane-distributed): wave -> this warp's pieces of the wave's weight
// range -> copies -> row segments (R-11) -> tiles of <= kWTile bytes
struct WaveGen {
  const PropMeta* pm;
  const uint64_t* P;
  uint8_t *V, *pool;
  uint64_t gw, nw;
  uint64_t item_cost, min_piece;
  // wave and piece
  uint64_t a, b, w0, w1, piece, np, pc, s, e;
  bool have_piece;
  // window: lane i <-> position k0 + i
  uint64_t k0, pk, pk1;
  PropMeta m;
  uint32_t j;
  // current copy
  bool in_copy;
  uint64_t o, y, r, c, W, src, dst, sp, dp;
  uint8_t *sb, *db;
  bool zero;

  __device__ __forceinline__ void begin_wave(const uint32_t* wstart, uint32_t w) {
    a = __ldg(wstart + w);
    b = __ldg(wstart + w + 1);
    w0 = __ldg(P + a);
    w1 = __ldg(P + b);
    piece = umax64((w1 - w0 + nw - 1) / nw, min_piece);
    np = w1 > w0 ? (w1 - w0 + piece - 1) / piece : 0;
    pc = gw;
    have_piece = in_copy = false;
  }

  __device__ __forceinline__ void load_window() {
    const uint64_t kk = k0 + (threadIdx.x & 31);
    pk = pk1 = ~0ull;
    m.info = 0;
    if (kk < b) {
      pk = __ldg(P + kk);
      pk1 = __ldg(P + kk + 1);
      m = pm[kk];
    }
  }

  // the warp's next piece of the wave: 32-ary search for the last position
  // k in [a, b) with P[k] <= s (its weight range holds s)
  __device__ __forceinline__ bool begin_piece() {
    if (pc >= np) return false;
    s = w0 + pc * piece;
    e = umin64(s + piece, w1);
    pc += nw;
    const uint32_t lane = threadIdx.x & 31;
    uint64_t lo = a, hi = b;
    while (hi - lo > 1) {
      const uint64_t step = (hi - lo + 31) >> 5, x = lo + lane * step;
      const uint32_t le = __ballot_sync(kFull, x < hi && __ldg(P + x) <= s);
      lo += (uint64_t)(__popc(le) - 1) * step;
      hi = umin64(lo + step, hi);
    }
    k0 = lo;
    j = ~0u;   // next_copy starts at window lane 0
    load_window();
    have_piece = true;
    return true;
  }

  // the next copy with bytes in the current piece (or the next piece)
  __device__ __forceinline__ bool next_copy() {
    in_copy = false;
    while (true) {
      if (!have_piece && !begin_piece()) return false;
      if (++j == 32) {
        k0 += 32;
        j = 0;
        load_window();
      }
      if (k0 + j >= b) {
        have_piece = false;
        continue;
      }
      const uint64_t pd = __shfl_sync(kFull, pk, j);
      if (pd >= e) {
        have_piece = false;
        continue;
      }
      const uint64_t pd1 = __shfl_sync(kFull, pk1, j);
      uint64_t x = umax64(s, pd) - pd, yy = umin64(e, pd1) - pd;
      x = x > item_cost ? x - item_cost : 0;
      yy = yy > item_cost ? yy - item_cost : 0;
      if (x >= yy) continue;   // nothing to move here (or a memmove entry, weight 0)
      const uint64_t info = __shfl_sync(kFull, m.info, j);
      W = __shfl_sync(kFull, m.W, j);
      src = __shfl_sync(kFull, m.src, j);
      dst = __shfl_sync(kFull, m.dst, j);
      sp = __shfl_sync(kFull, m.spitch, j);
      dp = __shfl_sync(kFull, m.dpitch, j);
      sb = ((info >> 41) & 1u) ? pool : V;
      db = ((info >> 42) & 1u) ? pool : V;
      zero = (info >> 43) & 1u;
      r = x < W ? 0 : x / W;
      c = x - r * W;
      o = x;
      y = yy;
      in_copy = true;
      return true;
    }
  }

  // issues the next tile into ring slot `slot`; false when the wave holds no more for this warp
  __device__ __forceinline__ bool next(WaveRing& ring, int slot) {
    if (!in_copy || o >= y)
      if (!next_copy()) return false;
    const uint64_t len = umin64(umin64(W - c, y - o), kWTile);
    const uint8_t* S = sb + src + r * sp + c;
    uint8_t* D = db + dst + r * dp + c;
    o += len;
    c += len;
    if (c == W) {
      ++r;
      c = 0;
    }
    if ((threadIdx.x & 31) == 0) {
      WTile t;
      t.D = (uint64_t)D;
      t.L = (uint32_t)len;
      if (zero) {
        t.so = 1u << 31;
        ring.info[slot] = t;
        mbar_arrive(&ring.bar[slot]);
      } else {
        const uint32_t so = (uint32_t)((uintptr_t)S & 15);
        const uint32_t span = (so + (uint32_t)len + 15u) & ~15u;
        t.so = so;
        ring.info[slot] = t;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive_tx(&ring.bar[slot], span);
        bulk_g2s_nohint(ring.data[slot], S - so, span, &ring.bar[slot]);
      }
    }
    return true;
  }
};

__device__ __forceinline__ uint4 funnel16(uint4 lo, uint4 hi, uint32_t m) {
  const uint32_t q = m >> 2, r = (m & 3) * 8;
  const uint32_t w0 = q == 0 ? lo.x : q == 1 ? lo.y : q == 2 ? lo.z : lo.w;
  const uint32_t w1 = q == 0 ? lo.y : q == 1 ? lo.z : q == 2 ? lo.w : hi.x;
  const uint32_t w2 = q == 0 ? lo.z : q == 1 ? lo.w : q == 2 ? hi.x : hi.y;
  const uint32_t w3 = q == 0 ? lo.w : q == 1 ? hi.x : q == 2 ? hi.y : hi.z;
  const uint32_t w4 = q == 0 ? hi.x : q == 1 ? hi.y : q == 2 ? hi.z : hi.w;
  return make_uint4(__funnelshift_r(w0, w1, r), __funnelshift_r(w1, w2, r), __funnelshift_r(w2, w3, r),
                    __funnelshift_r(w3, w4, r));
}

// writes one staged tile to its destination
__device__ __forceinline__ void wave_consume(const WTile& t, const uint8_t* buf) {
  const uint32_t lane = threadIdx.x & 31;
  uint8_t* D = reinterpret_cast<uint8_t*>(t.D);
  const uint32_t L = t.L;
  const bool zero = t.so >> 31;
  const uint32_t so = t.so & 31u;
  const uint32_t hd = min(L, (uint32_t)((16 - ((uintptr_t)D & 15)) & 15));
  const uint32_t nv = (L - hd) >> 4, tl = L - hd - 16 * nv;
  if (lane < hd) D[lane] = zero ? 0 : buf[so + lane];
  else if (lane >= 16 && lane - 16 < tl) D[hd + 16 * nv + lane - 16] = zero ? 0 : buf[so + hd + 16 * nv + lane - 16];
  uint4* d4 = reinterpret_cast<uint4*>(D + hd);
  const uint32_t base = so + hd, sh = base & 15;
  if (zero) {
    for (uint32_t v = lane; v < nv; v += 32) d4[v] = make_uint4(0, 0, 0, 0);
  } else if (sh == 0) {
    const uint4* s4 = reinterpret_cast<const uint4*>(buf + base);
    for (uint32_t v = lane; v < nv; v += 32) d4[v] = s4[v];
  } else {
    const uint4* s4 = reinterpret_cast<const uint4*>(buf + (base & ~15u));
    for (uint32_t v = lane; v < nv; v += 32) d4[v] = funnel16(s4[v], s4[v + 1], sh);
  }
}

__global__ void __launch_bounds__(kWRing * 32) k_prop_waves(const cg_copy_desc* __restrict__ descs,
                                                            const uint32_t* __restrict__ index,
                                                            const PropMeta* __restrict__ pm,
                                                            const uint64_t* __restrict__ P,
                                                            const uint32_t* __restrict__ wstart, uint32_t n_waves,
                                                            uint8_t* V, uint8_t* pool,
                                                            const uint64_t* __restrict__ dvoff,
                                                            const uint32_t* __restrict__ mm,
                                                            const uint32_t* __restrict__ mm_count, uint8_t* scratch,
                                                            uint32_t* overflow, uint64_t item_cost, uint64_t min_piece) {
  pdl_entry();
  extern __shared__ __align__(128) uint8_t smem[];
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WaveRing& ring = reinterpret_cast<WaveRing*>(smem)[wid];
  if (lane == 0) {
    for (int s = 0; s < kWStages; ++s) mbar_init(&ring.bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  WaveGen gen;
  gen.pm = pm;
  gen.P = P;
  gen.V = V;
  gen.pool = pool;
  gen.gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  gen.nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  gen.item_cost = item_cost;
  gen.min_piece = min_piece;
  const uint32_t nmm = *mm_count;
  uint32_t phase = 0;   // bit s = parity to wait for on slot s
  gen.begin_wave(wstart, 0);
  gen.begin_piece();
  for (uint32_t w = 0; w < n_waves; ++w) {
    int filled = 0;
    while (filled < kWStages && gen.next(ring, filled)) ++filled;
    for (int s = 0, left = filled; left > 0; s = (s + 1 == kWStages) ? 0 : s + 1) {
      mbar_wait(&ring.bar[s], (phase >> s) & 1u);
      phase ^= 1u << s;
      const WTile t = ring.info[s];
      wave_consume(t, ring.data[s]);
      __syncwarp();
      if (!gen.next(ring, s)) --left;
    }
    const uint64_t a = gen.a, b = gen.b;
    if (w + 1 < n_waves) {   // the next wave's first piece: search + metadata (static) before the barrier
      gen.begin_wave(wstart, w + 1);
      gen.begin_piece();
    }
    bool has_mm = nmm > 64;   // a short list is searched for this wave's entries first
    for (uint32_t k = 0; k < nmm && !has_mm; ++k) {
      const uint32_t pos = __ldcg(mm + k);
      has_mm = pos >= a && pos < b;
    }
    if (has_mm) {   // this wave's self-overlapping DtoDs, after its other copies
      grid.sync();
      for (uint32_t k = 0; k < nmm; ++k) {   // entry k on CTA k mod grid; unequal pitches: CTA 0 (shared scratch)
        const uint32_t pos = __ldcg(mm + k);
        if (pos < a || pos >= b) continue;
        const uint32_t i = __ldg(index + pos);
        const cg_copy_desc d = descs[i];
        const bool shared = d.src_pitch != d.dst_pitch && d.height > 1;
        if (shared ? blockIdx.x != 0 : k % gridDim.x != blockIdx.x) continue;
        block_memmove(d, i, __ldg(dvoff + 2 * i + 1), __ldg(dvoff + 2 * i), pool, scratch, overflow);
      }
    }
    if (w + 1 < n_waves) {
      grid.sync();
      // the next wave's bulk copies (async proxy) read bytes this wave stored (generic proxy)
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
  }
}

// ---------------------------------------------------------------------------
// plumbing: fresh shadow, marks, set_vbits check
// ---------------------------------------------------------------------------
__global__ void k_fill(uint4* __restrict__ p, uint64_t n16, uint32_t word) {
  pdl_entry();
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16;
       i += (uint64_t)gridDim.x * blockDim.x)
    stg_val16(p + i, word);
}

__global__ void __launch_bounds__(kThreads) k_mark_prep(const cg_mark* __restrict__ marks, uint64_t n,
                                                        uint64_t* __restrict__ weight) {
  pdl_entry();
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    weight[i] = marks[i].len ? marks[i].len + kApplyItemCost : 0;
}

// A bits [q0, q1) := bit (set or clear); partial words with atomics because a
// neighbouring mark of the same batch may own the other bits of the word
__device__ __forceinline__ void put_abits(const ShadowView& sv, uint64_t q0, uint64_t q1, bool set) {
  const int lane = threadIdx.x & 31;
  uint32_t* A4 = reinterpret_cast<uint32_t*>(sv.A);
  const uint64_t k0 = q0 >> 5, k1 = (q1 + 31) >> 5;
  for (uint64_t k = k0 + lane; k < k1; k += 32) {
    const uint32_t m = range_mask(k << 5, 32, q0, q1);
    if (m == 0xffffffffu) A4[k] = set ? 0xffffffffu : 0u;
    else if (set) atomicOr(A4 + k, m);
    else atomicAnd(A4 + k, ~m);
  }
}

__global__ void __launch_bounds__(kThreads) k_mark(const cg_mark* __restrict__ marks, uint64_t n,
                                                   const uint64_t* __restrict__ P,
                                                   const uint32_t* __restrict__ chunk_first, uint64_t t_min,
                                                   uint64_t max_chunks, ShadowView sv) {
  pdl_entry();
  const ChunkGeom g = chunk_geom(P, n, t_min, max_chunks);
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t c = gw; c < g.nchunks; c += nw) {
    const uint64_t w0 = c * g.T, w1 = umin64(w0 + g.T, g.total);
    for (uint64_t d = chunk_first[c]; d < n; ++d) {
      const uint64_t pd = P[d];
      if (pd >= w1) break;
      const uint64_t pd1 = P[d + 1];
      if (pd1 == pd) continue;
      uint64_t a = umax64(w0, pd) - pd, b = umin64(w1, pd1) - pd;
      a = a > kApplyItemCost ? a - kApplyItemCost : 0;
      b = b > kApplyItemCost ? b - kApplyItemCost : 0;
      if (a >= b) continue;
      const cg_mark mk = marks[d];
      const uint64_t x = mk.addr + a, end = mk.addr + b;
      const uint64_t y0 = umax64(x, sv.sb), y1 = umin64(end, sv.se);
      if (y0 >= y1) continue;
      if (sv.two_bit) {
        fill2_any<true>(sv, y0 - sv.sb, y1 - sv.sb,
                        mk.state == CG_DEFINED ? 0xAAAAAAAAu : mk.state == CG_UNDEFINED ? 0xFFFFFFFFu : 0u);
      } else {
        fill_v(sv, y0 - sv.sb, y1 - sv.sb, mk.state == CG_DEFINED ? 0x00u : 0xFFu);
        put_abits(sv, y0 - sv.sb, y1 - sv.sb, mk.state != CG_NOACCESS);
      }
    }
  }
}

__global__ void k_setv_check(ShadowView sv, uint64_t addr, uint64_t len, uint32_t* __restrict__ flag) {
  pdl_entry();
  const uint64_t y0 = umax64(addr, sv.sb), y1 = umin64(addr + len, sv.se);
  for (uint64_t q = y0 - sv.sb + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < y1 - sv.sb;
       q += (uint64_t)gridDim.x * blockDim.x) {
    bool bad;
    if (sv.sparse) {
      const uint64_t c = q >> kChunkShift;
      const uint32_t sec = sparse_secondary(sv, c);
      bad = sec == 0 || ((reinterpret_cast<const uint32_t*>(chunk_base(sv, c, sec))[q >> 4] >> (2 * (q & 15))) & 3u) ==
                            kSt2NoAccess;
    } else if (sv.two_bit) {
      bad = ((reinterpret_cast<const uint32_t*>(sv.V)[q >> 4] >> (2 * (q & 15))) & 3u) == kSt2NoAccess;
    } else {
      bad = !((sv.A[q >> 3] >> (q & 7)) & 1);
    }
    if (bad) atomicOr(flag, 1u);
  }
}

// ---------------------------------------------------------------------------
// NEXT-4: ERROR SUMMARY counts: one diagnostic per set flag
// ---------------------------------------------------------------------------
__global__ void k_summary(const cg_verdict* __restrict__ v, uint64_t n, uint32_t warn_mask,
                          unsigned long long* __restrict__ counts) {
  pdl_entry();
  uint64_t e = 0, w = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t f = v[i].flags;
    e += __popc(f & ~warn_mask);
    w += __popc(f & warn_mask);
  }
  e = warp_sum(e);
  w = warp_sum(w);
  if ((threadIdx.x & 31) == 0 && (e | w)) {
    atomicAdd(counts, (unsigned long long)e);
    atomicAdd(counts + 1, (unsigned long long)w);
  }
}

// ---------------------------------------------------------------------------
// e: straddler exchange (descriptors whose host range spans several shards)
// ---------------------------------------------------------------------------
// Raw partials of m straddlers -> structure of arrays for three collectives:
// mins[2m] = {first_unaddr, first_undef}, sums[5m] = {undef_count, dst_expected,
// dst_found, src_expected, src_found} (only the owner shard has nonzero device
// fields), maxs[m] = flags (validation flags are identical on every shard and
// only the owner adds device flags, so MAX = OR here).
__global__ void k_straddler_pack(const cg_verdict* __restrict__ v, uint64_t m, uint64_t* __restrict__ mins,
                                 uint64_t* __restrict__ sums, uint32_t* __restrict__ maxs) {
  pdl_entry();
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const cg_verdict x = v[i];
    mins[i] = x.first_unaddr;
    mins[m + i] = x.first_undef;
    sums[i] = x.undef_count;
    sums[m + i] = x.dst_expected;
    sums[2 * m + i] = x.dst_found;
    sums[3 * m + i] = x.src_expected;
    sums[4 * m + i] = x.src_found;
    maxs[i] = x.flags;
  }
}

// merged fields -> final verdicts (a5 after the exchange)
__global__ void k_straddler_finalize(const uint64_t* __restrict__ mins, const uint64_t* __restrict__ sums,
                                     const uint32_t* __restrict__ maxs, uint64_t m, cg_verdict* __restrict__ v,
                                     uint32_t err_mask) {
  pdl_entry();
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    cg_verdict x;
    x.first_unaddr = mins[i];
    x.first_undef = mins[m + i];
    x.undef_count = sums[i];
    x.dst_expected = sums[m + i];
    x.dst_found = sums[2 * m + i];
    x.src_expected = sums[3 * m + i];
    x.src_found = sums[4 * m + i];
    x.flags = maxs[i];
    finalize_fields(x.flags, x.status, x.first_unaddr, x.undef_count, err_mask);
    v[i] = x;
  }
}

__global__ void k_expand_1d(const cg_copy1d* __restrict__ in, uint64_t n, cg_copy_desc* __restrict__ out) {
  pdl_entry();
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const cg_copy1d a = in[i];
    cg_copy_desc d;
    d.kind = a.kind;
    d.reserved = a.reserved;
    d.seq = a.seq;
    d.width = a.bytes;
    d.height = 1;
    d.dst = a.dst;
    d.dst_x = d.dst_y = 0;
    d.dst_pitch = a.bytes;
    d.src = a.src;
    d.src_x = d.src_y = 0;
    d.src_pitch = a.bytes;
    out[i] = d;
  }
}

// verdicts with any flag (order not kept) -> (index, verdict) lists for the
// gather to the root; clean verdicts are canonical and are not sent
__global__ void k_compact_dirty(const cg_verdict* __restrict__ v, uint64_t n, uint64_t* __restrict__ idx,
                                cg_verdict* __restrict__ dirty, uint32_t* __restrict__ count, uint64_t idx_base) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  for (uint64_t b0 = (uint64_t)blockIdx.x * blockDim.x; b0 < n; b0 += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = b0 + threadIdx.x;
    const bool d = i < n && v[i].flags != 0;
    const uint32_t mask = __ballot_sync(kFull, d);
    if (mask) {
      const int leader = __ffs(mask) - 1;
      uint32_t base = 0;
      if (lane == leader) base = atomicAdd(count, (uint32_t)__popc(mask));
      base = __shfl_sync(kFull, base, leader);
      if (d) {
        const uint32_t k = base + __popc(mask & ((1u << lane) - 1u));
        idx[k] = idx_base + i;
        dirty[k] = v[i];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// a8: leak sweep
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_live(Table t, uint64_t* __restrict__ weight) {
  pdl_entry();
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < t.n;
       i += (uint64_t)gridDim.x * blockDim.x)
    weight[i] = t.fseq[i] == kInf ? 1 : 0;
}

__global__ void __launch_bounds__(kThreads) k_leak_scatter(Table t, const uint64_t* __restrict__ P,
                                                           cg_alloc_record* __restrict__ out, uint64_t cap,
                                                           uint64_t* __restrict__ count) {
  pdl_entry();
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < t.n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (t.fseq[i] == kInf && P[i] < cap) {
      cg_alloc_record r;
      r.base = t.base[i];
      r.size = t.end[i] - t.base[i];
      r.alloc_seq = t.aseq[i];
      out[P[i]] = r;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *count = P[t.n];
}

// The whole sweep in one cooperative launch: block b counts the live entries of
// its contiguous slice [lo, hi), one grid barrier, then b's output offset is the
// sum of the counts of blocks < b and the slice is compacted in base order
// (k_live + prefix sum + k_leak_scatter without the 4 intermediate launches).
__global__ void __launch_bounds__(kThreads) k_leak(Table t, uint64_t* __restrict__ bsum,
                                                   cg_alloc_record* __restrict__ out, uint64_t cap,
                                                   uint64_t* __restrict__ count) {
  pdl_entry();
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  __shared__ uint64_t s_warp[33];
  const uint64_t n = t.n;
  const uint64_t per = (n + gridDim.x - 1) / gridDim.x;
  const uint64_t lo = umin64(n, (uint64_t)blockIdx.x * per), hi = umin64(n, lo + per);
  uint64_t total;
  {
    uint64_t acc = 0;
    for (uint64_t k = lo + threadIdx.x; k < hi; k += blockDim.x) acc += t.fseq[k] == kInf ? 1 : 0;
    block_exclusive_scan(acc, s_warp, total);
    if (threadIdx.x == 0) bsum[blockIdx.x] = total;
  }
  grid.sync();
  uint64_t part = 0;
  for (uint32_t j = threadIdx.x; j < blockIdx.x; j += blockDim.x) part += __ldcg(bsum + j);
  block_exclusive_scan(part, s_warp, total);
  uint64_t carry = total;
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) *count = carry + __ldcg(bsum + blockIdx.x);
  for (uint64_t k0 = lo; k0 < hi; k0 += blockDim.x) {
    const uint64_t k = k0 + threadIdx.x;
    const bool live = k < hi && t.fseq[k] == kInf;
    const uint64_t ex = block_exclusive_scan(live ? 1 : 0, s_warp, total);
    if (live && carry + ex < cap) {
      cg_alloc_record r;
      r.base = t.base[k];
      r.size = t.end[k] - t.base[k];
      r.alloc_seq = t.aseq[k];
      out[carry + ex] = r;
    }
    carry += total;
  }
}

inline int blocks_for(uint64_t n, int threads, int cap) {
  uint64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  return (int)(b < (uint64_t)cap ? b : (uint64_t)cap);
}

}  // namespace

// kernel launch with the programmatic-stream-serialization attribute (PDL)
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  static const bool pdl = [] {   // env CG_PDL=0: plain stream order (A/B measurements)
    const char* e = getenv("CG_PDL");
    return !(e && e[0] == '0');
  }();
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

uint64_t scan_blocks(uint64_t n) { return (n + kScanTile - 1) / kScanTile; }

// prefix sum of p.weight[0..n) into p.P[0..n], then the chunk plan
static cudaError_t plan(const Launch& L, uint64_t n, const Plan& p, cudaStream_t s,
                        const uint32_t* n_dev = nullptr) {
  const uint64_t nb = std::max<uint64_t>(scan_blocks(n), 1);
  launch_pdl(k_scan_reduce, (unsigned)nb, kScanThreads, 0, s, p.weight, n, p.bsum, n_dev);
  launch_pdl(k_scan_top, 1, 1024, 0, s, p.bsum, n, p.P, n_dev);
  launch_pdl(k_scan_down, (unsigned)nb, kScanThreads, 0, s, p.weight, n, p.bsum, p.P, n_dev);
  launch_pdl(k_plan, L.num_sms * 4, kThreads, 0, s, p.P, n, p.t_min, p.max_chunks, p.chunk_first, n_dev);
  *L.counter += 4;
  return cudaGetLastError();
}

// a1-a4: prep, plan and the shadow scan
static cudaError_t check_front(const Launch& L, const cg_copy_desc* d, uint64_t n, cg_verdict* out, const Table& t,
                        const ShadowView& sv, const Plan& p, uint32_t err_mask, int fuse, cudaStream_t s) {
  // fuse: 0 check only, 1 fused scan (cg_check_copies' fused form), 2 cg_check_apply
  // (k_finish runs the CG_CHECK_AFTER checks and the CG_APPLY_LAST applies)
  const size_t smem = ((size_t)t.nsplit + 1) * sizeof(uint64_t);
  ScanMeta* meta = reinterpret_cast<ScanMeta*>(p.meta);
  L.stage(CG_STAGE_CHECK_PREP, true, s);
  // prep + plan in one cooperative launch for batches of up to 4M descriptors;
  // above, the plan's per-block loops of the persistent grid are latency-bound
  // and the separate prep + scan + plan kernels are faster (C5, 10M: 1.05 ->
  // 0.99 ms)
  constexpr uint64_t kFrontCoopMax = 1ull << 22;
  if (L.front_blocks > 0 && smem <= kFrontSmem && n <= kFrontCoopMax) {
    const Table tc = t;
    ShadowView svc = sv;
    uint64_t* weight = p.weight;
    uint64_t* dvoff = p.dvoff;
    uint32_t* counter = p.counter;
    uint32_t* defer = p.defer;
    uint64_t* P = p.P;
    uint64_t* bsum = p.fbsum;
    uint64_t t_min = p.t_min, max_chunks = p.max_chunks;
    uint32_t* chunk_first = p.chunk_first;
    uint32_t em = err_mask;
    int fu = fuse;
    uint32_t* late = p.late;
    void* args[] = {(void*)&d, (void*)&n, (void*)&tc, (void*)&out, (void*)&weight, (void*)&meta, (void*)&dvoff,
                    (void*)&svc, (void*)&counter, (void*)&defer, (void*)&P, (void*)&bsum, (void*)&t_min,
                    (void*)&max_chunks, (void*)&chunk_first, (void*)&em, (void*)&fu, (void*)&late};
    const cudaError_t e =
        cudaLaunchCooperativeKernel((const void*)k_front, dim3((unsigned)L.front_blocks), dim3(kThreads), args, smem, s);
    *L.counter += 1;
    L.stage(CG_STAGE_CHECK_PREP, false, s);
    if (e != cudaSuccess) return e;   // nothing after it may consume a stale plan
  } else {
    launch_pdl(k_check_prep, blocks_for(n, kThreads, L.num_sms * 4), kThreads, smem, s, d, n, t, out, p.weight, meta,
               p.dvoff, sv, p.counter, p.defer, err_mask, fuse, p.late);
    *L.counter += 1;
    L.stage(CG_STAGE_CHECK_PREP, false, s);
    L.stage(CG_STAGE_CHECK_PLAN, true, s);
    plan(L, n, p, s);
    L.stage(CG_STAGE_CHECK_PLAN, false, s);
  }
  L.stage(CG_STAGE_CHECK_SCAN, true, s);
  if (sv.small_limit) {   // the small pass (k_check_small), then the ring scan
    launch_pdl(sv.two_bit ? k_check_small<true> : k_check_small<false>, L.small_blocks, kSmallThreads, 0, s, meta, n, sv,
               out, err_mask, fuse ? 1 : 0, p.resid, p.counter + 2, p.last);
    *L.counter += 1;
  }
  auto scan = !sv.two_bit ? (fuse ? k_check_scan<false, true, false> : k_check_scan<false, false, false>)
              : sv.sparse ? (fuse ? k_check_scan<true, true, true> : k_check_scan<true, false, true>)
                          : (fuse ? k_check_scan<true, true, false> : k_check_scan<true, false, false>);
  launch_pdl(scan, L.scan_blocks, kRingWarps * 32, kScanSmem, s, meta, n, p.P, p.chunk_first, p.counter, p.t_min,
             p.max_chunks, sv, out, err_mask, fuse ? 1 : 0, p.resid, p.counter + 2, d, p.defer, p.last);
  L.stage(CG_STAGE_CHECK_SCAN, false, s);
  *L.counter += 1;
  return cudaGetLastError();
}

cudaError_t check_copies(const Launch& L, const cg_copy_desc* d, uint64_t n, cg_verdict* out, const Table& t,
                         const ShadowView& sv, const Plan& p, uint32_t err_mask, bool fuse, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  cudaError_t e = check_front(L, d, n, out, t, sv, p, err_mask, fuse ? 1 : 0, s);
  if (e != cudaSuccess) return e;
  ScanMeta* meta = reinterpret_cast<ScanMeta*>(p.meta);
  L.stage(CG_STAGE_CHECK_FINAL, true, s);
  launch_pdl(k_finalize_split, blocks_for(n, kThreads, L.num_sms * 8), kThreads, 0, s, 
      n, p.P, p.t_min, p.max_chunks, out, err_mask, meta, fuse ? 1 : 0, p.resid, p.counter + 2, sv.small_share);
  L.stage(CG_STAGE_CHECK_FINAL, false, s);
  *L.counter += 1;
  return cudaGetLastError();
}

// cg_check_apply: the fused scan, then k_finish (finalise + residual apply)
cudaError_t check_apply(const Launch& L, const cg_copy_desc* d, uint64_t n, cg_verdict* out, const Table& t,
                        const ShadowView& sv, const Plan& p, uint32_t err_mask, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  cudaError_t e = check_front(L, d, n, out, t, sv, p, err_mask, 2, s);
  if (e != cudaSuccess) return e;
  L.stage(CG_STAGE_APPLY, true, s);
  ScanMeta* meta = reinterpret_cast<ScanMeta*>(p.meta);
  uint64_t* P = p.P;
  uint64_t t_min = p.t_min, max_chunks = p.max_chunks;
  uint32_t* resid = p.resid;
  uint32_t* counter = p.counter;
  uint64_t* weight = p.weight;
  uint64_t* bsum = p.fbsum;
  uint32_t* chunk_first = p.chunk_first;
  ShadowView svc = sv;
  const uint32_t* late = p.late;
  uint32_t* last = p.last;
  void* args[] = {(void*)&d, (void*)&n, (void*)&P, (void*)&t_min, (void*)&max_chunks, (void*)&out, (void*)&err_mask,
                  (void*)&meta, (void*)&resid, (void*)&counter, (void*)&weight, (void*)&bsum, (void*)&chunk_first,
                  (void*)&svc, (void*)&late, (void*)&last};
  e = cudaLaunchCooperativeKernel(sv.two_bit ? (const void*)k_finish<true> : (const void*)k_finish<false>,
                                              dim3((unsigned)L.finish_blocks), dim3(kThreads), args, 0, s);
  L.stage(CG_STAGE_APPLY, false, s);
  *L.counter += 1;
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t apply_dtoh(const Launch& L, const cg_copy_desc* d, const cg_verdict* v, uint64_t n,
                       const ShadowView& sv, const Plan& p, bool after_fused, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  ScanMeta* meta = reinterpret_cast<ScanMeta*>(p.meta);
  const uint32_t* n_dev = after_fused ? p.counter + 2 : nullptr;   // residual list count
  L.stage(CG_STAGE_APPLY_PREP, true, s);
  if (after_fused) {
    launch_pdl(k_apply_list_prep, L.num_sms * 2, kThreads, 0, s, d, p.resid, n_dev, p.weight, meta, p.counter);
  } else {
    cudaMemsetAsync(p.weight, 0, n * sizeof(uint64_t), s);
    cudaMemsetAsync(p.counter + 1, 0, sizeof(uint32_t), s);
    launch_pdl(k_apply_prep, blocks_for(n, kThreads, L.num_sms * 8), kThreads, 0, s, d, v, n, p.weight, meta,
                                                                             p.counter + 1);
  }
  *L.counter += 1;
  L.stage(CG_STAGE_APPLY_PREP, false, s);
  L.stage(CG_STAGE_APPLY_PLAN, true, s);
  cudaError_t e = plan(L, n, p, s, n_dev);
  if (e != cudaSuccess) return e;
  L.stage(CG_STAGE_APPLY_PLAN, false, s);
  L.stage(CG_STAGE_APPLY, true, s);
  if (!after_fused) cudaMemsetAsync(p.counter, 0, sizeof(uint32_t), s);
  launch_pdl(sv.two_bit ? k_apply<true> : k_apply<false>, L.persist_blocks, kThreads, 0, s, meta, n, p.P, p.chunk_first, p.counter, p.t_min, p.max_chunks, sv,
                                                n_dev);
  L.stage(CG_STAGE_APPLY, false, s);
  *L.counter += 1;
  return cudaGetLastError();
}

cudaError_t mark_batch(const Launch& L, const cg_mark* d_marks, uint64_t n, const ShadowView& sv, const Plan& p,
                       cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  launch_pdl(k_mark_prep, blocks_for(n, kThreads, L.num_sms * 8), kThreads, 0, s, d_marks, n, p.weight);
  *L.counter += 1;
  cudaError_t e = plan(L, n, p, s);
  if (e != cudaSuccess) return e;
  launch_pdl(k_mark, L.persist_blocks, kThreads, 0, s, d_marks, n, p.P, p.chunk_first, p.t_min, p.max_chunks, sv);
  *L.counter += 1;
  return cudaGetLastError();
}

cudaError_t summarize(const cg_verdict* v, uint64_t n, uint32_t warn_mask, unsigned long long* d_counts,
                      cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(d_counts, 0, 2 * sizeof(unsigned long long), s);
  if (e != cudaSuccess || n == 0) return e;
  launch_pdl(k_summary, (unsigned)std::min<uint64_t>((n + kThreads - 1) / kThreads, 148 * 8), kThreads, 0, s, v, n, warn_mask,
                                                                                               d_counts);
  return cudaGetLastError();
}

cudaError_t fresh_shadow(const Launch& L, const ShadowView& sv, cudaStream_t s) {
  if (sv.two_bit) {   // every state NOACCESS
    launch_pdl(k_fill, L.num_sms * 8, kThreads, 0, s, reinterpret_cast<uint4*>(sv.V), sv.v_bytes / 16, 0u);
    *L.counter += 1;
    return cudaGetLastError();
  }
  const uint64_t nv = (sv.se - sv.sb) / 16, na = (sv.se - sv.sb) / 128;
  launch_pdl(k_fill, L.num_sms * 8, kThreads, 0, s, reinterpret_cast<uint4*>(sv.V), nv, 0xffffffffu);
  if (na) launch_pdl(k_fill, L.num_sms * 8, kThreads, 0, s, reinterpret_cast<uint4*>(sv.A), na, 0u);
  *L.counter += 2;
  return cudaGetLastError();
}

cudaError_t setv_check(const Launch& L, uint64_t addr, uint64_t len, const ShadowView& sv, uint32_t* d_flag,
                       cudaStream_t s) {
  cudaMemsetAsync(d_flag, 0, sizeof(uint32_t), s);
  launch_pdl(k_setv_check, blocks_for(len, kThreads, L.num_sms * 4), kThreads, 0, s, sv, addr, len, d_flag);
  *L.counter += 1;
  return cudaGetLastError();
}

cudaError_t leak_sweep(const Launch& L, const Table& t, const Plan& p, cg_alloc_record* out, uint64_t cap,
                       uint64_t* d_count, cudaStream_t s) {
  if (t.n == 0) return cudaMemsetAsync(d_count, 0, sizeof(uint64_t), s);
  L.stage(CG_STAGE_LEAK, true, s);
  if (L.leak_blocks > 0) {   // one cooperative launch
    Table tc = t;
    uint64_t* bsum = p.fbsum;
    void* args[] = {(void*)&tc, (void*)&bsum, (void*)&out, (void*)&cap, (void*)&d_count};
    const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)L.leak_blocks,
                                                                          (t.n + kThreads - 1) / kThreads));
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_leak, dim3(g), dim3(kThreads), args, 0, s);
    L.stage(CG_STAGE_LEAK, false, s);
    *L.counter += 1;
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
  }
  launch_pdl(k_live, blocks_for(t.n, kThreads, L.num_sms * 8), kThreads, 0, s, t, p.weight);
  const uint64_t nb = scan_blocks(t.n);
  launch_pdl(k_scan_reduce, (unsigned)nb, kScanThreads, 0, s, p.weight, t.n, p.bsum, nullptr);
  launch_pdl(k_scan_top, 1, 1024, 0, s, p.bsum, t.n, p.P, nullptr);
  launch_pdl(k_scan_down, (unsigned)nb, kScanThreads, 0, s, p.weight, t.n, p.bsum, p.P, nullptr);
  launch_pdl(k_leak_scatter, blocks_for(t.n, kThreads, L.num_sms * 8), kThreads, 0, s, t, p.P, out, cap, d_count);
  L.stage(CG_STAGE_LEAK, false, s);
  *L.counter += 5;
  return cudaGetLastError();
}

cudaError_t straddler_pack(const Launch& L, const cg_verdict* v, uint64_t m, uint64_t* mins, uint64_t* sums,
                           uint32_t* maxs, cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  launch_pdl(k_straddler_pack, blocks_for(m, kThreads, L.num_sms * 8), kThreads, 0, s, v, m, mins, sums, maxs);
  *L.counter += 1;
  return cudaGetLastError();
}

cudaError_t straddler_finalize(const Launch& L, const uint64_t* mins, const uint64_t* sums, const uint32_t* maxs,
                               uint64_t m, cg_verdict* v, uint32_t err_mask, cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  launch_pdl(k_straddler_finalize, blocks_for(m, kThreads, L.num_sms * 8), kThreads, 0, s, mins, sums, maxs, m, v,
                                                                                    err_mask);
  *L.counter += 1;
  return cudaGetLastError();
}

cudaError_t compact_dirty(const Launch& L, const cg_verdict* v, uint64_t n, uint64_t* idx, cg_verdict* dirty,
                          uint32_t* count, uint64_t idx_base, bool reset, cudaStream_t s) {
  if (reset) cudaMemsetAsync(count, 0, sizeof(uint32_t), s);
  if (n == 0) return cudaGetLastError();
  launch_pdl(k_compact_dirty, blocks_for(n, kThreads, L.num_sms * 8), kThreads, 0, s, v, n, idx, dirty, count, idx_base);
  *L.counter += 1;
  return cudaGetLastError();
}

cudaError_t expand_1d(const Launch& L, const cg_copy1d* in, uint64_t n, cg_copy_desc* out, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  launch_pdl(k_expand_1d, blocks_for(n, kThreads, L.num_sms * 8), kThreads, 0, s, in, n, out);
  *L.counter += 1;
  return cudaGetLastError();
}

cudaError_t propagate(const Launch& L, const cg_copy_desc* d, const cg_verdict* v, const uint32_t* index, uint64_t n,
                      const ShadowView& sv, uint8_t* pool, const Plan& p, uint8_t* scratch, uint32_t* overflow,
                      cudaStream_t s, bool reset_overflow) {
  if (n == 0) return cudaSuccess;
  PropMeta* pm = reinterpret_cast<PropMeta*>(p.meta);   // 48 B per item: the meta area holds max_descs of them
  uint32_t* cnt = p.counter + 1;
  uint32_t* mm_count = p.counter + 3;
  cudaMemsetAsync(p.weight, 0, n * sizeof(uint64_t), s);
  cudaMemsetAsync(p.counter, 0, 4 * sizeof(uint32_t), s);
  if (reset_overflow) cudaMemsetAsync(overflow, 0, sizeof(uint32_t), s);
  L.stage(CG_STAGE_APPLY_PREP, true, s);
  launch_pdl(k_prop_prep, blocks_for(n, kThreads, L.num_sms * 8), kThreads, 0, s, d, v, index, n, p.dvoff, sv.sb, p.weight, pm,
                                                                          cnt, p.resid, mm_count);
  L.stage(CG_STAGE_APPLY_PREP, false, s);
  L.stage(CG_STAGE_APPLY_PLAN, true, s);
  cudaError_t e = plan(L, n, p, s, cnt);
  if (e != cudaSuccess) return e;
  L.stage(CG_STAGE_APPLY_PLAN, false, s);
  L.stage(CG_STAGE_APPLY, true, s);
  cudaMemsetAsync(p.counter, 0, sizeof(uint32_t), s);
  launch_pdl(k_propagate, L.persist_blocks, kThreads, 0, s, pm, n, p.P, p.chunk_first, p.counter, p.t_min, p.max_chunks,
                                                    sv.V, pool, cnt);
  launch_pdl(k_memmove, 64, kThreads, 0, s, d, p.dvoff, p.resid, mm_count, pool, scratch, overflow, kStageBytes);
  L.stage(CG_STAGE_APPLY, false, s);
  *L.counter += 3;
  return cudaGetLastError();
}

cudaError_t propagate_direct(const Launch& L, const cg_copy_desc* d, const cg_verdict* v, const uint32_t* index,
                             uint64_t m, uint64_t max_bytes, const ShadowView& sv, uint8_t* pool, const Plan& p,
                             uint8_t* scratch, uint32_t* overflow, cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  uint32_t* mm_count = p.counter + 3;
  cudaMemsetAsync(mm_count, 0, sizeof(uint32_t), s);
  L.stage(CG_STAGE_APPLY, true, s);
  const uint64_t slices = std::max<uint64_t>(1, (max_bytes + kDirectSlice - 1) / kDirectSlice);
  if (m * slices > (uint64_t)L.num_sms * 512) {   // very many copies: a warp each
    launch_pdl(k_prop_direct_warp, blocks_for(m * 32, kThreads, 1 << 20), kThreads, 0, s, d, v, index, m, p.dvoff, sv.sb,
                                                                                   sv.V, pool, p.resid, mm_count);
  } else {   // CTA slices keep the larger copies of the later waves streaming
    launch_pdl(k_prop_direct, dim3((unsigned)m, (unsigned)slices), kThreads, 0, s, d, v, index, m, p.dvoff, sv.sb, sv.V, pool,
                                                                          p.resid, mm_count);
  }
  launch_pdl(k_memmove, 64, kThreads, 0, s, d, p.dvoff, p.resid, mm_count, pool, scratch, overflow, kStageBytes);
  L.stage(CG_STAGE_APPLY, false, s);
  *L.counter += 2;
  return cudaGetLastError();
}

cudaError_t propagate_waves(const Launch& L, const cg_copy_desc* d, const cg_verdict* v, const uint32_t* index,
                            uint64_t m, const uint32_t* d_wstart, uint32_t n_waves, const ShadowView& sv,
                            uint8_t* pool, const Plan& p, uint8_t* scratch, uint32_t* overflow, cudaStream_t s) {
  if (m == 0 || n_waves == 0) return cudaSuccess;
  PropMeta* pm = reinterpret_cast<PropMeta*>(p.meta);
  uint32_t* mm_count = p.counter + 3;
  cudaMemsetAsync(mm_count, 0, sizeof(uint32_t), s);
  L.stage(CG_STAGE_APPLY_PREP, true, s);
  static const uint64_t item_cost = [] {
    const char* e = getenv("CG_WAVE_COST");
    return e ? (uint64_t)atoll(e) : kWaveItemCost;
  }();
  static const uint64_t min_piece = [] {
    const char* e = getenv("CG_WAVE_PIECE");
    return e ? std::max<uint64_t>((uint64_t)atoll(e), 1) : kWaveMinPiece;
  }();
  launch_pdl(k_wave_prep, blocks_for(m, kThreads, L.num_sms * 8), kThreads, 0, s, d, v, index, m, p.dvoff, sv.sb, p.weight,
                                                                          pm, p.resid, mm_count, item_cost);
  L.stage(CG_STAGE_APPLY_PREP, false, s);
  L.stage(CG_STAGE_APPLY_PLAN, true, s);
  const uint64_t nb = std::max<uint64_t>(scan_blocks(m), 1);
  launch_pdl(k_scan_reduce, (unsigned)nb, kScanThreads, 0, s, p.weight, m, p.bsum, nullptr);
  launch_pdl(k_scan_top, 1, 1024, 0, s, p.bsum, m, p.P, nullptr);
  launch_pdl(k_scan_down, (unsigned)nb, kScanThreads, 0, s, p.weight, m, p.bsum, p.P, nullptr);
  L.stage(CG_STAGE_APPLY_PLAN, false, s);
  L.stage(CG_STAGE_APPLY, true, s);
  uint8_t* V = sv.V;
  const uint64_t* P = p.P;
  const uint64_t* dvoff = p.dvoff;
  const uint32_t* mm = p.resid;
  const uint32_t* mmc = mm_count;
  uint64_t ic = item_cost, mp = min_piece;
  void* args[] = {(void*)&d, (void*)&index, (void*)&pm, (void*)&P, (void*)&d_wstart, (void*)&n_waves, (void*)&V,
                  (void*)&pool, (void*)&dvoff, (void*)&mm, (void*)&mmc, (void*)&scratch, (void*)&overflow, (void*)&ic,
                  (void*)&mp};
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_prop_waves, dim3((unsigned)L.wave_blocks),
                                              dim3(kWRing * 32), args, kWaveSmem, s);
  L.stage(CG_STAGE_APPLY, false, s);
  *L.counter += 5;
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// the recovery pass of the self-overlapping 2D DtoDs the staging area could
// not hold (block_memmove's overflow list): staged through `scratch` of
// stage_cap bytes, after the rest of their batch / wave
cudaError_t memmove_list(const Launch& L, const cg_copy_desc* d, const uint64_t* dvoff, const uint32_t* list,
                         const uint32_t* count, uint8_t* pool, uint8_t* scratch, uint64_t stage_cap,
                         uint32_t* overflow, cudaStream_t s) {
  launch_pdl(k_memmove, 64, kThreads, 0, s, d, dvoff, list, count, pool, scratch, overflow, stage_cap);
  *L.counter += 1;
  return cudaGetLastError();
}

// the free stamps of a registry diff upload: pairs (position, free seq) ->
// fseq column and the walk record (prefix max, end, alloc seq, free seq)
__global__ void k_table_patch(uint64_t* __restrict__ fseq, uint64_t* __restrict__ walk,
                              const uint64_t* __restrict__ pairs, uint64_t k) {
  pdl_entry();
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t pos = pairs[2 * i], f = pairs[2 * i + 1];
    fseq[pos] = f;
    walk[4 * pos + 3] = f;
  }
}

cudaError_t table_patch(const Launch& L, uint64_t* fseq, uint64_t* walk, const uint64_t* d_pairs, uint64_t k,
                        cudaStream_t s) {
  launch_pdl(k_table_patch, blocks_for(k, kThreads, L.num_sms * 4), kThreads, 0, s, fseq, walk, d_pairs, k);
  *L.counter += 1;
  return cudaGetLastError();
}

size_t prop_meta_bytes() { return sizeof(PropMeta); }
uint64_t stage_bytes() { return kStageBytes; }

int persistent_blocks(int which) {
  int b = 0;
  if (which == 0) {
    b = 1 << 20;
    for (auto k : {k_check_scan<false, false, false>, k_check_scan<false, true, false>,
                   k_check_scan<true, false, false>, k_check_scan<true, true, false>, k_check_scan<true, false, true>,
                   k_check_scan<true, true, true>}) {
      int bk = 0;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kScanSmem);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bk, k, kRingWarps * 32, kScanSmem);
      b = std::min(b, bk);
    }
  } else if (which == 4) {   // k_front with the largest splitter array (4097 words)
    cudaFuncSetAttribute(k_front, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFrontSmem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_front, kThreads, kFrontSmem);
  } else if (which == 5) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_leak, kThreads, 0);
  } else if (which == 6) {
    int b2 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_check_small<false>, kSmallThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b2, k_check_small<true>, kSmallThreads, 0);
    b = std::min(b, b2);
  } else if (which == 3) {
    int b2 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_finish<false>, kThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b2, k_finish<true>, kThreads, 0);
    b = std::min(b, b2);
  } else if (which == 1) {
    // the bytes-format instantiation sizes the persistent grid (extra CTAs of
    // the 2-bit one just find the group counter exhausted)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_apply<false>, kThreads, 0);
  } else {
    cudaFuncSetAttribute(k_prop_waves, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kWaveSmem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_prop_waves, kWRing * 32, kWaveSmem);
  }
  return b;
}

size_t scan_meta_bytes() { return sizeof(ScanMeta); }

}  // namespace cgk
