// NEXT-2: concurrency hazards ("certain concurrent
// accesses when several threads are used"; SPEC check_concurrent S:258-266
// with the rule of S:285; readings R-31..R-35).
//
// A copy's access (one side, one address space) is a ConcurrentHazard iff the
// most recent earlier recorded access overlapping it belongs to another thread
// that has not synchronised since, and one of the two writes.
//
// Batched, exact and order-free on the GPU.  Per address space (host, device)
// the state between calls is the last-access map H: disjoint byte ranges, each
// tagged with the stamp that touched it last, sorted by stamp seq.  A batch of
// n copies (seq order) turns into query accesses Q (every valid side) and
// recorded accesses R = H + the sides of copies without an Error.  Every
// stamp p gets a unique key = 2*ord(p) + is_write, ord = index in seq order
// (H first, then the batch), so "p is earlier than q" is key_p < 2*ord_q and
// the newest overlapping stamp is the largest such key.  p overlaps q iff
//   (A) s_q <= s_p < e_q   -- a range query over R sorted by start: a merge-sort
//                              tree (level L: blocks of 2^L starts sorted by key),
//                              predecessor search per block;
//   (B) s_p <= s_q < e_p   -- a stabbing query at s_q: a segment tree over the
//                              elementary intervals of R's endpoints whose nodes
//                              hold the keys of the ranges they canonically cover.
// The new map is the winner (largest key) of every elementary interval, runs
// merged, re-sorted by key.  Cost per batch: O((|R| + |Q|) log^2) with sorts
// (cub radix sort) and one thread per query; no data-dependent serialisation.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <string>
#include <utility>
#include <vector>

#include "cg_internal.h"

namespace {

constexpr int kT = 256;
constexpr uint32_t kNoKey = 0xffffffffu;

inline unsigned grid_for(uint64_t n) { return (unsigned)std::max<uint64_t>(1, (n + kT - 1) / kT); }

__device__ __forceinline__ uint64_t lower_bound64(const uint64_t* a, uint64_t n, uint64_t x) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// largest element < lim of the ascending u32 array a[0, n), or kNoKey
__device__ __forceinline__ uint32_t pred32(const uint32_t* a, uint64_t n, uint32_t lim) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (a[mid] < lim) lo = mid + 1; else hi = mid;
  }
  return lo ? a[lo - 1] : kNoKey;
}

// the same over the keys of (node << kb | key) pairs of one node list
__device__ __forceinline__ uint32_t pred_pairs(const uint64_t* a, uint64_t b, uint64_t e, uint32_t lim, uint64_t kmask) {
  uint64_t lo = b, hi = e;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if ((uint32_t)(a[mid] & kmask) < lim) lo = mid + 1; else hi = mid;
  }
  return lo > b ? (uint32_t)(a[lo - 1] & kmask) : kNoKey;
}

__device__ __forceinline__ uint64_t warp_min64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w < v ? w : v;
  }
  return v;
}
__device__ __forceinline__ uint64_t warp_max64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}


__device__ __forceinline__ uint32_t kmax(uint32_t a, uint32_t b) {
  return a == kNoKey ? b : b == kNoKey ? a : (a > b ? a : b);
}

struct Space {            // one address space's arrays (device pointers)
  // last-access map (history), sorted by seq; double-buffered
  uint64_t *hs, *he, *hseq;
  uint32_t *hthr;
  uint8_t *hw;
  // queries
  uint64_t *qs, *qe;
  uint32_t *qkey, *qcopy;
  // recorded ranges (history first, then the batch)
  uint64_t *rs, *re;
  uint32_t *rkey;
};

// R-32: the accesses of one copy kind -> (space, side is dst, is_write)
__device__ __forceinline__ int copy_accesses(uint32_t kind, int sp[2], int dst[2], int wr[2]) {
  switch (kind) {
    case CG_HTOD: sp[0] = 0; dst[0] = 0; wr[0] = 0; sp[1] = 1; dst[1] = 1; wr[1] = 1; return 2;
    case CG_DTOH: sp[0] = 1; dst[0] = 0; wr[0] = 0; sp[1] = 0; dst[1] = 1; wr[1] = 1; return 2;
    case CG_DTOD: sp[0] = 1; dst[0] = 0; wr[0] = 0; sp[1] = 1; dst[1] = 1; wr[1] = 1; return 2;
    case CG_HTOA: sp[0] = 0; dst[0] = 0; wr[0] = 0; return 1;
    case CG_ATOH: sp[0] = 0; dst[0] = 1; wr[0] = 1; return 1;
    default: return 0;
  }
}



// block-level aggregation of the per-space key ranges: one atomic per block and value
__device__ __forceinline__ void block_range(unsigned long long* counts, const uint64_t mn[2], const uint64_t mx[2]) {
  __shared__ uint64_t red[kT / 32][4];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint64_t v[4] = {warp_min64(mn[0]), warp_max64(mx[0]), warp_min64(mn[1]), warp_max64(mx[1])};
  if (lane == 0)
    for (int k = 0; k < 4; ++k) red[w][k] = v[k];
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int j = 1; j < (int)(blockDim.x >> 5); ++j) {
      v[0] = min(v[0], red[j][0]);
      v[1] = max(v[1], red[j][1]);
      v[2] = min(v[2], red[j][2]);
      v[3] = max(v[3], red[j][3]);
    }
    for (int sp = 0; sp < 2; ++sp)
      if (v[2 * sp] <= v[2 * sp + 1]) {
        atomicMin(counts + 8 + 2 * sp, (unsigned long long)v[2 * sp]);
        atomicMax(counts + 9 + 2 * sp, (unsigned long long)v[2 * sp + 1]);
      }
  }
}

__global__ void __launch_bounds__(kT) k_hist_to_r(Space S0, Space S1, uint64_t nh0, uint64_t nh1,
                                                  unsigned long long* counts) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t mn[2] = {~0ull, ~0ull}, mx[2] = {0, 0};
  if (i < nh0) {
    S0.rs[i] = mn[0] = S0.hs[i];
    S0.re[i] = mx[0] = S0.he[i];
    S0.rkey[i] = 2u * (uint32_t)i + S0.hw[i];
  }
  if (i < nh1) {
    S1.rs[i] = mn[1] = S1.hs[i];
    S1.re[i] = mx[1] = S1.he[i];
    S1.rkey[i] = 2u * (uint32_t)i + S1.hw[i];
  }
  block_range(counts, mn, mx);
}

// one thread per copy: its accesses become queries; performed copies' accesses
// are appended to R (R-33, R-34).  Slots come from one block-wide exclusive
// scan of the four packed counters and one atomic per block and counter.
// counts: [qn0, qn1, rn0, rn1, ...]
__global__ void __launch_bounds__(kT) k_access(const cg_copy_desc* __restrict__ d, const cg_verdict* __restrict__ v,
                                               uint64_t n, Space S0, Space S1, uint64_t nh0, uint64_t nh1,
                                               unsigned long long* counts) {
  using Scan = cub::BlockScan<unsigned long long, kT>;
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ unsigned long long s_base[4];
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  int sp[2] = {0, 0}, dst[2] = {0, 0}, wr[2] = {0, 0};
  bool ok[2] = {false, false}, performed = false;
  uint64_t st[2] = {0, 0}, sn[2] = {0, 0};
  if (i < n) {
    const cg_copy_desc c = d[i];
    const int na = copy_accesses(c.kind, sp, dst, wr);
    performed = v[i].status == CG_OK;
    // the contract: seqs strictly increase inside the batch (counts[12] flags a violation)
    if (i > 0 && d[i - 1].seq >= c.seq) atomicOr(counts + 12, 1ull);
    if (i == 0) counts[13] = c.seq;       // the batch's first seq, checked against the previous batch
    if (i + 1 == n) counts[14] = c.seq;   // and its last
    for (int k = 0; k < na; ++k) {
      ok[k] = dst[k] ? cgk::fold_side(c.dst, c.dst_x, c.dst_y, c.dst_pitch, c.width, c.height, st[k], sn[k])
                     : cgk::fold_side(c.src, c.src_x, c.src_y, c.src_pitch, c.width, c.height, st[k], sn[k]);
      ok[k] = ok[k] && sn[k] != 0;
    }
  }
  // packed 16-bit counters: queries of space 0 / 1, recorded of space 0 / 1 (<= 2 each per thread)
  unsigned long long mine = 0;
  uint64_t mn[2] = {~0ull, ~0ull}, mx[2] = {0, 0};
  for (int k = 0; k < 2; ++k) {
    if (!ok[k]) continue;
    mine += 1ull << (16 * sp[k]);
    if (performed) {
      mine += 1ull << (16 * (2 + sp[k]));
      mn[sp[k]] = min(mn[sp[k]], st[k]);
      mx[sp[k]] = max(mx[sp[k]], st[k] + sn[k]);
    }
  }
  unsigned long long pre, tot;
  Scan(scan_tmp).ExclusiveSum(mine, pre, tot);
  if (threadIdx.x == 0)
    for (int c = 0; c < 4; ++c) {
      const unsigned long long t = (tot >> (16 * c)) & 0xffffull;
      s_base[c] = t ? atomicAdd(counts + c, t) : 0ull;
    }
  block_range(counts, mn, mx);   // contains the __syncthreads that publishes s_base
  unsigned long long q[2] = {s_base[0] + (pre & 0xffffull), s_base[1] + ((pre >> 16) & 0xffffull)};
  unsigned long long r[2] = {s_base[2] + ((pre >> 32) & 0xffffull), s_base[3] + ((pre >> 48) & 0xffffull)};
  for (int k = 0; k < 2; ++k) {
    if (!ok[k]) continue;
    const int space = sp[k];
    Space& S = space ? S1 : S0;
    const uint64_t nh = space ? nh1 : nh0;
    const uint32_t key = 2u * (uint32_t)(nh + i) + (uint32_t)wr[k];
    const unsigned long long qq = q[space]++;
    S.qs[qq] = st[k];
    S.qe[qq] = st[k] + sn[k];
    S.qkey[qq] = key;
    S.qcopy[qq] = (uint32_t)i;
    if (performed) {
      const unsigned long long rr = nh + r[space]++;
      S.rs[rr] = st[k];
      S.re[rr] = st[k] + sn[k];
      S.rkey[rr] = key;
    }
  }
}

// merge-sort tree: level L from level L-1 (blocks of 2^(L-1) sorted keys, pairwise merged)
__global__ void k_merge_level(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, uint64_t n, int L) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t half = 1ull << (L - 1);
  const uint64_t b = i >> (L - 1), sib = b ^ 1ull;
  const uint64_t r = i - (b << (L - 1));
  const uint64_t s0 = sib << (L - 1);
  const uint32_t key = in[i];
  uint64_t c = 0;
  if (s0 < n) {   // keys are unique: position = own rank + sibling keys below it
    const uint64_t s1 = s0 + half < n ? s0 + half : n;
    uint64_t lo = s0, hi = s1;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (in[mid] < key) lo = mid + 1; else hi = mid;
    }
    c = lo - s0;
  }
  out[(((b < sib) ? b : sib) << (L - 1)) + r + c] = key;
}

// keys of the sorted run [s0, min(s0 + h, n)) below key (0 if the run is empty)
__device__ __forceinline__ uint64_t count_below(const uint32_t* __restrict__ in, uint64_t s0, uint64_t h, uint64_t n,
                                                uint32_t key) {
  if (s0 >= n) return 0;
  uint64_t lo = s0, hi = s0 + h < n ? s0 + h : n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (in[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo - s0;
}

// levels L and L+1 at once from level L-1 (runs of h = 2^(L-1)): an element's
// place among its 2 and its 4 runs
__global__ void k_merge_2levels(const uint32_t* __restrict__ in, uint32_t* __restrict__ outL,
                                uint32_t* __restrict__ outL1, uint64_t n, int L) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int sh = L - 1;
  const uint64_t h = 1ull << sh, b = i >> sh, r = i - (b << sh), key_b = b;
  const uint32_t key = in[i];
  const uint64_t sib = key_b ^ 1ull, q0 = key_b & ~3ull, other = (key_b & 2ull) ? q0 : q0 + 2;
  const uint64_t c1 = count_below(in, sib << sh, h, n, key);
  const uint64_t c2 = count_below(in, other << sh, h, n, key) + count_below(in, (other + 1) << sh, h, n, key);
  outL[((b & ~1ull) << sh) + r + c1] = key;
  outL1[(q0 << sh) + r + c1 + c2] = key;
}

// levels 1..kSmemLevels of the merge-sort tree for one 2^kSmemLevels tile in shared memory
constexpr int kSmemLevels = 8;
__global__ void __launch_bounds__(1 << kSmemLevels) k_merge_tile(uint32_t* __restrict__ mst, uint64_t n, uint64_t cap,
                                                                 int levels) {
  __shared__ uint32_t buf[2][1 << kSmemLevels];
  const uint32_t t = threadIdx.x;
  const uint64_t base = (uint64_t)blockIdx.x << kSmemLevels;
  const uint32_t m = (uint32_t)min((uint64_t)1 << kSmemLevels, n - base);   // valid keys of this tile
  if (t < m) buf[0][t] = mst[base + t];
  __syncthreads();
  int cur = 0;
  for (int L = 1; L <= levels; ++L) {
    if (t < m) {
      const uint32_t half = 1u << (L - 1);
      const uint32_t b = t >> (L - 1), sib = b ^ 1u, r = t - (b << (L - 1)), s0 = sib << (L - 1);
      const uint32_t key = buf[cur][t];
      uint32_t c = 0;
      if (s0 < m) {
        uint32_t lo = s0, hi = min(s0 + half, m);
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (buf[cur][mid] < key) lo = mid + 1; else hi = mid;
        }
        c = lo - s0;
      }
      const uint32_t o = (min(b, sib) << (L - 1)) + r + c;
      buf[cur ^ 1][o] = key;
      mst[(uint64_t)L * cap + base + o] = key;
    }
    cur ^= 1;
    __syncthreads();
  }
}

__global__ void k_endpoints(const uint64_t* __restrict__ rs, const uint64_t* __restrict__ re, uint64_t n,
                            uint64_t* __restrict__ ep) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < n) { ep[2 * i] = rs[i]; ep[2 * i + 1] = re[i]; }
}

__device__ __forceinline__ void leaf_range(const uint64_t* coords, uint64_t m, uint64_t s, uint64_t e,
                                           uint64_t& l, uint64_t& r) {
  l = lower_bound64(coords, m, s);
  r = lower_bound64(coords, m, e);   // both are endpoints, so exact ranks
}

__global__ void k_cover_count(const uint64_t* __restrict__ rs, const uint64_t* __restrict__ re, uint64_t n,
                              const uint64_t* __restrict__ coords, const unsigned long long* __restrict__ m_dev,
                              uint64_t M, uint32_t* __restrict__ cnt, uint64_t* __restrict__ lr) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t l, r;
  leaf_range(coords, *m_dev, rs[i], re[i], l, r);
  lr[i] = (l << 32) | r;   // reused by k_cover_emit
  uint32_t k = 0;
  for (l += M, r += M; l < r; l >>= 1, r >>= 1) {
    if (l & 1) { ++k; ++l; }
    if (r & 1) { ++k; --r; }
  }
  cnt[i] = k;
}

__global__ void k_cover_emit(const uint64_t* __restrict__ lr, const uint32_t* __restrict__ rkey, uint64_t n,
                             uint64_t M, const uint32_t* __restrict__ off, uint64_t* __restrict__ pairs, int kb) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t l = lr[i] >> 32, r = lr[i] & 0xffffffffull;
  uint64_t o = off[i];
  const uint64_t key = rkey[i];
  for (l += M, r += M; l < r; l >>= 1, r >>= 1) {
    if (l & 1) pairs[o++] = (l++ << kb) | key;
    if (r & 1) pairs[o++] = (--r << kb) | key;
  }
}

// node list offsets: off(v) = first pair with node >= v.  The first pair of
// every node list is scattered to rev[nodes - node] (rev pre-filled with P),
// then an inclusive min-scan over rev fills the empty nodes: off(v) = scanned[nodes - v]
__global__ void k_fill_u32(uint32_t* __restrict__ a, uint64_t n, uint32_t val) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < n) a[i] = val;
}
__global__ void k_node_starts(const uint64_t* __restrict__ pairs, uint64_t P, int kb, uint64_t nodes,
                              uint32_t* __restrict__ rev) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= P) return;
  const uint64_t node = pairs[i] >> kb;
  if (i == 0 || (pairs[i - 1] >> kb) != node) rev[nodes - node] = (uint32_t)i;
}
struct MinU32 {
  __device__ __forceinline__ uint32_t operator()(uint32_t a, uint32_t b) const { return a < b ? a : b; }
};

struct Syncs {
  const uint32_t* thr;   // sorted by (thread, seq)
  const uint64_t* seq;
  uint64_t n;
};

// R-31: thread t synchronised after its stamp at seq a and before seq b
__device__ __forceinline__ bool synced(const Syncs& sy, uint32_t t, uint64_t a, uint64_t b) {
  uint64_t lo = 0, hi = sy.n;   // first (thread, seq) > (t, a)
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    const uint32_t mt = sy.thr[mid];
    if (mt < t || (mt == t && sy.seq[mid] <= a)) lo = mid + 1; else hi = mid;
  }
  return lo < sy.n && sy.thr[lo] == t && sy.seq[lo] < b;
}

struct Tree {
  const uint64_t* rs_sorted;   // R starts, ascending
  const uint32_t* mst;         // (levels) x cap keys
  uint64_t cap, rn;
  int levels;
  const uint64_t* coords;
  const unsigned long long* m_dev;
  const uint32_t* noff;   // reversed: the offset of node v is noff[nodes - v]
  uint64_t nodes;
  const uint64_t* pairs;
  uint64_t M;
  uint64_t kmask;   // key bits of a pair (node << kb | key)
};

__device__ uint32_t newest_overlap(const Tree& T, uint64_t s, uint64_t e, uint32_t lim) {
  uint32_t best = kNoKey;
  // (A) ranges starting inside [s, e)
  uint64_t a = lower_bound64(T.rs_sorted, T.rn, s), b = lower_bound64(T.rs_sorted, T.rn, e);
  for (int L = 0; a < b; ++L, a >>= 1, b >>= 1) {
    const uint32_t* lvl = T.mst + (uint64_t)L * T.cap;
    if (a & 1) {
      const uint64_t b0 = a << L, b1 = min((a + 1) << L, T.rn);
      best = kmax(best, pred32(lvl + b0, b1 - b0, lim));
      ++a;
    }
    if (b & 1) {
      --b;
      const uint64_t b0 = b << L, b1 = min((b + 1) << L, T.rn);
      best = kmax(best, pred32(lvl + b0, b1 - b0, lim));
    }
  }
  // (B) ranges covering s
  const uint64_t m = *T.m_dev;
  const uint64_t k1 = lower_bound64(T.coords, m, s + 1);   // coords[k] <= s < coords[k+1]
  if (k1 > 0 && k1 < m) {
    for (uint64_t v = T.M + (k1 - 1); v >= 1; v >>= 1)
      best = kmax(best, pred_pairs(T.pairs, T.noff[T.nodes - v], T.noff[T.nodes - v - 1], lim, T.kmask));
  }
  return best;
}

struct Stamps {   // winner lookup: key -> (thread, seq)
  const uint32_t* hthr;
  const uint64_t* hseq;
  uint64_t nh;
  const cg_copy_desc* d;
  const uint32_t* threads;
};

__device__ __forceinline__ void stamp_of(const Stamps& st, uint32_t key, uint32_t& thr, uint64_t& seq) {
  const uint64_t ord = key >> 1;
  if (ord < st.nh) { thr = st.hthr[ord]; seq = st.hseq[ord]; }
  else { thr = st.threads[ord - st.nh]; seq = st.d[ord - st.nh].seq; }
}

__global__ void k_query(Space S, uint64_t qn, Tree T, Stamps st, Syncs sy, cg_verdict* __restrict__ v) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= qn) return;
  const uint32_t qkey = S.qkey[i];
  const uint32_t best = newest_overlap(T, S.qs[i], S.qe[i], qkey & ~1u);
  if (best == kNoKey) return;
  uint32_t pt, qt;
  uint64_t ps, qs;
  stamp_of(st, best, pt, ps);
  stamp_of(st, qkey, qt, qs);
  if (pt != qt && !synced(sy, pt, ps, qs) && ((best | qkey) & 1u))
    atomicOr(&v[S.qcopy[i]].flags, (uint32_t)CG_F_CONCURRENT);
}

// winner of every elementary interval [coords[k], coords[k+1]) and run flags
__global__ void k_winners(Tree T, uint32_t* __restrict__ win) {
  const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t m = *T.m_dev;
  if (k + 1 >= m) return;
  uint32_t best = kNoKey;
  for (uint64_t v = T.M + k; v >= 1; v >>= 1) {
    const uint32_t b = T.noff[T.nodes - v], e = T.noff[T.nodes - v - 1];
    if (e > b) best = kmax(best, (uint32_t)(T.pairs[e - 1] & T.kmask));
  }
  win[k] = best;
}

__global__ void k_run_flags(const uint32_t* __restrict__ win, const unsigned long long* __restrict__ m_dev,
                            uint64_t cap, uint32_t* __restrict__ start) {
  const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (k >= cap) return;
  const uint64_t m = *m_dev;
  start[k] = (k + 1 < m && win[k] != kNoKey && (k == 0 || win[k - 1] != win[k])) ? 1u : 0u;
}

__global__ void k_emit_runs(const uint32_t* __restrict__ win, const uint32_t* __restrict__ start,
                            const uint32_t* __restrict__ pos, const uint64_t* __restrict__ coords,
                            const unsigned long long* __restrict__ m_dev, uint64_t cap, uint64_t* __restrict__ ts,
                            uint64_t* __restrict__ te, uint32_t* __restrict__ tkey, uint32_t* __restrict__ tidx) {
  const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (k >= cap) return;
  const uint64_t m = *m_dev;
  if (k + 1 >= m || win[k] == kNoKey) return;
  const uint32_t run = pos[k] + start[k] - 1;
  if (start[k]) { ts[run] = coords[k]; tkey[run] = win[k]; tidx[run] = run; }
  if (k + 2 >= m || win[k + 1] != win[k]) te[run] = coords[k + 1];
}

__global__ void k_gather_hist(const uint32_t* __restrict__ key_sorted, const uint32_t* __restrict__ idx_sorted,
                              const uint64_t* __restrict__ ts, const uint64_t* __restrict__ te, uint64_t nn,
                              Stamps st, uint64_t* __restrict__ hs, uint64_t* __restrict__ he,
                              uint64_t* __restrict__ hseq, uint32_t* __restrict__ hthr, uint8_t* __restrict__ hw) {
  const uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (j >= nn) return;
  const uint32_t key = key_sorted[j], r = idx_sorted[j];
  uint32_t t;
  uint64_t s;
  stamp_of(st, key, t, s);
  hs[j] = ts[r];
  he[j] = te[r];
  hseq[j] = s;
  hthr[j] = t;
  hw[j] = (uint8_t)(key & 1u);
}

}  // namespace

struct cg_conc {
  int device = 0;
  uint64_t max_n = 0, max_stamps = 0, cap = 0, qcap = 0;
  int levels = 1;
  uint64_t nh[2] = {0, 0};
  uint64_t last_seq = 0;   // largest seq of the batches checked so far
  uint64_t launches = 0;
  std::string err;
  std::vector<std::pair<uint32_t, uint64_t>> syncs;
  bool syncs_dirty = false;
  std::vector<void*> allocs;
  // history (double-buffered) per space
  uint64_t *hs[2][2], *he[2][2], *hseq[2][2];
  uint32_t *hthr[2][2];
  uint8_t *hw[2][2];
  int cur[2] = {0, 0};
  // shared per-batch buffers
  uint64_t *qs[2], *qe[2];
  uint32_t *qkey[2], *qcopy[2];
  uint64_t *rs, *re, *rs_sorted, *ep, *ep_sorted, *coords;
  uint32_t *rkey, *mst, *cnt, *off, *noff, *noff2, *win, *flag, *pos, *tkey, *tidx, *tkey2, *tidx2;
  uint64_t *ts, *te;
  uint64_t* pairs = nullptr;
  uint64_t* pairs2 = nullptr;
  uint64_t pairs_cap = 0;
  unsigned long long* counts;   // [qn0, qn1, rn0, rn1, m, ...]
  uint32_t* sthr = nullptr;
  uint64_t* sseq = nullptr;
  uint64_t sync_cap = 0;
  void* temp = nullptr;
  size_t temp_bytes = 0;
  unsigned long long* h_counts = nullptr;   // pinned

  cg_status fail(cg_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    err = buf;
    return s;
  }
  template <typename T>
  bool alloc(T*& p, uint64_t n) {
    void* q = nullptr;
    if (cudaMalloc(&q, std::max<uint64_t>(n, 1) * sizeof(T)) != cudaSuccess) return false;
    allocs.push_back(q);
    p = static_cast<T*>(q);
    return true;
  }
  cg_status cuda(cudaError_t e, const char* what) {
    return e == cudaSuccess ? CG_OK : fail(CG_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  }
  Space space(int sp) {
    Space S;
    const int c = cur[sp];
    S.hs = hs[sp][c]; S.he = he[sp][c]; S.hseq = hseq[sp][c]; S.hthr = hthr[sp][c]; S.hw = hw[sp][c];
    S.qs = qs[sp]; S.qe = qe[sp]; S.qkey = qkey[sp]; S.qcopy = qcopy[sp];
    S.rs = rs + (sp ? cap : 0); S.re = re + (sp ? cap : 0); S.rkey = rkey + (sp ? cap : 0);
    return S;
  }
  cg_status ensure_temp(size_t bytes) {
    if (bytes <= temp_bytes) return CG_OK;
    if (temp) cudaFree(temp);
    temp = nullptr;
    temp_bytes = 0;
    if (cudaMalloc(&temp, bytes) != cudaSuccess) return fail(CG_ERR_OUT_OF_MEMORY, "cub temp storage");
    temp_bytes = bytes;
    return CG_OK;
  }
  cg_status ensure_pairs(uint64_t P) {
    if (P <= pairs_cap) return CG_OK;
    if (pairs) cudaFree(pairs);
    if (pairs2) cudaFree(pairs2);
    pairs = pairs2 = nullptr;
    pairs_cap = 0;
    const uint64_t cap2 = std::max<uint64_t>(P, 1024) * 5 / 4;
    if (cudaMalloc(&pairs, cap2 * 8) != cudaSuccess || cudaMalloc(&pairs2, cap2 * 8) != cudaSuccess)
      return fail(CG_ERR_OUT_OF_MEMORY, "cover pairs");
    pairs_cap = cap2;
    return CG_OK;
  }
  cg_status upload_syncs(cudaStream_t s) {
    if (!syncs_dirty) return CG_OK;
    const uint64_t n = syncs.size();
    if (n > sync_cap) {
      if (sthr) cudaFree(sthr);
      if (sseq) cudaFree(sseq);
      sthr = nullptr;
      sseq = nullptr;
      sync_cap = std::max<uint64_t>(n * 2, 1024);
      if (cudaMalloc(&sthr, sync_cap * 4) != cudaSuccess || cudaMalloc(&sseq, sync_cap * 8) != cudaSuccess)
        return fail(CG_ERR_OUT_OF_MEMORY, "sync list");
    }
    std::vector<uint32_t> t(n);
    std::vector<uint64_t> q(n);
    for (uint64_t i = 0; i < n; ++i) { t[i] = syncs[i].first; q[i] = syncs[i].second; }
    cudaError_t e = cudaMemcpyAsync(sthr, t.data(), n * 4, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(sseq, q.data(), n * 8, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);   // the host vectors die here
    if (e != cudaSuccess) return cuda(e, "sync upload");
    syncs_dirty = false;
    return CG_OK;
  }
  ~cg_conc() {
    for (void* p : allocs) cudaFree(p);
    if (pairs) cudaFree(pairs);
    if (pairs2) cudaFree(pairs2);
    if (sthr) cudaFree(sthr);
    if (sseq) cudaFree(sseq);
    if (temp) cudaFree(temp);
    if (h_counts) cudaFreeHost(h_counts);
  }
  cg_status run_space(int sp, const cg_copy_desc* d, const uint32_t* threads, uint64_t n, cg_verdict* v,
                      uint64_t qn, uint64_t rn, int addr_bits, cudaStream_t s);
};

namespace {
uint64_t next_pow2(uint64_t x) {
  uint64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}
int ceil_log2(uint64_t x) {
  int L = 0;
  while ((1ull << L) < x) ++L;
  return L;
}
}  // namespace

cg_status cg_conc::run_space(int sp, const cg_copy_desc* d, const uint32_t* threads, uint64_t n, cg_verdict* v,
                             uint64_t qn, uint64_t rn, int addr_bits, cudaStream_t s) {
  const uint64_t nh0 = nh[sp];
  if (qn == 0) return CG_OK;   // no access of this space in the batch: nothing recorded either
  Space S = space(sp);
  Stamps st{S.hthr, S.hseq, nh0, d, threads};
  Syncs sy{sthr, sseq, syncs.size()};
  Tree T{};
  T.cap = cap;
  T.rn = rn;
  size_t tb = 0;
  cudaError_t e = cudaSuccess;
  const uint64_t M = next_pow2(std::max<uint64_t>(2 * rn, 2));
  if (rn) {
    // (A) merge-sort tree over R sorted by start
    // R's addresses share every bit above addr_bits: sort only the bits that differ
    cub::DeviceRadixSort::SortPairs(nullptr, tb, S.rs, rs_sorted, S.rkey, mst, (int)rn, 0, addr_bits, s);
    if (ensure_temp(tb) != CG_OK) return CG_ERR_OUT_OF_MEMORY;
    e = cub::DeviceRadixSort::SortPairs(temp, tb, S.rs, rs_sorted, S.rkey, mst, (int)rn, 0, addr_bits, s);
    if (e != cudaSuccess) return cuda(e, "sort R");
    const int L = ceil_log2(rn);
    const int Ls = std::min(L, kSmemLevels);   // levels inside 256-key tiles: one pass in shared memory
    if (Ls) {
      k_merge_tile<<<(unsigned)((rn + (1u << kSmemLevels) - 1) >> kSmemLevels), 1 << kSmemLevels, 0, s>>>(mst, rn, cap,
                                                                                                         Ls);
      ++launches;
    }
    for (int l = Ls + 1; l <= L;) {
      if (l + 1 <= L) {
        k_merge_2levels<<<grid_for(rn), kT, 0, s>>>(mst + (uint64_t)(l - 1) * cap, mst + (uint64_t)l * cap,
                                                    mst + (uint64_t)(l + 1) * cap, rn, l);
        l += 2;
      } else {
        k_merge_level<<<grid_for(rn), kT, 0, s>>>(mst + (uint64_t)(l - 1) * cap, mst + (uint64_t)l * cap, rn, l);
        ++l;
      }
      ++launches;
    }
    T.rs_sorted = rs_sorted;
    T.mst = mst;
    T.levels = L + 1;
    // (B) elementary intervals and cover lists
    k_endpoints<<<grid_for(rn), kT, 0, s>>>(S.rs, S.re, rn, ep);
    ++launches;
    tb = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tb, ep, ep_sorted, (int)(2 * rn), 0, addr_bits, s);
    if (ensure_temp(tb) != CG_OK) return CG_ERR_OUT_OF_MEMORY;
    e = cub::DeviceRadixSort::SortKeys(temp, tb, ep, ep_sorted, (int)(2 * rn), 0, addr_bits, s);
    if (e != cudaSuccess) return cuda(e, "sort endpoints");
    tb = 0;
    cub::DeviceSelect::Unique(nullptr, tb, ep_sorted, coords, counts + 4, (int)(2 * rn), s);
    if (ensure_temp(tb) != CG_OK) return CG_ERR_OUT_OF_MEMORY;
    e = cub::DeviceSelect::Unique(temp, tb, ep_sorted, coords, counts + 4, (int)(2 * rn), s);
    if (e != cudaSuccess) return cuda(e, "unique endpoints");
    k_cover_count<<<grid_for(rn), kT, 0, s>>>(S.rs, S.re, rn, coords, counts + 4, M, cnt, ts);
    ++launches;
    tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, off, (int)rn, s);
    if (ensure_temp(tb) != CG_OK) return CG_ERR_OUT_OF_MEMORY;
    e = cub::DeviceScan::ExclusiveSum(temp, tb, cnt, off, (int)rn, s);
    if (e != cudaSuccess) return cuda(e, "scan cover counts");
    uint32_t tail[2];
    e = cudaMemcpyAsync(&tail[0], off + rn - 1, 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&tail[1], cnt + rn - 1, 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda(e, "cover total");
    const uint64_t P = (uint64_t)tail[0] + tail[1];
    if (ensure_pairs(P) != CG_OK) return CG_ERR_OUT_OF_MEMORY;
    const int kb = std::max(ceil_log2(2 * (nh0 + n) + 2), 1);   // bits of a key (2 ord + is_write)
    k_cover_emit<<<grid_for(rn), kT, 0, s>>>(ts, S.rkey, rn, M, off, pairs2, kb);
    ++launches;
    const int end_bit = kb + ceil_log2(2 * M) + 1;
    tb = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tb, pairs2, pairs, (int)P, 0, end_bit, s);
    if (ensure_temp(tb) != CG_OK) return CG_ERR_OUT_OF_MEMORY;
    e = cub::DeviceRadixSort::SortKeys(temp, tb, pairs2, pairs, (int)P, 0, end_bit, s);
    if (e != cudaSuccess) return cuda(e, "sort cover pairs");
    k_fill_u32<<<grid_for(2 * M + 1), kT, 0, s>>>(noff2, 2 * M + 1, (uint32_t)P);
    k_node_starts<<<grid_for(P), kT, 0, s>>>(pairs, P, kb, 2 * M, noff2);
    launches += 2;
    tb = 0;
    cub::DeviceScan::InclusiveScan(nullptr, tb, noff2, noff, MinU32(), (int)(2 * M + 1), s);
    if (ensure_temp(tb) != CG_OK) return CG_ERR_OUT_OF_MEMORY;
    e = cub::DeviceScan::InclusiveScan(temp, tb, noff2, noff, MinU32(), (int)(2 * M + 1), s);
    if (e != cudaSuccess) return cuda(e, "node offsets");
    T.coords = coords;
    T.m_dev = counts + 4;
    T.noff = noff;
    T.nodes = 2 * M;
    T.pairs = pairs;
    T.M = M;
    T.kmask = (1ull << kb) - 1;
    k_query<<<grid_for(qn), kT, 0, s>>>(S, qn, T, st, sy, v);
    ++launches;
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda(e, "query kernels");
  }
  if (rn == nh0) return CG_OK;   // nothing performed: the map is unchanged
  // rebuild the last-access map: winners of the elementary intervals, runs merged
  const uint64_t ncap = 2 * rn;   // elementary intervals < number of coordinates <= 2 rn
  k_winners<<<grid_for(ncap), kT, 0, s>>>(T, win);
  k_run_flags<<<grid_for(ncap), kT, 0, s>>>(win, counts + 4, ncap, flag);
  launches += 2;
  tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, flag, pos, (int)ncap, s);
  if (ensure_temp(tb) != CG_OK) return CG_ERR_OUT_OF_MEMORY;
  e = cub::DeviceScan::ExclusiveSum(temp, tb, flag, pos, (int)ncap, s);
  if (e != cudaSuccess) return cuda(e, "scan runs");
  uint32_t tail[2];
  e = cudaMemcpyAsync(&tail[0], pos + ncap - 1, 4, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&tail[1], flag + ncap - 1, 4, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda(e, "run count");
  const uint64_t nn = (uint64_t)tail[0] + tail[1];
  if (nn > max_stamps) return fail(CG_ERR_OUT_OF_MEMORY, "last-access map needs %llu > max_stamps ranges",
                                   (unsigned long long)nn);
  k_emit_runs<<<grid_for(ncap), kT, 0, s>>>(win, flag, pos, coords, counts + 4, ncap, ts, te, tkey, tidx);
  ++launches;
  tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, tkey, tkey2, tidx, tidx2, (int)nn, 0, 32, s);
  if (ensure_temp(tb) != CG_OK) return CG_ERR_OUT_OF_MEMORY;
  e = cub::DeviceRadixSort::SortPairs(temp, tb, tkey, tkey2, tidx, tidx2, (int)nn, 0, 32, s);
  if (e != cudaSuccess) return cuda(e, "sort map");
  const int nx = cur[sp] ^ 1;
  k_gather_hist<<<grid_for(nn), kT, 0, s>>>(tkey2, tidx2, ts, te, nn, st, hs[sp][nx], he[sp][nx], hseq[sp][nx],
                                            hthr[sp][nx], hw[sp][nx]);
  ++launches;
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda(e, "rebuild kernels");
  cur[sp] = nx;
  nh[sp] = nn;
  return CG_OK;
}

extern "C" {

cg_status cg_conc_create(int device, uint64_t max_n, uint64_t max_stamps, cg_conc** out) {
  if (!out) return CG_ERR_INVALID_VALUE;
  *out = nullptr;
  if (max_n == 0 || max_stamps == 0 || 2 * max_n + max_stamps >= (1ull << 30)) return CG_ERR_INVALID_VALUE;
  int prev = -1;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess) return CG_ERR_CUDA;
  cg_conc* c = new cg_conc();
  c->device = device;
  c->max_n = max_n;
  c->max_stamps = max_stamps;
  c->qcap = 2 * max_n;
  c->cap = max_stamps + 2 * max_n;
  c->levels = ceil_log2(c->cap) + 1;
  const uint64_t cap = c->cap, ncap = 2 * cap;
  bool ok = true;
  for (int sp = 0; sp < 2 && ok; ++sp) {
    for (int b = 0; b < 2 && ok; ++b)
      ok = c->alloc(c->hs[sp][b], max_stamps) && c->alloc(c->he[sp][b], max_stamps) &&
           c->alloc(c->hseq[sp][b], max_stamps) && c->alloc(c->hthr[sp][b], max_stamps) &&
           c->alloc(c->hw[sp][b], max_stamps);
    ok = ok && c->alloc(c->qs[sp], c->qcap) && c->alloc(c->qe[sp], c->qcap) && c->alloc(c->qkey[sp], c->qcap) &&
         c->alloc(c->qcopy[sp], c->qcap);
  }
  ok = ok && c->alloc(c->rs, 2 * cap) && c->alloc(c->re, 2 * cap) && c->alloc(c->rkey, 2 * cap) &&
       c->alloc(c->rs_sorted, cap) && c->alloc(c->ep, ncap) && c->alloc(c->ep_sorted, ncap) &&
       c->alloc(c->coords, ncap) && c->alloc(c->mst, (uint64_t)c->levels * cap) && c->alloc(c->cnt, cap) &&
       c->alloc(c->off, cap) && c->alloc(c->noff, 2 * next_pow2(ncap) + 2) && c->alloc(c->noff2, 2 * next_pow2(ncap) + 2) && c->alloc(c->win, ncap) &&
       c->alloc(c->flag, ncap) && c->alloc(c->pos, ncap) && c->alloc(c->tkey, ncap) && c->alloc(c->tidx, ncap) &&
       c->alloc(c->tkey2, ncap) && c->alloc(c->tidx2, ncap) && c->alloc(c->ts, ncap) && c->alloc(c->te, ncap) &&
       c->alloc(c->counts, 16);
  ok = ok && cudaMallocHost(&c->h_counts, 16 * sizeof(unsigned long long)) == cudaSuccess;
  if (prev >= 0) cudaSetDevice(prev);
  if (!ok) {
    delete c;
    return CG_ERR_OUT_OF_MEMORY;
  }
  *out = c;
  return CG_OK;
}

cg_status cg_conc_destroy(cg_conc* c) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(c->device);
  delete c;
  if (prev >= 0) cudaSetDevice(prev);
  return CG_OK;
}

const char* cg_conc_last_error(const cg_conc* c) { return c ? c->err.c_str() : "null context"; }

cg_status cg_conc_sync(cg_conc* c, uint32_t thread, uint64_t seq) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  const std::pair<uint32_t, uint64_t> x{thread, seq};
  auto it = std::lower_bound(c->syncs.begin(), c->syncs.end(), x);
  if (it == c->syncs.end() || *it != x) c->syncs.insert(it, x);
  c->syncs_dirty = true;
  return CG_OK;
}

cg_status cg_conc_check(cg_conc* c, const cg_copy_desc* d_descs, const uint32_t* d_threads, uint64_t n,
                        cg_verdict* d_verdicts, void* stream) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  if (n == 0) return CG_OK;
  if (!d_descs || !d_threads || !d_verdicts) return c->fail(CG_ERR_INVALID_VALUE, "null array");
  if (n > c->max_n) return c->fail(CG_ERR_INVALID_VALUE, "n > max_n");
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(c->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cg_status st = c->upload_syncs(s);
  cudaError_t e = cudaSuccess;
  if (st == CG_OK) {
    // counts: queries per space, recorded batch accesses per space (R holds the map first)
    e = cudaMemsetAsync(c->counts, 0, 16 * sizeof(unsigned long long), s);
    for (int sp = 0; sp < 2 && e == cudaSuccess; ++sp)   // min start of R per space
      e = cudaMemsetAsync(c->counts + 8 + 2 * sp, 0xFF, sizeof(unsigned long long), s);
    Space S0 = c->space(0), S1 = c->space(1);
    const uint64_t mh = std::max(c->nh[0], c->nh[1]);
    if (e == cudaSuccess && mh) {
      k_hist_to_r<<<grid_for(mh), kT, 0, s>>>(S0, S1, c->nh[0], c->nh[1], c->counts);
      ++c->launches;
    }
    if (e == cudaSuccess) {
      k_access<<<grid_for(n), kT, 0, s>>>(d_descs, d_verdicts, n, S0, S1, c->nh[0], c->nh[1], c->counts);
      ++c->launches;
      e = cudaMemcpyAsync(c->h_counts, c->counts, 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) st = c->cuda(e, "access kernels");
  }
  for (int sp = 0; sp < 2 && st == CG_OK; ++sp) {
    if (sp == 0 && (c->h_counts[12] || c->h_counts[13] <= c->last_seq)) {
      st = c->fail(CG_ERR_INVALID_VALUE, "batch seqs must increase, and exceed those of earlier batches");
      break;
    }
    const uint64_t qn = c->h_counts[sp], rn = c->nh[sp] + c->h_counts[2 + sp];
    const uint64_t lo = c->h_counts[8 + 2 * sp], hi = c->h_counts[9 + 2 * sp];
    const int bits = lo < hi ? 64 - __builtin_clzll(lo ^ hi) : 1;   // the address bits R's keys differ in
    st = c->run_space(sp, d_descs, d_threads, n, d_verdicts, qn, rn, std::max(bits, 1), s);
  }
  if (st == CG_OK) c->last_seq = c->h_counts[14];
  if (prev >= 0) cudaSetDevice(prev);
  return st;
}

cg_status cg_conc_stamps(const cg_conc* c, uint64_t* n_host, uint64_t* n_device) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  if (n_host) *n_host = c->nh[0];
  if (n_device) *n_device = c->nh[1];
  return CG_OK;
}

uint64_t cg_conc_kernel_launches(const cg_conc* c) { return c ? c->launches : 0; }

}  // extern "C"
