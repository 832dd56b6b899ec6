// Internal interface between the C-ABI runtime (cg_runtime.cu) and the
// sm_100a kernels (cg_kernels.cu).  Not part of the public ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "cg.h"

namespace cgk {

constexpr uint64_t kNone = UINT64_MAX;
constexpr uint64_t kInf = UINT64_MAX;          // free_seq of a live allocation
constexpr uint64_t kMaxShardBytes = 1ull << 38;  // host bytes one context stores (config limit; scan weights < 2^40 each)
constexpr uint64_t kDeferBytes = 1ull << 36;     // sparse map: longer host sides go to the deferred pass
constexpr uint64_t kSmallBytesDefault = 4096;    // the small pass's limit (env CG_SMALL_BYTES, at most 4 KiB: its stage)
constexpr uint64_t kSmallStatDefault = 4096;     // its adaptive choice counts sides up to this (env CG_SMALL_STAT)
constexpr uint64_t kMaxDescs = 1ull << 24;       // per call (keeps sum of weights < 2^63)

// start = base + y*pitch + x; span = (w==0||h==0) ? 0 : (h-1)*pitch + w;
// valid iff start + span <= 2^64 - 1 (every partial sum is then exact).
__device__ __forceinline__ bool fold_side(uint64_t base, uint64_t x, uint64_t y, uint64_t pitch,
                                          uint64_t w, uint64_t h, uint64_t& start, uint64_t& span) {
  if (__umul64hi(y, pitch) != 0) return false;
  uint64_t s = y * pitch;
  uint64_t t = s + x;
  if (t < s) return false;
  uint64_t st = t + base;
  if (st < t) return false;
  uint64_t sp = 0;
  if (w != 0 && h != 0) {
    if (__umul64hi(h - 1, pitch) != 0) return false;
    uint64_t q = (h - 1) * pitch;
    sp = q + w;
    if (sp < q) return false;
  }
  uint64_t e = st + sp;
  if (e < st) return false;
  start = st;
  span = sp;
  return true;
}

// Host window [wb, we) and the shard [sb, se) whose shadow this GPU stores.
struct ShadowView {
  uint64_t wb, we, sb, se;
  uint8_t* V;   // bytes format: se - sb V bytes; 2-bit format: (se - sb) / 4 state bytes
  uint8_t* A;   // bytes format: (se - sb) / 8 bytes (unused in the 2-bit format)
  uint32_t two_bit;   // NEXT-4 compressed shadow (CG_SHADOW_2BIT, CG_SHADOW_SPARSE)
  // NEXT-4 sparse two-level map (CG_SHADOW_SPARSE): host byte q lives in the
  // 64 KiB chunk q >> 16, whose 16 KiB of states is secondary dir(chunk) of V
  // (secondary 0 = the distinguished all-NOACCESS one, never written); the
  // directory is an open-addressing table, Fibonacci-hashed, linear probing
  uint32_t sparse;
  uint32_t dir_bits;        // log2 of the slot count
  const uint64_t* dir_key;  // chunk + 1, 0 = empty slot
  const uint32_t* dir_val;  // secondary index
  uint64_t v_bytes;         // size of V (fresh-shadow fill)
  // sparse map: the chunks that have a secondary, ascending (the deferred
  // pass walks them instead of the whole 64-bit range of a huge copy)
  const uint64_t* chunk_list;
  uint64_t n_chunks;
  // the small pass (k_check_small) takes contiguous host sides of at most
  // this many bytes (0: none; env CG_SMALL_BYTES)
  uint64_t small_limit;
  // its on/off choice: 0 adaptive (from the previous check's share of sides of
  // at most small_stat bytes), 1 always, 2 never (env CG_SMALL_MODE, CG_SMALL_STAT)
  uint32_t small_mode;
  uint32_t small_share;   // adaptive: on when at least this percent of the sides were small (env CG_SMALL_SHARE)
  uint64_t small_stat;
};

constexpr uint64_t kChunkShift = 16;               // 64 KiB host bytes per chunk
constexpr uint64_t kSecondaryBytes = 1ull << 14;   // their 2-bit states
__host__ __device__ __forceinline__ uint64_t dir_hash(uint64_t chunk, uint32_t bits) {
  return (chunk * 0x9E3779B97F4A7C15ull) >> (64 - bits);
}

// NEXT-4 2-bit host states (R-36): host byte q <-> bits 2(q&15),
// 2(q&15)+1 of 32-bit word q>>4.  bit 0 set = some V bit undefined, state 0 =
// unaddressable (A = 0, V = 0xFF implied).
constexpr uint32_t kSt2NoAccess = 0u, kSt2Partial = 1u, kSt2Defined = 2u, kSt2Undefined = 3u;

// Allocation table: structure of arrays sorted by (base, alloc_seq), with the
// running maximum of end addresses.
struct Table {
  const uint64_t* base;
  const uint64_t* end;
  const uint64_t* aseq;
  const uint64_t* fseq;
  const uint64_t* pmax;
  const uint64_t* split;   // base[k * stride], k < nsplit (16-byte aligned, padded to even)
  const uint64_t* l2;      // base[4 k], k < ceil(n / 4) (64-byte aligned)
  const uint64_t* pool;    // NEXT-1: device V-pool offset of each entry (nullptr without tracking)
  const uint4* walk;       // per entry 32 B: (prefix max of ends, end, alloc seq, free seq), the lookup walk's reads
  uint64_t n;
  // NEXT-3 device arrays: sorted by (handle, alloc_seq)
  const uint64_t* ahandle;
  const uint64_t* atotal;
  const uint64_t* aaseq;
  const uint64_t* afseq;
  const uint64_t* apool;   // NEXT-1 x NEXT-3: device V-pool offset of each array's V-bits (nullptr without tracking)
  uint64_t na;
  uint32_t stride;   // splitter stride (every stride-th base is staged in smem)
  uint32_t nsplit;
  uint32_t two_round64;   // stride 64: two independent-load rounds (env CG_LOOKUP64=1; default: binary search)
};

// A planned pass over n weighted items: P = exclusive prefix sum of weights
// (P[n] = total), cut into chunks of T >= t_min weight units (T grows so that
// the number of chunks never exceeds max_chunks); chunk_first[c] = the item
// whose weight interval contains c*T.
struct Plan {
  uint64_t* weight;       // [n]
  uint64_t* P;            // [n + 1]
  uint64_t* bsum;         // [nblocks + 1]
  uint64_t* fbsum;        // [kFinishMaxBlocks] k_finish's per-block sums
  uint32_t* chunk_first;  // [max_chunks]
  void* meta;             // [n] ScanMeta (check plans only)
  uint32_t* counter;      // [0] group counter, [1] apply compaction count, [2] residual-list count,
                          // [3] memmove-list count, [4] deferred-list count, [5] deferred-list cursor
  uint32_t* resid;        // [n] fused check: DtoH descriptors left to the residual apply
  uint32_t* defer;        // [n] descriptors whose host side the deferred pass checks (R-10, R-12)
  uint32_t* late;         // [n] CG_CHECK_AFTER descriptors, checked by k_finish after the applies
  uint32_t* last;         // [n] CG_APPLY_LAST DtoH descriptors, applied by k_finish after the late checks
                          // (count, cursor: counter[6], [7])
  uint64_t* dvoff;        // [2n] NEXT-1: device V offsets (dst, src) found by the last check
  uint64_t max_chunks;
  uint64_t t_min;
};

// Optional per-stage event recording (cg_profile_begin / cg_profile_end).
struct Profiler {
  bool on = false;
  void (*mark)(void* self, int stage, bool begin, cudaStream_t s) = nullptr;
  void* self = nullptr;
};

struct Launch {
  int num_sms;
  int persist_blocks;     // persistent grid for the chunked kernels
  int scan_blocks;        // persistent grid of the TMA-ring scan
  int wave_blocks;        // cooperative grid of k_prop_waves (all co-resident)
  int finish_blocks;      // cooperative grid of k_finish
  int front_blocks;       // cooperative grid of k_front (0: prep + plan as separate launches)
  int leak_blocks = 0;    // cooperative grid of k_leak (0: the 5-launch sweep)
  int small_blocks = 0;   // grid of k_check_small (the small pass)
  uint64_t* counter;      // host counter of kernel launches
  Profiler* prof;
  void stage(int st, bool begin, cudaStream_t s) const {
    if (prof && prof->on) prof->mark(prof->self, st, begin, s);
  }
};

constexpr int kScanTile = 2048;   // items per block of the prefix scan

uint64_t scan_blocks(uint64_t n);
int persistent_blocks(int which);   // 0: k_check_scan, 1: k_apply, 2: k_prop_waves, 3: k_finish, 4: k_front, 5: k_leak, 6: k_check_small (per SM)
constexpr uint64_t kFinishMaxBlocks = 4096;
constexpr size_t kFrontSmem = (4096 + 2) * sizeof(uint64_t);   // k_front: the largest splitter array
size_t prop_meta_bytes();
uint64_t stage_bytes();
cudaError_t propagate(const Launch& L, const cg_copy_desc* d, const cg_verdict* v, const uint32_t* index, uint64_t n,
                      const ShadowView& sv, uint8_t* pool, const Plan& p, uint8_t* scratch, uint32_t* overflow,
                      cudaStream_t s, bool reset_overflow);
cudaError_t propagate_direct(const Launch& L, const cg_copy_desc* d, const cg_verdict* v, const uint32_t* index,
                             uint64_t m, uint64_t max_bytes, const ShadowView& sv, uint8_t* pool, const Plan& p,
                             uint8_t* scratch, uint32_t* overflow, cudaStream_t s);
cudaError_t propagate_waves(const Launch& L, const cg_copy_desc* d, const cg_verdict* v, const uint32_t* index,
                            uint64_t m, const uint32_t* d_wstart, uint32_t n_waves, const ShadowView& sv,
                            uint8_t* pool, const Plan& p, uint8_t* scratch, uint32_t* overflow, cudaStream_t s);
size_t scan_meta_bytes();
cudaError_t table_patch(const Launch& L, uint64_t* fseq, uint64_t* walk, const uint64_t* d_pairs, uint64_t k,
                        cudaStream_t s);
cudaError_t memmove_list(const Launch& L, const cg_copy_desc* d, const uint64_t* dvoff, const uint32_t* list,
                         const uint32_t* count, uint8_t* pool, uint8_t* scratch, uint64_t stage_cap,
                         uint32_t* overflow, cudaStream_t s);

cudaError_t check_copies(const Launch& L, const cg_copy_desc* d, uint64_t n, cg_verdict* out,
                         const Table& t, const ShadowView& sv, const Plan& p, uint32_t err_mask, bool fuse,
                         cudaStream_t s);
cudaError_t check_apply(const Launch& L, const cg_copy_desc* d, uint64_t n, cg_verdict* out, const Table& t,
                        const ShadowView& sv, const Plan& p, uint32_t err_mask, cudaStream_t s);
cudaError_t apply_dtoh(const Launch& L, const cg_copy_desc* d, const cg_verdict* v, uint64_t n,
                       const ShadowView& sv, const Plan& p, bool after_fused, cudaStream_t s);
cudaError_t straddler_pack(const Launch& L, const cg_verdict* v, uint64_t m, uint64_t* mins, uint64_t* sums,
                           uint32_t* maxs, cudaStream_t s);
cudaError_t straddler_finalize(const Launch& L, const uint64_t* mins, const uint64_t* sums, const uint32_t* maxs,
                               uint64_t m, cg_verdict* v, uint32_t err_mask, cudaStream_t s);
cudaError_t compact_dirty(const Launch& L, const cg_verdict* v, uint64_t n, uint64_t* idx, cg_verdict* dirty,
                          uint32_t* count, uint64_t idx_base, bool reset, cudaStream_t s);
cudaError_t expand_1d(const Launch& L, const cg_copy1d* in, uint64_t n, cg_copy_desc* out, cudaStream_t s);
cudaError_t mark_batch(const Launch& L, const cg_mark* d_marks, uint64_t n, const ShadowView& sv,
                       const Plan& p, cudaStream_t s);
cudaError_t fresh_shadow(const Launch& L, const ShadowView& sv, cudaStream_t s);
cudaError_t summarize(const cg_verdict* v, uint64_t n, uint32_t warn_mask, unsigned long long* d_counts,
                      cudaStream_t s);
cudaError_t setv_check(const Launch& L, uint64_t addr, uint64_t len, const ShadowView& sv,
                       uint32_t* d_flag, cudaStream_t s);
cudaError_t leak_sweep(const Launch& L, const Table& t, const Plan& p, cg_alloc_record* out,
                       uint64_t cap, uint64_t* d_count, cudaStream_t s);

}  // namespace cgk
