// C-ABI runtime of the batched Cudagrind transfer checker (include/cg.h).
//
// Owns: the context (window, shard, caller buffers carved into device tables
// and plan scratch), the registry host mirror (sorted,
// lifetime-stamped entries; live set for overlap / free validation), its
// upload to the device table, pinned staging, and the host epoch planner.
// Every step of the check itself runs in the kernels of cg_kernels.cu.

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "cg.h"
#include "cg_internal.h"


namespace {

constexpr uint64_t kAlign = 256;
constexpr uint64_t kChunkMin = 32 * 1024;        // t_min of the chunk plans (weight units)
constexpr uint64_t kMarkRun = 1u << 20;          // marks uploaded per run
constexpr uint64_t kHostChunks = 5;              // cg_check_host upload / check pipeline depth
constexpr uint32_t kHostSlots = 2;               // cg_check_host_submit staging slots (double buffering)

uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

struct Entry {
  uint64_t base, end, aseq, fseq, pool;   // pool: NEXT-1 device V offset of the allocation
};

struct ArrayEntry {   // NEXT-3 device array (SPEC register_array S:166-168)
  uint64_t handle, total, aseq, fseq, pool;   // pool: NEXT-1 offset of its V-bits (R-30)
};

struct Layout {
  uint64_t table, walk, patch, arrays, weight, P, bsum, fbsum, chunk, meta, resid, defer, late, last, dvoff, scratch, waves, ovl, marks, flags,
      leaks,
      desc_stage, chunk_list,
      verdict_stage, raw_stage,
      idx_stage, dirty_stage, dir, total;
  uint32_t dir_bits;
  uint64_t max_items, max_chunks;
};

bool valid_config(const cg_config* c) {
  if (!c) return false;
  if (c->shadow_format == CG_SHADOW_SPARSE) {   // NEXT-4 two-level map: capacity only, unsharded
    if (c->host_base != 0 || c->host_size == 0 || c->host_size % 65536 || c->shard_size || c->dev_vbuf) return false;
    if (c->max_descs == 0 || c->max_descs > cgk::kMaxDescs) return false;
    return c->max_allocs != 0 && c->max_allocs <= (1ull << 32);
  }
  if (c->host_size == 0 || c->host_base % 4096 || c->host_size % 4096) return false;
  if (c->host_base + c->host_size < c->host_base) return false;
  uint64_t sb = c->shard_size ? c->shard_base : c->host_base;
  uint64_t ss = c->shard_size ? c->shard_size : c->host_size;
  if (sb % 4096 || ss % 4096 || ss == 0) return false;
  if (ss > cgk::kMaxShardBytes) return false;   // one GPU stores at most 2^38 host bytes (no B200 holds more shadow)
  if (sb < c->host_base || sb + ss > c->host_base + c->host_size) return false;
  if (c->max_descs == 0 || c->max_descs > cgk::kMaxDescs) return false;
  if (c->max_allocs == 0 || c->max_allocs > (1ull << 32)) return false;
  if (c->shadow_format != CG_SHADOW_BYTES && c->shadow_format != CG_SHADOW_2BIT) return false;
  if (c->shadow_format == CG_SHADOW_2BIT && c->dev_vbuf) return false;   // NEXT-1 needs exact host V-bytes
  if (c->dev_vbuf && (c->dev_vsize == 0 || c->dev_vsize % 16 || (uintptr_t)c->dev_vbuf % 16 || (c->shard_size && (c->shard_base != c->host_base ||
                                                              c->shard_size != c->host_size))))
    return false;   // NEXT-1 tracking needs a pool and an unsharded context
  return true;
}

Layout layout_of(const cg_config* c) {
  Layout L{};
  L.max_items = std::max(c->max_descs, c->max_allocs);
  L.max_chunks = std::max<uint64_t>(1u << 20, 2 * c->max_descs);
  uint64_t off = 0;
  auto take = [&](uint64_t bytes) {
    uint64_t o = off;
    off = align_up(off + bytes, kAlign);
    return o;
  };
  L.table = take(6 * c->max_allocs * 8 + (4096 + 3) * 8 + (c->max_allocs / 4 + 16) * 8);   // SoA (+ pool offsets) + splitters + every 4th base
  L.walk = take(4 * c->max_allocs * 8);                      // (prefix max, end, alloc seq, free seq) per entry
  L.patch = take(2 * c->max_allocs * 8);                     // (position, free seq) pairs of a diff upload
  L.arrays = take(5 * c->max_allocs * 8);                    // NEXT-3 array table (SoA + pool offsets)
  L.weight = take(L.max_items * 8);
  L.P = take((L.max_items + 1) * 8);
  L.bsum = take((cgk::scan_blocks(L.max_items) + 1) * 8);
  L.fbsum = take(cgk::kFinishMaxBlocks * 8);   // k_finish's per-block sums
  L.chunk = take(L.max_chunks * 4);
  L.meta = take(c->max_descs * std::max(cgk::scan_meta_bytes(), cgk::prop_meta_bytes()));
  L.resid = take(c->max_descs * sizeof(uint32_t));
  L.defer = take(c->max_descs * sizeof(uint32_t));
  L.late = take(c->max_descs * sizeof(uint32_t));
  L.last = take(c->max_descs * sizeof(uint32_t));
  L.dvoff = c->dev_vbuf ? take(c->max_descs * 16) : 0;
  L.scratch = c->dev_vbuf ? take(cgk::stage_bytes()) : 0;
  L.waves = c->dev_vbuf ? take((c->max_descs + 1) * sizeof(uint32_t)) : 0;   // NEXT-1 wave offsets
  L.ovl = c->dev_vbuf ? take((c->max_descs + 2) * sizeof(uint32_t)) : 0;     // NEXT-1 staging overflow: flag, count, list
  L.marks = take(std::min<uint64_t>(c->max_descs, kMarkRun) * sizeof(cg_mark));
  L.flags = take(256);
  L.leaks = take(c->max_allocs * sizeof(cg_alloc_record));
  // host staging: kHostSlots slots (cg_check_host_submit double-buffers batches)
  L.desc_stage = c->host_staging ? take(kHostSlots * c->max_descs * sizeof(cg_copy_desc)) : 0;
  L.verdict_stage = c->host_staging ? take(kHostSlots * c->max_descs * sizeof(cg_verdict)) : 0;
  L.raw_stage = c->host_staging ? take(kHostSlots * c->max_descs * sizeof(cg_copy1d)) : 0;
  L.idx_stage = c->host_staging ? take(kHostSlots * c->max_descs * sizeof(uint64_t)) : 0;
  L.dirty_stage = c->host_staging ? take(kHostSlots * c->max_descs * sizeof(cg_verdict)) : 0;
  L.dir_bits = 0;
  L.dir = 0;
  if (c->shadow_format == CG_SHADOW_SPARSE) {   // directory: >= 2x the secondaries, power of two
    const uint64_t nsec = c->host_size / 65536 + 1;
    while ((1ull << L.dir_bits) < 2 * nsec) ++L.dir_bits;
    L.dir = take((1ull << L.dir_bits) * 12);
    L.chunk_list = take(nsec * 8);   // the chunks with a secondary, ascending (deferred pass)
  }
  L.total = off;
  return L;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace

struct cg_ctx {
  cg_config cfg;
  Layout lay;
  cgk::ShadowView sv;
  cgk::Launch launch;
  uint64_t launches = 0;
  uint8_t* ws = nullptr;
  // registry host mirror
  std::vector<Entry> table;                 // sorted by (base, aseq)
  std::map<uint64_t, uint64_t> live;        // base -> end of live allocations
  std::vector<ArrayEntry> arrays;           // NEXT-3: sorted by (handle, aseq)
  std::map<uint64_t, uint8_t> partial;      // NEXT-4 2-bit format: exact V-bytes of PARTIAL host bytes
  std::map<uint64_t, uint32_t> chunks;      // NEXT-4 sparse map: chunk -> secondary (1-based)
  std::vector<uint32_t> dir_host;           // directory image: 2^bits u64 keys then 2^bits u32 values
  bool dir_dirty = false;

  // sparse map: make sure every chunk of [a, b) has a secondary; false if the pool is full
  bool ensure_chunks(uint64_t a, uint64_t b) {
    const uint64_t cap = cfg.host_size / 65536;
    for (uint64_t c = a >> cgk::kChunkShift; c <= (b - 1) >> cgk::kChunkShift; ++c) {
      if (chunks.count(c)) continue;
      if (chunks.size() >= cap) return false;
      const uint32_t sec = (uint32_t)chunks.size() + 1;
      chunks.emplace(c, sec);
      const uint64_t slots = 1ull << lay.dir_bits;
      uint64_t* keys = reinterpret_cast<uint64_t*>(dir_host.data());
      uint32_t* vals = dir_host.data() + 2 * slots;
      for (uint64_t h = cgk::dir_hash(c, lay.dir_bits);; h = (h + 1) & (slots - 1)) {
        if (keys[h] == 0) {
          keys[h] = c + 1;
          vals[h] = sec;
          break;
        }
      }
      dir_dirty = true;
    }
    return true;
  }
  std::vector<uint64_t> chunk_ids;          // sorted chunk list image (sparse map)
  cg_status upload_dir(cudaStream_t s) {
    if (!dir_dirty) return CG_OK;
    cudaError_t e = cudaMemcpyAsync(ws + lay.dir, dir_host.data(), dir_host.size() * 4, cudaMemcpyHostToDevice, s);
    chunk_ids.clear();
    for (const auto& kv : chunks) chunk_ids.push_back(kv.first);
    if (e == cudaSuccess && !chunk_ids.empty())
      e = cudaMemcpyAsync(ws + lay.chunk_list, chunk_ids.data(), chunk_ids.size() * 8, cudaMemcpyHostToDevice, s);
    sv.n_chunks = chunk_ids.size();
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);   // the host image may change right after
    if (e != cudaSuccess) return cuda(e, "directory upload");
    dir_dirty = false;
    return CG_OK;
  }
  // device pointer of the state word holding host byte q (sparse: nullptr if its chunk has no secondary)
  uint32_t* state_word(uint64_t q) {
    if (!sv.sparse) return reinterpret_cast<uint32_t*>(sv.V) + (q >> 4);
    auto it = chunks.find(q >> cgk::kChunkShift);
    if (it == chunks.end()) return nullptr;
    return reinterpret_cast<uint32_t*>(sv.V + (uint64_t)it->second * cgk::kSecondaryBytes) +
           ((q & ((1ull << cgk::kChunkShift) - 1)) >> 4);
  }
  std::map<uint64_t, uint64_t> live_arrays; // handle -> total bytes
  uint64_t last_seq = 0;
  // registry diff upload state (sync_table)
  uint64_t dev_n = 0, min_pos = 0, dev_stride = 0, uploads = 0;
  std::vector<std::pair<uint64_t, uint64_t>> patches;   // (position, free seq) below min_pos
  std::vector<uint64_t> pmax_host;                      // prefix max of ends by position
  bool arrays_dirty = false;
  int stage_slot = 0;
  uint64_t* h_tab[2] = {nullptr, nullptr};              // pinned staging, double buffered
  uint64_t* h_wlk[2] = {nullptr, nullptr};
  uint64_t* h_arr[2] = {nullptr, nullptr};
  uint64_t* h_patch[2] = {nullptr, nullptr};
  cudaEvent_t staged_ev[2] = {nullptr, nullptr};
  uint64_t pool_cursor = 0;                 // NEXT-1 bump allocator in dev_vbuf
  const void* last_check = nullptr;         // descriptors of the last check (for cg_apply_copies)
  uint64_t last_check_n = 0;
  // pinned staging
  cg_mark* h_marks = nullptr;               // kMarkRun
  cudaEvent_t staged = nullptr;             // the mark staging (h_marks) has been read
  cudaStream_t copy_stream = nullptr;        // host -> device uploads of cg_check_host
  cudaStream_t out_stream = nullptr;         // device -> host dirty-verdict downloads (cg_check_host_wait)
  cudaEvent_t chunk_ev[kHostSlots][kHostChunks] = {};
  cudaEvent_t slot_free[kHostSlots] = {};    // the slot's last batch stopped reading its staging
  cudaEvent_t slot_done[kHostSlots] = {};    // ... and its dirty count is on the host
  bool slot_busy[kHostSlots] = {};
  uint32_t* h_count = nullptr;               // pinned, one dirty count per slot
  bool wave_kernel = true;                   // cg_apply_copies_waves: one cooperative launch (env CG_WAVE_KERNEL=0: per wave)
  std::vector<uint32_t> h_wstart;            // its wave offsets, rebased, before upload
  uint64_t host_chunks = 2;                   // cg_check_host pipeline (env CG_HOST_CHUNKS / CG_HOST_GEOMETRIC)
  bool host_geometric = true;
  std::string err;
  // profiling (cg_profile_begin / end)
  cgk::Profiler prof;
  struct Rec { int stage; cudaEvent_t a, b; };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t open_ev[CG_STAGE_COUNT] = {};

  cudaEvent_t get_event() {
    if (!pool.empty()) { cudaEvent_t e = pool.back(); pool.pop_back(); return e; }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  static void mark_cb(void* self, int stage, bool begin, cudaStream_t s) {
    cg_ctx* c = static_cast<cg_ctx*>(self);
    cudaEvent_t e = c->get_event();
    cudaEventRecord(e, s);
    if (begin) c->open_ev[stage] = e;
    else c->recs.push_back({stage, c->open_ev[stage], e});
  }

  uint64_t* d(uint64_t off) { return reinterpret_cast<uint64_t*>(ws + off); }

  cg_status fail(cg_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    err = buf;
    return s;
  }
  cg_status cuda(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return CG_OK;
    return fail(CG_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  }

  cgk::Plan plan() {
    cgk::Plan p;
    p.weight = d(lay.weight);
    p.P = d(lay.P);
    p.bsum = d(lay.bsum);
    p.fbsum = d(lay.fbsum);
    p.chunk_first = reinterpret_cast<uint32_t*>(ws + lay.chunk);
    p.meta = ws + lay.meta;
    p.counter = reinterpret_cast<uint32_t*>(ws + lay.flags + 128);
    p.resid = reinterpret_cast<uint32_t*>(ws + lay.resid);
    p.defer = reinterpret_cast<uint32_t*>(ws + lay.defer);
    p.late = reinterpret_cast<uint32_t*>(ws + lay.late);
    p.last = reinterpret_cast<uint32_t*>(ws + lay.last);
    p.dvoff = cfg.dev_vbuf ? reinterpret_cast<uint64_t*>(ws + lay.dvoff) : nullptr;
    p.max_chunks = lay.max_chunks;
    p.t_min = kChunkMin;
    return p;
  }

  cgk::Table dev_table() {
    cgk::Table t;
    const uint64_t cap = cfg.max_allocs;
    uint64_t* b = d(lay.table);
    t.base = b;
    t.end = b + cap;
    t.aseq = b + 2 * cap;
    t.fseq = b + 3 * cap;
    t.pmax = b + 4 * cap;
    t.pool = cfg.dev_vbuf ? b + 5 * cap : nullptr;
    t.walk = reinterpret_cast<const uint4*>(d(lay.walk));
    t.split = b + ((6 * cap + 1) & ~1ull);   // 16-byte aligned
    t.l2 = b + l2_offset(cap);
    t.n = table.size();
    uint64_t* a = d(lay.arrays);
    t.ahandle = a;
    t.atotal = a + cap;
    t.aaseq = a + 2 * cap;
    t.afseq = a + 3 * cap;
    t.apool = cfg.dev_vbuf ? a + 4 * cap : nullptr;
    t.na = arrays.size();
    const uint64_t stride = split_stride(t.n);
    t.stride = (uint32_t)stride;
    t.nsplit = (uint32_t)((t.n + stride - 1) / stride);
    static const bool two = [] {   // measured slower than the binary search for C5 (1.58 vs 1.45 ms): opt-in
      const char* e = getenv("CG_LOOKUP64");
      return e && e[0] == '1';
    }();
    t.two_round64 = two ? 1u : 0u;
    return t;
  }

  // Registry upload by difference ("device table by diff
  // upload"): the device table equals the mirror except positions [min_pos, n)
  // (inserts shift the entries after them; a bump allocator only appends, so
  // usually just the new tail) and the free stamps in `patches` (frees of
  // entries below min_pos: 16 bytes each, scattered by k_table_patch).  The
  // pinned staging is double buffered (an event per buffer), so an upload
  // waits only for the one two uploads back, normally long finished.
  cg_status sync_table(cudaStream_t s) {
    const uint64_t n = table.size(), cap = cfg.max_allocs;
    if (min_pos >= n && n == dev_n && patches.empty() && !arrays_dirty) return CG_OK;
    const int slot = stage_slot;
    stage_slot ^= 1;
    cudaError_t e = cudaEventSynchronize(staged_ev[slot]);   // this buffer's previous upload has been read
    if (e != cudaSuccess) return cuda(e, "cudaEventSynchronize");
    uint64_t* ht = h_tab[slot];
    uint64_t* hw = h_wlk[slot];
    uint64_t* dt = d(lay.table);
    const uint64_t stride = split_stride(n), nsplit = (n + stride - 1) / stride;
    const uint64_t so = (6 * cap + 1) & ~1ull;
    const uint64_t a = std::min(min_pos, n);
    if (a < n) {   // positions [a, n): SoA columns, prefix max of ends, walk records
      uint64_t pm = a ? pmax_host[a - 1] : 0;
      pmax_host.resize(n);
      for (uint64_t i = a; i < n; ++i) {
        const Entry& x = table[i];
        ht[i] = x.base;
        ht[cap + i] = x.end;
        ht[2 * cap + i] = x.aseq;
        ht[3 * cap + i] = x.fseq;
        pm = std::max(pm, x.end);
        pmax_host[i] = pm;
        ht[4 * cap + i] = pm;
        ht[5 * cap + i] = x.pool;
        hw[4 * i] = pm;
        hw[4 * i + 1] = x.end;
        hw[4 * i + 2] = x.aseq;
        hw[4 * i + 3] = x.fseq;
      }
      for (int k = 0; k < 6; ++k) {
        e = cudaMemcpyAsync(dt + k * cap + a, ht + k * cap + a, (n - a) * 8, cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) return cuda(e, "table upload");
      }
      e = cudaMemcpyAsync(d(lay.walk) + 4 * a, hw + 4 * a, (n - a) * 32, cudaMemcpyHostToDevice, s);
      if (e != cudaSuccess) return cuda(e, "walk upload");
    }
    if (a < n || n != dev_n) {   // splitters (every stride-th base) and every 4th base from a on
      const uint64_t k0 = stride == dev_stride ? std::min(a / stride, nsplit) : 0;
      for (uint64_t k = k0; k < nsplit; ++k) ht[so + k] = table[k * stride].base;
      ht[so + nsplit] = UINT64_MAX;   // padding for the 16-byte loads
      e = cudaMemcpyAsync(dt + so + k0, ht + so + k0, (nsplit + 1 - k0) * 8, cudaMemcpyHostToDevice, s);
      const uint64_t hl2 = so + 4099 + 4 * cap, nl2 = (n + 3) / 4, j0 = std::min(a / 4, nl2);
      for (uint64_t k = j0; k < nl2; ++k) ht[hl2 + k] = table[4 * k].base;
      if (e == cudaSuccess && nl2 > j0)
        e = cudaMemcpyAsync(dt + l2_offset(cap) + j0, ht + hl2 + j0, (nl2 - j0) * 8, cudaMemcpyHostToDevice, s);
      if (e != cudaSuccess) return cuda(e, "splitter upload");
      dev_stride = stride;
    }
    if (!patches.empty()) {   // free stamps below a: (position, free seq) pairs
      uint64_t* hp = h_patch[slot];
      uint64_t k = 0;
      for (const auto& pr : patches) {
        if (pr.first >= a) continue;
        hp[2 * k] = pr.first;
        hp[2 * k + 1] = pr.second;
        ++k;
      }
      if (k) {
        uint64_t* dp = d(lay.patch);
        e = cudaMemcpyAsync(dp, hp, k * 16, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess) e = cgk::table_patch(launch, dt + 3 * cap, d(lay.walk), dp, k, s);
        if (e != cudaSuccess) return cuda(e, "free-stamp patch");
      }
    }
    if (arrays_dirty && !arrays.empty()) {
      uint64_t* ha = h_arr[slot];
      const uint64_t na = arrays.size();
      for (uint64_t i = 0; i < na; ++i) {
        ha[i] = arrays[i].handle;
        ha[cap + i] = arrays[i].total;
        ha[2 * cap + i] = arrays[i].aseq;
        ha[3 * cap + i] = arrays[i].fseq;
        ha[4 * cap + i] = arrays[i].pool;
      }
      uint64_t* da = d(lay.arrays);
      for (int k = 0; k < 5; ++k) {
        e = cudaMemcpyAsync(da + k * cap, ha + k * cap, na * 8, cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) return cuda(e, "array table upload");
      }
    }
    cudaEventRecord(staged_ev[slot], s);
    dev_n = n;
    min_pos = n;
    patches.clear();
    arrays_dirty = false;
    ++uploads;
    return CG_OK;
  }
  // the registry changed at position pos (insert: pos and everything after it move)
  void touch_insert(uint64_t pos) {
    min_pos = std::min(min_pos, pos);
    patches.erase(std::remove_if(patches.begin(), patches.end(),
                                 [&](const std::pair<uint64_t, uint64_t>& p) { return p.first >= pos; }),
                  patches.end());
  }
  void touch_free(uint64_t pos, uint64_t fseq) {
    if (pos < min_pos) patches.emplace_back(pos, fseq);
  }

  // word offset of the every-4th-base array in the device table (64-byte aligned)
  static uint64_t l2_offset(uint64_t cap) { return ((((6 * cap + 1) & ~1ull) + 4099) + 7) & ~7ull; }

  static uint64_t split_stride(uint64_t n) {
    const uint64_t stride = std::max<uint64_t>(32, (n + 4095) / 4096);
    return (stride + 31) / 32 * 32;   // whole 256-byte blocks of bases per bucket
  }

  uint32_t err_mask() const {
    return cfg.undef_is_error ? 0xffffffffu : ~(uint32_t)CG_F_HOST_UNDEFINED;
  }
};

extern "C" {

cg_status cg_apply_copies(cg_ctx* c, const cg_copy_desc* d_descs, const cg_verdict* d_verdicts, uint64_t n,
                          void* stream);
cg_status cg_apply_flush(cg_ctx* c, void* stream);

uint64_t cg_workspace_size(const cg_config* cfg) {
  if (!valid_config(cfg)) return 0;
  return layout_of(cfg).total;
}

cg_status cg_ctx_create(const cg_config* cfg, cg_ctx** out) {
  if (!out) return CG_ERR_INVALID_VALUE;
  *out = nullptr;
  if (!valid_config(cfg)) return CG_ERR_INVALID_VALUE;
  const Layout lay = layout_of(cfg);
  const bool sparse = cfg->shadow_format == CG_SHADOW_SPARSE;
  const bool two_bit = cfg->shadow_format == CG_SHADOW_2BIT || sparse;
  if (!cfg->v_buf || (!two_bit && !cfg->a_buf) || !cfg->workspace) return CG_ERR_INVALID_VALUE;
  if (cfg->workspace_size < lay.total) return CG_ERR_INVALID_VALUE;
  if ((uintptr_t)cfg->v_buf % 16 || (!two_bit && (uintptr_t)cfg->a_buf % 16) || (uintptr_t)cfg->workspace % kAlign)
    return CG_ERR_INVALID_VALUE;
  DeviceGuard g(cfg->device);
  cg_ctx* c = new cg_ctx();
  c->cfg = *cfg;
  c->lay = lay;
  c->ws = static_cast<uint8_t*>(cfg->workspace);
  c->sv.wb = cfg->host_base;
  c->sv.we = cfg->host_base + cfg->host_size;
  c->sv.sb = cfg->shard_size ? cfg->shard_base : cfg->host_base;
  c->sv.se = c->sv.sb + (cfg->shard_size ? cfg->shard_size : cfg->host_size);
  c->sv.V = static_cast<uint8_t*>(cfg->v_buf);
  c->sv.A = two_bit ? nullptr : static_cast<uint8_t*>(cfg->a_buf);
  c->sv.two_bit = two_bit ? 1u : 0u;
  c->sv.sparse = sparse ? 1u : 0u;
  c->sv.v_bytes = sparse ? (cfg->host_size / 65536 + 1) * cgk::kSecondaryBytes : two_bit ? cfg->host_size / 4
                                                                                          : cfg->host_size;
  if (cfg->shard_size && !sparse) c->sv.v_bytes = two_bit ? cfg->shard_size / 4 : cfg->shard_size;
  c->sv.small_limit = cgk::kSmallBytesDefault;
  // the stage holds a side of at most 4 KiB (bytes format) / 16 KiB (2-bit states)
  if (const char* sl = getenv("CG_SMALL_BYTES"))
    c->sv.small_limit = std::min<uint64_t>(strtoull(sl, nullptr, 10), two_bit ? 16384 : 4096);
  c->sv.small_mode = 0;
  if (const char* sm = getenv("CG_SMALL_MODE")) c->sv.small_mode = (uint32_t)std::min<uint64_t>(strtoull(sm, nullptr, 10), 2);
  c->sv.small_share = two_bit ? 50u : 80u;
  if (const char* sh = getenv("CG_SMALL_SHARE")) c->sv.small_share = (uint32_t)std::min<uint64_t>(strtoull(sh, nullptr, 10), 100);
  c->sv.small_stat = cgk::kSmallStatDefault;
  if (const char* ss = getenv("CG_SMALL_STAT")) c->sv.small_stat = strtoull(ss, nullptr, 10);
  if (sparse) {   // the whole 64-bit space; the directory lives in the workspace
    c->sv.wb = c->sv.sb = 0;
    c->sv.we = c->sv.se = UINT64_MAX;
    c->sv.dir_bits = lay.dir_bits;
    c->sv.dir_key = reinterpret_cast<const uint64_t*>(c->ws + lay.dir);
    c->sv.dir_val = reinterpret_cast<const uint32_t*>(c->ws + lay.dir + (8ull << lay.dir_bits));
    c->sv.chunk_list = reinterpret_cast<const uint64_t*>(c->ws + lay.chunk_list);
    c->dir_host.assign((1ull << lay.dir_bits) * 3, 0u);   // keys (2 words each) + values
  }
  cudaDeviceProp prop;
  cudaError_t e = cudaGetDeviceProperties(&prop, cfg->device);
  if (e != cudaSuccess) {
    delete c;
    return CG_ERR_CUDA;
  }
  c->launch.num_sms = prop.multiProcessorCount;
  c->launch.persist_blocks = prop.multiProcessorCount * std::max(cgk::persistent_blocks(1), 1);
  c->launch.scan_blocks = prop.multiProcessorCount * std::max(cgk::persistent_blocks(0), 1);
  c->launch.wave_blocks = prop.multiProcessorCount * std::max(cgk::persistent_blocks(2), 1);
  c->launch.front_blocks = std::min(prop.multiProcessorCount * cgk::persistent_blocks(4), (int)cgk::kFinishMaxBlocks);
  if (const char* fr = getenv("CG_FRONT_COOP")) if (atoi(fr) == 0) c->launch.front_blocks = 0;
  c->launch.leak_blocks = std::min(prop.multiProcessorCount * cgk::persistent_blocks(5), (int)cgk::kFinishMaxBlocks);
  c->launch.small_blocks = prop.multiProcessorCount * std::max(cgk::persistent_blocks(6), 1);
  if (const char* lk = getenv("CG_LEAK_COOP")) if (atoi(lk) == 0) c->launch.leak_blocks = 0;

  c->launch.finish_blocks = std::min(prop.multiProcessorCount * std::max(cgk::persistent_blocks(3), 1),
                                     (int)cgk::kFinishMaxBlocks);
  c->launch.counter = &c->launches;
  c->prof.mark = &cg_ctx::mark_cb;
  c->prof.self = c;
  c->launch.prof = &c->prof;
  bool pinned_ok = cudaMallocHost(&c->h_marks, std::min<uint64_t>(cfg->max_descs, kMarkRun) * sizeof(cg_mark)) ==
                       cudaSuccess &&
                   cudaEventCreateWithFlags(&c->staged, cudaEventDisableTiming) == cudaSuccess;
  for (int k = 0; k < 2 && pinned_ok; ++k)
    pinned_ok = cudaMallocHost(&c->h_tab[k], 10 * cfg->max_allocs * 8 + (4096 + 5) * 8 + (cfg->max_allocs / 4 + 16) * 8) ==
                    cudaSuccess &&
                cudaMallocHost(&c->h_wlk[k], 4 * cfg->max_allocs * sizeof(uint64_t)) == cudaSuccess &&
                cudaMallocHost(&c->h_arr[k], 5 * cfg->max_allocs * sizeof(uint64_t)) == cudaSuccess &&
                cudaMallocHost(&c->h_patch[k], 2 * cfg->max_allocs * sizeof(uint64_t)) == cudaSuccess &&
                cudaEventCreateWithFlags(&c->staged_ev[k], cudaEventDisableTiming) == cudaSuccess &&
                cudaEventRecord(c->staged_ev[k], 0) == cudaSuccess;
  if (!pinned_ok) {
    cg_ctx_destroy(c);
    return CG_ERR_OUT_OF_MEMORY;
  }
  cudaEventRecord(c->staged, 0);
  if (const char* hc = getenv("CG_HOST_CHUNKS")) c->host_chunks = std::min<uint64_t>(std::max(atoi(hc), 1), kHostChunks);
  if (const char* hg = getenv("CG_HOST_GEOMETRIC")) c->host_geometric = atoi(hg) != 0;
  if (const char* wk = getenv("CG_WAVE_KERNEL")) c->wave_kernel = atoi(wk) != 0;
  if (cfg->host_staging) {
    if (cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->out_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaMallocHost(&c->h_count, kHostSlots * sizeof(uint32_t)) != cudaSuccess) {
      cg_ctx_destroy(c);
      return CG_ERR_CUDA;
    }
    for (auto& slot : c->chunk_ev)
      for (auto& ev : slot) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    for (uint32_t k = 0; k < kHostSlots; ++k) {
      cudaEventCreateWithFlags(&c->slot_free[k], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&c->slot_done[k], cudaEventDisableTiming);
      cudaEventRecord(c->slot_free[k], 0);
    }
  }
  e = cudaMemset(c->ws + lay.flags, 0, 256);   // counters, overflow flag
  if (e == cudaSuccess) e = cgk::fresh_shadow(c->launch, c->sv, 0);
  if (e == cudaSuccess && cfg->dev_vbuf) e = cudaMemset(cfg->dev_vbuf, 0xFF, cfg->dev_vsize);
  if (e == cudaSuccess && cfg->dev_vbuf) e = cudaMemset(c->ws + lay.ovl, 0, 8);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    cg_ctx_destroy(c);
    return CG_ERR_CUDA;
  }
  *out = c;
  return CG_OK;
}

cg_status cg_ctx_destroy(cg_ctx* c) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  DeviceGuard g(c->cfg.device);
  if (c->staged) {
    cudaEventSynchronize(c->staged);
    cudaEventDestroy(c->staged);
  }
  if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);
  if (c->out_stream) cudaStreamSynchronize(c->out_stream);
  for (auto& slot : c->chunk_ev)
    for (auto& ev : slot)
      if (ev) cudaEventDestroy(ev);
  for (uint32_t k = 0; k < kHostSlots; ++k) {
    if (c->slot_free[k]) cudaEventDestroy(c->slot_free[k]);
    if (c->slot_done[k]) cudaEventSynchronize(c->slot_done[k]), cudaEventDestroy(c->slot_done[k]);
  }
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  if (c->out_stream) cudaStreamDestroy(c->out_stream);
  if (c->h_count) cudaFreeHost(c->h_count);
  for (auto& r : c->recs) { c->pool.push_back(r.a); c->pool.push_back(r.b); }
  for (cudaEvent_t e : c->pool) cudaEventDestroy(e);
  for (int k = 0; k < 2; ++k) {
    if (c->staged_ev[k]) {
      cudaEventSynchronize(c->staged_ev[k]);
      cudaEventDestroy(c->staged_ev[k]);
    }
    if (c->h_tab[k]) cudaFreeHost(c->h_tab[k]);
    if (c->h_wlk[k]) cudaFreeHost(c->h_wlk[k]);
    if (c->h_arr[k]) cudaFreeHost(c->h_arr[k]);
    if (c->h_patch[k]) cudaFreeHost(c->h_patch[k]);
  }
  if (c->h_marks) cudaFreeHost(c->h_marks);
  delete c;
  return CG_OK;
}

const char* cg_last_error(const cg_ctx* c) { return c ? c->err.c_str() : "null context"; }

uint64_t cg_kernel_launches(const cg_ctx* c) { return c ? c->launches : 0; }

static const char* direction(uint32_t kind) {
  return kind == CG_HTOD ? "host->device" : kind == CG_DTOH ? "device->host" : kind == CG_HTOA ? "host->array"
         : kind == CG_ATOH ? "array->host" : "device->device";
}

uint64_t cg_format_verdict(const cg_verdict* v, uint32_t kind, char* buf, uint64_t cap) {
  std::string t;
  char line[256];
  auto add = [&](const char* fmt, auto... args) {
    snprintf(line, sizeof line, fmt, args...);
    t += line;
  };
  if (!v) return 0;
  const char* dir = direction(kind);
  const char* mem = kind == CG_HTOA || kind == CG_ATOH ? "device array" : "device memory";
  const unsigned long long de = v->dst_expected, df = v->dst_found, se = v->src_expected, sf = v->src_found;
  const unsigned long long fu = v->first_unaddr, fd = v->first_undef, uc = v->undef_count;
  if (v->flags & CG_F_DST_NOT_ALLOCATED) add("Error: Destination %s of %s copy is not allocated.\n", mem, dir);
  if (v->flags & CG_F_DST_TOO_SMALL)
    add("Error: Allocated %s too small for %s copy.\nExpected %llu allocated bytes but only found %llu.\n",
        mem, dir, de, df);
  if (v->flags & CG_F_SRC_NOT_ALLOCATED) add("Error: Source %s of %s copy is not allocated.\n", mem, dir);
  if (v->flags & CG_F_SRC_TOO_SMALL)
    add("Error: Allocated %s too small for %s copy.\nExpected %llu allocated bytes but only found %llu.\n",
        mem, dir, se, sf);
  if (v->flags & CG_F_HOST_UNADDRESSABLE)
    add("Error: Host memory of %s copy is not addressable (first unaddressable byte at offset %llu).\n", dir, fu);
  if (v->flags & CG_F_HOST_UNDEFINED)
    add("Warning: Undefined host data in %s copy (%llu undefined bytes, first at offset %llu).\n", dir, uc, fd);
  if (v->flags & CG_F_BAD_PITCH) add("Error: Pitch of %s copy smaller than width plus X offset.\n", dir);
  if (v->flags & CG_F_INVALID_RANGE) add("Error: Address range of %s copy overflows.\n", dir);
  if (v->flags & CG_F_BAD_KIND) add("Error: Unknown copy kind %u.\n", kind);
  if (cap) {
    const uint64_t m = std::min<uint64_t>(t.size(), cap - 1);
    if (buf) {
      std::memcpy(buf, t.data(), m);
      buf[m] = 0;
    }
  }
  return t.size();
}

cg_status cg_summarize(const cg_verdict* d_verdicts, uint64_t n, uint32_t undef_is_error, uint64_t* d_counts,
                       void* stream) {
  if (!d_counts || (n && !d_verdicts)) return CG_ERR_INVALID_VALUE;
  const uint32_t warn = CG_F_CONCURRENT | (undef_is_error ? 0u : (uint32_t)CG_F_HOST_UNDEFINED);
  cudaError_t e = cgk::summarize(d_verdicts, n, warn, reinterpret_cast<unsigned long long*>(d_counts),
                                 static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? CG_OK : CG_ERR_CUDA;
}

uint64_t cg_format_summary(uint64_t errors, uint64_t warnings, uint64_t suppressed, char* buf, uint64_t cap) {
  char line[160];
  const int k = snprintf(line, sizeof line, "ERROR SUMMARY: %llu errors, %llu warnings (%llu suppressed)\n",
                         (unsigned long long)errors, (unsigned long long)warnings, (unsigned long long)suppressed);
  if (cap && buf) {
    const uint64_t m = std::min<uint64_t>((uint64_t)k, cap - 1);
    std::memcpy(buf, line, m);
    buf[m] = 0;
  }
  return (uint64_t)k;
}

uint64_t cg_format_leak(const cg_alloc_record* r, char* buf, uint64_t cap) {
  if (!r) return 0;
  char line[128];
  const int k = snprintf(line, sizeof line, "Warning: Device memory leak of %llu bytes.\n", (unsigned long long)r->size);
  if (cap && buf) {
    const uint64_t m = std::min<uint64_t>((uint64_t)k, cap - 1);
    std::memcpy(buf, line, m);
    buf[m] = 0;
  }
  return (uint64_t)k;
}

cg_status cg_profile_begin(cg_ctx* c) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  c->prof.on = true;
  return CG_OK;
}

cg_status cg_profile_end(cg_ctx* c, double* ms, uint64_t* launches) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  DeviceGuard g(c->cfg.device);
  c->prof.on = false;
  double acc[CG_STAGE_COUNT] = {};
  uint64_t cnt[CG_STAGE_COUNT] = {};
  cg_status st = CG_OK;
  for (auto& r : c->recs) {
    cudaError_t e = cudaEventSynchronize(r.b);
    float t = 0.f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&t, r.a, r.b);
    if (e != cudaSuccess) st = c->cuda(e, "profile events");
    acc[r.stage] += t;
    cnt[r.stage] += 1;
    c->pool.push_back(r.a);
    c->pool.push_back(r.b);
  }
  c->recs.clear();
  for (int k = 0; k < CG_STAGE_COUNT; ++k) {
    if (ms) ms[k] = acc[k];
    if (launches) launches[k] = cnt[k];
  }
  return st;
}

static bool in_window(const cg_ctx* c, uint64_t addr, uint64_t len) {
  if (c->sv.sparse) return len <= UINT64_MAX - addr;
  return addr >= c->sv.wb && len <= c->sv.we - c->sv.wb && addr - c->sv.wb <= (c->sv.we - c->sv.wb) - len;
}

cg_status cg_host_mark_batch(cg_ctx* c, const cg_mark* h_marks, uint64_t n, uint32_t* h_status, void* stream) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  if (n == 0) return CG_OK;
  if (!h_marks) return c->fail(CG_ERR_INVALID_VALUE, "null marks");
  DeviceGuard g(c->cfg.device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint64_t cap = std::min<uint64_t>(c->cfg.max_descs, kMarkRun);
  cg_mark* dm = reinterpret_cast<cg_mark*>(c->ws + c->lay.marks);
  cg_status ret = CG_OK;
  // runs of pairwise-disjoint valid marks are applied in parallel, runs in order
  uint64_t i = 0;
  while (i < n) {
    std::map<uint64_t, uint64_t> run;   // start -> end of the marks of this run
    uint64_t j = i, k = 0;
    cudaError_t e = cudaEventSynchronize(c->staged);   // the previous run's upload has been read
    if (e != cudaSuccess) return c->cuda(e, "cudaEventSynchronize");
    while (j < n && k < cap) {
      const cg_mark& m = h_marks[j];
      const bool valid = m.state <= CG_DEFINED && (m.len == 0 || in_window(c, m.addr, m.len));
      if (h_status) h_status[j] = valid ? CG_OK : CG_ERR_INVALID_VALUE;
      if (!valid) {
        ret = c->fail(CG_ERR_INVALID_VALUE, "mark %llu invalid (state or range)", (unsigned long long)j);
        ++j;
        continue;
      }
      if (m.len) {
        const uint64_t a = m.addr, b = m.addr + m.len;
        auto it = run.upper_bound(a);
        bool overlap = (it != run.end() && it->first < b);
        if (!overlap && it != run.begin()) overlap = std::prev(it)->second > a;
        if (overlap) break;
        if (c->sv.sparse && m.state != CG_NOACCESS && !c->ensure_chunks(a, b)) {   // NEXT-4: pool full
          if (h_status) h_status[j] = CG_ERR_OUT_OF_MEMORY;
          ret = c->fail(CG_ERR_OUT_OF_MEMORY, "sparse host map: no secondary left for mark %llu",
                        (unsigned long long)j);
          ++j;
          continue;
        }
        run.emplace(a, b);
        c->h_marks[k++] = m;
      }
      ++j;
    }
    if (k) {
      if (c->upload_dir(s) != CG_OK) return CG_ERR_CUDA;
      e = cudaMemcpyAsync(dm, c->h_marks, k * sizeof(cg_mark), cudaMemcpyHostToDevice, s);
      if (e != cudaSuccess) return c->cuda(e, "marks upload");
      e = cgk::mark_batch(c->launch, dm, k, c->sv, c->plan(), s);
      if (e != cudaSuccess) return c->cuda(e, "mark kernels");
      cudaEventRecord(c->staged, s);
    }
    i = j;
  }
  return ret;
}

cg_status cg_host_mark(cg_ctx* c, uint64_t addr, uint64_t len, uint32_t state, void* stream) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  cg_mark m{addr, len, state, 0};
  return cg_host_mark_batch(c, &m, 1, nullptr, stream);
}

cg_status cg_host_set_vbits(cg_ctx* c, uint64_t addr, uint64_t len, const uint8_t* h_vbytes, void* stream) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  if (len == 0) return CG_OK;
  if (!h_vbytes) return c->fail(CG_ERR_INVALID_VALUE, "null vbytes");
  if (!in_window(c, addr, len)) return c->fail(CG_ERR_INVALID_VALUE, "set_vbits range outside the host window");
  DeviceGuard g(c->cfg.device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint64_t y0 = std::max(addr, c->sv.sb), y1 = std::min(addr + len, c->sv.se);
  if (y0 >= y1) return CG_OK;   // nothing of it in this shard
  uint32_t* flag = reinterpret_cast<uint32_t*>(c->ws + c->lay.flags);
  cudaError_t e = cgk::setv_check(c->launch, addr, len, c->sv, flag, s);
  uint32_t h_flag = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h_flag, flag, sizeof h_flag, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return c->cuda(e, "set_vbits check");
  if (h_flag) return c->fail(CG_ERR_INVALID_VALUE, "set_vbits on unaddressable bytes");
  if (c->sv.two_bit) {   // NEXT-4: read-modify-write the state words; exact partial V-bytes go to the host table
    const uint64_t q0 = y0 - c->sv.sb, q1 = y1 - c->sv.sb;
    for (uint64_t a = q0; a < q1;) {   // pieces that stay inside one chunk of the sparse map
      const uint64_t rem = c->sv.sparse ? (1ull << cgk::kChunkShift) - (a & ((1ull << cgk::kChunkShift) - 1)) : q1 - a;
      const uint64_t b = q1 - a <= rem ? q1 : a + rem;
      const uint64_t k0 = a >> 4, k1 = (b + 15) >> 4;
      uint32_t* S = c->state_word(a);   // addressable, so its chunk has a secondary
      std::vector<uint32_t> w(k1 - k0);
      e = cudaMemcpyAsync(w.data(), S, w.size() * 4, cudaMemcpyDeviceToHost, s);
      if (e == cudaSuccess) e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) return c->cuda(e, "set_vbits read");
      for (uint64_t q = a; q < b; ++q) {
        const uint8_t v = h_vbytes[q - q0 + (y0 - addr)];
        const uint32_t st = v == 0x00 ? cgk::kSt2Defined : v == 0xFF ? cgk::kSt2Undefined : cgk::kSt2Partial;
        uint32_t& x = w[(q >> 4) - k0];
        const int sh = 2 * (int)(q & 15);
        x = (x & ~(3u << sh)) | (st << sh);
        if (st == cgk::kSt2Partial) c->partial[q + c->sv.sb] = v;
        else c->partial.erase(q + c->sv.sb);
      }
      e = cudaMemcpyAsync(S, w.data(), w.size() * 4, cudaMemcpyHostToDevice, s);
      if (e == cudaSuccess) e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) return c->cuda(e, "set_vbits write");
      a = b;
    }
    return CG_OK;
  }
  e = cudaMemcpyAsync(c->sv.V + (y0 - c->sv.sb), h_vbytes + (y0 - addr), y1 - y0, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  return c->cuda(e, "set_vbits copy");
}

cg_status cg_host_shadow_read(cg_ctx* c, uint64_t addr, uint64_t len, uint8_t* h_a, uint8_t* h_v, void* stream) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  if (len == 0) return CG_OK;
  if (addr < c->sv.sb || addr > c->sv.se || len > c->sv.se - addr)
    return c->fail(CG_ERR_INVALID_VALUE, "shadow read outside this context's shard");
  if (c->sv.sparse && len > (1ull << 32)) return c->fail(CG_ERR_INVALID_VALUE, "sparse shadow read above 4 GiB");
  DeviceGuard g(c->cfg.device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint64_t q0 = addr - c->sv.sb, q1 = q0 + len;
  cudaError_t e = cudaSuccess;
  if (c->sv.two_bit) {
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return c->cuda(e, "shadow read");
    for (uint64_t a = q0; a < q1;) {   // pieces that stay inside one chunk of the sparse map
      const uint64_t rem = c->sv.sparse ? (1ull << cgk::kChunkShift) - (a & ((1ull << cgk::kChunkShift) - 1)) : q1 - a;
      const uint64_t b = q1 - a <= rem ? q1 : a + rem;
      const uint64_t k0 = a >> 4, k1 = (b + 15) >> 4;
      std::vector<uint32_t> w(k1 - k0, 0u);   // a chunk without a secondary reads as NOACCESS
      if (uint32_t* S = c->state_word(a)) {
        e = cudaMemcpy(w.data(), S, w.size() * 4, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) return c->cuda(e, "shadow read");
      }
      for (uint64_t q = a; q < b; ++q) {
        const uint32_t st = (w[(q >> 4) - k0] >> (2 * (q & 15))) & 3u;
      if (h_a) h_a[q - q0] = st != cgk::kSt2NoAccess;
      if (h_v) {
        uint8_t v = st == cgk::kSt2Defined ? 0x00 : 0xFF;
        if (st == cgk::kSt2Partial) {
          auto it = c->partial.find(q + c->sv.sb);
          v = it != c->partial.end() ? it->second : 0xFF;
        }
        h_v[q - q0] = v;
      }
      }
      a = b;
    }
    return CG_OK;
  }
  if (h_v) e = cudaMemcpyAsync(h_v, c->sv.V + q0, len, cudaMemcpyDeviceToHost, s);
  std::vector<uint8_t> a;
  if (e == cudaSuccess && h_a) {
    a.resize((q1 + 7) / 8 - q0 / 8);
    e = cudaMemcpyAsync(a.data(), c->sv.A + q0 / 8, a.size(), cudaMemcpyDeviceToHost, s);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return c->cuda(e, "shadow read");
  if (h_a)
    for (uint64_t q = q0; q < q1; ++q) h_a[q - q0] = (a[q / 8 - q0 / 8] >> (q & 7)) & 1u;
  return CG_OK;
}

cg_status cg_host_query_addressable(cg_ctx* c, uint64_t addr, uint64_t len, uint32_t* all_addressable, void* stream) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  if (!all_addressable) return c->fail(CG_ERR_INVALID_VALUE, "null output");
  *all_addressable = 1;
  if (len == 0) return CG_OK;
  if (!in_window(c, addr, len)) {
    *all_addressable = 0;
    return CG_OK;
  }
  const uint64_t y0 = std::max(addr, c->sv.sb), y1 = std::min(addr + len, c->sv.se);
  if (y0 >= y1) return CG_OK;
  DeviceGuard g(c->cfg.device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint32_t* flag = reinterpret_cast<uint32_t*>(c->ws + c->lay.flags);
  cudaError_t e = cgk::setv_check(c->launch, addr, len, c->sv, flag, s);
  uint32_t h_flag = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h_flag, flag, sizeof h_flag, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return c->cuda(e, "addressability query");
  *all_addressable = h_flag ? 0 : 1;
  return CG_OK;
}

cg_status cg_register_alloc(cg_ctx* c, uint64_t base, uint64_t size, uint64_t seq) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  if (size == 0 || base == 0) return c->fail(CG_ERR_INVALID_VALUE, "register: size 0 or base 0");
  if (size > UINT64_MAX - base) return c->fail(CG_ERR_INVALID_VALUE, "register: range overflows");
  if (seq <= c->last_seq) return c->fail(CG_ERR_INVALID_VALUE, "register: seq not increasing");
  const uint64_t end = base + size;
  auto it = c->live.lower_bound(base);
  if (it != c->live.end() && it->first < end)
    return c->fail(CG_ERR_INVALID_VALUE, "register: overlaps a live allocation");
  if (it != c->live.begin() && std::prev(it)->second > base)
    return c->fail(CG_ERR_INVALID_VALUE, "register: overlaps a live allocation");
  if (c->table.size() >= c->cfg.max_allocs) return c->fail(CG_ERR_OUT_OF_MEMORY, "allocation table full");
  uint64_t pool = 0;
  if (c->cfg.dev_vbuf) {   // NEXT-1: V-bits of the allocation, same alignment mod 256 as its base
    pool = (c->pool_cursor + 255) / 256 * 256 + (base & 255);
    if (pool + size > c->cfg.dev_vsize || pool + size < pool)
      return c->fail(CG_ERR_OUT_OF_MEMORY, "device V-bit pool full");
  }
  Entry x{base, end, seq, cgk::kInf, pool};
  if (c->cfg.dev_vbuf) c->pool_cursor = pool + size;
  auto pos = std::upper_bound(c->table.begin(), c->table.end(), base,
                              [](uint64_t b, const Entry& e) { return b < e.base; });
  c->touch_insert((uint64_t)(pos - c->table.begin()));
  c->table.insert(pos, x);
  c->live.emplace(base, end);
  c->last_seq = seq;
  return CG_OK;
}

cg_status cg_free(cg_ctx* c, uint64_t ptr, uint64_t seq) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  if (seq <= c->last_seq) return c->fail(CG_ERR_INVALID_VALUE, "free: seq not increasing");
  auto it = c->live.find(ptr);
  if (it == c->live.end()) return c->fail(CG_ERR_INVALID_VALUE, "InvalidFree: not a live base");
  auto pos = std::lower_bound(c->table.begin(), c->table.end(), ptr,
                              [](const Entry& e, uint64_t b) { return e.base < b; });
  for (; pos != c->table.end() && pos->base == ptr; ++pos) {
    if (pos->fseq == cgk::kInf) {
      pos->fseq = seq;
      c->touch_free((uint64_t)(pos - c->table.begin()), seq);
      break;
    }
  }
  c->live.erase(it);
  c->last_seq = seq;
  return CG_OK;
}

cg_status cg_registry_batch(cg_ctx* c, const cg_reg_event* h_events, uint64_t n, uint32_t* h_status) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  if (n && !h_events) return c->fail(CG_ERR_INVALID_VALUE, "null events");
  cg_status first = CG_OK;
  for (uint64_t i = 0; i < n; ++i) {
    const cg_reg_event& e = h_events[i];
    const cg_status st = e.op == CG_REG_ALLOC ? cg_register_alloc(c, e.addr, e.size, e.seq)
                         : e.op == CG_REG_FREE ? cg_free(c, e.addr, e.seq)
                                               : c->fail(CG_ERR_INVALID_VALUE, "unknown registry op");
    if (h_status) h_status[i] = (uint32_t)st;
    if (st != CG_OK && first == CG_OK) first = st;
  }
  return first;
}

cg_status cg_registry_compact(cg_ctx* c, uint64_t before_seq) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  auto it = std::remove_if(c->table.begin(), c->table.end(),
                           [&](const Entry& e) { return e.fseq != cgk::kInf && e.fseq <= before_seq; });
  if (it != c->table.end()) {
    c->touch_insert(0);   // entries move: re-upload all of them
    c->table.erase(it, c->table.end());
  }
  auto ia = std::remove_if(c->arrays.begin(), c->arrays.end(),
                           [&](const ArrayEntry& e) { return e.fseq != cgk::kInf && e.fseq <= before_seq; });
  if (ia != c->arrays.end()) {
    c->arrays.erase(ia, c->arrays.end());
    c->arrays_dirty = true;
  }
  return CG_OK;
}

uint64_t cg_array_bytes(uint64_t width, uint64_t height, uint64_t depth, uint32_t format, uint32_t channels) {
  static const uint64_t fb[8] = {1, 2, 4, 1, 2, 4, 2, 4};
  if (width == 0 || format > 7 || (channels != 1 && channels != 2 && channels != 4)) return 0;
  unsigned __int128 t = (unsigned __int128)width * (height ? height : 1) * (depth ? depth : 1);
  t *= fb[format] * channels;
  return t > (unsigned __int128)UINT64_MAX ? 0 : (uint64_t)t;
}

cg_status cg_register_array(cg_ctx* c, uint64_t handle, uint64_t width, uint64_t height, uint64_t depth,
                            uint32_t format, uint32_t channels, uint64_t seq) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  const uint64_t total = cg_array_bytes(width, height, depth, format, channels);
  if (total == 0) return c->fail(CG_ERR_INVALID_VALUE, "register_array: zero extent or bad descriptor");
  if (seq <= c->last_seq) return c->fail(CG_ERR_INVALID_VALUE, "register_array: seq not increasing");
  if (c->live_arrays.count(handle)) return c->fail(CG_ERR_INVALID_VALUE, "register_array: DuplicateHandle");
  if (c->arrays.size() >= c->cfg.max_allocs) return c->fail(CG_ERR_OUT_OF_MEMORY, "array table full");
  auto pos = std::upper_bound(c->arrays.begin(), c->arrays.end(), handle,
                              [](uint64_t h, const ArrayEntry& e) { return h < e.handle; });
  uint64_t pool = 0;
  if (c->cfg.dev_vbuf) {   // NEXT-1: the array's V-bits, fresh = undefined (the pool starts 0xFF, never reused)
    pool = (c->pool_cursor + 15) / 16 * 16;
    if (pool + total > c->cfg.dev_vsize || pool + total < pool)
      return c->fail(CG_ERR_OUT_OF_MEMORY, "device V-bit pool full");
    c->pool_cursor = pool + total;
  }
  c->arrays.insert(pos, ArrayEntry{handle, total, seq, cgk::kInf, pool});
  c->live_arrays.emplace(handle, total);
  c->last_seq = seq;
  c->arrays_dirty = true;
  return CG_OK;
}

cg_status cg_free_array(cg_ctx* c, uint64_t handle, uint64_t seq) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  if (seq <= c->last_seq) return c->fail(CG_ERR_INVALID_VALUE, "free_array: seq not increasing");
  auto it = c->live_arrays.find(handle);
  if (it == c->live_arrays.end()) return c->fail(CG_ERR_INVALID_VALUE, "free_array: UnknownHandle");
  auto pos = std::lower_bound(c->arrays.begin(), c->arrays.end(), handle,
                              [](const ArrayEntry& e, uint64_t h) { return e.handle < h; });
  for (; pos != c->arrays.end() && pos->handle == handle; ++pos) {
    if (pos->fseq == cgk::kInf) {
      pos->fseq = seq;
      break;
    }
  }
  c->live_arrays.erase(it);
  c->last_seq = seq;
  c->arrays_dirty = true;
  return CG_OK;
}

cg_status cg_array_report(cg_ctx* c, cg_alloc_record* h_out, uint64_t cap, uint64_t* n_out) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  if (!n_out || (cap && !h_out)) return c->fail(CG_ERR_INVALID_VALUE, "null output");
  uint64_t k = 0;
  for (const ArrayEntry& e : c->arrays) {
    if (e.fseq != cgk::kInf) continue;
    if (k < cap) h_out[k] = cg_alloc_record{e.handle, e.total, e.aseq};
    ++k;
  }
  *n_out = k;
  return CG_OK;
}

cg_status cg_check_copies(cg_ctx* c, const cg_copy_desc* d_descs, uint64_t n, cg_verdict* d_out, void* stream) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  if (n == 0) return CG_OK;
  if (!d_descs || !d_out) return c->fail(CG_ERR_INVALID_VALUE, "null descriptor or verdict array");
  if ((uintptr_t)d_descs % 16 || (uintptr_t)d_out % 16) return c->fail(CG_ERR_INVALID_VALUE, "arrays not 16-byte aligned");
  if (n > c->cfg.max_descs) return c->fail(CG_ERR_INVALID_VALUE, "n > max_descs");
  DeviceGuard g(c->cfg.device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cg_status st = c->sync_table(s);
  if (st != CG_OK) return st;
  cudaError_t e =
      cgk::check_copies(c->launch, d_descs, n, d_out, c->dev_table(), c->sv, c->plan(), c->err_mask(), false, s);
  c->last_check = d_descs;
  c->last_check_n = n;
  return c->cuda(e, "check kernels");
}

cg_status cg_apply_dtoh(cg_ctx* c, const cg_copy_desc* d_descs, const cg_verdict* d_verdicts, uint64_t n,
                        void* stream) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  if (c->cfg.dev_vbuf) return cg_apply_copies(c, d_descs, d_verdicts, n, stream);   // NEXT-1: a6 moves V-bits
  if (n == 0) return CG_OK;
  if (!d_descs || !d_verdicts) return c->fail(CG_ERR_INVALID_VALUE, "null descriptor or verdict array");
  if (n > c->cfg.max_descs) return c->fail(CG_ERR_INVALID_VALUE, "n > max_descs");
  DeviceGuard g(c->cfg.device);
  cudaError_t e =
      cgk::apply_dtoh(c->launch, d_descs, d_verdicts, n, c->sv, c->plan(), false, static_cast<cudaStream_t>(stream));
  return c->cuda(e, "apply kernels");
}

cg_status cg_apply_copies_subset(cg_ctx* c, const cg_copy_desc* d_descs, const cg_verdict* d_verdicts, uint64_t n,
                                 const uint32_t* d_index, uint64_t m, uint64_t max_bytes, void* stream) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  if (!c->cfg.dev_vbuf) return c->fail(CG_ERR_NOT_INITIALIZED, "no device V-bit tracking");
  if (n == 0 || m == 0) return CG_OK;
  if (!d_descs || !d_verdicts || !d_index) return c->fail(CG_ERR_INVALID_VALUE, "null descriptor, verdict or index array");
  if (m > n) return c->fail(CG_ERR_INVALID_VALUE, "m > n");
  if (d_descs != c->last_check || n != c->last_check_n)
    return c->fail(CG_ERR_INVALID_VALUE, "cg_apply_copies must follow the check of the same descriptors");
  DeviceGuard g(c->cfg.device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint32_t* overflow = reinterpret_cast<uint32_t*>(c->ws + c->lay.ovl);
  // asynchronous: a staging overflow stays flagged until cg_apply_flush.  Waves
  // of copies up to kDirectMax bytes take the plan-free warp-per-copy kernel.
  constexpr uint64_t kDirectMax = 1ull << 20;
  uint8_t* pool = static_cast<uint8_t*>(c->cfg.dev_vbuf);
  cudaError_t e = max_bytes && max_bytes <= kDirectMax
                      ? cgk::propagate_direct(c->launch, d_descs, d_verdicts, d_index, m, max_bytes, c->sv, pool,
                                              c->plan(), c->ws + c->lay.scratch, overflow, s)
                      : cgk::propagate(c->launch, d_descs, d_verdicts, d_index, m, c->sv, pool, c->plan(),
                                       c->ws + c->lay.scratch, overflow, s, false);
  return c->cuda(e, "propagate");
}

cg_status cg_apply_copies_waves(cg_ctx* c, const cg_copy_desc* d_descs, const cg_verdict* d_verdicts, uint64_t n,
                                const uint32_t* d_index, const uint64_t* h_wave_start, const uint64_t* h_max_bytes,
                                uint32_t n_waves, void* stream) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  if (n_waves && (!h_wave_start || !h_max_bytes)) return c->fail(CG_ERR_INVALID_VALUE, "null wave arrays");
  for (uint32_t w = 0; w < n_waves; ++w)
    if (h_wave_start[w + 1] < h_wave_start[w] || h_wave_start[w + 1] > n)
      return c->fail(CG_ERR_INVALID_VALUE, "wave offsets not increasing or beyond n");
  bool big = false;   // a wave that may hold a self-overlapping copy beyond the staging area: recovered per wave
  for (uint32_t w = 0; w < n_waves; ++w) big = big || h_max_bytes[w] > cgk::stage_bytes();
  if (c->wave_kernel && n_waves && c->cfg.dev_vbuf && !big) {   // every wave in one cooperative launch
    if (!d_descs || !d_verdicts || !d_index) return c->fail(CG_ERR_INVALID_VALUE, "null descriptor, verdict or index array");
    if (d_descs != c->last_check || n != c->last_check_n)
      return c->fail(CG_ERR_INVALID_VALUE, "cg_apply_copies must follow the check of the same descriptors");
    const uint64_t a = h_wave_start[0], m = h_wave_start[n_waves] - a;
    if (m) {
      DeviceGuard g(c->cfg.device);
      cudaStream_t s = static_cast<cudaStream_t>(stream);
      c->h_wstart.resize(n_waves + 1);
      for (uint32_t w = 0; w <= n_waves; ++w) c->h_wstart[w] = (uint32_t)(h_wave_start[w] - a);
      uint32_t* dw = reinterpret_cast<uint32_t*>(c->ws + c->lay.waves);
      cudaError_t e = cudaMemcpyAsync(dw, c->h_wstart.data(), (n_waves + 1) * sizeof(uint32_t),
                                      cudaMemcpyHostToDevice, s);
      if (e == cudaSuccess)
        e = cgk::propagate_waves(c->launch, d_descs, d_verdicts, d_index + a, m, dw, n_waves, c->sv,
                                 static_cast<uint8_t*>(c->cfg.dev_vbuf), c->plan(), c->ws + c->lay.scratch,
                                 reinterpret_cast<uint32_t*>(c->ws + c->lay.ovl), s);
      if (e != cudaSuccess) return c->cuda(e, "propagate waves");
    }
    return cg_apply_flush(c, stream);
  }
  for (uint32_t w = 0; w < n_waves; ++w) {   // in level order, all launches from this loop
    cg_status st = cg_apply_copies_subset(c, d_descs, d_verdicts, n, d_index + h_wave_start[w],
                                          h_wave_start[w + 1] - h_wave_start[w], h_max_bytes[w], stream);
    if (st == CG_OK && h_max_bytes[w] > cgk::stage_bytes()) st = cg_apply_flush(c, stream);   // before the next wave
    if (st != CG_OK) return st;
  }
  return cg_apply_flush(c, stream);
}

// NEXT-1: the self-overlapping 2D DtoDs with unequal pitches that did not fit
// the 8 MiB staging area were skipped and listed by the kernels; stage each
// through a scratch of its own size now (their batch / wave is conflict-free,
// so moving them after the rest of it is the sequential result)
static cg_status recover_memmoves(cg_ctx* c, const cg_copy_desc* d_descs, cudaStream_t s) {
  uint32_t* overflow = reinterpret_cast<uint32_t*>(c->ws + c->lay.ovl);
  uint32_t h[2] = {0, 0};
  cudaError_t e = cudaMemcpyAsync(h, overflow, sizeof h, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return c->cuda(e, "propagate");
  if (!h[0]) return CG_OK;
  std::vector<uint32_t> list(h[1]);
  e = cudaMemcpy(list.data(), overflow + 2, h[1] * sizeof(uint32_t), cudaMemcpyDeviceToHost);
  uint64_t need = 0;
  for (uint32_t i : list) {
    cg_copy_desc d{};
    if (e == cudaSuccess) e = cudaMemcpy(&d, d_descs + i, sizeof d, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) need = std::max(need, d.width * d.height);
  }
  uint8_t* scratch = nullptr;
  if (e == cudaSuccess) e = cudaMallocAsync(&scratch, need, s);
  if (e != cudaSuccess) return c->fail(CG_ERR_OUT_OF_MEMORY, "staging of a %llu-byte self-overlapping copy: %s",
                                       (unsigned long long)need, cudaGetErrorString(e));
  e = cudaMemsetAsync(overflow, 0, 8, s);   // flag and count; the list itself is read by the kernel below
  uint32_t* d_list = nullptr;
  if (e == cudaSuccess) e = cudaMallocAsync(&d_list, (h[1] + 1) * sizeof(uint32_t), s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_list + 1, list.data(), h[1] * sizeof(uint32_t), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_list, &h[1], sizeof(uint32_t), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess)
    e = cgk::memmove_list(c->launch, d_descs, c->plan().dvoff, d_list + 1, d_list, static_cast<uint8_t*>(c->cfg.dev_vbuf),
                          scratch, need, overflow, s);
  if (e == cudaSuccess) e = cudaFreeAsync(scratch, s);
  if (e == cudaSuccess) e = cudaFreeAsync(d_list, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  return c->cuda(e, "memmove recovery");
}

cg_status cg_apply_flush(cg_ctx* c, void* stream) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  if (!c->cfg.dev_vbuf) return CG_OK;
  DeviceGuard g(c->cfg.device);
  if (!c->last_check) return CG_OK;
  return recover_memmoves(c, static_cast<const cg_copy_desc*>(c->last_check), static_cast<cudaStream_t>(stream));
}

cg_status cg_apply_copies(cg_ctx* c, const cg_copy_desc* d_descs, const cg_verdict* d_verdicts, uint64_t n,
                          void* stream) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  if (!c->cfg.dev_vbuf) return cg_apply_dtoh(c, d_descs, d_verdicts, n, stream);
  if (n == 0) return CG_OK;
  if (!d_descs || !d_verdicts) return c->fail(CG_ERR_INVALID_VALUE, "null descriptor or verdict array");
  if (d_descs != c->last_check || n != c->last_check_n)
    return c->fail(CG_ERR_INVALID_VALUE, "cg_apply_copies must follow the check of the same descriptors");
  DeviceGuard g(c->cfg.device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint32_t* overflow = reinterpret_cast<uint32_t*>(c->ws + c->lay.ovl);
  cudaError_t e = cgk::propagate(c->launch, d_descs, d_verdicts, nullptr, n, c->sv,
                                 static_cast<uint8_t*>(c->cfg.dev_vbuf), c->plan(), c->ws + c->lay.scratch, overflow, s,
                                 false);
  if (e != cudaSuccess) return c->cuda(e, "propagate");
  return recover_memmoves(c, d_descs, s);
}

cg_status cg_device_vbits(cg_ctx* c, uint64_t addr, uint64_t len, uint8_t* h_out) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  if (!c->cfg.dev_vbuf) return c->fail(CG_ERR_NOT_INITIALIZED, "no device V-bit tracking");
  if (len && !h_out) return c->fail(CG_ERR_INVALID_VALUE, "null output");
  auto it = c->live.upper_bound(addr);
  if (it == c->live.begin()) return c->fail(CG_ERR_INVALID_VALUE, "not inside a live allocation");
  --it;
  if (addr >= it->second || len > it->second - addr) return c->fail(CG_ERR_INVALID_VALUE, "not inside a live allocation");
  auto pos = std::lower_bound(c->table.begin(), c->table.end(), it->first,
                              [](const Entry& e, uint64_t b) { return e.base < b; });
  for (; pos != c->table.end() && pos->base == it->first && pos->fseq != cgk::kInf; ++pos) {
  }
  DeviceGuard g(c->cfg.device);
  cudaError_t e = cudaMemcpy(h_out, static_cast<uint8_t*>(c->cfg.dev_vbuf) + pos->pool + (addr - pos->base), len,
                             cudaMemcpyDeviceToHost);
  return c->cuda(e, "device V download");
}

cg_status cg_array_vbits(cg_ctx* c, uint64_t handle, uint64_t offset, uint64_t len, uint8_t* h_out) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  if (!c->cfg.dev_vbuf) return c->fail(CG_ERR_NOT_INITIALIZED, "no device V-bit tracking");
  if (len && !h_out) return c->fail(CG_ERR_INVALID_VALUE, "null output");
  auto it = c->live_arrays.find(handle);
  if (it == c->live_arrays.end() || offset > it->second || len > it->second - offset)
    return c->fail(CG_ERR_INVALID_VALUE, "not inside a live array");
  auto pos = std::lower_bound(c->arrays.begin(), c->arrays.end(), handle,
                              [](const ArrayEntry& e, uint64_t h) { return e.handle < h; });
  for (; pos != c->arrays.end() && pos->handle == handle && pos->fseq != cgk::kInf; ++pos) {
  }
  DeviceGuard g(c->cfg.device);
  cudaError_t e = cudaMemcpy(h_out, static_cast<uint8_t*>(c->cfg.dev_vbuf) + pos->pool + offset, len,
                             cudaMemcpyDeviceToHost);
  return c->cuda(e, "array V download");
}

cg_status cg_check_apply(cg_ctx* c, const cg_copy_desc* d_descs, uint64_t n, cg_verdict* d_out, void* stream) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  if (n == 0) return CG_OK;
  if (!d_descs || !d_out) return c->fail(CG_ERR_INVALID_VALUE, "null descriptor or verdict array");
  if ((uintptr_t)d_descs % 16 || (uintptr_t)d_out % 16) return c->fail(CG_ERR_INVALID_VALUE, "arrays not 16-byte aligned");
  if (n > c->cfg.max_descs) return c->fail(CG_ERR_INVALID_VALUE, "n > max_descs");
  DeviceGuard g(c->cfg.device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cg_status st = c->sync_table(s);
  if (st != CG_OK) return st;
  if (c->cfg.dev_vbuf) {   // NEXT-1 tracking: check, then propagate (not fused)
    st = cg_check_copies(c, d_descs, n, d_out, stream);
    return st != CG_OK ? st : cg_apply_copies(c, d_descs, d_out, n, stream);
  }
  cudaError_t e = cgk::check_apply(c->launch, d_descs, n, d_out, c->dev_table(), c->sv, c->plan(), c->err_mask(), s);
  c->last_check = nullptr;
  return c->cuda(e, "check+apply kernels");
}

cg_status cg_check_copies_host(cg_ctx* c, const cg_copy_desc* h_descs, uint64_t n, cg_verdict* h_out, int apply,
                               void* stream) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  if (!c->cfg.host_staging) return c->fail(CG_ERR_NOT_INITIALIZED, "context created without host staging");
  if (n == 0) return CG_OK;
  if (!h_descs || !h_out) return c->fail(CG_ERR_INVALID_VALUE, "null host arrays");
  if (n > c->cfg.max_descs) return c->fail(CG_ERR_INVALID_VALUE, "n > max_descs");
  DeviceGuard g(c->cfg.device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (c->slot_busy[0]) return c->fail(CG_ERR_INVALID_VALUE, "staging slot 0 holds a submitted batch");
  cg_copy_desc* dd = reinterpret_cast<cg_copy_desc*>(c->ws + c->lay.desc_stage);
  cg_verdict* dv = reinterpret_cast<cg_verdict*>(c->ws + c->lay.verdict_stage);
  cudaError_t e = cudaStreamWaitEvent(s, c->slot_free[0], 0);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dd, h_descs, n * sizeof(cg_copy_desc), cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return c->cuda(e, "descriptor upload");
  cg_status st = apply == 2 ? cg_check_apply(c, dd, n, dv, stream) : cg_check_copies(c, dd, n, dv, stream);
  if (st != CG_OK) return st;
  if (apply == 1) {
    st = cg_apply_dtoh(c, dd, dv, n, stream);
    if (st != CG_OK) return st;
  }
  e = cudaMemcpyAsync(h_out, dv, n * sizeof(cg_verdict), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  return c->cuda(e, "verdict download");
}

cg_status cg_expand_copy1d(cg_ctx* c, const cg_copy1d* d_in, uint64_t n, cg_copy_desc* d_out, void* stream) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  if (n && (!d_in || !d_out)) return c->fail(CG_ERR_INVALID_VALUE, "null arrays");
  DeviceGuard g(c->cfg.device);
  return c->cuda(cgk::expand_1d(c->launch, d_in, n, d_out, static_cast<cudaStream_t>(stream)), "expand 1d");
}

static cg_status check_host_submit(cg_ctx* c, const void* h_descs, uint32_t format, uint64_t n, int apply,
                                   uint32_t slot, void* stream, bool chunked);

cg_status cg_check_host_submit(cg_ctx* c, const void* h_descs, uint32_t format, uint64_t n, int apply, uint32_t slot,
                               void* stream) {
  // one chunk: with batches in flight on both slots the whole upload already
  // runs under the previous batch's kernels
  return check_host_submit(c, h_descs, format, n, apply, slot, stream, false);
}

static cg_status check_host_submit(cg_ctx* c, const void* h_descs, uint32_t format, uint64_t n, int apply,
                                   uint32_t slot, void* stream, bool chunked) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  if (!c->cfg.host_staging) return c->fail(CG_ERR_NOT_INITIALIZED, "context created without host staging");
  if (slot >= kHostSlots) return c->fail(CG_ERR_INVALID_VALUE, "slot out of range");
  if (c->slot_busy[slot]) return c->fail(CG_ERR_INVALID_VALUE, "slot holds a batch not yet waited for");
  if (n && (!h_descs || format > CG_FMT_1D || apply < 0 || apply > 2))
    return c->fail(CG_ERR_INVALID_VALUE, "bad arguments");
  if (n > c->cfg.max_descs) return c->fail(CG_ERR_INVALID_VALUE, "n > max_descs");
  DeviceGuard g(c->cfg.device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint64_t md = c->cfg.max_descs;
  cg_copy_desc* dd = reinterpret_cast<cg_copy_desc*>(c->ws + c->lay.desc_stage) + slot * md;
  cg_verdict* dv = reinterpret_cast<cg_verdict*>(c->ws + c->lay.verdict_stage) + slot * md;
  cg_copy1d* draw = reinterpret_cast<cg_copy1d*>(c->ws + c->lay.raw_stage) + slot * md;
  uint64_t* didx = reinterpret_cast<uint64_t*>(c->ws + c->lay.idx_stage) + slot * md;
  cg_verdict* ddirty = reinterpret_cast<cg_verdict*>(c->ws + c->lay.dirty_stage) + slot * md;
  uint32_t* dcount = reinterpret_cast<uint32_t*>(c->ws + c->lay.flags + 192) + slot;
  const size_t esz = format == CG_FMT_1D ? sizeof(cg_copy1d) : sizeof(cg_copy_desc);
  uint8_t* dst = format == CG_FMT_1D ? reinterpret_cast<uint8_t*>(draw) : reinterpret_cast<uint8_t*>(dd);
  // geometric chunks (sizes 1 : 2 : 4 : ...): the first upload is short, and
  // every later chunk's upload (PCIe, ~50 GB/s) finishes while the previous
  // chunk is being checked (the check is slower per descriptor than the upload)
  const uint64_t nchunks = chunked && n >= (1u << 19) ? c->host_chunks : 1;
  uint64_t bound[kHostChunks + 1];
  bound[0] = 0;
  for (uint64_t k = 1; k <= nchunks; ++k)
    bound[k] = k == nchunks ? n
               : c->host_geometric ? n * ((1ull << k) - 1) / ((1ull << nchunks) - 1) : n * k / nchunks;
  // uploads on the copy stream, after the slot's previous batch stopped reading
  // its staging (not after all work on s: the previous batch of the other slot
  // is still being checked while this one uploads)
  cudaError_t e = cudaStreamWaitEvent(c->copy_stream, c->slot_free[slot], 0);
  for (uint64_t k = 0; k < nchunks && e == cudaSuccess; ++k) {
    const uint64_t a = bound[k], b = bound[k + 1];
    if (a >= b) continue;
    e = cudaMemcpyAsync(dst + a * esz, static_cast<const uint8_t*>(h_descs) + a * esz, (b - a) * esz,
                        cudaMemcpyHostToDevice, c->copy_stream);
    if (e == cudaSuccess) e = cudaEventRecord(c->chunk_ev[slot][k], c->copy_stream);
  }
  if (e != cudaSuccess) return c->cuda(e, "descriptor upload");
  e = cudaMemsetAsync(dcount, 0, sizeof(uint32_t), s);
  if (e != cudaSuccess) return c->cuda(e, "memset");
  for (uint64_t k = 0; k < nchunks; ++k) {
    const uint64_t a = bound[k], b = bound[k + 1];
    if (a >= b) continue;
    e = cudaStreamWaitEvent(s, c->chunk_ev[slot][k], 0);
    if (e == cudaSuccess && format == CG_FMT_1D) e = cgk::expand_1d(c->launch, draw + a, b - a, dd + a, s);
    if (e != cudaSuccess) return c->cuda(e, "chunk wait / expand");
    cg_status st = apply == 2 ? cg_check_apply(c, dd + a, b - a, dv + a, stream)
                              : cg_check_copies(c, dd + a, b - a, dv + a, stream);
    if (st == CG_OK && apply == 1) st = cg_apply_dtoh(c, dd + a, dv + a, b - a, stream);
    if (st != CG_OK) return st;
    e = cgk::compact_dirty(c->launch, dv + a, b - a, didx, ddirty, dcount, a, false, s);
    if (e != cudaSuccess) return c->cuda(e, "compact");
  }
  e = cudaEventRecord(c->slot_free[slot], s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(c->h_count + slot, dcount, sizeof(uint32_t), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaEventRecord(c->slot_done[slot], s);
  if (e != cudaSuccess) return c->cuda(e, "count download");
  c->slot_busy[slot] = true;
  return CG_OK;
}

cg_status cg_check_host_wait(cg_ctx* c, uint32_t slot, uint64_t* h_idx, cg_verdict* h_dirty, uint64_t cap,
                             uint64_t* n_dirty) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  if (slot >= kHostSlots || !c->slot_busy[slot]) return c->fail(CG_ERR_INVALID_VALUE, "no batch submitted to slot");
  if (!n_dirty || (cap && (!h_idx || !h_dirty))) return c->fail(CG_ERR_INVALID_VALUE, "null outputs");
  DeviceGuard g(c->cfg.device);
  c->slot_busy[slot] = false;
  cudaError_t e = cudaEventSynchronize(c->slot_done[slot]);
  if (e != cudaSuccess) return c->cuda(e, "batch wait");
  const uint64_t cnt = c->h_count[slot];
  *n_dirty = cnt;
  const uint64_t m = std::min<uint64_t>(cnt, cap), md = c->cfg.max_descs;
  if (m) {   // on the result stream: the next batch's kernels on the check stream keep running
    const uint64_t* didx = reinterpret_cast<const uint64_t*>(c->ws + c->lay.idx_stage) + slot * md;
    const cg_verdict* ddirty = reinterpret_cast<const cg_verdict*>(c->ws + c->lay.dirty_stage) + slot * md;
    e = cudaMemcpyAsync(h_idx, didx, m * sizeof(uint64_t), cudaMemcpyDeviceToHost, c->out_stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(h_dirty, ddirty, m * sizeof(cg_verdict), cudaMemcpyDeviceToHost, c->out_stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->out_stream);
    if (e != cudaSuccess) return c->cuda(e, "dirty download");
  }
  return CG_OK;
}

cg_status cg_check_host(cg_ctx* c, const void* h_descs, uint32_t format, uint64_t n, int apply, uint64_t* h_idx,
                        cg_verdict* h_dirty, uint64_t cap, uint64_t* n_dirty, void* stream) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  if (!c->cfg.host_staging) return c->fail(CG_ERR_NOT_INITIALIZED, "context created without host staging");
  if (!n_dirty || (cap && (!h_idx || !h_dirty))) return c->fail(CG_ERR_INVALID_VALUE, "null outputs");
  *n_dirty = 0;
  if (n == 0) return CG_OK;
  if (!h_descs || format > CG_FMT_1D || apply < 0 || apply > 2) return c->fail(CG_ERR_INVALID_VALUE, "bad arguments");
  const uint32_t slot = c->slot_busy[0] ? 1u : 0u;
  cg_status st = check_host_submit(c, h_descs, format, n, apply, slot, stream, true);
  if (st != CG_OK) return st;
  return cg_check_host_wait(c, slot, h_idx, h_dirty, cap, n_dirty);
}

cg_status cg_straddler_pack(cg_ctx* c, const cg_verdict* d_raw, uint64_t m, uint64_t* d_mins, uint64_t* d_sums,
                            uint32_t* d_maxs, void* stream) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  if (m == 0) return CG_OK;
  if (!d_raw || !d_mins || !d_sums || !d_maxs) return c->fail(CG_ERR_INVALID_VALUE, "null straddler arrays");
  DeviceGuard g(c->cfg.device);
  return c->cuda(cgk::straddler_pack(c->launch, d_raw, m, d_mins, d_sums, d_maxs, static_cast<cudaStream_t>(stream)),
                 "straddler pack");
}

cg_status cg_straddler_finalize(cg_ctx* c, const uint64_t* d_mins, const uint64_t* d_sums, const uint32_t* d_maxs,
                                uint64_t m, cg_verdict* d_out, void* stream) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  if (m == 0) return CG_OK;
  if (!d_out || !d_mins || !d_sums || !d_maxs) return c->fail(CG_ERR_INVALID_VALUE, "null straddler arrays");
  DeviceGuard g(c->cfg.device);
  return c->cuda(cgk::straddler_finalize(c->launch, d_mins, d_sums, d_maxs, m, d_out, c->err_mask(),
                                         static_cast<cudaStream_t>(stream)),
                 "straddler finalize");
}

cg_status cg_compact_dirty(cg_ctx* c, const cg_verdict* d_verdicts, uint64_t n, uint64_t* d_idx,
                           cg_verdict* d_dirty, uint32_t* d_count, void* stream) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  if (!d_count || (n && (!d_verdicts || !d_idx || !d_dirty))) return c->fail(CG_ERR_INVALID_VALUE, "null arrays");
  DeviceGuard g(c->cfg.device);
  return c->cuda(
      cgk::compact_dirty(c->launch, d_verdicts, n, d_idx, d_dirty, d_count, 0, true, static_cast<cudaStream_t>(stream)),
      "compact dirty");
}

cg_status cg_leak_sweep(cg_ctx* c, cg_alloc_record* d_out, uint64_t cap, uint64_t* d_count, void* stream) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  if (!d_count || (cap && !d_out)) return c->fail(CG_ERR_INVALID_VALUE, "null output");
  DeviceGuard g(c->cfg.device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cg_status st = c->sync_table(s);
  if (st != CG_OK) return st;
  cudaError_t e = cgk::leak_sweep(c->launch, c->dev_table(), c->plan(), d_out, cap, d_count, s);
  return c->cuda(e, "leak sweep");
}

cg_status cg_leak_report(cg_ctx* c, cg_alloc_record* h_out, uint64_t cap, uint64_t* n_out) {
  if (!c) return CG_ERR_INVALID_CONTEXT;
  if (!n_out || (cap && !h_out)) return c->fail(CG_ERR_INVALID_VALUE, "null output");
  DeviceGuard g(c->cfg.device);
  cg_alloc_record* d_rec = reinterpret_cast<cg_alloc_record*>(c->ws + c->lay.leaks);
  uint64_t* d_cnt = reinterpret_cast<uint64_t*>(c->ws + c->lay.flags + 64);
  cg_status st = cg_leak_sweep(c, d_rec, c->cfg.max_allocs, d_cnt, 0);
  uint64_t k = 0;
  if (st == CG_OK) {
    cudaError_t e = cudaMemcpy(&k, d_cnt, sizeof k, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && cap && k)
      e = cudaMemcpy(h_out, d_rec, std::min(cap, k) * sizeof(cg_alloc_record), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) st = c->cuda(e, "leak report download");
  }
  *n_out = k;
  return st;
}

// host -> device direction (HtoD, HtoA: the host side is read) vs device -> host
static bool reads_host(uint32_t kind) { return kind == CG_HTOD || kind == CG_HTOA; }
static bool writes_host(uint32_t kind) { return kind == CG_DTOH || kind == CG_ATOH; }

static bool host_range(const cg_copy_desc& d, uint64_t& lo, uint64_t& hi) {
  const bool htod = reads_host(d.kind);
  if (!htod && !writes_host(d.kind)) return false;
  const uint64_t base = htod ? d.src : d.dst, x = htod ? d.src_x : d.dst_x;
  const uint64_t y = htod ? d.src_y : d.dst_y, pitch = htod ? d.src_pitch : d.dst_pitch;
  if (d.width == 0 || d.height == 0) return false;
  unsigned __int128 st = (unsigned __int128)base + (unsigned __int128)y * pitch + x;
  unsigned __int128 sp = (unsigned __int128)(d.height - 1) * pitch + d.width;
  if (st + sp > (unsigned __int128)UINT64_MAX) return false;
  lo = (uint64_t)st;
  hi = (uint64_t)(st + sp);
  return true;
}

int cg_ctx_device(const cg_ctx* c) { return c ? c->cfg.device : -1; }

cg_status cg_shard_lists(const cg_copy_desc* h_descs, uint64_t n, uint64_t host_base, uint64_t host_size,
                         uint32_t world, uint32_t rank, cg_copy_desc* h_out, uint64_t* h_gidx, uint64_t* n_own,
                         uint64_t* m) {
  if (!n_own || !m || rank >= world || (n && (!h_descs || !h_out || !h_gidx))) return CG_ERR_INVALID_VALUE;
  std::vector<uint32_t> owner(n), first(n), last(n);
  cg_status st = cg_shard_plan(h_descs, n, host_base, host_size, world, owner.data(), first.data(), last.data());
  if (st != CG_OK) return st;
  uint64_t k = 0;
  for (uint64_t i = 0; i < n; ++i)
    if (first[i] == last[i] && owner[i] == rank) {
      h_out[k] = h_descs[i];
      h_out[k].reserved = 0;
      h_gidx[k++] = i;
    }
  *n_own = k;
  for (uint64_t i = 0; i < n; ++i)
    if (first[i] < last[i]) {
      h_out[k] = h_descs[i];
      h_out[k].reserved = CG_SHARD_RAW | (owner[i] == rank ? 0u : (uint32_t)CG_SHARD_NOT_OWNER);
      h_gidx[k++] = i;
    }
  *m = k - *n_own;
  uint64_t after = 0;
  return cg_plan_apply_after(h_out, k, &after);
}

cg_status cg_plan_apply_after(cg_copy_desc* h_descs, uint64_t n, uint64_t* n_after) {
  if (!n_after || (n && !h_descs)) return CG_ERR_INVALID_VALUE;
  std::vector<std::pair<uint64_t, uint64_t>> rd;   // HtoD / HtoA host ranges, merged
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t lo, hi;
    if (reads_host(h_descs[i].kind) && host_range(h_descs[i], lo, hi)) rd.emplace_back(lo, hi);
  }
  std::sort(rd.begin(), rd.end());
  std::vector<std::pair<uint64_t, uint64_t>> m;
  for (const auto& r : rd) {
    if (!m.empty() && r.first <= m.back().second) m.back().second = std::max(m.back().second, r.second);
    else m.push_back(r);
  }
  uint64_t k = 0;
  for (uint64_t i = 0; i < n; ++i) {
    cg_copy_desc& d = h_descs[i];
    d.reserved &= ~(uint32_t)CG_APPLY_AFTER;
    if (d.reserved & CG_SHARD_RAW) continue;   // a straddler is applied after the exchange anyway
    uint64_t lo, hi;
    if (!writes_host(d.kind) || !host_range(d, lo, hi)) continue;
    auto it = std::upper_bound(m.begin(), m.end(), std::make_pair(lo, UINT64_MAX));   // first range starting after lo
    bool hit = it != m.end() && it->first < hi;
    if (!hit && it != m.begin()) hit = std::prev(it)->second > lo;
    if (hit) {
      d.reserved |= CG_APPLY_AFTER;
      ++k;
    }
  }
  *n_after = k;
  return CG_OK;
}

cg_status cg_batch_disjoint(const cg_copy_desc* h_descs, uint64_t n, int* disjoint) {
  if (!disjoint || (n && !h_descs)) return CG_ERR_INVALID_VALUE;
  struct Iv {
    uint64_t lo, hi;
    bool htod;
  };
  std::vector<Iv> v;
  v.reserve(n);
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t lo, hi;
    if (host_range(h_descs[i], lo, hi)) v.push_back({lo, hi, reads_host(h_descs[i].kind)});
  }
  std::sort(v.begin(), v.end(), [](const Iv& a, const Iv& b) { return a.lo < b.lo; });
  uint64_t end_h = 0, end_d = 0;   // furthest end of HtoD / DtoH ranges starting earlier
  bool seen_h = false, seen_d = false;
  *disjoint = 1;
  for (const Iv& x : v) {
    if (x.htod) {
      if (seen_d && x.lo < end_d) { *disjoint = 0; break; }
      end_h = seen_h ? std::max(end_h, x.hi) : x.hi;
      seen_h = true;
    } else {
      if (seen_h && x.lo < end_h) { *disjoint = 0; break; }
      end_d = seen_d ? std::max(end_d, x.hi) : x.hi;
      seen_d = true;
    }
  }
  return CG_OK;
}

cg_status cg_shard_plan(const cg_copy_desc* h_descs, uint64_t n, uint64_t host_base, uint64_t host_size,
                        uint32_t world, uint32_t* h_owner, uint32_t* h_first, uint32_t* h_last) {
  if (world == 0 || host_size == 0 || host_size % world || (host_size / world) % 4096) return CG_ERR_INVALID_VALUE;
  if (n && (!h_descs || !h_owner || !h_first || !h_last)) return CG_ERR_INVALID_VALUE;
  const uint64_t shard = host_size / world, we = host_base + host_size;
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t lo, hi;
    uint32_t owner = (uint32_t)(i % world), first = owner, last = owner;
    if (host_range(h_descs[i], lo, hi)) {
      // owner: the shard holding the host start (clamped into the window)
      const uint64_t s0 = lo < host_base ? 0 : lo >= we ? host_size - 1 : lo - host_base;
      owner = (uint32_t)(s0 / shard);
      const uint64_t a = std::max(lo, host_base), b = std::min(hi, we);
      if (a < b) {   // shards holding shadow bytes of the range
        first = (uint32_t)((a - host_base) / shard);
        last = (uint32_t)((b - 1 - host_base) / shard);
        if (owner < first) first = owner;
        if (owner > last) last = owner;
      } else {
        first = last = owner;
      }
    }
    h_owner[i] = owner;
    h_first[i] = first;
    h_last[i] = last;
  }
  return CG_OK;
}

// folded [lo, hi) of one side (false on overflow or no bytes)
static bool side_range(const cg_copy_desc& d, bool dst, uint64_t& lo, uint64_t& hi) {
  const uint64_t base = dst ? d.dst : d.src, x = dst ? d.dst_x : d.src_x;
  const uint64_t y = dst ? d.dst_y : d.src_y, pitch = dst ? d.dst_pitch : d.src_pitch;
  if (d.width == 0 || d.height == 0) return false;
  unsigned __int128 st = (unsigned __int128)base + (unsigned __int128)y * pitch + x;
  unsigned __int128 sp = (unsigned __int128)(d.height - 1) * pitch + d.width;
  if (st + sp > (unsigned __int128)UINT64_MAX) return false;
  lo = (uint64_t)st;
  hi = (uint64_t)(st + sp);
  return true;
}

// the V-bit bytes a copy reads / writes (NEXT-1, R-28): host and device sides
// by address (2D: bounding range); an array side (R-29, R-30) by byte offset
// [offset, offset + W*H) in that array's own space
static bool array_side(const cg_copy_desc& d, bool dst, uint64_t& lo, uint64_t& hi) {
  const uint64_t off = dst ? d.dst_x : d.src_x;
  if (d.width == 0 || d.height == 0) return false;
  const unsigned __int128 nb = (unsigned __int128)d.width * d.height;
  if (off + nb > (unsigned __int128)UINT64_MAX) return false;
  lo = off;
  hi = (uint64_t)(off + nb);
  return true;
}
static bool copy_read(const cg_copy_desc& d, uint64_t& lo, uint64_t& hi) {
  return d.kind == CG_ATOH ? array_side(d, false, lo, hi) : side_range(d, false, lo, hi);
}
static bool copy_write(const cg_copy_desc& d, uint64_t& lo, uint64_t& hi) {
  return d.kind == CG_HTOA ? array_side(d, true, lo, hi) : side_range(d, true, lo, hi);
}

namespace {
struct IvSet {   // disjoint merged intervals
  std::map<uint64_t, uint64_t> m;
  bool overlaps(uint64_t lo, uint64_t hi) const {
    auto it = m.upper_bound(lo);
    if (it != m.end() && it->first < hi) return true;
    return it != m.begin() && std::prev(it)->second > lo;
  }
  void add(uint64_t lo, uint64_t hi) {
    auto it = m.upper_bound(lo);
    if (it != m.begin() && std::prev(it)->second >= lo) {
      --it;
      lo = it->first;
      hi = std::max(hi, it->second);
      it = m.erase(it);
    }
    while (it != m.end() && it->first <= hi) {
      hi = std::max(hi, it->second);
      it = m.erase(it);
    }
    m.emplace(lo, hi);
  }
};
}  // namespace

namespace {
// disjoint intervals of host or device addresses, each with the highest wave
// level (+1) that read (or wrote) it so far
struct LevelMap {
  std::map<uint64_t, std::pair<uint64_t, uint32_t>> m;   // start -> (end, level + 1)
  uint32_t max_over(uint64_t lo, uint64_t hi) const {
    uint32_t r = 0;
    auto it = m.upper_bound(lo);
    if (it != m.begin()) --it;
    for (; it != m.end() && it->first < hi; ++it)
      if (it->second.first > lo) r = std::max(r, it->second.second);
    return r;
  }
  void split(uint64_t x) {   // make x an interval boundary
    auto it = m.upper_bound(x);
    if (it == m.begin()) return;
    --it;
    if (it->first < x && it->second.first > x) {
      m.emplace(x, it->second);
      it->second.first = x;
    }
  }
  void erase(uint64_t lo, uint64_t hi) {
    split(lo);
    split(hi);
    m.erase(m.lower_bound(lo), m.lower_bound(hi));
  }
  void assign(uint64_t lo, uint64_t hi, uint32_t v) {
    erase(lo, hi);
    m.emplace(lo, std::make_pair(hi, v));
  }
  void paint_max(uint64_t lo, uint64_t hi, uint32_t v) {
    split(lo);
    split(hi);
    uint64_t cur = lo;
    for (auto it = m.lower_bound(lo); it != m.end() && it->first < hi; ++it) {
      if (it->first > cur) it = m.emplace_hint(it, cur, std::make_pair(it->first, v));   // the gap before it
      else it->second.second = std::max(it->second.second, v);
      cur = it->second.first;
    }
    if (cur < hi) m.emplace(cur, std::make_pair(hi, v));
  }
};
}  // namespace

cg_status cg_plan_waves(const cg_copy_desc* h_descs, uint64_t n, uint32_t* h_level, uint32_t* n_levels) {
  if (!n_levels || (n && (!h_descs || !h_level))) return CG_ERR_INVALID_VALUE;
  // per address space ([0] host, [1] device): the levels of earlier readers and
  // writers.  A write at level l dominates every earlier access of its range
  // (it conflicted with all of them), so it replaces the writer entries and
  // clears the reader entries there; reads merge by max.
  LevelMap rd[2], wr[2];
  std::map<uint64_t, LevelMap> ard, awr;   // per array handle (R-30): its byte offsets
  uint32_t top = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const cg_copy_desc& d = h_descs[i];
    h_level[i] = 0;
    if (d.kind < CG_HTOD || d.kind > CG_ATOH) continue;
    uint64_t rlo = 0, rhi = 0, wlo = 0, whi = 0;
    // the same read / write sets as cg_plan_batches_propagate (R-28, R-30)
    const bool r_ok = copy_read(d, rlo, rhi), w_ok = copy_write(d, wlo, whi);
    const int rs = reads_host(d.kind) ? 0 : 1, ws = writes_host(d.kind) ? 0 : 1;
    LevelMap& R = d.kind == CG_ATOH ? ard[d.src] : rd[rs];
    LevelMap& Rw = d.kind == CG_ATOH ? awr[d.src] : wr[rs];
    LevelMap& W = d.kind == CG_HTOA ? awr[d.dst] : wr[ws];
    LevelMap& Wr = d.kind == CG_HTOA ? ard[d.dst] : rd[ws];
    uint32_t lv = 0;   // = 1 + the highest conflicting earlier level (maps hold level + 1), 0 if none
    if (r_ok) lv = std::max(lv, Rw.max_over(rlo, rhi));                                      // RAW
    if (w_ok) lv = std::max(lv, std::max(Wr.max_over(wlo, whi), W.max_over(wlo, whi)));      // WAR, WAW
    h_level[i] = lv;
    if (r_ok) R.paint_max(rlo, rhi, lv + 1);
    if (w_ok) {
      Wr.erase(wlo, whi);
      W.assign(wlo, whi, lv + 1);
    }
    top = std::max(top, lv + 1);
  }
  *n_levels = n ? std::max(top, 1u) : 0;
  return CG_OK;
}

cg_status cg_plan_batches_propagate(const cg_copy_desc* h_descs, uint64_t n, uint64_t* h_cuts, uint64_t* n_cuts) {
  if (!n_cuts || (n && (!h_descs || !h_cuts))) return CG_ERR_INVALID_VALUE;
  IvSet hr, hw, dr, dw;   // host / device reads and writes of the open batch
  std::map<uint64_t, IvSet> ar, aw;   // per array handle: reads / writes of its V-bits (R-30)
  uint64_t k = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const cg_copy_desc& d = h_descs[i];
    if (d.kind < CG_HTOD || d.kind > CG_ATOH) continue;
    uint64_t rlo = 0, rhi = 0, wlo = 0, whi = 0;
    const bool r_ok = copy_read(d, rlo, rhi), w_ok = copy_write(d, wlo, whi);
    bool conflict;
    {
      IvSet& W = d.kind == CG_HTOA ? aw[d.dst] : writes_host(d.kind) ? hw : dw;   // the destination's space
      IvSet& Rw = d.kind == CG_ATOH ? aw[d.src] : reads_host(d.kind) ? hw : dw;   // writes in the source's space
      IvSet& Wr = d.kind == CG_HTOA ? ar[d.dst] : writes_host(d.kind) ? hr : dr;  // reads in the destination's
      conflict = (r_ok && Rw.overlaps(rlo, rhi)) || (w_ok && (Wr.overlaps(wlo, whi) || W.overlaps(wlo, whi)));
    }
    if (conflict) {
      h_cuts[k++] = i;
      hr.m.clear();
      hw.m.clear();
      dr.m.clear();
      dw.m.clear();
      ar.clear();
      aw.clear();
    }
    IvSet& R = d.kind == CG_ATOH ? ar[d.src] : reads_host(d.kind) ? hr : dr;    // the source's address space
    IvSet& W = d.kind == CG_HTOA ? aw[d.dst] : writes_host(d.kind) ? hw : dw;   // the destination's
    if (r_ok) R.add(rlo, rhi);
    if (w_ok) W.add(wlo, whi);
  }
  if (n) h_cuts[k++] = n;
  *n_cuts = k;
  return CG_OK;
}

cg_status cg_plan_batches_fused(cg_copy_desc* h_descs, uint64_t n, uint64_t* h_cuts, uint64_t* n_cuts) {
  if (!n_cuts || (n && (!h_descs || !h_cuts))) return CG_ERR_INVALID_VALUE;
  constexpr uint64_t kLateMax = 1ull << 20;   // larger dependent HtoDs end the batch instead
  constexpr uint32_t kBits = CG_CHECK_AFTER | CG_APPLY_AFTER | CG_APPLY_LAST;
  // the batch's DtoH ranges, its CG_CHECK_AFTER HtoD ranges, its CG_APPLY_LAST DtoH ranges
  IvSet dtoh, late, last;
  uint64_t k = 0, start = 0;
  auto cut = [&](uint64_t i) {   // end the batch before i; CG_APPLY_AFTER over [start, i)
    std::vector<cg_copy_desc> tmp(h_descs + start, h_descs + i);
    uint64_t after = 0;
    cg_plan_apply_after(tmp.data(), tmp.size(), &after);
    for (uint64_t j = start; j < i; ++j) {
      cg_copy_desc& d = h_descs[j];
      const uint32_t a = (d.reserved & CG_APPLY_LAST) ? 0u : (tmp[j - start].reserved & CG_APPLY_AFTER);
      d.reserved = (d.reserved & ~(uint32_t)CG_APPLY_AFTER) | a;
    }
    if (i == n) return;
    h_cuts[k++] = i;
    start = i;
    dtoh.m.clear();
    late.m.clear();
    last.m.clear();
  };
  for (uint64_t i = 0; i < n; ++i) {
    cg_copy_desc& d = h_descs[i];
    d.reserved &= ~kBits;
    uint64_t lo, hi;
    if (!host_range(d, lo, hi)) continue;
    if (reads_host(d.kind)) {
      if (last.overlaps(lo, hi)) cut(i);   // reads bytes applied only after the late checks
      if (dtoh.overlaps(lo, hi)) {
        if (hi - lo <= kLateMax) {
          d.reserved |= CG_CHECK_AFTER;
          late.add(lo, hi);
        } else {   // too large for the late pass: a new batch (the classic R-20 cut)
          cut(i);
        }
      }
    } else {
      if (late.overlaps(lo, hi)) {   // it writes bytes a CG_CHECK_AFTER HtoD must not see
        d.reserved |= CG_APPLY_LAST;
        last.add(lo, hi);
      }
      dtoh.add(lo, hi);
    }
  }
  if (n) {
    cut(n);
    h_cuts[k++] = n;
  }
  *n_cuts = k;
  return CG_OK;
}

cg_status cg_plan_batches(const cg_copy_desc* h_descs, uint64_t n, uint64_t* h_cuts, uint64_t* n_cuts) {
  if (!n_cuts || (n && (!h_descs || !h_cuts))) return CG_ERR_INVALID_VALUE;
  std::map<uint64_t, uint64_t> dtoh;   // merged DtoH host intervals of the open batch
  uint64_t k = 0;
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t lo, hi;
    if (!host_range(h_descs[i], lo, hi)) continue;
    if (reads_host(h_descs[i].kind)) {
      auto it = dtoh.upper_bound(lo);
      bool overlap = it != dtoh.end() && it->first < hi;
      if (!overlap && it != dtoh.begin()) overlap = std::prev(it)->second > lo;
      if (overlap) {
        h_cuts[k++] = i;
        dtoh.clear();
      }
    } else {
      // insert [lo, hi) merging neighbours
      auto it = dtoh.upper_bound(lo);
      if (it != dtoh.begin() && std::prev(it)->second >= lo) {
        --it;
        lo = it->first;
        hi = std::max(hi, it->second);
        it = dtoh.erase(it);
      }
      while (it != dtoh.end() && it->first <= hi) {
        hi = std::max(hi, it->second);
        it = dtoh.erase(it);
      }
      dtoh.emplace(lo, hi);
    }
  }
  if (n) h_cuts[k++] = n;
  *n_cuts = k;
  return CG_OK;
}

}  // extern "C"
