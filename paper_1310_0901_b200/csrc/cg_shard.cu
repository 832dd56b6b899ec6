// Host-address-range sharding inside the library (
// BASELINE north_star: "The shadow address space and copy batch are
// partitioned across the 8 B200s by host-address range, with an NCCL gather
// over NVLink only for the per-descriptor verdicts").
//
// A shard group is G contexts, each storing one shard of the global host
// window; the allocation table is replicated (every rank registers every
// allocation).  One sharded check of a batch, per rank, all asynchronous on
// the rank's stream with no host synchronisation:
//   1. cg_check_apply of the rank's list: its owned descriptors (host range in
//      its shard, or no host side and index mod G == rank), then the m
//      straddlers (host range over several shards, CG_SHARD_RAW, and
//      CG_SHARD_NOT_OWNER except on the owner): raw partials for those;
//   2. straddler pack -> three all-reduces (MIN of the two first offsets, SUM
//      of the count and the owner-only device fields, MAX of the flags, which
//      are identical everywhere or come from the owner only: MAX = OR) ->
//      straddler finalize (flags and status derived on every rank) -> each
//      rank applies its shard part of the straddling DtoH copies with status OK;
//   3. dirty verdicts of the owned part (and, on the root, of the straddlers)
//      compacted with their global indices into a fixed-capacity send buffer
//      (count, indices, verdicts: clean verdicts are canonical and not sent),
//      gathered to the root, merged there by a kernel into one dirty list (and
//      optionally scattered into a dense verdict array).
// Collectives: NCCL (one rank per process; libnccl.so.2 loaded with dlopen,
// normally the copy torch already loaded) or loopback (all G contexts in this
// process on one device: the reductions and the gather read the G ranks'
// device buffers directly).

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "cg.h"

namespace {

constexpr int kT = 256;
constexpr unsigned kFullMask = 0xffffffffu;

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
// dirty verdicts of v[0, n) -> send buffer: [0] u64 count (all dirty, also the
// ones past cap), then cap u64 global indices, then cap verdicts
__global__ void k_compact_gidx(const cg_verdict* __restrict__ v, uint64_t n, const uint64_t* __restrict__ gidx,
                               unsigned long long* __restrict__ count, uint64_t* __restrict__ idx,
                               cg_verdict* __restrict__ dirty, uint64_t cap) {
  const int lane = threadIdx.x & 31;
  for (uint64_t b0 = (uint64_t)blockIdx.x * blockDim.x; b0 < n; b0 += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = b0 + threadIdx.x;
    const bool d = i < n && v[i].flags != 0;
    const uint32_t mask = __ballot_sync(kFullMask, d);
    if (!mask) continue;
    const int leader = __ffs(mask) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(count, (unsigned long long)__popc(mask));
    base = __shfl_sync(kFullMask, base, leader);
    if (d) {
      const uint64_t k = base + __popc(mask & ((1u << lane) - 1u));
      if (k < cap) {   // the count keeps growing past cap: the overflow is detected
        idx[k] = gidx[i];
        dirty[k] = v[i];
      }
    }
  }
}

__global__ void k_zero_u64(unsigned long long* p, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    p[i] = 0;
}

// loopback all-reduce: rank 0's buffers := MIN / SUM / MAX over the G ranks'
struct Ptrs {
  uint64_t* mins[8];
  uint64_t* sums[8];
  uint32_t* maxs[8];
};
__global__ void k_reduce_loopback(Ptrs p, uint32_t world, uint64_t m) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < 5 * m; i += (uint64_t)gridDim.x * blockDim.x) {
    if (i < 2 * m) {
      uint64_t x = p.mins[0][i];
      for (uint32_t g = 1; g < world; ++g) x = min(x, p.mins[g][i]);
      p.mins[0][i] = x;
    }
    uint64_t s = p.sums[0][i];
    for (uint32_t g = 1; g < world; ++g) s += p.sums[g][i];
    p.sums[0][i] = s;
    if (i < m) {
      uint32_t f = p.maxs[0][i];
      for (uint32_t g = 1; g < world; ++g) f = max(f, p.maxs[g][i]);
      p.maxs[0][i] = f;
    }
  }
}

// root merge: the G gathered send buffers (count, cap indices, cap verdicts)
// -> one dirty list (out_idx / out_v, count in *out_n) and, if dense !=
// nullptr, the verdicts scattered into the dense array (whose clean entries
// were filled before).  *overflow = 1 if any count exceeds cap.
struct Bufs {
  const uint8_t* p[8];
};
__global__ void k_root_merge(Bufs bufs, uint32_t world, uint64_t cap, uint64_t* __restrict__ out_idx,
                             cg_verdict* __restrict__ out_v, unsigned long long* __restrict__ out_n,
                             cg_verdict* __restrict__ dense, uint32_t* __restrict__ overflow) {
  uint64_t off = 0;   // rank r's entries go to [sum of the earlier counts, + its count)
  for (uint32_t r = 0; r < world; ++r) {
    const uint8_t* b = bufs.p[r];
    const uint64_t c = *reinterpret_cast<const uint64_t*>(b);
    const uint64_t k = c < cap ? c : cap;
    if (c > cap && blockIdx.x == 0 && threadIdx.x == 0) *overflow = 1;
    const uint64_t* idx = reinterpret_cast<const uint64_t*>(b + 16);
    const cg_verdict* v = reinterpret_cast<const cg_verdict*>(b + 16 + 8 * cap);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += (uint64_t)gridDim.x * blockDim.x) {
      out_idx[off + i] = idx[i];
      out_v[off + i] = v[i];
      if (dense) dense[idx[i]] = v[i];
    }
    off += k;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *out_n = off;
}

__global__ void k_fill_clean(cg_verdict* __restrict__ v, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    cg_verdict x;
    x.first_unaddr = CG_NONE;
    x.first_undef = CG_NONE;
    x.undef_count = 0;
    x.dst_expected = x.dst_found = x.src_expected = x.src_found = 0;
    x.flags = x.status = 0;
    v[i] = x;
  }
}

int grid_for(uint64_t n) { return (int)std::max<uint64_t>(1, std::min<uint64_t>((n + kT - 1) / kT, 148 * 8)); }

// ---------------------------------------------------------------------------
// NCCL, loaded at run time
// ---------------------------------------------------------------------------
struct Nccl {
  void* h = nullptr;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclGetErrorString) errorString = nullptr;
  bool load(std::string& err) {
    if (h) return true;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) {
      err = "libnccl.so.2 not found";
      return false;
    }
#define CG_SYM(f, s)                                  \
  f = reinterpret_cast<decltype(f)>(dlsym(h, s));     \
  if (!f) {                                           \
    err = std::string("libnccl lacks ") + s;          \
    return false;                                     \
  }
    CG_SYM(getUniqueId, "ncclGetUniqueId")
    CG_SYM(commInitRank, "ncclCommInitRank")
    CG_SYM(commDestroy, "ncclCommDestroy")
    CG_SYM(allReduce, "ncclAllReduce")
    CG_SYM(send, "ncclSend")
    CG_SYM(recv, "ncclRecv")
    CG_SYM(groupStart, "ncclGroupStart")
    CG_SYM(groupEnd, "ncclGroupEnd")
    CG_SYM(errorString, "ncclGetErrorString")
#undef CG_SYM
    return true;
  }
};
Nccl g_nccl;

}  // namespace

struct cg_comm {
  int backend = CG_COMM_LOOPBACK;
  uint32_t world = 1, rank = 0;
  std::vector<cg_ctx*> ctxs;    // local ranks: 1 (NCCL) or world (loopback)
  int device = 0;
  ncclComm_t nccl = nullptr;
  uint64_t mcap = 0, cap = 0, stride = 0;
  // per local rank: mins[2 mcap], sums[5 mcap], maxs[mcap], send[stride]
  std::vector<uint8_t*> scratch;
  uint8_t* recv = nullptr;      // root: world * stride (NCCL); loopback reads the send buffers in place
  uint32_t* d_overflow = nullptr;
  uint64_t launches = 0;
  std::string err;
  cg_status fail(cg_status s, const std::string& m) {
    err = m;
    return s;
  }
  uint64_t* mins(uint32_t r) { return reinterpret_cast<uint64_t*>(scratch[r]); }
  uint64_t* sums(uint32_t r) { return mins(r) + 2 * mcap; }
  uint32_t* maxs(uint32_t r) { return reinterpret_cast<uint32_t*>(sums(r) + 5 * mcap); }
  uint8_t* send(uint32_t r) { return scratch[r] + align(8 * 7 * mcap + 4 * mcap); }
  static uint64_t align(uint64_t x) { return (x + 255) / 256 * 256; }
  uint64_t scratch_bytes() const { return align(8 * 7 * mcap + 4 * mcap) + stride; }
};

extern "C" {

cg_status cg_comm_nccl_id(uint8_t* h_id) {
  if (!h_id) return CG_ERR_INVALID_VALUE;
  std::string err;
  if (!g_nccl.load(err)) return CG_ERR_NCCL;
  ncclUniqueId id;
  if (g_nccl.getUniqueId(&id) != ncclSuccess) return CG_ERR_NCCL;
  static_assert(sizeof(ncclUniqueId) == CG_NCCL_ID_BYTES, "ncclUniqueId size");
  std::memcpy(h_id, &id, sizeof id);
  return CG_OK;
}

static cg_status comm_alloc(cg_comm* c, uint32_t local) {
  c->stride = cg_comm::align(16 + 8 * c->cap + sizeof(cg_verdict) * c->cap);
  for (uint32_t r = 0; r < local; ++r) {
    uint8_t* p = nullptr;
    if (cudaMalloc(&p, c->scratch_bytes()) != cudaSuccess) return c->fail(CG_ERR_OUT_OF_MEMORY, "comm scratch");
    c->scratch.push_back(p);
  }
  if (c->backend == CG_COMM_NCCL && cudaMalloc(&c->recv, c->world * c->stride) != cudaSuccess)
    return c->fail(CG_ERR_OUT_OF_MEMORY, "comm gather buffer");
  if (cudaMalloc(&c->d_overflow, 256) != cudaSuccess || cudaMemset(c->d_overflow, 0, 256) != cudaSuccess)
    return c->fail(CG_ERR_OUT_OF_MEMORY, "comm flags");
  return CG_OK;
}

cg_status cg_comm_destroy(cg_comm* c) {
  if (!c) return CG_ERR_INVALID_VALUE;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(c->device);
  if (c->nccl) g_nccl.commDestroy(c->nccl);
  for (uint8_t* p : c->scratch) cudaFree(p);
  if (c->recv) cudaFree(c->recv);
  if (c->d_overflow) cudaFree(c->d_overflow);
  cudaSetDevice(prev);
  delete c;
  return CG_OK;
}

cg_status cg_comm_create_nccl(cg_ctx* ctx, uint32_t world, uint32_t rank, const uint8_t* h_id,
                              uint64_t max_straddlers, uint64_t cap, cg_comm** out) {
  if (!out || !ctx || !h_id || world == 0 || world > 8 || rank >= world) return CG_ERR_INVALID_VALUE;
  *out = nullptr;
  cg_comm* c = new cg_comm();
  c->backend = CG_COMM_NCCL;
  c->world = world;
  c->rank = rank;
  c->ctxs.push_back(ctx);
  c->device = cg_ctx_device(ctx);
  c->mcap = std::max<uint64_t>(max_straddlers, 1);
  c->cap = std::max<uint64_t>(cap, 1);
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(c->device);
  if (!g_nccl.load(c->err)) {
    cudaSetDevice(prev);
    delete c;
    return CG_ERR_NCCL;
  }
  ncclUniqueId id;
  std::memcpy(&id, h_id, sizeof id);
  if (g_nccl.commInitRank(&c->nccl, (int)world, id, (int)rank) != ncclSuccess) {
    c->nccl = nullptr;
    cudaSetDevice(prev);
    cg_comm_destroy(c);
    return CG_ERR_NCCL;
  }
  const cg_status st = comm_alloc(c, 1);
  cudaSetDevice(prev);
  if (st != CG_OK) {
    cg_comm_destroy(c);
    return st;
  }
  *out = c;
  return CG_OK;
}

cg_status cg_comm_create_loopback(cg_ctx* const* ctxs, uint32_t world, uint64_t max_straddlers, uint64_t cap,
                                  cg_comm** out) {
  if (!out || !ctxs || world == 0 || world > 8) return CG_ERR_INVALID_VALUE;
  *out = nullptr;
  cg_comm* c = new cg_comm();
  c->backend = CG_COMM_LOOPBACK;
  c->world = world;
  for (uint32_t r = 0; r < world; ++r) {
    if (!ctxs[r]) {
      delete c;
      return CG_ERR_INVALID_VALUE;
    }
    c->ctxs.push_back(ctxs[r]);
  }
  c->device = cg_ctx_device(ctxs[0]);
  for (uint32_t r = 1; r < world; ++r)
    if (cg_ctx_device(ctxs[r]) != c->device) {
      delete c;
      return CG_ERR_INVALID_VALUE;   // loopback: one device
    }
  c->mcap = std::max<uint64_t>(max_straddlers, 1);
  c->cap = std::max<uint64_t>(cap, 1);
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(c->device);
  const cg_status st = comm_alloc(c, world);
  cudaSetDevice(prev);
  if (st != CG_OK) {
    cg_comm_destroy(c);
    return st;
  }
  *out = c;
  return CG_OK;
}

const char* cg_comm_last_error(const cg_comm* c) { return c ? c->err.c_str() : "null comm"; }

uint64_t cg_comm_kernel_launches(const cg_comm* c) { return c ? c->launches : 0; }

cg_status cg_comm_overflow(cg_comm* c, uint32_t* overflow) {
  if (!c || !overflow) return CG_ERR_INVALID_VALUE;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(c->device);
  uint32_t h = 0;
  cudaError_t e = cudaMemcpy(&h, c->d_overflow, sizeof h, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemset(c->d_overflow, 0, sizeof h);
  cudaSetDevice(prev);
  if (e != cudaSuccess) return c->fail(CG_ERR_CUDA, cudaGetErrorString(e));
  *overflow = h;
  return CG_OK;
}

static cg_status nccl_check(cg_comm* c, ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return CG_OK;
  return c->fail(CG_ERR_NCCL, std::string(what) + ": " + g_nccl.errorString(r));
}

cg_status cg_check_sharded(cg_comm* c, const cg_shard_batch* b, uint64_t* d_root_idx, cg_verdict* d_root_dirty,
                           uint64_t* d_root_count, cg_verdict* d_dense, uint64_t n_total, void* stream) {
  if (!c || !b) return CG_ERR_INVALID_VALUE;
  const uint32_t local = (uint32_t)c->ctxs.size();
  const uint64_t m = b[0].m;
  for (uint32_t r = 0; r < local; ++r)
    if (b[r].m != m || (b[r].n_own + m && (!b[r].d_descs || !b[r].d_out || !b[r].d_gidx)))
      return c->fail(CG_ERR_INVALID_VALUE, "batches: equal straddler counts and non-null arrays required");
  if (m > c->mcap) return c->fail(CG_ERR_INVALID_VALUE, "more straddlers than max_straddlers");
  const bool root_here = c->backend == CG_COMM_LOOPBACK || c->rank == 0;
  if (root_here && (!d_root_idx || !d_root_dirty || !d_root_count))
    return c->fail(CG_ERR_INVALID_VALUE, "root outputs required on the root");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(c->device);
  cg_status st = CG_OK;
  auto done = [&](cg_status x) {
    cudaSetDevice(prev);
    return x;
  };
  // 1. the check of every local rank's list (fused; raw straddler partials)
  for (uint32_t r = 0; r < local && st == CG_OK; ++r)
    if (b[r].n_own + m) st = cg_check_apply(c->ctxs[r], b[r].d_descs, b[r].n_own + m, b[r].d_out, stream);
  if (st != CG_OK) return done(c->fail(st, std::string("check: ") + cg_last_error(c->ctxs[0])));
  // 2. straddlers: pack, all-reduce, finalize, apply this shard's part
  if (m) {
    for (uint32_t r = 0; r < local && st == CG_OK; ++r)
      st = cg_straddler_pack(c->ctxs[r], b[r].d_out + b[r].n_own, m, c->mins(r), c->sums(r), c->maxs(r), stream);
    if (st != CG_OK) return done(c->fail(st, "straddler pack"));
    if (c->backend == CG_COMM_NCCL) {
      g_nccl.groupStart();
      ncclResult_t x = g_nccl.allReduce(c->mins(0), c->mins(0), 2 * m, ncclUint64, ncclMin, c->nccl, s);
      if (x == ncclSuccess) x = g_nccl.allReduce(c->sums(0), c->sums(0), 5 * m, ncclUint64, ncclSum, c->nccl, s);
      if (x == ncclSuccess) x = g_nccl.allReduce(c->maxs(0), c->maxs(0), m, ncclUint32, ncclMax, c->nccl, s);
      const ncclResult_t y = g_nccl.groupEnd();
      if ((st = nccl_check(c, x != ncclSuccess ? x : y, "straddler all-reduce")) != CG_OK) return done(st);
    } else if (local > 1) {
      Ptrs p{};
      for (uint32_t r = 0; r < local; ++r) {
        p.mins[r] = c->mins(r);
        p.sums[r] = c->sums(r);
        p.maxs[r] = c->maxs(r);
      }
      k_reduce_loopback<<<grid_for(5 * m), kT, 0, s>>>(p, local, m);
      ++c->launches;
    }
    for (uint32_t r = 0; r < local && st == CG_OK; ++r) {
      const uint32_t src = c->backend == CG_COMM_NCCL ? r : 0;   // loopback: the merged values sit in rank 0's buffers
      st = cg_straddler_finalize(c->ctxs[r], c->mins(src), c->sums(src), c->maxs(src), m, b[r].d_out + b[r].n_own,
                                 stream);
      if (st == CG_OK)
        st = cg_apply_dtoh(c->ctxs[r], b[r].d_descs + b[r].n_own, b[r].d_out + b[r].n_own, m, stream);
    }
    if (st != CG_OK) return done(c->fail(st, "straddler finalize / apply"));
  }
  // 3. dirty verdicts with global indices -> send buffers (the root's send
  //    buffer also takes the straddlers), gather to the root, merge there
  for (uint32_t r = 0; r < local; ++r) {
    uint8_t* sb = c->send(r);
    unsigned long long* cnt = reinterpret_cast<unsigned long long*>(sb);
    uint64_t* idx = reinterpret_cast<uint64_t*>(sb + 16);
    cg_verdict* dv = reinterpret_cast<cg_verdict*>(sb + 16 + 8 * c->cap);
    const bool root_rank = c->backend == CG_COMM_LOOPBACK ? r == 0 : c->rank == 0;
    const uint64_t k = b[r].n_own + (root_rank ? m : 0);
    k_zero_u64<<<1, 32, 0, s>>>(cnt, 1);
    if (k) k_compact_gidx<<<grid_for(k), kT, 0, s>>>(b[r].d_out, k, b[r].d_gidx, cnt, idx, dv, c->cap);
    c->launches += k ? 2 : 1;
  }
  const uint8_t* gathered = nullptr;
  if (c->backend == CG_COMM_NCCL) {
    if (c->world > 1) {
      g_nccl.groupStart();
      ncclResult_t x = ncclSuccess;
      if (c->rank == 0) {
        cudaMemcpyAsync(c->recv, c->send(0), c->stride, cudaMemcpyDeviceToDevice, s);
        for (uint32_t r = 1; r < c->world && x == ncclSuccess; ++r)
          x = g_nccl.recv(c->recv + r * c->stride, c->stride, ncclUint8, (int)r, c->nccl, s);
      } else {
        x = g_nccl.send(c->send(0), c->stride, ncclUint8, 0, c->nccl, s);
      }
      const ncclResult_t y = g_nccl.groupEnd();
      if ((st = nccl_check(c, x != ncclSuccess ? x : y, "verdict gather")) != CG_OK) return done(st);
      gathered = c->recv;
    } else {
      gathered = c->send(0);
    }
  }
  if (root_here) {
    if (d_dense) {
      k_fill_clean<<<grid_for(n_total), kT, 0, s>>>(d_dense, n_total);
      ++c->launches;
    }
    Bufs bufs{};
    for (uint32_t r = 0; r < c->world; ++r)
      bufs.p[r] = c->backend == CG_COMM_LOOPBACK ? c->send(r) : gathered + r * c->stride;
    k_root_merge<<<grid_for(c->cap), kT, 0, s>>>(bufs, c->world, c->cap, d_root_idx, d_root_dirty,
                                                 reinterpret_cast<unsigned long long*>(d_root_count), d_dense,
                                                 c->d_overflow);
    ++c->launches;
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return done(c->fail(CG_ERR_CUDA, cudaGetErrorString(e)));
  return done(CG_OK);
}

}  // extern "C"
