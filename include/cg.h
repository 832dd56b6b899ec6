/*
 * cg.h -- C ABI of the B200-native batched Cudagrind transfer checker.
 *
 * Cudagrind (Baumann & Gracia, arXiv 1310.0901) wraps "all CUDA Driver API
 * functions related to allocation, deallocation and transfer of memory" and
 * cross-checks their parameters "against this list [of device allocations]
 * as well as the knowledge of Valgrind about the ... host memory" (PAPER.md
 * §2.2, §3).  This library is the data-parallel core of those
 * checks: it receives what the wrappers observe -- device allocations/frees
 * and batches of copy descriptors -- and answers, on a B200, the paper's error
 * classes plus the DtoH definedness update and the leak
 * sweep (abstract).
 *
 * Conventions
 *  - Every function returns a cg_status (int).  Per-descriptor problems never
 *    fail a call: they are reported in the cg_verdict array ("report and
 *    continue").  Call-level problems (bad arguments, CUDA errors)
 *    return a nonzero status and set cg_last_error(ctx).
 *  - "d_" pointers are device pointers on the context's device; "h_" pointers
 *    are host pointers.  The library never frees caller memory.
 *  - "stream" is a cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream)
 *    or NULL for the legacy default stream.  Asynchronous calls only enqueue
 *    work; the caller synchronises.
 *  - A context is single-writer: calls on one context must
 *    not overlap from several host threads.
 *  - Arithmetic is unsigned 64-bit; there is no floating point anywhere.
 *
 * Host shadow format (readings R-1, R-2):
 *  - the host window is [host_base, host_base + host_size), host_base and
 *    host_size multiples of 4096;
 *  - V: one byte per host byte, bit k set = bit k of that byte undefined
 *    (Memcheck's V polarity); a byte is undefined iff its V-byte != 0;
 *  - A: one bit per host byte, bit (x-host_base)&7 of byte (x-host_base)>>3,
 *    1 = addressable;
 *  - host bytes outside the window are unaddressable (R-15); fresh state is
 *    A = 0, V = 0xFF.
 */
#ifndef CG_H_
#define CG_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (SPEC S:303-306 DriverStatus; CG_ERR_INVALID_VALUE mirrors
 *      CUDA_ERROR_INVALID_VALUE = 1, the "invalid argument" of P:188) ---- */
typedef int cg_status;
enum {
  CG_OK = 0,
  CG_ERR_INVALID_VALUE = 1,
  CG_ERR_INVALID_CONTEXT = 2,
  CG_ERR_OUT_OF_MEMORY = 3,
  CG_ERR_NOT_INITIALIZED = 4,
  CG_ERR_CUDA = 5,
  CG_ERR_NCCL = 6
};

/* ---- copy kinds: host/device, device/host, device/device ----
 * NEXT-3 (Fig. 2 caption P:88 "device arrays"): transfers
 * between host memory and a registered device array.  The array side is
 * (handle, byte offset): HTOA uses dst = handle, dst_x = offset; ATOH uses
 * src = handle, src_x = offset; its y / pitch are ignored.  The host side is a
 * pitched range like HTOD's source / DTOH's destination (pitch rule on the host
 * side only).  The array must be live at desc.seq (else *_NOT_ALLOCATED) and
 * offset + width*height <= its total bytes (else *_TOO_SMALL with expected =
 * width*height, found = total - offset or 0; R-29).  Array V-bits
 * (R-30, "array V-bits tracked in a per-array shadow"): without device
 * V-bit tracking an error-free ATOH makes its host range defined and an HTOA
 * only reads the host shadow (as DTOH / HTOD, R-5); with tracking
 * (cfg.dev_vbuf) every array gets its own V-bits in the pool (fresh =
 * undefined) and error-free HTOA / ATOH copy V-bits host -> array / array ->
 * host. */
enum { CG_HTOD = 1, CG_DTOH = 2, CG_DTOD = 3, CG_HTOA = 4, CG_ATOH = 5 };

/* ---- host mark states (SPEC S:355-358 host_alloc / host_write / host_free) ---- */
enum { CG_NOACCESS = 0, CG_UNDEFINED = 1, CG_DEFINED = 2 };

#define CG_NONE UINT64_MAX

/* ---- verdict flags, in SPEC's diagnostic order (R-14) ---- */
enum {
  CG_F_DST_NOT_ALLOCATED = 1u << 0,  /* P:80 copy into unallocated memory            */
  CG_F_DST_TOO_SMALL = 1u << 1,      /* P:82 copying more than was allocated          */
  CG_F_SRC_NOT_ALLOCATED = 1u << 2,  /* P:80 copy from unallocated memory             */
  CG_F_SRC_TOO_SMALL = 1u << 3,      /* P:82, Listing 5                         */
  CG_F_HOST_UNADDRESSABLE = 1u << 4, /* P:77/P:80 host range not addressable (A-bits) */
  CG_F_HOST_UNDEFINED = 1u << 5,     /* P:81 undefined host data sent (Warning)      */
  CG_F_BAD_PITCH = 1u << 6,          /* R-12: pitch < WidthInBytes + XInBytes         */
  CG_F_INVALID_RANGE = 1u << 7,      /* an address range overflows 64 bits      */
  CG_F_BAD_KIND = 1u << 8,           /* R-16: kind not in {HTOD, DTOH, DTOD, HTOA, ATOH} */
  CG_F_CONCURRENT = 1u << 9          /* NEXT-2: ConcurrentHazard, a Warning (cg_conc_check) */
};

/* One cuMemcpy{HtoD,DtoH,DtoD,2D} call, with the raw CUDA_MEMCPY2D fields
 * (P:62).  96 bytes, 8-byte aligned, array-of-structs.
 *  - 1D copies are 2D copies with height = 1, x = y = 0, pitch = width.
 *  - per side: start = base + y*pitch + x; span = (width==0 || height==0) ? 0
 *    : (height-1)*pitch + width; row r covers [start + r*pitch, +width).
 *  - seq: position of the call in the program's single global event order
 *    (SPEC SimState.seq); the allocation table is evaluated "as of" seq
 *    (an allocation e is visible iff e.alloc_seq < seq < e.free_seq). */
/* Shard mode bits of cg_copy_desc.reserved (host-address-range sharding
 * across GPUs; 0 on a single GPU):
 *  - CG_SHARD_NOT_OWNER: another shard owns the device side (no lookups here);
 *  - CG_SHARD_RAW: the descriptor's host range spans several shards; this
 *    shard writes only its raw partial (first_unaddr, first_undef, undef_count,
 *    device fields, flags without HOST_*; status 0) for cg_straddler_pack /
 *    cg_straddler_finalize after the collective merge. */
enum {
  CG_SHARD_NOT_OWNER = 1u << 0,
  CG_SHARD_RAW = 1u << 1,
  CG_APPLY_AFTER = 1u << 2,
  CG_CHECK_AFTER = 1u << 3,
  CG_APPLY_LAST = 1u << 4
};
/* CG_CHECK_AFTER (cg_check_apply only): this HTOD / HTOA descriptor reads host
 * bytes that an earlier DTOH / ATOH of the same batch writes, so it is
 * checked after every apply of the batch (no later DTOH / ATOH of the batch
 * may write its range).  Set by cg_plan_batches_fused; ignored by
 * cg_check_copies. */
/* CG_APPLY_AFTER (cg_check_apply only): this DTOH / ATOH descriptor's host
 * range overlaps the host range of an HTOD / HTOA descriptor of the same
 * batch, so its apply waits until every check of the batch has read the
 * shadow (the residual pass) instead of running inside the scan.  Set by
 * cg_plan_apply_after. */
/* CG_APPLY_LAST (cg_check_apply only): this DTOH / ATOH descriptor writes host
 * bytes that an earlier CG_CHECK_AFTER HTOD of the same batch reads, so its
 * apply runs after the CG_CHECK_AFTER checks (no later HTOD of the batch may
 * read its range).  Set by cg_plan_batches_fused; cg_check_copies (and the
 * sharded path) treat it as CG_APPLY_AFTER. */

typedef struct {
  uint32_t kind;       /* CG_HTOD / CG_DTOH / CG_DTOD / CG_HTOA / CG_ATOH */
  uint32_t reserved;   /* shard mode bits (CG_SHARD_*), 0 on one GPU   */
  uint64_t seq;
  uint64_t width;      /* WidthInBytes                                 */
  uint64_t height;     /* Height (1 for 1D)                            */
  uint64_t dst, dst_x, dst_y, dst_pitch;
  uint64_t src, src_x, src_y, src_pitch;
} cg_copy_desc;

/* Compact form of a 1D copy (cuMemcpyHtoD / DtoH / DtoD): 40 bytes; equal to
 * the cg_copy_desc {kind, seq, width = bytes, height = 1, dst, src,
 * pitches = bytes, x = y = 0}. */
typedef struct {
  uint32_t kind, reserved;
  uint64_t seq, dst, src, bytes;
} cg_copy1d;

/* descriptor formats accepted by cg_check_host */
enum { CG_FMT_2D = 0, CG_FMT_1D = 1 };

/* Result for one descriptor.  64 bytes.  Clean = {NONE, NONE, 0, 0,0,0,0, 0, 0}.
 *  - first_unaddr: lowest logical offset o = r*width + c of a host byte that is
 *    not addressable (SPEC check_addressable S:63-71), else CG_NONE;
 *  - first_undef / undef_count: HtoD only -- lowest offset / number of
 *    addressable host bytes with a nonzero V-byte (R-3, R-6);
 *  - *_expected / *_found: for *_TOO_SMALL only, the device span and the bytes
 *    from start to the end of the allocation containing start (Listing 5
 *    "Expected 8000000 allocated bytes but only found 4000000"; S:160,
 *    S:192); 0 otherwise (R-19);
 *  - status: CG_ERR_INVALID_VALUE iff an Error flag is set;
 *    every flag except HOST_UNDEFINED is an Error unless undef_is_error. */
typedef struct {
  uint64_t first_unaddr, first_undef, undef_count;
  uint64_t dst_expected, dst_found, src_expected, src_found;
  uint32_t flags, status;
} cg_verdict;

/* One live allocation in a leak report, ascending base. */
typedef struct {
  uint64_t base, size, alloc_seq;
} cg_alloc_record;

/* One host shadow update for cg_host_mark_batch.  24 bytes. */
typedef struct {
  uint64_t addr, len;
  uint32_t state;      /* CG_NOACCESS / CG_UNDEFINED / CG_DEFINED */
  uint32_t reserved;
} cg_mark;

/* Context configuration.  All device buffers are caller-owned (e.g. torch
 * tensors) and must stay alive until cg_ctx_destroy.
 *  - host_base/host_size: the global host window (multiples of 4096).
 *  - shard_base/shard_size: the part of the window whose shadow this context
 *    stores (host-address-range sharding across GPUs); 0/0 = the whole window.
 *    Multiples of 4096, inside the window.
 *  - v_buf: shard_size bytes; a_buf: shard_size/8 bytes; both 16-byte aligned.
 *  - workspace: >= cg_workspace_size(cfg) bytes, 256-byte aligned.
 *  - max_descs: largest n accepted by one check/apply/mark-batch call.
 *  - max_allocs: allocation-table capacity (live entries plus tombstones).
 *  - host_staging: nonzero reserves device staging in the workspace for
 *    cg_check_copies_host / cg_check_host[_submit] (two slots of descriptors,
 *    verdicts and dirty lists of max_descs each).
 *  - dev_vbuf / dev_vsize (NEXT-1; SPEC copy_vbits S:81-89):
 *    non-NULL enables device V-bit tracking.  Every registered allocation gets
 *    `size` bytes of device V-bits in this caller-owned pool (bump allocated,
 *    never reused; fresh = undefined) and cg_apply_copies moves V-bits
 *    through error-free copies (HtoD host->device, DtoD device->device with
 *    memmove semantics, DtoH device->host) instead of R-5's "DtoH marks the
 *    host range defined".  dev_vbuf must be 16-byte aligned and dev_vsize a
 *    multiple of 16 (the propagation stages 16-byte-aligned supersets of
 *    its ranges with bulk copies).  Requires an
 *    unsharded context.
 *  - shadow_format (NEXT-4): CG_SHADOW_BYTES (0) = one V byte per
 *    host byte + one A bit per host byte (v_buf / a_buf as above);
 *    CG_SHADOW_2BIT (1) = Memcheck-style compressed states, 2 bits per host
 *    byte {NOACCESS, PARTIAL, DEFINED, UNDEFINED} in v_buf (shard_size/4
 *    bytes, 16-byte aligned; a_buf unused, may be NULL).  Exact partial
 *    V-bytes (cg_host_set_vbits values other than 0x00 / 0xFF) are kept in a
 *    host-side table for cg_host_shadow_read; the checks only need "some bit
 *    undefined", which the state holds (R-36).  The scan then reads
 *    0.25 B per host byte for both kinds and the DtoH apply writes 0.25 B.
 *    Not combinable with dev_vbuf.
 *    CG_SHADOW_SPARSE (2) = the same states in a Memcheck-style two-level map
 *    over the whole 64-bit host address space: 64 KiB host chunks, each with
 *    a 16 KiB secondary of states allocated on first mark (a chunk without one
 *    is NOACCESS).  host_base must be 0 and host_size is the capacity in host
 *    bytes (a multiple of 65536): v_buf holds host_size/65536 + 1 secondaries
 *    (the first is the distinguished NOACCESS one).  Every host address is
 *    then "in the window"; marks that need more secondaries than the capacity
 *    fail with CG_ERR_OUT_OF_MEMORY.  Unsharded, no dev_vbuf. */
enum { CG_SHADOW_BYTES = 0, CG_SHADOW_2BIT = 1, CG_SHADOW_SPARSE = 2 };

typedef struct {
  uint64_t host_base, host_size;
  uint64_t shard_base, shard_size;
  uint64_t max_descs, max_allocs;
  uint32_t undef_is_error;  /* S:284 promotes HOST_UNDEFINED to an Error */
  uint32_t host_staging;
  int32_t device;           /* CUDA device ordinal                       */
  int32_t shadow_format;    /* CG_SHADOW_BYTES / CG_SHADOW_2BIT (NEXT-4) */
  void *v_buf, *a_buf, *workspace;
  uint64_t workspace_size;
  void *dev_vbuf;           /* NEXT-1 device V-bit pool (or NULL)        */
  uint64_t dev_vsize;
} cg_config;

typedef struct cg_ctx cg_ctx;

/* Bytes of device workspace a context with this configuration needs (0 if the
 * configuration is invalid). */
uint64_t cg_workspace_size(const cg_config *cfg);

/* Creates a context: validates cfg, carves the workspace, resets the shard's
 * shadow to the fresh state (A = 0, V = 0xFF) on the device.  Synchronous.
 * Errors: CG_ERR_INVALID_VALUE (null, misaligned or inconsistent window /
 * shard / buffers, workspace too small), CG_ERR_CUDA. */
cg_status cg_ctx_create(const cg_config *cfg, cg_ctx **out);

/* Frees the context (not the caller's buffers).  Does not run the leak sweep:
 * call cg_leak_report first (SPEC S:317 runs it at destroy; here it is explicit).
 * Errors: CG_ERR_INVALID_CONTEXT on NULL. */
cg_status cg_ctx_destroy(cg_ctx *ctx);

/* Message for the last call-level error on ctx ("" if none); owned by ctx. */
const char *cg_last_error(const cg_ctx *ctx);

/* Host shadow update (SPEC mark_addressable / mark_unaddressable S:45-62;
 * host_alloc / host_write / host_free S:355-363): every byte of
 * [addr, addr+len) gets NOACCESS (A=0, V=0xFF), UNDEFINED (A=1, V=0xFF) or
 * DEFINED (A=1, V=0x00).  Stream-ordered.  Only the part inside this context's
 * shard is stored.  Errors: CG_ERR_INVALID_VALUE if the range leaves the
 * window or state is unknown (nothing is changed). */
cg_status cg_host_mark(cg_ctx *ctx, uint64_t addr, uint64_t len, uint32_t state, void *stream);

/* n marks applied as if by n cg_host_mark calls in order.  h_marks is a host
 * array, copied before return.  An invalid mark (range leaving the window,
 * unknown state) is skipped and only it: its status (CG_ERR_INVALID_VALUE) is
 * written to h_status[i] when h_status is not NULL (CG_OK for applied marks).
 * Any n is accepted (uploaded in runs of at most min(max_descs, 2^20) marks).
 * Returns CG_OK if every mark was applied, else CG_ERR_INVALID_VALUE (also for
 * NULL h_marks, when nothing is applied). */
cg_status cg_host_mark_batch(cg_ctx *ctx, const cg_mark *h_marks, uint64_t n, uint32_t *h_status,
                             void *stream);

/* Sets exact V-bytes (partial-bit definedness) of
 * [addr, addr+len) from the host array h_vbytes (copied before return).
 * Synchronous on stream.  Errors: CG_ERR_INVALID_VALUE if any byte of the
 * range is unaddressable or outside the window (defined => addressable);
 * nothing is changed then. */
cg_status cg_host_set_vbits(cg_ctx *ctx, uint64_t addr, uint64_t len, const uint8_t *h_vbytes,
                            void *stream);

/* Synchronous read of the host shadow of [addr, addr+len), which must lie in
 * this context's shard, in the plain form of either format: h_a[i] = 1 if
 * byte addr+i is addressable else 0, h_v[i] = its V-byte (0xFF for
 * unaddressable bytes); either output may be NULL.  Inspection / tests.
 * Errors: CG_ERR_INVALID_VALUE (range outside the shard), CG_ERR_CUDA. */
cg_status cg_host_shadow_read(cg_ctx *ctx, uint64_t addr, uint64_t len, uint8_t *h_a, uint8_t *h_v, void *stream);

/* Synchronous query: *all_addressable = 1 iff every byte of [addr, addr+len)
 * that this context's shard stores is addressable and the range lies in the
 * window (a sharded cg_host_set_vbits asks every shard first).  Errors:
 * CG_ERR_INVALID_VALUE on NULL. */
cg_status cg_host_query_addressable(cg_ctx *ctx, uint64_t addr, uint64_t len, uint32_t *all_addressable,
                                    void *stream);

/* Registers a device allocation (Fig. 2 caption P:88: "Each allocation
 * generates a new entry into the list"; SPEC register_linear S:139-147).
 * seq must exceed the seq of every earlier successful cg_register_alloc /
 * cg_free.  Errors (no mutation): CG_ERR_INVALID_VALUE for size 0, base 0,
 * base+size > 2^64-1, overlap with a live allocation, non-increasing
 * seq; CG_ERR_OUT_OF_MEMORY when the table (live + tombstones) is full. */
cg_status cg_register_alloc(cg_ctx *ctx, uint64_t base, uint64_t size, uint64_t seq);

/* Frees the live allocation whose base is ptr (SPEC unregister_linear
 * S:148-156, mem_free S:332-340).  The entry stays in the table as a
 * tombstone with free_seq = seq so that descriptors with smaller seq still see
 * it.  Errors (no mutation): CG_ERR_INVALID_VALUE = InvalidFree (ptr is not a
 * live base: offset pointer, double free, 0) or non-increasing seq. */
cg_status cg_free(cg_ctx *ctx, uint64_t ptr, uint64_t seq);

/* A registry event for cg_registry_batch: op CG_REG_ALLOC (cg_register_alloc
 * of addr, size) or CG_REG_FREE (cg_free of addr).  32 bytes. */
enum { CG_REG_ALLOC = 1, CG_REG_FREE = 2 };
typedef struct {
  uint32_t op, reserved;
  uint64_t seq, addr, size;
} cg_reg_event;

/* n registry events applied in order, as n cg_register_alloc / cg_free calls
 * (one call crossing the ABI instead of n); h_status[i] (if not NULL) gets
 * event i's status.  The device table follows by difference at the next
 * check (new entries and changed free stamps only).  Returns CG_OK if every
 * event succeeded, else the first failing status (the others still apply). */
cg_status cg_registry_batch(cg_ctx *ctx, const cg_reg_event *h_events, uint64_t n, uint32_t *h_status);

/* Drops tombstones with free_seq <= before_seq (no later descriptor may have
 * seq < before_seq).  Synchronous host operation.  Tombstones count against
 * max_allocs until dropped: a long-running caller compacts at its epoch
 * boundaries (the replay driver does when half the capacity was registered
 * since the last compaction), else cg_register_alloc eventually returns
 * CG_ERR_OUT_OF_MEMORY. */
cg_status cg_registry_compact(cg_ctx *ctx, uint64_t before_seq);

/* NEXT-3: bytes of a CUDA array (SPEC register_array S:166-168):
 * width * max(height,1) * max(depth,1) * format_bytes * channels, with
 * format_bytes = {1,2,4,1,2,4,2,4}[format] (u8,u16,u32,i8,i16,i32,f16,f32) and
 * channels in {1,2,4}.  0 for width 0, an unknown format / channel count or a
 * product above 2^64-1. */
uint64_t cg_array_bytes(uint64_t width, uint64_t height, uint64_t depth, uint32_t format, uint32_t channels);

/* NEXT-3: registers a device array under its handle (cuArrayCreate /
 * cuArray3DCreate; the Fig. 2 caption P:88 lists arrays in the allocation list).  Shares the seq order of cg_register_alloc /
 * cg_free.  Errors (no mutation): CG_ERR_INVALID_VALUE for a zero extent
 * (cg_array_bytes == 0), a handle that is already live
 * (DuplicateHandle) or a non-increasing seq; CG_ERR_OUT_OF_MEMORY when the
 * array table (live + tombstones, capacity max_allocs) is full. */
cg_status cg_register_array(cg_ctx *ctx, uint64_t handle, uint64_t width, uint64_t height, uint64_t depth,
                            uint32_t format, uint32_t channels, uint64_t seq);

/* NEXT-3: frees the live array with this handle (cuArrayDestroy); it stays a
 * tombstone with free_seq = seq (dropped by cg_registry_compact).  Errors (no
 * mutation): CG_ERR_INVALID_VALUE = UnknownHandle or non-increasing seq. */
cg_status cg_free_array(cg_ctx *ctx, uint64_t handle, uint64_t seq);

/* NEXT-3: live arrays at the end of the program (the array half of the leak
 * report): records {handle, total bytes, alloc_seq} in ascending
 * handle order into the host array h_out (at most cap), *n_out = how many are
 * live.  Synchronous host operation. */
cg_status cg_array_report(cg_ctx *ctx, cg_alloc_record *h_out, uint64_t cap, uint64_t *n_out);

/* ---- NEXT-2: concurrency hazards ("certain concurrent
 * accesses when several threads are used"; SPEC check_concurrent S:258-266,
 * rule S:285; R-31..R-35) ----
 * A separate checker object that owns its device memory.  Every side of a
 * copy is an access of its address space (host / device; R-32) over its
 * folded [start, start+span) (R-33).  An access is a ConcurrentHazard iff the
 * newest earlier recorded access overlapping it was made by another thread
 * that has not called cg_conc_sync since, and one of the two writes.  Only
 * copies whose verdict status is CG_OK are recorded (R-34).  The state between
 * calls is, per address space, the last-access map: disjoint ranges tagged
 * with the stamp that touched them last. */
typedef struct cg_conc cg_conc;

/* max_n: largest batch of cg_conc_check; max_stamps: capacity of each address
 * space's last-access map (ranges).  2*max_n + max_stamps < 2^30.  Allocates
 * on `device` with cudaMalloc (freed by cg_conc_destroy).  Errors:
 * CG_ERR_INVALID_VALUE, CG_ERR_CUDA, CG_ERR_OUT_OF_MEMORY. */
cg_status cg_conc_create(int device, uint64_t max_n, uint64_t max_stamps, cg_conc **out);
cg_status cg_conc_destroy(cg_conc *c);
const char *cg_conc_last_error(const cg_conc *c);

/* ctx_synchronize by `thread` at `seq` (R-31: marks that thread's
 * earlier stamps synced for every later access).  Must be submitted before the
 * cg_conc_check of any copy with a larger seq.  Host-only. */
cg_status cg_conc_sync(cg_conc *c, uint32_t thread, uint64_t seq);

/* check_concurrent for a batch: d_descs (n cg_copy_desc, in seq order, every
 * seq larger than those of earlier batches) with their issuing threads
 * d_threads (n uint32) and the verdicts the transfer check wrote for them
 * (d_verdicts; status decides R-34's recording).  Sets CG_F_CONCURRENT in the
 * verdict flags of every hazardous copy (status unchanged, R-35), then updates
 * the last-access maps.  Overlaps inside the batch are resolved exactly (no
 * planner cut is needed).  Synchronous on stream.  Errors: CG_ERR_INVALID_VALUE
 * (null, n > max_n, seqs not strictly increasing or not above every seq of
 * the earlier batches -- nothing is flagged or recorded then), CG_ERR_OUT_OF_MEMORY (a map would exceed max_stamps: the
 * flags are written, the maps are left as before), CG_ERR_CUDA. */
cg_status cg_conc_check(cg_conc *c, const cg_copy_desc *d_descs, const uint32_t *d_threads, uint64_t n,
                        cg_verdict *d_verdicts, void *stream);

/* Ranges in the host / device last-access maps (inspection). */
cg_status cg_conc_stamps(const cg_conc *c, uint64_t *n_host, uint64_t *n_device);
uint64_t cg_conc_kernel_launches(const cg_conc *c);

/* The check for a batch of n descriptors:
 * validation, batched interval search in the allocation table as of each
 * desc.seq, host A/V shadow scan, verdicts.
 * Contract: every registry event with seq < max(desc.seq) has been submitted;
 * the host shadow is read as of the call (snapshot), so the batch must be
 * hazard-free (no HtoD may overlap an earlier DtoH of the same batch; see
 * cg_plan_batches).  d_descs: device array of n cg_copy_desc; d_out: device
 * array of n cg_verdict (fully overwritten); both 16-byte aligned.
 * Asynchronous on stream.
 * Errors: CG_ERR_INVALID_VALUE (null, misaligned, n > max_descs), CG_ERR_CUDA. */
cg_status cg_check_copies(cg_ctx *ctx, const cg_copy_desc *d_descs, uint64_t n, cg_verdict *d_out,
                          void *stream);

/* The DtoH shadow update (BASELINE north_star (3));
 * with device V-bit tracking (cfg.dev_vbuf) this is cg_apply_copies:
 * for every descriptor with kind == CG_DTOH or CG_ATOH and verdict status ==
 * CG_OK, every written host byte becomes defined (V := 0x00); other descriptors are ignored
 * (no mutation on error).  Asynchronous on stream.
 * Errors: as cg_check_copies. */
cg_status cg_apply_dtoh(cg_ctx *ctx, const cg_copy_desc *d_descs, const cg_verdict *d_verdicts,
                        uint64_t n, void *stream);

/* The a6 step generalised (NEXT-1): without device V-bit tracking identical
 * to cg_apply_dtoh; with it, every descriptor whose verdict is OK moves its
 * V-bits (HtoD: host -> device pool, DtoD: pool -> pool as if staged through a
 * scratch buffer, DtoH: pool -> host; HtoA: host -> array V-bits, AtoH: array
 * V-bits -> host, R-30).  Must follow the cg_check_copies call of
 * the same descriptor array (it uses the device V offsets that check found);
 * the batch must be hazard-free for propagation (cg_plan_batches with
 * CG_PLAN_PROPAGATE).  With tracking it synchronises on stream at the end.
 * A self-overlapping 2D DtoD with unequal pitches is staged through an 8 MiB
 * area; a larger one is staged, after the rest of the batch, through a device
 * buffer of its own size the call allocates and frees (cudaMallocAsync).
 * Errors: as cg_apply_dtoh; CG_ERR_INVALID_VALUE if the preceding check was of
 * other descriptors; CG_ERR_OUT_OF_MEMORY if that staging buffer cannot be had. */
cg_status cg_apply_copies(cg_ctx *ctx, const cg_copy_desc *d_descs, const cg_verdict *d_verdicts, uint64_t n,
                          void *stream);

/* NEXT-1 propagation of a subset: the m descriptors d_index[0..m) (device
 * uint32 indices into the n descriptors of the preceding cg_check_copies, each
 * at most once) move their V-bits as in cg_apply_copies.  With the waves of
 * cg_plan_waves this propagates a batch whose copies read or write each
 * other's bytes: wave by wave, in level order.  max_bytes: the largest
 * width*height among the m copies if the caller knows it (waves of copies up
 * to 1 MiB then run one warp per copy without a plan), else 0.
 * Asynchronous on stream: a
 * self-overlapping 2D DtoD that does not fit the staging area is moved by the
 * next cg_apply_flush.  Errors: CG_ERR_INVALID_VALUE (null, m > n, not
 * the checked descriptors), CG_ERR_NOT_INITIALIZED without tracking, CG_ERR_CUDA. */
cg_status cg_apply_copies_subset(cg_ctx *ctx, const cg_copy_desc *d_descs, const cg_verdict *d_verdicts, uint64_t n,
                                 const uint32_t *d_index, uint64_t m, uint64_t max_bytes, void *stream);

/* Synchronises stream and moves the V-bits of the self-overlapping 2D DtoDs
 * the cg_apply_copies_subset calls since the last flush could not stage (more
 * than 8 MiB), each through a device buffer of its size; call it between a
 * wave holding such a copy and a later wave that depends on it
 * (cg_apply_copies_waves does).  Errors: CG_ERR_OUT_OF_MEMORY, CG_ERR_CUDA. */
cg_status cg_apply_flush(cg_ctx *ctx, void *stream);

/* All waves of a batch in one call: wave w is d_index[h_wave_start[w] ..
 * h_wave_start[w+1]) with largest copy h_max_bytes[w] (host arrays of
 * n_waves + 1 and n_waves entries), propagated in order by
 * cg_apply_copies_subset, then cg_apply_flush.  Synchronous. */
cg_status cg_apply_copies_waves(cg_ctx *ctx, const cg_copy_desc *d_descs, const cg_verdict *d_verdicts, uint64_t n,
                                const uint32_t *d_index, const uint64_t *h_wave_start, const uint64_t *h_max_bytes,
                                uint32_t n_waves, void *stream);

/* NEXT-1 wave planner (host): h_level[i] = 1 + the highest level of an
 * earlier descriptor of the batch whose V-bit reads / writes conflict with
 * descriptor i's (read-after-write, write-after-read, write-after-write on
 * host or device bytes, the sets of cg_plan_batches_propagate; R-28), 0 if
 * none; *n_levels = number of levels.  Propagating level 0, then 1, ... with
 * cg_apply_copies_subset equals propagating the copies one by one in order.
 * Errors: CG_ERR_INVALID_VALUE on NULL. */
cg_status cg_plan_waves(const cg_copy_desc *h_descs, uint64_t n, uint32_t *h_level, uint32_t *n_levels);

/* Downloads the device V-bits of [addr, addr+len) (inside one allocation live
 * now) to h_out (NEXT-1 state inspection).  Synchronous.  Errors:
 * CG_ERR_NOT_INITIALIZED without tracking; CG_ERR_INVALID_VALUE if the range
 * is not inside one live allocation. */
cg_status cg_device_vbits(cg_ctx *ctx, uint64_t addr, uint64_t len, uint8_t *h_out);

/* NEXT-1 x NEXT-3: downloads the V-bits of bytes [offset, offset+len) of the
 * live array `handle` (its per-array shadow; R-30) to h_out.
 * Synchronous.  Errors: CG_ERR_NOT_INITIALIZED without tracking;
 * CG_ERR_INVALID_VALUE if there is no such live array or the range leaves it. */
cg_status cg_array_vbits(cg_ctx *ctx, uint64_t handle, uint64_t offset, uint64_t len, uint8_t *h_out);

/* cg_check_copies followed by cg_apply_dtoh, fused: the shadow scan applies
 * every DtoH descriptor that fits one of its work groups as soon as its verdict
 * is final, and a residual apply pass handles the rest.  Same results as the
 * two calls PROVIDED that every DtoH descriptor whose host range overlaps an
 * HtoD host range of the batch carries CG_APPLY_AFTER (cg_plan_apply_after
 * sets exactly those; a batch where cg_batch_disjoint holds needs none).
 * Asynchronous on stream.  Errors: as cg_check_copies. */
cg_status cg_check_apply(cg_ctx *ctx, const cg_copy_desc *d_descs, uint64_t n, cg_verdict *d_out,
                         void *stream);

/* Host helper: *disjoint = 1 iff no HtoD host range of the n descriptors
 * overlaps any DtoH host range of them (the precondition of cg_check_apply).
 * Errors: CG_ERR_INVALID_VALUE on NULL. */
cg_status cg_batch_disjoint(const cg_copy_desc *h_descs, uint64_t n, int *disjoint);

/* Host helper for cg_check_apply: sets CG_APPLY_AFTER in h_descs[i].reserved
 * for every DTOH / ATOH descriptor whose host range (bounding range for 2D)
 * overlaps the host range of any HTOD / HTOA descriptor of the n (in either
 * order) and clears it elsewhere; *n_after = how many carry it.  Errors:
 * CG_ERR_INVALID_VALUE on NULL. */
cg_status cg_plan_apply_after(cg_copy_desc *h_descs, uint64_t n, uint64_t *n_after);

/* End-to-end entry point with HOST buffers: copies h_descs to the device,
 * runs cg_check_copies (apply = 0), cg_check_copies + cg_apply_dtoh
 * (apply = 1) or cg_check_apply (apply = 2, same precondition) and copies the
 * verdicts back to h_out.  Synchronous.  Requires cfg.host_staging and staging
 * slot 0 free (no batch submitted to it and not waited for).  Errors: as
 * cg_check_copies; CG_ERR_NOT_INITIALIZED without host staging. */
cg_status cg_check_copies_host(cg_ctx *ctx, const cg_copy_desc *h_descs, uint64_t n, cg_verdict *h_out,
                               int apply, void *stream);

/* Expands n compact 1D descriptors (device array d_in) into cg_copy_desc
 * records (device array d_out); asynchronous.  Errors: CG_ERR_INVALID_VALUE on
 * NULL. */
cg_status cg_expand_copy1d(cg_ctx *ctx, const cg_copy1d *d_in, uint64_t n, cg_copy_desc *d_out, void *stream);

/* End-to-end entry point with HOST buffers and a compact result: uploads the
 * n host descriptors (format CG_FMT_2D: cg_copy_desc, CG_FMT_1D: cg_copy1d),
 * checks them -- apply = 0: cg_check_copies, 1: + cg_apply_dtoh, 2:
 * cg_check_apply (needs an apply-disjoint batch) -- and downloads only the
 * dirty verdicts: h_idx[k] (descriptor index) and h_dirty[k] for
 * k < min(*n_dirty, cap), in unspecified order; every other descriptor's
 * verdict is the clean one.  The batch is processed in up to 4 chunks whose
 * host->device copies run on a second stream under the previous chunk's
 * kernels (pinned host memory makes them asynchronous).  Synchronous.
 * Requires cfg.host_staging.  Errors: as cg_check_copies; CG_ERR_NOT_INITIALIZED
 * without host staging. */
cg_status cg_check_host(cg_ctx *ctx, const void *h_descs, uint32_t format, uint64_t n, int apply, uint64_t *h_idx,
                        cg_verdict *h_dirty, uint64_t cap, uint64_t *n_dirty, void *stream);

/* The same in two halves, for a stream of batches (double buffering): the
 * context has two staging slots.  cg_check_host_submit enqueues batch n's
 * upload (copy stream, waiting only until the slot's previous batch stopped
 * reading its staging), check (stream) and dirty-verdict compaction into
 * staging slot `slot` (0 or 1) and returns without waiting, so the next
 * batch's upload overlaps this batch's kernels.  cg_check_host_wait(slot)
 * waits for that batch and downloads its dirty verdicts (on a third stream:
 * kernels of a batch submitted later keep running).  Batches are checked in
 * submission order on the stream, exactly as consecutive cg_check_host calls.
 * h_descs (pinned for the upload to be asynchronous) must stay unchanged until
 * the wait returns.  A slot takes one batch at a time.  Errors: as
 * cg_check_host; CG_ERR_INVALID_VALUE for a slot > 1, a submit to a slot whose
 * batch was not waited for, or a wait on a slot with no batch. */
cg_status cg_check_host_submit(cg_ctx *ctx, const void *h_descs, uint32_t format, uint64_t n, int apply,
                               uint32_t slot, void *stream);
cg_status cg_check_host_wait(cg_ctx *ctx, uint32_t slot, uint64_t *h_idx, cg_verdict *h_dirty, uint64_t cap,
                             uint64_t *n_dirty);

/* Straddler exchange, step 1 (device, asynchronous): the m raw partial
 * verdicts d_raw (CG_SHARD_RAW descriptors, in the same order on every shard)
 * become three arrays for collectives: d_mins[2m] (reduce with MIN, u64),
 * d_sums[5m] (SUM, u64), d_maxs[m] (MAX, u32).  Errors: CG_ERR_INVALID_VALUE
 * on NULL. */
cg_status cg_straddler_pack(cg_ctx *ctx, const cg_verdict *d_raw, uint64_t m, uint64_t *d_mins,
                            uint64_t *d_sums, uint32_t *d_maxs, void *stream);

/* Straddler exchange, step 2: after the three all-reduces over all shards,
 * writes the m final verdicts (flags and status derived exactly as for an
 * unsharded descriptor) to d_out.  Errors: CG_ERR_INVALID_VALUE on NULL. */
cg_status cg_straddler_finalize(cg_ctx *ctx, const uint64_t *d_mins, const uint64_t *d_sums,
                                const uint32_t *d_maxs, uint64_t m, cg_verdict *d_out, void *stream);

/* Verdicts with any flag set -> d_idx[k] (position in d_verdicts) and
 * d_dirty[k], k < *d_count (a device u32; order not specified).  Clean
 * verdicts are canonical ({NONE, NONE, 0, 0, 0, 0, 0, 0, 0}), so (count, idx,
 * dirty) reconstruct the array -- the payload of the verdict gather to the
 * root.  d_idx / d_dirty need room for n entries.  Asynchronous. */
cg_status cg_compact_dirty(cg_ctx *ctx, const cg_verdict *d_verdicts, uint64_t n, uint64_t *d_idx,
                           cg_verdict *d_dirty, uint32_t *d_count, void *stream);

/* Host helper for host-address-range sharding over `world` equal shards of
 * the window [host_base, host_base + host_size): per descriptor, the owner
 * shard (the one holding the host start, clamped into the window; index mod
 * world without a host side) and the first/last shard holding shadow bytes of
 * its host range (first < last: a straddler).  Errors: CG_ERR_INVALID_VALUE if
 * the shards are not multiples of 4096 or on NULL. */
cg_status cg_shard_plan(const cg_copy_desc *h_descs, uint64_t n, uint64_t host_base, uint64_t host_size,
                        uint32_t world, uint32_t *h_owner, uint32_t *h_first, uint32_t *h_last);

/* ---- host-address-range shards inside the library (
 * BASELINE north_star: the shadow address space and the copy batch are
 * partitioned across GPUs by host-address range, with an NCCL gather of the
 * per-descriptor verdicts) ----
 * A shard group is G <= 8 contexts whose shards split the same global window,
 * every one holding the whole (replicated) allocation table.  cg_comm is the
 * group's collective backend: NCCL (one rank = one context per process; the
 * library loads libnccl.so.2 with dlopen -- in a torch process the copy torch
 * loaded) or LOOPBACK (all G contexts in this process, on one device; the
 * collectives read the G ranks' device buffers directly). */
typedef struct cg_comm cg_comm;
enum { CG_COMM_NCCL = 0, CG_COMM_LOOPBACK = 1 };
#define CG_NCCL_ID_BYTES 128

/* CUDA device ordinal of a context (or -1 for NULL). */
int cg_ctx_device(const cg_ctx *ctx);

/* A fresh NCCL unique id (128 bytes into h_id) -- on rank 0; the caller hands
 * it to every rank (e.g. a torch.distributed broadcast).  CG_ERR_NCCL if
 * libnccl cannot be loaded. */
cg_status cg_comm_nccl_id(uint8_t *h_id);

/* NCCL backend for this process's context `ctx`, rank `rank` of `world`
 * (<= 8); every rank calls it with the same id (collective).
 * max_straddlers: the most straddling descriptors one cg_check_sharded call
 * may carry; cap: the most dirty verdicts one rank sends to the root per call
 * (fixed-size gather buffers; more are counted and reported by
 * cg_comm_overflow).  The comm allocates its own device scratch (cudaMalloc,
 * freed by cg_comm_destroy).  Errors: CG_ERR_INVALID_VALUE, CG_ERR_NCCL,
 * CG_ERR_OUT_OF_MEMORY. */
cg_status cg_comm_create_nccl(cg_ctx *ctx, uint32_t world, uint32_t rank, const uint8_t *h_id,
                              uint64_t max_straddlers, uint64_t cap, cg_comm **out);

/* LOOPBACK backend over the world (<= 8) contexts ctxs[0..world) of this
 * process, all on one device; rank r = ctxs[r], rank 0 is the root. */
cg_status cg_comm_create_loopback(cg_ctx *const *ctxs, uint32_t world, uint64_t max_straddlers, uint64_t cap,
                                  cg_comm **out);
cg_status cg_comm_destroy(cg_comm *comm);
const char *cg_comm_last_error(const cg_comm *comm);
uint64_t cg_comm_kernel_launches(const cg_comm *comm);

/* Synchronous: *overflow = 1 if, since the last query, some rank had more
 * dirty verdicts than `cap` in a cg_check_sharded call (the root's list is
 * then incomplete; the ranks' own verdict arrays are still exact); resets it. */
cg_status cg_comm_overflow(cg_comm *comm, uint32_t *overflow);

/* One local rank's part of a sharded batch (cg_shard_lists builds it). */
typedef struct {
  const cg_copy_desc *d_descs;   /* n_own owned descriptors, then the m straddlers (device) */
  uint64_t n_own, m;             /* m: equal on every rank, same straddlers in the same order */
  const uint64_t *d_gidx;        /* n_own + m global indices of the listed descriptors (device) */
  cg_verdict *d_out;             /* n_own + m verdicts, final after the call (device) */
} cg_shard_batch;

/* The sharded check of one batch (a hazard-free R-20 epoch), for every local
 * rank of comm (batches[r]; NCCL: one), asynchronous on stream with no host
 * synchronisation: the fused check + DtoH apply of each rank's list, the
 * straddler exchange (pack, three all-reduces: MIN of the first offsets, SUM
 * of the count and of the owner-only device fields, MAX = OR of the flags;
 * finalize on every rank; each rank applies its shard part of the straddling
 * DtoH copies with status OK), then every rank's dirty verdicts with their
 * global indices gathered to the root (rank 0) and merged there by a kernel
 * into d_root_idx / d_root_dirty (capacity world * cap) with the count in
 * *d_root_count (device u64), and, if d_dense is not NULL, scattered into the
 * dense d_dense[n_total] (clean entries canonical).  Root outputs are only
 * read on the root (may be NULL elsewhere).  Errors: CG_ERR_INVALID_VALUE
 * (unequal m, m > max_straddlers, NULL), CG_ERR_NCCL, CG_ERR_CUDA, and those
 * of cg_check_apply. */
cg_status cg_check_sharded(cg_comm *comm, const cg_shard_batch *batches, uint64_t *d_root_idx,
                           cg_verdict *d_root_dirty, uint64_t *d_root_count, cg_verdict *d_dense, uint64_t n_total,
                           void *stream);

/* Host planner of a sharded batch: rank `rank`'s list of the n descriptors
 * h_descs (an R-20 epoch) over `world` equal shards of [host_base, host_base +
 * host_size): the descriptors it owns (cg_shard_plan: host range in its shard
 * only, or no host side and index mod world == rank) in order, then every
 * straddler in order with CG_SHARD_RAW (and CG_SHARD_NOT_OWNER unless it owns
 * it), CG_APPLY_AFTER set as cg_plan_apply_after sets it on the list.  h_out /
 * h_gidx need room for n entries; *n_own, *m receive the counts.  Errors:
 * CG_ERR_INVALID_VALUE (as cg_shard_plan). */
cg_status cg_shard_lists(const cg_copy_desc *h_descs, uint64_t n, uint64_t host_base, uint64_t host_size,
                         uint32_t world, uint32_t rank, cg_copy_desc *h_out, uint64_t *h_gidx, uint64_t *n_own,
                         uint64_t *m);

/* Leak sweep on the device: writes the live allocations
 * (ascending base) to d_out (at most cap records) and their total number to
 * *d_count (a device u64).  Asynchronous on stream. */
cg_status cg_leak_sweep(cg_ctx *ctx, cg_alloc_record *d_out, uint64_t cap, uint64_t *d_count, void *stream);

/* Synchronous leak report (abstract P:12): runs the device sweep
 * and copies min(cap, k) records to h_out; *n_out = k.  Errors:
 * CG_ERR_INVALID_VALUE if n_out is NULL (h_out may be NULL when cap == 0). */
cg_status cg_leak_report(cg_ctx *ctx, cg_alloc_record *h_out, uint64_t cap, uint64_t *n_out);

/* Epoch planner (host): splits n descriptors (host array, in call order) into
 * consecutive batches such that no HtoD's host range overlaps the host range
 * of an earlier DtoH in the same batch (the batch contract above; reading
 * R-20, conservative on 2D bounding intervals).  Writes the end index of every
 * batch to h_cuts (at most n entries; the last is n) and their number to
 * *n_cuts.  Errors: CG_ERR_INVALID_VALUE on NULL. */
cg_status cg_plan_batches(const cg_copy_desc *h_descs, uint64_t n, uint64_t *h_cuts, uint64_t *n_cuts);

/* Batches for cg_check_apply (fused), in place: like cg_plan_batches, but an
 * HtoD that reads bytes an earlier DtoH of the batch writes does not end the
 * batch: it gets CG_CHECK_AFTER (checked after the batch's applies) when its
 * host range is at most 1 MiB; a DtoH that writes bytes of such an HtoD gets
 * CG_APPLY_LAST (applied after the CG_CHECK_AFTER checks, so every one of them
 * sees exactly the applies of the DtoH copies before it), and an HtoD that
 * reads bytes of a CG_APPLY_LAST DtoH ends the batch; every other DtoH whose
 * range an HtoD of its batch reads gets CG_APPLY_AFTER.  The result of cg_check_apply over each batch
 * equals the sequential replay.  Writes the end of every batch to h_cuts (the
 * last is n), their number to *n_cuts.  Errors: CG_ERR_INVALID_VALUE on NULL. */
cg_status cg_plan_batches_fused(cg_copy_desc *h_descs, uint64_t n, uint64_t *h_cuts, uint64_t *n_cuts);

/* As cg_plan_batches, for device V-bit tracking (NEXT-1): a batch is cut
 * before any copy whose reads (HtoD host source, DtoD/DtoH device source)
 * overlap an earlier write of the batch (DtoH host target, HtoD/DtoD device
 * target) or whose writes overlap an earlier read or write -- so every copy's
 * propagation in a batch can run in parallel (a DtoD overlapping itself is
 * fine).  Conservative on 2D bounding intervals. */
cg_status cg_plan_batches_propagate(const cg_copy_desc *h_descs, uint64_t n, uint64_t *h_cuts, uint64_t *n_cuts);

/* Diagnostic text (SPEC format_text S:454-462): renders
 * one line pair per set flag of *v, in flag order, for a copy of the given
 * kind, into buf (NUL-terminated, truncated to cap).  The TooSmall text is the
 * paper's Listing 5 verbatim: "Error: Allocated device memory too
 * small for device->host copy.\nExpected 8000000 allocated bytes but only
 * found 4000000."; the other messages follow SPEC's "Error: <message>." /
 * "Warning: <message>." template.  Returns the number of characters needed
 * (excluding the NUL), like snprintf. */
uint64_t cg_format_verdict(const cg_verdict *v, uint32_t kind, char *buf, uint64_t cap);

/* "Warning: Device memory leak of <size> bytes."; as above. */
uint64_t cg_format_leak(const cg_alloc_record *r, char *buf, uint64_t cap);

/* NEXT-4 ERROR SUMMARY (Listing 4 P:219 for the shape):
 * counts the diagnostics of n verdicts on the device -- one per set flag;
 * HOST_UNDEFINED (unless undef_is_error) and CONCURRENT are Warnings,
 * every other flag an Error.  d_counts: device array of 2 uint64
 * {errors, warnings}, overwritten.  Stateless, asynchronous on stream.
 * Registry errors (InvalidFree) and leaks are counted by the caller from the
 * call statuses and cg_leak_report.  Errors: CG_ERR_INVALID_VALUE, CG_ERR_CUDA. */
cg_status cg_summarize(const cg_verdict *d_verdicts, uint64_t n, uint32_t undef_is_error, uint64_t *d_counts,
                       void *stream);

/* "ERROR SUMMARY: <e> errors, <w> warnings (<s> suppressed)\n";
 * returns the length, writes at most cap-1 bytes + NUL. */
uint64_t cg_format_summary(uint64_t errors, uint64_t warnings, uint64_t suppressed, char *buf, uint64_t cap);

/* Number of kernels this context has launched so far (for bench accounting). */
uint64_t cg_kernel_launches(const cg_ctx *ctx);

/* Per-stage device timing (bench instrumentation).  After cg_profile_begin,
 * every asynchronous call brackets each of its stages with CUDA events on the
 * call's stream.  cg_profile_end synchronises, writes the accumulated
 * milliseconds and launch counts of the stages to ms[CG_STAGE_COUNT] and
 * launches[CG_STAGE_COUNT] (either may be NULL) and stops recording. */
enum {
  CG_STAGE_CHECK_PREP = 0,   /* a1+a3: k_check_prep                      */
  CG_STAGE_CHECK_PLAN = 1,   /* a2: prefix sum + chunk plan              */
  CG_STAGE_CHECK_SCAN = 2,   /* a4+a5: k_check_scan (the shadow scan)    */
  CG_STAGE_CHECK_FINAL = 3,  /* a5: k_finalize_split                     */
  CG_STAGE_APPLY_PREP = 4,   /* a6: k_apply_prep                         */
  CG_STAGE_APPLY_PLAN = 5,   /* a6: prefix sum + chunk plan              */
  CG_STAGE_APPLY = 6,        /* a6: k_apply (the DtoH shadow update)     */
  CG_STAGE_LEAK = 7,         /* a8: leak sweep                           */
  CG_STAGE_COUNT = 8
};
cg_status cg_profile_begin(cg_ctx *ctx);
cg_status cg_profile_end(cg_ctx *ctx, double *ms, uint64_t *launches);

#ifdef __cplusplus
}
#endif
#endif /* CG_H_ */
