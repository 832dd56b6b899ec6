/*
 * cg_oracle.c -- plain, slow, sequential CPU oracle for the batched Cudagrind
 * transfer checker.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_1310_0901_b200/csrc) and never includes it; every constant below is
 * restated from the paper / SURVEY.md, not imported.
 *
 * What it computes (§3):
 * events are replayed one at a time, in trace order, exactly as a wrapper
 * around each driver call would see them:
 *   O1 host_mark        -- S:45-62
 *   O2 host_set_vbits   -- S:79
 *   O3 register         -- Fig. 2 caption P:88
 *   O4 free             -- S:148-156
 *   O5 copy check+apply -- P:80-82, S:157-165, S:192, S:63-80, S:222-248,
 *                          S:278-281; readings R-1..R-16
 *   O6 leak report      -- P:12 (abstract)
 *   O7 concurrency      -- NEXT-2: P:83, S:216-219, S:258-266, S:285;
 *                          DESIGN.md readings R-31..R-35
 *
 * State (SURVEY §8(c) "State"):
 *   host window [h0, h0+s);  A: one addressability bit per host byte, bit
 *   (x-h0)&7 of byte (x-h0)>>3, 1 = addressable (R-2);  V: one byte of
 *   validity bits per host byte, bit set = bit undefined (R-1);  fresh state
 *   A=0 (unaddressable), V=0xFF.  The device allocation list is an
 *   unsorted array searched linearly -- the paper's Fig. 2 "list".
 *
 * Parity pins: see tests/test_oracle_*.py (paper worked example P:137-146 ->
 * P:234-235, SPEC examples, closed forms, invariants, numpy brute force).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_NONE UINT64_MAX

/* event ops (tracegen/__init__.py) */
enum { OR_MARK = 1, OR_SETV = 2, OR_REG = 3, OR_FREE = 4, OR_COPY = 5, OR_REGA = 6, OR_FREEA = 7, OR_SYNC = 8 };
/* copy kinds: host->device, device->host, device->device, and the
 * device-array transfers HtoA / AtoH (NEXT-3: Fig. 2 caption P:88) */
enum { OR_HTOD = 1, OR_DTOH = 2, OR_DTOD = 3, OR_HTOA = 4, OR_ATOH = 5 };
/* host mark states (host_alloc / host_write / host_free) */
enum { OR_NOACCESS = 0, OR_UNDEFINED = 1, OR_DEFINED = 2 };

/* diagnostic flags in SPEC's emission order (reading R-14) */
#define F_DST_NOT_ALLOCATED   (1u << 0)
#define F_DST_TOO_SMALL       (1u << 1)
#define F_SRC_NOT_ALLOCATED   (1u << 2)
#define F_SRC_TOO_SMALL       (1u << 3)   /* P:82, Listing 5 */
#define F_HOST_UNADDRESSABLE  (1u << 4)   /* P:80 (host side, via Memcheck A-bits) */
#define F_HOST_UNDEFINED      (1u << 5)   /* P:81 (Warning, footnote) */
#define F_BAD_PITCH           (1u << 6)   /* R-12 */
#define F_INVALID_RANGE       (1u << 7)
#define F_BAD_KIND            (1u << 8)   /* R-16 */
#define F_CONCURRENT          (1u << 9)   /* P:83, S:260 ConcurrentHazard (Warning) */

typedef struct {
    uint32_t op, kind;
    uint64_t seq, width, height;
    uint64_t dst, dst_x, dst_y, dst_pitch;
    uint64_t src, src_x, src_y, src_pitch;
} or_event;                                    /* 96 bytes */

typedef struct {
    uint64_t first_unaddr, first_undef, undef_count;
    uint64_t dst_expected, dst_found, src_expected, src_found;
    uint32_t flags, status;
} or_verdict;                                  /* 64 bytes */

typedef struct { uint64_t base, size, seq; } or_alloc;

/* NEXT-2 AccessStamp of one recorded access: the byte range it
 * touched in one address space, its thread, seq and direction */
typedef struct { uint64_t lo, hi, seq; uint32_t thread, is_write; } or_stamp;
typedef struct { uint64_t seq; uint32_t thread; } or_sync_ev;

typedef struct {
    uint64_t h0, s;
    uint8_t *A;            /* s/8 bytes */
    uint8_t *V;            /* s bytes   */
    or_alloc *live;        /* unsorted list of live allocations (Fig. 2) */
    uint8_t **dv;          /* NEXT-1: device V-bytes of live[i] (track mode), else NULL */
    uint64_t n_live, cap_live;
    int track;             /* NEXT-1: propagate V-bits through copies (SPEC copy_vbits) */
    or_alloc *arr;         /* NEXT-3: unsorted list of live device arrays {handle, total_bytes, seq} */
    uint8_t **av;          /* NEXT-3 x NEXT-1: V-bytes of arr[i] (track mode), else NULL */
    uint64_t n_arr, cap_arr;
    uint64_t last_reg_seq;
    int undef_is_error;    /* CLI flag promotes HostUndefined */
    int conc;              /* NEXT-2: run check_concurrent on every copy */
    or_stamp *stamps[2];   /* NEXT-2: every recorded access, in order; [0] host, [1] device space */
    uint64_t n_stamps[2], cap_stamps[2];
    or_sync_ev *syncs;     /* NEXT-2: ctx_synchronize events */
    uint64_t n_syncs, cap_syncs;
} or_state;

/* ---------------------------------------------------------------- state */
or_state *or_create(uint64_t h0, uint64_t s, int undef_is_error) {
    or_state *st = (or_state *)calloc(1, sizeof(or_state));
    if (!st) return NULL;
    st->h0 = h0; st->s = s; st->undef_is_error = undef_is_error;
    st->A = (uint8_t *)calloc(s / 8 + 1, 1);          /* A = 0: unaddressable */
    st->V = (uint8_t *)malloc(s ? s : 1);
    if (!st->A || !st->V) { free(st->A); free(st->V); free(st); return NULL; }
    memset(st->V, 0xFF, s);                            /* V = all undefined  */
    st->cap_live = 16;
    st->live = (or_alloc *)malloc(st->cap_live * sizeof(or_alloc));
    st->dv = (uint8_t **)calloc(st->cap_live, sizeof(uint8_t *));
    return st;
}

/* NEXT-1: device
 * allocations carry V-bits too (fresh: undefined); an error-free HtoD copies
 * host V-bits to the device, DtoD device to device (as if staged through a
 * scratch buffer), DtoH device to host -- instead of R-5's "DtoH marks
 * the host range defined".  Must be set before the first registration. */
void or_track_device(or_state *st, int on) { st->track = on; }

void or_destroy(or_state *st) {
    if (!st) return;
    for (uint64_t i = 0; i < st->n_live; i++) free(st->dv[i]);
    for (uint64_t i = 0; i < st->n_arr; i++) free(st->av[i]);
    free(st->A); free(st->V); free(st->live); free(st->dv); free(st->arr); free(st->av);
    free(st->stamps[0]); free(st->stamps[1]); free(st->syncs); free(st);
}

uint8_t *or_A(or_state *st) { return st->A; }
uint8_t *or_V(or_state *st) { return st->V; }

static int in_window(const or_state *st, uint64_t x) {
    return x >= st->h0 && x - st->h0 < st->s;
}

static int a_get(const or_state *st, uint64_t x) {        /* x inside window */
    uint64_t i = x - st->h0;
    return (st->A[i >> 3] >> (i & 7)) & 1;
}

static void a_put(or_state *st, uint64_t x, int bit) {
    uint64_t i = x - st->h0;
    if (bit) st->A[i >> 3] |= (uint8_t)(1u << (i & 7));
    else     st->A[i >> 3] &= (uint8_t)~(1u << (i & 7));
}

/* addr(x) of SURVEY §8(a)-a4: inside the window and A-bit set (R-15) */
static int addressable(const or_state *st, uint64_t x) {
    return in_window(st, x) && a_get(st, x);
}

/* ------------------------------------------------------- O1 host_mark */
/* returns 0 on success, 1 (INVALID_VALUE) if the range leaves the window */
int or_mark(or_state *st, uint64_t addr, uint64_t len, uint32_t state) {
    if (state > OR_DEFINED) return 1;
    if (len == 0) return 0;
    if (addr < st->h0 || len > st->s || addr - st->h0 > st->s - len) return 1;
    for (uint64_t k = 0; k < len; k++) {
        uint64_t x = addr + k;
        a_put(st, x, state != OR_NOACCESS);
        st->V[x - st->h0] = (state == OR_DEFINED) ? 0x00 : 0xFF;
    }
    return 0;
}

/* --------------------------------------------------- O2 host_set_vbits */
int or_set_vbits(or_state *st, uint64_t addr, uint64_t len, const uint8_t *vb) {
    if (len == 0) return 0;
    if (addr < st->h0 || len > st->s || addr - st->h0 > st->s - len) return 1;
    for (uint64_t k = 0; k < len; k++)                 /* defined => addressable */
        if (!a_get(st, addr + k)) return 1;
    for (uint64_t k = 0; k < len; k++) st->V[addr + k - st->h0] = vb[k];
    return 0;
}

/* -------------------------------------------------------- O3 register */
int or_register(or_state *st, uint64_t base, uint64_t size, uint64_t seq) {
    if (seq <= st->last_reg_seq) return 1;               /* seq strictly increasing */
    if (size == 0 || base == 0) return 1;
    if (size > UINT64_MAX - base) return 1;               /* end must fit in 64 bits */
    for (uint64_t i = 0; i < st->n_live; i++) {            /* S:143 OverlapWithLive */
        const or_alloc *e = &st->live[i];
        if (base < e->base + e->size && e->base < base + size) return 1;
    }
    if (st->n_live == st->cap_live) {
        st->cap_live *= 2;
        st->live = (or_alloc *)realloc(st->live, st->cap_live * sizeof(or_alloc));
        st->dv = (uint8_t **)realloc(st->dv, st->cap_live * sizeof(uint8_t *));
    }
    st->live[st->n_live].base = base;
    st->live[st->n_live].size = size;
    st->live[st->n_live].seq = seq;
    st->dv[st->n_live] = NULL;
    if (st->track) {                                      /* fresh device memory is undefined */
        st->dv[st->n_live] = (uint8_t *)malloc(size);
        memset(st->dv[st->n_live], 0xFF, size);
    }
    st->n_live++;
    st->last_reg_seq = seq;
    return 0;
}

/* ---------------------------------------------- NEXT-3 device arrays */
/* SPEC ArrayDescriptor: total_bytes = width * max(height,1) *
 * max(depth,1) * format_bytes * channels; formats u8,u16,u32,s8,s16,s32,f16,
 * f32 (codes 0..7) are 1,2,4,1,2,4,2,4 bytes; channels in {1,2,4}; width >= 1.
 * Returns 0 for an invalid descriptor. */
uint64_t or_array_bytes(uint64_t width, uint64_t height, uint64_t depth, uint64_t format, uint64_t channels) {
    static const uint64_t fb[8] = {1, 2, 4, 1, 2, 4, 2, 4};
    if (width == 0 || format > 7 || (channels != 1 && channels != 2 && channels != 4)) return 0;
    unsigned __int128 t = (unsigned __int128)width * (height ? height : 1);
    t *= (depth ? depth : 1);
    t *= fb[format] * channels;
    return t > (unsigned __int128)UINT64_MAX ? 0 : (uint64_t)t;
}

/* register_array: DuplicateHandle (a live array has this handle),
 * zero-extent descriptor or non-increasing seq -> 1, no mutation */
int or_register_array(or_state *st, uint64_t handle, uint64_t total, uint64_t seq) {
    if (seq <= st->last_reg_seq || total == 0) return 1;
    for (uint64_t i = 0; i < st->n_arr; i++)
        if (st->arr[i].base == handle) return 1;
    if (st->n_arr == st->cap_arr) {
        st->cap_arr = st->cap_arr ? 2 * st->cap_arr : 16;
        st->arr = (or_alloc *)realloc(st->arr, st->cap_arr * sizeof(or_alloc));
        st->av = (uint8_t **)realloc(st->av, st->cap_arr * sizeof(uint8_t *));
    }
    st->arr[st->n_arr].base = handle;
    st->arr[st->n_arr].size = total;
    st->arr[st->n_arr].seq = seq;
    st->av[st->n_arr] = NULL;
    if (st->track) {                       /* S:252 per-array shadow; fresh = undefined */
        st->av[st->n_arr] = (uint8_t *)malloc(total);
        memset(st->av[st->n_arr], 0xFF, total);
    }
    st->n_arr++;
    st->last_reg_seq = seq;
    return 0;
}

/* unregister_array: UnknownHandle -> 1, no mutation */
int or_free_array(or_state *st, uint64_t handle, uint64_t seq) {
    if (seq <= st->last_reg_seq) return 1;
    for (uint64_t i = 0; i < st->n_arr; i++) {
        if (st->arr[i].base == handle) {
            free(st->av[i]);
            st->arr[i] = st->arr[st->n_arr - 1];
            st->av[i] = st->av[st->n_arr - 1];
            st->n_arr--;
            st->last_reg_seq = seq;
            return 0;
        }
    }
    return 1;
}

uint64_t or_array_leaks(or_state *st, or_alloc *out, uint64_t cap) {
    for (uint64_t i = 0; i < st->n_arr && i < cap; i++) out[i] = st->arr[i];
    return st->n_arr;
}

/* ------------------------------------------------------------ O4 free */
int or_free(or_state *st, uint64_t ptr, uint64_t seq) {
    if (seq <= st->last_reg_seq) return 1;
    for (uint64_t i = 0; i < st->n_live; i++) {
        if (st->live[i].base == ptr) {                    /* S:150 base match only */
            free(st->dv[i]);
            st->live[i] = st->live[st->n_live - 1];
            st->dv[i] = st->dv[st->n_live - 1];
            st->n_live--;
            st->last_reg_seq = seq;
            return 0;
        }
    }
    return 1;                                             /* InvalidFree, no mutation */
}

/* ----------------------------------------------------------- O5 copy */
/* start = base + Y*pitch + X  (CUDA_MEMCPY2D start address, R-11);
 * span  = 0 if W==0 or H==0, else (H-1)*pitch + W;
 * the side is a valid range iff start+span fits in 64 bits (R-10). */
static int side_range(uint64_t base, uint64_t x, uint64_t y, uint64_t pitch,
                      uint64_t w, uint64_t h, uint64_t *start, uint64_t *span) {
    unsigned __int128 st = (unsigned __int128)base + (unsigned __int128)y * pitch + x;
    unsigned __int128 sp = (w == 0 || h == 0) ? 0
                         : (unsigned __int128)(h - 1) * pitch + w;
    if (st + sp > (unsigned __int128)UINT64_MAX) return 0;
    *start = (uint64_t)st;
    *span = (uint64_t)sp;
    return 1;
}

/* coverage anchored on the allocation containing start */
static void device_side(const or_state *st, uint64_t start, uint64_t span,
                        uint32_t f_na, uint32_t f_small, uint32_t *flags,
                        uint64_t *expected, uint64_t *found) {
    for (uint64_t i = 0; i < st->n_live; i++) {
        const or_alloc *e = &st->live[i];
        if (e->base <= start && start < e->base + e->size) {
            uint64_t avail = e->base + e->size - start;
            if (avail < span) { *flags |= f_small; *expected = span; *found = avail; }
            return;
        }
    }
    *flags |= f_na;
}

/* device V-bytes at device address x (inside a live allocation) */
static uint8_t *device_vbits(const or_state *st, uint64_t x) {
    for (uint64_t i = 0; i < st->n_live; i++) {
        const or_alloc *e = &st->live[i];
        if (e->base <= x && x < e->base + e->size) return st->dv[i] + (x - e->base);
    }
    return NULL;
}

/* device V-bytes of [x, x+len) into out (test view; 1 if not inside one live allocation) */
int or_device_vbits(const or_state *st, uint64_t x, uint64_t len, uint8_t *out) {
    for (uint64_t i = 0; i < st->n_live; i++) {
        const or_alloc *e = &st->live[i];
        if (e->base <= x && x < e->base + e->size) {
            if (len > e->base + e->size - x || !st->dv[i]) return 1;
            memcpy(out, st->dv[i] + (x - e->base), len);
            return 0;
        }
    }
    return 1;
}

/* (iii) the host-side scan of one copy: every logical byte o = r*W + c
 * (row-major, R-11) at address x = start + r*pitch + c, in increasing o.
 * first_unaddr = the first o whose byte is not addressable (outside the window
 * counts as unaddressable, R-15); if `defined` is asked (HtoD), first_undef /
 * undef_count over the addressable bytes with a nonzero V-byte (R-1, R-3).
 * The loop visits o in increasing order, so once first_unaddr is set a byte
 * outside the window can change nothing (it is not counted as undefined and
 * cannot lower first_unaddr): such bytes are skipped -- the rest of a row past
 * the window end, the part of a row before the window start, whole rows before
 * the window, and (pitch > 0, so rows only move up) every row from the first
 * one that starts at or past the window end.  This keeps copies of any size
 * (R-10 allows up to 2^64-1 logical bytes) bounded by the window. */
static void host_scan(const or_state *st, uint64_t start, uint64_t pitch, uint64_t W, uint64_t H,
                      int defined, or_verdict *v) {
    const uint64_t wend = st->h0 + st->s;
    for (uint64_t r = 0; r < H && W; r++) {
        const uint64_t xr = start + r * pitch;
        if (v->first_unaddr != OR_NONE) {
            if (pitch > 0 && xr >= wend) break;
            if (pitch > 0 && xr + W <= st->h0) {       /* rows r .. r+k end before the window */
                r += (st->h0 - xr - W) / pitch;
                continue;
            }
        }
        for (uint64_t c = 0; c < W; c++) {
            const uint64_t x = xr + c, o = r * W + c;
            if (!in_window(st, x) && v->first_unaddr != OR_NONE) {
                if (x >= wend) break;                   /* the rest of the row is further out */
                c = st->h0 - xr - 1;                    /* continue at the window start */
                continue;
            }
            if (!addressable(st, x)) {
                if (v->first_unaddr == OR_NONE) v->first_unaddr = o;
            } else if (defined && st->V[x - st->h0] != 0) {
                if (v->first_undef == OR_NONE) v->first_undef = o;
                v->undef_count++;
            }
        }
    }
}

/* array V-bytes [off, off+len) of the live array `handle` into out (test view;
 * 1 if there is none, it has no V-bytes or the range leaves it) */
int or_array_vbits(const or_state *st, uint64_t handle, uint64_t off, uint64_t len, uint8_t *out) {
    for (uint64_t i = 0; i < st->n_arr; i++) {
        if (st->arr[i].base != handle) continue;
        if (!st->av[i] || off > st->arr[i].size || len > st->arr[i].size - off) return 1;
        memcpy(out, st->av[i] + off, len);
        return 0;
    }
    return 1;
}

/* NEXT-3 check_array_transfer: the array side is (handle, byte
 * offset) = (dst, dst_x) for HtoA and (src, src_x) for AtoH; the array holds
 * the W*H logical bytes contiguously from the offset.  Unknown handle ->
 * *_NOT_ALLOCATED; offset + W*H > total_bytes -> *_TOO_SMALL with expected =
 * W*H and found = total_bytes - offset (0 past the end).  The host side is
 * checked as for HtoD / DtoH (pitch rule on the host side only). */
static void check_array_copy(const or_state *st, const or_event *ev, or_verdict *v) {
    const int htoa = ev->kind == OR_HTOA;
    const uint64_t W = ev->width, H = ev->height;
    const uint64_t handle = htoa ? ev->dst : ev->src, off = htoa ? ev->dst_x : ev->src_x;
    const uint64_t hb = htoa ? ev->src : ev->dst, hx = htoa ? ev->src_x : ev->dst_x;
    const uint64_t hy = htoa ? ev->src_y : ev->dst_y, hp = htoa ? ev->src_pitch : ev->dst_pitch;
    if ((unsigned __int128)hp < (unsigned __int128)W + hx) v->flags |= F_BAD_PITCH;
    uint64_t hs = 0, hspan = 0;
    const int hok = side_range(hb, hx, hy, hp, W, H, &hs, &hspan);
    const unsigned __int128 nb = (unsigned __int128)W * H;
    const int nbytes_ok = nb <= (unsigned __int128)UINT64_MAX;       /* R-10: logical bytes fit 64 bits */
    const int aok = (unsigned __int128)off + nb <= (unsigned __int128)UINT64_MAX;
    if (!hok || !nbytes_ok || !aok) v->flags |= F_INVALID_RANGE;
    if (aok && nbytes_ok) {
        int found = 0;
        for (uint64_t i = 0; i < st->n_arr; i++) {
            if (st->arr[i].base != handle) continue;
            found = 1;
            const uint64_t total = st->arr[i].size;
            if (off + (uint64_t)nb > total) {
                v->flags |= htoa ? F_DST_TOO_SMALL : F_SRC_TOO_SMALL;
                if (htoa) { v->dst_expected = (uint64_t)nb; v->dst_found = off < total ? total - off : 0; }
                else      { v->src_expected = (uint64_t)nb; v->src_found = off < total ? total - off : 0; }
            }
        }
        if (!found) v->flags |= htoa ? F_DST_NOT_ALLOCATED : F_SRC_NOT_ALLOCATED;
    }
    if (hok && nbytes_ok) host_scan(st, hs, hp, W, H, htoa, v);
    if (v->first_unaddr != OR_NONE) v->flags |= F_HOST_UNADDRESSABLE;
    if (v->undef_count > 0 && v->first_unaddr == OR_NONE) v->flags |= F_HOST_UNDEFINED;
    const uint32_t errors = v->flags & ~(st->undef_is_error ? 0u : F_HOST_UNDEFINED);
    v->status = errors ? 1u : 0u;
}

/* O5 (i)-(iv): the checks of one copy; reads the state, changes nothing */
static void check_only(const or_state *st, const or_event *ev, or_verdict *v) {
    v->first_unaddr = OR_NONE; v->first_undef = OR_NONE; v->undef_count = 0;
    v->dst_expected = v->dst_found = v->src_expected = v->src_found = 0;
    v->flags = 0; v->status = 0;
    uint32_t kind = ev->kind;
    uint64_t W = ev->width, H = ev->height;
    if (kind < OR_HTOD || kind > OR_ATOH) {
        v->flags = F_BAD_KIND; v->status = 1; return;
    }
    if (kind == OR_HTOA || kind == OR_ATOH) { check_array_copy(st, ev, v); return; }
    /* (i) validation: pitch rule (pitch >= WidthInBytes + XInBytes) and ranges */
    if ((unsigned __int128)ev->dst_pitch < (unsigned __int128)W + ev->dst_x ||
        (unsigned __int128)ev->src_pitch < (unsigned __int128)W + ev->src_x)
        v->flags |= F_BAD_PITCH;
    uint64_t ds = 0, dspan = 0, ss = 0, sspan = 0;
    int dok = side_range(ev->dst, ev->dst_x, ev->dst_y, ev->dst_pitch, W, H, &ds, &dspan);
    int sok = side_range(ev->src, ev->src_x, ev->src_y, ev->src_pitch, W, H, &ss, &sspan);
    /* R-10 ("InvalidRange on overflow"): a side whose
     * start + span, or a copy whose logical byte count W*H (the offsets
     * reported below), does not fit in 64 bits is an invalid range */
    int nbytes_ok = ((unsigned __int128)W * H <= (unsigned __int128)UINT64_MAX);
    if (!dok || !sok || !nbytes_ok) v->flags |= F_INVALID_RANGE;

    /* (ii) device endpoints, dst then src */
    if (kind == OR_HTOD || kind == OR_DTOD)
        if (dok) device_side(st, ds, dspan, F_DST_NOT_ALLOCATED, F_DST_TOO_SMALL,
                             &v->flags, &v->dst_expected, &v->dst_found);
    if (kind == OR_DTOH || kind == OR_DTOD)
        if (sok) device_side(st, ss, sspan, F_SRC_NOT_ALLOCATED, F_SRC_TOO_SMALL,
                             &v->flags, &v->src_expected, &v->src_found);

    /* (iii) host side: HtoD reads src, DtoH writes dst.  Row-major logical
     * offsets o = r*W + c at address x = start + r*pitch + c (R-11). */
    if ((kind == OR_HTOD && sok && nbytes_ok) || (kind == OR_DTOH && dok && nbytes_ok)) {
        uint64_t hstart = (kind == OR_HTOD) ? ss : ds;
        uint64_t hpitch = (kind == OR_HTOD) ? ev->src_pitch : ev->dst_pitch;
        host_scan(st, hstart, hpitch, W, H, kind == OR_HTOD, v);
    }
    /* (iv) flags and status (R-4, R-8) */
    if (v->first_unaddr != OR_NONE) v->flags |= F_HOST_UNADDRESSABLE;
    if (v->undef_count > 0 && v->first_unaddr == OR_NONE) v->flags |= F_HOST_UNDEFINED;
    uint32_t errors = v->flags & ~(st->undef_is_error ? 0u : F_HOST_UNDEFINED);
    v->status = errors ? 1u : 0u;
}

/* (v) without device V-bits: the host bytes an error-free DtoH / AtoH wrote
 * become defined (R-5, R-7) -- those of them inside [lo, hi) (the whole
 * window in the sequential replay; one thread's slice in the parallel one) */
static void apply_defined(or_state *st, const or_event *ev, uint64_t lo, uint64_t hi) {
    const uint64_t W = ev->width, H = ev->height;
    const uint64_t hs = ev->dst + ev->dst_y * ev->dst_pitch + ev->dst_x;   /* fits: no Error */
    for (uint64_t r = 0; r < H && W; r++) {
        const uint64_t xr = hs + r * ev->dst_pitch;
        const uint64_t c0 = lo > xr ? lo - xr : 0;                 /* the row's columns inside [lo, hi) */
        const uint64_t c1 = hi > xr ? (hi - xr < W ? hi - xr : W) : 0;
        for (uint64_t c = c0; c < c1; c++) st->V[xr + c - st->h0] = 0x00;
    }
}

/* NEXT-3 x NEXT-1 ("array V-bits tracked in a per-array shadow", R-30):
 * the V-bytes of the live array with this handle, at the byte offset */
static uint8_t *array_vbits(const or_state *st, uint64_t handle, uint64_t off) {
    for (uint64_t i = 0; i < st->n_arr; i++)
        if (st->arr[i].base == handle) return st->av[i] + off;
    return NULL;
}

/* (v') NEXT-1: with device V-bits, an error-free copy moves V-bits (SPEC
 * copy_vbits S:81-89): host -> device, device -> device (staged: memmove,
 * S:84), device -> host, and with arrays host -> array / array -> host (R-30) */
static void move_vbits(or_state *st, const or_event *ev) {
    const uint32_t kind = ev->kind;
    const uint64_t W = ev->width, H = ev->height;
    if (!W || !H) return;
    const uint64_t ds = ev->dst + ev->dst_y * ev->dst_pitch + ev->dst_x;
    const uint64_t ss = ev->src + ev->src_y * ev->src_pitch + ev->src_x;
    uint8_t *dd = NULL, *sd = NULL;   /* device / array V of dst / src at their start */
    if (kind == OR_HTOD || kind == OR_DTOD) dd = device_vbits(st, ds);
    if (kind == OR_DTOH || kind == OR_DTOD) sd = device_vbits(st, ss);
    if (kind == OR_HTOA) dd = array_vbits(st, ev->dst, ev->dst_x);
    if (kind == OR_ATOH) sd = array_vbits(st, ev->src, ev->src_x);
    const int host_src = kind == OR_HTOD || kind == OR_HTOA, host_dst = kind == OR_DTOH || kind == OR_ATOH;
    /* an array side is W*H contiguous bytes from its offset (R-29): pitch W, no y */
    const uint64_t sp = kind == OR_ATOH ? W : ev->src_pitch, dp = kind == OR_HTOA ? W : ev->dst_pitch;
    const uint64_t hs = kind == OR_HTOA ? ev->src + ev->src_y * ev->src_pitch + ev->src_x : ss;
    const uint64_t hd = kind == OR_ATOH ? ev->dst + ev->dst_y * ev->dst_pitch + ev->dst_x : ds;
    uint8_t *tmp = (uint8_t *)malloc(W * H);           /* logical order, staged */
    for (uint64_t r = 0; r < H; r++)
        for (uint64_t c = 0; c < W; c++)
            tmp[r * W + c] = host_src ? st->V[hs + r * sp + c - st->h0] : sd[r * sp + c];
    for (uint64_t r = 0; r < H; r++)
        for (uint64_t c = 0; c < W; c++) {
            if (host_dst) st->V[hd + r * dp + c - st->h0] = tmp[r * W + c];
            else dd[r * dp + c] = tmp[r * W + c];
        }
    free(tmp);
}

/* O5: check one copy, then (no Error) its effect on the shadow */
void or_check_copy(or_state *st, const or_event *ev, or_verdict *v) {
    check_only(st, ev, v);
    if (v->status != 0) return;                              /* R-7: the copy fails, nothing moves */
    if (st->track) move_vbits(st, ev);
    else if (ev->kind == OR_DTOH || ev->kind == OR_ATOH) apply_defined(st, ev, st->h0, st->h0 + st->s);
}

/* ------------------------------------------------------ O7 concurrency */
/* NEXT-2 ("certain concurrent accesses when several
 * threads are used"; SPEC check_concurrent S:258-266 with the rule of S:285):
 * a copy's access is a ConcurrentHazard (Warning) iff the most recent earlier
 * recorded access overlapping it was made by a different thread, that thread
 * has not synchronised since (ctx_synchronize), and one of the two
 * writes.  Readings: R-31 one context per thread, so a sync by
 * thread t marks exactly t's stamps; R-32 every side of a copy is an access
 * (host read of HtoD/HtoA, device write of HtoD, device read of DtoH/DtoD,
 * host write of DtoH/AtoH, device write of DtoD) -- array sides are not
 * stamped; R-33 the access range is the side's folded [start, start+span)
 * (2D: the bounding range), empty or overflowing sides make no access;
 * R-34 every copy with a valid kind is checked, only copies without an Error
 * (the ones the driver performs) record stamps, after their check; two
 * stamps of the same copy count as one access that writes if either writes. */
void or_track_concurrency(or_state *st, int on) { st->conc = on; }

void or_sync(or_state *st, uint32_t thread, uint64_t seq) {
    if (st->n_syncs == st->cap_syncs) {
        st->cap_syncs = st->cap_syncs ? 2 * st->cap_syncs : 16;
        st->syncs = (or_sync_ev *)realloc(st->syncs, st->cap_syncs * sizeof(or_sync_ev));
    }
    st->syncs[st->n_syncs].seq = seq;
    st->syncs[st->n_syncs].thread = thread;
    st->n_syncs++;
}

/* synced_after -- thread t synchronised after its stamp at seq a and before seq b */
static int synced_between(const or_state *st, uint32_t t, uint64_t a, uint64_t b) {
    for (uint64_t i = 0; i < st->n_syncs; i++)
        if (st->syncs[i].thread == t && st->syncs[i].seq > a && st->syncs[i].seq < b) return 1;
    return 0;
}

/* S:260 for one new access against every stamp recorded so far */
static int conc_hazard(const or_state *st, int space, uint64_t lo, uint64_t hi, int is_write,
                       uint32_t thread, uint64_t seq) {
    int found = 0, prev_write = 0;
    uint64_t best = 0;
    uint32_t prev_thread = 0;
    for (uint64_t i = 0; i < st->n_stamps[space]; i++) {
        const or_stamp *p = &st->stamps[space][i];
        if (p->lo >= hi || lo >= p->hi || p->seq >= seq) continue;   /* no overlap / not earlier */
        if (!found || p->seq > best) {
            found = 1; best = p->seq; prev_thread = p->thread; prev_write = (int)p->is_write;
        } else if (p->seq == best) {
            prev_write |= (int)p->is_write;                          /* R-34 */
        }
    }
    if (!found) return 0;
    return prev_thread != thread && !synced_between(st, prev_thread, best, seq) && (prev_write || is_write);
}

static void add_stamp(or_state *st, int space, uint64_t lo, uint64_t hi, int is_write, uint32_t thread,
                      uint64_t seq) {
    if (st->n_stamps[space] == st->cap_stamps[space]) {
        st->cap_stamps[space] = st->cap_stamps[space] ? 2 * st->cap_stamps[space] : 64;
        st->stamps[space] = (or_stamp *)realloc(st->stamps[space], st->cap_stamps[space] * sizeof(or_stamp));
    }
    or_stamp *p = &st->stamps[space][st->n_stamps[space]++];
    p->lo = lo; p->hi = hi; p->seq = seq; p->thread = thread; p->is_write = (uint32_t)is_write;
}

/* R-32: the accesses of one copy: (space, side is dst, is_write) */
static int copy_accesses(uint32_t kind, int space[2], int dst[2], int wr[2]) {
    switch (kind) {
    case OR_HTOD: space[0] = 0; dst[0] = 0; wr[0] = 0; space[1] = 1; dst[1] = 1; wr[1] = 1; return 2;
    case OR_DTOH: space[0] = 1; dst[0] = 0; wr[0] = 0; space[1] = 0; dst[1] = 1; wr[1] = 1; return 2;
    case OR_DTOD: space[0] = 1; dst[0] = 0; wr[0] = 0; space[1] = 1; dst[1] = 1; wr[1] = 1; return 2;
    case OR_HTOA: space[0] = 0; dst[0] = 0; wr[0] = 0; return 1;
    case OR_ATOH: space[0] = 0; dst[0] = 1; wr[0] = 1; return 1;
    default: return 0;
    }
}

static void check_concurrent(or_state *st, const or_event *e, uint32_t thread, or_verdict *v) {
    int space[2], dst[2], wr[2];
    uint64_t lo[2], hi[2];
    int ok[2] = {0, 0};
    const int na = copy_accesses(e->kind, space, dst, wr);
    for (int k = 0; k < na; k++) {
        uint64_t start, span;
        const int fits = dst[k] ? side_range(e->dst, e->dst_x, e->dst_y, e->dst_pitch, e->width, e->height, &start, &span)
                                : side_range(e->src, e->src_x, e->src_y, e->src_pitch, e->width, e->height, &start, &span);
        if (!fits || span == 0) continue;                                /* R-33 */
        ok[k] = 1; lo[k] = start; hi[k] = start + span;
        if (conc_hazard(st, space[k], lo[k], hi[k], wr[k], thread, e->seq)) v->flags |= F_CONCURRENT;
    }
    if (v->status == 0)                                                 /* R-34 */
        for (int k = 0; k < na; k++)
            if (ok[k]) add_stamp(st, space[k], lo[k], hi[k], wr[k], thread, e->seq);
}

/* one copy by a given thread: O5 then, in concurrency mode, O7 */
void or_check_copy_mt(or_state *st, const or_event *ev, uint32_t thread, or_verdict *v) {
    or_check_copy(st, ev, v);
    if (st->conc) check_concurrent(st, ev, thread, v);
}

/* ------------------------------------------------------ O6 leak report */
static int cmp_base(const void *a, const void *b) {
    uint64_t x = ((const or_alloc *)a)->base, y = ((const or_alloc *)b)->base;
    return x < y ? -1 : x > y;
}

uint64_t or_leaks(or_state *st, or_alloc *out, uint64_t cap) {
    or_alloc *tmp = (or_alloc *)malloc((st->n_live + 1) * sizeof(or_alloc));
    memcpy(tmp, st->live, st->n_live * sizeof(or_alloc));
    qsort(tmp, st->n_live, sizeof(or_alloc), cmp_base);
    for (uint64_t i = 0; i < st->n_live && i < cap; i++) out[i] = tmp[i];
    free(tmp);
    return st->n_live;
}

/* --------------------------------------------------------------- replay */
/* Replays n events in order.  out_v receives one verdict per COPY event (in
 * order); out_status receives one status per event (call status for
 * MARK/SETV/REG/FREE, verdict status for COPY). Returns the number of copies. */
uint64_t or_replay_mt(or_state *st, const or_event *ev, uint64_t n, const uint8_t *blob, const uint32_t *threads,
                      or_verdict *out_v, uint32_t *out_status);

uint64_t or_replay(or_state *st, const or_event *ev, uint64_t n, const uint8_t *blob,
                   or_verdict *out_v, uint32_t *out_status) {
    return or_replay_mt(st, ev, n, blob, NULL, out_v, out_status);
}

/* as or_replay; threads[i] is the thread of event i (NULL: all thread 0);
 * SYNC events are ctx_synchronize of their thread */
uint64_t or_replay_mt(or_state *st, const or_event *ev, uint64_t n, const uint8_t *blob, const uint32_t *threads,
                      or_verdict *out_v, uint32_t *out_status) {
    uint64_t nc = 0;
    for (uint64_t i = 0; i < n; i++) {
        const or_event *e = &ev[i];
        uint32_t s = 0;
        switch (e->op) {
        case OR_MARK: s = (uint32_t)or_mark(st, e->dst, e->width, e->kind); break;
        case OR_SETV: s = (uint32_t)or_set_vbits(st, e->dst, e->width, blob + e->src); break;
        case OR_REG:  s = (uint32_t)or_register(st, e->dst, e->width, e->seq); break;
        case OR_FREE: s = (uint32_t)or_free(st, e->dst, e->seq); break;
        case OR_REGA:
            s = (uint32_t)or_register_array(st, e->dst, or_array_bytes(e->width, e->height, e->dst_x, e->dst_y,
                                                                     e->dst_pitch), e->seq);
            break;
        case OR_FREEA: s = (uint32_t)or_free_array(st, e->dst, e->seq); break;
        case OR_SYNC: or_sync(st, threads ? threads[i] : 0, e->seq); break;
        case OR_COPY:
            or_check_copy(st, e, &out_v[nc]);
            if (st->conc) check_concurrent(st, e, threads ? threads[i] : 0, &out_v[nc]);
            s = out_v[nc].status;
            nc++;
            break;
        default: s = 1; break;
        }
        if (out_status) out_status[i] = s;
    }
    return nc;
}

/* ------------------------------------------------ T-thread replay (timing) */
/* The same replay on T host threads (SURVEY §8(d) "CPU oracle timing": the
 * per-descriptor check loop parallelised inside epochs; its result must equal
 * the 1-thread or_replay, which tests/ and bench.py assert).  An epoch is a
 * maximal run of consecutive COPY events in which no HtoD / HtoA reads a host
 * page (4 KiB) that an earlier DtoH / AtoH of the run writes (bounding ranges,
 * conservative): inside it every check reads the state as it was at the
 * epoch's start -- the registry does not change (registry events end an
 * epoch), DtoH checks read only A, which no copy changes, and no HtoD reads a
 * byte an earlier copy of the epoch defines -- so phase 1 runs the checks of
 * the epoch in parallel (check_only: read-only), then phase 2 applies the
 * error-free DtoH / AtoH copies, thread t writing only host bytes in its slice
 * of the window (apply_defined, so no byte is written by two threads); the
 * order of the applies does not matter (they all write 0x00).  Device V-bit
 * tracking and the concurrency checks stay sequential (or_replay). */
#include <pthread.h>

typedef struct {
    or_state *st;
    const or_event *ev;
    const uint64_t *idx;      /* event index of each copy of the epoch */
    or_verdict *out;          /* verdict of each copy of the epoch */
    uint64_t m;
    int t, T, phase;
} or_par_job;

static void *par_worker(void *arg) {
    or_par_job *j = (or_par_job *)arg;
    if (j->phase == 1) {
        for (uint64_t k = (uint64_t)j->t; k < j->m; k += (uint64_t)j->T)
            check_only(j->st, &j->ev[j->idx[k]], &j->out[k]);
    } else {
        const uint64_t slice = (j->st->s + (uint64_t)j->T - 1) / (uint64_t)j->T;
        const uint64_t lo = j->st->h0 + slice * (uint64_t)j->t;
        const uint64_t hi = (uint64_t)j->t + 1 == (uint64_t)j->T ? j->st->h0 + j->st->s : lo + slice;
        for (uint64_t k = 0; k < j->m; k++) {
            const or_event *e = &j->ev[j->idx[k]];
            if (j->out[k].status == 0 && (e->kind == OR_DTOH || e->kind == OR_ATOH)) apply_defined(j->st, e, lo, hi);
        }
    }
    return NULL;
}

static void par_run(or_state *st, const or_event *ev, const uint64_t *idx, or_verdict *out, uint64_t m, int T,
                    int phase) {
    pthread_t th[256];
    or_par_job jobs[256];
    if (T > 256) T = 256;
    for (int t = 0; t < T; t++) {
        jobs[t] = (or_par_job){st, ev, idx, out, m, t, T, phase};
        if (t) pthread_create(&th[t], NULL, par_worker, &jobs[t]);
    }
    par_worker(&jobs[0]);
    for (int t = 1; t < T; t++) pthread_join(th[t], NULL);
}

/* host bounding range of a copy, clipped to the window, as window offsets [q0, q1) */
static int host_bounds(const or_state *st, const or_event *e, int dst, uint64_t *q0, uint64_t *q1) {
    uint64_t start, span;
    const int ok = dst ? side_range(e->dst, e->dst_x, e->dst_y, e->dst_pitch, e->width, e->height, &start, &span)
                       : side_range(e->src, e->src_x, e->src_y, e->src_pitch, e->width, e->height, &start, &span);
    if (!ok || span == 0) return 0;
    const uint64_t we = st->h0 + st->s, a = start < st->h0 ? st->h0 : start;
    const uint64_t b = start + span > we ? we : start + span;
    if (a >= b) return 0;
    *q0 = a - st->h0;
    *q1 = b - st->h0;
    return 1;
}

/* one bit per host byte: set / test / clear [q0, q1) */
static void bits_set(uint64_t *m, uint64_t q0, uint64_t q1, int on) {
    for (uint64_t q = q0; q < q1;) {
        if ((q & 63) == 0 && q + 64 <= q1) { m[q >> 6] = on ? ~0ull : 0; q += 64; continue; }
        if (on) m[q >> 6] |= 1ull << (q & 63); else m[q >> 6] &= ~(1ull << (q & 63));
        q++;
    }
}
static int bits_any(const uint64_t *m, uint64_t q0, uint64_t q1) {
    for (uint64_t q = q0; q < q1;) {
        if ((q & 63) == 0 && q + 64 <= q1) { if (m[q >> 6]) return 1; q += 64; continue; }
        if ((m[q >> 6] >> (q & 63)) & 1) return 1;
        q++;
    }
    return 0;
}

uint64_t or_replay_parallel(or_state *st, const or_event *ev, uint64_t n, const uint8_t *blob, int nthreads,
                            or_verdict *out_v, uint32_t *out_status) {
    if (st->track || st->conc || nthreads <= 1) return or_replay(st, ev, n, blob, out_v, out_status);
    uint64_t *written = (uint64_t *)calloc(st->s / 64 + 1, 8);   /* host bytes a DtoH of the epoch writes */
    uint64_t *idx = (uint64_t *)malloc(sizeof(uint64_t) * (n ? n : 1));
    uint64_t nc = 0, i = 0;
    while (i < n) {
        if (ev[i].op != OR_COPY) {           /* sequential, as or_replay */
            or_replay(st, &ev[i], 1, blob, NULL, out_status ? &out_status[i] : NULL);
            i++;
            continue;
        }
        uint64_t j = i, m = 0;
        for (; j < n && ev[j].op == OR_COPY; j++) {
            const or_event *e = &ev[j];
            uint64_t q0, q1;
            if ((e->kind == OR_HTOD || e->kind == OR_HTOA) && host_bounds(st, e, 0, &q0, &q1) &&
                bits_any(written, q0, q1))
                break;                       /* reads a byte an earlier DtoH may define: next epoch */
            if ((e->kind == OR_DTOH || e->kind == OR_ATOH) && host_bounds(st, e, 1, &q0, &q1))
                bits_set(written, q0, q1, 1);
            idx[m++] = j;
        }
        par_run(st, ev, idx, out_v + nc, m, nthreads, 1);
        par_run(st, ev, idx, out_v + nc, m, nthreads, 2);
        for (uint64_t k = 0; k < m; k++) {
            const or_event *e = &ev[idx[k]];
            uint64_t q0, q1;
            if (out_status) out_status[idx[k]] = out_v[nc + k].status;
            if ((e->kind == OR_DTOH || e->kind == OR_ATOH) && host_bounds(st, e, 1, &q0, &q1))
                bits_set(written, q0, q1, 0);
        }
        nc += m;
        i = j;
    }
    free(written); free(idx);
    return nc;
}
