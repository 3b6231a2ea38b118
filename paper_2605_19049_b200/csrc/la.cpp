// la.cpp — host side of the C ABI declared in include/la.h: configuration
// validation, sizing, the opaque handle with its exact host occupancy mirror,
// all-or-nothing argument checking, and kernel launches on the caller's
// stream.  No device memory is allocated here and nothing synchronises
// except la_device_status.
#include "../../include/la.h"

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "internal.h"

using namespace labuf;

namespace {


thread_local std::string g_last_error;

la_status fail(la_status st, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return st;
}

la_status cuda_fail(cudaError_t e, const char *what) {
    return fail(LA_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

size_t dt_size(int dt) { return dt == LA_DT_F32 ? 4 : 2; }

constexpr size_t kAlign = 1024;

}  // namespace

la_status labuf_set_error(la_status st, const char *msg) { return fail(st, "%s", msg); }

struct la_buf {
    la_config cfg;
    la_sizes sz;
    Dims dm;
    Ptrs p;
    int device;
    std::vector<int32_t> occ, len, mode, pending;   // host mirror
    int64_t launches = 0;
    int overlap = 0;                                 // la_set_overlap
    int auto_flush = 0;                              // la_set_auto_flush
    alignas(64) unsigned char tmap[128];             // CUtensorMap of the state (tensor-core pass)
    int tmap_state = 0;                              // 0 not built, 1 ok, 2 unavailable
};

namespace {

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
    return fn;
}

// The state viewed as a 2-D fp32 tensor [R*Hv*128 rows][128], read in
// 128-row x 32-column boxes with the 128-byte swizzle the tensor-core pass
// of kernels (3)/prefill consumes.  Built once per handle, on first use.
const void *state_tmap(la_buf *b) {
    if (b->tmap_state == 0) {
        b->tmap_state = 2;
        if (auto enc = tmap_encoder()) {
            const cuuint64_t dims[2] = {(cuuint64_t)kD, (cuuint64_t)b->dm.R * b->dm.Hv * kD};
            const cuuint64_t strides[1] = {(cuuint64_t)kD * 4};
            const cuuint32_t box[2] = {32, 128};
            const cuuint32_t estr[2] = {1, 1};
            if (enc(reinterpret_cast<CUtensorMap *>(b->tmap), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, b->p.state,
                    dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
                b->tmap_state = 1;
        }
    }
    return b->tmap_state == 1 ? b->tmap : nullptr;
}

// Launch overlap bookkeeping.  With programmatic dependent launch a kernel's
// CTAs may start while the kernel immediately before it on the same stream
// drains; every kernel of the library calls griddepcontrol.launch_dependents
// only after its own griddepcontrol.wait, so no older kernel can still be
// running.  A kernel may therefore request its state tiles before the wait
// only if that immediate predecessor did not write the same state.  The
// record is kept per STREAM (process-wide), for the library's own launches:
// the last launch on the stream, whose state it was and whether it wrote it.
// g_enqueue_mu is held from the decision through the launch and the record,
// so concurrent callers on one stream (different handles, different threads)
// see the records in stream order.
struct LastLaunch {
    const void *state = nullptr;
    bool wrote = false;
};
std::mutex g_enqueue_mu;
std::unordered_map<cudaStream_t, LastLaunch> g_last_on_stream;

template <class Args>
void overlap_flags(const la_buf *b, cudaStream_t s, Args &a) {
    a.pdl = b->overlap;
    bool prev_wrote_mine = false;
    auto it = g_last_on_stream.find(s);
    if (it != g_last_on_stream.end()) prev_wrote_mine = it->second.wrote && it->second.state == b->p.state;
    a.pdl_early = b->overlap && !prev_wrote_mine;
}
void note_launch(const la_buf *b, cudaStream_t s, bool wrote_state) {
    LastLaunch &l = g_last_on_stream[s];
    l.state = b->p.state;
    l.wrote = wrote_state;
}

la_status check_config(const la_config *c) {
    if (!c) return fail(LA_ERR_INVALID, "null config");
    if (c->max_slots < 1) return fail(LA_ERR_INVALID, "max_slots must be >= 1");
    if (c->n_qk_heads < 1 || c->n_v_heads < 1) return fail(LA_ERR_INVALID, "head counts must be >= 1");
    if (c->d_k != kD || c->d_v != kD) return fail(LA_ERR_UNSUPPORTED, "d_k = d_v = 128 only (got %d, %d)", c->d_k, c->d_v);
    if (c->n_v_heads % c->n_qk_heads != 0) return fail(LA_ERR_UNSUPPORTED, "n_v_heads %% n_qk_heads != 0");
    const int g = c->n_v_heads / c->n_qk_heads;
    if (g != 1 && g != 2 && g != 4) return fail(LA_ERR_UNSUPPORTED, "n_v_heads / n_qk_heads must be 1, 2 or 4");
    if (c->chunk < 1 || c->chunk > 64) return fail(LA_ERR_INVALID, "chunk must be in [1, 64]");
    if (c->max_drafts < 0 || c->max_drafts > kMaxNewPerLaunch) return fail(LA_ERR_INVALID, "max_drafts must be in [0, 16]");
    if (c->short_cap < 0 || c->short_cap > kD) return fail(LA_ERR_INVALID, "short_cap must be in [0, 128]");
    if (c->in_dtype != LA_DT_F32 && c->in_dtype != LA_DT_BF16) return fail(LA_ERR_UNSUPPORTED, "in_dtype must be F32 or BF16");
    if (c->u_dtype != LA_DT_F32 && c->u_dtype != LA_DT_F16) return fail(LA_ERR_UNSUPPORTED, "u_dtype must be F32 or F16 (never BF16, reading Z11)");
    if (c->u_dtype == LA_DT_F16 && c->in_dtype != LA_DT_BF16) return fail(LA_ERR_UNSUPPORTED, "u_dtype F16 requires in_dtype BF16");
    if (c->keep_raw != 0 && c->keep_raw != 1) return fail(LA_ERR_INVALID, "keep_raw must be 0 or 1");
    if (c->validate != 0 && c->validate != 1) return fail(LA_ERR_INVALID, "validate must be 0 or 1");
    return LA_OK;
}

void compute_sizes(const la_config *c, la_sizes *s) {
    memset(s, 0, sizeof(*s));
    const size_t R = c->max_slots, Hk = c->n_qk_heads, Hv = c->n_v_heads, d = kD;
    // records per (slot, head), padded to a multiple of 4 so the per-head log
    // decays can be staged with 16-byte bulk copies
    const int T = (std::max(c->chunk + c->max_drafts, c->short_cap) + 3) & ~3;
    s->capacity = T;
    s->align = kAlign;
    s->state_bytes = R * Hv * d * d * 4;
    size_t o = 0;
    s->off_k = o; o = round_up(o + R * Hk * T * d * dt_size(c->in_dtype), kAlign);
    s->off_u = o; o = round_up(o + R * Hv * T * d * dt_size(c->u_dtype), kAlign);
    s->off_g = o; o = round_up(o + R * Hv * T * 4, kAlign);
    if (c->keep_raw) {
        s->off_v = o; o = round_up(o + R * Hv * T * d * dt_size(c->in_dtype), kAlign);
        s->off_b = o; o = round_up(o + R * Hv * T * 4, kAlign);
    }
    s->buffer_bytes = o;
    s->meta_bytes = round_up(4 * R * 4 + 16, 256);
    s->record_bytes = Hk * d * dt_size(c->in_dtype) + Hv * d * dt_size(c->u_dtype) + Hv * 4 +
                      (c->keep_raw ? Hv * d * dt_size(c->in_dtype) + Hv * 4 : 0);
}

bool aligned(const void *p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

la_status check_handle(la_buf *b) {
    if (!b) return fail(LA_ERR_INVALID, "null handle");
    return LA_OK;
}

la_status check_range(la_buf *b, int32_t first, int32_t n) {
    if (first < 0 || n < 0 || (int64_t)first + n > b->cfg.max_slots)
        return fail(LA_ERR_INVALID, "slot range [%d, %d) outside [0, %d)", first, first + n, b->cfg.max_slots);
    return LA_OK;
}

la_status check_inputs(const void *q, const void *k, const void *v, const float *alpha,
                       const float *beta, const float *o, bool o_required) {
    if (!q || !k || !v || !alpha || !beta) return fail(LA_ERR_INVALID, "null input pointer");
    if (o_required && !o) return fail(LA_ERR_INVALID, "null output pointer");
    if (!aligned(q, 16) || !aligned(k, 16) || !aligned(v, 16) || !aligned(alpha, 4) ||
        !aligned(beta, 4) || (o && !aligned(o, 16)))
        return fail(LA_ERR_INVALID, "inputs must be 16-byte aligned");
    return LA_OK;
}

la_status set_device(la_buf *b) {
    int cur = -1;
    cudaError_t e = cudaGetDevice(&cur);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (cur != b->device) {
        e = cudaSetDevice(b->device);
        if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    }
    return LA_OK;
}

// Enqueue the chunk-attend kernel for tokens [tok_base, tok_base + n_tok) of
// per-slot arrays holding tok_total tokens, split into launches of at most
// max_new_per_launch(g) tokens and kMaxSlotsPerLaunch slots.  Launches of a
// token split see the earlier tokens as buffered records: the device counter
// advanced for decode/direct/prefill, an explicit offset (j_add) for verify.
cudaError_t run_chunk(la_buf *b, int first, int n, int n_tok, int j0_cap, int tok_base, int tok_total,
                      int kind, const void *q, const void *k, const void *v, const float *alpha,
                      const float *beta, float *o, cudaStream_t s, int fold = 0) {
    const int mx = max_new_per_launch(b->dm.g);
    const size_t isz = dt_size(b->cfg.in_dtype);
    const size_t d = kD;
    // pass 0 checks every launch configuration (shared memory, grid) without
    // enqueueing anything, so a configuration error leaves the handle and the
    // device untouched (all-or-nothing); pass 1 enqueues
    for (int pass = 0; pass < 2; ++pass) {
        for (int off = 0; off < n_tok; off += mx) {
            const int m = std::min(mx, n_tok - off);
            for (int s0 = 0; s0 < n; s0 += kMaxSlotsPerLaunch) {
                ChunkArgs a;
                a.dm = b->dm; a.p = b->p;
                a.first = first + s0; a.n = std::min(kMaxSlotsPerLaunch, n - s0);
                a.n_new = m; a.j0_cap = j0_cap + off;
                a.j_add = (kind == CK_VERIFY) ? off : 0;
                a.tok_total = tok_total; a.tok_offset = tok_base + off; a.kind = kind;
                const size_t sq = (size_t)s0 * tok_total;          // token rows skipped
                a.q = static_cast<const char *>(q) + sq * b->dm.Hk * d * isz;
                a.k = static_cast<const char *>(k) + sq * b->dm.Hk * d * isz;
                a.v = static_cast<const char *>(v) + sq * b->dm.Hv * d * isz;
                a.alpha = alpha + sq * b->dm.Hv;
                a.beta = beta + sq * b->dm.Hv;
                a.o = o ? o + sq * b->dm.Hv * d : nullptr;
                a.tmap = (kind == CK_VERIFY || kind == CK_PREFILL) && m >= 2 ? state_tmap(b) : nullptr;
                a.fold = fold;
                a.dry = pass == 0;
                overlap_flags(b, s, a);
                cudaError_t e = launch_chunk(a, s, &b->launches);
                if (e != cudaSuccess) return e;
                if (pass == 1) note_launch(b, s, fold != 0);
            }
        }
    }
    return cudaSuccess;
}

// Folds (flush, commit, compression) in slot batches of kMaxSlotsPerLaunch
// (the slot index is a grid dimension).
cudaError_t run_fold(la_buf *b, FoldArgs a, cudaStream_t s) {
    const int first = a.first, n = a.n;
    const int *nacc = a.nacc;
    for (int s0 = 0; s0 < n; s0 += kMaxSlotsPerLaunch) {
        a.first = first + s0;
        a.n = std::min(kMaxSlotsPerLaunch, n - s0);
        a.nacc = nacc ? nacc + s0 : nullptr;
        overlap_flags(b, s, a);
        cudaError_t e = launch_fold(a, s, &b->launches);
        if (e != cudaSuccess) return e;
        note_launch(b, s, true);
    }
    return cudaSuccess;
}

// Recurrent kernels (5a)/(5b)/commit in slot batches; per-slot arrays
// (inputs [n][n_draft][...], outputs, temporary states, n_accepted) advance
// with the batch.
template <class Launch>
cudaError_t run_rec(la_buf *b, RecArgs a, cudaStream_t s, bool wrote, Launch launch) {
    const int first = a.first, n = a.n, N = a.n_draft;
    const size_t isz = dt_size(b->cfg.in_dtype), d = kD, Hk = b->dm.Hk, Hv = b->dm.Hv;
    const RecArgs a0 = a;
    for (int s0 = 0; s0 < n; s0 += kMaxSlotsPerLaunch) {
        const size_t sq = (size_t)s0 * N;
        a.first = first + s0;
        a.n = std::min(kMaxSlotsPerLaunch, n - s0);
        if (a0.q) {
            a.q = static_cast<const char *>(a0.q) + sq * Hk * d * isz;
            a.k = static_cast<const char *>(a0.k) + sq * Hk * d * isz;
            a.v = static_cast<const char *>(a0.v) + sq * Hv * d * isz;
            a.alpha = a0.alpha + sq * Hv;
            a.beta = a0.beta + sq * Hv;
            a.o = a0.o + sq * Hv * d;
        }
        if (a0.temp) a.temp = a0.temp + sq * Hv * d * d;
        if (a0.nacc) a.nacc = a0.nacc + s0;
        overlap_flags(b, s, a);
        cudaError_t e = launch(a, s, &b->launches);
        if (e != cudaSuccess) return e;
        note_launch(b, s, wrote);
    }
    return cudaSuccess;
}

}  // namespace

extern "C" {

la_status la_buf_query(const la_config *cfg, la_sizes *out) {
    la_status st = check_config(cfg);
    if (st != LA_OK) return st;
    if (!out) return fail(LA_ERR_INVALID, "null sizes output");
    compute_sizes(cfg, out);
    return LA_OK;
}

la_status la_buf_create(const la_config *cfg, void *state, void *buffer, void *meta, int32_t device,
                        la_buf **out) {
    la_status st = check_config(cfg);
    if (st != LA_OK) return st;
    if (!out) return fail(LA_ERR_INVALID, "null handle output");
    if (!state || !buffer || !meta) return fail(LA_ERR_INVALID, "null device pointer");
    if (!aligned(state, kAlign) || !aligned(buffer, kAlign) || !aligned(meta, 256))
        return fail(LA_ERR_INVALID, "state/buffer must be 1024-byte aligned, meta 256-byte aligned");
    if (device < 0) return fail(LA_ERR_INVALID, "bad device ordinal");
    la_buf *b = new la_buf();
    b->cfg = *cfg;
    compute_sizes(cfg, &b->sz);
    b->device = device;
    Dims &dm = b->dm;
    dm.R = cfg->max_slots; dm.Hk = cfg->n_qk_heads; dm.Hv = cfg->n_v_heads;
    dm.g = cfg->n_v_heads / cfg->n_qk_heads; dm.T = b->sz.capacity; dm.C = cfg->chunk;
    dm.in_dt = cfg->in_dtype; dm.u_dt = cfg->u_dtype; dm.keep_raw = cfg->keep_raw;
    dm.validate = cfg->validate;
    Ptrs &p = b->p;
    char *bb = static_cast<char *>(buffer);
    p.state = static_cast<float *>(state);
    p.K = bb + b->sz.off_k;
    p.U = bb + b->sz.off_u;
    p.G = reinterpret_cast<float *>(bb + b->sz.off_g);
    p.V = cfg->keep_raw ? bb + b->sz.off_v : nullptr;
    p.B = cfg->keep_raw ? reinterpret_cast<float *>(bb + b->sz.off_b) : nullptr;
    int32_t *m = static_cast<int32_t *>(meta);
    const int R = cfg->max_slots;
    p.occ = m; p.len = m + R; p.mode = m + 2 * R; p.ticket = m + 3 * R;
    p.status = reinterpret_cast<unsigned *>(m + 4 * R);
    b->occ.assign(R, 0); b->len.assign(R, 0); b->mode.assign(R, 0); b->pending.assign(R, 0);
    *out = b;
    return LA_OK;
}

la_status la_buf_destroy(la_buf *buf) {
    if (!buf) return fail(LA_ERR_INVALID, "null handle");
    delete buf;
    return LA_OK;
}

la_status la_request_reset(la_buf *b, int32_t first, int32_t n, int32_t mode, int32_t zero_state,
                           la_stream stream) {
    la_status st;
    if ((st = check_handle(b)) != LA_OK || (st = check_range(b, first, n)) != LA_OK) return st;
    if (mode != LA_MODE_CHUNKWISE && mode != LA_MODE_DIRECT) return fail(LA_ERR_INVALID, "bad mode");
    if (mode == LA_MODE_DIRECT && b->cfg.short_cap == 0) return fail(LA_ERR_MODE, "direct mode disabled (short_cap = 0)");
    if (n == 0) return LA_OK;
    if ((st = set_device(b)) != LA_OK) return st;
    std::lock_guard<std::mutex> lk(g_enqueue_mu);
    for (int s0 = 0; s0 < n; s0 += kMaxSlotsPerLaunch) {
        cudaError_t e = launch_reset(b->dm, b->p, first + s0, std::min(kMaxSlotsPerLaunch, n - s0), mode,
                                     zero_state ? 1 : 0, static_cast<cudaStream_t>(stream), &b->launches);
        if (e != cudaSuccess) return cuda_fail(e, "reset launch");
        note_launch(b, static_cast<cudaStream_t>(stream), zero_state != 0);
    }
    // status word: cleared by a reset covering slot 0
    if (first == 0) {
        cudaError_t e = cudaMemsetAsync(b->p.status, 0, sizeof(unsigned), static_cast<cudaStream_t>(stream));
        if (e != cudaSuccess) return cuda_fail(e, "status clear");
    }
    for (int r = first; r < first + n; ++r) {
        b->occ[r] = 0; b->len[r] = 0; b->mode[r] = mode; b->pending[r] = 0;
    }
    return LA_OK;
}

la_status la_decode_step(la_buf *b, int32_t first, int32_t n, const void *q, const void *k,
                         const void *v, const float *alpha, const float *beta, float *o,
                         la_stream stream) {
    la_status st;
    if ((st = check_handle(b)) != LA_OK || (st = check_range(b, first, n)) != LA_OK) return st;
    if ((st = check_inputs(q, k, v, alpha, beta, o, true)) != LA_OK) return st;
    int j0_cap = 0;
    bool fills = false;
    for (int r = first; r < first + n; ++r) {
        if (b->mode[r] != LA_MODE_CHUNKWISE) return fail(LA_ERR_MODE, "slot %d is not CHUNKWISE", r);
        if (b->pending[r]) return fail(LA_ERR_MODE, "slot %d has a pending verify (commit first)", r);
        if (b->occ[r] >= b->cfg.chunk) return fail(LA_ERR_CAPACITY, "slot %d buffer full (call la_flush)", r);
        j0_cap = std::max(j0_cap, b->occ[r]);
        fills |= b->occ[r] + 1 == b->cfg.chunk;
    }
    if (n == 0) return LA_OK;
    if ((st = set_device(b)) != LA_OK) return st;
    const int fold = (b->auto_flush && fills && b->cfg.chunk <= 32) ? 1 : 0;
    std::lock_guard<std::mutex> lk(g_enqueue_mu);
    cudaError_t e = run_chunk(b, first, n, 1, j0_cap, 0, 1, CK_DECODE, q, k, v, alpha, beta, o,
                              static_cast<cudaStream_t>(stream), fold);
    if (e != cudaSuccess) return cuda_fail(e, "decode launch");
    for (int r = first; r < first + n; ++r) {
        b->occ[r] += 1;
        if (fold && b->occ[r] == b->cfg.chunk) b->occ[r] = 0;   // folded in the same kernel
    }
    return LA_OK;
}

la_status la_flush(la_buf *b, int32_t first, int32_t n, int32_t kind, la_stream stream) {
    la_status st;
    if ((st = check_handle(b)) != LA_OK || (st = check_range(b, first, n)) != LA_OK) return st;
    const bool raw = (kind & LA_FLUSH_RAW) != 0;
    kind &= ~LA_FLUSH_RAW;
    if (kind != LA_FLUSH_FULL && kind != LA_FLUSH_FORCE) return fail(LA_ERR_INVALID, "bad flush kind");
    if (raw && !b->cfg.keep_raw) return fail(LA_ERR_INVALID, "LA_FLUSH_RAW needs a handle created with keep_raw = 1");
    bool any = false, all = true;
    int kcap = 0;
    for (int r = first; r < first + n; ++r) {
        if (b->pending[r]) return fail(LA_ERR_MODE, "slot %d has a pending verify (commit first)", r);
        int nr = 0;
        if (kind == LA_FLUSH_FULL)
            nr = (b->mode[r] == LA_MODE_CHUNKWISE && b->occ[r] == b->cfg.chunk) ? b->occ[r] : 0;
        else
            nr = b->mode[r] == LA_MODE_CHUNKWISE ? b->occ[r] : b->len[r];
        any |= nr > 0;
        all &= nr > 0 && !(kind == LA_FLUSH_FORCE && b->mode[r] == LA_MODE_DIRECT);
        kcap = std::max(kcap, nr);
    }
    if (!any) return LA_OK;   // empty flush is not an error (SPEC flush_and_free)
    if ((st = set_device(b)) != LA_OK) return st;
    FoldArgs a;
    a.dm = b->dm; a.p = b->p; a.first = first; a.n = n;
    a.kind = kind == LA_FLUSH_FULL ? FK_FULL : FK_FORCE; a.nacc = nullptr; a.n_draft = 0; a.kcap = kcap; a.spec = all;
    a.raw = raw ? 1 : 0;
    std::lock_guard<std::mutex> lk(g_enqueue_mu);
    cudaError_t e = run_fold(b, a, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "flush launch");
    for (int r = first; r < first + n; ++r) {
        if (kind == LA_FLUSH_FULL) {
            if (b->mode[r] == LA_MODE_CHUNKWISE && b->occ[r] == b->cfg.chunk) b->occ[r] = 0;
        } else if (b->mode[r] == LA_MODE_CHUNKWISE) {
            b->occ[r] = 0;
        } else if (b->len[r] > 0) {
            b->mode[r] = LA_MODE_CHUNKWISE; b->len[r] = 0; b->occ[r] = 0;
        }
    }
    return LA_OK;
}

la_status la_verify_drafts(la_buf *b, int32_t first, int32_t n, int32_t n_draft, const void *q,
                           const void *k, const void *v, const float *alpha, const float *beta,
                           float *o, la_stream stream) {
    la_status st;
    if ((st = check_handle(b)) != LA_OK || (st = check_range(b, first, n)) != LA_OK) return st;
    if ((st = check_inputs(q, k, v, alpha, beta, o, true)) != LA_OK) return st;
    if (n_draft < 1 || n_draft > b->cfg.max_drafts)
        return fail(LA_ERR_INVALID, "n_draft %d outside [1, %d]", n_draft, b->cfg.max_drafts);
    int j0_cap = 0;
    for (int r = first; r < first + n; ++r) {
        if (b->mode[r] != LA_MODE_CHUNKWISE) return fail(LA_ERR_MODE, "slot %d is not CHUNKWISE", r);
        if (b->pending[r]) return fail(LA_ERR_MODE, "slot %d already has a pending verify", r);
        if (b->occ[r] + n_draft > b->sz.capacity) return fail(LA_ERR_CAPACITY, "slot %d: occ + n_draft > capacity", r);
        j0_cap = std::max(j0_cap, b->occ[r]);
    }
    if (n == 0) return LA_OK;
    if ((st = set_device(b)) != LA_OK) return st;
    std::lock_guard<std::mutex> lk(g_enqueue_mu);
    cudaError_t e = run_chunk(b, first, n, n_draft, j0_cap, 0, n_draft, CK_VERIFY, q, k, v, alpha, beta, o,
                              static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "verify launch");
    for (int r = first; r < first + n; ++r) b->pending[r] = n_draft;
    return LA_OK;
}

la_status la_commit_accepted(la_buf *b, int32_t first, int32_t n, const int32_t *n_accepted,
                             la_stream stream) {
    la_status st;
    if ((st = check_handle(b)) != LA_OK || (st = check_range(b, first, n)) != LA_OK) return st;
    if (!n_accepted) return fail(LA_ERR_INVALID, "null n_accepted");
    if (n == 0) return LA_OK;
    const int nd = b->pending[first];
    for (int r = first; r < first + n; ++r)
        if (b->pending[r] == 0 || b->pending[r] != nd)
            return fail(LA_ERR_MODE, "slot %d has no pending verify of %d drafts", r, nd);
    if ((st = set_device(b)) != LA_OK) return st;
    FoldArgs a;
    a.dm = b->dm; a.p = b->p; a.first = first; a.n = n;
    int occ_max = 0;
    for (int r = first; r < first + n; ++r) occ_max = std::max(occ_max, b->occ[r]);
    a.kind = FK_COMMIT; a.nacc = n_accepted; a.n_draft = nd; a.kcap = occ_max + nd; a.spec = 0;
    std::lock_guard<std::mutex> lk(g_enqueue_mu);
    cudaError_t e = run_fold(b, a, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "commit launch");
    for (int r = first; r < first + n; ++r) { b->occ[r] = 0; b->pending[r] = 0; }
    return LA_OK;
}

la_status la_direct_short(la_buf *b, int32_t first, int32_t n, int32_t n_new, const void *q,
                          const void *k, const void *v, const float *alpha, const float *beta,
                          float *o, la_stream stream) {
    la_status st;
    if ((st = check_handle(b)) != LA_OK || (st = check_range(b, first, n)) != LA_OK) return st;
    if ((st = check_inputs(q, k, v, alpha, beta, o, true)) != LA_OK) return st;
    if (n_new < 1) return fail(LA_ERR_INVALID, "n_new must be >= 1");
    int j0_cap = 0;
    for (int r = first; r < first + n; ++r) {
        if (b->mode[r] != LA_MODE_DIRECT) return fail(LA_ERR_MODE, "slot %d is not DIRECT", r);
        if (b->len[r] + n_new > b->cfg.short_cap) return fail(LA_ERR_CAPACITY, "slot %d: len + n_new > short_cap", r);
        j0_cap = std::max(j0_cap, b->len[r]);
    }
    if (n == 0) return LA_OK;
    if ((st = set_device(b)) != LA_OK) return st;
    std::lock_guard<std::mutex> lk(g_enqueue_mu);
    cudaError_t e = run_chunk(b, first, n, n_new, j0_cap, 0, n_new, CK_DIRECT, q, k, v, alpha, beta, o,
                              static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "direct launch");
    for (int r = first; r < first + n; ++r) b->len[r] += n_new;
    return LA_OK;
}

la_status la_prefill(la_buf *b, int32_t first, int32_t n, int32_t n_tok, const void *q, const void *k,
                     const void *v, const float *alpha, const float *beta, float *o, la_stream stream) {
    la_status st;
    if ((st = check_handle(b)) != LA_OK || (st = check_range(b, first, n)) != LA_OK) return st;
    if ((st = check_inputs(q, k, v, alpha, beta, o, false)) != LA_OK) return st;
    if (n_tok < 0) return fail(LA_ERR_INVALID, "n_tok must be >= 0");
    for (int r = first; r < first + n; ++r) {
        if (b->mode[r] != LA_MODE_CHUNKWISE) return fail(LA_ERR_MODE, "slot %d is not CHUNKWISE", r);
        if (b->pending[r]) return fail(LA_ERR_MODE, "slot %d has a pending verify", r);
        if (b->occ[r] != 0) return fail(LA_ERR_MODE, "slot %d: prefill needs an empty buffer (occ = %d)", r, b->occ[r]);
    }
    if (n == 0 || n_tok == 0) return LA_OK;
    if ((st = set_device(b)) != LA_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int C = b->cfg.chunk;
    std::lock_guard<std::mutex> lk(g_enqueue_mu);
    for (int c0 = 0; c0 < n_tok; c0 += C) {
        const int cn = std::min(C, n_tok - c0);
        cudaError_t e = run_chunk(b, first, n, cn, 0, c0, n_tok, CK_PREFILL, q, k, v, alpha, beta, o, s);
        if (e != cudaSuccess) return cuda_fail(e, "prefill chunk launch (the handle's slots are undefined: reset them)");
        FoldArgs f;
        f.dm = b->dm; f.p = b->p; f.first = first; f.n = n; f.kind = FK_FORCE; f.nacc = nullptr; f.n_draft = 0;
        f.kcap = cn; f.spec = 1;
        e = run_fold(b, f, s);
        if (e != cudaSuccess) return cuda_fail(e, "prefill fold launch (the handle's slots are undefined: reset them)");
    }
    return LA_OK;
}

la_status la_recurrent_step(la_buf *b, int32_t first, int32_t n, const void *q, const void *k,
                            const void *v, const float *alpha, const float *beta, float *o,
                            la_stream stream) {
    la_status st;
    if ((st = check_handle(b)) != LA_OK || (st = check_range(b, first, n)) != LA_OK) return st;
    if ((st = check_inputs(q, k, v, alpha, beta, o, true)) != LA_OK) return st;
    for (int r = first; r < first + n; ++r)
        if (b->mode[r] != LA_MODE_CHUNKWISE || b->occ[r] != 0 || b->pending[r])
            return fail(LA_ERR_MODE, "slot %d: recurrent step needs a CHUNKWISE slot with an empty buffer", r);
    if (n == 0) return LA_OK;
    if ((st = set_device(b)) != LA_OK) return st;
    RecArgs a{};
    a.dm = b->dm; a.p = b->p; a.first = first; a.n = n; a.n_draft = 1;
    a.q = q; a.k = k; a.v = v; a.alpha = alpha; a.beta = beta; a.o = o;
    std::lock_guard<std::mutex> lk(g_enqueue_mu);
    cudaError_t e = run_rec(b, a, static_cast<cudaStream_t>(stream), true, launch_recurrent_step);
    if (e != cudaSuccess) return cuda_fail(e, "recurrent step launch");
    return LA_OK;
}

la_status la_recurrent_verify(la_buf *b, int32_t first, int32_t n, int32_t n_draft, const void *q,
                              const void *k, const void *v, const float *alpha, const float *beta,
                              float *temp, float *o, la_stream stream) {
    la_status st;
    if ((st = check_handle(b)) != LA_OK || (st = check_range(b, first, n)) != LA_OK) return st;
    if ((st = check_inputs(q, k, v, alpha, beta, o, true)) != LA_OK) return st;
    if (!temp || !aligned(temp, 16)) return fail(LA_ERR_INVALID, "temp must be a 16-byte aligned device pointer");
    if (n_draft < 1 || n_draft > kMaxNewPerLaunch) return fail(LA_ERR_INVALID, "n_draft outside [1, 16]");
    for (int r = first; r < first + n; ++r)
        if (b->mode[r] != LA_MODE_CHUNKWISE || b->occ[r] != 0 || b->pending[r])
            return fail(LA_ERR_MODE, "slot %d: recurrent verify needs a CHUNKWISE slot with an empty buffer", r);
    if (n == 0) return LA_OK;
    if ((st = set_device(b)) != LA_OK) return st;
    RecArgs a{};
    a.dm = b->dm; a.p = b->p; a.first = first; a.n = n; a.n_draft = n_draft;
    a.q = q; a.k = k; a.v = v; a.alpha = alpha; a.beta = beta; a.o = o; a.temp = temp;
    std::lock_guard<std::mutex> lk(g_enqueue_mu);
    cudaError_t e = run_rec(b, a, static_cast<cudaStream_t>(stream), false, launch_recurrent_verify);
    if (e != cudaSuccess) return cuda_fail(e, "recurrent verify launch");
    return LA_OK;
}

la_status la_recurrent_commit(la_buf *b, int32_t first, int32_t n, int32_t n_draft,
                              const int32_t *n_accepted, const float *temp, la_stream stream) {
    la_status st;
    if ((st = check_handle(b)) != LA_OK || (st = check_range(b, first, n)) != LA_OK) return st;
    if (!n_accepted || !temp || !aligned(temp, 16)) return fail(LA_ERR_INVALID, "null/misaligned pointer");
    if (n_draft < 1 || n_draft > kMaxNewPerLaunch) return fail(LA_ERR_INVALID, "n_draft outside [1, 16]");
    for (int r = first; r < first + n; ++r)
        if (b->mode[r] != LA_MODE_CHUNKWISE || b->occ[r] != 0 || b->pending[r])
            return fail(LA_ERR_MODE, "slot %d: recurrent commit needs a CHUNKWISE slot with an empty buffer", r);
    if (n == 0) return LA_OK;
    if ((st = set_device(b)) != LA_OK) return st;
    RecArgs a{};
    a.dm = b->dm; a.p = b->p; a.first = first; a.n = n; a.n_draft = n_draft;
    a.nacc = n_accepted; a.temp = const_cast<float *>(temp);
    std::lock_guard<std::mutex> lk(g_enqueue_mu);
    cudaError_t e = run_rec(b, a, static_cast<cudaStream_t>(stream), true, launch_recurrent_commit);
    if (e != cudaSuccess) return cuda_fail(e, "recurrent commit launch");
    return LA_OK;
}

la_status la_set_auto_flush(la_buf *b, int32_t enable) {
    la_status st;
    if ((st = check_handle(b)) != LA_OK) return st;
    if (enable != 0 && enable != 1) return fail(LA_ERR_INVALID, "enable must be 0 or 1");
    b->auto_flush = enable;
    return LA_OK;
}

la_status la_set_overlap(la_buf *b, int32_t enable) {
    la_status st;
    if ((st = check_handle(b)) != LA_OK) return st;
    if (enable != 0 && enable != 1) return fail(LA_ERR_INVALID, "enable must be 0 or 1");
    b->overlap = enable;
    return LA_OK;
}

la_status la_state_get(la_buf *b, int32_t slot, float *dst, la_stream stream) {
    la_status st;
    if ((st = check_handle(b)) != LA_OK || (st = check_range(b, slot, 1)) != LA_OK) return st;
    if (!dst) return fail(LA_ERR_INVALID, "null dst");
    if ((st = set_device(b)) != LA_OK) return st;
    const size_t bytes = (size_t)b->dm.Hv * kD * kD * 4;
    cudaError_t e = cudaMemcpyAsync(dst, b->p.state + (size_t)slot * b->dm.Hv * kD * kD, bytes,
                                    cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "state_get copy");
    return LA_OK;
}

la_status la_state_set(la_buf *b, int32_t slot, const float *src, la_stream stream) {
    la_status st;
    if ((st = check_handle(b)) != LA_OK || (st = check_range(b, slot, 1)) != LA_OK) return st;
    if (!src) return fail(LA_ERR_INVALID, "null src");
    if (b->mode[slot] != LA_MODE_CHUNKWISE || b->occ[slot] != 0 || b->pending[slot])
        return fail(LA_ERR_MODE, "slot %d: state_set needs a CHUNKWISE slot with an empty buffer", slot);
    if ((st = set_device(b)) != LA_OK) return st;
    std::lock_guard<std::mutex> lk(g_enqueue_mu);
    const size_t bytes = (size_t)b->dm.Hv * kD * kD * 4;
    cudaError_t e = cudaMemcpyAsync(b->p.state + (size_t)slot * b->dm.Hv * kD * kD, src, bytes,
                                    cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "state_set copy");
    note_launch(b, static_cast<cudaStream_t>(stream), true);
    return LA_OK;
}

la_status la_slot_info(la_buf *b, int32_t slot, int32_t *occ, int32_t *len, int32_t *mode,
                       int32_t *pending_drafts) {
    la_status st;
    if ((st = check_handle(b)) != LA_OK || (st = check_range(b, slot, 1)) != LA_OK) return st;
    if (occ) *occ = b->occ[slot];
    if (len) *len = b->len[slot];
    if (mode) *mode = b->mode[slot];
    if (pending_drafts) *pending_drafts = b->pending[slot];
    return LA_OK;
}

la_status la_device_status(la_buf *b, la_stream stream, uint32_t *flags, int32_t *occ_host,
                           int32_t *len_host, int32_t *mode_host) {
    la_status st;
    if ((st = check_handle(b)) != LA_OK) return st;
    if ((st = set_device(b)) != LA_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "stream synchronize");
    const int R = b->cfg.max_slots;
    unsigned f = 0;
    e = cudaMemcpy(&f, b->p.status, sizeof(unsigned), cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && occ_host) e = cudaMemcpy(occ_host, b->p.occ, R * 4, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && len_host) e = cudaMemcpy(len_host, b->p.len, R * 4, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && mode_host) e = cudaMemcpy(mode_host, b->p.mode, R * 4, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "status read");
    if (flags) *flags = f;
    return LA_OK;
}

int64_t la_kernel_launches(const la_buf *b) { return b ? b->launches : -1; }

const char *la_last_error(void) { return g_last_error.c_str(); }

}  // extern "C"
