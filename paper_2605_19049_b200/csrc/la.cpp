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
// work lists of an index-array batch (la_decode_mixed): chunkwise slots and
// their input rows, direct slots and their input rows, slots to flush, slots
// to compress
constexpr int kWorkLists = 6;
enum { WL_CW = 0, WL_CW_POS = 1, WL_DR = 2, WL_DR_POS = 3, WL_FL = 4, WL_CP = 5 };

}  // namespace

la_status labuf_set_error(la_status st, const char *msg) { return fail(st, "%s", msg); }

struct la_buf {
    la_config cfg;
    la_sizes sz;
    Dims dm;
    Ptrs p;
    int device;
    std::vector<int32_t> occ, len, mode, pending;   // host mirror
    std::vector<uint8_t> occ_ub;                     // 1: occ is an upper bound (after la_commit_append)
    std::vector<int32_t> branch_nd;                  // pending branch verify: drafts per branch (0: plain verify)
    // pools: record blocks per slot, state index per slot
    // (-1: none); LIFO free stacks, back() = next id (initially ascending)
    bool paged = false, state_pool = false;
    std::vector<std::vector<int32_t>> blocks;
    std::vector<int32_t> sidx;
    std::vector<int32_t> free_blocks, free_states;
    int *meta_i = nullptr;                           // device meta as int32
    std::vector<int32_t> wl_dev;                     // what the device work lists hold (-1: unknown)
    // la_decode_mixed scratch (reused across calls: no per-call allocation)
    std::vector<int> mx_cw, mx_cwp, mx_dr, mx_drp, mx_fl, mx_cp;
    std::vector<uint32_t> mx_seen;
    uint32_t mx_stamp = 0;
    size_t i_sidx = 0, i_btab = 0, i_wl = 0;         // int32 offsets in meta
    int64_t launches = 0;
    int overlap = 0;                                 // la_set_overlap
    int auto_flush = 0;                              // la_set_auto_flush
    int prefill_chunk = 0;                           // la_set_prefill_chunk (0: chunk)
    alignas(64) unsigned char tmap[128];             // CUtensorMap of the state (tensor-core pass)
    int tmap_state = 0;                              // 0 not built, 1 ok, 2 unavailable
    alignas(64) unsigned char tmapk[128];            // CUtensorMap of the bf16 key records (direct step)
    int tmapk_state = 0;
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

// The state viewed as a 2-D fp32 tensor [S*Hv*128 rows][128], read in
// 32-row x 32-column boxes with the 128-byte swizzle the tensor-core state
// passes of kernels (3)/prefill consume (conflict-free fragment reads).  Built once per handle, on first use.
const void *state_tmap(la_buf *b) {
    if (b->tmap_state == 0) {
        b->tmap_state = 2;
        if (b->sz.n_states <= 0) return nullptr;
        if (auto enc = tmap_encoder()) {
            const cuuint64_t dims[2] = {(cuuint64_t)kD, (cuuint64_t)b->sz.n_states * b->dm.Hv * kD};
            const cuuint64_t strides[1] = {(cuuint64_t)kD * 4};
            const cuuint32_t box[2] = {32, 32};   // 32 columns (128 B, swizzled) x 32 rows: one d_v tile
            const cuuint32_t estr[2] = {1, 1};
            if (enc(reinterpret_cast<CUtensorMap *>(b->tmap), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, b->p.state,
                    dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
                b->tmap_state = 1;
        }
    }
    return b->tmap_state == 1 ? b->tmap : nullptr;
}

// The bf16 key records of a contiguous handle viewed as a 2-D tensor
// [R*Hk*T rows][128], read in 16-row x 64-column boxes (128 B, 128-byte
// swizzle): the conflict-free ldmatrix operand of the direct step's key rows
// on the tensor cores.  Built once per handle, on first use.
const void *key_tmap(la_buf *b) {
    if (b->tmapk_state == 0) {
        b->tmapk_state = 2;
        if (b->paged || b->cfg.in_dtype != LA_DT_BF16) return nullptr;
        if (auto enc = tmap_encoder()) {
            const cuuint64_t dims[2] = {(cuuint64_t)kD, (cuuint64_t)b->dm.R * b->dm.Hk * b->dm.T};
            const cuuint64_t strides[1] = {(cuuint64_t)kD * 2};
            const cuuint32_t box[2] = {64, 16};
            const cuuint32_t estr[2] = {1, 1};
            if (enc(reinterpret_cast<CUtensorMap *>(b->tmapk), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, b->p.K, dims,
                    strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
                b->tmapk_state = 1;
        }
    }
    return b->tmapk_state == 1 ? b->tmapk : nullptr;
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
    // (pooled handles resolve slots, states and blocks after the wait: no early loads)
    a.pdl_early = b->overlap && !prev_wrote_mine && !b->paged && !b->state_pool;
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
    if (c->block_tokens != 0 && (c->block_tokens < 4 || c->block_tokens > 128 || c->block_tokens % 4))
        return fail(LA_ERR_INVALID, "block_tokens must be 0 or a multiple of 4 in [4, 128]");
    if (c->block_tokens != 0 && c->n_blocks < 1) return fail(LA_ERR_INVALID, "a paged handle needs n_blocks >= 1");
    if (c->state_slots < -1) return fail(LA_ERR_INVALID, "state_slots must be >= -1");
    if (c->variant < LA_VARIANT_GDN || c->variant > LA_VARIANT_VANILLA) return fail(LA_ERR_INVALID, "bad variant");
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
    // record blocks: one per slot of T records, or a pool of n_blocks blocks
    const size_t bt = c->block_tokens ? c->block_tokens : T;
    const size_t nb = c->block_tokens ? c->n_blocks : R;
    s->block_tokens = (int32_t)bt;
    s->n_blocks = (int32_t)nb;
    s->max_blocks = (int32_t)((T + bt - 1) / bt);
    s->n_states = c->state_slots == 0 ? c->max_slots : std::max(c->state_slots, 0);
    s->state_bytes = (size_t)s->n_states * Hv * d * d * 4;
    size_t o = 0;
    s->off_k = o; o = round_up(o + nb * Hk * bt * d * dt_size(c->in_dtype), kAlign);
    s->off_u = o; o = round_up(o + nb * Hv * bt * d * dt_size(c->u_dtype), kAlign);
    s->off_g = o; o = round_up(o + nb * Hv * bt * 4, kAlign);
    if (c->keep_raw) {
        s->off_v = o; o = round_up(o + nb * Hv * bt * d * dt_size(c->in_dtype), kAlign);
        s->off_b = o; o = round_up(o + nb * Hv * bt * 4, kAlign);
    }
    s->buffer_bytes = o;
    // meta: occ, len, mode, ticket [R], status; state index [R]; block table
    // [R][max_blocks]; work lists [kWorkLists][R]
    size_t m = 4 * R * 4 + 16;
    s->off_sidx = m; m += R * 4;
    s->off_btab = m; m += R * (size_t)s->max_blocks * 4;
    s->off_wl = m;   m += kWorkLists * R * 4;
    s->meta_bytes = round_up(m, 256);
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

la_status check_chunkwise(la_buf *b, int r) {
    if (b->mode[r] != LA_MODE_CHUNKWISE) return fail(LA_ERR_MODE, "slot %d is not CHUNKWISE", r);
    if (b->sidx[r] < 0) return fail(LA_ERR_MODE, "slot %d holds no state (reset it as CHUNKWISE)", r);
    return LA_OK;
}
// every slot of [first, first + n) holds exactly the same, exactly known count
bool uniform_exact(const la_buf *b, int first, int n, const std::vector<int> &cnt) {
    for (int r = first; r < first + n; ++r)
        if (b->occ_ub[r] || cnt[r] != cnt[first]) return false;
    return n > 0;
}
// calls that need the exact occupancy (decode, FULL flush, prefill, mixed, recurrent)
la_status check_exact(la_buf *b, int r) {
    if (b->occ_ub[r])
        return fail(LA_ERR_MODE, "slot %d: occupancy known only as a bound after la_commit_append (flush FORCE first)", r);
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
                      const float *beta, float *o, cudaStream_t s, int fold = 0,
                      const int *slots = nullptr, const int *pos = nullptr, int passes = 3, int seg = 0,
                      bool j0_uniform = false, int pfold = 0) {
    const int mx = max_new_per_launch(b->dm.g);
    const size_t isz = dt_size(b->cfg.in_dtype);
    const size_t d = kD;
    // pass 0 checks every launch configuration (shared memory, grid) without
    // enqueueing anything, so a configuration error leaves the handle and the
    // device untouched (all-or-nothing); pass 1 enqueues.  Index-array
    // batches (slots/pos: device work lists) address the inputs by row.
    for (int pass = 0; pass < 2; ++pass) {
        if (!(passes & (1 << pass))) continue;
        for (int off = 0; off < n_tok; off += mx) {
            const int m = std::min(mx, n_tok - off);
            for (int s0 = 0; s0 < n; s0 += kMaxSlotsPerLaunch) {
                ChunkArgs a;
                a.dm = b->dm; a.p = b->p;
                a.first = first + s0; a.n = std::min(kMaxSlotsPerLaunch, n - s0);
                a.n_new = m; a.j0_cap = j0_cap + off;
                a.j0_fixed = (j0_uniform && !slots) ? j0_cap + off : -1;
                a.j_add = (kind == CK_VERIFY) ? off : 0;
                a.tok_total = tok_total; a.tok_offset = tok_base + off; a.kind = kind;
                const size_t sq = slots ? 0 : (size_t)s0 * tok_total;          // token rows skipped
                a.q = static_cast<const char *>(q) + sq * b->dm.Hk * d * isz;
                a.k = static_cast<const char *>(k) + sq * b->dm.Hk * d * isz;
                a.v = static_cast<const char *>(v) + sq * b->dm.Hv * d * isz;
                a.alpha = alpha + sq * b->dm.Hv;
                a.beta = beta + sq * b->dm.Hv;
                a.o = o ? o + sq * b->dm.Hv * d : nullptr;
                a.slots = slots ? slots + s0 : nullptr;
                a.pos = pos ? pos + s0 : nullptr;
                a.tmap = (kind == CK_VERIFY || kind == CK_PREFILL) && m >= 2 ? state_tmap(b) : nullptr;
                a.tmapk = (kind == CK_DIRECT && m == 1 && !slots) ? key_tmap(b) : nullptr;
                a.fold = fold;
                a.pfold = (pfold && m >= 2 && a.tmap) ? 1 : 0;
                a.seg = seg;
                a.dry = pass == 0;
                overlap_flags(b, s, a);
                if (slots) a.pdl_early = 0;   // the slot list itself comes from a previous grid
                cudaError_t e = launch_chunk(a, s, &b->launches);
                if (e != cudaSuccess) return e;
                if (pass == 1) note_launch(b, s, fold != 0 || a.pfold != 0);   // (a folding launch writes the state)
            }
        }
    }
    return cudaSuccess;
}

// Folds (flush, commit, compression) in slot batches of kMaxSlotsPerLaunch
// (the slot index is a grid dimension), over a range or a device slot list.
cudaError_t run_fold(la_buf *b, FoldArgs a, cudaStream_t s) {
    const int first = a.first, n = a.n;
    const int *nacc = a.nacc, *slots = a.slots;
    for (int s0 = 0; s0 < n; s0 += kMaxSlotsPerLaunch) {
        a.first = first + s0;
        a.n = std::min(kMaxSlotsPerLaunch, n - s0);
        a.nacc = nacc ? nacc + s0 : nullptr;
        a.slots = slots ? slots + s0 : nullptr;
        overlap_flags(b, s, a);
        if (slots) a.pdl_early = 0;
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

// ---------------------------------------------------------------- pools
// Host decisions (which block / state a slot gets) are made here and
// delivered to the device in stream order by the staging kernel: (meta int32
// index, value) entries passed as kernel parameters.
struct Stage {
    std::vector<int2> e;
    void put(size_t idx, int v) { e.push_back(make_int2((int)idx, v)); }
};

int blocks_for(const la_buf *b, int npos) { return b->paged ? (npos + b->dm.bt - 1) / b->dm.bt : 0; }

// Grow the slots' block lists to cover their record positions [0, npos):
// check (ok == nullptr: take) -- the check happens before anything mutates
struct Grow { int slot, npos; };
la_status check_blocks(la_buf *b, const std::vector<Grow> &g) {
    if (!b->paged) return LA_OK;
    size_t need = 0;
    for (const Grow &x : g) need += (size_t)std::max(0, blocks_for(b, x.npos) - (int)b->blocks[x.slot].size());
    if (need > b->free_blocks.size())
        return fail(LA_ERR_CAPACITY, "record block pool exhausted: %zu blocks needed, %zu free", need,
                    b->free_blocks.size());
    return LA_OK;
}
void take_blocks(la_buf *b, const std::vector<Grow> &g, Stage &st) {
    if (!b->paged) return;
    for (const Grow &x : g) {
        std::vector<int32_t> &bl = b->blocks[x.slot];
        while ((int)bl.size() < blocks_for(b, x.npos)) {
            const int id = b->free_blocks.back();
            b->free_blocks.pop_back();
            st.put(b->i_btab + (size_t)x.slot * b->dm.maxb + bl.size(), id);
            bl.push_back(id);
        }
    }
}
// return the slot's blocks beyond the first `keep` to the pool (LIFO)
void drop_blocks(la_buf *b, int r, int keep) {
    std::vector<int32_t> &bl = b->blocks[r];
    while ((int)bl.size() > keep) {
        b->free_blocks.push_back(bl.back());
        bl.pop_back();
    }
}
la_status check_states(la_buf *b, size_t need) {
    if (need == 0) return LA_OK;
    if (!b->state_pool || b->sz.n_states == 0) return fail(LA_ERR_CAPACITY, "the handle has no states (state_slots = -1)");
    if (need > b->free_states.size())
        return fail(LA_ERR_CAPACITY, "state pool exhausted: %zu states needed, %zu free", need, b->free_states.size());
    return LA_OK;
}
void take_state(la_buf *b, int r, Stage &st) {
    if (b->sidx[r] >= 0) return;
    const int id = b->free_states.back();
    b->free_states.pop_back();
    b->sidx[r] = id;
    st.put(b->i_sidx + r, id);
}
void drop_state(la_buf *b, int r) {
    if (!b->state_pool || b->sidx[r] < 0) return;
    b->free_states.push_back(b->sidx[r]);
    b->sidx[r] = -1;
}
cudaError_t run_stage(la_buf *b, Stage &st, cudaStream_t s) {
    for (size_t o = 0; o < st.e.size(); o += kStageMax) {
        const int n = (int)std::min(st.e.size() - o, (size_t)kStageMax);
        cudaError_t e = launch_stage(b->meta_i, st.e.data() + o, n, 1, s, &b->launches);
        if (e != cudaSuccess) return e;
        note_launch(b, s, true);   // state indices / tables moved: no early state loads next
    }
    st.e.clear();
    return cudaSuccess;
}
// stage work list `w` (only entries that differ from what the device holds)
void stage_list(la_buf *b, int w, const std::vector<int> &vals, Stage &st) {
    const size_t R = b->cfg.max_slots;
    for (size_t j = 0; j < vals.size(); ++j) {
        int32_t &dev = b->wl_dev[w * R + j];
        if (dev != vals[j]) {
            st.put(b->i_wl + w * R + j, vals[j]);
            dev = vals[j];
        }
    }
}
const int *wl_ptr(const la_buf *b, int w) { return b->meta_i + b->i_wl + (size_t)w * b->cfg.max_slots; }

// range -> Grow list of the slots' positions [0, base[r] + add)
std::vector<Grow> grow_range(la_buf *b, int first, int n, const std::vector<int32_t> &base, int add) {
    std::vector<Grow> g;
    if (!b->paged) return g;
    g.reserve(n);
    for (int r = first; r < first + n; ++r) g.push_back({r, base[r] + add});
    return g;
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
    b->occ_ub.assign(R, 0);
    b->branch_nd.assign(R, 0);
    dm.bt = b->sz.block_tokens; dm.maxb = b->sz.max_blocks;
    dm.bt_shift = -1;
    for (int sh = 0; sh < 31; ++sh)
        if ((1 << sh) == dm.bt) dm.bt_shift = sh;
    dm.variant = cfg->variant;
    b->meta_i = m;
    b->i_sidx = b->sz.off_sidx / 4; b->i_btab = b->sz.off_btab / 4; b->i_wl = b->sz.off_wl / 4;
    b->paged = cfg->block_tokens != 0;
    b->state_pool = cfg->state_slots != 0;
    p.sidx = b->state_pool ? m + b->i_sidx : nullptr;
    p.btab = b->paged ? m + b->i_btab : nullptr;
    b->blocks.assign(R, {});
    // without a state pool slot r owns state r; with one, slots start empty
    b->sidx.assign(R, -1);
    if (!b->state_pool)
        for (int r = 0; r < R; ++r) b->sidx[r] = r;
    b->wl_dev.assign((size_t)kWorkLists * R, -1);
    for (int i = b->sz.n_blocks - 1; b->paged && i >= 0; --i) b->free_blocks.push_back(i);
    for (int i = b->sz.n_states - 1; b->state_pool && i >= 0; --i) b->free_states.push_back(i);
    *out = b;
    return LA_OK;
}

la_status la_buf_destroy(la_buf *buf) {
    if (!buf) return fail(LA_ERR_INVALID, "null handle");
    delete buf;
    return LA_OK;
}

static la_status reset_impl(la_buf *b, int32_t first, int32_t n, int32_t mode, int32_t zero_state,
                            la_stream stream, bool release) {
    la_status st;
    if ((st = check_handle(b)) != LA_OK || (st = check_range(b, first, n)) != LA_OK) return st;
    if (mode != LA_MODE_CHUNKWISE && mode != LA_MODE_DIRECT) return fail(LA_ERR_INVALID, "bad mode");
    if (!release && mode == LA_MODE_DIRECT && b->cfg.short_cap == 0)
        return fail(LA_ERR_MODE, "direct mode disabled (short_cap = 0)");
    if (n == 0) return LA_OK;
    // state pool: CHUNKWISE slots keep or take a state, DIRECT slots return theirs
    size_t need = 0;
    if (b->state_pool && mode == LA_MODE_CHUNKWISE)
        for (int r = first; r < first + n; ++r) need += b->sidx[r] < 0;
    if ((st = check_states(b, need)) != LA_OK) return st;
    if ((st = set_device(b)) != LA_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    std::lock_guard<std::mutex> lk(g_enqueue_mu);
    Stage stg;
    for (int r = first; r < first + n; ++r) {
        drop_blocks(b, r, 0);                     // the buffer empties: blocks back to the pool
        if (mode == LA_MODE_DIRECT) drop_state(b, r);
        else take_state(b, r, stg);
    }
    cudaError_t e = run_stage(b, stg, s);
    if (e != cudaSuccess) return cuda_fail(e, "stage launch");
    // zeroing a state needs one: DIRECT slots of a state pool hold none
    const int zero = zero_state && !(b->state_pool && mode == LA_MODE_DIRECT) ? 1 : 0;
    for (int s0 = 0; s0 < n; s0 += kMaxSlotsPerLaunch) {
        e = launch_reset(b->dm, b->p, first + s0, std::min(kMaxSlotsPerLaunch, n - s0), mode, zero, s,
                         &b->launches);
        if (e != cudaSuccess) return cuda_fail(e, "reset launch");
        note_launch(b, s, zero != 0);
    }
    // status word: cleared by a reset covering slot 0
    if (first == 0 && !release) {
        e = cudaMemsetAsync(b->p.status, 0, sizeof(unsigned), s);
        if (e != cudaSuccess) return cuda_fail(e, "status clear");
    }
    for (int r = first; r < first + n; ++r) {
        b->occ[r] = 0; b->len[r] = 0; b->mode[r] = mode; b->pending[r] = 0; b->occ_ub[r] = 0; b->branch_nd[r] = 0;
    }
    return LA_OK;
}

la_status la_request_reset(la_buf *b, int32_t first, int32_t n, int32_t mode, int32_t zero_state,
                           la_stream stream) {
    return reset_impl(b, first, n, mode, zero_state, stream, false);
}

la_status la_request_release(la_buf *b, int32_t first, int32_t n, la_stream stream) {
    return reset_impl(b, first, n, LA_MODE_DIRECT, 0, stream, true);
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
        if ((st = check_chunkwise(b, r)) != LA_OK || (st = check_exact(b, r)) != LA_OK) return st;
        if (b->pending[r]) return fail(LA_ERR_MODE, "slot %d has a pending verify (commit first)", r);
        if (b->occ[r] >= b->cfg.chunk) return fail(LA_ERR_CAPACITY, "slot %d buffer full (call la_flush)", r);
        j0_cap = std::max(j0_cap, b->occ[r]);
        fills |= b->occ[r] + 1 == b->cfg.chunk;
    }
    if (n == 0) return LA_OK;
    if ((st = set_device(b)) != LA_OK) return st;
    // (the fused fold is a contiguous-handle option)
    const int fold = (b->auto_flush && fills && b->cfg.chunk <= 32 && !b->paged && !b->state_pool) ? 1 : 0;
    const std::vector<Grow> g = grow_range(b, first, n, b->occ, 1);
    if ((st = check_blocks(b, g)) != LA_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    std::lock_guard<std::mutex> lk(g_enqueue_mu);
    const bool uni = uniform_exact(b, first, n, b->occ);
    cudaError_t e = run_chunk(b, first, n, 1, j0_cap, 0, 1, CK_DECODE, q, k, v, alpha, beta, o, s, fold,
                              nullptr, nullptr, 1, 0, uni);
    if (e != cudaSuccess) return cuda_fail(e, "decode launch configuration");
    Stage stg;
    take_blocks(b, g, stg);
    if ((e = run_stage(b, stg, s)) != cudaSuccess) return cuda_fail(e, "stage launch");
    e = run_chunk(b, first, n, 1, j0_cap, 0, 1, CK_DECODE, q, k, v, alpha, beta, o, s, fold, nullptr, nullptr, 2, 0,
                  uni);
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
    if (raw && b->cfg.variant != LA_VARIANT_GDN) return fail(LA_ERR_UNSUPPORTED, "LA_FLUSH_RAW is the GDN UT transform");
    bool any = false, all = true;
    int kcap = 0;
    for (int r = first; r < first + n; ++r) {
        if (b->pending[r]) return fail(LA_ERR_MODE, "slot %d has a pending verify (commit first)", r);
        if (kind == LA_FLUSH_FULL && (st = check_exact(b, r)) != LA_OK) return st;
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
    // compression of DIRECT slots (FORCE): each needs a state from the pool
    size_t need = 0;
    if (kind == LA_FLUSH_FORCE)
        for (int r = first; r < first + n; ++r) need += b->mode[r] == LA_MODE_DIRECT && b->len[r] > 0 && b->sidx[r] < 0;
    if ((st = check_states(b, need)) != LA_OK) return st;
    for (int r = first; r < first + n; ++r)
        if (b->mode[r] == LA_MODE_CHUNKWISE && b->sidx[r] < 0 && b->occ[r] > 0)
            return fail(LA_ERR_MODE, "slot %d holds no state", r);
    if ((st = set_device(b)) != LA_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    FoldArgs a;
    a.dm = b->dm; a.p = b->p; a.first = first; a.n = n;
    a.kind = kind == LA_FLUSH_FULL ? FK_FULL : FK_FORCE; a.nacc = nullptr; a.n_draft = 0; a.kcap = kcap; a.spec = all;
    a.raw = raw ? 1 : 0;
    if (raw && !(a.tmap = state_tmap(b))) return fail(LA_ERR_CUDA, "no tensor map for the state (driver entry point missing)");
    std::lock_guard<std::mutex> lk(g_enqueue_mu);
    Stage stg;
    if (kind == LA_FLUSH_FORCE)
        for (int r = first; r < first + n; ++r)
            if (b->mode[r] == LA_MODE_DIRECT && b->len[r] > 0) take_state(b, r, stg);
    cudaError_t e = run_stage(b, stg, s);
    if (e != cudaSuccess) return cuda_fail(e, "stage launch");
    e = run_fold(b, a, s);
    if (e != cudaSuccess) return cuda_fail(e, "flush launch");
    for (int r = first; r < first + n; ++r) {
        if (kind == LA_FLUSH_FULL) {
            if (b->mode[r] == LA_MODE_CHUNKWISE && b->occ[r] == b->cfg.chunk) b->occ[r] = 0;
        } else if (b->mode[r] == LA_MODE_CHUNKWISE) {
            b->occ[r] = 0;
            b->occ_ub[r] = 0;
        } else if (b->len[r] > 0) {
            b->mode[r] = LA_MODE_CHUNKWISE; b->len[r] = 0; b->occ[r] = 0;
            // the compressed records are dead: keep the blocks a chunkwise buffer uses
            drop_blocks(b, r, blocks_for(b, b->cfg.chunk + b->cfg.max_drafts));
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
        if ((st = check_chunkwise(b, r)) != LA_OK) return st;
        if (b->pending[r]) return fail(LA_ERR_MODE, "slot %d already has a pending verify", r);
        if (b->occ[r] + n_draft > b->sz.capacity) return fail(LA_ERR_CAPACITY, "slot %d: occ + n_draft > capacity", r);
        j0_cap = std::max(j0_cap, b->occ[r]);
    }
    if (n == 0) return LA_OK;
    if ((st = set_device(b)) != LA_OK) return st;
    const std::vector<Grow> g = grow_range(b, first, n, b->occ, n_draft);
    if ((st = check_blocks(b, g)) != LA_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    std::lock_guard<std::mutex> lk(g_enqueue_mu);
    const bool uni = uniform_exact(b, first, n, b->occ);
    cudaError_t e = run_chunk(b, first, n, n_draft, j0_cap, 0, n_draft, CK_VERIFY, q, k, v, alpha, beta, o, s, 0,
                              nullptr, nullptr, 1, 0, uni);
    if (e != cudaSuccess) return cuda_fail(e, "verify launch configuration");
    Stage stg;
    take_blocks(b, g, stg);
    if ((e = run_stage(b, stg, s)) != cudaSuccess) return cuda_fail(e, "stage launch");
    e = run_chunk(b, first, n, n_draft, j0_cap, 0, n_draft, CK_VERIFY, q, k, v, alpha, beta, o, s, 0,
                  nullptr, nullptr, 2, 0, uni);
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
    for (int r = first; r < first + n; ++r) {
        if (b->pending[r] == 0 || b->pending[r] != nd)
            return fail(LA_ERR_MODE, "slot %d has no pending verify of %d drafts", r, nd);
        if (b->branch_nd[r]) return fail(LA_ERR_MODE, "slot %d: a branch verify is committed by la_commit_branch", r);
    }
    if ((st = set_device(b)) != LA_OK) return st;
    FoldArgs a;
    a.dm = b->dm; a.p = b->p; a.first = first; a.n = n;
    int occ_max = 0, occ_min = INT32_MAX;
    for (int r = first; r < first + n; ++r) {
        occ_max = std::max(occ_max, b->occ[r]);
        occ_min = std::min(occ_min, b->occ[r]);
    }
    // every slot holding buffered records folds (n = occ + n_acc >= 1): the
    // state tiles can be requested at entry (multi-round speculation)
    a.kind = FK_COMMIT; a.nacc = n_accepted; a.n_draft = nd; a.kcap = occ_max + nd; a.spec = occ_min > 0;
    std::lock_guard<std::mutex> lk(g_enqueue_mu);
    cudaError_t e = run_fold(b, a, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "commit launch");
    for (int r = first; r < first + n; ++r) { b->occ[r] = 0; b->pending[r] = 0; b->occ_ub[r] = 0; }
    return LA_OK;
}

la_status la_verify_branches(la_buf *b, int32_t first, int32_t n, int32_t n_branch, int32_t n_draft,
                             const void *q, const void *k, const void *v, const float *alpha, const float *beta,
                             float *o, la_stream stream) {
    la_status st;
    if ((st = check_handle(b)) != LA_OK || (st = check_range(b, first, n)) != LA_OK) return st;
    if ((st = check_inputs(q, k, v, alpha, beta, o, true)) != LA_OK) return st;
    const int tot = n_branch * n_draft;
    if (n_branch < 1 || n_draft < 1 || tot > b->cfg.max_drafts || tot > kMaxNewPerLaunch)
        return fail(LA_ERR_INVALID, "n_branch x n_draft = %d x %d outside [1, min(max_drafts, 16)]", n_branch, n_draft);
    int j0_cap = 0;
    for (int r = first; r < first + n; ++r) {
        if ((st = check_chunkwise(b, r)) != LA_OK) return st;
        if (b->pending[r]) return fail(LA_ERR_MODE, "slot %d already has a pending verify", r);
        if (b->occ[r] + tot > b->sz.capacity) return fail(LA_ERR_CAPACITY, "slot %d: occ + branches x drafts > capacity", r);
        j0_cap = std::max(j0_cap, b->occ[r]);
    }
    if (n == 0) return LA_OK;
    if ((st = set_device(b)) != LA_OK) return st;
    const std::vector<Grow> g = grow_range(b, first, n, b->occ, tot);
    if ((st = check_blocks(b, g)) != LA_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    std::lock_guard<std::mutex> lk(g_enqueue_mu);
    cudaError_t e = run_chunk(b, first, n, tot, j0_cap, 0, tot, CK_VERIFY, q, k, v, alpha, beta, o, s, 0,
                              nullptr, nullptr, 1, n_draft);
    if (e != cudaSuccess) return cuda_fail(e, "branch verify launch configuration");
    Stage stg;
    take_blocks(b, g, stg);
    if ((e = run_stage(b, stg, s)) != cudaSuccess) return cuda_fail(e, "stage launch");
    e = run_chunk(b, first, n, tot, j0_cap, 0, tot, CK_VERIFY, q, k, v, alpha, beta, o, s, 0, nullptr, nullptr, 2,
                  n_draft);
    if (e != cudaSuccess) return cuda_fail(e, "branch verify launch");
    for (int r = first; r < first + n; ++r) { b->pending[r] = tot; b->branch_nd[r] = n_draft; }
    return LA_OK;
}

la_status la_commit_branch(la_buf *b, int32_t first, int32_t n, const int32_t *branch, const int32_t *n_accepted,
                           la_stream stream) {
    la_status st;
    if ((st = check_handle(b)) != LA_OK || (st = check_range(b, first, n)) != LA_OK) return st;
    if (!branch || !n_accepted) return fail(LA_ERR_INVALID, "null branch / n_accepted");
    if (n == 0) return LA_OK;
    const int tot = b->pending[first], nd = b->branch_nd[first];
    int occ_max = 0;
    for (int r = first; r < first + n; ++r) {
        if (!b->pending[r] || !b->branch_nd[r] || b->pending[r] != tot || b->branch_nd[r] != nd)
            return fail(LA_ERR_MODE, "slot %d has no pending branch verify of the range's shape", r);
        occ_max = std::max(occ_max, b->occ[r]);
    }
    if ((st = set_device(b)) != LA_OK) return st;
    FoldArgs a;
    a.dm = b->dm; a.p = b->p; a.first = first; a.n = n;
    a.kind = FK_BRANCH; a.nacc = n_accepted; a.branch = branch; a.n_draft = nd; a.n_branch = tot / nd;
    a.kcap = occ_max + nd; a.spec = 0;
    std::lock_guard<std::mutex> lk(g_enqueue_mu);
    cudaError_t e = run_fold(b, a, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "branch commit launch");
    for (int r = first; r < first + n; ++r) { b->occ[r] = 0; b->pending[r] = 0; b->branch_nd[r] = 0; b->occ_ub[r] = 0; }
    return LA_OK;
}

la_status la_commit_append(la_buf *b, int32_t first, int32_t n, const int32_t *n_accepted, la_stream stream) {
    la_status st;
    if ((st = check_handle(b)) != LA_OK || (st = check_range(b, first, n)) != LA_OK) return st;
    if (!n_accepted) return fail(LA_ERR_INVALID, "null n_accepted");
    if (n == 0) return LA_OK;
    const int nd = b->pending[first];
    int occ_max = 0;
    for (int r = first; r < first + n; ++r) {
        if (b->pending[r] == 0 || b->pending[r] != nd || b->branch_nd[r])
            return fail(LA_ERR_MODE, "slot %d has no pending (non-branch) verify of %d drafts", r, nd);
        occ_max = std::max(occ_max, b->occ[r]);
    }
    // append while the buffer stays within the chunk and can take another
    // round of max_drafts drafts; else fold everything (la_commit_accepted)
    if (occ_max + nd > b->cfg.chunk || occ_max + nd + b->cfg.max_drafts > b->sz.capacity)
        return la_commit_accepted(b, first, n, n_accepted, stream);
    if ((st = set_device(b)) != LA_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    std::lock_guard<std::mutex> lk(g_enqueue_mu);
    cudaError_t e = launch_commit_append(b->dm, b->p, first, n, n_accepted, nd, b->overlap, s, &b->launches);
    if (e != cudaSuccess) return cuda_fail(e, "append-commit launch");
    note_launch(b, s, false);
    for (int r = first; r < first + n; ++r) { b->occ[r] += nd; b->pending[r] = 0; b->occ_ub[r] = 1; }
    return LA_OK;
}

la_status la_state_fork(la_buf *b, int32_t src, int32_t dst, int32_t n_records, la_stream stream) {
    la_status st;
    if ((st = check_handle(b)) != LA_OK || (st = check_range(b, src, 1)) != LA_OK ||
        (st = check_range(b, dst, 1)) != LA_OK)
        return st;
    if (src == dst) return fail(LA_ERR_INVALID, "src == dst");
    if ((st = check_chunkwise(b, dst)) != LA_OK) return st;
    if (b->occ[dst] != 0 || b->pending[dst] || b->occ_ub[dst])
        return fail(LA_ERR_MODE, "slot %d: fork destination needs an empty buffer", dst);
    if (b->occ_ub[src]) return fail(LA_ERR_MODE, "slot %d: occupancy known only as a bound", src);
    const int have = b->mode[src] == LA_MODE_CHUNKWISE ? b->occ[src] : b->len[src];
    if (n_records < 1 || n_records > have)
        return fail(LA_ERR_INVALID, "n_records %d outside [1, %d] (slot %d's buffered records)", n_records, have, src);
    if (b->mode[src] == LA_MODE_CHUNKWISE && b->sidx[src] < 0) return fail(LA_ERR_MODE, "slot %d holds no state", src);
    if ((st = set_device(b)) != LA_OK) return st;
    FoldArgs a;
    a.dm = b->dm; a.p = b->p; a.first = src; a.n = 1;
    a.kind = FK_FORK; a.nacc = nullptr; a.n_draft = 0; a.kcap = n_records; a.spec = 0;
    a.fork_n = n_records; a.fork_dst = dst;
    std::lock_guard<std::mutex> lk(g_enqueue_mu);
    cudaError_t e = run_fold(b, a, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "fork launch");
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
    const std::vector<Grow> g = grow_range(b, first, n, b->len, n_new);
    if ((st = check_blocks(b, g)) != LA_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    std::lock_guard<std::mutex> lk(g_enqueue_mu);
    const bool uni = uniform_exact(b, first, n, b->len);
    cudaError_t e = run_chunk(b, first, n, n_new, j0_cap, 0, n_new, CK_DIRECT, q, k, v, alpha, beta, o, s, 0,
                              nullptr, nullptr, 1, 0, uni);
    if (e != cudaSuccess) return cuda_fail(e, "direct launch configuration");
    Stage stg;
    take_blocks(b, g, stg);
    if ((e = run_stage(b, stg, s)) != cudaSuccess) return cuda_fail(e, "stage launch");
    e = run_chunk(b, first, n, n_new, j0_cap, 0, n_new, CK_DIRECT, q, k, v, alpha, beta, o, s, 0, nullptr, nullptr, 2,
                  0, uni);
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
        if ((st = check_chunkwise(b, r)) != LA_OK || (st = check_exact(b, r)) != LA_OK) return st;
        if (b->pending[r]) return fail(LA_ERR_MODE, "slot %d has a pending verify", r);
        if (b->occ[r] != 0) return fail(LA_ERR_MODE, "slot %d: prefill needs an empty buffer (occ = %d)", r, b->occ[r]);
    }
    if (n == 0 || n_tok == 0) return LA_OK;
    if ((st = set_device(b)) != LA_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // prefill chunk (la_set_prefill_chunk; default the handle's C): longer
    // chunks cut state traffic (64 tokens: 6 state passes per 64 tokens
    // instead of 12 with 16) but the later 16-token launches of a chunk carry
    // the chunk's earlier records (key rows, records sum) -- measured slower
    // at 64 with this kernel
    const int C = b->prefill_chunk ? b->prefill_chunk : b->cfg.chunk;
    const std::vector<Grow> g = grow_range(b, first, n, b->occ, std::min(C, n_tok));
    if ((st = check_blocks(b, g)) != LA_OK) return st;
    std::lock_guard<std::mutex> lk(g_enqueue_mu);
    {
        Stage stg;
        take_blocks(b, g, stg);
        cudaError_t e = run_stage(b, stg, s);
        if (e != cudaSuccess) return cuda_fail(e, "stage launch");
    }
    for (int c0 = 0; c0 < n_tok; c0 += C) {
        const int cn = std::min(C, n_tok - c0);
        // a chunk of 2..16 tokens is one warp-MMA launch that also folds its
        // records into the state (the buffer is empty at every chunk start):
        // one state read and one write per chunk instead of two reads
        const bool pf = cn >= 2 && cn <= max_new_per_launch(b->dm.g) && state_tmap(b) != nullptr;
        cudaError_t e = run_chunk(b, first, n, cn, 0, c0, n_tok, CK_PREFILL, q, k, v, alpha, beta, o, s, 0, nullptr,
                                  nullptr, 3, 0, false, pf ? 1 : 0);
        if (e != cudaSuccess) return cuda_fail(e, "prefill chunk launch (the handle's slots are undefined: reset them)");
        if (pf) continue;
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
        if (b->mode[r] != LA_MODE_CHUNKWISE || b->sidx[r] < 0 || b->occ[r] != 0 || b->pending[r])
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
        if (b->mode[r] != LA_MODE_CHUNKWISE || b->sidx[r] < 0 || b->occ[r] != 0 || b->pending[r])
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
        if (b->mode[r] != LA_MODE_CHUNKWISE || b->sidx[r] < 0 || b->occ[r] != 0 || b->pending[r])
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

la_status la_decode_mixed(la_buf *b, int32_t n, const int32_t *slots, const void *q, const void *k,
                          const void *v, const float *alpha, const float *beta, float *o, la_stream stream) {
    la_status st;
    if ((st = check_handle(b)) != LA_OK) return st;
    const int R = b->cfg.max_slots, C = b->cfg.chunk;
    if (n < 0 || n > R) return fail(LA_ERR_INVALID, "n %d outside [0, max_slots]", n);
    if (n == 0) return LA_OK;
    if (!slots) return fail(LA_ERR_INVALID, "null slots");
    if ((st = check_inputs(q, k, v, alpha, beta, o, true)) != LA_OK) return st;
    // route every slot to its form (host mirror): chunkwise decode (+ eager
    // flush of a buffer it fills), KV-only decode, or compression at
    // len == short_cap followed by chunkwise decode
    std::vector<int> &cw = b->mx_cw, &cw_pos = b->mx_cwp, &dr = b->mx_dr, &dr_pos = b->mx_drp, &fl = b->mx_fl,
                     &cp = b->mx_cp;
    cw.clear(); cw_pos.clear(); dr.clear(); dr_pos.clear(); fl.clear(); cp.clear();
    if (b->mx_seen.size() != (size_t)R) b->mx_seen.assign(R, 0);
    if (++b->mx_stamp == 0) { std::fill(b->mx_seen.begin(), b->mx_seen.end(), 0u); b->mx_stamp = 1; }
    const uint32_t stamp = b->mx_stamp;
    std::vector<Grow> g;
    if (b->paged) g.reserve(n);
    int j0_cw = 0, j0_dr = 0, cp_cap = 0;
    size_t need_states = 0;
    for (int i = 0; i < n; ++i) {
        const int r = slots[i];
        if (r < 0 || r >= R) return fail(LA_ERR_INVALID, "slots[%d] = %d outside [0, %d)", i, r, R);
        if (b->mx_seen[r] == stamp) return fail(LA_ERR_INVALID, "slot %d appears twice in the batch", r);
        b->mx_seen[r] = stamp;
        if (b->pending[r]) return fail(LA_ERR_MODE, "slot %d has a pending verify (commit first)", r);
        if (b->mode[r] == LA_MODE_CHUNKWISE) {
            if (b->sidx[r] < 0) return fail(LA_ERR_MODE, "slot %d holds no state (reset it as CHUNKWISE)", r);
            if ((st = check_exact(b, r)) != LA_OK) return st;
            if (b->occ[r] >= C) return fail(LA_ERR_CAPACITY, "slot %d buffer full (call la_flush)", r);
            j0_cw = std::max(j0_cw, b->occ[r]);
            g.push_back({r, b->occ[r] + 1});
            if (b->occ[r] + 1 == C) fl.push_back(r);
            cw.push_back(r); cw_pos.push_back(i);
        } else if (b->len[r] < b->cfg.short_cap) {
            j0_dr = std::max(j0_dr, b->len[r]);
            g.push_back({r, b->len[r] + 1});
            dr.push_back(r); dr_pos.push_back(i);
        } else {
            cp.push_back(r);
            cp_cap = std::max(cp_cap, b->len[r]);
            need_states += b->sidx[r] < 0;
            g.push_back({r, 1});
            if (C == 1) fl.push_back(r);
            cw.push_back(r); cw_pos.push_back(i);
        }
    }
    if ((st = check_states(b, need_states)) != LA_OK) return st;
    // blocks: compressed slots keep what a chunkwise buffer uses, the rest return first
    size_t freed = 0;
    const int keep = blocks_for(b, C + b->cfg.max_drafts);
    for (int r : cp) freed += (size_t)std::max(0, (int)b->blocks[r].size() - std::max(keep, 1));
    {
        size_t need = 0;
        for (const Grow &x : g) need += (size_t)std::max(0, blocks_for(b, x.npos) - (int)b->blocks[x.slot].size());
        if (b->paged && need > b->free_blocks.size() + freed)
            return fail(LA_ERR_CAPACITY, "record block pool exhausted: %zu blocks needed, %zu free", need,
                        b->free_blocks.size() + freed);
    }
    if ((st = set_device(b)) != LA_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    std::lock_guard<std::mutex> lk(g_enqueue_mu);
    // launch configurations first (all-or-nothing)
    const int *W_CW = wl_ptr(b, WL_CW), *W_CWP = wl_ptr(b, WL_CW_POS), *W_DR = wl_ptr(b, WL_DR),
              *W_DRP = wl_ptr(b, WL_DR_POS), *W_FL = wl_ptr(b, WL_FL), *W_CP = wl_ptr(b, WL_CP);
    // a group whose slots and input rows are both consecutive launches as a
    // plain range (no work-list loads in front of every CTA's state request):
    // the slots' own range and the inputs offset to its first row
    auto consecutive = [](const std::vector<int> &x) {
        for (size_t i = 1; i < x.size(); ++i)
            if (x[i] != x[0] + (int)i) return false;
        return !x.empty();
    };
    const size_t isz = dt_size(b->cfg.in_dtype), dd = kD;
    const int Hk = b->dm.Hk, Hv = b->dm.Hv;
    auto launch_group = [&](const std::vector<int> &sl, const std::vector<int> &pos, int j0c, int kind,
                            const int *W, const int *WP, int passes) -> cudaError_t {
        if (consecutive(sl) && consecutive(pos)) {
            const size_t p0 = (size_t)pos[0];
            return run_chunk(b, sl[0], (int)sl.size(), 1, j0c, 0, 1, kind,
                             static_cast<const char *>(q) + p0 * Hk * dd * isz, static_cast<const char *>(k) + p0 * Hk * dd * isz,
                             static_cast<const char *>(v) + p0 * Hv * dd * isz, alpha + p0 * Hv, beta + p0 * Hv,
                             o ? o + p0 * Hv * dd : nullptr, s, 0, nullptr, nullptr, passes);
        }
        return run_chunk(b, 0, (int)sl.size(), 1, j0c, 0, 1, kind, q, k, v, alpha, beta, o, s, 0, W, WP, passes);
    };
    cudaError_t e = cudaSuccess;
    if (!cw.empty()) e = launch_group(cw, cw_pos, j0_cw, CK_DECODE, W_CW, W_CWP, 1);
    if (e == cudaSuccess && !dr.empty()) e = launch_group(dr, dr_pos, j0_dr, CK_DIRECT, W_DR, W_DRP, 1);
    if (e != cudaSuccess) return cuda_fail(e, "mixed decode launch configuration");
    // pools and work lists -> one staging pass
    Stage stg;
    for (int r : cp) {
        take_state(b, r, stg);
        drop_blocks(b, r, std::max(keep, 1));
    }
    take_blocks(b, g, stg);
    stage_list(b, WL_CW, cw, stg);
    stage_list(b, WL_CW_POS, cw_pos, stg);
    stage_list(b, WL_DR, dr, stg);
    stage_list(b, WL_DR_POS, dr_pos, stg);
    stage_list(b, WL_FL, fl, stg);
    stage_list(b, WL_CP, cp, stg);
    if ((e = run_stage(b, stg, s)) != cudaSuccess) return cuda_fail(e, "stage launch");
    if (!cp.empty()) {   // compression: fold the len records into a zero state, mode -> CHUNKWISE
        FoldArgs a;
        a.dm = b->dm; a.p = b->p; a.first = 0; a.n = (int)cp.size(); a.slots = W_CP;
        a.kind = FK_FORCE; a.nacc = nullptr; a.n_draft = 0; a.kcap = cp_cap; a.spec = 0;
        if ((e = run_fold(b, a, s)) != cudaSuccess) return cuda_fail(e, "compression launch");
    }
    if (!cw.empty() && (e = launch_group(cw, cw_pos, j0_cw, CK_DECODE, W_CW, W_CWP, 2)) != cudaSuccess)
        return cuda_fail(e, "mixed decode launch");
    if (!dr.empty() && (e = launch_group(dr, dr_pos, j0_dr, CK_DIRECT, W_DR, W_DRP, 2)) != cudaSuccess)
        return cuda_fail(e, "mixed direct launch");
    if (!fl.empty()) {   // eager flush of the buffers this step filled (Z15)
        FoldArgs a;
        a.dm = b->dm; a.p = b->p; a.first = 0; a.n = (int)fl.size(); a.slots = W_FL;
        if (consecutive(fl)) { a.first = fl[0]; a.slots = nullptr; }
        a.kind = FK_FULL; a.nacc = nullptr; a.n_draft = 0; a.kcap = C; a.spec = 1;
        if ((e = run_fold(b, a, s)) != cudaSuccess) return cuda_fail(e, "flush launch");
    }
    for (int r : cp) { b->mode[r] = LA_MODE_CHUNKWISE; b->len[r] = 0; b->occ[r] = 0; }
    for (int r : cw) b->occ[r] = (b->occ[r] + 1 == C) ? 0 : b->occ[r] + 1;
    for (int r : dr) b->len[r] += 1;
    return LA_OK;
}

la_status la_pool_info(la_buf *b, int32_t *free_blocks, int32_t *total_blocks, int32_t *free_states,
                       int32_t *total_states, int32_t slot, int32_t *slot_blocks, int32_t *slot_state) {
    la_status st;
    if ((st = check_handle(b)) != LA_OK) return st;
    if (slot >= 0 && (st = check_range(b, slot, 1)) != LA_OK) return st;
    if (free_blocks) *free_blocks = b->paged ? (int32_t)b->free_blocks.size() : 0;
    if (total_blocks) *total_blocks = b->paged ? b->sz.n_blocks : 0;
    if (free_states) *free_states = b->state_pool ? (int32_t)b->free_states.size() : 0;
    if (total_states) *total_states = b->sz.n_states;
    if (slot >= 0) {
        if (slot_blocks) *slot_blocks = b->paged ? (int32_t)b->blocks[slot].size() : 1;
        if (slot_state) *slot_state = b->sidx[slot];
    }
    return LA_OK;
}

la_status la_set_auto_flush(la_buf *b, int32_t enable) {
    la_status st;
    if ((st = check_handle(b)) != LA_OK) return st;
    if (enable != 0 && enable != 1) return fail(LA_ERR_INVALID, "enable must be 0 or 1");
    b->auto_flush = enable;
    return LA_OK;
}

la_status la_set_prefill_chunk(la_buf *b, int32_t tokens) {
    la_status st;
    if ((st = check_handle(b)) != LA_OK) return st;
    if (tokens != 0 && (tokens < 1 || tokens > std::min(64, (int)b->sz.capacity)))
        return fail(LA_ERR_INVALID, "prefill chunk %d outside [1, min(64, T = %d)] (0: chunk)", tokens, b->sz.capacity);
    b->prefill_chunk = tokens;
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
    if (b->sidx[slot] < 0) return fail(LA_ERR_MODE, "slot %d holds no state", slot);
    if ((st = set_device(b)) != LA_OK) return st;
    const size_t bytes = (size_t)b->dm.Hv * kD * kD * 4;
    cudaError_t e = cudaMemcpyAsync(dst, b->p.state + (size_t)b->sidx[slot] * b->dm.Hv * kD * kD, bytes,
                                    cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "state_get copy");
    return LA_OK;
}

la_status la_state_set(la_buf *b, int32_t slot, const float *src, la_stream stream) {
    la_status st;
    if ((st = check_handle(b)) != LA_OK || (st = check_range(b, slot, 1)) != LA_OK) return st;
    if (!src) return fail(LA_ERR_INVALID, "null src");
    if (b->mode[slot] != LA_MODE_CHUNKWISE || b->sidx[slot] < 0 || b->occ[slot] != 0 || b->pending[slot])
        return fail(LA_ERR_MODE, "slot %d: state_set needs a CHUNKWISE slot with an empty buffer", slot);
    if ((st = set_device(b)) != LA_OK) return st;
    std::lock_guard<std::mutex> lk(g_enqueue_mu);
    const size_t bytes = (size_t)b->dm.Hv * kD * kD * 4;
    cudaError_t e = cudaMemcpyAsync(b->p.state + (size_t)b->sidx[slot] * b->dm.Hv * kD * kD, src, bytes,
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
