// internal.h — kernel argument blocks and launcher declarations shared by the
// host library (la.cpp) and the kernels (*.cu).  Internal; not the C ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace labuf {

constexpr int kD = 128;          // d_k = d_v
constexpr int kRows = 32;        // d_v rows per V head per recurrent-kernel CTA
constexpr int kUSub = 32;        // U records are stored tile-major: [R][Hv][d/kUSub][T][kUSub]
constexpr int kMaxNewPerLaunch = 16;
constexpr int kMaxSlotsPerLaunch = 4096;
// new tokens per chunk-kernel launch (the log-decay scan runs in one warp)
inline int max_new_per_launch(int /*g*/) { return kMaxNewPerLaunch; }

enum DType : int { DT_F32 = 0, DT_BF16 = 1, DT_F16 = 2 };

// Record addressing.  Records live in blocks of `bt` token positions:
// K [nblk][Hk][bt][d], U [nblk][Hv][d/kUSub][bt][kUSub], G [nblk][Hv][bt],
// V [nblk][Hv][bt][d], B [nblk][Hv][bt].  Contiguous handles (block_tokens =
// 0) are the special case bt = T, one block per slot, block id = slot, no
// table; paged handles look position p of slot r up in the block table:
// block btab[r * maxb + p / bt], offset p % bt.
// States: slot r's state is state[sidx[r]] with a state pool, state[r]
// without (sidx == nullptr).
struct Dims {
    int R, Hk, Hv, g, T, C;
    int in_dt, u_dt, keep_raw, validate;
    int bt, maxb;        // tokens per record block; blocks per slot (table row length)
    int bt_shift;        // log2(bt) when bt is a power of two (block / offset by shift and mask), else -1
    int variant;         // 0 GDN (gate + delta rule), 1 gated LA (no delta), 2 vanilla LA
};

// Launch overlap (la_set_overlap, programmatic dependent launch): pdl = the
// kernel is launched as a programmatic dependent of the previous kernel on
// the stream and reads nothing another grid may write before
// griddepcontrol.wait; pdl_early = the previous kernel cannot have written
// this handle's state, so the state tiles are requested BEFORE the wait and
// stream in while that kernel drains.  Every kernel triggers its dependents
// (griddepcontrol.launch_dependents) once all its CTAs are running.
struct Ptrs {
    float *state;            // [R][Hv][d][d]
    void *K;                 // [R][Hk][T][d] in_dt
    void *U;                 // [R][Hv][T][d] u_dt
    float *G;                // [R][Hv][T]
    void *V;                 // [R][Hv][T][d] in_dt (keep_raw)
    float *B;                // [R][Hv][T]        (keep_raw)
    int *occ, *len, *mode, *ticket;
    unsigned *status;
    const int *sidx;         // [R] state index per slot, or nullptr (identity)
    const int *btab;         // [R][maxb] record block table, or nullptr (contiguous)
};

#ifdef __CUDACC__
// (block id, offset) of record position pos of slot r
__device__ __forceinline__ int2 rec_at(const Dims &dm, const Ptrs &p, int r, int pos) {
    if (!p.btab) return make_int2(r, pos);
    if (dm.bt_shift >= 0)   // (no integer division: the usual power-of-two block size)
        return make_int2(p.btab[(size_t)r * dm.maxb + (pos >> dm.bt_shift)], pos & (dm.bt - 1));
    return make_int2(p.btab[(size_t)r * dm.maxb + pos / dm.bt], pos % dm.bt);
}
#endif

// What the chunk-attend kernel does with the counters and the state.
enum ChunkKind : int {
    CK_DECODE = 0,   // state, append at occ, occ += n_new           (kernel 1)
    CK_VERIFY = 1,   // state, write drafts at occ.., occ unchanged  (kernel 3)
    CK_DIRECT = 2,   // no state, append at len, len += n_new        (kernel 4)
    CK_PREFILL = 3,  // state, append at occ, occ += n_new (then fold)
};

struct ChunkArgs {
    Dims dm;
    Ptrs p;
    int first, n;       // slot range
    int n_new;          // tokens processed per slot in this launch (<= kMaxNewPerLaunch)
    int j0_cap;         // max over the range of the buffered count j0 (sizes smem)
    int j_add;          // added to the device count (verify split into several launches)
    int j0_fixed = -1;  // >= 0: every slot of the (contiguous) range holds exactly this many
                        // records (host mirror exact): the kernel requests them at once
                        // instead of reading the device counter first
    int seg = 0;        // branch verify: new tokens form independent branches of `seg` tokens
                        // (causal and cumulative decay only within a branch); 0 = one sequence
    int tok_total;      // tokens per slot in the caller's q/k/v/alpha/beta/o arrays
    int tok_offset;     // first token of this launch inside those arrays
    int kind;
    const void *q, *k, *v;
    const float *alpha, *beta;
    float *o;           // may be null (prefill without outputs)
    const int *slots = nullptr;   // index-array batch: slot of CTA row zi (else first + zi)
    const int *pos = nullptr;     // ... and its row in the caller's inputs / outputs (else zi)
    int dry = 0;        // 1: check the launch configuration only, enqueue nothing
    int pdl = 0, pdl_early = 0;   // see Ptrs/launch overlap below
    int fold = 0;                 // decode: fold a slot's buffer in the step that fills it
    int pfold = 0;                // prefill chunk from an empty buffer (warp-MMA kinds): fold the chunk's
                                  // records into the state tile in the same kernel (no records written)
    const void *tmapk = nullptr;  // direct one-token step: host CUtensorMap of the bf16 key records as
                                  // [R*Hk*T][128] (16 x 64 boxes, 128 B swizzle) -- key rows on the tensor cores
    const void *tmap = nullptr;   // host CUtensorMap of the state as [R*Hv*128][128] fp32
                                  // (128 x 32 boxes, 128 B swizzle) for the tensor-core state pass
};

enum FoldKind : int {
    FK_FULL = 0,     // chunkwise slots with occ == C
    FK_FORCE = 1,    // chunkwise slots with occ > 0; direct slots: compress, S0 = 0
    FK_COMMIT = 2,   // chunkwise: n = occ + clamp(n_acc[r], 0, n_draft)
    FK_BRANCH = 4,   // commit of branch b: records [0, occ) + [occ + b n_draft, occ + b n_draft + n_acc)
    FK_FORK = 3,     // state of slot `dst` <- fold of slot r's first fork_n records (S0: r's state, or 0
                     // for a DIRECT slot); slot r and its counters untouched
};

struct FoldArgs {
    Dims dm;
    Ptrs p;
    int first, n;
    int kind;
    const int *nacc;    // FK_COMMIT
    int n_draft;
    int kcap;           // host bound on the records any slot of the launch folds
    int spec;           // host mirror: every slot of the range folds (issue the state copy at entry)
    int kc;             // staging chunk (set by launch_fold)
    int raw = 0;        // mode ii: recompute u from the raw records (keep_raw) by the UT transform
    int pdl = 0, pdl_early = 0;
    const int *slots = nullptr;   // index-array batch (else first + zi)
    int fork_n = 0, fork_dst = -1;  // FK_FORK
    const int *branch = nullptr;    // FK_BRANCH: accepted branch per slot
    int n_branch = 1;               // FK_BRANCH: branches of n_draft drafts
    const void *tmap = nullptr;     // raw (mode ii): host CUtensorMap of the state (see ChunkArgs::tmap)
};
cudaError_t launch_commit_append(const Dims &dm, const Ptrs &p, int first, int n, const int *nacc, int n_draft,
                                 int pdl, cudaStream_t s, int64_t *launches);

struct RecArgs {
    Dims dm;
    Ptrs p;
    int first, n;
    int n_draft;        // 1 for the decode step
    const void *q, *k, *v;
    const float *alpha, *beta;
    float *o;
    float *temp;        // recurrent verify: [n][n_draft][Hv][d][d]
    const int *nacc;    // recurrent commit
    int pdl = 0, pdl_early = 0;
};

// Launchers: return cudaSuccess or the launch error; *launches += kernels.
cudaError_t launch_chunk(const ChunkArgs &a, cudaStream_t s, int64_t *launches);
cudaError_t launch_fold(const FoldArgs &a, cudaStream_t s, int64_t *launches);
// mode ii (fold_ut.cu): one CTA of 8 warps per (V head, slot); FULL / FORCE only
cudaError_t launch_fold_ut(const FoldArgs &a, cudaStream_t s);
cudaError_t launch_recurrent_step(const RecArgs &a, cudaStream_t s, int64_t *launches);
cudaError_t launch_recurrent_verify(const RecArgs &a, cudaStream_t s, int64_t *launches);
cudaError_t launch_recurrent_commit(const RecArgs &a, cudaStream_t s, int64_t *launches);
// Writes dst[idx[i]] = val[i] for the staged host entries (block tables,
// state indices, work lists): small host decisions delivered in stream order
// as kernel parameters (no host buffer outlives the call; graph-capturable).
constexpr int kStageMax = 3000;
constexpr int kStageSmall = 256;   // the usual per-step update fits a 2 KiB parameter block
template <int CAP>
struct StageArgsT {
    int *dst;
    int n;
    int2 e[CAP];   // (index, value)
};
using StageArgs = StageArgsT<kStageMax>;
// n entries from e[] (n <= kStageMax); the smallest parameter block that holds them
cudaError_t launch_stage(int *dst, const int2 *e, int n, int pdl, cudaStream_t s, int64_t *launches);
cudaError_t launch_reset(const Dims &dm, const Ptrs &p, int first, int n, int mode, int zero_state,
                         cudaStream_t s, int64_t *launches);

}  // namespace labuf
