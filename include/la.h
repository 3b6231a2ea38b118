/*
 * la.h — C ABI of the KV-buffered Gated DeltaNet decode library (labuf).
 *
 * Implements the IO-aware serving mechanism of arxiv 2605.19049 for Gated
 * DeltaNet (GDN) linear attention on NVIDIA B200 (sm_100a).  Citations
 * "P:n" are lines of the paper text; "Eq. k" counts its numbered
 * display equations in order; "Zk" are the readings listed in DESIGN.md.
 *
 * ---------------------------------------------------------------- math
 * Per request slot r and V head h (QK head floor(h*Hk/Hv)), with column
 * vectors and the state S in R^{d_v x d_k} (the transpose of the paper's
 * row-vector S, reading Z1), the method reaches exactly (up to rounding) the
 * GDN recurrence:
 *     S_t = alpha_t S_{t-1} (I - beta_t k_t k_t^T) + beta_t v_t k_t^T,
 *     o_t = S_t q_t.
 * It keeps, per slot and head, a KV buffer of records (k_i, u_i, G_i), where
 *     u_i = beta_i (v_i - e^{G_i} S0 k_i - sum_{l<i} e^{G_i-G_l} (k_i.k_l) u_l)
 * is the delta value and G_i the cumulative log decay
 * since the last fold (reading Z2).  Outputs are computed from one read of
 * S0 plus the buffer, and the buffer is folded into the state in
 * batch:  S <- e^{G_last} S0 + sum_i e^{G_last - G_i} u_i k_i^T.
 *
 * ---------------------------------------------------------------- layout
 * Device memory is caller-owned (allocate it with torch.empty or cudaMalloc;
 * sizes from la_buf_query).  All pointers are DEVICE pointers unless noted.
 *   state   fp32 [S][Hv][d_v][d_k]   (d_k contiguous; 64 KiB per (state,head));
 *           S = R (state of slot r at index r) or, with a state pool
 *           (state_slots > 0), S = state_slots states assigned to slots on
 *           demand (state_slots = -1: no states, a KV-only handle)
 *   buffer  the record blocks, at offsets reported by la_buf_query:
 *           K [nb][Hk][bt][d_k] in_dtype, U [nb][Hv][d_v/32][bt][32] u_dtype,
 *           G [nb][Hv][bt] fp32, and when keep_raw: V [nb][Hv][bt][d_v]
 *           in_dtype, B [nb][Hv][bt] fp32.  Contiguous handles
 *           (block_tokens = 0): nb = R, bt = T = max(chunk + max_drafts,
 *           short_cap) rounded up to 4, block r = slot r's records.  Paged
 *           handles (block_tokens > 0): nb = n_blocks blocks of
 *           bt = block_tokens records from one pool; a slot holds the blocks
 *           its records need (position p -> its block p / bt, offset p % bt),
 *           allocated by the library on append and returned on reset/release
 *   meta    int32 occ[R], len[R], mode[R], ticket[R], uint32 status, then
 *           (at the offsets in la_sizes) the state index per slot, the block
 *           table [R][max_blocks] and the work lists of index-array batches.
 *           Must be zero-filled before la_buf_create.
 * Per-call tensors (row-major, batch = contiguous slot range [first, first+n)):
 *   q, k  [n][n_tok][Hk][d_k] in_dtype;  v [n][n_tok][Hv][d_v] in_dtype;
 *   alpha, beta fp32 [n][n_tok][Hv];   o fp32 [n][n_tok][Hv][d_v]
 *   (n_tok = 1 for decode / recurrent step, n_draft for verify, n_new for
 *   direct, n_tok for prefill).  Inputs must be 16-byte aligned.
 *
 * ---------------------------------------------------------------- contract
 * Streams: every call enqueues asynchronously on `stream` (a cudaStream_t;
 *   NULL = legacy default stream) and never synchronises, except
 *   la_device_status.  Calls on one handle must be stream-ordered and issued
 *   from one host thread at a time.
 * Errors: every function returns la_status.  On any return other than LA_OK
 *   nothing was enqueued and the host occupancy mirror is unchanged
 *   (all-or-nothing; every launch configuration of a call is checked before
 *   the first kernel is enqueued); la_last_error() returns a thread-local
 *   message.  The one exception is LA_ERR_CUDA from a launch that the driver
 *   rejects after earlier kernels of the same call were enqueued (e.g. a
 *   sticky error from an earlier fault): the slots of the call are then in
 *   an undefined state and must be reset with la_request_reset.
 * Batches of more than 4096 slots are split into several launches (the slot
 *   index is a grid dimension).
 * Occupancy: the library keeps an exact host mirror of occ/len/mode per slot;
 *   it advances deterministically (decode +1, flush/commit -> 0, direct +n_new,
 *   prefill -> 0) and never needs device values.  Device copies in `meta`
 *   are what the kernels read, so whole cycles can be captured in CUDA graphs;
 *   a replayed graph must cover closed cycles (the mirror does not see
 *   replays).
 * Determinism: identical inputs give bit-identical outputs (no float atomics).
 * Pools: block and state allocation is a host
 *   decision (LIFO free lists over ascending ids, so the same call sequence
 *   gives the same ids); the block table and state indices are delivered to
 *   the device in stream order by a small staging kernel whose entries travel
 *   as kernel parameters.  Pool exhaustion is LA_ERR_CAPACITY before anything
 *   is enqueued.  Invariants: free + held = pool size (blocks and states); a
 *   block or state is held by at most one slot.
 */
#ifndef LABUF_LA_H
#define LABUF_LA_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define LA_API __attribute__((visibility("default")))
#else
#define LA_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct la_buf la_buf;   /* opaque host handle; owns NO device memory */
typedef void *la_stream;        /* cudaStream_t */

typedef enum {
    LA_OK = 0,
    LA_ERR_INVALID = 1,      /* null/misaligned pointer, bad range or count   */
    LA_ERR_UNSUPPORTED = 2,  /* d != 128, Hv % Hk != 0, unsupported dtype mix  */
    LA_ERR_CAPACITY = 3,     /* buffer would overflow (forgot la_flush, ...)   */
    LA_ERR_MODE = 4,         /* wrong slot mode / pending verify / no verify   */
    LA_ERR_CUDA = 5,         /* CUDA launch or runtime error                  */
    LA_ERR_NCCL = 6          /* NCCL error (tensor-parallel helpers)          */
} la_status;

typedef enum { LA_DT_F32 = 0, LA_DT_BF16 = 1, LA_DT_F16 = 2 } la_dtype;
/* Linear-attention variant of a handle (Table 1):
 *   GDN     S_t = alpha_t S_{t-1} (I - beta_t k_t k_t^T) + beta_t v_t k_t^T
 *   GATED   S_t = alpha_t S_{t-1} + v_t k_t^T   (scalar-gated LA, no delta rule;
 *           beta ignored)
 *   VANILLA S_t = S_{t-1} + v_t k_t^T           (alpha, beta ignored)
 * The buffered value is u_t = v_t for the two delta-free variants; every
 * kernel, the fold and the recurrent baselines honour the variant. */
typedef enum { LA_VARIANT_GDN = 0, LA_VARIANT_GATED = 1, LA_VARIANT_VANILLA = 2 } la_variant;
typedef enum { LA_MODE_CHUNKWISE = 0, LA_MODE_DIRECT = 1 } la_mode;
typedef enum {
    LA_FLUSH_FULL = 0,   /* fold only slots whose buffer holds `chunk` records */
    LA_FLUSH_FORCE = 1,  /* fold every non-empty slot; a DIRECT slot is compressed
                            into a fresh state and switches to CHUNKWISE */
    LA_FLUSH_RAW = 2     /* flag, OR-ed into FULL/FORCE: mode ii.  The delta values
                            are recomputed from the raw records (k, v, beta, G) and
                            S0 by the UT transform -- W = K S0^T, the n x n forward
                            substitution T = [I + strictLower(Diag(beta)(Gamma (.)
                            K K^T))]^{-1}, U = T Diag(beta)(V - Diag(e^G) W)
                            (K~ as corrected by reading Z4) -- then
                            folded as in mode i.  Needs keep_raw = 1, else
                            LA_ERR_INVALID. */
} la_flush_kind;

/* Device status bits (la_device_status), set only when config.validate = 1. */
#define LA_STATUS_BAD_ALPHA   0x1u  /* alpha not in (0, 1]  (reading Z9)      */
#define LA_STATUS_BAD_BETA    0x2u  /* beta not in [0, 1]                      */
#define LA_STATUS_NONFINITE   0x4u  /* non-finite q/k/v                         */
#define LA_STATUS_BAD_NACC    0x8u  /* n_accepted outside [0, n_draft] (clamped) */

typedef struct {
    int32_t max_slots;   /* R >= 1                                            */
    int32_t n_qk_heads;  /* Hk >= 1                                           */
    int32_t n_v_heads;   /* Hv, Hv % Hk == 0, Hv/Hk in {1,2,4}                */
    int32_t d_k, d_v;    /* must be 128                               */
    int32_t chunk;       /* buffer size C in [1, 64] (best near 2 sqrt d) */
    int32_t max_drafts;  /* N_max in [0, 16]                                  */
    int32_t short_cap;   /* direct-mode capacity in [0, 128] (<= d)     */
    int32_t in_dtype;    /* la_dtype of q,k,v: LA_DT_BF16 or LA_DT_F32        */
    int32_t u_dtype;     /* la_dtype of buffered u: F32, or F16 with BF16 in  */
    int32_t keep_raw;    /* 1: also store v and beta per record               */
    int32_t validate;    /* 1: device-side value checks -> status word        */
    int32_t block_tokens;/* 0: contiguous per-slot records; else paged record
                            blocks of this many tokens, a multiple of 4 in
                            [4, 128] (the paper: 8 or 16; = C or N,
                            P:224)                                          */
    int32_t n_blocks;    /* paged: blocks in the pool (>= 1); else ignored    */
    int32_t state_slots; /* 0: one state per slot; > 0: a pool of that many
                            states, assigned on demand; -1: no states          */
    int32_t variant;     /* la_variant (0 = GDN)                              */
} la_config;

typedef struct {
    size_t state_bytes;  /* fp32 [R][Hv][d_v][d_k]                            */
    size_t buffer_bytes; /* K, U, G [, V, B] records                          */
    size_t meta_bytes;   /* int32 occ, len, mode, ticket [R] + uint32 status  */
    size_t align;        /* required base alignment of all three (1024)       */
    int32_t capacity;    /* T, records per (slot, head)                       */
    size_t off_k, off_u, off_g, off_v, off_b;   /* offsets inside `buffer`    */
    size_t record_bytes; /* bytes per record per slot-layer (all heads)       */
    int32_t block_tokens;/* bt: records per block (T when contiguous)         */
    int32_t n_blocks;    /* nb: blocks in the buffer (R when contiguous)      */
    int32_t max_blocks;  /* blocks a slot can hold: ceil(T / bt)              */
    int32_t n_states;    /* states in `state`                                 */
    size_t off_sidx, off_btab, off_wl;   /* byte offsets inside `meta`        */
} la_sizes;

/* Sizing query; no device access.  LA_ERR_INVALID/UNSUPPORTED on bad config. */
LA_API la_status la_buf_query(const la_config *cfg, la_sizes *out);

/* Create a handle over caller-owned device memory.  `state`, `buffer`, `meta`
 * must be `align`-aligned device pointers of at least the queried sizes and
 * outlive the handle.  Does not initialise device memory: call
 * la_request_reset on every slot before use.  `device` is the CUDA ordinal. */
LA_API la_status la_buf_create(const la_config *cfg, void *state, void *buffer, void *meta,
                        int32_t device, la_buf **out);
LA_API la_status la_buf_destroy(la_buf *buf);   /* frees host memory only */

/* Reset slots [first, first+n): occ = len = 0, mode as given, and (if
 * zero_state) the state set to 0.  Clears a pending verify.  Paged handles:
 * the slots' record blocks return to the pool.  State pool: a CHUNKWISE slot
 * keeps or receives a state (LA_ERR_CAPACITY if the pool is empty), a DIRECT
 * slot returns its state. */
LA_API la_status la_request_reset(la_buf *buf, int32_t first, int32_t n, int32_t mode,
                           int32_t zero_state, la_stream stream);

/* Release slots [first, first+n) (request finished): their record blocks and
 * state return to the pools; the slots become empty DIRECT slots (len 0)
 * that hold nothing.  Enqueues nothing unless the slots held something. */
LA_API la_status la_request_release(la_buf *buf, int32_t first, int32_t n, la_stream stream);

/* Mixed-form decode step over an index-array batch (SURVEY
 * NEXT-3): slots[i] (HOST int32 [n], distinct) receives the token at row i
 * of q, k, v [n][Hk|Hv][d], alpha, beta [n][Hv]; o[i] [Hv][d_v] gets its
 * output.  Each slot decodes in its current form:
 *   CHUNKWISE: buffered decode (kernel 1); a buffer it fills is folded at the
 *              end of the call (kernel 2, eager flush, reading Z15);
 *   DIRECT with len < short_cap: KV-only decode (kernel 4);
 *   DIRECT with len == short_cap: first compressed into a state (fold with
 *              S0 = 0: "once the context length L >= d ... compress"),
 *              then decoded as CHUNKWISE.
 * Blocks and states are taken from the pools as needed (LA_ERR_CAPACITY,
 * all-or-nothing, if they run out).  Requires no pending verify and, for
 * CHUNKWISE slots, occ < chunk. */
LA_API la_status la_decode_mixed(la_buf *buf, int32_t n, const int32_t *slots, const void *q,
                          const void *k, const void *v, const float *alpha, const float *beta,
                          float *o, la_stream stream);

/* Pool occupancy (host mirror, no device access): free / total blocks and
 * states, and the blocks slot `slot` holds (slot < 0: skip). */
LA_API la_status la_pool_info(la_buf *buf, int32_t *free_blocks, int32_t *total_blocks,
                       int32_t *free_states, int32_t *total_states, int32_t slot,
                       int32_t *slot_blocks, int32_t *slot_state);

/* Buffered decode step, kernel (1).  For each slot in the
 * range (CHUNKWISE, occ < chunk, no pending verify): computes u_t and
 * o_t = e^{G_t} S0 q_t + sum_i e^{G_t-G_i} (q_t.k_i) u_i + (q_t.k_t) u_t from
 * one read of the state, appends (k_t, u_t, G_t) at position occ, occ += 1.
 * Does not fold: call la_flush(LA_FLUSH_FULL) after the step that fills the
 * buffer.  LA_ERR_CAPACITY if some slot has occ == chunk. */
LA_API la_status la_decode_step(la_buf *buf, int32_t first, int32_t n, const void *q,
                         const void *k, const void *v, const float *alpha,
                         const float *beta, float *o, la_stream stream);

/* Flush, kernel (2): S <- e^{G_last} S0 +
 * sum_{i<occ} e^{G_last-G_i} u_i k_i^T on the 5th-gen tensor cores
 * (tcgen05, split-TF32, accumulator in TMEM), occ <- 0.  kind may carry
 * LA_FLUSH_RAW (mode ii: u recomputed by the UT transform).  FULL folds slots
 * with occ == chunk, FORCE every non-empty slot (DIRECT slots: compression
 * with S0 = 0, mode -> CHUNKWISE).  A range with nothing to fold is a no-op
 * (not an error). */
LA_API la_status la_flush(la_buf *buf, int32_t first, int32_t n, int32_t kind, la_stream stream);

/* Parallel draft verification, kernel (3): outputs of
 * n_draft drafts per slot from one read of the state, the buffered records
 * and the drafts themselves (n_draft x n_draft forward substitution).  Draft
 * records are written at positions occ .. occ+n_draft-1 but occ does not move
 * and no temporary state exists.  Requires 1 <= n_draft <= max_drafts,
 * occ + n_draft <= T, no pending verify.  Marks the range pending. */
LA_API la_status la_verify_drafts(la_buf *buf, int32_t first, int32_t n, int32_t n_draft,
                           const void *q, const void *k, const void *v,
                           const float *alpha, const float *beta, float *o,
                           la_stream stream);

/* Accepted-prefix commit (Eq. 8): folds records
 * [0, occ + n_accepted[r]) into the state (kernel (2)), occ <- 0.
 * n_accepted: DEVICE int32 [n], clamped to [0, n_draft] (status bit when
 * validate=1).  occ + n_accepted = 0 leaves the state bit-identical.
 * LA_ERR_MODE unless every slot in the range has a pending verify of the
 * same n_draft. */
LA_API la_status la_commit_accepted(la_buf *buf, int32_t first, int32_t n,
                             const int32_t *n_accepted, la_stream stream);

/* Branch (beam) candidates: n_branch candidate
 * branches of n_draft tokens each, all extending the slot's current buffer,
 * verified in one launch: inputs [n][n_branch * n_draft][...] branch-major;
 * token p of branch b sees the state, the buffered records and tokens
 * 0..p of its own branch only (the decay restarts per branch).  Records are
 * written at occ + b * n_draft + p; nothing is folded and no per-branch state
 * exists.  n_branch * n_draft <= min(max_drafts, 16). */
LA_API la_status la_verify_branches(la_buf *buf, int32_t first, int32_t n, int32_t n_branch,
                             int32_t n_draft, const void *q, const void *k, const void *v,
                             const float *alpha, const float *beta, float *o, la_stream stream);

/* Commit of the accepted branch: folds records [0, occ) and the first
 * n_accepted[r] records of branch branch[r] (DEVICE int32 [n] each, clamped;
 * status bit with validate = 1) into the state; occ <- 0.  LA_ERR_MODE unless
 * the range has a pending branch verify of one shape. */
LA_API la_status la_commit_branch(la_buf *buf, int32_t first, int32_t n, const int32_t *branch,
                           const int32_t *n_accepted, la_stream stream);

/* Multi-round buffered speculation: commit the accepted
 * prefix by APPENDING it -- the accepted drafts' records (k, u, G) are
 * already the recurrence's records (u_t depends only on tokens <= t),
 * so the device occupancy advances by n_accepted[r] and nothing is folded.
 * The state is folded only when the buffer could not take another round of
 * max_drafts drafts (then exactly as la_commit_accepted: records
 * [0, occ + n_accepted)).  The host mirror then holds an upper bound of the
 * occupancy (it never reads n_accepted): until a fold, the slots accept only
 * la_verify_drafts, commits and la_flush(FORCE) (LA_ERR_MODE otherwise).
 * Same argument rules as la_commit_accepted. */
LA_API la_status la_commit_append(la_buf *buf, int32_t first, int32_t n,
                           const int32_t *n_accepted, la_stream stream);

/* State rebuild / fork for KV-based prefix caching: the state of
 * slot `dst` becomes the state slot `src` had after its first n_records
 * buffered records: e^{G_{n-1}} S0 + sum_{i<n} e^{G_{n-1}-G_i} u_i k_i^T with
 * S0 = src's state (CHUNKWISE src) or 0 (DIRECT src: the state rebuilt from
 * the cached KVs alone).  src is not modified; dst must be a
 * CHUNKWISE slot with an empty buffer (e.g. just reset), dst != src,
 * 1 <= n_records <= src's buffered count. */
LA_API la_status la_state_fork(la_buf *buf, int32_t src, int32_t dst, int32_t n_records,
                        la_stream stream);

/* Direct (KV-only) short-context decoding, kernel (4) (P:200-213,
 * P:374-378): for DIRECT slots, outputs of n_new new tokens computed only
 * from the buffered records of the whole context and the new tokens
 * (n_new x n_new forward substitution); no state is read or written.
 * Appends the records, len += n_new.  n_new = 1 is a decode step, n_new = P
 * a short prefill.  LA_ERR_CAPACITY if len + n_new > short_cap. */
LA_API la_status la_direct_short(la_buf *buf, int32_t first, int32_t n, int32_t n_new,
                          const void *q, const void *k, const void *v,
                          const float *alpha, const float *beta, float *o,
                          la_stream stream);

/* Chunkwise prefill: folds a prompt of n_tok tokens into
 * the state of CHUNKWISE slots with occ == 0, in chunks of P tokens (the
 * handle's chunk, or la_set_prefill_chunk): each chunk runs the
 * forward-substitution kernel (the UT transform of P:395-397, state mat-vecs
 * on the tensor cores, 16 tokens per launch) and the tensor-core fold
 * (P:407).  o may be NULL; otherwise it receives the prompt outputs
 * [n][n_tok][Hv][d_v].  Leaves occ = 0. */
LA_API la_status la_prefill(la_buf *buf, int32_t first, int32_t n, int32_t n_tok,
                     const void *q, const void *k, const void *v,
                     const float *alpha, const float *beta, float *o,
                     la_stream stream);

/* Conventional recurrent decode, kernel (5a) (Table 2):
 * reads and writes the whole state every token.  In-run IO baseline.
 * Requires CHUNKWISE slots with occ == 0. */
LA_API la_status la_recurrent_step(la_buf *buf, int32_t first, int32_t n, const void *q,
                            const void *k, const void *v, const float *alpha,
                            const float *beta, float *o, la_stream stream);

/* Conventional recurrent speculative verification, kernel (5b) (P:94,
 * P:183): reads S once, takes n_draft sequential steps and writes one
 * temporary state per draft: temp fp32 [n][n_draft][Hv][d_v][d_k]. */
LA_API la_status la_recurrent_verify(la_buf *buf, int32_t first, int32_t n, int32_t n_draft,
                              const void *q, const void *k, const void *v,
                              const float *alpha, const float *beta, float *temp,
                              float *o, la_stream stream);

/* Baseline commit: the slot's state is replaced by the temporary state of the
 * last accepted draft (Fig. 3); n_accepted = 0 leaves it unchanged.
 * Requires CHUNKWISE slots with an empty buffer and no pending verify. */
LA_API la_status la_recurrent_commit(la_buf *buf, int32_t first, int32_t n, int32_t n_draft,
                              const int32_t *n_accepted, const float *temp,
                              la_stream stream);

/* Launch overlap (programmatic dependent launch, B200 griddepcontrol): with
 * enable = 1 every kernel of this handle is launched as a programmatic
 * dependent of the previous kernel on the stream, so its CTAs start while
 * that kernel drains; when the previous kernel cannot have written this
 * handle's state (the library tracks its own launches: a fold, reset,
 * recurrent step/commit or la_state_set of the same handle on the same
 * stream disables it), the state tiles are requested before
 * griddepcontrol.wait and stream in during that drain.  Inputs, counters,
 * records and outputs are always accessed after the wait.
 * Contract when enabled: a kernel that is NOT a la_* call and writes this
 * handle's state must not be the kernel enqueued immediately before a la_*
 * call of the handle on the same stream (put an event/sync or any la_* call
 * in between).  Default 0 (off).  LA_ERR_INVALID on enable not 0/1. */
LA_API la_status la_set_overlap(la_buf *buf, int32_t enable);

/* Prefill chunk length P of la_prefill: 0 = the handle's chunk (default),
 * else 1 <= P <= min(64, T).  LA_ERR_INVALID otherwise. */
LA_API la_status la_set_prefill_chunk(la_buf *buf, int32_t tokens);

/* Fused flush: with enable = 1 and
 * chunk <= 32, a la_decode_step that fills a slot's buffer (occ reaches
 * chunk) folds the slot's `chunk` records into its state inside the decode
 * kernel -- S <- e^{G_last} S0 + sum_i e^{G_last-G_i} u_i k_i^T on CUDA cores
 * (fp32), from the S0 rows the step has already read -- and leaves occ = 0;
 * the separate flush and its second read of the state disappear.  A
 * la_flush(FULL) after such a step is an empty no-op.  Outputs are those of
 * the unfused path (same buffered u, fold within fp32 rounding).  Default 0.
 * LA_ERR_INVALID on enable not 0/1. */
LA_API la_status la_set_auto_flush(la_buf *buf, int32_t enable);

/* Canonical state export/import of one slot: fp32 [Hv][d_v][d_k], device
 * pointers, async on `stream`.  la_state_set requires a CHUNKWISE slot with
 * an empty buffer and no pending verify (the buffered records were computed
 * against the old state), else LA_ERR_MODE. */
LA_API la_status la_state_get(la_buf *buf, int32_t slot, float *dst, la_stream stream);
LA_API la_status la_state_set(la_buf *buf, int32_t slot, const float *src, la_stream stream);

/* Host mirror of one slot (no device access). */
LA_API la_status la_slot_info(la_buf *buf, int32_t slot, int32_t *occ, int32_t *len,
                       int32_t *mode, int32_t *pending_drafts);

/* Synchronises `stream`, returns the device status word in *flags, and
 * copies the device occ/len/mode of all slots into the optional host arrays
 * (each int32[R], may be NULL). */
LA_API la_status la_device_status(la_buf *buf, la_stream stream, uint32_t *flags,
                           int32_t *occ_host, int32_t *len_host, int32_t *mode_host);

/* Number of kernels this handle has launched since creation (all la_* calls). */
LA_API int64_t la_kernel_launches(const la_buf *buf);

/* Thread-local message of the last non-LA_OK return on this thread. */
LA_API const char *la_last_error(void);

/* ----------------------------------------------- tensor-parallel helpers
 * Heads are partitioned over ranks (each handle created with Hk/G, Hv/G);
 * head outputs are gathered with one NCCL all-gather per layer (DESIGN.md
 * "Multi-GPU").  The only collective in the library. */
LA_API la_status la_tp_unique_id(void *id_out /* 128 bytes, host */);
LA_API la_status la_tp_init(const void *unique_id /* 128 bytes, host */, int32_t rank,
                     int32_t world, int32_t device, void **comm_out);
LA_API la_status la_tp_allgather(void *comm, const void *send, void *recv,
                          size_t bytes_per_rank, la_stream stream);
LA_API la_status la_tp_destroy(void *comm);

#ifdef __cplusplus
}
#endif
#endif /* LABUF_LA_H */
