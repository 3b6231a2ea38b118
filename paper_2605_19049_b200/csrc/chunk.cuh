// chunk.cu — kernels (1) buffered decode, (3) parallel draft verification,
// (4) direct short-context decoding, and the prefill chunk step.
//
// All compute, for n_new new tokens t of one request slot r and one V head
// (QK head = h / g), against j0 buffered records (k_i, u_i, G_i):
//
//   G_t = G_{t-1} + ln alpha_t                  (cumulative log decay, reading Z2)
//   a_t = S0 k_t,  b_t = S0 q_t                 (one read of the state tile; absent for direct)
//   u_t = beta_t (v_t - e^{G_t} a_t - sum_{i<j0+t} e^{G_t-G_i} (k_t.k_i) u_i)
//   o_t = e^{G_t} b_t + sum_{i<=j0+t} e^{G_t-G_i} (q_t.k_i) u_i
//
// which is the single-token chunkwise form P:403-406 (decode, subscripts per
// readings Z2/Z3), the chunkwise matrix form P:392-399 solved by forward
// substitution over the new tokens (verify, prefill: the UT transform of
// P:395-397), and the parallel form P:374-386 with S0 = 0 (direct).
// New records (k_t, u_t, G_t) are appended at position j0 + t.
//
// B200 structure (measured, tools/microbench_bulk.cu): HBM is saturated by
// many small CTAs that each put their whole working set in flight with a
// few bulk copies (cp.async.bulk -> SASS UBLKCP) on one mbarrier — 7.4 TB/s
// even with 1 KB pieces — while a single issuing thread per SM cannot issue
// small copies fast enough.  So: one CTA of TPC warps per (row-tile group,
// V head, slot).  At entry its warps issue the copies — the TPC x 32 rows
// of fp32 state of the head (ONE contiguous copy, 16 KiB per tile), the
// tiles' u sub-tiles of all buffered records (contiguous by the tile-major U
// layout), the QK head's key rows, the log decays and the new tokens — and
// several CTAs per SM overlap one CTA's compute with the others' loads.
// Compute: warp w owns d_v tile w (32 rows).  (A) Every state row and every
// key row is reduced against k_t and q_t by 4-lane teams (8 rows per warp
// step; each lane owns eight parity-swizzled 16-byte column chunks, so the
// shared-memory reads are conflict-free; packed FFMA2 dot products; 2 shuffle
// levels per value); the key rows are shared out over the CTA's warps.  One block
// barrier.  (B) The forward substitution over the new tokens with one lane
// per d_v row, and the o / u / record stores.
#pragma once
#include <cuda.h>

#include <cstdlib>

#include "device.cuh"
#include "internal.h"

namespace labuf {

constexpr int kChunkTPC = 2;        // d_v tiles (warps) per CTA for the state kinds
constexpr int kMmaWPT = 1;  // (must be 1: the substitution lane of a row holds its MMA results)          // warps per d_v tile for the multi-token (warp-MMA) kinds (2: measured
                                    // slower for verify: N = 4 163 -> 176 us, N = 8 265 -> 293 us)
constexpr int kDirectTPC = 4;       // ... and for direct slots (the key rows dominate)

__host__ __device__ inline uint32_t al128(uint32_t x) { return (x + 127u) & ~127u; }
// row length of the record-major coefficient arrays Ck / Cq
__host__ __device__ constexpr int ntp(int nt) { return nt == 1 ? 1 : (nt + 3) / 4 * 4; }

struct CtaLayout {
    uint32_t S, U, K, Gs, q, k, v, kq32, Ck, Cq, av, bv, Gn, Bn, Y, Kf, Bm, Ap, Kp, bar, bytes;
};

// fused fold (decode with auto-flush): A operand U~ [row][record], rows of
// kAuS floats (conflict-free ldmatrix; records <= kFusedFoldMaxC = 32)
constexpr int kAuS = 36;
// warp-MMA state pass: B operand rows (k_t, q_t of the new tokens, zero padded
// to whole n8 tiles), row stride padded to 132 floats (conflict-free
// fragment reads); fp32 tokens keep a hi and a lo copy
constexpr int kBmStride = 132;
constexpr int kKp = 136;   // bf16 row stride of the key-rows MMA operands (272 B)
__host__ __device__ constexpr int mma_nrows(int nt) { return (2 * nt + 7) / 8 * 8; }

// tensor-core state pass: B operand rows (k_t, q_t of every new token, zero
// padded to the MMA N granule of 16 at M = 128)
__host__ __device__ constexpr int tc_nmma(int nt) { return (2 * nt + 15) / 16 * 16; }

__host__ __device__ inline CtaLayout cta_layout(int TPC, int nt, bool has_state, int jcap, int isz, int usz,
                                                bool tc = false, bool fold = false, bool mma = false, int minb = 1) {
    CtaLayout L;
    const int J = jcap + nt;
    uint32_t o = 0;
    // (tc / mma: 1 KiB of slack so the 128-byte-swizzled state tile starts 1024-aligned)
    // (tc: 1 KiB of slack for the 1024-aligned swizzled tile; the MMA kinds rely
    // on the dynamic shared memory base being 1024-aligned -- measured on B200,
    // tools/probe_smem_align.cu -- and trap otherwise)
    L.S = o;  o = al128(o + (has_state ? (uint32_t)(TPC * 32 * kD * 4) + (tc ? 1024u : 0u) : 0u));
    L.U = o;  o = al128(o + (uint32_t)(TPC * 32 * jcap * usz));
    // (direct one-token step: the key rows arrive by 2-D TMA, 16-record boxes of
    //  64 bf16 columns with the 128-byte swizzle -- 1 KiB aligned, whole boxes)
    const bool ktma_ = !has_state && nt == 1 && isz == 2 && !mma && !tc;
    if (ktma_) o = (o + 1023u) & ~1023u;
    L.K = o;  o = al128(o + (uint32_t)((ktma_ ? (jcap + 15) / 16 * 16 : jcap) * kD * isz));
    L.Gs = o; o = al128(o + (uint32_t)(((jcap + 3) & ~3) * 4));
    // (key-rows MMA kinds: q_t, k_t land straight in the padded rows Ap)
    const bool krm_ = mma && isz == 2;
    L.q = o;  o = al128(o + (krm_ ? 0u : (uint32_t)(nt * kD * isz)));
    L.k = o;  o = al128(o + (krm_ ? 0u : (uint32_t)(nt * kD * isz)));
    L.v = o;  o = al128(o + (uint32_t)(nt * TPC * 32 * isz));
    // fp32 k_t, q_t: the kinds that do not keep them in registers (KQ_REG)
    const bool kq_reg = nt == 1 && (has_state || minb < 5);
    L.kq32 = o; o = al128(o + (!kq_reg && isz == 2 && !mma ? (uint32_t)(nt * 2 * kD * 4) : 0u));
    // Ck / Cq are record-major [i][t] (rows of ntp(nt) floats): the records sum
    // reads all tokens' coefficients of a record with 16-byte loads
    L.Ck = o; o = al128(o + (uint32_t)(ntp(nt) * J * 4));
    L.Cq = o; o = al128(o + (uint32_t)(ntp(nt) * J * 4));
    // (the MMA kinds keep S0 k_t, S0 q_t in registers and shuffle them to the rows)
    // (self-folding prefill chunks of 8+ tokens stash S0 k_t, S0 q_t here once
    //  instead of shuffling them to the substitution lanes per token; measured:
    //  prefill 7.55 -> 7.39 ms, but verify N = 8 149.5 -> 201.6 us from the
    //  extra shared memory, so not for verify)
    const bool stash_ = has_state && mma && fold && nt >= 8;
    L.av = o; o = al128(o + (uint32_t)(has_state && (!mma || stash_) ? TPC * nt * 32 * 4 : 0));
    L.bv = o; o = al128(o + (uint32_t)(has_state && (!mma || stash_) ? TPC * nt * 32 * 4 : 0));
    L.Gn = o; o = al128(o + (uint32_t)(nt * 4));
    L.Bn = o; o = al128(o + (uint32_t)(nt * 4));
    L.Y = o;  o = al128(o + (tc ? (uint32_t)(tc_nmma(nt) * kD * 4 * (isz == 4 ? 2 : 1)) : 0u));
    L.Kf = o;   // (unused: the fused fold builds its operand in registers)
    // (fp32 tokens only: bf16 tokens feed the state pass from the bf16 rows Ap)
    L.Bm = o; o = al128(o + (mma && isz == 4 ? (uint32_t)(mma_nrows(nt) * kBmStride * 4 * 2) : 0u));
    // key rows on the tensor cores (bf16 inputs): the 2 nt vectors and the J
    // keys as bf16 rows padded to 272 B (conflict-free ldmatrix)
    const bool krm = mma && isz == 2;
    L.Ap = o; o = al128(o + (krm ? (uint32_t)(2 * nt * kKp * 2) : 0u));   // (fragment rows past 2 nt clamp)
    L.Kp = o; o = al128(o + (krm ? (uint32_t)(jcap * kKp * 2) : 0u));   // the buffered records' keys
    L.bar = o; o += 64;
    L.bytes = al128(o);
    return L;
}

// ---------------------------------------------------------------- row loads
// A 4-lane team reduces one 128-wide row.  Lane `seg` (0..3) owns the eight
// 16-byte column chunks ch(c) = seg + 4 (c ^ p), c < 8, where p is the row
// parity of its team: the two rows read in one 128-bit shared-memory phase
// (8 lanes) then touch 8 distinct bank groups.  k_t / q_t chunks are held in
// registers in the same per-lane order, so the pairing is static.
__device__ __forceinline__ int chunk_of(int seg, int p, int c) { return seg + 4 * (c ^ p); }

template <typename T>
__device__ __forceinline__ void load_row8(const T *row, int seg, int p, float4 (&x)[8]) {
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = load4(row + 4 * chunk_of(seg, p, c));
}

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d)
        : "l"(*reinterpret_cast<uint64_t *>(&a)), "l"(*reinterpret_cast<uint64_t *>(&b)),
          "l"(*reinterpret_cast<uint64_t *>(&c)));
    return *reinterpret_cast<float2 *>(&d);
}
// sum_c x[c] . y[c] as two packed fp32 accumulators (SASS FFMA2)
__device__ __forceinline__ float dot8x4(const float4 (&x)[8], const float4 (&y)[8]) {
    float2 a0 = make_float2(0.f, 0.f), a1 = make_float2(0.f, 0.f);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        a0 = ffma2(make_float2(x[c].x, x[c].y), make_float2(y[c].x, y[c].y), a0);
        a1 = ffma2(make_float2(x[c].z, x[c].w), make_float2(y[c].z, y[c].w), a1);
    }
    return (a0.x + a0.y) + (a1.x + a1.y);
}

// Sum V values over the 4 lanes of a team (xor 1, 2).  V < 4: every lane gets
// every sum, returned for value index x = seg (lanes seg >= V get -1).
// V >= 4: transposed butterfly, lane seg ends with the V/4 sums of value
// indices x = i + (V/4) seg.
template <int V>
struct TeamOut {
    static constexpr int N = V >= 4 ? V / 4 : 1;
};
template <int V>
__device__ __forceinline__ void team_reduce(float (&v)[V], int seg, float (&res)[TeamOut<V>::N],
                                            int (&xid)[TeamOut<V>::N]) {
    if constexpr (V < 4) {
#pragma unroll
        for (int j = 0; j < V; ++j) {
            float x = v[j];
            x += __shfl_xor_sync(0xffffffffu, x, 1);
            x += __shfl_xor_sync(0xffffffffu, x, 2);
            v[j] = x;
        }
        float r = v[0];
#pragma unroll
        for (int j = 1; j < V; ++j)
            if (seg == j) r = v[j];
        res[0] = r;
        xid[0] = seg < V ? seg : -1;
    } else {
        int n = V;
#pragma unroll
        for (int s = 2; s >= 1; s >>= 1) {
            const bool upper = (seg & s) != 0;
            const int h = n / 2;
#pragma unroll
            for (int i = 0; i < V / 2; ++i) {
                if (i < h) {
                    const float send = upper ? v[i] : v[i + h];
                    const float keep = upper ? v[i + h] : v[i];
                    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
                }
            }
            n = h;
        }
#pragma unroll
        for (int i = 0; i < V / 4; ++i) {
            res[i] = v[i];
            xid[i] = i + (V / 4) * seg;
        }
    }
}

// TC (multi-token kinds with a state): the state mat-vecs a_t = S0 k_t,
// b_t = S0 q_t of all new tokens are ONE M = 128 (d_v rows) x N (k_t, q_t
// columns) x K = 128 contraction on the tensor cores: the state tile arrives
// by 2-D TMA in the 128-byte-swizzled K-major layout the MMA reads, the
// tokens are staged K-major, and fp32 accuracy comes from split TF32 (the
// MMA reads the top 19 bits; pass 2 multiplies the exact remainder
// S0 - trunc(S0), written in place once pass 1 has read the tile; fp32
// tokens add a pass with their own remainder).
__device__ __forceinline__ float trunc_tf32(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

// FOLD (decode with auto-flush, la_set_auto_flush): when the step fills the
// slot's buffer (J == C), the CTA -- which holds the S0 rows of its tiles,
// every buffered key and its rows' delta values -- folds the C records into
// those rows itself (P:407 on CUDA cores, fp32), and writes S_new: the
// separate flush, and its second read of the state, disappear.
constexpr int kFusedFoldMaxC = 32;
// new tokens from which the state mat-vecs run on the tensor cores
constexpr int kTcMinTokens = 8;

#ifdef LABUF_CK_PROF
// per-CTA timeline of the last chunk-kernel launch (globaltimer ns, SM id):
// 0 entry, 1 tokens (+ state) landed, 2 records landed, 3 exit, 4 state landed (MMA kinds),
// 5 state pass done, 6 before the substitution, 7 after it -- tools/ck_prof.py
__device__ unsigned long long g_ck_prof[8192][9];
__device__ __forceinline__ unsigned long long ck_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define CK_MARK(i)                                                                                   \
    do {                                                                                             \
        const int cta_ = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);             \
        if (threadIdx.x == 0 && cta_ < 8192) {                                                       \
            g_ck_prof[cta_][i] = ck_now();                                                           \
            if (i == 0) { unsigned sm_; asm("mov.u32 %0, %%smid;" : "=r"(sm_)); g_ck_prof[cta_][8] = sm_; } \
        }                                                                                            \
    } while (0)
#else
#define CK_MARK(i) do { } while (0)
#endif

template <typename InT, typename UT, int TPC, int WPT, int NT, bool HAS_STATE, int MINB, bool TC, bool FOLD = false,
          bool MMA = false, bool PG = false>
__global__ void __launch_bounds__(TPC * WPT * 32, MINB) chunk_cta_kernel(const ChunkArgs a,
                                                                        const __grid_constant__ CUtensorMap tmap) {
    static_assert(!TC || (HAS_STATE && TPC == 4 && WPT == 1), "tensor-core pass: whole head per CTA");
    // FOLD: the decode kind folds a filled buffer (NT = 1), or -- with MMA -- a
    // prefill chunk from an empty buffer folds its own records (PFOLD)
    static_assert(!FOLD || MMA || (NT == 1 && HAS_STATE && WPT == 1 && !TC), "fused fold: decode kind only");
    constexpr bool PFOLD = FOLD && MMA;
    constexpr bool DFOLD = FOLD && !MMA;
    static_assert(!MMA || (HAS_STATE && (WPT == 1 || WPT == 2) && NT >= 2 && !TC),
                  "warp-MMA pass: multi-token state kinds");
    constexpr int NMMA = tc_nmma(NT);
    constexpr int NTHR = TPC * WPT * 32;
    constexpr int RPW = 32 / WPT;                // d_v rows per warp
    constexpr int V = 2 * NT;                    // reduced values per row: (k_t, q_t) dots
    constexpr int NOUT = TeamOut<V>::N;
    // k_t, q_t chunks held in registers (decode, and direct at the 4-CTA budget;
    // the 5-CTA direct instantiation reads them from shared memory: registers)
    constexpr bool KQ_REG = NT == 1 && (HAS_STATE || MINB < 5);
    constexpr int isz = (int)sizeof(InT), usz = (int)sizeof(UT);
    static_assert(NT <= 32, "decay scan runs inside one warp");
    static_assert(NTHR >= 64, "warp 0 requests the records, warp 1 the new tokens");

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    CK_MARK(0);
    const int seg = lane & 3, team = lane >> 2, par = team & 1;
    const int wt = warp / WPT, half = warp % WPT;  // the warp's d_v tile and row block in it
    const Dims dm = a.dm;
    const int T = dm.T, Hv = dm.Hv, Hk = dm.Hk;
    const int tg = blockIdx.x, h = blockIdx.y, zi = blockIdx.z;
    // index-array batches: the slot and the caller's input row of CTA row zi
    // (staged by a previous grid: L2 loads, and never before the PDL wait --
    // the host clears pdl_early for list launches)
    // PG (pools / index lists) is a separate instantiation: the contiguous
    // range path keeps its exact address arithmetic and load batching
    if constexpr (PG) {   // slot lists, state indices and block tables may come from the previous grid
        if (a.pdl) pdl_wait();
    }
    const int r = PG && a.slots ? __ldcg(a.slots + zi) : a.first + zi, hk = h / dm.g;
    const int xrow = PG && a.pos ? __ldcg(a.pos + zi) : zi;
    const size_t sb = PG && a.p.sidx ? (size_t)__ldcg(a.p.sidx + r) : (size_t)r;   // state slot
    const int tile0 = tg * TPC;                  // first 32-row d_v tile of the CTA
    const int n_new = a.n_new;
    const bool direct = (a.kind == CK_DIRECT);
    constexpr int NTP = ntp(NT);                 // row stride of Ck/Cq ([record][token])

    extern __shared__ __align__(1024) unsigned char smem[];
    const CtaLayout L = cta_layout(TPC, NT, HAS_STATE, a.j0_cap, isz, usz, TC, FOLD, MMA, MINB);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + L.bar);
    uint64_t *recs = full + 1;                  // second barrier: the buffered records
    int *j0_s = reinterpret_cast<int *>(smem + L.bar + 16);
    uint64_t *mmab = full + 3;                  // tensor-core pass completions
    // MMA kinds: the new tokens complete on their own barrier, so the B operand,
    // the key rows and the records are processed while the state is in flight
    uint64_t *tokb = MMA ? full + 5 : full;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + L.bar + 32);
    unsigned char *S_base = smem + L.S;
    if constexpr (TC) S_base += (1024u - (smem_u32(S_base) & 1023u)) & 1023u;
    if constexpr (MMA) {
        if (smem_u32(S_base) & 1023u) __trap();   // the swizzled TMA tile needs 1024-byte alignment
    }
    const float *S_s = reinterpret_cast<const float *>(S_base);
    const UT *U_s = reinterpret_cast<const UT *>(smem + L.U);
    const InT *K_s = reinterpret_cast<const InT *>(smem + L.K);
    const float *G_s = reinterpret_cast<const float *>(smem + L.Gs);
    // new tokens' q_t / k_t rows: token t at q_s + t * TS (key-rows MMA kinds: rows
    // 2t + 1 / 2t of the padded bf16 operand Ap)
    constexpr bool KRM = MMA && isz == 2;
    // direct one-token step on a contiguous handle: key rows by TMA + mma.sync
    // (runtime: the host passes the key tensor map in `tmap`, a.tmapk != null)
    constexpr bool KTMA = !HAS_STATE && NT == 1 && isz == 2 && !MMA && !TC && !PG;
    constexpr int TS = KRM ? 2 * kKp : kD;
    const InT *q_s = KRM ? reinterpret_cast<const InT *>(smem + L.Ap) + kKp : reinterpret_cast<const InT *>(smem + L.q);
    const InT *k_s = KRM ? reinterpret_cast<const InT *>(smem + L.Ap) : reinterpret_cast<const InT *>(smem + L.k);
    const InT *v_s = reinterpret_cast<const InT *>(smem + L.v);
    float *Ck = reinterpret_cast<float *>(smem + L.Ck);
    float *Cq = reinterpret_cast<float *>(smem + L.Cq);
    float *av = reinterpret_cast<float *>(smem + L.av);
    float *bv = reinterpret_cast<float *>(smem + L.bv);
    float *Gn_s = reinterpret_cast<float *>(smem + L.Gn);
    float *Bn_s = reinterpret_cast<float *>(smem + L.Bn);

    const InT *qin = static_cast<const InT *>(a.q);
    const InT *kin = static_cast<const InT *>(a.k);
    const InT *vin = static_cast<const InT *>(a.v);
    auto tok_of = [&](int t) { return (size_t)xrow * a.tok_total + a.tok_offset + t; };

    // ---- 0. Two mbarriers.  `full`: the fixed-size operands (state tiles,
    //         new tokens), requested at once (thread 0: the state, warp 1:
    //         q_t, k_t, v_t).  `recs`: the buffered records (U, K, G), which
    //         need the slot's count j0; thread 0 alone reads it, requests the
    //         records and publishes j0 through `recs`, then takes the slot
    //         ticket (every CTA of the slot has read the counter before the
    //         last ticket is drawn).  The state mat-vecs run while the records
    //         are still in flight.
    const uint32_t tok_bytes = (uint32_t)(n_new * (2 * kD * isz + TPC * 32 * isz));
    const uint32_t fixed_bytes = (HAS_STATE ? (uint32_t)(TPC * 32 * kD * 4) : 0u) + (MMA ? 0u : tok_bytes);
    auto issue_state = [&]() {
        if constexpr (TC || MMA) {
            // 32-row x 32-column boxes, 128-byte swizzle: column group kb of the
            // CTA's TPC x 32 rows at S_base + kb * TPC * 4 KiB (row-major inside)
            const int row0 = (int)((sb * Hv + h) * kD) + tile0 * 32;
#pragma unroll
            for (int kb = 0; kb < 4; ++kb)
#pragma unroll
                for (int x = 0; x < TPC; ++x)
                    tma_load_2d(S_base + kb * (TPC * 32 * 128) + x * 4096, &tmap, kb * 32, row0 + x * 32, full);
        } else {
            bulk_g2s(smem + L.S, a.p.state + ((sb * Hv + h) * kD + (size_t)tile0 * 32) * kD,
                     TPC * 32 * kD * 4, full);
        }
    };
    if constexpr (TC) {
        if (warp == 0) tmem_alloc<32>(tmem_slot);
    }
    if (tid == 0) {
        mbar_init(full, 1);
        mbar_init(recs, 1);
        if (TC) mbar_init(mmab, 1);
        if (MMA) mbar_init(tokb, 1);
        fence_mbar_init();
        if (HAS_STATE && a.pdl_early) {
            // the state tile is not written by the grid this one overlaps
            // (launch overlap), so it streams in while that grid drains
            mbar_arrive_expect_tx(full, fixed_bytes);
            issue_state();
        }
    }
    if (a.pdl) pdl_wait();   // inputs, counters and records may come from the previous grid
    pdl_trigger();
    // alpha / beta of the new tokens (lane t), in flight with the copies
    float al_l = 1.f, be_l = 0.f;
    if (lane < n_new) {
        al_l = a.alpha[tok_of(lane) * Hv + h];
        be_l = a.beta[tok_of(lane) * Hv + h];
    }
    __syncthreads();
    int ticket = 0;
    if (PG && warp == 0) {
        // lane 0: the state (unless early), the slot's count j0; the j0-dependent
        // records are requested by the lanes in parallel, one copy per (record
        // block, field): the tiles' u sub-tiles, the QK head's key rows, the
        // log decays
        int j0v = 0;
        if (lane == 0) {
            if (!(HAS_STATE && a.pdl_early)) {
                mbar_arrive_expect_tx(full, fixed_bytes);
                if (HAS_STATE) issue_state();
            }
            j0v = (direct ? a.p.len : a.p.occ)[r] + a.j_add;
            *j0_s = j0v;
        }
        j0v = __shfl_sync(0xffffffffu, j0v, 0);
        const int bt = dm.bt, nb = (j0v + bt - 1) / bt;
        if (lane == 0) {
            uint32_t gbytes = 0;
            for (int b = 0; b < nb; ++b) gbytes += (uint32_t)(((min(bt, j0v - b * bt) + 3) & ~3) * 4);
            mbar_arrive_expect_tx(recs, (uint32_t)(TPC * 32 * j0v * usz) + (uint32_t)(j0v * kD * isz) + gbytes);
        }
        __syncwarp();
        constexpr int NF = TPC + 2;
        for (int c = lane; c < nb * NF; c += 32) {
            const int b = c / NF, f = c % NF, cnt = min(bt, j0v - b * bt);
            const size_t blk = a.p.btab ? (size_t)__ldcg(a.p.btab + (size_t)r * dm.maxb + b) : (size_t)r;
            if (f < TPC)
                bulk_g2s(smem + L.U + ((size_t)f * j0v + (size_t)b * bt) * kUSub * usz,
                         static_cast<const UT *>(a.p.U) + (((blk * Hv + h) * (kD / kUSub) + tile0 + f) * bt) * kUSub,
                         (uint32_t)(cnt * kUSub * usz), recs);
            else if (f == TPC)
                bulk_g2s(smem + L.K + (size_t)b * bt * kD * isz,
                         static_cast<const InT *>(a.p.K) + (blk * Hk + hk) * bt * kD, (uint32_t)(cnt * kD * isz), recs);
            else
                bulk_g2s(smem + L.Gs + (size_t)b * bt * 4, a.p.G + (blk * Hv + h) * bt,
                         (uint32_t)(((cnt + 3) & ~3) * 4), recs);
        }
        if (lane == 0 && a.kind != CK_VERIFY) ticket = atomicAdd(&a.p.ticket[r], 1);
    } else if (!PG && tid == 0) {
        // contiguous handle: one region of T records per slot
        if (!(HAS_STATE && a.pdl_early)) {
            mbar_arrive_expect_tx(full, fixed_bytes);
            if (HAS_STATE) issue_state();
        }
        // (host-exact uniform count: the records are requested without the counter round trip)
        const int j0v = a.j0_fixed >= 0 ? a.j0_fixed : (direct ? a.p.len : a.p.occ)[r] + a.j_add;
        const int jbv = (j0v + 3) & ~3;
        *j0_s = j0v;
        const uint32_t kbytes = (KTMA && a.tmapk) ? (uint32_t)((j0v + 15) / 16 * 4096) : (uint32_t)(j0v * kD * isz);
        mbar_arrive_expect_tx(recs, (uint32_t)(TPC * 32 * j0v * usz) + kbytes + (j0v ? (uint32_t)(jbv * 4) : 0u));
        if (j0v) {
            for (int x = 0; x < TPC; ++x)
                bulk_g2s(smem + L.U + (size_t)x * j0v * kUSub * usz,
                         static_cast<const UT *>(a.p.U) + ((((size_t)r * Hv + h) * (kD / kUSub) + tile0 + x) * T) * kUSub,
                         (uint32_t)(j0v * kUSub * usz), recs);
            if (KTMA && a.tmapk) {
                // key rows as 16-record x 64-column boxes, 128-byte swizzle (conflict-
                // free ldmatrix); rows past j0 are other records or zero fill (unused)
                const int nb = (j0v + 15) / 16, jp = (a.j0_cap + 15) / 16 * 16;
                const int row = (r * Hk + hk) * T;
                for (int b = 0; b < nb; ++b) {
                    tma_load_2d(smem + L.K + b * 2048, &tmap, 0, row + b * 16, recs);
                    tma_load_2d(smem + L.K + jp * 128 + b * 2048, &tmap, 64, row + b * 16, recs);
                }
            } else {
                bulk_g2s(smem + L.K, static_cast<const InT *>(a.p.K) + ((size_t)r * Hk + hk) * T * kD,
                         (uint32_t)(j0v * kD * isz), recs);
            }
            bulk_g2s(smem + L.Gs, a.p.G + ((size_t)r * Hv + h) * T, (uint32_t)(jbv * 4), recs);
        }
        if (a.kind != CK_VERIFY) ticket = atomicAdd(&a.p.ticket[r], 1);
    } else if (warp == 1) {
        // new tokens: q_t, k_t rows of the QK head and the tiles' v_t slice
        // (warp 1's lanes, so they issue in parallel with warp 0)
        if constexpr (MMA) {
            if (lane == 0) mbar_arrive_expect_tx(tokb, tok_bytes);
            __syncwarp();
        }
        for (int c = lane; c < 3 * n_new; c += 32) {
            const int t = c % n_new, kind = c / n_new;
            if (kind == 0)
                bulk_g2s(const_cast<InT *>(q_s) + (size_t)t * TS, qin + (tok_of(t) * Hk + hk) * kD, kD * isz, tokb);
            else if (kind == 1)
                bulk_g2s(const_cast<InT *>(k_s) + (size_t)t * TS, kin + (tok_of(t) * Hk + hk) * kD, kD * isz, tokb);
            else
                bulk_g2s(smem + L.v + (size_t)t * TPC * 32 * isz, vin + (tok_of(t) * Hv + h) * kD + tile0 * 32,
                         TPC * 32 * isz, tokb);
        }
    }

    // ---- 1. cumulative log decay increments of the new tokens (lane t), in registers
    unsigned bad = 0;
    float x_l = 0.f;
    if (lane < n_new) {
        x_l = dm.variant == 2 ? 0.f : logf(al_l);   // vanilla LA: no decay (alpha ignored)
        if (dm.validate && warp == 0) {
            if (dm.variant != 2 && !(al_l > 0.f && al_l <= 1.f)) bad |= 0x1u;
            if (!(be_l >= 0.f && be_l <= 1.f)) bad |= 0x2u;
        }
    }
    // (branch verify: the scan restarts at every branch of a.seg tokens)
    const int segl = a.seg > 0 ? a.seg : NT;
#pragma unroll
    for (int off = 1; off < NT; off <<= 1) {
        const float y = __shfl_up_sync(0xffffffffu, x_l, off);
        if (lane % segl >= off) x_l += y;
    }
    mbar_wait(tokb, 0);   // (non-MMA kinds: tokb == full, the state and the tokens)
    CK_MARK(1);
    // multi-token launches read k_t / q_t once per row step: widen them to
    // fp32 once per CTA ([t][k | q][128])
    // (with the warp-MMA pass the fp32 B rows double as the widened k_t / q_t)
    constexpr bool KQ32 = !KQ_REG && isz == 2 && !MMA;
    constexpr bool KQB = MMA && isz == 2;
    float *kq32 = reinterpret_cast<float *>(smem + L.kq32);
    float *Bm = reinterpret_cast<float *>(smem + L.Bm);
    if constexpr (MMA && isz == 4) {
        // B operand of the warp-MMA pass for fp32 tokens: row n = k_t (n = 2t) /
        // q_t (n = 2t + 1), zero rows past 2 n_new, split hi (top 19 bits) + lo
        // (bf16 tokens: the padded bf16 rows Ap serve both MMA passes as they land)
        constexpr int NB = mma_nrows(NT);
        for (int e = tid; e < NB * (kD / 8); e += NTHR) {
            const int n = e >> 4, c = (e & 15) * 8, t = n >> 1;
            float x[8];
            if (t < n_new) {
                const InT *src = ((n & 1) ? q_s : k_s) + t * TS + c;
                const float4 lo4 = load4(src), hi4 = load4(src + 4);
                x[0] = lo4.x; x[1] = lo4.y; x[2] = lo4.z; x[3] = lo4.w;
                x[4] = hi4.x; x[5] = hi4.y; x[6] = hi4.z; x[7] = hi4.w;
            } else {
#pragma unroll
                for (int i = 0; i < 8; ++i) x[i] = 0.f;
            }
            float hi[8], lo[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) { hi[i] = trunc_tf32(x[i]); lo[i] = x[i] - hi[i]; }
            float4 *dst = reinterpret_cast<float4 *>(Bm + n * kBmStride + c);
            dst[0] = make_float4(hi[0], hi[1], hi[2], hi[3]);
            dst[1] = make_float4(hi[4], hi[5], hi[6], hi[7]);
            float4 *dl = reinterpret_cast<float4 *>(Bm + (NB + n) * kBmStride + c);
            dl[0] = make_float4(lo[0], lo[1], lo[2], lo[3]);
            dl[1] = make_float4(lo[4], lo[5], lo[6], lo[7]);
        }
    }
    if constexpr (KQ32) {
        for (int e = tid; e < n_new * kD; e += NTHR) {
            const int t = e / kD, c = e % kD;
            kq32[(t * 2 + 0) * kD + c] = to_f(k_s[e]);
            kq32[(t * 2 + 1) * kD + c] = to_f(q_s[e]);
        }
    }
    if constexpr (KQ32 || (MMA && isz == 4)) __syncthreads();
    uint32_t tmem = 0;
    float *Yh = reinterpret_cast<float *>(smem + L.Y);
    float *Yl = Yh + NMMA * kD;
    auto mma_pass = [&](const float *Y, bool acc) {
        const uint32_t idesc = idesc_tf32(128, NMMA);
#pragma unroll
        for (int kk = 0; kk < kD / 8; ++kk) {
            const uint64_t da = umma_desc_sw128(smem_u32(S_base) + (kk >> 2) * (TPC * 32 * 128) + (kk & 3) * 32);
            const uint64_t db = umma_desc_noswz(smem_u32(Y) + kk * 256, 128, kD * 32);
            tc_mma_tf32(tmem, da, db, idesc, (acc || kk > 0) ? 1u : 0u);
        }
    };
    if constexpr (TC) {
        // B operand: row n = (k_t | q_t) of token n / 2, K-major SWIZZLE_NONE
        // (8-row x 16-byte core matrices, K-adjacent at +128 B, row groups at +4 KiB)
        for (int e = tid; e < NMMA * kD; e += NTHR) {
            const int n = e / kD, c = e % kD, t = n >> 1;
            float x = 0.f;
            if (t < n_new) x = to_f(((n & 1) ? q_s : k_s)[t * kD + c]);
            const int off = (n >> 3) * (kD * 32 / 4) + (c >> 2) * 32 + (n & 7) * 4 + (c & 3);
            if constexpr (isz == 4) {
                const float hi = trunc_tf32(x);
                Yh[off] = hi;
                Yl[off] = x - hi;
            } else {
                Yh[off] = x;     // bf16 values are exact in tf32
            }
        }
        fence_proxy_async_smem();
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
        tmem = *tmem_slot;
        if (tid == 0) {
            mma_pass(Yh, false);                    // trunc(S0) . Y_hi
            if constexpr (isz == 4) mma_pass(Yl, true);   // trunc(S0) . Y_lo
            tc_commit(mmab);
        }
    }
    int j0 = 0, J = 0;
    // MMA kinds: the state pass accumulators (S0 k_t, S0 q_t per row) live on in registers
    float macc[MMA ? 2 / WPT : 1][MMA ? mma_nrows(NT) / 8 : 1][4];
    float gn_l = 0.f;
    // ---- 2. rows with 4-lane teams, 8 rows per warp step:
    //      state rows of the warp's tile: a = S0 k_t, b = S0 q_t;
    //      key rows i (shared out over the warps):
    //        Ck[t][i] = e^{G_t-G_i} (k_t.k_i) (i < j0+t),  Cq[t][i] = e^{G_t-G_i} (q_t.k_i) (i <= j0+t)  (Z3)
    {
        float4 kx[KQ_REG ? 8 : 1], qx[KQ_REG ? 8 : 1];
        if constexpr (KQ_REG) {
            load_row8(k_s, seg, par, kx);
            load_row8(q_s, seg, par, qx);
        }
        // dots of row x with k_t and q_t (this lane's 32 columns)
        auto row_dots = [&](const float4 (&x)[8], float (&vals)[V]) {
            if constexpr (KQ_REG) {
                vals[0] = dot8x4(x, kx);
                vals[1] = dot8x4(x, qx);
            } else {
#pragma unroll
                for (int t = 0; t < NT; ++t) {
                    float4 y[8];
                    if constexpr (KQB) load_row8(Bm + (size_t)(t * 2) * kBmStride, seg, par, y);
                    else if constexpr (KQ32) load_row8(kq32 + (size_t)(t * 2) * kD, seg, par, y);
                    else load_row8(k_s + (size_t)t * kD, seg, par, y);
                    vals[2 * t] = dot8x4(x, y);
                    if constexpr (KQB) load_row8(Bm + (size_t)(t * 2 + 1) * kBmStride, seg, par, y);
                    else if constexpr (KQ32) load_row8(kq32 + (size_t)(t * 2 + 1) * kD, seg, par, y);
                    else load_row8(q_s + (size_t)t * kD, seg, par, y);
                    vals[2 * t + 1] = dot8x4(x, y);
                }
            }
        };
        // state rows of the warp's tile: 4 steps of 8 rows (one token), or --
        // when k_t / q_t come from shared memory (several tokens) -- 2 steps
        // of 2 x 8 rows, so every k_t / q_t chunk load serves two rows
        if constexpr (TC) {
            // (the tensor-core pass is in flight; see after the key rows)
        } else if constexpr (MMA) {
            // (the warp-MMA pass runs once the state lands, after the key rows)
        } else if constexpr (HAS_STATE && KQ_REG) {
#pragma unroll 4
            for (int st = 0; st < RPW / 8; ++st) {
                const int rf = half * RPW + st * 8 + team;
                float4 x[8];
                load_row8(S_s + (size_t)(wt * 32 + rf) * kD, seg, par, x);
                float vals[V];
                row_dots(x, vals);
                float res[NOUT];
                int xid[NOUT];
                team_reduce<V>(vals, seg, res, xid);
#pragma unroll
                for (int o = 0; o < NOUT; ++o) {
                    const int t = xid[o] >> 1;
                    if (xid[o] >= 0 && t < n_new) ((xid[o] & 1) ? bv : av)[(wt * NT + t) * 32 + rf] = res[o];
                }
            }
        } else if constexpr (HAS_STATE && V <= 8 && WPT == 1) {
            // 2 or 4 new tokens (verify): lane owns columns 4 lane .. 4 lane + 3 of
            // all V = 2 NT vectors (k_t, q_t) in registers and reads whole state
            // rows (one conflict-free 16-byte read per row); RB = 32 / V rows per
            // batch give 32 partial sums per lane, summed across the warp by one
            // transposed butterfly (lane l ends with value l = (row l / V, vector l % V))
            constexpr int RB = 32 / V;
            float4 vec[V];
#pragma unroll
            for (int v = 0; v < V; ++v) {
                if constexpr (KQ32) vec[v] = *reinterpret_cast<const float4 *>(kq32 + (size_t)v * kD + 4 * lane);
                else vec[v] = load4(((v & 1) ? q_s : k_s) + (size_t)(v >> 1) * kD + 4 * lane);
            }
#pragma unroll 1
            for (int rb = 0; rb < 32; rb += RB) {
                float vals[32];
#pragma unroll
                for (int rr = 0; rr < RB; ++rr) {
                    const float4 s4 = *reinterpret_cast<const float4 *>(S_s + (size_t)(wt * 32 + rb + rr) * kD + 4 * lane);
#pragma unroll
                    for (int v = 0; v < V; ++v)
                        vals[rr * V + v] = fmaf(s4.x, vec[v].x, fmaf(s4.y, vec[v].y, fmaf(s4.z, vec[v].z, s4.w * vec[v].w)));
                }
                const float red = transposed_reduce<32>(vals, lane);
                const int row = rb + lane / V, v = lane % V, t = v >> 1;
                if (t < n_new) ((v & 1) ? bv : av)[(wt * NT + t) * 32 + row] = red;
            }
        } else if constexpr (HAS_STATE) {
            static_assert(RPW % 16 == 0, "two row blocks per step");
            constexpr int NOUT2 = TeamOut<2 * V>::N;
            for (int st = 0; st < RPW / 16; ++st) {
                const int rf0 = half * RPW + st * 16 + team, rf1 = rf0 + 8;
                float4 x0[8], x1[8];
                load_row8(S_s + (size_t)(wt * 32 + rf0) * kD, seg, par, x0);
                load_row8(S_s + (size_t)(wt * 32 + rf1) * kD, seg, par, x1);
                float vals[2 * V];
#pragma unroll
                for (int t = 0; t < NT; ++t) {
                    float4 y[8];
                    if constexpr (KQ32) load_row8(kq32 + (size_t)(t * 2) * kD, seg, par, y);
                    else load_row8(k_s + (size_t)t * kD, seg, par, y);
                    vals[2 * t] = dot8x4(x0, y);
                    vals[V + 2 * t] = dot8x4(x1, y);
                    if constexpr (KQ32) load_row8(kq32 + (size_t)(t * 2 + 1) * kD, seg, par, y);
                    else load_row8(q_s + (size_t)t * kD, seg, par, y);
                    vals[2 * t + 1] = dot8x4(x0, y);
                    vals[V + 2 * t + 1] = dot8x4(x1, y);
                }
                float res[NOUT2];
                int xid[NOUT2];
                team_reduce<2 * V>(vals, seg, res, xid);
#pragma unroll
                for (int o = 0; o < NOUT2; ++o) {
                    const int xv = xid[o] % V, rf = xid[o] < V ? rf0 : rf1;
                    const int t = xv >> 1;
                    if (xid[o] >= 0 && t < n_new) ((xv & 1) ? bv : av)[(wt * NT + t) * 32 + rf] = res[o];
                }
            }
        }
        // ---- the buffered records: j0, log decays
        mbar_wait(recs, 0);
        CK_MARK(2);
        j0 = *j0_s;
        J = j0 + n_new;
        gn_l = (j0 > 0 ? G_s[j0 - 1] : 0.f) + x_l;
        if (warp == 0 && lane < n_new) {
            Gn_s[lane] = gn_l;
            Bn_s[lane] = be_l;
        }
        // key rows, shared out over the warps in steps of 8
        const int KS = (J + 7) / 8;
        if constexpr (MMA && isz == 2) {
            // on the tensor cores: raw dots D[v][i] = vec_v . key_i (v = 2t: k_t, 2t+1:
            // q_t) = Ap [2NT x 128] . Kp^T, mma.sync m16n8k16 bf16 (products exact, fp32
            // accumulate); keys = the j0 records then the new tokens' keys
            constexpr int NW = TPC * WPT, MT2 = (2 * NT + 15) / 16;
            InT *Kp = reinterpret_cast<InT *>(smem + L.Kp);
            for (int e = tid; e < j0 * (kD / 8); e += NTHR) {   // the records' keys, padded rows
                const int i = e >> 4, c = (e & 15) * 8;
                *reinterpret_cast<uint4 *>(Kp + i * kKp + c) = *reinterpret_cast<const uint4 *>(K_s + (size_t)i * kD + c);
            }
            __syncthreads();   // Kp, Gn_s (and the token rows Ap) visible
            const int g = lane >> 2, t4 = lane & 3, lr = lane & 7, lm = lane >> 3;
            const uint32_t ap0 = smem_u32(smem + L.Ap) + (uint32_t)((lm >> 1) * 8 * 2);
            const uint32_t apk = smem_u32(smem + L.Ap) + (uint32_t)((lm & 1) * 8 * 2);
            const uint32_t kpb = smem_u32(Kp) + (uint32_t)((lm & 1) * 8 * 2);
            for (int nt = warp; nt < KS; nt += NW) {
#pragma unroll
                for (int mt = 0; mt < MT2; ++mt) {
                    float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                    for (int kk = 0; kk < kD / 16; ++kk) {
                        uint32_t av4[4], bv2[2];
                        // (rows past 2 NT repeat the last vector: their outputs are dropped)
                        const int arow = min(mt * 16 + lr + (lm & 1) * 8, 2 * NT - 1);
                        ldsm_x4(av4, ap0 + (uint32_t)((arow * kKp + kk * 16) * 2));
                        // key row i: a buffered record (Kp) or new token i - j0 (row 2 (i - j0) of Ap;
                        // rows past J repeat a valid row, their outputs are dropped)
                        const int ki = nt * 8 + lr;
                        const uint32_t brow = ki < j0 ? kpb + (uint32_t)(ki * kKp * 2)
                                                      : apk + (uint32_t)(2 * min(ki - j0, n_new - 1) * kKp * 2);
                        ldsm_x2(bv2, brow + (uint32_t)(kk * 16 * 2));
                        mma_bf16_16x8x16(acc, av4, bv2[0], bv2[1]);
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int v = mt * 16 + g + (q >> 1) * 8, i = nt * 8 + 2 * t4 + (q & 1);
                        const int t = v >> 1;
                        const bool isq = v & 1;
                        if (t < n_new && i < J) {
                            bool valid = isq ? (i <= j0 + t) : (i < j0 + t);
                            if (a.seg > 0 && i >= j0 && (i - j0) / segl != t / segl) valid = false;   // another branch
                            const float cf = valid ? expf(Gn_s[t] - (i < j0 ? G_s[i] : Gn_s[i - j0])) * acc[q] : 0.f;
                            (isq ? Cq : Ck)[i * NTP + t] = cf;
                        }
                    }
                }
            }
        } else if (KTMA && a.tmapk) {
            // key rows on the tensor cores: D[i][n] = k_i . vec_n (n = 0: k_t, 1: q_t),
            // mma.sync m16n8k16 bf16 (products exact, fp32 accumulate); A = the
            // swizzled key boxes by ldmatrix (conflict-free), B = the token rows
            const int g = lane >> 2, t4 = lane & 3, lr = lane & 7, lm = lane >> 3;
            const int jp = (a.j0_cap + 15) / 16 * 16;
            const uint32_t kbase = smem_u32(K_s);
            const float gt = __shfl_sync(0xffffffffu, gn_l, 0);
            const InT *vrow = g == 0 ? k_s : q_s;
            for (int mt = warp; mt * 16 < j0; mt += TPC * WPT) {
                float acc[4] = {0.f, 0.f, 0.f, 0.f};
                const int arow = mt * 16 + lr + (lm & 1) * 8;
#pragma unroll
                for (int kk = 0; kk < kD / 16; ++kk) {
                    const int chunk = (kk & 3) * 2 + (lm >> 1);
                    uint32_t av4[4];
                    ldsm_x4(av4, kbase + (uint32_t)((kk >> 2) * jp * 128 + arow * 128 + ((chunk ^ (arow & 7)) << 4)));
                    uint32_t b0 = 0u, b1 = 0u;
                    if (g < 2) {
                        b0 = *reinterpret_cast<const uint32_t *>(vrow + kk * 16 + 2 * t4);
                        b1 = *reinterpret_cast<const uint32_t *>(vrow + kk * 16 + 8 + 2 * t4);
                    }
                    mma_bf16_16x8x16(acc, av4, b0, b1);
                }
                if (t4 == 0) {
#pragma unroll
                    for (int hf = 0; hf < 2; ++hf) {
                        const int i = mt * 16 + g + 8 * hf;
                        if (i < j0) {   // (rows past j0: other records or zero fill)
                            const float w = expf(gt - G_s[i]);
                            Ck[i * NTP] = w * acc[2 * hf];
                            Cq[i * NTP] = w * acc[2 * hf + 1];
                        }
                    }
                }
            }
            // the new token's own key (record j0): q_t . k_t, weight e^0
            if (warp == TPC * WPT - 1) {
                const float dqk = warp_sum(dot4(load4(k_s + 4 * lane), load4(q_s + 4 * lane)));
                if (lane == 0) Cq[j0 * NTP] = dqk;
            }
        } else
        for (int ks = warp; ks < KS; ks += TPC * WPT) {
            const int i = ks * 8 + team;
            float4 x[8];
            if (i < J) {
                load_row8(i < j0 ? K_s + (size_t)i * kD : k_s + (size_t)(i - j0) * kD, seg, par, x);
            } else {
#pragma unroll
                for (int c = 0; c < 8; ++c) x[c] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
            float vals[V];
            row_dots(x, vals);
            float res[NOUT];
            int xid[NOUT];
            team_reduce<V>(vals, seg, res, xid);
            const int inew = (i - j0) > 0 ? (i - j0) : 0;
#pragma unroll
            for (int o = 0; o < NOUT; ++o) {
                const int t = xid[o] >= 0 ? (xid[o] >> 1) : 0;
                const bool isq = xid[o] & 1;
                const float gt = __shfl_sync(0xffffffffu, gn_l, t);
                const float gnew = __shfl_sync(0xffffffffu, gn_l, inew < NT ? inew : 0);
                if (xid[o] >= 0 && i < J && t < n_new) {
                    bool valid = isq ? (i <= j0 + t) : (i < j0 + t);
                    if (a.seg > 0 && i >= j0 && (i - j0) / segl != t / segl) valid = false;   // another branch
                    float cf = 0.f;
                    if (valid) cf = expf(gt - (i < j0 ? G_s[i] : gnew)) * res[o];
                    (isq ? Cq : Ck)[i * NTP + t] = cf;
                }
            }
        }
    }
    if constexpr (MMA) {
        mbar_wait(full, 0);   // the state tile (TMA, swizzled)
        CK_MARK(4);
        float (&acc)[2 / WPT][mma_nrows(NT) / 8][4] = macc;
        // warp-level tensor cores (mma.sync m16n8k8 tf32, fp32 accumulate):
        // D[32 rows x 2NT] = S0 tile [32 x 128] . [k_t | q_t] [128 x 2NT];
        // A fragments straight from the 128-byte-swizzled tile (conflict-
        // free), split TF32: S0 = hi + lo (hi = top 19 bits), 2 passes for
        // bf16 tokens (exact in tf32), 3 for fp32 tokens (+ hi . B_lo)
        constexpr int NB = mma_nrows(NT), NJ = NB / 8;
        constexpr int MTW = 2 / WPT;                 // m16 tiles of the 32-row tile per warp
#pragma unroll
        for (int mt = 0; mt < MTW; ++mt)
#pragma unroll
            for (int j = 0; j < NJ; ++j) acc[mt][j][0] = acc[mt][j][1] = acc[mt][j][2] = acc[mt][j][3] = 0.f;
        // ldmatrix addressing: lane i feeds row (i % 8) of 8x8 matrix i / 8 --
        // A: matrices = (rows 0-7 | 8-15) x (k 0-3 | 4-7) of the m16 x k8
        // fragment, in the 128-byte swizzle (16-byte chunk ^= row % 8: the 8
        // rows of a matrix hit 8 bank groups); B: (k 0-3 | 4-7) of the 8
        // vectors of an n-tile (rows of 132 floats: conflict-free)
        const int lr = lane & 7, lm = lane >> 3;
        uint32_t aoff[4];
#pragma unroll
        for (int c8 = 0; c8 < 4; ++c8)
            aoff[c8] = (uint32_t)((lr + (lm & 1) * 8) * 128 + (((2 * c8 + (lm >> 1)) ^ lr) << 4));
        const uint32_t abase = smem_u32(S_base) + wt * 4096;
        const uint32_t bbase = smem_u32(Bm) + (uint32_t)((lr * kBmStride + (lm & 1) * 4) * 4);
#pragma unroll
        for (int kk = 0; kk < kD / 8; ++kk) {
            uint32_t ahi[MTW][4], alo[MTW][4];
#pragma unroll
            for (int mt = 0; mt < MTW; ++mt) {
                uint32_t x[4];
                ldsm_x4(x, abase + (kk >> 2) * (TPC * 4096) + (half * MTW + mt) * 2048 + aoff[kk & 3]);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t hi = x[q] & 0xFFFFE000u;
                    ahi[mt][q] = hi;
                    alo[mt][q] = __float_as_uint(__uint_as_float(x[q]) - __uint_as_float(hi));
                }
            }
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                uint32_t b[2];
                if constexpr (isz == 2) {   // bf16 row (vector j*8+g): exact in tf32, widened in registers
                    const unsigned short *br = reinterpret_cast<const unsigned short *>(smem + L.Ap) +
                                               min(j * 8 + (lane >> 2), 2 * NT - 1) * kKp + kk * 8 + (lane & 3);
                    b[0] = (uint32_t)br[0] << 16;
                    b[1] = (uint32_t)br[4] << 16;
                } else {
                    ldsm_x2(b, bbase + (uint32_t)((j * 8 * kBmStride + kk * 8) * 4));
                }
#pragma unroll
                for (int mt = 0; mt < MTW; ++mt) {
                    mma_tf32_16x8x8(acc[mt][j], ahi[mt], b[0], b[1]);
                    mma_tf32_16x8x8(acc[mt][j], alo[mt], b[0], b[1]);
                }
                if constexpr (isz == 4) {   // + S0_hi . B_lo
                    uint32_t bl[2];
                    ldsm_x2(bl, bbase + (uint32_t)(((NB + j * 8) * kBmStride + kk * 8) * 4));
#pragma unroll
                    for (int mt = 0; mt < MTW; ++mt) mma_tf32_16x8x8(acc[mt][j], ahi[mt], bl[0], bl[1]);
                }
            }
        }
        // D[row][2 t + {0, 1}] = (S0 k_t, S0 q_t) of token t = 4 j + t4: stays in
        // registers; the substitution shuffles each row's values to its lane
        // (8+ tokens: stashed per (token, row) instead -- 2 loads per token)
        if constexpr (NT >= 8 && FOLD) {
            const int g = lane >> 2, t4 = lane & 3;
#pragma unroll
            for (int mt = 0; mt < MTW; ++mt)
#pragma unroll
                for (int j = 0; j < NJ; ++j)
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int t = 4 * j + t4, rr = (half * MTW + mt) * 16 + g + 8 * (q >> 1);
                        if (t < NT) ((q & 1) ? bv : av)[(wt * NT + t) * 32 + rr] = acc[mt][j][q];
                    }
        }
    }
    if constexpr (TC) {
        // pass 2 on the exact remainder S0 - trunc(S0), written in place once
        // pass 1 has read the tile (the split is elementwise: layout-agnostic)
        mbar_wait(mmab, 0);
        float4 *S4 = reinterpret_cast<float4 *>(S_base);
        for (int e = tid; e < TPC * 32 * kD / 4; e += NTHR) {
            float4 x = S4[e];
            x.x -= trunc_tf32(x.x);
            x.y -= trunc_tf32(x.y);
            x.z -= trunc_tf32(x.z);
            x.w -= trunc_tf32(x.w);
            S4[e] = x;
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) {
            tc_fence_after();
            mma_pass(Yh, true);                     // (S0 - trunc(S0)) . Y_hi
            tc_commit(mmab);
        }
        mbar_wait(mmab, 1);
        tc_fence_after();
        // D row m = d_v row 32 w + lane: warp w reads TMEM lanes 32w..32w+31
        float dv[32];
        tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16), dv);
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            if (t < n_new) {
                av[(warp * NT + t) * 32 + lane] = dv[2 * t];
                bv[(warp * NT + t) * 32 + lane] = dv[2 * t + 1];
            }
        }
    }
    CK_MARK(5);
    if (dm.validate) {
        for (int e = tid; e < n_new * kD; e += NTHR) {
            const float kk = to_f(k_s[(e / kD) * TS + e % kD]), qq = to_f(q_s[(e / kD) * TS + e % kD]);
            if (!(isfinite(kk) && isfinite(qq))) bad |= 0x4u;
        }
    }
    if constexpr (TC) tc_fence_before();
    __syncthreads();
    if constexpr (TC) {
        if (warp == 0) {
            tc_fence_after();
            tmem_dealloc<32>(tmem);
        }
    }

    CK_MARK(6);
    // ---- 3. forward substitution over the new tokens.  Lane -> d_v row
    //         (half * RPW + lane % RPW) of the warp's tile; the WPT lanes of a
    //         row split the buffered records by i % WPT and combine by shuffle.
    {
        const int sub = lane / RPW, row = half * RPW + lane % RPW, tile = tile0 + wt;
        const int drow = tile * 32 + row;
        const UT *ut = U_s + (size_t)wt * j0 * kUSub + row;
        // record position j0 + t of the slot: (block, offset)
        auto recpos = [&](int t) -> int2 {
            if (!PG || !a.p.btab) return make_int2(r, j0 + t);
            return make_int2(__ldcg(a.p.btab + (size_t)r * dm.maxb + (dm.bt_shift >= 0 ? (j0 + t) >> dm.bt_shift : (j0 + t) / dm.bt)),
                                 dm.bt_shift >= 0 ? (j0 + t) & (dm.bt - 1) : (j0 + t) % dm.bt);
        };
        float un[NT];
        // per-token e^{G_t} (lane t computes it once; broadcast by shuffle) and
        // the output / record addresses of token 0 (token t is a fixed stride on)
        const float eg_l = expf(gn_l);
        const size_t ostr = (size_t)Hv * kD;
        float *const obase = a.o ? a.o + (tok_of(0) * Hv + h) * kD + drow : nullptr;
        UT *const ubase = static_cast<UT *>(a.p.U) + ((((size_t)r * Hv + h) * (kD / kUSub) + tile) * dm.bt + j0) * kUSub + row;
        // records part of every token's sums, record-outer for several tokens:
        // each u_i is loaded once and the tokens' coefficients of record i come
        // in 16-byte loads
        float rk[NT], rq[NT];
        if constexpr (NT > 1) {
#pragma unroll
            for (int t = 0; t < NT; ++t) rk[t] = rq[t] = 0.f;
            for (int i = sub; i < j0; i += WPT) {
                const float u0 = to_f(ut[(size_t)i * kUSub]);
#pragma unroll
                for (int tc = 0; tc < NTP / 4; ++tc) {
                    const float4 c4 = *reinterpret_cast<const float4 *>(Ck + i * NTP + 4 * tc);
                    const float4 d4 = *reinterpret_cast<const float4 *>(Cq + i * NTP + 4 * tc);
                    const float cv[4] = {c4.x, c4.y, c4.z, c4.w}, dv4[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
                    for (int x = 0; x < 4; ++x) {
                        if (4 * tc + x < NT) {
                            rk[4 * tc + x] = fmaf(cv[x], u0, rk[4 * tc + x]);
                            rq[4 * tc + x] = fmaf(dv4[x], u0, rq[4 * tc + x]);
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            if (t < n_new) {
                const float *ck = Ck + t;   // coefficient of record i: ck[i * NTP]
                const float *cq = Cq + t;
                float ak0 = 0.f, ak1 = 0.f, aq0 = 0.f, aq1 = 0.f;
                if constexpr (NT == 1) {
                    int i = sub;
                    for (; i + WPT < j0; i += 2 * WPT) {
                        const float u0 = to_f(ut[(size_t)i * kUSub]);
                        const float u1 = to_f(ut[(size_t)(i + WPT) * kUSub]);
                        ak0 = fmaf(ck[i], u0, ak0);
                        aq0 = fmaf(cq[i], u0, aq0);
                        ak1 = fmaf(ck[i + WPT], u1, ak1);
                        aq1 = fmaf(cq[i + WPT], u1, aq1);
                    }
                    if (i < j0) {
                        const float u0 = to_f(ut[(size_t)i * kUSub]);
                        ak0 = fmaf(ck[i], u0, ak0);
                        aq0 = fmaf(cq[i], u0, aq0);
                    }
                } else {
                    ak0 = rk[t];
                    aq0 = rq[t];
                }
                float acc_k = ak0 + ak1, acc_q = aq0 + aq1;
#pragma unroll
                for (int m = RPW; m < 32; m <<= 1) {
                    acc_k += __shfl_xor_sync(0xffffffffu, acc_k, m);
                    acc_q += __shfl_xor_sync(0xffffffffu, acc_q, m);
                }
#pragma unroll
                for (int tp = 0; tp < t; ++tp) {
                    acc_k = fmaf(ck[(j0 + tp) * NTP], un[tp], acc_k);
                    acc_q = fmaf(cq[(j0 + tp) * NTP], un[tp], acc_q);
                }
                const float vt = to_f(v_s[t * TPC * 32 + wt * 32 + row]);
                const float bt = Bn_s[t];
                const float eG = __shfl_sync(0xffffffffu, eg_l, t);
                float u, o;
                if constexpr (MMA && NT >= 8 && FOLD) {
                    u = bt * (vt - fmaf(eG, av[(wt * NT + t) * 32 + row], acc_k));
                    o = fmaf(eG, bv[(wt * NT + t) * 32 + row], acc_q);
                } else if constexpr (MMA) {
                    // (S0 k_t, S0 q_t) of this row from the fragment holder: lane
                    // 4 (row % 8) + t % 4 holds rows g, g + 8 of each m-tile
                    static_assert(!MMA || WPT == 1, "row = lane");
                    const int src = 4 * (row & 7) + (t & 3), j = t >> 2;
                    const float a00 = __shfl_sync(0xffffffffu, macc[0][j][0], src);
                    const float a08 = __shfl_sync(0xffffffffu, macc[0][j][2], src);
                    const float a10 = __shfl_sync(0xffffffffu, macc[MMA ? 1 : 0][j][0], src);
                    const float a18 = __shfl_sync(0xffffffffu, macc[MMA ? 1 : 0][j][2], src);
                    const float b00 = __shfl_sync(0xffffffffu, macc[0][j][1], src);
                    const float b08 = __shfl_sync(0xffffffffu, macc[0][j][3], src);
                    const float b10 = __shfl_sync(0xffffffffu, macc[MMA ? 1 : 0][j][1], src);
                    const float b18 = __shfl_sync(0xffffffffu, macc[MMA ? 1 : 0][j][3], src);
                    const float ar = row < 16 ? (row & 8 ? a08 : a00) : (row & 8 ? a18 : a10);
                    const float br = row < 16 ? (row & 8 ? b08 : b00) : (row & 8 ? b18 : b10);
                    u = bt * (vt - fmaf(eG, ar, acc_k));
                    o = fmaf(eG, br, acc_q);
                } else if (HAS_STATE) {
                    u = bt * (vt - fmaf(eG, av[(wt * NT + t) * 32 + row], acc_k));
                    o = fmaf(eG, bv[(wt * NT + t) * 32 + row], acc_q);
                } else {
                    u = bt * (vt - acc_k);
                    o = acc_q;
                }
                if (dm.variant != 0) u = vt;   // no delta rule: the buffered value is v_t itself
                const UT us = from_f<UT>(u);
                un[t] = to_f(us);                      // the stored (rounded) value
                o = fmaf(cq[(j0 + t) * NTP], un[t], o);
                if (sub == 0) {
                    if (dm.validate && !isfinite(vt)) bad |= 0x4u;
                    if (obase) obase[t * ostr] = o;
                    const int2 rp = recpos(t);
                    const size_t bh = (size_t)rp.x * Hv + h;
                    if constexpr (PFOLD) {
                        // (folded in this kernel: the delta value is not buffered)
                    } else if (!PG || !a.p.btab) ubase[t * kUSub] = us;   // (contiguous records: position j0 + t of slot r)
                    else static_cast<UT *>(a.p.U)[((bh * (kD / kUSub) + tile) * dm.bt + rp.y) * kUSub + row] = us;
                    if (dm.keep_raw) {
                        static_cast<InT *>(a.p.V)[(bh * dm.bt + rp.y) * kD + drow] = v_s[t * TPC * 32 + wt * 32 + row];
                        if (tile == 0 && row == 0) a.p.B[bh * dm.bt + rp.y] = bt;
                    }
                }
            }
        }
        if constexpr (DFOLD) {
            if (J == dm.C) {   // CTA-uniform
                // S_new = e^{G_t} S0 + U~ K,  U~[row][i] = e^{G_t-G_i} u_i[row] on the
                // warp-level tensor cores: per warp D[32 rows x 128] = U~ [32 x J] . K [J x 128]
                // (split TF32: U~ hi + lo; bf16 keys exact, fp32 keys hi + lo), J padded to 8
                const float gt = Gn_s[0];
                const float eG = expf(gt);
                const int g = lane >> 2, t4 = lane & 3;
                const int KS = (J + 7) / 8;
                auto key = [&](int i, int c) -> float { return i < J ? to_f(i < j0 ? K_s[i * kD + c] : k_s[c]) : 0.f; };
                float *Sw = const_cast<float *>(S_s) + (size_t)wt * 32 * kD;
                // A = U~ fragments in registers, once: U~[row][i] = e^{G_t-G_i} u_i[row] from the
                // staged records (i < j0) and the new token's u_t (i = j0, lane `row` holds it)
                const UT *uw = U_s + (size_t)wt * j0 * kUSub;
                uint32_t fhi[kFusedFoldMaxC / 8][2][4], flo[kFusedFoldMaxC / 8][2][4];
#pragma unroll
                for (int ks = 0; ks < kFusedFoldMaxC / 8; ++ks) {
                    if (ks < KS) {
#pragma unroll
                        for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                const int rr = mt * 16 + g + (q & 1) * 8, i = ks * 8 + t4 + (q >> 1) * 4;
                                const float un_r = __shfl_sync(0xffffffffu, un[0], rr);
                                float x = 0.f;
                                if (i < j0) x = expf(gt - G_s[i]) * to_f(uw[(size_t)i * kUSub + rr]);
                                else if (i == j0) x = un_r;
                                const uint32_t hi = __float_as_uint(x) & 0xFFFFE000u;
                                fhi[ks][mt][q] = hi;
                                flo[ks][mt][q] = __float_as_uint(x - __uint_as_float(hi));
                            }
                        }
                    }
                }
#pragma unroll 1
                for (int ng = 0; ng < kD / 32; ++ng) {
                    float acc[2][4][4];
#pragma unroll
                    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                        for (int nt = 0; nt < 4; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = acc[mt][nt][2] = acc[mt][nt][3] = 0.f;
#pragma unroll
                    for (int ks = 0; ks < kFusedFoldMaxC / 8; ++ks) {
                        if (ks >= KS) break;
                        const uint32_t (&ahi)[2][4] = fhi[ks];
                        const uint32_t (&alo)[2][4] = flo[ks];
#pragma unroll
                        for (int nt = 0; nt < 4; ++nt) {
                            const int c = ng * 32 + nt * 8 + g;
                            const float b0 = key(ks * 8 + t4, c), b1 = key(ks * 8 + t4 + 4, c);
                            const uint32_t h0 = __float_as_uint(b0) & 0xFFFFE000u, h1 = __float_as_uint(b1) & 0xFFFFE000u;
#pragma unroll
                            for (int mt = 0; mt < 2; ++mt) {
                                mma_tf32_16x8x8(acc[mt][nt], ahi[mt], h0, h1);
                                mma_tf32_16x8x8(acc[mt][nt], alo[mt], h0, h1);
                                if constexpr (isz == 4)   // fp32 keys: + U~_hi . K_lo
                                    mma_tf32_16x8x8(acc[mt][nt], ahi[mt],
                                                    __float_as_uint(b0 - __uint_as_float(h0)),
                                                    __float_as_uint(b1 - __uint_as_float(h1)));
                            }
                        }
                    }
                    // epilogue: rows g, g + 8 of each m-tile, columns 2 t4, 2 t4 + 1
#pragma unroll
                    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                        for (int nt = 0; nt < 4; ++nt) {
                            const int c = ng * 32 + nt * 8 + 2 * t4;
                            float2 *p0 = reinterpret_cast<float2 *>(Sw + (size_t)(mt * 16 + g) * kD + c);
                            float2 *p1 = reinterpret_cast<float2 *>(Sw + (size_t)(mt * 16 + g + 8) * kD + c);
                            const float2 s0 = *p0, s1 = *p1;
                            *p0 = make_float2(fmaf(eG, s0.x, acc[mt][nt][0]), fmaf(eG, s0.y, acc[mt][nt][1]));
                            *p1 = make_float2(fmaf(eG, s1.x, acc[mt][nt][2]), fmaf(eG, s1.y, acc[mt][nt][3]));
                        }
                }
            }
        }
        if constexpr (PFOLD) {
            {   // a prefill chunk from an empty buffer (j0 == 0)
                // S_new = e^{G_last} S0 + sum_t e^{G_last - G_t} u_t k_t^T for the
                // chunk's n_new records, in the swizzled state tile, per warp
                // D[32 rows x 128] = Y [32 x n_new] . K [n_new x 128] on mma.sync tf32
                // (Y = e^{G_last - G_t} u_t split hi + lo; bf16 keys exact, fp32 keys
                // hi + lo); the record index inside each 8-token k-step is permuted
                // (slot t <-> token 2t, slot t + 4 <-> 2t + 1) so a B fragment is the
                // key pair of two consecutive tokens; the A fragments are gathered
                // from the rows' lanes by shuffles
                const int g = lane >> 2, t4 = lane & 3;
                const float gl = Gn_s[n_new - 1], eGl = expf(gl);
                constexpr int KSN = (NT + 7) / 8;
                float yv[NT];
#pragma unroll
                for (int t = 0; t < NT; ++t) yv[t] = t < n_new ? expf(gl - Gn_s[t]) * un[t] : 0.f;
                uint32_t yh[KSN][2][4], yl[KSN][2][4];
#pragma unroll
                for (int ks = 0; ks < KSN; ++ks)
#pragma unroll
                    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            // a_q = Y[row mt*16 + g + 8 (q & 1)][token ks*8 + 2 t4 + (q >> 1)]
                            const int src = mt * 16 + g + 8 * (q & 1), e = q >> 1;
                            float v = 0.f;
#pragma unroll
                            for (int tt = 0; tt < 4; ++tt) {
                                const int t = ks * 8 + 2 * tt + e;
                                const float x = __shfl_sync(0xffffffffu, t < NT ? yv[t < NT ? t : 0] : 0.f, src);
                                if (tt == t4) v = x;
                            }
                            const uint32_t hi = __float_as_uint(v) & 0xFFFFE000u;
                            yh[ks][mt][q] = hi;
                            yl[ks][mt][q] = __float_as_uint(v - __uint_as_float(hi));
                        }
                auto kval = [&](int t, int c) -> float { return t < n_new ? to_f(k_s[(size_t)t * TS + c]) : 0.f; };
#pragma unroll 1
                for (int ng = 0; ng < kD / 32; ++ng) {
                    float acc[2][4][4] = {};
#pragma unroll
                    for (int ks = 0; ks < KSN; ++ks) {
#pragma unroll
                        for (int nt = 0; nt < 4; ++nt) {
                            const int c = ng * 32 + nt * 8 + g;
                            const float b0 = kval(ks * 8 + 2 * t4, c), b1 = kval(ks * 8 + 2 * t4 + 1, c);
                            const uint32_t h0 = __float_as_uint(b0) & 0xFFFFE000u, h1 = __float_as_uint(b1) & 0xFFFFE000u;
#pragma unroll
                            for (int mt = 0; mt < 2; ++mt) {
                                mma_tf32_16x8x8(acc[mt][nt], yh[ks][mt], h0, h1);
                                mma_tf32_16x8x8(acc[mt][nt], yl[ks][mt], h0, h1);
                                if constexpr (isz == 4)   // fp32 keys: + Y_hi . K_lo
                                    mma_tf32_16x8x8(acc[mt][nt], yh[ks][mt], __float_as_uint(b0 - __uint_as_float(h0)),
                                                    __float_as_uint(b1 - __uint_as_float(h1)));
                            }
                        }
                    }
                    // S = e^{G_last} S + D at rows R = wt*32 + mt*16 + g (+8), columns c, c + 1
                    unsigned char *Sb = const_cast<unsigned char *>(S_base);
#pragma unroll
                    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                        for (int nt = 0; nt < 4; ++nt) {
                            const int c = ng * 32 + nt * 8 + 2 * t4;
#pragma unroll
                            for (int rh = 0; rh < 2; ++rh) {
                                const int R = wt * 32 + mt * 16 + g + 8 * rh;
                                float2 *p = reinterpret_cast<float2 *>(
                                    Sb + (c >> 5) * (TPC * 4096) + R * 128 + ((((c & 31) >> 2) ^ (R & 7)) << 4) + (c & 3) * 4);
                                const float2 sv = *p;
                                *p = make_float2(fmaf(eGl, sv.x, acc[mt][nt][2 * rh]), fmaf(eGl, sv.y, acc[mt][nt][2 * rh + 1]));
                            }
                        }
                }
            }
        }
    }
    if constexpr (PFOLD) {
        {   // the CTA's folded rows leave as TMA box stores
            fence_proxy_async_smem();
            __syncthreads();
            if (tid == 0) {
                const int row0 = (int)((sb * Hv + h) * kD) + tile0 * 32;
#pragma unroll
                for (int kb = 0; kb < 4; ++kb)
#pragma unroll
                    for (int x = 0; x < TPC; ++x)
                        tma_store_2d(&tmap, S_base + kb * (TPC * 4096) + x * 4096, kb * 32, row0 + x * 32);
                bulk_commit();
            }
        }
    }
    if constexpr (DFOLD) {
        if (J == dm.C) {   // CTA-uniform: one bulk store of the CTA's folded rows
            fence_proxy_async_smem();
            __syncthreads();
            if (tid == 0) {
                bulk_s2g(a.p.state + ((sb * Hv + h) * kD + (size_t)tile0 * 32) * kD, S_s, TPC * 32 * kD * 4);
                bulk_commit();
            }
        }
    }
    CK_MARK(7);
    // ---- 4. records: k_t once per QK head, G_t per V head (first tile group)
    if (tg == 0) {
        if constexpr (PG) {
            auto recpos = [&](int t) -> int2 {
                if (!a.p.btab) return make_int2(r, j0 + t);
                return make_int2(__ldcg(a.p.btab + (size_t)r * dm.maxb + (dm.bt_shift >= 0 ? (j0 + t) >> dm.bt_shift : (j0 + t) / dm.bt)),
                                 dm.bt_shift >= 0 ? (j0 + t) & (dm.bt - 1) : (j0 + t) % dm.bt);
            };
            if (h % dm.g == 0) {
                for (int idx = tid; idx < n_new * kD; idx += NTHR) {
                    const int2 rp = recpos(idx / kD);
                    static_cast<InT *>(a.p.K)[(((size_t)rp.x * Hk + hk) * dm.bt + rp.y) * kD + idx % kD] =
                        k_s[(idx / kD) * TS + idx % kD];
                }
            }
            if (tid < n_new) {
                const int2 rp = recpos(tid);
                a.p.G[((size_t)rp.x * Hv + h) * dm.bt + rp.y] = Gn_s[tid];
            }
        } else {
            if (h % dm.g == 0) {
                InT *Kdst = static_cast<InT *>(a.p.K) + (((size_t)r * Hk + hk) * T + j0) * kD;
                for (int idx = tid; idx < n_new * kD; idx += NTHR) Kdst[idx] = k_s[(idx / kD) * TS + idx % kD];
            }
            if (tid < n_new) a.p.G[((size_t)r * Hv + h) * T + j0 + tid] = Gn_s[tid];
        }
    }
    if (a.kind != CK_VERIFY && tid == 0 && ticket == (int)(gridDim.x * gridDim.y) - 1) {
        a.p.ticket[r] = 0;
        if (direct) a.p.len[r] = J;
        else a.p.occ[r] = ((DFOLD && J == dm.C) || PFOLD) ? 0 : J;
    }
    if (bad) atomicOr(a.p.status, bad);
    CK_MARK(3);
    if constexpr (DFOLD) {
        if (J == dm.C && tid == 0) bulk_wait_read0();   // shared memory stays live until the store has read it
    }
    if constexpr (PFOLD) {
        if (tid == 0) bulk_wait_read0();
    }
}

// ---------------------------------------------------------------- launch
template <typename InT, typename UT, int TPC, int WPT, int NT, bool HAS_STATE, int MBO = 0, bool TC = false,
          bool FOLD = false, bool MMA = false>
static cudaError_t launch_cfg(const ChunkArgs &a, cudaStream_t s) {
    constexpr int MINB = MBO ? MBO : (NT <= 2 ? (HAS_STATE ? 12 / (TPC * WPT) : 2) : 1);
    const CtaLayout L = cta_layout(TPC, NT, HAS_STATE, a.j0_cap, sizeof(InT), sizeof(UT), TC, FOLD, MMA, MINB < 1 ? 1 : MINB);
    if (L.bytes > 227 * 1024) return cudaErrorInvalidConfiguration;
    if (a.n > kMaxSlotsPerLaunch) return cudaErrorInvalidConfiguration;
    // pools / index lists: the PG instantiation (not for the TC or fused-fold kinds)
    const bool pg = a.slots || a.pos || a.p.btab || a.p.sidx;
    if (pg && (TC || (FOLD && !MMA))) return cudaErrorInvalidValue;
    auto kfn = pg ? chunk_cta_kernel<InT, UT, TPC, WPT, NT, HAS_STATE, MINB < 1 ? 1 : MINB, TC && !TC, FOLD && MMA, MMA, true>
                  : chunk_cta_kernel<InT, UT, TPC, WPT, NT, HAS_STATE, MINB < 1 ? 1 : MINB, TC, FOLD, MMA, false>;
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.bytes);
    if (e != cudaSuccess) return e;
    if (a.dry) return cudaSuccess;
    // the whole L1 / shared carveout for shared memory: CTAs per SM are bounded
    // by registers and shared memory only, never by the driver's default split
    e = cudaFuncSetAttribute(kfn, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;   // configuration check only (all-or-nothing pre-pass)
    CUtensorMap tm;
    if (TC || MMA) tm = *static_cast<const CUtensorMap *>(a.tmap);
    else if (!HAS_STATE && a.tmapk) tm = *static_cast<const CUtensorMap *>(a.tmapk);   // (direct: the key records)
    else memset(&tm, 0, sizeof(tm));
    return launch_k(kfn, dim3(4 / TPC, a.dm.Hv, a.n), dim3(TPC * WPT * 32), L.bytes, s, a.pdl != 0, a, tm);
}

template <typename InT, typename UT, int TPC, int WPT, bool HAS_STATE, int MBO = 0, bool TC = false, bool MMA = false>
static cudaError_t launch_nt(const ChunkArgs &a, cudaStream_t s) {
    if (!TC && !MMA && a.n_new == 1) return launch_cfg<InT, UT, TPC, WPT, 1, HAS_STATE, MBO, TC>(a, s);
    if constexpr (MMA) {   // (prefill chunk that folds its own records)
        if (a.pfold) {
            if (a.n_new <= 2) return launch_cfg<InT, UT, TPC, WPT, 2, HAS_STATE, MBO, TC, true, MMA>(a, s);
            if (a.n_new <= 4) return launch_cfg<InT, UT, TPC, WPT, 4, HAS_STATE, MBO, TC, true, MMA>(a, s);
            if (a.n_new <= 8) return launch_cfg<InT, UT, TPC, WPT, 8, HAS_STATE, MBO, TC, true, MMA>(a, s);
            return launch_cfg<InT, UT, TPC, WPT, 16, HAS_STATE, MBO, TC, true, MMA>(a, s);
        }
    }
    if (a.n_new <= 2) return launch_cfg<InT, UT, TPC, WPT, 2, HAS_STATE, MBO, TC, false, MMA>(a, s);
    if (a.n_new <= 4) return launch_cfg<InT, UT, TPC, WPT, 4, HAS_STATE, MBO, TC, false, MMA>(a, s);
    if (a.n_new <= 8) return launch_cfg<InT, UT, TPC, WPT, 8, HAS_STATE, MBO, TC, false, MMA>(a, s);
    return launch_cfg<InT, UT, TPC, WPT, 16, HAS_STATE, MBO, TC, false, MMA>(a, s);
}

// Per-dtype, per-kind launchers, each instantiated in its own translation
// unit (chunk_<dtype>_<kind>.cu) so the template instantiations compile in
// parallel.
template <typename InT, typename UT>
cudaError_t launch_direct(const ChunkArgs &a, cudaStream_t s) {
    // direct: at most 128 registers so 4 CTAs (16 warps) share an SM (measured
    // 338 -> 281 us at config 4; 5 CTAs spill more and lose)
    // (short contexts: 5 CTAs per SM at <= 102 registers, k_t / q_t from shared
    //  memory -- measured faster up to ~64 records; longer ones keep the
    //  4-CTA budget with k_t / q_t in registers, faster at 100+ records)
    if (a.j0_cap + a.n_new <= 64) return launch_nt<InT, UT, kDirectTPC, 1, false, 5>(a, s);
    return launch_nt<InT, UT, kDirectTPC, 1, false, 4>(a, s);
}

template <typename InT, typename UT>
cudaError_t launch_state(const ChunkArgs &a, cudaStream_t s) {
    // (1 or 4 tiles per CTA and 2 warps per tile were measured and rejected,
    //  DESIGN.md section 6)
    if (a.fold) {   // decode with the fused fold (host: some slot fills, C <= 32)
        if (a.kind != CK_DECODE || a.n_new != 1 || a.dm.C > kFusedFoldMaxC) return cudaErrorInvalidValue;
        return launch_cfg<InT, UT, kChunkTPC, 1, 1, true, 0, false, true>(a, s);
    }
    // 2 or more new tokens (verify, prefill chunks): the state mat-vecs on the
    // warp-level tensor cores in the 2-warp CTA (mma.sync tf32, no TMEM);
    // the CUDA-core pass is the fallback without a tensor map
    // (8 or more tokens: the whole head per CTA -- the key rows are computed
    // once per head; measured verify N = 8 162 -> 150 us, N = 4 109 -> 123)
    if (a.n_new >= 8 && a.tmap && !a.pfold) return launch_nt<InT, UT, 4, kMmaWPT, true, 0, false, true>(a, s);
    if (a.n_new >= 2 && a.tmap) return launch_nt<InT, UT, kChunkTPC, kMmaWPT, true, 0, false, true>(a, s);
    return launch_nt<InT, UT, kChunkTPC, 1, true>(a, s);
}

cudaError_t launch_direct_f32(const ChunkArgs &a, cudaStream_t s);
cudaError_t launch_direct_bf16(const ChunkArgs &a, cudaStream_t s);
cudaError_t launch_direct_bf16h(const ChunkArgs &a, cudaStream_t s);
cudaError_t launch_state_f32(const ChunkArgs &a, cudaStream_t s);
cudaError_t launch_state_bf16(const ChunkArgs &a, cudaStream_t s);
cudaError_t launch_state_bf16h(const ChunkArgs &a, cudaStream_t s);

}  // namespace labuf
