// fold.cu — kernel (2): batched state update on the 5th-generation tensor cores.
//
//   S_new = e^{G_last} S0 + sum_{i<n} e^{G_last - G_i} u_i k_i^T
//
// n = occ (flush), occ + n_accepted (accepted-prefix commit, Eq. 8), or
// len with S0 = 0 (compression of a direct-mode slot into a state).
// The rank-n update is the one dense contraction of the path:
//   D[c][j] = sum_i  k_i[c] * (w_i u_i[j]),   M = d_k = 128 (TMEM lanes),
//   N = 64 (half of d_v per CTA), K = n tokens in chunks of up to 32,
// issued as tcgen05.mma.kind::tf32 from K-major SWIZZLE_NONE shared-memory
// operands with the fp32 accumulator in TMEM.  fp32 accuracy comes from
// split-TF32 (x = hi + lo): bf16 keys are exact in tf32, so 2 passes
// (K*Whi + K*Wlo); fp32 keys need 3 (Khi*Whi + Khi*Wlo + Klo*Whi).
//
// B200 structure: one CTA of 4 warps per (half of d_v, V head, slot).  At
// entry warp 0 allocates the TMEM accumulator while thread 0 reads the
// slot's counters and puts the 32 KiB S0 half-tile in flight with one bulk
// copy; every thread then loads ALL of its key / delta-value operand
// elements for the chunk in one batch (one memory round trip), converts and
// splits them into the UMMA layouts in shared memory, and thread 0 issues
// the MMAs.  The epilogue reads TMEM (lane = key index c, conflict-free in
// the row-major state tile), adds e^{G_last} S0 in shared memory and one
// bulk store writes S_new back.  Shared memory is sized from the host-known
// largest record count, so 4 CTAs share an SM at C = 16.
#include <cstdlib>

#include "device.cuh"
#include "internal.h"

namespace labuf {

constexpr int kFoldKCMax = 16;   // tokens per MMA staging chunk (max)
constexpr int kFoldThreads = 128;

struct FoldSmem {
    uint32_t S, A, Alo, Bhi, Blo, bar, total;
};
__host__ __device__ inline FoldSmem fold_smem_layout(bool fp32_in, int nj, int kc) {
    FoldSmem L;
    uint32_t o = 0;
    L.S = o;   o += (uint32_t)nj * kD * 4;                 // nj state rows
    L.A = o;   o += (uint32_t)kD * kc * 4;
    L.Alo = o; o += fp32_in ? (uint32_t)kD * kc * 4 : 0;
    L.Bhi = o; o += (uint32_t)nj * kc * 4;
    L.Blo = o; o += (uint32_t)nj * kc * 4;
    L.bar = o; o += 64;
    L.total = o;
    return L;
}

// byte offset of element (row, k) in a K-major SWIZZLE_NONE operand with kc
// columns: 8x(16 B) core matrices, K-adjacent at +128 B (LBO), 8-row groups
// at +kc*32 B (SBO).
__device__ __forceinline__ uint32_t kmaj_off(int row, int k, int kc) {
    return (uint32_t)((row >> 3) * (kc * 32) + (k >> 2) * 128 + (row & 7) * 16 + (k & 3) * 4);
}

// Which records a fold launch folds for slot r (uniform over the slot's
// CTAs): meta[0] = n, meta[1] = S0 is zero (compression), meta[2..3] = the
// branch remap (FK_BRANCH: record i >= meta[2] is record i + meta[3]),
// meta[4] = the last folded record's log decay G_last.
__device__ __forceinline__ size_t recb_h(int2 ba, int Hv, int h, int bt) { return ((size_t)ba.x * Hv + h) * bt + ba.y; }

template <bool PG>
__device__ __forceinline__ void fold_counters(const FoldArgs &a, int r, int zi, int h, int *meta) {
    const Dims &dm = a.dm;
    const int mode = a.p.mode[r], occ = a.p.occ[r], len = a.p.len[r];
    int n = 0;
    bool zero_s0 = false;
    meta[2] = 1 << 30;
    meta[3] = 0;
    if (a.kind == FK_FULL) {
        n = (mode == 0 && occ == dm.C) ? occ : 0;
    } else if (a.kind == FK_FORCE) {
        if (mode == 1) { n = len; zero_s0 = true; } else n = occ;
    } else if (a.kind == FK_FORK) {
        n = a.fork_n;
        zero_s0 = mode == 1;
    } else if (a.kind == FK_BRANCH) {
        int na = a.nacc[zi], br = a.branch[zi];
        if (na < 0 || na > a.n_draft || br < 0 || br >= a.n_branch) {
            if (dm.validate) atomicOr(a.p.status, 0x8u);
            na = na < 0 ? 0 : (na > a.n_draft ? a.n_draft : na);
            br = br < 0 ? 0 : (br >= a.n_branch ? a.n_branch - 1 : br);
        }
        n = occ + na;
        meta[2] = occ;
        meta[3] = br * a.n_draft;
    } else {  // FK_COMMIT
        int na = a.nacc[zi];
        if (na < 0 || na > a.n_draft) {
            if (dm.validate) atomicOr(a.p.status, 0x8u);
            na = na < 0 ? 0 : a.n_draft;
        }
        n = occ + na;
    }
    meta[0] = n;
    meta[1] = zero_s0;
    // the last folded record's log decay, read here with the counters (off
    // the post-barrier critical path); branch commits remap past occ
    if (n > 0) {
        const int last = (a.kind == FK_BRANCH && n - 1 >= occ) ? n - 1 + meta[3] : n - 1;
        const int2 ba = PG ? rec_at(dm, a.p, r, last) : make_int2(r, last);
        meta[4] = __float_as_int(a.p.G[((size_t)ba.x * dm.Hv + h) * dm.bt + ba.y]);
    }
}

// (Mode ii, the UT transform from the raw records, is fold_ut.cu.)
template <typename InT, typename UT, bool FP32_IN, int kFoldNJ, int KCM, bool PG>
__global__ void __launch_bounds__(kFoldThreads, kFoldNJ == 128 ? 2 : (kFoldNJ == 32 && KCM == 16 ? 8 : 4)) fold_kernel(const FoldArgs a) {
    constexpr int NPAR = kFoldThreads / kFoldNJ;   // token parities per B row
    const int jh = blockIdx.x, h = blockIdx.y, zi = blockIdx.z;
    if constexpr (PG) {   // slot lists, state indices and block tables may come from the previous grid
        if (a.pdl) pdl_wait();
    }
    const int r = PG && a.slots ? __ldcg(a.slots + zi) : a.first + zi;
    const int tid = threadIdx.x, warp = tid >> 5;
    const Dims dm = a.dm;
    const int Hv = dm.Hv, bt = dm.bt;
    const int hk = h / dm.g;
    const int KC = a.kc;                           // staging chunk (multiple of 8, <= 32)

    extern __shared__ __align__(1024) unsigned char smem[];
    const FoldSmem L = fold_smem_layout(FP32_IN, kFoldNJ, KC);
    float *S_s = reinterpret_cast<float *>(smem + L.S);
    unsigned char *A = smem + L.A, *Alo = smem + L.Alo, *Bhi = smem + L.Bhi, *Blo = smem + L.Blo;
    uint64_t *bar_ld = reinterpret_cast<uint64_t *>(smem + L.bar);
    uint64_t *bar_mma = bar_ld + 1;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bar_ld + 2);
    int *meta = reinterpret_cast<int *>(bar_ld + 3);      // n, zero_s0, branch occ / offset, G_last
    const size_t sb = PG && a.p.sidx ? (size_t)__ldcg(a.p.sidx + r) : (size_t)r;
    float *state_tile = a.p.state + ((sb * Hv + h) * kD + (size_t)jh * kFoldNJ) * kD;
    // where S_new goes: the slot's own state, or (FK_FORK) the destination slot's
    float *state_out = state_tile;
    if (a.kind == FK_FORK) {
        const size_t db = PG && a.p.sidx ? (size_t)__ldcg(a.p.sidx + a.fork_dst) : (size_t)a.fork_dst;
        state_out = a.p.state + ((db * Hv + h) * kD + (size_t)jh * kFoldNJ) * kD;
    }

    // per-thread operand coordinates: A column c = tid (all KC tokens);
    // B row j = tid % NJ, tokens i = ip (mod NPAR)
    const int c = tid, jb = tid % kFoldNJ, ip = tid / kFoldNJ;
    const int jr = jh * kFoldNJ + jb;
    // record i of the slot (block table or the slot's own region): key row,
    // this thread's delta value u_i[jr] (U is tile-major
    // [blk][Hv][d/kUSub][bt][kUSub]), log decay, raw value, beta
    // (PG: block table lookups; else the slot's own region, block = slot)
    // (FK_BRANCH: record i >= occ of the folded prefix is the accepted branch's
    //  record occ + b n_draft + (i - occ); set once the counters are read)
    int bocc = 1 << 30, boff = 0;
    auto at = [&](int i) -> int2 {
        const int ii = i >= bocc ? i + boff : i;
        return PG ? rec_at(dm, a.p, r, ii) : make_int2(r, ii);
    };
    auto recb = [&](int2 ba) -> size_t { return ((size_t)ba.x * Hv + h) * bt + ba.y; };
    auto rec = [&](int i) -> size_t { return recb(at(i)); };   // (block * Hv + h) * bt + offset
    auto Kb = [&](int2 ba) { return static_cast<const InT *>(a.p.K) + (((size_t)ba.x * dm.Hk + hk) * bt + ba.y) * kD; };
    auto Ub = [&](int2 ba) {
        return static_cast<const UT *>(a.p.U) +
               ((((size_t)ba.x * Hv + h) * (kD / kUSub) + jr / kUSub) * bt + ba.y) * kUSub + jr % kUSub;
    };
    // operands of one chunk: K^T column c, u_i[j], G_i — the first chunk is
    // requested at entry, bounded by the host's record count (in-capacity
    // reads past a slot's own count are never used).  Block tables: one lookup
    // for the chunk's first record; the records that share its block (all of
    // them for chunks of <= 16 inside 16-token blocks) are addressed from it
    float kv[KCM], uv[KCM / NPAR], gv[KCM / NPAR];
    auto load_chunk = [&](int kc0, int kn) {
        // records kc0 .. kc0 + lim - 1 follow b0 in one block (a branch remap
        // inside the chunk: every record through at())
        const int2 b0 = at(kc0);
        const int lim = (kc0 < bocc && kc0 + KCM > bocc) ? 0 : ((PG && a.p.btab) ? bt - b0.y : (1 << 30));
        auto ba_of = [&](int i) -> int2 { return i < lim ? make_int2(b0.x, b0.y + i) : at(kc0 + i); };
#pragma unroll
        for (int i = 0; i < KCM; ++i) kv[i] = (i < kn) ? to_f(Kb(ba_of(i))[c]) : 0.f;
#pragma unroll
        for (int q = 0; q < KCM / NPAR; ++q) {
            const int i = NPAR * q + ip;
            const int2 ba = ba_of(i);
            uv[q] = (i < kn) ? to_f(*Ub(ba)) : 0.f;
            gv[q] = (i < kn) ? a.p.G[recb(ba)] : 0.f;
        }
    };

    // ---- which records fold (uniform over all CTAs of the slot); S0 in flight
    //      at once when the host mirror says every slot of the range folds
    if (warp == 0) tmem_alloc<kFoldNJ>(tmem_slot);
    if (tid == 32) {
        mbar_init(bar_ld, 1);
        mbar_init(bar_mma, 1);
        fence_mbar_init();
        if (a.spec) {
            mbar_arrive_expect_tx(bar_ld, kFoldNJ * kD * 4);
            if (a.pdl_early) bulk_g2s(S_s, state_tile, kFoldNJ * kD * 4, bar_ld);
        }
    }
    if (a.pdl) pdl_wait();   // counters, records (and the state unless pdl_early) may come from the previous grid
    pdl_trigger();
    if (tid == 32) {
        if (a.spec && !a.pdl_early) bulk_g2s(S_s, state_tile, kFoldNJ * kD * 4, bar_ld);
        fold_counters<PG>(a, r, zi, h, meta);
        if (!a.spec && meta[0] > 0 && !meta[1]) {
            mbar_arrive_expect_tx(bar_ld, kFoldNJ * kD * 4);
            bulk_g2s(S_s, state_tile, kFoldNJ * kD * 4, bar_ld);
        }
    }
    if (a.kind != FK_BRANCH) {
        load_chunk(0, min(KC, a.kcap));
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const int n = meta[0];
    const bool zero_s0 = meta[1] != 0;
    if (a.kind == FK_BRANCH) {   // the record remap needs the counters: load after them
        bocc = meta[2];
        boff = meta[3];
        load_chunk(0, min(KC, n));
    }
    const uint32_t tmem = *tmem_slot;
    if (n == 0) {   // nothing to fold: state untouched, counters unchanged
        if (a.spec) mbar_wait(bar_ld, 0);   // the speculative copy must land before exit
        if (warp == 0) tmem_dealloc<kFoldNJ>(tmem);
        return;
    }
    const float g_last = __int_as_float(meta[4]);
    const uint32_t idesc = idesc_tf32(128, kFoldNJ);
    uint32_t mma_phase = 0;

    for (int kc0 = 0; kc0 < n; kc0 += KC) {
        const int kn = min(KC, n - kc0);
        const int kpad = (kn + 7) & ~7;
        if (kc0 > 0) {
            mbar_wait(bar_mma, mma_phase);
            mma_phase ^= 1;
            load_chunk(kc0, kn);
        }
        // ---- A = K^T chunk: row c (d_k), column i (token), zero padded to kpad
#pragma unroll
        for (int i = 0; i < KCM; ++i) {
            if (i < kpad) {
                // columns past this slot's count are zero (the speculative
                // loads may hold other records, even non-finite garbage)
                const float x = i < kn ? kv[i] : 0.f;
                const uint32_t off = kmaj_off(c, i, KC);
                if (FP32_IN) {
                    const float hi = tf32_rna(x);
                    *reinterpret_cast<float *>(A + off) = hi;
                    *reinterpret_cast<float *>(Alo + off) = x - hi;
                } else {
                    *reinterpret_cast<float *>(A + off) = x;   // bf16 values are exact in tf32
                }
            }
        }
        // ---- B = (w_i u_i)^T chunk: row j (d_v), column i, split hi + lo
#pragma unroll
        for (int q = 0; q < KCM / NPAR; ++q) {
            const int i = NPAR * q + ip;
            if (i < kpad) {
                const float y = (i < kn) ? expf(g_last - gv[q]) * uv[q] : 0.f;
                const float hi = tf32_rna(y);
                const uint32_t off = kmaj_off(jb, i, KC);
                *reinterpret_cast<float *>(Bhi + off) = hi;
                *reinterpret_cast<float *>(Blo + off) = y - hi;
            }
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) {
            tc_fence_after();
            for (int kk = 0; kk < kpad / 8; ++kk) {
                const uint32_t koff = kk * 256;   // 8 tf32 = 2 core matrices along K
                const uint64_t da = umma_desc_noswz(smem_u32(A) + koff, 128, KC * 32);
                const uint64_t dbh = umma_desc_noswz(smem_u32(Bhi) + koff, 128, KC * 32);
                const uint64_t dbl = umma_desc_noswz(smem_u32(Blo) + koff, 128, KC * 32);
                tc_mma_tf32(tmem, da, dbh, idesc, (kc0 > 0 || kk > 0) ? 1u : 0u);
                tc_mma_tf32(tmem, da, dbl, idesc, 1u);
                if (FP32_IN) {
                    const uint64_t dal = umma_desc_noswz(smem_u32(Alo) + koff, 128, KC * 32);
                    tc_mma_tf32(tmem, dal, dbh, idesc, 1u);
                }
            }
            tc_commit(bar_mma);
        }
        __syncwarp();
    }
    mbar_wait(bar_mma, mma_phase);
    tc_fence_after();
    if (!zero_s0) mbar_wait(bar_ld, 0);

    // ---- epilogue: S_new[j][c] = e^{G_last} S0[j][c] + D[c][j]; thread owns key index c
    const float eG = expf(g_last);
#pragma unroll
    for (int cc = 0; cc < kFoldNJ / 32; ++cc) {
        float v[32];
        tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(cc * 32), v);
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) {
            float *p = S_s + (size_t)(cc * 32 + jj) * kD + c;
            *p = zero_s0 ? v[jj] : fmaf(eG, *p, v[jj]);
        }
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
        bulk_s2g(state_out, S_s, kFoldNJ * kD * 4);
        bulk_commit();
    }
    if (warp == 0) tmem_dealloc<kFoldNJ>(tmem);

    // ---- counters: last CTA of the slot resets the buffer
    if (tid == 0) {
        const int nct = gridDim.x * gridDim.y;
        if (a.kind != FK_FORK && atomicAdd(&a.p.ticket[r], 1) == nct - 1) {
            a.p.ticket[r] = 0;
            a.p.occ[r] = 0;
            if (zero_s0) { a.p.mode[r] = 0; a.p.len[r] = 0; }
        }
        bulk_wait_read0();   // shared memory must stay live until the store has read it
    }
}

// Warp-MMA form of kernel (2): the same fold with the rank-n update on
// mma.sync (m16n8k8 tf32, fp32 accumulate in registers) and no TMEM.
// Allocating TMEM costs every CTA ~0.5 us of SM-serialised time
// (tools/microbench_tmem.cu), ~30 us per SM over a config-2 flush's 8192
// CTAs; this form drops it.  One 4-warp CTA per (32 d_v rows, V head,
// slot): the 16 KiB S0 tile streams into shared memory with one bulk copy
// and the chunk's key rows and u values with cp.async, so the registers hold
// only the accumulators (64 registers: 8 CTAs per SM, 128 KiB of state in
// flight per SM; 7 with block tables).
// Warp w owns key columns c in [32 w, 32 w + 32).  The MMA rows (M) are key
// columns and the columns (N) d_v rows, both permuted so that every
// thread's accumulators are whole float4 rows of the state: M row g / g + 8
// of m-tile mt is column c0 + 2 mt + 0 / 1 (c0 = 32 w + 4 g), N column n of
// n-tile nt is d_v row 4 n + nt.  Thread (g, t) then holds S[j][c0 .. c0 +
// 3] for j = 8 t + 4 p + nt (p, nt in 0..1 x 0..3); the epilogue adds
// e^{G_last} S0 from shared memory (float4, conflict-free) and stores the
// rows straight to HBM (128 B per 8 lanes).  fp32 accuracy: split-TF32 as
// in the tcgen05 form (bf16 keys exact; fp32 keys split too).
template <typename InT, typename UT, bool FP32_IN, bool PG, int MINB>
__global__ void __launch_bounds__(kFoldThreads, MINB) fold_wm_kernel(const FoldArgs a) {
    static_assert(kUSub == 32, "one U sub-tile per CTA");
    constexpr int KB = kD * (int)sizeof(InT);   // bytes per key row
    constexpr int UB = 32 * (int)sizeof(UT);    // bytes of u_i per CTA
    const int jh = blockIdx.x, h = blockIdx.y, zi = blockIdx.z;
    if constexpr (PG) {
        if (a.pdl) pdl_wait();
    }
    const int r = PG && a.slots ? __ldcg(a.slots + zi) : a.first + zi;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const Dims dm = a.dm;
    const int Hv = dm.Hv, bt = dm.bt, hk = h / dm.g;
    __shared__ __align__(128) float S_s[32 * kD];
    __shared__ __align__(128) unsigned char K_s[16 * KB];
    __shared__ __align__(128) unsigned char U_s[16 * UB];
    __shared__ uint64_t bar_ld;
    __shared__ int meta[5];
    const size_t sb = PG && a.p.sidx ? (size_t)__ldcg(a.p.sidx + r) : (size_t)r;
    const float *state_tile = a.p.state + ((sb * Hv + h) * kD + (size_t)jh * 32) * kD;
    float *state_out = const_cast<float *>(state_tile);
    if (a.kind == FK_FORK) {
        const size_t db = PG && a.p.sidx ? (size_t)__ldcg(a.p.sidx + a.fork_dst) : (size_t)a.fork_dst;
        state_out = a.p.state + ((db * Hv + h) * kD + (size_t)jh * 32) * kD;
    }
    const int c0 = warp * 32 + 4 * g;

    int bocc = 1 << 30, boff = 0;
    auto at = [&](int i) -> int2 {
        const int ii = i >= bocc ? i + boff : i;
        return PG ? rec_at(dm, a.p, r, ii) : make_int2(r, ii);
    };
    // chunk kc0 .. kc0 + kn - 1: key rows and u values into shared memory
    // (cp.async), this thread's log decays G for tokens t + 4 s into gv
    float gv[4];
    auto load_chunk = [&](int kc0, int kn) {
        const int2 b0 = at(kc0);
        const int lim = (kc0 < bocc && kc0 + 16 > bocc) ? 0 : ((PG && a.p.btab) ? bt - b0.y : (1 << 30));
        auto ba_of = [&](int i) -> int2 { return i < lim ? make_int2(b0.x, b0.y + i) : at(kc0 + i); };
#pragma unroll
        for (int q = 0; q < 16 * KB / 16 / kFoldThreads; ++q) {
            const int idx = q * kFoldThreads + tid, i = idx / (KB / 16), seg = idx % (KB / 16);
            if (i < kn) {
                const int2 ba = ba_of(i);
                cp_async16(K_s + i * KB + seg * 16,
                           reinterpret_cast<const unsigned char *>(a.p.K) +
                               ((((size_t)ba.x * dm.Hk + hk) * bt + ba.y) * kD) * sizeof(InT) + seg * 16);
            }
        }
        if (tid < 16 * UB / 16) {
            const int i = tid / (UB / 16), seg = tid % (UB / 16);
            if (i < kn) {
                const int2 ba = ba_of(i);
                cp_async16(U_s + i * UB + seg * 16,
                           reinterpret_cast<const unsigned char *>(a.p.U) +
                               (((((size_t)ba.x * Hv + h) * (kD / kUSub) + jh) * bt + ba.y) * kUSub) * sizeof(UT) + seg * 16);
            }
        }
        cp_async_commit();
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const int i = t + 4 * s;
            gv[s] = i < kn ? a.p.G[recb_h(ba_of(i), Hv, h, bt)] : 0.f;
        }
    };

    if (tid == 32) {
        mbar_init(&bar_ld, 1);
        fence_mbar_init();
        if (a.spec) {
            mbar_arrive_expect_tx(&bar_ld, 32 * kD * 4);
            if (a.pdl_early) bulk_g2s(S_s, state_tile, 32 * kD * 4, &bar_ld);
        }
    }
    if (a.pdl) pdl_wait();   // counters, records (and the state unless pdl_early) may come from the previous grid
    pdl_trigger();
    if (tid == 32) {
        if (a.spec && !a.pdl_early) bulk_g2s(S_s, state_tile, 32 * kD * 4, &bar_ld);
        fold_counters<PG>(a, r, zi, h, meta);
        if (!a.spec && meta[0] > 0 && !meta[1]) {
            mbar_arrive_expect_tx(&bar_ld, 32 * kD * 4);
            bulk_g2s(S_s, state_tile, 32 * kD * 4, &bar_ld);
        }
    }
    if (a.kind != FK_BRANCH) load_chunk(0, min(16, a.kcap));
    __syncthreads();
    const int n = meta[0];
    const bool zero_s0 = meta[1] != 0;
    if (n == 0) {   // nothing to fold: state untouched, counters unchanged
        cp_async_wait_all();
        if (a.spec) mbar_wait(&bar_ld, 0);   // the speculative copy must land before exit
        return;
    }
    if (a.kind == FK_BRANCH) {
        bocc = meta[2];
        boff = meta[3];
        load_chunk(0, min(16, n));
    }
    const float g_last = __int_as_float(meta[4]);
    float acc[2][4][4] = {};   // [mt][nt][fragment]
#pragma unroll 1
    for (int kc0 = 0; kc0 < n; kc0 += 16) {
        const int kn = min(16, n - kc0);
        if (kc0 > 0) {
            __syncthreads();   // every warp is done with the previous chunk
            load_chunk(kc0, kn);
        }
        cp_async_wait_all();
        __syncthreads();
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
            if (8 * ks >= kn) break;
            // tokens A = 8 ks + t (k = t), B = A + 4 (k = t + 4); past the
            // slot's count: zero keys and weights (shared memory holds garbage)
            const int ia = 8 * ks + t, ib = ia + 4;
            const bool va = ia < kn, vb = ib < kn;
            const float wa = va ? expf(g_last - gv[2 * ks]) : 0.f;
            const float wb = vb ? expf(g_last - gv[2 * ks + 1]) : 0.f;
            const float4 ua = load4(reinterpret_cast<const UT *>(U_s + ia * UB) + 4 * g);
            const float4 ub = load4(reinterpret_cast<const UT *>(U_s + ib * UB) + 4 * g);
            // (rows past the loaded count may hold another CTA's bytes: select, never scale)
            const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
            const float4 ka = va ? load4(reinterpret_cast<const InT *>(K_s + ia * KB) + c0) : z4;
            const float4 kb = vb ? load4(reinterpret_cast<const InT *>(K_s + ib * KB) + c0) : z4;
            const float af[2][4] = {{ka.x, ka.y, kb.x, kb.y}, {ka.z, ka.w, kb.z, kb.w}};
            uint32_t ah[2][4], al[2][4];
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float hi = FP32_IN ? tf32_rna(af[mt][e]) : af[mt][e];   // bf16 keys are exact in tf32
                    ah[mt][e] = __float_as_uint(hi);
                    al[mt][e] = __float_as_uint(af[mt][e] - hi);
                }
            // d_v row 4 g + nt of tokens A / B: one n-tile at a time (few live registers)
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
                const float ya = va ? wa * (nt == 0 ? ua.x : nt == 1 ? ua.y : nt == 2 ? ua.z : ua.w) : 0.f;
                const float yb = vb ? wb * (nt == 0 ? ub.x : nt == 1 ? ub.y : nt == 2 ? ub.z : ub.w) : 0.f;
                const float ha = tf32_rna(ya), hb = tf32_rna(yb);
                const uint32_t bh0 = __float_as_uint(ha), bl0 = __float_as_uint(ya - ha);
                const uint32_t bh1 = __float_as_uint(hb), bl1 = __float_as_uint(yb - hb);
#pragma unroll
                for (int mt = 0; mt < 2; ++mt) {
                    mma_tf32_16x8x8(acc[mt][nt], ah[mt], bl0, bl1);
                    if (FP32_IN) mma_tf32_16x8x8(acc[mt][nt], al[mt], bh0, bh1);
                    mma_tf32_16x8x8(acc[mt][nt], ah[mt], bh0, bh1);
                }
            }
        }
    }
    // ---- epilogue: S_new[j][c] = e^{G_last} S0[j][c] + D[c][j]
    if (!zero_s0) mbar_wait(&bar_ld, 0);
    const float eG = expf(g_last);
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
            const int j = 8 * t + 4 * p + nt;
            float4 v = make_float4(acc[0][nt][p], acc[0][nt][p + 2], acc[1][nt][p], acc[1][nt][p + 2]);
            if (!zero_s0) {
                const float4 x = *reinterpret_cast<const float4 *>(S_s + j * kD + c0);
                v = make_float4(fmaf(eG, x.x, v.x), fmaf(eG, x.y, v.y), fmaf(eG, x.z, v.z), fmaf(eG, x.w, v.w));
            }
            __stcs(reinterpret_cast<float4 *>(state_out + j * kD + c0), v);
        }

    // ---- counters: last CTA of the slot resets the buffer
    if (tid == 0) {
        const int nct = gridDim.x * gridDim.y;
        if (a.kind != FK_FORK && atomicAdd(&a.p.ticket[r], 1) == nct - 1) {
            a.p.ticket[r] = 0;
            a.p.occ[r] = 0;
            if (zero_s0) { a.p.mode[r] = 0; a.p.len[r] = 0; }
        }
    }
}

template <typename InT, typename UT, bool FP32_IN, int MINB>
static cudaError_t launch_fold_wm(const FoldArgs &a, cudaStream_t s) {
    const bool pg = a.slots || a.p.btab || a.p.sidx;
    // (block-table addressing needs a few more registers: one CTA per SM fewer, no spills)
    auto kfn = pg ? fold_wm_kernel<InT, UT, FP32_IN, true, MINB - 1> : fold_wm_kernel<InT, UT, FP32_IN, false, MINB>;
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;
    return launch_k(kfn, dim3(kD / 32, a.dm.Hv, a.n), dim3(kFoldThreads), 0, s, a.pdl != 0, a);
}

template <typename InT, typename UT, bool FP32_IN, int NJ, int KCM>
static cudaError_t launch_fold_cfg(const FoldArgs &a, cudaStream_t s) {
    const FoldSmem L = fold_smem_layout(FP32_IN, NJ, a.kc);
    const bool pg = a.slots || a.p.btab || a.p.sidx;
    auto kfn = pg ? fold_kernel<InT, UT, FP32_IN, NJ, KCM, true> : fold_kernel<InT, UT, FP32_IN, NJ, KCM, false>;
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
    if (e != cudaSuccess) return e;
    // the whole L1 / shared carveout for shared memory: CTAs per SM are bounded
    // by registers and shared memory only, never by the driver's default split
    e = cudaFuncSetAttribute(kfn, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;
    return launch_k(kfn, dim3(kD / NJ, a.dm.Hv, a.n), dim3(kFoldThreads), L.total, s, a.pdl != 0, a);
}

template <typename InT, typename UT, bool FP32_IN>
static cudaError_t launch_fold_t(const FoldArgs &a, cudaStream_t s) {
    // Flushes and compressions take the warp-MMA form (no TMEM allocation
    // per CTA): config-2 flush 59.1 -> 57.1 us, config 5 (paged, mixed)
    // 40.0 -> 36.1 ms per step.  Accepted-draft commits keep the tcgen05 form
    // with 64-row CTAs: their state request waits for the counters (the host
    // cannot tell which slots fold), and there the 64-row tcgen05 CTA wins
    // (config-3 commit 136 vs 145 us; profiles/r2h); commits where every
    // slot holds buffered records (a.spec) take the warp-MMA form too.
    // LABUF_FOLD=tc|wm
    // forces one form (A/B).
    static const int fold_form = [] {
        const char *e = getenv("LABUF_FOLD");
        return !e ? -1 : (e[0] == 't' ? 0 : 1);
    }();
    if (fold_form == 1 || (fold_form < 0 && ((a.kind != FK_COMMIT && a.kind != FK_BRANCH) || a.spec))) return launch_fold_wm<InT, UT, FP32_IN, 8>(a, s);
    const int nj = a.spec ? 32 : 64;
    if (nj == 64) return launch_fold_cfg<InT, UT, FP32_IN, 64, kFoldKCMax>(a, s);
    return launch_fold_cfg<InT, UT, FP32_IN, 32, kFoldKCMax>(a, s);
}

cudaError_t launch_fold(const FoldArgs &a_in, cudaStream_t s, int64_t *launches) {
    if (a_in.n <= 0) return cudaSuccess;
    FoldArgs a = a_in;
    if (a.n > kMaxSlotsPerLaunch) return cudaErrorInvalidConfiguration;
    // staging chunk: the largest record count of the launch, rounded to the
    // MMA K granule (8), at most 32 (longer folds loop over chunks)
    int kc = (a.kcap + 7) & ~7;
    // staging chunk of at most 16 tokens: longer folds (C = 22, 32, commits of
    // occ + n_acc > 16) loop over 16-token chunks in the small-footprint CTA
    // (8 per SM) -- measured C = 22: 99 -> 75 us, C = 32: 104 -> 85 us per
    // flush against 32-token chunks at 4 CTAs/SM.
    a.kc = kc < 8 ? 8 : (kc > kFoldKCMax ? kFoldKCMax : kc);
    cudaError_t e;
    if (a.raw)
        e = launch_fold_ut(a, s);
    else if (a.dm.in_dt == DT_F32)
        e = launch_fold_t<float, float, true>(a, s);
    else if (a.dm.u_dt == DT_F16)
        e = launch_fold_t<__nv_bfloat16, __half, false>(a, s);
    else
        e = launch_fold_t<__nv_bfloat16, float, false>(a, s);
    if (e == cudaSuccess) ++*launches;
    return e;
}

}  // namespace labuf
