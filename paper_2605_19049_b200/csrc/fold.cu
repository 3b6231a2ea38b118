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
        const int mode = a.p.mode[r], occ = a.p.occ[r], len = a.p.len[r];
        int n = 0;
        bool zero_s0 = false;
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
            meta[4] = __float_as_int(a.p.G[((size_t)ba.x * Hv + h) * bt + ba.y]);
        }
        if (!a.spec && n > 0 && !zero_s0) {
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
    // d_v rows per CTA.  Every CTA of a TMEM-allocating kernel costs ~0.5 us
    // of SM-serialised launch/allocation time on B200 (tools/microbench_tmem.cu:
    // 3.7 ns per CTA GPU-wide vs 0.64 ns for a plain kernel), so launches where
    // many CTAs fold little or nothing (commits: zero or few accepted drafts)
    // take 64-row CTAs (half the CTAs): config-3 commit 164 -> 127 us.  Full
    // flushes keep 32-row CTAs (more CTAs per SM in flight): 57 vs 62 us.
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
