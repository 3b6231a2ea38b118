// fold_ut.cu — kernel (2 RAW): flush mode ii.  The delta values are not read
// from the buffer but recomputed from the raw records (k_i, v_i, beta_i, G_i)
// and the state by the chunkwise UT transform of P:392-399 (K~ corrected per
// reading Z4), then folded into the state:
//
//   L      = strictLower(Diag(beta) (Gamma (.) K K^T))          Gamma_il = e^{G_i - G_l}
//   A      = (I + L)^{-1}
//   K~     = A Diag(beta) Diag(gamma) K,   V~ = A Diag(beta) V    gamma_i = e^{G_i}
//   U      = V~ - K~ S^T                                          (u_i rows)
//   S_new  = gamma_last S + sum_i e^{G_last - G_i} u_i k_i^T
//
// over chunks of up to 16 records (G relative to the chunk's entering state;
// a longer fold chains chunks through the state held in shared memory).
//
// B200 structure: a persistent CTA per SM walks its (V head, slot) units
// with the state double-buffered, so the next unit's 64 KiB state and raw
// records stream in while the current unit computes.
//   * producer warp: per unit, once the buffer is free, reads the slot's
//     counters, requests the state as 16 TMA boxes (32 x 32 fp32, 128-byte
//     swizzle) on four mbarriers (one per 32-row block) and the first 16
//     raw key / value rows by bulk copies, and stages beta, G;
//   * 8 compute warps, per unit: everything that does not need the state
//     first -- the 16 x 16 Gram K K^T on mma.sync (2 warps), the inverse of
//     the unit lower-triangular I + L by forward substitution on the identity
//     (one warp, lane = column), K~ and V~ on CUDA cores -- then each warp
//     streams its own 16 d_v rows as soon as their 32-row block has landed:
//       U^T = V~^T - S K~^T   (m16n8k8 tf32, A = the state rows straight from
//                              the swizzled tile by ldmatrix, split TF32:
//                              S_hi K~_hi + S_lo K~_hi + S_hi K~_lo),
//       D^T = Y^T K           (Y = e^{G_last - G_i} u_i, hi + lo; the U^T
//                              accumulator fragment IS the A fragment of this
//                              product once the record index inside each
//                              8-record tile is permuted (slot t <-> record 2t,
//                              slot t+4 <-> record 2t+1): no shuffles),
//       S_new = gamma_last S + D^T, written from registers straight to HBM
//     (8-byte stores, full 32-byte sectors), and releases its rows of the
//     buffer to the producer.
// The fold, the one dense contraction, runs on the warp-level tensor cores
// (HMMA).  Measured at config 2: tcgen05 M128 x N128
// fold in TMEM, one CTA per unit: 103 us; mma.sync, one CTA per unit
// (2 per SM): 90 us, and the same kernel with the arithmetic removed 45 us
// -- the units' compute and memory phases did not overlap, hence this
// persistent, double-buffered form.
#include <cuda.h>

#include "device.cuh"
#include "internal.h"

namespace labuf {

constexpr int kUtCh = 16;            // records per UT chunk
constexpr int kUtCompute = 256;      // 8 compute warps: one m16 tile of d_v rows each
constexpr int kUtThreads = 288;      // + 1 producer warp
constexpr int kUtS = 132;            // fp32 record rows padded to 132 floats (conflict-free ldmatrix)
constexpr int kUtKc = 24;            // keys transposed [c][record], 24-float rows (conflict-free 8-byte reads)

struct UtSmem {
    uint32_t S, RK, RV, Ks, Vs, Kc, Ls, Qs, Ps, Gs, Bs, GB, bar, meta, total;
};
__host__ __device__ inline UtSmem ut_smem_layout(int isz) {
    UtSmem L;
    uint32_t o = 0;
    L.S = o;   o += 2 * kD * kD * 4;               // 2 states: 4 column groups x 128 rows x 128 B, SW128
    L.RK = o;  o += 2 * kUtCh * kD * isz;          // 2 x raw key rows of the first chunk (bulk copies)
    L.RV = o;  o += 2 * kUtCh * kD * isz;          // 2 x raw value rows
    L.Ks = o;  o += kUtCh * kUtS * 4;              // keys (fp32), then K~ in place
    L.Vs = o;  o += kUtCh * kUtS * 4;              // values (fp32), then V~ in place
    L.Kc = o;  o += kD * kUtKc * 4;                // keys [c][record]: the fold's B operand
    L.Ls = o;  o += kUtCh * 17 * 4;                // L (row stride 17)
    L.Qs = o;  o += kUtCh * kUtCh * 4;             // A Diag(beta gamma)
    L.Ps = o;  o += kUtCh * kUtCh * 4;             // A Diag(beta)
    L.Gs = o;  o += kUtCh * 4;                     // G_i relative to the chunk's entering state
    L.Bs = o;  o += kUtCh * 4;                     // beta_i
    L.GB = o;  o += 2 * 2 * kUtCh * 4;             // 2 x staged (G, beta) of the first chunk
    L.bar = o; o += 14 * 8;                        // full_S[2][4], empty_S[2], full_raw[2], empty_raw[2]
    L.meta = o; o += 2 * 2 * 4;                    // 2 x (n, zero_s0)
    L.total = o;
    return L;
}

// byte offset of state element (d_v row j, d_k column c) in a TMA tile:
// column group c / 32 (16 KiB each), row j (128 B), 16-byte chunk ^= j % 8
__device__ __forceinline__ uint32_t ut_sw(int j, int c) {
    return (uint32_t)((c >> 5) * 16384 + j * 128 + ((((c & 31) >> 2) ^ (j & 7)) << 4) + (c & 3) * 4);
}
__device__ __forceinline__ void split_tf32(uint32_t x, uint32_t &hi, uint32_t &lo) {
    hi = x & 0xFFFFE000u;
    lo = __float_as_uint(__uint_as_float(x) - __uint_as_float(hi));
}
// 16 bytes of a record row as 4 (fp32) or 8 (bf16) floats
__device__ __forceinline__ void widen16(const uint4 &u, const float *, float (&f)[8]) {
    f[0] = __uint_as_float(u.x); f[1] = __uint_as_float(u.y); f[2] = __uint_as_float(u.z); f[3] = __uint_as_float(u.w);
}
__device__ __forceinline__ void widen16(const uint4 &u, const __nv_bfloat16 *, float (&f)[8]) {
    f[0] = __uint_as_float(u.x << 16); f[1] = __uint_as_float(u.x & 0xFFFF0000u);
    f[2] = __uint_as_float(u.y << 16); f[3] = __uint_as_float(u.y & 0xFFFF0000u);
    f[4] = __uint_as_float(u.z << 16); f[5] = __uint_as_float(u.z & 0xFFFF0000u);
    f[6] = __uint_as_float(u.w << 16); f[7] = __uint_as_float(u.w & 0xFFFF0000u);
}
__device__ __forceinline__ void cbar() { named_bar_sync(1, kUtCompute); }   // the 8 compute warps
#ifdef LABUF_UT_PROF
__device__ long long g_ut_prof[2][8][12];
extern "C" __attribute__((visibility("default"))) int la_debug_ut_prof(long long *dst) {
    return (int)cudaMemcpyFromSymbol(dst, g_ut_prof, sizeof(g_ut_prof));
}
#define UT_MARK(i) do { if (blockIdx.x == 0 && (warp == 0 || warp == 6) && lane == 0 && k < 8) g_ut_prof[warp == 6][k][i] = clock64(); } while (0)
#else
#define UT_MARK(i) do { } while (0)
#endif

template <typename InT, bool FP32_IN, bool PG>
__global__ void __launch_bounds__(kUtThreads, 1)
    fold_ut_kernel(const FoldArgs a, const __grid_constant__ CUtensorMap tmap) {
    constexpr int isz = (int)sizeof(InT);
    constexpr int EPC = 16 / isz;                    // record elements per 16-byte piece
    constexpr int PPR = kD / EPC;                    // pieces per record row (16 bf16, 32 fp32)
    constexpr int PPT = kUtCh * PPR / kUtCompute;    // pieces per thread per operand (1 bf16, 2 fp32)
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const Dims dm = a.dm;
    const int Hv = dm.Hv, bt = dm.bt;
    const int n_units = a.n * Hv;

    extern __shared__ __align__(1024) unsigned char smem[];
    const UtSmem L = ut_smem_layout(isz);
    float *Ks = reinterpret_cast<float *>(smem + L.Ks), *Vs = reinterpret_cast<float *>(smem + L.Vs);
    float *Kc = reinterpret_cast<float *>(smem + L.Kc);
    float *Ls = reinterpret_cast<float *>(smem + L.Ls), *Qs = reinterpret_cast<float *>(smem + L.Qs);
    float *Ps = reinterpret_cast<float *>(smem + L.Ps);
    float *Gs = reinterpret_cast<float *>(smem + L.Gs), *Bs = reinterpret_cast<float *>(smem + L.Bs);
    float *GB = reinterpret_cast<float *>(smem + L.GB);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + L.bar);
    uint64_t *full_S = bars, *empty_S = bars + 8, *full_raw = bars + 10, *empty_raw = bars + 12;
    int *meta = reinterpret_cast<int *>(smem + L.meta);

    // unit u: V head u % Hv of slot row u / Hv
    auto slot_of = [&](int u) -> int { return PG && a.slots ? __ldcg(a.slots + u / Hv) : a.first + u / Hv; };
    auto state_row0 = [&](int r, int h) -> int {
        const size_t sb = PG && a.p.sidx ? (size_t)__ldcg(a.p.sidx + r) : (size_t)r;
        return (int)((sb * Hv + h) * kD);
    };
    auto at = [&](int r, int i) -> int2 { return PG ? rec_at(dm, a.p, r, i) : make_int2(r, i); };
    auto issue_state = [&](int b, int row0) {
#pragma unroll
        for (int x = 0; x < 4; ++x) {
            mbar_arrive_expect_tx(full_S + 4 * b + x, 32 * kD * 4);
#pragma unroll
            for (int kb = 0; kb < 4; ++kb)
                tma_load_2d(smem + L.S + b * 65536 + kb * 16384 + x * 4096, &tmap, kb * 32, row0 + x * 32,
                            full_S + 4 * b + x);
        }
    };
    const int stride = gridDim.x;

    if (tid == 0) {
        for (int i = 0; i < 8; ++i) mbar_init(full_S + i, 1);
        mbar_init(empty_S, 8);
        mbar_init(empty_S + 1, 8);
        mbar_init(full_raw, 2);
        mbar_init(full_raw + 1, 2);
        mbar_init(empty_raw, 1);
        mbar_init(empty_raw + 1, 1);
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == kUtCompute / 32) {
        // ================================================================ producer
        if constexpr (PG) pdl_wait();
        const bool early = !PG && a.spec && a.pdl_early;   // every unit folds: states before the wait
        if (early && lane == 0)
            for (int k = 0; k < 2; ++k) {
                const int u = blockIdx.x + k * stride;
                if (u < n_units) issue_state(k, state_row0(slot_of(u), u % Hv));
            }
        if constexpr (!PG) pdl_wait();
        pdl_trigger();
        // one unit of lookahead: the next unit's counters (and, for contiguous
        // records, its first decays / betas) are requested before this unit's
        // buffers are waited for, so no global round trip sits in the loop
        const int kspec = min(kUtCh, a.kcap);
        int nx_mode = 0, nx_occ = 0, nx_len = 0;
        float nx_g = 0.f, nx_b = 0.f;
        auto prefetch = [&](int u) {
            const int r = slot_of(u), h = u % Hv;
            nx_mode = a.p.mode[r];
            nx_occ = a.p.occ[r];
            nx_len = a.p.len[r];
            if (!PG && lane < kspec) {
                const size_t o = ((size_t)r * Hv + h) * bt + lane;
                nx_g = a.p.G[o];
                nx_b = a.p.B[o];
            }
        };
        if ((int)blockIdx.x < n_units) prefetch(blockIdx.x);
        for (int k = 0;; ++k) {
            const int u = blockIdx.x + k * stride;
            if (u >= n_units) break;
            const int b = k & 1, m = k >> 1;
            const int r = slot_of(u), h = u % Hv, hk = h / dm.g;
            const int mode = nx_mode, occ = nx_occ, len = nx_len;
            float gv = nx_g, bv = nx_b;
            if (u + stride < n_units) prefetch(u + stride);
            int n = 0, zero_s0 = 0;
            if (a.kind == FK_FULL)
                n = (mode == 0 && occ == dm.C) ? occ : 0;
            else if (mode == 1) {   // FK_FORCE: a direct slot compresses into a state, S0 = 0
                n = len;
                zero_s0 = 1;
            } else
                n = occ;
            const int kn0 = min(kUtCh, n);
            if (PG && lane < kn0) {   // block-table records: after the counters
                const int2 ba = at(r, lane);
                const size_t o = ((size_t)ba.x * Hv + h) * bt + ba.y;
                gv = a.p.G[o];
                bv = a.p.B[o];
            }
            if (lane >= kn0) gv = bv = 0.f;
            if (m > 0) mbar_wait(empty_raw + b, (m - 1) & 1);   // raw staging b released
            if (lane < kUtCh) {
                GB[b * 2 * kUtCh + lane] = gv;
                GB[b * 2 * kUtCh + kUtCh + lane] = bv;
            }
            if (lane == 0) {
                meta[2 * b] = n;
                meta[2 * b + 1] = zero_s0;
                if (kn0 > 0) {
                    mbar_arrive_expect_tx(full_raw + b, (uint32_t)(2 * kn0 * kD * isz));
                    unsigned char *rk = smem + L.RK + b * kUtCh * kD * isz;
                    unsigned char *rv = smem + L.RV + b * kUtCh * kD * isz;
                    for (int p = 0; p < kn0;) {   // runs of consecutive positions inside one record block
                        const int2 ba = at(r, p);
                        const int run = PG ? min(kn0 - p, bt - ba.y) : kn0;
                        const InT *K = static_cast<const InT *>(a.p.K) + (((size_t)ba.x * dm.Hk + hk) * bt + ba.y) * kD;
                        const InT *V = static_cast<const InT *>(a.p.V) + (((size_t)ba.x * Hv + h) * bt + ba.y) * kD;
                        bulk_g2s(rk + p * kD * isz, K, run * kD * isz, full_raw + b);
                        bulk_g2s(rv + p * kD * isz, V, run * kD * isz, full_raw + b);
                        p += run;
                    }
                } else {
                    mbar_arrive(full_raw + b);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(full_raw + b);   // G, beta, meta written
            // state buffer b: free once every compute warp released unit k - 2
            if (lane == 0 && !(early && k < 2)) {
                if (m > 0) mbar_wait(empty_S + b, (m - 1) & 1);
                if (n > 0 && !zero_s0)
                    issue_state(b, state_row0(r, h));
                else
                    for (int x = 0; x < 4; ++x) mbar_arrive(full_S + 4 * b + x);
            }
        }
        return;
    }

    // ==================================================================== compute warps
    pdl_wait();
    pdl_trigger();
    const int g = lane >> 2, t4 = lane & 3, lr = lane & 7, lm = lane >> 3;
    const int c = tid & (kD - 1), hh = tid >> 7;
    for (int k = 0;; ++k) {
        const int u = blockIdx.x + k * stride;
        if (u >= n_units) break;
        const int b = k & 1, ph = (k >> 1) & 1;
        const int r = slot_of(u), h = u % Hv, hk = h / dm.g;
        unsigned char *Sb = smem + L.S + b * 65536;
        UT_MARK(0);
        mbar_wait(full_raw + b, ph);
        UT_MARK(1);
        const int n = meta[2 * b];
        const bool zero_s0 = meta[2 * b + 1] != 0;
        if (n == 0 || zero_s0) {   // the producer arrived on the state barriers without a copy
            for (int x = 0; x < 4; ++x) mbar_wait(full_S + 4 * b + x, ph);
            if (zero_s0)
                for (int x = tid; x < kD * kD / 4; x += kUtCompute)
                    reinterpret_cast<float4 *>(Sb)[x] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        if (n == 0) {
            __syncwarp();
            if (tid == 0) mbar_arrive(empty_raw + b);
            if (lane == 0) mbar_arrive(empty_S + b);
            continue;
        }
        float *const Sg = a.p.state + (size_t)state_row0(r, h) * kD;   // this unit's state in HBM
        for (int s0 = 0; s0 < n; s0 += kUtCh) {
            const int kn = min(kUtCh, n - s0);
            const int nkt = (kn + 7) >> 3;   // 8-record tiles
            // ---- operands of the chunk -> fp32 rows (zero past kn)
            if (s0 == 0) {
                const unsigned char *rk = smem + L.RK + b * kUtCh * kD * isz;
                const unsigned char *rv = smem + L.RV + b * kUtCh * kD * isz;
#pragma unroll
                for (int q = 0; q < PPT; ++q) {
                    const int p = tid + kUtCompute * q, i = p / PPR, e = (p % PPR) * EPC;
                    const bool ok = i < kn;
                    float fk[8], fv[8];
                    widen16(ok ? *reinterpret_cast<const uint4 *>(rk + (i * kD + e) * isz) : make_uint4(0u, 0u, 0u, 0u),
                            static_cast<const InT *>(nullptr), fk);
                    widen16(ok ? *reinterpret_cast<const uint4 *>(rv + (i * kD + e) * isz) : make_uint4(0u, 0u, 0u, 0u),
                            static_cast<const InT *>(nullptr), fv);
#pragma unroll
                    for (int x = 0; x < EPC; x += 4) {
                        *reinterpret_cast<float4 *>(Ks + i * kUtS + e + x) = make_float4(fk[x], fk[x + 1], fk[x + 2], fk[x + 3]);
                        *reinterpret_cast<float4 *>(Vs + i * kUtS + e + x) = make_float4(fv[x], fv[x + 1], fv[x + 2], fv[x + 3]);
                    }
                }
                if (tid < kUtCh) {
                    Gs[tid] = GB[b * 2 * kUtCh + tid];
                    Bs[tid] = GB[b * 2 * kUtCh + kUtCh + tid];
                }
            } else {   // later chunks of a long fold: straight from HBM
                cbar();   // every warp is done with the previous chunk's operands
#pragma unroll
                for (int q = 0; q < PPT; ++q) {
                    const int p = tid + kUtCompute * q, i = p / PPR, e = (p % PPR) * EPC;
                    uint4 kr = make_uint4(0u, 0u, 0u, 0u), vr = kr;
                    if (i < kn) {
                        const int2 ba = at(r, s0 + i);
                        kr = __ldg(reinterpret_cast<const uint4 *>(static_cast<const InT *>(a.p.K) +
                                                                   (((size_t)ba.x * dm.Hk + hk) * bt + ba.y) * kD + e));
                        vr = __ldg(reinterpret_cast<const uint4 *>(static_cast<const InT *>(a.p.V) +
                                                                   (((size_t)ba.x * Hv + h) * bt + ba.y) * kD + e));
                    }
                    float fk[8], fv[8];
                    widen16(kr, static_cast<const InT *>(nullptr), fk);
                    widen16(vr, static_cast<const InT *>(nullptr), fv);
#pragma unroll
                    for (int x = 0; x < EPC; x += 4) {
                        *reinterpret_cast<float4 *>(Ks + i * kUtS + e + x) = make_float4(fk[x], fk[x + 1], fk[x + 2], fk[x + 3]);
                        *reinterpret_cast<float4 *>(Vs + i * kUtS + e + x) = make_float4(fv[x], fv[x + 1], fv[x + 2], fv[x + 3]);
                    }
                }
                if (tid < kUtCh) {
                    float gv = 0.f, bv = 0.f;
                    if (tid < kn) {
                        const int2 ba = at(r, s0 + tid);
                        const size_t o = ((size_t)ba.x * Hv + h) * bt + ba.y;
                        gv = a.p.G[o];
                        bv = a.p.B[o];
                    }
                    const int2 bb = at(r, s0 - 1);
                    const float gbase = a.p.G[((size_t)bb.x * Hv + h) * bt + bb.y];
                    Gs[tid] = tid < kn ? gv - gbase : 0.f;
                    Bs[tid] = bv;
                }
            }
            cbar();
            UT_MARK(2);
            if (s0 == 0 && tid == 0) mbar_arrive(empty_raw + b);   // raw staging b consumed

            // (1) L = strictLower(Diag(beta) (Gamma (.) K K^T)): warp nt computes
            //     Gram columns 8 nt .. 8 nt + 7 (m16n8k8 tf32; bf16 products exact)
            if (warp < 2) {
                // HMMA latency on sm_100a is ~90 cycles (measured, tools/ut_prof.py):
                // four independent partial sums instead of one chain
                float acc4[4][4] = {};
                if (warp < nkt) {
                    const uint32_t ab = smem_u32(Ks) + (uint32_t)(((lr + (lm & 1) * 8) * kUtS + (lm >> 1) * 4) * 4);
                    const uint32_t bb = smem_u32(Ks) + (uint32_t)(((warp * 8 + lr) * kUtS + (lm & 1) * 4) * 4);
#pragma unroll
                    for (int kk = 0; kk < kD / 8; ++kk) {
                        uint32_t ka[4], kb[2];
                        ldsm_x4(ka, ab + kk * 32);
                        ldsm_x2(kb, bb + kk * 32);
                        if constexpr (FP32_IN) {
                            uint32_t ah[4], al[4], bh[2], bl[2];
#pragma unroll
                            for (int q = 0; q < 4; ++q) split_tf32(ka[q], ah[q], al[q]);
                            split_tf32(kb[0], bh[0], bl[0]);
                            split_tf32(kb[1], bh[1], bl[1]);
                            mma_tf32_16x8x8(acc4[kk & 1], ah, bh[0], bh[1]);
                            mma_tf32_16x8x8(acc4[2], al, bh[0], bh[1]);
                            mma_tf32_16x8x8(acc4[3], ah, bl[0], bl[1]);
                        } else {
                            mma_tf32_16x8x8(acc4[kk & 3], ka, kb[0], kb[1]);
                        }
                    }
                }
                float acc[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[q] = (acc4[0][q] + acc4[1][q]) + (acc4[2][q] + acc4[3][q]);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int i = g + 8 * (q >> 1), l = warp * 8 + 2 * t4 + (q & 1);
                    Ls[i * 17 + l] = l < i ? Bs[i] * __expf(Gs[i] - Gs[l]) * acc[q] : 0.f;
                }
            }
            // ... meanwhile every thread takes its key / value column into
            //     registers and writes the transposed keys (the fold's B operand)
            float kc[kUtCh], vc[kUtCh];
#pragma unroll
            for (int l = 0; l < kUtCh; ++l) {
                kc[l] = Ks[l * kUtS + c];
                vc[l] = Vs[l * kUtS + c];
            }
            {
                float kh[8];   // this thread's half of the column (select, not a dynamic register index)
#pragma unroll
                for (int x = 0; x < 8; ++x) kh[x] = hh ? kc[8 + x] : kc[x];
                *reinterpret_cast<float4 *>(Kc + c * kUtKc + hh * 8) = make_float4(kh[0], kh[1], kh[2], kh[3]);
                *reinterpret_cast<float4 *>(Kc + c * kUtKc + hh * 8 + 4) = make_float4(kh[4], kh[5], kh[6], kh[7]);
            }
            cbar();
            UT_MARK(3);
            // (2) A = (I + L)^{-1} column by column (lane l: forward substitution on
            //     e_l); P = A Diag(beta), Q = A Diag(beta gamma)
            if (warp == 0 && lane < kUtCh) {
                float x[kUtCh];
#pragma unroll
                for (int i = 0; i < kUtCh; ++i) {
                    float a0 = i == lane ? 1.f : 0.f, a1 = 0.f;
#pragma unroll
                    for (int mm = 0; mm < i; mm += 2) {
                        a0 = fmaf(-Ls[i * 17 + mm], x[mm], a0);
                        if (mm + 1 < i) a1 = fmaf(-Ls[i * 17 + mm + 1], x[mm + 1], a1);
                    }
                    x[i] = a0 + a1;
                }
                const float bl = Bs[lane], ql = bl * expf(Gs[lane]);
#pragma unroll
                for (int i = 0; i < kUtCh; ++i) {
                    Ps[i * kUtCh + lane] = x[i] * bl;
                    Qs[i * kUtCh + lane] = x[i] * ql;
                }
            }
            cbar();
            UT_MARK(4);
            // (3) K~ = Q K, V~ = P V in place of K, V (thread: column c, rows 2 m + hh;
            //     Q, P lower triangular; the columns were read into registers above)
#pragma unroll
            for (int mm = 0; mm < kUtCh / 2; ++mm) {
                const int i = 2 * mm + hh;
                const float4 *q4 = reinterpret_cast<const float4 *>(Qs + i * kUtCh);
                const float4 *p4 = reinterpret_cast<const float4 *>(Ps + i * kUtCh);
                float ak = 0.f, av = 0.f;
#pragma unroll
                for (int l4 = 0; l4 < kUtCh / 4; ++l4) {
                    if (4 * l4 <= 2 * mm + 1) {
                        const float4 qq = q4[l4], pp = p4[l4];
                        ak = fmaf(qq.x, kc[4 * l4], fmaf(qq.y, kc[4 * l4 + 1], fmaf(qq.z, kc[4 * l4 + 2], fmaf(qq.w, kc[4 * l4 + 3], ak))));
                        av = fmaf(pp.x, vc[4 * l4], fmaf(pp.y, vc[4 * l4 + 1], fmaf(pp.z, vc[4 * l4 + 2], fmaf(pp.w, vc[4 * l4 + 3], av))));
                    }
                }
                Ks[i * kUtS + c] = ak;
                Vs[i * kUtS + c] = av;
            }
            cbar();
            UT_MARK(5);

            // (4) warp w: d_v rows j = 16 w .. 16 w + 15 (32-row block w / 2)
            if (s0 == 0 && !zero_s0) mbar_wait(full_S + 4 * b + (warp >> 1), ph);
            UT_MARK(6);
            float acc[2][4];   // U^T [row g (+8)][record 8 nt + 2 t4 (+1)], from V~^T
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    acc[nt][q] = Vs[(nt * 8 + 2 * t4 + (q & 1)) * kUtS + warp * 16 + g + 8 * (q >> 1)];
            {
                // six independent chains: (record tile) x (S_hi K~_hi, S_lo K~_hi, S_hi K~_lo)
                float pacc[2][3][4] = {};
                uint32_t aoff[4];
#pragma unroll
                for (int c8 = 0; c8 < 4; ++c8)
                    aoff[c8] = (uint32_t)((lr + (lm & 1) * 8) * 128 + (((2 * c8 + (lm >> 1)) ^ lr) << 4));
                const uint32_t abase = smem_u32(Sb) + warp * 2048;
                const uint32_t bbase = smem_u32(Ks) + (uint32_t)((lr * kUtS + (lm & 1) * 4) * 4);
#pragma unroll 8
                for (int kk = 0; kk < kD / 8; ++kk) {
                    uint32_t x[4], ah[4], al[4];
                    ldsm_x4(x, abase + (kk >> 2) * 16384 + aoff[kk & 3]);
#pragma unroll
                    for (int q = 0; q < 4; ++q) split_tf32(x[q], ah[q], al[q]);
#pragma unroll
                    for (int nt = 0; nt < 2; ++nt) {
                        if (nt < nkt) {   // U^T -= S K~^T (B = -K~, split)
                            uint32_t bq[2], bh[2], bl[2];
                            ldsm_x2(bq, bbase + (uint32_t)((nt * 8 * kUtS + kk * 8) * 4));
                            split_tf32(bq[0] ^ 0x80000000u, bh[0], bl[0]);
                            split_tf32(bq[1] ^ 0x80000000u, bh[1], bl[1]);
                            mma_tf32_16x8x8(pacc[nt][0], ah, bh[0], bh[1]);
                            mma_tf32_16x8x8(pacc[nt][1], al, bh[0], bh[1]);
                            mma_tf32_16x8x8(pacc[nt][2], ah, bl[0], bl[1]);
                        }
                    }
                }
#pragma unroll
                for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                    for (int q = 0; q < 4; ++q) acc[nt][q] += pacc[nt][0][q] + (pacc[nt][1][q] + pacc[nt][2][q]);
            }
            // (5) Y = e^{G_last - G_i} u_i in the same fragments, split hi + lo; as the A
            //     fragment of D^T = Y^T K: a = {Y[g][2t], Y[g+8][2t], Y[g][2t+1], Y[g+8][2t+1]}
            const float gl = Gs[kn - 1], eg = __expf(gl);
            uint32_t yh[2][4], yl[2][4];
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
                const float w0 = __expf(gl - Gs[nt * 8 + 2 * t4]), w1 = __expf(gl - Gs[nt * 8 + 2 * t4 + 1]);
                const float y[4] = {w0 * acc[nt][0], w0 * acc[nt][2], w1 * acc[nt][1], w1 * acc[nt][3]};
#pragma unroll
                for (int q = 0; q < 4; ++q) split_tf32(__float_as_uint(y[q]), yh[nt][q], yl[nt][q]);
            }
            // (6) D^T[j][c] = sum_i Y[i][j] k_i[c] per 8-column tile of d_k, then
            //     S_new = gamma_last S + D^T: into the tile (a later chunk follows) or
            //     straight to HBM (pairs of columns: 8-byte stores, 32-byte sectors)
            const int j0 = warp * 16 + g;
            const bool last = s0 + kUtCh >= n;
#pragma unroll 4
            for (int ct = 0; ct < kD / 8; ++ct) {
                float dp[2][3][4] = {};   // independent chains: (record tile) x (pass)
#pragma unroll
                for (int nt = 0; nt < 2; ++nt) {
                    if (nt < nkt) {   // b = {K[8 nt + 2 t][c], K[8 nt + 2 t + 1][c]}, c = 8 ct + g
                        const float2 kb = *reinterpret_cast<const float2 *>(Kc + (ct * 8 + g) * kUtKc + nt * 8 + 2 * t4);
                        if constexpr (FP32_IN) {
                            uint32_t bh0, bl0, bh1, bl1;
                            split_tf32(__float_as_uint(kb.x), bh0, bl0);
                            split_tf32(__float_as_uint(kb.y), bh1, bl1);
                            mma_tf32_16x8x8(dp[nt][0], yh[nt], bh0, bh1);
                            mma_tf32_16x8x8(dp[nt][1], yl[nt], bh0, bh1);
                            mma_tf32_16x8x8(dp[nt][2], yh[nt], bl0, bl1);
                        } else {   // bf16 keys are exact in tf32
                            mma_tf32_16x8x8(dp[nt][0], yh[nt], __float_as_uint(kb.x), __float_as_uint(kb.y));
                            mma_tf32_16x8x8(dp[nt][1], yl[nt], __float_as_uint(kb.x), __float_as_uint(kb.y));
                        }
                    }
                }
                float d[4];
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    d[q] = (dp[0][0][q] + dp[1][0][q]) + ((dp[0][1][q] + dp[1][1][q]) + (dp[0][2][q] + dp[1][2][q]));
                const int cc = ct * 8 + 2 * t4;
                float2 *p0 = reinterpret_cast<float2 *>(Sb + ut_sw(j0, cc));
                float2 *p1 = reinterpret_cast<float2 *>(Sb + ut_sw(j0 + 8, cc));
                float2 s0v = *p0, s1v = *p1;
                s0v.x = fmaf(eg, s0v.x, d[0]); s0v.y = fmaf(eg, s0v.y, d[1]);
                s1v.x = fmaf(eg, s1v.x, d[2]); s1v.y = fmaf(eg, s1v.y, d[3]);
                if (last) {
                    *reinterpret_cast<float2 *>(Sg + (size_t)j0 * kD + cc) = s0v;
                    *reinterpret_cast<float2 *>(Sg + (size_t)(j0 + 8) * kD + cc) = s1v;
                } else {
                    *p0 = s0v;
                    *p1 = s1v;
                }
            }
        }
        UT_MARK(8);
        fence_proxy_async_smem();   // generic writes to the buffer (zero fill, chained chunks) before the next TMA
        __syncwarp();
        if (lane == 0) mbar_arrive(empty_S + b);   // this warp's rows of buffer b are done
        cbar();                                     // every warp done with the unit's operands
        UT_MARK(9);
        // ---- counters: the last unit of the slot resets the buffer
        if (tid == 0 && atomicAdd(&a.p.ticket[r], 1) == Hv - 1) {
            a.p.ticket[r] = 0;
            a.p.occ[r] = 0;
            if (zero_s0) { a.p.mode[r] = 0; a.p.len[r] = 0; }
        }
    }
}

static int sm_count() {
    static int n[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    if (n[dev] == 0) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        n[dev] = v > 0 ? v : 148;
    }
    return n[dev];
}

template <typename InT, bool FP32_IN>
static cudaError_t launch_ut_t(const FoldArgs &a, cudaStream_t s) {
    const UtSmem L = ut_smem_layout((int)sizeof(InT));
    const bool pg = a.slots || a.p.btab || a.p.sidx;
    auto kfn = pg ? fold_ut_kernel<InT, FP32_IN, true> : fold_ut_kernel<InT, FP32_IN, false>;
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
    if (e != cudaSuccess) return e;
    const CUtensorMap tm = *static_cast<const CUtensorMap *>(a.tmap);
    const int units = a.n * a.dm.Hv;
    const int grid = units < sm_count() ? units : sm_count();
    return launch_k(kfn, dim3(grid), dim3(kUtThreads), L.total, s, a.pdl != 0, a, tm);
}

cudaError_t launch_fold_ut(const FoldArgs &a, cudaStream_t s) {
    if (!a.tmap || (a.kind != FK_FULL && a.kind != FK_FORCE)) return cudaErrorInvalidValue;
    if (a.dm.in_dt == DT_F32) return launch_ut_t<float, true>(a, s);
    return launch_ut_t<__nv_bfloat16, false>(a, s);
}

}  // namespace labuf
