// fold_ut.cu — kernel (2 RAW): flush mode ii.  The delta values are not read
// from the buffer but recomputed from the raw records (k_i, v_i, beta_i, G_i)
// and the state by the chunkwise UT transform of P:392-399 (K~ corrected per
// reading Z4), then folded into the state:
//
//   L      = strictLower(Diag(beta) (Gamma (.) K K^T))          Gamma_il = e^{G_i - G_l}
//   A      = (I + L)^{-1}
//   K~     = A Diag(beta) Diag(gamma) K,   V~ = A Diag(beta) V    gamma_i = e^{G_i}
//   U      = V~ - K~ S^T = V~ - Q W,  Q = A Diag(beta gamma), W = K S^T   (u_i rows)
//   S_new  = gamma_last S + sum_i e^{G_last - G_i} u_i k_i^T
//
// over chunks of up to 16 records (G relative to the chunk's entering state;
// a longer fold chains chunks through the state held in shared memory).
// K~ S^T is evaluated as Q (K S^T): the keys are exact in TF32 when they are
// bf16, so W takes two split-TF32 passes instead of three, and the 16 x 16
// Q W product is a handful of MMAs.
//
// B200 structure: ONE CTA of 8 warps per (V head, slot), so the UT transform
// (Gram, triangular inverse, Q, V~) is computed once per head; 2 CTAs per SM.
//   * entry: the 64 KiB state is requested as 16 TMA boxes (32 x 32 fp32,
//     128-byte swizzle) on four mbarriers, one per 32-row block, and every
//     thread requests its raw record pieces (one 16-byte load of a key row,
//     one of a value row);
//   * everything that does not need the state runs while it is in flight:
//     the 16 x 16 Gram K K^T on mma.sync (2 warps), the inverse of the unit
//     lower-triangular I + L by forward substitution on the identity (one
//     warp, lane = column; -Q stored as TF32 hi + lo pieces), V~ on CUDA cores;
//   * then each warp streams its own 16 d_v rows, starting as soon as their
//     32-row block has landed, with no further block-wide barrier:
//       W^T = S K^T           (m16n8k8 tf32, A = the state rows straight from
//                              the swizzled tile by ldmatrix, split TF32),
//       U^T = V~^T - W^T Q^T  (the W^T accumulator fragment IS the A fragment
//                              of this product once the record index inside
//                              each 8-record tile is permuted (slot t <->
//                              record 2t, slot t+4 <-> record 2t+1)),
//       D^T = Y^T K           (bf16 keys: m16n8k16 bf16 with Y split into three
//                              bf16 pieces, the U^T accumulator pairs being the
//                              bf16 A fragment as they stand -- 48 instead of 64
//                              MMAs per warp, 80.3 -> 78.2 us; fp32 keys: tf32,
//                              Y hi + lo, the same permutation trick),
//       S = gamma_last S + D in the tile, and the warp pair's 32 rows leave by
//     4 TMA box stores while the other warps still compute.
// Every product keeps several independent accumulators.  The warp-level
// tensor cores (HMMA, ~277 TFLOP/s tf32 on B200) are the bound of the
// compute phase: 140 HMMA per warp per chunk (tools/ut_prof.py phase trace).
// Measured at config 2: the tcgen05 version (M = 128 x
// N = 128 fold in TMEM after a block-wide barrier, TMEM allocated per CTA)
// 103 us; a persistent double-buffered version (one CTA per SM, producer
// warp) 111 us -- 8 warps per SM cannot hide the per-unit chain that two
// 8-warp CTAs per SM overlap; this version 80 us.  Shared memory ≈ 100 KiB.
#include <cuda.h>

#include "device.cuh"
#include "internal.h"

namespace labuf {

constexpr int kUtCh = 16;          // records per UT chunk
constexpr int kUtThreads = 256;    // 8 warps: one m16 tile of d_v rows each
constexpr int kUtS = 132;          // fp32 record rows padded to 132 floats (conflict-free ldmatrix)
constexpr int kUtKc = 24;          // keys transposed [c][record], 24-float rows (conflict-free 8-byte reads)
constexpr int kUtQn = 24;          // -Q pieces [i][l], 24-float rows (conflict-free 8-byte reads)

struct UtSmem {
    uint32_t S, Ks, Vs, Kc, Ls, Ps, Qn, Gs, Bs, bar, total;
};
__host__ __device__ inline UtSmem ut_smem_layout() {
    UtSmem L;
    uint32_t o = 0;
    L.S = o;   o += kD * kD * 4;               // state: 4 column groups x 128 rows x 128 B, SW128
    L.Ks = o;  o += kUtCh * kUtS * 4;          // keys (fp32)
    L.Vs = o;  o += kUtCh * kUtS * 4;          // values (fp32), then V~ in place
    L.Kc = o;  o += kD * kUtKc * 4;            // keys [c][record]: the fold's B operand
    L.Ls = o;  o += kUtCh * 17 * 4;            // L (row stride 17)
    L.Ps = o;  o += kUtCh * kUtCh * 4;         // A Diag(beta)
    L.Qn = o;  o += 2 * kUtCh * kUtQn * 4;     // -Q as TF32 hi, lo pieces (rows of 24 floats)
    L.Gs = o;  o += kUtCh * 4;                 // G_i relative to the chunk's entering state
    L.Bs = o;  o += kUtCh * 4;                 // beta_i
    L.bar = o; o += 64;
    L.total = o;
    return L;
}

// byte offset of state element (d_v row j, d_k column c) in the TMA tile:
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

#ifdef LABUF_UT_PROF
// phase timestamps (clock64) of warps 0 and 6 of CTAs 0..7: tools/ut_prof.py
__device__ long long g_ut_prof[2][8][12];
extern "C" __attribute__((visibility("default"))) int la_debug_ut_prof(long long *dst) {
    return (int)cudaMemcpyFromSymbol(dst, g_ut_prof, sizeof(g_ut_prof));
}
#define UT_MARK(i)                                                                                  \
    do {                                                                                            \
        const int cta_ = blockIdx.x + gridDim.x * blockIdx.y;                                       \
        if (cta_ < 8 && (warp == 0 || warp == 6) && lane == 0) g_ut_prof[warp == 6][cta_][i] = clock64(); \
    } while (0)
#else
#define UT_MARK(i) do { } while (0)
#endif

template <typename InT, bool FP32_IN, bool PG>
__global__ void __launch_bounds__(kUtThreads, 2)
    fold_ut_kernel(const FoldArgs a, const __grid_constant__ CUtensorMap tmap) {
    constexpr int EPC = 16 / (int)sizeof(InT);       // record elements per 16-byte piece
    constexpr int PPR = kD / EPC;                    // pieces per record row (16 bf16, 32 fp32)
    constexpr int PPT = kUtCh * PPR / kUtThreads;    // pieces per thread per operand (1 bf16, 2 fp32)
    const int h = blockIdx.x, zi = blockIdx.y;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    UT_MARK(0);
    if constexpr (PG) {   // slot lists, state indices and block tables may come from the previous grid
        if (a.pdl) pdl_wait();
    }
    const int r = PG && a.slots ? __ldcg(a.slots + zi) : a.first + zi;
    const Dims dm = a.dm;
    const int Hv = dm.Hv, bt = dm.bt, hk = h / dm.g;

    extern __shared__ __align__(1024) unsigned char smem[];
    const UtSmem L = ut_smem_layout();
    float *S_s = reinterpret_cast<float *>(smem + L.S);
    float *Ks = reinterpret_cast<float *>(smem + L.Ks), *Qn = reinterpret_cast<float *>(smem + L.Qn);
    float *Vs = reinterpret_cast<float *>(smem + L.Vs), *Kc = reinterpret_cast<float *>(smem + L.Kc);
    float *Ls = reinterpret_cast<float *>(smem + L.Ls);
    float *Ps = reinterpret_cast<float *>(smem + L.Ps);
    float *Gs = reinterpret_cast<float *>(smem + L.Gs), *Bs = reinterpret_cast<float *>(smem + L.Bs);
    uint64_t *bar_S = reinterpret_cast<uint64_t *>(smem + L.bar);   // 4: one per 32-row block
    int *meta = reinterpret_cast<int *>(bar_S + 4);                 // n, zero_s0
    const size_t sb = PG && a.p.sidx ? (size_t)__ldcg(a.p.sidx + r) : (size_t)r;
    const int row0 = (int)((sb * Hv + h) * kD);

    auto issue_state = [&]() {
#pragma unroll
        for (int x = 0; x < 4; ++x) {
            mbar_arrive_expect_tx(bar_S + x, 32 * kD * 4);
#pragma unroll
            for (int kb = 0; kb < 4; ++kb)
                tma_load_2d(smem + L.S + kb * 16384 + x * 4096, &tmap, kb * 32, row0 + x * 32, bar_S + x);
        }
    };
    // record position i of the slot: (block, offset) -- the block table or the slot's own region
    auto at = [&](int i) -> int2 { return PG ? rec_at(dm, a.p, r, i) : make_int2(r, i); };

    // raw operands: 16-byte pieces p = tid + 256 q of the chunk's key / value rows
    uint4 kr[PPT], vr[PPT];
    float gr = 0.f, br = 0.f, gbase = 0.f;
    auto load_raw = [&](int s0, int kn) {
#pragma unroll
        for (int q = 0; q < PPT; ++q) {
            const int p = tid + kUtThreads * q, i = p / PPR, e = (p % PPR) * EPC;
            kr[q] = vr[q] = make_uint4(0u, 0u, 0u, 0u);
            if (i < kn) {
                const int2 ba = at(s0 + i);
                kr[q] = __ldg(reinterpret_cast<const uint4 *>(static_cast<const InT *>(a.p.K) +
                                                              (((size_t)ba.x * dm.Hk + hk) * bt + ba.y) * kD + e));
                vr[q] = __ldg(reinterpret_cast<const uint4 *>(static_cast<const InT *>(a.p.V) +
                                                              (((size_t)ba.x * Hv + h) * bt + ba.y) * kD + e));
            }
        }
        if (tid < kUtCh) {
            gr = br = gbase = 0.f;
            if (tid < kn) {
                const int2 ba = at(s0 + tid);
                const size_t o = ((size_t)ba.x * Hv + h) * bt + ba.y;
                gr = a.p.G[o];
                br = a.p.B[o];
            }
            if (s0 > 0) {
                const int2 ba = at(s0 - 1);
                gbase = a.p.G[((size_t)ba.x * Hv + h) * bt + ba.y];
            }
        }
    };
    // rows >= kn are zero in every operand (loads past a slot's own count are never used)
    auto store_raw = [&](int kn) {
#pragma unroll
        for (int q = 0; q < PPT; ++q) {
            const int p = tid + kUtThreads * q, i = p / PPR, e = (p % PPR) * EPC;
            float fk[8], fv[8];
            widen16(kr[q], static_cast<const InT *>(nullptr), fk);
            widen16(vr[q], static_cast<const InT *>(nullptr), fv);
            const bool ok = i < kn;
#pragma unroll
            for (int u = 0; u < EPC; u += 4) {
                *reinterpret_cast<float4 *>(Ks + i * kUtS + e + u) =
                    ok ? make_float4(fk[u], fk[u + 1], fk[u + 2], fk[u + 3]) : make_float4(0.f, 0.f, 0.f, 0.f);
                *reinterpret_cast<float4 *>(Vs + i * kUtS + e + u) =
                    ok ? make_float4(fv[u], fv[u + 1], fv[u + 2], fv[u + 3]) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        if (tid < kUtCh) {
            Gs[tid] = tid < kn ? gr - gbase : 0.f;
            Bs[tid] = tid < kn ? br : 0.f;
        }
    };

    // ---- which records fold (uniform over the slot's CTAs); the state in
    //      flight at once when the host mirror says every slot of the range folds
    if (tid == 32) {
#pragma unroll
        for (int x = 0; x < 4; ++x) mbar_init(bar_S + x, 1);
        fence_mbar_init();
        if (a.spec && a.pdl_early) issue_state();
    }
    if (a.pdl) pdl_wait();   // counters, records (and the state unless pdl_early) may come from the previous grid
    pdl_trigger();
    if (tid == 32) {
        if (a.spec && !a.pdl_early) issue_state();
        const int mode = a.p.mode[r], occ = a.p.occ[r], len = a.p.len[r];
        int n = 0;
        bool zero_s0 = false;
        if (a.kind == FK_FULL)
            n = (mode == 0 && occ == dm.C) ? occ : 0;
        else if (mode == 1) {   // FK_FORCE: a direct slot compresses into a state, S0 = 0
            n = len;
            zero_s0 = true;
        } else
            n = occ;
        meta[0] = n;
        meta[1] = zero_s0;
        if (!a.spec && n > 0 && !zero_s0) issue_state();
    }
    const int kspec = PG ? 0 : min(kUtCh, a.kcap);   // first chunk requested before the counters are known
    if (kspec > 0) load_raw(0, kspec);
    __syncthreads();
    const int n = meta[0];
    const bool zero_s0 = meta[1] != 0;
    if (n == 0) {   // nothing to fold: state untouched, counters unchanged
        if (a.spec)   // the speculative copies must land before exit
            for (int x = 0; x < 4; ++x) mbar_wait(bar_S + x, 0);
        return;
    }
    if (zero_s0)
        for (int x = tid; x < kD * kD / 4; x += kUtThreads) reinterpret_cast<float4 *>(S_s)[x] = make_float4(0.f, 0.f, 0.f, 0.f);

    const int g = lane >> 2, t4 = lane & 3, lr = lane & 7, lm = lane >> 3;
    const int c = tid & (kD - 1), hh = tid >> 7;
    for (int s0 = 0; s0 < n; s0 += kUtCh) {
        const int kn = min(kUtCh, n - s0);
        const int nkt = (kn + 7) >> 3;   // 8-record tiles
        if (s0 > 0) __syncthreads();     // every warp is done with the previous chunk's operands
        if (s0 > 0 || kspec == 0) load_raw(s0, kn);
        store_raw(kn);
        __syncthreads();
        UT_MARK(1);

        // (1) L = strictLower(Diag(beta) (Gamma (.) K K^T)): warp nt computes
        //     Gram columns 8 nt .. 8 nt + 7 (m16n8k8 tf32; bf16 products exact),
        //     four independent partial sums
        if (warp < 2) {
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
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int i = g + 8 * (q >> 1), l = warp * 8 + 2 * t4 + (q & 1);
                const float kk_il = (acc4[0][q] + acc4[1][q]) + (acc4[2][q] + acc4[3][q]);
                Ls[i * 17 + l] = l < i ? Bs[i] * __expf(Gs[i] - Gs[l]) * kk_il : 0.f;
            }
        }
        // ... meanwhile every thread takes its key / value column into registers
        //     and writes the transposed keys (the fold's B operand)
        float kc[kUtCh], vc[kUtCh];
#pragma unroll
        for (int l = 0; l < kUtCh; ++l) {
            kc[l] = Ks[l * kUtS + c];
            vc[l] = Vs[l * kUtS + c];
        }
        {
            float kh[8];   // this thread's half of the column (select, not a dynamic register index)
#pragma unroll
            for (int u = 0; u < 8; ++u) kh[u] = hh ? kc[8 + u] : kc[u];
            if constexpr (FP32_IN) {
                *reinterpret_cast<float4 *>(Kc + c * kUtKc + hh * 8) = make_float4(kh[0], kh[1], kh[2], kh[3]);
                *reinterpret_cast<float4 *>(Kc + c * kUtKc + hh * 8 + 4) = make_float4(kh[4], kh[5], kh[6], kh[7]);
            } else {   // bf16 keys: record pairs as bf16x2 words, 12-word rows (conflict-free B reads)
                uint4 w;
                w.x = (__float_as_uint(kh[0]) >> 16) | (__float_as_uint(kh[1]) & 0xFFFF0000u);
                w.y = (__float_as_uint(kh[2]) >> 16) | (__float_as_uint(kh[3]) & 0xFFFF0000u);
                w.z = (__float_as_uint(kh[4]) >> 16) | (__float_as_uint(kh[5]) & 0xFFFF0000u);
                w.w = (__float_as_uint(kh[6]) >> 16) | (__float_as_uint(kh[7]) & 0xFFFF0000u);
                *reinterpret_cast<uint4 *>(reinterpret_cast<uint32_t *>(Kc) + c * 12 + hh * 4) = w;
            }
        }
        __syncthreads();
        UT_MARK(2);
        // (2) A = (I + L)^{-1} column by column (lane l: forward substitution on
        //     e_l); P = A Diag(beta), Q = A Diag(beta gamma)
        if (warp == 0 && lane < kUtCh) {
            float x[kUtCh];
#pragma unroll
            for (int i = 0; i < kUtCh; ++i) {
                float a0 = i == lane ? 1.f : 0.f, a1 = 0.f;
#pragma unroll
                for (int m = 0; m < i; m += 2) {
                    a0 = fmaf(-Ls[i * 17 + m], x[m], a0);
                    if (m + 1 < i) a1 = fmaf(-Ls[i * 17 + m + 1], x[m + 1], a1);
                }
                x[i] = a0 + a1;
            }
            const float bl = Bs[lane], ql = bl * expf(Gs[lane]);
#pragma unroll
            for (int i = 0; i < kUtCh; ++i) {
                Ps[i * kUtCh + lane] = x[i] * bl;
                uint32_t qh, qlo;
                split_tf32(__float_as_uint(x[i] * ql) ^ 0x80000000u, qh, qlo);
                Qn[i * kUtQn + lane] = __uint_as_float(qh);
                Qn[kUtCh * kUtQn + i * kUtQn + lane] = __uint_as_float(qlo);
            }
        }
        __syncthreads();
        UT_MARK(3);
        // (3) V~ = P V in place of V (thread: column c, rows 2 m + hh; P lower
        //     triangular; the column was read into registers above)
#pragma unroll
        for (int m = 0; m < kUtCh / 2; ++m) {
            const int i = 2 * m + hh;
            const float4 *p4 = reinterpret_cast<const float4 *>(Ps + i * kUtCh);
            float av = 0.f;
#pragma unroll
            for (int l4 = 0; l4 < kUtCh / 4; ++l4) {
                if (4 * l4 <= 2 * m + 1) {
                    const float4 pp = p4[l4];
                    av = fmaf(pp.x, vc[4 * l4], fmaf(pp.y, vc[4 * l4 + 1], fmaf(pp.z, vc[4 * l4 + 2], fmaf(pp.w, vc[4 * l4 + 3], av))));
                }
            }
            Vs[i * kUtS + c] = av;
        }
        __syncthreads();
        UT_MARK(4);

        // (4) warp w: d_v rows j = 16 w .. 16 w + 15 (32-row block w / 2)
        if (s0 == 0 && !zero_s0) mbar_wait(bar_S + (warp >> 1), 0);
        UT_MARK(5);
        float acc[2][4];   // U^T [row g (+8)][record 8 nt + 2 t4 (+1)], from V~^T
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int q = 0; q < 4; ++q)
                acc[nt][q] = Vs[(nt * 8 + 2 * t4 + (q & 1)) * kUtS + warp * 16 + g + 8 * (q >> 1)];
        {
            // W^T = S K^T (W = K S^T of the UT transform, P:397 with K~ = Q K):
            // independent chains per (record tile, pass); bf16 keys are exact in
            // TF32 (S_hi K + S_lo K), fp32 keys add S_hi K_lo
            constexpr int NP = FP32_IN ? 3 : 2;
            float wp[2][NP][4] = {};
            uint32_t aoff[4];
#pragma unroll
            for (int c8 = 0; c8 < 4; ++c8)
                aoff[c8] = (uint32_t)((lr + (lm & 1) * 8) * 128 + (((2 * c8 + (lm >> 1)) ^ lr) << 4));
            const uint32_t abase = smem_u32(S_s) + warp * 2048;
            const uint32_t bbase = smem_u32(Ks) + (uint32_t)((lr * kUtS + (lm & 1) * 4) * 4);
#pragma unroll 4
            for (int kk = 0; kk < kD / 8; ++kk) {
                uint32_t x[4], ah[4], al[4];
                ldsm_x4(x, abase + (kk >> 2) * 16384 + aoff[kk & 3]);
#pragma unroll
                for (int q = 0; q < 4; ++q) split_tf32(x[q], ah[q], al[q]);
#pragma unroll
                for (int nt = 0; nt < 2; ++nt) {
                    if (nt < nkt) {
                        uint32_t bk[2];
                        ldsm_x2(bk, bbase + (uint32_t)((nt * 8 * kUtS + kk * 8) * 4));
                        if constexpr (FP32_IN) {
                            uint32_t bh[2], bl[2];
                            split_tf32(bk[0], bh[0], bl[0]);
                            split_tf32(bk[1], bh[1], bl[1]);
                            mma_tf32_16x8x8(wp[nt][0], ah, bh[0], bh[1]);
                            mma_tf32_16x8x8(wp[nt][1], al, bh[0], bh[1]);
                            mma_tf32_16x8x8(wp[nt][NP - 1], ah, bl[0], bl[1]);
                        } else {
                            mma_tf32_16x8x8(wp[nt][0], ah, bk[0], bk[1]);
                            mma_tf32_16x8x8(wp[nt][1], al, bk[0], bk[1]);
                        }
                    }
                }
            }
            // U^T += W^T (-Q)^T: the W^T accumulator fragment is the A fragment
            // of this product with the record index permuted inside each 8-record
            // tile (slot t <-> record 2t, slot t+4 <-> record 2t+1); B = -Q rows
            // (hi, lo), 8-byte reads; W split hi + lo in registers
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
                if (ks < nkt) {
                    float w[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        w[q] = wp[ks][0][q] + wp[ks][1][q];
                        if constexpr (FP32_IN) w[q] += wp[ks][NP - 1][q];
                    }
                    const float wa[4] = {w[0], w[2], w[1], w[3]};
                    uint32_t wh[4], wl[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) split_tf32(__float_as_uint(wa[q]), wh[q], wl[q]);
#pragma unroll
                    for (int nt = 0; nt < 2; ++nt) {
                        if (nt < nkt) {
                            const float2 qh = *reinterpret_cast<const float2 *>(Qn + (nt * 8 + g) * kUtQn + ks * 8 + 2 * t4);
                            const float2 ql = *reinterpret_cast<const float2 *>(Qn + kUtCh * kUtQn + (nt * 8 + g) * kUtQn + ks * 8 + 2 * t4);
                            mma_tf32_16x8x8(acc[nt], wh, __float_as_uint(qh.x), __float_as_uint(qh.y));
                            mma_tf32_16x8x8(acc[nt], wl, __float_as_uint(qh.x), __float_as_uint(qh.y));
                            mma_tf32_16x8x8(acc[nt], wh, __float_as_uint(ql.x), __float_as_uint(ql.y));
                        }
                    }
                }
            }
        }
        UT_MARK(6);
        const float gl = Gs[kn - 1], eg = __expf(gl);
        const int j0 = warp * 16 + g;
        if constexpr (!FP32_IN) {
            // (5') bf16 keys: D^T = Y^T K on m16n8k16 bf16 (products exact, fp32
            //      accumulate) with Y split into three bf16 pieces (24 significant
            //      bits): the U^T accumulator pairs {Y[row][2t], Y[row][2t+1]} are the
            //      bf16 A fragment as they stand; B = the packed key-pair words
            uint32_t ya[3][4];
            {
                float wv[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) wv[e] = __expf(gl - Gs[(e >> 1) * 8 + 2 * t4 + (e & 1)]);
                // fragment q: rows g (q even) / g + 8 (q odd), records 2 t (+1) of tile q >> 1
                const float yv[4][2] = {{wv[0] * acc[0][0], wv[1] * acc[0][1]}, {wv[0] * acc[0][2], wv[1] * acc[0][3]},
                                        {wv[2] * acc[1][0], wv[3] * acc[1][1]}, {wv[2] * acc[1][2], wv[3] * acc[1][3]}};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    float x0 = yv[q][0], x1 = yv[q][1];
#pragma unroll
                    for (int pc = 0; pc < 3; ++pc) {
                        const __nv_bfloat162 b2 = __floats2bfloat162_rn(x0, x1);
                        ya[pc][q] = *reinterpret_cast<const uint32_t *>(&b2);
                        x0 -= __low2float(b2);
                        x1 -= __high2float(b2);
                    }
                }
            }
            const uint32_t *Kw = reinterpret_cast<const uint32_t *>(Kc);
#pragma unroll 4
            for (int ct = 0; ct < kD / 8; ++ct) {
                float dp[3][4] = {};
                const uint32_t *kr = Kw + (ct * 8 + g) * 12 + t4;
                const uint32_t b0 = kr[0], b1 = kr[4];
#pragma unroll
                for (int pc = 0; pc < 3; ++pc) mma_bf16_16x8x16(dp[pc], ya[pc], b0, b1);
                float d[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) d[q] = dp[0][q] + (dp[1][q] + dp[2][q]);
                const int cc = ct * 8 + 2 * t4;
                float2 *p0 = reinterpret_cast<float2 *>(smem + L.S + ut_sw(j0, cc));
                float2 *p1 = reinterpret_cast<float2 *>(smem + L.S + ut_sw(j0 + 8, cc));
                float2 s0v = *p0, s1v = *p1;
                s0v.x = fmaf(eg, s0v.x, d[0]); s0v.y = fmaf(eg, s0v.y, d[1]);
                s1v.x = fmaf(eg, s1v.x, d[2]); s1v.y = fmaf(eg, s1v.y, d[3]);
                *p0 = s0v;
                *p1 = s1v;
            }
        } else {
        // (5) Y = e^{G_last - G_i} u_i in the same fragments, split hi + lo; as the A
        //     fragment of D^T = Y^T K: a = {Y[g][2t], Y[g+8][2t], Y[g][2t+1], Y[g+8][2t+1]}
        uint32_t yh[2][4], yl[2][4];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
            const float w0 = __expf(gl - Gs[nt * 8 + 2 * t4]), w1 = __expf(gl - Gs[nt * 8 + 2 * t4 + 1]);
            const float y[4] = {w0 * acc[nt][0], w0 * acc[nt][2], w1 * acc[nt][1], w1 * acc[nt][3]};
#pragma unroll
            for (int q = 0; q < 4; ++q) split_tf32(__float_as_uint(y[q]), yh[nt][q], yl[nt][q]);
        }
        // (6) D^T[j][c] = sum_i Y[i][j] k_i[c] per 8-column tile of d_k (independent
        //     chains per (record tile, pass)), then S = gamma_last S + D^T in the tile
        //     (pairs of columns: 8-byte accesses)
#pragma unroll 4
        for (int ct = 0; ct < kD / 8; ++ct) {
            float dp[2][3][4] = {};
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
            float2 *p0 = reinterpret_cast<float2 *>(smem + L.S + ut_sw(j0, cc));
            float2 *p1 = reinterpret_cast<float2 *>(smem + L.S + ut_sw(j0 + 8, cc));
            float2 s0v = *p0, s1v = *p1;
            s0v.x = fmaf(eg, s0v.x, d[0]); s0v.y = fmaf(eg, s0v.y, d[1]);
            s1v.x = fmaf(eg, s1v.x, d[2]); s1v.y = fmaf(eg, s1v.y, d[3]);
            *p0 = s0v;
            *p1 = s1v;
        }
        }
        UT_MARK(7);
    }
    // ---- the warp pair's 32 rows leave as soon as both warps are done
    fence_proxy_async_smem();
    named_bar_sync(1 + (warp >> 1), 64);
    if ((warp & 1) == 0 && lane == 0) {
        const int x = warp >> 1;
#pragma unroll
        for (int kb = 0; kb < 4; ++kb)
            tma_store_2d(&tmap, smem + L.S + kb * 16384 + x * 4096, kb * 32, row0 + x * 32);
        bulk_commit();
        // ---- counters: the last CTA of the slot resets the buffer
        if (x == 0 && atomicAdd(&a.p.ticket[r], 1) == (int)gridDim.x - 1) {
            a.p.ticket[r] = 0;
            a.p.occ[r] = 0;
            if (zero_s0) { a.p.mode[r] = 0; a.p.len[r] = 0; }
        }
        bulk_wait_read0();   // shared memory must stay live until the stores have read it
    }
    UT_MARK(8);
}

template <typename InT, bool FP32_IN>
static cudaError_t launch_ut_t(const FoldArgs &a, cudaStream_t s) {
    const UtSmem L = ut_smem_layout();
    const bool pg = a.slots || a.p.btab || a.p.sidx;
    auto kfn = pg ? fold_ut_kernel<InT, FP32_IN, true> : fold_ut_kernel<InT, FP32_IN, false>;
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(kfn, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;
    const CUtensorMap tm = *static_cast<const CUtensorMap *>(a.tmap);
    return launch_k(kfn, dim3(a.dm.Hv, a.n), dim3(kUtThreads), L.total, s, a.pdl != 0, a, tm);
}

cudaError_t launch_fold_ut(const FoldArgs &a, cudaStream_t s) {
    if (!a.tmap || (a.kind != FK_FULL && a.kind != FK_FORCE)) return cudaErrorInvalidValue;
    if (a.dm.in_dt == DT_F32) return launch_ut_t<float, true>(a, s);
    return launch_ut_t<__nv_bfloat16, false>(a, s);
}

}  // namespace labuf
