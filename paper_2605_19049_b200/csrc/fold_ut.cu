// fold_ut.cu — kernel (2 RAW): flush mode ii.  The delta values are not read
// from the buffer but recomputed from the raw records (k_i, v_i, beta_i, G_i)
// and the state by the chunkwise UT transform of P:392-399 (K~ corrected per
// reading Z4), then folded into the state on the 5th-generation tensor cores:
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
// B200 structure: ONE CTA of 8 warps per (V head, slot), so the UT transform
// (Gram, triangular inverse, K~, V~) is computed once per head and the TMEM
// allocation is paid once per head (≈ 0.5 µs of SM-serialised time per
// allocating CTA, tools/microbench_tmem.cu), not once per 32-row tile.
//   * entry: the 64 KiB state arrives by 16 TMA boxes (32 x 32 fp32, 128-byte
//     swizzle) while every thread loads its raw records (8 keys, 8 values);
//   * everything that does not need the state runs while it is in flight:
//     the 16 x 16 Gram K K^T on mma.sync (2 warps), the inverse of the unit
//     lower-triangular I + L by forward substitution on the identity (one
//     warp, lane = column), K~ and V~ on CUDA cores;
//   * U^T = V~^T - S K~^T: one m16 tile of d_v rows per warp, A = the state
//     straight from the swizzled TMA tile by ldmatrix, B = K~ rows, split
//     TF32 (S_hi K~_hi + S_lo K~_hi + S_hi K~_lo: fp32-accurate products), the
//     accumulator initialised with V~^T;
//   * the results, scaled by e^{G_last - G_i}, are written straight from the
//     fragments as the B operand (hi + lo) of one tcgen05.mma.kind::tf32
//     M = 128 (d_k) x N = 128 (d_v) x K = 16 fold with the accumulator in TMEM;
//   * epilogue: tcgen05.ld, S = gamma_last S + D in the swizzled tile (lane =
//     key index c: conflict-free), 16 TMA box stores.
// Shared memory ≈ 108 KiB (bf16 records): 2 CTAs per SM.
#include <cuda.h>

#include "device.cuh"
#include "internal.h"

namespace labuf {

constexpr int kUtCh = 16;          // records per UT chunk
constexpr int kUtThreads = 256;    // 8 warps: one m16 tile of d_v rows each
constexpr int kUtS = 132;          // fp32 record rows padded to 132 floats (conflict-free ldmatrix)

struct UtSmem {
    uint32_t S, X, Kt, Vt, A, Alo, Ls, Qs, Ps, Gs, Bs, bar, total;
};
__host__ __device__ inline UtSmem ut_smem_layout(bool fp32_in) {
    UtSmem L;
    uint32_t o = 0;
    L.S = o;   o += kD * kD * 4;               // state: 4 column groups x 128 rows x 128 B, SW128
    L.X = o;   o += 2 * kUtCh * kUtS * 4;      // raw keys + raw values; then the fold's B (hi, lo)
    L.Kt = o;  o += kUtCh * kUtS * 4;          // K~
    L.Vt = o;  o += kUtCh * kUtS * 4;          // V~
    L.A = o;   o += kD * kUtCh * 4;            // fold A = K^T (K-major, no swizzle)
    L.Alo = o; o += fp32_in ? kD * kUtCh * 4 : 0;
    L.Ls = o;  o += kUtCh * 17 * 4;            // L (row stride 17)
    L.Qs = o;  o += kUtCh * kUtCh * 4;         // A Diag(beta gamma)
    L.Ps = o;  o += kUtCh * kUtCh * 4;         // A Diag(beta)
    L.Gs = o;  o += kUtCh * 4;                 // G_i relative to the chunk's entering state
    L.Bs = o;  o += kUtCh * 4;                 // beta_i
    L.bar = o; o += 64;
    L.total = o;
    return L;
}

// byte offset of element (row, k) in a K-major SWIZZLE_NONE operand of 16
// columns: 8x(16 B) core matrices, K-adjacent at +128 B, 8-row groups at +512 B
__device__ __forceinline__ uint32_t ut_kmaj(int row, int k) {
    return (uint32_t)((row >> 3) * 512 + (k >> 2) * 128 + (row & 7) * 16 + (k & 3) * 4);
}
// byte offset of state element (d_v row j, d_k column c) in the TMA tile:
// column group c / 32 (16 KiB each), row j (128 B), 16-byte chunk ^= j % 8
__device__ __forceinline__ uint32_t ut_sw(int j, int c) {
    return (uint32_t)((c >> 5) * 16384 + j * 128 + ((((c & 31) >> 2) ^ (j & 7)) << 4) + (c & 3) * 4);
}
__device__ __forceinline__ void tma_store_2d(const void *tmap, const void *src_smem, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];"
                 ::"l"(tmap), "r"(smem_u32(src_smem)), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void split_tf32(uint32_t x, uint32_t &hi, uint32_t &lo) {
    hi = x & 0xFFFFE000u;
    lo = __float_as_uint(__uint_as_float(x) - __uint_as_float(hi));
}

template <typename InT, bool FP32_IN, bool PG>
__global__ void __launch_bounds__(kUtThreads, 2)
    fold_ut_kernel(const FoldArgs a, const __grid_constant__ CUtensorMap tmap) {
    const int h = blockIdx.x, zi = blockIdx.y;
    if constexpr (PG) {   // slot lists, state indices and block tables may come from the previous grid
        if (a.pdl) pdl_wait();
    }
    const int r = PG && a.slots ? __ldcg(a.slots + zi) : a.first + zi;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const Dims dm = a.dm;
    const int Hv = dm.Hv, bt = dm.bt, hk = h / dm.g;

    extern __shared__ __align__(1024) unsigned char smem[];
    const UtSmem L = ut_smem_layout(FP32_IN);
    float *S_s = reinterpret_cast<float *>(smem + L.S);
    float *Ks = reinterpret_cast<float *>(smem + L.X), *Vs = Ks + kUtCh * kUtS;
    unsigned char *Bhi = smem + L.X, *Blo = smem + L.X + kD * kUtCh * 4;
    float *Kt = reinterpret_cast<float *>(smem + L.Kt), *Vt = reinterpret_cast<float *>(smem + L.Vt);
    unsigned char *Aop = smem + L.A, *Alo = smem + L.Alo;
    float *Ls = reinterpret_cast<float *>(smem + L.Ls), *Qs = reinterpret_cast<float *>(smem + L.Qs);
    float *Ps = reinterpret_cast<float *>(smem + L.Ps);
    float *Gs = reinterpret_cast<float *>(smem + L.Gs), *Bs = reinterpret_cast<float *>(smem + L.Bs);
    uint64_t *bar_ld = reinterpret_cast<uint64_t *>(smem + L.bar);
    uint64_t *bar_mma = bar_ld + 1;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bar_ld + 2);
    int *meta = reinterpret_cast<int *>(bar_ld + 3);   // n, zero_s0
    const size_t sb = PG && a.p.sidx ? (size_t)__ldcg(a.p.sidx + r) : (size_t)r;
    const int row0 = (int)((sb * Hv + h) * kD);

    auto issue_state = [&]() {
        mbar_arrive_expect_tx(bar_ld, kD * kD * 4);
#pragma unroll
        for (int kb = 0; kb < 4; ++kb)
#pragma unroll
            for (int x = 0; x < 4; ++x)
                tma_load_2d(smem + L.S + kb * 16384 + x * 4096, &tmap, kb * 32, row0 + x * 32, bar_ld);
    };
    // record position i of the slot: (block, offset) -- the block table or the slot's own region
    auto at = [&](int i) -> int2 { return PG ? rec_at(dm, a.p, r, i) : make_int2(r, i); };

    // per-thread raw operands: column c of records hh*8 .. hh*8+7 of the chunk
    const int c = tid & (kD - 1), hh = tid >> 7;
    float kr[8], vr[8], gr = 0.f, br = 0.f, gbase = 0.f;
    auto load_raw = [&](int s0, int kn) {
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const int i = hh * 8 + m;
            kr[m] = vr[m] = 0.f;
            if (i < kn) {
                const int2 ba = at(s0 + i);
                kr[m] = to_f(static_cast<const InT *>(a.p.K)[(((size_t)ba.x * dm.Hk + hk) * bt + ba.y) * kD + c]);
                vr[m] = to_f(static_cast<const InT *>(a.p.V)[(((size_t)ba.x * Hv + h) * bt + ba.y) * kD + c]);
            }
        }
        if (tid < kUtCh) {
            gr = br = 0.f;
            if (tid < kn) {
                const int2 ba = at(s0 + tid);
                const size_t o = ((size_t)ba.x * Hv + h) * bt + ba.y;
                gr = a.p.G[o];
                br = a.p.B[o];
            }
            gbase = 0.f;
            if (s0 > 0) {
                const int2 ba = at(s0 - 1);
                gbase = a.p.G[((size_t)ba.x * Hv + h) * bt + ba.y];
            }
        }
    };
    // rows >= kn are zero in every operand (loads past a slot's own count are never used)
    auto store_raw = [&](int kn) {
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const int i = hh * 8 + m;
            const float x = i < kn ? kr[m] : 0.f;
            Ks[i * kUtS + c] = x;
            Vs[i * kUtS + c] = i < kn ? vr[m] : 0.f;
            const uint32_t off = ut_kmaj(c, i);
            if constexpr (FP32_IN) {
                const float hi = tf32_rna(x);
                *reinterpret_cast<float *>(Aop + off) = hi;
                *reinterpret_cast<float *>(Alo + off) = x - hi;
            } else {
                *reinterpret_cast<float *>(Aop + off) = x;   // bf16 keys are exact in tf32
            }
        }
        if (tid < kUtCh) {
            Gs[tid] = tid < kn ? gr - gbase : 0.f;
            Bs[tid] = tid < kn ? br : 0.f;
        }
    };

    // ---- which records fold (uniform over the slot's CTAs); the state in
    //      flight at once when the host mirror says every slot of the range folds
    if (warp == 0) tmem_alloc<128>(tmem_slot);
    if (tid == 32) {
        mbar_init(bar_ld, 1);
        mbar_init(bar_mma, 1);
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
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const int n = meta[0];
    const bool zero_s0 = meta[1] != 0;
    const uint32_t tmem = *tmem_slot;
    if (n == 0) {   // nothing to fold: state untouched, counters unchanged
        if (a.spec) mbar_wait(bar_ld, 0);   // the speculative copy must land before exit
        if (warp == 0) tmem_dealloc<128>(tmem);
        return;
    }
    if (zero_s0)
        for (int x = tid; x < kD * kD / 4; x += kUtThreads) reinterpret_cast<float4 *>(S_s)[x] = make_float4(0.f, 0.f, 0.f, 0.f);

    const int g = lane >> 2, t4 = lane & 3, lr = lane & 7, lm = lane >> 3;
    const uint32_t idesc = idesc_tf32(128, 128);
    uint32_t mma_phase = 0;
    for (int s0 = 0; s0 < n; s0 += kUtCh) {
        const int kn = min(kUtCh, n - s0);
        const int nkt = (kn + 7) >> 3;   // 8-record k / n tiles
        if (s0 > 0 || kspec == 0) load_raw(s0, kn);
        store_raw(kn);
        __syncthreads();

        // (1) L = strictLower(Diag(beta) (Gamma (.) K K^T)): warp nt computes
        //     Gram columns 8 nt .. 8 nt + 7 (m16n8k8 tf32; bf16 products exact)
        if (warp < 2) {
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
            if (warp < nkt) {
                const uint32_t ab = smem_u32(Ks) + (uint32_t)(((lr + (lm & 1) * 8) * kUtS + (lm >> 1) * 4) * 4);
                const uint32_t bb = smem_u32(Ks) + (uint32_t)(((warp * 8 + lr) * kUtS + (lm & 1) * 4) * 4);
#pragma unroll 4
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
                        mma_tf32_16x8x8(acc, ah, bh[0], bh[1]);
                        mma_tf32_16x8x8(acc, al, bh[0], bh[1]);
                        mma_tf32_16x8x8(acc, ah, bl[0], bl[1]);
                    } else {
                        mma_tf32_16x8x8(acc, ka, kb[0], kb[1]);
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int i = g + 8 * (q >> 1), l = warp * 8 + 2 * t4 + (q & 1);
                Ls[i * 17 + l] = l < i ? Bs[i] * __expf(Gs[i] - Gs[l]) * acc[q] : 0.f;
            }
        }
        __syncthreads();
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
                Qs[i * kUtCh + lane] = x[i] * ql;
            }
        }
        __syncthreads();
        // (3) K~ = Q K, V~ = P V (thread: column c, rows 2 m + hh; Q, P lower triangular)
        {
            float kc[kUtCh], vc[kUtCh];
#pragma unroll
            for (int l = 0; l < kUtCh; ++l) {
                kc[l] = Ks[l * kUtS + c];
                vc[l] = Vs[l * kUtS + c];
            }
#pragma unroll
            for (int m = 0; m < kUtCh / 2; ++m) {
                const int i = 2 * m + hh;
                const float4 *q4 = reinterpret_cast<const float4 *>(Qs + i * kUtCh);
                const float4 *p4 = reinterpret_cast<const float4 *>(Ps + i * kUtCh);
                float ak = 0.f, av = 0.f;
#pragma unroll
                for (int l4 = 0; l4 < kUtCh / 4; ++l4) {
                    if (4 * l4 <= 2 * m + 1) {
                        const float4 qq = q4[l4], pp = p4[l4];
                        ak = fmaf(qq.x, kc[4 * l4], fmaf(qq.y, kc[4 * l4 + 1], fmaf(qq.z, kc[4 * l4 + 2], fmaf(qq.w, kc[4 * l4 + 3], ak))));
                        av = fmaf(pp.x, vc[4 * l4], fmaf(pp.y, vc[4 * l4 + 1], fmaf(pp.z, vc[4 * l4 + 2], fmaf(pp.w, vc[4 * l4 + 3], av))));
                    }
                }
                Kt[i * kUtS + c] = ak;
                Vt[i * kUtS + c] = av;
            }
        }
        __syncthreads();
        if (s0 == 0 && !zero_s0) mbar_wait(bar_ld, 0);

        // (4) U^T = V~^T - S K~^T: warp w, d_v rows 16 w .. 16 w + 15, records in
        //     n tiles of 8; A = S from the swizzled tile, B = -K~ (split TF32)
        {
            float acc[2][4];
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    acc[nt][q] = Vt[(nt * 8 + 2 * t4 + (q & 1)) * kUtS + warp * 16 + g + 8 * (q >> 1)];
            uint32_t aoff[4];
#pragma unroll
            for (int c8 = 0; c8 < 4; ++c8)
                aoff[c8] = (uint32_t)((lr + (lm & 1) * 8) * 128 + (((2 * c8 + (lm >> 1)) ^ lr) << 4));
            const uint32_t abase = smem_u32(S_s) + warp * 2048;
            const uint32_t bbase = smem_u32(Kt) + (uint32_t)((lr * kUtS + (lm & 1) * 4) * 4);
#pragma unroll 4
            for (int kk = 0; kk < kD / 8; ++kk) {
                uint32_t x[4], ah[4], al[4];
                ldsm_x4(x, abase + (kk >> 2) * 16384 + aoff[kk & 3]);
#pragma unroll
                for (int q = 0; q < 4; ++q) split_tf32(x[q], ah[q], al[q]);
#pragma unroll
                for (int nt = 0; nt < 2; ++nt) {
                    if (nt < nkt) {
                        uint32_t b[2], bh[2], bl[2];
                        ldsm_x2(b, bbase + (uint32_t)((nt * 8 * kUtS + kk * 8) * 4));
                        split_tf32(b[0], bh[0], bl[0]);
                        split_tf32(b[1], bh[1], bl[1]);
                        bh[0] ^= 0x80000000u; bh[1] ^= 0x80000000u;
                        bl[0] ^= 0x80000000u; bl[1] ^= 0x80000000u;
                        mma_tf32_16x8x8(acc[nt], ah, bh[0], bh[1]);
                        mma_tf32_16x8x8(acc[nt], al, bh[0], bh[1]);
                        mma_tf32_16x8x8(acc[nt], ah, bl[0], bl[1]);
                    }
                }
            }
            // (5) fold operand B = (e^{G_last - G_i} u_i)^T: row j (d_v), column i, hi + lo
            const float gl = Gs[kn - 1];
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int i = nt * 8 + 2 * t4 + (q & 1), j = warp * 16 + g + 8 * (q >> 1);
                    const float y = i < kn ? __expf(gl - Gs[i]) * acc[nt][q] : 0.f;
                    const float hi = tf32_rna(y);
                    const uint32_t off = ut_kmaj(j, i);
                    *reinterpret_cast<float *>(Bhi + off) = hi;
                    *reinterpret_cast<float *>(Blo + off) = y - hi;
                }
        }
        fence_proxy_async_smem();
        __syncthreads();
        // (6) D[c][j] = sum_i k_i[c] y_i[j]: M = 128 (d_k), N = 128 (d_v), K = 8 per k tile
        if (tid == 0) {
            tc_fence_after();
            for (int kt = 0; kt < nkt; ++kt) {
                const uint32_t koff = kt * 256;   // 8 tf32 = 2 core matrices along K
                const uint64_t da = umma_desc_noswz(smem_u32(Aop) + koff, 128, 512);
                const uint64_t dbh = umma_desc_noswz(smem_u32(Bhi) + koff, 128, 512);
                const uint64_t dbl = umma_desc_noswz(smem_u32(Blo) + koff, 128, 512);
                tc_mma_tf32(tmem, da, dbh, idesc, kt > 0 ? 1u : 0u);
                tc_mma_tf32(tmem, da, dbl, idesc, 1u);
                if constexpr (FP32_IN) {
                    const uint64_t dal = umma_desc_noswz(smem_u32(Alo) + koff, 128, 512);
                    tc_mma_tf32(tmem, dal, dbh, idesc, 1u);
                }
            }
            tc_commit(bar_mma);
        }
        mbar_wait(bar_mma, mma_phase);
        mma_phase ^= 1;
        tc_fence_after();
        // (7) S = gamma_last S + D: warp w reads TMEM lanes 32 (w % 4) .. (key index c)
        //     and d_v columns 64 (w / 4) .. + 63
        {
            const float eg = __expf(Gs[kn - 1]);
            const int q4 = warp & 3, cw = 32 * q4 + lane;
#pragma unroll
            for (int xh = 0; xh < 2; ++xh) {
                float v[32];
                const int j0 = (warp >> 2) * 64 + xh * 32;
                tmem_ld32(tmem + ((uint32_t)(32 * q4) << 16) + (uint32_t)j0, v);
#pragma unroll
                for (int jj = 0; jj < 32; ++jj) {
                    float *p = reinterpret_cast<float *>(smem + L.S + ut_sw(j0 + jj, cw));
                    *p = fmaf(eg, *p, v[jj]);
                }
            }
        }
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
#pragma unroll
        for (int kb = 0; kb < 4; ++kb)
#pragma unroll
            for (int x = 0; x < 4; ++x)
                tma_store_2d(&tmap, smem + L.S + kb * 16384 + x * 4096, kb * 32, row0 + x * 32);
        bulk_commit();
    }
    if (warp == 0) tmem_dealloc<128>(tmem);
    // ---- counters: the last CTA of the slot resets the buffer
    if (tid == 0) {
        if (atomicAdd(&a.p.ticket[r], 1) == (int)gridDim.x - 1) {
            a.p.ticket[r] = 0;
            a.p.occ[r] = 0;
            if (zero_s0) { a.p.mode[r] = 0; a.p.len[r] = 0; }
        }
        bulk_wait_read0();   // shared memory must stay live until the stores have read it
    }
}

template <typename InT, bool FP32_IN>
static cudaError_t launch_ut_t(const FoldArgs &a, cudaStream_t s) {
    const UtSmem L = ut_smem_layout(FP32_IN);
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
