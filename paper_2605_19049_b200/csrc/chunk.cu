// chunk.cu — kernels (1) buffered decode, (3) parallel draft verification,
// (4) direct short-context decoding, and the prefill chunk step.
//
// All compute, for n_new new tokens t of one request slot r and the g V
// heads of one QK head, against j0 buffered records (k_i, u_i, G_i):
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
// B200 structure: one light CTA per (d_v tile of ROWS rows x g V heads, QK
// head, slot).  At entry the lanes of warp 0 issue one bulk copy each
// (cp.async.bulk -> SASS UBLKCP) for every operand of the CTA — the fp32
// state tile, the buffered u sub-tiles, key rows and log decays, and the new
// tokens — onto a single mbarrier, so a CTA's whole working set is in flight
// at once and several CTAs per SM keep HBM busy.  The CTA then computes from
// shared memory with one block barrier (before the forward substitution).
#include "device.cuh"
#include "internal.h"

namespace labuf {

struct CtaLayout {
    uint32_t S, U, K, Gs, q, k, v, Ck, Cq, av, bv, Gn, Bn, bar, bytes;
};

__host__ __device__ inline uint32_t al128(uint32_t x) { return (x + 127u) & ~127u; }

__host__ __device__ inline CtaLayout cta_layout(int G, int ROWS, int nt, bool has_state, int jcap,
                                                int isz, int usz) {
    CtaLayout L;
    const int J = jcap + nt;
    uint32_t o = 0;
    L.S = o;  o = al128(o + (has_state ? (uint32_t)(G * ROWS * kD * 4) : 0u));
    L.U = o;  o = al128(o + (uint32_t)(G * ROWS * jcap * usz));
    L.K = o;  o = al128(o + (uint32_t)(jcap * kD * isz));
    L.Gs = o; o = al128(o + (uint32_t)(G * ((jcap + 3) & ~3) * 4));
    L.q = o;  o = al128(o + (uint32_t)(nt * kD * isz));
    L.k = o;  o = al128(o + (uint32_t)(nt * kD * isz));
    L.v = o;  o = al128(o + (uint32_t)(nt * G * ROWS * isz));
    L.Ck = o; o = al128(o + (uint32_t)(G * nt * J * 4));
    L.Cq = o; o = al128(o + (uint32_t)(G * nt * J * 4));
    L.av = o; o = al128(o + (uint32_t)(has_state ? G * nt * ROWS * 4 : 0));
    L.bv = o; o = al128(o + (uint32_t)(has_state ? G * nt * ROWS * 4 : 0));
    L.Gn = o; o = al128(o + (uint32_t)(G * nt * 4));
    L.Bn = o; o = al128(o + (uint32_t)(G * nt * 4));
    L.bar = o; o += 16;
    L.bytes = al128(o);
    return L;
}

template <int NT>
struct MatvecGroups {
    // rows per reduction group so that 2 * NT * RG values fit one transposed reduction
    static constexpr int RG = (16 / NT) > 0 ? 16 / NT : 1;
};

template <typename InT, typename UT, int G, int ROWS, int NT, bool HAS_STATE, int MINB>
__global__ void __launch_bounds__(256, MINB) chunk_cta_kernel(const ChunkArgs a) {
    constexpr int NTHR = 256, NWARP = 8;
    constexpr int GR = G * ROWS;                 // rows of this CTA (flattened over heads)
    constexpr int SUB = ROWS / kUSub;            // u sub-tiles per head
    constexpr int RPW = GR / NWARP;              // mat-vec rows per warp
    constexpr int RG = MatvecGroups<NT>::RG < RPW ? MatvecGroups<NT>::RG : RPW;
    constexpr int NV = 2 * NT * RG;
    static_assert(GR <= NTHR, "one thread per (head,row) in the forward substitution");
    static_assert(RPW % RG == 0, "row grouping");
    static_assert(G * NT <= 32, "decay scan runs inside one warp");

    const int tile = blockIdx.x, hk = blockIdx.y, zi = blockIdx.z;
    const int r = a.first + zi;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const Dims dm = a.dm;
    const int T = dm.T, Hv = dm.Hv, Hk = dm.Hk;
    const int n_new = a.n_new;
    const bool direct = (a.kind == CK_DIRECT);
    constexpr int isz = (int)sizeof(InT), usz = (int)sizeof(UT);
    const int *cnt = direct ? a.p.len : a.p.occ;
    const int j0 = cnt[r] + a.j_add;
    const int jb = (j0 + 3) & ~3;
    const int Jst = a.j0_cap + NT;               // row stride of Ck/Cq

    extern __shared__ __align__(1024) unsigned char smem[];
    const CtaLayout L = cta_layout(G, ROWS, NT, HAS_STATE, a.j0_cap, isz, usz);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + L.bar);
    const float *S_s = reinterpret_cast<const float *>(smem + L.S);
    const UT *U_s = reinterpret_cast<const UT *>(smem + L.U);
    const InT *K_s = reinterpret_cast<const InT *>(smem + L.K);
    const float *G_s = reinterpret_cast<const float *>(smem + L.Gs);
    const InT *q_s = reinterpret_cast<const InT *>(smem + L.q);
    const InT *k_s = reinterpret_cast<const InT *>(smem + L.k);
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

    // ---- 1. warp 0: one bulk copy per lane for every operand of the CTA
    if (warp == 0) {
        if (lane == 0) {
            mbar_init(full, 1);
            fence_mbar_init();
            uint32_t total = (HAS_STATE ? (uint32_t)(GR * kD * 4) : 0u) + (uint32_t)(GR * j0 * usz) +
                             (uint32_t)(j0 * kD * isz) + (j0 ? (uint32_t)(G * jb * 4) : 0u) +
                             (uint32_t)(n_new * (2 * kD * isz + GR * isz));
            mbar_arrive_expect_tx(full, total);
        }
        __syncwarp();
        const int nS = HAS_STATE ? G : 0, nU = j0 ? G * SUB : 0, nK = j0 ? 1 : 0, nG = j0 ? G : 0;
        const int nQ = n_new;
        const int ncopy = nS + nU + nK + nG + 2 * nQ + nQ * G;
        unsigned char *sm = smem;
        for (int c = lane; c < ncopy; c += 32) {
            int x = c;
            if (x < nS) {
                bulk_g2s(sm + L.S + (size_t)x * ROWS * kD * 4,
                         a.p.state + (((size_t)r * Hv + hk * G + x) * kD + (size_t)tile * ROWS) * kD,
                         ROWS * kD * 4, full);
                continue;
            }
            x -= nS;
            if (x < nU) {
                const int hh = x / SUB, sb = x % SUB;
                const UT *src = static_cast<const UT *>(a.p.U) +
                                ((((size_t)r * Hv + hk * G + hh) * (kD / kUSub) + tile * SUB + sb) * T) * kUSub;
                bulk_g2s(sm + L.U + (size_t)(hh * SUB + sb) * j0 * kUSub * usz, src,
                         (uint32_t)(j0 * kUSub * usz), full);
                continue;
            }
            x -= nU;
            if (x < nK) {
                bulk_g2s(sm + L.K, static_cast<const InT *>(a.p.K) + ((size_t)r * Hk + hk) * T * kD,
                         (uint32_t)(j0 * kD * isz), full);
                continue;
            }
            x -= nK;
            if (x < nG) {
                bulk_g2s(sm + L.Gs + (size_t)x * jb * 4, a.p.G + ((size_t)r * Hv + hk * G + x) * T,
                         (uint32_t)(jb * 4), full);
                continue;
            }
            x -= nG;
            if (x < 2 * nQ) {
                const int t = x % nQ;
                const size_t tok = (size_t)zi * a.tok_total + a.tok_offset + t;
                bulk_g2s(sm + (x < nQ ? L.q : L.k) + (size_t)t * kD * isz,
                         (x < nQ ? qin : kin) + (tok * Hk + hk) * kD, kD * isz, full);
                continue;
            }
            x -= 2 * nQ;
            {
                const int t = x / G, hh = x % G;
                const size_t tok = (size_t)zi * a.tok_total + a.tok_offset + t;
                bulk_g2s(sm + L.v + (size_t)(t * G + hh) * ROWS * isz,
                         vin + (tok * Hv + hk * G + hh) * kD + (size_t)tile * ROWS, ROWS * isz, full);
            }
        }
    }

    // ---- 2. every warp: cumulative log decay of the new tokens in registers
    //         (lane l <-> token t = l / G, head hh = l % G), while the copies fly
    float gn_l = 0.f, be_l = 0.f;
    unsigned bad = 0;
    {
        const bool own = lane < G * n_new;
        const int hh = lane % G, t = lane / G;
        float x = 0.f;
        if (own) {
            const size_t tok = (size_t)zi * a.tok_total + a.tok_offset + t;
            const float al = a.alpha[tok * Hv + hk * G + hh];
            be_l = a.beta[tok * Hv + hk * G + hh];
            x = logf(al);
            if (dm.validate) {
                if (!(al > 0.f && al <= 1.f)) bad |= 0x1u;
                if (!(be_l >= 0.f && be_l <= 1.f)) bad |= 0x2u;
            }
        }
#pragma unroll
        for (int off = 1; off < NT; off <<= 1) {
            const float y = __shfl_up_sync(0xffffffffu, x, off * G);
            if (lane >= off * G) x += y;
        }
        const float g0 = (own && j0 > 0) ? a.p.G[((size_t)r * Hv + hk * G + hh) * T + j0 - 1] : 0.f;
        gn_l = g0 + x;
        if (warp == 0 && own) {
            Gn_s[hh * NT + t] = gn_l;
            Bn_s[hh * NT + t] = be_l;
        }
    }
    // (the block barrier below orders mbarrier init before any other warp waits)
    __syncthreads();
    mbar_wait(full, 0);

    // ---- 3. key scores -> decay-weighted coefficients (Z3)
    //   Ck[h][t][i] = e^{G_t-G_i} (k_t . k_i), i <  j0+t ;  Cq: (q_t . k_i), i <= j0+t
    {
        const int J = j0 + n_new;
        for (int i = warp; i < J; i += NWARP) {
            const float4 ki = load4((i < j0 ? K_s + (size_t)i * kD : k_s + (size_t)(i - j0) * kD) + 4 * lane);
            float vals[2 * NT];
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                vals[2 * t] = dot4(ki, load4(k_s + (size_t)t * kD + 4 * lane));
                vals[2 * t + 1] = dot4(ki, load4(q_s + (size_t)t * kD + 4 * lane));
            }
            const float red = transposed_reduce<2 * NT>(vals, lane);
            // lane l holds value (t = l>>1, isq = l&1); weights per head from the scan lanes
#pragma unroll
            for (int hh = 0; hh < G; ++hh) {
                const int t = (lane >> 1) % NT;
                const float gt = __shfl_sync(0xffffffffu, gn_l, t * G + hh);
                const float gnew = __shfl_sync(0xffffffffu, gn_l, ((i - j0) > 0 ? (i - j0) : 0) * G + hh);
                if (lane < 2 * n_new) {
                    const bool isq = lane & 1;
                    const bool valid = isq ? (i <= j0 + t) : (i < j0 + t);
                    float c = 0.f;
                    if (valid) c = expf(gt - (i < j0 ? G_s[hh * jb + i] : gnew)) * red;
                    (isq ? Cq : Ck)[(hh * NT + t) * Jst + i] = c;
                }
            }
        }
    }
    // ---- 4. state mat-vecs a_t = S0 k_t, b_t = S0 q_t (transposed warp reduction)
    if (HAS_STATE) {
#pragma unroll
        for (int rg0 = 0; rg0 < RPW; rg0 += RG) {
            float4 s4[RG];
#pragma unroll
            for (int rr = 0; rr < RG; ++rr)
                s4[rr] = reinterpret_cast<const float4 *>(S_s + (size_t)(warp * RPW + rg0 + rr) * kD)[lane];
            float vals[NV];
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const float4 k4 = load4(k_s + (size_t)t * kD + 4 * lane);
                const float4 q4 = load4(q_s + (size_t)t * kD + 4 * lane);
#pragma unroll
                for (int rr = 0; rr < RG; ++rr) {
                    vals[(rr * NT + t) * 2 + 0] = dot4(s4[rr], k4);
                    vals[(rr * NT + t) * 2 + 1] = dot4(s4[rr], q4);
                }
            }
            const float red = transposed_reduce<NV>(vals, lane);
            if (lane < NV) {
                const int ab = lane & 1, t = (lane >> 1) % NT, rr = (lane >> 1) / NT;
                const int rf = warp * RPW + rg0 + rr;
                if (t < n_new) (ab ? bv : av)[((rf / ROWS) * NT + t) * ROWS + rf % ROWS] = red;
            }
        }
    }
    if (dm.validate && tid < n_new * kD) {
        const float kk = to_f(k_s[tid]), qq = to_f(q_s[tid]);
        if (!(isfinite(kk) && isfinite(qq))) bad |= 0x4u;
    }
    __syncthreads();

    // ---- 5. slot counter: every CTA of the slot has read it (it did so before
    //         the barrier above); the last one advances it.  Off the critical
    //         path (last warp), no fence: the next launch consumes it.
    if (a.kind != CK_VERIFY && tid == NTHR - 1) {
        if (atomicAdd(&a.p.ticket[r], 1) == (int)(gridDim.x * gridDim.y) - 1) {
            a.p.ticket[r] = 0;
            if (direct) a.p.len[r] = j0 + n_new;
            else a.p.occ[r] = j0 + n_new;
        }
    }

    // ---- 6. forward substitution over the new tokens, one thread per (head, row)
    if (tid < GR) {
        const int hh = tid / ROWS, row = tid % ROWS, h = hk * G + hh;
        const int drow = tile * ROWS + row;
        const int sb = row / kUSub, rr = row % kUSub;
        const UT *ut = U_s + (size_t)(hh * SUB + sb) * j0 * kUSub + rr;
        UT *Uout = static_cast<UT *>(a.p.U) +
                   ((((size_t)r * Hv + h) * (kD / kUSub) + tile * SUB + sb) * T + j0) * kUSub + rr;
        float un[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            if (t < n_new) {
                const float *ck = Ck + (hh * NT + t) * Jst;
                const float *cq = Cq + (hh * NT + t) * Jst;
                float acc_k = 0.f, acc_q = 0.f;
#pragma unroll 4
                for (int i = 0; i < j0; ++i) {
                    const float ui = to_f(ut[(size_t)i * kUSub]);
                    acc_k = fmaf(ck[i], ui, acc_k);
                    acc_q = fmaf(cq[i], ui, acc_q);
                }
#pragma unroll
                for (int tp = 0; tp < t; ++tp) {
                    acc_k = fmaf(ck[j0 + tp], un[tp], acc_k);
                    acc_q = fmaf(cq[j0 + tp], un[tp], acc_q);
                }
                const size_t tok = (size_t)zi * a.tok_total + a.tok_offset + t;
                const float vt = to_f(v_s[(t * G + hh) * ROWS + row]);
                const float bt = Bn_s[hh * NT + t];
                const float eG = expf(Gn_s[hh * NT + t]);
                float u, o;
                if (HAS_STATE) {
                    u = bt * (vt - fmaf(eG, av[(hh * NT + t) * ROWS + row], acc_k));
                    o = fmaf(eG, bv[(hh * NT + t) * ROWS + row], acc_q);
                } else {
                    u = bt * (vt - acc_k);
                    o = acc_q;
                }
                const UT us = from_f<UT>(u);
                un[t] = to_f(us);                      // the stored (rounded) value
                o = fmaf(cq[j0 + t], un[t], o);
                if (dm.validate && !isfinite(vt)) bad |= 0x4u;
                if (a.o) a.o[(tok * Hv + h) * kD + drow] = o;
                Uout[(size_t)t * kUSub] = us;
                if (dm.keep_raw) {
                    static_cast<InT *>(a.p.V)[(((size_t)r * Hv + h) * T + j0 + t) * kD + drow] =
                        v_s[(t * G + hh) * ROWS + row];
                    if (tile == 0 && row == 0) a.p.B[((size_t)r * Hv + h) * T + j0 + t] = bt;
                }
            }
        }
    }
    // ---- 7. append k_t and G_t records (tile 0 of each QK head)
    if (tile == 0) {
        InT *Kdst = static_cast<InT *>(a.p.K) + (((size_t)r * Hk + hk) * T + j0) * kD;
        for (int idx = tid; idx < n_new * kD; idx += NTHR) Kdst[idx] = k_s[idx];
        if (tid < G * n_new) {
            const int hh = tid / n_new, t = tid % n_new;
            a.p.G[((size_t)r * Hv + hk * G + hh) * T + j0 + t] = Gn_s[hh * NT + t];
        }
    }
    if (bad) atomicOr(a.p.status, bad);
}

// ---------------------------------------------------------------- launch
template <typename InT, typename UT, int G, int ROWS, int NT, bool HAS_STATE>
static cudaError_t launch_cfg(const ChunkArgs &a, cudaStream_t s) {
    const CtaLayout L = cta_layout(G, ROWS, NT, HAS_STATE, a.j0_cap, sizeof(InT), sizeof(UT));
    if (L.bytes > 227 * 1024) return cudaErrorInvalidConfiguration;
    constexpr int MINB = NT <= 2 ? 3 : (NT <= 8 ? 2 : 1);
    auto kfn = chunk_cta_kernel<InT, UT, G, ROWS, NT, HAS_STATE, MINB>;
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.bytes);
    if (e != cudaSuccess) return e;
    kfn<<<dim3(kD / ROWS, a.dm.Hk, a.n), 256, L.bytes, s>>>(a);
    return cudaGetLastError();
}

template <typename InT, typename UT, int G, bool HAS_STATE>
static cudaError_t launch_nt(const ChunkArgs &a, cudaStream_t s) {
    constexpr int ROWS = HAS_STATE ? 32 : (256 / G > kD ? kD : 256 / G);
    constexpr int NTMAX = 32 / G < 16 ? 32 / G : 16;
    constexpr int NT8 = NTMAX < 8 ? NTMAX : 8;
    if (a.n_new == 1) return launch_cfg<InT, UT, G, ROWS, 1, HAS_STATE>(a, s);
    if (a.n_new <= 2) return launch_cfg<InT, UT, G, ROWS, 2, HAS_STATE>(a, s);
    if (a.n_new <= 4) return launch_cfg<InT, UT, G, ROWS, 4, HAS_STATE>(a, s);
    if (a.n_new <= 8) return launch_cfg<InT, UT, G, ROWS, NT8, HAS_STATE>(a, s);
    return launch_cfg<InT, UT, G, ROWS, NTMAX, HAS_STATE>(a, s);
}

template <typename InT, typename UT>
static cudaError_t launch_t(const ChunkArgs &a, cudaStream_t s) {
    const bool st = a.kind != CK_DIRECT;
    switch (a.dm.g) {
        case 1: return st ? launch_nt<InT, UT, 1, true>(a, s) : launch_nt<InT, UT, 1, false>(a, s);
        case 2: return st ? launch_nt<InT, UT, 2, true>(a, s) : launch_nt<InT, UT, 2, false>(a, s);
        case 4: return st ? launch_nt<InT, UT, 4, true>(a, s) : launch_nt<InT, UT, 4, false>(a, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_chunk(const ChunkArgs &a, cudaStream_t s, int64_t *launches) {
    if (a.n <= 0 || a.n_new <= 0) return cudaSuccess;
    if (a.n_new > max_new_per_launch(a.dm.g)) return cudaErrorInvalidValue;
    cudaError_t e;
    if (a.dm.in_dt == DT_F32)
        e = launch_t<float, float>(a, s);
    else if (a.dm.u_dt == DT_F16)
        e = launch_t<__nv_bfloat16, __half>(a, s);
    else
        e = launch_t<__nv_bfloat16, float>(a, s);
    if (e == cudaSuccess) ++*launches;
    return e;
}

}  // namespace labuf
