// chunk.cu — kernels (1) buffered decode, (3) parallel draft verification,
// (4) direct short-context decoding, and the prefill chunk step.
//
// All four compute, for n_new new tokens t of one request slot r and the g
// V heads of one QK head, against j0 buffered records (k_i, u_i, G_i):
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
// CTA = (d_v tile of kRows rows, QK head, slot).  The state tile of the g V
// heads (g * kRows * 512 B, contiguous per head) is staged in shared memory
// by the bulk-copy engine behind an mbarrier while the CTA computes the
// key-key dot products; the buffered u tile arrives by cp.async.
#include "device.cuh"
#include "internal.h"

namespace labuf {

struct ChunkSmem {
    size_t bar, S, kn, qn, Gb, Gn, Ck, Cq, av, bv, Ut, un, total;
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

__host__ __device__ inline ChunkSmem chunk_smem_layout(int G, bool has_state, int n_new, int TG,
                                                       int j0_cap, int u_bytes) {
    ChunkSmem L;
    const int npad = (n_new + TG - 1) / TG * TG;
    const int J = j0_cap + n_new;
    size_t o = 0;
    L.bar = o; o += 128;
    L.S = o; o += has_state ? (size_t)G * kRows * kD * 4 : 0;
    L.kn = o; o += (size_t)npad * kD * 4;
    L.qn = o; o += (size_t)npad * kD * 4;
    L.Gb = o; o = align16(o + (size_t)G * j0_cap * 4);
    L.Gn = o; o = align16(o + (size_t)G * n_new * 4);
    L.Ck = o; o = align16(o + (size_t)G * n_new * J * 4);
    L.Cq = o; o = align16(o + (size_t)G * n_new * J * 4);
    L.av = o; o = align16(o + (size_t)G * n_new * kRows * 4);
    L.bv = o; o = align16(o + (size_t)G * n_new * kRows * 4);
    L.Ut = o; o = align16(o + (size_t)G * j0_cap * kRows * u_bytes);
    L.un = o; o = align16(o + (size_t)G * n_new * kRows * 4);
    L.total = o;
    return L;
}

template <typename InT, typename UT, int G, int TG>
__global__ void __launch_bounds__(256) chunk_attend_kernel(const ChunkArgs a) {
    constexpr int ROWS = kRows;
    constexpr int GR = G * ROWS;            // rows of this CTA, flattened over heads
    constexpr int RPW = GR / 8;             // rows per warp (8 warps)
    constexpr int RG = (RPW < (TG == 1 ? 8 : 4)) ? RPW : (TG == 1 ? 8 : 4);
    constexpr int NV = 2 * RG * TG;         // partial values per reduction
    static_assert(RPW % RG == 0, "row grouping");

    const int tile = blockIdx.x, hk = blockIdx.y, zi = blockIdx.z;
    const int r = a.first + zi;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const Dims dm = a.dm;
    const int T = dm.T, Hv = dm.Hv, Hk = dm.Hk;
    const bool has_state = (a.kind != CK_DIRECT);
    const int n_new = a.n_new;
    const int npad = (n_new + TG - 1) / TG * TG;
    const int j0 = (a.kind == CK_DIRECT) ? a.p.len[r] : a.p.occ[r];
    const int J = j0 + n_new;
    const int Jcap = a.j0_cap + n_new;

    extern __shared__ __align__(128) unsigned char smem[];
    const ChunkSmem L = chunk_smem_layout(G, has_state, n_new, TG, a.j0_cap, (int)sizeof(UT));
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + L.bar);
    float *S_s = reinterpret_cast<float *>(smem + L.S);
    float *kn = reinterpret_cast<float *>(smem + L.kn);
    float *qn = reinterpret_cast<float *>(smem + L.qn);
    float *Gb = reinterpret_cast<float *>(smem + L.Gb);
    float *Gn = reinterpret_cast<float *>(smem + L.Gn);
    float *Ck = reinterpret_cast<float *>(smem + L.Ck);
    float *Cq = reinterpret_cast<float *>(smem + L.Cq);
    float *av = reinterpret_cast<float *>(smem + L.av);
    float *bv = reinterpret_cast<float *>(smem + L.bv);
    UT *Ut = reinterpret_cast<UT *>(smem + L.Ut);
    float *un = reinterpret_cast<float *>(smem + L.un);

    const InT *qin = static_cast<const InT *>(a.q);
    const InT *kin = static_cast<const InT *>(a.k);
    const InT *vin = static_cast<const InT *>(a.v);
    const InT *Kbuf = static_cast<const InT *>(a.p.K);
    UT *Ubuf = static_cast<UT *>(a.p.U);
    unsigned bad = 0;

    // ---- 1. state tile -> smem (bulk copy engine), buffered u tile -> smem (cp.async)
    if (has_state && tid == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
        mbar_arrive_expect_tx(bar, (uint32_t)(GR * kD * 4));
#pragma unroll
        for (int hh = 0; hh < G; ++hh) {
            const int h = hk * G + hh;
            const float *src = a.p.state + (((size_t)r * Hv + h) * kD + (size_t)tile * ROWS) * kD;
            bulk_g2s(S_s + (size_t)hh * ROWS * kD, src, ROWS * kD * 4, bar);
        }
    }
    {
        constexpr int CPR = ROWS * (int)sizeof(UT) / 16;   // 16-byte chunks per row segment
        const int total = G * j0 * CPR;
        for (int idx = tid; idx < total; idx += 256) {
            const int c = idx % CPR;
            const int i = (idx / CPR) % j0;
            const int hh = idx / (CPR * j0);
            const int h = hk * G + hh;
            const UT *src = Ubuf + (((size_t)r * Hv + h) * T + i) * kD + (size_t)tile * ROWS;
            UT *dst = Ut + ((size_t)hh * a.j0_cap + i) * ROWS;
            cp_async16(reinterpret_cast<char *>(dst) + c * 16,
                       reinterpret_cast<const char *>(src) + c * 16);
        }
        cp_async_commit();
    }

    // ---- 2. new tokens' q, k (fp32 in smem, zero-padded to npad), buffered G
    for (int idx = tid; idx < npad * (kD / 4); idx += 256) {
        const int t = idx / (kD / 4), c4 = idx % (kD / 4);
        float4 kk = make_float4(0.f, 0.f, 0.f, 0.f), qq = kk;
        if (t < n_new) {
            const size_t tok = (size_t)zi * a.tok_total + a.tok_offset + t;
            kk = load4(kin + (tok * Hk + hk) * kD + 4 * c4);
            qq = load4(qin + (tok * Hk + hk) * kD + 4 * c4);
            if (dm.validate && !(finite4(kk) && finite4(qq))) bad |= 0x4u;
        }
        reinterpret_cast<float4 *>(kn)[idx] = kk;
        reinterpret_cast<float4 *>(qn)[idx] = qq;
    }
    for (int idx = tid; idx < G * j0; idx += 256) {
        const int hh = idx / j0, i = idx % j0;
        Gb[hh * a.j0_cap + i] = a.p.G[((size_t)r * Hv + hk * G + hh) * T + i];
    }
    __syncthreads();

    // ---- 3. cumulative log decay of the new tokens (one thread per V head)
    if (tid < G) {
        const int h = hk * G + tid;
        float gacc = (j0 > 0) ? Gb[tid * a.j0_cap + j0 - 1] : 0.f;
        for (int t = 0; t < n_new; ++t) {
            const size_t tok = (size_t)zi * a.tok_total + a.tok_offset + t;
            const float al = a.alpha[tok * Hv + h];
            if (dm.validate) {
                const float be = a.beta[tok * Hv + h];
                if (!(al > 0.f && al <= 1.f)) bad |= 0x1u;
                if (!(be >= 0.f && be <= 1.f)) bad |= 0x2u;
            }
            gacc += logf(al);
            Gn[tid * n_new + t] = gacc;
        }
    }
    __syncthreads();

    // ---- 4. key-key / query-key dot products -> decay-weighted coefficients
    //   Ck[h][t][i] = e^{G_t - G_i} (k_t . k_i)  for i <  j0 + t
    //   Cq[h][t][i] = e^{G_t - G_i} (q_t . k_i)  for i <= j0 + t
    for (int i = warp; i < J; i += 8) {
        float4 ki;
        if (i < j0)
            ki = load4(Kbuf + (((size_t)r * Hk + hk) * T + i) * kD + 4 * lane);
        else
            ki = reinterpret_cast<const float4 *>(kn + (size_t)(i - j0) * kD)[lane];
        for (int t = 0; t < n_new; ++t) {
            if (i > j0 + t) continue;   // warp-uniform
            float vals[2];
            vals[0] = dot4(ki, reinterpret_cast<const float4 *>(kn + (size_t)t * kD)[lane]);
            vals[1] = dot4(ki, reinterpret_cast<const float4 *>(qn + (size_t)t * kD)[lane]);
            const float red = transposed_reduce<2>(vals, lane);   // lane&1: 0 -> kk, 1 -> qk
            if (lane < 2 * G) {
                const int hh = lane >> 1;
                const float gt = Gn[hh * n_new + t];
                const float gi = (i < j0) ? Gb[hh * a.j0_cap + i] : Gn[hh * n_new + (i - j0)];
                const float w = expf(gt - gi);
                float *dst = ((lane & 1) ? Cq : Ck) + ((size_t)hh * n_new + t) * Jcap + i;
                *dst = ((lane & 1) || i < j0 + t) ? w * red : 0.f;
            }
        }
    }

    // ---- 5. state mat-vecs a_t = S0 k_t, b_t = S0 q_t (transposed warp reduction)
    if (has_state) {
        mbar_wait(bar, 0);
        for (int rg0 = 0; rg0 < RPW; rg0 += RG) {
            float4 s4[RG];
#pragma unroll
            for (int rr = 0; rr < RG; ++rr)
                s4[rr] = reinterpret_cast<const float4 *>(S_s + (size_t)(warp * RPW + rg0 + rr) * kD)[lane];
            for (int tg0 = 0; tg0 < npad; tg0 += TG) {
                float vals[NV];
#pragma unroll
                for (int tt = 0; tt < TG; ++tt) {
                    const float4 k4 = reinterpret_cast<const float4 *>(kn + (size_t)(tg0 + tt) * kD)[lane];
                    const float4 q4 = reinterpret_cast<const float4 *>(qn + (size_t)(tg0 + tt) * kD)[lane];
#pragma unroll
                    for (int rr = 0; rr < RG; ++rr) {
                        vals[(rr * TG + tt) * 2 + 0] = dot4(s4[rr], k4);
                        vals[(rr * TG + tt) * 2 + 1] = dot4(s4[rr], q4);
                    }
                }
                const float red = transposed_reduce<NV>(vals, lane);
                if (lane < NV) {
                    const int ab = lane & 1, tt = (lane >> 1) % TG, rr = (lane >> 1) / TG;
                    const int t = tg0 + tt;
                    const int rf = warp * RPW + rg0 + rr;
                    const int hh = rf / ROWS, row = rf % ROWS;
                    if (t < n_new) (ab ? bv : av)[((size_t)hh * n_new + t) * ROWS + row] = red;
                }
            }
        }
    }
    cp_async_wait_all();
    __syncthreads();

    // ---- 6. forward substitution over the new tokens, one thread per (head, row)
    if (tid < GR) {
        const int hh = tid / ROWS, row = tid % ROWS;
        const int h = hk * G + hh;
        const int drow = tile * ROWS + row;
        for (int t = 0; t < n_new; ++t) {
            const size_t tok = (size_t)zi * a.tok_total + a.tok_offset + t;
            const float vt = to_f(vin[(tok * Hv + h) * kD + drow]);
            if (dm.validate && !isfinite(vt)) bad |= 0x4u;
            const float bt = a.beta[tok * Hv + h];
            const float eG = expf(Gn[hh * n_new + t]);
            const float *ck = Ck + ((size_t)hh * n_new + t) * Jcap;
            const float *cq = Cq + ((size_t)hh * n_new + t) * Jcap;
            float acc_k = 0.f, acc_q = 0.f;
            const UT *ut = Ut + (size_t)hh * a.j0_cap * ROWS + row;
#pragma unroll 4
            for (int i = 0; i < j0; ++i) {
                const float ui = to_f(ut[(size_t)i * ROWS]);
                acc_k = fmaf(ck[i], ui, acc_k);
                acc_q = fmaf(cq[i], ui, acc_q);
            }
            for (int tp = 0; tp < t; ++tp) {
                const float ui = un[((size_t)hh * n_new + tp) * ROWS + row];
                acc_k = fmaf(ck[j0 + tp], ui, acc_k);
                acc_q = fmaf(cq[j0 + tp], ui, acc_q);
            }
            float ut_new;
            float o;
            if (has_state) {
                const float at = av[((size_t)hh * n_new + t) * ROWS + row];
                const float btv = bv[((size_t)hh * n_new + t) * ROWS + row];
                ut_new = bt * (vt - fmaf(eG, at, acc_k));
                o = fmaf(eG, btv, acc_q);
            } else {
                ut_new = bt * (vt - acc_k);
                o = acc_q;
            }
            const UT us = from_f<UT>(ut_new);
            const float ur = to_f(us);                   // the stored (rounded) value
            un[((size_t)hh * n_new + t) * ROWS + row] = ur;
            o = fmaf(cq[j0 + t], ur, o);
            if (a.o) a.o[(tok * Hv + h) * kD + drow] = o;
            Ubuf[(((size_t)r * Hv + h) * T + j0 + t) * kD + drow] = us;
            if (dm.keep_raw) {
                static_cast<InT *>(a.p.V)[(((size_t)r * Hv + h) * T + j0 + t) * kD + drow] =
                    vin[(tok * Hv + h) * kD + drow];
                if (tile == 0 && row == 0) a.p.B[((size_t)r * Hv + h) * T + j0 + t] = bt;
            }
        }
    }

    // ---- 7. append k_t and G_t records (tile 0 of each QK head)
    if (tile == 0) {
        InT *Kdst = static_cast<InT *>(a.p.K);
        for (int idx = tid; idx < n_new * kD; idx += 256) {
            const int t = idx / kD, c = idx % kD;
            const size_t tok = (size_t)zi * a.tok_total + a.tok_offset + t;
            Kdst[(((size_t)r * Hk + hk) * T + j0 + t) * kD + c] = kin[(tok * Hk + hk) * kD + c];
        }
        for (int idx = tid; idx < G * n_new; idx += 256) {
            const int hh = idx / n_new, t = idx % n_new;
            a.p.G[((size_t)r * Hv + hk * G + hh) * T + j0 + t] = Gn[hh * n_new + t];
        }
    }
    if (bad) atomicOr(a.p.status, bad);

    // ---- 8. advance the slot counter once every CTA of the slot has read it
    if (a.kind != CK_VERIFY) {
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            const int nct = gridDim.x * gridDim.y;
            if (atomicAdd(&a.p.ticket[r], 1) == nct - 1) {
                a.p.ticket[r] = 0;
                if (a.kind == CK_DIRECT) a.p.len[r] = j0 + n_new;
                else a.p.occ[r] = j0 + n_new;
            }
        }
    }
}

template <typename InT, typename UT, int G>
static cudaError_t launch_chunk_g(const ChunkArgs &a, cudaStream_t s) {
    const bool has_state = a.kind != CK_DIRECT;
    dim3 grid(kD / kRows, a.dm.Hk, a.n);
    if (a.n_new == 1) {
        const ChunkSmem L = chunk_smem_layout(G, has_state, 1, 1, a.j0_cap, sizeof(UT));
        auto kfn = chunk_attend_kernel<InT, UT, G, 1>;
        cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)L.total);
        if (e != cudaSuccess) return e;
        kfn<<<grid, 256, L.total, s>>>(a);
    } else {
        const ChunkSmem L = chunk_smem_layout(G, has_state, a.n_new, 4, a.j0_cap, sizeof(UT));
        auto kfn = chunk_attend_kernel<InT, UT, G, 4>;
        cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)L.total);
        if (e != cudaSuccess) return e;
        kfn<<<grid, 256, L.total, s>>>(a);
    }
    return cudaGetLastError();
}

template <typename InT, typename UT>
static cudaError_t launch_chunk_t(const ChunkArgs &a, cudaStream_t s) {
    switch (a.dm.g) {
        case 1: return launch_chunk_g<InT, UT, 1>(a, s);
        case 2: return launch_chunk_g<InT, UT, 2>(a, s);
        case 4: return launch_chunk_g<InT, UT, 4>(a, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_chunk(const ChunkArgs &a, cudaStream_t s, int64_t *launches) {
    if (a.n <= 0 || a.n_new <= 0) return cudaSuccess;
    cudaError_t e;
    if (a.dm.in_dt == DT_F32)
        e = launch_chunk_t<float, float>(a, s);
    else if (a.dm.u_dt == DT_F16)
        e = launch_chunk_t<__nv_bfloat16, __half>(a, s);
    else
        e = launch_chunk_t<__nv_bfloat16, float>(a, s);
    if (e == cudaSuccess) ++*launches;
    return e;
}

}  // namespace labuf
