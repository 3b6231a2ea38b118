// recurrent.cu — kernels (5a) and (5b): the conventional recurrent GDN path
// that existing serving systems run ("fused into a single
// kernel"), kept as the in-run IO baseline.  They use the same streaming
// machinery as kernel (1) (bulk-copy state tiles, transposed warp
// reductions) so "buffered beats recurrent" is not a straw man.
//
// Row j of the state evolves independently (north-star form):
//   m_j = alpha (S0[j] . k);  u_j = beta (v_j - m_j);
//   S[j] <- alpha S0[j] + u_j k;  o_j = S[j] . q = alpha (S0[j] . q) + u_j (k . q)
#include <cstring>

#include "device.cuh"
#include "internal.h"

namespace labuf {

__device__ __forceinline__ size_t sidx_of(const Ptrs &p, int r) {
    return p.sidx ? (size_t)__ldcg(p.sidx + r) : (size_t)r;
}

// ------------------------------------------------------------------ (5a)
// CTA = (d_v tile of kRows rows, QK head, slot) over the g V heads of the
// QK head.  Reads the state tile once, writes it once.
template <typename InT, int G>
__global__ void __launch_bounds__(256) recurrent_step_kernel(const RecArgs a) {
    constexpr int ROWS = kRows, GR = G * ROWS, RPW = GR / 8;
    constexpr int RG = RPW < 8 ? RPW : 8;
    constexpr int NV = 2 * RG;
    const int tile = blockIdx.x, hk = blockIdx.y, zi = blockIdx.z;
    const int r = a.first + zi;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int Hv = a.dm.Hv, Hk = a.dm.Hk;

    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
    float *S_s = reinterpret_cast<float *>(smem + 128);
    float *av = S_s + GR * kD;       // S0 k
    float *bv = av + GR;             // S0 q
    float *us = bv + GR;             // u
    float *kq = us + GR;             // k . q

    if (a.p.sidx && a.pdl) pdl_wait();   // state indices may come from the previous grid
    float *tiles[G];
#pragma unroll
    for (int hh = 0; hh < G; ++hh)
        tiles[hh] = a.p.state + ((sidx_of(a.p, r) * Hv + hk * G + hh) * kD + (size_t)tile * ROWS) * kD;
    if (tid == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
        mbar_arrive_expect_tx(bar, GR * kD * 4);
        if (a.pdl_early)
#pragma unroll
            for (int hh = 0; hh < G; ++hh) bulk_g2s(S_s + hh * ROWS * kD, tiles[hh], ROWS * kD * 4, bar);
    }
    if (a.pdl) pdl_wait();
    pdl_trigger();
    if (tid == 0 && !a.pdl_early) {
#pragma unroll
        for (int hh = 0; hh < G; ++hh) bulk_g2s(S_s + hh * ROWS * kD, tiles[hh], ROWS * kD * 4, bar);
    }
    const InT *kin = static_cast<const InT *>(a.k) + ((size_t)zi * Hk + hk) * kD;
    const InT *qin = static_cast<const InT *>(a.q) + ((size_t)zi * Hk + hk) * kD;
    const float4 k4 = load4(kin + 4 * lane);
    const float4 q4 = load4(qin + 4 * lane);
    if (warp == 0) {
        const float x = warp_sum(dot4(k4, q4));
        if (lane == 0) *kq = x;
    }
    __syncthreads();
    mbar_wait(bar, 0);
    for (int rg0 = 0; rg0 < RPW; rg0 += RG) {
        float vals[NV];
#pragma unroll
        for (int rr = 0; rr < RG; ++rr) {
            const float4 s4 = reinterpret_cast<const float4 *>(S_s + (size_t)(warp * RPW + rg0 + rr) * kD)[lane];
            vals[2 * rr] = dot4(s4, k4);
            vals[2 * rr + 1] = dot4(s4, q4);
        }
        const float red = transposed_reduce<NV>(vals, lane);
        if (lane < NV) (lane & 1 ? bv : av)[warp * RPW + rg0 + (lane >> 1)] = red;
    }
    __syncthreads();
    if (tid < GR) {
        const int hh = tid / ROWS, row = tid % ROWS, h = hk * G + hh;
        const int drow = tile * ROWS + row;
        const float al = a.dm.variant == 2 ? 1.f : a.alpha[(size_t)zi * Hv + h], be = a.beta[(size_t)zi * Hv + h];
        const float vt = to_f(static_cast<const InT *>(a.v)[((size_t)zi * Hv + h) * kD + drow]);
        const float u = a.dm.variant ? vt : be * (vt - al * av[tid]);   // (no delta rule: u = v)
        us[tid] = u;
        a.o[((size_t)zi * Hv + h) * kD + drow] = fmaf(al, bv[tid], u * (*kq));
    }
    __syncthreads();
    // S_new row = alpha S0 row + u k, in place, then one bulk store per head
    for (int rr = 0; rr < RPW; ++rr) {
        const int rf = warp * RPW + rr;
        const int h = hk * G + rf / ROWS;
        const float al = a.dm.variant == 2 ? 1.f : a.alpha[(size_t)zi * Hv + h];
        float4 *p = reinterpret_cast<float4 *>(S_s + (size_t)rf * kD) + lane;
        float4 s = *p;
        const float u = us[rf];
        s.x = fmaf(u, k4.x, al * s.x);
        s.y = fmaf(u, k4.y, al * s.y);
        s.z = fmaf(u, k4.z, al * s.z);
        s.w = fmaf(u, k4.w, al * s.w);
        *p = s;
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
#pragma unroll
        for (int hh = 0; hh < G; ++hh) bulk_s2g(tiles[hh], S_s + hh * ROWS * kD, ROWS * kD * 4);
        bulk_commit();
        bulk_wait0();
    }
}

// ------------------------------------------------------------------ (5b)
// N sequential recurrent steps from one state read; writes N temporary
// states [n][N][Hv][d][d] and N outputs.  CTA = (d_v tile of
// kRows rows, V head, slot), 4 warps x 8 rows; the rows stay in registers
// across the drafts.  Every operand is staged at entry (state tile by one
// bulk copy; k_t, q_t, v_t of all drafts by bulk copies; alpha, beta) so the
// draft loop has no global loads, and each temporary state leaves through a
// double-buffered shared-memory tile and ONE bulk store (the TMA engine, not
// per-lane stores, drains the N x 16 KiB of writes per CTA) -- the same
// machinery as kernel (5a), so the baseline streams at the copy roofline.
template <typename InT>
__global__ void __launch_bounds__(128) recurrent_verify_kernel(const RecArgs a) {
    constexpr int ROWS = kRows, RPW = ROWS / 4, isz = (int)sizeof(InT);
    static_assert(RPW == 8, "4 warps x 8 rows");
    const int tile = blockIdx.x, h = blockIdx.y, zi = blockIdx.z;
    const int r = a.first + zi;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int Hv = a.dm.Hv, Hk = a.dm.Hk, N = a.n_draft, hk = h / a.dm.g;

    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
    float *buf = reinterpret_cast<float *>(smem + 128);             // [2][ROWS][kD]
    InT *kq_s = reinterpret_cast<InT *>(buf + 2 * ROWS * kD);        // [N][k | q][kD]
    InT *v_s = kq_s + (size_t)N * 2 * kD;                            // [N][ROWS]
    float *al_s = reinterpret_cast<float *>(v_s + (size_t)N * ROWS); // [N]
    float *be_s = al_s + 16;
    float *kqd = be_s + 16;                                          // k_t . q_t

    if (a.p.sidx && a.pdl) pdl_wait();   // state indices may come from the previous grid
    const float *src = a.p.state + ((sidx_of(a.p, r) * Hv + h) * kD + (size_t)tile * ROWS) * kD;
    const uint32_t bytes = ROWS * kD * 4 + (uint32_t)N * (2 * kD + ROWS) * isz;
    if (tid == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
        if (a.pdl_early) {
            mbar_arrive_expect_tx(bar, bytes);
            bulk_g2s(buf, src, ROWS * kD * 4, bar);
        }
    }
    if (a.pdl) pdl_wait();
    pdl_trigger();
    __syncthreads();   // barrier initialised
    const InT *qin = static_cast<const InT *>(a.q);
    const InT *kin = static_cast<const InT *>(a.k);
    const InT *vin = static_cast<const InT *>(a.v);
    if (tid == 0) {
        if (!a.pdl_early) {
            mbar_arrive_expect_tx(bar, bytes);
            bulk_g2s(buf, src, ROWS * kD * 4, bar);
        }
    } else if (warp == 1) {
        for (int c = lane; c < 3 * N; c += 32) {
            const int t = c % N, kind = c / N;
            const size_t tok = (size_t)zi * N + t;
            if (kind < 2)
                bulk_g2s(kq_s + ((size_t)t * 2 + kind) * kD, (kind ? qin : kin) + (tok * Hk + hk) * kD, kD * isz, bar);
            else
                bulk_g2s(v_s + (size_t)t * ROWS, vin + (tok * Hv + h) * kD + tile * ROWS, ROWS * isz, bar);
        }
    } else if (warp == 2 && lane < N) {
        const size_t tok = (size_t)zi * N + lane;
        al_s[lane] = a.alpha[tok * Hv + h];
        be_s[lane] = a.beta[tok * Hv + h];
    }
    mbar_wait(bar, 0);
    for (int t = warp; t < N; t += 4) {
        const float x = warp_sum(dot4(load4(kq_s + (size_t)t * 2 * kD + 4 * lane), load4(kq_s + ((size_t)t * 2 + 1) * kD + 4 * lane)));
        if (lane == 0) kqd[t] = x;
    }
    float4 s[RPW];
#pragma unroll
    for (int rr = 0; rr < RPW; ++rr) s[rr] = reinterpret_cast<const float4 *>(buf + (size_t)(warp * RPW + rr) * kD)[lane];
    __syncthreads();   // kqd visible; every warp holds its rows
    const int rl = (lane & 15) >> 1;              // the row whose (k | q) dot this lane ends with
    const int drow = tile * ROWS + warp * RPW + rl;
    for (int t = 0; t < N; ++t) {
        const float4 k4 = load4(kq_s + (size_t)t * 2 * kD + 4 * lane);
        const float4 q4 = load4(kq_s + ((size_t)t * 2 + 1) * kD + 4 * lane);
        float vals[2 * RPW];
#pragma unroll
        for (int rr = 0; rr < RPW; ++rr) {
            vals[2 * rr] = dot4(s[rr], k4);
            vals[2 * rr + 1] = dot4(s[rr], q4);
        }
        const float red = transposed_reduce<2 * RPW>(vals, lane);   // lane l: (row (l%16)/2, k|q = l&1)
        const float al = a.dm.variant == 2 ? 1.f : al_s[t], be = be_s[t];
        const float vr = to_f(v_s[t * ROWS + warp * RPW + rl]);
        const float uk = a.dm.variant ? vr : be * (vr - al * red);   // valid on even lanes
        const float u = __shfl_sync(0xffffffffu, uk, lane & ~1);
        if (lane < 16 && (lane & 1)) {
            const size_t tok = (size_t)zi * N + t;
            a.o[(tok * Hv + h) * kD + drow] = fmaf(al, red, u * kqd[t]);
        }
        float *dst = buf + (size_t)(t & 1) * ROWS * kD;
#pragma unroll
        for (int rr = 0; rr < RPW; ++rr) {
            const float ur = __shfl_sync(0xffffffffu, u, 2 * rr);
            float4 x = s[rr];
            x.x = fmaf(ur, k4.x, al * x.x);
            x.y = fmaf(ur, k4.y, al * x.y);
            x.z = fmaf(ur, k4.z, al * x.z);
            x.w = fmaf(ur, k4.w, al * x.w);
            s[rr] = x;
            reinterpret_cast<float4 *>(dst + (size_t)(warp * RPW + rr) * kD)[lane] = x;
        }
        fence_proxy_async_smem();
        if (tid == 0) bulk_wait_read0();   // the store of draft t-1 has read the other buffer
        __syncthreads();
        if (tid == 0) {
            bulk_s2g(a.temp + ((((size_t)zi * N + t) * Hv + h) * kD + (size_t)tile * ROWS) * kD, dst, ROWS * kD * 4);
            bulk_commit();
        }
    }
    if (tid == 0) bulk_wait_read0();   // shared memory stays live until the last store has read it
}

// Commit of the baseline: state <- temp[n_acc - 1] (Fig. 3).
__global__ void __launch_bounds__(256) recurrent_commit_kernel(const RecArgs a) {
    if (a.pdl) pdl_wait();
    pdl_trigger();
    const int h = blockIdx.y, zi = blockIdx.z, r = a.first + zi;
    int na = a.nacc[zi];
    if (na < 0 || na > a.n_draft) {
        if (a.dm.validate && threadIdx.x == 0 && blockIdx.x == 0) atomicOr(a.p.status, 0x8u);
        na = na < 0 ? 0 : a.n_draft;
    }
    if (na == 0) return;
    const float4 *src = reinterpret_cast<const float4 *>(
        a.temp + (((size_t)zi * a.n_draft + na - 1) * a.dm.Hv + h) * kD * kD);
    float4 *dst = reinterpret_cast<float4 *>(a.p.state + (sidx_of(a.p, r) * a.dm.Hv + h) * kD * kD);
    const int per = kD * kD / 4 / gridDim.x;
    const int base = blockIdx.x * per;
    for (int i = threadIdx.x; i < per; i += 256) dst[base + i] = src[base + i];
}

template <int G, typename InT>
static cudaError_t launch_rs(const RecArgs &a, cudaStream_t s) {
    const size_t smem = 128 + (size_t)G * kRows * kD * 4 + 3 * G * kRows * 4 + 16;
    auto kfn = recurrent_step_kernel<InT, G>;
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    return launch_k(kfn, dim3(kD / kRows, a.dm.Hk, a.n), dim3(256), smem, s, a.pdl != 0, a);
}
template <typename InT>
static cudaError_t launch_rv(const RecArgs &a, cudaStream_t s) {
    const size_t smem = 128 + 2 * (size_t)kRows * kD * 4 + (size_t)a.n_draft * (2 * kD + kRows) * sizeof(InT) + 48 * 4;
    auto kfn = recurrent_verify_kernel<InT>;
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    return launch_k(kfn, dim3(kD / kRows, a.dm.Hv, a.n), dim3(128), smem, s, a.pdl != 0, a);
}

template <typename InT>
static cudaError_t dispatch_step(const RecArgs &a, cudaStream_t s, bool verify) {
    if (verify) return launch_rv<InT>(a, s);
    switch (a.dm.g) {
        case 1: return launch_rs<1, InT>(a, s);
        case 2: return launch_rs<2, InT>(a, s);
        case 4: return launch_rs<4, InT>(a, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_recurrent_step(const RecArgs &a, cudaStream_t s, int64_t *launches) {
    if (a.n <= 0) return cudaSuccess;
    cudaError_t e = a.dm.in_dt == DT_F32 ? dispatch_step<float>(a, s, false)
                                         : dispatch_step<__nv_bfloat16>(a, s, false);
    if (e == cudaSuccess) ++*launches;
    return e;
}
cudaError_t launch_recurrent_verify(const RecArgs &a, cudaStream_t s, int64_t *launches) {
    if (a.n <= 0) return cudaSuccess;
    cudaError_t e = a.dm.in_dt == DT_F32 ? dispatch_step<float>(a, s, true)
                                         : dispatch_step<__nv_bfloat16>(a, s, true);
    if (e == cudaSuccess) ++*launches;
    return e;
}
cudaError_t launch_recurrent_commit(const RecArgs &a, cudaStream_t s, int64_t *launches) {
    if (a.n <= 0) return cudaSuccess;
    cudaError_t e = launch_k(recurrent_commit_kernel, dim3(8, a.dm.Hv, a.n), dim3(256), 0, s, a.pdl != 0, a);
    if (e == cudaSuccess) ++*launches;
    return e;
}

// ------------------------------------------------------------------ append commit
// Multi-round speculation: the accepted drafts stay buffered, occ += n_acc.
__global__ void commit_append_kernel(Ptrs p, Dims dm, int first, int n, const int *nacc, int n_draft) {
    pdl_wait();
    pdl_trigger();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int na = nacc[i];
    if (na < 0 || na > n_draft) {
        if (dm.validate) atomicOr(p.status, 0x8u);
        na = na < 0 ? 0 : n_draft;
    }
    p.occ[first + i] += na;
}

cudaError_t launch_commit_append(const Dims &dm, const Ptrs &p, int first, int n, const int *nacc, int n_draft,
                                 int pdl, cudaStream_t s, int64_t *launches) {
    if (n <= 0) return cudaSuccess;
    cudaError_t e = launch_k(commit_append_kernel, dim3((n + 255) / 256), dim3(256), 0, s, pdl != 0, p, dm, first, n,
                             nacc, n_draft);
    if (e == cudaSuccess) ++*launches;
    return e;
}

// ------------------------------------------------------------------ stage
template <int CAP>
__global__ void stage_kernel(const __grid_constant__ StageArgsT<CAP> a) {
    if (a.n > 0) pdl_wait();   // the previous grid may still read the entries being replaced
    pdl_trigger();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += gridDim.x * blockDim.x)
        a.dst[a.e[i].x] = a.e[i].y;
}

template <int CAP>
static cudaError_t stage_cap(int *dst, const int2 *e, int n, cudaStream_t s) {
    StageArgsT<CAP> a;
    a.dst = dst;
    a.n = n;
    memcpy(a.e, e, n * sizeof(int2));
    return launch_k(stage_kernel<CAP>, dim3((n + 255) / 256), dim3(256), 0, s, true, a);
}

cudaError_t launch_stage(int *dst, const int2 *e, int n, int /*pdl*/, cudaStream_t s, int64_t *launches) {
    if (n <= 0) return cudaSuccess;
    if (n > kStageMax) return cudaErrorInvalidValue;
    cudaError_t err = n <= kStageSmall ? stage_cap<kStageSmall>(dst, e, n, s) : stage_cap<kStageMax>(dst, e, n, s);
    if (err == cudaSuccess) ++*launches;
    return err;
}

// ------------------------------------------------------------------ reset
__global__ void reset_kernel(Ptrs p, Dims dm, int first, int n, int mode, int zero_state) {
    const int zi = blockIdx.y, r = first + zi;
    if (zero_state) {
        float4 *st = reinterpret_cast<float4 *>(p.state + sidx_of(p, r) * dm.Hv * kD * kD);
        const size_t total = (size_t)dm.Hv * kD * kD / 4;
        for (size_t i = blockIdx.x * 256 + threadIdx.x; i < total; i += (size_t)gridDim.x * 256)
            st[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        p.occ[r] = 0;
        p.len[r] = 0;
        p.mode[r] = mode;
        p.ticket[r] = 0;
    }
}

cudaError_t launch_reset(const Dims &dm, const Ptrs &p, int first, int n, int mode, int zero_state,
                         cudaStream_t s, int64_t *launches) {
    if (n <= 0) return cudaSuccess;
    reset_kernel<<<dim3(zero_state ? 32 : 1, n), 256, 0, s>>>(p, dm, first, n, mode, zero_state);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) ++*launches;
    return e;
}

}  // namespace labuf
