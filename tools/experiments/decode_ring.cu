// EXPERIMENT (not built): persistent decode with a state-buffer ring, measured
// 35.6 us per decode launch vs 25.6 for chunk_cta_kernel at config 2 (profiles/r2c/ab_runs/abring_persistent_decode.txt);
// kept for the record.  It was compiled from paper_2605_19049_b200/csrc with chunk.cuh.
// decode_ring.cu — kernel (1), the buffered decode step (NT = 1), as a
// persistent CTA per SM with a ring of state buffers.
//
// Same arithmetic as the decode kind of chunk_cta_kernel (chunk.cuh, the
// single-token chunkwise form P:403-406 with readings Z2/Z3): per unit
// (slot r, V head h, 64 d_v rows)
//   a = S0 k_t, b = S0 q_t                               (the state rows, once)
//   G_t = G_{j0-1} + ln alpha_t
//   u_t = beta_t (v_t - e^{G_t} a - sum_{i<j0} e^{G_t-G_i} (k_t.k_i) u_i)
//   o_t = e^{G_t} b + sum_{i<j0} e^{G_t-G_i} (q_t.k_i) u_i + (q_t.k_t) u_t
// and the record (k_t, u_t, G_t) appended at position j0.
//
// Why a ring (measured, tools/ck_prof.py): the non-persistent kernel holds a
// CTA's 32 KiB state tile for its whole life -- the load (~2 us under full
// bandwidth) AND ~1.9 us of compute of which only the first ~0.7 us (the
// state rows) needs the tile -- so ~45 % of the shared memory that could
// hold bytes in flight idles.  Here a producer warp keeps NS state buffers
// filling, and each consumer warp pair releases its state buffer as soon as
// its rows are reduced, finishing the records, substitution and stores from
// a separate (small) record buffer while the next tile streams into the
// state buffer.
#include "chunk.cuh"

namespace labuf {

constexpr int kRingPairs = 4;                 // consumer warp pairs (2 x 32 rows each)
constexpr int kRingNS = 5;                    // state buffers (32 KiB each)
constexpr int kRingNR = kRingPairs + 2;       // record buffers
constexpr int kRingThreads = 32 * (2 * kRingPairs + 1);

struct RingSmem {
    uint32_t S, R, rec_bytes, U, K, G, q, k, v, ab, P, bar, total;
};
// record buffer r: U (2 tiles x jcap x 32 u), K (jcap rows), G, q_t, k_t, v_t slice, (alpha, beta)
__host__ __device__ inline RingSmem ring_layout(int jcap, int isz, int usz) {
    RingSmem L;
    uint32_t o = 0;
    L.S = o;  o += kRingNS * 64 * kD * 4;
    uint32_t r = 0;
    L.U = r;  r = al128(r + (uint32_t)(2 * jcap * kUSub * usz));
    L.K = r;  r = al128(r + (uint32_t)(jcap * kD * isz));
    L.G = r;  r = al128(r + (uint32_t)(((jcap + 3) & ~3) * 4));
    L.q = r;  r = al128(r + (uint32_t)(kD * isz));
    L.k = r;  r = al128(r + (uint32_t)(kD * isz));
    L.v = r;  r = al128(r + (uint32_t)(64 * isz));
    L.ab = r; r = al128(r + 16);
    L.rec_bytes = r;
    L.R = o;  o += kRingNR * r;
    // per pair: a, b of its 64 rows, the coefficient rows Ck, Cq (j0 + 1)
    L.P = o;  o += kRingPairs * al128((uint32_t)(2 * 64 * 4 + 2 * (jcap + 1 + 3) * 4));
    L.bar = o; o += (2 * kRingNS + 2 * kRingNR) * 8;
    L.total = o;
    return L;
}

template <typename InT, typename UT>
__global__ void __launch_bounds__(kRingThreads, 1) decode_ring_kernel(const ChunkArgs a) {
    constexpr int isz = (int)sizeof(InT), usz = (int)sizeof(UT);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const Dims dm = a.dm;
    const int T = dm.T, Hv = dm.Hv, Hk = dm.Hk;
    const int n_units = a.n * Hv * 2;           // (slot row, V head, 64-row half)
    extern __shared__ __align__(1024) unsigned char smem[];
    const RingSmem L = ring_layout(a.j0_cap, isz, usz);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + L.bar);
    uint64_t *full_S = bars, *empty_S = bars + kRingNS, *full_R = bars + 2 * kRingNS,
             *empty_R = bars + 2 * kRingNS + kRingNR;
    const int stride = gridDim.x;
    auto unit = [&](int u, int &zi, int &h, int &tg) { zi = u / (2 * Hv); h = (u >> 1) % Hv; tg = u & 1; };

    if (tid == 0) {
        for (int i = 0; i < kRingNS; ++i) { mbar_init(full_S + i, 1); mbar_init(empty_S + i, 2); }
        for (int i = 0; i < kRingNR; ++i) { mbar_init(full_R + i, 2); mbar_init(empty_R + i, 2); }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == 2 * kRingPairs) {
        // ==================================================== producer warp
        auto issue_state = [&](int k) {
            int zi, h, tg;
            unit(blockIdx.x + k * stride, zi, h, tg);
            const int r = a.first + zi;
            mbar_arrive_expect_tx(full_S + k % kRingNS, 64 * kD * 4);
            bulk_g2s(smem + L.S + (k % kRingNS) * (64 * kD * 4),
                     a.p.state + (((size_t)r * Hv + h) * kD + (size_t)tg * 64) * kD, 64 * kD * 4, full_S + k % kRingNS);
        };
        const bool early = a.pdl_early != 0;
        if (early && lane == 0)   // the states this grid starts with stream in while the previous grid drains
            for (int k = 0; k < kRingNS && (int)blockIdx.x + k * stride < n_units; ++k) issue_state(k);
        if (a.pdl) pdl_wait();
        pdl_trigger();
        // one unit of lookahead for the scalars (count, alpha, beta)
        int nx_j0 = 0;
        float nx_al = 1.f, nx_be = 0.f;
        auto prefetch = [&](int u) {
            int zi, h, tg;
            unit(u, zi, h, tg);
            const int r = a.first + zi;
            if (lane == 0) nx_j0 = a.j0_fixed >= 0 ? a.j0_fixed : a.p.occ[r];
            if (lane == 1) nx_al = a.alpha[(size_t)zi * Hv + h];
            if (lane == 2) nx_be = a.beta[(size_t)zi * Hv + h];
        };
        if ((int)blockIdx.x < n_units) prefetch(blockIdx.x);
        for (int k = 0;; ++k) {
            const int u = blockIdx.x + k * stride;
            if (u >= n_units) break;
            int zi, h, tg;
            unit(u, zi, h, tg);
            const int r = a.first + zi, hk = h / dm.g;
            const int j0 = __shfl_sync(0xffffffffu, nx_j0, 0);
            const float al = nx_al, be = nx_be;
            if (u + stride < n_units) prefetch(u + stride);
            const int bs = k % kRingNS, br = k % kRingNR;
            // state buffer: free once the pair that used it for unit k - NS reduced its rows
            if (lane == 0 && !(early && k < kRingNS)) {
                if (k >= kRingNS) mbar_wait(empty_S + bs, ((k / kRingNS) - 1) & 1);
                issue_state(k);
            }
            // record buffer: free once unit k - NR finished
            if (k >= kRingNR) mbar_wait(empty_R + br, ((k / kRingNR) - 1) & 1);
            unsigned char *Rb = smem + L.R + br * L.rec_bytes;
            if (lane == 1) reinterpret_cast<float *>(Rb + L.ab)[0] = al;
            if (lane == 2) reinterpret_cast<float *>(Rb + L.ab)[1] = be;
            if (lane == 0) reinterpret_cast<int *>(Rb + L.ab)[2] = j0;
            if (lane == 0) {
                const int jbv = (j0 + 3) & ~3;
                const uint32_t bytes = (uint32_t)(2 * j0 * kUSub * usz + j0 * kD * isz + (j0 ? jbv * 4 : 0) +
                                                  2 * kD * isz + 64 * isz);
                mbar_arrive_expect_tx(full_R + br, bytes);
                if (j0) {
                    for (int x = 0; x < 2; ++x)
                        bulk_g2s(Rb + L.U + x * j0 * kUSub * usz,
                                 static_cast<const UT *>(a.p.U) + ((((size_t)r * Hv + h) * (kD / kUSub) + tg * 2 + x) * T) * kUSub,
                                 (uint32_t)(j0 * kUSub * usz), full_R + br);
                    bulk_g2s(Rb + L.K, static_cast<const InT *>(a.p.K) + ((size_t)r * Hk + hk) * T * kD,
                             (uint32_t)(j0 * kD * isz), full_R + br);
                    bulk_g2s(Rb + L.G, a.p.G + ((size_t)r * Hv + h) * T, (uint32_t)(jbv * 4), full_R + br);
                }
                bulk_g2s(Rb + L.q, static_cast<const InT *>(a.q) + ((size_t)zi * Hk + hk) * kD, kD * isz, full_R + br);
                bulk_g2s(Rb + L.k, static_cast<const InT *>(a.k) + ((size_t)zi * Hk + hk) * kD, kD * isz, full_R + br);
                bulk_g2s(Rb + L.v, static_cast<const InT *>(a.v) + ((size_t)zi * Hv + h) * kD + tg * 64, 64 * isz,
                         full_R + br);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(full_R + br);   // (alpha, beta, j0 written)
        }
        return;
    }

    // ======================================================== consumer pairs
    if (a.pdl) pdl_wait();
    pdl_trigger();
    const int pair = warp >> 1, wt = warp & 1;   // the pair's warp = 32-row tile of the unit's 64 rows
    const int seg = lane & 3, team = lane >> 2, par = team & 1;
    float *av = reinterpret_cast<float *>(smem + L.P + pair * al128((uint32_t)(2 * 64 * 4 + 2 * (a.j0_cap + 1 + 3) * 4)));
    float *bv = av + 64;
    float *Ck = bv + 64;
    float *Cq = Ck + ((a.j0_cap + 1 + 3) & ~3);
    auto pbar = [&]() { named_bar_sync(1 + pair, 64); };
    unsigned bad = 0;
    for (int k = pair;; k += kRingPairs) {
        const int u = blockIdx.x + k * stride;
        if (u >= n_units) break;
        int zi, h, tg;
        unit(u, zi, h, tg);
        const int r = a.first + zi, hk = h / dm.g;
        const int bs = k % kRingNS, br = k % kRingNR;
        const unsigned char *Rb = smem + L.R + br * L.rec_bytes;
        const float *S_s = reinterpret_cast<const float *>(smem + L.S + bs * (64 * kD * 4));
        const UT *U_s = reinterpret_cast<const UT *>(Rb + L.U);
        const InT *K_s = reinterpret_cast<const InT *>(Rb + L.K);
        const float *G_s = reinterpret_cast<const float *>(Rb + L.G);
        const InT *q_s = reinterpret_cast<const InT *>(Rb + L.q), *k_s = reinterpret_cast<const InT *>(Rb + L.k);
        const InT *v_s = reinterpret_cast<const InT *>(Rb + L.v);
        mbar_wait(full_R + br, (k / kRingNR) & 1);
        const float al = reinterpret_cast<const float *>(Rb + L.ab)[0], be = reinterpret_cast<const float *>(Rb + L.ab)[1];
        const int j0 = reinterpret_cast<const int *>(Rb + L.ab)[2], J = j0 + 1;
        const float x_l = dm.variant == 2 ? 0.f : logf(al);
        const float gt = (j0 > 0 ? G_s[j0 - 1] : 0.f) + x_l;
        if (dm.validate && wt == 0 && lane == 0) {
            if (dm.variant != 2 && !(al > 0.f && al <= 1.f)) bad |= 0x1u;
            if (!(be >= 0.f && be <= 1.f)) bad |= 0x2u;
        }
        float4 kx[8], qx[8];
        load_row8(k_s, seg, par, kx);
        load_row8(q_s, seg, par, qx);
        // ---- the state rows of this warp's 32-row tile (4-lane teams, 8 rows per step)
        mbar_wait(full_S + bs, (k / kRingNS) & 1);
#pragma unroll 4
        for (int st = 0; st < 4; ++st) {
            const int rf = st * 8 + team;
            float4 x[8];
            load_row8(S_s + (size_t)(wt * 32 + rf) * kD, seg, par, x);
            float vals[2] = {dot8x4(x, kx), dot8x4(x, qx)};
            float res[1];
            int xid[1];
            team_reduce<2>(vals, seg, res, xid);
            if (xid[0] >= 0) (xid[0] ? bv : av)[wt * 32 + rf] = res[0];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty_S + bs);   // the state buffer goes back to the producer
        // ---- key rows (k_t.k_i, q_t.k_i, i < J), shared out over the pair's warps, weighted (Z3)
        for (int ks = wt; ks * 8 < J; ks += 2) {
            const int i = ks * 8 + team;
            float4 x[8];
            if (i < J) {
                load_row8(i < j0 ? K_s + (size_t)i * kD : k_s, seg, par, x);
            } else {
#pragma unroll
                for (int c = 0; c < 8; ++c) x[c] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
            float vals[2] = {dot8x4(x, kx), dot8x4(x, qx)};
            float res[1];
            int xid[1];
            team_reduce<2>(vals, seg, res, xid);
            if (xid[0] >= 0 && i < J) {
                const bool isq = xid[0] == 1;
                const bool valid = isq ? (i <= j0) : (i < j0);
                (isq ? Cq : Ck)[i] = valid ? expf(gt - (i < j0 ? G_s[i] : gt)) * res[0] : 0.f;
            }
        }
        pbar();
        // ---- substitution: lane = d_v row of the warp's tile
        {
            const int row = lane, drow = tg * 64 + wt * 32 + row;
            const UT *ut = U_s + (size_t)wt * j0 * kUSub + row;
            float ak0 = 0.f, ak1 = 0.f, aq0 = 0.f, aq1 = 0.f;
            int i = 0;
            for (; i + 1 < j0; i += 2) {
                const float u0 = to_f(ut[(size_t)i * kUSub]), u1 = to_f(ut[(size_t)(i + 1) * kUSub]);
                ak0 = fmaf(Ck[i], u0, ak0);
                aq0 = fmaf(Cq[i], u0, aq0);
                ak1 = fmaf(Ck[i + 1], u1, ak1);
                aq1 = fmaf(Cq[i + 1], u1, aq1);
            }
            if (i < j0) {
                const float u0 = to_f(ut[(size_t)i * kUSub]);
                ak0 = fmaf(Ck[i], u0, ak0);
                aq0 = fmaf(Cq[i], u0, aq0);
            }
            const float eG = expf(gt);
            const float vt = to_f(v_s[wt * 32 + row]);
            float uu = be * (vt - fmaf(eG, av[wt * 32 + row], ak0 + ak1));
            if (dm.variant != 0) uu = vt;   // no delta rule: the buffered value is v_t itself
            const UT us = from_f<UT>(uu);
            const float un = to_f(us);
            const float o = fmaf(Cq[j0], un, fmaf(eG, bv[wt * 32 + row], aq0 + aq1));
            if (dm.validate && !isfinite(vt)) bad |= 0x4u;
            if (a.o) a.o[((size_t)zi * Hv + h) * kD + drow] = o;
            const size_t bh = (size_t)r * Hv + h;
            static_cast<UT *>(a.p.U)[((bh * (kD / kUSub) + tg * 2 + wt) * T + j0) * kUSub + row] = us;
            if (dm.keep_raw) {
                static_cast<InT *>(a.p.V)[(bh * T + j0) * kD + drow] = v_s[wt * 32 + row];
                if (tg == 0 && wt == 0 && row == 0) a.p.B[bh * T + j0] = be;
            }
        }
        // ---- records: k_t once per QK head, G_t per V head (first half)
        if (tg == 0) {
            const int t64 = wt * 32 + lane;
            if (h % dm.g == 0) {
                InT *Kdst = static_cast<InT *>(a.p.K) + (((size_t)r * Hk + hk) * T + j0) * kD;
                Kdst[t64] = k_s[t64];
                Kdst[t64 + 64] = k_s[t64 + 64];
            }
            if (t64 == 0) a.p.G[((size_t)r * Hv + h) * T + j0] = gt;
        }
        if (dm.validate) {
            const int t64 = wt * 32 + lane;
            const float kk0 = to_f(k_s[t64]), kk1 = to_f(k_s[t64 + 64]), qq0 = to_f(q_s[t64]), qq1 = to_f(q_s[t64 + 64]);
            if (!(isfinite(kk0) && isfinite(kk1) && isfinite(qq0) && isfinite(qq1))) bad |= 0x4u;
        }
        pbar();   // the pair is done with the record buffer, Ck / Cq and a / b
        if (lane == 0) mbar_arrive(empty_R + br);
        // ---- the slot's counter: the last of its 2 Hv units advances occ
        if (wt == 0 && lane == 0 && atomicAdd(&a.p.ticket[r], 1) == 2 * Hv - 1) {
            a.p.ticket[r] = 0;
            a.p.occ[r] = J;
        }
    }
    if (bad) atomicOr(a.p.status, bad);
}

static int ring_sm_count() {
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

template <typename InT, typename UT>
static cudaError_t launch_ring_t(const ChunkArgs &a, cudaStream_t s) {
    const RingSmem L = ring_layout(a.j0_cap, (int)sizeof(InT), (int)sizeof(UT));
    if (L.total > 227 * 1024) return cudaErrorInvalidConfiguration;
    auto kfn = decode_ring_kernel<InT, UT>;
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
    if (e != cudaSuccess || a.dry) return e;
    const int units = a.n * a.dm.Hv * 2;
    const int grid = units < ring_sm_count() ? units : ring_sm_count();
    return launch_k(kfn, dim3(grid), dim3(kRingThreads), L.total, s, a.pdl != 0, a);
}

// decode step (NT = 1) of a contiguous range: the ring kernel
cudaError_t launch_decode_ring(const ChunkArgs &a, cudaStream_t s) {
    if (a.dm.in_dt == DT_F32) return launch_ring_t<float, float>(a, s);
    if (a.dm.u_dt == DT_F16) return launch_ring_t<__nv_bfloat16, __half>(a, s);
    return launch_ring_t<__nv_bfloat16, float>(a, s);
}

}  // namespace labuf
