// microbench_bulk.cu — HBM streaming microbenchmarks on B200 (tool, not the
// product): how fast can one SM pull data into shared memory with
// cp.async.bulk (UBLKCP) in different arrangements, versus plain 16-byte
// loads?  Used to size the decode kernel's pipeline.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        tools/microbench_bulk.cu -o /tmp/mb && /tmp/mb
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c));
}
__device__ __forceinline__ void expect_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t *b, uint32_t par) {
    uint32_t done;
    do {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                     : "=r"(done) : "r"(sa(b)), "r"(par) : "memory");
    } while (!done);
}
__device__ __forceinline__ void bulk(void *dst, const void *src, uint32_t bytes, uint64_t *b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sa(dst)), "l"(src), "r"(bytes), "r"(sa(b)) : "memory");
}

// A: persistent ring.  item = `chunk` bytes split into `pieces` copies.
__global__ void ring_kernel(const char *src, size_t total, int chunk, int pieces, int ns, float *sink) {
    extern __shared__ __align__(1024) unsigned char sm[];
    uint64_t *full = (uint64_t *)sm, *empty = full + 16;
    unsigned char *buf = sm + 256;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ncons = blockDim.x / 32 - 1;
    if (threadIdx.x == 0) {
        for (int s = 0; s < ns; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const size_t n_items = total / chunk;
    if (warp == ncons) {
        if (lane == 0) {
            int it = 0;
            for (size_t item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
                const int s = it % ns;
                if (it >= ns) wait(&empty[s], ((it / ns) - 1) & 1);
                expect_tx(&full[s], chunk);
                const int pb = chunk / pieces;
                for (int p = 0; p < pieces; ++p)
                    bulk(buf + (size_t)s * chunk + p * pb, src + item * chunk + p * pb, pb, &full[s]);
            }
        }
        return;
    }
    // consumers: warp w takes items it = w, w + ncons, ...  (ns % ncons == 0)
    float acc = 0.f;
    int it = warp;
    for (size_t item = blockIdx.x + (size_t)warp * gridDim.x; item < n_items; item += (size_t)ncons * gridDim.x, it += ncons) {
        const int s = it % ns;
        wait(&full[s], (it / ns) & 1);
        acc += ((const float *)(buf + (size_t)s * chunk))[lane];
        __syncwarp();
        if (lane == 0) arrive(&empty[s]);
    }
    if (acc == 12345.f) *sink = acc;
}

// C: one item per CTA (non-persistent), several CTAs per SM.
__global__ void oneshot_kernel(const char *src, int chunk, int pieces, float *sink) {
    extern __shared__ __align__(1024) unsigned char sm[];
    uint64_t *full = (uint64_t *)sm;
    unsigned char *buf = sm + 128;
    if (threadIdx.x == 0) {
        mbar_init(full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        expect_tx(full, chunk);
        const int pb = chunk / pieces;
        for (int p = 0; p < pieces; ++p) bulk(buf + p * pb, src + (size_t)blockIdx.x * chunk + p * pb, pb, full);
    }
    __syncthreads();
    wait(full, 0);
    float v = ((const float *)buf)[threadIdx.x];
    if (v == 12345.f) *sink = v;
}

// D: plain 16-byte loads, grid-stride.
__global__ void ldg_kernel(const float4 *src, size_t n4, float *sink) {
    float acc = 0.f;
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const size_t st = (size_t)gridDim.x * blockDim.x;
    for (; i + 3 * st < n4; i += 4 * st) {
        float4 a = __ldg(src + i), b = __ldg(src + i + st), c = __ldg(src + i + 2 * st), d = __ldg(src + i + 3 * st);
        acc += a.x + b.y + c.z + d.w;
    }
    if (acc == 12345.f) *sink = acc;
}

int main() {
    const size_t total = (size_t)2 << 30;   // 2 GiB >> L2
    char *src; float *sink;
    CK(cudaMalloc(&src, total));
    CK(cudaMalloc(&sink, 4));
    CK(cudaMemset(src, 0, total));
    int nsm; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto timeit = [&](auto launch) {
        launch(); CK(cudaDeviceSynchronize());
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0); launch(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
            float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
        }
        return total / (best * 1e-3) / 1e9;
    };
    CK(cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    CK(cudaFuncSetAttribute(oneshot_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    printf("A ring (persistent, 1 CTA/SM, 1 producer lane)\n");
    const int chunks[] = {4096, 8192, 16384, 32768};
    for (int chunk : chunks)
        for (int ns : {2, 4, 8, 12})
            for (int ncons : {1, 4})
                for (int pieces : {1, 8}) {
                    if ((size_t)chunk * ns + 256 > 227 * 1024 || ns % ncons) continue;
                    const int smem = chunk * ns + 256;
                    double gbs = timeit([&] { ring_kernel<<<nsm, (ncons + 1) * 32, smem>>>(src, total, chunk, pieces, ns, sink); });
                    printf("  chunk %6d ns %2d cons %d pieces %d  -> %7.0f GB/s  (%5.1f KB in flight/SM)\n", chunk, ns, ncons, pieces, gbs, chunk * ns / 1024.0);
                }
    printf("A2 ring, 2 CTAs/SM\n");
    for (int chunk : {16384, 32768})
        for (int ns : {2, 3, 4, 6})
            for (int pieces : {1, 8}) {
                if ((size_t)chunk * ns + 256 > 113 * 1024) continue;
                const int smem = chunk * ns + 256;
                double gbs = timeit([&] { ring_kernel<<<2 * nsm, 2 * 32, smem>>>(src, total, chunk, pieces, ns, sink); });
                printf("  chunk %6d ns %2d pieces %d  -> %7.0f GB/s\n", chunk, ns, pieces, gbs);
            }
    printf("C oneshot (grid = total / chunk)\n");
    for (int chunk : {8192, 16384, 32768, 65536})
        for (int pieces : {1, 8}) {
            const int smem = chunk + 128;
            double gbs = timeit([&] { oneshot_kernel<<<total / chunk, 128, smem>>>(src, chunk, pieces, sink); });
            printf("  chunk %6d pieces %d -> %7.0f GB/s\n", chunk, pieces, gbs);
        }
    printf("D ldg float4\n");
    for (int bpsm : {4, 8, 16}) {
        double gbs = timeit([&] { ldg_kernel<<<nsm * bpsm, 256>>>((const float4 *)src, total / 16, sink); });
        printf("  %d blocks/SM x 256 thr -> %7.0f GB/s\n", bpsm, gbs);
    }
    return 0;
}
