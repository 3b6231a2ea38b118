// TMEM allocation cost microbenchmark (B200): CTAs that only allocate and
// free TMEM, in the fold kernel's grid shape, with variations.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_tmem tools/microbench_tmem.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int NCOLS, bool RELINQ, bool DEALLOC_BY_SAME_WARP_EARLY>
__global__ void k(int *p) {
    __shared__ unsigned slot;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&slot)), "n"(NCOLS));
        if (RELINQ) asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "n"(NCOLS));
    if (threadIdx.x == 0 && p[blockIdx.x & 7] == 12345) p[0] = 1;
}
// a kernel that CAN allocate but (at run time) does not
template <bool RELINQ>
__global__ void noalloc_k(int *p) {
    __shared__ unsigned slot;
    if (threadIdx.x < 32 && p[0] == 12345) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"((unsigned)__cvta_generic_to_shared(&slot)));
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(slot));
    }
    if (RELINQ && threadIdx.x < 32) asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    if (threadIdx.x == 0 && p[blockIdx.x & 7] == 12345) p[0] = 1;
}
// one CTA per SM looping: pure alloc/dealloc latency
__global__ void loop_k(int *p, long long *cyc) {
    __shared__ unsigned slot;
    long long t0 = clock64();
    for (int i = 0; i < 64; ++i) {
        if (threadIdx.x < 32)
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"((unsigned)__cvta_generic_to_shared(&slot)));
        __syncthreads();
        if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(slot));
        __syncthreads();
    }
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

template <typename F>
void run(const char *name, F f, int grid) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        for (int i = 0; i < 10; ++i) f();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms * 100.f < best ? ms * 100.f : best;
    }
    printf("%-40s grid %6d: %8.2f us per launch, %6.2f ns per CTA (%s)\n", name, grid, best, best * 1e3 / grid,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int *p;
    long long *cyc;
    cudaMalloc(&p, 64);
    cudaMemset(p, 0, 64);
    cudaMalloc(&cyc, 148 * 8);
    const int smem = 28 * 1024;
    cudaFuncSetAttribute(k<32, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k<32, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k<128, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int g : {4096, 32768}) {
        run("alloc32 + relinquish + dealloc", [&] { k<32, true, false><<<g, 128, smem>>>(p); }, g);
        run("alloc32 + dealloc (no relinquish)", [&] { k<32, false, false><<<g, 128, smem>>>(p); }, g);
        run("alloc128 + relinquish + dealloc", [&] { k<128, true, false><<<g, 128, smem>>>(p); }, g);
    }
    cudaFuncSetAttribute(noalloc_k<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(noalloc_k<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    run("no alloc, relinquish", [&] { noalloc_k<true><<<32768, 128, smem>>>(p); }, 32768);
    run("no alloc, no relinquish", [&] { noalloc_k<false><<<32768, 128, smem>>>(p); }, 32768);
    loop_k<<<148, 128>>>(p, cyc);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("loop: alloc+dealloc round trip %.0f cycles (1 CTA per SM) (%s)\n", h[0] / 64.0,
           cudaGetErrorString(cudaGetLastError()));
    return 0;
}
