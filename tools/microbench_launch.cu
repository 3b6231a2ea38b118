// CTA launch-rate microbenchmark: near-empty kernels with the hot path's
// grid / block / dynamic shared memory shapes, timed with CUDA events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_launch tools/microbench_launch.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void empty_k(int *p) {
    extern __shared__ int sm[];
    if (threadIdx.x == 0 && p[blockIdx.x & 7] == 12345) sm[0] = 1, p[0] = sm[0];
}
__global__ void tmem_k(int *p) {
    __shared__ unsigned slot;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"((unsigned)__cvta_generic_to_shared(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(slot));
    if (threadIdx.x == 0 && p[blockIdx.x & 7] == 12345) p[0] = 1;
}

int main() {
    int *p;
    cudaMalloc(&p, 64);
    cudaMemset(p, 0, 64);
    struct Cfg { int grid, block, smem, tm; } cfgs[] = {
        {4096, 64, 0, 0}, {4096, 64, 41 * 1024, 0}, {16384, 64, 41 * 1024, 0}, {32768, 128, 0, 0},
        {32768, 128, 28 * 1024, 0}, {32768, 128, 28 * 1024, 1}, {4096, 128, 28 * 1024, 1},
        {8192, 32, 20 * 1024, 0}, {1184, 128, 28 * 1024, 0}};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (auto c : cfgs) {
        cudaFuncSetAttribute(empty_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
        cudaFuncSetAttribute(tmem_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
        float best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(e0);
            for (int i = 0; i < 10; ++i) {
                if (c.tm) tmem_k<<<c.grid, c.block, c.smem>>>(p);
                else empty_k<<<c.grid, c.block, c.smem>>>(p);
            }
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms * 100.f < best ? ms * 100.f : best;
        }
        printf("grid %6d block %4d smem %6d tmem %d : %8.2f us per launch, %6.2f ns per CTA (%s)\n", c.grid, c.block,
               c.smem, c.tm, best, best * 1e3 / c.grid, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
