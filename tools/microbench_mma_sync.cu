// Throughput of the warp-level mma.sync tensor-core path on sm_100a
// (m16n8k8 tf32 and m16n8k16 bf16, fp32 accumulate), register operands,
// 8 independent accumulators per warp.  Decides whether a small-CTA state
// pass (verify / prefill: S0 [rows x 128] times 2N token vectors) can use
// mma.sync instead of tcgen05 (no TMEM allocation per CTA).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_mma tools/microbench_mma_sync.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <bool BF16>
__global__ void kern(float *out, int iters) {
    float acc[8][4] = {};
    uint32_t a[4], b[2];
    for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(1.0f + threadIdx.x * 1e-3f + i);
    for (int i = 0; i < 2; ++i) b[i] = __float_as_uint(0.5f + threadIdx.x * 1e-3f + i);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (BF16)
                asm volatile(
                    "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                    : "+f"(acc[j][0]), "+f"(acc[j][1]), "+f"(acc[j][2]), "+f"(acc[j][3])
                    : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
            else
                asm volatile(
                    "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                    : "+f"(acc[j][0]), "+f"(acc[j][1]), "+f"(acc[j][2]), "+f"(acc[j][3])
                    : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
        }
    }
    float s = 0.f;
    for (int j = 0; j < 8; ++j)
        for (int i = 0; i < 4; ++i) s += acc[j][i];
    if (s == 12345.f) out[threadIdx.x] = s;
}

int main() {
    float *out;
    cudaMalloc(&out, 4096);
    const int iters = 4096;
    for (int bf = 0; bf < 2; ++bf) {
        for (int warps : {4, 8, 16}) {
            dim3 grid(148 * 4), block(32 * warps);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(e0);
                if (bf) kern<true><<<grid, block>>>(out, iters);
                else kern<false><<<grid, block>>>(out, iters);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
            }
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double k = bf ? 16 : 8;
            const double flops = 2.0 * 16 * 8 * k * 8 * iters * (double)grid.x * warps;
            printf("%s warps/CTA %2d: %.1f TFLOP/s (%.3f ms)\n", bf ? "bf16 m16n8k16" : "tf32 m16n8k8 ", warps,
                   flops / ms / 1e9, ms);
        }
    }
    return 0;
}
