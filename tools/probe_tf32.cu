// Does mma.sync .tf32 (sm_100a) truncate or round fp32 operands with nonzero
// low 13 bits?  A = 1 + 2^-11 + 2^-12 (tf32 keeps 10 mantissa bits), B = 1.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/probe_tf32 tools/probe_tf32.cu
#include <cstdio>
#include <cstdint>
__global__ void k(float *out, float av) {
    float d[4] = {0.f, 0.f, 0.f, 0.f};
    const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
    // A[16x8]: only A[0][0] = av; B[8x8]: only B[0][0] = 1
    uint32_t a[4] = {0u, 0u, 0u, 0u};
    if (g == 0 && t == 0) a[0] = __float_as_uint(av);
    uint32_t b0 = (g == 0 && t == 0) ? __float_as_uint(1.f) : 0u, b1 = 0u;
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
    if (lane == 0) out[0] = d[0];
}
int main() {
    float *o, h;
    cudaMalloc(&o, 4);
    const float vals[3] = {1.f + 0.000732421875f /* 2^-11 + 2^-12 */, 1.f + 0.0003662109375f /* 2^-12 + 2^-13 */, -1.f - 0.000732421875f};
    for (float v : vals) {
        k<<<1, 32>>>(o, v);
        cudaMemcpy(&h, o, 4, cudaMemcpyDeviceToHost);
        const float tr = __builtin_bit_cast(float, __builtin_bit_cast(uint32_t, v) & 0xFFFFE000u);
        printf("A = %.10f  mma = %.10f  trunc = %.10f  %s\n", v, h, tr, h == tr ? "TRUNCATES" : "rounds/other");
    }
    return 0;
}
