// Where does dynamic shared memory start inside a CTA's shared window on
// sm_100a?  (Decides whether the 1 KiB alignment slack for 128-byte-swizzled
// TMA tiles is needed.)  nvcc -gencode arch=compute_100a,code=sm_100a -o tools/probe_smem_align tools/probe_smem_align.cu
#include <cstdio>
#include <cstdint>
__global__ void k(unsigned *out) {
    extern __shared__ __align__(1024) unsigned char smem[];
    if (threadIdx.x == 0) out[blockIdx.x] = (unsigned)__cvta_generic_to_shared(smem);
}
int main() {
    unsigned *d, h[64];
    cudaMalloc(&d, 64 * 4);
    for (int sz : {4096, 40000, 45000, 100000}) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sz);
        k<<<64, 64, sz>>>(d);
        cudaMemcpy(h, d, 64 * 4, cudaMemcpyDeviceToHost);
        unsigned mx = 0;
        for (int i = 0; i < 64; ++i) mx |= h[i] & 1023u;
        printf("dyn %6d B: base %u, OR of (base mod 1024) over 64 CTAs = %u\n", sz, h[0], mx);
    }
    return 0;
}
