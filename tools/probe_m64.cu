// Probe: where does tcgen05.mma.cta_group::1.kind::tf32 with M = 64 put the
// accumulator rows in TMEM?  D[m][n] = m (A[m][0] = m, B[n][0] = 1, rest 0);
// 4 warps read lanes 32w..32w+31, columns 0..15 and print D row per lane.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2605_19049_b200/csrc -o tools/probe_m64 tools/probe_m64.cu
#include <cstdio>
#include "device.cuh"
using namespace labuf;

__global__ void probe(float *out) {
    __shared__ __align__(1024) float A[64 * 8];
    __shared__ __align__(1024) float B[16 * 8];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // K-major SWIZZLE_NONE: (row, k) at (row>>3)*SBO + (k>>2)*LBO + (row&7)*16 + (k&3)*4 bytes, LBO = 128, SBO = 256
    for (int e = tid; e < 64 * 8; e += 128) {
        const int m = e / 8, k = e % 8;
        A[((m >> 3) * 256 + (k >> 2) * 128 + (m & 7) * 16 + (k & 3) * 4) / 4] = (k == 0) ? (float)m : 0.f;
    }
    for (int e = tid; e < 16 * 8; e += 128) {
        const int n = e / 8, k = e % 8;
        B[((n >> 3) * 256 + (k >> 2) * 128 + (n & 7) * 16 + (k & 3) * 4) / 4] = (k == 0) ? 1.f + n : 0.f;
    }
    if (warp == 0) tmem_alloc<32>(&slot);
    if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    // clear TMEM columns 0..31 of all lanes with a sentinel first (st not needed: read before/after)
    if (tid == 0) {
        const uint64_t da = umma_desc_noswz(smem_u32(A), 128, 256);
        const uint64_t db = umma_desc_noswz(smem_u32(B), 128, 256);
        tc_mma_tf32(tmem, da, db, idesc_tf32(64, 16), 0u);
        tc_commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    float v[32];
    tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16), v);
    for (int c = 0; c < 32; ++c) out[(warp * 32 + lane) * 32 + c] = v[c];
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<32>(tmem);
}

int main() {
    float *d;
    cudaMalloc(&d, 128 * 32 * 4);
    cudaMemset(d, 0xff, 128 * 32 * 4);
    probe<<<1, 128>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    printf("err %s\n", cudaGetErrorString(e));
    float h[128 * 32];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    for (int lane = 0; lane < 128; ++lane) {
        printf("lane %3d:", lane);
        for (int c = 0; c < 18; ++c) printf(" %5.0f", h[lane * 32 + c]);
        printf("\n");
    }
    return 0;
}
