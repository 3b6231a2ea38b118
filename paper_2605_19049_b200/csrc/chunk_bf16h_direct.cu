// chunk_bf16h_direct.cu — one (dtype, kind) slice of the chunk-attend kernel instantiations
// (kernels (1), (3), (4) and the prefill chunk step; see chunk.cuh).
#include "chunk.cuh"

namespace labuf {
cudaError_t launch_direct_bf16h(const ChunkArgs &a, cudaStream_t s) { return launch_direct<__nv_bfloat16, __half>(a, s); }
}  // namespace labuf

#ifdef LABUF_CK_PROF
// per-CTA timeline of the last bf16 / fp16-u direct launch (tools/ck_prof.py)
extern "C" __attribute__((visibility("default"))) int la_debug_ck_prof_direct(unsigned long long *dst) {
    return (int)cudaMemcpyFromSymbol(dst, labuf::g_ck_prof, sizeof(labuf::g_ck_prof));
}
#endif
