// chunk_bf16_state.cu — one (dtype, kind) slice of the chunk-attend kernel instantiations
// (kernels (1), (3), (4) and the prefill chunk step; see chunk.cuh).
#include "chunk.cuh"

namespace labuf {
cudaError_t launch_state_bf16(const ChunkArgs &a, cudaStream_t s) { return launch_state<__nv_bfloat16, float>(a, s); }
}  // namespace labuf

#ifdef LABUF_CK_PROF
// per-CTA timeline of the last bf16 state-kind launch (tools/ck_prof.py)
extern "C" __attribute__((visibility("default"))) int la_debug_ck_prof(unsigned long long *dst) {
    return (int)cudaMemcpyFromSymbol(dst, labuf::g_ck_prof, sizeof(labuf::g_ck_prof));
}
#endif
