// chunk_f32_state.cu — one (dtype, kind) slice of the chunk-attend kernel instantiations
// (kernels (1), (3), (4) and the prefill chunk step; see chunk.cuh).
#include "chunk.cuh"

namespace labuf {
cudaError_t launch_state_f32(const ChunkArgs &a, cudaStream_t s) { return launch_state<float, float>(a, s); }
}  // namespace labuf
