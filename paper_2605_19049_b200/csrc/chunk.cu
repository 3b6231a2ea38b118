// chunk.cu — launch dispatch of the chunk-attend kernel (chunk.cuh): kernels
// (1) buffered decode, (3) parallel draft verification, (4) direct
// short-context decoding and the prefill chunk step, by input / delta-value
// dtype and by kind (the instantiations live in chunk_<dtype>_<kind>.cu).
#include "chunk.cuh"

namespace labuf {

cudaError_t launch_chunk(const ChunkArgs &a, cudaStream_t s, int64_t *launches) {
    if (a.n <= 0 || a.n_new <= 0) return cudaSuccess;
    if (a.n_new > max_new_per_launch(a.dm.g)) return cudaErrorInvalidValue;
    const bool direct = a.kind == CK_DIRECT;
    cudaError_t e;
    if (a.dm.in_dt == DT_F32)
        e = direct ? launch_direct_f32(a, s) : launch_state_f32(a, s);
    else if (a.dm.u_dt == DT_F16)
        e = direct ? launch_direct_bf16h(a, s) : launch_state_bf16h(a, s);
    else
        e = direct ? launch_direct_bf16(a, s) : launch_state_bf16(a, s);
    if (e == cudaSuccess && !a.dry) ++*launches;
    return e;
}

}  // namespace labuf
