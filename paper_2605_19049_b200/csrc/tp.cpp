// tp.cpp — tensor-parallel-over-heads helpers (la_tp_*): the only collective
// in the library.  Each rank owns a contiguous range of QK heads and their V
// heads (GQA pairs stay on one GPU); after a layer's decode, head outputs are
// gathered with one ncclAllGather into a head-major [G][n][Hv/G][d_v] buffer.
// The data-parallel mode (requests partitioned over GPUs) uses no collective
// at all.  NCCL is resolved at run time with dlopen so the library has no
// link-time NCCL dependency (torch's own libnccl.so.2 is reused when loaded)
// and no build-time one either: the few NCCL ABI types used are declared
// here (they are part of NCCL's stable C ABI), so the library builds where
// no nccl.h is installed.  LABUF_NCCL_LIB names the shared object to load
// when libnccl.so.2 is not on the loader path.
#include "../../include/la.h"

#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

extern "C" const char *la_last_error(void);

namespace {

// NCCL C ABI (nccl.h): result codes, the 128-byte unique id, the opaque
// communicator handle and the uint8 data type tag
typedef int ncclResult_t;
constexpr ncclResult_t ncclSuccess = 0;
typedef struct { char internal[128]; } ncclUniqueId;
typedef struct ncclComm *ncclComm_t;
typedef int ncclDataType_t;
constexpr ncclDataType_t ncclUint8 = 1;

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId *);
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    const char *(*GetErrorString)(ncclResult_t);
    bool ok = false;
};

NcclApi g_api;
std::once_flag g_once;
std::string g_load_error;

void load_nccl() {
    // an already loaded libnccl.so.2 (torch imports its bundled copy) is
    // found by soname first
    const char *env = getenv("LABUF_NCCL_LIB");
    const char *candidates[] = {env ? env : "libnccl.so.2", "libnccl.so.2", "libnccl.so"};
    void *h = nullptr;
    for (const char *c : candidates) {
        h = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
        if (h) break;
    }
    if (!h) { g_load_error = std::string("dlopen libnccl.so.2 failed: ") + dlerror(); return; }
    g_api.GetUniqueId = (decltype(g_api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    g_api.CommInitRank = (decltype(g_api.CommInitRank))dlsym(h, "ncclCommInitRank");
    g_api.AllGather = (decltype(g_api.AllGather))dlsym(h, "ncclAllGather");
    g_api.CommDestroy = (decltype(g_api.CommDestroy))dlsym(h, "ncclCommDestroy");
    g_api.GetErrorString = (decltype(g_api.GetErrorString))dlsym(h, "ncclGetErrorString");
    g_api.ok = g_api.GetUniqueId && g_api.CommInitRank && g_api.AllGather && g_api.CommDestroy &&
               g_api.GetErrorString;
    if (!g_api.ok) g_load_error = "libnccl.so.2 lacks required symbols";
}

}  // namespace

// defined in la.cpp
la_status labuf_set_error(la_status st, const char *msg);

extern "C" {

la_status la_tp_unique_id(void *id_out) {
    if (!id_out) return labuf_set_error(LA_ERR_INVALID, "null id output");
    std::call_once(g_once, load_nccl);
    if (!g_api.ok) return labuf_set_error(LA_ERR_NCCL, g_load_error.c_str());
    ncclUniqueId id;
    ncclResult_t r = g_api.GetUniqueId(&id);
    if (r != ncclSuccess) return labuf_set_error(LA_ERR_NCCL, g_api.GetErrorString(r));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    memcpy(id_out, &id, sizeof(id));
    return LA_OK;
}

la_status la_tp_init(const void *unique_id, int32_t rank, int32_t world, int32_t device, void **comm_out) {
    if (!unique_id || !comm_out) return labuf_set_error(LA_ERR_INVALID, "null pointer");
    if (world < 1 || rank < 0 || rank >= world) return labuf_set_error(LA_ERR_INVALID, "bad rank/world");
    std::call_once(g_once, load_nccl);
    if (!g_api.ok) return labuf_set_error(LA_ERR_NCCL, g_load_error.c_str());
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return labuf_set_error(LA_ERR_CUDA, cudaGetErrorString(e));
    ncclUniqueId id;
    memcpy(&id, unique_id, sizeof(id));
    ncclComm_t comm;
    ncclResult_t r = g_api.CommInitRank(&comm, world, id, rank);
    if (r != ncclSuccess) return labuf_set_error(LA_ERR_NCCL, g_api.GetErrorString(r));
    *comm_out = comm;
    return LA_OK;
}

la_status la_tp_allgather(void *comm, const void *send, void *recv, size_t bytes_per_rank,
                          la_stream stream) {
    if (!comm || !send || !recv) return labuf_set_error(LA_ERR_INVALID, "null pointer");
    if (!g_api.ok) return labuf_set_error(LA_ERR_NCCL, "NCCL not initialised (la_tp_init)");
    ncclResult_t r = g_api.AllGather(send, recv, bytes_per_rank, ncclUint8,
                                     static_cast<ncclComm_t>(comm), static_cast<cudaStream_t>(stream));
    if (r != ncclSuccess) return labuf_set_error(LA_ERR_NCCL, g_api.GetErrorString(r));
    return LA_OK;
}

la_status la_tp_destroy(void *comm) {
    if (!comm) return labuf_set_error(LA_ERR_INVALID, "null comm");
    if (!g_api.ok) return labuf_set_error(LA_ERR_NCCL, "NCCL not initialised");
    ncclResult_t r = g_api.CommDestroy(static_cast<ncclComm_t>(comm));
    if (r != ncclSuccess) return labuf_set_error(LA_ERR_NCCL, g_api.GetErrorString(r));
    return LA_OK;
}

}  // extern "C"
