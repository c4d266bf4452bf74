// Run-time binding of NCCL (libnccl.so.2): the library is only needed for
// multi-GPU runs, and torch may already have a libnccl.so.2 loaded in the
// process, which dlopen then reuses.
#pragma once

#include <nccl.h>

namespace tw {

struct NcclApi {
    bool loaded = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                              ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

// Loads on first call; throws tw::Error(TW_ERR_NCCL) when unavailable.
const NcclApi& nccl();
void nccl_check(ncclResult_t r, const char* what);
#define TW_NCCL(x) ::tw::nccl_check((x), #x)

} // namespace tw
