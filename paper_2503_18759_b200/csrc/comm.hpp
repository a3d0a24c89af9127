// NCCL access for sharded contexts.  libnccl is dlopen'ed on first use so
// the single-GPU library has no link-time NCCL dependency and shares the
// process's already-loaded NCCL (torch ships one) when there is one.
#pragma once

#include <cstddef>
#include <string>

#include <cuda_runtime.h>
#include <nccl.h>

namespace cpdb {

struct Nccl {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                                  ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    bool ok = false;
    std::string why;
};

// Loads libnccl.so.2 once; returns the table (ok == false with `why` set on
// failure).
const Nccl& nccl();

}  // namespace cpdb
