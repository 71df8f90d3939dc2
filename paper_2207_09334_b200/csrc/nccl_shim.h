// Minimal run-time binding of NCCL (dlopen): the library loads on hosts
// without NCCL and only resolves it when a sharded engine asks for it.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

namespace ss {

struct NcclApi {
    ncclResult_t (*getUniqueId)(ncclUniqueId *);
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int);
    ncclResult_t (*commDestroy)(ncclComm_t);
    ncclResult_t (*groupStart)();
    ncclResult_t (*groupEnd)();
    ncclResult_t (*send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    const char *(*getErrorString)(ncclResult_t);
};

// Returns nullptr (and sets ss_last_error) if NCCL cannot be loaded.
const NcclApi *nccl_api();

}  // namespace ss
