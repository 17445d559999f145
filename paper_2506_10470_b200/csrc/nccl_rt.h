// nccl_rt.h -- NCCL entry points resolved at run time (dlopen), used only by
// the multi-process pipeline (one process per GPU = one stage).
#pragma once
#include <cuda_runtime.h>

#include <string>

#ifndef TDP_NO_NCCL
#include <nccl.h>

namespace tdp {
struct NcclApi {
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*commDestroy)(ncclComm_t);
  const char* (*getErrorString)(ncclResult_t);
};
// nullptr (and *err set) if libnccl cannot be loaded.
const NcclApi* nccl_api(std::string* err);
}  // namespace tdp
#endif
