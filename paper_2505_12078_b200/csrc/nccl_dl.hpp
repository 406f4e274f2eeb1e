// NCCL entry points resolved at run time (dlopen of libnccl.so.2): the
// sharded solver's collectives enqueue on the solver's stream from C++ with no
// host callback.  Under Python the process already holds torch's NCCL (same
// soname), so the library uses that copy; a C++ caller gets the system one.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

namespace spock {

struct NcclDl {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

// the resolved table; throws std::runtime_error when NCCL cannot be loaded
const NcclDl& nccl_dl();
// throws std::runtime_error on a failed NCCL call
void nccl_check(ncclResult_t r, const char* what);

}  // namespace spock
