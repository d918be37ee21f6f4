// nccl_dyn.h -- NCCL entry points resolved at run time (dlopen), only when a distributed
// context or an NCCL id is requested. Linking libnccl at build time would pin whichever
// libnccl.so.2 the loader finds first for the whole process (e.g. the system 2.27 ahead
// of the torch-bundled 2.28 torch needs). Resolution order: a libnccl.so.2 already
// loaded in the process (torch's), $EXAGEO_NCCL_LIBRARY, then the loader's search path.
#pragma once
#include <nccl.h>

#include <string>

namespace exageo {
namespace nccl {

bool load(std::string* err);

extern ncclResult_t (*GetUniqueId)(ncclUniqueId*);
extern ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
extern ncclResult_t (*CommDestroy)(ncclComm_t);
extern ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
extern ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
extern ncclResult_t (*Reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t, cudaStream_t);
extern ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*);
extern ncclResult_t (*GroupStart)();
extern ncclResult_t (*GroupEnd)();
extern const char* (*GetErrorString)(ncclResult_t);

}  // namespace nccl
}  // namespace exageo
