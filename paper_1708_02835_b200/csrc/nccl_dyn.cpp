// nccl_dyn.cpp -- see nccl_dyn.h.
#include "nccl_dyn.h"

#include <dlfcn.h>

#include <cstdlib>
#include <mutex>

namespace exageo {
namespace nccl {

ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
ncclResult_t (*Reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t, cudaStream_t) = nullptr;
ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
ncclResult_t (*GroupStart)() = nullptr;
ncclResult_t (*GroupEnd)() = nullptr;
const char* (*GetErrorString)(ncclResult_t) = nullptr;

namespace {
std::mutex g_mu;
void* g_handle = nullptr;
std::string g_err;

template <class F>
bool sym(void* h, const char* name, F& fp) {
  fp = reinterpret_cast<F>(dlsym(h, name));
  if (!fp) g_err = std::string("NCCL symbol missing: ") + name;
  return fp != nullptr;
}
}  // namespace

bool load(std::string* err) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_handle) return true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
  if (!h) {
    if (const char* p = std::getenv("EXAGEO_NCCL_LIBRARY")) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
  }
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    const char* e = dlerror();
    g_err = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
    if (err) *err = g_err;
    return false;
  }
  bool ok = sym(h, "ncclGetUniqueId", GetUniqueId) && sym(h, "ncclCommInitRank", CommInitRank) &&
            sym(h, "ncclCommDestroy", CommDestroy) && sym(h, "ncclBroadcast", Broadcast) &&
            sym(h, "ncclAllReduce", AllReduce) && sym(h, "ncclReduce", Reduce) && sym(h, "ncclCommSplit", CommSplit) &&
            sym(h, "ncclGroupStart", GroupStart) && sym(h, "ncclGroupEnd", GroupEnd) &&
            sym(h, "ncclGetErrorString", GetErrorString);
  if (!ok) {
    if (err) *err = g_err;
    return false;
  }
  g_handle = h;
  return true;
}

}  // namespace nccl
}  // namespace exageo
