// nccl_dl.cuh -- NCCL resolved lazily with dlopen so libdinr.so never forces a second copy of
// libnccl.so.2 into a process: in a torch process the already-loaded library is reused.
// Path: $DINR_NCCL_LIB if set (the Python binding points it at torch's bundled NCCL), else
// the loader's "libnccl.so.2".
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <string>

namespace dinr {

struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

inline NcclApi &nccl() {
  static NcclApi api = [] {
    NcclApi a;
    const char *path = std::getenv("DINR_NCCL_LIB");
    void *h = dlopen(path && *path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.err = std::string("dlopen(libnccl.so.2) failed: ") + dlerror();
      return a;
    }
    a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))dlsym(h, "ncclCommInitRank");
    a.AllReduce = (decltype(a.AllReduce))dlsym(h, "ncclAllReduce");
    a.CommDestroy = (decltype(a.CommDestroy))dlsym(h, "ncclCommDestroy");
    a.GetErrorString = (decltype(a.GetErrorString))dlsym(h, "ncclGetErrorString");
    a.ok = a.GetUniqueId && a.CommInitRank && a.AllReduce && a.CommDestroy && a.GetErrorString;
    if (!a.ok) a.err = "libnccl.so.2 lacks a required symbol";
    return a;
  }();
  return api;
}

}  // namespace dinr
