// nccl_dl.h -- NCCL resolved at run time (dlopen), so that libdespot loads and
// runs single-GPU work without NCCL and a sharded process uses the libnccl
// it already has (torch's), else $DESPOT_NCCL_LIB, else the loader's search
// path.  Types come from nccl.h; no NCCL symbol is linked.
#pragma once
#include <dlfcn.h>

#include <cstdlib>
#include <mutex>
#include <string>

#include "nccl.h"

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
  int version = 0;
  bool ok = false;
  std::string err;
};

inline NcclApi& nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // already in the process (torch)
    if (!h)
      if (const char* e = getenv("DESPOT_NCCL_LIB")) h = dlopen(e, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* d = dlerror();
      api.err = std::string("cannot load libnccl.so.2: ") + (d ? d : "?");
      return;
    }
#define HD_NCCL_SYM(n)                                                       \
  api.n = reinterpret_cast<decltype(api.n)>(dlsym(h, "nccl" #n));            \
  if (!api.n) {                                                              \
    api.err = "libnccl.so.2 lacks nccl" #n;                                  \
    return;                                                                  \
  }
    HD_NCCL_SYM(GetUniqueId)
    HD_NCCL_SYM(CommInitRank)
    HD_NCCL_SYM(CommDestroy)
    HD_NCCL_SYM(CommAbort)
    HD_NCCL_SYM(AllReduce)
    HD_NCCL_SYM(AllGather)
    HD_NCCL_SYM(GroupStart)
    HD_NCCL_SYM(GroupEnd)
    HD_NCCL_SYM(GetErrorString)
    HD_NCCL_SYM(GetVersion)
#undef HD_NCCL_SYM
    api.GetVersion(&api.version);
    api.ok = true;
  });
  return api;
}
