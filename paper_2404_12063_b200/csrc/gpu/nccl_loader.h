// NCCL reached through dlopen (vpinn_gpu.cu's multi-GPU fallback path):
// no link-time dependency, a libnccl already loaded into the process (e.g.
// by torch) is reused.  Included after host_runtime.h (Fail).
#pragma once

#include <dlfcn.h>

#include <string>

#include <nccl.h>

namespace {

struct NcclUid {
  char b[NCCL_UNIQUE_ID_BYTES];
};
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*get_unique_id)(NcclUid*) = nullptr;
  ncclResult_t (*comm_init_rank)(void**, int, NcclUid, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, void*,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(void*) = nullptr;
  const char* (*get_error)(ncclResult_t) = nullptr;
};
NcclApi& nccl() {
  static NcclApi api;
  if (!api.h) {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw Fail{VPINN_ERR_DEVICE, std::string("cannot load libnccl: ") + dlerror()};
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.get_error = reinterpret_cast<decltype(api.get_error)>(dlsym(h, "ncclGetErrorString"));
    if (!api.get_unique_id || !api.comm_init_rank || !api.all_reduce || !api.comm_destroy)
      throw Fail{VPINN_ERR_DEVICE, "libnccl lacks the required symbols"};
    api.h = h;
  }
  return api;
}
#define NK(x)                                                                         \
  do {                                                                                \
    ncclResult_t r_ = (x);                                                            \
    if (r_ != ncclSuccess)                                                            \
      throw Fail{VPINN_ERR_DEVICE, std::string("nccl: ") +                            \
                                       (nccl().get_error ? nccl().get_error(r_) : "?")}; \
  } while (0)

}  // namespace
