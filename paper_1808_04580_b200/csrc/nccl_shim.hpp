// nccl_shim.hpp -- NCCL entry points resolved lazily with dlopen.
//
// The library must coexist with PyTorch, which bundles its own (newer)
// libnccl.so.2 with the same SONAME: a link-time dependency would bind
// whichever copy loads first and break the other.  Resolving at first use
// picks the copy already mapped in the process (torch's when torch is
// imported, the system one otherwise).  Only sharded handles touch NCCL.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <string>

#include "common.cuh"

namespace fgsb {

struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

inline const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = dlerror() ? dlerror() : "dlopen(libnccl.so.2) failed";
      return;
    }
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
  });
  if (!api.all_reduce || !api.comm_init_rank || !api.get_unique_id || !api.comm_destroy)
    fail(FGS_ENCCL, "NCCL unavailable: " + (err.empty() ? std::string("missing symbols") : err));
  return api;
}

inline void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    const NcclApi& a = nccl();
    fail(FGS_ENCCL, std::string(what) + ": " + (a.error_string ? a.error_string(r) : "nccl error"));
  }
}

}  // namespace fgsb
