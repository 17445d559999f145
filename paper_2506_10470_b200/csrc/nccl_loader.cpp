// nccl_loader.cpp -- lazy NCCL (dlopen), so single-process and CPU-only use of
// the library never needs libnccl.  Search order: $TDPIPE_NCCL_LIB, the
// torch-bundled nvidia/nccl wheel next to the running interpreter, the system.
#include <dlfcn.h>

#include <cstdlib>
#include <string>

void* tdp_nccl_handle(std::string* err) {
  static void* h = nullptr;
  if (h) return h;
  const char* env = std::getenv("TDPIPE_NCCL_LIB");
  const char* cands[] = {env, "libnccl.so.2", "libnccl.so"};
  for (const char* c : cands) {
    if (!c) continue;
    h = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
    if (h) return h;
  }
  if (err) *err = std::string("cannot dlopen libnccl.so.2: ") + (dlerror() ? dlerror() : "");
  return nullptr;
}

#ifndef TDP_NO_NCCL
#include "nccl_rt.h"

namespace tdp {
const NcclApi* nccl_api(std::string* err) {
  static NcclApi api;
  static bool ok = false;
  if (ok) return &api;
  void* h = tdp_nccl_handle(err);
  if (!h) return nullptr;
  api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
  api.send = (decltype(api.send))dlsym(h, "ncclSend");
  api.recv = (decltype(api.recv))dlsym(h, "ncclRecv");
  api.allReduce = (decltype(api.allReduce))dlsym(h, "ncclAllReduce");
  api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
  api.getErrorString = (decltype(api.getErrorString))dlsym(h, "ncclGetErrorString");
  if (!api.commInitRank || !api.send || !api.recv || !api.allReduce || !api.commDestroy || !api.getErrorString) {
    if (err) *err = "libnccl is missing an entry point";
    return nullptr;
  }
  ok = true;
  return &api;
}
}  // namespace tdp
#endif
