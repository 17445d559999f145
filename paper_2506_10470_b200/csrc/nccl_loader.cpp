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
