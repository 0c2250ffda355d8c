#include <dlfcn.h>

#include <mutex>
#include <string>

#include "cuda_api.hpp"

namespace cgf::drv {

#define CGF_DRV_DEF(fn) decltype(&::fn) fn = nullptr;
CGF_DRV_FUNCS(CGF_DRV_DEF)
#undef CGF_DRV_DEF

#define CGF_STR2(x) #x
#define CGF_STR(x) CGF_STR2(x)

bool load(std::string* why) {
  static std::once_flag once;
  static bool ok = false;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libcuda.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("no CUDA driver (libcuda.so.1): ") + dlerror();
      return;
    }
    ok = true;
    // cuda.h maps e.g. cuMemAlloc -> cuMemAlloc_v2; CGF_STR expands the macro.
#define CGF_DRV_LOAD(fn)                                            \
    fn = reinterpret_cast<decltype(&::fn)>(dlsym(h, CGF_STR(fn)));  \
    if (!fn) { ok = false; err = std::string("libcuda lacks ") + CGF_STR(fn); }
    CGF_DRV_FUNCS(CGF_DRV_LOAD)
#undef CGF_DRV_LOAD
  });
  if (!ok && why) *why = err;
  return ok;
}

}  // namespace cgf::drv
