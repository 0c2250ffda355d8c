#include "jit.hpp"
#include "cuda_api.hpp"

#include <dlfcn.h>
#include <nvrtc.h>
#include <sys/stat.h>

#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <map>
#include <mutex>
#include <sstream>
#include <vector>

namespace cgf {

void cu_check(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return;
  const char* name = nullptr;
  const char* msg = nullptr;
  drv::cuGetErrorName(r, &name);
  drv::cuGetErrorString(r, &msg);
  throw CudaError(std::string(what) + ": " + (name ? name : "?") + " (" + (msg ? msg : "") + ")");
}

CUcontext ensure_context(int device) {
  std::string why;
  if (!drv::load(&why)) throw CudaError(why);
  static std::once_flag once;
  std::call_once(once, [] { CU_CHECK(drv::cuInit(0)); });
  CUcontext ctx = nullptr;
  CU_CHECK(drv::cuCtxGetCurrent(&ctx));
  if (ctx && device < 0) return ctx;
  if (device < 0) {
    const char* env = std::getenv("CGF_DEVICE");
    device = env ? std::atoi(env) : 0;
  }
  CUdevice dev;
  CU_CHECK(drv::cuDeviceGet(&dev, device));
  CU_CHECK(drv::cuDevicePrimaryCtxRetain(&ctx, dev));
  CU_CHECK(drv::cuCtxSetCurrent(ctx));
  return ctx;
}

namespace {

std::uint64_t fnv1a(const std::string& s) {
  std::uint64_t h = 1469598103934665603ull;
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

const std::vector<std::string>& nvrtc_opts() {
  static const std::vector<std::string> o = {
      "--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo", "--fmad=true",
      "-default-device", "--extra-device-vectorization"};
  return o;
}

std::string pkg_dir() {
  Dl_info info;
  if (dladdr(reinterpret_cast<void*>(&pkg_dir), &info) && info.dli_fname) {
    std::string p = info.dli_fname;
    const auto slash = p.rfind('/');
    if (slash != std::string::npos) return p.substr(0, slash);
  }
  return ".";
}

}  // namespace

std::string nvrtc_options_string() {
  std::string s;
  for (const auto& o : nvrtc_opts()) s += o + " ";
  return s;
}

std::string cache_dir() {
  const char* env = std::getenv("CGF_KCACHE");
  std::string d = env ? env : pkg_dir() + "/_kcache";
  ::mkdir(d.c_str(), 0755);
  return d;
}

std::string compile_cubin(const std::string& source, const std::string& name) {
  int maj = 0, min = 0;
  nvrtcVersion(&maj, &min);
  const std::string key = source + "\n//" + nvrtc_options_string() + std::to_string(maj) + "." + std::to_string(min);
  char hex[32];
  std::snprintf(hex, sizeof hex, "%016llx", static_cast<unsigned long long>(fnv1a(key)));
  const std::string path = cache_dir() + "/" + name + "_" + hex + ".cubin";
  {
    std::ifstream in(path, std::ios::binary);
    if (in) {
      std::stringstream ss;
      ss << in.rdbuf();
      if (!ss.str().empty()) return ss.str();
    }
  }
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, source.c_str(), (name + ".cu").c_str(), 0, nullptr, nullptr) != NVRTC_SUCCESS)
    throw JitError("nvrtcCreateProgram failed");
  std::vector<const char*> opts;
  for (const auto& o : nvrtc_opts()) opts.push_back(o.c_str());
  const nvrtcResult rc = nvrtcCompileProgram(prog, static_cast<int>(opts.size()), opts.data());
  if (rc != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    nvrtcGetProgramLog(prog, log.data());
    nvrtcDestroyProgram(&prog);
    // Keep the failing source next to the cache for inspection.
    std::ofstream(cache_dir() + "/" + name + "_" + hex + ".failed.cu") << source;
    throw JitError("NVRTC compile of " + name + " failed: " + log.substr(0, 4000));
  }
  size_t n = 0;
  nvrtcGetCUBINSize(prog, &n);
  std::string cubin(n, '\0');
  nvrtcGetCUBIN(prog, cubin.data());
  nvrtcDestroyProgram(&prog);
  const std::string tmp = path + ".tmp" + std::to_string(::getpid());
  {
    std::ofstream out(tmp, std::ios::binary);
    out << cubin;
  }
  std::rename(tmp.c_str(), path.c_str());
  return cubin;
}

Kernel load_kernel(const KernelSource& ks) {
  static std::mutex mu;
  static std::map<std::pair<CUcontext, std::string>, Kernel> loaded;
  CUcontext ctx = ensure_context();
  const std::string key = ks.name + "#" + std::to_string(fnv1a(ks.source));
  std::lock_guard<std::mutex> g(mu);
  auto it = loaded.find({ctx, key});
  if (it != loaded.end()) return it->second;
  const std::string cubin = compile_cubin(ks.source, ks.module.empty() ? ks.name : ks.module);
  CUmodule mod;
  CU_CHECK(drv::cuModuleLoadData(&mod, cubin.data()));
  Kernel k;
  CU_CHECK(drv::cuModuleGetFunction(&k.fn, mod, ks.name.c_str()));
  k.threads = ks.threads;
  k.smem_bytes = ks.smem_bytes;
  k.name = ks.name;
  if (ks.smem_bytes > 48 * 1024)
    CU_CHECK(drv::cuFuncSetAttribute(k.fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, ks.smem_bytes));
  int per_sm = 0;
  CU_CHECK(drv::cuOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k.fn, ks.threads, ks.smem_bytes));
  CUdevice dev;
  CU_CHECK(drv::cuCtxGetDevice(&dev));
  int sms = 0;
  CU_CHECK(drv::cuDeviceGetAttribute(&sms, CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT, dev));
  if (per_sm < 1) throw JitError("kernel " + ks.name + " cannot be resident (smem " + std::to_string(ks.smem_bytes) + ")");
  k.max_grid = per_sm * sms;
  loaded.emplace(std::make_pair(ctx, key), k);
  return k;
}

}  // namespace cgf
