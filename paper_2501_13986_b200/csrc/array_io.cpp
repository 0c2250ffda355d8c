// The reference's array files (array_io.cpp:15-68): raw little-endian values
// in <base>.bin plus a JSON sidecar <base>.json = {"cols":C,"dtype":"fp32"|
// "fp64","rows":R} — the inputs / outputs of its CLI's compile / verify /
// bench workflow. Here for host buffers and, streamed through pinned staging in
// 64 MB pieces, straight into device memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <cctype>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>

#include "../../include/cgf.h"
#include "problem.hpp"

namespace {

const char* dname(int dtype) { return dtype == CGF_F64 ? "fp64" : "fp32"; }
std::size_t esize(int dtype) { return dtype == CGF_F64 ? 8 : 4; }

void check_dtype(int dtype) {
  if (dtype != CGF_F32 && dtype != CGF_F64) throw std::invalid_argument("bad dtype");
}

struct Meta {
  std::int64_t rows = 0, cols = 0;
  std::string dtype;
};

// The sidecar is one small JSON object; read its three keys.
Meta read_meta(const std::string& base) {
  std::ifstream in(base + ".json");
  if (!in) throw std::runtime_error("cannot read " + base + ".json");
  std::stringstream ss;
  ss << in.rdbuf();
  const std::string t = ss.str();
  auto field = [&](const char* key) -> std::string {
    const std::string k = std::string("\"") + key + "\"";
    std::size_t p = t.find(k);
    if (p == std::string::npos) throw cgf::ParseError(base + ".json: missing key " + k);
    p = t.find(':', p + k.size());
    if (p == std::string::npos) throw cgf::ParseError(base + ".json: malformed");
    ++p;
    while (p < t.size() && (t[p] == ' ' || t[p] == '\t' || t[p] == '\n' || t[p] == '\r')) ++p;
    std::size_t e = p;
    if (p < t.size() && t[p] == '"') {
      e = t.find('"', p + 1);
      if (e == std::string::npos) throw cgf::ParseError(base + ".json: malformed");
      return t.substr(p + 1, e - p - 1);
    }
    while (e < t.size() && (std::isdigit(static_cast<unsigned char>(t[e])) || t[e] == '-')) ++e;
    return t.substr(p, e - p);
  };
  Meta m;
  try {
    m.rows = std::stoll(field("rows"));
    m.cols = std::stoll(field("cols"));
  } catch (const std::logic_error&) {
    throw cgf::ParseError(base + ".json: rows / cols must be integers");
  }
  m.dtype = field("dtype");
  return m;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return CGF_OK;
  } catch (const cgf::ParseError& e) {
    cgf::set_last_error(e.what());
    return CGF_E_PARSE;
  } catch (const cgf::ShapeError& e) {
    cgf::set_last_error(e.what());
    return CGF_E_SHAPE;
  } catch (const cgf::CudaError& e) {
    cgf::set_last_error(e.what());
    return CGF_E_CUDA;
  } catch (const std::invalid_argument& e) {
    cgf::set_last_error(e.what());
    return CGF_E_INVALID;
  } catch (const std::exception& e) {
    cgf::set_last_error(e.what());
    return CGF_E_INTERNAL;
  }
}

void cuda_check(cudaError_t r, const char* what) {
  if (r != cudaSuccess) throw cgf::CudaError(std::string(what) + ": " + cudaGetErrorString(r));
}

}  // namespace

extern "C" {

int cgf_array_save(const char* base, int dtype, const void* data, int64_t rows, int64_t cols) {
  return guarded([&] {
    check_dtype(dtype);
    if (!base || (rows * cols > 0 && !data)) throw std::invalid_argument("null pointer");
    if (rows < 0 || cols < 0) throw cgf::ShapeError("negative array shape");
    const std::string b = base;
    std::ofstream bin(b + ".bin", std::ios::binary);
    if (!bin) throw std::runtime_error("cannot write " + b + ".bin");
    bin.write(static_cast<const char*>(data), static_cast<std::streamsize>(esize(dtype) * rows * cols));
    std::ofstream meta(b + ".json");
    if (!meta) throw std::runtime_error("cannot write " + b + ".json");
    meta << "{\"cols\":" << cols << ",\"dtype\":\"" << dname(dtype) << "\",\"rows\":" << rows << "}\n";
  });
}

int cgf_array_meta(const char* base, int64_t shape[2], int* dtype) {
  return guarded([&] {
    if (!base || !shape || !dtype) throw std::invalid_argument("null pointer");
    const Meta m = read_meta(base);
    if (m.dtype != "fp32" && m.dtype != "fp64") throw cgf::ParseError(std::string(base) + ".json: unknown dtype " + m.dtype);
    shape[0] = m.rows;
    shape[1] = m.cols;
    *dtype = m.dtype == "fp64" ? CGF_F64 : CGF_F32;
  });
}

// Loads into a host buffer of `capacity` elements, or (device != 0) into a
// device buffer through pinned staging; the file's dtype must be `dtype`.
int cgf_array_load(const char* base, int dtype, void* dst, int64_t capacity, int device, void* stream) {
  return guarded([&] {
    check_dtype(dtype);
    if (!base) throw std::invalid_argument("null pointer");
    const std::string b = base;
    const Meta m = read_meta(b);
    if (m.dtype != dname(dtype))
      throw std::runtime_error(b + ": dtype is " + m.dtype + ", expected " + dname(dtype));
    const std::int64_t n = m.rows * m.cols;
    if (n > capacity) throw cgf::ShapeError(b + ": " + std::to_string(n) + " elements exceed the buffer's " +
                                            std::to_string(capacity));
    if (n > 0 && !dst) throw std::invalid_argument("null pointer");
    std::ifstream bin(b + ".bin", std::ios::binary);
    if (!bin) throw std::runtime_error("cannot read " + b + ".bin");
    const std::size_t bytes = esize(dtype) * static_cast<std::size_t>(n);
    if (!device) {
      bin.read(static_cast<char*>(dst), static_cast<std::streamsize>(bytes));
      if (bin.gcount() != static_cast<std::streamsize>(bytes))
        throw std::runtime_error(b + ".bin: file shorter than the sidecar promises");
      return;
    }
    // device: double-buffered pinned pieces, the read of piece i+1 overlapping the copy of piece i
    const std::size_t piece = 64ull << 20;
    void* pin[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    struct Free {
      void** p; cudaEvent_t* e;
      ~Free() { for (int i = 0; i < 2; ++i) { if (p[i]) cudaFreeHost(p[i]); if (e[i]) cudaEventDestroy(e[i]); } }
    } guard{pin, done};
    for (int i = 0; i < 2; ++i) {
      cuda_check(cudaMallocHost(&pin[i], piece), "cudaMallocHost");
      cuda_check(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming), "cudaEventCreate");
    }
    std::size_t off = 0;
    for (int i = 0; off < bytes; i ^= 1) {
      const std::size_t k = std::min(piece, bytes - off);
      cuda_check(cudaEventSynchronize(done[i]), "cudaEventSynchronize");  // the piece's last copy finished
      bin.read(static_cast<char*>(pin[i]), static_cast<std::streamsize>(k));
      if (bin.gcount() != static_cast<std::streamsize>(k))
        throw std::runtime_error(b + ".bin: file shorter than the sidecar promises");
      cuda_check(cudaMemcpyAsync(static_cast<char*>(dst) + off, pin[i], k, cudaMemcpyHostToDevice, st), "cudaMemcpyAsync");
      cuda_check(cudaEventRecord(done[i], st), "cudaEventRecord");
      off += k;
    }
    cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
  });
}

}  // extern "C"
