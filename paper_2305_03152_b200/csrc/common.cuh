// Shared plumbing for the vipkit_b200 C-ABI library: status codes mapped to
// the reference's exception hierarchy (/root/reference/proj/include/vipkit/
// error.hpp:8-38), a thread-local error message, CUDA error checking and a
// small RAII device buffer.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <utility>

#include "../../include/vipkit_b200.h"

namespace vk {

// One exception type carrying a vk_status; the C-ABI boundary converts it to
// the status code + message (the reference throws typed vipkit::*_error).
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void raise(int code, const std::string& msg) { throw Error(code, msg); }

void set_last_error(const std::string& msg);

template <class F>
int guard(F&& f) {
  try {
    f();
    return VK_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return VK_ERR_INTERNAL;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return VK_ERR_INTERNAL;
  }
}

#define VK_CUDA(expr)                                                                   \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess)                                                              \
      ::vk::raise(VK_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e) +     \
                                   " (" __FILE__ ":" + std::to_string(__LINE__) + ")"); \
  } while (0)

#define VK_LAUNCH_CHECK() VK_CUDA(cudaGetLastError())

// Scoped device switch: the library never leaves the caller's current device
// changed.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    VK_CUDA(cudaGetDevice(&prev));
    if (prev != dev) VK_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
  }
};

// Owning device allocation.
struct DevBuf {
  void* p = nullptr;
  std::size_t bytes = 0;
  DevBuf() = default;
  explicit DevBuf(std::size_t b) { alloc(b); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(std::exchange(o.p, nullptr)), bytes(std::exchange(o.bytes, 0)) {}
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = std::exchange(o.p, nullptr);
      bytes = std::exchange(o.bytes, 0);
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(std::size_t b) {
    release();
    bytes = b;
    if (b) {
      cudaError_t e = cudaMalloc(&p, b);
      if (e != cudaSuccess) {
        p = nullptr;
        bytes = 0;
        raise(VK_ERR_CUDA, "cudaMalloc(" + std::to_string(b) + " B): " + cudaGetErrorString(e));
      }
    }
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// Pinned host staging buffer.
struct PinnedBuf {
  void* p = nullptr;
  std::size_t bytes = 0;
  PinnedBuf() = default;
  PinnedBuf(const PinnedBuf&) = delete;
  PinnedBuf& operator=(const PinnedBuf&) = delete;
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
  void ensure(std::size_t b) {
    if (b <= bytes) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    VK_CUDA(cudaMallocHost(&p, b));
    bytes = b;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

inline unsigned ceil_div(std::uint64_t a, std::uint64_t b) { return static_cast<unsigned>((a + b - 1) / b); }

int sm_count(int device);

}  // namespace vk
