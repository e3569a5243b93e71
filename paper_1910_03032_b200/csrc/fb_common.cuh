// Shared helpers for the fbb200 library: status handling, launch counting,
// device buffers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>
#include <vector>

#include "../../include/fbb200.h"

namespace fb {

void set_error(const std::string& msg);
int64_t& launch_counter();

inline void count_launch() { ++launch_counter(); }

#define FB_TRY_CUDA(expr)                                                              \
  do {                                                                                 \
    cudaError_t _e = (expr);                                                           \
    if (_e != cudaSuccess) {                                                           \
      ::fb::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));             \
      return (_e == cudaErrorMemoryAllocation) ? FB_ERR_OOM : FB_ERR_CUDA;             \
    }                                                                                  \
  } while (0)

bool debug_sync();  // FB_DEBUG_SYNC=1: synchronise and check after every launch
void debug_canary_register(const int* dev_ptr, int n);
void debug_canary_unregister(const int* dev_ptr);
bool debug_canary_check(const char* where);

#define FB_CHECK_LAUNCH()                                                              \
  do {                                                                                 \
    ::fb::count_launch();                                                              \
    cudaError_t _e = cudaGetLastError();                                               \
    if (_e == cudaSuccess && ::fb::debug_sync()) {                                     \
      _e = cudaDeviceSynchronize();                                                    \
      if (_e == cudaSuccess)                                                           \
        ::fb::debug_canary_check((std::string(__FILE__) + ":" + std::to_string(__LINE__)).c_str()); \
    }                                                                                  \
    if (_e != cudaSuccess) {                                                           \
      ::fb::set_error(std::string("kernel launch (") + __FILE__ + ":" +               \
                      std::to_string(__LINE__) + "): " + cudaGetErrorString(_e));      \
      return FB_ERR_CUDA;                                                              \
    }                                                                                  \
  } while (0)

#define FB_REQUIRE(cond, msg)                                                          \
  do {                                                                                 \
    if (!(cond)) {                                                                     \
      ::fb::set_error(msg);                                                            \
      return FB_ERR_ARG;                                                               \
    }                                                                                  \
  } while (0)

// Owning device buffer.
template <typename T>
struct DevBuf {
  T* ptr = nullptr;
  int64_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { reset(); }
  void reset() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    n = 0;
  }
  // Allocates n elements plus `pad_bytes` of slack (bulk L2 prefetches may
  // round a range up to 16 bytes).
  cudaError_t alloc(int64_t count, size_t pad_bytes = 256) {
    reset();
    n = count;
    if (count == 0) return cudaSuccess;
    return cudaMalloc(reinterpret_cast<void**>(&ptr), size_t(count) * sizeof(T) + pad_bytes);
  }
  cudaError_t upload(const T* host, int64_t count) {
    cudaError_t e = alloc(count);
    if (e != cudaSuccess || count == 0) return e;
    return cudaMemcpy(ptr, host, size_t(count) * sizeof(T), cudaMemcpyHostToDevice);
  }
  size_t bytes() const { return size_t(n) * sizeof(T); }
};

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline int ceil_div(int64_t a, int64_t b) { return int((a + b - 1) / b); }

}  // namespace fb
