// Shared helpers for the libmfg_b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <atomic>
#include <string>

#include "../../include/mfg_b200.h"

namespace mfg {

void set_error(const std::string& msg);
extern std::atomic<int64_t> g_launches;

#define MFG_CUDA_CHECK(expr)                                                   \
  do {                                                                         \
    cudaError_t _e = (expr);                                                   \
    if (_e != cudaSuccess) {                                                   \
      ::mfg::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));    \
      return MFG_ERR_CUDA;                                                     \
    }                                                                          \
  } while (0)

// Check the most recent launch and count it.
#define MFG_LAUNCH_CHECK()                                                     \
  do {                                                                         \
    ::mfg::g_launches.fetch_add(1, std::memory_order_relaxed);                 \
    cudaError_t _e = cudaGetLastError();                                       \
    if (_e != cudaSuccess) {                                                   \
      ::mfg::set_error(std::string("kernel launch: ") + cudaGetErrorString(_e)); \
      return MFG_ERR_CUDA;                                                     \
    }                                                                          \
  } while (0)

#define MFG_REQUIRE(cond, msg)                                                 \
  do {                                                                         \
    if (!(cond)) {                                                             \
      ::mfg::set_error(msg);                                                   \
      return MFG_ERR_ARG;                                                      \
    }                                                                          \
  } while (0)

constexpr int kWarp = 32;
constexpr int kNumSMs = 148;

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// Bump allocator over a caller-provided workspace.
struct Carver {
  char* base;
  size_t cap;
  size_t off = 0;
  bool ok = true;
  Carver(void* b, size_t c) : base(static_cast<char*>(b)), cap(c) {}
  template <typename T>
  T* take(size_t count) {
    size_t bytes = align_up(count * sizeof(T));
    if (off + bytes > cap) {
      ok = false;
      return nullptr;
    }
    T* p = reinterpret_cast<T*>(base + off);
    off += bytes;
    return p;
  }
};

// Size-only twin of Carver for the *_workspace queries.
struct Sizer {
  size_t off = 0;
  template <typename T>
  T* take(size_t count) {
    off += align_up(count * sizeof(T));
    return nullptr;
  }
};

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

template <typename T>
__device__ __forceinline__ T shfl_xor(T v, int m) {
  return __shfl_xor_sync(0xffffffffu, v, m);
}

// Deterministic fp64 block reduction (fixed tree); result valid in thread 0.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* smem) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) smem[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NT / 32; ++i) s += smem[i];
  }
  __syncthreads();
  return s;
}

}  // namespace mfg
