// Shared helpers for the hfb200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/hfb200.h"

namespace hf {

void set_error(const char* fmt, ...);

// Number of kernels this library has launched (graph launches count their
// kernel nodes); bench.py reports it as gpu_launches.
void count_launches(long k);

#define HF_CUDA(x)                                                                    \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      ::hf::set_error("%s: %s (%s:%d)", #x, cudaGetErrorString(e_), __FILE__, __LINE__); \
      return HF_ERR_CUDA;                                                             \
    }                                                                                 \
  } while (0)

#define HF_LAUNCH_CHECK()                                                             \
  do {                                                                                \
    cudaError_t e_ = cudaGetLastError();                                              \
    if (e_ != cudaSuccess) {                                                          \
      ::hf::set_error("kernel launch: %s (%s:%d)", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return HF_ERR_CUDA;                                                             \
    }                                                                                 \
  } while (0)

constexpr unsigned FULL = 0xffffffffu;

inline int sm_count() {
  static int cached = 0;
  if (!cached) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
    if (cached <= 0) cached = 148;
  }
  return cached;
}

// Bump allocator over a caller-provided workspace (256-byte aligned slices).
struct Carve {
  char* base;
  size_t used;
  size_t cap;
  template <typename T>
  T* take(size_t count) {
    size_t off = (used + 255) & ~size_t(255);
    used = off + count * sizeof(T);
    return reinterpret_cast<T*>(base + off);
  }
  bool ok() const { return used <= cap; }
};

// Loads that bypass L1: data written by other SMs inside the same launch
// (last-block reductions read every block's partials).
__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }

// Exclusive scan over int32 counts into int32 offsets (3-phase, deterministic).
int exclusive_scan_i32(const int32_t* in, int32_t* out, int32_t n, int32_t* block_sums,
                       int32_t* total_dev, cudaStream_t s);
size_t scan_scratch_elems(int32_t n);

}  // namespace hf
