// ABI plumbing: error reporting, version, device queries, and the
// deterministic int32 exclusive scan used by the CSR builders.
#include <stdarg.h>
#include <stdio.h>

#include <atomic>

#include "common.cuh"

namespace hf {

static thread_local char g_err[1024] = "";
static std::atomic<long> g_launches{0};

void count_launches(long k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

// ---------------------------------------------------------------- scan
constexpr int SCAN_T = 1024;
constexpr int SCAN_PER = 4;
constexpr int SCAN_TILE = SCAN_T * SCAN_PER;

__device__ __forceinline__ int32_t block_incl_scan(int32_t v, int32_t* sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    int32_t t = __shfl_up_sync(FULL, v, off);
    if (lane >= off) v += t;
  }
  if (lane == 31) sm[warp] = v;
  __syncthreads();
  if (warp == 0) {
    int32_t w = (lane < (int)(blockDim.x >> 5)) ? sm[lane] : 0;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      int32_t t = __shfl_up_sync(FULL, w, off);
      if (lane >= off) w += t;
    }
    sm[lane] = w;
  }
  __syncthreads();
  if (warp > 0) v += sm[warp - 1];
  __syncthreads();
  return v;
}

// Phase 1: per-tile exclusive scan, tile sums into bsum.
// In-place safe (in == out): each thread reads its own elements before writing them.
__global__ void __launch_bounds__(SCAN_T) k_scan_tiles(const int32_t* in, int32_t* out, int n,
                                                       int32_t* __restrict__ bsum) {
  __shared__ int32_t sm[32];
  const size_t base = (size_t)blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_PER;
  int32_t v[SCAN_PER];
  int32_t s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_PER; ++k) {
    v[k] = (base + k < (size_t)n) ? in[base + k] : 0;
    s += v[k];
  }
  const int32_t incl = block_incl_scan(s, sm);
  int32_t run = incl - s;
#pragma unroll
  for (int k = 0; k < SCAN_PER; ++k) {
    if (base + k < (size_t)n) out[base + k] = run;
    run += v[k];
  }
  if (threadIdx.x == blockDim.x - 1) bsum[blockIdx.x] = incl;
}

// Phase 2: scan the tile sums (nb <= SCAN_TILE), write the grand total.
__global__ void __launch_bounds__(SCAN_T) k_scan_sums(int32_t* bsum, int nb, int32_t* total) {
  __shared__ int32_t sm[32];
  const int base = threadIdx.x * SCAN_PER;
  int32_t v[SCAN_PER];
  int32_t s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_PER; ++k) {
    v[k] = (base + k < nb) ? bsum[base + k] : 0;
    s += v[k];
  }
  const int32_t incl = block_incl_scan(s, sm);
  int32_t run = incl - s;
#pragma unroll
  for (int k = 0; k < SCAN_PER; ++k) {
    if (base + k < nb) bsum[base + k] = run;
    run += v[k];
  }
  if (threadIdx.x == blockDim.x - 1) *total = incl;
}

__global__ void k_scan_add(int32_t* out, int n, const int32_t* __restrict__ bsum) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < (size_t)n) out[i] += bsum[i / SCAN_TILE];
}

size_t scan_scratch_elems(int32_t n) {
  const size_t nb = ((size_t)n + SCAN_TILE - 1) / SCAN_TILE;
  return nb + (nb > (size_t)SCAN_TILE ? scan_scratch_elems((int32_t)nb) : 32);
}

// Exclusive scan of any int32 length: tile scan, recursive scan of the tile sums
// (in place, next level's sums after them), then add-back.  Fixed order, so the
// result is deterministic.
int exclusive_scan_i32(const int32_t* in, int32_t* out, int32_t n, int32_t* block_sums,
                       int32_t* total_dev, cudaStream_t s) {
  if (n <= 0) {
    HF_CUDA(cudaMemsetAsync(total_dev, 0, sizeof(int32_t), s));
    return HF_OK;
  }
  const int nb = (n + SCAN_TILE - 1) / SCAN_TILE;
  count_launches(1);
  k_scan_tiles<<<nb, SCAN_T, 0, s>>>(in, out, n, block_sums);
  if (nb > SCAN_TILE) {
    int rc = exclusive_scan_i32(block_sums, block_sums, nb, block_sums + nb, total_dev, s);
    if (rc) return rc;
  } else {
    count_launches(1);
    k_scan_sums<<<1, SCAN_T, 0, s>>>(block_sums, nb, total_dev);
  }
  if (nb > 1) {
    count_launches(1);
    k_scan_add<<<(n + 255) / 256, 256, 0, s>>>(out, n, block_sums);
  }
  HF_LAUNCH_CHECK();
  return HF_OK;
}

}  // namespace hf

extern "C" const char* hf_version(void) { return "hfb200 0.1.0 (sm_100a)"; }

extern "C" const char* hf_last_error(void) { return hf::g_err; }

extern "C" long long hf_launch_count(void) { return hf::g_launches.load(); }

extern "C" int hf_device_sm_count(int32_t* out) {
  if (!out) return HF_ERR_ARG;
  int dev = 0, v = 0;
  HF_CUDA(cudaGetDevice(&dev));
  HF_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
  *out = v;
  return HF_OK;
}

extern "C" size_t hf_scan_workspace_bytes(int32_t n) {
  return hf::scan_scratch_elems(n < 0 ? 0 : n) * sizeof(int32_t);
}

extern "C" int hf_exclusive_scan_i32(const int32_t* in, int32_t* out, int32_t n, int32_t* total,
                                     void* ws, size_t ws_bytes, void* stream) {
  if (n < 0 || !total || (n > 0 && (!in || !out || !ws))) {
    hf::set_error("hf_exclusive_scan_i32: bad argument");
    return HF_ERR_ARG;
  }
  if (ws_bytes < hf_scan_workspace_bytes(n)) {
    hf::set_error("scan workspace too small");
    return HF_ERR_WORKSPACE;
  }
  return hf::exclusive_scan_i32(in, out, n, reinterpret_cast<int32_t*>(ws), total,
                                reinterpret_cast<cudaStream_t>(stream));
}
