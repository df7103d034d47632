// Microbenchmark: throughput of cp.async.bulk (TMA 1D) row-range copies into
// shared memory with S stages in flight per block, for a band-local access
// pattern like the SpMM's (5 ranges of ~16 rows of 512 B around a moving row).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void mbar_init(uint64_t* b, int c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned phase) {
  asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" :: "r"((unsigned)__cvta_generic_to_shared(b)), "r"(phase) : "memory");
}

template <int S>
__global__ void __launch_bounds__(256, 1) k(const double* __restrict__ V, int n, int ntiles, int plane, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  double* buf = reinterpret_cast<double*>(sm + 128);
  const int ROWB = 512, TR = 16, W = 96;  // 96 rows per stage
  if (threadIdx.x == 0) { for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  auto issue = [&](int i, int s) {
    int t = blockIdx.x + i * gridDim.x;
    if (t >= ntiles) return;
    long r0 = (long)t * TR;
    long starts[5] = {r0 - 1, r0 - 123, r0 + 123, r0 - plane, r0 + plane};
    int lens[5] = {18, 16, 16, 16, 16};
    mbar_expect(&bar[s], 82 * ROWB);
    int off = 0;
    for (int q = 0; q < 5; ++q) {
      long st = starts[q]; if (st < 0) st = 0; if (st + lens[q] > n) st = n - lens[q];
      bulk_g2s(buf + (size_t)s * W * 64 + off * 64, V + st * 64, lens[q] * ROWB, &bar[s]);
      off += lens[q];
    }
  };
  int nmine = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
  if (threadIdx.x == 0) for (int s = 0; s < S - 1 && s < nmine; ++s) issue(s, s);
  double acc = 0;
  for (int i = 0; i < nmine; ++i) {
    int s = i % S;
    if (threadIdx.x == 0 && i + S - 1 < nmine) issue(i + S - 1, (i + S - 1) % S);
    mbar_wait(&bar[s], (i / S) & 1);
    // consume: each thread reads a few doubles
    const double* b = buf + (size_t)s * W * 64;
    for (int e = threadIdx.x; e < 82 * 64; e += 256 * 8) acc += b[e];
    __syncthreads();
  }
  if (acc == 12345.0) out[0] = acc;
}

int main() {
  const int n = 1001184, plane = 15200;
  double* V; cudaMalloc(&V, (size_t)n * 64 * 8); cudaMemset(V, 0, (size_t)n * 64 * 8);
  double* out; cudaMalloc(&out, 8);
  int ntiles = n / 16 - 2000;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
#define RUN(S) { size_t smem = 128 + (size_t)S * 96 * 512; cudaFuncSetAttribute(k<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
  for (int bps = 1; bps <= 2; ++bps) { if (smem * bps > 227 * 1024) continue; int g = sms * bps; \
    k<S><<<g, 256, smem>>>(V, n, ntiles, plane, out); cudaEventRecord(a); for (int r = 0; r < 5; ++r) k<S><<<g, 256, smem>>>(V, n, ntiles, plane, out); cudaEventRecord(b); cudaEventSynchronize(b); \
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5; double bytes = (double)ntiles * 82 * 512; \
    printf("S=%d blocks/SM=%d: %.3f ms  %.1f TB/s into smem (%s)\n", S, bps, ms, bytes / ms / 1e9, cudaGetErrorString(cudaGetLastError())); } }
  RUN(1) RUN(2) RUN(3) RUN(4)
  return 0;
}
