// Microbenchmark: an SpMM-shaped gather through TMA tile::gather4 into shared
// memory.  P is n x 64 fp64; row i of the output sums the 7-point stencil rows
// {i-plane, i-line, i-1, i, i+1, i+line, i+plane} (the pruned C2 operator's
// shape).  One producer warp issues 4-row gathers for tiles of 16 rows into an
// NS-stage ring (mbarrier full/empty); 16 consumer warps each reduce one row
// (2 columns per lane) from shared memory and store it.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 gather4.cu -o gather4
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int KP = 64, ROWB = KP * 8, TR = 16, NE = 7, EPT = TR * NE, NCW = 16;
#ifndef NS
#define NS 3
#endif

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned ph) {
  asm volatile(
      "{\n .reg .pred p;\n W_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(sa(b)),
      "r"(ph)
      : "memory");
}

__global__ void __launch_bounds__(32 * (NCW + 1), 1)
    k_g4(const __grid_constant__ CUtensorMap tm, int n, int line, int plane, double* __restrict__ Q) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[NS], empty[NS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&empty[s])), "r"(NCW));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int ntiles = (n + TR - 1) / TR;
  const int mine = (ntiles - (int)blockIdx.x + gridDim.x - 1) / gridDim.x;
  const int off[NE] = {-plane, -line, -1, 0, 1, line, plane};
  if (warp == 0) {
    if (lane == 0) {
      for (int k = 0; k < mine; ++k) {
        const int s = k % NS;
        if (k >= NS) mbar_wait(&empty[s], ((k / NS) - 1) & 1);
        const int t = blockIdx.x + k * gridDim.x;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])),
                     "r"(EPT * ROWB)
                     : "memory");
        unsigned char* dst = smem + (size_t)s * EPT * ROWB;
        for (int j = 0; j < EPT / 4; ++j) {
          int r[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int e = 4 * j + q, row = t * TR + e / NE;
            int c = row + off[e % NE];
            c = c < 0 ? 0 : (c >= n ? n - 1 : c);
            r[q] = c;
          }
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(sa(dst + (size_t)j * 4 * ROWB)),
              "l"(&tm), "r"(0), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(sa(&full[s]))
              : "memory");
        }
      }
    }
    return;
  }
  const int cw = warp - 1;
  const double w[NE] = {-1.0, -1.0, -1.0, 6.5, -1.0, -1.0, -1.0};
  for (int k = 0; k < mine; ++k) {
    const int s = k % NS;
    mbar_wait(&full[s], (k / NS) & 1);
    const int t = blockIdx.x + k * gridDim.x, row = t * TR + cw;
    const double* st = reinterpret_cast<const double*>(smem + (size_t)s * EPT * ROWB) + (size_t)cw * NE * KP +
                       lane * 2;
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const double2 g = *reinterpret_cast<const double2*>(st + e * KP);
      a0 = fma(w[e], g.x, a0);
      a1 = fma(w[e], g.y, a1);
    }
    if (row < n) *reinterpret_cast<double2*>(Q + (size_t)row * KP + lane * 2) = make_double2(a0, a1);
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[s])) : "memory");
  }
}

// reference: the same stencil with plain gathers, one row per warp
__global__ void k_ref(const double* __restrict__ P, int n, int line, int plane, double* __restrict__ Q) {
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= n) return;
  const int off[NE] = {-plane, -line, -1, 0, 1, line, plane};
  const double w[NE] = {-1.0, -1.0, -1.0, 6.5, -1.0, -1.0, -1.0};
  double a0 = 0.0, a1 = 0.0;
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    int c = row + off[e];
    c = c < 0 ? 0 : (c >= n ? n - 1 : c);
    const double2 g = __ldg(reinterpret_cast<const double2*>(P + (size_t)c * KP + lane * 2));
    a0 = fma(w[e], g.x, a0);
    a1 = fma(w[e], g.y, a1);
  }
  *reinterpret_cast<double2*>(Q + (size_t)row * KP + lane * 2) = make_double2(a0, a1);
}

// CSR-driven gathers, no pipelining, high occupancy: one row per LPR lanes,
// CPL = 64/LPR columns per lane; entries e < 8 held by lane e and shuffled.
template <int LPR>
__global__ void __launch_bounds__(256) k_csr(const int* __restrict__ ip, const int* __restrict__ ix,
                                             const double* __restrict__ va, const double* __restrict__ P,
                                             int n, double* __restrict__ Q) {
  constexpr int CPL = KP / LPR, GB = 8;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int row = gt / LPR, gl = threadIdx.x % LPR;
  const bool ok = row < n;
  int st = 0, ln = 0;
  if (ok) {
    st = __ldg(ip + row);
    ln = __ldg(ip + row + 1) - st;
  }
  int ci = 0;
  double cv = 0.0;
  if (gl < ln) {
    ci = __ldg(ix + st + gl);
    cv = __ldg(va + st + gl);
  }
  double acc[CPL];
#pragma unroll
  for (int k = 0; k < CPL; ++k) acc[k] = 0.0;
  double g[GB][CPL];
#pragma unroll
  for (int e = 0; e < GB; ++e) {
    const int cc = __shfl_sync(0xffffffffu, ci, e, LPR);
    if (e < ln) {
      if constexpr (CPL == 4) {
        asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
            : "=d"(g[e][0]), "=d"(g[e][1]), "=d"(g[e][2]), "=d"(g[e][3])
            : "l"(P + (size_t)cc * KP + gl * CPL));
      } else {
        const double2 t = __ldg(reinterpret_cast<const double2*>(P + (size_t)cc * KP + gl * CPL));
        g[e][0] = t.x;
        g[e][1] = t.y;
      }
    }
  }
#pragma unroll
  for (int e = 0; e < GB; ++e) {
    const double vv = __shfl_sync(0xffffffffu, cv, e, LPR);
    if (e < ln) {
#pragma unroll
      for (int k = 0; k < CPL; ++k) acc[k] = fma(vv, g[e][k], acc[k]);
    }
  }
  if (ok) {
#pragma unroll
    for (int k = 0; k < CPL; ++k) Q[(size_t)row * KP + gl * CPL + k] = acc[k];
  }
}

// ELL (8 slots per row, padded with (row, 0.0)): the gathers depend on one load
// (the row's slot indices), not on indptr -> indices.  One row per warp.
__global__ void __launch_bounds__(256) k_ell(const int* __restrict__ ex, const double* __restrict__ ev,
                                             const double* __restrict__ P, int n, double* __restrict__ Q) {
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= n) return;
  const int ci = __ldg(ex + (size_t)row * 8 + (lane & 7));
  const double cv = __ldg(ev + (size_t)row * 8 + (lane & 7));
  double g[8][2];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int cc = __shfl_sync(0xffffffffu, ci, e);
    const double2 t = __ldg(reinterpret_cast<const double2*>(P + (size_t)cc * KP + lane * 2));
    g[e][0] = t.x;
    g[e][1] = t.y;
  }
  double a0 = 0.0, a1 = 0.0;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const double vv = __shfl_sync(0xffffffffu, cv, e);
    a0 = fma(vv, g[e][0], a0);
    a1 = fma(vv, g[e][1], a1);
  }
  *reinterpret_cast<double2*>(Q + (size_t)row * KP + lane * 2) = make_double2(a0, a1);
}

// the same, persistent, with the next row's slot indices prefetched
__global__ void __launch_bounds__(256) k_ellp(const int* __restrict__ ex, const double* __restrict__ ev,
                                              const double* __restrict__ P, int n, double* __restrict__ Q) {
  const int lane = threadIdx.x & 31;
  const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  int row = w0;
  int ci = 0;
  double cv = 0.0;
  if (row < n) {
    ci = __ldg(ex + (size_t)row * 8 + (lane & 7));
    cv = __ldg(ev + (size_t)row * 8 + (lane & 7));
  }
  for (; row < n; row += nw) {
    const int nx = row + nw;
    int ciN = 0;
    double cvN = 0.0;
    if (nx < n) {
      ciN = __ldg(ex + (size_t)nx * 8 + (lane & 7));
      cvN = __ldg(ev + (size_t)nx * 8 + (lane & 7));
    }
    double g[8][2];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int cc = __shfl_sync(0xffffffffu, ci, e);
      const double2 t = __ldg(reinterpret_cast<const double2*>(P + (size_t)cc * KP + lane * 2));
      g[e][0] = t.x;
      g[e][1] = t.y;
    }
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const double vv = __shfl_sync(0xffffffffu, cv, e);
      a0 = fma(vv, g[e][0], a0);
      a1 = fma(vv, g[e][1], a1);
    }
    *reinterpret_cast<double2*>(Q + (size_t)row * KP + lane * 2) = make_double2(a0, a1);
    ci = ciN;
    cv = cvN;
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int n = 1001184, line = 124, plane = 12000;
  double *P, *Q, *Q2;
  cudaMalloc(&P, (size_t)n * ROWB);
  cudaMalloc(&Q, (size_t)n * ROWB);
  cudaMalloc(&Q2, (size_t)n * ROWB);
  std::vector<double> h((size_t)n * KP);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (double)((i * 2654435761u) % 1000) * 1e-3;
  cudaMemcpy(P, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  if (!enc) {
    printf("no cuTensorMapEncodeTiled\n");
    return 1;
  }
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)KP, (cuuint64_t)n};
  cuuint64_t strides[1] = {(cuuint64_t)ROWB};
  cuuint32_t box[2] = {(cuuint32_t)KP, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, P, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("encode failed %d\n", (int)r);
    return 1;
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t sm = (size_t)NS * EPT * ROWB;
  cudaFuncSetAttribute(k_g4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int it = 0; it < 3; ++it) k_g4<<<sms, 32 * (NCW + 1), sm>>>(tm, n, line, plane, Q);
  k_ref<<<(n * 32 + 255) / 256, 256>>>(P, n, line, plane, Q2);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<double> h1((size_t)n * KP), h2((size_t)n * KP);
  cudaMemcpy(h1.data(), Q, h1.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(h2.data(), Q2, h2.size() * 8, cudaMemcpyDeviceToHost);
  size_t bad = 0;
  for (size_t i = 0; i < h1.size(); ++i) bad += h1[i] != h2[i];
  const int R = 20;
  cudaEventRecord(a);
  for (int it = 0; it < R; ++it) k_g4<<<sms, 32 * (NCW + 1), sm>>>(tm, n, line, plane, Q);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventRecord(a);
  for (int it = 0; it < R; ++it) k_ref<<<(n * 32 + 255) / 256, 256>>>(P, n, line, plane, Q2);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms2 = 0;
  cudaEventElapsedTime(&ms2, a, b);
  // CSR of the same stencil (duplicates from clamping kept)
  std::vector<int> hip(n + 1), hix((size_t)n * NE);
  std::vector<double> hva((size_t)n * NE);
  {
    const int offs[NE] = {-plane, -line, -1, 0, 1, line, plane};
    const double ws[NE] = {-1.0, -1.0, -1.0, 6.5, -1.0, -1.0, -1.0};
    for (int i = 0; i < n; ++i) {
      hip[i] = i * NE;
      for (int e = 0; e < NE; ++e) {
        int c = i + offs[e];
        c = c < 0 ? 0 : (c >= n ? n - 1 : c);
        hix[(size_t)i * NE + e] = c;
        hva[(size_t)i * NE + e] = ws[e];
      }
    }
    hip[n] = n * NE;
  }
  int *dip, *dix;
  double* dva;
  cudaMalloc(&dip, hip.size() * 4);
  cudaMalloc(&dix, hix.size() * 4);
  cudaMalloc(&dva, hva.size() * 8);
  cudaMemcpy(dip, hip.data(), hip.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dix, hix.data(), hix.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dva, hva.data(), hva.size() * 8, cudaMemcpyHostToDevice);
  float msc[2];
  size_t badc[2];
  for (int v = 0; v < 2; ++v) {
    auto run = [&]() {
      if (v == 0) k_csr<32><<<(n * 32 + 255) / 256, 256>>>(dip, dix, dva, P, n, Q);
      else k_csr<16><<<(n * 16 + 255) / 256, 256>>>(dip, dix, dva, P, n, Q);
    };
    run();
    cudaDeviceSynchronize();
    cudaMemcpy(h1.data(), Q, h1.size() * 8, cudaMemcpyDeviceToHost);
    badc[v] = 0;
    for (size_t i = 0; i < h1.size(); ++i) badc[v] += h1[i] != h2[i];
    cudaEventRecord(a);
    for (int it = 0; it < R; ++it) run();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&msc[v], a, b);
  }
  {
    std::vector<int> ex((size_t)n * 8);
    std::vector<double> ev((size_t)n * 8);
    for (int i = 0; i < n; ++i)
      for (int e = 0; e < 8; ++e) {
        ex[(size_t)i * 8 + e] = e < NE ? hix[(size_t)i * NE + e] : i;
        ev[(size_t)i * 8 + e] = e < NE ? hva[(size_t)i * NE + e] : 0.0;
      }
    int* dex;
    double* dev_;
    cudaMalloc(&dex, ex.size() * 4);
    cudaMalloc(&dev_, ev.size() * 8);
    cudaMemcpy(dex, ex.data(), ex.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dev_, ev.data(), ev.size() * 8, cudaMemcpyHostToDevice);
    for (int v = 0; v < 3; ++v) {
      auto run = [&]() {
        if (v == 0) k_ell<<<(n * 32 + 255) / 256, 256>>>(dex, dev_, P, n, Q);
        else if (v == 1) k_ellp<<<sms * 8, 256>>>(dex, dev_, P, n, Q);
        else k_ellp<<<sms * 6, 256>>>(dex, dev_, P, n, Q);
      };
      run();
      cudaDeviceSynchronize();
      cudaMemcpy(h1.data(), Q, h1.size() * 8, cudaMemcpyDeviceToHost);
      size_t bad2 = 0;
      for (size_t i = 0; i < h1.size(); ++i) bad2 += h1[i] != h2[i];
      cudaEventRecord(a);
      for (int it = 0; it < R; ++it) run();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float m = 0;
      cudaEventElapsedTime(&m, a, b);
      printf("ell variant %d: %.4f ms (mismatch %zu)\n", v, m / R, bad2);
    }
  }
  printf("csr LPR=32: %.4f ms (mismatch %zu)  csr LPR=16: %.4f ms (mismatch %zu)\n", msc[0] / R, badc[0],
         msc[1] / R, badc[1]);
  printf("NS=%d gather4 %.4f ms  plain-gather %.4f ms  mismatches %zu  (algorithmic %.2f GB moved)\n", NS, ms / R,
         ms2 / R, bad, 16.0 * n * KP / 1e9);
  return 0;
}
