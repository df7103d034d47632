// Post-solve lead-field kernels for sm_100a (leadfield.py:104-237).
//
//   k_bt_t           raw response block C - B'T[:, cols]       (leadfield.py:107)
//   k_lf_tile        LF tile = W (G'T)'_tile  — the (G'T)' tile is gathered
//                    from T rows into shared memory (<= 8 nonzeros per source
//                    column), then multiplied by W = -R M^-1 on the fp64 tensor
//                    path (DMMA: mma.sync.m8n8k4.f64).   (leadfield.py:128-129)
//   k_eit_sens       per-DOF sensitivities Q[p, m, :] = T' K_m u_p  (leadfield.py:179-207)
#include "common.cuh"

namespace hf {
namespace tail {

// ---------------------------------------------------------------- response
__global__ void k_bt_t(int L, int col0, int ncols, const int32_t* __restrict__ ptr,
                       const int32_t* __restrict__ idx, const double* __restrict__ val,
                       const double* __restrict__ T, int ldt, const double* __restrict__ Cdiag,
                       double* __restrict__ Mraw) {
  const int l = blockIdx.x;
  for (int c = threadIdx.x; c < ncols; c += blockDim.x) {
    double acc = 0.0;  // (B'T)[l, c], ascending node order as csc_matvecs
    for (int q = ptr[l]; q < ptr[l + 1]; ++q) acc += val[q] * T[(size_t)idx[q] * ldt + c];
    const double cl = (l == col0 + c) ? Cdiag[l] : 0.0;
    Mraw[(size_t)l * ncols + c] = cl - acc;
  }
}

// ---------------------------------------------------------------- DMMA tile GEMM
constexpr int LF_THREADS = 256;
constexpr int LF_NC = 32;  // source columns per CTA
constexpr int LF_SBS = LF_NC + 4;  // smem row stride: conflict-free B fragments

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// MODE 0: B-operand tile gathered from T through G' (CSR, row c = source column c).
// MODE 1: B-operand tile read from dense Qc (ncols x L row-major).
// Output out[l * ldo + c] for l < L, c < ncols.
template <int MODE>
__global__ void __launch_bounds__(LF_THREADS)
    k_lf_tile(int L, int K, int Kp, int ncols, const double* __restrict__ T, int ldt,
              const int32_t* __restrict__ gptr, const int32_t* __restrict__ gidx,
              const double* __restrict__ gval, const double* __restrict__ Qc,
              const double* __restrict__ W, int ldw, double* __restrict__ out, int ldo) {
  extern __shared__ double sB[];  // [Kp][LF_SBS]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c0 = blockIdx.x * LF_NC;
  // phase 1: B tile
  for (int o = tid; o < Kp * LF_NC; o += LF_THREADS) {
    const int k = o % Kp, cc = o / Kp, c = c0 + cc;
    double acc = 0.0;
    if (k < K && c < ncols) {
      if (MODE == 0) {
        for (int q = gptr[c]; q < gptr[c + 1]; ++q)
          acc += __ldg(gval + q) * __ldg(T + (size_t)__ldg(gidx + q) * ldt + k);
      } else {
        acc = __ldg(Qc + (size_t)c * K + k);
      }
    }
    sB[k * LF_SBS + cc] = acc;
  }
  __syncthreads();
  // phase 2: out tile (L x LF_NC) = W (L x K) * sB (K x LF_NC); warp owns row
  // blocks rb = warp, warp+8, ... and all LF_NC/8 column blocks.
  const int g = lane >> 2, t4 = lane & 3;
  const int nrb = (L + 7) / 8;
  for (int rb = warp; rb < nrb; rb += LF_THREADS / 32) {
    double d[LF_NC / 8][2];
#pragma unroll
    for (int j = 0; j < LF_NC / 8; ++j) d[j][0] = d[j][1] = 0.0;
    const int row = rb * 8 + g;
    const double* wrow = W + (size_t)row * ldw;
    for (int k0 = 0; k0 < Kp; k0 += 4) {
      const int kk = k0 + t4;
      const double a = (row < L && kk < K) ? __ldg(wrow + kk) : 0.0;
#pragma unroll
      for (int j = 0; j < LF_NC / 8; ++j) {
        const double b = sB[kk * LF_SBS + j * 8 + g];
        dmma_8x8x4(d[j][0], d[j][1], a, b);
      }
    }
#pragma unroll
    for (int j = 0; j < LF_NC / 8; ++j) {
      const int c = c0 + j * 8 + t4 * 2;
      if (row < L) {
        if (c < ncols) out[(size_t)row * ldo + c] = d[j][0];
        if (c + 1 < ncols) out[(size_t)row * ldo + c + 1] = d[j][1];
      }
    }
  }
}

// ---------------------------------------------------------------- EIT sensitivities
constexpr int ES_THREADS = 256;
constexpr int ES_EB = 8;         // elements staged per batch
constexpr int ES_MAXO = 16;      // outputs per thread per CTA (P*L chunk <= 4096)
constexpr int ES_CHUNK = ES_THREADS * ES_MAXO;

#define MUL(a, b) __dmul_rn((a), (b))
#define ADD(a, b) __dadd_rn((a), (b))
#define SUB(a, b) __dsub_rn((a), (b))

// unit-sigma block of an element with grounded rows/cols zeroed
// (leadfield.py:189-196); same explicitly rounded arithmetic as hf_p1_blocks.
__device__ void unit_block(const double* __restrict__ nodes, const int32_t* __restrict__ conn,
                           int ground, double K[16]) {
  double p[4][3];
  for (int a = 0; a < 4; ++a)
    for (int r = 0; r < 3; ++r) p[a][r] = nodes[3 * (size_t)conn[a] + r];
  double J[3][3];
  for (int r = 0; r < 3; ++r)
    for (int k = 0; k < 3; ++k) J[r][k] = SUB(p[k + 1][r], p[0][r]);
  const double c0 = SUB(MUL(J[1][1], J[2][2]), MUL(J[1][2], J[2][1]));
  const double c1 = SUB(MUL(J[1][0], J[2][2]), MUL(J[1][2], J[2][0]));
  const double c2 = SUB(MUL(J[1][0], J[2][1]), MUL(J[1][1], J[2][0]));
  const double det = ADD(SUB(MUL(J[0][0], c0), MUL(J[0][1], c1)), MUL(J[0][2], c2));
  const double vol = __ddiv_rn(det, 6.0);
  double g[4][3];
  g[1][0] = __ddiv_rn(SUB(MUL(J[1][1], J[2][2]), MUL(J[1][2], J[2][1])), det);
  g[1][1] = __ddiv_rn(SUB(MUL(J[0][2], J[2][1]), MUL(J[0][1], J[2][2])), det);
  g[1][2] = __ddiv_rn(SUB(MUL(J[0][1], J[1][2]), MUL(J[0][2], J[1][1])), det);
  g[2][0] = __ddiv_rn(SUB(MUL(J[1][2], J[2][0]), MUL(J[1][0], J[2][2])), det);
  g[2][1] = __ddiv_rn(SUB(MUL(J[0][0], J[2][2]), MUL(J[0][2], J[2][0])), det);
  g[2][2] = __ddiv_rn(SUB(MUL(J[0][2], J[1][0]), MUL(J[0][0], J[1][2])), det);
  g[3][0] = __ddiv_rn(SUB(MUL(J[1][0], J[2][1]), MUL(J[1][1], J[2][0])), det);
  g[3][1] = __ddiv_rn(SUB(MUL(J[0][1], J[2][0]), MUL(J[0][0], J[2][1])), det);
  g[3][2] = __ddiv_rn(SUB(MUL(J[0][0], J[1][1]), MUL(J[0][1], J[1][0])), det);
  for (int k = 0; k < 3; ++k) g[0][k] = -ADD(ADD(g[1][k], g[2][k]), g[3][k]);
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      double v = MUL(ADD(ADD(MUL(g[i][0], g[j][0]), MUL(g[i][1], g[j][1])), MUL(g[i][2], g[j][2])), vol);
      if (conn[i] == ground || conn[j] == ground) v = 0.0;
      K[4 * i + j] = v;
    }
}

__global__ void __launch_bounds__(ES_THREADS)
    k_eit_sens(const double* __restrict__ nodes, const int32_t* __restrict__ tetra,
               const int32_t* __restrict__ dof_elems, const int32_t* __restrict__ dof_ptr,
               int n_dofs, int ground, const double* __restrict__ T, int ldt, int L,
               const double* __restrict__ U, int ldu, int P, double* __restrict__ Q) {
  extern __shared__ double sh[];
  double* sT = sh;                         // [EB][4][L]
  double* sS = sT + ES_EB * 4 * L;         // [EB][4][P]
  double* sK = sS + ES_EB * 4 * P;         // [EB][16]
  double* sU = sK + ES_EB * 16;            // [EB][4][P]
  __shared__ int32_t sC[ES_EB][4];
  const int m = blockIdx.x;
  const int o0 = blockIdx.y * ES_CHUNK;
  const int PL = P * L;
  const int tid = threadIdx.x;
  double acc[ES_MAXO];
#pragma unroll
  for (int k = 0; k < ES_MAXO; ++k) acc[k] = 0.0;
  const int e0 = dof_ptr[m], e1 = dof_ptr[m + 1];
  for (int eb = e0; eb < e1; eb += ES_EB) {
    const int ne = min(ES_EB, e1 - eb);
    if (tid < ne * 4) {
      const int e = dof_elems[eb + tid / 4];
      sC[tid / 4][tid % 4] = tetra[4 * (size_t)e + (tid % 4)];
    }
    __syncthreads();
    if (tid < ne) unit_block(nodes, sC[tid], ground, sK + 16 * tid);
    for (int o = tid; o < ne * 4 * L; o += ES_THREADS) {
      const int l = o % L, ei = o / L;
      sT[o] = __ldg(T + (size_t)sC[ei / 4][ei % 4] * ldt + l);
    }
    for (int o = tid; o < ne * 4 * P; o += ES_THREADS) {
      const int p = o % P, ei = o / P;
      sU[o] = __ldg(U + (size_t)sC[ei / 4][ei % 4] * ldu + p);
    }
    __syncthreads();
    // s[e,i,p] = sum_j K_e[i,j] u[conn_ej, p]   (einsum "eij,ej->ei")
    for (int o = tid; o < ne * 4 * P; o += ES_THREADS) {
      const int p = o % P, ei = o / P, e = ei / 4, i = ei % 4;
      const double* K = sK + 16 * e + 4 * i;
      const double* u = sU + (size_t)e * 4 * P + p;
      sS[o] = K[0] * u[0] + K[1] * u[P] + K[2] * u[2 * P] + K[3] * u[3 * P];
    }
    __syncthreads();
    // contrib[p, l] = sum_i T[conn_ei, l] s[e,i,p]; Q[p, m, l] += contrib (np.add.at order)
    for (int e = 0; e < ne; ++e) {
#pragma unroll
      for (int k = 0; k < ES_MAXO; ++k) {
        const int o = o0 + tid + k * ES_THREADS;
        if (o < PL) {
          const int p = o / L, l = o % L;
          const double* tt = sT + (size_t)e * 4 * L + l;
          const double* ss = sS + (size_t)e * 4 * P + p;
          const double contrib = tt[0] * ss[0] + tt[L] * ss[P] + tt[2 * L] * ss[2 * P] + tt[3 * L] * ss[3 * P];
          acc[k] += contrib;
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int k = 0; k < ES_MAXO; ++k) {
    const int o = o0 + tid + k * ES_THREADS;
    if (o < PL) {
      const int p = o / L, l = o % L;
      Q[((size_t)p * n_dofs + m) * L + l] = acc[k];
    }
  }
}

}  // namespace tail
}  // namespace hf

using namespace hf;

extern "C" int hf_response_matrix(const hf_csr* Bt, const double* T, int32_t ldt, int32_t L,
                                  int32_t col0, int32_t ncols, const double* Cdiag, double* Mraw,
                                  void* stream) {
  if (!Bt || !T || !Cdiag || !Mraw || L <= 0 || Bt->n_rows != L || ncols < 0 || ldt < ncols ||
      col0 < 0 || col0 + ncols > L) {
    set_error("hf_response_matrix: bad argument");
    return HF_ERR_ARG;
  }
  if (ncols == 0) return HF_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int th = ncols < 256 ? ((ncols + 31) / 32) * 32 : 256;
  tail::k_bt_t<<<L, th, 0, s>>>(L, col0, ncols, Bt->indptr, Bt->indices, Bt->val, T, ldt, Cdiag,
                                Mraw);
  HF_LAUNCH_CHECK();
  count_launches(1);
  return HF_OK;
}

static int lf_launch(int mode, const double* T, int ldt, int L, int K, const hf_csr* Gt,
                     const double* Qc, int ncols, const double* W, int ldw, double* out, int ldo,
                     cudaStream_t s) {
  if (L <= 0 || K <= 0 || K > 1024 || ncols < 0 || ldw < K) {
    set_error("lead-field tail: unsupported L=%d K=%d", L, K);
    return HF_ERR_ARG;
  }
  if (ncols == 0) return HF_OK;
  count_launches(1);
  const int Kp = ((K + 7) / 8) * 8;
  const size_t smem = sizeof(double) * Kp * tail::LF_SBS;
  const int grid = (ncols + tail::LF_NC - 1) / tail::LF_NC;
  if (mode == 0) {
    HF_CUDA(cudaFuncSetAttribute(tail::k_lf_tile<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    tail::k_lf_tile<0><<<grid, tail::LF_THREADS, smem, s>>>(L, K, Kp, ncols, T, ldt, Gt->indptr,
                                                            Gt->indices, Gt->val, nullptr, W, ldw,
                                                            out, ldo);
  } else {
    HF_CUDA(cudaFuncSetAttribute(tail::k_lf_tile<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    tail::k_lf_tile<1><<<grid, tail::LF_THREADS, smem, s>>>(L, K, Kp, ncols, nullptr, 0, nullptr,
                                                            nullptr, nullptr, Qc, W, ldw, out, ldo);
  }
  HF_LAUNCH_CHECK();
  return HF_OK;
}

extern "C" int hf_lf_tail(const double* T, int32_t ldt, int32_t K, const hf_csr* Gt,
                          const double* W, int32_t L, int32_t ldw, double* LF, void* stream) {
  if (!T || !Gt || !W || !LF || ldt < K) {
    set_error("hf_lf_tail: bad argument");
    return HF_ERR_ARG;
  }
  return lf_launch(0, T, ldt, L, K, Gt, nullptr, Gt->n_rows, W, ldw, LF, Gt->n_rows,
                   reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int hf_dense_lf(const double* Qc, int32_t ncols, int32_t K, const double* W,
                           int32_t L, int32_t ldw, double* out, int32_t ldo, void* stream) {
  if (!Qc || !W || !out || ldo < ncols) {
    set_error("hf_dense_lf: bad argument");
    return HF_ERR_ARG;
  }
  return lf_launch(1, nullptr, 0, L, K, nullptr, Qc, ncols, W, ldw, out, ldo,
                   reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int hf_eit_sens(const double* nodes, const int32_t* tetra, const int32_t* dof_elems,
                           const int32_t* dof_ptr, int32_t n_dofs, int32_t ground, const double* T,
                           int32_t ldt, int32_t L, const double* U, int32_t ldu, int32_t P,
                           double* Q, void* stream) {
  if (!nodes || !tetra || !dof_elems || !dof_ptr || !T || !U || !Q || L <= 0 || P <= 0 ||
      ldt < L || ldu < P) {
    set_error("hf_eit_sens: bad argument");
    return HF_ERR_ARG;
  }
  if (n_dofs == 0) return HF_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const size_t smem = sizeof(double) * (tail::ES_EB * 4 * (size_t)L + tail::ES_EB * 4 * (size_t)P * 2 +
                                        tail::ES_EB * 16);
  if (smem > 200 * 1024) {
    set_error("hf_eit_sens: L=%d, P=%d exceed the shared-memory tile", L, P);
    return HF_ERR_ARG;
  }
  HF_CUDA(cudaFuncSetAttribute(tail::k_eit_sens, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem));
  const int chunks = (P * L + tail::ES_CHUNK - 1) / tail::ES_CHUNK;
  dim3 grid(n_dofs, chunks);
  tail::k_eit_sens<<<grid, tail::ES_THREADS, smem, s>>>(nodes, tetra, dof_elems, dof_ptr, n_dofs,
                                                        ground, T, ldt, L, U, ldu, P, Q);
  HF_LAUNCH_CHECK();
  count_launches(1);
  return HF_OK;
}
