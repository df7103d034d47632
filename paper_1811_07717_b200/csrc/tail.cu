// Post-solve lead-field kernels for sm_100a (leadfield.py:104-237).
//
//   k_bt_t           raw response block C - B'T[:, cols]       (leadfield.py:107)
//   k_lf_tile        LF tile = W (G'T)'_tile  — the (G'T)' tile is gathered
//                    from T rows into shared memory (<= 8 nonzeros per source
//                    column), then multiplied by W = -R M^-1 on the fp64 tensor
//                    path (DMMA: mma.sync.m8n8k4.f64).   (leadfield.py:128-129)
//   k_eit_sens       per-DOF sensitivities Q[p, m, :] = T' K_m u_p  (leadfield.py:179-207)
#include <algorithm>

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

// Q_m (P x L) = S' Tg over the DOF's element corners k = (e, i):
//   S[k, p]  = sum_j K_e[i, j] u[conn_ej, p]     (einsum "eij,ej->ei", leadfield.py:203)
//   Tg[k, l] = T[conn_ei, l]                      (T[conn], leadfield.py:198)
// i.e. np.add.at(Q[p], owner, Tg' s) (leadfield.py:204-206) as one GEMM with
// K = 4 |E_m| per DOF, run on the fp64 tensor pipe (DMMA m8n8k4).  One CTA per
// (DOF, block of <= 64 electrode columns, block of <= 64 patterns); elements in
// chunks of ES_EC: per chunk the CTA computes the unit-sigma blocks, gathers the
// chunk's U and T rows into shared memory, forms S, and every warp accumulates
// its 8x8 output tiles with DMMA.  Shared rows are padded to a stride = 4 mod 16
// doubles so the A/B fragment loads are bank-conflict free.
constexpr int ES_EC = 16;             // elements per chunk -> K = 64 per chunk
constexpr int ES_K = 4 * ES_EC;
constexpr int ES_MAXP = 64, ES_MAXL = 64;
constexpr int ES_WARPS = ES_THREADS / 32;
constexpr int ES_MAXT = (ES_MAXP / 8) * (ES_MAXL / 8) / ES_WARPS;  // output tiles per warp

__host__ __device__ inline int es_stride(int w) { return ((w + 7) / 8) * 8 + ((((w + 7) / 8) * 8) % 16 == 0 ? 4 : 12); }

__global__ void __launch_bounds__(ES_THREADS, 2)
    k_eit_sens(const double* __restrict__ nodes, const int32_t* __restrict__ tetra,
               const int32_t* __restrict__ dof_elems, const int32_t* __restrict__ dof_ptr,
               int n_dofs, int ground, const double* __restrict__ T, int ldt, int L,
               const double* __restrict__ U, int ldu, int P, double* __restrict__ Q) {
  extern __shared__ double sh[];
  const int m = blockIdx.x;
  const int l0 = blockIdx.y * ES_MAXL, p0 = blockIdx.z * ES_MAXP;
  const int nl = min(ES_MAXL, L - l0), np_ = min(ES_MAXP, P - p0);
  const int SP = es_stride(np_), SL = es_stride(nl);
  double* sS = sh;                      // [ES_K][SP]
  double* sT = sS + ES_K * SP;          // [ES_K][SL]
  double* sU = sT + ES_K * SL;          // [ES_K][np_]
  double* sK = sU + ES_K * np_;         // [ES_EC][16]
  __shared__ int32_t sC[ES_EC][4];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int MT = (np_ + 7) / 8, NTt = (nl + 7) / 8, ntile = MT * NTt;
  double acc[ES_MAXT][2];
#pragma unroll
  for (int j = 0; j < ES_MAXT; ++j) acc[j][0] = acc[j][1] = 0.0;
  const int e0 = dof_ptr[m], e1 = dof_ptr[m + 1];
  for (int eb = e0; eb < e1; eb += ES_EC) {
    const int ne = min(ES_EC, e1 - eb);
    if (tid < ES_EC * 4) {
      const int e = tid / 4;
      sC[e][tid % 4] = e < ne ? tetra[4 * (size_t)dof_elems[eb + e] + (tid % 4)] : -1;
    }
    __syncthreads();
    if (tid < ne) unit_block(nodes, sC[tid], ground, sK + 16 * tid);
    for (int o = tid; o < ES_K * np_; o += ES_THREADS) {  // U rows of the chunk's corners
      const int k = o / np_, p = o % np_;
      const int node = sC[k / 4][k % 4];
      sU[o] = node >= 0 ? __ldg(U + (size_t)node * ldu + p0 + p) : 0.0;
    }
    for (int o = tid; o < ES_K * nl; o += ES_THREADS) {  // T rows of the chunk's corners
      const int k = o / nl, l = o % nl;
      const int node = sC[k / 4][k % 4];
      sT[k * SL + l] = node >= 0 ? __ldg(T + (size_t)node * ldt + l0 + l) : 0.0;
    }
    __syncthreads();
    for (int o = tid; o < ES_K * np_; o += ES_THREADS) {  // S = K_e u_e
      const int k = o / np_, p = o % np_, e = k / 4, i = k % 4;
      double v = 0.0;
      if (e < ne) {
        const double* K = sK + 16 * e + 4 * i;
        const double* u = sU + (size_t)(4 * e) * np_ + p;
        v = K[0] * u[0];
        v = fma(K[1], u[np_], v);
        v = fma(K[2], u[2 * np_], v);
        v = fma(K[3], u[3 * np_], v);
      }
      sS[k * SP + p] = v;
    }
    // zero the padded output rows/columns' operands (p >= np_, l >= nl) once per chunk
    for (int o = tid; o < ES_K * (MT * 8 - np_); o += ES_THREADS) {
      const int w = MT * 8 - np_;
      sS[(o / w) * SP + np_ + o % w] = 0.0;
    }
    for (int o = tid; o < ES_K * (NTt * 8 - nl); o += ES_THREADS) {
      const int w = NTt * 8 - nl;
      sT[(o / w) * SL + nl + o % w] = 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < ES_MAXT; ++j) {
      const int ti = warp + ES_WARPS * j;
      if (ti >= ntile) break;
      const int mt = ti % MT, nt = ti / MT;
      const double* ap = sS + (size_t)t4 * SP + mt * 8 + g;  // A[row p][k] = S[k][p]
      const double* bp = sT + (size_t)t4 * SL + nt * 8 + g;  // B[k][col l] = Tg[k][l]
#pragma unroll 4
      for (int k0 = 0; k0 < ES_K; k0 += 4)
        dmma_8x8x4(acc[j][0], acc[j][1], ap[(size_t)k0 * SP], bp[(size_t)k0 * SL]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < ES_MAXT; ++j) {
    const int ti = warp + ES_WARPS * j;
    if (ti >= ntile) break;
    const int mt = ti % MT, nt = ti / MT;
    const int p = mt * 8 + g, l = nt * 8 + 2 * t4;
    if (p < np_) {
      double* q = Q + ((size_t)(p0 + p) * n_dofs + m) * L + l0;
      if (l < nl) q[l] = acc[j][0];
      if (l + 1 < nl) q[l + 1] = acc[j][1];
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
  const int nl = std::min(L, tail::ES_MAXL), np_ = std::min(P, tail::ES_MAXP);
  const size_t smem = sizeof(double) * ((size_t)tail::ES_K * (tail::es_stride(np_) + tail::es_stride(nl) + np_) +
                                        16 * tail::ES_EC);
  HF_CUDA(cudaFuncSetAttribute(tail::k_eit_sens, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem));
  dim3 grid(n_dofs, (L + tail::ES_MAXL - 1) / tail::ES_MAXL, (P + tail::ES_MAXP - 1) / tail::ES_MAXP);
  tail::k_eit_sens<<<grid, tail::ES_THREADS, smem, s>>>(nodes, tetra, dof_elems, dof_ptr, n_dofs,
                                                        ground, T, ldt, L, U, ldu, P, Q);
  HF_LAUNCH_CHECK();
  count_launches(1);
  return HF_OK;
}
