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

// ---------------------------------------------------------------- sparse x dense
// out (n x ncols, row-major) = A (CSR n x k) D (k x ncols, row-major): the EIT
// pattern right-hand sides B V (leadfield.py:223), rows summed in CSR order as
// scipy's csr_matvecs does (a product, then an add).
__global__ void k_csr_dense(int n, int ncols, const int32_t* __restrict__ ptr,
                            const int32_t* __restrict__ idx, const double* __restrict__ val,
                            const double* __restrict__ D, int ldd, double* __restrict__ out, int ldo) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (size_t)n * ncols) return;
  const int i = (int)(t / ncols), c = (int)(t % ncols);
  double acc = 0.0;
  for (int q = ptr[i]; q < ptr[i + 1]; ++q)
    acc = __dadd_rn(acc, __dmul_rn(val[q], D[(size_t)idx[q] * ldd + c]));
  out[(size_t)i * ldo + c] = acc;
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
constexpr int ES_EC = 16;             // elements per chunk -> K = 64 per chunk (one corner per 4 threads)
constexpr int ES_K = 4 * ES_EC;
constexpr int ES_MAXP = 32, ES_MAXL = 64;  // patterns x electrode columns per CTA
constexpr int ES_WARPS = ES_THREADS / 32;
static_assert(ES_MAXP == 32 && ES_MAXL == 64 && ES_WARPS == 8, "8 warps x 16x16 blocks = 32 x 64");

__host__ __device__ inline int es_stride(int w) { return ((w + 7) / 8) * 8 + ((((w + 7) / 8) * 8) % 16 == 0 ? 4 : 12); }

// Unit-sigma blocks of every DOF element, in dof_elems order (one thread each):
// the divisions of unit_block run massively parallel here instead of on 16
// threads of a sensitivity CTA.  Kbuf: (sum of DOF sizes) x 16.
__global__ void k_dof_blocks(const double* __restrict__ nodes, const int32_t* __restrict__ tetra,
                             const int32_t* __restrict__ dof_elems, int n_elems, int ground,
                             double* __restrict__ Kbuf) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_elems) return;
  int32_t conn[4];
  const int e = dof_elems[i];
#pragma unroll
  for (int a = 0; a < 4; ++a) conn[a] = tetra[4 * (size_t)e + a];
  double K[16];
  unit_block(nodes, conn, ground, K);
#pragma unroll
  for (int q = 0; q < 16; ++q) Kbuf[(size_t)i * 16 + q] = K[q];
}

__global__ void __launch_bounds__(ES_THREADS, 3)
    k_eit_sens(const double* __restrict__ Kbuf, const int32_t* __restrict__ tetra,
               const int32_t* __restrict__ dof_elems, const int32_t* __restrict__ dof_ptr,
               int n_dofs, const double* __restrict__ T, int ldt, int L,
               const double* __restrict__ U, int ldu, int P, double* __restrict__ Q) {
  extern __shared__ double sh[];
  const int m = blockIdx.x;
  const int l0 = blockIdx.y * ES_MAXL, p0 = blockIdx.z * ES_MAXP;
  const int nl = min(ES_MAXL, L - l0), np_ = min(ES_MAXP, P - p0);
  const int SP = es_stride(np_), SL = es_stride(nl);
  double* sS = sh;                      // [ES_K][SP]
  double* sT = sS + ES_K * SP;          // [ES_K][SL]
  double* sU = sT + ES_K * SL;          // [ES_K][SP]
  double* sK = sU + ES_K * SP;          // [ES_EC][16]
  __shared__ int32_t sC[2][ES_K];       // corner nodes of this chunk and the next
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int wm = warp & 1, wn = warp >> 1;  // this warp's 16 x 16 output block
  // gather layout: 4 threads per chunk corner k = tid / 4; thread gq of a corner owns
  // columns gq, gq + 4, ... so a warp's accesses are 8 corners x 4 consecutive
  // doubles: one sector per corner in global memory, conflict-free in shared memory
  const int gk = tid >> 2, gq = tid & 3;
  double acc[4][2];  // tiles (rows +0/+8, columns +0/+8) of the warp's block
#pragma unroll
  for (int j = 0; j < 4; ++j) acc[j][0] = acc[j][1] = 0.0;
  const int e0 = dof_ptr[m], e1 = dof_ptr[m + 1];
  auto load_conn = [&](int eb, int buf) {
    if (tid < ES_K) {
      const int e = eb + tid / 4;
      sC[buf][tid] = e < e1 ? tetra[4 * (size_t)dof_elems[e] + (tid & 3)] : -1;
    }
  };
  load_conn(e0, 0);
  // padded operand rows/columns (p >= np_, l >= nl) stay zero for the whole CTA
  for (int o = tid; o < ES_K * SP; o += ES_THREADS) sS[o] = 0.0;
  for (int o = tid; o < ES_K * SL; o += ES_THREADS) sT[o] = 0.0;
  __syncthreads();
  int buf = 0;
  for (int eb = e0; eb < e1; eb += ES_EC, buf ^= 1) {
    const int ne = min(ES_EC, e1 - eb);
    // 1) this thread's T and U row segments into registers: every load in flight at once
    const int node = sC[buf][gk];
    double tv[ES_MAXL / 4], uv[ES_MAXP / 4];
#pragma unroll
    for (int i = 0; i < ES_MAXL / 4; ++i)
      tv[i] = (node >= 0 && gq + 4 * i < nl) ? __ldg(T + (size_t)node * ldt + l0 + gq + 4 * i) : 0.0;
#pragma unroll
    for (int i = 0; i < ES_MAXP / 4; ++i)
      uv[i] = (node >= 0 && gq + 4 * i < np_) ? __ldg(U + (size_t)node * ldu + p0 + gq + 4 * i) : 0.0;
    // 2) the chunk's element blocks (k_dof_blocks), one entry per thread
    const double kv = tid < 16 * ne ? __ldg(Kbuf + (size_t)(eb - dof_ptr[0]) * 16 + tid) : 0.0;
    // 3) next chunk's corners
    load_conn(eb + ES_EC, buf ^ 1);
#pragma unroll
    for (int i = 0; i < ES_MAXL / 4; ++i)
      if (gq + 4 * i < nl) sT[gk * SL + gq + 4 * i] = tv[i];
#pragma unroll
    for (int i = 0; i < ES_MAXP / 4; ++i)
      if (gq + 4 * i < np_) sU[gk * SP + gq + 4 * i] = uv[i];
    sK[tid] = kv;
    __syncthreads();
    // 4) S[k, p] = K_e[i, :] u_e[:, p]
    {
      const int e = gk / 4, i = gk & 3;
      if (e < ne) {
        const double* K = sK + 16 * e + 4 * i;
        const double* u = sU + (size_t)(4 * e) * SP;
        for (int pp = gq; pp < np_; pp += 4) {
          double v = K[0] * u[pp];
          v = fma(K[1], u[SP + pp], v);
          v = fma(K[2], u[2 * SP + pp], v);
          v = fma(K[3], u[3 * SP + pp], v);
          sS[gk * SP + pp] = v;
        }
      } else {
        for (int pp = gq; pp < np_; pp += 4) sS[gk * SP + pp] = 0.0;
      }
    }
    __syncthreads();
    // 5) Q tiles += S' Tg on the fp64 tensor pipe.  Warp w owns the 2 x 2 block of
    //    8x8 output tiles (rows 16 (w % 2) .., columns 16 (w / 2) ..): per k-step two A
    //    and two B fragments feed four DMMAs, whose chains advance together.
#pragma unroll 4
    for (int k0 = 0; k0 < ES_K; k0 += 4) {
      const double* ar = sS + (size_t)(k0 + t4) * SP + wm * 16 + g;  // A[row p][k] = S[k][p]
      const double* br = sT + (size_t)(k0 + t4) * SL + wn * 16 + g;  // B[k][col l] = Tg[k][l]
      const double a0 = ar[0], a1 = ar[8], b0 = br[0], b1 = br[8];
      dmma_8x8x4(acc[0][0], acc[0][1], a0, b0);
      dmma_8x8x4(acc[1][0], acc[1][1], a1, b0);
      dmma_8x8x4(acc[2][0], acc[2][1], a0, b1);
      dmma_8x8x4(acc[3][0], acc[3][1], a1, b1);
    }
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int p = wm * 16 + (j & 1) * 8 + g, l = wn * 16 + (j >> 1) * 8 + 2 * t4;
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

extern "C" size_t hf_eit_sens_workspace_bytes(int64_t n_dof_elems) {
  return (size_t)(n_dof_elems + 1) * 16 * sizeof(double) + 256;
}

extern "C" int hf_eit_sens(const double* nodes, const int32_t* tetra, const int32_t* dof_elems,
                           const int32_t* dof_ptr, int32_t n_dofs, int32_t ground, const double* T,
                           int32_t ldt, int32_t L, const double* U, int32_t ldu, int32_t P,
                           double* Q, void* ws, size_t ws_bytes, void* stream) {
  if (!nodes || !tetra || !dof_elems || !dof_ptr || !T || !U || !Q || !ws || L <= 0 || P <= 0 ||
      ldt < L || ldu < P || n_dofs < 0) {
    set_error("hf_eit_sens: bad argument");
    return HF_ERR_ARG;
  }
  if (n_dofs == 0) return HF_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int32_t ends[2] = {0, 0};
  HF_CUDA(cudaMemcpyAsync(&ends[0], dof_ptr, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  HF_CUDA(cudaMemcpyAsync(&ends[1], dof_ptr + n_dofs, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  HF_CUDA(cudaStreamSynchronize(s));
  const int64_t ne = (int64_t)ends[1] - ends[0];
  if (ws_bytes < hf_eit_sens_workspace_bytes(ne)) {
    set_error("hf_eit_sens: workspace too small");
    return HF_ERR_WORKSPACE;
  }
  double* Kbuf = reinterpret_cast<double*>(ws);
  if (ne > 0) {
    tail::k_dof_blocks<<<(int)((ne + 255) / 256), 256, 0, s>>>(nodes, tetra, dof_elems + ends[0], (int)ne,
                                                               ground, Kbuf);
    HF_LAUNCH_CHECK();
    count_launches(1);
  }
  const int nl = std::min(L, tail::ES_MAXL), np_ = std::min(P, tail::ES_MAXP);
  const size_t smem = sizeof(double) * ((size_t)tail::ES_K * (2 * tail::es_stride(np_) + tail::es_stride(nl)) +
                                        16 * tail::ES_EC);
  HF_CUDA(cudaFuncSetAttribute(tail::k_eit_sens, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem));
  dim3 grid(n_dofs, (L + tail::ES_MAXL - 1) / tail::ES_MAXL, (P + tail::ES_MAXP - 1) / tail::ES_MAXP);
  tail::k_eit_sens<<<grid, tail::ES_THREADS, smem, s>>>(Kbuf, tetra, dof_elems, dof_ptr, n_dofs, T,
                                                        ldt, L, U, ldu, P, Q);
  HF_LAUNCH_CHECK();
  count_launches(1);
  return HF_OK;
}

extern "C" int hf_csr_dense(const hf_csr* A, const double* D, int32_t ldd, int32_t ncols, double* out,
                            int32_t ldo, void* stream) {
  if (!A || !D || !out || ncols < 0 || ldd < ncols || ldo < ncols) {
    set_error("hf_csr_dense: bad argument");
    return HF_ERR_ARG;
  }
  const size_t work = (size_t)A->n_rows * ncols;
  if (work == 0) return HF_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  tail::k_csr_dense<<<(unsigned)((work + 255) / 256), 256, 0, s>>>(A->n_rows, ncols, A->indptr, A->indices,
                                                                    A->val, D, ldd, out, ldo);
  HF_LAUNCH_CHECK();
  count_launches(1);
  return HF_OK;
}
