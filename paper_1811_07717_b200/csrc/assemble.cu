// P1 tetrahedral stiffness assembly for sm_100a (fem.py:31-224).
//
//   k_blocks       one thread per element: 3x3 Jacobian, volume, P1 gradients,
//                  4x4 block V g_i.sigma g_j (fem.py:31-93) and the AssemblyError
//                  checks (fem.py:56-67, 82-83).
//   incidence      node -> (element, local vertex) lists by counting sort, each
//                  list sorted ascending so every later sum runs in element order.
//   k_row_count /  one warp per matrix row: the row's column set is the union of
//   k_row_fill     the nodes of its incident elements (scipy's COO->CSR pattern
//                  of fem.py:96-102, explicit zeros kept), minus the grounded
//                  column (fem.py:219-224).  Values are gathered, not scattered:
//                  lane p sums the blocks of the incident elements that hold
//                  column p in ascending element order, then adds the electrode
//                  contact terms in triangle order (fem.py:206-211).  No atomics
//                  touch values, so the result is bit-reproducible.
#include "common.cuh"

namespace hf {
namespace asmb {

constexpr int ROW_WARPS = 8;          // warps per block in the row kernels
constexpr int MAX_INC = 128;          // incident elements per node supported
constexpr int MAX_CAND = 4 * MAX_INC; // candidate columns per row

// Element arithmetic uses explicitly rounded operations (no FMA contraction):
// mirrored Kuhn tetrahedra then produce bitwise-opposite off-diagonal
// contributions, which cancel to exact zeros in the row sums — the explicit
// zeros of the reference's pattern (fem.py:96-102) — instead of 1e-20 residue
// that the SpMM would have to stream.
#define MUL(a, b) __dmul_rn((a), (b))
#define ADD(a, b) __dadd_rn((a), (b))
#define SUB(a, b) __dsub_rn((a), (b))

__device__ __forceinline__ double det3(const double a[3][3]) {
  const double c0 = SUB(MUL(a[1][1], a[2][2]), MUL(a[1][2], a[2][1]));
  const double c1 = SUB(MUL(a[1][0], a[2][2]), MUL(a[1][2], a[2][0]));
  const double c2 = SUB(MUL(a[1][0], a[2][1]), MUL(a[1][1], a[2][0]));
  return ADD(SUB(MUL(a[0][0], c0), MUL(a[0][1], c1)), MUL(a[0][2], c2));
}

__device__ __forceinline__ double dot3(const double* a, const double* b) {
  return ADD(ADD(MUL(a[0], b[0]), MUL(a[1], b[1])), MUL(a[2], b[2]));
}

// vol, grads (4x3) of element with vertex coordinates p[4][3]  (fem.py:31-41)
__device__ __forceinline__ double p1_gradients(const double p[4][3], double g[4][3]) {
  double J[3][3];  // columns are edge vectors p_k - p_0
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k) J[r][k] = SUB(p[k + 1][r], p[0][r]);
  const double det = det3(J);
  // inverse = adj(J)/det; row k of the inverse is grad(lambda_{k+1})
  g[1][0] = __ddiv_rn(SUB(MUL(J[1][1], J[2][2]), MUL(J[1][2], J[2][1])), det);
  g[1][1] = __ddiv_rn(SUB(MUL(J[0][2], J[2][1]), MUL(J[0][1], J[2][2])), det);
  g[1][2] = __ddiv_rn(SUB(MUL(J[0][1], J[1][2]), MUL(J[0][2], J[1][1])), det);
  g[2][0] = __ddiv_rn(SUB(MUL(J[1][2], J[2][0]), MUL(J[1][0], J[2][2])), det);
  g[2][1] = __ddiv_rn(SUB(MUL(J[0][0], J[2][2]), MUL(J[0][2], J[2][0])), det);
  g[2][2] = __ddiv_rn(SUB(MUL(J[0][2], J[1][0]), MUL(J[0][0], J[1][2])), det);
  g[3][0] = __ddiv_rn(SUB(MUL(J[1][0], J[2][1]), MUL(J[1][1], J[2][0])), det);
  g[3][1] = __ddiv_rn(SUB(MUL(J[0][1], J[2][0]), MUL(J[0][0], J[2][1])), det);
  g[3][2] = __ddiv_rn(SUB(MUL(J[0][0], J[1][1]), MUL(J[0][1], J[1][0])), det);
#pragma unroll
  for (int k = 0; k < 3; ++k) g[0][k] = -ADD(ADD(g[1][k], g[2][k]), g[3][k]);
  return __ddiv_rn(det, 6.0);
}

__device__ __forceinline__ void load_element(const double* __restrict__ nodes,
                                             const int32_t* __restrict__ tetra, int e,
                                             double p[4][3]) {
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int v = tetra[4 * (size_t)e + a];
#pragma unroll
    for (int r = 0; r < 3; ++r) p[a][r] = nodes[3 * (size_t)v + r];
  }
}

// K_e for scalar sigma (fem.py:87,91) or tensor rows (fem.py:92-93)
__global__ void k_blocks(const double* __restrict__ nodes, const int32_t* __restrict__ tetra,
                         const int32_t* __restrict__ elements, int m_sub,
                         const double* __restrict__ sigma, int sigma_cols, double sigma_scalar,
                         double* __restrict__ blocks, double* __restrict__ vols,
                         int* __restrict__ flags) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m_sub) return;
  const int e = elements ? elements[t] : t;
  double p[4][3], g[4][3];
  load_element(nodes, tetra, e, p);
  const double vol = p1_gradients(p, g);
  if (vols) vols[t] = vol;
  int fl = 0;
  if (!(vol > 0.0)) fl |= 1;
  double* out = blocks + 16 * (size_t)t;
  if (sigma_cols == 6) {
    const double* s = sigma + 6 * (size_t)t;  // sigma rows align with the subset
    const double S[3][3] = {{s[0], s[3], s[4]}, {s[3], s[1], s[5]}, {s[4], s[5], s[2]}};
    const double d1 = S[0][0], d2 = SUB(MUL(S[0][0], S[1][1]), MUL(S[0][1], S[0][1])), d3 = det3(S);
    if (d1 <= 0.0 || d2 <= 0.0 || d3 <= 0.0) fl |= 4;  // Sylvester, fem.py:62-67
    double Sg[4][3];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int k = 0; k < 3; ++k) Sg[j][k] = dot3(S[k], g[j]);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        out[4 * i + j] = MUL(dot3(g[i], Sg[j]), vol);
  } else {
    double sg;
    if (sigma_cols == 1) {
      sg = sigma[t];
      if (sg < 0.0) fl |= 2;  // fem.py:57-59
    } else {
      sg = sigma_scalar;
    }
    const double w = MUL(vol, sg);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        out[4 * i + j] = MUL(dot3(g[i], g[j]), w);
  }
  if (fl) atomicOr(flags, fl);
}

// ---------------------------------------------------------------- incidence
__global__ void k_inc_count(const int32_t* __restrict__ conn, int width, int count,
                            int32_t* __restrict__ cnt) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (size_t)count * width) return;
  atomicAdd(&cnt[conn[t]], 1);
}

__global__ void k_inc_fill(const int32_t* __restrict__ conn, int width, int count,
                           const int32_t* __restrict__ off, int32_t* __restrict__ cur,
                           int32_t* __restrict__ inc) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (size_t)count * width) return;
  const int v = conn[t];
  const int pos = off[v] + atomicAdd(&cur[v], 1);
  inc[pos] = (int32_t)t;  // = owner*width + local slot; owner ascending after sort
}

// Sort each node's incidence list ascending (lists are short: ~24 on a Kuhn grid).
__global__ void k_inc_sort(int n, const int32_t* __restrict__ off, const int32_t* __restrict__ cnt,
                           int32_t* __restrict__ inc) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  int32_t* a = inc + off[v];
  const int len = cnt[v];
  for (int i = 1; i < len; ++i) {
    const int32_t x = a[i];
    int j = i - 1;
    while (j >= 0 && a[j] > x) {
      a[j + 1] = a[j];
      --j;
    }
    a[j + 1] = x;
  }
}

// ---------------------------------------------------------------- rows
// Candidate columns of row i into smem; returns count (or -1 over capacity).
__device__ __forceinline__ int row_candidates(int i, const int32_t* __restrict__ tetra,
                                              const int32_t* __restrict__ off,
                                              const int32_t* __restrict__ cnt,
                                              const int32_t* __restrict__ inc, int32_t* cand) {
  const int lane = threadIdx.x & 31;
  const int deg = cnt[i];
  if (deg > MAX_INC) return -1;
  const int32_t* lst = inc + off[i];
  for (int q = lane; q < 4 * deg; q += 32) {
    const int e = lst[q >> 2] >> 2;
    cand[q] = tetra[4 * (size_t)e + (q & 3)];
  }
  __syncwarp();
  return 4 * deg;
}

// Is cand[j] the first occurrence of its value, and not the grounded column?
__device__ __forceinline__ bool first_occ(const int32_t* cand, int j, int ground) {
  const int v = cand[j];
  if (v == ground) return false;
  for (int k = 0; k < j; ++k)
    if (cand[k] == v) return false;
  return true;
}

__global__ void __launch_bounds__(ROW_WARPS * 32)
    k_row_count(int n, const int32_t* __restrict__ tetra, const int32_t* __restrict__ off,
                const int32_t* __restrict__ cnt, const int32_t* __restrict__ inc, int ground,
                int32_t* __restrict__ rowcnt, int* __restrict__ err) {
  __shared__ int32_t s_cand[ROW_WARPS][MAX_CAND];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x * ROW_WARPS + warp;
  if (i >= n) return;
  if (i == ground) {
    if (lane == 0) rowcnt[i] = 1;
    return;
  }
  int32_t* cand = s_cand[warp];
  const int c = row_candidates(i, tetra, off, cnt, inc, cand);
  if (c < 0) {
    if (lane == 0) {
      atomicOr(err, 1);
      rowcnt[i] = 0;
    }
    return;
  }
  int u = 0;
  for (int j = lane; j < c; j += 32) u += first_occ(cand, j, ground);
  u = __reduce_add_sync(FULL, u);
  if (lane == 0) rowcnt[i] = u;
}

__global__ void __launch_bounds__(ROW_WARPS * 32)
    k_row_fill(int n, const int32_t* __restrict__ tetra, const double* __restrict__ blocks,
               const int32_t* __restrict__ off, const int32_t* __restrict__ cnt,
               const int32_t* __restrict__ inc, const int32_t* __restrict__ etri,
               const double* __restrict__ ecoef, const int32_t* __restrict__ toff,
               const int32_t* __restrict__ tcnt, const int32_t* __restrict__ tinc, int ground,
               const int32_t* __restrict__ indptr, int32_t* __restrict__ indices,
               double* __restrict__ val, int* __restrict__ err) {
  __shared__ int32_t s_cand[ROW_WARPS][MAX_CAND];
  __shared__ int32_t s_cols[ROW_WARPS][MAX_CAND];
  __shared__ uint8_t s_first[ROW_WARPS][MAX_CAND];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x * ROW_WARPS + warp;
  if (i >= n) return;
  const int base = indptr[i];
  if (i == ground) {  // identity row (fem.py:223)
    if (lane == 0) {
      indices[base] = i;
      val[base] = 1.0;
    }
    return;
  }
  int32_t* cand = s_cand[warp];
  int32_t* cols = s_cols[warp];
  const int c = row_candidates(i, tetra, off, cnt, inc, cand);
  if (c < 0) return;  // reported by k_row_count
  // first-occurrence flags, then the rank of each distinct value -> sorted columns
  uint8_t* first = s_first[warp];
  for (int j = lane; j < c; j += 32) first[j] = first_occ(cand, j, ground);
  __syncwarp();
  for (int j = lane; j < c; j += 32) {
    if (!first[j]) continue;
    const int v = cand[j];
    int rank = 0;
    for (int k = 0; k < c; ++k) rank += (first[k] && cand[k] < v);
    cols[rank] = v;
  }
  __syncwarp();
  const int len = indptr[i + 1] - base;
  const int deg = cnt[i];
  const int32_t* lst = inc + off[i];
  const int tdeg = tcnt ? tcnt[i] : 0;
  const int32_t* tl = tinc ? tinc + toff[i] : nullptr;
  for (int p = lane; p < len; p += 32) {
    const int col = cols[p];
    double acc = 0.0;
    // volume part, ascending element order
    for (int q = 0; q < deg; ++q) {
      const int ent = lst[q];
      const int e = ent >> 2, li = ent & 3;
      const int32_t* te = tetra + 4 * (size_t)e;
#pragma unroll
      for (int lk = 0; lk < 4; ++lk)
        if (te[lk] == col) acc += blocks[16 * (size_t)e + 4 * li + lk];
    }
    // electrode contact terms, triangle order (fem.py:207-211)
    for (int q = 0; q < tdeg; ++q) {
      const int ent = tl[q];
      const int t = ent / 3, la = ent % 3;
      const int32_t* tt = etri + 3 * (size_t)t;
#pragma unroll
      for (int lb = 0; lb < 3; ++lb)
        if (tt[lb] == col) acc += MUL(ecoef[t], (la == lb ? 2.0 : 1.0) / 12.0);
    }
    indices[base + p] = col;
    val[base + p] = acc;
  }
  // every triangle neighbour must be in the row (triangle edges are tet edges)
  for (int q = lane; q < tdeg; q += 32) {
    const int t = tl[q] / 3;
    for (int lb = 0; lb < 3; ++lb) {
      const int col = etri[3 * (size_t)t + lb];
      if (col == ground) continue;
      bool found = false;
      for (int p = 0; p < len; ++p) found |= (cols[p] == col);
      if (!found) atomicOr(err, 2);
    }
  }
}

struct Ws {
  int32_t *ecnt, *eoff, *ecur, *einc;
  int32_t *tcnt, *toff, *tcur, *tinc;
  int32_t *rowcnt, *scratch, *tot;
  int* err;
  size_t bytes;
};

inline Ws carve(void* base, int n, int m, int nt) {
  Carve cv{reinterpret_cast<char*>(base), 0, ~size_t(0)};
  Ws w;
  w.ecnt = cv.take<int32_t>((size_t)n + 1);
  w.eoff = cv.take<int32_t>((size_t)n + 1);
  w.ecur = cv.take<int32_t>((size_t)n + 1);
  w.einc = cv.take<int32_t>((size_t)m * 4 + 1);
  w.tcnt = cv.take<int32_t>((size_t)n + 1);
  w.toff = cv.take<int32_t>((size_t)n + 1);
  w.tcur = cv.take<int32_t>((size_t)n + 1);
  w.tinc = cv.take<int32_t>((size_t)nt * 3 + 1);
  w.rowcnt = cv.take<int32_t>((size_t)n + 1);
  w.scratch = cv.take<int32_t>(scan_scratch_elems(n));
  w.tot = cv.take<int32_t>(8);
  w.err = cv.take<int>(8);
  w.bytes = cv.used + 256;
  return w;
}

int build_incidence(const int32_t* conn, int width, int count, int n, int32_t* cnt,
                           int32_t* off, int32_t* cur, int32_t* inc, int32_t* scratch,
                           int32_t* tot, cudaStream_t s) {
  HF_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (n + 1), s));
  HF_CUDA(cudaMemsetAsync(cur, 0, sizeof(int32_t) * (n + 1), s));
  const size_t tot_entries = (size_t)count * width;
  if (tot_entries) {
    const int g = (int)((tot_entries + 255) / 256);
    k_inc_count<<<g, 256, 0, s>>>(conn, width, count, cnt);
    count_launches(1);
    HF_LAUNCH_CHECK();
  }
  int rc = exclusive_scan_i32(cnt, off, n, scratch, tot, s);
  if (rc) return rc;
  if (tot_entries) {
    const int g = (int)((tot_entries + 255) / 256);
    k_inc_fill<<<g, 256, 0, s>>>(conn, width, count, off, cur, inc);
    k_inc_sort<<<(n + 127) / 128, 128, 0, s>>>(n, off, cnt, inc);
    count_launches(2);
    HF_LAUNCH_CHECK();
  }
  return HF_OK;
}

}  // namespace asmb
}  // namespace hf

using namespace hf;

extern "C" int hf_p1_blocks(const double* nodes, const int32_t* tetra, int32_t m,
                            const int32_t* elements, int32_t m_sub, const double* sigma,
                            int32_t sigma_cols, double sigma_scalar, double* blocks, double* vols,
                            int32_t* flags, void* stream) {
  if (!nodes || !tetra || !blocks || !flags || m_sub < 0 ||
      !(sigma_cols == 0 || sigma_cols == 1 || sigma_cols == 6) || (sigma_cols && !sigma)) {
    set_error("hf_p1_blocks: bad argument");
    return HF_ERR_ARG;
  }
  (void)m;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // flags need one device int: use the first slot past the blocks' tail? No —
  // keep the ABI allocation-free by reusing `vols`-independent scratch: the
  // caller passes blocks sized m_sub*16+1 doubles; the extra double holds flags.
  int* dflag = reinterpret_cast<int*>(blocks + 16 * (size_t)m_sub);
  HF_CUDA(cudaMemsetAsync(dflag, 0, sizeof(int), s));
  if (m_sub > 0) {
    asmb::k_blocks<<<(m_sub + 127) / 128, 128, 0, s>>>(nodes, tetra, elements, m_sub, sigma,
                                                       sigma_cols, sigma_scalar, blocks, vols,
                                                       dflag);
    HF_LAUNCH_CHECK();
    count_launches(1);
  }
  int hf = 0;
  HF_CUDA(cudaMemcpyAsync(&hf, dflag, sizeof(int), cudaMemcpyDeviceToHost, s));
  HF_CUDA(cudaStreamSynchronize(s));
  *flags = hf;
  return HF_OK;
}

extern "C" size_t hf_p1_assemble_workspace_bytes(int32_t n, int32_t m, int32_t n_etri) {
  return asmb::carve(nullptr, n, m, n_etri).bytes;
}

extern "C" int hf_p1_assemble_prepare(const int32_t* tetra, int32_t n, int32_t m,
                                      const int32_t* etri, int32_t n_etri, int32_t ground,
                                      int32_t* indptr, int64_t* nnz_out, void* ws,
                                      size_t ws_bytes, void* stream) {
  if (!tetra || !indptr || !nnz_out || !ws || n <= 0 || m < 0 || n_etri < 0 ||
      (n_etri > 0 && !etri)) {
    set_error("hf_p1_assemble_prepare: bad argument");
    return HF_ERR_ARG;
  }
  asmb::Ws w = asmb::carve(ws, n, m, n_etri);
  if (w.bytes > ws_bytes) {
    set_error("assembly workspace too small: need %zu have %zu", w.bytes, ws_bytes);
    return HF_ERR_WORKSPACE;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  HF_CUDA(cudaMemsetAsync(w.err, 0, sizeof(int) * 8, s));
  int rc = asmb::build_incidence(tetra, 4, m, n, w.ecnt, w.eoff, w.ecur, w.einc, w.scratch,
                                 w.tot, s);
  if (rc) return rc;
  rc = asmb::build_incidence(etri, 3, n_etri, n, w.tcnt, w.toff, w.tcur, w.tinc, w.scratch,
                             w.tot + 1, s);
  if (rc) return rc;
  const int g = (n + asmb::ROW_WARPS - 1) / asmb::ROW_WARPS;
  asmb::k_row_count<<<g, asmb::ROW_WARPS * 32, 0, s>>>(n, tetra, w.eoff, w.ecnt, w.einc, ground,
                                                        w.rowcnt, w.err);
  HF_LAUNCH_CHECK();
  count_launches(1);
  rc = exclusive_scan_i32(w.rowcnt, indptr, n, w.scratch, w.tot + 2, s);
  if (rc) return rc;
  HF_CUDA(cudaMemcpyAsync(indptr + n, w.tot + 2, sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  int32_t h[2] = {0, 0};
  HF_CUDA(cudaMemcpyAsync(&h[0], w.tot + 2, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  HF_CUDA(cudaMemcpyAsync(&h[1], w.err, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  HF_CUDA(cudaStreamSynchronize(s));
  if (h[1] & 1) {
    set_error("a node is incident to more than %d elements", asmb::MAX_INC);
    return HF_ERR_CAPACITY;
  }
  *nnz_out = h[0];
  return HF_OK;
}

extern "C" int hf_p1_assemble_fill(const int32_t* tetra, int32_t n, int32_t m,
                                   const double* blocks, const int32_t* etri, const double* ecoef,
                                   int32_t n_etri, int32_t ground, const int32_t* indptr,
                                   int32_t* indices, double* val, void* ws, size_t ws_bytes,
                                   void* stream) {
  if (!tetra || !blocks || !indptr || !indices || !val || !ws || (n_etri > 0 && (!etri || !ecoef))) {
    set_error("hf_p1_assemble_fill: bad argument");
    return HF_ERR_ARG;
  }
  asmb::Ws w = asmb::carve(ws, n, m, n_etri);
  if (w.bytes > ws_bytes) {
    set_error("assembly workspace too small");
    return HF_ERR_WORKSPACE;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int g = (n + asmb::ROW_WARPS - 1) / asmb::ROW_WARPS;
  asmb::k_row_fill<<<g, asmb::ROW_WARPS * 32, 0, s>>>(
      n, tetra, blocks, w.eoff, w.ecnt, w.einc, n_etri ? etri : nullptr, ecoef,
      n_etri ? w.toff : nullptr, n_etri ? w.tcnt : nullptr, n_etri ? w.tinc : nullptr, ground,
      indptr, indices, val, w.err);
  HF_LAUNCH_CHECK();
  count_launches(1);
  int32_t herr = 0;
  HF_CUDA(cudaMemcpyAsync(&herr, w.err, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  HF_CUDA(cudaStreamSynchronize(s));
  if (herr & 2) {
    set_error("an electrode triangle edge is not an element edge");
    return HF_ERR_ARG;
  }
  return HF_OK;
}
