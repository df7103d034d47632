// Mesh topology and the Whitney source matrix on the device — the "next" rows
// of SURVEY.md §8f that feed the lead-field path:
//
//   hf_boundary_faces   TetMesh.element_faces / boundary_triangles (meshgen.py:101-134)
//   hf_whitney_gt       _face_incidence + build_source_model + whitney_source_matrix
//                       + assemble_G (fem.py:291-422), emitted as G' (source columns
//                       as CSR rows), the layout hf_lf_tail consumes.
//
// Both replace a global sort/unique over the 4m element faces by node->element
// incidence lists: the element across face (a,b,c) of e is the other element
// in a's list that also holds b and c.  Outputs are ordered exactly like the
// reference (ascending element-face index; ascending node per G column).
#include "common.cuh"

namespace hf {
namespace topo {

__constant__ int FACE[4][3] = {{1, 2, 3}, {0, 3, 2}, {0, 1, 3}, {0, 2, 1}};  // meshgen.py:107-111

#define MUL(a, b) __dmul_rn((a), (b))
#define ADD(a, b) __dadd_rn((a), (b))
#define SUB(a, b) __dsub_rn((a), (b))

__device__ __forceinline__ bool holds(const int32_t* te, int v) {
  return te[0] == v || te[1] == v || te[2] == v || te[3] == v;
}

// element sharing face {a, b, c} with e, or -1 (boundary face)
__device__ __forceinline__ int neighbour(int e, int a, int b, int c, const int32_t* __restrict__ tetra,
                                         const int32_t* __restrict__ off,
                                         const int32_t* __restrict__ cnt,
                                         const int32_t* __restrict__ inc) {
  const int32_t* lst = inc + off[a];
  const int len = cnt[a];
  for (int q = 0; q < len; ++q) {
    const int k = lst[q] >> 2;
    if (k == e) continue;
    const int32_t* tk = tetra + 4 * (size_t)k;
    if (holds(tk, b) && holds(tk, c)) return k;
  }
  return -1;
}

// per element: bit j set when face j is a boundary face; count of such faces
__global__ void k_boundary_count(int m, const int32_t* __restrict__ tetra,
                                 const int32_t* __restrict__ off, const int32_t* __restrict__ cnt,
                                 const int32_t* __restrict__ inc, int32_t* __restrict__ bits,
                                 int32_t* __restrict__ counts) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m) return;
  const int32_t* te = tetra + 4 * (size_t)e;
  int b = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int a = te[FACE[j][0]], bb = te[FACE[j][1]], c = te[FACE[j][2]];
    if (neighbour(e, a, bb, c, tetra, off, cnt, inc) < 0) b |= 1 << j;
  }
  bits[e] = b;
  counts[e] = __popc(b);
}

__global__ void k_boundary_fill(int m, const int32_t* __restrict__ bits,
                                const int32_t* __restrict__ pos, int32_t* __restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m) return;
  int o = pos[e];
  const int b = bits[e];
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (b & (1 << j)) out[o++] = 4 * e + j;
}

// ---------------------------------------------------------------- Whitney G
constexpr int GROWS = 8;  // nodes of a source element and of its 4 face neighbours

struct SourceStencil {
  int rows[GROWS];
  double gw[GROWS][4];  // G_w[row, 4s + j] (fem.py:342-364)
  int nrows;
  double coeff[4][3];   // min-norm face combination for unit axis moments (fem.py:411-413)
};

__device__ __forceinline__ void load_node(const double* __restrict__ nodes, int v, double p[3]) {
  p[0] = nodes[3 * (size_t)v];
  p[1] = nodes[3 * (size_t)v + 1];
  p[2] = nodes[3 * (size_t)v + 2];
}

__device__ void build_stencil(int e, const double* __restrict__ nodes,
                              const int32_t* __restrict__ tetra, const int32_t* __restrict__ off,
                              const int32_t* __restrict__ cnt, const int32_t* __restrict__ inc,
                              SourceStencil& S) {
  double mom[4][3];
  int slot_elem[4][2];
  double slot_sgn[4][2];
  const int32_t* te = tetra + 4 * (size_t)e;
  for (int j = 0; j < 4; ++j) {
    int f0 = te[FACE[j][0]], f1 = te[FACE[j][1]], f2 = te[FACE[j][2]];
    // sorted face nodes: the rows of np.unique(np.sort(faces)) (fem.py:293-294)
    if (f0 > f1) { const int t = f0; f0 = f1; f1 = t; }
    if (f1 > f2) { const int t = f1; f1 = f2; f2 = t; }
    if (f0 > f1) { const int t = f0; f0 = f1; f1 = t; }
    double p0[3], p1[3], p2[3];
    load_node(nodes, f0, p0);
    load_node(nodes, f1, p1);
    load_node(nodes, f2, p2);
    double fc[3], u[3], v[3];
    for (int r = 0; r < 3; ++r) {
      fc[r] = __ddiv_rn(ADD(ADD(p0[r], p1[r]), p2[r]), 3.0);  // face centre (fem.py:325)
      u[r] = SUB(p1[r], p0[r]);
      v[r] = SUB(p2[r], p0[r]);
    }
    const double nc[3] = {SUB(MUL(u[1], v[2]), MUL(u[2], v[1])), SUB(MUL(u[2], v[0]), MUL(u[0], v[2])),
                          SUB(MUL(u[0], v[1]), MUL(u[1], v[0]))};  // np.cross (fem.py:326-327)
    const int k = neighbour(e, f0, f1, f2, tetra, off, cnt, inc);
    // face_elems: slot 0 is the lower element index (stable argsort, fem.py:297-303)
    slot_elem[j][0] = (k >= 0 && k < e) ? k : e;
    slot_elem[j][1] = (k < 0) ? -1 : (k < e ? e : k);
    for (int r = 0; r < 3; ++r) mom[j][r] = 0.0;
    for (int sl = 0; sl < 2; ++sl) {
      const int q = slot_elem[j][sl];
      slot_sgn[j][sl] = 0.0;
      if (q < 0) continue;
      const int32_t* tq = tetra + 4 * (size_t)q;
      int opp = tq[0];
      for (int a = 0; a < 4; ++a)
        if (tq[a] != f0 && tq[a] != f1 && tq[a] != f2) opp = tq[a];
      double po[3];
      load_node(nodes, opp, po);
      const double w[3] = {SUB(fc[0], po[0]), SUB(fc[1], po[1]), SUB(fc[2], po[2])};
      const double dot = ADD(ADD(MUL(nc[0], w[0]), MUL(nc[1], w[1])), MUL(nc[2], w[2]));
      const double sgn = dot > 0.0 ? 1.0 : -1.0;  // fem.py:332
      slot_sgn[j][sl] = sgn;
      double cq[3] = {0.0, 0.0, 0.0};
      for (int a = 0; a < 4; ++a) {
        double pa[3];
        load_node(nodes, tq[a], pa);
        for (int r = 0; r < 3; ++r) cq[r] = ADD(cq[r], pa[r]);
      }
      for (int r = 0; r < 3; ++r) {  // moments += sgn (centroid_k - a_k) / 3   (fem.py:336-337)
        const double cen = __ddiv_rn(cq[r], 4.0);
        mom[j][r] = ADD(mom[j][r], __ddiv_rn(MUL(sgn, SUB(cen, po[r])), 3.0));
      }
    }
  }
  // coeff (4x3) = min-norm solution of  M' coeff = I,  M = mom (4x3):
  // coeff = M (M'M)^-1  (np.linalg.lstsq for a full-rank 3x4 system)
  double g[3][3];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double sacc = 0.0;
      for (int j = 0; j < 4; ++j) sacc = fma(mom[j][a], mom[j][b], sacc);
      g[a][b] = sacc;
    }
  const double det = g[0][0] * (g[1][1] * g[2][2] - g[1][2] * g[2][1]) -
                     g[0][1] * (g[1][0] * g[2][2] - g[1][2] * g[2][0]) +
                     g[0][2] * (g[1][0] * g[2][1] - g[1][1] * g[2][0]);
  double gi[3][3];
  gi[0][0] = (g[1][1] * g[2][2] - g[1][2] * g[2][1]) / det;
  gi[0][1] = (g[0][2] * g[2][1] - g[0][1] * g[2][2]) / det;
  gi[0][2] = (g[0][1] * g[1][2] - g[0][2] * g[1][1]) / det;
  gi[1][0] = (g[1][2] * g[2][0] - g[1][0] * g[2][2]) / det;
  gi[1][1] = (g[0][0] * g[2][2] - g[0][2] * g[2][0]) / det;
  gi[1][2] = (g[0][2] * g[1][0] - g[0][0] * g[1][2]) / det;
  gi[2][0] = (g[1][0] * g[2][1] - g[1][1] * g[2][0]) / det;
  gi[2][1] = (g[0][1] * g[2][0] - g[0][0] * g[2][1]) / det;
  gi[2][2] = (g[0][0] * g[1][1] - g[0][1] * g[1][0]) / det;
  for (int j = 0; j < 4; ++j)
    for (int c = 0; c < 3; ++c) {
      double sacc = 0.0;
      for (int a = 0; a < 3; ++a) sacc = fma(mom[j][a], gi[a][c], sacc);
      S.coeff[j][c] = sacc;
    }
  // rows: nodes of every adjoining element, ascending; G_w values (+-1/4 per element)
  int nr = 0;
  for (int j = 0; j < 4; ++j)
    for (int sl = 0; sl < 2; ++sl) {
      const int q = slot_elem[j][sl];
      if (q < 0) continue;
      for (int a = 0; a < 4; ++a) {
        const int v = tetra[4 * (size_t)q + a];
        bool seen = false;
        for (int r = 0; r < nr; ++r) seen |= (S.rows[r] == v);
        if (!seen && nr < GROWS) S.rows[nr++] = v;
      }
    }
  for (int a = 1; a < nr; ++a) {  // insertion sort
    const int v = S.rows[a];
    int b = a - 1;
    while (b >= 0 && S.rows[b] > v) {
      S.rows[b + 1] = S.rows[b];
      --b;
    }
    S.rows[b + 1] = v;
  }
  S.nrows = nr;
  for (int r = 0; r < nr; ++r)
    for (int j = 0; j < 4; ++j) {
      double wsum = 0.0;  // duplicates of (row, 4s+j) summed in slot order
      for (int sl = 0; sl < 2; ++sl) {
        const int q = slot_elem[j][sl];
        if (q >= 0 && holds(tetra + 4 * (size_t)q, S.rows[r])) wsum = ADD(wsum, slot_sgn[j][sl] / 4.0);
      }
      S.gw[r][j] = wsum;
    }
}

__global__ void k_whitney_count(int S_, const int32_t* __restrict__ src, const double* __restrict__ nodes,
                                const int32_t* __restrict__ tetra, const int32_t* __restrict__ off,
                                const int32_t* __restrict__ cnt, const int32_t* __restrict__ inc,
                                int ncomp, int32_t* __restrict__ colcnt) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S_) return;
  SourceStencil st;
  build_stencil(src[s], nodes, tetra, off, cnt, inc, st);
  for (int c = 0; c < ncomp; ++c) colcnt[ncomp * s + c] = st.nrows;
}

__global__ void k_whitney_fill(int S_, const int32_t* __restrict__ src, const double* __restrict__ nodes,
                               const int32_t* __restrict__ tetra, const int32_t* __restrict__ off,
                               const int32_t* __restrict__ cnt, const int32_t* __restrict__ inc,
                               int ncomp, const double* __restrict__ orient,
                               const int32_t* __restrict__ gptr, int32_t* __restrict__ gidx,
                               double* __restrict__ gval) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S_) return;
  SourceStencil st;
  build_stencil(src[s], nodes, tetra, off, cnt, inc, st);
  for (int c = 0; c < ncomp; ++c) {
    double w[4];
    for (int j = 0; j < 4; ++j) {
      if (ncomp == 3) {
        w[j] = st.coeff[j][c];
      } else {  // constrained: coeff @ orientation (fem.py:414-416)
        const double* o = orient + 3 * (size_t)s;
        w[j] = fma(st.coeff[j][2], o[2], fma(st.coeff[j][1], o[1], st.coeff[j][0] * o[0]));
      }
    }
    const int base = gptr[ncomp * s + c];
    for (int r = 0; r < st.nrows; ++r) {
      double v = 0.0;  // (G_w W)[row, col]: sum over the 4 face functions (fem.py:419-420)
      for (int j = 0; j < 4; ++j) v = fma(st.gw[r][j], w[j], v);
      gidx[base + r] = st.rows[r];
      gval[base + r] = v;
    }
  }
}

}  // namespace topo

namespace asmb {
int build_incidence(const int32_t* conn, int width, int count, int n, int32_t* cnt, int32_t* off,
                    int32_t* cur, int32_t* inc, int32_t* scratch, int32_t* tot, cudaStream_t s);
}

}  // namespace hf

using namespace hf;

namespace {
struct TopoWs {
  int32_t *cnt, *off, *cur, *inc, *scratch, *tot, *bits, *counts, *pos;
  size_t bytes;
};
TopoWs carve_topo(void* base, int n, int m, int ncols) {
  Carve cv{reinterpret_cast<char*>(base), 0, ~size_t(0)};
  TopoWs w;
  const int big = (m > ncols ? m : ncols);
  w.cnt = cv.take<int32_t>((size_t)n + 1);
  w.off = cv.take<int32_t>((size_t)n + 1);
  w.cur = cv.take<int32_t>((size_t)n + 1);
  w.inc = cv.take<int32_t>((size_t)m * 4 + 1);
  w.scratch = cv.take<int32_t>(scan_scratch_elems(big > n ? big : n));
  w.tot = cv.take<int32_t>(8);
  w.bits = cv.take<int32_t>((size_t)big + 1);
  w.counts = cv.take<int32_t>((size_t)big + 1);
  w.pos = cv.take<int32_t>((size_t)big + 1);
  w.bytes = cv.used + 256;
  return w;
}
}  // namespace

namespace hf {
namespace topo {
// ---------------------------------------------------------------- electrodes / ground
// Centroids of boundary triangles, numpy's mean of 3 rows: ((a + b) + c) / 3
// (ElectrodeSet.from_centers, fem.py:163).
__global__ void k_tri_centroids(const double* __restrict__ nodes, const int32_t* __restrict__ tri,
                                int nt, double* __restrict__ cent) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nt) return;
  const int a = tri[3 * (size_t)t], b = tri[3 * (size_t)t + 1], c = tri[3 * (size_t)t + 2];
#pragma unroll
  for (int r = 0; r < 3; ++r)
    cent[3 * (size_t)t + r] =
        __ddiv_rn(__dadd_rn(__dadd_rn(nodes[3 * (size_t)a + r], nodes[3 * (size_t)b + r]),
                            nodes[3 * (size_t)c + r]),
                  3.0);
}

__global__ void k_mark_nodes(const int32_t* __restrict__ tri, int nt, unsigned bit,
                             unsigned* __restrict__ mark) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (size_t)nt * 3) return;
  atomicOr(&mark[tri[t]], bit);
}

__global__ void k_first_free(int n, const unsigned* __restrict__ mark, int* __restrict__ best) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < n && mark[v] == 1u) atomicMin(best, v);
}

}  // namespace topo
}  // namespace hf

extern "C" int hf_triangle_centroids(const double* nodes, const int32_t* tri, int32_t n_tri,
                                     double* cent, void* stream) {
  if (n_tri < 0 || (n_tri > 0 && (!nodes || !tri || !cent))) {
    hf::set_error("hf_triangle_centroids: bad argument");
    return HF_ERR_ARG;
  }
  if (n_tri == 0) return HF_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  hf::topo::k_tri_centroids<<<(n_tri + 255) / 256, 256, 0, s>>>(nodes, tri, n_tri, cent);
  HF_LAUNCH_CHECK();
  hf::count_launches(1);
  return HF_OK;
}

extern "C" size_t hf_ground_node_workspace_bytes(int32_t n) { return 4 * ((size_t)n + 2) + 256; }

extern "C" int hf_ground_node(const int32_t* bfaces, int32_t n_bfaces, const int32_t* etri,
                              int32_t n_etri, int32_t n, void* ws, int32_t* ground, void* stream) {
  if (!bfaces || !ws || !ground || n <= 0 || n_bfaces < 0 || n_etri < 0 || (n_etri > 0 && !etri)) {
    hf::set_error("hf_ground_node: bad argument");
    return HF_ERR_ARG;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  unsigned* mark = reinterpret_cast<unsigned*>(ws);
  int* best = reinterpret_cast<int*>(mark + n + 1);
  HF_CUDA(cudaMemsetAsync(mark, 0, sizeof(unsigned) * (n + 1), s));
  const int big = 0x7f7f7f7f;  // > any int32 node index this ABI accepts
  HF_CUDA(cudaMemsetAsync(best, 0x7f, sizeof(int), s));
  if (n_bfaces)
    hf::topo::k_mark_nodes<<<(3 * n_bfaces + 255) / 256, 256, 0, s>>>(bfaces, n_bfaces, 1u, mark);
  if (n_etri)
    hf::topo::k_mark_nodes<<<(3 * n_etri + 255) / 256, 256, 0, s>>>(etri, n_etri, 2u, mark);
  hf::topo::k_first_free<<<(n + 255) / 256, 256, 0, s>>>(n, mark, best);
  HF_LAUNCH_CHECK();
  hf::count_launches(1 + (n_bfaces > 0) + (n_etri > 0));
  int h = big;
  HF_CUDA(cudaMemcpyAsync(&h, best, sizeof(int), cudaMemcpyDeviceToHost, s));
  HF_CUDA(cudaStreamSynchronize(s));
  *ground = (h == big) ? -1 : h;
  return HF_OK;
}

extern "C" size_t hf_topology_workspace_bytes(int32_t n, int32_t m, int32_t ncols) {
  return carve_topo(nullptr, n, m, ncols).bytes;
}

extern "C" int hf_boundary_faces(const int32_t* tetra, int32_t n, int32_t m, int32_t* face_idx,
                                 int64_t* n_faces, void* ws, size_t ws_bytes, void* stream) {
  if (!tetra || !face_idx || !n_faces || !ws || n <= 0 || m < 0) {
    set_error("hf_boundary_faces: bad argument");
    return HF_ERR_ARG;
  }
  TopoWs w = carve_topo(ws, n, m, 0);
  if (w.bytes > ws_bytes) {
    set_error("topology workspace too small");
    return HF_ERR_WORKSPACE;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int rc = asmb::build_incidence(tetra, 4, m, n, w.cnt, w.off, w.cur, w.inc, w.scratch, w.tot, s);
  if (rc) return rc;
  if (m > 0) {
    topo::k_boundary_count<<<(m + 255) / 256, 256, 0, s>>>(m, tetra, w.off, w.cnt, w.inc, w.bits,
                                                           w.counts);
    HF_LAUNCH_CHECK();
    count_launches(1);
  }
  rc = exclusive_scan_i32(w.counts, w.pos, m, w.scratch, w.tot + 1, s);
  if (rc) return rc;
  if (m > 0) {
    topo::k_boundary_fill<<<(m + 255) / 256, 256, 0, s>>>(m, w.bits, w.pos, face_idx);
    HF_LAUNCH_CHECK();
    count_launches(1);
  }
  int32_t total = 0;
  HF_CUDA(cudaMemcpyAsync(&total, w.tot + 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  HF_CUDA(cudaStreamSynchronize(s));
  *n_faces = total;
  return HF_OK;
}

extern "C" int hf_whitney_gt(const double* nodes, const int32_t* tetra, int32_t n, int32_t m,
                             const int32_t* src_elems, int32_t n_src, const double* orient,
                             int32_t* gptr, int32_t* gidx, double* gval, int64_t* nnz_out,
                             void* ws, size_t ws_bytes, void* stream) {
  if (!nodes || !tetra || !src_elems || !gptr || !nnz_out || !ws || n <= 0 || n_src < 0) {
    set_error("hf_whitney_gt: bad argument");
    return HF_ERR_ARG;
  }
  const int ncomp = orient ? 1 : 3;
  const int ncols = ncomp * n_src;
  TopoWs w = carve_topo(ws, n, m, ncols);
  if (w.bytes > ws_bytes) {
    set_error("topology workspace too small");
    return HF_ERR_WORKSPACE;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int rc = asmb::build_incidence(tetra, 4, m, n, w.cnt, w.off, w.cur, w.inc, w.scratch, w.tot, s);
  if (rc) return rc;
  const int g = (n_src + 127) / 128;
  if (n_src > 0) {
    topo::k_whitney_count<<<g, 128, 0, s>>>(n_src, src_elems, nodes, tetra, w.off, w.cnt, w.inc,
                                             ncomp, w.counts);
    HF_LAUNCH_CHECK();
    count_launches(1);
  }
  rc = exclusive_scan_i32(w.counts, gptr, ncols, w.scratch, w.tot + 2, s);
  if (rc) return rc;
  HF_CUDA(cudaMemcpyAsync(gptr + ncols, w.tot + 2, sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  int32_t total = 0;
  HF_CUDA(cudaMemcpyAsync(&total, w.tot + 2, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  HF_CUDA(cudaStreamSynchronize(s));
  *nnz_out = total;
  if (gidx && gval && n_src > 0) {
    topo::k_whitney_fill<<<g, 128, 0, s>>>(n_src, src_elems, nodes, tetra, w.off, w.cnt, w.inc,
                                            ncomp, orient, gptr, gidx, gval);
    HF_LAUNCH_CHECK();
    count_launches(1);
  }
  return HF_OK;
}
