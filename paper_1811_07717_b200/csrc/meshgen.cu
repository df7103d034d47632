// Labelled uniform tetrahedral mesh generation on the device (SURVEY.md §8f
// "next" row #4): generate_mesh (meshgen.py:186-244), _apply_priorities
// (meshgen.py:247-269) and the point-location query they call,
// Segmentation.locate (geometry.py:359-374) -> Compartment.contains
// (geometry.py:332-341) -> SurfaceMesh._contains_impl / _cast
// (geometry.py:168-249).
//
// locate: one thread per point walks the compartments innermost first and,
// inside a compartment, its sub-surfaces; a surface test is the reference's
// ray-parity loop over its fixed directions (retry on a grazing or coplanar
// hit, stop on an on-surface hit).  The per-(direction, triangle) constants
// of _cast (h = d x e2, k = e1 x d, n, c_h, c_k, c_n, f, parallel, tol*|n|)
// are computed on the host with the reference's own numpy expressions and
// read here as warp-uniform rows, so each thread only evaluates the three
// affine forms p.h, p.k, p.n per triangle.  The dot products follow the
// rounding of the BLAS product the reference uses (p0 h0 rounded, then two
// FMAs); every other operation is an explicitly rounded fp64 op, as numpy
// evaluates it.  All thresholds (1e-10 barycentric margin, 1e-9 x diameter
// distance) sit twelve orders of magnitude above one rounding, so labels are
// the reference's (tests/test_gpu_meshgen.py checks them element for element).
#include <algorithm>

#include "common.cuh"

namespace hf {
namespace mg {

constexpr int LOC_T = 128;
constexpr int RAYW = 16;  // doubles per (direction, triangle) row

__device__ __forceinline__ double dot3_blas(double p0, double p1, double p2, const double* h) {
  double a = __dmul_rn(p0, h[0]);
  a = fma(p1, h[1], a);
  return fma(p2, h[2], a);
}

// One _cast pass of one point against one surface along one direction
// (geometry.py:203-249).  Returns parity in bit 0, suspect in bit 1, on-surface in bit 2.
__device__ __forceinline__ int cast_one(double p0, double p1, double p2, const double* __restrict__ rows,
                                        int nt, double tol) {
  const double eb = 1e-10;
  const double one_p = 1.0 + eb, one_m = 1.0 - eb;
  int parity = 0;
  bool suspect = false, on = false;
  for (int j = 0; j < nt; ++j) {
    const double* r = rows + (size_t)j * RAYW;
    const double hh[3] = {__ldg(r + 0), __ldg(r + 1), __ldg(r + 2)};
    const double kk[3] = {__ldg(r + 3), __ldg(r + 4), __ldg(r + 5)};
    const double nn[3] = {__ldg(r + 6), __ldg(r + 7), __ldg(r + 8)};
    const double c_h = __ldg(r + 9), c_k = __ldg(r + 10), c_n = __ldg(r + 11);
    const double f = __ldg(r + 12), par = __ldg(r + 13), tn = __ldg(r + 14);
    const double u = __dmul_rn(__dsub_rn(dot3_blas(p0, p1, p2, hh), c_h), f);
    const double v = __dmul_rn(__dsub_rn(dot3_blas(p0, p1, p2, kk), c_k), f);
    const double dn = __dsub_rn(dot3_blas(p0, p1, p2, nn), c_n);
    const double t = __dmul_rn(dn, f);
    const double w = __dadd_rn(u, v);
    const bool ok = par == 0.0;
    const bool in_tri = (u >= -eb) && (v >= -eb) && (w <= one_p);
    const bool strict = (u > eb) && (v > eb) && (w < one_m);
    parity ^= (ok && strict && t > tol) ? 1 : 0;
    on |= ok && in_tri && fabs(t) <= tol;
    suspect |= ok && in_tri && !strict && t > tol;
    suspect |= !ok && fabs(dn) <= tn;
  }
  return parity | (suspect ? 2 : 0) | (on ? 4 : 0);
}

// SurfaceMesh.contains for one point (geometry.py:147-184).
__device__ bool surface_contains(const hf_segmentation& sg, int s, double p0, double p1, double p2) {
  const double* b = sg.box + (size_t)s * 8;
  const double tol = b[6];
  if (!(p0 >= b[0] - tol && p1 >= b[1] - tol && p2 >= b[2] - tol && p0 <= b[3] + tol &&
        p1 <= b[4] + tol && p2 <= b[5] + tol))
    return false;
  const int t0 = sg.tri_off[s], nt = sg.tri_off[s + 1] - t0;
  const double* base = sg.rays + (size_t)t0 * sg.n_dir * RAYW;
  int last = 0;
  for (int d = 0; d < sg.n_dir; ++d) {
    const int r = cast_one(p0, p1, p2, base + (size_t)d * nt * RAYW, nt, tol);
    if (r & 4) return true;         // on the surface counts as inside
    if (!(r & 2)) return r & 1;     // settled by this direction
    last = r & 1;                   // grazed: retry with the next direction
  }
  return last;  // every direction grazed: the last parity (geometry.py:179-180)
}

__global__ void __launch_bounds__(LOC_T) k_locate(hf_segmentation sg, const double* __restrict__ pts,
                                                  int np_, int32_t* __restrict__ labels) {
  const int i = blockIdx.x * LOC_T + threadIdx.x;
  if (i >= np_) return;
  const double p0 = pts[3 * (size_t)i], p1 = pts[3 * (size_t)i + 1], p2 = pts[3 * (size_t)i + 2];
  int lab = -1;
  for (int k = 0; k < sg.n_comp && lab < 0; ++k)
    for (int s = sg.comp_surf[k]; s < sg.comp_surf[k + 1]; ++s)
      if (surface_contains(sg, s, p0, p1, p2)) {
        lab = k;
        break;
      }
  labels[i] = lab;
}

// ---------------------------------------------------------------- grid
// _KUHN_TETS (meshgen.py:23-40) and corner offsets j -> (j&1, j>>1&1, j>>2&1).
__constant__ int c_kuhn[6][4] = {{0, 1, 3, 7}, {0, 1, 7, 5}, {0, 2, 7, 3},
                                 {0, 2, 6, 7}, {0, 4, 5, 7}, {0, 4, 7, 6}};

__global__ void k_grid_tets(const double* __restrict__ xs, const double* __restrict__ ys,
                            const double* __restrict__ zs, int nx, int ny, int nz,
                            int32_t* __restrict__ tetra, double* __restrict__ cent) {
  const long e = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long ncube = (long)nx * ny * nz;
  if (e >= ncube * 6) return;
  const long cube = e / 6;
  const int k = (int)(e % 6);
  const int cx = (int)(cube % nx), cy = (int)((cube / nx) % ny), cz = (int)(cube / ((long)nx * ny));
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int j = c_kuhn[k][q];
    const int ix = cx + (j & 1), iy = cy + ((j >> 1) & 1), iz = cz + ((j >> 2) & 1);
    tetra[4 * e + q] = ix + (nx + 1) * (iy + (ny + 1) * iz);
    const double x = xs[ix], y = ys[iy], z = zs[iz];
    if (q == 0) {
      s0 = x;
      s1 = y;
      s2 = z;
    } else {  // ((a + b) + c) + d, as numpy's mean over the corner axis
      s0 = __dadd_rn(s0, x);
      s1 = __dadd_rn(s1, y);
      s2 = __dadd_rn(s2, z);
    }
  }
  cent[3 * e] = s0 * 0.25;
  cent[3 * e + 1] = s1 * 0.25;
  cent[3 * e + 2] = s2 * 0.25;
}

__global__ void k_keep_flags(const int32_t* __restrict__ lab, int m, int32_t* __restrict__ flag) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < m) flag[e] = lab[e] >= 0;
}

__global__ void k_mark_used(const int32_t* __restrict__ tetra, const int32_t* __restrict__ lab, int m,
                            int32_t* __restrict__ used) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m || lab[e] < 0) return;
#pragma unroll
  for (int q = 0; q < 4; ++q) used[tetra[4 * (size_t)e + q]] = 1;  // benign same-value race
}

// np.unique(tetra, return_inverse=True): used grid nodes in ascending order, and
// the element corners renumbered to their rank (meshgen.py:229-232).
__global__ void k_compact_tets(const int32_t* __restrict__ tetra, const int32_t* __restrict__ lab,
                               const int32_t* __restrict__ epos, const int32_t* __restrict__ nid,
                               int m, int32_t* __restrict__ tout, int32_t* __restrict__ lout) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m || lab[e] < 0) return;
  const int o = epos[e];
#pragma unroll
  for (int q = 0; q < 4; ++q) tout[4 * (size_t)o + q] = nid[tetra[4 * (size_t)e + q]];
  lout[o] = lab[e];
}

__global__ void k_compact_nodes(const int32_t* __restrict__ used, const int32_t* __restrict__ nid,
                                int ngrid, int nx, int ny, const double* __restrict__ xs,
                                const double* __restrict__ ys, const double* __restrict__ zs,
                                double* __restrict__ nodes) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= ngrid || !used[g]) return;
  const int ix = g % (nx + 1), iy = (g / (nx + 1)) % (ny + 1), iz = g / ((nx + 1) * (ny + 1));
  const size_t o = nid[g];
  nodes[3 * o] = xs[ix];
  nodes[3 * o + 1] = ys[iy];
  nodes[3 * o + 2] = zs[iz];
}

// _apply_priorities (meshgen.py:247-269), one thread per element.
__global__ void k_priorities(const int32_t* __restrict__ tetra, int m, const int32_t* __restrict__ nl,
                             const int32_t* __restrict__ pri, int32_t* __restrict__ labels) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m) return;
  int l[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) l[q] = nl[tetra[4 * (size_t)e + q]];
  const int first = max(max(l[0], l[1]), max(l[2], l[3]));
  bool multi = false;
#pragma unroll
  for (int q = 0; q < 4; ++q) multi |= (l[q] != first) && (l[q] >= 0);
  if (!multi || first < 0) return;
  const int cur = labels[e];
  int best = pri[cur];
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (l[q] >= 0) best = min(best, pri[l[q]]);
  if (pri[cur] == best) return;
  int pick = 0x7fffffff;
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (l[q] >= 0 && pri[l[q]] == best) pick = min(pick, l[q]);
  labels[e] = pick;  // cur has pri > best, so it is never the pick
}

}  // namespace mg
}  // namespace hf

using namespace hf;

extern "C" int hf_locate(const hf_segmentation* seg, const double* points, int32_t n_points,
                         int32_t* labels, void* stream) {
  if (!seg || n_points < 0 || (n_points > 0 && (!points || !labels)) || seg->n_comp < 0 ||
      seg->n_dir < 1) {
    set_error("hf_locate: bad argument");
    return HF_ERR_ARG;
  }
  if (n_points == 0) return HF_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  mg::k_locate<<<(n_points + mg::LOC_T - 1) / mg::LOC_T, mg::LOC_T, 0, s>>>(*seg, points, n_points,
                                                                          labels);
  count_launches(1);
  HF_LAUNCH_CHECK();
  return HF_OK;
}

extern "C" int hf_grid_tets(const double* xs, const double* ys, const double* zs, int32_t nx,
                            int32_t ny, int32_t nz, int32_t* tetra, double* centroids, void* stream) {
  const long m = 6L * nx * ny * nz;
  if (!xs || !ys || !zs || !tetra || !centroids || nx < 1 || ny < 1 || nz < 1 || m >= (1L << 31) ||
      (long)(nx + 1) * (ny + 1) * (nz + 1) >= (1L << 31)) {
    set_error("hf_grid_tets: bad argument");
    return HF_ERR_ARG;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  mg::k_grid_tets<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(xs, ys, zs, nx, ny, nz, tetra,
                                                               centroids);
  count_launches(1);
  HF_LAUNCH_CHECK();
  return HF_OK;
}

extern "C" size_t hf_mesh_compact_workspace_bytes(int32_t m_all, int32_t n_grid) {
  const size_t a = (size_t)(m_all > 0 ? m_all : 0), g = (size_t)(n_grid > 0 ? n_grid : 0);
  return (2 * a + 2 * g + scan_scratch_elems((int32_t)a) + scan_scratch_elems((int32_t)g) + 16) *
             sizeof(int32_t) + 8 * 256;
}

extern "C" int hf_mesh_compact(const int32_t* tetra_all, const int32_t* cent_label, int32_t m_all,
                               const double* xs, const double* ys, const double* zs, int32_t nx,
                               int32_t ny, int32_t nz, int32_t* tetra_out, int32_t* labels_out,
                               double* nodes_out, int64_t* m_out, int64_t* n_out, void* ws,
                               size_t ws_bytes, void* stream) {
  const long ngl = (long)(nx + 1) * (ny + 1) * (nz + 1);
  if (!tetra_all || !cent_label || !tetra_out || !labels_out || !nodes_out || !m_out || !n_out ||
      !ws || m_all < 0 || ngl >= (1L << 31)) {
    set_error("hf_mesh_compact: bad argument");
    return HF_ERR_ARG;
  }
  const int ng = (int)ngl;
  if (ws_bytes < hf_mesh_compact_workspace_bytes(m_all, ng)) {
    set_error("hf_mesh_compact: workspace too small");
    return HF_ERR_WORKSPACE;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  Carve cv{reinterpret_cast<char*>(ws), 0, ws_bytes};
  int32_t* flag = cv.take<int32_t>((size_t)m_all + 1);
  int32_t* epos = cv.take<int32_t>((size_t)m_all + 1);
  int32_t* used = cv.take<int32_t>((size_t)ng + 1);
  int32_t* nid = cv.take<int32_t>((size_t)ng + 1);
  int32_t* scr = cv.take<int32_t>(std::max(scan_scratch_elems(m_all), scan_scratch_elems(ng)));
  int32_t* tot = cv.take<int32_t>(4);
  const unsigned gm = (unsigned)((m_all + 255) / 256), gg = (unsigned)((ng + 255) / 256);
  if (m_all > 0) mg::k_keep_flags<<<gm, 256, 0, s>>>(cent_label, m_all, flag);
  if (int rc = exclusive_scan_i32(flag, epos, m_all, scr, tot, s)) return rc;
  HF_CUDA(cudaMemsetAsync(used, 0, sizeof(int32_t) * ng, s));
  if (m_all > 0) mg::k_mark_used<<<gm, 256, 0, s>>>(tetra_all, cent_label, m_all, used);
  if (int rc = exclusive_scan_i32(used, nid, ng, scr, tot + 1, s)) return rc;
  if (m_all > 0)
    mg::k_compact_tets<<<gm, 256, 0, s>>>(tetra_all, cent_label, epos, nid, m_all, tetra_out,
                                          labels_out);
  mg::k_compact_nodes<<<gg, 256, 0, s>>>(used, nid, ng, nx, ny, xs, ys, zs, nodes_out);
  count_launches(4);
  HF_LAUNCH_CHECK();
  int32_t h[2] = {0, 0};
  HF_CUDA(cudaMemcpyAsync(h, tot, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  HF_CUDA(cudaStreamSynchronize(s));
  *m_out = h[0];
  *n_out = h[1];
  return HF_OK;
}

extern "C" int hf_apply_priorities(const int32_t* tetra, int32_t m, const int32_t* node_label,
                                   const int32_t* priority, int32_t* labels, void* stream) {
  if (m < 0 || (m > 0 && (!tetra || !node_label || !priority || !labels))) {
    set_error("hf_apply_priorities: bad argument");
    return HF_ERR_ARG;
  }
  if (m == 0) return HF_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  mg::k_priorities<<<(m + 255) / 256, 256, 0, s>>>(tetra, m, node_label, priority, labels);
  count_launches(1);
  HF_LAUNCH_CHECK();
  return HF_OK;
}
