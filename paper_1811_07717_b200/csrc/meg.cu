// MEG lead field on the same FEM system (BASELINE.json configs[2], C3).
//
// The reference has no MEG: this is the standard FEM reciprocity
// formulation, parity unpinned.  With u = -A^-1 G q the potential of a dipole
// source (the EEG path's source matrix G, fem.py:391-422, whose sign makes the
// EEG lead field -R M^-1 T'G, leadfield.py:129), the flux of the
// secondary currents -sigma grad u through coil c (position r_c, normal n_c) is
//   B_sec,c = sum_j u_j S[c, j],
//   S[c, j] = -mu0/4pi sum_{e ∋ j} sigma_e V_e grad(phi_j)|_e . ((r_c - x_e) x n_c) / |r_c - x_e|^3
// (one-point quadrature at the element centroid x_e), so the MEG transfer
// matrix is T_meg = A^-1 S' — one RHS column per sensor through the same
// multi-RHS PCG as the electrodes — and the lead field is
//   L = L_primary - T_meg' G,
//   L_primary[s, 3k + a] = mu0/4pi sum_{c in s} w_c ((r_c - r_k) x n_c)_a / |r_c - r_k|^3.
// A sensor is a weighted set of point coils (magnetometer: one coil; planar
// gradiometer: two coils, weights +-1/baseline).
//
//   k_meg_elem     per element: centroid and sigma V grad(phi_a), a = 0..3
//   k_meg_rhs      S' (n x ncols row-major) node by node over the node -> element
//                  incidence lists, elements in ascending order (deterministic)
//   k_meg_primary  L_primary (ncols x 3 S)
#include <math.h>

#include "common.cuh"

namespace hf {
namespace asmb {
int build_incidence(const int32_t* conn, int width, int count, int n, int32_t* cnt, int32_t* off,
                    int32_t* cur, int32_t* inc, int32_t* scratch, int32_t* tot, cudaStream_t s);
}
namespace meg {

constexpr double MU0_4PI = 1e-7;
constexpr int EW = 16;  // doubles per element record: centroid (3), sigma V grad phi_a (4 x 3), pad

__global__ void k_meg_elem(const double* __restrict__ nodes, const int32_t* __restrict__ tetra,
                           const double* __restrict__ sigma, int m, double* __restrict__ rec) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m) return;
  double p[4][3];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int r = 0; r < 3; ++r) p[a][r] = nodes[3 * (size_t)tetra[4 * (size_t)e + a] + r];
  double J[3][3];  // columns p_k - p_0 (fem.py:33-35)
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k) J[r][k] = p[k + 1][r] - p[0][r];
  const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                     J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                     J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
  const double inv = 1.0 / det;
  double g[4][3];  // rows of J^-1 are grad phi_1..3; grad phi_0 = -sum
  g[1][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) * inv;
  g[1][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * inv;
  g[1][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * inv;
  g[2][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) * inv;
  g[2][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * inv;
  g[2][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * inv;
  g[3][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) * inv;
  g[3][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * inv;
  g[3][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * inv;
#pragma unroll
  for (int k = 0; k < 3; ++k) g[0][k] = -(g[1][k] + g[2][k] + g[3][k]);
  const double w = sigma[e] * det / 6.0;  // sigma_e V_e
  double* o = rec + (size_t)e * EW;
#pragma unroll
  for (int r = 0; r < 3; ++r) o[r] = 0.25 * (p[0][r] + p[1][r] + p[2][r] + p[3][r]);
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int k = 0; k < 3; ++k) o[3 + 3 * a + k] = w * g[a][k];
}

// One block per node; thread t handles sensor columns t + 128 i (i < MAXC).
// coils: {rx, ry, rz, nx, ny, nz, weight, pad} x n_coils; column s owns coils
// [coil_ptr[s], coil_ptr[s+1]).  The node's incidences (ascending element
// order) are staged 64 at a time in shared memory.
constexpr int RHS_THREADS = 128, MAXC = 4, INC_CHUNK = 64;

__global__ void __launch_bounds__(RHS_THREADS)
    k_meg_rhs(int n, int ground, const int32_t* __restrict__ off, const int32_t* __restrict__ cnt,
              const int32_t* __restrict__ inc, const double* __restrict__ rec,
              const double* __restrict__ coils, const int32_t* __restrict__ coil_ptr, int ncols,
              double* __restrict__ Bt, int ldb) {
  const int j = blockIdx.x;
  __shared__ double s_x[INC_CHUNK][3];  // element centroids
  __shared__ double s_g[INC_CHUNK][3];  // sigma V grad phi_j on the element
  const int deg = cnt[j], o0 = off[j];
  double acc[MAXC];
#pragma unroll
  for (int t = 0; t < MAXC; ++t) acc[t] = 0.0;
  for (int q0 = 0; q0 < deg; q0 += INC_CHUNK) {
    const int nq = min(INC_CHUNK, deg - q0);
    __syncthreads();
    if (threadIdx.x < nq) {
      const int id = inc[o0 + q0 + threadIdx.x];  // element * 4 + local corner
      const double* r = rec + (size_t)(id >> 2) * EW;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        s_x[threadIdx.x][k] = r[k];
        s_g[threadIdx.x][k] = r[3 + 3 * (id & 3) + k];
      }
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < MAXC; ++t) {
      const int s = threadIdx.x + RHS_THREADS * t;
      if (s >= ncols) break;
      for (int c = coil_ptr[s]; c < coil_ptr[s + 1]; ++c) {
        const double* cl = coils + 8 * (size_t)c;
        double sub = 0.0;
        for (int q = 0; q < nq; ++q) {
          const double dx = cl[0] - s_x[q][0], dy = cl[1] - s_x[q][1], dz = cl[2] - s_x[q][2];
          const double r2 = dx * dx + dy * dy + dz * dz;
          const double ir3 = rsqrt(r2) / r2;
          // ((r_c - x_e) x n_c) . g
          const double cx = dy * cl[5] - dz * cl[4], cy = dz * cl[3] - dx * cl[5],
                       cz = dx * cl[4] - dy * cl[3];
          sub += (cx * s_g[q][0] + cy * s_g[q][1] + cz * s_g[q][2]) * ir3;
        }
        acc[t] += cl[6] * sub;
      }
    }
  }
#pragma unroll
  for (int t = 0; t < MAXC; ++t) {
    const int s = threadIdx.x + RHS_THREADS * t;
    if (s < ncols) Bt[(size_t)j * ldb + s] = (j == ground) ? 0.0 : -MU0_4PI * acc[t];
  }
}

__global__ void k_meg_primary(const double* __restrict__ coils, const int32_t* __restrict__ coil_ptr,
                              int ncols, const double* __restrict__ pos, int S,
                              double* __restrict__ Lp) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;  // source
  const int s = blockIdx.y;                             // sensor column
  if (k >= S) return;
  const double px = pos[3 * (size_t)k], py = pos[3 * (size_t)k + 1], pz = pos[3 * (size_t)k + 2];
  double a[3] = {0.0, 0.0, 0.0};
  for (int c = coil_ptr[s]; c < coil_ptr[s + 1]; ++c) {
    const double* cl = coils + 8 * (size_t)c;
    const double dx = cl[0] - px, dy = cl[1] - py, dz = cl[2] - pz;
    const double r2 = dx * dx + dy * dy + dz * dz;
    const double f = cl[6] * MU0_4PI * rsqrt(r2) / r2;
    a[0] += f * (dy * cl[5] - dz * cl[4]);
    a[1] += f * (dz * cl[3] - dx * cl[5]);
    a[2] += f * (dx * cl[4] - dy * cl[3]);
  }
  double* o = Lp + (size_t)s * 3 * S + 3 * (size_t)k;
  o[0] = a[0];
  o[1] = a[1];
  o[2] = a[2];
}

struct Ws {
  int32_t *cnt, *off, *cur, *inc, *scratch, *tot;
  double* rec;
  size_t bytes;
};

inline Ws carve(void* base, int n, int m) {
  Carve cv{reinterpret_cast<char*>(base), 0, ~size_t(0)};
  Ws w;
  w.cnt = cv.take<int32_t>((size_t)n + 1);
  w.off = cv.take<int32_t>((size_t)n + 1);
  w.cur = cv.take<int32_t>((size_t)n + 1);
  w.inc = cv.take<int32_t>((size_t)4 * m + 1);
  w.scratch = cv.take<int32_t>(scan_scratch_elems(n));
  w.tot = cv.take<int32_t>(8);
  w.rec = cv.take<double>((size_t)m * EW);
  w.bytes = cv.used + 256;
  return w;
}

}  // namespace meg
}  // namespace hf

using namespace hf;

extern "C" size_t hf_meg_workspace_bytes(int32_t n, int32_t m) { return meg::carve(nullptr, n, m).bytes; }

extern "C" int hf_meg_rhs(const double* nodes, const int32_t* tetra, const double* sigma, int32_t n,
                          int32_t m, int32_t ground, const double* coils, const int32_t* coil_ptr,
                          int32_t ncols, double* Bt, int32_t ldb, void* ws, size_t ws_bytes,
                          void* stream) {
  if (!nodes || !tetra || !sigma || !coils || !coil_ptr || !Bt || !ws || n <= 0 || m <= 0 ||
      ncols <= 0 || ncols > meg::RHS_THREADS * meg::MAXC || ldb < ncols) {
    set_error("hf_meg_rhs: bad argument");
    return HF_ERR_ARG;
  }
  if (ws_bytes < hf_meg_workspace_bytes(n, m)) {
    set_error("hf_meg_rhs: workspace too small");
    return HF_ERR_WORKSPACE;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  meg::Ws w = meg::carve(ws, n, m);
  meg::k_meg_elem<<<(m + 255) / 256, 256, 0, s>>>(nodes, tetra, sigma, m, w.rec);
  HF_LAUNCH_CHECK();
  count_launches(1);
  if (int rc = asmb::build_incidence(tetra, 4, m, n, w.cnt, w.off, w.cur, w.inc, w.scratch, w.tot, s))
    return rc;
  meg::k_meg_rhs<<<n, meg::RHS_THREADS, 0, s>>>(n, ground, w.off, w.cnt, w.inc, w.rec, coils, coil_ptr, ncols, Bt,
                                   ldb);
  HF_LAUNCH_CHECK();
  count_launches(1);
  return HF_OK;
}

extern "C" int hf_meg_primary(const double* coils, const int32_t* coil_ptr, int32_t ncols,
                              const double* positions, int32_t n_sources, double* Lp, void* stream) {
  if (!coils || !coil_ptr || !positions || !Lp || ncols <= 0 || n_sources < 0) {
    set_error("hf_meg_primary: bad argument");
    return HF_ERR_ARG;
  }
  if (n_sources == 0) return HF_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  dim3 grid((n_sources + 127) / 128, ncols);
  meg::k_meg_primary<<<grid, 128, 0, s>>>(coils, coil_ptr, ncols, positions, n_sources, Lp);
  HF_LAUNCH_CHECK();
  count_launches(1);
  return HF_OK;
}
