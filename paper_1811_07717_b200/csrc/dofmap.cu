// Nearest-centre partition of the EIT conductivity DOFs on the device —
// SURVEY.md §8f "next" row #3, the owner = argmin(d, axis=1) step of
// build_dof_map (leadfield.py:96-99).  The reference materialises the
// (E, m, 3) difference array (459 GiB at C4); here every element centroid is
// compared with every centre straight from shared memory.
//
// Bit parity with numpy: d_ij = sqrt((dx*dx + dy*dy) + dz*dz) with
// dx = p_x - c_x, each operation rounded separately (np.linalg.norm's
// add.reduce of x*x over the 3-axis, numpy/linalg/_linalg.py `norm`), and the
// FIRST index among equal d wins (np.argmin).  The square root is only
// evaluated when the squared distance drops below the best one seen so far:
// sqrt is monotone, so a larger square can never give a strictly smaller root,
// and a smaller square whose root ties the current minimum keeps the earlier
// index exactly as argmin does.
#include "common.cuh"

namespace hf {
namespace dof {

constexpr int NC_T = 256;    // threads per block
constexpr int NC_PPT = 2;    // points per thread (each centre read from smem serves both)
constexpr int NC_TILE = 2048;  // centres per shared-memory tile (48 KB)

__global__ void __launch_bounds__(NC_T) k_nearest(const double* __restrict__ pts, int E,
                                                 const double* __restrict__ ctr, int m,
                                                 int32_t* __restrict__ owner,
                                                 double* __restrict__ dist) {
  __shared__ double cx[NC_TILE], cy[NC_TILE], cz[NC_TILE];
  double px[NC_PPT], py[NC_PPT], pz[NC_PPT], bs[NC_PPT], br[NC_PPT];
  int bi[NC_PPT];
  const size_t base = (size_t)blockIdx.x * NC_T * NC_PPT + threadIdx.x;
#pragma unroll
  for (int u = 0; u < NC_PPT; ++u) {
    const size_t i = base + (size_t)u * NC_T;
    const bool ok = i < (size_t)E;
    px[u] = ok ? pts[3 * i] : 0.0;
    py[u] = ok ? pts[3 * i + 1] : 0.0;
    pz[u] = ok ? pts[3 * i + 2] : 0.0;
    bs[u] = __longlong_as_double(0x7ff0000000000000LL);  // +inf
    br[u] = bs[u];
    bi[u] = 0;
  }
  for (int t0 = 0; t0 < m; t0 += NC_TILE) {
    const int nt = min(NC_TILE, m - t0);
    __syncthreads();
    for (int j = threadIdx.x; j < nt; j += NC_T) {
      cx[j] = ctr[3 * (size_t)(t0 + j)];
      cy[j] = ctr[3 * (size_t)(t0 + j) + 1];
      cz[j] = ctr[3 * (size_t)(t0 + j) + 2];
    }
    __syncthreads();
#pragma unroll 4
    for (int j = 0; j < nt; ++j) {
      const double x = cx[j], y = cy[j], z = cz[j];
#pragma unroll
      for (int u = 0; u < NC_PPT; ++u) {
        const double dx = __dsub_rn(px[u], x), dy = __dsub_rn(py[u], y), dz = __dsub_rn(pz[u], z);
        const double s =
            __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
        if (s < bs[u]) {  // rare: a new smallest square
          bs[u] = s;
          const double r = __dsqrt_rn(s);
          if (r < br[u]) {
            br[u] = r;
            bi[u] = t0 + j;
          }
        }
      }
    }
  }
#pragma unroll
  for (int u = 0; u < NC_PPT; ++u) {
    const size_t i = base + (size_t)u * NC_T;
    if (i < (size_t)E) {
      owner[i] = bi[u];
      if (dist != nullptr) dist[i] = br[u];
    }
  }
}

}  // namespace dof
}  // namespace hf

using namespace hf;

extern "C" int hf_nearest_center(const double* points, int32_t n_points, const double* centers,
                                 int32_t n_centers, int32_t* owner, double* dist, void* stream) {
  if (n_points < 0 || n_centers <= 0 || !centers || (n_points > 0 && (!points || !owner))) {
    set_error("hf_nearest_center: bad argument");
    return HF_ERR_ARG;
  }
  if (n_points == 0) return HF_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int per = dof::NC_T * dof::NC_PPT;
  const int nb = (n_points + per - 1) / per;
  dof::k_nearest<<<nb, dof::NC_T, 0, s>>>(points, n_points, centers, n_centers, owner, dist);
  HF_LAUNCH_CHECK();
  count_launches(1);
  return HF_OK;
}

// ---------------------------------------------------------------- DOF map partition (next row #3)
// The host steps of build_dof_map (leadfield.py:80-101) around the nearest-centre
// search, on the device: element centroids with numpy's rounding
// (mean over 4 corners = (((a + b) + c) + d) / 4, meshgen.py:TetMesh.centroids),
// and the partition sets = cand[owner == k] for every k, as one stable radix sort
// of the candidates by owner (ascending element order inside each set, as the
// reference's boolean mask gives) plus the set offsets.
#include <cub/device/device_radix_sort.cuh>

namespace hf {
namespace dof {

__global__ void k_tet_centroids(const double* __restrict__ nodes, const int32_t* __restrict__ tetra,
                                const int32_t* __restrict__ elems, int count,
                                double* __restrict__ cent) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const size_t e = elems ? (size_t)elems[i] : (size_t)i;
  const int32_t* t = tetra + 4 * e;
  const double* a = nodes + 3 * (size_t)t[0];
  const double* b = nodes + 3 * (size_t)t[1];
  const double* c = nodes + 3 * (size_t)t[2];
  const double* d = nodes + 3 * (size_t)t[3];
#pragma unroll
  for (int r = 0; r < 3; ++r)
    cent[3 * (size_t)i + r] = __dmul_rn(__dadd_rn(__dadd_rn(__dadd_rn(a[r], b[r]), c[r]), d[r]), 0.25);
}

__global__ void k_set_bounds(const int32_t* __restrict__ sorted_owner, int n, int n_sets,
                             int32_t* __restrict__ ptr) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k > n_sets) return;
  int lo = 0, hi = n;  // first position with owner >= k
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (sorted_owner[mid] < k) lo = mid + 1; else hi = mid;
  }
  ptr[k] = lo;
}

}  // namespace dof
}  // namespace hf

extern "C" int hf_tet_centroids(const double* nodes, const int32_t* tetra, const int32_t* elems,
                                int32_t count, double* cent, void* stream) {
  if (count < 0 || (count > 0 && (!nodes || !tetra || !cent))) {
    set_error("hf_tet_centroids: bad argument");
    return HF_ERR_ARG;
  }
  if (count == 0) return HF_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  dof::k_tet_centroids<<<(count + 255) / 256, 256, 0, s>>>(nodes, tetra, elems, count, cent);
  HF_LAUNCH_CHECK();
  count_launches(1);
  return HF_OK;
}

static size_t partition_sort_bytes(int32_t n) {
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, (const int32_t*)nullptr, (int32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, n);
  return tmp;
}

extern "C" size_t hf_dof_partition_workspace_bytes(int32_t n_cand) {
  return partition_sort_bytes(n_cand) + 4 * ((size_t)n_cand + 64) + 512;
}

extern "C" int hf_dof_partition(const int32_t* cand, const int32_t* owner, int32_t n_cand,
                                int32_t n_sets, int32_t* sorted_cand, int32_t* set_ptr, void* ws,
                                size_t ws_bytes, void* stream) {
  if (!cand || !owner || !sorted_cand || !set_ptr || !ws || n_cand < 0 || n_sets < 1) {
    set_error("hf_dof_partition: bad argument");
    return HF_ERR_ARG;
  }
  if (ws_bytes < hf_dof_partition_workspace_bytes(n_cand)) {
    set_error("hf_dof_partition: workspace too small");
    return HF_ERR_WORKSPACE;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  Carve cv{reinterpret_cast<char*>(ws), 0, ws_bytes};
  int32_t* sorted_owner = cv.take<int32_t>((size_t)n_cand + 1);
  size_t tmp_bytes = partition_sort_bytes(n_cand);
  void* tmp = cv.take<char>(tmp_bytes + 1);
  int bits = 1;
  while ((1 << bits) <= n_sets && bits < 31) ++bits;
  HF_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, owner, sorted_owner, cand, sorted_cand,
                                          n_cand, 0, bits, s));
  dof::k_set_bounds<<<(n_sets + 256) / 256, 256, 0, s>>>(sorted_owner, n_cand, n_sets, set_ptr);
  HF_LAUNCH_CHECK();
  count_launches(2);
  return HF_OK;
}
