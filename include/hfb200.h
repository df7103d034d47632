/*
 * hfb200.h — C ABI of the B200-native FEM lead-field engine.
 *
 * One shared library (paper_1811_07717_b200/_lib/libhfb200.so) exports the
 * entry points below.  Every pointer argument marked "device" is a CUDA device
 * pointer on the current device; "host" pointers are ordinary host memory.
 * `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 * No function allocates device memory: callers size the workspace with the
 * matching *_workspace_bytes() query and pass it in.  Every function returns
 * an hf_status; hf_last_error() gives a human-readable message for the last
 * failure on the calling thread.
 *
 * Each entry point replaces one interface of the reference package
 * `headfem` (files relative to /root/reference/pkg/src/headfem/):
 *
 *   hf_ldp                 solver.py:50-61     ldp(A)
 *   hf_csr_bandwidth       (internal)          gather reach of A, sizes the PCG batch width
 *   hf_pcg_multi           solver.py:64-111    pcg_solve(A, b, cfg), one column per RHS
 *                          solver.py:114-141   transfer_matrix(A, B, cfg, threads)
 *   hf_pcg_stream          solver.py:114-141   transfer_matrix with columns streamed through kp slots
 *   hf_pcg_profile         (bench)             per-kernel CUDA-event timing of a PCG round
 *   hf_csr_prune_*         (internal)          zero-free copy of A for the SpMM
 *   hf_p1_blocks           fem.py:31-93        element_gradients + stiffness_blocks
 *   hf_p1_assemble_*       fem.py:96-109       _scatter_blocks / volume_stiffness
 *                          fem.py:197-224      assemble_A (+ electrode terms, _ground)
 *   hf_response_matrix     leadfield.py:104-109 electrode_response: M = C - B'T (column block)
 *   hf_lf_tail             leadfield.py:122-134 eeg_leadfield: L = W (G'T)'  with W = -R M^-1
 *   hf_dense_lf            leadfield.py:230-237 eit_leadfield column blocks  W Q[p]'
 *   hf_eit_sens            leadfield.py:179-207 _dof_sensitivities: Q[p,m,:] = T' K_m u_p
 *   hf_csr_dense           leadfield.py:223    eit_leadfield's pattern right-hand sides B V
 *   hf_boundary_faces      meshgen.py:101-134  TetMesh.boundary_triangles
 *   hf_whitney_gt          fem.py:291-422      assemble_G (Whitney source matrix), as G'
 *   hf_nearest_center      leadfield.py:96-99  build_dof_map: owner = argmin ||c_i - centre_j||
 *                          fem.py:157-173      ElectrodeSet.from_centers (nearest centre + distance)
 *   hf_triangle_centroids  fem.py:163          boundary-triangle centroids of from_centers
 *   hf_tet_centroids       leadfield.py:96     build_dof_map's element centroids
 *   hf_dof_partition       leadfield.py:99-100 build_dof_map's sets: cand[owner == k] for every k
 *   hf_ground_node         fem.py:188-194      ground_node
 *   hf_locate              geometry.py:147-374 Segmentation.locate (ray-parity point location)
 *   hf_grid_tets           meshgen.py:205-223  generate_mesh's Kuhn grid + element centroids
 *   hf_mesh_compact        meshgen.py:224-235  keep labelled elements, np.unique node renumbering
 *   hf_apply_priorities    meshgen.py:247-269  _apply_priorities
 *   hf_meg_rhs             (none: SPEC.md:8)   MEG transfer right-hand sides S' (C3, parity unpinned)
 *   hf_meg_primary         (none: SPEC.md:8)   MEG primary-field lead field (C3, parity unpinned)
 *
 * See INTEGRATION.md for the ctypes binding the reference would use.
 */
#ifndef HFB200_H
#define HFB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HF_OK = 0,
  HF_ERR_ARG = 1,          /* bad argument (shape, null pointer, unsupported width) */
  HF_ERR_CUDA = 2,         /* CUDA runtime error (message in hf_last_error) */
  HF_ERR_WORKSPACE = 3,    /* workspace too small */
  HF_ERR_CAPACITY = 4,     /* a node touches more elements than the row builder supports */
  HF_ERR_INTERNAL = 5      /* solver control did not terminate */
} hf_status;

/* Compressed sparse rows; int32 indices as scipy produces them (solver.py:55,87). */
typedef struct {
  int32_t n_rows;
  int32_t n_cols;
  int64_t nnz;
  const int32_t* indptr;   /* device, n_rows+1 */
  const int32_t* indices;  /* device, nnz, sorted within each row */
  const double* val;       /* device, nnz */
} hf_csr;

/* Per-column terminal states reported by hf_pcg_multi. */
enum {
  HF_COL_DONE = 2,         /* converged: true residual <= tol (solver.py:94-100) */
  HF_COL_FAILED = 3,       /* max_iter reached (solver.py:108-111) */
  HF_COL_ZERO = 4,         /* ||b|| == 0: x = 0, 0 iterations (solver.py:75-76) */
  HF_COL_FROZEN = 5        /* replay stopped at freeze_at[j] (best-iterate recovery) */
};

/* Version / diagnostics. */
const char* hf_version(void);
const char* hf_last_error(void);
int hf_device_sm_count(int32_t* sm_count);
/* Kernels launched by this library so far (graph launches count their nodes). */
long long hf_launch_count(void);
/* Deterministic int32 exclusive scan of n counts into out (any n >= 0);
 * *total (device int32) receives the sum.  This is the CSR row-pointer step
 * (the cumsum inside scipy's coo -> csr conversion that fem.py:122-124 and
 * meshgen.py:114-130 go through).  Scratch: hf_scan_workspace_bytes(n). */
size_t hf_scan_workspace_bytes(int32_t n);
int hf_exclusive_scan_i32(const int32_t* in, int32_t* out, int32_t n, int32_t* total, void* ws,
                          size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------- solver */

/* d_i = sum_j |a_ij|  (solver.py:50-61).  zero_count is one device int32 of
 * scratch; *n_zero_rows (host) receives the number of rows with d_i == 0 (the
 * caller raises SingularPreconditionerError).  Synchronises `stream`. */
int hf_ldp(const hf_csr* A, double* d, int32_t* zero_count, int32_t* n_zero_rows, void* stream);

/* Matrix bandwidth max_i max(i - first col, last col - i) of a CSR with sorted
 * rows (the reach of the SpMM's gathers; the solver sizes its batch width so
 * the rows one sweep touches twice stay in L2).  scratch: one device int32;
 * *bandwidth (host).  Synchronises `stream`. */
int hf_csr_bandwidth(const hf_csr* A, int32_t* scratch, int32_t* bandwidth, void* stream);

/* Zero-free copy of A used by the SpMM (explicit zeros add 0*x, an exact
 * no-op for finite x).  Two steps: count (returns nnz of the copy on host),
 * then fill into caller-allocated arrays.  ws: hf_csr_prune_workspace_bytes. */
size_t hf_csr_prune_workspace_bytes(int32_t n_rows);
int hf_csr_prune_count(const hf_csr* A, void* ws, size_t ws_bytes, int64_t* nnz_out, void* stream);
int hf_csr_prune_fill(const hf_csr* A, void* ws, size_t ws_bytes, int32_t* indptr_out,
                      int32_t* indices_out, double* val_out, void* stream);

/* Multi-RHS LDP-PCG: kp independent column recurrences of solver.py:64-111
 * advanced together through one SpMM per iteration.
 *   B, X       device, n x kp row-major (column j of the reference = X[:, j]);
 *              kp in {2,4,8,16,32,64}; unused columns must be zero in B.
 *              A column's result does not depend on kp or on the other columns
 *              (canonical reductions: every dot product is summed in one order
 *              that depends on n only), so T is bit-identical however the
 *              columns are batched or sharded over ranks.
 *   d          device, n (LDP diagonal, or ones for preconditioner="none")
 *   freeze_at  device, kp int32, or NULL.  If given, column j stops right after
 *              iteration freeze_at[j] (freeze_at[j] < 0: run normally) — used to
 *              replay a failed column to its best iterate.
 *   iters, status, best_iter  host, kp int32 each
 *   true_res, best_res        host, kp double each
 * Workspace: hf_pcg_workspace_bytes(n, kp, A->nnz) bytes.  n < 2^30.
 * Result per column: status HF_COL_*; iters = converged iteration count;
 * true_res = ||b - A x|| / ||b|| at exit; best_res/best_iter = smallest
 * recurrence residual seen and the iteration it occurred at. */
size_t hf_pcg_workspace_bytes(int32_t n, int32_t kp, int64_t nnz);
int hf_pcg_multi(const hf_csr* A, const double* d, const double* B, int32_t n, int32_t kp,
                 double tol, int32_t max_iter, const int32_t* freeze_at, double* X,
                 int32_t* iters, int32_t* status, double* true_res, double* best_res,
                 int32_t* best_iter, void* ws, size_t ws_bytes, void* stream);

/* Column streaming: the same solver for ncols >= 1 columns of B (device n x ldb
 * row-major, columns 0..ncols-1) through kp slots.  When a slot's column finishes,
 * its x goes to column j of X (device n x ldb) and the slot takes the next column
 * at the next chunk boundary, so no slot waits for the slowest column of a batch.
 * Columns are handed out longest-expected-first (ascending b'Ab / b'Db, estimated
 * on a row sample) and slots are scheduled on the device; neither changes a column's
 * arithmetic: per-column iterates are bit-identical to hf_pcg_multi's (canonical
 * reductions).
 * iters, status, best_iter (int32) and true_res, best_res (double): host, ncols
 * each.  FAILED columns hold x at max_iter: replay them with hf_pcg_multi and
 * freeze_at = best_iter for the best iterate (solver.py:92-93, 108-111).
 * Workspace: hf_pcg_stream_workspace_bytes(n, kp, ncols). */
size_t hf_pcg_stream_workspace_bytes(int32_t n, int32_t kp, int32_t ncols);
int hf_pcg_stream(const hf_csr* A, const double* d, const double* B, int32_t ldb, int32_t ncols,
                  int32_t n, int32_t kp, double tol, int32_t max_iter, double* X, int32_t* iters,
                  int32_t* status, double* true_res, double* best_res, int32_t* best_iter,
                  void* ws, size_t ws_bytes, void* stream);

/* Timing probe for the roofline report: runs `rounds` PCG rounds of the same
 * kernels as hf_pcg_multi (tolerance 0, so no column stops) and writes the
 * average duration in ms, measured with CUDA events on `stream`, of
 * {SpMM, r update, p update / x round averaged over the ring} to ms3;
 * *flags (host int32) = 6 | (XD << 8), XD = the x-deferral depth.
 * Same workspace as hf_pcg_multi. */
int hf_pcg_profile(const hf_csr* A, const double* d, const double* B, int32_t n, int32_t kp,
                   int32_t rounds, double* X, float* ms3, int32_t* fused, void* ws,
                   size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------- assembly */

/* Element blocks K_e[i][j] = V g_i . sigma g_j (fem.py:31-93).
 *   nodes  device n x 3 f64;  tetra device m x 4 int32
 *   elements  device int32 subset of size m_sub, or NULL (all m elements)
 *   sigma  device: m_sub (sigma_cols == 1) or m_sub x 6 (sigma_cols == 6) f64 aligned
 *          with the subset, or NULL
 *          with sigma_cols == 0 for the uniform value sigma_scalar
 *   blocks device m_sub x 16 + 1 f64 (row-major 4x4 per element; the trailing
 *          slot is scratch for the flag word)
 *   vols   device m_sub f64 (may be NULL)
 *   flags  host int32: bit0 non-positive volume, bit1 negative scalar sigma,
 *          bit2 non positive-definite tensor (AssemblyError in fem.py:56-67,82-83) */
int hf_p1_blocks(const double* nodes, const int32_t* tetra, int32_t m, const int32_t* elements,
                 int32_t m_sub, const double* sigma, int32_t sigma_cols, double sigma_scalar,
                 double* blocks, double* vols, int32_t* flags, void* stream);

/* CSR assembly of the P1 stiffness matrix with scipy's pattern (fem.py:96-102):
 * rows/columns of every element pair, sorted, duplicates summed in a fixed
 * (ascending element) order, explicit zeros kept.  Optional electrode contact
 * terms (fem.py:206-211): triangle t adds ecoef[t] * [[2,1,1],[1,2,1],[1,1,2]]/12
 * on its nodes, in triangle order, after the volume sum.  ground >= 0 deletes
 * row/column `ground` and sets a_gg = 1 (fem.py:219-224).
 *   step 1 (prepare): blocks (from hf_p1_blocks, m x 16), incidence lists and
 *           row counts; writes indptr (device, n+1) and *nnz_out (host).
 *   step 2 (fill):   writes indices (device, nnz) and val (device, nnz). */
size_t hf_p1_assemble_workspace_bytes(int32_t n, int32_t m, int32_t n_etri);
int hf_p1_assemble_prepare(const int32_t* tetra, int32_t n, int32_t m, const int32_t* etri,
                           int32_t n_etri, int32_t ground, int32_t* indptr, int64_t* nnz_out,
                           void* ws, size_t ws_bytes, void* stream);
int hf_p1_assemble_fill(const int32_t* tetra, int32_t n, int32_t m, const double* blocks,
                        const int32_t* etri, const double* ecoef, int32_t n_etri, int32_t ground,
                        const int32_t* indptr, int32_t* indices, double* val, void* ws,
                        size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------- lead field */

/* Raw electrode response block M[:, col0:col0+ncols] = C - B' T (leadfield.py:107;
 * the caller symmetrises M = (M + M')/2 on the host, leadfield.py:108, after
 * gathering the column blocks of every rank).
 *   Bt   CSR of B' (L x n) on device (row l = electrode l's nodes, ascending)
 *   T    device n x ldt row-major holding the ncols transfer columns col0..
 *   Cdiag device L (C = diag(1/Z), fem.py:256);  Mraw device L x ncols row-major */
int hf_response_matrix(const hf_csr* Bt, const double* T, int32_t ldt, int32_t L, int32_t col0,
                       int32_t ncols, const double* Cdiag, double* Mraw, void* stream);

/* EEG lead field tail (leadfield.py:128-129):  LF = W (G' T)'  where T holds K
 * transfer columns (device n x ldt), W = -R M^-1 restricted to those K columns
 * (device L x ldw row-major, L x K used) and G' is CSR (ncols x n, row c =
 * source column c, <= 8 entries each).  LF device L x ncols row-major.  With
 * K = L this is the whole lead field; with a column block it is one rank's
 * partial sum.  The (G'T)' tile is gathered into shared memory and multiplied
 * on the fp64 tensor path (DMMA, mma.sync m8n8k4 f64). */
int hf_lf_tail(const double* T, int32_t ldt, int32_t K, const hf_csr* Gt, const double* W,
               int32_t L, int32_t ldw, double* LF, void* stream);

/* Dense variant for the EIT Jacobian (leadfield.py:230-237):
 * out[l, c] = sum_{k<K} W[l*ldw + k] * Qc[c*K + k] for l < L, c < ncols, with Qc
 * device ncols x K row-major (i.e. out = W[:, :K] Qc').  out device L x ldo
 * row-major.  K = L for one device; K = the electrode block on a rank, with W
 * pointing at the block's first column (distributed EIT partial sums). */
int hf_dense_lf(const double* Qc, int32_t ncols, int32_t K, const double* W, int32_t L,
                int32_t ldw, double* out, int32_t ldo, void* stream);

/* EIT sensitivities Q[p, m, l] = sum_{e in dof m} sum_i T[conn_ei, l] (K_e u_e,p)_i
 * with unit-conductivity K_e whose ground rows/columns are zeroed
 * (leadfield.py:179-207).
 *   dof_elems device (sum of DOF sizes) int32, dof_ptr device n_dofs+1 int32
 *   T device n x ldt (L used), U device n x ldu (P used)
 *   Q device P x n_dofs x L row-major
 *   ws device workspace of hf_eit_sens_workspace_bytes(dof_ptr[n_dofs] - dof_ptr[0])
 *      bytes (the DOF elements' unit blocks)
 * The contraction runs on the fp64 tensor pipe (DMMA m8n8k4), one GEMM with
 * K = 4 |E_m| per DOF. */
/* out (device n_rows x ldo row-major, ncols used) = A (CSR) D (device A->n_cols x ldd
 * row-major): the EIT pattern right-hand sides B M^-1 I (leadfield.py:223). */
int hf_csr_dense(const hf_csr* A, const double* D, int32_t ldd, int32_t ncols, double* out,
                 int32_t ldo, void* stream);

size_t hf_eit_sens_workspace_bytes(int64_t n_dof_elems);
int hf_eit_sens(const double* nodes, const int32_t* tetra, const int32_t* dof_elems,
                const int32_t* dof_ptr, int32_t n_dofs, int32_t ground, const double* T,
                int32_t ldt, int32_t L, const double* U, int32_t ldu, int32_t P, double* Q,
                void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------- topology (next rows, §8f) */

/* Boundary faces of a tetrahedral mesh (meshgen.py:101-134): face k of element e
 * is opposite local vertex k, ids f = 4e + k; a face is on the boundary when no
 * other element holds its three nodes.  face_idx (device, capacity 4m) receives
 * the boundary face ids ascending (the reference's flatnonzero order);
 * *n_faces (host) their number.  ws: hf_topology_workspace_bytes(n, m, 0). */
size_t hf_topology_workspace_bytes(int32_t n, int32_t m, int32_t ncols);
int hf_boundary_faces(const int32_t* tetra, int32_t n, int32_t m, int32_t* face_idx,
                      int64_t* n_faces, void* ws, size_t ws_bytes, void* stream);

/* Source matrix G of assemble_G (fem.py:291-422) as its transpose G' in CSR:
 * row c = source column c (3 per source, x/y/z, unconstrained; or 1 per source
 * when orient (device S x 3) is given, constrained), columns = mesh nodes
 * ascending (the <= 8 nodes of the source element and its face neighbours).
 * Two calls: with gidx/gval NULL it writes gptr (device, ncols+1) and *nnz_out;
 * then with gidx/gval (device, nnz) it fills them.
 * ws: hf_topology_workspace_bytes(n, m, ncols). */
int hf_whitney_gt(const double* nodes, const int32_t* tetra, int32_t n, int32_t m,
                  const int32_t* src_elems, int32_t n_src, const double* orient, int32_t* gptr,
                  int32_t* gidx, double* gval, int64_t* nnz_out, void* ws, size_t ws_bytes,
                  void* stream);

/* owner[i] = argmin_j ||points_i - centers_j|| (first index on ties) with the
 * reference's arithmetic: sqrt((dx*dx + dy*dy) + dz*dz), each op rounded
 * (build_dof_map, leadfield.py:96-99).  points (n_points x 3), centers
 * (n_centers x 3) row-major fp64, owner int32; all device.  No workspace. */
int hf_nearest_center(const double* points, int32_t n_points, const double* centers,
                      int32_t n_centers, int32_t* owner, double* dist, void* stream);
/* dist (device n_points f64, or NULL): the winning distance, as np.linalg.norm
 * computes it — ElectrodeSet.from_centers' coverage test d <= radius
 * (fem.py:164-167) uses the same routine on boundary-triangle centroids. */

/* Element centroids (((a + b) + c) + d) / 4 (TetMesh.centroids' numpy rounding) of
 * elems[0..count) (device int32, or NULL for elements 0..count-1); cent device count x 3. */
int hf_tet_centroids(const double* nodes, const int32_t* tetra, const int32_t* elems, int32_t count,
                     double* cent, void* stream);

/* build_dof_map's sets (leadfield.py:99-100): sorted_cand = cand stably sorted by owner
 * (each set keeps ascending element order), set_ptr[k] = first position of set k
 * (n_sets + 1 entries).  All device int32; ws: hf_dof_partition_workspace_bytes(n_cand). */
size_t hf_dof_partition_workspace_bytes(int32_t n_cand);
int hf_dof_partition(const int32_t* cand, const int32_t* owner, int32_t n_cand, int32_t n_sets,
                     int32_t* sorted_cand, int32_t* set_ptr, void* ws, size_t ws_bytes, void* stream);

/* Centroids ((a + b) + c) / 3 of n_tri triangles (device n_tri x 3 int32 node ids),
 * numpy's mean over 3 rows (fem.py:163).  cent device n_tri x 3 f64. */
int hf_triangle_centroids(const double* nodes, const int32_t* tri, int32_t n_tri, double* cent,
                          void* stream);

/* ground_node (fem.py:188-194): the lowest boundary node (nodes of bfaces, device
 * n_bfaces x 3 int32) not covered by an electrode triangle (etri, device n_etri x 3
 * int32); *ground (host) = -1 if there is none.  ws: hf_ground_node_workspace_bytes(n). */
size_t hf_ground_node_workspace_bytes(int32_t n);
int hf_ground_node(const int32_t* bfaces, int32_t n_bfaces, const int32_t* etri, int32_t n_etri,
                   int32_t n, void* ws, int32_t* ground, void* stream);

/* ---------------------------------------------------------------- mesh generation (next row #4, §8f) */

/* A segmentation for hf_locate (geometry.py:317-374): compartments innermost
 * first, each a union of closed surfaces.  All arrays device.
 *   comp_surf  n_comp+1   surfaces of compartment k: comp_surf[k] .. comp_surf[k+1]-1
 *   tri_off    n_surf+1   triangles of surface s: tri_off[s] .. tri_off[s+1]-1
 *   box        n_surf x 8 {lo.x, lo.y, lo.z, hi.x, hi.y, hi.z, tol, 0}, tol = 1e-9 * diameter
 *   rays       16 doubles per (surface, direction, triangle), surface s's block at row
 *              tri_off[s] * n_dir, direction d at + d * n_tri(s): {h(3), k(3), n(3), c_h, c_k,
 *              c_n, f, parallel (1/0), tol * 2 * area, 0} exactly as SurfaceMesh._cast
 *              derives them for direction d (geometry.py:203-224). */
typedef struct {
  int32_t n_comp, n_surf, n_dir;
  const int32_t* comp_surf;
  const int32_t* tri_off;
  const double* box;
  const double* rays;
} hf_segmentation;

/* labels[i] = innermost compartment containing points[i] (on-surface counts as
 * inside), -1 outside all (Segmentation.locate, geometry.py:359-374).
 * points device n x 3 fp64, labels device int32.  No workspace. */
int hf_locate(const hf_segmentation* seg, const double* points, int32_t n_points, int32_t* labels,
              void* stream);

/* generate_mesh's grid (meshgen.py:205-223): nx*ny*nz cubes, cx fastest, 6 Kuhn
 * tetrahedra per cube in _KUHN_TETS order; tetra (device 6*ncube x 4 int32) holds
 * grid node ids ix + (nx+1)(iy + (ny+1) iz), centroids (device 6*ncube x 3) the
 * corner means.  xs/ys/zs (device, nx+1 / ny+1 / nz+1) are the grid coordinates. */
int hf_grid_tets(const double* xs, const double* ys, const double* zs, int32_t nx, int32_t ny,
                 int32_t nz, int32_t* tetra, double* centroids, void* stream);

/* Keep the elements with label >= 0 in order, number the used grid nodes
 * ascending and renumber the corners (the np.unique(return_inverse) of
 * meshgen.py:229-232).  tetra_out (capacity m_all x 4), labels_out (m_all),
 * nodes_out (capacity (nx+1)(ny+1)(nz+1) x 3) device; *m_out, *n_out host.
 * ws: hf_mesh_compact_workspace_bytes(m_all, (nx+1)(ny+1)(nz+1)). */
size_t hf_mesh_compact_workspace_bytes(int32_t m_all, int32_t n_grid);
int hf_mesh_compact(const int32_t* tetra_all, const int32_t* cent_label, int32_t m_all,
                    const double* xs, const double* ys, const double* zs, int32_t nx, int32_t ny,
                    int32_t nz, int32_t* tetra_out, int32_t* labels_out, double* nodes_out,
                    int64_t* m_out, int64_t* n_out, void* ws, size_t ws_bytes, void* stream);

/* _apply_priorities (meshgen.py:247-269) in place on labels (device m), from the
 * node labels (device n) and the compartment priorities (device n_comp). */
int hf_apply_priorities(const int32_t* tetra, int32_t m, const int32_t* node_label,
                        const int32_t* priority, int32_t* labels, void* stream);

/* ---------------------------------------------------------------- MEG (C3)
 * No reference counterpart (the reference excludes MEG): the FEM
 * reciprocity formulation on the EEG path's system (csrc/meg.cu header).
 * coils device n_coils x 8 f64 {rx, ry, rz, nx, ny, nz, weight, 0};
 * coil_ptr device ncols+1 int32 (sensor s = coils coil_ptr[s]..coil_ptr[s+1]-1). */
size_t hf_meg_workspace_bytes(int32_t n, int32_t m);
/* S' (device n x ldb row-major, ncols <= 512 used): the secondary-current flux
 * operator of every sensor, row `ground` zeroed.  sigma device m f64 (scalar). */
int hf_meg_rhs(const double* nodes, const int32_t* tetra, const double* sigma, int32_t n, int32_t m,
               int32_t ground, const double* coils, const int32_t* coil_ptr, int32_t ncols,
               double* Bt, int32_t ldb, void* ws, size_t ws_bytes, void* stream);
/* Lp device ncols x 3*n_sources: primary flux of unit x/y/z dipoles at positions
 * (device n_sources x 3). */
int hf_meg_primary(const double* coils, const int32_t* coil_ptr, int32_t ncols,
                   const double* positions, int32_t n_sources, double* Lp, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HFB200_H */
