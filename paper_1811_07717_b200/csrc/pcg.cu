// Multi-RHS LDP-PCG for sm_100a.
//
// Restates solver.py:64-111 (pcg_solve) for kp right-hand sides at once: every
// column keeps its own recurrence (alpha, beta, residual replacement, true-
// residual confirmation, best iterate), exactly as transfer_matrix runs them
// one by one (solver.py:114-141); the columns only share the matrix stream.
//
// Layout: every n-vector block (X, R, Q, B and the ring of P blocks) is n x kp
// row-major, so the kp values of one mesh node are contiguous.  A row group of
// LPR lanes owns one row; each lane owns CPL consecutive columns and moves them
// as one 256-bit (CPL = 4) or 128-bit (CPL = 2) access.
//
// One PCG round is three kernels:
//   k_spmm      q = A p over a padded ELL copy of A, partial p.q   -> alpha
//   k_update_r  r -= alpha q, partial r.r and r.(r/d)              -> res, beta, state
//   k_update_p  p_{k+1} = r/d + beta p_k into the next slot of a ring of XD p
//               blocks; every XD-th round k_update_xring also replays
//               x += alpha_j p_j over the ring (x touched once per XD rounds).
// Columns whose recurrence residual drops below tol freeze in state CHECK; at
// the end of every chunk of rounds the check path (k_spmm in residual mode,
// k_replace, k_replace_p) computes b - A x, and finishes the column or
// replaces r and resumes it, exactly as solver.py:94-102.
//
// Canonical reductions.  A column's arithmetic must not depend on the batch
// width kp or on which other columns share the batch (so T is bit-identical
// for any batch, rank count or `threads`, the multi-GPU analogue of
// test_solver.py:131-137).  Every per-row value is computed by the same
// explicit operations for every kp, and every dot product is summed in one
// fixed order that only depends on n:
//   rows are dealt in tiles of TR = 32 rows, tile t -> block t % G with
//   G = min(GRID, tiles) blocks (GRID = 296, a constant, not the SM count);
//   row group g of a block (tile row g) accumulates its rows sequentially over
//   the block's tiles in sweep order; the 32 row-group sums of a block are
//   added by a balanced binary tree (warp shuffles for the groups inside a
//   warp, then shared memory across warps); the last block to finish sums the
//   G block partials in RSEG = 8 fixed segments (sequential inside a
//   segment) and adds the segments by a balanced tree.
// Every reducing kernel is launched with one row group per tile row
// (32 x LPR threads), so the same order falls out of any kp.
#include <math.h>

#include <algorithm>
#include <vector>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"

namespace hf {
namespace pcg {

constexpr int TR = 32;        // rows per tile: the canonical reduction unit
constexpr int GRID = 296;     // blocks of every reducing kernel (2 per SM on the 148-SM B200)
constexpr int RSEG = 8;       // segments of the last-block reduction
constexpr int CHUNK = 8;      // PCG rounds per captured graph
constexpr int LOOKAHEAD = 3;  // chunks queued beyond the one whose status is read
constexpr int ELL_W = 8;      // slots per row of the ELL copy of A
constexpr int ELL_LONG = 1 << 30;  // slot 0 flag: the row has entries beyond the slots
constexpr int ELL_OPT = 5;         // first slot gathered only when it holds an entry

enum : int {
  S_RUN = 0,
  S_CHECK = 1,
  S_DONE = HF_COL_DONE,
  S_FAILED = HF_COL_FAILED,
  S_ZERO = HF_COL_ZERO,
  S_FROZEN = HF_COL_FROZEN,
  S_REPLACE = 6
};

// summary[] slots
enum : int {
  SUM_RUN = 0,
  SUM_CHECK = 1,
  SUM_REPLACE = 2,
  SUM_PM = 4,    // columns whose p advances this round
  SUM_XANY = 5,  // x updates pending since the last x round
  SUM_N = 8
};

// Deferred x update.  x_{k+1} = x_k + alpha_k p_k needs nothing else of round
// k, so the x stream is touched once every XD rounds: the p of each round
// goes to its own buffer of a ring of XD (p_{k+1} into slot (k+1) % XD, the
// old p stays), alpha and the x mask of each round go to their own slot, and
// the x round (slot XD-1) replays x += alpha_j p_j for j = 0..XD-1 in order:
// the same sequence of roundings as one update per round, with x read and
// written once per XD rounds (80 -> 72 + 8/XD bytes per row per column per
// round).  XD divides CHUNK, so x is current at every check path.  A column
// that stops running keeps its last p in slot pbuf[j] (where the check path's
// replacement finds it).
constexpr int XD = 8;
static_assert(CHUNK % XD == 0, "x rounds fall on chunk ends");

struct Ctl {
  int n, G;
  double tol;
  int max_iter;
  double *normb, *rz, *alpha, *beta, *best_res, *true_res;
  int *iters, *best_iter, *state, *xmask, *pmask, *freeze;
  double *part0, *part1;
  double2* dd;  // per row {d_i, 1/d_i}, written by k_init
  unsigned int* counter;
  int* summary;
  int rnd;    // round within the chunk
  int* pbuf;  // per column: ring slot of its p once it stops running
};

// Thread layout of a kernel at batch width KP with CPL columns per lane: one row
// group of LPR lanes per tile row, so a reducing kernel runs 32 x LPR threads.
// Kernels may pick different CPL: the reduction order only depends on the tile
// and row-group structure, not on how a row's columns are split over lanes.
template <int KP_, int CPL_>
struct Lay {
  static_assert(KP_ >= 2 && KP_ <= 64 && (KP_ & (KP_ - 1)) == 0, "kp in {2,...,64}");
  static constexpr int KP = KP_;
  static constexpr int CPL = CPL_;
  static constexpr int LPR = KP / CPL;            // lanes per row
  static constexpr int NT = TR * LPR;             // threads of a reducing kernel
  static constexpr int NW = NT / 32;              // warps of a reducing kernel
  static constexpr int SPL = LPR >= ELL_W ? 1 : ELL_W / LPR;  // ELL slots held per lane
  static constexpr int RED = (NW * KP * 2 > RSEG * KP * 2) ? NW * KP * 2 : RSEG * KP * 2;
};

// Streaming kernels: one 256/128/64-bit access per lane; kp <= 16 keeps 1 column
// per lane so a reducing kernel still runs 16 lanes per row (512 threads at kp = 16).
template <int KP>
struct Map : Lay<KP, (KP >= 64) ? 4 : (KP == 32 ? 2 : 1)> {
  using B = Lay<KP, (KP >= 64) ? 4 : (KP == 32 ? 2 : 1)>;
  // tiles in flight per thread in the streaming kernels (register budget: 64)
  static constexpr int U = (B::CPL == 4) ? 1 : (B::CPL == 2 ? 2 : 4);
};

// The SpMM moves 256-bit gathers from kp = 32 on (kp = 32: 8 lanes per row,
// 256 threads; 6% faster at C2 and 16% at C5 than 128-bit lanes) and 128 bits
// below (kp = 16: 8 lanes per row, two tiles per step in flight, see k_spmm).
template <int KP>
using SpmmLay = Lay<KP, (KP >= 32) ? 4 : 2>;

__host__ __device__ inline int n_tiles(int n) { return (n + TR - 1) / TR; }

// Column slices of a row move as one 256-bit access (LDG/STG.E.256 on
// sm_100a) when a lane owns 4 columns, else as a 128-bit access.
template <int CPL>
__device__ __forceinline__ void ld_cols(const double* p, double (&v)[CPL]) {
  if constexpr (CPL == 1) {
    v[0] = *p;
  } else if constexpr (CPL == 4) {
    asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
                 : "l"(p));
  } else {
    const double2 t = *reinterpret_cast<const double2*>(p);
    v[0] = t.x;
    v[1] = t.y;
  }
}
template <int CPL>
__device__ __forceinline__ void ldg_cols(const double* __restrict__ p, double (&v)[CPL]) {
  if constexpr (CPL == 1) {
    v[0] = __ldg(p);
  } else if constexpr (CPL == 4) {
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
        : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
        : "l"(p));
  } else {
    const double2 t = __ldg(reinterpret_cast<const double2*>(p));
    v[0] = t.x;
    v[1] = t.y;
  }
}
template <int CPL>
__device__ __forceinline__ void st_cols(double* p, const double (&v)[CPL]) {
  if constexpr (CPL == 1) {
    *p = v[0];
  } else if constexpr (CPL == 4) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v[0]), "d"(v[1]),
                 "d"(v[2]), "d"(v[3])
                 : "memory");
  } else {
    *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
  }
}

// z = x / d with the row's precomputed reciprocal and one residual
// correction (3 flops instead of a ~10-instruction fp64 division): the
// corrected quotient is the correctly rounded x / d except in rare
// double-rounding ties, where it is one ulp away.  dd = {d_i, 1/d_i}.
__device__ __forceinline__ double zdiv(double x, double2 dd) {
  const double q0 = __dmul_rn(x, dd.y);
  const double res = __fma_rn(-q0, dd.x, x);
  return __fma_rn(res, dd.y, q0);
}

// Per-row recurrence arithmetic, written with explicit roundings so every
// template instantiation computes the same bits (no compiler contraction
// choices): r - alpha q, z + beta p, x + alpha p and the dot-product terms.
__device__ __forceinline__ double axpy(double a, double x, double y) { return __fma_rn(a, x, y); }
__device__ __forceinline__ double dot_acc(double acc, double a, double b) { return __fma_rn(a, b, acc); }

// ------------------------------------------------------------ canonical reductions
// Block partials: v[q][k] is this thread's running sum (its row group, column
// glane*CPL + k).  Balanced tree over the block's 32 row groups; the block's
// partial row goes to part{q}[blockIdx.x * KP + col].
template <class M, int NV>
__device__ __forceinline__ void block_partials(double (&v)[NV][M::CPL], double* sm,
                                               const Ctl& c) {
  constexpr int KP = M::KP;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int glane = tid % M::LPR;
#pragma unroll
  for (int q = 0; q < NV; ++q)
#pragma unroll
    for (int k = 0; k < M::CPL; ++k) {
      double x = v[q][k];
#pragma unroll
      for (int off = M::LPR; off < 32; off <<= 1) x = __dadd_rn(x, __shfl_xor_sync(FULL, x, off));
      v[q][k] = x;
    }
  if (lane < M::LPR) {
#pragma unroll
    for (int q = 0; q < NV; ++q)
#pragma unroll
      for (int k = 0; k < M::CPL; ++k) sm[(q * M::NW + warp) * KP + glane * M::CPL + k] = v[q][k];
  }
  __syncthreads();
  if (tid < NV * KP) {
    const int q = tid / KP, col = tid % KP;
    double a[M::NW];
#pragma unroll
    for (int w = 0; w < M::NW; ++w) a[w] = sm[(q * M::NW + w) * KP + col];
#pragma unroll
    for (int s = 1; s < M::NW; s <<= 1)
#pragma unroll
      for (int w = 0; w + s < M::NW; w += 2 * s) a[w] = __dadd_rn(a[w], a[w + s]);
    (q == 0 ? c.part0 : c.part1)[(size_t)blockIdx.x * KP + col] = a[0];
  }
}

// Last-block detection; the last block reduces the G block partials in RSEG
// fixed segments and a balanced tree over them into tot[q*KP + col] (shared).
// The reduction is on the critical path of every round (the next kernel waits
// for it), so each thread keeps 8 loads per quantity in flight instead of
// walking its segment one L2 round trip at a time.
template <class M, int NV>
__device__ __forceinline__ bool last_block_reduce(const Ctl& c, double* sm, double* tot) {
  constexpr int KP = M::KP;
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(c.counter, 1u) == (unsigned)(c.G - 1));
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
  const int tid = threadIdx.x;
  const int per = (c.G + RSEG - 1) / RSEG;
  for (int o = tid; o < RSEG * KP; o += M::NT) {
    const int s = o / KP, col = o % KP;
    const int b0 = s * per, b1 = min(c.G, b0 + per);
    double a[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) a[q] = 0.0;
    for (int bb = b0; bb < b1; bb += 8) {
      double x[NV][8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int q = 0; q < NV; ++q)
          x[q][u] = (bb + u < b1) ? ld_cg((q == 0 ? c.part0 : c.part1) + (size_t)(bb + u) * KP + col)
                                  : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (bb + u < b1) {
#pragma unroll
          for (int q = 0; q < NV; ++q) a[q] = __dadd_rn(a[q], x[q][u]);
        }
    }
#pragma unroll
    for (int q = 0; q < NV; ++q) sm[(q * RSEG + s) * KP + col] = a[q];
  }
  __syncthreads();
  if (tid < NV * KP) {
    const int q = tid / KP, col = tid % KP;
    double a[RSEG];
#pragma unroll
    for (int s = 0; s < RSEG; ++s) a[s] = sm[(q * RSEG + s) * KP + col];
#pragma unroll
    for (int s = 1; s < RSEG; s <<= 1)
#pragma unroll
      for (int w = 0; w + s < RSEG; w += 2 * s) a[w] = __dadd_rn(a[w], a[w + s]);
    tot[q * KP + col] = a[0];
  }
  __syncthreads();
  if (tid == 0) *c.counter = 0u;
  return true;
}

// Column-state census of the last block (every thread calls it; thread j < KP
// passes column j's new state): summary counters without a serial walk over
// the states in global memory.
template <int KP>
__device__ __forceinline__ void census(const Ctl& c, int st) {
  const bool mine = threadIdx.x < KP;
  const int nrun = __syncthreads_count(mine && st == S_RUN);
  const int nchk = __syncthreads_count(mine && st == S_CHECK);
  if (threadIdx.x == 0) {
    c.summary[SUM_RUN] = nrun;
    c.summary[SUM_CHECK] = nchk;
  }
}

// ---------------------------------------------------------------- init
// x = 0; r = b; z = r/d; p = z; rz = r.z; ||b||   (solver.py:74-85)
template <int KP>
__global__ void __launch_bounds__(Map<KP>::NT)
    k_init(Ctl c, const double* __restrict__ B, const double* __restrict__ d, double* X,
           double* R, double* P) {
  using M = Map<KP>;
  __shared__ double sm[M::RED];
  __shared__ double tot[2 * KP];
  const int tid = threadIdx.x, grp = tid / M::LPR, glane = tid % M::LPR;
  const int nt = n_tiles(c.n);
  double v[2][M::CPL];
#pragma unroll
  for (int k = 0; k < M::CPL; ++k) v[0][k] = v[1][k] = 0.0;
  for (int t = blockIdx.x; t < nt; t += c.G) {
    const int row = t * TR + grp;
    if (row >= c.n) continue;
    const size_t o = (size_t)row * KP + glane * M::CPL;
    double b[M::CPL], z[M::CPL], zero[M::CPL];
    ld_cols<M::CPL>(B + o, b);
    const double dd = d[row];
    if (glane == 0) c.dd[row] = make_double2(dd, 1.0 / dd);
#pragma unroll
    for (int k = 0; k < M::CPL; ++k) {
      z[k] = __ddiv_rn(b[k], dd);
      zero[k] = 0.0;
      v[0][k] = dot_acc(v[0][k], b[k], b[k]);
      v[1][k] = dot_acc(v[1][k], b[k], z[k]);
    }
    st_cols<M::CPL>(X + o, zero);
    st_cols<M::CPL>(R + o, b);
    st_cols<M::CPL>(P + o, z);
  }
  block_partials<M, 2>(v, sm, c);
  if (!last_block_reduce<M, 2>(c, sm, tot)) return;
  int st = -1;
  if (tid < KP) {
    const int j = tid;
    const double nb = sqrt(tot[j]);
    c.normb[j] = nb;
    c.rz[j] = tot[KP + j];
    c.alpha[j] = 0.0;
    c.beta[j] = 0.0;
    c.best_res[j] = 1.0;  // best = (1.0, x0, 0)   solver.py:85
    c.best_iter[j] = 0;
    c.iters[j] = 0;
    c.true_res[j] = 0.0;
    c.xmask[j] = 0;
    c.pmask[j] = 0;
    st = S_RUN;
    if (nb == 0.0)
      st = S_ZERO;  // solver.py:75-76
    else if (c.freeze != nullptr && c.freeze[j] == 0)
      st = S_FROZEN;
    c.state[j] = st;
  }
  census<KP>(c, st);
  if (tid == 0) c.summary[SUM_REPLACE] = 0;
}

// ---------------------------------------------------------------- column streaming
// hf_pcg_stream runs more columns than the kp slots of a batch: a slot whose
// column finished is harvested (its x and results copied out) and refilled with
// the next column at a chunk boundary, so no slot idles while the slowest column
// of a batch finishes.  One kernel does both, the slot lists passed by value (no
// staging copy to wait for): harvest[j] = destination column of slot j's x, -1
// none; refill[j] = source column, -2 = none (state ZERO; b = x = r = p = 0 on
// the first fill), -1 = keep.
// The refill is k_init restricted to the refilled slots: the same per-row
// arithmetic and the same canonical b.b / b.z reductions, so a column's iterates
// are bit-identical to a batch solve of it.
struct SlotLists {
  int refill[64];
  int harvest[64];
};

struct Harvest {  // per-column results of hf_pcg_stream
  double* X;      // n x ldb
  int *iters, *state, *best_iter;
  double *true_res, *best_res;
};

template <int KP>
__global__ void __launch_bounds__(Map<KP>::NT)
    k_refill(Ctl c, const SlotLists sl, const double* __restrict__ Ball, int ldb, Harvest hv, double* Bs,
             const double* __restrict__ d, double* X, double* R, double* P, int init_dd) {
  using M = Map<KP>;
  __shared__ double sm[M::RED];
  __shared__ double tot[2 * KP];
  const int tid = threadIdx.x, grp = tid / M::LPR, glane = tid % M::LPR;
  if (blockIdx.x == 0 && tid < KP && sl.harvest[tid] >= 0) {  // results, before the last block resets them
    const int j = tid, col = sl.harvest[j];
    hv.iters[col] = c.iters[j];
    hv.state[col] = c.state[j];
    hv.true_res[col] = c.true_res[j];
    hv.best_res[col] = c.best_res[j];
    hv.best_iter[col] = c.best_iter[j];
  }
  int col[M::CPL], hcol[M::CPL];
  bool any = false;
#pragma unroll
  for (int k = 0; k < M::CPL; ++k) {
    col[k] = sl.refill[glane * M::CPL + k];
    hcol[k] = sl.harvest[glane * M::CPL + k];
    // b = 0 is written only by the first fill (empty slots of ncols < kp)
    if (col[k] == -2 && !init_dd) col[k] = -3;
    any |= col[k] != -1 || hcol[k] >= 0;
  }
  const int nt = n_tiles(c.n);
  double v[2][M::CPL];
#pragma unroll
  for (int k = 0; k < M::CPL; ++k) v[0][k] = v[1][k] = 0.0;
  if (any || init_dd) {
    for (int t = blockIdx.x; t < nt; t += c.G) {
      const int row = t * TR + grp;
      if (row >= c.n) continue;
      const size_t o = (size_t)row * KP + glane * M::CPL;
      const double dd = d[row];
      if (init_dd && glane == 0) c.dd[row] = make_double2(dd, 1.0 / dd);
#pragma unroll
      for (int k = 0; k < M::CPL; ++k) {
        if (hcol[k] >= 0) hv.X[(size_t)row * ldb + hcol[k]] = X[o + k];
        if (col[k] < 0 && col[k] != -2) continue;
        const double b = col[k] >= 0 ? Ball[(size_t)row * ldb + col[k]] : 0.0;
        const double z = __ddiv_rn(b, dd);
        v[0][k] = dot_acc(v[0][k], b, b);
        v[1][k] = dot_acc(v[1][k], b, z);
        Bs[o + k] = b;
        X[o + k] = 0.0;
        R[o + k] = b;
        P[o + k] = z;
      }
    }
  }
  block_partials<M, 2>(v, sm, c);
  if (!last_block_reduce<M, 2>(c, sm, tot)) return;
  int st = -1;
  if (tid < KP) {
    const int j = tid;
    st = c.state[j];
    if (sl.refill[j] != -1) {
      const double nb = sqrt(tot[j]);
      c.normb[j] = nb;
      c.rz[j] = tot[KP + j];
      c.beta[j] = 0.0;
      c.best_res[j] = 1.0;
      c.best_iter[j] = 0;
      c.iters[j] = 0;
      c.true_res[j] = 0.0;
      c.pmask[j] = 0;
      st = nb == 0.0 ? S_ZERO : S_RUN;
      c.state[j] = st;
    }
  }
  census<KP>(c, st);
}

// Device-side slot scheduler of hf_pcg_stream, the last node of every captured
// chunk (after the check path, so DONE / FAILED are final): every block derives
// the same decisions from the slot states, then it is k_refill with those lists.
// A finished slot takes the next column (slot order), or retires when none is
// left; its results go out now, a retired slot's x at the final harvest.
struct Sched {
  int* slot_col;     // column in each slot, -1 = none
  int* retired;      // 1 = finished, nothing left to take, x not yet harvested
  int* next;         // next position of `order` to hand out
  int* nfin;         // finished columns (harvested or retired); the host stops at ncols
  const int* order;  // hand-out order of the columns (longest expected first)
  int ncols;
};

// Hand-out order.  A slot idles once no column is left, so the columns that need
// the most iterations should start first.  Jacobi-preconditioned CG takes longest
// on smooth right-hand sides, whose Rayleigh quotient b'Ab / b'Db is small (C3:
// Spearman -0.74 against the iteration counts, tools/order_probe.py), so columns
// go out in ascending b'Ab / b'Db.  Only the schedule changes: a column's
// arithmetic does not depend on its slot or start time.  Per block b: partial
// sums over rows 16 b, 16 (b + G), ... of b_i (A b)_i and d_i b_i^2 for every column
// (thread t owns columns t, t + NT, ...), in shared memory; k_col_rq_sum adds the
// G partials per column in block order (deterministic).
constexpr int RQ_NT = 256, RQ_MAXC = 2048;
constexpr int RQ_STRIDE = 16;  // every 16th row: an estimate is enough to order columns
__global__ void __launch_bounds__(RQ_NT)
    k_col_rq(int n, const int* __restrict__ eci, const double* __restrict__ ecv, const int32_t* __restrict__ indptr,
             const int32_t* __restrict__ indices, const double* __restrict__ val, const double* __restrict__ d,
             const double* __restrict__ B, int ldb, int ncols, double* part) {
  __shared__ double s_num[RQ_MAXC], s_den[RQ_MAXC];
  for (int c = threadIdx.x; c < ncols; c += RQ_NT) s_num[c] = s_den[c] = 0.0;
  for (int i = blockIdx.x * RQ_STRIDE; i < n; i += gridDim.x * RQ_STRIDE) {
    const int c0 = __ldg(eci + (size_t)i * ELL_W);
    const bool lng = (c0 & ELL_LONG) != 0;
    const double di = d[i];
    for (int c = threadIdx.x; c < ncols; c += RQ_NT) {
      double ab = 0.0;
#pragma unroll
      for (int e = 0; e < ELL_W; ++e) {
        const int ce = __ldg(eci + (size_t)i * ELL_W + e) & (ELL_LONG - 1);
        if (e >= ELL_OPT && __ldg(eci + (size_t)i * ELL_W + e) < 0) continue;
        ab = __fma_rn(__ldg(ecv + (size_t)i * ELL_W + e), __ldg(B + (size_t)ce * ldb + c), ab);
      }
      if (lng)
        for (int j = indptr[i] + ELL_W; j < indptr[i + 1]; ++j)
          ab = __fma_rn(val[j], __ldg(B + (size_t)indices[j] * ldb + c), ab);
      const double bi = __ldg(B + (size_t)i * ldb + c);
      s_num[c] = __fma_rn(bi, ab, s_num[c]);
      s_den[c] = __fma_rn(di * bi, bi, s_den[c]);
    }
  }
  for (int c = threadIdx.x; c < ncols; c += RQ_NT) {
    part[(size_t)blockIdx.x * 2 * ncols + c] = s_num[c];
    part[(size_t)blockIdx.x * 2 * ncols + ncols + c] = s_den[c];
  }
}

__global__ void k_col_rq_sum(int nblocks, int ncols, const double* __restrict__ part, double* rq) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncols) return;
  double num = 0.0, den = 0.0;
  for (int b = 0; b < nblocks; ++b) {
    num += part[(size_t)b * 2 * ncols + c];
    den += part[(size_t)b * 2 * ncols + ncols + c];
  }
  rq[c] = den > 0.0 ? num / den : INFINITY;  // b = 0: last (it finishes at once)
}

// Tail compaction.  Once no column is left to hand out, finished slots leave
// holes and the kernels keep moving every lane that still holds a running
// column; when the running columns would fit in at least two fewer 4-slot lane
// groups, one pass harvests every finished slot's x and moves the running
// columns from the high slots into the lowest free ones (x, r, b and the p in
// ring slot 0 — where a running column's p is at a chunk end — plus its control
// words), so lanes above them go idle.  A column's arithmetic does not depend
// on its slot (canonical reductions), so its results stay bit-identical.
// Returns false (nothing done, no block touched anything) when not worth it.
template <int KP>
__device__ bool compact_tail(Ctl& c, Sched& sc, int ntake, const int* s_take, int* s_harv, int* s_src,
                             int ldb, Harvest& hv, double* Bs, double* X, double* R, double* P, double* sm,
                             double* tot) {
  using M = Map<KP>;
  __shared__ int s_go;
  const int tid = threadIdx.x, grp = tid / M::LPR, glane = tid % M::LPR;
  if (tid == 0) {
    int m = 0, groups = 0, gmask = 0;
    int active[KP];
    for (int j = 0; j < KP; ++j) {
      active[j] = sc.slot_col[j] >= 0 && !sc.retired[j] && !s_take[j];
      m += active[j];
      if (active[j]) gmask |= 1 << (j / 4);
    }
    for (int q = 0; q < KP / 4; ++q) groups += (gmask >> q) & 1;
    s_go = m > 0 && groups - (m + 3) / 4 >= 2;
    if (s_go) {
      int src = m;
      for (int j = 0; j < KP; ++j) {
        s_harv[j] = (sc.slot_col[j] >= 0 && !active[j]) ? sc.slot_col[j] : -1;  // finished: x out
        s_src[j] = -1;
      }
      for (int f = 0; f < m; ++f) {
        if (active[f]) continue;
        while (!active[src]) ++src;
        s_src[f] = src++;
      }
    }
  }
  __syncthreads();
  if (!s_go) return false;
  int hcol[M::CPL], from[M::CPL];
  bool any = false;
#pragma unroll
  for (int k = 0; k < M::CPL; ++k) {
    hcol[k] = s_harv[glane * M::CPL + k];
    from[k] = s_src[glane * M::CPL + k];
    any |= hcol[k] >= 0 || from[k] >= 0;
  }
  if (any) {
    const int nt = n_tiles(c.n);
    for (int t = blockIdx.x; t < nt; t += c.G) {
      const int row = t * TR + grp;
      if (row >= c.n) continue;
      const size_t o = (size_t)row * KP + glane * M::CPL, r0 = (size_t)row * KP;
#pragma unroll
      for (int k = 0; k < M::CPL; ++k) {
        if (hcol[k] >= 0) hv.X[(size_t)row * ldb + hcol[k]] = X[o + k];
        if (from[k] < 0) continue;
        X[o + k] = X[r0 + from[k]];
        R[o + k] = R[r0 + from[k]];
        Bs[o + k] = Bs[r0 + from[k]];
        P[o + k] = P[r0 + from[k]];  // ring slot 0
      }
    }
  }
  // no reduction: the partials only carry the last-block election
  double v[1][M::CPL];
#pragma unroll
  for (int k = 0; k < M::CPL; ++k) v[0][k] = 0.0;
  block_partials<M, 1>(v, sm, c);
  if (!last_block_reduce<M, 1>(c, sm, tot)) return true;
  __syncthreads();
  if (tid == 0) {
    for (int f = 0; f < KP; ++f) {
      if (s_harv[f] >= 0) {  // harvested: the slot is empty
        sc.slot_col[f] = -1;
        sc.retired[f] = 0;
        c.state[f] = S_ZERO;
      }
    }
    for (int f = 0; f < KP; ++f) {
      const int a = s_src[f];
      if (a < 0) continue;
      c.state[f] = c.state[a];
      c.normb[f] = c.normb[a];
      c.rz[f] = c.rz[a];
      c.beta[f] = c.beta[a];
      c.best_res[f] = c.best_res[a];
      c.best_iter[f] = c.best_iter[a];
      c.iters[f] = c.iters[a];
      c.true_res[f] = c.true_res[a];
      c.pmask[f] = c.pmask[a];
      c.pbuf[f] = c.pbuf[a];
      sc.slot_col[f] = sc.slot_col[a];
      sc.retired[f] = 0;
      sc.slot_col[a] = -1;
      sc.retired[a] = 0;
      c.state[a] = S_ZERO;
    }
    *sc.nfin += ntake;
  }
  __syncthreads();
  census<KP>(c, tid < KP ? c.state[tid] : -1);
  return true;
}

template <int KP>
__global__ void __launch_bounds__(Map<KP>::NT)
    k_sched(Ctl c, Sched sc, const double* __restrict__ Ball, int ldb, Harvest hv, double* Bs,
            const double* __restrict__ d, double* X, double* R, double* P) {
  using M = Map<KP>;
  __shared__ double sm[M::RED];
  __shared__ double tot[2 * KP];
  __shared__ int s_take[KP], s_ref[KP], s_harv[KP];
  const int tid = threadIdx.x, grp = tid / M::LPR, glane = tid % M::LPR;
  const int nx = *sc.next;
  int take = 0;
  if (tid < KP) {
    const int st = c.state[tid];
    take = (st == S_DONE || st == S_FAILED || st == S_ZERO) && sc.slot_col[tid] >= 0 && !sc.retired[tid];
    s_take[tid] = take;
  }
  const int ntake = __syncthreads_count(take);
  if (ntake == 0) return;  // the common case: nothing finished in this chunk
  int refill = 0;
  if (tid < KP) {
    int rank = 0;
    for (int i = 0; i < tid; ++i) rank += s_take[i];
    const int pos = nx + rank;
    s_ref[tid] = (take && pos < sc.ncols) ? sc.order[pos] : -1;
    s_harv[tid] = (take && pos < sc.ncols) ? sc.slot_col[tid] : -1;
    refill = s_ref[tid] >= 0;
  }
  const int nref = __syncthreads_count(refill);
  if (blockIdx.x == 0 && tid < KP && s_take[tid]) {  // results, before the last block resets them
    const int j = tid, col = sc.slot_col[j];
    hv.iters[col] = c.iters[j];
    hv.state[col] = c.state[j];
    hv.true_res[col] = c.true_res[j];
    hv.best_res[col] = c.best_res[j];
    hv.best_iter[col] = c.best_iter[j];
  }
  if (nref == 0) {  // no column left (every block sees it)
    if (compact_tail<KP>(c, sc, ntake, s_take, s_harv, s_ref, ldb, hv, Bs, X, R, P, sm, tot)) return;
    if (blockIdx.x == 0) {  // block 0 retires the finished slots
      __syncthreads();
      if (tid < KP && s_take[tid]) sc.retired[tid] = 1;
      if (tid == 0) *sc.nfin += ntake;
    }
    return;
  }
  int col[M::CPL], hcol[M::CPL];
  bool any = false;
#pragma unroll
  for (int k = 0; k < M::CPL; ++k) {
    col[k] = s_ref[glane * M::CPL + k];
    hcol[k] = s_harv[glane * M::CPL + k];
    any |= col[k] >= 0;
  }
  const int nt = n_tiles(c.n);
  double v[2][M::CPL];
#pragma unroll
  for (int k = 0; k < M::CPL; ++k) v[0][k] = v[1][k] = 0.0;
  if (any) {
    for (int t = blockIdx.x; t < nt; t += c.G) {
      const int row = t * TR + grp;
      if (row >= c.n) continue;
      const size_t o = (size_t)row * KP + glane * M::CPL;
      const double dd = d[row];
#pragma unroll
      for (int k = 0; k < M::CPL; ++k) {
        if (col[k] < 0) continue;
        hv.X[(size_t)row * ldb + hcol[k]] = X[o + k];
        const double b = Ball[(size_t)row * ldb + col[k]];
        const double z = __ddiv_rn(b, dd);
        v[0][k] = dot_acc(v[0][k], b, b);
        v[1][k] = dot_acc(v[1][k], b, z);
        Bs[o + k] = b;
        X[o + k] = 0.0;
        R[o + k] = b;
        P[o + k] = z;
      }
    }
  }
  block_partials<M, 2>(v, sm, c);
  if (!last_block_reduce<M, 2>(c, sm, tot)) return;
  int st = -1;
  if (tid < KP) {
    const int j = tid;
    st = c.state[j];
    if (s_ref[j] >= 0) {
      const double nb = sqrt(tot[j]);
      c.normb[j] = nb;
      c.rz[j] = tot[KP + j];
      c.beta[j] = 0.0;
      c.best_res[j] = 1.0;
      c.best_iter[j] = 0;
      c.iters[j] = 0;
      c.true_res[j] = 0.0;
      c.pmask[j] = 0;
      st = nb == 0.0 ? S_ZERO : S_RUN;
      c.state[j] = st;
      sc.slot_col[j] = s_ref[j];
    } else if (s_take[j]) {
      sc.retired[j] = 1;
    }
  }
  if (tid == 0) {
    *sc.next = nx + nref;
    *sc.nfin += ntake;
  }
  census<KP>(c, st);
}

// ---------------------------------------------------------------- SpMM over an ELL copy
// The SpMM runs on a padded ELL copy of the zero-free matrix (8 slots per row,
// built once per solve by k_ell_fill).  Empty slots 0..ELL_OPT-1 hold (row
// itself, 0.0): their gather hits L1 (the row's own p) and their FMA adds an
// exact zero, so they are gathered and multiplied unconditionally; empty slots
// from ELL_OPT on hold -1 and are skipped (an interior Kuhn row fills 7).  The
// diagonal sits in slot 0, so the epilogue's p_i is its gather.  Rows with
// more than 8 entries keep entries 0..7 in the slots and flag bit 30 of slot
// 0's column; their entries 8.. come from the CSR.  Sum order, for every kp:
// slots 7..0, then entries 8.. in order.  A/B timings of the variants are in
// DESIGN.md §3.
constexpr int ELL_HB = 4;   // gathers in flight per batch

__global__ void k_ell_fill(int n, const int32_t* __restrict__ indptr,
                           const int32_t* __restrict__ indices, const double* __restrict__ val,
                           int* __restrict__ eci, double* __restrict__ ecv) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int st = indptr[i], ln = indptr[i + 1] - st;
  int c[ELL_W];
  double v[ELL_W];
  for (int e = 0; e < ELL_W; ++e) {
    c[e] = e >= ELL_OPT ? -1 : i;
    v[e] = 0.0;
    if (e < ln) {
      c[e] = indices[st + e];
      v[e] = val[st + e];
    }
  }
  for (int e = 1; e < ELL_W && e < ln; ++e)  // the diagonal (when slot-held) to slot 0
    if (c[e] == i) {
      const int tc = c[0];
      const double tv = v[0];
      c[0] = c[e];
      v[0] = v[e];
      c[e] = tc;
      v[e] = tv;
      break;
    }
  if (ln > ELL_W) c[0] |= ELL_LONG;
  for (int e = 0; e < ELL_W; ++e) {
    eci[(size_t)i * ELL_W + e] = c[e];
    ecv[(size_t)i * ELL_W + e] = v[e];
  }
}

struct Ell {
  const int* __restrict__ ci;
  const double* __restrict__ cv;
  const int32_t* __restrict__ indptr;  // the CSR the ELL copy was built from (long rows)
  const int32_t* __restrict__ indices;
  const double* __restrict__ val;
};

// MODE_PQ:    q = A p for RUN columns, partial p.q -> alpha = rz / p.q   (solver.py:87-88)
// MODE_RESID: s = b - A x (into Q) for CHECK columns, partial s.s -> true residual,
//             DONE / FAILED / REPLACE                                   (solver.py:94-102)
enum { MODE_PQ = 0, MODE_RESID = 1 };

template <int KP, int MODE>
__global__ void __launch_bounds__(SpmmLay<KP>::NT, 2)
    k_spmm(Ctl c, Ell A, const double* __restrict__ V, const double* __restrict__ Bv,
           double* __restrict__ Q) {
  using M = SpmmLay<KP>;
  constexpr int CPL = M::CPL, LPR = M::LPR, SPL = M::SPL;
  // tiles per step: narrow batches move few bytes per gather, so a row group keeps
  // two rows' gathers in flight (the rows are still summed in tile order)
  constexpr int UT = (KP <= 16) ? 2 : 1;
  // how a row's 8 slots reach its lanes: at kp = 64 every lane reads them itself (L1
  // broadcast, prefetched a step ahead), narrower batches stage them through shared
  // memory (A/B timed: DESIGN.md §3.1)
  constexpr bool SLOT_LDG = (KP >= 64);
  __shared__ double sm[M::RED];
  __shared__ double tot[KP];
  __shared__ int s_act[KP];
  constexpr int SLOTS = SLOT_LDG ? 1 : 2 * UT * TR;  // shared slot staging (unused at kp = 64)
  __shared__ __align__(16) int s_ci_[SLOTS][ELL_W];
  __shared__ __align__(16) double s_cv_[SLOTS][ELL_W];
  auto s_ci = reinterpret_cast<int(*)[UT][TR][ELL_W]>(&s_ci_[0][0]);
  auto s_cv = reinterpret_cast<double(*)[UT][TR][ELL_W]>(&s_cv_[0][0]);
  if (MODE == MODE_PQ && c.summary[SUM_RUN] == 0) return;
  if (MODE == MODE_RESID && c.summary[SUM_CHECK] == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) c.summary[SUM_REPLACE] = 0;
    return;
  }
  const int tid = threadIdx.x, gl = tid % LPR, grp = tid / LPR;
  for (int j = tid; j < KP; j += M::NT)
    s_act[j] = (c.state[j] == (MODE == MODE_PQ ? S_RUN : S_CHECK));
  __syncthreads();
  double m[CPL];  // 1 for the lane's active columns: masks their dot terms
  bool act[CPL];
  bool any = false;
#pragma unroll
  for (int k = 0; k < CPL; ++k) {
    act[k] = s_act[gl * CPL + k] != 0;
    m[k] = act[k] ? 1.0 : 0.0;
    any |= act[k];
  }
  const int nt = n_tiles(c.n);
  const int slot = gl < ELL_W ? gl : ELL_W - 1;
  const double* __restrict__ Vl = V + gl * CPL;
  double v[1][CPL];
#pragma unroll
  for (int k = 0; k < CPL; ++k) v[0][k] = 0.0;
  auto tile_row = [&](int tt) {  // tile tt's row of this row group (-1: none)
    const int r = tt * TR + grp;
    return (tt < nt && r < c.n) ? r : -1;
  };
  auto load_slots = [&](int r, int (&cs)[SPL], double (&vs)[SPL]) {
#pragma unroll
    for (int k = 0; k < SPL; ++k) {
      cs[k] = 0;
      vs[k] = 0.0;
      if (r >= 0) {
        cs[k] = __ldg(A.ci + (size_t)r * ELL_W + slot + k * LPR);
        vs[k] = __ldg(A.cv + (size_t)r * ELL_W + slot + k * LPR);
      }
    }
  };
  int row[UT], ci[UT][SPL];
  double cv[UT][SPL];
#pragma unroll
  for (int u = 0; u < UT; ++u) {
    row[u] = tile_row(blockIdx.x + u * c.G);
    if (!SLOT_LDG) load_slots(row[u], ci[u], cv[u]);
  }
  int b = 0;
  for (int t = blockIdx.x; t < nt; t += UT * c.G, b ^= 1) {
    int rowN[UT], ciN[UT][SPL];
    double cvN[UT][SPL];
#pragma unroll
    for (int u = 0; u < UT; ++u) {  // next step's slots in flight during this one
      rowN[u] = tile_row(t + (UT + u) * c.G);
      if (!SLOT_LDG) load_slots(rowN[u], ciN[u], cvN[u]);
    }
    if constexpr (SLOT_LDG) {
      // every lane reads its row's 8 slots itself (L1 broadcast, one line per two rows),
      // the next tile's rows prefetched into L1 one step ahead
      if (gl == 0) {
#pragma unroll
        for (int u = 0; u < UT; ++u)
          if (rowN[u] >= 0) {
            asm volatile("prefetch.global.L1 [%0];" ::"l"(A.ci + (size_t)rowN[u] * ELL_W));
            asm volatile("prefetch.global.L1 [%0];" ::"l"(A.cv + (size_t)rowN[u] * ELL_W));
          }
      }
    } else {
      if (gl < ELL_W) {
#pragma unroll
        for (int u = 0; u < UT; ++u)
#pragma unroll
          for (int k = 0; k < SPL; ++k) {
            s_ci[b][u][grp][gl + k * LPR] = ci[u][k];
            s_cv[b][u][grp][gl + k * LPR] = cv[u][k];
          }
      }
      __syncwarp();
    }
    int cc[UT][ELL_W], c0x[UT];
    bool live[UT];
#pragma unroll
    for (int u = 0; u < UT; ++u) {
      const int rr = row[u] >= 0 ? row[u] : 0;
      const int4 c0 = SLOT_LDG ? __ldg(reinterpret_cast<const int4*>(A.ci + (size_t)rr * ELL_W))
                               : *reinterpret_cast<const int4*>(&s_ci[b][u][grp][0]);
      const int4 c1 = SLOT_LDG ? __ldg(reinterpret_cast<const int4*>(A.ci + (size_t)rr * ELL_W + 4))
                               : *reinterpret_cast<const int4*>(&s_ci[b][u][grp][4]);
      c0x[u] = c0.x;
      cc[u][0] = c0.x & (ELL_LONG - 1);
      cc[u][1] = c0.y;
      cc[u][2] = c0.z;
      cc[u][3] = c0.w;
      cc[u][4] = c1.x;
      cc[u][5] = c1.y;
      cc[u][6] = c1.z;
      cc[u][7] = c1.w;
      live[u] = row[u] >= 0 && any;
    }
    double a[UT][CPL], g0[UT][CPL];  // g0: slot 0's gather, p_i when slot 0 is the diagonal
    bool anylive = false;
#pragma unroll
    for (int u = 0; u < UT; ++u) {
      anylive |= live[u];
#pragma unroll
      for (int k = 0; k < CPL; ++k) a[u][k] = 0.0;
    }
    if (anylive) {
#pragma unroll
    for (int bt = ELL_W / ELL_HB - 1; bt >= 0; --bt) {
      double g[UT][ELL_HB][CPL];
#pragma unroll
      for (int u = 0; u < UT; ++u)
#pragma unroll
        for (int k = 0; k < ELL_HB; ++k) {
          const int e = bt * ELL_HB + k;
          if (e >= ELL_OPT) {  // optional slot: zero when empty
#pragma unroll
            for (int q = 0; q < CPL; ++q) g[u][k][q] = 0.0;
            if (live[u] && cc[u][e] >= 0) ldg_cols<CPL>(Vl + (size_t)cc[u][e] * KP, g[u][k]);
          } else if (live[u]) {
            ldg_cols<CPL>(Vl + (size_t)(unsigned)cc[u][e] * KP, g[u][k]);
          }
        }
#pragma unroll
      for (int u = 0; u < UT; ++u) {
        if (bt == 0) {
#pragma unroll
          for (int q = 0; q < CPL; ++q) g0[u][q] = g[u][0][q];
        }
        const double2* vp =
            SLOT_LDG ? reinterpret_cast<const double2*>(A.cv + (size_t)(row[u] >= 0 ? row[u] : 0) * ELL_W)
                     : reinterpret_cast<const double2*>(&s_cv[b][u][grp][0]);
        // consume the batch last-issued first (slot order 7..0)
#pragma unroll
        for (int k2 = ELL_HB / 2 - 1; k2 >= 0; --k2) {
          const double2 vv = SLOT_LDG ? __ldg(vp + bt * ELL_HB / 2 + k2) : vp[bt * ELL_HB / 2 + k2];
#pragma unroll
          for (int q = 0; q < CPL; ++q) a[u][q] = __fma_rn(vv.y, g[u][2 * k2 + 1][q], a[u][q]);
#pragma unroll
          for (int q = 0; q < CPL; ++q) a[u][q] = __fma_rn(vv.x, g[u][2 * k2][q], a[u][q]);
        }
      }
    }
    }
#pragma unroll
    for (int u = 0; u < UT; ++u) {  // epilogues in tile order (the canonical dot order)
      if (!live[u]) continue;
      const int r = row[u];
      if (c0x[u] & ELL_LONG) {  // entries 8.. of a long row, in order
        const int st = __ldg(A.indptr + r), en = __ldg(A.indptr + r + 1);
        for (int j = st + ELL_W; j < en; ++j) {
          const int ce = __ldg(A.indices + j);
          const double ve = __ldg(A.val + j);
          double q2[CPL];
          ldg_cols<CPL>(Vl + (size_t)ce * KP, q2);
#pragma unroll
          for (int q = 0; q < CPL; ++q) a[u][q] = __fma_rn(ve, q2[q], a[u][q]);
        }
      }
      const size_t o = (size_t)r * KP + gl * CPL;
      if constexpr (MODE == MODE_PQ) {
        st_cols<CPL>(Q + o, a[u]);
        double pr[CPL];
        if (cc[u][0] == r) {
#pragma unroll
          for (int q = 0; q < CPL; ++q) pr[q] = g0[u][q];
        } else {
          ldg_cols<CPL>(V + o, pr);
        }
#pragma unroll
        for (int q = 0; q < CPL; ++q) v[0][q] = __fma_rn(__dmul_rn(pr[q], a[u][q]), m[q], v[0][q]);
      } else {
        double bb[CPL], sres[CPL];
        ld_cols<CPL>(Bv + o, bb);
#pragma unroll
        for (int q = 0; q < CPL; ++q) {
          sres[q] = __dsub_rn(bb[q], a[u][q]);
          if (act[q]) v[0][q] = dot_acc(v[0][q], sres[q], sres[q]);
        }
        st_cols<CPL>(Q + o, sres);
      }
    }
#pragma unroll
    for (int u = 0; u < UT; ++u) {
      row[u] = rowN[u];
#pragma unroll
      for (int k = 0; k < SPL; ++k) {
        ci[u][k] = ciN[u][k];
        cv[u][k] = cvN[u][k];
      }
    }
  }
  block_partials<M, 1>(v, sm, c);
  if (!last_block_reduce<M, 1>(c, sm, tot)) return;
  if constexpr (MODE == MODE_PQ) {
    if (tid < KP && s_act[tid]) c.alpha[tid] = c.rz[tid] / tot[tid];
  } else {
    int st = -1;
    if (tid < KP) {
      const int j = tid;
      st = c.state[j];
      if (st == S_CHECK) {
        const double tr = sqrt(tot[j]) / c.normb[j];
        c.true_res[j] = tr;
        if (tr <= c.tol)
          st = S_DONE;
        else if (c.iters[j] >= c.max_iter)
          st = S_FAILED;
        else
          st = S_REPLACE;
        c.state[j] = st;
      }
    }
    const int nrep = __syncthreads_count(tid < KP && st == S_REPLACE);
    census<KP>(c, st);
    if (tid == 0) c.summary[SUM_REPLACE] = nrep;
  }
}

// r -= alpha q ; res = |r|/|b| ; best ; tolerance / max_iter ; beta   (solver.py:90-106)
// The tiles are swept backward: the sweep starts on the q rows the SpMM wrote
// last (still in L2) and ends on the r rows the p update reads first.
template <int KP>
__global__ void __launch_bounds__(Map<KP>::NT, 2)
    k_update_r(Ctl c, const double* __restrict__ Q, double* R) {
  using M = Map<KP>;
  __shared__ double sm[M::RED];
  __shared__ double tot[2 * KP];
  __shared__ double s_alpha[KP];
  __shared__ int s_act[KP];
  if (c.summary[SUM_RUN] == 0) {
    if (blockIdx.x == 0) {  // no x update this round (its history slot is read by the x round)
      for (int j = threadIdx.x; j < KP; j += M::NT) c.xmask[j] = 0;
      if (threadIdx.x == 0) {
        c.summary[SUM_PM] = 0;
        if (c.rnd % XD == 0) c.summary[SUM_XANY] = 0;
      }
    }
    return;
  }
  const int tid = threadIdx.x, grp = tid / M::LPR, glane = tid % M::LPR;
  for (int j = tid; j < KP; j += M::NT) {
    const int a = (c.state[j] == S_RUN);
    s_act[j] = a;
    s_alpha[j] = a ? c.alpha[j] : 0.0;
  }
  __syncthreads();
  bool act[M::CPL];
  double al[M::CPL];
  bool any = false;
#pragma unroll
  for (int k = 0; k < M::CPL; ++k) {
    act[k] = s_act[glane * M::CPL + k];
    al[k] = s_alpha[glane * M::CPL + k];
    any |= act[k];
  }
  const int nt = n_tiles(c.n);
  double v[2][M::CPL];
#pragma unroll
  for (int k = 0; k < M::CPL; ++k) v[0][k] = v[1][k] = 0.0;
  if (any) {
    constexpr int U = M::U;
    for (int j0 = blockIdx.x; j0 < nt; j0 += U * c.G) {
      double r[U][M::CPL], q[U][M::CPL];
      double2 dd[U];
      int rows[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {  // all loads first: U rows in flight
        const int tt = j0 + u * c.G;
        rows[u] = (tt < nt) ? (nt - 1 - tt) * TR + grp : c.n;
        if (rows[u] < c.n) {
          const size_t o = (size_t)rows[u] * KP + glane * M::CPL;
          ld_cols<M::CPL>(R + o, r[u]);
          ld_cols<M::CPL>(Q + o, q[u]);
          dd[u] = c.dd[rows[u]];
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (rows[u] >= c.n) continue;
#pragma unroll
        for (int k = 0; k < M::CPL; ++k) {
          if (act[k]) {
            r[u][k] = axpy(-al[k], q[u][k], r[u][k]);
            v[0][k] = dot_acc(v[0][k], r[u][k], r[u][k]);
            v[1][k] = dot_acc(v[1][k], r[u][k], zdiv(r[u][k], dd[u]));
          }
        }
        st_cols<M::CPL>(R + (size_t)rows[u] * KP + glane * M::CPL, r[u]);
      }
    }
  }
  block_partials<M, 2>(v, sm, c);
  if (!last_block_reduce<M, 2>(c, sm, tot)) return;
  int xm = 0, pm = 0, st = -1;
  if (tid < KP) {
    const int j = tid;
    st = c.state[j];
    if (st == S_RUN) {
      const int k = c.iters[j] + 1;
      c.iters[j] = k;
      const double res = sqrt(tot[j]) / c.normb[j];
      if (res < c.best_res[j]) {  // solver.py:92-93
        c.best_res[j] = res;
        c.best_iter[j] = k;
      }
      xm = 1;
      if (c.freeze != nullptr && c.freeze[j] == k) {
        st = S_FROZEN;
      } else if (res <= c.tol) {  // solver.py:94
        st = S_CHECK;
      } else if (k >= c.max_iter) {  // loop exhausted, solver.py:108
        st = S_FAILED;
      } else {
        const double rzn = tot[KP + j];  // solver.py:103-106
        c.beta[j] = rzn / c.rz[j];
        c.rz[j] = rzn;
        pm = 1;
      }
      c.state[j] = st;
      if (!pm) c.pbuf[j] = c.rnd % XD;  // its last p stays in this slot
    }
    c.xmask[j] = xm;
    c.pmask[j] = pm;
  }
  const int npm = __syncthreads_count(pm);
  const int nxm = __syncthreads_count(xm);
  census<KP>(c, st);
  if (tid == 0) {
    c.summary[SUM_PM] = npm;
    c.summary[SUM_XANY] = (c.rnd % XD == 0) ? nxm : c.summary[SUM_XANY] + nxm;
  }
}

// ---------------------------------------------------------------- p / x updates (no reductions)
// Round r of a chunk: p_{k+1} = r/d + beta p_k into ring slot (r+1) % XD, the
// old p stays in slot r % XD for the x round.
template <int KP>
__global__ void __launch_bounds__(Map<KP>::NT)
    k_update_p(Ctl c, const double* __restrict__ Pcur, double* __restrict__ Pnext,
               const double* __restrict__ R) {
  using M = Map<KP>;
  __shared__ double s_beta[KP];
  __shared__ int s_pm[KP];
  if (c.summary[SUM_PM] == 0) return;
  const int tid = threadIdx.x, grp = tid / M::LPR, glane = tid % M::LPR;
  for (int j = tid; j < KP; j += M::NT) {
    s_pm[j] = c.pmask[j];
    s_beta[j] = c.beta[j];
  }
  __syncthreads();
  bool pm[M::CPL];
  double be[M::CPL];
  bool anyp = false;
#pragma unroll
  for (int k = 0; k < M::CPL; ++k) {
    const int j = glane * M::CPL + k;
    pm[k] = s_pm[j];
    be[k] = s_beta[j];
    anyp |= pm[k];
  }
  if (!anyp) return;  // no column of this lane advances: its slot of Pnext is never read
  const int nt = n_tiles(c.n);
  constexpr int U = M::U;
  for (int t0 = blockIdx.x; t0 < nt; t0 += U * c.G) {
    double p[U][M::CPL], r[U][M::CPL];
    double2 dd[U];
    int rows[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      rows[u] = (t0 + u * c.G < nt) ? (t0 + u * c.G) * TR + grp : c.n;
      if (rows[u] < c.n) {
        const size_t o = (size_t)rows[u] * KP + glane * M::CPL;
        ld_cols<M::CPL>(Pcur + o, p[u]);
        ld_cols<M::CPL>(R + o, r[u]);
        dd[u] = c.dd[rows[u]];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (rows[u] >= c.n) continue;
#pragma unroll
      for (int k = 0; k < M::CPL; ++k)
        if (pm[k]) p[u][k] = axpy(be[k], p[u][k], zdiv(r[u][k], dd[u]));
      st_cols<M::CPL>(Pnext + (size_t)rows[u] * KP + glane * M::CPL, p[u]);
    }
  }
}

// The x round (slot XD-1): x += alpha_j p_j for j = 0..XD-1 in round order
// (each with that round's mask), then p_{k+1} into slot 0.  One block per SM
// with a 128-register budget at 4-column lanes: a lane keeps x, XD p slices
// and r in flight.
template <int KP>
__global__ void __launch_bounds__(Map<KP>::NT, (Map<KP>::NT >= 512 ? 1 : 2))
    k_update_xring(Ctl c, double* __restrict__ X, double* __restrict__ Pring, size_t nk,
                   const double* __restrict__ R, const double* __restrict__ alpha_h,
                   const int* __restrict__ xmask_h) {
  using M = Map<KP>;
  __shared__ double s_alpha[XD][KP];
  __shared__ int s_xm[XD][KP];
  __shared__ double s_beta[KP];
  __shared__ int s_pm[KP];
  if (c.summary[SUM_XANY] == 0 && c.summary[SUM_PM] == 0) return;
  const int tid = threadIdx.x, grp = tid / M::LPR, glane = tid % M::LPR;
  for (int j = tid; j < XD * KP; j += M::NT) {
    const int xm = xmask_h[j];
    s_xm[j / KP][j % KP] = xm;
    s_alpha[j / KP][j % KP] = xm ? alpha_h[j] : 0.0;
  }
  for (int j = tid; j < KP; j += M::NT) {
    s_pm[j] = c.pmask[j];
    s_beta[j] = c.beta[j];
  }
  __syncthreads();
  constexpr int CUR = XD - 1;  // this round's slot; p_{k+1} goes to slot 0
  unsigned lx = 0;             // ring slots this lane's columns need for x
  bool anyp = false;
#pragma unroll
  for (int k = 0; k < M::CPL; ++k) {
    const int j = glane * M::CPL + k;
#pragma unroll
    for (int q = 0; q < XD; ++q) lx |= s_xm[q][j] ? (1u << q) : 0u;
    anyp |= s_pm[j] != 0;
  }
  const bool anyx = lx != 0;
  if (anyp) lx |= 1u << CUR;
  if (!lx) return;
  const int nt = n_tiles(c.n);
  for (int t = blockIdx.x; t < nt; t += c.G) {
    const int row = t * TR + grp;
    if (row >= c.n) continue;
    const size_t o = (size_t)row * KP + glane * M::CPL;
    double x[M::CPL], p[XD][M::CPL], r[M::CPL];
    double2 dd;
    if (anyx) ld_cols<M::CPL>(X + o, x);
#pragma unroll
    for (int q = 0; q < XD; ++q)
      if ((lx >> q) & 1u) ld_cols<M::CPL>(Pring + (size_t)q * nk + o, p[q]);
    if (anyp) {
      ld_cols<M::CPL>(R + o, r);
      dd = c.dd[row];
    }
    if (anyx) {
#pragma unroll
      for (int q = 0; q < XD; ++q)
#pragma unroll
        for (int k = 0; k < M::CPL; ++k) {
          const int j = glane * M::CPL + k;
          if (s_xm[q][j]) x[k] = axpy(s_alpha[q][j], p[q][k], x[k]);
        }
      st_cols<M::CPL>(X + o, x);
    }
    if (anyp) {
      double pn[M::CPL];
#pragma unroll
      for (int k = 0; k < M::CPL; ++k) {
        const int j = glane * M::CPL + k;
        pn[k] = s_pm[j] ? axpy(s_beta[j], p[CUR][k], zdiv(r[k], dd)) : p[CUR][k];
      }
      st_cols<M::CPL>(Pring + o, pn);
    }
  }
}

// ---------------------------------------------------------------- check path
// r = s for REPLACE columns, rz_next = r.(r/d), beta, resume   (solver.py:101-106)
template <int KP>
__global__ void __launch_bounds__(Map<KP>::NT, 2)
    k_replace(Ctl c, const double* __restrict__ Q, double* R) {
  using M = Map<KP>;
  __shared__ double sm[M::RED];
  __shared__ double tot[KP];
  __shared__ int s_act[KP];
  if (c.summary[SUM_REPLACE] == 0) return;
  const int tid = threadIdx.x, grp = tid / M::LPR, glane = tid % M::LPR;
  for (int j = tid; j < KP; j += M::NT) s_act[j] = (c.state[j] == S_REPLACE);
  __syncthreads();
  bool act[M::CPL];
  bool any = false;
#pragma unroll
  for (int k = 0; k < M::CPL; ++k) {
    act[k] = s_act[glane * M::CPL + k];
    any |= act[k];
  }
  const int nt = n_tiles(c.n);
  double v[1][M::CPL];
#pragma unroll
  for (int k = 0; k < M::CPL; ++k) v[0][k] = 0.0;
  if (any) {
    for (int t = blockIdx.x; t < nt; t += c.G) {
      const int row = t * TR + grp;
      if (row >= c.n) continue;
      const size_t o = (size_t)row * KP + glane * M::CPL;
      double r[M::CPL], q[M::CPL];
      ld_cols<M::CPL>(R + o, r);
      ld_cols<M::CPL>(Q + o, q);
      const double2 dd = c.dd[row];
#pragma unroll
      for (int k = 0; k < M::CPL; ++k)
        if (act[k]) {
          r[k] = q[k];
          v[0][k] = dot_acc(v[0][k], r[k], zdiv(r[k], dd));
        }
      st_cols<M::CPL>(R + o, r);
    }
  }
  block_partials<M, 1>(v, sm, c);
  if (!last_block_reduce<M, 1>(c, sm, tot)) return;
  int st = -1;
  if (tid < KP) {
    const int j = tid;
    int pm = 0;
    st = c.state[j];
    if (st == S_REPLACE) {
      const double rzn = tot[j];
      c.beta[j] = rzn / c.rz[j];
      c.rz[j] = rzn;
      st = S_RUN;
      c.state[j] = st;
      pm = 1;
    }
    c.xmask[j] = 0;
    c.pmask[j] = pm;
  }
  census<KP>(c, st);
}

// A replaced column resumes with p = r/d + beta p from the slot its last p
// stayed in (pbuf) into slot 0.
template <int KP>
__global__ void __launch_bounds__(Map<KP>::NT)
    k_replace_p(Ctl c, double* __restrict__ Pring, size_t nk, const double* __restrict__ R) {
  using M = Map<KP>;
  __shared__ int s_pm[KP], s_buf[KP];
  __shared__ double s_beta[KP];
  if (c.summary[SUM_REPLACE] == 0) return;
  const int tid = threadIdx.x, grp = tid / M::LPR, glane = tid % M::LPR;
  for (int j = tid; j < KP; j += M::NT) {
    s_pm[j] = c.pmask[j];
    s_buf[j] = c.pbuf[j];
    s_beta[j] = c.beta[j];
  }
  __syncthreads();
  bool anyp = false;
#pragma unroll
  for (int k = 0; k < M::CPL; ++k) anyp |= s_pm[glane * M::CPL + k] != 0;
  if (!anyp) return;
  const int nt = n_tiles(c.n);
  for (int t = blockIdx.x; t < nt; t += c.G) {
    const int row = t * TR + grp;
    if (row >= c.n) continue;
    const size_t o = (size_t)row * KP + glane * M::CPL;
    double r[M::CPL];
    ld_cols<M::CPL>(R + o, r);
    const double2 dd = c.dd[row];
#pragma unroll
    for (int k = 0; k < M::CPL; ++k) {
      const int j = glane * M::CPL + k;
      if (!s_pm[j]) continue;
      const double pold = Pring[(size_t)s_buf[j] * nk + o + k];
      Pring[o + k] = axpy(s_beta[j], pold, zdiv(r[k], dd));
    }
  }
}

// ---------------------------------------------------------------- host driver
struct Layout {
  double *R, *P, *Q, *part0, *part1;
  double2* dd;
  double *normb, *rz, *alpha, *beta, *best_res, *true_res;
  int *iters, *best_iter, *state, *xmask, *pmask, *freeze;
  int* pbuf;
  unsigned int* counter;
  int* summary;
  int* ell_ci;  // 8 slots per row (see k_ell_fill)
  double* ell_cv;
  size_t bytes;
};

inline Layout carve(void* ws, int n, int kp) {
  Carve cv{reinterpret_cast<char*>(ws), 0, ~size_t(0)};
  Layout L;
  const size_t nk = (size_t)n * kp;
  L.R = cv.take<double>(nk);
  L.P = cv.take<double>(nk * XD);  // ring of XD p blocks
  L.Q = cv.take<double>(nk);
  L.part0 = cv.take<double>((size_t)GRID * kp);
  L.part1 = cv.take<double>((size_t)GRID * kp);
  L.dd = cv.take<double2>((size_t)n);
  L.normb = cv.take<double>(kp);
  L.rz = cv.take<double>(kp);
  L.alpha = cv.take<double>((size_t)(XD + 1) * kp);  // per-round slots
  L.beta = cv.take<double>(kp);
  L.best_res = cv.take<double>(kp);
  L.true_res = cv.take<double>(kp);
  L.iters = cv.take<int>(kp);
  L.best_iter = cv.take<int>(kp);
  L.state = cv.take<int>(kp);
  L.xmask = cv.take<int>((size_t)(XD + 1) * kp);  // per-round slots + check-path scratch
  L.pbuf = cv.take<int>(kp);
  L.pmask = cv.take<int>(kp);
  L.freeze = cv.take<int>(kp);
  L.counter = cv.take<unsigned int>(4);
  L.summary = cv.take<int>(SUM_N);
  L.ell_ci = cv.take<int>((size_t)n * ELL_W);
  L.ell_cv = cv.take<double>((size_t)n * ELL_W);
  L.bytes = cv.used + 256;
  return L;
}

__global__ void k_bandwidth(int n, const int32_t* __restrict__ indptr,
                            const int32_t* __restrict__ indices, int* __restrict__ bw) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int s = indptr[i], e = indptr[i + 1];
  if (s < e) atomicMax(bw, max(i - indices[s], indices[e - 1] - i));
}

// Blocks of a kernel without reductions: enough to fill every SM.
template <class K>
int stream_grid(K kernel, int nt, int threads) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0);
  const int g = std::max(1, per_sm) * sm_count();
  return std::max(1, std::min(g, nt));
}

struct Grids {
  Ctl c;    // reducing kernels: G = min(GRID, tiles)
  Ctl cp;   // k_update_p
  Ctl cx;   // k_update_xring
  Ctl crp;  // k_replace_p
  Ell ell;
};

template <int KP>
int setup(const Layout& L, const hf_csr* A, int n, double tol, int max_iter, Grids& g,
          cudaStream_t stream) {
  using M = Map<KP>;
  Ctl& c = g.c;
  memset(&c, 0, sizeof(c));
  const int nt = n_tiles(n);
  c.n = n;
  c.G = std::min(GRID, nt);
  c.tol = tol;
  c.max_iter = max_iter;
  c.normb = L.normb; c.rz = L.rz; c.alpha = L.alpha; c.beta = L.beta;
  c.best_res = L.best_res; c.true_res = L.true_res; c.iters = L.iters;
  c.best_iter = L.best_iter; c.state = L.state; c.xmask = L.xmask; c.pmask = L.pmask;
  c.freeze = nullptr; c.part0 = L.part0; c.part1 = L.part1; c.dd = L.dd;
  c.counter = L.counter; c.summary = L.summary;
  c.rnd = 0; c.pbuf = L.pbuf;
  g.cp = c;
  g.cp.G = stream_grid(k_update_p<KP>, nt, M::NT);
  g.cx = c;
  g.cx.G = stream_grid(k_update_xring<KP>, nt, M::NT);
  g.crp = c;
  g.crp.G = stream_grid(k_replace_p<KP>, nt, M::NT);
  // ELL copy of the SpMM matrix (once per solve)
  k_ell_fill<<<(n + 255) / 256, 256, 0, stream>>>(n, A->indptr, A->indices, A->val, L.ell_ci,
                                                   L.ell_cv);
  HF_LAUNCH_CHECK();
  count_launches(1);
  g.ell = Ell{L.ell_ci, L.ell_cv, A->indptr, A->indices, A->val};
  return HF_OK;
}

// One PCG round r of a chunk: SpMM, r update, then the p update (or, every XD-th
// round, the x round).  ev (profiling only): recorded after each of the three.
template <int KP>
inline void launch_round(const Grids& g0, const Layout& L, double* X, int r, cudaStream_t q,
                         cudaEvent_t* ev) {
  using M = Map<KP>;
  Grids g = g0;
  const size_t nk = (size_t)g.c.n * KP;
  const int slot = r % XD;
  for (Ctl* k : {&g.c, &g.cp, &g.cx}) {
    k->rnd = r;
    k->alpha = L.alpha + (size_t)slot * KP;
    k->xmask = L.xmask + (size_t)slot * KP;
  }
  double* Pc = L.P + (size_t)slot * nk;
  k_spmm<KP, MODE_PQ><<<g.c.G, SpmmLay<KP>::NT, 0, q>>>(g.c, g.ell, Pc, nullptr, L.Q);
  if (ev) cudaEventRecord(ev[1], q);
  k_update_r<KP><<<g.c.G, M::NT, 0, q>>>(g.c, L.Q, L.R);
  if (ev) cudaEventRecord(ev[2], q);
  if (slot == XD - 1)
    k_update_xring<KP><<<g.cx.G, M::NT, 0, q>>>(g.cx, X, L.P, nk, L.R, L.alpha, L.xmask);
  else
    k_update_p<KP><<<g.cp.G, M::NT, 0, q>>>(g.cp, Pc, L.P + (size_t)(slot + 1) * nk, L.R);
  if (ev) cudaEventRecord(ev[3], q);
}

// The check path after a chunk: s = b - A x, true residuals, replacement.
template <int KP>
inline void launch_check(const Grids& g0, const Layout& L, const double* B, double* X,
                         cudaStream_t q) {
  using M = Map<KP>;
  Grids g = g0;
  g.c.xmask = L.xmask + (size_t)XD * KP;  // scratch: the round slots stay untouched
  k_spmm<KP, MODE_RESID><<<g.c.G, SpmmLay<KP>::NT, 0, q>>>(g.c, g.ell, X, B, L.Q);
  k_replace<KP><<<g.c.G, M::NT, 0, q>>>(g.c, L.Q, L.R);
  k_replace_p<KP><<<g.crp.G, M::NT, 0, q>>>(g.crp, L.P, (size_t)g.c.n * KP, L.R);
}

constexpr long PER_CHUNK = 3 * CHUNK + 3;  // kernels per captured chunk

// Capture stream and pinned status words, one per host thread and device (a
// cudaHostAlloc can stall for tens of milliseconds; a capture stream belongs
// to one device).
struct ThreadRes {
  int dev = -1;
  cudaStream_t cap = nullptr;
};
static thread_local ThreadRes t_res[16];
static thread_local int* t_hsum = nullptr;

inline int thread_resources(cudaStream_t* cap, int** hsum) {
  int dev = 0;
  HF_CUDA(cudaGetDevice(&dev));
  ThreadRes& r = t_res[dev & 15];
  if (r.cap == nullptr || r.dev != dev) {
    HF_CUDA(cudaStreamCreateWithFlags(&r.cap, cudaStreamNonBlocking));
    r.dev = dev;
  }
  if (t_hsum == nullptr)  // summary words, then the per-slot states of hf_pcg_stream
    HF_CUDA(cudaHostAlloc(&t_hsum, sizeof(int) * (SUM_N + 64), cudaHostAllocPortable));
  *cap = r.cap;
  *hsum = t_hsum;
  return HF_OK;
}

template <int KP>
int run(const hf_csr* A, const double* d, const double* B, int n, double tol, int max_iter,
        const int32_t* freeze_at, double* X, int32_t* iters, int32_t* status, double* true_res,
        double* best_res, int32_t* best_iter, void* ws, size_t ws_bytes, cudaStream_t stream) {
  using M = Map<KP>;
  Layout L = carve(ws, n, KP);
  if (L.bytes > ws_bytes) {
    set_error("pcg workspace too small: need %zu, have %zu", L.bytes, ws_bytes);
    return HF_ERR_WORKSPACE;
  }
  Grids g;
  if (int rc = setup<KP>(L, A, n, tol, max_iter, g, stream)) return rc;
  if (freeze_at != nullptr) {
    HF_CUDA(cudaMemcpyAsync(L.freeze, freeze_at, sizeof(int) * KP, cudaMemcpyDeviceToDevice, stream));
    for (Ctl* k : {&g.c, &g.cp, &g.cx, &g.crp}) k->freeze = L.freeze;
  }
  HF_CUDA(cudaMemsetAsync(L.counter, 0, sizeof(unsigned int) * 4, stream));
  HF_CUDA(cudaMemsetAsync(L.xmask, 0, sizeof(int) * (XD + 1) * KP, stream));
  HF_CUDA(cudaMemsetAsync(L.summary, 0, sizeof(int) * SUM_N, stream));
  k_init<KP><<<g.c.G, M::NT, 0, stream>>>(g.c, B, d, X, L.R, L.P);
  HF_LAUNCH_CHECK();
  count_launches(1);

  cudaStream_t cap = nullptr;
  int* h_sum = nullptr;
  if (int rc = thread_resources(&cap, &h_sum)) return rc;
  struct Guard {
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    cudaEvent_t ev[LOOKAHEAD + 1] = {};
    ~Guard() {
      if (ge) cudaGraphExecDestroy(ge);
      if (g) cudaGraphDestroy(g);
      for (auto e : ev)
        if (e) cudaEventDestroy(e);
    }
  } guard;
  HF_CUDA(cudaMemcpyAsync(h_sum, L.summary, sizeof(int) * SUM_N, cudaMemcpyDeviceToHost, stream));
  HF_CUDA(cudaStreamSynchronize(stream));

  if (h_sum[SUM_RUN] > 0) {
    // Capture one chunk: CHUNK rounds, the check path, then the status copy.
    HF_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    for (int r = 0; r < CHUNK; ++r) launch_round<KP>(g, L, X, r, cap, nullptr);
    launch_check<KP>(g, L, B, X, cap);
    cudaMemcpyAsync(h_sum, L.summary, sizeof(int) * SUM_N, cudaMemcpyDeviceToHost, cap);
    const cudaError_t le = cudaGetLastError();
    const cudaError_t ce = cudaStreamEndCapture(cap, &guard.g);
    if (ce != cudaSuccess || le != cudaSuccess) {
      set_error("graph capture failed: %s / %s", cudaGetErrorString(ce), cudaGetErrorString(le));
      return HF_ERR_CUDA;
    }
    HF_CUDA(cudaGraphInstantiate(&guard.ge, guard.g, 0));
    for (auto& e : guard.ev) HF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    // Every chunk advances each running column by at least one iteration (a
    // column that reaches the tolerance in a chunk's first round and is
    // replaced at its end is the slowest case), so max_iter + LOOKAHEAD + a
    // few chunks always suffice; more means the control logic is broken.
    const long max_chunks = (long)max_iter + LOOKAHEAD + 8;
    long i = 0;
    bool finished = false;
    // Keep LOOKAHEAD chunks queued ahead of the status being read, so a late
    // host wake-up never leaves the GPU idle; chunks queued after the last
    // column finished exit at once (every kernel is gated on the status).
    for (; i < max_chunks; ++i) {
      HF_CUDA(cudaGraphLaunch(guard.ge, stream));
      count_launches(PER_CHUNK);
      HF_CUDA(cudaEventRecord(guard.ev[i % (LOOKAHEAD + 1)], stream));
      if (i >= LOOKAHEAD) {
        HF_CUDA(cudaEventSynchronize(guard.ev[(i - LOOKAHEAD) % (LOOKAHEAD + 1)]));
        volatile int* hs = h_sum;
        if (hs[SUM_RUN] == 0 && hs[SUM_CHECK] == 0) {
          finished = true;
          break;
        }
      }
    }
    HF_CUDA(cudaStreamSynchronize(stream));
    if (!finished) {
      volatile int* hs = h_sum;
      if (!(hs[SUM_RUN] == 0 && hs[SUM_CHECK] == 0)) {
        set_error("pcg control did not terminate after %ld chunks", i);
        return HF_ERR_INTERNAL;
      }
    }
  }
  // Per-column results back to the host.
  HF_CUDA(cudaMemcpyAsync(iters, L.iters, sizeof(int) * KP, cudaMemcpyDeviceToHost, stream));
  HF_CUDA(cudaMemcpyAsync(status, L.state, sizeof(int) * KP, cudaMemcpyDeviceToHost, stream));
  HF_CUDA(cudaMemcpyAsync(true_res, L.true_res, sizeof(double) * KP, cudaMemcpyDeviceToHost, stream));
  HF_CUDA(cudaMemcpyAsync(best_res, L.best_res, sizeof(double) * KP, cudaMemcpyDeviceToHost, stream));
  HF_CUDA(cudaMemcpyAsync(best_iter, L.best_iter, sizeof(int) * KP, cudaMemcpyDeviceToHost, stream));
  HF_CUDA(cudaStreamSynchronize(stream));
  return HF_OK;
}

// Column streaming (hf_pcg_stream): L >= 1 columns of Ball through kp slots.  The
// slots are scheduled on the device (k_sched ends every chunk), so a finished slot
// takes its next column at the end of the chunk it finished in; the host only
// keeps LOOKAHEAD chunks queued and stops once every column is finished, then
// harvests the retired slots' x in one pass.
template <int KP>
int run_stream(const hf_csr* A, const double* d, const double* Ball, int ldb, int ncols, int n,
               double tol, int max_iter, double* Xall, int32_t* iters, int32_t* status,
               double* true_res, double* best_res, int32_t* best_iter, void* ws, size_t ws_bytes,
               cudaStream_t stream) {
  using M = Map<KP>;
  Layout L = carve(ws, n, KP);
  Carve cv{reinterpret_cast<char*>(ws), L.bytes, ~size_t(0)};
  double* Bs = cv.take<double>((size_t)n * KP);  // the slots' right-hand sides (check path)
  double* X = cv.take<double>((size_t)n * KP);
  Harvest hv;
  hv.X = Xall;
  hv.iters = cv.take<int>(ncols);
  hv.state = cv.take<int>(ncols);
  hv.best_iter = cv.take<int>(ncols);
  hv.true_res = cv.take<double>(ncols);
  hv.best_res = cv.take<double>(ncols);
  Sched sched;
  int* d_order = cv.take<int>(ncols);
  const bool ordered = ncols > KP && ncols <= RQ_MAXC;
  double* rq_part = ordered ? cv.take<double>((size_t)GRID * 2 * ncols) : nullptr;
  double* rq = ordered ? cv.take<double>(ncols) : nullptr;
  sched.order = d_order;
  sched.slot_col = cv.take<int>(2 * KP + 2);  // slot_col, retired, next, nfin: one block
  sched.retired = sched.slot_col + KP;
  sched.next = sched.slot_col + 2 * KP;
  sched.nfin = sched.next + 1;
  sched.ncols = ncols;
  if (cv.used + 256 > ws_bytes) {
    set_error("pcg stream workspace too small: need %zu, have %zu", cv.used + 256, ws_bytes);
    return HF_ERR_WORKSPACE;
  }
  Grids g;
  if (int rc = setup<KP>(L, A, n, tol, max_iter, g, stream)) return rc;
  cudaStream_t cap = nullptr;
  int* h_sum = nullptr;
  if (int rc = thread_resources(&cap, &h_sum)) return rc;
  int* h_nfin = h_sum + SUM_N;  // finished-column count of the status read (pinned)
  struct Guard {
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    cudaEvent_t ev[LOOKAHEAD + 1] = {};
    ~Guard() {
      if (ge) cudaGraphExecDestroy(ge);
      if (g) cudaGraphDestroy(g);
      for (auto e : ev)
        if (e) cudaEventDestroy(e);
    }
  } guard;
  HF_CUDA(cudaMemsetAsync(L.counter, 0, sizeof(unsigned int) * 4, stream));
  HF_CUDA(cudaMemsetAsync(L.xmask, 0, sizeof(int) * (XD + 1) * KP, stream));
  HF_CUDA(cudaMemsetAsync(L.summary, 0, sizeof(int) * SUM_N, stream));
  HF_CUDA(cudaMemsetAsync(L.state, 0, sizeof(int) * KP, stream));
  // hand-out order: ascending Rayleigh quotient (longest expected first), ties by index
  std::vector<int> order(ncols);
  for (int j = 0; j < ncols; ++j) order[j] = j;
  if (ordered) {
    k_col_rq<<<GRID, RQ_NT, 0, stream>>>(n, g.ell.ci, g.ell.cv, A->indptr, A->indices, A->val, d, Ball, ldb,
                                         ncols, rq_part);
    k_col_rq_sum<<<(ncols + 255) / 256, 256, 0, stream>>>(GRID, ncols, rq_part, rq);
    HF_LAUNCH_CHECK();
    count_launches(2);
    std::vector<double> h_rq(ncols);
    HF_CUDA(cudaMemcpyAsync(h_rq.data(), rq, sizeof(double) * ncols, cudaMemcpyDeviceToHost, stream));
    HF_CUDA(cudaStreamSynchronize(stream));
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return h_rq[a] < h_rq[b]; });
  }
  HF_CUDA(cudaMemcpyAsync(d_order, order.data(), sizeof(int) * ncols, cudaMemcpyHostToDevice, stream));
  // first fill: slot j <- order[j] (b = 0 and state ZERO for slots beyond ncols)
  SlotLists sl;
  std::vector<int> ctl(2 * KP + 2, 0);  // slot_col, retired, next, nfin
  for (int j = 0; j < 64; ++j) sl.refill[j] = sl.harvest[j] = -1;
  for (int j = 0; j < KP; ++j) {
    sl.refill[j] = j < ncols ? order[j] : -2;
    ctl[j] = j < ncols ? order[j] : -1;
  }
  ctl[2 * KP] = std::min(KP, ncols);
  HF_CUDA(cudaMemcpyAsync(sched.slot_col, ctl.data(), sizeof(int) * ctl.size(), cudaMemcpyHostToDevice, stream));
  k_refill<KP><<<g.c.G, M::NT, 0, stream>>>(g.c, sl, Ball, ldb, hv, Bs, d, X, L.R, L.P, 1);
  HF_LAUNCH_CHECK();
  count_launches(1);
  HF_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
  for (int r = 0; r < CHUNK; ++r) launch_round<KP>(g, L, X, r, cap, nullptr);
  launch_check<KP>(g, L, Bs, X, cap);
  k_sched<KP><<<g.c.G, M::NT, 0, cap>>>(g.c, sched, Ball, ldb, hv, Bs, d, X, L.R, L.P);
  cudaMemcpyAsync(h_sum, L.summary, sizeof(int) * SUM_N, cudaMemcpyDeviceToHost, cap);
  cudaMemcpyAsync(h_nfin, sched.nfin, sizeof(int), cudaMemcpyDeviceToHost, cap);
  const cudaError_t le = cudaGetLastError();
  const cudaError_t ce = cudaStreamEndCapture(cap, &guard.g);
  if (ce != cudaSuccess || le != cudaSuccess) {
    set_error("graph capture failed: %s / %s", cudaGetErrorString(ce), cudaGetErrorString(le));
    return HF_ERR_CUDA;
  }
  HF_CUDA(cudaGraphInstantiate(&guard.ge, guard.g, 0));
  for (auto& e : guard.ev) HF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  // every column needs at most max_iter + 1 chunks in its slot and takes its slot
  // at the end of the chunk its predecessor finished in
  const long per_col = (long)max_iter + 2 * LOOKAHEAD + 8;
  const long max_chunks = per_col * ((ncols + KP - 1) / KP + 1);
  int nfin = 0;
  long i = 0;
  for (; i < max_chunks && nfin < ncols; ++i) {
    HF_CUDA(cudaGraphLaunch(guard.ge, stream));
    count_launches(PER_CHUNK + 1);
    HF_CUDA(cudaEventRecord(guard.ev[i % (LOOKAHEAD + 1)], stream));
    if (i < LOOKAHEAD) continue;
    HF_CUDA(cudaEventSynchronize(guard.ev[(i - LOOKAHEAD) % (LOOKAHEAD + 1)]));
    nfin = *(volatile int*)h_nfin;
  }
  HF_CUDA(cudaStreamSynchronize(stream));
  nfin = *(volatile int*)h_nfin;
  if (nfin < ncols) {
    set_error("pcg stream control did not finish: %d of %d columns after %ld chunks", nfin, ncols, i);
    return HF_ERR_INTERNAL;
  }
  // the retired slots' x, in one pass
  HF_CUDA(cudaMemcpyAsync(ctl.data(), sched.slot_col, sizeof(int) * 2 * KP, cudaMemcpyDeviceToHost, stream));
  HF_CUDA(cudaStreamSynchronize(stream));
  for (int j = 0; j < KP; ++j) {
    sl.refill[j] = -1;
    sl.harvest[j] = ctl[KP + j] ? ctl[j] : -1;
  }
  k_refill<KP><<<g.c.G, M::NT, 0, stream>>>(g.c, sl, Ball, ldb, hv, Bs, d, X, L.R, L.P, 0);
  HF_LAUNCH_CHECK();
  count_launches(1);
  HF_CUDA(cudaMemcpyAsync(iters, hv.iters, sizeof(int) * ncols, cudaMemcpyDeviceToHost, stream));
  HF_CUDA(cudaMemcpyAsync(status, hv.state, sizeof(int) * ncols, cudaMemcpyDeviceToHost, stream));
  HF_CUDA(cudaMemcpyAsync(true_res, hv.true_res, sizeof(double) * ncols, cudaMemcpyDeviceToHost, stream));
  HF_CUDA(cudaMemcpyAsync(best_res, hv.best_res, sizeof(double) * ncols, cudaMemcpyDeviceToHost, stream));
  HF_CUDA(cudaMemcpyAsync(best_iter, hv.best_iter, sizeof(int) * ncols, cudaMemcpyDeviceToHost, stream));
  HF_CUDA(cudaStreamSynchronize(stream));
  return HF_OK;
}

inline size_t stream_bytes(int n, int kp, int ncols) {
  Layout L = carve(nullptr, n, kp);
  Carve cv{nullptr, L.bytes, ~size_t(0)};
  cv.take<double>((size_t)n * kp);
  cv.take<double>((size_t)n * kp);
  for (int q = 0; q < 3; ++q) cv.take<int>(ncols);
  for (int q = 0; q < 2; ++q) cv.take<double>(ncols);
  cv.take<int>(ncols);
  if (ncols > kp && ncols <= RQ_MAXC) {
    cv.take<double>((size_t)GRID * 2 * ncols);
    cv.take<double>(ncols);
  }
  cv.take<int>(2 * kp + 2);
  return cv.used + 512;
}

// Per-kernel timing of `rounds` PCG rounds with CUDA events on the launch
// stream (bench.py roofline).  tol = 0 keeps every column running.  ms3 =
// {k_spmm, k_update_r, k_update_p / k_update_xring averaged over the ring}.
template <int KP>
int profile(const hf_csr* A, const double* d, const double* B, int n, int rounds, double* X,
            float* ms3, int* flags_out, void* ws, size_t ws_bytes, cudaStream_t stream) {
  using M = Map<KP>;
  Layout L = carve(ws, n, KP);
  if (L.bytes > ws_bytes) {
    set_error("pcg workspace too small");
    return HF_ERR_WORKSPACE;
  }
  Grids g;
  if (int rc = setup<KP>(L, A, n, 0.0, 1 << 30, g, stream)) return rc;
  *flags_out = 6 | (XD << 8);  // ELL SpMM, x deferred over XD rounds
  rounds = (rounds + XD - 1) / XD * XD;  // whole x-deferral cycles
  HF_CUDA(cudaMemsetAsync(L.counter, 0, sizeof(unsigned int) * 4, stream));
  HF_CUDA(cudaMemsetAsync(L.xmask, 0, sizeof(int) * (XD + 1) * KP, stream));
  HF_CUDA(cudaMemsetAsync(L.summary, 0, sizeof(int) * SUM_N, stream));
  k_init<KP><<<g.c.G, M::NT, 0, stream>>>(g.c, B, d, X, L.R, L.P);
  HF_LAUNCH_CHECK();
  count_launches(1 + 3L * rounds);
  cudaEvent_t ev[4];
  for (auto& e : ev) HF_CUDA(cudaEventCreate(&e));
  double acc[3] = {0, 0, 0};
  for (int r = 0; r < rounds; ++r) {
    cudaEventRecord(ev[0], stream);
    launch_round<KP>(g, L, X, r % CHUNK, stream, ev);
    HF_CUDA(cudaEventSynchronize(ev[3]));
    for (int k = 0; k < 3; ++k) {
      float t = 0.f;
      cudaEventElapsedTime(&t, ev[k], ev[k + 1]);
      acc[k] += t;
    }
  }
  for (auto& e : ev) cudaEventDestroy(e);
  HF_LAUNCH_CHECK();
  for (int k = 0; k < 3; ++k) ms3[k] = (float)(acc[k] / (rounds > 0 ? rounds : 1));
  return HF_OK;
}

// ---------------------------------------------------------------- ldp / prune
__global__ void k_ldp(int n, const int32_t* __restrict__ indptr, const double* __restrict__ val,
                      double* __restrict__ d, int* __restrict__ nzero) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int j = indptr[i]; j < indptr[i + 1]; ++j) s = __dadd_rn(s, fabs(val[j]));  // solver.py:55
  d[i] = s;
  if (s == 0.0) atomicAdd(nzero, 1);
}

__global__ void k_prune_count(int n, const int32_t* __restrict__ indptr,
                              const double* __restrict__ val, int32_t* __restrict__ cnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int c = 0;
  for (int j = indptr[i]; j < indptr[i + 1]; ++j) c += (val[j] != 0.0);
  cnt[i] = c;
}

__global__ void k_prune_fill(int n, const int32_t* __restrict__ indptr,
                             const int32_t* __restrict__ indices, const double* __restrict__ val,
                             const int32_t* __restrict__ off, int32_t* __restrict__ optr,
                             int32_t* __restrict__ oidx, double* __restrict__ oval, int total) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > n) return;
  if (i == n) {
    optr[n] = total;
    return;
  }
  int o = off[i];
  optr[i] = o;
  for (int j = indptr[i]; j < indptr[i + 1]; ++j) {
    const double v = val[j];
    if (v != 0.0) {
      oidx[o] = indices[j];
      oval[o] = v;
      ++o;
    }
  }
}

}  // namespace pcg
}  // namespace hf

using namespace hf;

extern "C" size_t hf_pcg_workspace_bytes(int32_t n, int32_t kp, int64_t nnz) {
  (void)nnz;
  return pcg::carve(nullptr, n, kp).bytes;
}

#define HF_PCG_WIDTHS(X) X(2) X(4) X(8) X(16) X(32) X(64)

extern "C" int hf_pcg_multi(const hf_csr* A, const double* d, const double* B, int32_t n,
                            int32_t kp, double tol, int32_t max_iter, const int32_t* freeze_at,
                            double* X, int32_t* iters, int32_t* status, double* true_res,
                            double* best_res, int32_t* best_iter, void* ws, size_t ws_bytes,
                            void* stream) {
  if (!A || !d || !B || !X || !iters || !status || !true_res || !best_res || !best_iter || !ws) {
    set_error("hf_pcg_multi: null argument");
    return HF_ERR_ARG;
  }
  if (n <= 0 || A->n_rows != n || A->n_cols != n || max_iter < 1 || !(tol > 0.0)) {
    set_error("hf_pcg_multi: bad shape or settings (n=%d rows=%d cols=%d max_iter=%d)", n,
              A->n_rows, A->n_cols, max_iter);
    return HF_ERR_ARG;
  }
  if (n >= (1 << 30)) {
    set_error("hf_pcg_multi: n=%d exceeds the ELL column range", n);
    return HF_ERR_ARG;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
#define HF_PCG_CASE(K)                                                                         \
  case K:                                                                                      \
    return pcg::run<K>(A, d, B, n, tol, max_iter, freeze_at, X, iters, status, true_res,       \
                       best_res, best_iter, ws, ws_bytes, s);
  switch (kp) {
    HF_PCG_WIDTHS(HF_PCG_CASE)
    default:
      set_error("hf_pcg_multi: unsupported column width kp=%d", kp);
      return HF_ERR_ARG;
  }
#undef HF_PCG_CASE
}

extern "C" size_t hf_pcg_stream_workspace_bytes(int32_t n, int32_t kp, int32_t ncols) {
  return pcg::stream_bytes(n, kp, ncols);
}

extern "C" int hf_pcg_stream(const hf_csr* A, const double* d, const double* B, int32_t ldb,
                             int32_t ncols, int32_t n, int32_t kp, double tol, int32_t max_iter,
                             double* X, int32_t* iters, int32_t* status, double* true_res,
                             double* best_res, int32_t* best_iter, void* ws, size_t ws_bytes,
                             void* stream) {
  if (!A || !d || !B || !X || !iters || !status || !true_res || !best_res || !best_iter || !ws) {
    set_error("hf_pcg_stream: null argument");
    return HF_ERR_ARG;
  }
  if (n <= 0 || A->n_rows != n || A->n_cols != n || max_iter < 1 || !(tol > 0.0) || ncols < 1 ||
      ldb < ncols) {
    set_error("hf_pcg_stream: bad shape or settings (n=%d ncols=%d ldb=%d)", n, ncols, ldb);
    return HF_ERR_ARG;
  }
  if (n >= (1 << 30)) {
    set_error("hf_pcg_stream: n=%d exceeds the ELL column range", n);
    return HF_ERR_ARG;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
#define HF_STREAM_CASE(K)                                                                      \
  case K:                                                                                      \
    return pcg::run_stream<K>(A, d, B, ldb, ncols, n, tol, max_iter, X, iters, status,         \
                              true_res, best_res, best_iter, ws, ws_bytes, s);
  switch (kp) {
    HF_PCG_WIDTHS(HF_STREAM_CASE)
    default:
      set_error("hf_pcg_stream: unsupported kp=%d", kp);
      return HF_ERR_ARG;
  }
#undef HF_STREAM_CASE
}

extern "C" int hf_pcg_profile(const hf_csr* A, const double* d, const double* B, int32_t n,
                              int32_t kp, int32_t rounds, double* X, float* ms3, int32_t* flags,
                              void* ws, size_t ws_bytes, void* stream) {
  if (!A || !d || !B || !X || !ms3 || !flags || !ws || n <= 0 || rounds < 1) {
    set_error("hf_pcg_profile: bad argument");
    return HF_ERR_ARG;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
#define HF_PROF_CASE(K) \
  case K:               \
    return pcg::profile<K>(A, d, B, n, rounds, X, ms3, flags, ws, ws_bytes, s);
  switch (kp) {
    HF_PCG_WIDTHS(HF_PROF_CASE)
    default:
      set_error("hf_pcg_profile: unsupported kp=%d", kp);
      return HF_ERR_ARG;
  }
#undef HF_PROF_CASE
}

extern "C" int hf_csr_bandwidth(const hf_csr* A, int32_t* scratch, int32_t* bandwidth,
                                void* stream) {
  if (!A || !scratch || !bandwidth) {
    set_error("hf_csr_bandwidth: null argument");
    return HF_ERR_ARG;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  HF_CUDA(cudaMemsetAsync(scratch, 0, sizeof(int32_t), s));
  const int n = A->n_rows;
  if (n > 0) pcg::k_bandwidth<<<(n + 255) / 256, 256, 0, s>>>(n, A->indptr, A->indices, scratch);
  count_launches(1);
  HF_LAUNCH_CHECK();
  HF_CUDA(cudaMemcpyAsync(bandwidth, scratch, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  HF_CUDA(cudaStreamSynchronize(s));
  return HF_OK;
}

extern "C" int hf_ldp(const hf_csr* A, double* d, int32_t* zero_count, int32_t* n_zero_rows,
                      void* stream) {
  if (!A || !d || !zero_count || !n_zero_rows) {
    set_error("hf_ldp: null argument");
    return HF_ERR_ARG;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  HF_CUDA(cudaMemsetAsync(zero_count, 0, sizeof(int32_t), s));
  const int n = A->n_rows;
  if (n > 0) pcg::k_ldp<<<(n + 255) / 256, 256, 0, s>>>(n, A->indptr, A->val, d, zero_count);
  count_launches(1);
  HF_LAUNCH_CHECK();
  int hz = 0;
  HF_CUDA(cudaMemcpyAsync(&hz, zero_count, sizeof(int), cudaMemcpyDeviceToHost, s));
  HF_CUDA(cudaStreamSynchronize(s));
  *n_zero_rows = hz;
  return HF_OK;
}

extern "C" size_t hf_csr_prune_workspace_bytes(int32_t n_rows) {
  const size_t e = (size_t)n_rows + 1;
  return (2 * e + scan_scratch_elems(n_rows) + 64) * sizeof(int32_t) + 1024;
}

static int prune_scan(const hf_csr* A, void* ws, size_t ws_bytes, int32_t** off_out,
                      int32_t* total, cudaStream_t s) {
  const int n = A->n_rows;
  if (ws_bytes < hf_csr_prune_workspace_bytes(n)) {
    set_error("prune workspace too small");
    return HF_ERR_WORKSPACE;
  }
  Carve cv{reinterpret_cast<char*>(ws), 0, ws_bytes};
  int32_t* cnt = cv.take<int32_t>((size_t)n + 1);
  int32_t* off = cv.take<int32_t>((size_t)n + 1);
  int32_t* scratch = cv.take<int32_t>(scan_scratch_elems(n));
  int32_t* tot = cv.take<int32_t>(4);
  pcg::k_prune_count<<<(n + 255) / 256, 256, 0, s>>>(n, A->indptr, A->val, cnt);
  count_launches(1);
  HF_LAUNCH_CHECK();
  int rc = exclusive_scan_i32(cnt, off, n, scratch, tot, s);
  if (rc) return rc;
  HF_CUDA(cudaMemcpyAsync(total, tot, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  HF_CUDA(cudaStreamSynchronize(s));
  *off_out = off;
  return HF_OK;
}

extern "C" int hf_csr_prune_count(const hf_csr* A, void* ws, size_t ws_bytes, int64_t* nnz_out,
                                  void* stream) {
  if (!A || !ws || !nnz_out) {
    set_error("hf_csr_prune_count: null argument");
    return HF_ERR_ARG;
  }
  int32_t* off = nullptr;
  int32_t total = 0;
  int rc = prune_scan(A, ws, ws_bytes, &off, &total, reinterpret_cast<cudaStream_t>(stream));
  if (rc) return rc;
  *nnz_out = total;
  return HF_OK;
}

extern "C" int hf_csr_prune_fill(const hf_csr* A, void* ws, size_t ws_bytes, int32_t* indptr_out,
                                 int32_t* indices_out, double* val_out, void* stream) {
  if (!A || !ws || !indptr_out) {
    set_error("hf_csr_prune_fill: null argument");
    return HF_ERR_ARG;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int32_t* off = nullptr;
  int32_t total = 0;
  int rc = prune_scan(A, ws, ws_bytes, &off, &total, s);
  if (rc) return rc;
  const int n = A->n_rows;
  pcg::k_prune_fill<<<(n + 256) / 256, 256, 0, s>>>(n, A->indptr, A->indices, A->val, off,
                                                     indptr_out, indices_out, val_out, total);
  count_launches(1);
  HF_LAUNCH_CHECK();
  return HF_OK;
}
