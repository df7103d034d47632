// Multi-RHS LDP-PCG for sm_100a.
//
// Restates solver.py:64-111 (pcg_solve) for kp right-hand sides at once: every
// column keeps its own recurrence (alpha, beta, residual replacement, true-
// residual confirmation, best iterate), exactly as transfer_matrix runs them
// one by one (solver.py:114-141); the columns only share the matrix stream.
//
// Layout: every n-vector block (X, R, P, Q, B) is n x kp row-major, so the kp
// values of one mesh node are contiguous (one 128-byte line per 16 columns).
// A row group of LPR lanes owns one mesh node; each lane owns CPL consecutive
// columns and moves them as double2.
//
// One PCG round is three kernels (and three grid-wide reductions):
//   k_spmm_pq   q = A p                      , partial p.q   -> alpha
//   k_update_r  r -= alpha q                 , partial r.r, r.(r/d) -> res, beta, state
//   k_update_xp x += alpha p ; p = r/d + beta p
// which is 80 bytes per node per column per iteration of vector traffic plus
// one CSR read per round.  The x update is deferred to the
// third kernel so x, p and r are each read once.
//
// Columns whose recurrence residual drops below tol freeze in state CHECK; at
// the end of every chunk of rounds the check path computes b - A x for them
// (k_spmm_resid), and either finishes the column or replaces r and resumes it
// (k_replace + k_update_xp), exactly as solver.py:94-102.  Freezing a column
// never changes its arithmetic, only when it is scheduled.
//
// Reductions are deterministic: fixed row->block mapping, fixed in-block tree,
// and the last block to finish sums the per-block partials in block order.
#include <math.h>

#include <algorithm>
#include <vector>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"

namespace hf {
namespace pcg {

constexpr int BLOCK = 512;
constexpr int NWARP = BLOCK / 32;
constexpr int BLOCKS_PER_SM = 2;
constexpr int CHUNK = 8;      // PCG rounds per captured graph
constexpr int LOOKAHEAD = 3;  // chunks queued beyond the one whose status is read

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
  SUM_MASKED = 3,
  SUM_PM = 4,    // columns whose p advances this round
  SUM_XANY = 5,  // x updates pending since the last x round (deferred x)
  SUM_N = 8
};

// Deferred x update.  x_{k+1} = x_k + alpha_k p_k needs nothing else of round
// k, so the x stream is touched once every XD rounds: the p of each round
// goes to its own buffer of a ring of XD (p_{k+1} into slot (k+1) % XD, the
// old p stays), alpha and the x mask of each round go to their own slot, and
// the x round (slot XD-1) replays x += alpha_j p_j for j = 0..XD-1 in order:
// the same sequence of roundings as one update per round, with x read and
// written once per XD rounds instead of every round (80 -> 72 + 8/XD bytes
// per row per column per round).  XD divides CHUNK, so x is current at every
// check path.  A column that stops running keeps its last p in slot pbuf[j]
// (where the check path's replacement finds it).
constexpr int XD = 8;
static_assert(CHUNK % XD == 0, "x rounds fall on chunk ends");

struct Ctl {
  int n, kp, G;
  int nb, tpb, delta;  // k_xs band schedule: bands, tiles per block per band, band reach
  int* xdone;          // k_xs: blocks done with each band's x/p update
  double tol;
  int max_iter;
  double *normb, *rz, *alpha, *beta, *best_res, *true_res;
  int *iters, *best_iter, *state, *xmask, *pmask, *freeze;
  double *part0, *part1;
  double2* dd;  // per row {d_i, 1/d_i}, written by k_init
  unsigned int* counter;
  int* summary;
  int rnd, xd;  // round within the chunk; x-deferral depth (1: x every round)
  int rev;      // ELL rounds: the r update sweeps backward (see r_sweep_bwd)
  int* pbuf;    // per column: ring slot of its p once it stops running
};

struct Csr {
  const int32_t* __restrict__ indptr;
  const int32_t* __restrict__ indices;
  const double* __restrict__ val;
};

template <int KP>
struct Map {
  static constexpr int CPL = (KP >= 64) ? 4 : 2;  // columns per lane: one 256/128-bit access
  static constexpr int LPR = KP / CPL;            // lanes per row
  static constexpr int RB = BLOCK / LPR;                    // rows per block pass
  static constexpr int SPLIT = BLOCK / KP;                  // last-block reduction splits
  static constexpr int RED = (NWARP * KP > BLOCK) ? NWARP * KP : BLOCK;
  // row tiles in flight per thread in the streaming kernels (register budget: 64)
  static constexpr int UR = (CPL == 4) ? 1 : 2;  // k_update_r
  static constexpr int UX = (CPL == 4) ? 1 : 2;  // k_update_xp
};

// Rows are dealt to blocks in tiles of RB rows, round-robin (tile t -> block
// t % G): the whole grid sweeps the mesh as one narrow band, so the rows a
// gather touches one z-plane up or down are still in L2 (a contiguous chunk
// per block made every block's neighbours far apart in time: 4x DRAM re-reads).
__host__ __device__ inline int n_tiles(int n, int rb) { return (n + rb - 1) / rb; }

// Sweep direction.  The rows a kernel touches last are still in L2 when the
// next kernel starts, so in ELL rounds the r update sweeps the tiles backward:
// it starts on the q rows the SpMM wrote last, and ends on the r rows the p
// update (forward) reads first.  The SpMM stays forward (a backward SpMM was
// 5% slower).  C2: p/x update 0.338 -> 0.335 ms, build +0.9%.
__device__ __forceinline__ bool r_sweep_bwd(int rev) { return rev != 0; }

// Column slices of a row move as one 256-bit access (LDG/STG.E.256 on
// sm_100a) when a lane owns 4 columns, else as a 128-bit access.
template <int CPL>
__device__ __forceinline__ void ld_cols(const double* p, double (&v)[CPL]) {
  if constexpr (CPL == 4) {
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
  if constexpr (CPL == 4) {
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
  if constexpr (CPL == 4) {
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
  const double q0 = x * dd.y;
  const double res = fma(-q0, dd.x, x);
  return fma(res, dd.y, q0);
}

// Sum NV per-column values over the block in a fixed order and store the
// block's partial row (KP values per quantity) at part[nv][blockIdx.x*KP].
// (lane g of a row group of LPR lanes holds columns g*CPL .. g*CPL+CPL-1)
template <int KP, int NV, int CPL, int LPR>
__device__ __forceinline__ void block_partials_map(double (&v)[NV][CPL], double* sm,
                                                   double* part0, double* part1) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int glane = tid % LPR;
#pragma unroll
  for (int q = 0; q < NV; ++q)
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      double x = v[q][c];
#pragma unroll
      for (int off = 16; off >= LPR; off >>= 1) x += __shfl_xor_sync(FULL, x, off);
      v[q][c] = x;
    }
  if (lane < LPR) {
#pragma unroll
    for (int q = 0; q < NV; ++q)
#pragma unroll
      for (int c = 0; c < CPL; ++c) sm[(q * NWARP + warp) * KP + glane * CPL + c] = v[q][c];
  }
  __syncthreads();
  for (int col = tid; col < KP; col += BLOCK) {
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double s = 0.0;
      for (int w = 0; w < NWARP; ++w) s += sm[(q * NWARP + w) * KP + col];
      (q == 0 ? part0 : part1)[(size_t)blockIdx.x * KP + col] = s;
    }
  }
}

template <int KP, int NV>
__device__ __forceinline__ void block_partials(double (&v)[NV][Map<KP>::CPL], double* sm,
                                               double* part0, double* part1) {
  block_partials_map<KP, NV, Map<KP>::CPL, Map<KP>::LPR>(v, sm, part0, part1);
}

// Last-block detection; the last block reduces the partials of every block in
// block order into tot[q*KP + col] (shared memory).  Returns true in the last block.
template <int KP, int NV>
__device__ __forceinline__ bool last_block_reduce(const Ctl& c, double* sm, double* tot) {
  using M = Map<KP>;
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(c.counter, 1u) == (unsigned)(c.G - 1));
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
  const int tid = threadIdx.x;
  const int col = tid % KP, sp = tid / KP;
  const int per = (c.G + M::SPLIT - 1) / M::SPLIT;
  const int b0 = sp * per, b1 = min(c.G, b0 + per);
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    const double* part = (q == 0) ? c.part0 : c.part1;
    double a0 = 0.0;
    for (int b = b0; b < b1; ++b) a0 += ld_cg(part + (size_t)b * KP + col);
    sm[(q * M::SPLIT + sp) * KP + col] = a0;
  }
  __syncthreads();
  if (tid < KP) {
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double s = 0.0;
      for (int k = 0; k < M::SPLIT; ++k) s += sm[(q * M::SPLIT + k) * KP + tid];
      tot[q * KP + tid] = s;
    }
  }
  __syncthreads();
  if (tid == 0) *c.counter = 0u;
  return true;
}

__device__ __forceinline__ void recount(const Ctl& c, int kp) {
  // single thread: refresh the run/check counters from the states
  int nrun = 0, nchk = 0;
  for (int j = 0; j < kp; ++j) {
    nrun += (c.state[j] == S_RUN);
    nchk += (c.state[j] == S_CHECK);
  }
  c.summary[SUM_RUN] = nrun;
  c.summary[SUM_CHECK] = nchk;
}

// ---------------------------------------------------------------- init
// x = 0; r = b; z = r/d; p = z; rz = r.z; ||b||   (solver.py:74-85)
template <int KP>
__global__ void __launch_bounds__(BLOCK, BLOCKS_PER_SM)
    k_init(Ctl c, const double* __restrict__ B, const double* __restrict__ d, double* X,
           double* R, double* P) {
  using M = Map<KP>;
  __shared__ double sm[2 * M::RED];
  __shared__ double tot[2 * KP];
  const int tid = threadIdx.x, gl = tid / M::LPR, glane = tid % M::LPR;
  const int nt = n_tiles(c.n, M::RB);
  double v[2][M::CPL];
#pragma unroll
  for (int k = 0; k < M::CPL; ++k) v[0][k] = v[1][k] = 0.0;
  for (int t = blockIdx.x; t < nt; t += c.G) {
    const int row = t * M::RB + gl;
    if (row >= c.n) continue;
    const size_t o = (size_t)row * KP + glane * M::CPL;
    double b[M::CPL], z[M::CPL], zero[M::CPL];
    ld_cols<M::CPL>(B + o, b);
    const double dd = d[row];
    if (glane == 0) c.dd[row] = make_double2(dd, 1.0 / dd);
#pragma unroll
    for (int k = 0; k < M::CPL; ++k) {
      z[k] = b[k] / dd;
      zero[k] = 0.0;
      v[0][k] += b[k] * b[k];
      v[1][k] += b[k] * z[k];
    }
    st_cols<M::CPL>(X + o, zero);
    st_cols<M::CPL>(R + o, b);
    st_cols<M::CPL>(P + o, z);
  }
  block_partials<KP, 2>(v, sm, c.part0, c.part1);
  if (!last_block_reduce<KP, 2>(c, sm, tot)) return;
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
    int st = S_RUN;
    if (nb == 0.0)
      st = S_ZERO;  // solver.py:75-76
    else if (c.freeze != nullptr && c.freeze[j] == 0)
      st = S_FROZEN;
    c.state[j] = st;
  }
  __syncthreads();
  if (tid == 0) {
    recount(c, KP);
    c.summary[SUM_REPLACE] = 0;
    c.summary[SUM_MASKED] = 0;
  }
}

// ---------------------------------------------------------------- SpMM
// The SpMM kernels are latency-bound gathers: they run one 512-thread block
// per SM with a 128-register budget and keep R rows x GB gathers in flight
// per lane group (all loads issued before any FMA consumes them).
constexpr int ELL_W = 8;  // slots per row of the ELL SpMM copy (= the gather batch)
#ifndef HF_GB
#define HF_GB 8
#endif
constexpr int GB = HF_GB;  // gathers per batch

template <int KP>
struct Spmm {
  static constexpr int R = 1;  // rows per row group per step (pipelined across steps)
  // 4-column lanes hold 8 x 256-bit gathers in registers: one block per SM
  // with a 128-register budget; 2-column lanes fit two blocks per SM.
  static constexpr int BPS = (Map<KP>::LPR >= 4) ? 1 : 2;
  // (index, value) pairs each lane of a row group holds for the pipeline
  static constexpr int EPL = (Map<KP>::LPR >= 16) ? 1 : 2;  // CAP = LPR*EPL >= 8 entries
  static constexpr bool PIPELINED = Map<KP>::LPR >= 4;
};

// acc[r] = sum_j a_ij * V[col_j, lane columns] for the R rows of this row group.
// The rows' (index, value) pairs are loaded cooperatively by the group and
// broadcast with shuffles; loop bounds are warp-uniform so shuffles never
// diverge.  `any` false skips the gathers (no active column in this lane).
template <int KP, int R>
__device__ __forceinline__ void gather_rows(const Csr& A, const double* __restrict__ V,
                                            const int (&row)[R], bool any,
                                            double (&acc)[R][Map<KP>::CPL]) {
  using M = Map<KP>;
  constexpr int CPL = M::CPL, LPR = M::LPR;
  const int glane = threadIdx.x % LPR;
  int start[R], len[R];
  int maxlen = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) {
#pragma unroll
    for (int k = 0; k < CPL; ++k) acc[r][k] = 0.0;
    start[r] = 0;
    len[r] = 0;
    if (row[r] >= 0) {
      start[r] = A.indptr[row[r]];
      len[r] = A.indptr[row[r] + 1] - start[r];
    }
    maxlen = max(maxlen, len[r]);
  }
  if (LPR < 32) maxlen = (int)__reduce_max_sync(FULL, (unsigned)maxlen);
  const double* __restrict__ Vl = V + glane * CPL;
  for (int c0 = 0; c0 < maxlen; c0 += LPR) {
    int ci[R];
    double cv[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int jj = c0 + glane;
      ci[r] = 0;
      cv[r] = 0.0;
      if (jj < len[r]) {
        ci[r] = __ldg(A.indices + start[r] + jj);
        cv[r] = __ldg(A.val + start[r] + jj);
      }
    }
    if (LPR == 1) {  // one row per thread: the thread walks its own entries
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (c0 < len[r] && any) {
          double g[CPL];
          ldg_cols<CPL>(Vl + (size_t)ci[r] * KP, g);
#pragma unroll
          for (int k = 0; k < CPL; ++k) acc[r][k] = fma(cv[r], g[k], acc[r][k]);
        }
      continue;
    }
    const int nchunk = min(LPR, maxlen - c0);
    for (int b = 0; b < nchunk; b += GB) {
      double g[R][GB][CPL];
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int t = 0; t < GB; ++t) {
          const int e = b + t;
          const int cc = __shfl_sync(FULL, ci[r], e & (LPR - 1), LPR);
          if (e < nchunk && c0 + e < len[r] && any) {
            ldg_cols<CPL>(Vl + (size_t)cc * KP, g[r][t]);
          } else {
#pragma unroll
            for (int k = 0; k < CPL; ++k) g[r][t][k] = 0.0;
          }
        }
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int t = 0; t < GB; ++t) {
          const int e = b + t;
          const double vv = __shfl_sync(FULL, cv[r], e & (LPR - 1), LPR);
          if (e < nchunk && c0 + e < len[r]) {
#pragma unroll
            for (int k = 0; k < CPL; ++k) acc[r][k] = fma(vv, g[r][t][k], acc[r][k]);
          }
        }
    }
  }
}

// Tile schedules: slot s of a block -> tile index (>= the tile count: idle).
struct LinearSched {  // tiles blockIdx.x + s*G (the whole grid sweeps one band)
  int G;
  __device__ __forceinline__ int tile(int s) const { return blockIdx.x + s * G; }
};
struct BandSched {  // band-major: band b holds G*tpb tiles, tpb per block (k_xs)
  int G, tpb;
  __device__ __forceinline__ int tile(int s) const {
    return (s / tpb) * G * tpb + blockIdx.x + G * (s % tpb);
  }
};
struct NoHook {
  __device__ __forceinline__ void operator()(int) const {}
};

template <int KP>
__device__ __forceinline__ void load_meta(const Ctl& c, const Csr& A, int tile, int nt, int& row,
                                          int& st, int& ln) {
  using M = Map<KP>;
  const int rw = tile * M::RB + threadIdx.x / M::LPR;
  row = (tile < nt && rw < c.n) ? rw : -1;
  st = 0;
  ln = 0;
  if (row >= 0) {
    st = __ldg(A.indptr + row);
    ln = __ldg(A.indptr + row + 1) - st;
  }
}

template <int KP>
__device__ __forceinline__ void load_entries(const Csr& A, int st, int ln,
                                             int (&ci)[Spmm<KP>::EPL],
                                             double (&cv)[Spmm<KP>::EPL]) {
  constexpr int LPR = Map<KP>::LPR;
  const int glane = threadIdx.x % LPR;
#pragma unroll
  for (int q = 0; q < Spmm<KP>::EPL; ++q) {
    const int e = q * LPR + glane;
    ci[q] = 0;
    cv[q] = 0.0;
    if (e < ln) {
      ci[q] = __ldg(A.indices + st + e);
      cv[q] = __ldg(A.val + st + e);
    }
  }
}

template <int CPL, bool NC>
__device__ __forceinline__ void gather_cols(const double* p, double (&v)[CPL]) {
  if constexpr (NC)
    ldg_cols<CPL>(p, v);
  else
    ld_cols<CPL>(p, v);  // coherent: V is written inside the same launch (k_xs)
}

// Sweep over a block's slots: calls hook(s) at the top of slot s, then
// epi(row, acc) with acc = sum_j a_ij V[col_j, lane columns] for the slot's row
// (row < 0: idle).  For row groups of >= 8 lanes the CSR stream is
// software-pipelined in registers: row pointers 3 slots ahead, (index, value)
// pairs 2 slots ahead (lane g of a row group holds entries g, g+LPR, ...), an
// L2 bulk prefetch of each row's largest-index neighbour 1 slot ahead (on a
// grid-ordered mesh the +z neighbour, the row the sweep touches first, i.e.
// the DRAM miss), and the current slot's gathers issued GB at a time before
// any FMA consumes them.  So a row costs one memory latency instead of three
// dependent ones (indptr -> indices -> gathered rows).
template <int KP, bool NC, class Sched, class Hook, class Epi>
__device__ __forceinline__ void spmm_slots(const Ctl& c, const Csr& A, const double* V, bool any,
                                           int nslots, const Sched& sc, Hook&& hook, Epi&& epi) {
  using M = Map<KP>;
  static_assert(Spmm<KP>::R == 1, "one row per row group per slot");
  constexpr int LPR = M::LPR, CPL = M::CPL, EPL = Spmm<KP>::EPL;
  constexpr int CAP = LPR * EPL;  // entries per row served from registers
  const int nt = n_tiles(c.n, M::RB);
  const int glane = threadIdx.x % LPR;
  const double* Vl = V + glane * CPL;
  auto tile_of = [&](int s) { return s < nslots ? sc.tile(s) : nt; };
  if constexpr (!Spmm<KP>::PIPELINED) {
    for (int s = 0; s < nslots; ++s) {
      hook(s);
      int row[1];
      const int t = tile_of(s);
      const int rw = t * M::RB + threadIdx.x / LPR;
      row[0] = (t < nt && rw < c.n) ? rw : -1;
      double acc[1][CPL];
      gather_rows<KP, 1>(A, V, row, any, acc);
      epi(row[0], acc[0]);
    }
  } else {
    int row, st, ln, ci[EPL];
    double cv[EPL];
    int rowN, stN, lnN, ciN[EPL];
    double cvN[EPL];
    int rowNN, stNN, lnNN;
    load_meta<KP>(c, A, tile_of(0), nt, row, st, ln);
    load_entries<KP>(A, st, ln, ci, cv);
    load_meta<KP>(c, A, tile_of(1), nt, rowN, stN, lnN);
    load_entries<KP>(A, stN, lnN, ciN, cvN);
    load_meta<KP>(c, A, tile_of(2), nt, rowNN, stNN, lnNN);
    for (int s = 0; s < nslots; ++s) {
      int ciNN[EPL], rowN3, stN3, lnN3;
      double cvNN[EPL];
      load_entries<KP>(A, stNN, lnNN, ciNN, cvNN);             // slot s+2 pairs
      load_meta<KP>(c, A, tile_of(s + 3), nt, rowN3, stN3, lnN3);  // slot s+3 pointers
      hook(s);
      if (any) {
        const int e = lnN - 1;  // sorted columns: the last entry is the largest index
        if (e >= 0 && e < CAP && glane == e % LPR) {
          const int cc = (e / LPR == 0) ? ciN[0] : ciN[EPL - 1];
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(V + (size_t)cc * KP),
                       "r"(KP * 8)
                       : "memory");
        }
      }
      double acc[CPL];
#pragma unroll
      for (int k = 0; k < CPL; ++k) acc[k] = 0.0;
      int maxlen = ln;
      if (LPR < 32) maxlen = (int)__reduce_max_sync(FULL, (unsigned)maxlen);
      const int lim = any ? min(ln, CAP) : 0;  // entries gathered from registers
      const int inreg = min(maxlen, CAP);
      // entry e sits in lane e % LPR, register slot e / LPR (compile-time per t)
#pragma unroll
      for (int b = 0; b < CAP; b += GB) {
        if (b >= inreg) break;
        double g[GB][CPL];
#pragma unroll
        for (int t = 0; t < GB; ++t) {
          const int e = b + t;
          if (e >= CAP) break;
          const int cc = __shfl_sync(FULL, ci[e / LPR], e % LPR, LPR);
          if (e < lim) gather_cols<CPL, NC>(Vl + (size_t)cc * KP, g[t]);
        }
        // consume the batch last-issued first: the first FMA waits on the last
        // gather, so the scheduler cannot start FMAs before every gather is issued
#pragma unroll
        for (int t = GB - 1; t >= 0; --t) {
          const int e = b + t;
          if (e >= CAP) continue;
          const double vv = __shfl_sync(FULL, cv[e / LPR], e % LPR, LPR);
          if (e < lim) {
#pragma unroll
            for (int k = 0; k < CPL; ++k) acc[k] = fma(vv, g[t][k], acc[k]);
          }
        }
      }
      if (maxlen > CAP) {  // long rows: remaining entries straight from memory
        for (int e = CAP; e < ln; ++e) {
          const int cc = __ldg(A.indices + st + e);
          const double vv = __ldg(A.val + st + e);
          if (any) {
            double g[CPL];
            gather_cols<CPL, NC>(Vl + (size_t)cc * KP, g);
#pragma unroll
            for (int k = 0; k < CPL; ++k) acc[k] = fma(vv, g[k], acc[k]);
          }
        }
      }
      epi(row, acc);
      row = rowN;
      st = stN;
      ln = lnN;
#pragma unroll
      for (int q = 0; q < EPL; ++q) {
        ci[q] = ciN[q];
        cv[q] = cvN[q];
        ciN[q] = ciNN[q];
        cvN[q] = cvNN[q];
      }
      rowN = rowNN;
      stN = stNN;
      lnN = lnNN;
      rowNN = rowN3;
      stNN = stN3;
      lnNN = lnN3;
    }
  }
}

template <int KP, class Epi>
__device__ __forceinline__ void spmm_sweep(const Ctl& c, const Csr& A, const double* __restrict__ V,
                                           bool any, Epi&& epi) {
  const int nt = n_tiles(c.n, Map<KP>::RB);
  const int nslots = (nt - (int)blockIdx.x + c.G - 1) / c.G;
  spmm_slots<KP, true>(c, A, V, any, nslots, LinearSched{c.G}, NoHook{}, epi);
}

// q = A p, partial p.q, alpha = rz / p.q       (solver.py:87-88)
template <int KP>
__global__ void __launch_bounds__(BLOCK, Spmm<KP>::BPS)
    k_spmm_pq(Ctl c, Csr A, const double* __restrict__ P, double* __restrict__ Q, int mode) {
  // mode 0: every RUN column; mode 1: the columns the check path just resumed
  // (pmask), so that q = A p exists for them before the next k_update_r.
  using M = Map<KP>;
  __shared__ double sm[M::RED];
  __shared__ double tot[KP];
  __shared__ int s_act[KP];
  if (c.summary[mode == 0 ? SUM_RUN : SUM_REPLACE] == 0) return;
  const int tid = threadIdx.x, glane = tid % M::LPR;
  for (int j = tid; j < KP; j += BLOCK)
    s_act[j] = (mode == 0) ? (c.state[j] == S_RUN) : (c.pmask[j] != 0);
  __syncthreads();
  bool act[M::CPL];
  bool any = false;
#pragma unroll
  for (int k = 0; k < M::CPL; ++k) {
    act[k] = s_act[glane * M::CPL + k];
    any |= act[k];
  }
  const int nt = n_tiles(c.n, M::RB);
  double v[1][M::CPL];
#pragma unroll
  for (int k = 0; k < M::CPL; ++k) v[0][k] = 0.0;
  spmm_sweep<KP>(c, A, P, any, [&](int row, double (&acc)[M::CPL]) {
    if (!any || row < 0) return;
    const size_t o = (size_t)row * KP + glane * M::CPL;
    st_cols<M::CPL>(Q + o, acc);
    double p[M::CPL];
    ldg_cols<M::CPL>(P + o, p);
#pragma unroll
    for (int k = 0; k < M::CPL; ++k)
      if (act[k]) v[0][k] += p[k] * acc[k];
  });
  block_partials<KP, 1>(v, sm, c.part0, nullptr);
  if (!last_block_reduce<KP, 1>(c, sm, tot)) return;
  if (tid < KP) {
    if (s_act[tid]) c.alpha[tid] = c.rz[tid] / tot[tid];
  }
}

// ---------------------------------------------------------------- SpMM over an ELL copy
// k_spmm_ell2: q = A p, p.q and alpha like k_spmm_pq, from a padded ELL copy of
// the SpMM matrix (8 slots per row, built once per solve by k_ell_fill2).  The
// row pointers drop out of the dependency chain: a row's gathers wait on one
// coalesced slot load prefetched a step ahead.  Lanes own 2 columns (128-bit
// gathers), so 32 warps/SM keep the gathers in flight by occupancy.  The
// predicated first version (k_spmm_ell: empty slots skipped per slot, slots
// distributed by shuffles) and its variants are A/B-timed in DESIGN.md §3.
#ifndef HF_ELL
#define HF_ELL 1
#endif
#ifndef HF_ELL_BPS
#define HF_ELL_BPS 2
#endif
#ifndef HF_ELL_LEAN_HB
#define HF_ELL_LEAN_HB 4
#endif
#ifndef HF_ELL_CPL
#define HF_ELL_CPL 4
#endif
#ifndef HF_ELL_MAXKP
#define HF_ELL_MAXKP 64  // widest batch served by the ELL kernel (128: 4-column lanes, one row per warp)
#endif
#ifndef HF_ELL_CPL4_MIN
#define HF_ELL_CPL4_MIN 32  // smallest kp with 4-column lanes
#endif
template <int KP>
struct Ell {
  // columns per lane: 4 (256-bit gathers; two rows per warp at kp = 64) for kp >= 32, else 2.
  // At C2 kp = 64, 4 columns per lane halve the instructions and slot broadcasts per row:
  // SpMM 0.269 -> 0.247 ms (0.269 -> 0.263 with batches of 2 gathers)
  static constexpr int CPL = (HF_ELL_CPL == 4 && KP >= HF_ELL_CPL4_MIN) ? 4 : 2;
  static constexpr int LPR = KP / CPL;    // lanes per row (>= 8: lane e holds slot e)
  static constexpr int RB = BLOCK / LPR;  // rows per block step
  static constexpr int HB = HF_ELL_LEAN_HB;  // gathers per batch
  static constexpr bool OK = (KP >= 16 && KP <= HF_ELL_MAXKP);
};

// The ELL copy is built so that slots can be gathered and multiplied
// unconditionally: empty slots 0..ELL_OPT-1 hold (row itself, 0.0), whose
// gather hits L1 (the row's own p) and whose FMA adds an exact zero; empty
// slots from ELL_OPT on hold -1 and are skipped (an interior row fills 7).  The
// diagonal sits in slot 0, so the epilogue's p_i is its gather.  Rows with more
// than 8 entries keep entries 0..7 in the slots and flag bit 30 of slot 0's
// column; their entries 8.. come from the CSR.  Sum order: slots 7..0, then
// entries 8.. in order.  ~110 instructions per row instead of ~210 (predicated
// gathers, zero fills and conditional-FMA selects made the predicated kernel
// issue-bound at 66%).
constexpr int ELL_LONG = 1 << 30;
#ifndef HF_ELL_OPT_FROM
#define HF_ELL_OPT_FROM 5
#endif
constexpr int ELL_OPT = HF_ELL_OPT_FROM;  // first slot gathered only when it holds an entry

__global__ void k_ell_fill2(int n, const int32_t* __restrict__ indptr,
                            const int32_t* __restrict__ indices, const double* __restrict__ val,
                            int* __restrict__ eci, double* __restrict__ ecv) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int st = indptr[i], ln = indptr[i + 1] - st;
  int c[ELL_W];
  double v[ELL_W];
  for (int e = 0; e < ELL_W; ++e) {
    // empty slot: (row, 0.0), gathered unconditionally; slots >= ELL_OPT are
    // gathered only when they hold an entry (-1 = empty)
    c[e] = e >= ELL_OPT ? -1 : i;
    v[e] = 0.0;
    if (e < ln) {
      c[e] = indices[st + e];
      v[e] = val[st + e];
    }
  }
  // the diagonal (when slot-held) goes to slot 0: the epilogue's p_i is its gather
  for (int e = 1; e < ELL_W && e < ln; ++e)
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

template <int KP>
__global__ void __launch_bounds__(BLOCK, HF_ELL_BPS)
    k_spmm_ell2(Ctl c, Csr A, const int* __restrict__ eci, const double* __restrict__ ecv,
                const double* __restrict__ P, double* __restrict__ Q) {
  using E = Ell<KP>;
  constexpr int CPL = E::CPL, LPR = E::LPR, RB = E::RB;
  constexpr int HB = E::HB;  // gathers in flight per batch (batches run 7.. first)
  __shared__ double sm[NWARP * KP > BLOCK ? NWARP * KP : BLOCK];
  __shared__ double tot[KP];
  __shared__ int s_act[KP];
  __shared__ __align__(16) int s_ci[2][RB][ELL_W];
  __shared__ __align__(16) double s_cv[2][RB][ELL_W];
  if (c.summary[SUM_RUN] == 0) return;
  const int tid = threadIdx.x, gl = tid % LPR, grp = tid / LPR;
  for (int j = tid; j < KP; j += BLOCK) s_act[j] = (c.state[j] == S_RUN);
  __syncthreads();
  double m[CPL];  // 1 for the lane's running columns: masks their p.q terms
  bool any = false;
#pragma unroll
  for (int k = 0; k < CPL; ++k) {
    const int a = s_act[gl * CPL + k];
    m[k] = a ? 1.0 : 0.0;
    any |= a != 0;
  }
  const int nt = (c.n + RB - 1) / RB;
  // slots per lane: a row group of LPR >= 8 lanes has lane e hold slot e; with
  // LPR = 4 (kp 16, 4-column lanes) lane e holds slots e and e + 4
  constexpr int SPL = LPR >= ELL_W ? 1 : ELL_W / LPR;
  const int slot = gl < ELL_W ? gl : ELL_W - 1;
  const double* __restrict__ Pl = P + gl * CPL;
  double v[1][CPL];
#pragma unroll
  for (int k = 0; k < CPL; ++k) v[0][k] = 0.0;
  auto tile_row = [&](int tt) {  // tile tt's row of this row group (-1: none)
    const int r = tt * RB + grp;
    return (tt < nt && r < c.n) ? r : -1;
  };
  int t = blockIdx.x;
  int row = tile_row(t);
  int ci[SPL];
  double cv[SPL];
  auto load_slots = [&](int r, int (&cs)[SPL], double (&vs)[SPL]) {
#pragma unroll
    for (int k = 0; k < SPL; ++k) {
      cs[k] = 0;
      vs[k] = 0.0;
      if (r >= 0) {
        cs[k] = __ldg(eci + (size_t)r * ELL_W + slot + k * LPR);
        vs[k] = __ldg(ecv + (size_t)r * ELL_W + slot + k * LPR);
      }
    }
  };
  load_slots(row, ci, cv);
  int b = 0;
  for (; t < nt; t += c.G, b ^= 1) {
    const int rowN = tile_row(t + c.G);
    int ciN[SPL];
    double cvN[SPL];
    load_slots(rowN, ciN, cvN);  // next step's slots in flight during this one
    if (gl < ELL_W) {
#pragma unroll
      for (int k = 0; k < SPL; ++k) {
        s_ci[b][grp][gl + k * LPR] = ci[k];
        s_cv[b][grp][gl + k * LPR] = cv[k];
      }
    }
    __syncwarp();
    if (row >= 0 && any) {
      const int4 c0 = *reinterpret_cast<const int4*>(&s_ci[b][grp][0]);
      const int4 c1 = *reinterpret_cast<const int4*>(&s_ci[b][grp][4]);
      const int cc[ELL_W] = {c0.x & (ELL_LONG - 1), c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
      const double2* vp = reinterpret_cast<const double2*>(&s_cv[b][grp][0]);
      double a[CPL];
#pragma unroll
      for (int k = 0; k < CPL; ++k) a[k] = 0.0;
      double g0[CPL];  // slot 0's gather: p_i when slot 0 is the diagonal
#pragma unroll
      for (int bt = ELL_W / HB - 1; bt >= 0; --bt) {
        double g[HB][CPL];
#pragma unroll
        for (int k = 0; k < HB; ++k) {
          const int e = bt * HB + k;
          if (e >= ELL_OPT) {  // optional slot: zero when empty
#pragma unroll
            for (int q = 0; q < CPL; ++q) g[k][q] = 0.0;
            if (cc[e] >= 0) ldg_cols<CPL>(Pl + (size_t)cc[e] * KP, g[k]);
          } else {
            ldg_cols<CPL>(Pl + (size_t)(unsigned)cc[e] * KP, g[k]);
          }
        }
        if (bt == 0) {
#pragma unroll
          for (int q = 0; q < CPL; ++q) g0[q] = g[0][q];
        }
#pragma unroll
        for (int k2 = HB / 2 - 1; k2 >= 0; --k2) {
          const double2 vv = vp[bt * HB / 2 + k2];
#pragma unroll
          for (int q = 0; q < CPL; ++q) a[q] = fma(vv.y, g[2 * k2 + 1][q], a[q]);
#pragma unroll
          for (int q = 0; q < CPL; ++q) a[q] = fma(vv.x, g[2 * k2][q], a[q]);
        }
      }
      if (c0.x & ELL_LONG) {  // entries 8.. of a long row, in order
        const int st = __ldg(A.indptr + row), en = __ldg(A.indptr + row + 1);
        for (int j = st + ELL_W; j < en; ++j) {
          const int ce = __ldg(A.indices + j);
          const double ve = __ldg(A.val + j);
          double q2[CPL];
          ldg_cols<CPL>(Pl + (size_t)ce * KP, q2);
#pragma unroll
          for (int q = 0; q < CPL; ++q) a[q] = fma(ve, q2[q], a[q]);
        }
      }
      const size_t o = (size_t)row * KP + gl * CPL;
      st_cols<CPL>(Q + o, a);
      double pr[CPL];
      if (cc[0] == row) {
#pragma unroll
        for (int q = 0; q < CPL; ++q) pr[q] = g0[q];
      } else {
        ldg_cols<CPL>(P + o, pr);
      }
#pragma unroll
      for (int q = 0; q < CPL; ++q) v[0][q] = fma(pr[q] * a[q], m[q], v[0][q]);
    }
    row = rowN;
#pragma unroll
    for (int k = 0; k < SPL; ++k) {
      ci[k] = ciN[k];
      cv[k] = cvN[k];
    }
  }
  block_partials_map<KP, 1, CPL, LPR>(v, sm, c.part0, nullptr);
  if (!last_block_reduce<KP, 1>(c, sm, tot)) return;
  if (tid < KP) {
    if (s_act[tid]) c.alpha[tid] = c.rz[tid] / tot[tid];
  }
}

// r -= alpha q ; res = |r|/|b| ; best ; tolerance / max_iter ; beta   (solver.py:90-106)
template <int KP>
__global__ void __launch_bounds__(BLOCK, BLOCKS_PER_SM)
    k_update_r(Ctl c, const double* __restrict__ Q, double* R) {
  using M = Map<KP>;
  __shared__ double sm[2 * M::RED];
  __shared__ double tot[2 * KP];
  __shared__ double s_alpha[KP];
  __shared__ int s_act[KP];
  if (c.summary[SUM_RUN] == 0) {
    if (blockIdx.x == 0) {  // no x update this round (its history slot is read by the x round)
      for (int j = threadIdx.x; j < KP; j += BLOCK) c.xmask[j] = 0;
      if (threadIdx.x == 0) {
        c.summary[SUM_MASKED] = 0;
        c.summary[SUM_PM] = 0;
        if (c.rnd % c.xd == 0) c.summary[SUM_XANY] = 0;
      }
    }
    return;
  }
  const int tid = threadIdx.x, gl = tid / M::LPR, glane = tid % M::LPR;
  for (int j = tid; j < KP; j += BLOCK) {
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
  const int nt = n_tiles(c.n, M::RB);
  double v[2][M::CPL];
#pragma unroll
  for (int k = 0; k < M::CPL; ++k) v[0][k] = v[1][k] = 0.0;
  if (any) {
    constexpr int U = M::UR;
    const bool bwd = r_sweep_bwd(c.rev);
    for (int t0 = blockIdx.x; t0 < nt; t0 += U * c.G) {
      double r[U][M::CPL], q[U][M::CPL];
      double2 dd[U];
      int rows[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {  // all loads first: U rows in flight
        const int tt = t0 + u * c.G;
        rows[u] = (tt < nt) ? (bwd ? nt - 1 - tt : tt) * M::RB + gl : c.n;
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
            r[u][k] = r[u][k] - al[k] * q[u][k];
            v[0][k] += r[u][k] * r[u][k];
            v[1][k] += r[u][k] * zdiv(r[u][k], dd[u]);
          }
        }
        st_cols<M::CPL>(R + (size_t)rows[u] * KP + glane * M::CPL, r[u]);
      }
    }
  }
  block_partials<KP, 2>(v, sm, c.part0, c.part1);
  if (!last_block_reduce<KP, 2>(c, sm, tot)) return;
  if (tid < KP) {
    const int j = tid;
    int xm = 0, pm = 0;
    if (c.state[j] == S_RUN) {
      const int k = c.iters[j] + 1;
      c.iters[j] = k;
      const double res = sqrt(tot[j]) / c.normb[j];
      if (res < c.best_res[j]) {  // solver.py:92-93
        c.best_res[j] = res;
        c.best_iter[j] = k;
      }
      xm = 1;
      if (c.freeze != nullptr && c.freeze[j] == k) {
        c.state[j] = S_FROZEN;
      } else if (res <= c.tol) {  // solver.py:94
        c.state[j] = S_CHECK;
      } else if (k >= c.max_iter) {  // loop exhausted, solver.py:108
        c.state[j] = S_FAILED;
      } else {
        const double rzn = tot[KP + j];  // solver.py:103-106
        c.beta[j] = rzn / c.rz[j];
        c.rz[j] = rzn;
        pm = 1;
      }
      if (!pm && c.pbuf != nullptr) c.pbuf[j] = c.rnd % c.xd;  // its last p stays in this slot
    }
    c.xmask[j] = xm;
    c.pmask[j] = pm;
  }
  __syncthreads();
  if (tid == 0) {
    recount(c, KP);
    int masked = 0, npm = 0, nxm = 0;
    for (int j = 0; j < KP; ++j) {
      masked += c.xmask[j] | c.pmask[j];
      npm += c.pmask[j];
      nxm += c.xmask[j];
    }
    c.summary[SUM_MASKED] = masked;
    c.summary[SUM_PM] = npm;
    c.summary[SUM_XANY] = (c.rnd % c.xd == 0) ? nxm : c.summary[SUM_XANY] + nxm;
  }
}

// x += alpha p (xmask) ; p = r/d + beta p (pmask)      (solver.py:89,103,107)
template <int KP>
__global__ void __launch_bounds__(BLOCK, BLOCKS_PER_SM)
    k_update_xp(Ctl c, int gate, double* X, double* P, const double* __restrict__ R) {
  using M = Map<KP>;
  __shared__ double s_alpha[KP], s_beta[KP];
  __shared__ int s_xm[KP], s_pm[KP];
  if (c.summary[gate] == 0) return;
  const int tid = threadIdx.x, gl = tid / M::LPR, glane = tid % M::LPR;
  for (int j = tid; j < KP; j += BLOCK) {
    s_xm[j] = c.xmask[j];
    s_pm[j] = c.pmask[j];
    s_alpha[j] = c.alpha[j];
    s_beta[j] = c.beta[j];
  }
  __syncthreads();
  bool xm[M::CPL], pm[M::CPL];
  double al[M::CPL], be[M::CPL];
  bool anyx = false, anyp = false;
#pragma unroll
  for (int k = 0; k < M::CPL; ++k) {
    const int j = glane * M::CPL + k;
    xm[k] = s_xm[j];
    pm[k] = s_pm[j];
    al[k] = s_alpha[j];
    be[k] = s_beta[j];
    anyx |= xm[k];
    anyp |= pm[k];
  }
  if (!anyx && !anyp) return;
  const int nt = n_tiles(c.n, M::RB);
  constexpr int U = M::UX;
  for (int t0 = blockIdx.x; t0 < nt; t0 += U * c.G) {
    double p[U][M::CPL], x[U][M::CPL], r[U][M::CPL];
    double2 dd[U];
    int rows[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {  // all loads first: U rows in flight
      rows[u] = (t0 + u * c.G < nt) ? (t0 + u * c.G) * M::RB + gl : c.n;
      if (rows[u] < c.n) {
        const size_t o = (size_t)rows[u] * KP + glane * M::CPL;
        ld_cols<M::CPL>(P + o, p[u]);
        if (anyx) ld_cols<M::CPL>(X + o, x[u]);
        if (anyp) {
          ld_cols<M::CPL>(R + o, r[u]);
          dd[u] = c.dd[rows[u]];
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (rows[u] >= c.n) continue;
      const size_t o = (size_t)rows[u] * KP + glane * M::CPL;
      if (anyx) {
#pragma unroll
        for (int k = 0; k < M::CPL; ++k)
          if (xm[k]) x[u][k] = x[u][k] + al[k] * p[u][k];
        st_cols<M::CPL>(X + o, x[u]);
      }
      if (anyp) {
#pragma unroll
        for (int k = 0; k < M::CPL; ++k)
          if (pm[k]) p[u][k] = zdiv(r[u][k], dd[u]) + be[k] * p[u][k];
        st_cols<M::CPL>(P + o, p[u]);
      }
    }
  }
}

// ---------------------------------------------------------------- deferred-x rounds
// Round r of a chunk with x deferred (XD > 1): p_{k+1} = r/d + beta p_k into
// ring slot (r+1) % XD, the old p stays in slot r % XD for the x round.
template <int KP>
__global__ void __launch_bounds__(BLOCK, BLOCKS_PER_SM)
    k_update_p(Ctl c, const double* __restrict__ Pcur, double* __restrict__ Pnext,
               const double* __restrict__ R) {
  using M = Map<KP>;
  __shared__ double s_beta[KP];
  __shared__ int s_pm[KP];
  if (c.summary[SUM_PM] == 0) return;
  const int tid = threadIdx.x, gl = tid / M::LPR, glane = tid % M::LPR;
  for (int j = tid; j < KP; j += BLOCK) {
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
  const int nt = n_tiles(c.n, M::RB);
  constexpr int U = M::UX;
  for (int t0 = blockIdx.x; t0 < nt; t0 += U * c.G) {
    double p[U][M::CPL], r[U][M::CPL];
    double2 dd[U];
    int rows[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      rows[u] = (t0 + u * c.G < nt) ? (t0 + u * c.G) * M::RB + gl : c.n;
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
        if (pm[k]) p[u][k] = zdiv(r[u][k], dd[u]) + be[k] * p[u][k];
      st_cols<M::CPL>(Pnext + (size_t)rows[u] * KP + glane * M::CPL, p[u]);
    }
  }
}

// The x round (slot XD-1): x += alpha_j p_j for j = 0..XD-1 in round order
// (each with that round's mask), then p_{k+1} into slot 0.  One block per SM
// with a 128-register budget: a lane keeps x, XD p slices, r in flight.
template <int KP>
__global__ void __launch_bounds__(BLOCK, 1)
    k_update_xring(Ctl c, double* __restrict__ X, double* __restrict__ Pring, size_t nk,
                   const double* __restrict__ R, const double* __restrict__ alpha_h,
                   const int* __restrict__ xmask_h) {
  using M = Map<KP>;
  __shared__ double s_alpha[XD][KP];
  __shared__ int s_xm[XD][KP];
  __shared__ double s_beta[KP];
  __shared__ int s_pm[KP];
  if (c.summary[SUM_XANY] == 0 && c.summary[SUM_PM] == 0) return;
  const int tid = threadIdx.x, gl = tid / M::LPR, glane = tid % M::LPR;
  for (int j = tid; j < XD * KP; j += BLOCK) {
    const int xm = xmask_h[j];
    s_xm[j / KP][j % KP] = xm;
    s_alpha[j / KP][j % KP] = xm ? alpha_h[j] : 0.0;
  }
  for (int j = tid; j < KP; j += BLOCK) {
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
  const int nt = n_tiles(c.n, M::RB);
  for (int t = blockIdx.x; t < nt; t += c.G) {
    const int row = t * M::RB + gl;
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
          if (s_xm[q][j]) x[k] = x[k] + s_alpha[q][j] * p[q][k];
        }
      st_cols<M::CPL>(X + o, x);
    }
    if (anyp) {
      double pn[M::CPL];
#pragma unroll
      for (int k = 0; k < M::CPL; ++k) {
        const int j = glane * M::CPL + k;
        pn[k] = s_pm[j] ? zdiv(r[k], dd) + s_beta[j] * p[CUR][k] : p[CUR][k];
      }
      st_cols<M::CPL>(Pring + o, pn);
    }
  }
}

// Check path with x deferred: a replaced column resumes with p = r/d + beta p
// from the slot its last p stayed in (pbuf) into slot 0.
template <int KP>
__global__ void __launch_bounds__(BLOCK, BLOCKS_PER_SM)
    k_replace_p(Ctl c, double* __restrict__ Pring, size_t nk, const double* __restrict__ R) {
  using M = Map<KP>;
  __shared__ int s_pm[KP], s_buf[KP];
  __shared__ double s_beta[KP];
  if (c.summary[SUM_REPLACE] == 0) return;
  const int tid = threadIdx.x, gl = tid / M::LPR, glane = tid % M::LPR;
  for (int j = tid; j < KP; j += BLOCK) {
    s_pm[j] = c.pmask[j];
    s_buf[j] = c.pbuf[j];
    s_beta[j] = c.beta[j];
  }
  __syncthreads();
  bool anyp = false;
#pragma unroll
  for (int k = 0; k < M::CPL; ++k) anyp |= s_pm[glane * M::CPL + k] != 0;
  if (!anyp) return;
  const int nt = n_tiles(c.n, M::RB);
  for (int t = blockIdx.x; t < nt; t += c.G) {
    const int row = t * M::RB + gl;
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
      Pring[o + k] = zdiv(r[k], dd) + s_beta[j] * pold;
    }
  }
}

// ---------------------------------------------------------------- windowed SpMM (TMA)
// On a grid-ordered mesh the rows one tile of TR consecutive rows gathers form
// a handful of contiguous row ranges (x, y+-1, z+-1 neighbours).  A planner
// (once per operator) records, per tile, those ranges (merged across gaps of
// <= WGAP rows) and each entry's slot in the concatenated window.  The SpMM
// then moves every window with one TMA bulk copy per range
// (cp.async.bulk.shared::cluster.global) into shared memory, double-buffered
// per half block on mbarriers, and reads the neighbour rows from shared
// memory: no register-staged gathers, no L1 traffic, each neighbour row
// fetched once per tile.  Tiles whose window does not fit (irregular meshes)
// fall back to direct gathers.  The sums run over the same entries in the
// same order as k_spmm_pq, so q is bitwise identical.
constexpr int WIN_BYTES = 54 * 1024;  // shared-memory window per tile stage (108 rows at kp=64)
constexpr int RCAP = 8;               // row ranges per window
constexpr int WGAP = 2;               // ranges closer than this merge
constexpr int WCAND = 512;            // columns per tile the planner handles
constexpr int WHALF = BLOCK / 2;      // threads per tile (half block)

template <int KP>
struct Win {
  static constexpr int TR = WHALF / Map<KP>::LPR;  // rows per tile
  static constexpr int ROWB = KP * 8;              // bytes per P row
  static constexpr int WROWS = WIN_BYTES / ROWB;   // window capacity (rows)
  static constexpr int CAP = Map<KP>::LPR;         // entries per row held in registers
};

// tinfo[t] = {nranges (-1: fallback), slot of the tile's first row, window bytes, 0}
__global__ void __launch_bounds__(256) k_plan_windows(int n, int tr, int wrows, int rowb,
                                                      const int32_t* __restrict__ indptr,
                                                      const int32_t* __restrict__ indices,
                                                      int4* __restrict__ tinfo,
                                                      int2* __restrict__ tranges,
                                                      uint16_t* __restrict__ eslot) {
  __shared__ int s_c[8][WCAND];
  __shared__ int s_u[8][WCAND];
  __shared__ short s_slot[8][WCAND];
  __shared__ unsigned char s_f[8][WCAND];
  __shared__ int s_ok[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.x * 8 + warp;
  const int ntile = (n + tr - 1) / tr;
  if (t >= ntile) return;
  const int r0 = t * tr, r1 = min(n, r0 + tr);
  const int e0 = indptr[r0], E = indptr[r1] - e0;
  if (E <= 0 || E > WCAND) {
    if (lane == 0) tinfo[t] = make_int4(-1, 0, 0, 0);
    return;
  }
  int* c = s_c[warp];
  int* u = s_u[warp];
  short* slot = s_slot[warp];
  unsigned char* f = s_f[warp];
  for (int i = lane; i < E; i += 32) c[i] = indices[e0 + i];
  __syncwarp();
  for (int i = lane; i < E; i += 32) {
    bool first = true;
    for (int j = 0; j < i; ++j)
      if (c[j] == c[i]) {
        first = false;
        break;
      }
    f[i] = first;
  }
  __syncwarp();
  int nu = 0;
  for (int i = lane; i < E; i += 32) {
    if (!f[i]) continue;
    int rank = 0;
    for (int j = 0; j < E; ++j) rank += (f[j] && c[j] < c[i]);
    u[rank] = c[i];
    ++nu;
  }
  nu = __reduce_add_sync(FULL, nu);
  __syncwarp();
  if (lane == 0) {  // ranges over the sorted unique columns
    int nr = 0, off = 0, ok = 1, own0 = -1;
    int rs = u[0], re = u[0];
    auto close = [&](int k_end) {
      (void)k_end;
      if (nr < RCAP) tranges[t * RCAP + nr] = make_int2(rs, re - rs + 1);
      off += re - rs + 1;
      ++nr;
    };
    int run_off = 0;
    for (int k = 0; k < nu; ++k) {
      if (k > 0 && u[k] - re > WGAP + 1) {
        close(k);
        run_off = off;
        rs = u[k];
      }
      re = u[k];
      slot[k] = (short)(run_off + (u[k] - rs));
      if (u[k] == r0) own0 = slot[k];
    }
    close(nu);
    if (nr > RCAP || off > wrows || own0 < 0) ok = 0;
    tinfo[t] = ok ? make_int4(nr, own0, off * rowb, 0) : make_int4(-1, 0, 0, 0);
    s_ok[warp] = ok;
  }
  __syncwarp();
  if (!s_ok[warp]) return;
  for (int i = lane; i < E; i += 32) {
    int rank = 0;
    for (int j = 0; j < E; ++j) rank += (f[j] && c[j] < c[i]);
    eslot[e0 + i] = (uint16_t)slot[rank];
  }
}

__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_addr(b)),
      "r"(parity)
      : "memory");
}

// q = A p (mode as k_spmm_pq) through TMA-staged windows.  Each half block
// owns every other tile of the block's sweep (tiles blockIdx.x + G*(2i + h)).
template <int KP>
__global__ void __launch_bounds__(BLOCK, 1)
    k_spmm_win(Ctl c, Csr A, const uint16_t* __restrict__ eslot, const int4* __restrict__ tinfo,
               const int2* __restrict__ tranges, const double* __restrict__ P,
               double* __restrict__ Q, int mode) {
  using M = Map<KP>;
  using Wn = Win<KP>;
  constexpr int LPR = M::LPR, CPL = M::CPL, TR = Wn::TR, ROWB = Wn::ROWB, CAP = Wn::CAP;
  extern __shared__ __align__(1024) unsigned char wsm[];  // [half][stage] windows
  __shared__ __align__(8) uint64_t bar[2][2];
  __shared__ double sm[M::RED];
  __shared__ double tot[KP];
  __shared__ int s_act[KP];
  if (c.summary[mode == 0 ? SUM_RUN : SUM_REPLACE] == 0) return;
  const int tid = threadIdx.x, h = tid / WHALF, ht = tid % WHALF;
  const int gl = ht / LPR, glane = ht % LPR;
  for (int j = tid; j < KP; j += BLOCK)
    s_act[j] = (mode == 0) ? (c.state[j] == S_RUN) : (c.pmask[j] != 0);
  if (ht == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bar[h][0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bar[h][1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  bool act[CPL];
  bool any = false;
#pragma unroll
  for (int k = 0; k < CPL; ++k) {
    act[k] = s_act[glane * CPL + k];
    any |= act[k];
  }
  const int nt = (c.n + TR - 1) / TR;
  const int my = (nt - (int)blockIdx.x + c.G - 1) / c.G;  // tiles of this block
  const int steps = (my + 1) / 2;                          // per half (uniform)
  auto tile_of = [&](int i) {
    const int k = 2 * i + h;
    return k < my ? (int)blockIdx.x + c.G * k : nt;
  };
  unsigned char* win0 = wsm + (size_t)h * 2 * WIN_BYTES;
  // Producer = warp 0 of the half.  The window descriptor of step i+1 (tile
  // info in every lane, range r in lane r) is loaded one step early, so the
  // copies for step i+1 issue at the top of step i without a dependent load.
  const bool pw = ht < 32;
  const int lane = ht & 31;
  int4 ninfo = make_int4(-1, 0, 0, 0);
  int2 nrng = make_int2(0, 0);
  auto load_desc = [&](int i) {
    const int t = tile_of(i);
    ninfo = make_int4(-1, 0, 0, 0);
    nrng = make_int2(0, 0);
    if (t < nt) {
      ninfo = tinfo[t];
      if (lane < RCAP && ninfo.x > lane) nrng = tranges[t * RCAP + lane];
    }
  };
  auto issue = [&](int i) {  // warp 0: window of step i (descriptor in ninfo/nrng) into stage i & 1
    if (ninfo.x < 0) return;
    uint64_t* b = &bar[h][i & 1];
    unsigned char* dst = win0 + (size_t)(i & 1) * WIN_BYTES;
    int off = 0;
    for (int r = 0; r < ninfo.x; ++r) {
      const int st = __shfl_sync(FULL, nrng.x, r);
      const int len = __shfl_sync(FULL, nrng.y, r);
      if (lane == 0) {
        if (r == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)),
                       "r"(ninfo.z)
                       : "memory");
        }
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_addr(dst + (size_t)off * ROWB)),
            "l"(P + (size_t)st * KP), "r"(len * ROWB), "r"(smem_addr(b))
            : "memory");
      }
      off += len;
    }
  };
  // CSR metadata pipelined one step ahead: row pointers and (slot, value) pairs
  auto meta = [&](int i, int& row, int& st, int& ln, int& fb) {
    const int t = tile_of(i);
    row = -1, st = 0, ln = 0, fb = 1;
    if (t >= nt) return;
    fb = tinfo[t].x < 0;
    const int rw = t * TR + gl;
    if (rw >= c.n) return;
    row = rw;
    st = __ldg(A.indptr + rw);
    ln = __ldg(A.indptr + rw + 1) - st;
  };
  auto entries = [&](int st, int ln, int fb, int& ci, double& cv) {
    ci = 0;
    cv = 0.0;
    if (glane < ln) {
      ci = fb ? __ldg(A.indices + st + glane) : (int)__ldg(eslot + st + glane);
      cv = __ldg(A.val + st + glane);
    }
  };
  if (pw) {
    load_desc(0);
    issue(0);
    load_desc(1);
  }
  int row, st, ln, fb, ci;
  double cv;
  meta(0, row, st, ln, fb);
  entries(st, ln, fb, ci, cv);
  int rowN, stN, lnN, fbN;
  meta(1, rowN, stN, lnN, fbN);
  double v[1][CPL];
#pragma unroll
  for (int k = 0; k < CPL; ++k) v[0][k] = 0.0;
  const double* Pl = P + glane * CPL;
  unsigned phase = 0;  // bit s: parity of stage s's next completion (fallback tiles skip a use)
  for (int i = 0; i < steps; ++i) {
    if (pw) {
      issue(i + 1);
      load_desc(i + 2);
    }
    int ciN, rowNN, stNN, lnNN, fbNN;
    double cvN;
    entries(stN, lnN, fbN, ciN, cvN);
    meta(i + 2, rowNN, stNN, lnNN, fbNN);
    const int t = tile_of(i);
    const unsigned char* win = win0 + (size_t)(i & 1) * WIN_BYTES;
    double acc[CPL];
#pragma unroll
    for (int k = 0; k < CPL; ++k) acc[k] = 0.0;
    int maxlen = (int)__reduce_max_sync(FULL, (unsigned)ln);
    const int lim = any ? ln : 0;
    if (!fb) {
      if (t < nt) {
        mbar_wait(&bar[h][i & 1], (phase >> (i & 1)) & 1u);
        phase ^= 1u << (i & 1);
      }
      const double* wl = reinterpret_cast<const double*>(win) + glane * CPL;
      for (int e = 0; e < min(maxlen, CAP); ++e) {
        const int sl = __shfl_sync(FULL, ci, e, LPR);
        const double vv = __shfl_sync(FULL, cv, e, LPR);
        if (e < lim) {
          const double* g = wl + (size_t)sl * KP;
#pragma unroll
          for (int k = 0; k < CPL; k += 2) {
            const double2 gg = *reinterpret_cast<const double2*>(g + k);
            acc[k] = fma(vv, gg.x, acc[k]);
            acc[k + 1] = fma(vv, gg.y, acc[k + 1]);
          }
        }
      }
      for (int e = CAP; e < lim; ++e) {  // rows longer than the lane group
        const int sl = __ldg(eslot + st + e);
        const double vv = __ldg(A.val + st + e);
        const double* g = wl + (size_t)sl * KP;
#pragma unroll
        for (int k = 0; k < CPL; ++k) acc[k] = fma(vv, g[k], acc[k]);
      }
    } else {  // direct gathers
      for (int e = 0; e < min(maxlen, CAP); ++e) {
        const int cc = __shfl_sync(FULL, ci, e, LPR);
        const double vv = __shfl_sync(FULL, cv, e, LPR);
        if (e < lim) {
          double g[CPL];
          ldg_cols<CPL>(Pl + (size_t)cc * KP, g);
#pragma unroll
          for (int k = 0; k < CPL; ++k) acc[k] = fma(vv, g[k], acc[k]);
        }
      }
      for (int e = CAP; e < lim; ++e) {
        const int cc = __ldg(A.indices + st + e);
        const double vv = __ldg(A.val + st + e);
        double g[CPL];
        ldg_cols<CPL>(Pl + (size_t)cc * KP, g);
#pragma unroll
        for (int k = 0; k < CPL; ++k) acc[k] = fma(vv, g[k], acc[k]);
      }
    }
    if (any && row >= 0) {
      const size_t o = (size_t)row * KP + glane * CPL;
      st_cols<CPL>(Q + o, acc);
      double p[CPL];
      if (!fb) {
        const int4 ti = tinfo[t];
        const double* g = reinterpret_cast<const double*>(win) +
                          (size_t)(ti.y + row - t * TR) * KP + glane * CPL;
#pragma unroll
        for (int k = 0; k < CPL; ++k) p[k] = g[k];
      } else {
        ldg_cols<CPL>(P + o, p);
      }
#pragma unroll
      for (int k = 0; k < CPL; ++k)
        if (act[k]) v[0][k] += p[k] * acc[k];
    }
    asm volatile("bar.sync %0, %1;" ::"r"(1 + h), "r"(WHALF) : "memory");  // stage i&1 free
    row = rowN;
    st = stN;
    ln = lnN;
    fb = fbN;
    ci = ciN;
    cv = cvN;
    rowN = rowNN;
    stN = stNN;
    lnN = lnNN;
    fbN = fbNN;
  }
  block_partials<KP, 1>(v, sm, c.part0, nullptr);
  if (!last_block_reduce<KP, 1>(c, sm, tot)) return;
  if (tid < KP) {
    if (s_act[tid]) c.alpha[tid] = c.rz[tid] / tot[tid];
  }
}

// ---------------------------------------------------------------- fused x/p update + SpMM
// One launch does round k's  x += alpha p, p = r/d + beta p  and round k+1's
// q = A p, p.q.  Rows are grouped in bands of G*tpb tiles.  Every block first
// updates its tiles of band b (k_update_xp's arithmetic), publishes that on
// xdone[b], and gathers for band j only after all blocks have published every
// band j' <= j + delta (delta bands cover the matrix bandwidth).  The p rows
// the SpMM gathers were therefore written moments earlier and are still in
// L2: the SpMM's DRAM read of P disappears and the launch count per round
// drops from 3 to 2.  Per-column arithmetic and every reduction order equal
// the three-kernel path (same tiles per block, same in-block trees).
// Requires all G blocks co-resident: launched cooperatively.
template <int KP>
__global__ void __launch_bounds__(BLOCK, Spmm<KP>::BPS)
    k_xs(Ctl c, Csr A, double* X, double* P, const double* __restrict__ R, double* Q) {
  using M = Map<KP>;
  __shared__ double sm[M::RED];
  __shared__ double tot[KP];
  __shared__ double s_alpha[KP], s_beta[KP];
  __shared__ int s_xm[KP], s_pm[KP];
  if (c.summary[SUM_MASKED] == 0) return;  // uniform: every block returns
  const int tid = threadIdx.x, gl = tid / M::LPR, glane = tid % M::LPR;
  for (int j = tid; j < KP; j += BLOCK) {
    s_xm[j] = c.xmask[j];
    s_pm[j] = c.pmask[j];
    s_alpha[j] = c.alpha[j];
    s_beta[j] = c.beta[j];
  }
  __syncthreads();
  // per-column factors stay in shared memory (registers are the SpMM's)
  const int j0 = glane * M::CPL;
  bool anyx = false, anyp = false;
#pragma unroll
  for (int k = 0; k < M::CPL; ++k) {
    anyx |= s_xm[j0 + k] != 0;
    anyp |= s_pm[j0 + k] != 0;
  }
  const int nt = n_tiles(c.n, M::RB);
  const BandSched sc{c.G, c.tpb};
  // x/p update of this block's tiles of band b, then publish it
  auto xphase = [&](int b) {
    if (anyx || anyp) {
      for (int i = 0; i < c.tpb; ++i) {
        const int t = sc.tile(b * c.tpb + i);
        const int row = t * M::RB + gl;
        if (t >= nt || row >= c.n) continue;
        const size_t o = (size_t)row * KP + glane * M::CPL;
        double p[M::CPL], x[M::CPL], r[M::CPL];
        double2 dd;
        ld_cols<M::CPL>(P + o, p);
        if (anyx) ld_cols<M::CPL>(X + o, x);
        if (anyp) {
          ld_cols<M::CPL>(R + o, r);
          dd = c.dd[row];
        }
        if (anyx) {
#pragma unroll
          for (int k = 0; k < M::CPL; ++k)
            if (s_xm[j0 + k]) x[k] = x[k] + s_alpha[j0 + k] * p[k];
          st_cols<M::CPL>(X + o, x);
        }
        if (anyp) {
#pragma unroll
          for (int k = 0; k < M::CPL; ++k)
            if (s_pm[j0 + k]) p[k] = zdiv(r[k], dd) + s_beta[j0 + k] * p[k];
          st_cols<M::CPL>(P + o, p);
        }
      }
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) atomicAdd(c.xdone + b, 1);
  };
  auto wait_band = [&](int b) {
    if (tid == 0) {
      const volatile int* f = c.xdone + b;
      while (*f < c.G) __nanosleep(64);
      __threadfence();
    }
    __syncthreads();
  };
  const int nb = c.nb, dl = c.delta;
  for (int b = 0; b <= dl && b < nb; ++b) xphase(b);
  int xnext = dl + 1;  // next band this block updates
  auto hook = [&](int s) {
    if (s % c.tpb) return;
    const int j = s / c.tpb;  // band whose rows this slot starts
    if (xnext < nb && xnext <= j + dl + 1) xphase(xnext++);
    wait_band(min(j + dl, nb - 1));
  };
  double v[1][M::CPL];
#pragma unroll
  for (int k = 0; k < M::CPL; ++k) v[0][k] = 0.0;
  spmm_slots<KP, false>(c, A, P, anyp, nb * c.tpb, sc, hook, [&](int row, double (&acc)[M::CPL]) {
    if (!anyp || row < 0) return;
    const size_t o = (size_t)row * KP + glane * M::CPL;
    st_cols<M::CPL>(Q + o, acc);
    double p[M::CPL];
    ld_cols<M::CPL>(P + o, p);
#pragma unroll
    for (int k = 0; k < M::CPL; ++k)
      if (s_pm[j0 + k]) v[0][k] += p[k] * acc[k];
  });
  while (xnext < nb) xphase(xnext++);  // (only when the slot loop ended early)
  block_partials<KP, 1>(v, sm, c.part0, nullptr);
  if (!last_block_reduce<KP, 1>(c, sm, tot)) return;
  if (tid < KP) {
    if (s_pm[tid]) c.alpha[tid] = c.rz[tid] / tot[tid];
  }
  for (int b = tid; b < nb; b += BLOCK) c.xdone[b] = 0;  // every block has left its waits
}

// ---------------------------------------------------------------- check path
// s = b - A x for CHECK columns (into Q), true residual, DONE / FAILED / REPLACE
// (solver.py:94-102)
template <int KP>
__global__ void __launch_bounds__(BLOCK, Spmm<KP>::BPS)
    k_spmm_resid(Ctl c, Csr A, const double* __restrict__ B, const double* __restrict__ X,
                 double* __restrict__ Q) {
  using M = Map<KP>;
  __shared__ double sm[M::RED];
  __shared__ double tot[KP];
  __shared__ int s_act[KP];
  if (c.summary[SUM_CHECK] == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) c.summary[SUM_REPLACE] = 0;
    return;
  }
  const int tid = threadIdx.x, glane = tid % M::LPR;
  for (int j = tid; j < KP; j += BLOCK) s_act[j] = (c.state[j] == S_CHECK);
  __syncthreads();
  bool act[M::CPL];
  bool any = false;
#pragma unroll
  for (int k = 0; k < M::CPL; ++k) {
    act[k] = s_act[glane * M::CPL + k];
    any |= act[k];
  }
  const int nt = n_tiles(c.n, M::RB);
  double v[1][M::CPL];
#pragma unroll
  for (int k = 0; k < M::CPL; ++k) v[0][k] = 0.0;
  spmm_sweep<KP>(c, A, X, any, [&](int row, double (&acc)[M::CPL]) {
    if (!any || row < 0) return;
    const size_t o = (size_t)row * KP + glane * M::CPL;
    double b[M::CPL], q[M::CPL];
    ld_cols<M::CPL>(B + o, b);
    ld_cols<M::CPL>(Q + o, q);
#pragma unroll
    for (int k = 0; k < M::CPL; ++k)
      if (act[k]) {
        q[k] = b[k] - acc[k];
        v[0][k] += q[k] * q[k];
      }
    st_cols<M::CPL>(Q + o, q);
  });
  block_partials<KP, 1>(v, sm, c.part0, nullptr);
  if (!last_block_reduce<KP, 1>(c, sm, tot)) return;
  if (tid < KP) {
    const int j = tid;
    if (c.state[j] == S_CHECK) {
      const double t = sqrt(tot[j]) / c.normb[j];
      c.true_res[j] = t;
      if (t <= c.tol)
        c.state[j] = S_DONE;
      else if (c.iters[j] >= c.max_iter)
        c.state[j] = S_FAILED;
      else
        c.state[j] = S_REPLACE;
    }
  }
  __syncthreads();
  if (tid == 0) {
    int nrep = 0;
    for (int j = 0; j < KP; ++j) nrep += (c.state[j] == S_REPLACE);
    c.summary[SUM_REPLACE] = nrep;
    recount(c, KP);
  }
}

// r = s for REPLACE columns, rz_next = r.(r/d), beta, resume   (solver.py:101-106)
template <int KP>
__global__ void __launch_bounds__(BLOCK, BLOCKS_PER_SM)
    k_replace(Ctl c, const double* __restrict__ Q, double* R) {
  using M = Map<KP>;
  __shared__ double sm[M::RED];
  __shared__ double tot[KP];
  __shared__ int s_act[KP];
  if (c.summary[SUM_REPLACE] == 0) return;
  const int tid = threadIdx.x, gl = tid / M::LPR, glane = tid % M::LPR;
  for (int j = tid; j < KP; j += BLOCK) s_act[j] = (c.state[j] == S_REPLACE);
  __syncthreads();
  bool act[M::CPL];
  bool any = false;
#pragma unroll
  for (int k = 0; k < M::CPL; ++k) {
    act[k] = s_act[glane * M::CPL + k];
    any |= act[k];
  }
  const int nt = n_tiles(c.n, M::RB);
  double v[1][M::CPL];
#pragma unroll
  for (int k = 0; k < M::CPL; ++k) v[0][k] = 0.0;
  if (any) {
    for (int t = blockIdx.x; t < nt; t += c.G) {
      const int row = t * M::RB + gl;
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
          v[0][k] += r[k] * zdiv(r[k], dd);
        }
      st_cols<M::CPL>(R + o, r);
    }
  }
  block_partials<KP, 1>(v, sm, c.part0, nullptr);
  if (!last_block_reduce<KP, 1>(c, sm, tot)) return;
  if (tid < KP) {
    const int j = tid;
    int pm = 0;
    if (c.state[j] == S_REPLACE) {
      const double rzn = tot[j];
      c.beta[j] = rzn / c.rz[j];
      c.rz[j] = rzn;
      c.state[j] = S_RUN;
      pm = 1;
    }
    c.xmask[j] = 0;
    c.pmask[j] = pm;
  }
  __syncthreads();
  if (tid == 0) recount(c, KP);
}

// ---------------------------------------------------------------- host driver

inline int grid_for(int n, int kp, int blocks_per_sm = BLOCKS_PER_SM) {
  const int lpr = (kp >= 64) ? kp / 4 : kp / 2;  // Map<KP>::LPR
  const int rb = BLOCK / lpr;
  int g = sm_count() * blocks_per_sm;
  const int need = (n + rb - 1) / rb;
  if (need < g) g = need;
  return g < 1 ? 1 : g;
}

struct Layout {
  double *R, *P, *Q, *part0, *part1;
  double2* dd;
  double *normb, *rz, *alpha, *beta, *best_res, *true_res;
  int *iters, *best_iter, *state, *xmask, *pmask, *freeze;
  int* pbuf;  // deferred x: ring slot of each stopped column's p
  unsigned int* counter;
  int* summary;
  int* xdone;  // k_xs band counters (one per band; bands <= tiles)
  int* bw;     // matrix bandwidth scratch
  int4* tinfo;       // k_spmm_win tile windows
  int2* tranges;
  uint16_t* eslot;
  int* ell_ci;     // k_spmm_ell2: 8 slots per row (see k_ell_fill2)
  double* ell_cv;
  size_t bytes;
};

inline int win_tile_rows(int kp) {  // Win<KP>::TR
  const int lpr = (kp >= 64) ? kp / 4 : kp / 2;  // Map<KP>::LPR
  return WHALF / lpr;
}

inline Layout carve(void* ws, int n, int kp, int64_t nnz) {
  Carve cv{reinterpret_cast<char*>(ws), 0, ~size_t(0)};
  Layout L;
  const size_t nk = (size_t)n * kp;
  const int gmax = sm_count() * 4;  // the most blocks any PCG kernel launches
  L.R = cv.take<double>(nk);
  L.P = cv.take<double>(nk * XD);  // ring of XD p blocks (deferred x); slot 0 otherwise
  L.Q = cv.take<double>(nk);
  L.part0 = cv.take<double>((size_t)gmax * kp);
  L.part1 = cv.take<double>((size_t)gmax * kp);
  L.dd = cv.take<double2>((size_t)n);
  L.normb = cv.take<double>(kp);
  L.rz = cv.take<double>(kp);
  L.alpha = cv.take<double>((size_t)(XD + 1) * kp);  // per-round slots (deferred x)
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
  L.xdone = cv.take<int>((size_t)n + 2);
  L.bw = cv.take<int>(2);
  const size_t ntw = (size_t)(n + win_tile_rows(kp) - 1) / win_tile_rows(kp);
  L.tinfo = cv.take<int4>(ntw + 1);
  L.tranges = cv.take<int2>((ntw + 1) * RCAP);
  L.eslot = cv.take<uint16_t>((size_t)nnz + 8);
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

// The fused x/p-update + SpMM round (k_xs) is correct but, with the SpMM's
// 128-register budget, its streaming half runs at 16 warps/SM and loses to
// the three-kernel round (1.28 vs 1.00 ms at C2, kp=64).  Opt in with
// HFB200_FUSED=1 while it is being reworked (warp-specialised x/p warps).
// k_spmm_ell2 for kp 16..64 (default); HFB200_ELL=0 selects the CSR kernel k_spmm_pq.
inline bool ell_enabled() {
  const char* v = getenv("HFB200_ELL");
  return HF_ELL && !(v && v[0] == '0');
}

// x deferred over a ring of XD p blocks (default); HFB200_XDEFER=0 updates x every round.
inline bool xdefer_enabled() {
  const char* v = getenv("HFB200_XDEFER");
  return !(v && v[0] == '0');
}

inline bool fused_enabled() {
  const char* v = getenv("HFB200_FUSED");
  return v && v[0] == '1';
}

// Control block and grids for one solve.  c: streaming kernels; cs: SpMM and
// fused kernels (one block per SM for 4-column lanes) with the band schedule.
// The TMA-windowed SpMM (k_spmm_win) is correct but, with one window in
// flight per half block, it waits on its mbarriers ~35% of the time and runs
// at 0.54 ms vs 0.33 ms for the register-pipelined gathers (C2, kp=64).
// Opt in with HFB200_WIN=1 while its pipeline is deepened.
inline bool win_enabled() {
  const char* v = getenv("HFB200_WIN");
  return v && v[0] == '1';
}

template <int KP>
int setup(const Layout& L, const hf_csr* A, int n, double tol, int max_iter, Ctl& c, Ctl& cs,
          Ctl& ce, bool& fused, bool& win, bool& ell, cudaStream_t stream) {
  memset(&c, 0, sizeof(c));
  c.n = n;
  c.kp = KP;
  c.G = grid_for(n, KP);
  c.tol = tol;
  c.max_iter = max_iter;
  c.normb = L.normb; c.rz = L.rz; c.alpha = L.alpha; c.beta = L.beta;
  c.best_res = L.best_res; c.true_res = L.true_res; c.iters = L.iters;
  c.best_iter = L.best_iter; c.state = L.state; c.xmask = L.xmask; c.pmask = L.pmask;
  c.freeze = nullptr; c.part0 = L.part0; c.part1 = L.part1; c.dd = L.dd;
  c.counter = L.counter; c.summary = L.summary; c.xdone = L.xdone;
  c.rnd = 0; c.xd = 1; c.pbuf = nullptr; c.rev = 0;
  cs = c;
  cs.G = grid_for(n, KP, Spmm<KP>::BPS);
  win = (KP >= 32) && win_enabled();
  if (win) {  // per-tile TMA windows of the SpMM (once per solve)
    const int tr = Win<KP>::TR;
    const int ntw = (n + tr - 1) / tr;
    k_plan_windows<<<(ntw + 7) / 8, 256, 0, stream>>>(n, tr, Win<KP>::WROWS, Win<KP>::ROWB,
                                                       A->indptr, A->indices, L.tinfo, L.tranges,
                                                       L.eslot);
    HF_LAUNCH_CHECK();
    count_launches(1);
    HF_CUDA(cudaFuncSetAttribute(k_spmm_win<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 4 * WIN_BYTES));
    cs.G = grid_for(n, KP, 1);
  }
  fused = Spmm<KP>::PIPELINED && fused_enabled() && !win;
  if (fused) {  // band schedule from the matrix bandwidth (max |col - row|)
    HF_CUDA(cudaMemsetAsync(L.bw, 0, sizeof(int), stream));
    k_bandwidth<<<(n + 255) / 256, 256, 0, stream>>>(n, A->indptr, A->indices, L.bw);
    HF_LAUNCH_CHECK();
    count_launches(1);
    int bw = 0;
    HF_CUDA(cudaMemcpyAsync(&bw, L.bw, sizeof(int), cudaMemcpyDeviceToHost, stream));
    HF_CUDA(cudaStreamSynchronize(stream));
    const long rows_per_tileset = (long)cs.G * Map<KP>::RB;
    const int nt = n_tiles(n, Map<KP>::RB);
    cs.tpb = (int)std::max<long>(1, (bw + rows_per_tileset - 1) / rows_per_tileset);
    const long band_rows = rows_per_tileset * cs.tpb;
    cs.delta = bw == 0 ? 0 : (int)((bw + band_rows - 1) / band_rows);
    cs.nb = (int)((nt + (long)cs.G * cs.tpb - 1) / ((long)cs.G * cs.tpb));
    HF_CUDA(cudaMemsetAsync(L.xdone, 0, sizeof(int) * (cs.nb + 1), stream));
  }
  if (!fused && xdefer_enabled()) {
    c.xd = XD;
    c.pbuf = L.pbuf;
    cs.xd = XD;
    cs.pbuf = L.pbuf;
  }
  ce = cs;
  ell = false;
  if constexpr (Ell<KP>::OK) {
    ell = !fused && !win && ell_enabled() && n < (1 << 30);  // lean ELL: bit 30 flags long rows
    if (ell) {  // ELL copy of the SpMM matrix (once per solve)
      const int nt = (n + Ell<KP>::RB - 1) / Ell<KP>::RB;
      ce.G = std::max(1, std::min(sm_count() * HF_ELL_BPS, nt));
      k_ell_fill2<<<(n + 255) / 256, 256, 0, stream>>>(n, A->indptr, A->indices, A->val, L.ell_ci,
                                                       L.ell_cv);
      HF_LAUNCH_CHECK();
      count_launches(1);
    }
  }
  return HF_OK;
}

// The unfused round's SpMM: the TMA-window, ELL or CSR kernel.
template <int KP>
inline void launch_round_spmm(const Ctl& cs, const Ctl& ce, const Csr& csr, const Layout& L,
                              const double* P, bool win, bool ell, cudaStream_t q) {
  if (win) {
    k_spmm_win<KP><<<cs.G, BLOCK, 4 * WIN_BYTES, q>>>(cs, csr, L.eslot, L.tinfo, L.tranges, P,
                                                       L.Q, 0);
    return;
  }
  if constexpr (Ell<KP>::OK) {
    if (ell) {
      k_spmm_ell2<KP><<<ce.G, BLOCK, 0, q>>>(ce, csr, L.ell_ci, L.ell_cv, P, L.Q);
      return;
    }
  }
  k_spmm_pq<KP><<<cs.G, BLOCK, 0, q>>>(cs, csr, P, L.Q, 0);
}

// One unfused PCG round r of a chunk: SpMM, r update, then the x/p update
// (x every round, or deferred over the p ring: p-only rounds and the x round).
template <int KP>
inline void launch_round_timed(const Ctl& c0, const Ctl& cs0, const Ctl& ce0, const Csr& csr,
                               const Layout& L, double* X, int r, bool win, bool ell,
                               cudaStream_t q, cudaEvent_t* ev) {
  // ev (profiling only): recorded after the SpMM, the r update and the x/p update
  Ctl c = c0, cs = cs0, ce = ce0;
  const size_t nk = (size_t)c.n * KP;
  for (Ctl* k : {&c, &cs, &ce}) {
    k->rnd = r;
    k->rev = ell ? 1 : 0;
  }
  if (c.xd == 1) {
    launch_round_spmm<KP>(cs, ce, csr, L, L.P, win, ell, q);
    if (ev) cudaEventRecord(ev[1], q);
    k_update_r<KP><<<c.G, BLOCK, 0, q>>>(c, L.Q, L.R);
    if (ev) cudaEventRecord(ev[2], q);
    k_update_xp<KP><<<c.G, BLOCK, 0, q>>>(c, SUM_MASKED, X, L.P, L.R);
    if (ev) cudaEventRecord(ev[3], q);
    return;
  }
  const int slot = r % XD;
  for (Ctl* k : {&c, &cs, &ce}) {
    k->rnd = r;
    k->alpha = L.alpha + (size_t)slot * KP;
    k->xmask = L.xmask + (size_t)slot * KP;
  }
  double* Pc = L.P + (size_t)slot * nk;
  launch_round_spmm<KP>(cs, ce, csr, L, Pc, win, ell, q);
  if (ev) cudaEventRecord(ev[1], q);
  k_update_r<KP><<<c.G, BLOCK, 0, q>>>(c, L.Q, L.R);
  if (ev) cudaEventRecord(ev[2], q);
  if (slot == XD - 1) {
    const int gx = std::max(1, std::min(sm_count(), n_tiles(c.n, Map<KP>::RB)));
    Ctl cx = c;
    cx.G = gx;
    k_update_xring<KP><<<gx, BLOCK, 0, q>>>(cx, X, L.P, nk, L.R, L.alpha, L.xmask);
  } else {
    k_update_p<KP><<<c.G, BLOCK, 0, q>>>(c, Pc, L.P + (size_t)(slot + 1) * nk, L.R);
  }
  if (ev) cudaEventRecord(ev[3], q);
}

template <int KP>
inline void launch_round(const Ctl& c, const Ctl& cs, const Ctl& ce, const Csr& csr,
                         const Layout& L, double* X, int r, bool win, bool ell, cudaStream_t q) {
  launch_round_timed<KP>(c, cs, ce, csr, L, X, r, win, ell, q, nullptr);
}

// The check path after a chunk: s = b - A x, true residuals, replacement.
template <int KP>
inline void launch_check(const Ctl& c0, const Ctl& cs, const Csr& csr, const Layout& L,
                         const double* B, double* X, cudaStream_t q) {
  Ctl c = c0;
  k_spmm_resid<KP><<<cs.G, BLOCK, 0, q>>>(cs, csr, B, X, L.Q);
  if (c.xd == 1) {
    k_replace<KP><<<c.G, BLOCK, 0, q>>>(c, L.Q, L.R);
    k_update_xp<KP><<<c.G, BLOCK, 0, q>>>(c, SUM_REPLACE, X, L.P, L.R);
    return;
  }
  c.xmask = L.xmask + (size_t)XD * KP;  // scratch: the round slots stay untouched
  k_replace<KP><<<c.G, BLOCK, 0, q>>>(c, L.Q, L.R);
  k_replace_p<KP><<<c.G, BLOCK, 0, q>>>(c, L.P, (size_t)c.n * KP, L.R);
}

template <int KP>
cudaError_t launch_xs(const Ctl& cs, const Csr& csr, double* X, double* P, const double* R,
                      double* Q, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs.G);
  cfg.blockDim = dim3(BLOCK);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;  // all blocks co-resident: band waits cannot deadlock
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_xs<KP>, cs, csr, X, P, R, Q);
}

template <int KP>
int run(const hf_csr* A, const double* d, const double* B, int n, double tol, int max_iter,
        const int32_t* freeze_at, double* X, int32_t* iters, int32_t* status, double* true_res,
        double* best_res, int32_t* best_iter, void* ws, size_t ws_bytes, cudaStream_t stream) {
  Layout L = carve(ws, n, KP, A->nnz);
  if (L.bytes > ws_bytes) {
    set_error("pcg workspace too small: need %zu, have %zu", L.bytes, ws_bytes);
    return HF_ERR_WORKSPACE;
  }
  Ctl c, cs, ce;
  bool fused = false, win = false, ell = false;
  Csr csr{A->indptr, A->indices, A->val};
  if (int rc = setup<KP>(L, A, n, tol, max_iter, c, cs, ce, fused, win, ell, stream)) return rc;
  if (freeze_at != nullptr) {
    HF_CUDA(cudaMemcpyAsync(L.freeze, freeze_at, sizeof(int) * KP, cudaMemcpyDeviceToDevice, stream));
    c.freeze = L.freeze;
    cs.freeze = L.freeze;
    ce.freeze = L.freeze;
  }
  HF_CUDA(cudaMemsetAsync(L.counter, 0, sizeof(unsigned int) * 4, stream));
  HF_CUDA(cudaMemsetAsync(L.xmask, 0, sizeof(int) * (XD + 1) * KP, stream));
  HF_CUDA(cudaMemsetAsync(L.summary, 0, sizeof(int) * SUM_N, stream));
  k_init<KP><<<c.G, BLOCK, 0, stream>>>(c, B, d, X, L.R, L.P);
  HF_LAUNCH_CHECK();
  count_launches(1);
  if (fused) {  // q = A p of the first round; later rounds get it from k_xs
    k_spmm_pq<KP><<<cs.G, BLOCK, 0, stream>>>(cs, csr, L.P, L.Q, 0);
    HF_LAUNCH_CHECK();
    count_launches(1);
  }

  // Pinned status words and the capture stream are allocated once per host
  // thread and reused: cudaHostAlloc can stall for tens of milliseconds.
  static thread_local int* h_sum_tls = nullptr;
  static thread_local cudaStream_t cap_tls = nullptr;
  if (!h_sum_tls) HF_CUDA(cudaHostAlloc(&h_sum_tls, sizeof(int) * SUM_N, cudaHostAllocDefault));
  if (!cap_tls) HF_CUDA(cudaStreamCreateWithFlags(&cap_tls, cudaStreamNonBlocking));
  int* h_sum = h_sum_tls;
  struct Guard {
    int* h;
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    cudaStream_t cs = nullptr;
    cudaEvent_t ev[LOOKAHEAD + 1] = {};
    ~Guard() {
      if (ge) cudaGraphExecDestroy(ge);
      if (g) cudaGraphDestroy(g);
      for (auto e : ev)
        if (e) cudaEventDestroy(e);
    }
  } guard{h_sum};
  HF_CUDA(cudaMemcpyAsync(h_sum, L.summary, sizeof(int) * SUM_N, cudaMemcpyDeviceToHost, stream));
  HF_CUDA(cudaStreamSynchronize(stream));

  if (h_sum[SUM_RUN] > 0) {
    // Capture one chunk: CHUNK rounds, then the check path, then the status copy.
    // Unfused round: spmm_pq, update_r, update_xp.  Fused round: update_r,
    // k_xs (= update_xp of this round + spmm_pq of the next).
    auto enqueue_chunk = [&](cudaStream_t q) -> cudaError_t {
      cudaError_t le = cudaSuccess;
      for (int r = 0; r < CHUNK; ++r) {
        if (fused) {
          k_update_r<KP><<<c.G, BLOCK, 0, q>>>(c, L.Q, L.R);
          cudaError_t e = launch_xs<KP>(cs, csr, X, L.P, L.R, L.Q, q);
          if (e != cudaSuccess) le = e;
        } else {
          launch_round<KP>(c, cs, ce, csr, L, X, r, win, ell, q);
        }
      }
      if (fused) {
        k_spmm_resid<KP><<<cs.G, BLOCK, 0, q>>>(cs, csr, B, X, L.Q);
        k_replace<KP><<<c.G, BLOCK, 0, q>>>(c, L.Q, L.R);
        k_update_xp<KP><<<c.G, BLOCK, 0, q>>>(c, SUM_REPLACE, X, L.P, L.R);
      } else {
        launch_check<KP>(c, cs, csr, L, B, X, q);
      }
      if (fused) k_spmm_pq<KP><<<cs.G, BLOCK, 0, q>>>(cs, csr, L.P, L.Q, 1);
      cudaMemcpyAsync(h_sum, L.summary, sizeof(int) * SUM_N, cudaMemcpyDeviceToHost, q);
      return le;
    };
    const char* ng = getenv("HFB200_NOGRAPH");
    const bool use_graph = !(ng && ng[0] == '1');
    if (use_graph) {
      guard.cs = cap_tls;
      HF_CUDA(cudaStreamBeginCapture(guard.cs, cudaStreamCaptureModeThreadLocal));
      cudaError_t le = enqueue_chunk(guard.cs);
      cudaError_t ce = cudaStreamEndCapture(guard.cs, &guard.g);
      if (ce != cudaSuccess || le != cudaSuccess) {
        set_error("graph capture failed: %s / %s", cudaGetErrorString(ce), cudaGetErrorString(le));
        return HF_ERR_CUDA;
      }
      HF_CUDA(cudaGraphInstantiate(&guard.ge, guard.g, 0));
    }
    for (auto& e : guard.ev) HF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    // HFB200_TRACE=1: per-chunk GPU durations on stderr (diagnostics only)
    const char* tr = getenv("HFB200_TRACE");
    const bool trace = tr && tr[0] == '1';
    std::vector<cudaEvent_t> tev;
    const long per_chunk = fused ? 2 * CHUNK + 4 : 3 * CHUNK + 3;
    // Every chunk costs at least one iteration of some column (or finishes a
    // CHECK); bound the loop generously and report if control never settles.
    const long max_chunks = 4L * (max_iter / CHUNK + 2) + 64;
    long i = 0;
    bool finished = false;
    // Keep LOOKAHEAD chunks queued ahead of the status being read, so a late
    // host wake-up never leaves the GPU idle; chunks queued after the last
    // column finished exit at once (every kernel is gated on the status).
    for (; i < max_chunks; ++i) {
      if (trace) {
        tev.emplace_back();
        cudaEventCreate(&tev.back());
        cudaEventRecord(tev.back(), stream);
      }
      if (use_graph) {
        HF_CUDA(cudaGraphLaunch(guard.ge, stream));
      } else {
        HF_CUDA(enqueue_chunk(stream));
        HF_LAUNCH_CHECK();
      }
      count_launches(per_chunk);
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
    if (trace && tev.size() > 1) {
      fprintf(stderr, "[hfb200] chunk ms:");
      for (size_t k = 1; k < tev.size(); ++k) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, tev[k - 1], tev[k]);
        fprintf(stderr, " %.2f", ms);
      }
      fprintf(stderr, "\n");
      for (auto e : tev) cudaEventDestroy(e);
    }
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

// Per-kernel timing of `rounds` PCG rounds with CUDA events on the launch
// stream (bench.py roofline).  tol = 0 keeps every column running.  ms3 =
// {k_spmm_pq, k_update_r, k_update_xp}, or {k_xs, k_update_r, 0} when fused.
template <int KP>
int profile(const hf_csr* A, const double* d, const double* B, int n, int rounds, double* X,
            float* ms3, int* fused_out, void* ws, size_t ws_bytes, cudaStream_t stream) {
  Layout L = carve(ws, n, KP, A->nnz);
  if (L.bytes > ws_bytes) {
    set_error("pcg workspace too small");
    return HF_ERR_WORKSPACE;
  }
  Ctl c, cs, ce;
  bool fused = false, win = false, ell = false;
  Csr csr{A->indptr, A->indices, A->val};
  if (int rc = setup<KP>(L, A, n, 0.0, 1 << 30, c, cs, ce, fused, win, ell, stream)) return rc;
  *fused_out = (fused ? 1 : 0) | (ell ? 6 : 0) | (c.xd << 8);  // 4: the lean ELL kernel
  if (c.xd > 1) rounds = (rounds + XD - 1) / XD * XD;  // whole x-deferral cycles
  HF_CUDA(cudaMemsetAsync(L.counter, 0, sizeof(unsigned int) * 4, stream));
  HF_CUDA(cudaMemsetAsync(L.xmask, 0, sizeof(int) * (XD + 1) * KP, stream));
  HF_CUDA(cudaMemsetAsync(L.summary, 0, sizeof(int) * SUM_N, stream));
  k_init<KP><<<c.G, BLOCK, 0, stream>>>(c, B, d, X, L.R, L.P);
  if (fused) k_spmm_pq<KP><<<cs.G, BLOCK, 0, stream>>>(cs, csr, L.P, L.Q, 0);
  HF_LAUNCH_CHECK();
  count_launches((fused ? 2 : 1) + (fused ? 2L : 3L) * rounds);
  cudaEvent_t ev[4];
  for (auto& e : ev) HF_CUDA(cudaEventCreate(&e));
  double acc[3] = {0, 0, 0};
  for (int r = 0; r < rounds; ++r) {
    if (fused) {
      cudaEventRecord(ev[0], stream);
      HF_CUDA(launch_xs<KP>(cs, csr, X, L.P, L.R, L.Q, stream));
      cudaEventRecord(ev[1], stream);
      k_update_r<KP><<<c.G, BLOCK, 0, stream>>>(c, L.Q, L.R);
      cudaEventRecord(ev[2], stream);
      cudaEventRecord(ev[3], stream);
    } else {  // the events split launch_round's three launches
      cudaEventRecord(ev[0], stream);
      launch_round_timed<KP>(c, cs, ce, csr, L, X, r % CHUNK, win, ell, stream, ev);
    }
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
  for (int j = indptr[i]; j < indptr[i + 1]; ++j) s += fabs(val[j]);  // solver.py:55
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
  return pcg::carve(nullptr, n, kp, nnz).bytes;
}

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
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
#define HF_PCG_CASE(K)                                                                         \
  case K:                                                                                      \
    return pcg::run<K>(A, d, B, n, tol, max_iter, freeze_at, X, iters, status, true_res,       \
                       best_res, best_iter, ws, ws_bytes, s);
  switch (kp) {
    HF_PCG_CASE(2)
    HF_PCG_CASE(4)
    HF_PCG_CASE(8)
    HF_PCG_CASE(16)
    HF_PCG_CASE(32)
    HF_PCG_CASE(64)
    HF_PCG_CASE(128)
    default:
      set_error("hf_pcg_multi: unsupported column width kp=%d", kp);
      return HF_ERR_ARG;
  }
#undef HF_PCG_CASE
}

extern "C" int hf_pcg_profile(const hf_csr* A, const double* d, const double* B, int32_t n,
                              int32_t kp, int32_t rounds, double* X, float* ms3, int32_t* fused,
                              void* ws, size_t ws_bytes, void* stream) {
  if (!A || !d || !B || !X || !ms3 || !fused || !ws || n <= 0 || rounds < 1) {
    set_error("hf_pcg_profile: bad argument");
    return HF_ERR_ARG;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  switch (kp) {
    case 2: return pcg::profile<2>(A, d, B, n, rounds, X, ms3, fused, ws, ws_bytes, s);
    case 4: return pcg::profile<4>(A, d, B, n, rounds, X, ms3, fused, ws, ws_bytes, s);
    case 8: return pcg::profile<8>(A, d, B, n, rounds, X, ms3, fused, ws, ws_bytes, s);
    case 16: return pcg::profile<16>(A, d, B, n, rounds, X, ms3, fused, ws, ws_bytes, s);
    case 32: return pcg::profile<32>(A, d, B, n, rounds, X, ms3, fused, ws, ws_bytes, s);
    case 64: return pcg::profile<64>(A, d, B, n, rounds, X, ms3, fused, ws, ws_bytes, s);
    case 128: return pcg::profile<128>(A, d, B, n, rounds, X, ms3, fused, ws, ws_bytes, s);
    default:
      set_error("hf_pcg_profile: unsupported kp=%d", kp);
      return HF_ERR_ARG;
  }
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
