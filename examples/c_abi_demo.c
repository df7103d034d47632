/*
 * c_abi_demo.c — the C ABI (include/hfb200.h) used from plain C99, no Python:
 * transfer_matrix (solver.py:114-141) for a 1-D Laplacian with L right-hand
 * sides, once through hf_pcg_multi (one batch of kp columns) and once through
 * hf_pcg_stream (L columns streamed through fewer slots), checked on the host.
 *
 *   gcc -std=c99 -O2 examples/c_abi_demo.c -I include -I /usr/local/cuda/include \
 *       -L paper_1811_07717_b200/_lib -lhfb200 -L /usr/local/cuda/lib64 -lcudart -lm \
 *       -Wl,-rpath,$PWD/paper_1811_07717_b200/_lib -o /tmp/c_abi_demo && /tmp/c_abi_demo
 *
 * Exit status 0 when every column converged with a true residual <= tol and
 * the two entry points agree bit for bit.
 */
#include <cuda_runtime_api.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "hfb200.h"

#define CHECK_CUDA(x)                                                     \
  do {                                                                    \
    cudaError_t e_ = (x);                                                 \
    if (e_ != cudaSuccess) {                                              \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));            \
      return 2;                                                           \
    }                                                                     \
  } while (0)
#define CHECK_HF(x)                                                       \
  do {                                                                    \
    int s_ = (x);                                                         \
    if (s_ != HF_OK) {                                                    \
      fprintf(stderr, "%s: status %d: %s\n", #x, s_, hf_last_error());    \
      return 3;                                                           \
    }                                                                     \
  } while (0)

enum { N = 3000, L = 40, KP_BATCH = 64, KP_STREAM = 8 };

int main(void) {
  const double tol = 1e-10;
  const int max_iter = (int)(5.0 * sqrt((double)N)) + 1000; /* PcgConfig's rule, solver.py:24-47 */
  /* A: tridiagonal (-1, 2 + 1e-3, -1), sorted CSR */
  int32_t* ip = malloc(sizeof(int32_t) * (N + 1));
  int32_t* ix = malloc(sizeof(int32_t) * 3 * N);
  double* vv = malloc(sizeof(double) * 3 * N);
  int32_t nnz = 0;
  for (int i = 0; i < N; ++i) {
    ip[i] = nnz;
    if (i > 0) { ix[nnz] = i - 1; vv[nnz++] = -1.0; }
    ix[nnz] = i; vv[nnz++] = 2.0 + 1e-3;
    if (i + 1 < N) { ix[nnz] = i + 1; vv[nnz++] = -1.0; }
  }
  ip[N] = nnz;
  /* B: n x L row-major, smooth and rough columns; column 7 is zero */
  double* B = calloc((size_t)N * KP_BATCH, sizeof(double));
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < L; ++j)
      B[(size_t)i * KP_BATCH + j] = (j == 7) ? 0.0 : sin(0.001 * (j + 1) * i) + ((i * (j + 3)) % 17 == 0);

  int32_t *d_ip, *d_ix, *d_zero;
  double *d_vv, *d_d, *d_B, *d_X, *d_Xs;
  CHECK_CUDA(cudaMalloc((void**)&d_ip, sizeof(int32_t) * (N + 1)));
  CHECK_CUDA(cudaMalloc((void**)&d_ix, sizeof(int32_t) * nnz));
  CHECK_CUDA(cudaMalloc((void**)&d_vv, sizeof(double) * nnz));
  CHECK_CUDA(cudaMalloc((void**)&d_zero, sizeof(int32_t)));
  CHECK_CUDA(cudaMalloc((void**)&d_d, sizeof(double) * N));
  CHECK_CUDA(cudaMalloc((void**)&d_B, sizeof(double) * N * KP_BATCH));
  CHECK_CUDA(cudaMalloc((void**)&d_X, sizeof(double) * N * KP_BATCH));
  CHECK_CUDA(cudaMalloc((void**)&d_Xs, sizeof(double) * N * KP_BATCH));
  CHECK_CUDA(cudaMemcpy(d_ip, ip, sizeof(int32_t) * (N + 1), cudaMemcpyHostToDevice));
  CHECK_CUDA(cudaMemcpy(d_ix, ix, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice));
  CHECK_CUDA(cudaMemcpy(d_vv, vv, sizeof(double) * nnz, cudaMemcpyHostToDevice));
  CHECK_CUDA(cudaMemcpy(d_B, B, sizeof(double) * N * KP_BATCH, cudaMemcpyHostToDevice));
  hf_csr A = {N, N, nnz, d_ip, d_ix, d_vv};

  int32_t zero_rows = 0;
  CHECK_HF(hf_ldp(&A, d_d, d_zero, &zero_rows, NULL)); /* solver.py:50-61 */
  if (zero_rows) return 4;

  /* one batch: kp = 64 slots, columns L..63 zero */
  int32_t it[KP_BATCH], st[KP_BATCH], bi[KP_BATCH];
  double tr[KP_BATCH], br[KP_BATCH];
  size_t wsb = hf_pcg_workspace_bytes(N, KP_BATCH, nnz);
  void* ws;
  CHECK_CUDA(cudaMalloc(&ws, wsb));
  CHECK_HF(hf_pcg_multi(&A, d_d, d_B, N, KP_BATCH, tol, max_iter, NULL, d_X, it, st, tr, br, bi, ws, wsb,
                        NULL));
  CHECK_CUDA(cudaFree(ws));

  /* streamed: the same L columns (row stride 64) through 8 slots */
  int32_t its[L], sts[L], bis[L];
  double trs[L], brs[L];
  size_t wss = hf_pcg_stream_workspace_bytes(N, KP_STREAM, L);
  CHECK_CUDA(cudaMalloc(&ws, wss));
  CHECK_CUDA(cudaMemset(d_Xs, 0, sizeof(double) * N * KP_BATCH));
  CHECK_HF(hf_pcg_stream(&A, d_d, d_B, KP_BATCH, L, N, KP_STREAM, tol, max_iter, d_Xs, its, sts, trs, brs,
                         bis, ws, wss, NULL));
  CHECK_CUDA(cudaFree(ws));

  double* X = malloc(sizeof(double) * N * KP_BATCH);
  double* Xs = malloc(sizeof(double) * N * KP_BATCH);
  CHECK_CUDA(cudaMemcpy(X, d_X, sizeof(double) * N * KP_BATCH, cudaMemcpyDeviceToHost));
  CHECK_CUDA(cudaMemcpy(Xs, d_Xs, sizeof(double) * N * KP_BATCH, cudaMemcpyDeviceToHost));

  int bad = 0;
  double worst = 0.0;
  for (int j = 0; j < L; ++j) {
    double rr = 0.0, bb = 0.0;
    for (int i = 0; i < N; ++i) {
      double ax = 0.0;
      for (int k = ip[i]; k < ip[i + 1]; ++k) ax += vv[k] * X[(size_t)ix[k] * KP_BATCH + j];
      const double b = B[(size_t)i * KP_BATCH + j];
      rr += (b - ax) * (b - ax);
      bb += b * b;
      if (Xs[(size_t)i * KP_BATCH + j] != X[(size_t)i * KP_BATCH + j]) ++bad; /* bitwise */
    }
    const double rel = bb > 0.0 ? sqrt(rr / bb) : 0.0;
    if (rel > worst) worst = rel;
    const int want = (j == 7) ? HF_COL_ZERO : HF_COL_DONE;
    if (st[j] != want || sts[j] != want || its[j] != it[j] || trs[j] != tr[j] || rel > 2 * tol) ++bad;
  }
  printf("c_abi_demo: n=%d, %d columns, iterations %d..%d, worst true residual %.2e, mismatches %d\n", N, L,
         it[0], it[L - 1], worst, bad);
  cudaFree(d_ip); cudaFree(d_ix); cudaFree(d_vv); cudaFree(d_zero); cudaFree(d_d);
  cudaFree(d_B); cudaFree(d_X); cudaFree(d_Xs);
  free(ip); free(ix); free(vv); free(B); free(X); free(Xs);
  return bad ? 1 : 0;
}
