"""LDP-PCG on the B200: drop-in for headfem/solver.py.

Public names and behaviour follow the reference:
  PcgConfig        solver.py:24-47
  ldp              solver.py:50-61
  pcg_solve        solver.py:64-111
  transfer_matrix  solver.py:114-141
The columns of a transfer matrix are solved together by hf_pcg_multi (one
SpMM per iteration for up to 64 right-hand sides) while each column
keeps its own recurrence, so results do not depend on `threads` or on which
columns share a batch.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
import torch

from . import _native as N
from .device import DeviceCsr, PcgOperator, device, ldp_device, to_host, width_for
from .errors import ConvergenceError, ParameterError, SingularPreconditionerError

MAX_BATCH = 64  # RHS columns per multi-RHS solve (the widest kernel instantiation)


@dataclass(frozen=True)
class PcgConfig:
    """Solver settings; ``max_iterations=None`` resolves to 5 sqrt(n) + 1000."""

    tolerance: float = 1e-8
    max_iterations: int | None = None
    preconditioner: str = "ldp"

    def __post_init__(self):
        if self.tolerance <= 0:
            raise ParameterError("tolerance must be positive")
        if self.max_iterations is not None and self.max_iterations < 1:
            raise ParameterError("max_iterations must be >= 1")
        if self.preconditioner not in ("ldp", "none"):
            raise ParameterError(f"unknown preconditioner '{self.preconditioner}'")

    def resolve_max_iterations(self, n):
        if self.max_iterations is not None:
            return self.max_iterations
        return int(5 * np.sqrt(n)) + 1000


def _max_iter(cfg, n):
    return int(cfg.resolve_max_iterations(n))


@dataclass
class SolveInfo:
    """Per-column outcome of a multi-RHS solve."""

    iterations: np.ndarray
    status: np.ndarray
    true_residual: np.ndarray
    best_residual: np.ndarray
    best_iteration: np.ndarray
    max_iter: int


def _as_device_csr(A):
    if isinstance(A, DeviceCsr):
        return A
    if sp.issparse(A):
        return DeviceCsr.from_scipy(A)
    return DeviceCsr.from_scipy(sp.csr_matrix(np.asarray(A, dtype=float)))


def operator(A, cfg=PcgConfig()):
    """Prepare A (scipy / ndarray / DeviceCsr) for repeated solves."""
    if isinstance(A, PcgOperator):
        return A
    dA = _as_device_csr(A)
    if dA.shape[0] != dA.shape[1]:
        raise ParameterError("matrix must be square")
    return PcgOperator(dA, cfg.preconditioner)


def _run_batch(op, Bb, tol, max_iter, freeze=None):
    """One hf_pcg_multi call on an n x kp block; returns X and host arrays."""
    n, kp = Bb.shape
    X = torch.empty_like(Bb)
    ws = torch.empty(N.lib.hf_pcg_workspace_bytes(n, kp, op.Ac.nnz), dtype=torch.uint8, device=Bb.device)
    it = np.zeros(kp, dtype=np.int32)
    stt = np.zeros(kp, dtype=np.int32)
    tr = np.zeros(kp, dtype=np.float64)
    br = np.zeros(kp, dtype=np.float64)
    bi = np.zeros(kp, dtype=np.int32)
    fz = None
    if freeze is not None:
        fz = torch.from_numpy(np.ascontiguousarray(freeze, dtype=np.int32)).to(Bb.device)
    P = N.C.c_void_p
    N.check("hf_pcg_multi", N.lib.hf_pcg_multi(
        N.C.byref(op.Ac.struct), N.ptr(op.d), N.ptr(Bb), n, kp, float(tol), int(max_iter),
        N.ptr(fz), N.ptr(X), P(it.ctypes.data), P(stt.ctypes.data), P(tr.ctypes.data),
        P(br.ctypes.data), P(bi.ctypes.data), N.ptr(ws), ws.numel(), N.stream_handle()))
    return X, it, stt, tr, br, bi


def solve_block(op, B, cfg=PcgConfig(), batch=MAX_BATCH, out=None):
    """Solve A X = B for an n x k device block B (float64, any k).

    Returns (X, SolveInfo).  Failed columns (status FAILED) come back holding
    their best iterate, recovered by a deterministic replay of the column to
    its best iteration (the reference keeps a copy of x instead, solver.py:92-93).
    """
    n, k = B.shape
    if n != op.n:
        raise ValueError(f"right-hand side has {n} rows, operator has {op.n}")
    max_iter = _max_iter(cfg, n)
    X = out if out is not None else torch.empty((n, k), dtype=torch.float64, device=B.device)
    info = SolveInfo(np.zeros(k, np.int64), np.zeros(k, np.int64), np.zeros(k), np.ones(k),
                     np.zeros(k, np.int64), max_iter)
    batch = max(1, op.batch_width(k, batch))
    if k > batch:  # more columns than slots: stream them through the slots
        return _solve_streamed(op, B, cfg, width_for(batch), max_iter, X, info)
    for c0 in range(0, k, batch):
        c1 = min(k, c0 + batch)
        kb = c1 - c0
        kp = width_for(max(kb, 2))
        Bb = torch.zeros((n, kp), dtype=torch.float64, device=B.device)
        Bb[:, :kb] = B[:, c0:c1]
        Xb, it, stt, tr, br, bi = _run_batch(op, Bb, cfg.tolerance, max_iter)
        failed = np.flatnonzero(stt[:kb] == N.HF_COL_FAILED)
        if failed.size:
            freeze = np.zeros(kp, dtype=np.int32)  # other columns stop at x = 0
            freeze[failed] = bi[failed]
            Xr = _run_batch(op, Bb, cfg.tolerance, max_iter, freeze=freeze)[0]
            idx = torch.from_numpy(failed).to(B.device)
            Xb[:, idx] = Xr[:, idx]
        X[:, c0:c1] = Xb[:, :kb]
        info.iterations[c0:c1] = it[:kb]
        info.status[c0:c1] = stt[:kb]
        info.true_residual[c0:c1] = tr[:kb]
        info.best_residual[c0:c1] = br[:kb]
        info.best_iteration[c0:c1] = bi[:kb]
    return X, info


def _solve_streamed(op, B, cfg, kp, max_iter, X, info):
    """hf_pcg_stream: the k columns of B flow through kp slots, a finished column's
    slot taking the next one at a chunk boundary (no slot waits for the slowest
    column of a batch).  A column's iterates are bit-identical to a batch solve;
    failed columns are replayed to their best iterate in batches."""
    n, k = B.shape
    Bc = B if B.is_contiguous() else B.contiguous()
    if not X.is_contiguous():  # a strided `out`: solve into a dense block, then copy
        Xd, info = _solve_streamed(op, Bc, cfg, kp, max_iter, torch.empty_like(Bc), info)
        X.copy_(Xd)
        return X, info
    ws = torch.empty(N.lib.hf_pcg_stream_workspace_bytes(n, kp, k), dtype=torch.uint8, device=B.device)
    it = np.zeros(k, dtype=np.int32)
    stt = np.zeros(k, dtype=np.int32)
    tr = np.zeros(k, dtype=np.float64)
    br = np.zeros(k, dtype=np.float64)
    bi = np.zeros(k, dtype=np.int32)
    P = N.C.c_void_p
    N.check("hf_pcg_stream", N.lib.hf_pcg_stream(
        N.C.byref(op.Ac.struct), N.ptr(op.d), N.ptr(Bc), k, k, n, kp, float(cfg.tolerance), int(max_iter),
        N.ptr(X), P(it.ctypes.data), P(stt.ctypes.data), P(tr.ctypes.data), P(br.ctypes.data),
        P(bi.ctypes.data), N.ptr(ws), ws.numel(), N.stream_handle()))
    del ws
    failed = np.flatnonzero(stt == N.HF_COL_FAILED)
    for f0 in range(0, failed.size, kp):
        cols = failed[f0:f0 + kp]
        kw = width_for(max(len(cols), 2))
        Bb = torch.zeros((n, kw), dtype=torch.float64, device=B.device)
        idx = torch.from_numpy(cols).to(B.device)
        Bb[:, :len(cols)] = Bc[:, idx]
        freeze = np.zeros(kw, dtype=np.int32)  # other slots stop at x = 0
        freeze[:len(cols)] = bi[cols]
        Xr = _run_batch(op, Bb, cfg.tolerance, max_iter, freeze=freeze)[0]
        X[:, idx] = Xr[:, :len(cols)]
    info.iterations[:] = it
    info.status[:] = stt
    info.true_residual[:] = tr
    info.best_residual[:] = br
    info.best_iteration[:] = bi
    return X, info


def _check_preconditioner(op, any_nonzero):
    if any_nonzero and op.n_zero_rows:
        raise SingularPreconditionerError(f"{op.n_zero_rows} zero row(s) in the operator")


def _raise_failed(info, X, cfg, column_tag):
    failed = np.flatnonzero(info.status == N.HF_COL_FAILED)
    if failed.size == 0:
        return
    j = int(failed[0])  # first failing column in index order (pool.map order)
    best = float(info.best_residual[j])
    exc = ConvergenceError(
        f"PCG did not reach {cfg.tolerance:g} in {info.max_iter} iterations "
        f"(best residual {best:.3e})",
        best_x=X[:, j].cpu().numpy(), residual=best, iterations=info.max_iter)
    exc.local_column = j  # index within this call's block (ordering across ranks)
    if column_tag:
        exc.column = j
    raise exc


def ldp(A):
    """Lumped diagonal preconditioner d_i = sum_j |a_ij| (solver.py:50-61)."""
    shape = A.shape
    if shape[0] != shape[1]:
        raise ParameterError("matrix must be square")
    d, nz = ldp_device(_as_device_csr(A))
    if nz:
        raise SingularPreconditionerError(f"{nz} zero row(s) in the operator")
    return d.cpu().numpy()


def pcg_solve(A, b, cfg=PcgConfig()):
    """(x, iterations, true relative residual) for SPD A (solver.py:64-111)."""
    b = np.asarray(b, dtype=float).ravel()
    n = len(b)
    if np.linalg.norm(b) == 0:
        return np.zeros(n), 0, 0.0
    op = operator(A, cfg)
    _check_preconditioner(op, True)
    Bd = torch.from_numpy(b.reshape(n, 1)).to(device())
    X, info = solve_block(op, Bd, cfg)
    _raise_failed(info, X, cfg, column_tag=False)
    return X[:, 0].cpu().numpy(), int(info.iterations[0]), float(info.true_residual[0])


def rhs_block(B, n_rows=None, dev=None):
    """Dense device block (n x L, float64) from a scipy sparse or dense B."""
    dev = dev or device()
    if sp.issparse(B):
        Bc = sp.coo_matrix(B)
        out = torch.zeros(Bc.shape, dtype=torch.float64, device=dev)
        if Bc.nnz:
            r = torch.from_numpy(Bc.row.astype(np.int64)).to(dev)
            c = torch.from_numpy(Bc.col.astype(np.int64)).to(dev)
            v = torch.from_numpy(Bc.data.astype(np.float64)).to(dev)
            out.index_put_((r, c), v, accumulate=True)
        return out
    return torch.from_numpy(np.ascontiguousarray(B, dtype=np.float64)).to(dev)


def _column_nonzero(B):
    if sp.issparse(B):
        Bc = sp.csc_matrix(B)
        return np.asarray(abs(Bc).sum(axis=0)).ravel() > 0
    return np.any(np.asarray(B) != 0, axis=0)


def transfer_device(A, B, cfg=PcgConfig()):
    """T = A^-1 B kept on the device (n x L torch tensor) plus SolveInfo."""
    op = operator(A, cfg)
    L = B.shape[1]
    nonzero = _column_nonzero(B) if not torch.is_tensor(B) else (B != 0).any(dim=0).cpu().numpy()
    _check_preconditioner(op, bool(np.any(nonzero)))
    Bd = B if torch.is_tensor(B) else rhs_block(B)
    if L == 0:
        return torch.empty((op.n, 0), dtype=torch.float64, device=Bd.device), None
    T, info = solve_block(op, Bd, cfg)
    _raise_failed(info, T, cfg, column_tag=True)
    return T, info


def transfer_matrix(A, B, cfg=PcgConfig(), threads=1):
    """Dense T with column l solving A t = B[:, l] (solver.py:114-141).

    `threads` is accepted for signature compatibility; the result never
    depends on it (every column keeps its own recurrence)."""
    B = B.tocsc() if sp.issparse(B) else np.asarray(B, dtype=float)
    n, L = B.shape
    if L == 0:
        return np.empty((n, 0))
    nonzero = _column_nonzero(B)
    if not np.any(nonzero):
        return np.zeros((n, L))
    T, _ = transfer_device(A, B, cfg)
    return to_host(T.contiguous())


__all__ = ["PcgConfig", "SolveInfo", "ldp", "pcg_solve", "transfer_matrix", "transfer_device",
           "solve_block", "operator", "rhs_block"]
