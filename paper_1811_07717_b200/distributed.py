"""Electrode-column sharding of the EEG lead-field build over ranks.

One process per GPU.  Rank r owns the contiguous electrode block
`column_blocks(L, world)[r]`, holds a replica of the mesh and assembles its
own copy of A (assembly is cheap and deterministic, so every rank builds the
identical matrix without moving it), and solves only its columns.  The two
exchanges are small:

  1. all-gather of the raw response blocks (C - B'T)[:, block]  (L x L total)
     -> every rank forms M = (M + M')/2 and W = -R M^-1 on the host;
  2. sum-reduce to rank 0 of the partial lead fields W[:, block] (G'T_block)'
     (L x 3S), computed by hf_lf_tail on each rank.

`sharded_eit_leadfield` adds the EIT pattern solves, sharded by pattern, and
one all-gather of U (n x P); see its docstring.

A column's iterates never depend on which rank or batch solves it (the
solver's reductions are canonical, pcg.cu), so the transfer columns are
bit-identical to the single-GPU build; only the final sum over ranks changes
the LF at rounding level.  A convergence failure on any rank is raised on
every rank, before the next collective, as the same ConvergenceError.

`sharded_leadfield` only uses the engine's stage methods and torch.distributed
collectives, so the same orchestration runs with NCCL on GPUs and with gloo on
CPU tensors (tests/test_distributed.py).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .engine import column_blocks
from .leadfield import response_operator, symmetrize


def sharded_leadfield(engine, world=None, rank=None, group=None):
    """Run the sharded build; returns the full LF (torch, L x ncols) on rank 0, None elsewhere."""
    world = dist.get_world_size(group) if world is None else world
    rank = dist.get_rank(group) if rank is None else rank
    L = engine.L
    blocks = column_blocks(L, world)
    A = engine.assemble()
    T = _solve_consistently(lambda: engine.solve(A), engine.c0, L, blocks, group, tag=True)
    Mraw = _all_gather_columns(engine.response_block(T), blocks, group)  # L x L
    M = symmetrize(Mraw.cpu().numpy())
    W = response_operator(M, engine.R)
    LFp = engine.lf_partial(T, W).contiguous()
    _reduce_sum(LFp, group)
    return LFp if rank == 0 else None


def _host_collectives(group):
    """gloo moves CPU tensors only: stage device tensors through the host for it."""
    return dist.get_backend(group) == "gloo"


def _reduce_sum(X, group):
    if _host_collectives(group) and X.is_cuda:
        h = X.cpu()
        dist.reduce(h, dst=0, op=dist.ReduceOp.SUM, group=group)
        X.copy_(h)
    else:
        dist.reduce(X, dst=0, op=dist.ReduceOp.SUM, group=group)


def _all_gather_columns(X, blocks, group):
    """Concatenate the column blocks every rank holds (padded to equal width for the collective)."""
    width = max(c1 - c0 for c0, c1 in blocks)
    dev = "cpu" if _host_collectives(group) else X.device
    pad = torch.zeros((X.shape[0], width), dtype=X.dtype, device=dev)
    pad[:, :X.shape[1]] = X.to(dev)
    parts = [torch.empty_like(pad) for _ in blocks]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:, :c1 - c0] for p, (c0, c1) in zip(parts, blocks)], dim=1).to(X.device)


def _solve_consistently(solve, c0, n_cols, blocks, group, tag):
    """Run this rank's solve; if any rank's columns fail, every rank raises before the
    next collective, so no rank is left waiting in it.  Convergence failures become
    the same ConvergenceError on every rank (the reference's transfer_matrix reports
    the first failing column in index order, solver.py:129-136): the lowest failing
    global column wins and its owner broadcasts best_x, residual and iterations.
    Any other exception is re-raised where it happened and reported as a
    RuntimeError on the other ranks."""
    from .errors import ConvergenceError

    err, other, X = None, None, None
    try:
        X = solve()
    except ConvergenceError as exc:
        err = exc
    except Exception as exc:  # noqa: BLE001 - re-raised below, after the agreement
        other = exc
    mine = n_cols if err is None else c0 + int(getattr(err, "local_column", 0))
    flag = torch.tensor([mine, 1 if other is not None else 0], dtype=torch.int64)
    if not _host_collectives(group):
        flag = flag.cuda()
    first_t = flag[:1].clone()
    any_other = flag[1:].clone()
    dist.all_reduce(first_t, op=dist.ReduceOp.MIN, group=group)
    dist.all_reduce(any_other, op=dist.ReduceOp.MAX, group=group)
    if int(any_other.item()):
        if other is not None:
            raise other
        raise RuntimeError("the sharded solve failed on another rank")
    first = int(first_t.item())
    if first >= n_cols:
        return X
    owner = next(r for r, (b0, b1) in enumerate(blocks) if b0 <= first < b1)
    meta = torch.zeros(3, dtype=torch.float64)
    if err is not None and mine == first:
        meta[:] = torch.tensor([float(len(err.best_x)), float(err.residual), float(err.iterations)])
    if not _host_collectives(group):
        meta = meta.cuda()
    dist.broadcast(meta, src=_global_rank(owner, group), group=group)
    n, residual, iters = int(meta[0].item()), float(meta[1].item()), int(meta[2].item())
    best = torch.zeros(n, dtype=torch.float64)
    if err is not None and mine == first:
        best = torch.from_numpy(err.best_x.copy())
    if not _host_collectives(group):
        best = best.cuda()
    dist.broadcast(best, src=_global_rank(owner, group), group=group)
    out = ConvergenceError(f"PCG did not converge in {iters} iterations (best residual {residual:.3e})",
                           best_x=best.cpu().numpy(), residual=residual, iterations=iters)
    if tag:
        out.column = first
    raise out


def _global_rank(r, group):
    return r if group is None else dist.get_global_rank(group, r)


def sharded_eit_leadfield(engine, dofs, currents, world=None, rank=None, group=None):
    """EIT lead field (leadfield.py:210-237) over ranks (EIT bullet).

    Electrodes stay sharded as in the EEG build: rank r solves T[:, block_r].
    Then
      1. all-gather of the raw M blocks -> M, W = -R M^-1 and V = M^-1 I (host);
      2. the P pattern solves u_p = A^-1 B V[:, p] are sharded by pattern, and
         all-gathered (n x P) — the only n-sized exchange;
      3. every rank forms its electrode block's Q and W[:, block] Q[p]' and the
         partial Jacobians are sum-reduced to rank 0.
    Returns the LeadField on rank 0, None elsewhere."""
    import numpy as np

    from .leadfield import LeadField, _solve_response, check_current_patterns

    world = dist.get_world_size(group) if world is None else world
    rank = dist.get_rank(group) if rank is None else rank
    L = engine.L
    I = check_current_patterns(currents, L)
    P = I.shape[1]
    A = engine.assemble()
    T = _solve_consistently(lambda: engine.solve(A), engine.c0, L, column_blocks(L, world), group,
                            tag=True)
    Mraw = _all_gather_columns(engine.response_block(T), column_blocks(L, world), group)
    M = symmetrize(Mraw.cpu().numpy())
    W = response_operator(M, engine.R)
    V = _solve_response(M, I)                                  # L x P
    pblocks = column_blocks(P, world)
    p0, p1 = pblocks[rank]
    def solve_u():
        if p1 > p0:
            return engine.solve_rhs(A, np.asarray(engine.B @ V[:, p0:p1]))  # n x Pb
        return T.new_zeros((T.shape[0], 0))  # more ranks than patterns
    # pattern solves follow pcg_solve's semantics (leadfield.py:227): no column tag
    Ub = _solve_consistently(solve_u, p0, P, pblocks, group, tag=False)
    U = _all_gather_columns(Ub, pblocks, group)
    cols = engine.eit_partial(dofs, T, U, W).contiguous()      # P*L x n_dofs
    _reduce_sum(cols, group)
    if rank != 0:
        return None
    return LeadField(matrix=cols.cpu().numpy(), positions=dofs.centers, orientations=None,
                     modality="eit", n_patterns=P,
                     background_sigma=np.array(engine.mesh.sigma, copy=True),
                     background_data=(engine.R @ V).T.ravel())


def init_from_env(backend="nccl"):
    """torchrun-style init (RANK, WORLD_SIZE, LOCAL_RANK, MASTER_ADDR/PORT)."""
    import os

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    elif backend == "nccl" and torch.cuda.is_available():
        torch.cuda.set_device(local)
    return rank, world, local

