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

Iterates of a column never depend on which rank or batch solves it, so the
transfer columns are bit-identical to the single-GPU build; only the final
sum over ranks changes the LF at rounding level.

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
    T = engine.solve(A)
    Mraw = _all_gather_columns(engine.response_block(T), blocks, group)  # L x L
    M = symmetrize(Mraw.cpu().numpy())
    W = response_operator(M, engine.R)
    LFp = engine.lf_partial(T, W).contiguous()
    dist.reduce(LFp, dst=0, op=dist.ReduceOp.SUM, group=group)
    return LFp if rank == 0 else None


def _all_gather_columns(X, blocks, group):
    """Concatenate the column blocks every rank holds (padded to equal width for the collective)."""
    width = max(c1 - c0 for c0, c1 in blocks)
    pad = torch.zeros((X.shape[0], width), dtype=X.dtype, device=X.device)
    pad[:, :X.shape[1]] = X
    parts = [torch.empty_like(pad) for _ in blocks]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:, :c1 - c0] for p, (c0, c1) in zip(parts, blocks)], dim=1)


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
    T = engine.solve(A)
    Mraw = _all_gather_columns(engine.response_block(T), column_blocks(L, world), group)
    M = symmetrize(Mraw.cpu().numpy())
    W = response_operator(M, engine.R)
    V = _solve_response(M, I)                                  # L x P
    pblocks = column_blocks(P, world)
    p0, p1 = pblocks[rank]
    if p1 > p0:
        Ub = engine.solve_rhs(A, np.asarray(engine.B @ V[:, p0:p1]))  # n x Pb
    else:  # more ranks than patterns
        Ub = T.new_zeros((T.shape[0], 0))
    U = _all_gather_columns(Ub, pblocks, group)
    cols = engine.eit_partial(dofs, T, U, W).contiguous()      # P*L x n_dofs
    dist.reduce(cols, dst=0, op=dist.ReduceOp.SUM, group=group)
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

