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
    Mb = engine.response_block(T)                       # L x Lb
    width = max(c1 - c0 for c0, c1 in blocks)
    pad = torch.zeros((L, width), dtype=Mb.dtype, device=Mb.device)
    pad[:, :Mb.shape[1]] = Mb
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    Mraw = torch.cat([p[:, :c1 - c0] for p, (c0, c1) in zip(parts, blocks)], dim=1)
    M = symmetrize(Mraw.cpu().numpy())
    W = response_operator(M, engine.R)
    LFp = engine.lf_partial(T, W).contiguous()
    dist.reduce(LFp, dst=0, op=dist.ReduceOp.SUM, group=group)
    return LFp if rank == 0 else None


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

