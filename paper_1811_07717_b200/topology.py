"""Mesh topology and the source matrix on the device (SURVEY.md §8f "next" rows).

  boundary_triangles_device   TetMesh.boundary_triangles (meshgen.py:114-130)
  assemble_Gt_device          assemble_G (fem.py:391-422) as G' in HBM

Both run through libhfb200 (hf_boundary_faces, hf_whitney_gt) on node ->
element incidence lists, replacing the reference's sort/unique over every
element face (51 s for boundary_triangles and 65 s for assemble_G at C2).
"""
from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .device import DeviceCsr
from .errors import LocationError
from .fem import DeviceMesh

_FACES = np.array([[1, 2, 3], [0, 3, 2], [0, 1, 3], [0, 2, 1]])


def boundary_triangles_device(mesh):
    """(faces (b,3) int64, owners (b,)) — outward boundary faces in element-face order."""
    dm = DeviceMesh.of(mesh)
    dev = dm.nodes.device
    ws = torch.empty(N.lib.hf_topology_workspace_bytes(dm.n, dm.m, 0), dtype=torch.uint8, device=dev)
    idx = torch.empty(max(4 * dm.m, 1), dtype=torch.int32, device=dev)
    nb = N.C.c_int64(0)
    N.check("hf_boundary_faces", N.lib.hf_boundary_faces(
        N.ptr(dm.tetra), dm.n, dm.m, N.ptr(idx), N.C.byref(nb), N.ptr(ws), ws.numel(),
        N.stream_handle()))
    f = idx[: int(nb.value)].cpu().numpy().astype(np.int64)
    owners = f // 4
    faces = np.asarray(mesh.tetra)[owners[:, None], _FACES[f % 4]]
    return faces, owners


def assemble_Gt_device(mesh, sources):
    """G' (ncomp*S x n) CSR in HBM; row c is source column c of assemble_G."""
    dm = DeviceMesh.of(mesh)
    dev = dm.nodes.device
    el = np.asarray(sources.element_ids, dtype=np.int64)
    if el.size and (el.min() < 0 or el.max() >= dm.m):
        raise LocationError("source element index outside the mesh")
    S = len(el)
    constrained = getattr(sources, "mode", "unconstrained") == "constrained"
    ncols = S if constrained else 3 * S
    src = torch.from_numpy(el.astype(np.int32)).to(dev)
    orient = None
    if constrained:
        orient = torch.from_numpy(np.ascontiguousarray(sources.orientations, dtype=np.float64)).to(dev)
    ws = torch.empty(N.lib.hf_topology_workspace_bytes(dm.n, dm.m, ncols), dtype=torch.uint8,
                     device=dev)
    gptr = torch.empty(ncols + 1, dtype=torch.int32, device=dev)
    nnz = N.C.c_int64(0)
    st = N.stream_handle()
    args = (N.ptr(dm.nodes), N.ptr(dm.tetra), dm.n, dm.m, N.ptr(src), S, N.ptr(orient), N.ptr(gptr))
    N.check("hf_whitney_gt", N.lib.hf_whitney_gt(*args, None, None, N.C.byref(nnz), N.ptr(ws),
                                                 ws.numel(), st))
    k = int(nnz.value)
    gidx = torch.empty(max(k, 1), dtype=torch.int32, device=dev)[:k]
    gval = torch.empty(max(k, 1), dtype=torch.float64, device=dev)[:k]
    N.check("hf_whitney_gt", N.lib.hf_whitney_gt(*args, N.ptr(gidx), N.ptr(gval), N.C.byref(nnz),
                                                 N.ptr(ws), ws.numel(), st))
    return DeviceCsr(gptr, gidx, gval, (ncols, dm.n))


__all__ = ["boundary_triangles_device", "assemble_Gt_device"]
