"""Mesh topology and the source matrix on the device (SURVEY.md §8f "next" rows).

  boundary_triangles_device   TetMesh.boundary_triangles (meshgen.py:114-130)
  assemble_Gt_device          assemble_G (fem.py:391-422) as G' in HBM
  electrodes_from_centers     ElectrodeSet.from_centers (fem.py:157-173)
  ground_node_device          ground_node (fem.py:188-194)

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


def electrodes_from_centers(mesh, centers, radius, impedances):
    """ElectrodeSet.from_centers (fem.py:157-173) with the distance matrix on the
    device: boundary-triangle centroids (hf_triangle_centroids), nearest centre and
    its distance (hf_nearest_center: np.linalg.norm's rounding, np.argmin's
    first-index ties), coverage d <= radius.  Same triangle sets as the reference."""
    from .errors import ElectrodeError
    from .model import ElectrodeSet

    centers = np.atleast_2d(np.asarray(centers, dtype=float))
    dm = DeviceMesh.of(mesh)
    dev = dm.nodes.device
    bfaces, _ = mesh.boundary_triangles()
    nb = len(bfaces)
    tri = torch.from_numpy(np.ascontiguousarray(bfaces, dtype=np.int32)).to(dev)
    cent = torch.empty((max(nb, 1), 3), dtype=torch.float64, device=dev)
    st = N.stream_handle()
    N.check("hf_triangle_centroids", N.lib.hf_triangle_centroids(N.ptr(dm.nodes), N.ptr(tri), nb,
                                                                 N.ptr(cent), st))
    ctr = torch.from_numpy(centers).to(dev)
    owner = torch.empty(max(nb, 1), dtype=torch.int32, device=dev)
    dist = torch.empty(max(nb, 1), dtype=torch.float64, device=dev)
    N.check("hf_nearest_center", N.lib.hf_nearest_center(N.ptr(cent), nb, N.ptr(ctr), len(centers),
                                                         N.ptr(owner), N.ptr(dist), st))
    nearest = owner[:nb].cpu().numpy().astype(np.int64)
    covered = dist[:nb].cpu().numpy() <= radius
    order = np.flatnonzero(covered)
    order = order[np.argsort(nearest[order], kind="stable")]
    bounds = np.searchsorted(nearest[order], np.arange(len(centers) + 1))
    ids = [order[bounds[k]:bounds[k + 1]] for k in range(len(centers))]
    for k, t in enumerate(ids):
        if t.size == 0:
            raise ElectrodeError(f"electrode {k} at {centers[k]} covers no boundary triangle "
                                 f"within radius {radius}")
    return ElectrodeSet(mesh, ids, impedances)


def ground_node_device(mesh, electrodes):
    """ground_node (fem.py:188-194): lowest boundary node not under an electrode."""
    from .errors import AssemblyError
    from .model import electrode_contacts

    dm = DeviceMesh.of(mesh)
    dev = dm.nodes.device
    bfaces, _ = mesh.boundary_triangles()
    bf = torch.from_numpy(np.ascontiguousarray(bfaces, dtype=np.int32)).to(dev)
    etri, _ = electrode_contacts(electrodes)
    et = torch.from_numpy(np.ascontiguousarray(etri, dtype=np.int32)).to(dev) if len(etri) else None
    ws = torch.empty(N.lib.hf_ground_node_workspace_bytes(dm.n), dtype=torch.uint8, device=dev)
    g = N.C.c_int32(-1)
    N.check("hf_ground_node", N.lib.hf_ground_node(N.ptr(bf), len(bfaces), N.ptr(et), len(etri), dm.n,
                                                   N.ptr(ws), N.C.byref(g), N.stream_handle()))
    if g.value < 0:
        raise AssemblyError("electrodes cover every boundary node; cannot choose a grounding node")
    return int(g.value)


__all__ = ["boundary_triangles_device", "assemble_Gt_device", "electrodes_from_centers",
           "ground_node_device"]
