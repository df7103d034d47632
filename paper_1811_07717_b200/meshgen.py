"""Labelled tetrahedral mesh generation on the B200 (SURVEY.md §8f "next" row #4).

  locate          Segmentation.locate (geometry.py:359-374)   -> hf_locate
  generate_mesh   generate_mesh (meshgen.py:186-244)           -> hf_grid_tets, hf_locate,
                  _apply_priorities (meshgen.py:247-269)          hf_mesh_compact,
                                                                  hf_apply_priorities

The host does only O(surface) work: the per-(direction, triangle) constants
of SurfaceMesh._cast (geometry.py:203-224), computed with the reference's own
numpy expressions, and the grid coordinates lo + h * arange(...).  Every
per-point and per-element step runs in libhfb200.  The result is the
reference's mesh: the same nodes, element order, labels and sigma
(tests/test_gpu_meshgen.py compares them array for array).
"""
from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .device import device
from .errors import EmptyMeshError, ParameterError
from .geometry import RAY_DIRECTIONS, surface_geometry
from .model import TetMesh

RAYW = 16


class DeviceSegmentation:
    """hf_segmentation tables in HBM for a list of compartments (each a list of surfaces)."""

    def __init__(self, compartments, dev=None):
        dev = dev or device()
        comp_surf, tri_off, boxes, blocks = [0], [0], [], []
        dirs = RAY_DIRECTIONS
        for surfs in compartments:
            for s in surfs:
                nodes = np.ascontiguousarray(s.nodes, dtype=float)
                tri = np.ascontiguousarray(s.triangles, dtype=np.int64)
                v0, e1, e2, n, areas, bbox, diameter = surface_geometry(nodes, tri)
                tol = 1e-9 * (diameter or 1.0)                     # geometry.py:159
                boxes.append([*bbox[0], *bbox[1], tol, 0.0])
                nrm_tol = tol * (2.0 * areas)                      # geometry.py:222,242
                scale2 = np.linalg.norm(e1, axis=1) * np.linalg.norm(e2, axis=1)
                c_n = np.einsum("ij,ij->i", v0, n)
                for d in dirs:                                     # geometry.py:211-224
                    h = np.cross(d, e2)
                    k = np.cross(e1, d)
                    a = np.einsum("ij,ij->i", e1, h)
                    parallel = np.abs(a) <= 1e-12 * scale2
                    f = np.where(parallel, 1.0, 1.0 / np.where(parallel, 1.0, a))
                    row = np.zeros((len(tri), RAYW))
                    row[:, 0:3], row[:, 3:6], row[:, 6:9] = h, k, n
                    row[:, 9] = np.einsum("ij,ij->i", v0, h)
                    row[:, 10] = np.einsum("ij,ij->i", v0, k)
                    row[:, 11] = c_n
                    row[:, 12] = f
                    row[:, 13] = parallel
                    row[:, 14] = nrm_tol
                    blocks.append(row)
                tri_off.append(tri_off[-1] + len(tri))
            comp_surf.append(len(tri_off) - 1)
        self.n_comp, self.n_surf, self.n_dir = len(compartments), len(tri_off) - 1, len(dirs)
        t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(dev)  # noqa: E731
        self.comp_surf = t(comp_surf, np.int32)
        self.tri_off = t(tri_off, np.int32)
        self.box = t(np.array(boxes).reshape(-1, 8) if boxes else np.zeros((0, 8)), np.float64)
        self.rays = t(np.concatenate(blocks) if blocks else np.zeros((0, RAYW)), np.float64)
        self.struct = N.HfSegmentation(self.n_comp, self.n_surf, self.n_dir, N.ptr(self.comp_surf),
                                       N.ptr(self.tri_off), N.ptr(self.box), N.ptr(self.rays))

    @classmethod
    def of(cls, seg):
        ds = getattr(seg, "_hfb200_device", None)
        if ds is None or ds.rays.device != device():
            ds = cls([c.surfaces for c in seg.compartments])
            try:
                object.__setattr__(seg, "_hfb200_device", ds)
            except (AttributeError, TypeError):
                pass
        return ds

    def locate(self, pts_dev, labels=None):
        n = pts_dev.shape[0]
        if labels is None:
            labels = torch.empty(n, dtype=torch.int32, device=pts_dev.device)
        N.check("hf_locate", N.lib.hf_locate(N.C.byref(self.struct), N.ptr(pts_dev), n,
                                             N.ptr(labels), N.stream_handle()))
        return labels


def locate_surfaces(compartments, points):
    """Labels of `points` against compartments given as lists of surfaces."""
    ds = DeviceSegmentation(compartments)
    pts = torch.from_numpy(np.array(points, dtype=np.float64, order="C").reshape(-1, 3)).to(ds.rays.device)
    return ds.locate(pts).cpu().numpy().astype(np.int64)


def locate(seg, points):
    """Segmentation.locate (geometry.py:359-374): int64 labels, -1 outside."""
    pts = np.atleast_2d(np.asarray(points, dtype=float))
    ds = DeviceSegmentation.of(seg)
    p = torch.from_numpy(np.array(pts, dtype=np.float64, order="C")).to(ds.rays.device)
    return ds.locate(p).cpu().numpy().astype(np.int64)


def conductivity_table(seg):
    """Per-compartment sigma rows (meshgen.py:172-183)."""
    if any(not np.isscalar(c.conductivity) for c in seg.compartments):
        table = np.zeros((len(seg.compartments), 6))
        for k, comp in enumerate(seg.compartments):
            if np.isscalar(comp.conductivity):
                table[k, :3] = comp.conductivity
            else:
                table[k] = comp.conductivity
        return table
    return np.array([c.conductivity for c in seg.compartments])


class DeviceGrid:
    """generate_mesh's output while still in HBM (tetra int32, labels int32)."""

    def __init__(self, nodes, tetra, labels, sigma_table):
        self.nodes, self.tetra, self.labels, self.sigma_table = nodes, tetra, labels, sigma_table

    def to_mesh(self, mesh_cls=TetMesh):
        lab = self.labels.cpu().numpy().astype(np.int64)
        return mesh_cls(self.nodes.cpu().numpy(), self.tetra.cpu().numpy().astype(np.int64), lab,
                        self.sigma_table[lab])


def generate_mesh_device(seg, h):
    """generate_mesh (meshgen.py:186-244) with every per-element step on the device."""
    if not np.isfinite(h) or h <= 0:
        raise ParameterError(f"resolution must be positive, got {h}")
    lo, hi = seg.bounding_box()
    extent = hi - lo
    if not np.all(np.isfinite(extent)) or np.any(extent <= 0):
        raise ParameterError("segmentation bounding box is degenerate")
    nx, ny, nz = (int(v) for v in np.maximum(1, np.ceil(extent / h - 1e-12).astype(int)))
    ds = DeviceSegmentation.of(seg)
    dev = ds.rays.device
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)  # noqa: E731
    xs, ys, zs = (t(lo[a] + h * np.arange(c + 1)) for a, c in enumerate((nx, ny, nz)))
    m_all = 6 * nx * ny * nz
    if m_all >= 2 ** 31 or (nx + 1) * (ny + 1) * (nz + 1) >= 2 ** 31:
        raise ParameterError(f"grid {nx}x{ny}x{nz} exceeds the int32 element/node range")
    st = N.stream_handle()
    tet_all = torch.empty((m_all, 4), dtype=torch.int32, device=dev)
    cent = torch.empty((m_all, 3), dtype=torch.float64, device=dev)
    N.check("hf_grid_tets", N.lib.hf_grid_tets(N.ptr(xs), N.ptr(ys), N.ptr(zs), nx, ny, nz,
                                               N.ptr(tet_all), N.ptr(cent), st))
    cl = ds.locate(cent)
    del cent
    ng = (nx + 1) * (ny + 1) * (nz + 1)
    ws = torch.empty(N.lib.hf_mesh_compact_workspace_bytes(m_all, ng), dtype=torch.uint8, device=dev)
    tet = torch.empty((m_all, 4), dtype=torch.int32, device=dev)
    lab = torch.empty(m_all, dtype=torch.int32, device=dev)
    nodes = torch.empty((ng, 3), dtype=torch.float64, device=dev)
    mo, no = N.C.c_int64(0), N.C.c_int64(0)
    N.check("hf_mesh_compact", N.lib.hf_mesh_compact(
        N.ptr(tet_all), N.ptr(cl), m_all, N.ptr(xs), N.ptr(ys), N.ptr(zs), nx, ny, nz, N.ptr(tet),
        N.ptr(lab), N.ptr(nodes), N.C.byref(mo), N.C.byref(no), N.ptr(ws), ws.numel(), st))
    del tet_all, cl, ws
    m, n = int(mo.value), int(no.value)
    if m == 0:
        raise EmptyMeshError(f"no element centroid inside any compartment at h={h}")
    tet, lab, nodes = tet[:m], lab[:m], nodes[:n]
    node_label = ds.locate(nodes)
    pri = torch.tensor([int(c.priority) for c in seg.compartments], dtype=torch.int32, device=dev)
    N.check("hf_apply_priorities", N.lib.hf_apply_priorities(N.ptr(tet), m, N.ptr(node_label),
                                                             N.ptr(pri), N.ptr(lab), st))
    return DeviceGrid(nodes, tet, lab, conductivity_table(seg))


def generate_mesh(seg, h):
    """Drop-in for headfem.meshgen.generate_mesh: returns a TetMesh."""
    return generate_mesh_device(seg, h).to_mesh()


__all__ = ["DeviceSegmentation", "locate", "locate_surfaces", "generate_mesh",
           "generate_mesh_device", "conductivity_table", "DeviceGrid"]
