"""Surface segmentations: the input types of mesh generation (geometry.py of
the reference), mirrored for standalone use on the GPU box.

  SurfaceMesh      geometry.py:49-265   closed, oriented triangle surface
  Compartment      geometry.py:317-349  union of sub-surfaces + sigma/priority/active
  Segmentation     geometry.py:352-374  compartments innermost first; locate() on the device
  icosphere        geometry.py:501-535
  box_surface      geometry.py:538-556
  RAY_DIRECTIONS   geometry.py:25-32    the fixed parity-ray directions

The engine reads only `nodes`/`triangles` of each surface and the
compartments' `conductivity`/`priority`, so the reference's own objects work
too; every derived quantity is recomputed with the reference's numpy
expressions (bit-identical inputs to the device kernels).
"""
from __future__ import annotations

import numpy as np

from .errors import FormatError, TopologyError

_rng = np.random.default_rng(20240517)
RAY_DIRECTIONS = np.vstack([np.array([0.32574285, 0.54028471, 0.77595762]), _rng.normal(size=(19, 3))])
RAY_DIRECTIONS /= np.linalg.norm(RAY_DIRECTIONS, axis=1, keepdims=True)
RAY_DIRECTIONS.setflags(write=False)
del _rng

MAX_COMPARTMENTS = 27


def surface_geometry(nodes, triangles):
    """(v0, e1, e2, raw_normals, areas, bbox, diameter) as SurfaceMesh._build_geometry
    computes them (geometry.py:113-138)."""
    p = nodes[triangles]
    e1 = p[:, 1] - p[:, 0]
    e2 = p[:, 2] - p[:, 0]
    cross = np.cross(e1, e2)
    areas = 0.5 * np.linalg.norm(cross, axis=1)
    bbox = np.array([nodes.min(axis=0), nodes.max(axis=0)])
    diameter = float(np.linalg.norm(bbox[1] - bbox[0]))
    return np.ascontiguousarray(p[:, 0]), np.ascontiguousarray(e1), np.ascontiguousarray(e2), \
        cross, areas, bbox, diameter


class SurfaceMesh:
    """Closed, consistently oriented triangle surface (geometry.py:49-265)."""

    def __init__(self, nodes, triangles, name="surface"):
        nodes = np.ascontiguousarray(nodes, dtype=float)
        triangles = np.ascontiguousarray(triangles, dtype=np.int64)
        if nodes.ndim != 2 or nodes.shape[1] != 3:
            raise FormatError(f"nodes must be (n, 3), got {nodes.shape}")
        if triangles.ndim != 2 or triangles.shape[1] != 3:
            raise FormatError(f"triangles must be (m, 3), got {triangles.shape}")
        if not np.all(np.isfinite(nodes)):
            raise FormatError("non-finite node coordinate")
        if triangles.size and (triangles.min() < 0 or triangles.max() >= len(nodes)):
            bad = triangles[(triangles < 0) | (triangles >= len(nodes))][0]
            raise IndexError(f"triangle references node {bad} outside 0..{len(nodes) - 1}")
        self.nodes, self.triangles, self.name = nodes, triangles, str(name)
        self.nodes.setflags(write=False)
        self.triangles.setflags(write=False)
        self._validate_topology()
        v0, e1, e2, cross, areas, bbox, diameter = surface_geometry(nodes, triangles)
        scale = float(np.max(np.ptp(nodes, axis=0))) or 1.0
        if np.any(areas <= 1e-16 * scale * scale):
            raise FormatError(f"surface '{self.name}' has "
                              f"{np.count_nonzero(areas <= 1e-16 * scale * scale)} degenerate triangle(s)")
        signed_vol = np.einsum("ij,ij->", v0, cross) / 6.0
        self._orient = 1.0 if signed_vol >= 0 else -1.0
        self.areas = areas
        self.normals = self._orient * cross / (2.0 * areas[:, None])
        self.bbox = bbox
        self.enclosed_volume = abs(signed_vol)

    def _validate_topology(self):
        tri = self.triangles
        if len(tri) < 4:
            raise TopologyError("a closed surface needs at least 4 triangles")
        edges = np.concatenate([tri[:, [0, 1]], tri[:, [1, 2]], tri[:, [2, 0]]])
        if np.any(edges[:, 0] == edges[:, 1]):
            raise TopologyError("triangle with a repeated vertex")
        _, counts = np.unique(np.sort(edges, axis=1), axis=0, return_counts=True)
        if np.any(counts != 2):
            raise TopologyError(f"surface '{self.name}' is not closed: "
                                f"{np.count_nonzero(counts != 2)} edge(s) not shared by exactly 2 triangles")
        _, dcounts = np.unique(edges, axis=0, return_counts=True)
        if np.any(dcounts != 1):
            raise TopologyError(f"surface '{self.name}' is not consistently oriented")

    def contains(self, points):
        """Inside-or-on-surface test on the device (geometry.py:147-166)."""
        from .meshgen import locate_surfaces

        pts = np.atleast_2d(np.asarray(points, dtype=float))
        out = locate_surfaces([[self]], pts) >= 0
        return bool(out[0]) if np.asarray(points).ndim == 1 else out

    def __repr__(self):
        return f"SurfaceMesh('{self.name}', {len(self.nodes)} nodes, {len(self.triangles)} triangles)"


class Compartment:
    """One tissue compartment (geometry.py:317-349)."""

    def __init__(self, surfaces, conductivity, priority=0, active=False, name=None):
        if isinstance(surfaces, SurfaceMesh):
            surfaces = (surfaces,)
        surfaces = tuple(surfaces)
        if not surfaces:
            raise FormatError("compartment needs at least one surface")
        cond = np.asarray(conductivity, dtype=float)
        if cond.ndim == 0:
            cond = float(cond)
        elif cond.shape != (6,):
            raise FormatError("conductivity must be a scalar or a 6-entry tensor row "
                              "(s11, s22, s33, s12, s13, s23)")
        self.surfaces, self.conductivity = surfaces, cond
        self.priority, self.active = int(priority), bool(active)
        self.name = name if name is not None else surfaces[0].name

    @property
    def is_tensor(self):
        return not np.isscalar(self.conductivity)

    def contains(self, points):
        from .meshgen import locate_surfaces

        pts = np.atleast_2d(np.asarray(points, dtype=float))
        out = locate_surfaces([self.surfaces], pts) >= 0
        return bool(out[0]) if np.asarray(points).ndim == 1 else out


class Segmentation:
    """Ordered multi-compartment segmentation, innermost first (geometry.py:352-374)."""

    def __init__(self, compartments):
        compartments = tuple(compartments)
        if not compartments:
            raise FormatError("segmentation needs at least one compartment")
        if len(compartments) > MAX_COMPARTMENTS:
            raise FormatError(f"at most {MAX_COMPARTMENTS} compartments supported, "
                              f"got {len(compartments)}")
        self.compartments = compartments

    def __len__(self):
        return len(self.compartments)

    def __getitem__(self, i):
        return self.compartments[i]

    @property
    def has_tensor(self):
        return any(c.is_tensor for c in self.compartments)

    def bounding_box(self):
        los = [np.asarray(s.nodes).min(axis=0) for c in self.compartments for s in c.surfaces]
        his = [np.asarray(s.nodes).max(axis=0) for c in self.compartments for s in c.surfaces]
        return np.min(los, axis=0), np.max(his, axis=0)

    def locate(self, points):
        """Innermost enclosing compartment per point, -1 outside (device, hf_locate)."""
        from .meshgen import locate

        return locate(self, points)


def icosphere(radius=1.0, subdivisions=2, center=(0.0, 0.0, 0.0), name="sphere"):
    """Subdivided icosahedron, outward oriented (geometry.py:501-535): the same
    vertex and face order as the reference (midpoints created ab, bc, ca per face)."""
    phi = (1.0 + np.sqrt(5.0)) / 2.0
    verts = np.array([[-1, phi, 0], [1, phi, 0], [-1, -phi, 0], [1, -phi, 0],
                      [0, -1, phi], [0, 1, phi], [0, -1, -phi], [0, 1, -phi],
                      [phi, 0, -1], [phi, 0, 1], [-phi, 0, -1], [-phi, 0, 1]], dtype=float)
    faces = np.array([[0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11],
                      [1, 5, 9], [5, 11, 4], [11, 10, 2], [10, 7, 6], [7, 1, 8],
                      [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9],
                      [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]], dtype=np.int64)
    verts /= np.linalg.norm(verts, axis=1, keepdims=True)
    for _ in range(int(subdivisions)):
        index, vlist, out = {}, list(verts), []

        def mid(i, j):
            key = (i, j) if i < j else (j, i)
            if key not in index:
                m = vlist[i] + vlist[j]
                m /= np.linalg.norm(m)
                index[key] = len(vlist)
                vlist.append(m)
            return index[key]

        for a, b, c in faces:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            out += [[a, ab, ca], [b, bc, ab], [c, ca, bc], [ab, bc, ca]]
        verts, faces = np.array(vlist), np.array(out, dtype=np.int64)
    return SurfaceMesh(verts * float(radius) + np.asarray(center, dtype=float), faces, name=name)


def box_surface(lo=(0.0, 0.0, 0.0), hi=(1.0, 1.0, 1.0), name="box"):
    """Axis-aligned box, 12 outward triangles (geometry.py:538-556)."""
    (x0, y0, z0), (x1, y1, z1) = np.asarray(lo, dtype=float), np.asarray(hi, dtype=float)
    nodes = np.array([[x0, y0, z0], [x1, y0, z0], [x1, y1, z0], [x0, y1, z0],
                      [x0, y0, z1], [x1, y0, z1], [x1, y1, z1], [x0, y1, z1]])
    faces = np.array([[0, 2, 1], [0, 3, 2], [4, 5, 6], [4, 6, 7], [0, 1, 5], [0, 5, 4],
                      [2, 3, 7], [2, 7, 6], [0, 4, 7], [0, 7, 3], [1, 2, 6], [1, 6, 5]],
                     dtype=np.int64)
    return SurfaceMesh(nodes, faces, name=name)


def layered_sphere_segmentation(radii, conductivities, priorities=None, active_shells=(0,),
                                subdivisions=3):
    """Concentric icosphere head model, innermost first (experiments.py:46-57)."""
    return Segmentation([
        Compartment(icosphere(r, subdivisions, name=f"shell{k}"), conductivity=s,
                    priority=priorities[k] if priorities is not None else 0,
                    active=k in active_shells, name=f"shell{k}")
        for k, (r, s) in enumerate(zip(radii, conductivities))])


__all__ = ["SurfaceMesh", "Compartment", "Segmentation", "icosphere", "box_surface",
           "layered_sphere_segmentation", "RAY_DIRECTIONS", "surface_geometry"]
