"""Synthetic benchmark inputs (BASELINE.json configs) built without the reference.

`sphere_mesh` is the analytic-label Kuhn grid of SURVEY.md Appendix A.4: the
grid, node numbering (x fastest), cube order and the Kuhn 6-tetrahedron table
of generate_mesh (meshgen.py:23-42, 209-244), with elements labelled by the
radius of their centroid instead of icosphere ray casting.  It is a valid
TetMesh input for both the reference and this engine.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass

import numpy as np

from . import model


def kuhn_table():
    """6 tetrahedra per cube as corner ids (bit k = axis k offset), positive volume."""
    tets = []
    for perm in itertools.permutations((0, 1, 2)):
        ids, acc = [0], 0
        for axis in perm:
            acc |= 1 << axis
            ids.append(acc)
        if sum(a > b for a, b in itertools.combinations(perm, 2)) % 2 == 1:
            ids[2], ids[3] = ids[3], ids[2]
        tets.append(ids)
    return np.array(tets, dtype=np.int64)


KUHN = kuhn_table()
CORNERS = np.array([[(j >> a) & 1 for a in range(3)] for j in range(8)], dtype=np.int64)

# BASELINE.json configs
C1_RADII, C1_COND = (0.079, 0.086, 0.092), (0.33, 0.0064, 0.43)
C2_RADII, C2_COND = (0.079, 0.082, 0.087, 0.092), (0.33, 1.79, 0.0064, 0.43)


def sphere_mesh(radii, conductivities, h):
    """Concentric-sphere Kuhn mesh; label k = innermost shell containing the centroid."""
    R = radii[-1]
    lo = np.full(3, -R)
    nx = int(np.ceil(2 * R / h - 1e-12))
    xs = lo[0] + h * np.arange(nx + 1)
    gz, gy, gx = np.meshgrid(xs, xs, xs, indexing="ij")
    grid = np.column_stack([gx.ravel(), gy.ravel(), gz.ravel()])
    cz, cy, cx = np.meshgrid(*(np.arange(nx),) * 3, indexing="ij")
    base = (cx + (nx + 1) * (cy + (nx + 1) * cz)).ravel()
    off = CORNERS[:, 0] + (nx + 1) * (CORNERS[:, 1] + (nx + 1) * CORNERS[:, 2])
    # cube-centre radius prefilter (a tet centroid lies within h*sqrt(3)/2 of its cube centre)
    cc = grid[base] + 0.5 * h
    near = np.linalg.norm(cc, axis=1) <= R + h
    base = base[near]
    tetra = (base[:, None] + off[None, :])[:, KUHN].reshape(-1, 4)
    r = np.linalg.norm(grid[tetra].mean(axis=1), axis=1)
    lab = np.full(len(r), -1, dtype=np.int64)
    for k in reversed(range(len(radii))):
        lab[r <= radii[k]] = k
    keep = lab >= 0
    used, tet = np.unique(tetra[keep], return_inverse=True)
    cond = np.asarray(conductivities, dtype=float)
    return model.TetMesh(grid[used], tet.reshape(-1, 4), lab[keep], cond[lab[keep]])


def fibonacci_sphere_points(n, radius=1.0, center=(0.0, 0.0, 0.0)):
    """Golden-angle spiral electrode sites (simulate.py:196-204)."""
    i = np.arange(n) + 0.5
    phi = np.arccos(1.0 - 2.0 * i / n)
    theta = np.pi * (1.0 + 5.0 ** 0.5) * i
    pts = np.column_stack([np.sin(phi) * np.cos(theta), np.sin(phi) * np.sin(theta), np.cos(phi)])
    return radius * pts + np.asarray(center, dtype=float)


@dataclass
class EegProblem:
    mesh: model.TetMesh
    electrodes: model.ElectrodeSet
    sources: model.SourceSpace
    G: object
    B: object
    C: object
    R: np.ndarray
    ground: int
    name: str


def eeg_problem(name="c2", n_electrodes=None, n_sources=None, h=None, seed=1, device=False,
                with_G=True):
    """C1 / C2 / C5 EEG problem: mesh, electrodes, unconstrained sources, G, B, C, R.

    device=True builds the boundary faces and the source matrix with the CUDA
    kernels (G is then G' in HBM, a DeviceCsr); otherwise on the host."""
    if name == "c1":
        radii, cond = C1_RADII, C1_COND
        h = h or 0.004
        L, S, rad = n_electrodes or 32, n_sources or 1000, 0.014
    elif name == "c2":
        radii, cond = C2_RADII, C2_COND
        h = h or 0.0015
        L, S, rad = n_electrodes or 128, n_sources or 10_000, 0.01
    elif name == "c5":
        radii, cond = C2_RADII, C2_COND
        h = h or 0.00088
        L, S, rad = n_electrodes or 256, n_sources or 50_000, 0.006
    else:
        raise ValueError(name)
    mesh = sphere_mesh(radii, cond, h)
    if device:  # boundary faces and G' from the device kernels (topology.py)
        from .topology import assemble_Gt_device, boundary_triangles_device, electrodes_from_centers

        mesh._boundary = boundary_triangles_device(mesh)
    centers = fibonacci_sphere_points(L, radii[-1])
    if device:  # nearest-centre coverage on the device (topology.electrodes_from_centers)
        el = electrodes_from_centers(mesh, centers, radius=rad, impedances=1e3)
    else:
        el = model.ElectrodeSet.from_centers(mesh, centers, radius=rad, impedances=1e3)
    src = model.place_sources(mesh, [0], S, seed=seed)
    G = None
    if with_G:
        G = assemble_Gt_device(mesh, src) if device else model.assemble_G(mesh, src)
    B, C, R = model.assemble_B_C_R(mesh, el)
    if device:
        from .topology import ground_node_device

        g = ground_node_device(mesh, el)
    else:
        g = model.ground_node(mesh, el)
    return EegProblem(mesh, el, src, G, B, C, R, g, name)
