"""Oracle restatement of mesh generation (test infrastructure only).

point location   SurfaceMesh.contains / _contains_impl / _cast   geometry.py:147-249
                 Compartment.contains, Segmentation.locate          geometry.py:332-374
generate_mesh    meshgen.py:186-244, _apply_priorities meshgen.py:247-269

A segmentation is given as a list of compartments, each a tuple
(surfaces, conductivity, priority) with surfaces a list of (nodes, triangles).
Pinned to tests/golden/meshgen_cases.npz (made by the reference itself).
"""
from __future__ import annotations

import numpy as np

_rng = np.random.default_rng(20240517)  # geometry.py:25-32
RAY_DIRECTIONS = np.vstack([np.array([0.32574285, 0.54028471, 0.77595762]), _rng.normal(size=(19, 3))])
RAY_DIRECTIONS /= np.linalg.norm(RAY_DIRECTIONS, axis=1, keepdims=True)

EB = 1e-10  # barycentric margin, geometry.py:226


def _geometry(nodes, tris):
    p = nodes[tris]
    e1, e2 = p[:, 1] - p[:, 0], p[:, 2] - p[:, 0]
    n = np.cross(e1, e2)
    areas = 0.5 * np.linalg.norm(n, axis=1)
    lo, hi = nodes.min(axis=0), nodes.max(axis=0)
    return p[:, 0], e1, e2, n, areas, lo, hi, float(np.linalg.norm(hi - lo))


def _cast(g, pts, d, tol):
    """(parity, suspect, on_surface) of each point for ray direction d (geometry.py:203-249)."""
    v0, e1, e2, n, areas = g[:5]
    h, k = np.cross(d, e2), np.cross(e1, d)
    a = np.einsum("ij,ij->i", e1, h)
    par = np.abs(a) <= 1e-12 * np.linalg.norm(e1, axis=1) * np.linalg.norm(e2, axis=1)
    f = np.where(par, 1.0, 1.0 / np.where(par, 1.0, a))
    u = (pts @ h.T - np.einsum("ij,ij->i", v0, h)) * f
    v = (pts @ k.T - np.einsum("ij,ij->i", v0, k)) * f
    dn = pts @ n.T - np.einsum("ij,ij->i", v0, n)
    t = dn * f
    w = u + v
    ok = ~par[None, :]
    in_tri = (u >= -EB) & (v >= -EB) & (w <= 1.0 + EB)
    strict = (u > EB) & (v > EB) & (w < 1.0 - EB)
    parity = np.count_nonzero(ok & strict & (t > tol), axis=1) & 1
    on = np.any(ok & in_tri & (np.abs(t) <= tol), axis=1)
    graze = np.any(ok & in_tri & ~strict & (t > tol), axis=1)
    copl = np.any(par[None, :] & (np.abs(dn) <= tol * (2.0 * areas)[None, :]), axis=1)
    return parity.astype(bool), graze | copl, on


def surface_contains(nodes, tris, pts):
    """Inside-or-on test of one closed surface (geometry.py:147-184)."""
    g = _geometry(np.asarray(nodes, float), np.asarray(tris))
    lo, hi, diam = g[5], g[6], g[7]
    tol = 1e-9 * (diam or 1.0)
    inside = np.zeros(len(pts), dtype=bool)
    cand = np.flatnonzero(np.all((pts >= lo - tol) & (pts <= hi + tol), axis=1))
    last = np.zeros(len(pts), dtype=bool)
    for d in RAY_DIRECTIONS:
        if cand.size == 0:
            break
        parity, suspect, on = _cast(g, pts[cand], d, tol)
        inside[cand[on]] = True
        settled = ~suspect & ~on
        inside[cand[settled]] = parity[settled]
        last[cand] = parity
        cand = cand[suspect & ~on]
    inside[cand] = last[cand]
    return inside


def locate(compartments, pts):
    """Innermost compartment containing each point, -1 outside (geometry.py:359-374)."""
    pts = np.atleast_2d(np.asarray(pts, float))
    labels = np.full(len(pts), -1, dtype=np.int64)
    open_ = np.arange(len(pts))
    for k, (surfaces, _, _) in enumerate(compartments):
        hit = np.zeros(len(open_), dtype=bool)
        for nodes, tris in surfaces:
            hit |= surface_contains(nodes, tris, pts[open_])
        labels[open_[hit]] = k
        open_ = open_[~hit]
    return labels


_KUHN = np.array([[0, 1, 3, 7], [0, 1, 7, 5], [0, 2, 7, 3], [0, 2, 6, 7], [0, 4, 5, 7], [0, 4, 7, 6]])
_CORNERS = np.array([[(j >> a) & 1 for a in range(3)] for j in range(8)])


def generate_mesh(compartments, h):
    """(nodes, tetra, labels, sigma) of generate_mesh (meshgen.py:186-244)."""
    allnodes = np.vstack([np.asarray(nd, float) for s, _, _ in compartments for nd, _ in s])
    lo, hi = allnodes.min(axis=0), allnodes.max(axis=0)
    nx, ny, nz = np.maximum(1, np.ceil((hi - lo) / h - 1e-12).astype(int))
    xs, ys, zs = (lo[a] + h * np.arange(c + 1) for a, c in enumerate((nx, ny, nz)))
    gz, gy, gx = np.meshgrid(zs, ys, xs, indexing="ij")
    grid = np.column_stack([gx.ravel(), gy.ravel(), gz.ravel()])
    cz, cy, cx = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    base = (cx + (nx + 1) * (cy + (ny + 1) * cz)).ravel()
    off = _CORNERS[:, 0] + (nx + 1) * (_CORNERS[:, 1] + (ny + 1) * _CORNERS[:, 2])
    tetra = (base[:, None] + off[None, :])[:, _KUHN].reshape(-1, 4)
    lab = locate(compartments, grid[tetra].mean(axis=1))
    keep = lab >= 0
    used, inv = np.unique(tetra[keep], return_inverse=True)
    tetra, lab, nodes = inv.reshape(-1, 4), lab[keep], grid[used]
    nl = locate(compartments, nodes)[tetra]
    pri = np.array([p for _, _, p in compartments])
    first = nl.max(axis=1)
    multi = np.any((nl != first[:, None]) & (nl >= 0), axis=1) & (first >= 0)
    for e in np.flatnonzero(multi):  # meshgen.py:259-268
        cands = {int(v) for v in nl[e] if v >= 0} | {int(lab[e])}
        best = min(pri[c] for c in cands)
        if pri[lab[e]] != best:
            lab[e] = min(c for c in cands if pri[c] == best)
    conds = [np.atleast_1d(np.asarray(c, float)) for _, c, _ in compartments]
    if any(c.size == 6 for c in conds):
        table = np.zeros((len(conds), 6))
        for k, c in enumerate(conds):
            table[k, :c.size if c.size == 6 else 3] = c
    else:
        table = np.array([c[0] for c in conds])
    return nodes, tetra, lab, table[lab]
