"""Oracle restatement of the P1 assembly in headfem/fem.py (test infrastructure only).

element_gradients / stiffness_blocks   fem.py:31-93
volume_stiffness (_scatter_blocks)     fem.py:96-109
assemble_A (+ electrodes, _ground)     fem.py:185-224

The CSR pattern follows scipy's COO->CSR (sorted columns, duplicates summed,
explicit zeros kept).  Grounding deletes the row/column entries and sets the
diagonal to 1, as the LIL assignments of fem.py:219-224 do.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

SURF_MASS = np.array([[2.0, 1.0, 1.0], [1.0, 2.0, 1.0], [1.0, 1.0, 2.0]]) / 12.0  # fem.py:185


def element_gradients(nodes, tetra):
    p = nodes[tetra]
    jac = np.stack([p[:, 1] - p[:, 0], p[:, 2] - p[:, 0], p[:, 3] - p[:, 0]], axis=2)
    vols = np.linalg.det(jac) / 6.0
    inv = np.linalg.inv(jac)
    grads = np.empty((len(p), 4, 3))
    grads[:, 1:, :] = inv
    grads[:, 0, :] = -inv.sum(axis=1)
    return vols, grads


def _tensors(sigma):
    t = np.empty((len(sigma), 3, 3))
    t[:, 0, 0], t[:, 1, 1], t[:, 2, 2] = sigma[:, 0], sigma[:, 1], sigma[:, 2]
    t[:, 0, 1] = t[:, 1, 0] = sigma[:, 3]
    t[:, 0, 2] = t[:, 2, 0] = sigma[:, 4]
    t[:, 1, 2] = t[:, 2, 1] = sigma[:, 5]
    return t


def stiffness_blocks(nodes, tetra, sigma, elements=None):
    """(m,4,4) blocks V g_i.sigma g_j; sigma a scalar, (m,) or (m,6)."""
    vols, grads = element_gradients(nodes, tetra)
    if elements is not None:
        vols, grads = vols[elements], grads[elements]
        if not np.isscalar(sigma):
            sigma = np.asarray(sigma)[elements]
    if np.any(vols <= 0):
        raise ValueError("non-positive element volume")
    if np.isscalar(sigma) or np.asarray(sigma).ndim == 1:
        s = sigma if np.isscalar(sigma) else np.asarray(sigma, dtype=float)
        return np.einsum("eik,ejk->eij", grads, grads) * (vols * s)[:, None, None]
    tens = _tensors(np.asarray(sigma, dtype=float))
    return np.einsum("eik,ekl,ejl->eij", grads, tens, grads) * vols[:, None, None]


def volume_stiffness(nodes, tetra, sigma, elements=None):
    blocks = stiffness_blocks(nodes, tetra, sigma, elements)
    conn = tetra if elements is None else tetra[elements]
    rows = np.repeat(conn, 4, axis=1).ravel()
    cols = np.tile(conn, (1, 4)).ravel()
    return sp.coo_matrix((blocks.ravel(), (rows, cols)), shape=(len(nodes),) * 2).tocsr()


def boundary_nodes(tetra):
    faces = np.stack([tetra[:, [1, 2, 3]], tetra[:, [0, 3, 2]], tetra[:, [0, 1, 3]],
                      tetra[:, [0, 2, 1]]], axis=1).reshape(-1, 3)
    key = np.sort(faces, axis=1)
    _, inv, counts = np.unique(key, axis=0, return_inverse=True, return_counts=True)
    return np.unique(faces[counts[inv.ravel()] == 1])


def ground_node(tetra, electrode_triangles):
    """Lowest boundary node not under an electrode (fem.py:188-194)."""
    covered = np.unique(np.concatenate([t.ravel() for t in electrode_triangles]))
    free = np.setdiff1d(boundary_nodes(tetra), covered)
    return int(free[0])


def assemble_A(nodes, tetra, sigma, electrode_triangles, triangle_areas, impedances, areas,
               ground=True):
    """Grounded CEM stiffness (fem.py:197-224), returned as canonical CSR."""
    K = volume_stiffness(nodes, tetra, sigma)
    n = len(nodes)
    rows, cols, vals = [K.tocoo().row], [K.tocoo().col], [K.tocoo().data]
    for tris, at, z, a_l in zip(electrode_triangles, triangle_areas, impedances, areas):
        scale = 1.0 / (z * a_l)
        for tri, a in zip(tris, at):
            blk = scale * a * SURF_MASS
            rows.append(np.repeat(tri, 3))
            cols.append(np.tile(tri, 3))
            vals.append(blk.ravel())
    A = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(n, n)).tocsr()
    g = None
    if ground and len(electrode_triangles):
        g = ground_node(tetra, electrode_triangles)
        A = A.tocoo()
        keep = (A.row != g) & (A.col != g)
        r = np.concatenate([A.row[keep], [g]])
        c = np.concatenate([A.col[keep], [g]])
        v = np.concatenate([A.data[keep], [1.0]])
        A = sp.coo_matrix((v, (r, c)), shape=(n, n)).tocsr()
    A.sort_indices()
    return A, g
