"""Oracle restatement of headfem/leadfield.py (test infrastructure only).

electrode_response   leadfield.py:104-109
solve_response       leadfield.py:112-119
eeg_leadfield        leadfield.py:122-134
eit_forward          leadfield.py:165-176
build_dof_map        leadfield.py:80-101 (chunked / k-d tree: the reference's (E, m, 3) array
                     needs 459 GiB at C4)
dof_sensitivities    leadfield.py:179-207
eit_leadfield        leadfield.py:210-237
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

from .fem import stiffness_blocks
from .solver import PcgSettings, pcg_solve, transfer_matrix


def electrode_response(A, B, C, cfg=PcgSettings()):
    T = transfer_matrix(A, B, cfg)
    M = C.toarray() - B.T @ T
    M = 0.5 * (M + M.T)
    return T, M


def solve_response(M, rhs):
    lu, piv = sla.lu_factor(M)
    if np.any(np.abs(np.diag(lu)) < 1e-300):
        raise np.linalg.LinAlgError("electrode response matrix is singular")
    return sla.lu_solve((lu, piv), rhs)


def eeg_leadfield(A, B, C, R, G, cfg=PcgSettings()):
    T, M = electrode_response(A, B, C, cfg)
    TtG = np.asarray((G.T @ T).T if sp.issparse(G) else G.T @ T)
    return -(R @ solve_response(M, TtG)), T, M


def eit_forward(M, R, currents):
    I = np.asarray(currents, dtype=float)
    I2 = I[:, None] if I.ndim == 1 else I
    y = R @ solve_response(M, I2)
    return y[:, 0] if I.ndim == 1 else y


def dof_sensitivities(nodes, tetra, element_sets, ground, U, T):
    all_elems = np.concatenate([np.asarray(e) for e in element_sets])
    owner = np.concatenate([np.full(len(e), k) for k, e in enumerate(element_sets)])
    blocks = stiffness_blocks(nodes, tetra, 1.0, elements=all_elems)
    conn = tetra[all_elems]
    gmask = conn == ground
    if gmask.any():
        blocks = blocks.copy()
        blocks[np.repeat(gmask[:, :, None], 4, axis=2)] = 0.0
        blocks[np.repeat(gmask[:, None, :], 4, axis=1)] = 0.0
    Tg = T[conn]
    P, L = U.shape[1], T.shape[1]
    Q = np.zeros((P, len(element_sets), L))
    for p in range(P):
        ue = U[:, p][conn]
        s = np.einsum("eij,ej->ei", blocks, ue)
        contrib = np.einsum("eil,ei->el", Tg, s)
        np.add.at(Q[p], owner, contrib)
    return Q


def eit_leadfield(nodes, tetra, A, B, C, R, ground, element_sets, currents, cfg=PcgSettings()):
    I = np.asarray(currents, dtype=float)
    I = I[:, None] if I.ndim == 1 else I
    T, M = electrode_response(A, B, C, cfg)
    V = solve_response(M, I)
    y_bg = R @ V
    BV = np.asarray(B @ V)
    P = I.shape[1]
    U = np.empty((A.shape[0], P))
    for p in range(P):
        U[:, p], _, _ = pcg_solve(A, BV[:, p], cfg)
    Q = dof_sensitivities(nodes, tetra, element_sets, ground, U, T)
    L = B.shape[1]
    cols = np.empty((P * L, len(element_sets)))
    for p in range(P):
        cols[p * L:(p + 1) * L, :] = -(R @ solve_response(M, Q[p].T))
    return cols, y_bg.T.ravel()


def _nearest_center_exact(cc, centers, chunk=8192):
    """argmin_j ||cc_i - centers_j|| with the reference's arithmetic and first-index
    ties (leadfield.py:98-99), without the (E, m, 3) array: a k-d tree proposes the
    two nearest centres; where the runner-up is more than 1e-9 relatively farther the
    nearest is unique far beyond rounding, and the near-ties are re-evaluated with
    np.linalg.norm over all centres exactly as the reference does."""
    from scipy.spatial import cKDTree

    m = len(centers)
    if m == 1:
        return np.zeros(len(cc), dtype=np.int64)
    tree = cKDTree(centers)
    dist, idx = tree.query(cc, k=2, workers=-1)
    owner = idx[:, 0].astype(np.int64)
    close = np.flatnonzero(dist[:, 1] <= dist[:, 0] * (1.0 + 1e-9) + 1e-300)
    for a in range(0, len(close), chunk):
        sel = close[a:a + chunk]
        d = np.linalg.norm(cc[sel][:, None, :] - centers[None, :, :], axis=2)
        owner[sel] = np.argmin(d, axis=1)
    return owner


def build_dof_map(mesh, compartments, n_dofs, seed=0, method="tree", chunk=8192):
    """(element sets, centres) of build_dof_map (leadfield.py:80-101): the same draw,
    the same per-entry distance arithmetic and first-index argmin, in element chunks
    ("dense", the reference's comparison) or through an exact k-d tree ("tree")."""
    cand = np.flatnonzero(np.isin(mesh.labels, np.asarray(compartments)))
    rng = np.random.default_rng(seed)
    vols = mesh.volumes[cand]
    chosen = rng.choice(cand, size=int(n_dofs), replace=False, p=vols / vols.sum())
    centroids = mesh.nodes[mesh.tetra].mean(axis=1)
    centers = centroids[chosen]
    cc = centroids[cand]
    if method == "tree":
        owner = _nearest_center_exact(cc, centers, chunk)
    else:
        owner = np.empty(len(cand), dtype=np.int64)
        step = max(1, chunk * 64 // max(int(n_dofs), 1))
        for a in range(0, len(cand), step):
            d = np.linalg.norm(cc[a:a + step][:, None, :] - centers[None, :, :], axis=2)
            owner[a:a + step] = np.argmin(d, axis=1)
    order = np.argsort(owner, kind="stable")
    bounds = np.searchsorted(owner[order], np.arange(int(n_dofs) + 1))
    sets = tuple(cand[order[bounds[k]:bounds[k + 1]]] for k in range(int(n_dofs)))
    return sets, centers
