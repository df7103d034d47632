"""Host-side input types of the lead-field path.

The engine consumes the reference's own objects (headfem TetMesh,
ElectrodeSet, CemSystem — any object with the same attributes works).  This
module mirrors those types for standalone use (the GPU box has no
reference): same attributes, same validation, same results, written
vectorised so building a 1M-node system takes seconds instead of minutes.

  TetMesh                 meshgen.py:51-145  (boundary_triangles via packed keys)
  ElectrodeSet            fem.py:121-182
  ground_node             fem.py:188-194
  assemble_B_C_R          fem.py:227-258
  face_incidence          fem.py:291-304
  assemble_G              fem.py:307-422  (Whitney stencil, batched min-norm lstsq)
  place_sources           meshgen.py:351-391 (unconstrained mode)
  CemSystem               fem.py:428-444
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .errors import AssemblyError, ElectrodeError, LocationError, ParameterError

_FACES = np.array([[1, 2, 3], [0, 3, 2], [0, 1, 3], [0, 2, 1]])  # face k opposite vertex k


def tet_volumes(nodes, tetra):
    p = nodes[tetra]
    return np.linalg.det(p[:, 1:] - p[:, :1]) / 6.0


def _pack_sorted_faces(key):
    """int64 code per sorted node triple, ordered like the lexicographic rows."""
    key = key.astype(np.int64)
    nmax = int(key.max()) + 1 if key.size else 1
    bits = max(1, (nmax - 1).bit_length())
    if 3 * bits <= 63:
        return (key[:, 0] << (2 * bits)) | (key[:, 1] << bits) | key[:, 2], None
    return None, key


def face_keys(tetra):
    faces = tetra[:, _FACES].reshape(-1, 3)
    return faces, np.sort(faces, axis=1)


def _unique_rows(key):
    packed, raw = _pack_sorted_faces(key)
    if packed is not None:
        uniq_codes, inv, counts = np.unique(packed, return_inverse=True, return_counts=True)
        order = None
        return uniq_codes, inv.ravel(), counts, order
    uniq, inv, counts = np.unique(raw, axis=0, return_inverse=True, return_counts=True)
    return uniq, inv.ravel(), counts, None


class TetMesh:
    """Labelled tetrahedral mesh (meshgen.py:51-145)."""

    def __init__(self, nodes, tetra, labels, sigma):
        nodes = np.ascontiguousarray(nodes, dtype=float)
        tetra = np.ascontiguousarray(tetra, dtype=np.int64)
        labels = np.ascontiguousarray(labels, dtype=np.int64)
        sigma = np.ascontiguousarray(sigma, dtype=float)
        if tetra.ndim != 2 or tetra.shape[1] != 4:
            raise ParameterError(f"tetra must be (m, 4), got {tetra.shape}")
        if tetra.size and (tetra.min() < 0 or tetra.max() >= len(nodes)):
            raise IndexError("tetrahedron references a missing node")
        if len(labels) != len(tetra):
            raise ParameterError("labels length must equal element count")
        if len(sigma) != len(tetra):
            raise ParameterError("sigma length must equal element count")
        if sigma.ndim == 2 and sigma.shape[1] != 6:
            raise ParameterError("tensor sigma must have 6 columns")
        vols = tet_volumes(nodes, tetra)
        if np.any(vols <= 0):
            raise ParameterError(f"{np.count_nonzero(vols <= 0)} element(s) with non-positive volume")
        self.nodes, self.tetra, self.labels, self.sigma, self.volumes = nodes, tetra, labels, sigma, vols
        for arr in (self.nodes, self.tetra, self.labels, self.sigma, self.volumes):
            arr.setflags(write=False)
        self._boundary = None

    n_nodes = property(lambda self: len(self.nodes))
    n_elements = property(lambda self: len(self.tetra))
    is_tensor = property(lambda self: self.sigma.ndim == 2)

    def centroids(self):
        return self.nodes[self.tetra].mean(axis=1)

    def element_faces(self):
        return self.tetra[:, _FACES].reshape(-1, 3)

    def boundary_triangles(self):
        """Faces used by one element, in element-face order (meshgen.py:114-130)."""
        if self._boundary is None:
            faces, key = face_keys(self.tetra)
            _, inv, counts, _ = _unique_rows(key)
            idx = np.flatnonzero(counts[inv] == 1)
            self._boundary = (faces[idx], idx // 4)
        return self._boundary

    def boundary_nodes(self):
        if getattr(self, "_bnodes", None) is None:  # cached with the boundary faces (meshgen.py:122-134)
            self._bnodes = np.unique(self.boundary_triangles()[0])
            self._bnodes.setflags(write=False)
        return self._bnodes

    def with_sigma(self, sigma):
        return TetMesh(self.nodes, self.tetra, self.labels, sigma)

    def with_nodes(self, nodes):
        return TetMesh(nodes, self.tetra, self.labels, self.sigma)

    def __repr__(self):
        return f"TetMesh({self.n_nodes} nodes, {self.n_elements} elements)"


class MeshArrays:
    """A mesh handed over as raw host arrays — nodes (n,3) f64, tetra (m,4),
    sigma — with no validation and nothing cached across objects: the input of
    an end-to-end build from host buffers.  Its boundary faces come from the
    device (hf_boundary_faces, bit-exact with meshgen.py:114-130) the first
    time they are asked for."""

    def __init__(self, nodes, tetra, sigma, labels=None):
        self.nodes = np.asarray(nodes, dtype=float)
        self.tetra = np.asarray(tetra)
        self.sigma = np.asarray(sigma, dtype=float)
        self.labels = labels
        self._boundary = None

    n_nodes = property(lambda self: len(self.nodes))
    n_elements = property(lambda self: len(self.tetra))

    def boundary_triangles(self):
        if self._boundary is None:
            from .topology import boundary_triangles_device

            self._boundary = boundary_triangles_device(self)
        return self._boundary

    boundary_nodes = TetMesh.boundary_nodes


def triangle_areas(nodes, triangles):
    p = nodes[triangles]
    return 0.5 * np.linalg.norm(np.cross(p[:, 1] - p[:, 0], p[:, 2] - p[:, 0]), axis=1)


class ElectrodeSet:
    """Disjoint boundary-triangle sets with contact impedances (fem.py:121-182)."""

    def __init__(self, mesh, triangle_ids, impedances):
        bfaces, _ = mesh.boundary_triangles()
        n_el = len(triangle_ids)
        imp = np.broadcast_to(np.asarray(impedances, dtype=float), (n_el,)).copy()
        if np.any(imp <= 0):
            raise ElectrodeError("contact impedances must be positive")
        seen = (np.concatenate([np.asarray(t, dtype=np.int64) for t in triangle_ids])
                if n_el else np.array([], dtype=np.int64))
        if seen.size != len(np.unique(seen)):
            raise ElectrodeError("electrode triangle sets overlap")
        if seen.size and (seen.min() < 0 or seen.max() >= len(bfaces)):
            raise ElectrodeError("electrode triangle index outside the boundary")
        areas_all = triangle_areas(mesh.nodes, bfaces)
        self.triangle_ids = tuple(np.asarray(t, dtype=np.int64) for t in triangle_ids)
        self.triangles = tuple(bfaces[t] for t in self.triangle_ids)
        self.triangle_areas = tuple(areas_all[t] for t in self.triangle_ids)
        self.areas = np.array([a.sum() for a in self.triangle_areas])
        if np.any(self.areas <= 0):
            raise ElectrodeError("electrode with zero covered area")
        self.impedances = imp
        self.count = n_el

    @classmethod
    def from_centers(cls, mesh, centers, radius, impedances, chunk=65536):
        centers = np.atleast_2d(np.asarray(centers, dtype=float))
        bfaces, _ = mesh.boundary_triangles()
        cent = mesh.nodes[bfaces].mean(axis=1)
        nearest = np.empty(len(cent), dtype=np.int64)
        dmin = np.empty(len(cent))
        for a in range(0, len(cent), chunk):  # same per-entry arithmetic as fem.py:164-166
            d = np.linalg.norm(cent[a:a + chunk, None, :] - centers[None, :, :], axis=2)
            nearest[a:a + chunk] = np.argmin(d, axis=1)
            dmin[a:a + chunk] = d[np.arange(len(d)), nearest[a:a + chunk]]
        covered = dmin <= radius
        ids = [np.flatnonzero(covered & (nearest == k)) for k in range(len(centers))]
        for k, t in enumerate(ids):
            if t.size == 0:
                raise ElectrodeError(f"electrode {k} at {centers[k]} covers no boundary triangle "
                                     f"within radius {radius}")
        return cls(mesh, ids, impedances)

    @property
    def node_set(self):
        if getattr(self, "_node_set", None) is None:
            ns = (np.array([], dtype=np.int64) if self.count == 0
                  else np.unique(np.concatenate([t.ravel() for t in self.triangles])))
            ns.setflags(write=False)
            self._node_set = ns
        return self._node_set

    def __len__(self):
        return self.count


def ground_node(mesh, electrodes):
    """Lowest-index boundary node not covered by any electrode (fem.py:188-194)."""
    free = np.setdiff1d(mesh.boundary_nodes(), electrodes.node_set)
    if free.size == 0:
        raise AssemblyError("electrodes cover every boundary node; cannot choose a grounding node")
    return int(free[0])


def electrode_contacts(electrodes):
    """(triangles (t,3) int32, coef (t,)) with coef = (1/(Z_l A_l)) * A_t in the
    electrode/triangle order of fem.py:207-211."""
    tris, coef = [], []
    for t, at, z, a_l in zip(electrodes.triangles, electrodes.triangle_areas,
                             electrodes.impedances, electrodes.areas):
        scale = 1.0 / (z * a_l)
        tris.append(np.asarray(t, dtype=np.int32).reshape(-1, 3))
        coef.append(scale * np.asarray(at, dtype=float))
    if not tris:
        return np.zeros((0, 3), np.int32), np.zeros(0)
    return np.concatenate(tris), np.concatenate(coef)


def assemble_B_C_R(mesh, electrodes):
    """Electrode coupling blocks B (n x L CSR), C = diag(1/Z), R = I - 11'/L (fem.py:227-258)."""
    n, L = mesh.n_nodes, electrodes.count
    if L == 0:
        raise ElectrodeError("no electrodes defined")
    rows, cols, vals = [], [], []
    for l, (tris, areas, z, a_l) in enumerate(zip(electrodes.triangles, electrodes.triangle_areas,
                                                  electrodes.impedances, electrodes.areas)):
        if areas.sum() <= 0:
            raise ElectrodeError(f"electrode {l} has zero covered area")
        rows.append(tris.ravel())
        cols.append(np.full(tris.size, l, dtype=np.int64))
        vals.append(np.repeat(areas / (3.0 * z * a_l), 3))
    B = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(n, L)).tocsr()
    C = sp.diags(1.0 / electrodes.impedances, format="csr")
    R = np.eye(L) - np.full((L, L), 1.0 / L)
    return B, C, R


# ---------------------------------------------------------------- sources

@dataclass(frozen=True)
class SourceSpace:
    """Source positions / element ids (meshgen.py:148-169)."""

    positions: np.ndarray
    orientations: np.ndarray | None
    element_ids: np.ndarray
    mode: str

    n_sources = property(lambda self: len(self.positions))
    n_components = property(lambda self: 1 if self.mode == "constrained" else 3)


def place_sources(mesh, active_labels, n, seed=0):
    """Unconstrained sources drawn volume-weighted in the active labels,
    uniform inside each element — the same random stream as meshgen.py:351-391."""
    if n < 1:
        raise ParameterError("need at least one source")
    cand = np.flatnonzero(np.isin(mesh.labels, np.asarray(active_labels)))
    rng = np.random.default_rng(seed)
    vols = mesh.volumes[cand]
    elements = rng.choice(cand, size=n, p=vols / vols.sum())
    u = np.sort(rng.random((n, 3)), axis=1)
    bary = np.column_stack([u[:, 0], u[:, 1] - u[:, 0], u[:, 2] - u[:, 1], 1.0 - u[:, 2]])
    positions = np.einsum("nk,nkj->nj", bary, mesh.nodes[mesh.tetra[elements]])
    return SourceSpace(positions=positions, orientations=None, element_ids=elements,
                       mode="unconstrained")


def face_incidence(mesh):
    """(face id per element face (m,4), elements of each face (F,2), sorted face
    nodes (F,3)) — fem.py:291-304; face_elems[:,0] is the lower element index."""
    faces, key = face_keys(mesh.tetra)
    packed, raw = _pack_sorted_faces(key)
    if packed is not None:
        uniq_codes, first, inv, counts = np.unique(packed, return_index=True, return_inverse=True,
                                                   return_counts=True)
        uniq = key[first]
    else:
        uniq, first, inv, counts = np.unique(raw, axis=0, return_index=True, return_inverse=True,
                                             return_counts=True)
    inv = inv.ravel()
    owners = np.repeat(np.arange(mesh.n_elements), 4)
    order = np.argsort(inv, kind="stable")
    starts = np.concatenate([[0], np.cumsum(counts)[:-1]])
    face_elems = np.full((len(counts), 2), -1, dtype=np.int64)
    face_elems[:, 0] = owners[order[starts]]
    second = counts == 2
    face_elems[second, 1] = owners[order[starts[second] + 1]]
    return inv.reshape(-1, 4), face_elems, uniq


def assemble_G(mesh, sources, incidence=None):
    """Source matrix (n x 3S unconstrained / n x S constrained), fem.py:391-422.

    Whitney face functions of each source element (fem.py:307-364) combined by
    the minimum-norm solution of moments' coeff = I (np.linalg.lstsq(rcond=None)
    equals the pseudo-inverse with cutoff eps*max(3,4)), computed for all
    sources at once.
    """
    elements = np.asarray(sources.element_ids, dtype=np.int64)
    if elements.size and (elements.min() < 0 or elements.max() >= mesh.n_elements):
        raise LocationError("source element index outside the mesh")
    inv4, face_elems, uniq = incidence if incidence is not None else face_incidence(mesh)
    nodes, tetra = mesh.nodes, mesh.tetra
    S = len(elements)
    fid = inv4[elements]                       # (S,4)
    fnodes = uniq[fid]                         # (S,4,3) sorted face nodes
    fc = nodes[fnodes].mean(axis=2)            # (S,4,3)
    p0, p1, p2 = nodes[fnodes[..., 0]], nodes[fnodes[..., 1]], nodes[fnodes[..., 2]]
    ncanon = np.cross(p1 - p0, p2 - p0)
    adj = face_elems[fid]                      # (S,4,2)
    centroids = mesh.centroids()
    moments = np.zeros((S, 4, 3))
    signs = np.zeros((S, 4, 2))
    for slot in range(2):
        k = adj[..., slot]
        ok = k >= 0
        kk = np.where(ok, k, 0)
        tk = tetra[kk]                                         # (S,4,4)
        is_face = (tk[..., :, None] == fnodes[..., None, :]).any(axis=-1)  # (S,4,4)
        opp = np.take_along_axis(tk, np.argmin(is_face, axis=-1)[..., None], axis=-1)[..., 0]
        sgn = np.where(np.einsum("sjk,sjk->sj", ncanon, fc - nodes[opp]) > 0, 1.0, -1.0)
        sgn = np.where(ok, sgn, 0.0)
        signs[..., slot] = sgn
        moments += sgn[..., None] * (centroids[kk] - nodes[opp]) / 3.0
    Mt = np.transpose(moments, (0, 2, 1))       # (S,3,4)
    coeff = np.linalg.pinv(Mt, rcond=np.finfo(float).eps * 4)  # (S,4,3)
    if sources.mode == "constrained":
        coeff = np.einsum("sjc,sc->sj", coeff, sources.orientations)[..., None]
    ncomp = coeff.shape[2]
    rows, cols, vals = [], [], []
    for slot in range(2):
        k = adj[..., slot]
        ok = k >= 0
        tk = tetra[np.where(ok, k, 0)]                        # (S,4,4)
        w = (signs[..., slot] / 4.0)[..., None] * coeff       # (S,4,ncomp)
        for c in range(ncomp):
            r = tk.reshape(S, 16)
            v = np.repeat(w[..., c], 4, axis=1).reshape(S, 16)
            m = np.repeat(ok, 4, axis=1).reshape(S, 16)
            colid = np.repeat((np.arange(S) * ncomp + c)[:, None], 16, axis=1)
            rows.append(r[m]), cols.append(colid[m]), vals.append(v[m])
    G = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(mesh.n_nodes, ncomp * S)).tocsr()
    G.sum_duplicates()
    G.sort_indices()
    return G


@dataclass(frozen=True)
class CemSystem:
    """Assembled CEM blocks (fem.py:428-444)."""

    mesh: object
    electrodes: object
    A: object
    B: sp.csr_matrix
    C: sp.csr_matrix
    R: np.ndarray
    ground: int
    G: object = None
    source_space: object = None

    @property
    def n_electrodes(self):
        return self.electrodes.count
