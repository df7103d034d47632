"""Rebuild systems from the golden fixtures (no reference needed at run time)."""
from __future__ import annotations

import os

import numpy as np
import scipy.sparse as sp

from paper_1811_07717_b200 import model

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name), allow_pickle=False))


def csr(fx, prefix):
    shape = tuple(int(v) for v in fx[f"{prefix}_shape"])
    return sp.csr_matrix((fx[f"{prefix}_data"], fx[f"{prefix}_indices"], fx[f"{prefix}_indptr"]),
                         shape=shape)


def mesh_from_fixture(fx):
    return model.TetMesh(fx["nodes"], fx["tetra"].astype(np.int64), fx["labels"], fx["sigma"])


def electrodes_from_fixture(mesh, fx):
    ptr = fx["tri_ptr"]
    ids = [fx["tri_ids"][ptr[k]:ptr[k + 1]] for k in range(len(ptr) - 1)]
    return model.ElectrodeSet(mesh, ids, fx["impedances"])


def system_from_fixture(fx, use_reference_A=True):
    """(mesh, electrodes, CemSystem with the reference's A/B/C/G, sources)."""
    mesh = mesh_from_fixture(fx)
    el = electrodes_from_fixture(mesh, fx)
    B, C, R = model.assemble_B_C_R(mesh, el)
    A = csr(fx, "A") if (use_reference_A and "A_data" in fx) else None
    G = csr(fx, "G") if "G_data" in fx else None
    src = None
    if "src_elements" in fx:
        src = model.SourceSpace(positions=fx["src_positions"], orientations=None,
                                element_ids=fx["src_elements"], mode="unconstrained")
    sysm = model.CemSystem(mesh=mesh, electrodes=el, A=A, B=B, C=C, R=R,
                           ground=int(fx["ground"]), G=G, source_space=src)
    return mesh, el, sysm, src


def seg_parts(fx, key):
    """[(surfaces [(nodes, tris)], conductivity, priority)] of a stored segmentation."""
    out = []
    for c in range(int(fx[f"{key}_ncomp"])):
        surfs = [(fx[f"{key}_c{c}_s{s}_nodes"], fx[f"{key}_c{c}_s{s}_tris"])
                 for s in range(int(fx[f"{key}_c{c}_nsurf"]))]
        cond = fx[f"{key}_c{c}_cond"]
        out.append((surfs, float(cond[0]) if cond.size == 1 else cond, int(fx[f"{key}_c{c}_prio"])))
    return out


def segmentation(fx, key):
    """The stored segmentation as the package's geometry mirror types."""
    from paper_1811_07717_b200 import geometry as G

    return G.Segmentation([G.Compartment([G.SurfaceMesh(nd, tr) for nd, tr in surfs], cond,
                                         priority=pri)
                           for surfs, cond, pri in seg_parts(fx, key)])
