"""Golden vectors for mesh generation, made by running
the UNMODIFIED reference in this container:

    PYTHONPATH=/root/reference/pkg/src OPENBLAS_NUM_THREADS=1 python tests/golden/make_meshgen_golden.py

Writes tests/golden/meshgen_cases.npz:
  ray_dirs                         geometry._RAY_DIRECTIONS
  loc<k>_*                         Segmentation.locate on hand-picked point sets
                                   (surface nodes/triangles per compartment, points, labels)
  gm<k>_*                          generate_mesh(seg, h): nodes, tetra, labels, sigma
The segmentations are the reference tests' own fixtures (tests/conftest.py,
tests/test_meshgen.py, tests/test_geometry.py).  The C1 mesh (generate_mesh at
h = 4 mm on the 3-shell sphere) is already in c1.npz.
"""
import os

import numpy as np
from headfem import geometry as G
from headfem.meshgen import generate_mesh

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "meshgen_cases.npz")

TET_NODES = np.array([[1.0, 1.0, 1.0], [1.0, -1.0, -1.0], [-1.0, 1.0, -1.0], [-1.0, -1.0, 1.0]])
TET_TRIS = np.array([[0, 1, 2], [0, 3, 1], [0, 2, 3], [1, 3, 2]])


def segs():
    tet = G.SurfaceMesh(TET_NODES, TET_TRIS, name="tet")
    cube = G.box_surface(name="cube")
    nested = G.Segmentation([
        G.Compartment(G.icosphere(0.5, 2, name="inner"), 0.33, priority=0, active=True),
        G.Compartment(G.icosphere(1.0, 2, name="outer"), 0.43, priority=0)])
    prio = G.Segmentation([
        G.Compartment(G.box_surface((0, 0, 0), (1, 1, 1), name="a"), 1.0, priority=2),
        G.Compartment(G.box_surface((0.75, 0, 0), (1.75, 1, 1), name="b"), 1.0, priority=1)])
    tensor = G.Segmentation([
        G.Compartment(G.icosphere(0.5, 1), np.array([1.0, 2.0, 3.0, 0.1, 0.0, 0.0])),
        G.Compartment(G.icosphere(1.0, 1), 0.5)])
    blobs = G.Segmentation([G.Compartment(
        (G.icosphere(0.3, 2, center=(-0.5, 0, 0)), G.icosphere(0.3, 2, center=(0.5, 0, 0))), 1.0,
        active=True), G.Compartment(G.icosphere(1.0, 2), 0.2, priority=1)])
    layered = G.Segmentation([
        G.Compartment(G.icosphere(r, 3, name=f"shell{k}"), s, priority=p, active=k == 0)
        for k, (r, s, p) in enumerate(zip((0.079, 0.082, 0.087, 0.092), (0.33, 1.79, 0.0064, 0.43),
                                          (2, 1, 0, 3)))])
    return dict(tet=G.Segmentation([G.Compartment(tet, 1.0)]),
                cube=G.Segmentation([G.Compartment(cube, 1.0, active=True)]),
                nested=nested, prio=prio, tensor=tensor, blobs=blobs, layered=layered)


def put_seg(d, key, seg):
    d[f"{key}_ncomp"] = np.array(len(seg))
    for c, comp in enumerate(seg.compartments):
        d[f"{key}_c{c}_nsurf"] = np.array(len(comp.surfaces))
        d[f"{key}_c{c}_cond"] = np.atleast_1d(np.asarray(comp.conductivity, dtype=float))
        d[f"{key}_c{c}_prio"] = np.array(comp.priority)
        for s, surf in enumerate(comp.surfaces):
            d[f"{key}_c{c}_s{s}_nodes"] = surf.nodes
            d[f"{key}_c{c}_s{s}_tris"] = surf.triangles


def main():
    rng = np.random.default_rng(7)
    d = {"ray_dirs": G._RAY_DIRECTIONS}
    S = segs()
    lattice = np.stack(np.meshgrid(*(np.linspace(-0.25, 1.25, 7),) * 3, indexing="ij"), -1).reshape(-1, 3)
    cases = {
        "tet": np.vstack([TET_NODES, TET_NODES.mean(0), rng.uniform(-1.2, 1.2, (400, 3)),
                          0.5 * (TET_NODES[:, None] + TET_NODES[None]).reshape(-1, 3)]),
        "cube": np.vstack([lattice, rng.uniform(-0.1, 1.1, (400, 3))]),  # faces, edges, corners
        "nested": np.vstack([S["nested"][0].surfaces[0].nodes, S["nested"][1].surfaces[0].nodes,
                             rng.uniform(-1.1, 1.1, (3000, 3)), np.zeros((1, 3))]),
        "blobs": np.vstack([rng.uniform(-1.0, 1.0, (3000, 3)), [[0.0, 0.0, 0.0], [0.8, 0, 0]]]),
        "layered": rng.uniform(-0.095, 0.095, (20000, 3)),
    }
    for k, (name, pts) in enumerate(cases.items()):
        put_seg(d, f"loc{k}", S[name])
        d[f"loc{k}_points"] = pts
        d[f"loc{k}_labels"] = S[name].locate(pts)
        print(name, np.bincount(d[f"loc{k}_labels"] + 1))
    gm = [("cube", 0.25), ("cube", 0.3), ("nested", 0.25), ("nested", 0.22), ("prio", 0.5),
          ("tensor", 0.4), ("blobs", 0.15), ("layered", 0.009)]
    for k, (name, h) in enumerate(gm):
        mesh = generate_mesh(S[name], h)
        put_seg(d, f"gm{k}", S[name])
        d[f"gm{k}_h"] = np.array(h)
        for a in ("nodes", "tetra", "labels", "sigma"):
            d[f"gm{k}_{a}"] = getattr(mesh, a)
        print(name, h, mesh)
    np.savez_compressed(OUT, **d)


if __name__ == "__main__":
    main()
