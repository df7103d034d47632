"""Device topology and source matrix against the reference (meshgen.py:114-130,
fem.py:291-422): boundary faces bit-exact (same faces, same order), G' with
the reference's pattern and values to rounding."""
import hashlib

import numpy as np
import pytest
import scipy.sparse as sp

from tests.fixtures import csr, load, mesh_from_fixture

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def topo(cuda):
    from paper_1811_07717_b200 import topology

    return topology


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", ["sphere_small.npz", "layered_h12.npz", "layered_h14_tensor.npz",
                                  "c1.npz"])
def test_boundary_faces_match_reference(topo, name):
    fx = load(name)
    mesh = mesh_from_fixture(fx)
    faces, owners = topo.boundary_triangles_device(mesh)
    assert sha(faces.astype(np.int64)) == str(fx["bfaces_sha"])
    assert sha(owners.astype(np.int64)) == str(fx["bowners_sha"])


@pytest.mark.parametrize("name", ["sphere_small.npz", "layered_h12.npz", "c1.npz"])
def test_whitney_Gt_matches_reference(topo, name):
    from paper_1811_07717_b200 import model

    fx = load(name)
    mesh = mesh_from_fixture(fx)
    src = model.SourceSpace(positions=fx["src_positions"], orientations=None,
                            element_ids=fx["src_elements"], mode="unconstrained")
    Gt = topo.assemble_Gt_device(mesh, src).to_scipy()
    Gr = sp.csr_matrix(csr(fx, "G").T)
    Gr.sort_indices()
    np.testing.assert_array_equal(Gt.indptr, Gr.indptr)
    np.testing.assert_array_equal(Gt.indices, Gr.indices)
    np.testing.assert_allclose(Gt.data, Gr.data, rtol=1e-9, atol=1e-12 * np.abs(Gr.data).max())


def test_whitney_constrained_is_oriented_combination(topo):
    """Constrained columns are the orientation-weighted Cartesian columns (fem.py:414-416)."""
    from paper_1811_07717_b200 import model

    fx = load("layered_h12.npz")
    mesh = mesh_from_fixture(fx)
    el = fx["src_elements"][:50]
    o = np.random.default_rng(0).normal(size=(50, 3))
    o /= np.linalg.norm(o, axis=1, keepdims=True)
    su = model.SourceSpace(positions=fx["src_positions"][:50], orientations=None, element_ids=el,
                           mode="unconstrained")
    sc = model.SourceSpace(positions=fx["src_positions"][:50], orientations=o, element_ids=el,
                           mode="constrained")
    Gu = topo.assemble_Gt_device(mesh, su).to_scipy().toarray()
    Gc = topo.assemble_Gt_device(mesh, sc).to_scipy().toarray()
    expect = np.einsum("scn,sc->sn", Gu.reshape(50, 3, -1), o)
    np.testing.assert_allclose(Gc, expect, rtol=1e-12, atol=1e-14 * np.abs(expect).max())


def test_leadfield_with_device_G(topo):
    """LF built from the device G' equals the reference LF (C1 fixture)."""
    from paper_1811_07717_b200.engine import EegEngine
    from paper_1811_07717_b200 import model
    from paper_1811_07717_b200.solver import PcgConfig
    from tests.fixtures import electrodes_from_fixture

    fx = load("layered_h12.npz")
    mesh = mesh_from_fixture(fx)
    el = electrodes_from_fixture(mesh, fx)
    src = model.SourceSpace(positions=fx["src_positions"], orientations=None,
                            element_ids=fx["src_elements"], mode="unconstrained")
    eng = EegEngine(mesh, el, topo.assemble_Gt_device(mesh, src), PcgConfig(float(fx["tol"])))
    lf = eng.build(to_host=True)
    ref = fx["LF"]
    assert np.linalg.norm(lf - ref) / np.linalg.norm(ref) <= 1e-6


@pytest.mark.parametrize("name", ["sphere_small.npz", "layered_h12.npz", "c1.npz"])
def test_electrodes_and_ground_on_device_match_reference(cuda, name):
    """ElectrodeSet.from_centers (fem.py:157-173) and ground_node (fem.py:188-194)
    on the device: the reference's triangle sets and grounding node."""
    import numpy as np

    from paper_1811_07717_b200 import model, synthetic
    from paper_1811_07717_b200.topology import (boundary_triangles_device, electrodes_from_centers,
                                                ground_node_device)
    from tests.fixtures import electrodes_from_fixture, load, mesh_from_fixture

    fx = load(name)
    mesh = mesh_from_fixture(fx)
    mesh._boundary = boundary_triangles_device(mesh)
    ref = electrodes_from_fixture(mesh, fx)
    L = ref.count
    radius = {"sphere_small.npz": 0.05, "layered_h12.npz": 0.014, "c1.npz": 0.014}[name]
    R = 0.1 if name == "sphere_small.npz" else 0.092
    el = electrodes_from_centers(mesh, synthetic.fibonacci_sphere_points(L, R), radius, fx["impedances"])
    host = model.ElectrodeSet.from_centers(mesh, synthetic.fibonacci_sphere_points(L, R), radius,
                                           fx["impedances"])
    for a, b, c in zip(el.triangle_ids, ref.triangle_ids, host.triangle_ids):
        np.testing.assert_array_equal(a, b)
        np.testing.assert_array_equal(a, c)
    assert ground_node_device(mesh, el) == int(fx["ground"]) == model.ground_node(mesh, el)
