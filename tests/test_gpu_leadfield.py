"""Lead-field parity with the reference's golden outputs (leadfield.py:104-237):
relative Frobenius error <= 1e-6 (BASELINE.json north star), per-column
iteration counts within +-1, and the reference's own invariances."""
import numpy as np
import pytest

from tests.fixtures import load, system_from_fixture

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng(cuda):
    import paper_1811_07717_b200 as e

    return e


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("name", ["sphere_small.npz", "layered_h12.npz", "layered_h14_tensor.npz"])
def test_eeg_leadfield_matches_reference(eng, name):
    fx = load(name)
    _, _, sysm, _ = system_from_fixture(fx)
    cfg = eng.PcgConfig(tolerance=float(fx["tol"]))
    lf = eng.eeg_leadfield(sysm, cfg)
    assert lf.matrix.shape == fx["LF"].shape
    assert rel(lf.matrix, fx["LF"]) <= 1e-6
    # columns zero-mean by construction of R
    means = np.abs(lf.matrix.mean(axis=0))
    assert np.all(means <= 1e-10 * np.maximum(np.linalg.norm(lf.matrix, axis=0), 1e-300))


def test_electrode_response_matches_reference(eng):
    fx = load("layered_h12.npz")
    _, _, sysm, _ = system_from_fixture(fx)
    T, M = eng.electrode_response(sysm, eng.PcgConfig(tolerance=float(fx["tol"])))
    assert T.flags.c_contiguous
    assert rel(T, fx["T"]) < 1e-6
    np.testing.assert_allclose(M, M.T, atol=1e-12 * np.abs(M).max())
    assert rel(M, fx["M"]) < 1e-8


def test_eeg_leadfield_end_to_end_from_gpu_assembly(eng):
    """A assembled on the device feeds the solve: same LF as the reference's A."""
    from paper_1811_07717_b200.model import CemSystem

    fx = load("layered_h12.npz")
    mesh, el, sysm, _ = system_from_fixture(fx)
    A = eng.assemble_A(mesh, el)
    sys2 = CemSystem(mesh=mesh, electrodes=el, A=A, B=sysm.B, C=sysm.C, R=sysm.R,
                     ground=sysm.ground, G=sysm.G, source_space=sysm.source_space)
    lf = eng.eeg_leadfield(sys2, eng.PcgConfig(tolerance=float(fx["tol"])))
    assert rel(lf.matrix, fx["LF"]) <= 1e-6


def test_electrode_permutation_permutes_rows(eng):
    from paper_1811_07717_b200.model import CemSystem, ElectrodeSet, assemble_B_C_R

    fx = load("layered_h12.npz")
    mesh, el, sysm, _ = system_from_fixture(fx)
    perm = np.random.default_rng(0).permutation(el.count)
    el2 = ElectrodeSet(mesh, [el.triangle_ids[k] for k in perm], el.impedances[perm])
    B, C, R = assemble_B_C_R(mesh, el2)
    sys2 = CemSystem(mesh=mesh, electrodes=el2, A=sysm.A, B=B, C=C, R=R, ground=sysm.ground,
                     G=sysm.G, source_space=sysm.source_space)
    cfg = eng.PcgConfig(tolerance=1e-12)
    lf, lf2 = eng.eeg_leadfield(sysm, cfg), eng.eeg_leadfield(sys2, cfg)
    np.testing.assert_allclose(lf2.matrix, lf.matrix[perm], rtol=1e-9,
                               atol=1e-12 * np.abs(lf.matrix).max())


def test_missing_G_rejected(eng):
    from paper_1811_07717_b200.model import CemSystem

    fx = load("sphere_small.npz")
    _, _, s, _ = system_from_fixture(fx)
    s2 = CemSystem(mesh=s.mesh, electrodes=s.electrodes, A=s.A, B=s.B, C=s.C, R=s.R,
                   ground=s.ground, G=None)
    with pytest.raises(eng.SingularSystemError):
        eng.eeg_leadfield(s2)


def test_eit_leadfield_matches_reference(eng):
    fx = load("sphere_small.npz")
    _, _, sysm, _ = system_from_fixture(fx)
    dofs = eng.EitDofMap(element_sets=tuple(np.split(fx["eit_dof_elems"], fx["eit_dof_ptr"][1:-1])),
                         centers=fx["eit_centers"])
    lf = eng.eit_leadfield(sysm, dofs, fx["eit_currents"], eng.PcgConfig(tolerance=float(fx["tol"])))
    assert rel(lf.matrix, fx["eit_LF"]) <= 1e-6
    np.testing.assert_allclose(lf.background_data, fx["eit_bg"], rtol=1e-8, atol=1e-14)
    assert lf.n_patterns == fx["eit_currents"].shape[1]


def test_eit_layered_matches_reference(eng):
    fx = load("layered_h12.npz")
    _, _, sysm, _ = system_from_fixture(fx)
    dofs = eng.EitDofMap(element_sets=tuple(np.split(fx["eit_dof_elems"], fx["eit_dof_ptr"][1:-1])),
                         centers=fx["eit_centers"])
    lf = eng.eit_leadfield(sysm, dofs, fx["eit_currents"], eng.PcgConfig(tolerance=float(fx["tol"])))
    assert rel(lf.matrix, fx["eit_LF"]) <= 1e-6


def test_eit_forward_linearity(eng):
    fx = load("sphere_small.npz")
    _, _, sysm, _ = system_from_fixture(fx)
    I = np.array([1.0, -0.25, -0.5, -0.25, 0.0, 0.0])
    tm = eng.electrode_response(sysm, eng.PcgConfig(tolerance=1e-12))
    y1 = eng.eit_forward(sysm, I, tm=tm)
    y3 = eng.eit_forward(sysm, 3.0 * I, tm=tm)
    np.testing.assert_allclose(y3, 3.0 * y1, rtol=1e-12)
    with pytest.raises(eng.CurrentPatternError):
        eng.eit_forward(sysm, np.array([1.0, 0, 0, 0, 0, 0]), tm=tm)


def test_c1_leadfield_matches_reference(eng):
    """Config C1 of BASELINE.json: 55,545 nodes, 32 electrodes, 1k sources."""
    from paper_1811_07717_b200.model import CemSystem
    from paper_1811_07717_b200.solver import operator, solve_block

    fx = load("c1.npz")
    mesh, el, sysm, _ = system_from_fixture(fx)
    A = eng.assemble_A(mesh, el)
    sys2 = CemSystem(mesh=mesh, electrodes=el, A=A, B=sysm.B, C=sysm.C, R=sysm.R,
                     ground=sysm.ground, G=sysm.G, source_space=sysm.source_space)
    cfg = eng.PcgConfig(tolerance=float(fx["tol"]))
    lf = eng.eeg_leadfield(sys2, cfg)
    assert rel(lf.matrix, fx["LF"]) <= 1e-6
    from paper_1811_07717_b200.solver import rhs_block

    _, info = solve_block(operator(A, cfg), rhs_block(sysm.B), cfg)
    assert np.all(np.abs(info.iterations - fx["iters"]) <= 1), (info.iterations, fx["iters"])


def _dense_owner(cc, centers):
    """The reference's owner computation (leadfield.py:98-99) in row chunks."""
    out = []
    for a in range(0, len(cc), 4096):
        d = np.linalg.norm(cc[a:a + 4096][:, None, :] - centers[None, :, :], axis=2)
        out.append(np.argmin(d, axis=1))
    return np.concatenate(out)


def test_dof_map_device_matches_reference(eng):
    """build_dof_map on the GPU gives the reference's element sets (layered_h12 golden)."""
    from paper_1811_07717_b200.leadfield import build_dof_map
    from tests.fixtures import mesh_from_fixture

    fx = load("layered_h12.npz")
    mesh = mesh_from_fixture(fx)
    dofs = build_dof_map(mesh, [0, 1], 20, seed=2)
    np.testing.assert_array_equal(np.concatenate(dofs.element_sets), fx["eit_dof_elems"])
    np.testing.assert_array_equal(np.cumsum([0] + [len(e) for e in dofs.element_sets]),
                                  fx["eit_dof_ptr"])
    np.testing.assert_array_equal(dofs.centers, fx["eit_centers"])


@pytest.mark.parametrize("n_dofs", [1, 7, 500, 3000])
def test_nearest_center_bitwise_argmin(eng, n_dofs):
    """Every owner equals numpy's argmin of the reference's distance array (C1 mesh, 303k elements;
    3000 centres span two shared-memory tiles)."""
    from paper_1811_07717_b200.leadfield import nearest_center_device
    from tests.fixtures import mesh_from_fixture

    mesh = mesh_from_fixture(load("c1.npz"))
    cc = mesh.centroids()
    rng = np.random.default_rng(n_dofs)
    centers = cc[rng.choice(len(cc), size=n_dofs, replace=False)]
    sel = rng.choice(len(cc), size=40_000, replace=False)
    np.testing.assert_array_equal(nearest_center_device(cc[sel], centers),
                                  _dense_owner(cc[sel], centers))


def test_nearest_center_ties_take_first_index(eng):
    from paper_1811_07717_b200.leadfield import nearest_center_device

    centers = np.array([[1.0, 0, 0], [-1.0, 0, 0], [1.0, 0, 0], [0, 3.0, 0]])
    pts = np.array([[0.0, 0, 0], [0, 1.0, 0], [0, 0, 5.0], [2.0, 0, 0], [0, 3.0, 0]])
    own = nearest_center_device(pts, centers)
    np.testing.assert_array_equal(own, _dense_owner(pts, centers))
    np.testing.assert_array_equal(own, [0, 0, 0, 0, 3])
    # squares that differ by one ulp but share the rounded root keep the earlier centre
    base = np.array([[0.0, 0.0, 0.0]])
    s = 2.0
    c2 = np.array([[np.sqrt(np.nextafter(s, 3)), 0, 0], [np.sqrt(s), 0, 0]])
    np.testing.assert_array_equal(nearest_center_device(base, c2), _dense_owner(base, c2))


def test_tet_centroids_bitwise_and_partition(eng):
    """hf_tet_centroids equals TetMesh.centroids() bit for bit (numpy's rounding of the
    4-corner mean), and the device DOF map (centroids, nearest centre, partition) equals
    the host path's sets on the C1 mesh."""
    import torch

    from paper_1811_07717_b200 import _native as N
    from paper_1811_07717_b200.fem import DeviceMesh
    from paper_1811_07717_b200.leadfield import build_dof_map
    from tests.fixtures import mesh_from_fixture

    mesh = mesh_from_fixture(load("c1.npz"))
    dm = DeviceMesh.of(mesh)
    out = torch.empty((mesh.n_elements, 3), dtype=torch.float64, device="cuda")
    N.check("hf_tet_centroids", N.lib.hf_tet_centroids(N.ptr(dm.nodes), N.ptr(dm.tetra), None,
                                                       mesh.n_elements, N.ptr(out), N.stream_handle()))
    np.testing.assert_array_equal(out.cpu().numpy(), mesh.centroids())
    import oracle

    dev = build_dof_map(mesh, [0, 1], 700, seed=5)
    host_sets, host_centers = oracle.build_dof_map(mesh, [0, 1], 700, seed=5, method="tree")
    np.testing.assert_array_equal(dev.centers, host_centers)
    assert all(np.array_equal(a, b) for a, b in zip(dev.element_sets, host_sets))
