"""The CPU oracle (oracle/) pinned against golden vectors produced by the
reference package itself (tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle
from tests.fixtures import csr, load

SYSTEMS = ["sphere_small.npz", "layered_h12.npz", "layered_h14_tensor.npz"]


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.fixture(scope="module")
def cases():
    return load("solver_cases.npz")


@pytest.mark.parametrize("name", ["dense50", "bound40s0", "bound40s1", "bound40s2", "none60", "ldp60"])
def test_pcg_matches_reference_bitwise(cases, name):
    """Same recurrence, same numpy/scipy calls: identical iterates."""
    A, b, x_ref = cases[f"{name}_A"], cases[f"{name}_b"], cases[f"{name}_x"]
    it_ref, res_ref, tol, mi, pre = cases[f"{name}_meta"]
    cfg = oracle.PcgSettings(tolerance=tol, max_iterations=None if mi < 0 else int(mi),
                             preconditioner="ldp" if pre else "none")
    x, it, res = oracle.pcg_solve(sp.csr_matrix(A), b, cfg)
    assert it == it_ref
    np.testing.assert_array_equal(x, x_ref)
    assert res == res_ref


def test_best_iterate_failure(cases):
    with pytest.raises(oracle.ConvergenceFailure) as exc:
        oracle.pcg_solve(sp.csr_matrix(cases["fail30_A"]), np.ones(30),
                         oracle.PcgSettings(tolerance=1e-14, max_iterations=3))
    np.testing.assert_array_equal(exc.value.best_x, cases["fail30_best_x"])
    assert exc.value.residual == cases["fail30_meta"][0]
    assert exc.value.iterations == 3


def test_transfer_matrix_zero_column(cases):
    T = oracle.transfer_matrix(sp.csr_matrix(cases["tm40_A"]), cases["tm40_B"],
                               oracle.PcgSettings(tolerance=1e-9))
    np.testing.assert_array_equal(T, cases["tm40_T"])


@pytest.mark.parametrize("name", SYSTEMS)
def test_assembly_pattern_and_values(name):
    fx = load(name)
    from tests.fixtures import electrodes_from_fixture, mesh_from_fixture

    mesh = mesh_from_fixture(fx)
    el = electrodes_from_fixture(mesh, fx)
    A, g = oracle.assemble_A(mesh.nodes, mesh.tetra, mesh.sigma, list(el.triangles),
                             el.triangle_areas, el.impedances, el.areas)
    Ar = csr(fx, "A")
    assert g == int(fx["ground"])
    np.testing.assert_array_equal(A.indptr, Ar.indptr)
    np.testing.assert_array_equal(A.indices, Ar.indices)
    np.testing.assert_allclose(A.data, Ar.data, rtol=1e-12, atol=1e-14 * np.abs(Ar.data).max())
    K = oracle.volume_stiffness(mesh.nodes, mesh.tetra, mesh.sigma)
    Kr = csr(fx, "K")
    np.testing.assert_array_equal(K.indptr, Kr.indptr)
    np.testing.assert_array_equal(K.indices, Kr.indices)


@pytest.mark.parametrize("name", SYSTEMS)
def test_leadfield_and_iterations(name):
    fx = load(name)
    A, B = csr(fx, "A"), csr(fx, "B")
    C = sp.diags(fx["Cdiag"], format="csr")
    L = B.shape[1]
    R = np.eye(L) - np.full((L, L), 1.0 / L)
    cfg = oracle.PcgSettings(tolerance=float(fx["tol"]))
    lf, T, M = oracle.eeg_leadfield(A, B, C, R, csr(fx, "G"), cfg)
    assert rel(lf, fx["LF"]) < 1e-12
    np.testing.assert_allclose(M, fx["M"], rtol=1e-12, atol=1e-14 * np.abs(fx["M"]).max())
    _, its = oracle.transfer_matrix(A, B, cfg, return_iterations=True)
    np.testing.assert_array_equal(its, fx["iters"])
    # the reference's own noise floor (tol 1e-8 vs 1e-12) is far below the 1e-6 bar
    if "LF_tol12" in fx and float(fx["tol"]) == 1e-8:
        assert rel(fx["LF"], fx["LF_tol12"]) < 1e-7


def test_eit_leadfield_matches_reference():
    fx = load("sphere_small.npz")
    A, B = csr(fx, "A"), csr(fx, "B")
    C = sp.diags(fx["Cdiag"], format="csr")
    L = B.shape[1]
    R = np.eye(L) - np.full((L, L), 1.0 / L)
    sets = np.split(fx["eit_dof_elems"], fx["eit_dof_ptr"][1:-1])
    cols, bg = oracle.eit_leadfield(fx["nodes"], fx["tetra"].astype(np.int64), A, B, C, R,
                                    int(fx["ground"]), sets, fx["eit_currents"],
                                    oracle.PcgSettings(tolerance=float(fx["tol"])))
    assert rel(cols, fx["eit_LF"]) < 1e-10
    np.testing.assert_allclose(bg, fx["eit_bg"], rtol=1e-10, atol=1e-15)


def test_c1_summary_fixture_is_consistent():
    fx = load("c1.npz")
    assert fx["nodes"].shape == (55545, 3)
    assert int(fx["A_nnz"]) == 792439
    assert fx["LF"].shape == (32, 3000)
    assert 300 < fx["iters"].min() <= fx["iters"].max() < 400
