"""Parity at the benchmark's full size (BASELINE.json configs[1], C2: 1,001,184
nodes, 128 electrodes, 10k sources), on the same inputs bench.py times.

The CPU oracle cannot solve all 128 columns here (~20 s per column), so the
checks are: the device CSR pattern and ground node bit-exact against the
oracle's assembly (fem.py:96-109, 197-224); two transfer columns against the
oracle's PCG on that matrix (solver.py:64-111; rel <= 1e-6, iterations +-1);
and the lead field's size-independent properties (finite, zero-mean columns
by construction of R, leadfield.py:122-134; every column converged with a
true residual <= tol)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-8


@pytest.fixture(scope="module")
def c2(cuda):
    import torch

    from paper_1811_07717_b200 import synthetic
    from paper_1811_07717_b200.engine import EegEngine
    from paper_1811_07717_b200.solver import PcgConfig

    prob = synthetic.eeg_problem("c2", device=True)
    engine = EegEngine(prob.mesh, prob.electrodes, prob.G, PcgConfig(tolerance=TOL),
                       prob.B, prob.C, prob.R)
    A = engine.assemble()
    T = engine.solve(A)
    info = engine.last_info
    M = None
    from paper_1811_07717_b200.leadfield import response_operator, symmetrize

    M = symmetrize(engine.response_block(T).cpu().numpy())
    W = response_operator(M, engine.R)
    LF = engine.lf_partial(T, W).cpu().numpy()
    cols = [0, 77]
    Tcols = T[:, cols].cpu().numpy()
    del T
    torch.cuda.empty_cache()
    return dict(prob=prob, engine=engine, A=A.to_scipy(), info=info, LF=LF, cols=cols, Tcols=Tcols)


def test_c2_assembly_matches_oracle(c2):
    import oracle

    prob, Ad = c2["prob"], c2["A"]
    el = prob.electrodes
    Ao, g = oracle.assemble_A(prob.mesh.nodes, prob.mesh.tetra, prob.mesh.sigma, list(el.triangles),
                              el.triangle_areas, el.impedances, el.areas)
    assert Ad.shape == Ao.shape == (1_001_184, 1_001_184)
    assert int(g) == int(c2["engine"].ground)
    np.testing.assert_array_equal(Ad.indptr, Ao.indptr)
    np.testing.assert_array_equal(Ad.indices, Ao.indices)
    # values: the reference's duplicate-summation order is scipy's (unstable), so rounding only
    scale = np.abs(Ao.data).max()
    assert np.abs(Ad.data - Ao.data).max() <= 1e-12 * scale


def test_c2_transfer_columns_match_oracle(c2):
    import oracle

    A, B = c2["A"], c2["prob"].B.tocsc()
    for j, col in enumerate(c2["cols"]):
        b = B[:, col].toarray().ravel()
        x, it, res = oracle.pcg_solve(A, b, oracle.PcgSettings(tolerance=TOL))
        t = c2["Tcols"][:, j]
        assert np.linalg.norm(t - x) / np.linalg.norm(x) <= 1e-6
        assert abs(int(c2["info"].iterations[col]) - it) <= 1
        assert res <= TOL


def test_c2_leadfield_properties(c2):
    LF, info = c2["LF"], c2["info"]
    assert LF.shape == (128, 30_000)
    assert np.isfinite(LF).all()
    means = np.abs(LF.mean(axis=0))
    assert np.all(means <= 1e-10 * np.maximum(np.linalg.norm(LF, axis=0), 1e-300))
    assert np.all(info.true_residual <= TOL)
    n = 1_001_184
    assert np.all(info.iterations > 0) and np.all(info.iterations < int(5 * np.sqrt(n)) + 1000)


def test_c4_eit_leadfield_sampled_against_oracle(c2):
    """C4 (BASELINE.json configs[3]) on the C2 mesh: 64 electrodes, 32 adjacent-pair
    patterns, 5,000 DOFs.  DOF sets identical to the exact host k-d-tree path
    (leadfield.py:80-101), sampled sensitivity columns vs the oracle's
    _dof_sensitivities (leadfield.py:179-207), zero-mean pattern blocks."""
    import torch

    import oracle
    from paper_1811_07717_b200 import model, synthetic
    from paper_1811_07717_b200.leadfield import (
        _electrode_response_device, _solve_response, adjacent_pair_patterns, build_dof_map,
        dof_sensitivities_device, eit_leadfield)
    from paper_1811_07717_b200.solver import PcgConfig, solve_block

    mesh = c2["prob"].mesh
    el = model.ElectrodeSet.from_centers(mesh, synthetic.fibonacci_sphere_points(64, 0.092),
                                         radius=0.012, impedances=1e3)
    dofs = build_dof_map(mesh, [0, 1], 5000, seed=2, method="device")
    tree = build_dof_map(mesh, [0, 1], 5000, seed=2, method="tree")
    assert all(np.array_equal(a, b) for a, b in zip(dofs.element_sets, tree.element_sets))
    I = adjacent_pair_patterns(64)[:, :32]
    B, C, R = model.assemble_B_C_R(mesh, el)
    from paper_1811_07717_b200.fem import assemble_A

    A = assemble_A(mesh, el)
    sysm = model.CemSystem(mesh=mesh, electrodes=el, A=A, B=B, C=C, R=R,
                           ground=model.ground_node(mesh, el))
    cfg = PcgConfig(TOL)
    lf = eit_leadfield(sysm, dofs, I, cfg)
    assert lf.matrix.shape == (32 * 64, 5000) and np.isfinite(lf.matrix).all()
    blocks = lf.matrix.reshape(32, 64, -1)
    assert np.abs(blocks.sum(axis=1)).max() <= 1e-10 * np.abs(lf.matrix).max()
    dsys, T, M, _ = _electrode_response_device(sysm, cfg)
    V = _solve_response(M, I)
    U, _ = solve_block(dsys.op, dsys.Bd @ torch.from_numpy(np.ascontiguousarray(V)).cuda(), cfg)
    Q = dof_sensitivities_device(mesh, dofs, sysm.ground, T, U, 64, 32)
    pick = [0, 1234, 4999]
    Qo = oracle.dof_sensitivities(mesh.nodes, mesh.tetra, [dofs.element_sets[k] for k in pick],
                                  sysm.ground, U.cpu().numpy(), T.cpu().numpy())
    Qg = Q[:, pick, :].cpu().numpy()
    assert np.linalg.norm(Qg - Qo) / np.linalg.norm(Qo) < 1e-12
