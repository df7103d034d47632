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
