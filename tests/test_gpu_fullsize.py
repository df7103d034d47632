"""Parity at the benchmark's full sizes against the reference itself.

C2 (BASELINE.json configs[1]: 1,001,184 nodes, 128 electrodes, 10k sources) is
the bench workload.  tests/golden/c2_fullsize.npz holds the output of
/root/reference's headfem run unmodified on the same system
(tests/golden/make_fullsize_golden.py): all 128 transfer columns solved by the
reference's pcg_solve, its electrode_response and eeg_leadfield.  Checked here:

* inputs: mesh arrays, electrode triangles, source elements, A's CSR pattern
  and the ground node bit-exact with the reference (meshgen.py:51-145,
  fem.py:157-173, meshgen.py:351-391, fem.py:197-224);
* every one of the 128 columns: iteration count within +-1 of the reference
  and true residual <= tol (solver.py:64-111); T on every 997th row, the column
  norms and T' w within 1e-6 (relative) of the reference's T;
* M = C - B'T (leadfield.py:104-109) and the lead field (leadfield.py:122-134):
  a fixed 2,000-column subset, LF @ Omega for a seeded 30,000 x 8 Omega and
  ||LF||_F, all within 1e-6 relative Frobenius error.

C5 (configs[4], 4.9M nodes, 256 electrodes): three transfer columns against
the reference's pcg_solve (tests/golden/c5_fullsize.npz).  C4 (configs[3],
EIT on the C2 mesh): the DOF map against the exact host path and the
Jacobian's columns for 64 DOFs against the oracle's _dof_sensitivities and
column formula built from the device's own T and U (leadfield.py:179-237).
"""
import hashlib
import os

import numpy as np
import pytest

from tests.fixtures import GOLDEN

pytestmark = pytest.mark.gpu

TOL = 1e-8
REL = 1e-6


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


def golden(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.fail(f"{path} missing: run tests/golden/make_fullsize_golden.py where /root/reference exists")
    return dict(np.load(path, allow_pickle=False))


@pytest.fixture(scope="module")
def c2(cuda):
    import torch

    from paper_1811_07717_b200 import synthetic
    from paper_1811_07717_b200.engine import EegEngine
    from paper_1811_07717_b200.leadfield import response_operator, symmetrize
    from paper_1811_07717_b200.solver import PcgConfig

    gd = golden("c2_fullsize.npz")
    prob = synthetic.eeg_problem("c2", device=True)
    engine = EegEngine(prob.mesh, prob.electrodes, prob.G, PcgConfig(tolerance=TOL),
                       prob.B, prob.C, prob.R)
    A = engine.assemble()
    T = engine.solve(A)
    info = engine.last_info
    M = symmetrize(engine.response_block(T).cpu().numpy())
    W = response_operator(M, engine.R)
    LF = engine.lf_partial(T, W).cpu().numpy()
    rows = torch.from_numpy(gd["T_rows"]).to(T.device)
    w = torch.from_numpy(np.random.default_rng(7).standard_normal(T.shape[0])).to(T.device)
    out = dict(gd=gd, prob=prob, engine=engine, A=A.to_scipy(), info=info, M=M, LF=LF,
               T_sample=T[rows].cpu().numpy(), T_norm=torch.linalg.norm(T, dim=0).cpu().numpy(),
               T_w=(T.T @ w).cpu().numpy(), Tcols=T[:, [0, 77]].cpu().numpy())
    del T
    torch.cuda.empty_cache()
    return out


def test_c2_inputs_bit_exact_with_reference(c2):
    gd, prob, A = c2["gd"], c2["prob"], c2["A"]
    mesh, el = prob.mesh, prob.electrodes
    assert mesh.n_nodes == int(gd["n_nodes"]) == 1_001_184
    assert sha(np.asarray(mesh.nodes)) == str(gd["nodes_sha"])
    assert sha(np.asarray(mesh.tetra, dtype=np.int64)) == str(gd["tetra_sha"])
    ptr = np.cumsum([0] + [len(t) for t in el.triangle_ids])
    np.testing.assert_array_equal(ptr, gd["tri_ptr"])
    assert sha(np.concatenate(el.triangle_ids).astype(np.int64)) == str(gd["tri_ids_sha"])
    np.testing.assert_array_equal(np.asarray(prob.sources.element_ids, dtype=np.int64), gd["src_elements"])
    assert A.nnz == int(gd["A_nnz"]) == 14_739_218
    assert sha(A.indptr.astype(np.int32)) == str(gd["A_sha_indptr"])
    assert sha(A.indices.astype(np.int32)) == str(gd["A_sha_indices"])
    assert int(c2["engine"].ground) == int(gd["ground"])
    assert c2["engine"].Gt.nnz == int(gd["G_nnz"])


def test_c2_every_column_matches_reference(c2):
    """All 128 columns: iterations +-1, converged, T samples within 1e-6."""
    gd, info = c2["gd"], c2["info"]
    np.testing.assert_array_equal(gd["columns"], np.arange(128))
    d_it = np.abs(info.iterations.astype(np.int64) - gd["iters"])
    assert d_it.max() <= 1, (info.iterations, gd["iters"])
    assert np.all(info.true_residual <= TOL) and np.all(gd["true_res"] <= TOL)
    Ts, Tg = c2["T_sample"], gd["T_sample"]
    per_col = np.linalg.norm(Ts - Tg, axis=0) / np.linalg.norm(Tg, axis=0)
    assert per_col.max() <= REL, per_col.max()
    assert np.max(np.abs(c2["T_norm"] - gd["T_norm"]) / gd["T_norm"]) <= REL
    assert np.max(np.abs(c2["T_w"] - gd["T_w"]) / np.abs(gd["T_w"]).max()) <= REL
    print(f"\nC2 iterations: |d| max {d_it.max()}, mean {d_it.mean():.2f}; T sample rel max {per_col.max():.2e}")


def test_c2_response_and_leadfield_match_reference(c2):
    gd, LF = c2["gd"], c2["LF"]
    assert LF.shape == tuple(gd["LF_shape"]) == (128, 30_000)
    assert rel(c2["M"], gd["M"]) <= REL
    e_sub = rel(LF[:, gd["LF_cols"]], gd["LF_sub"])
    omega = np.random.default_rng(13).standard_normal((LF.shape[1], 8))
    e_om = rel(LF @ omega, gd["LF_omega"])
    e_fro = abs(np.linalg.norm(LF) - float(gd["LF_fro"])) / float(gd["LF_fro"])
    assert e_sub <= REL and e_om <= REL and e_fro <= REL, (e_sub, e_om, e_fro)
    means = np.abs(LF.mean(axis=0))
    assert np.all(means <= 1e-10 * np.maximum(np.linalg.norm(LF, axis=0), 1e-300))
    print(f"\nC2 LF vs reference: subset {e_sub:.2e}, LF.Omega {e_om:.2e}, ||LF|| {e_fro:.2e}; "
          f"M {rel(c2['M'], gd['M']):.2e}")


def test_c2_assembly_values_match_oracle(c2):
    """Values to rounding (the reference's duplicate-sum order is scipy's unstable sort)."""
    import oracle

    prob, Ad = c2["prob"], c2["A"]
    el = prob.electrodes
    Ao, g = oracle.assemble_A(prob.mesh.nodes, prob.mesh.tetra, prob.mesh.sigma, list(el.triangles),
                              el.triangle_areas, el.impedances, el.areas)
    np.testing.assert_array_equal(Ad.indptr, Ao.indptr)
    np.testing.assert_array_equal(Ad.indices, Ao.indices)
    assert np.abs(Ad.data - Ao.data).max() <= 1e-12 * np.abs(Ao.data).max()


def test_c5_columns_match_reference(cuda):
    """C5: 4,886,489 nodes; columns 0, 1 and 255 against the reference's pcg_solve."""
    import torch

    from paper_1811_07717_b200 import synthetic
    from paper_1811_07717_b200.fem import assemble_A_device
    from paper_1811_07717_b200.solver import PcgConfig, transfer_device

    gd = golden("c5_fullsize.npz")
    prob = synthetic.eeg_problem("c5", device=True, with_G=False)
    mesh = prob.mesh
    assert mesh.n_nodes == int(gd["n_nodes"])
    assert sha(np.asarray(mesh.nodes)) == str(gd["nodes_sha"])
    assert sha(np.asarray(mesh.tetra, dtype=np.int64)) == str(gd["tetra_sha"])
    el = prob.electrodes
    np.testing.assert_array_equal(np.cumsum([0] + [len(t) for t in el.triangle_ids]), gd["tri_ptr"])
    assert sha(np.concatenate(el.triangle_ids).astype(np.int64)) == str(gd["tri_ids_sha"])
    A, g = assemble_A_device(mesh, el)
    assert A.nnz == int(gd["A_nnz"]) and int(g) == int(gd["ground"])
    assert sha(A.indptr.cpu().numpy()) == str(gd["A_sha_indptr"])
    assert sha(A.indices.cpu().numpy()) == str(gd["A_sha_indices"])
    cols = [int(c) for c in gd["columns"]]
    T, info = transfer_device(A, prob.B.tocsc()[:, cols], PcgConfig(tolerance=TOL))
    d_it = np.abs(info.iterations.astype(np.int64) - gd["iters"])
    assert d_it.max() <= 1, (info.iterations, gd["iters"])
    assert np.all(info.true_residual <= TOL)
    rows = torch.from_numpy(gd["T_rows"]).to(T.device)
    Ts = T[rows].cpu().numpy()
    per_col = np.linalg.norm(Ts - gd["T_sample"], axis=0) / np.linalg.norm(gd["T_sample"], axis=0)
    assert per_col.max() <= REL, per_col
    w = torch.from_numpy(np.random.default_rng(7).standard_normal(T.shape[0])).to(T.device)
    Tw = (T.T @ w).cpu().numpy()
    assert np.max(np.abs(Tw - gd["T_w"]) / np.abs(gd["T_w"])) <= REL
    print(f"\nC5 columns {cols}: iterations {info.iterations.tolist()} vs {gd['iters'].tolist()}, "
          f"T sample rel max {per_col.max():.2e}")


def test_c4_eit_jacobian_against_oracle(c2):
    """C4 (BASELINE.json configs[3]) on the C2 mesh: 64 electrodes, 32 adjacent-pair
    patterns, 5,000 DOFs.  DOF sets identical to the exact host k-d-tree path
    (leadfield.py:80-101); the Jacobian's columns for 64 DOFs against the oracle's
    _dof_sensitivities (leadfield.py:179-207) and column formula
    cols[p*L:(p+1)*L] = -R M^-1 Q[p]' (leadfield.py:230-237) evaluated on the
    device's own T, U and M."""
    import torch

    import oracle
    from paper_1811_07717_b200 import model, synthetic
    from paper_1811_07717_b200.fem import assemble_A
    from paper_1811_07717_b200.leadfield import (
        _electrode_response_device, _solve_response, adjacent_pair_patterns, build_dof_map,
        eit_leadfield)
    from paper_1811_07717_b200.solver import PcgConfig, solve_block

    mesh = c2["prob"].mesh
    el = model.ElectrodeSet.from_centers(mesh, synthetic.fibonacci_sphere_points(64, 0.092),
                                         radius=0.012, impedances=1e3)
    dofs = build_dof_map(mesh, [0, 1], 5000, seed=2)
    tree_sets, tree_centers = oracle.build_dof_map(mesh, [0, 1], 5000, seed=2, method="tree")
    assert all(np.array_equal(a, b) for a, b in zip(dofs.element_sets, tree_sets))
    np.testing.assert_array_equal(dofs.centers, tree_centers)
    I = adjacent_pair_patterns(64)[:, :32]
    B, C, R = model.assemble_B_C_R(mesh, el)
    A = assemble_A(mesh, el)
    sysm = model.CemSystem(mesh=mesh, electrodes=el, A=A, B=B, C=C, R=R,
                           ground=model.ground_node(mesh, el))
    cfg = PcgConfig(TOL)
    lf = eit_leadfield(sysm, dofs, I, cfg)
    assert lf.matrix.shape == (32 * 64, 5000) and np.isfinite(lf.matrix).all()
    blocks = lf.matrix.reshape(32, 64, -1)
    assert np.abs(blocks.sum(axis=1)).max() <= 1e-10 * np.abs(lf.matrix).max()
    # the oracle on the device's own T, U, M
    dsys, T, M, _ = _electrode_response_device(sysm, cfg)
    V = _solve_response(M, I)
    U, _ = solve_block(dsys.op, dsys.Bd @ torch.from_numpy(np.ascontiguousarray(V)).cuda(), cfg)
    pick = np.linspace(0, 4999, 64).astype(int)
    Qo = oracle.dof_sensitivities(mesh.nodes, mesh.tetra, [dofs.element_sets[k] for k in pick],
                                  sysm.ground, U.cpu().numpy(), T.cpu().numpy())
    Jo = np.concatenate([-(R @ oracle.solve_response(M, Qo[p].T)) for p in range(32)], axis=0)
    Jg = lf.matrix[:, pick]
    e = rel(Jg, Jo)
    assert e <= 1e-10, e
    print(f"\nC4 Jacobian (64 DOFs x 2048 rows) vs oracle on device T/U: rel {e:.2e}")
