"""C3 (BASELINE.json configs[2]): the MEG lead field.  The reference has no MEG
(SPEC.md:8), so nothing here is pinned to it.  Checked instead:

* hf_meg_rhs against a numpy restatement of the same formula (csrc/meg.cu);
* the physics, as the reference checks its EEG lead field against the analytic
  sphere potential (test_leadfield.py:131-159, within 15%): on a concentric-
  sphere mesh the full MEG lead field (primary + volume currents) must match
  Sarvas' closed form for a spherically symmetric conductor, and the volume
  currents must nearly cancel for radial magnetometers;
* the transfer columns satisfy A T = S' and are width-independent like the
  EEG ones.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def sarvas(sensors, positions):
    """Sarvas (1987) field of unit x/y/z dipoles, flux through each sensor's coils."""
    ns = sensors.n_sensors
    L = np.zeros((ns, 3 * len(positions)))
    for s in range(ns):
        for c in range(sensors.coil_ptr[s], sensors.coil_ptr[s + 1]):
            r, n, w = sensors.coils[c, :3], sensors.coils[c, 3:6], sensors.coils[c, 6]
            av = r[None, :] - positions
            a = np.linalg.norm(av, axis=1)
            rr = np.linalg.norm(r)
            ar = av @ r
            F = a * (rr * a + rr ** 2 - positions @ r)
            gF = ((a ** 2 / rr + ar / a + 2 * a + 2 * rr)[:, None] * r[None, :]
                  - (a + 2 * rr + ar / a)[:, None] * positions)
            for k in range(3):
                q = np.zeros(3)
                q[k] = 1.0
                qxr0 = np.cross(q[None, :], positions)
                B = 1e-7 / F[:, None] ** 2 * (F[:, None] * qxr0 - (qxr0 @ r)[:, None] * gF)
                L[s, k::3] += w * (B @ n)
    return L


@pytest.fixture(scope="module")
def setup(cuda):
    from paper_1811_07717_b200 import meg, model, synthetic

    mesh = synthetic.sphere_mesh(synthetic.C1_RADII, synthetic.C1_COND, 0.004)
    src = model.place_sources(mesh, [0], 60, seed=4)
    keep = np.linalg.norm(src.positions, axis=1) < 0.06  # away from the staircase surface
    src = model.SourceSpace(positions=src.positions[keep], orientations=None,
                            element_ids=src.element_ids[keep], mode="unconstrained")
    sensors = meg.helmet_306()
    eng = meg.MegEngine(mesh, sensors, src, meg.PcgConfig(1e-10))
    return mesh, src, sensors, eng


def test_helmet_306():
    from paper_1811_07717_b200 import meg

    s = meg.helmet_306()
    assert s.n_sensors == 306 and s.kinds.count("mag") == 102
    assert np.allclose(np.linalg.norm(s.coils[:, 3:6], axis=1), 1.0)


def test_meg_rhs_matches_numpy(setup):
    mesh, src, sensors, eng = setup
    S = eng.rhs().cpu().numpy()
    nodes, tet, sig = mesh.nodes, mesh.tetra, mesh.sigma
    p = nodes[tet]
    J = np.transpose(p[:, 1:] - p[:, :1], (0, 2, 1))       # columns p_k - p_0
    det = np.linalg.det(J)
    inv = np.linalg.inv(J)                                    # rows: grad phi_1..3
    g = np.concatenate([-inv.sum(axis=1, keepdims=True), inv], axis=1)  # (m, 4, 3)
    w = (sig * det / 6.0)[:, None, None] * g
    xc = p.mean(axis=1)
    cols = [0, 1, 2, 150, 305]
    for s in cols:
        acc = np.zeros((len(tet), 4))
        for c in range(sensors.coil_ptr[s], sensors.coil_ptr[s + 1]):
            r, n, wt = sensors.coils[c, :3], sensors.coils[c, 3:6], sensors.coils[c, 6]
            d = r[None, :] - xc
            v = np.cross(d, n[None, :]) / np.linalg.norm(d, axis=1)[:, None] ** 3
            acc += wt * np.einsum("eak,ek->ea", w, v)
        ref = -1e-7 * np.bincount(tet.ravel(), weights=acc.ravel(), minlength=mesh.n_nodes)
        ref[eng.ground] = 0.0
        assert np.linalg.norm(S[:, s] - ref) <= 1e-11 * np.linalg.norm(ref), s


def test_meg_leadfield_matches_sarvas_sphere(setup):
    mesh, src, sensors, eng = setup
    L = eng.build(to_host=True)
    ref = sarvas(sensors, src.positions)
    err = np.linalg.norm(L - ref) / np.linalg.norm(ref)
    mags = [i for i, k in enumerate(sensors.kinds) if k == "mag"]
    Lp = eng.primary().cpu().numpy()
    sec = np.linalg.norm(L[mags] - Lp[mags]) / np.linalg.norm(Lp[mags])
    print(f"\nMEG LF vs Sarvas: {err:.3e}; radial-magnetometer volume-current share {sec:.3e}")
    assert err <= 0.15
    assert sec <= 0.05
    assert np.all(eng.last_info.true_residual <= 1e-10)


def test_meg_transfer_columns(setup):
    import torch

    from paper_1811_07717_b200.device import PcgOperator
    from paper_1811_07717_b200.solver import PcgConfig, solve_block

    mesh, src, sensors, eng = setup
    A = eng.assemble()
    S = eng.rhs()
    cfg = PcgConfig(1e-10)
    T, info = solve_block(PcgOperator(A), S, cfg)
    T3, _ = solve_block(PcgOperator(A), S[:, 100:103].contiguous(), cfg)
    assert torch.equal(T[:, 100:103], T3)
    As = A.to_scipy()
    Tn, Sn = T.cpu().numpy(), S.cpu().numpy()
    res = np.linalg.norm(As @ Tn - Sn, axis=0) / np.linalg.norm(Sn, axis=0)
    assert res.max() <= 1e-10
