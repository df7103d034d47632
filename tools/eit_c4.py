"""C4 (BASELINE.json configs[3]): linearised EIT lead field on the 1M-node C2
mesh — 64 electrodes, 32 adjacent-pair patterns, 5,000 conductivity DOFs.

Times each stage on the device and checks a sample of DOF columns of the
sensitivity tensor Q against the oracle's restatement of
_dof_sensitivities (leadfield.py:179-207) evaluated for those DOFs only.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_1811_07717_b200 import model, synthetic  # noqa: E402
from paper_1811_07717_b200.engine import EegEngine  # noqa: E402
from paper_1811_07717_b200.leadfield import (  # noqa: E402
    adjacent_pair_patterns, build_dof_map, dof_sensitivities_device, eit_leadfield)
from paper_1811_07717_b200.solver import PcgConfig  # noqa: E402


def main():
    t0 = time.time()
    mesh = synthetic.sphere_mesh(synthetic.C2_RADII, synthetic.C2_COND, 0.0015)
    el = model.ElectrodeSet.from_centers(mesh, synthetic.fibonacci_sphere_points(64, 0.092),
                                         radius=0.012, impedances=1e3)
    build_dof_map(mesh, [0, 1], 50, seed=2)  # warm-up (context, module load)
    t1 = time.time()
    dofs = build_dof_map(mesh, [0, 1], 5000, seed=2)
    t2 = time.time()
    tree_sets, _ = oracle.build_dof_map(mesh, [0, 1], 5000, seed=2, method="tree")
    t3 = time.time()
    same = all(np.array_equal(a, b) for a, b in zip(dofs.element_sets, tree_sets))
    print(f"build_dof_map C4: device {t2 - t1:.3f}s, host k-d tree {t3 - t2:.1f}s, "
          f"identical sets: {same}", flush=True)
    I = adjacent_pair_patterns(64)[:, :32]
    B, C, R = model.assemble_B_C_R(mesh, el)
    print(f"inputs {time.time() - t0:.1f}s: {mesh}, {len(el)} electrodes, "
          f"{sum(len(e) for e in dofs.element_sets):,} DOF elements", flush=True)
    cfg = PcgConfig(1e-8)
    eng = EegEngine(mesh, el, sp_eye(mesh.n_nodes), cfg, B, C, R)
    A = eng.assemble()
    sysm = model.CemSystem(mesh=mesh, electrodes=el, A=A, B=B, C=C, R=R,
                           ground=model.ground_node(mesh, el))
    for rep in range(2):
        torch.cuda.synchronize()
        t = time.time()
        lf = eit_leadfield(sysm, dofs, I, cfg)
        torch.cuda.synchronize()
        print(f"eit_leadfield (C4) {time.time() - t:.2f}s  LF {lf.matrix.shape}", flush=True)
    # stage timing of the sensitivity kernel alone, and a sampled oracle check
    from paper_1811_07717_b200.leadfield import _electrode_response_device, _solve_response
    from paper_1811_07717_b200.solver import solve_block
    dsys, T, M, _ = _electrode_response_device(sysm, cfg)
    V = _solve_response(M, I)
    U, _ = solve_block(dsys.op, dsys.Bd @ torch.from_numpy(np.ascontiguousarray(V)).cuda(), cfg)
    torch.cuda.synchronize()
    t = time.time()
    Q = dof_sensitivities_device(mesh, dofs, sysm.ground, T, U, 64, 32)
    torch.cuda.synchronize()
    print(f"k_eit_sens: {(time.time() - t) * 1e3:.1f} ms for Q {tuple(Q.shape)}", flush=True)
    pick = [0, 1234, 4999]
    Qo = oracle.dof_sensitivities(mesh.nodes, mesh.tetra, [dofs.element_sets[k] for k in pick],
                                  sysm.ground, U.cpu().numpy(), T.cpu().numpy())
    Qg = Q[:, pick, :].cpu().numpy()
    err = np.linalg.norm(Qg - Qo) / np.linalg.norm(Qo)
    print(f"sampled Q vs oracle: rel err {err:.2e}", flush=True)
    assert err < 1e-12
    zero_mean = np.abs(lf.matrix.reshape(32, 64, -1).sum(axis=1)).max() / np.abs(lf.matrix).max()
    print(f"pattern-block zero mean: {zero_mean:.1e}")


def sp_eye(n):
    import scipy.sparse as sp

    return sp.csr_matrix((n, 1))


if __name__ == "__main__":
    main()
