"""Generate the golden fixtures from the reference package itself.

Run here (the reference is importable in this container, not on the GPU box):

    python tests/golden/make_golden.py [--c1]

Every array stored below is an output of /root/reference/pkg/src/headfem run
unmodified; the fixtures pin both the oracle restatement (oracle/) and the
CUDA path.  `--c1` additionally builds the full C1 configuration of
BASELINE.json (3-layer sphere, ~55k nodes, 32 electrodes, 1k sources), which
takes a few minutes.
"""
from __future__ import annotations

import argparse
import hashlib
import os
import sys
import time

import numpy as np
import scipy.sparse as sp

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def csr_parts(prefix, M):
    M = sp.csr_matrix(M)
    return {f"{prefix}_indptr": M.indptr.astype(np.int32), f"{prefix}_indices": M.indices.astype(np.int32),
            f"{prefix}_data": M.data, f"{prefix}_shape": np.array(M.shape)}


def solver_cases(hf):
    from headfem.errors import ConvergenceError
    from headfem.solver import PcgConfig, pcg_solve, transfer_matrix

    def random_spd(n, seed, cond=100.0):  # the reference tests' fixture recipe
        rng = np.random.default_rng(seed)
        Q, _ = np.linalg.qr(rng.normal(size=(n, n)))
        lam = np.geomspace(1.0, cond, n)
        return Q @ np.diag(lam) @ Q.T

    out = {}
    cases = [("dense50", 50, 42, 100.0, 1, 1e-10, None, "ldp"),
             ("bound40s0", 40, 0, 10.0, 0, 1e-10, None, "ldp"),
             ("bound40s1", 40, 1, 10.0, 1, 1e-10, None, "ldp"),
             ("bound40s2", 40, 2, 10.0, 2, 1e-10, None, "ldp"),
             ("none60", 60, 9, 100.0, 9, 1e-10, None, "none"),
             ("ldp60", 60, 9, 100.0, 9, 1e-10, None, "ldp")]
    for name, n, seed, cond, bseed, tol, mi, pre in cases:
        A = random_spd(n, seed, cond)
        b = np.random.default_rng(bseed).normal(size=n)
        x, it, res = pcg_solve(sp.csr_matrix(A), b, PcgConfig(tolerance=tol, max_iterations=mi,
                                                               preconditioner=pre))
        out[f"{name}_A"] = A
        out[f"{name}_b"] = b
        out[f"{name}_x"] = x
        out[f"{name}_meta"] = np.array([it, res, tol, -1 if mi is None else mi,
                                        1 if pre == "ldp" else 0])
    # best-iterate failure (test_solver.py:62-70)
    A = random_spd(30, 3, 1e4)
    try:
        pcg_solve(sp.csr_matrix(A), np.ones(30), PcgConfig(tolerance=1e-14, max_iterations=3))
        raise SystemExit("expected ConvergenceError")
    except ConvergenceError as e:
        out["fail30_A"] = A
        out["fail30_best_x"] = e.best_x
        out["fail30_meta"] = np.array([e.residual, e.iterations])
    # multi-column transfer with a zero column
    A = random_spd(40, 5)
    B = sp.random(40, 5, density=0.4, random_state=5, format="csr").toarray()
    B[:, 2] = 0.0
    T = transfer_matrix(sp.csr_matrix(A), B, PcgConfig(tolerance=1e-9))
    out["tm40_A"], out["tm40_B"], out["tm40_T"] = A, B, T
    return out


def system_fixture(mesh, el, src, tol=1e-8, eit=None, store_A=True, store_T=True):
    from headfem.fem import assemble_cem_system
    from headfem.leadfield import eeg_leadfield, eit_leadfield, electrode_response
    from headfem.solver import PcgConfig, pcg_solve

    t0 = time.time()
    sysm = assemble_cem_system(mesh, el, src)
    t_asm = time.time() - t0
    cfg = PcgConfig(tolerance=tol)
    out = {"nodes": mesh.nodes, "tetra": mesh.tetra.astype(np.int32),
           "labels": mesh.labels.astype(np.int32), "sigma": mesh.sigma,
           "tri_ptr": np.cumsum([0] + [len(t) for t in el.triangle_ids]).astype(np.int64),
           "tri_ids": np.concatenate(el.triangle_ids).astype(np.int64),
           "impedances": el.impedances, "ground": np.array(sysm.ground),
           "A_sha_indptr": np.array(sha(sysm.A.indptr.astype(np.int32))),
           "A_sha_indices": np.array(sha(sysm.A.indices.astype(np.int32))),
           "A_nnz": np.array(sysm.A.nnz), "tol": np.array(tol),
           "t_assemble": np.array(t_asm)}
    bf, owners = mesh.boundary_triangles()
    out["bfaces_sha"] = np.array(sha(bf.astype(np.int64)))
    out["bowners_sha"] = np.array(sha(owners.astype(np.int64)))
    out["n_bfaces"] = np.array(len(bf))
    if store_A:
        out.update(csr_parts("A", sysm.A))
        out["bfaces"] = bf.astype(np.int32)
        out["bowners"] = owners.astype(np.int32)
        K = __import__("headfem.fem", fromlist=["volume_stiffness"]).volume_stiffness(mesh)
        out.update(csr_parts("K", K))
    out.update(csr_parts("B", sysm.B))
    out["Cdiag"] = sysm.C.diagonal()
    if src is not None:
        out.update(csr_parts("G", sysm.G))
        out["src_elements"] = np.asarray(src.element_ids, dtype=np.int64)
        out["src_positions"] = src.positions
    # per-column iteration counts through the reference's own pcg_solve
    Bc = sysm.B.tocsc()
    its = []
    t0 = time.time()
    for l in range(sysm.B.shape[1]):
        _, it, _ = pcg_solve(sysm.A, Bc[:, [l]].toarray().ravel(), cfg)
        its.append(it)
    out["iters"] = np.array(its)
    out["t_pcg_columns"] = np.array(time.time() - t0)
    T, M = electrode_response(sysm, cfg)
    out["M"] = M
    if store_T:
        out["T"] = T
    if src is not None:
        t0 = time.time()
        lf = eeg_leadfield(sysm, cfg)
        out["t_eeg_leadfield"] = np.array(time.time() - t0)
        out["LF"] = lf.matrix
        lf12 = eeg_leadfield(sysm, PcgConfig(tolerance=1e-12))
        out["LF_tol12"] = lf12.matrix
    if eit is not None:
        dofs, I = eit
        lf = eit_leadfield(sysm, dofs, I, cfg)
        out["eit_currents"] = I
        out["eit_dof_ptr"] = np.cumsum([0] + [len(e) for e in dofs.element_sets]).astype(np.int64)
        out["eit_dof_elems"] = np.concatenate(dofs.element_sets).astype(np.int64)
        out["eit_centers"] = dofs.centers
        out["eit_LF"] = lf.matrix
        out["eit_bg"] = lf.background_data
    return out


def sphere_small():
    from headfem.fem import ElectrodeSet
    from headfem.geometry import Compartment, Segmentation, icosphere
    from headfem.leadfield import adjacent_pair_patterns, build_dof_map
    from headfem.meshgen import generate_mesh, place_sources
    from headfem.simulate import fibonacci_sphere_points

    seg = Segmentation([Compartment(icosphere(0.1, 2), 0.33, active=True)])
    mesh = generate_mesh(seg, 0.045)
    el = ElectrodeSet.from_centers(mesh, fibonacci_sphere_points(6, 0.1), radius=0.05, impedances=1e3)
    src = place_sources(mesh, seg, 4, mode="unconstrained", seed=0)
    dofs = build_dof_map(mesh, [0], n_dofs=4, seed=1)
    I = adjacent_pair_patterns(6)[:, :3]
    out = system_fixture(mesh, el, src, tol=1e-12, eit=(dofs, I))
    out["dofmap_seed"] = np.array(1)
    return out


def layered(h, n_el, n_src, radius=0.014, eit=True, tensor=False, tol=1e-8):
    from headfem.experiments import layered_sphere_segmentation
    from headfem.fem import ElectrodeSet
    from headfem.leadfield import adjacent_pair_patterns, build_dof_map
    from headfem.meshgen import generate_mesh, place_sources
    from headfem.simulate import fibonacci_sphere_points

    seg = layered_sphere_segmentation((0.079, 0.086, 0.092), (0.33, 0.0064, 0.43), (2, 0, 3), (0,), 3)
    mesh = generate_mesh(seg, h)
    if tensor:
        rng = np.random.default_rng(3)
        s = np.zeros((mesh.n_elements, 6))
        s[:, :3] = mesh.sigma[:, None] * rng.uniform(0.8, 1.2, (mesh.n_elements, 3))
        s[:, 3] = 0.1 * mesh.sigma * rng.uniform(-1, 1, mesh.n_elements)
        mesh = mesh.with_sigma(s)
    el = ElectrodeSet.from_centers(mesh, fibonacci_sphere_points(n_el, 0.092), radius=radius,
                                   impedances=1e3)
    src = place_sources(mesh, seg, n_src, mode="unconstrained", seed=1)
    e = None
    if eit:
        dofs = build_dof_map(mesh, [0, 1], n_dofs=20, seed=2)
        e = (dofs, adjacent_pair_patterns(n_el)[:, :4])
    return system_fixture(mesh, el, src, tol=tol, eit=e)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c1", action="store_true")
    args = ap.parse_args()
    sys.path.insert(0, REF)
    import headfem as hf

    np.savez_compressed(os.path.join(OUT, "solver_cases.npz"), **solver_cases(hf))
    print("solver_cases ok")
    np.savez_compressed(os.path.join(OUT, "sphere_small.npz"), **sphere_small())
    print("sphere_small ok")
    np.savez_compressed(os.path.join(OUT, "layered_h12.npz"), **layered(0.012, 16, 200))
    print("layered_h12 ok")
    np.savez_compressed(os.path.join(OUT, "layered_h14_tensor.npz"),
                        **layered(0.014, 8, 50, radius=0.02, eit=False, tensor=True))
    print("layered_h14_tensor ok")
    if args.c1:
        t0 = time.time()
        d = layered(0.004, 32, 1000, eit=False)
        for k in ("A_indptr", "A_indices", "A_data", "A_shape", "K_indptr", "K_indices", "K_data",
                  "K_shape", "T", "bfaces", "bowners", "LF_tol12"):
            d.pop(k, None)
        np.savez_compressed(os.path.join(OUT, "c1.npz"), **d)
        print(f"c1 ok ({time.time() - t0:.1f}s)")


if __name__ == "__main__":
    main()
