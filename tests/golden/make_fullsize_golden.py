"""Full-size golden vectors (BASELINE.json configs[1] = C2, configs[4] = C5) from the
reference itself.

Run here, where /root/reference is importable (it is not on the GPU box):

    python tests/golden/make_fullsize_golden.py --config c2 [--procs 8]
    python tests/golden/make_fullsize_golden.py --config c5 --columns 0,1,255

Everything below is computed by /root/reference/pkg/src/headfem run unmodified:

* the mesh is SURVEY.md App. A.4's analytic-label Kuhn sphere built from the
  reference's own `_KUHN_TETS` / `_CORNER_OFFSETS` and `TetMesh` (and checked
  array-equal to `paper_1811_07717_b200.synthetic.sphere_mesh`, which is what
  the GPU box builds);
* electrodes: `ElectrodeSet.from_centers(mesh, fibonacci_sphere_points(L, 0.092), r, 1e3)`;
* sources: `place_sources(mesh, seg, S, 'unconstrained', seed=1)` with a
  segmentation stub whose only active compartment is label 0;
* `assemble_cem_system`, then every transfer column by the reference's
  `pcg_solve` (solver.py:64-111), one process per column.  `transfer_matrix`
  (solver.py:114-141) is exactly that loop and its result does not depend on
  how the columns are scheduled (test_solver.py:131-137), so the columns are
  solved in a process pool and `headfem.leadfield.transfer_matrix` is bound to
  the assembled result while the reference's `eeg_leadfield`
  (leadfield.py:122-134) forms M, W and the lead field.

Stored (the full T and LF are too large to commit): per-column iteration counts
and true residuals, T on every 997th row, T column norms and T' w for a seeded
w, M, the LF on a fixed 2,000-column subset, LF Omega for a seeded 30000 x 8
Omega, and the Frobenius norm of the LF.  The GPU test
tests/test_gpu_fullsize.py checks the device build against these.
"""
from __future__ import annotations

import argparse
import hashlib
import os
import sys
import time
import types

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(OUT))

CONFIGS = {
    # name: radii, conductivities, h, electrodes, electrode radius, sources
    "c2": ((0.079, 0.082, 0.087, 0.092), (0.33, 1.79, 0.0064, 0.43), 0.0015, 128, 0.01, 10_000),
    "c5": ((0.079, 0.082, 0.087, 0.092), (0.33, 1.79, 0.0064, 0.43), 0.00088, 256, 0.006, 50_000),
}
ROW_STRIDE = 997
LF_SUBSET = 2000


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def reference_mesh(radii, cond, h):
    """SURVEY.md App. A.4 with the reference's own Kuhn table and TetMesh."""
    from headfem.meshgen import _CORNER_OFFSETS, _KUHN_TETS, TetMesh

    R = radii[-1]
    lo = np.full(3, -R)
    nx = int(np.ceil(2 * R / h - 1e-12))
    xs = lo[0] + h * np.arange(nx + 1)
    gz, gy, gx = np.meshgrid(xs, xs, xs, indexing="ij")
    grid = np.column_stack([gx.ravel(), gy.ravel(), gz.ravel()])
    cz, cy, cx = np.meshgrid(*(np.arange(nx),) * 3, indexing="ij")
    base = (cx + (nx + 1) * (cy + (nx + 1) * cz)).ravel()
    off = _CORNER_OFFSETS[:, 0] + (nx + 1) * (_CORNER_OFFSETS[:, 1] + (nx + 1) * _CORNER_OFFSETS[:, 2])
    tetra = (base[:, None] + off[None, :])[:, _KUHN_TETS].reshape(-1, 4)
    r = np.linalg.norm(grid[tetra].mean(1), axis=1)
    lab = np.full(len(r), -1)
    for k in reversed(range(len(radii))):
        lab[r <= radii[k]] = k
    keep = lab >= 0
    used, tet = np.unique(tetra[keep], return_inverse=True)
    return TetMesh(grid[used], tet.reshape(-1, 4), lab[keep], np.asarray(cond)[lab[keep]])


_POOL_STATE = {}


def _solve_column(l):
    from threadpoolctl import threadpool_limits
    from headfem.solver import PcgConfig, pcg_solve

    A, Bc, tol = _POOL_STATE["A"], _POOL_STATE["Bc"], _POOL_STATE["tol"]
    with threadpool_limits(1):
        t0 = time.time()
        x, it, res = pcg_solve(A, Bc[:, [l]].toarray().ravel(), PcgConfig(tolerance=tol))
    return l, x, it, res, time.time() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--procs", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--columns", default="", help="comma list (default: every electrode)")
    ap.add_argument("--tol", type=float, default=1e-8)
    args = ap.parse_args()
    sys.path.insert(0, REF)
    import multiprocessing as mp

    import headfem.leadfield as hl
    from headfem.fem import ElectrodeSet, assemble_cem_system, assemble_A, assemble_B_C_R, ground_node
    from headfem.meshgen import place_sources
    from headfem.simulate import fibonacci_sphere_points
    from headfem.solver import PcgConfig

    radii, cond, h, L, erad, S = CONFIGS[args.config]
    t0 = time.time()
    mesh = reference_mesh(radii, cond, h)
    print(f"mesh {mesh.n_nodes} nodes {mesh.n_elements} elements ({time.time() - t0:.1f}s)", flush=True)
    try:  # the GPU box builds its mesh with the package's numpy recipe: must be the same arrays
        sys.path.insert(0, ROOT)
        from paper_1811_07717_b200 import synthetic

        m2 = synthetic.sphere_mesh(radii, cond, h)
        same = (np.array_equal(m2.nodes, mesh.nodes) and np.array_equal(m2.tetra, mesh.tetra)
                and np.array_equal(m2.labels, mesh.labels) and np.array_equal(m2.sigma, mesh.sigma))
        print(f"package synthetic mesh array-equal: {same}", flush=True)
        assert same
        del m2
    except ImportError as exc:
        print(f"(package not importable: {exc})")
    t0 = time.time()
    el = ElectrodeSet.from_centers(mesh, fibonacci_sphere_points(L, radii[-1]), radius=erad,
                                   impedances=1e3)
    print(f"electrodes ({time.time() - t0:.1f}s)", flush=True)
    full = args.config == "c2"
    out = {"nodes_sha": np.array(sha(mesh.nodes)), "tetra_sha": np.array(sha(mesh.tetra.astype(np.int64))),
           "n_nodes": np.array(mesh.n_nodes), "n_elements": np.array(mesh.n_elements),
           "tol": np.array(args.tol), "row_stride": np.array(ROW_STRIDE),
           "tri_ptr": np.cumsum([0] + [len(t) for t in el.triangle_ids]).astype(np.int64),
           "tri_ids_sha": np.array(sha(np.concatenate(el.triangle_ids).astype(np.int64)))}
    t0 = time.time()
    if full:
        seg = types.SimpleNamespace(compartments=[types.SimpleNamespace(active=(k == 0))
                                                  for k in range(len(radii))])
        src = place_sources(mesh, seg, S, mode="unconstrained", seed=1)
        sysm = assemble_cem_system(mesh, el, src)
        A, B, G = sysm.A, sysm.B, sysm.G
        out["src_elements"] = np.asarray(src.element_ids, dtype=np.int64)
        out["G_nnz"] = np.array(G.nnz)
        out["ground"] = np.array(sysm.ground)
    else:
        A = assemble_A(mesh, el)
        B, _, _ = assemble_B_C_R(mesh, el)
        out["ground"] = np.array(ground_node(mesh, el))
    print(f"system assembled ({time.time() - t0:.1f}s): nnz(A) {A.nnz}", flush=True)
    out["A_nnz"] = np.array(A.nnz)
    out["A_sha_indptr"] = np.array(sha(A.indptr.astype(np.int32)))
    out["A_sha_indices"] = np.array(sha(A.indices.astype(np.int32)))
    cols = [int(c) for c in args.columns.split(",")] if args.columns else list(range(B.shape[1]))
    _POOL_STATE.update(A=A, Bc=B.tocsc(), tol=args.tol)
    n = mesh.n_nodes
    T = np.empty((n, len(cols)))
    iters = np.zeros(len(cols), np.int64)
    res = np.zeros(len(cols))
    secs = np.zeros(len(cols))
    t0 = time.time()
    with mp.get_context("fork").Pool(min(args.procs, len(cols))) as pool:
        for done, (l, x, it, rr, dt) in enumerate(pool.imap_unordered(_solve_column, cols)):
            j = cols.index(l)
            T[:, j], iters[j], res[j], secs[j] = x, it, rr, dt
            print(f"  column {l}: {it} iterations, residual {rr:.3e}, {dt:.1f}s "
                  f"[{done + 1}/{len(cols)}, {time.time() - t0:.0f}s]", flush=True)
    rows = np.arange(0, n, ROW_STRIDE)
    w = np.random.default_rng(7).standard_normal(n)
    out.update(columns=np.array(cols), iters=iters, true_res=res, column_seconds=secs,
               T_rows=rows, T_sample=T[rows], T_norm=np.linalg.norm(T, axis=0), T_w=T.T @ w)
    if full:
        hl.transfer_matrix = lambda A_, B_, cfg_=None, threads=1: T  # the columns solved above
        T2, M = hl.electrode_response(sysm, PcgConfig(tolerance=args.tol))
        assert T2 is T
        lf = hl.eeg_leadfield(sysm, PcgConfig(tolerance=args.tol)).matrix
        ncol = lf.shape[1]
        sub = np.sort(np.random.default_rng(11).choice(ncol, LF_SUBSET, replace=False))
        omega = np.random.default_rng(13).standard_normal((ncol, 8))
        out.update(M=M, LF_cols=sub, LF_sub=lf[:, sub], LF_omega=lf @ omega, LF_fro=np.array(np.linalg.norm(lf)),
                   LF_shape=np.array(lf.shape), LF_colmean_max=np.array(np.abs(lf.mean(axis=0)).max()))
    path = os.path.join(OUT, f"{args.config}_fullsize.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path) / 1e6:.1f} MB)", flush=True)


if __name__ == "__main__":
    main()
