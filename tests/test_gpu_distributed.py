"""The sharded build on the device.

* NCCL with world_size 1 (one GPU per process is all a gpurun box offers);
* world_size 2 and 3 over gloo with every rank a separate process running its
  CUDA stages (assembly, PCG of its electrode block, response block, partial
  lead field, EIT pattern solves and sensitivities) on cuda:0 — the collectives
  stage through the host, the kernels are the product's.  The transfer columns
  must be bit-identical to the one-process build (canonical reductions), the
  lead field equal to rounding, and a convergence failure must surface as the
  same ConvergenceError on every rank;
* a 3-way split evaluated rank by rank in one process."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    from paper_1811_07717_b200 import synthetic

    return synthetic.eeg_problem("c1", h=0.006, n_electrodes=12, n_sources=200)


def test_nccl_world1_matches_single_process(cuda):
    import torch
    import torch.distributed as dist

    from paper_1811_07717_b200.distributed import sharded_leadfield
    from paper_1811_07717_b200.engine import EegEngine
    from paper_1811_07717_b200.solver import PcgConfig

    prob = _problem()
    cfg = PcgConfig(1e-10)
    ref = EegEngine(prob.mesh, prob.electrodes, prob.G, cfg).build(to_host=True)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        eng = EegEngine(prob.mesh, prob.electrodes, prob.G, cfg, columns=(0, prob.electrodes.count))
        lf = sharded_leadfield(eng, 1, 0).cpu().numpy()
    finally:
        dist.destroy_process_group()
    np.testing.assert_array_equal(lf, ref)


def test_column_blocks_reassemble_the_leadfield(cuda):
    """Rank-by-rank stages of a 3-way split (collectives replaced by host
    concatenation / summation) equal the one-rank build to rounding, and the
    transfer columns are bit-identical."""
    from paper_1811_07717_b200.engine import EegEngine, column_blocks
    from paper_1811_07717_b200.leadfield import response_operator, symmetrize
    from paper_1811_07717_b200.solver import PcgConfig

    prob = _problem()
    cfg = PcgConfig(1e-10)
    full = EegEngine(prob.mesh, prob.electrodes, prob.G, cfg)
    A = full.assemble()
    T_full = full.solve(A).cpu().numpy()
    ref = full.build(to_host=True)
    L = prob.electrodes.count
    engines = [EegEngine(prob.mesh, prob.electrodes, prob.G, cfg, columns=b)
               for b in column_blocks(L, 3)]
    Ts, Ms = [], []
    for e in engines:
        T = e.solve(e.assemble())
        Ts.append(T)
        Ms.append(e.response_block(T).cpu().numpy())
    Tcat = np.concatenate([t.cpu().numpy() for t in Ts], axis=1)
    # canonical reductions: a column's bits do not depend on its block (kp 4 vs 16)
    np.testing.assert_array_equal(Tcat, T_full)
    W = response_operator(symmetrize(np.concatenate(Ms, axis=1)), full.R)
    lf = sum(e.lf_partial(T, W).cpu().numpy() for e, T in zip(engines, Ts))
    assert np.linalg.norm(lf - ref) / np.linalg.norm(ref) < 1e-10


def test_eit_nccl_world1_and_rank_split_match_reference(cuda):
    """sharded_eit_leadfield through NCCL (world 1) and a 3-way electrode/pattern
    split evaluated rank by rank both reproduce the reference's EIT Jacobian."""
    import torch
    import torch.distributed as dist

    from paper_1811_07717_b200.distributed import sharded_eit_leadfield
    from paper_1811_07717_b200.engine import EegEngine, column_blocks
    from paper_1811_07717_b200.leadfield import (EitDofMap, _solve_response, response_operator,
                                                 symmetrize)
    from paper_1811_07717_b200.solver import PcgConfig
    from tests.fixtures import electrodes_from_fixture, load, mesh_from_fixture

    fx = load("layered_h12.npz")
    mesh = mesh_from_fixture(fx)
    el = electrodes_from_fixture(mesh, fx)
    cfg = PcgConfig(float(fx["tol"]))
    dofs = EitDofMap(element_sets=tuple(np.split(fx["eit_dof_elems"], fx["eit_dof_ptr"][1:-1])),
                     centers=fx["eit_centers"])
    I = fx["eit_currents"]
    ref = fx["eit_LF"]
    rel = lambda a: np.linalg.norm(a - ref) / np.linalg.norm(ref)  # noqa: E731
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        lf = sharded_eit_leadfield(EegEngine(mesh, el, None, cfg), dofs, I, 1, 0)
    finally:
        dist.destroy_process_group()
    assert rel(lf.matrix) <= 1e-6
    np.testing.assert_allclose(lf.background_data, fx["eit_bg"], rtol=1e-8, atol=1e-14)
    # 3 ranks by hand: T blocks, M from the blocks, U blocks, summed partial Jacobians
    L, P = el.count, I.shape[1]
    engs = [EegEngine(mesh, el, None, cfg, columns=b) for b in column_blocks(L, 3)]
    A = engs[0].assemble()
    Ts = [e.solve(A) for e in engs]
    M = symmetrize(torch.cat([e.response_block(T) for e, T in zip(engs, Ts)], 1).cpu().numpy())
    W = response_operator(M, engs[0].R)
    V = _solve_response(M, I)
    U = torch.cat([engs[0].solve_rhs(A, engs[0].B @ V[:, p0:p1])
                   for p0, p1 in column_blocks(P, 3)], 1)
    cols = sum(e.eit_partial(dofs, T, U, W) for e, T in zip(engs, Ts)).cpu().numpy()
    assert rel(cols) <= 1e-6


def _cuda_worker(rank, world, port, out, kind, max_iter):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    from paper_1811_07717_b200.distributed import sharded_eit_leadfield, sharded_leadfield
    from paper_1811_07717_b200.engine import EegEngine, column_blocks
    from paper_1811_07717_b200.errors import ConvergenceError
    from paper_1811_07717_b200.leadfield import EitDofMap
    from paper_1811_07717_b200.solver import PcgConfig
    from tests.fixtures import electrodes_from_fixture, load, mesh_from_fixture

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if kind == "eeg":
            prob = _problem()
            cfg = PcgConfig(1e-10, max_iterations=max_iter)
            blocks = column_blocks(prob.electrodes.count, world)
            eng = EegEngine(prob.mesh, prob.electrodes, prob.G, cfg, columns=blocks[rank])
            try:
                lf = sharded_leadfield(eng, world, rank)
            except ConvergenceError as exc:
                np.savez(f"{out}_err{rank}.npz", column=exc.column, best=exc.best_x,
                         res=exc.residual, it=exc.iterations)
                return
            np.save(f"{out}_T{rank}.npy", eng.solve(eng.assemble()).cpu().numpy())
            if rank == 0:
                np.save(f"{out}_lf.npy", lf.cpu().numpy())
        else:
            fx = load("layered_h12.npz")
            mesh = mesh_from_fixture(fx)
            el = electrodes_from_fixture(mesh, fx)
            cfg = PcgConfig(float(fx["tol"]))
            dofs = EitDofMap(element_sets=tuple(np.split(fx["eit_dof_elems"], fx["eit_dof_ptr"][1:-1])),
                             centers=fx["eit_centers"])
            eng = EegEngine(mesh, el, None, cfg, columns=column_blocks(el.count, world)[rank])
            lf = sharded_eit_leadfield(eng, dofs, fx["eit_currents"], world, rank)
            if rank == 0:
                np.savez(f"{out}_eit.npz", m=lf.matrix, bg=lf.background_data)
    finally:
        dist.destroy_process_group()


def _spawn(world, tmp_path, kind, max_iter=None):
    import torch.multiprocessing as mp

    out = str(tmp_path / "r")
    mp.spawn(_cuda_worker, args=(world, _free_port(), out, kind, max_iter), nprocs=world, join=True)
    return out


@pytest.mark.parametrize("world", [2, 3])
def test_multirank_cuda_eeg_matches_single_process(cuda, tmp_path, world):
    from paper_1811_07717_b200.engine import EegEngine
    from paper_1811_07717_b200.solver import PcgConfig

    prob = _problem()
    cfg = PcgConfig(1e-10)
    full = EegEngine(prob.mesh, prob.electrodes, prob.G, cfg)
    T_full = full.solve(full.assemble()).cpu().numpy()
    ref = full.build(to_host=True)
    out = _spawn(world, tmp_path, "eeg")
    Tcat = np.concatenate([np.load(f"{out}_T{r}.npy") for r in range(world)], axis=1)
    np.testing.assert_array_equal(Tcat, T_full)
    lf = np.load(f"{out}_lf.npy")
    assert lf.shape == ref.shape
    assert np.linalg.norm(lf - ref) / np.linalg.norm(ref) < 1e-12


@pytest.mark.parametrize("world", [2, 3])
def test_multirank_cuda_eit_matches_reference(cuda, tmp_path, world):
    from tests.fixtures import load

    fx = load("layered_h12.npz")
    out = _spawn(world, tmp_path, "eit")
    got = np.load(f"{out}_eit.npz")
    ref = fx["eit_LF"]
    assert got["m"].shape == ref.shape
    assert np.linalg.norm(got["m"] - ref) / np.linalg.norm(ref) <= 1e-6
    np.testing.assert_allclose(got["bg"], fx["eit_bg"], rtol=1e-8, atol=1e-14)


def test_multirank_convergence_error_is_raised_on_every_rank(cuda, tmp_path):
    """max_iterations too small: every rank raises the same ConvergenceError (first
    failing global column, its best iterate) before any collective can hang."""
    from paper_1811_07717_b200.engine import EegEngine
    from paper_1811_07717_b200.errors import ConvergenceError
    from paper_1811_07717_b200.solver import PcgConfig

    prob = _problem()
    with pytest.raises(ConvergenceError) as exc:
        EegEngine(prob.mesh, prob.electrodes, prob.G, PcgConfig(1e-10, max_iterations=5)).build()
    out = _spawn(2, tmp_path, "eeg", max_iter=5)
    errs = [np.load(f"{out}_err{r}.npz") for r in range(2)]
    for e in errs:
        assert int(e["column"]) == exc.value.column == 0
        assert int(e["it"]) == 5
        np.testing.assert_array_equal(e["best"], exc.value.best_x)
