"""The sharded build's NCCL path on the device (world_size 1: one GPU per
process is all a gpurun box offers; the multi-rank orchestration itself is
covered by the gloo tests).  The NCCL result must equal the single-process
build, and a 2-way column split evaluated rank by rank (no collectives, one
process) must reproduce it to rounding."""
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
    # block solves differ from the full solve only through the batch width
    # (kp) of the reduction tree: equal to rounding, same iteration counts
    assert np.linalg.norm(Tcat - T_full) / np.linalg.norm(T_full) < 1e-12
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
