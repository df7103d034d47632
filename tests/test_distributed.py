"""Multi-rank electrode sharding (distributed.sharded_leadfield) on CPU with
gloo, world_size 2 and 3.  The per-rank stages are the oracle's CPU
restatements (the GPU engine exposes the same stage methods), so this checks
the orchestration: block split, M all-gather + symmetrisation, W, partial LF
sum-reduce — against the reference's golden lead field."""
import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp
import torch
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleEngine:
    """CPU stand-in for engine.EegEngine with the same stage API."""

    def __init__(self, fx, columns):
        import oracle
        from tests.fixtures import csr

        self.oracle = oracle
        self.A, self.B, self.G = csr(fx, "A"), csr(fx, "B"), csr(fx, "G")
        self.L = self.B.shape[1]
        self.R = np.eye(self.L) - np.full((self.L, self.L), 1.0 / self.L)
        self.Cdiag = fx["Cdiag"]
        self.c0, self.c1 = columns
        self.cfg = oracle.PcgSettings(tolerance=float(fx["tol"]))
        from tests.fixtures import mesh_from_fixture

        self.mesh = mesh_from_fixture(fx)
        self.ground = int(fx["ground"])

    def assemble(self):
        return self.A

    def solve(self, A):
        return torch.from_numpy(self.oracle.transfer_matrix(A, self.B[:, self.c0:self.c1], self.cfg))

    def response_block(self, T):
        Tn = T.numpy()
        C = np.zeros((self.L, self.c1 - self.c0))
        for j in range(self.c0, self.c1):
            C[j, j - self.c0] = self.Cdiag[j]
        return torch.from_numpy(C - self.B.T @ Tn)

    def lf_partial(self, T, W):
        TtG = np.asarray((self.G.T @ T.numpy()).T)
        return torch.from_numpy(W[:, self.c0:self.c1] @ TtG)

    # EIT stages (distributed.sharded_eit_leadfield)
    def solve_rhs(self, A, rhs):
        return torch.from_numpy(self.oracle.transfer_matrix(A, sp.csc_matrix(rhs), self.cfg))

    def eit_partial(self, dofs, T, U, W):
        Q = self.oracle.dof_sensitivities(self.mesh.nodes, self.mesh.tetra, dofs.element_sets,
                                          self.ground, U.numpy(), T.numpy())
        Wb = W[:, self.c0:self.c1]
        return torch.from_numpy(np.concatenate([Wb @ Q[p].T for p in range(Q.shape[0])]))


def _worker(rank, world, port, name, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_1811_07717_b200.distributed import sharded_leadfield
    from paper_1811_07717_b200.engine import column_blocks
    from tests.fixtures import load

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fx = load(name)
        L = fx["B_shape"][1]
        eng = OracleEngine(fx, column_blocks(int(L), world)[rank])
        lf = sharded_leadfield(eng, world, rank)
        if rank == 0:
            np.save(out, lf.numpy())
        else:
            assert lf is None
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_leadfield_gloo(tmp_path, world):
    from tests.fixtures import load

    name = "layered_h12.npz"
    out = str(tmp_path / "lf.npy")
    mp.spawn(_worker, args=(world, _free_port(), name, out), nprocs=world, join=True)
    lf = np.load(out)
    ref = load(name)["LF"]
    assert np.linalg.norm(lf - ref) / np.linalg.norm(ref) <= 1e-6
    assert lf.shape == ref.shape
    _ = sp


def _eit_worker(rank, world, port, name, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_1811_07717_b200.distributed import sharded_eit_leadfield
    from paper_1811_07717_b200.engine import column_blocks
    from paper_1811_07717_b200.leadfield import EitDofMap
    from tests.fixtures import load

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fx = load(name)
        L = int(fx["B_shape"][1])
        eng = OracleEngine(fx, column_blocks(L, world)[rank])
        dofs = EitDofMap(element_sets=tuple(np.split(fx["eit_dof_elems"], fx["eit_dof_ptr"][1:-1])),
                         centers=fx["eit_centers"])
        lf = sharded_eit_leadfield(eng, dofs, fx["eit_currents"], world, rank)
        if rank == 0:
            np.savez(out, m=lf.matrix, bg=lf.background_data, p=lf.n_patterns)
        else:
            assert lf is None
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_eit_leadfield_gloo(tmp_path, world):
    """EIT over ranks: electrode-sharded T, pattern-sharded U + all-gather, summed Jacobian."""
    from tests.fixtures import load

    name = "layered_h12.npz"
    out = str(tmp_path / "eit.npz")
    mp.spawn(_eit_worker, args=(world, _free_port(), name, out), nprocs=world, join=True)
    got = np.load(out)
    fx = load(name)
    ref = fx["eit_LF"]
    assert got["m"].shape == ref.shape
    assert np.linalg.norm(got["m"] - ref) / np.linalg.norm(ref) <= 1e-6
    np.testing.assert_allclose(got["bg"], fx["eit_bg"], rtol=1e-8, atol=1e-14)
    assert int(got["p"]) == fx["eit_currents"].shape[1]


def _fail_worker(rank, world, port, out):
    """Rank 1 fails at its second column (global column 5); rank 0 converges."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_1811_07717_b200.distributed import sharded_leadfield
    from paper_1811_07717_b200.engine import column_blocks
    from paper_1811_07717_b200.errors import ConvergenceError

    class FailingEngine:
        L = 8

        def __init__(self, cols):
            self.c0, self.c1 = cols

        def assemble(self):
            return None

        def solve(self, A):
            if self.c0 == 4:
                exc = ConvergenceError("no convergence", best_x=np.arange(6.0) + 0.5, residual=0.25,
                                       iterations=17)
                exc.local_column = 1
                exc.column = self.c0 + 1
                raise exc
            return torch.zeros((6, self.c1 - self.c0), dtype=torch.float64)

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        eng = FailingEngine(column_blocks(8, world)[rank])
        try:
            sharded_leadfield(eng, world, rank)
            np.save(out + f"{rank}.npy", np.array([-1.0]))
        except ConvergenceError as exc:
            np.save(out + f"{rank}.npy", np.concatenate([[exc.column, exc.residual, exc.iterations], exc.best_x]))
    finally:
        dist.destroy_process_group()


def test_convergence_failure_raised_on_every_rank(tmp_path):
    """One rank's ConvergenceError surfaces on every rank, with the global column and
    the owner's best iterate, before any further collective (no rank hangs)."""
    out = str(tmp_path / "e")
    mp.spawn(_fail_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    for r in range(2):
        got = np.load(out + f"{r}.npy")
        np.testing.assert_array_equal(got, np.concatenate([[5.0, 0.25, 17.0], np.arange(6.0) + 0.5]))


def test_helmet_306_geometry():
    from paper_1811_07717_b200 import meg

    s = meg.helmet_306()
    assert s.n_sensors == 306 and s.kinds.count("mag") == 102
    assert s.kinds.count("grad1") == s.kinds.count("grad2") == 102
    np.testing.assert_allclose(np.linalg.norm(s.coils[:, 3:6], axis=1), 1.0)
    assert np.all(s.coils[:, 2] >= -0.02 - 1e-12)  # the cap
    grads = [i for i, k in enumerate(s.kinds) if k != "mag"]
    for i in grads:  # a planar gradiometer: two coils, opposite weights, 16.8 mm apart
        a, b = s.coil_ptr[i], s.coil_ptr[i + 1]
        assert b - a == 2 and s.coils[a, 6] == -s.coils[a + 1, 6]
        assert abs(np.linalg.norm(s.coils[a, :3] - s.coils[a + 1, :3]) - 0.0168) < 1e-12
