"""Parity of the CUDA LDP-PCG (hf_pcg_multi through the package API) with the
reference's golden outputs and the oracle (solver.py:50-141)."""
import numpy as np
import pytest
import scipy.sparse as sp

from tests.fixtures import load

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng(cuda):
    import paper_1811_07717_b200 as e

    return e


@pytest.fixture(scope="module")
def cases():
    return load("solver_cases.npz")


def random_spd(n, seed, cond=100.0):
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.normal(size=(n, n)))
    return Q @ np.diag(np.geomspace(1.0, cond, n)) @ Q.T


class TestLdp:
    def test_identity(self, eng):
        np.testing.assert_array_equal(eng.ldp(sp.eye(5, format="csr")), np.ones(5))

    def test_formula(self, eng):
        np.testing.assert_array_equal(eng.ldp(np.array([[2.0, -1.0], [-1.0, 2.0]])), [3.0, 3.0])

    def test_zero_row(self, eng):
        with pytest.raises(eng.SingularPreconditionerError):
            eng.ldp(sp.csr_matrix(np.array([[1.0, 0.0], [0.0, 0.0]])))

    def test_matches_oracle_on_mesh(self, eng):
        import oracle
        from tests.fixtures import csr

        A = csr(load("layered_h12.npz"), "A")
        # scipy's row sum and the kernel's sequential sum differ only in rounding
        np.testing.assert_allclose(eng.ldp(A), oracle.ldp(A), rtol=2e-15, atol=0)


class TestPcg:
    @pytest.mark.parametrize("name", ["dense50", "bound40s0", "bound40s1", "bound40s2", "none60",
                                      "ldp60"])
    def test_golden(self, eng, cases, name):
        A, b, x_ref = cases[f"{name}_A"], cases[f"{name}_b"], cases[f"{name}_x"]
        it_ref, res_ref, tol, mi, pre = cases[f"{name}_meta"]
        cfg = eng.PcgConfig(tolerance=tol, max_iterations=None if mi < 0 else int(mi),
                            preconditioner="ldp" if pre else "none")
        x, it, res = eng.pcg_solve(sp.csr_matrix(A), b, cfg)
        assert abs(it - it_ref) <= 1
        assert res <= tol
        # both are within tol of the solution; 1e-6 is far above their gap
        assert np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref) < 1e-6

    def test_identity_one_iteration(self, eng):
        b = np.array([3.0, -1.0, 2.0])
        x, it, res = eng.pcg_solve(sp.eye(3, format="csr"), b)
        np.testing.assert_allclose(x, b, rtol=1e-14)
        assert it == 1

    def test_two_by_two_closed_form(self, eng):
        A = sp.csr_matrix(np.array([[4.0, 1.0], [1.0, 3.0]]))
        x, _, _ = eng.pcg_solve(A, np.array([1.0, 2.0]), eng.PcgConfig(tolerance=1e-14))
        np.testing.assert_allclose(x, [1.0 / 11.0, 7.0 / 11.0], rtol=1e-12)

    def test_zero_rhs(self, eng):
        x, it, res = eng.pcg_solve(sp.eye(4, format="csr"), np.zeros(4))
        np.testing.assert_array_equal(x, 0.0)
        assert it == 0 and res == 0.0

    def test_best_iterate_matches_reference(self, eng, cases):
        A = cases["fail30_A"]
        with pytest.raises(eng.ConvergenceError) as exc:
            eng.pcg_solve(sp.csr_matrix(A), np.ones(30),
                          eng.PcgConfig(tolerance=1e-14, max_iterations=3))
        err = exc.value
        res_ref, it_ref = cases["fail30_meta"]
        assert err.iterations == 3 == it_ref
        assert err.residual <= 1.0
        assert abs(err.residual - res_ref) <= 1e-10 * res_ref
        np.testing.assert_allclose(err.best_x, cases["fail30_best_x"], rtol=1e-10, atol=1e-14)
        assert err.column is None

    def test_one_by_one(self, eng):
        x, it, res = eng.pcg_solve(sp.csr_matrix(np.array([[2.0]])), np.array([4.0]))
        np.testing.assert_allclose(x, [2.0], rtol=1e-15)
        assert it == 1 and res == 0.0

    def test_non_square_rejected(self, eng):
        with pytest.raises(eng.ParameterError):
            eng.pcg_solve(sp.csr_matrix(np.ones((3, 2))), np.ones(3))

    def test_singular_preconditioner_only_with_nonzero_rhs(self, eng):
        A = sp.csr_matrix(np.array([[1.0, 0.0], [0.0, 0.0]]))
        x, it, _ = eng.pcg_solve(A, np.zeros(2))      # b = 0 returns before ldp (solver.py:75-77)
        assert it == 0
        with pytest.raises(eng.SingularPreconditionerError):
            eng.pcg_solve(A, np.array([1.0, 0.0]))

    @pytest.mark.parametrize("n,k", [(3, 130), (5, 64), (17, 33)])
    def test_tiny_systems_many_columns(self, eng, n, k):
        A = sp.csr_matrix(random_spd(n, seed=n, cond=10.0))
        B = np.random.default_rng(k).normal(size=(n, k))
        T = eng.transfer_matrix(A, B, eng.PcgConfig(tolerance=1e-12))
        np.testing.assert_allclose(A @ T, B, rtol=0, atol=1e-10 * np.abs(B).max())

    def test_config_validation(self, eng):
        for kw in ({"tolerance": 0.0}, {"max_iterations": 0}, {"preconditioner": "amg"}):
            with pytest.raises(eng.ParameterError):
                eng.PcgConfig(**kw)


class TestTransferMatrix:
    def test_identity(self, eng):
        B = sp.random(20, 4, density=0.3, random_state=7, format="csr")
        T = eng.transfer_matrix(sp.eye(20, format="csr"), B)
        np.testing.assert_allclose(T, B.toarray(), atol=1e-12)

    def test_scaling(self, eng):
        B = sp.random(15, 3, density=0.5, random_state=2, format="csr")
        T = eng.transfer_matrix(2.0 * sp.eye(15, format="csr"), B, eng.PcgConfig(tolerance=1e-14))
        np.testing.assert_allclose(T, B.toarray() / 2.0, rtol=1e-12)

    def test_golden_with_zero_column(self, eng, cases):
        A, B, T_ref = cases["tm40_A"], cases["tm40_B"], cases["tm40_T"]
        T = eng.transfer_matrix(sp.csr_matrix(A), B, eng.PcgConfig(tolerance=1e-9))
        assert T.flags.c_contiguous and T.shape == (40, 5)
        np.testing.assert_array_equal(T[:, 2], 0.0)
        for l in range(5):
            if l == 2:
                continue
            assert np.linalg.norm(A @ T[:, l] - B[:, l]) / np.linalg.norm(B[:, l]) <= 1e-9
            assert np.linalg.norm(T[:, l] - T_ref[:, l]) / np.linalg.norm(T_ref[:, l]) < 1e-6

    def test_convergence_error_reports_column(self, eng):
        A = sp.csr_matrix(random_spd(25, seed=1, cond=1e6))
        B = sp.csr_matrix(np.ones((25, 2)))
        with pytest.raises(eng.ConvergenceError) as exc:
            eng.transfer_matrix(A, B, eng.PcgConfig(tolerance=1e-15, max_iterations=2))
        assert exc.value.column == 0

    def test_threads_do_not_change_result(self, eng):
        A = sp.csr_matrix(random_spd(30, seed=8))
        B = sp.random(30, 5, density=0.4, random_state=8, format="csr")
        np.testing.assert_array_equal(eng.transfer_matrix(A, B, threads=1),
                                      eng.transfer_matrix(A, B, threads=4))

    def test_batch_membership_does_not_change_columns(self, eng):
        """A column's iterates do not depend on the other columns of its batch."""
        from tests.fixtures import csr

        fx = load("layered_h12.npz")
        A, B = csr(fx, "A"), csr(fx, "B").toarray()
        T_all = eng.transfer_matrix(A, B)              # 16 columns -> kp = 16
        T_sub = eng.transfer_matrix(A, B[:, 2:13])     # 11 columns -> kp = 16
        np.testing.assert_array_equal(T_all[:, 3], T_sub[:, 1])
        B2 = B.copy()
        B2[:, 5] *= 3.0                                # another column changes, column 3 does not
        np.testing.assert_array_equal(T_all[:, 3], eng.transfer_matrix(A, B2)[:, 3])

    def test_batch_width_does_not_change_columns(self, eng):
        """Canonical reductions (pcg.cu header): a column's bits are the same at
        every SpMM width kp = 2..64, so T does not depend on how many columns a
        call, a batch or a rank holds (the multi-GPU analogue of the reference's
        test_threads_do_not_change_result, test_solver.py:131-137)."""
        from paper_1811_07717_b200.solver import operator, rhs_block, solve_block
        from tests.fixtures import csr

        fx = load("layered_h12.npz")
        A, B = csr(fx, "A"), csr(fx, "B").toarray()      # 16 electrodes
        B64 = np.concatenate([B] * 4, axis=1)            # kp = 64
        T64 = eng.transfer_matrix(A, B64)
        T16 = eng.transfer_matrix(A, B)                  # kp = 16
        np.testing.assert_array_equal(T64[:, :16], T16)
        np.testing.assert_array_equal(T64[:, 16:32], T16)
        T3 = eng.transfer_matrix(A, B[:, :3])            # kp = 4
        np.testing.assert_array_equal(T3, T16[:, :3])
        for kk, kp in ((7, 8), (20, 32)):
            Tk = eng.transfer_matrix(A, B64[:, :kk])
            np.testing.assert_array_equal(Tk, T64[:, :kk])
        x, it, res = eng.pcg_solve(A, B[:, 5])           # kp = 2
        np.testing.assert_array_equal(x, T16[:, 5])
        cfg = eng.PcgConfig()
        _, i64 = solve_block(operator(A, cfg), rhs_block(B64), cfg)
        _, i1 = solve_block(operator(A, cfg), rhs_block(B[:, 5:6]), cfg)
        assert i64.iterations[5] == i1.iterations[0] == it
        assert i64.true_residual[5] == i1.true_residual[0] == res

    def test_batch_width_does_not_change_best_iterate(self, eng):
        """The replayed best iterate of a failing column is the same at any width."""
        A = sp.csr_matrix(random_spd(60, seed=3, cond=1e8))
        B = np.random.default_rng(3).normal(size=(60, 40))
        cfg = eng.PcgConfig(tolerance=1e-15, max_iterations=13)
        got = []
        for k in (1, 3, 40):
            with pytest.raises(eng.ConvergenceError) as exc:
                eng.transfer_matrix(A, B[:, :k], cfg)
            got.append(exc.value)
        for e in got[1:]:
            np.testing.assert_array_equal(e.best_x, got[0].best_x)
            assert e.column == got[0].column == 0 and e.residual == got[0].residual

    def test_unattainable_tolerance_raises_convergence_error(self, eng):
        """tol below attainable accuracy: the recurrence residual keeps dropping
        under tol while the true residual stays above it, so the column advances
        one iteration per chunk; the solver must still end at max_iter with the
        reference's ConvergenceError (solver.py:108-111), not a control error."""
        A = sp.csr_matrix(np.array([[4.0, 1.0], [1.0, 3.0]]))
        cfg = eng.PcgConfig(tolerance=1e-17, max_iterations=40)
        with pytest.raises(eng.ConvergenceError) as exc:
            eng.pcg_solve(A, np.array([1.0, 2.0]), cfg)
        assert exc.value.iterations == 40
        assert exc.value.best_x.shape == (2,)

    @pytest.mark.parametrize("k", [1, 3, 16, 40, 70, 130])
    def test_widths(self, eng, k):
        """Every SpMM width (kp = 2..64, and the batch split) against the oracle."""
        import oracle
        from tests.fixtures import csr

        fx = load("layered_h14_tensor.npz")
        A = csr(fx, "A")
        rng = np.random.default_rng(k)
        B = rng.normal(size=(A.shape[0], k))
        B[fx["ground"]] = 0.0
        cfg = eng.PcgConfig(tolerance=1e-10)
        T = eng.transfer_matrix(A, B, cfg)
        for l in sorted({0, k // 2, k - 1}):
            x, it, _ = oracle.pcg_solve(A, B[:, l], oracle.PcgSettings(tolerance=1e-10))
            assert np.linalg.norm(T[:, l] - x) / np.linalg.norm(x) < 1e-7
            assert np.linalg.norm(A @ T[:, l] - B[:, l]) / np.linalg.norm(B[:, l]) <= 1e-10

    @pytest.mark.parametrize("k", [2, 8, 16, 32, 64])
    def test_ell_long_rows(self, eng, k):
        """The ELL SpMM on an SPD matrix whose rows hold 1..20 entries (rows of
        more than 8 take the flagged-slot + CSR path) against a direct solve."""
        import scipy.sparse.linalg as spla

        rng = np.random.default_rng(k)
        n = 3000
        rows, cols = [], []
        for i in range(n):
            m = int(rng.choice([0, 1, 2, 3, 6, 9, 19], p=[.05, .2, .3, .2, .1, .1, .05]))
            cc = rng.choice(n, size=m, replace=False)
            rows += [i] * m
            cols += list(cc)
        M = sp.coo_matrix((rng.uniform(-1, 1, len(rows)), (rows, cols)), shape=(n, n)).tocsr()
        M = M + M.T
        A = (M + sp.diags(np.asarray(abs(M).sum(axis=1)).ravel() + 1.0)).tocsr()
        lens = np.diff(A.indptr)
        assert lens.max() > 16 and (lens <= 8).any()
        B = rng.normal(size=(n, k))
        T = eng.transfer_matrix(A, B, eng.PcgConfig(tolerance=1e-12))
        ref = spla.splu(A.tocsc()).solve(B)
        assert np.linalg.norm(T - ref) / np.linalg.norm(ref) < 1e-10
        assert np.linalg.norm(A @ T - B) / np.linalg.norm(B) < 1e-11

    def test_iterations_match_reference_per_column(self, eng):
        from paper_1811_07717_b200.solver import operator, rhs_block, solve_block
        from tests.fixtures import csr

        fx = load("layered_h12.npz")
        cfg = eng.PcgConfig(tolerance=float(fx["tol"]))
        op = operator(csr(fx, "A"), cfg)
        _, info = solve_block(op, rhs_block(csr(fx, "B")), cfg)
        assert np.all(np.abs(info.iterations - fx["iters"]) <= 1), (info.iterations, fx["iters"])
        assert np.all(info.true_residual <= cfg.tolerance)

    @pytest.mark.parametrize("k", [3, 16, 40, 70])
    def test_deferred_x_matches_oracle(self, eng, k):
        """x deferred over the ring of XD p blocks, with columns converging
        mid-chunk and residual replacements (tol 1e-13), a zero column riding
        along: each column against the oracle's per-round x update."""
        import oracle
        from paper_1811_07717_b200.solver import operator, rhs_block, solve_block
        from tests.fixtures import csr

        fx = load("layered_h14_tensor.npz")
        A = csr(fx, "A")
        B = np.random.default_rng(10 + k).normal(size=(A.shape[0], k))
        B[fx["ground"]] = 0.0
        B[:, k // 2] = 0.0
        for tol in (1e-8, 1e-13):
            cfg = eng.PcgConfig(tolerance=tol)
            X, info = solve_block(operator(A, cfg), rhs_block(B), cfg)
            X = X.cpu().numpy()
            np.testing.assert_array_equal(X[:, k // 2], 0.0)
            assert info.iterations[k // 2] == 0
            for l in sorted({0, k - 1}):
                x, it, _ = oracle.pcg_solve(A, B[:, l], oracle.PcgSettings(tolerance=tol))
                assert abs(int(info.iterations[l]) - it) <= 1
                assert np.linalg.norm(X[:, l] - x) / np.linalg.norm(x) < 50 * tol
                assert info.true_residual[l] <= tol


class TestStream:
    """hf_pcg_stream (columns streamed through kp slots) against batch solves:
    every column's x and per-column results bit-identical."""

    @staticmethod
    def _solve(A, B, cfg, batch):
        from paper_1811_07717_b200.solver import operator, rhs_block, solve_block

        X, info = solve_block(operator(A, cfg), rhs_block(B), cfg, batch=batch)
        return X.cpu().numpy(), info

    @staticmethod
    def _same(a, b):
        Xa, ia = a
        Xb, ib = b
        np.testing.assert_array_equal(Xa, Xb)
        for f in ("iterations", "status", "true_residual", "best_residual", "best_iteration"):
            np.testing.assert_array_equal(getattr(ia, f), getattr(ib, f), err_msg=f)

    @pytest.mark.parametrize("slots", [2, 8, 32])
    def test_stream_equals_batch(self, eng, slots):
        from tests.fixtures import csr

        fx = load("layered_h14_tensor.npz")
        A = csr(fx, "A")
        rng = np.random.default_rng(slots)
        k = 45
        B = rng.normal(size=(A.shape[0], k)) * np.geomspace(1e-3, 1e3, k)
        B[:, ::7] *= rng.uniform(0, 1, size=(A.shape[0], 1)) ** 8   # harder columns
        B[fx["ground"]] = 0.0
        B[:, [0, 11, 44]] = 0.0                                      # zero columns, first and last
        cfg = eng.PcgConfig(tolerance=1e-10)
        ref = self._solve(A, B, cfg, 64)
        got = self._solve(A, B, cfg, slots)
        self._same(got, ref)
        assert (ref[1].status == eng._native.HF_COL_ZERO).sum() == 3

    def test_stream_failed_columns_replay_best_iterate(self, eng):
        from tests.fixtures import csr

        fx = load("layered_h14_tensor.npz")
        A = csr(fx, "A")
        rng = np.random.default_rng(5)
        B = rng.normal(size=(A.shape[0], 30))
        B[fx["ground"]] = 0.0
        full = self._solve(A, B, eng.PcgConfig(tolerance=1e-12), 64)[1].iterations
        cap = int(np.median(full))
        cfg = eng.PcgConfig(tolerance=1e-12, max_iterations=cap)
        ref = self._solve(A, B, cfg, 64)
        fails = (ref[1].status == eng._native.HF_COL_FAILED).sum()
        assert 0 < fails < 30
        self._same(self._solve(A, B, cfg, 4), ref)

    def test_stream_into_strided_output(self, eng):
        import torch

        from paper_1811_07717_b200.solver import operator, rhs_block, solve_block
        from tests.fixtures import csr

        fx = load("layered_h12.npz")
        A, B = csr(fx, "A"), csr(fx, "B").toarray()
        cfg = eng.PcgConfig(tolerance=1e-10)
        Bd = rhs_block(B)
        big = torch.full((Bd.shape[0], 2 * Bd.shape[1]), float("nan"), dtype=torch.float64, device=Bd.device)
        out = big[:, ::2]                                   # strided view
        X, _ = solve_block(operator(A, cfg), Bd, cfg, batch=4, out=out)
        assert X.data_ptr() == out.data_ptr()
        ref, _ = solve_block(operator(A, cfg), Bd, cfg, batch=64)
        assert torch.equal(out, ref) and torch.isnan(big[:, 1::2]).all()

    def test_stream_fewer_columns_than_slots(self, eng):
        from paper_1811_07717_b200.solver import _solve_streamed, operator, rhs_block, SolveInfo
        from tests.fixtures import csr

        fx = load("layered_h12.npz")
        A, B = csr(fx, "A"), csr(fx, "B").toarray()[:, :3]
        cfg = eng.PcgConfig(tolerance=1e-10)
        op = operator(A, cfg)
        Bd = rhs_block(B)
        n, k = Bd.shape
        mi = int(cfg.resolve_max_iterations(n))
        X = Bd.new_empty((n, k))
        info = SolveInfo(np.zeros(k, np.int64), np.zeros(k, np.int64), np.zeros(k), np.ones(k),
                         np.zeros(k, np.int64), mi)
        X, info = _solve_streamed(op, Bd, cfg, 16, mi, X, info)
        self._same((X.cpu().numpy(), info), self._solve(A, B, cfg, 64))


def test_csr_bandwidth_and_batch_width(cuda):
    """hf_csr_bandwidth = max_i max(i - first col, last col - i) of the SpMM copy;
    the batch width follows it (PcgOperator.batch_width)."""
    import scipy.sparse as sp

    from paper_1811_07717_b200.device import DeviceCsr, PcgOperator

    rng = np.random.default_rng(5)
    n = 2000
    M = sp.random(n, n, density=0.002, random_state=rng, format="csr")
    A = (M + M.T + sp.diags(np.full(n, 10.0))).tocsr()
    A.sort_indices()
    ref = max(max(i - A.indices[A.indptr[i]], A.indices[A.indptr[i + 1] - 1] - i) for i in range(n))
    op = PcgOperator(DeviceCsr.from_scipy(A))
    assert op.bandwidth == ref
    assert op.batch_width(128, 64) == 64  # a 2000-row window is far below L2
