"""Parity of the CUDA P1 assembly with the reference (fem.py:31-224):
bit-exact CSR pattern (explicit zeros, grounding), values to rounding."""
import hashlib

import numpy as np
import pytest
import scipy.sparse as sp

from tests.fixtures import csr, electrodes_from_fixture, load, mesh_from_fixture

pytestmark = pytest.mark.gpu

FIXTURES = ["sphere_small.npz", "layered_h12.npz", "layered_h14_tensor.npz"]


@pytest.fixture(scope="module")
def eng(cuda):
    import paper_1811_07717_b200 as e

    return e


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", FIXTURES)
def test_assemble_A_matches_reference(eng, name):
    fx = load(name)
    mesh = mesh_from_fixture(fx)
    el = electrodes_from_fixture(mesh, fx)
    A = eng.assemble_A(mesh, el)
    Ar = csr(fx, "A")
    np.testing.assert_array_equal(A.indptr, Ar.indptr)
    np.testing.assert_array_equal(A.indices, Ar.indices)
    scale = np.abs(Ar.data).max()
    np.testing.assert_allclose(A.data, Ar.data, rtol=1e-11, atol=1e-13 * scale)
    assert A.indptr.dtype == np.int32 and A.indices.dtype == np.int32
    g = int(fx["ground"])
    row = A.getrow(g)
    assert row.nnz == 1 and row.indices[0] == g and row.data[0] == 1.0


@pytest.mark.parametrize("name", FIXTURES)
def test_volume_stiffness_matches_reference(eng, name):
    fx = load(name)
    mesh = mesh_from_fixture(fx)
    K = eng.volume_stiffness(mesh)
    Kr = csr(fx, "K")
    np.testing.assert_array_equal(K.indptr, Kr.indptr)
    np.testing.assert_array_equal(K.indices, Kr.indices)
    np.testing.assert_allclose(K.data, Kr.data, rtol=1e-11, atol=1e-13 * np.abs(Kr.data).max())
    # explicit zeros of the Kuhn stencil are kept, exactly where scipy keeps them
    assert np.count_nonzero(K.data == 0.0) > 0 or name == "sphere_small.npz"


def test_assembly_is_bit_reproducible(eng):
    fx = load("layered_h12.npz")
    mesh = mesh_from_fixture(fx)
    el = electrodes_from_fixture(mesh, fx)
    A1, A2 = eng.assemble_A(mesh, el), eng.assemble_A(mesh, el)
    np.testing.assert_array_equal(A1.data, A2.data)


def test_stiffness_blocks_match_oracle(eng):
    import oracle

    fx = load("layered_h14_tensor.npz")
    mesh = mesh_from_fixture(fx)
    Kb = eng.stiffness_blocks(mesh)
    Ko = oracle.stiffness_blocks(mesh.nodes, mesh.tetra, mesh.sigma)
    np.testing.assert_allclose(Kb, Ko, rtol=1e-10, atol=1e-13 * np.abs(Ko).max())
    el = np.array([5, 1, 100, 7])
    np.testing.assert_allclose(eng.stiffness_blocks(mesh, sigma=1.0, elements=el),
                               oracle.stiffness_blocks(mesh.nodes, mesh.tetra, 1.0, elements=el),
                               rtol=1e-10, atol=1e-13)


def test_subset_volume_stiffness(eng):
    import oracle

    fx = load("sphere_small.npz")
    mesh = mesh_from_fixture(fx)
    el = np.arange(0, mesh.n_elements, 3)
    K = eng.volume_stiffness(mesh, sigma=1.0, elements=el)
    Ko = oracle.volume_stiffness(mesh.nodes, mesh.tetra, 1.0, elements=el)
    np.testing.assert_array_equal(K.indices, Ko.indices)
    np.testing.assert_allclose(K.toarray(), Ko.toarray(), rtol=1e-11, atol=1e-15)


def single_tet(sigma):
    from paper_1811_07717_b200.model import TetMesh

    nodes = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], dtype=float)
    s = np.asarray([sigma]) if np.isscalar(sigma) else np.asarray(sigma)[None, :]
    return TetMesh(nodes, np.array([[0, 1, 2, 3]]), np.array([0]), s)


def test_single_tet_electrode_block(eng):
    from paper_1811_07717_b200.model import ElectrodeSet

    mesh = single_tet(0.0)
    bfaces, _ = mesh.boundary_triangles()
    z0 = [i for i, f in enumerate(bfaces) if np.allclose(mesh.nodes[f][:, 2], 0.0)]
    Z = 2.5
    A = eng.assemble_A(mesh, ElectrodeSet(mesh, [np.array(z0)], Z), ground=False).toarray()
    tri = bfaces[z0[0]]
    for i in tri:
        assert A[i, i] == pytest.approx(1.0 / (6.0 * Z), rel=1e-14)
        for j in tri:
            if i != j:
                assert A[i, j] == pytest.approx(1.0 / (12.0 * Z), rel=1e-14)


def test_negative_sigma_rejected(eng):
    with pytest.raises(eng.AssemblyError):
        eng.volume_stiffness(single_tet(-1.0))


def test_non_pd_tensor_rejected(eng):
    with pytest.raises(eng.AssemblyError):
        eng.volume_stiffness(single_tet([1.0, 1.0, -1.0, 0.0, 0.0, 0.0]))


def test_isotropic_tensor_equals_scalar(eng):
    Ki = eng.volume_stiffness(single_tet(0.73)).toarray()
    Kt = eng.volume_stiffness(single_tet([0.73, 0.73, 0.73, 0, 0, 0])).toarray()
    np.testing.assert_allclose(Kt, Ki, atol=1e-15 * np.abs(Ki).max())


def test_c1_pattern_hash(eng):
    """Full C1 mesh (55,545 nodes): the grounded A's int32 indptr/indices hash
    equal to the reference's."""
    fx = load("c1.npz")
    mesh = mesh_from_fixture(fx)
    el = electrodes_from_fixture(mesh, fx)
    A = eng.assemble_A(mesh, el)
    assert A.nnz == int(fx["A_nnz"])
    assert sha(A.indptr.astype(np.int32)) == str(fx["A_sha_indptr"])
    assert sha(A.indices.astype(np.int32)) == str(fx["A_sha_indices"])
    _ = sp


@pytest.mark.parametrize("n", [0, 1, 4095, 4096, 4097, 16_777_217, 40_000_003])
def test_exclusive_scan_any_length(eng, n):
    """CSR row-pointer scan: exact, including lengths past two tile levels (C5 has 28.7M elements)."""
    import torch
    from paper_1811_07717_b200 import _native as N

    g = torch.Generator(device="cuda").manual_seed(n)
    x = torch.randint(0, 4, (max(n, 1),), generator=g, device="cuda", dtype=torch.int32)[:n]
    out = torch.empty_like(x)
    tot = torch.zeros(1, dtype=torch.int32, device="cuda")
    ws = torch.empty(max(N.lib.hf_scan_workspace_bytes(n), 1), dtype=torch.uint8, device="cuda")
    N.check("hf_exclusive_scan_i32", N.lib.hf_exclusive_scan_i32(
        N.ptr(x), N.ptr(out), n, N.ptr(tot), N.ptr(ws), ws.numel(), N.stream_handle()))
    c = torch.cumsum(x.long(), 0)
    assert int(tot.item()) == (int(c[-1]) if n else 0)
    if n:
        assert torch.equal(out.long(), c - x.long())
