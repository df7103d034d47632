"""Host-side logic on CPU: the C-ABI library loads and exports every symbol the
header declares; the input builders mirror the reference bit for bit; config
validation and sharding arithmetic."""
import hashlib
import os
import re

import numpy as np
import pytest

from tests.fixtures import csr, electrodes_from_fixture, load, mesh_from_fixture

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def header_symbols():
    text = open(os.path.join(ROOT, "include", "hfb200.h")).read()
    return sorted(set(re.findall(r"\b(hf_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_1811_07717_b200 import _native as N

    declared = header_symbols()
    assert len(declared) >= 17
    for name in declared:
        assert hasattr(N.lib, name), name
    assert sorted(N.EXPORTED) == declared
    assert N.lib.hf_version().decode().startswith("hfb200")


def test_library_is_sm100a():
    import subprocess

    from paper_1811_07717_b200 import _native as N

    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_workspace_queries_need_no_gpu():
    from paper_1811_07717_b200 import _native as N

    assert N.lib.hf_pcg_workspace_bytes(1000, 32, 15000) > 1000 * 32 * 8 * 3
    assert N.lib.hf_p1_assemble_workspace_bytes(1000, 5000, 10) > 0
    assert N.lib.hf_csr_prune_workspace_bytes(1000) > 0


def test_pcg_config_validation():
    import paper_1811_07717_b200 as eng

    for kw in ({"tolerance": 0.0}, {"max_iterations": 0}, {"preconditioner": "amg"}):
        with pytest.raises(eng.ParameterError):
            eng.PcgConfig(**kw)
    assert eng.PcgConfig().resolve_max_iterations(1_001_184) == 6002  # int(5 sqrt n) + 1000


@pytest.mark.parametrize("name", ["sphere_small.npz", "layered_h12.npz", "layered_h14_tensor.npz",
                                  "c1.npz"])
def test_boundary_ground_and_B_match_reference(name):
    from paper_1811_07717_b200 import model

    fx = load(name)
    mesh = mesh_from_fixture(fx)
    bf, ow = mesh.boundary_triangles()
    assert sha(bf.astype(np.int64)) == str(fx["bfaces_sha"])
    assert sha(ow.astype(np.int64)) == str(fx["bowners_sha"])
    el = electrodes_from_fixture(mesh, fx)
    assert model.ground_node(mesh, el) == int(fx["ground"])
    B, C, R = model.assemble_B_C_R(mesh, el)
    assert (B != csr(fx, "B")).nnz == 0
    np.testing.assert_array_equal(C.diagonal(), fx["Cdiag"])


@pytest.mark.parametrize("name", ["sphere_small.npz", "layered_h12.npz", "c1.npz"])
def test_assemble_G_matches_reference(name):
    """Vectorised Whitney source matrix: same pattern, values to rounding."""
    from paper_1811_07717_b200 import model

    fx = load(name)
    mesh = mesh_from_fixture(fx)
    src = model.SourceSpace(positions=fx["src_positions"], orientations=None,
                            element_ids=fx["src_elements"], mode="unconstrained")
    G = model.assemble_G(mesh, src)
    Gr = csr(fx, "G").copy()
    Gr.sort_indices()
    np.testing.assert_array_equal(G.indptr, Gr.indptr)
    np.testing.assert_array_equal(G.indices, Gr.indices)
    np.testing.assert_allclose(G.data, Gr.data, rtol=1e-9, atol=1e-13 * np.abs(Gr.data).max())


def test_electrodes_from_centers_match_reference():
    from paper_1811_07717_b200 import model, synthetic

    fx = load("layered_h12.npz")
    mesh = mesh_from_fixture(fx)
    el = model.ElectrodeSet.from_centers(mesh, synthetic.fibonacci_sphere_points(16, 0.092),
                                         radius=0.014, impedances=1e3)
    ref = electrodes_from_fixture(mesh, fx)
    for a, b in zip(el.triangle_ids, ref.triangle_ids):
        np.testing.assert_array_equal(a, b)


def test_dof_map_oracle_paths_match_reference():
    """The oracle's chunked and k-d-tree restatements of build_dof_map give the
    reference's sets (the product's device path is checked against both on the GPU)."""
    import oracle

    fx = load("layered_h12.npz")
    mesh = mesh_from_fixture(fx)
    for method in ("tree", "dense"):
        sets, centers = oracle.build_dof_map(mesh, [0, 1], 20, seed=2, method=method, chunk=64)
        np.testing.assert_array_equal(np.concatenate(sets), fx["eit_dof_elems"])
        np.testing.assert_array_equal(np.cumsum([0] + [len(e) for e in sets]), fx["eit_dof_ptr"])
        np.testing.assert_array_equal(centers, fx["eit_centers"])


def test_build_dof_map_has_no_cpu_fallback():
    import torch

    from paper_1811_07717_b200.leadfield import build_dof_map

    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        build_dof_map(mesh_from_fixture(load("layered_h12.npz")), [0, 1], 20, seed=2)


def test_column_blocks():
    from paper_1811_07717_b200.engine import column_blocks

    for L, w in [(128, 8), (128, 3), (5, 8), (256, 8)]:
        b = column_blocks(L, w)
        assert b[0][0] == 0 and b[-1][1] == L
        assert all(b[i][1] == b[i + 1][0] for i in range(w - 1))
        sizes = [c1 - c0 for c0, c1 in b]
        assert max(sizes) - min(sizes) <= 1


def test_synthetic_c1_mesh_is_a_valid_kuhn_grid():
    from paper_1811_07717_b200 import synthetic

    mesh = synthetic.sphere_mesh(synthetic.C1_RADII, synthetic.C1_COND, 0.012)
    h = 0.012
    np.testing.assert_allclose(mesh.volumes, h ** 3 / 6, rtol=1e-9)
    assert set(np.unique(mesh.labels)) == {0, 1, 2}


def test_install_rebinds_reference_entry_points():
    """With the reference importable (this container), install() patches the
    module attributes headfem resolves at call time and uninstall() restores."""
    import sys

    ref = "/root/reference/pkg/src"
    if not os.path.isdir(ref):
        pytest.skip("reference not present")
    sys.path.insert(0, ref)
    try:
        import headfem
        import headfem.leadfield as hl
        import headfem.solver as hs

        import paper_1811_07717_b200 as eng

        import headfem.geometry as hg
        import headfem.meshgen as hm

        orig, orig_gm, orig_loc = hs.pcg_solve, hm.generate_mesh, hg.Segmentation.locate
        eng.install(headfem)
        assert hs.pcg_solve is eng.pcg_solve and hl.transfer_matrix is eng.transfer_matrix
        assert hl.eeg_leadfield is eng.eeg_leadfield
        assert hm.generate_mesh is not orig_gm and headfem.generate_mesh is hm.generate_mesh
        assert hg.Segmentation.locate is not orig_loc
        eng.uninstall()
        assert hs.pcg_solve is orig and hm.generate_mesh is orig_gm
        assert hg.Segmentation.locate is orig_loc
    finally:
        sys.path.remove(ref)


def test_batch_width_policy():
    """kp stays at the cap unless the SpMM's two-plane window (4 x bandwidth x kp
    x 8 B) would exceed L2_WINDOW; never below 16, never above the column count."""
    from types import SimpleNamespace

    from paper_1811_07717_b200.device import PcgOperator

    bw = lambda b: SimpleNamespace(bandwidth=b)  # noqa: E731
    assert PcgOperator.batch_width(bw(12_232), 128, 64) == 64   # C2
    assert PcgOperator.batch_width(bw(35_031), 256, 64) == 32   # C5
    assert PcgOperator.batch_width(bw(10 ** 7), 256, 64) == 16  # floor
    assert PcgOperator.batch_width(bw(100), 5, 64) == 5


def test_abi_rejects_bad_arguments_without_a_gpu():
    """Argument validation happens before any CUDA call: every entry point returns
    HF_ERR_ARG (1) with a message on null pointers / bad shapes / unsupported widths."""
    import ctypes as C

    from paper_1811_07717_b200 import _native as N

    L = N.lib
    P = None
    arr = (C.c_int32 * 8)()
    dbl = (C.c_double * 8)()
    csr = N.HfCsr(10, 10, 30, 1, 1, 1)  # dummy (non-null) pointers
    # hf_pcg_multi: null argument, bad shape, unsupported kp
    assert L.hf_pcg_multi(None, P, P, 10, 4, 1e-8, 10, P, P, arr, arr, dbl, dbl, arr, P, 0, P) == 1
    assert b"null argument" in L.hf_last_error()
    rc = L.hf_pcg_multi(C.byref(csr), 1, 1, 11, 4, 1e-8, 10, P, 1, arr, arr, dbl, dbl, arr, 1, 0, P)
    assert rc == 1 and b"bad shape" in L.hf_last_error()
    rc = L.hf_pcg_multi(C.byref(csr), 1, 1, 10, 128, 1e-8, 10, P, 1, arr, arr, dbl, dbl, arr, 1, 0, P)
    assert rc == 1 and b"kp=128" in L.hf_last_error()
    rc = L.hf_pcg_multi(C.byref(csr), 1, 1, 10, 4, 0.0, 10, P, 1, arr, arr, dbl, dbl, arr, 1, 0, P)
    assert rc == 1  # tol must be > 0 (PcgConfig's rule)
    # hf_pcg_stream: null argument, ldb < ncols, unsupported kp
    assert L.hf_pcg_stream(None, 1, 1, 8, 8, 10, 4, 1e-8, 10, 1, arr, arr, dbl, dbl, arr, 1, 0, P) == 1
    assert b"null argument" in L.hf_last_error()
    rc = L.hf_pcg_stream(C.byref(csr), 1, 1, 4, 8, 10, 4, 1e-8, 10, 1, arr, arr, dbl, dbl, arr, 1, 0, P)
    assert rc == 1 and b"ldb=4" in L.hf_last_error()
    rc = L.hf_pcg_stream(C.byref(csr), 1, 1, 8, 8, 10, 3, 1e-8, 10, 1, arr, arr, dbl, dbl, arr, 1, 0, P)
    assert rc == 1 and b"kp=3" in L.hf_last_error()
    assert L.hf_ldp(None, P, P, None, P) == 1
    assert L.hf_eit_sens(P, P, P, P, 1, 0, P, 4, 4, P, 4, 2, P, P, 0, P) == 1
    assert L.hf_meg_rhs(P, P, P, 10, 10, 0, P, P, 600, P, 600, P, 0, P) == 1
    assert L.hf_lf_tail(P, 4, 4, None, P, 4, 4, P, P) == 1
    assert L.hf_ground_node(P, 0, P, 0, 10, P, None, P) == 1
    assert L.hf_dof_partition(P, P, 10, 0, P, P, P, 0, P) == 1


def test_abi_workspace_queries_cover_new_entry_points():
    from paper_1811_07717_b200 import _native as N

    assert N.lib.hf_eit_sens_workspace_bytes(4_105_824) >= 4_105_824 * 16 * 8
    # the stream workspace = a batch workspace's blocks + the slots' b and x + per-column results
    assert N.lib.hf_pcg_stream_workspace_bytes(1000, 64, 300) > 2 * 1000 * 64 * 8 + 300 * 28
    assert N.lib.hf_meg_workspace_bytes(1000, 5800) > 5800 * 16 * 8
    assert N.lib.hf_ground_node_workspace_bytes(1000) >= 4 * 1002
    assert N.lib.hf_dof_partition_workspace_bytes(100_000) > 100_000 * 4
