"""Mesh generation on the device (hf_locate, hf_grid_tets, hf_mesh_compact,
hf_apply_priorities) against the reference's own outputs: point labels and
generated meshes array-for-array equal (nodes, element order, labels, sigma),
including the C1 mesh (55,545 nodes) the golden lead-field fixtures use."""
import numpy as np
import pytest

from tests.fixtures import load, segmentation

pytestmark = pytest.mark.gpu

FX = load("meshgen_cases.npz")
LOC = sorted({k.split("_")[0] for k in FX if k.startswith("loc")})
GM = sorted({k.split("_")[0] for k in FX if k.startswith("gm")})
SHELLS = dict(radii=(0.079, 0.086, 0.092), conds=(0.33, 0.0064, 0.43), prios=(2, 0, 3))


@pytest.fixture(scope="module")
def mg(cuda):
    from paper_1811_07717_b200 import meshgen

    return meshgen


@pytest.mark.parametrize("key", LOC)
def test_locate_matches_reference(mg, key):
    seg = segmentation(FX, key)
    np.testing.assert_array_equal(mg.locate(seg, FX[f"{key}_points"]), FX[f"{key}_labels"])


@pytest.mark.parametrize("key", GM)
def test_generate_mesh_matches_reference(mg, key):
    mesh = mg.generate_mesh(segmentation(FX, key), float(FX[f"{key}_h"]))
    np.testing.assert_array_equal(mesh.nodes, FX[f"{key}_nodes"])
    np.testing.assert_array_equal(mesh.tetra, FX[f"{key}_tetra"])
    np.testing.assert_array_equal(mesh.labels, FX[f"{key}_labels"])
    np.testing.assert_array_equal(mesh.sigma, FX[f"{key}_sigma"])


@pytest.mark.parametrize("name,h", [("layered_h12.npz", 0.012), ("c1.npz", 0.004)])
def test_generate_mesh_layered_fixtures(mg, name, h):
    from paper_1811_07717_b200.geometry import layered_sphere_segmentation

    fx = load(name)
    seg = layered_sphere_segmentation(SHELLS["radii"], SHELLS["conds"], SHELLS["prios"], (0,), 3)
    mesh = mg.generate_mesh(seg, h)
    np.testing.assert_array_equal(mesh.nodes, fx["nodes"])
    np.testing.assert_array_equal(mesh.tetra, fx["tetra"])
    np.testing.assert_array_equal(mesh.labels, fx["labels"])
    if fx["sigma"].ndim == 1:
        np.testing.assert_array_equal(mesh.sigma, fx["sigma"])


def test_segmentation_locate_method_and_single_point(mg):
    seg = segmentation(FX, "loc2")
    pts = FX["loc2_points"]
    np.testing.assert_array_equal(seg.locate(pts), FX["loc2_labels"])
    assert seg.compartments[0].contains(np.zeros(3)) is True
    assert seg.compartments[0].surfaces[0].contains(np.array([5.0, 0, 0])) is False


def test_generate_mesh_errors(mg):
    from paper_1811_07717_b200.errors import EmptyMeshError, ParameterError
    from paper_1811_07717_b200.geometry import Compartment, Segmentation, icosphere

    seg = segmentation(FX, "gm0")
    for h in (0.0, -1.0, float("nan")):
        with pytest.raises(ParameterError):
            mg.generate_mesh(seg, h)
    tiny = icosphere(0.05, 1, center=(0.9, 0.9, 0.9))
    big = icosphere(0.05, 1, center=(0.05, 0.05, 0.05))
    with pytest.raises(EmptyMeshError):  # test_meshgen.py:89-94
        mg.generate_mesh(Segmentation([Compartment(tiny, 1.0), Compartment(big, 1.0)]), 2.5)


def test_c2_scale_generate_mesh_consistent(mg):
    """4-shell sphere at h = 3 mm (~150k nodes): device labels equal a device
    re-location of the centroids wherever no priority rule applies, and every
    element has positive volume."""
    from paper_1811_07717_b200.geometry import layered_sphere_segmentation

    seg = layered_sphere_segmentation((0.079, 0.082, 0.087, 0.092), (0.33, 1.79, 0.0064, 0.43),
                                      (2, 1, 0, 3), (0,), 3)
    mesh = mg.generate_mesh(seg, 0.003)
    assert mesh.n_nodes > 100_000 and np.all(mesh.volumes > 0)
    cl = mg.locate(seg, mesh.centroids())
    nl = mg.locate(seg, mesh.nodes)[mesh.tetra]
    plain = np.all((nl == nl[:, :1]) | (nl < 0), axis=1)
    np.testing.assert_array_equal(mesh.labels[plain], cl[plain])


def test_segmentation_to_leadfield_matches_reference(mg):
    """Segmentation -> generate_mesh (device) -> EEG lead field (device), against the
    reference's lead field for the same segmentation (sphere_small: icosphere(0.1, 2),
    h = 0.045; tests/golden/make_golden.py:149-163)."""
    import paper_1811_07717_b200 as eng
    from paper_1811_07717_b200 import model
    from paper_1811_07717_b200.geometry import Compartment, Segmentation, icosphere

    from tests.fixtures import electrodes_from_fixture

    fx = load("sphere_small.npz")
    mesh = mg.generate_mesh(Segmentation([Compartment(icosphere(0.1, 2), 0.33, active=True)]), 0.045)
    np.testing.assert_array_equal(mesh.tetra, fx["tetra"])
    el = electrodes_from_fixture(mesh, fx)
    B, C, R = model.assemble_B_C_R(mesh, el)
    src = model.SourceSpace(positions=fx["src_positions"], orientations=None,
                            element_ids=fx["src_elements"], mode="unconstrained")
    G = model.assemble_G(mesh, src)
    sysm = model.CemSystem(mesh=mesh, electrodes=el, A=eng.assemble_A(mesh, el), B=B, C=C, R=R,
                           ground=model.ground_node(mesh, el), G=G, source_space=src)
    lf = eng.eeg_leadfield(sysm, eng.PcgConfig(tolerance=float(fx["tol"])))
    ref = fx["LF"]
    assert np.linalg.norm(lf.matrix - ref) / np.linalg.norm(ref) <= 1e-6
