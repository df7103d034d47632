"""CPU: the mesh-generation oracle (oracle/meshgen.py) and the geometry mirror
against golden vectors made by the reference (tests/golden/make_meshgen_golden.py)."""
import numpy as np
import pytest

import oracle.meshgen as OM
from tests.fixtures import load, seg_parts

FX = load("meshgen_cases.npz")
LOC = sorted({k.split("_")[0] for k in FX if k.startswith("loc")})
GM = sorted({k.split("_")[0] for k in FX if k.startswith("gm")})


def test_ray_directions_match_reference():
    from paper_1811_07717_b200.geometry import RAY_DIRECTIONS

    np.testing.assert_array_equal(OM.RAY_DIRECTIONS, FX["ray_dirs"])
    np.testing.assert_array_equal(RAY_DIRECTIONS, FX["ray_dirs"])


@pytest.mark.parametrize("key", LOC)
def test_oracle_locate(key):
    np.testing.assert_array_equal(OM.locate(seg_parts(FX, key), FX[f"{key}_points"]), FX[f"{key}_labels"])


@pytest.mark.parametrize("key", GM)
def test_oracle_generate_mesh(key):
    nodes, tetra, labels, sigma = OM.generate_mesh(seg_parts(FX, key), float(FX[f"{key}_h"]))
    np.testing.assert_array_equal(nodes, FX[f"{key}_nodes"])
    np.testing.assert_array_equal(tetra, FX[f"{key}_tetra"])
    np.testing.assert_array_equal(labels, FX[f"{key}_labels"])
    np.testing.assert_array_equal(sigma, FX[f"{key}_sigma"])


def test_icosphere_mirror_matches_reference_surfaces():
    from paper_1811_07717_b200.geometry import icosphere

    # layered case: shells 0.079 .. 0.092, subdivisions 3 (experiments.py:46-57)
    for c, r in enumerate((0.079, 0.082, 0.087, 0.092)):
        s = icosphere(r, 3)
        np.testing.assert_array_equal(s.nodes, FX[f"gm7_c{c}_s0_nodes"])
        np.testing.assert_array_equal(s.triangles, FX[f"gm7_c{c}_s0_tris"])


def test_surface_validation_errors():
    from paper_1811_07717_b200.errors import FormatError, TopologyError
    from paper_1811_07717_b200.geometry import SurfaceMesh

    nodes = FX["loc0_c0_s0_nodes"]
    tris = FX["loc0_c0_s0_tris"]
    with pytest.raises(TopologyError):
        SurfaceMesh(nodes, tris[:3])
    with pytest.raises(TopologyError):
        SurfaceMesh(nodes, tris[:, ::-1].copy()[[0, 1, 2]].tolist() + [tris[3].tolist()])
    with pytest.raises(IndexError):
        SurfaceMesh(nodes, tris + 10)
    with pytest.raises(FormatError):
        SurfaceMesh(nodes[:, :2], tris)
