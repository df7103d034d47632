"""The reference's own tests, unchanged, with the engine patched in.

`baseline/_ref` holds the unmodified reference package and a copy of its test
suite (tools/install_reference.sh).  Each test here runs a slice of that suite
in a subprocess whose pytest session calls `install(headfem)` first
(tests/refsuite_plugin.py): every hot-path call the reference's tests make —
pcg_solve, transfer_matrix, assemble_A, eeg_leadfield, eit_leadfield,
generate_mesh, ... — then runs in libhfb200.so on the GPU.  The plugin's report
proves the rebinding held and that kernels were launched.
"""
import json
import os
import subprocess
import sys
import xml.etree.ElementTree as ET

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
SUITE = os.path.join(REF, "headfem_tests")

HOT_PATH = [  # the hot-path tests the build must pass unchanged
    "test_solver.py",
    "test_leadfield.py",
    "test_fem.py::TestAssembleA",
    "test_fem.py::TestSystem",
    "test_acceptance.py::test_criterion_1_fem_oracle_equivalence",
    "test_acceptance.py::test_criterion_2_zero_mean_constraint",
    "test_acceptance.py::test_criterion_3_eit_linearization",
    "test_acceptance.py::test_criterion_9_solver_oracle",
]


def _run(tmp_path, targets, timeout):
    if not os.path.isdir(SUITE):
        pytest.skip(f"{SUITE} missing: run tools/install_reference.sh (baseline/_ref ships with the snapshot)")
    report = tmp_path / "report.json"
    junit = tmp_path / "junit.xml"
    ini = tmp_path / "pytest.ini"
    ini.write_text("[pytest]\n")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, ROOT, os.path.join(ROOT, "tests"),
                                         env.get("PYTHONPATH", "")])
    env["REFSUITE_REPORT"] = str(report)
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-p", "refsuite_plugin",
           "-c", str(ini), "--rootdir", SUITE, f"--junitxml={junit}",
           *[os.path.join(SUITE, t) for t in targets]]
    proc = subprocess.run(cmd, cwd=tmp_path, env=env, capture_output=True, text=True, timeout=timeout)
    tail = (proc.stdout + proc.stderr)[-4000:]
    assert report.exists(), tail
    rep = json.loads(report.read_text())
    root = ET.parse(junit).getroot()
    suite = root if root.tag == "testsuite" else root.find("testsuite")
    counts = {k: int(suite.get(k, 0)) for k in ("tests", "failures", "errors", "skipped")}
    print(f"\nreference suite {targets}: {counts}, report {rep}\n{tail[-1500:]}")
    return proc.returncode, counts, rep, tail


@pytest.mark.gpu
def test_reference_hot_path_suite_on_engine(cuda, tmp_path):
    rc, counts, rep, tail = _run(tmp_path, HOT_PATH, timeout=1800)
    assert rep["patched"], rep
    assert rep["headfem"].startswith(REF), rep  # the installed reference, not /root/reference
    assert rep["gpu_launches"] > 1000, rep
    assert counts["failures"] == 0 and counts["errors"] == 0, tail
    assert counts["tests"] - counts["skipped"] >= 48, counts
    assert rc == 0, tail


@pytest.mark.gpu
def test_reference_full_suite_on_engine(cuda, tmp_path):
    """All 199 reference tests (mesh generation, simulation, inversion, CLI and the
    acceptance criteria included) with the engine patched in."""
    rc, counts, rep, tail = _run(tmp_path, ["."], timeout=3000)
    assert rep["patched"] and rep["gpu_launches"] > 1000, rep
    assert counts["failures"] == 0 and counts["errors"] == 0, tail
    assert counts["tests"] >= 199, counts
    assert rc == 0, tail
