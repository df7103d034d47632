"""pytest plugin: run the reference's own test suite with the B200 engine patched in.

Loaded with `-p refsuite_plugin` by tests/test_gpu_reference_suite.py on the GPU
box, where the unmodified reference lives in baseline/_ref (headfem + its tests,
tools/install_reference.sh).  `install(headfem)` runs before the test modules are
collected, so their `from headfem.solver import pcg_solve`-style imports bind the
engine's functions.  At the end of the session the plugin records whether the
rebinding held and how many libhfb200 kernels were launched, so the caller can
prove the suite ran on the GPU and not on the reference's numpy path.
"""
from __future__ import annotations

import json
import os

_STATE = {}


def pytest_configure(config):
    import headfem

    import paper_1811_07717_b200 as eng
    from paper_1811_07717_b200 import _native as N

    eng.install(headfem)
    _STATE["launch0"] = int(N.lib.hf_launch_count())
    import headfem.leadfield as hl
    import headfem.solver as hs

    _STATE["patched"] = bool(hs.pcg_solve is eng.pcg_solve and hl.transfer_matrix is eng.transfer_matrix
                             and hl.eeg_leadfield is eng.eeg_leadfield
                             and headfem.fem.assemble_A is eng.assemble_A)
    _STATE["headfem"] = headfem.__file__


def pytest_sessionfinish(session, exitstatus):
    from paper_1811_07717_b200 import _native as N

    out = os.environ.get("REFSUITE_REPORT")
    if out:
        with open(out, "w") as f:
            json.dump({"patched": _STATE.get("patched"), "headfem": _STATE.get("headfem"),
                       "gpu_launches": int(N.lib.hf_launch_count()) - _STATE.get("launch0", 0),
                       "exitstatus": int(exitstatus)}, f)
