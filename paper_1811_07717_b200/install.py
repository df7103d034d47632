"""Patch the reference package so its lead-field path runs on this engine.

The reference resolves its hot-path callees as module attributes at call
time: solver.pcg_solve/transfer_matrix/ldp, the copies bound
into leadfield.py:28-29, fem.volume_stiffness/assemble_A/stiffness_blocks and
the bindings held by cli.py, experiments.py and simulate.py.  `install`
rebinds every one of them and returns a handle; `uninstall` restores them.
"""
from __future__ import annotations

import importlib

_PATCHES = {
    "solver": ("ldp", "pcg_solve", "transfer_matrix"),
    "fem": ("stiffness_blocks", "volume_stiffness", "assemble_A"),
    "leadfield": ("stiffness_blocks", "pcg_solve", "transfer_matrix", "electrode_response",
                  "eeg_leadfield", "eit_forward", "eit_leadfield"),
    "cli": ("eeg_leadfield", "eit_leadfield", "eit_forward", "assemble_A", "transfer_matrix"),
    "experiments": ("eeg_leadfield", "eit_leadfield", "eit_forward", "assemble_A"),
    "simulate": ("eit_forward", "assemble_A", "eeg_leadfield"),
    "": ("ldp", "pcg_solve", "transfer_matrix", "assemble_A", "volume_stiffness",
         "eeg_leadfield", "eit_forward", "eit_leadfield", "electrode_response"),
}
_saved = []


def _engine(name):
    from . import fem, leadfield, solver
    for mod in (solver, fem, leadfield):
        if hasattr(mod, name):
            return getattr(mod, name)
    raise AttributeError(name)


def install(headfem=None):
    """Rebind headfem's lead-field entry points to the B200 engine."""
    if headfem is None:
        headfem = importlib.import_module("headfem")
    for sub, names in _PATCHES.items():
        try:
            mod = importlib.import_module(f"{headfem.__name__}.{sub}") if sub else headfem
        except ImportError:
            continue
        for name in names:
            if hasattr(mod, name):
                _saved.append((mod, name, getattr(mod, name)))
                setattr(mod, name, _engine(name))
    return headfem


def uninstall():
    while _saved:
        mod, name, fn = _saved.pop()
        setattr(mod, name, fn)
