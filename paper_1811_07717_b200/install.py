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
                  "eeg_leadfield", "eit_forward", "eit_leadfield", "build_dof_map"),
    "cli": ("eeg_leadfield", "eit_leadfield", "eit_forward", "assemble_A", "transfer_matrix",
            "generate_mesh", "build_dof_map"),
    "experiments": ("eeg_leadfield", "eit_leadfield", "eit_forward", "assemble_A", "generate_mesh",
                    "build_dof_map"),
    "meshgen": ("generate_mesh",),
    "simulate": ("eit_forward", "assemble_A", "eeg_leadfield"),
    "": ("ldp", "pcg_solve", "transfer_matrix", "assemble_A", "volume_stiffness",
         "eeg_leadfield", "eit_forward", "eit_leadfield", "electrode_response", "generate_mesh",
         "build_dof_map"),
}
_saved = []


def _engine(name, headfem=None):
    from . import fem, leadfield, meshgen, solver
    if name == "build_dof_map":  # returns the caller's own EitDofMap type
        dof_cls = importlib.import_module(f"{headfem.__name__}.leadfield").EitDofMap

        def build_dof_map(mesh, compartments, n_dofs, seed=0):
            m = leadfield.build_dof_map(mesh, compartments, n_dofs, seed)
            out = dof_cls(element_sets=m.element_sets, centers=m.centers)
            object.__setattr__(out, "_device", getattr(m, "_device", None))  # the device arrays
            return out

        build_dof_map.__doc__ = leadfield.build_dof_map.__doc__
        return build_dof_map
    if name == "generate_mesh":  # returns the caller's own TetMesh type
        mesh_cls = importlib.import_module(f"{headfem.__name__}.meshgen").TetMesh

        def generate_mesh(seg, h):
            return meshgen.generate_mesh_device(seg, h).to_mesh(mesh_cls)

        generate_mesh.__doc__ = meshgen.generate_mesh.__doc__
        return generate_mesh
    for mod in (solver, fem, leadfield):
        if hasattr(mod, name):
            return getattr(mod, name)
    raise AttributeError(name)


def install(headfem=None):
    """Rebind headfem's lead-field entry points to the B200 engine."""
    if headfem is None:
        headfem = importlib.import_module("headfem")
    made = {}
    for sub, names in _PATCHES.items():
        try:
            mod = importlib.import_module(f"{headfem.__name__}.{sub}") if sub else headfem
        except ImportError:
            continue
        for name in names:
            if hasattr(mod, name):
                _saved.append((mod, name, getattr(mod, name)))
                if name not in made:
                    made[name] = _engine(name, headfem)
                setattr(mod, name, made[name])
    # Segmentation.locate is a method (meshgen.py:227,239 and geometry.py:406 call it)
    geo = importlib.import_module(f"{headfem.__name__}.geometry")
    _saved.append((geo.Segmentation, "locate", geo.Segmentation.locate))
    geo.Segmentation.locate = _locate_method
    return headfem


def _locate_method(self, points):
    """Segmentation.locate (geometry.py:359-374) on the device (hf_locate)."""
    from .meshgen import locate

    return locate(self, points)


def uninstall():
    while _saved:
        mod, name, fn = _saved.pop()
        setattr(mod, name, fn)
