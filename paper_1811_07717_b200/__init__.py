"""B200-native FEM lead-field engine (drop-in for the lead-field path of `headfem`).

Hot path, all in libhfb200.so (sm_100a, C ABI in include/hfb200.h):
  * P1 stiffness CSR assembly              -> fem.assemble_A / volume_stiffness
  * multi-RHS LDP-PCG transfer solve       -> solver.pcg_solve / transfer_matrix
  * lead-field contractions (EEG, EIT)     -> leadfield.eeg_leadfield / eit_leadfield

`install(headfem)` rebinds the reference package's entry points to this
engine so existing callers (CLI, experiments, tests) run on the GPU.
"""
from .errors import (
    AssemblyError,
    ConvergenceError,
    CurrentPatternError,
    DofError,
    ParameterError,
    SingularPreconditionerError,
    SingularSystemError,
)
from .solver import PcgConfig, ldp, pcg_solve, transfer_matrix
from .fem import assemble_A, stiffness_blocks, volume_stiffness
from .leadfield import (
    EitDofMap,
    LeadField,
    adjacent_pair_patterns,
    build_dof_map,
    check_current_patterns,
    eeg_leadfield,
    eit_forward,
    eit_leadfield,
    electrode_response,
)
from .install import install, uninstall

__version__ = "0.1.0"
__all__ = [name for name in dir() if not name.startswith("_")]
