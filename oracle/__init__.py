"""CPU oracle for the lead-field hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in numpy/scipy, the algorithm of the reference package
`headfem` (/root/reference/pkg/src/headfem) for the path the B200 engine
replaces: P1 stiffness assembly (fem.py), LDP-PCG (solver.py) and the
lead-field contractions (leadfield.py).  Every function cites the reference
lines it follows.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import it, and only as the checker (or as the timed CPU baseline).  The
product package `paper_1811_07717_b200` never imports it and fails loudly when
its CUDA library is missing.

Parity pin: the restatement is checked against golden vectors produced by the
reference itself (tests/golden/make_golden.py imports headfem from
/root/reference and writes tests/golden/*.npz); tests/test_oracle_golden.py
holds the comparison.
"""

from .solver import ConvergenceFailure, PcgSettings, ldp, pcg_solve, transfer_matrix
from .fem import assemble_A, ground_node, stiffness_blocks, volume_stiffness
from .leadfield import (
    build_dof_map,
    dof_sensitivities,
    eeg_leadfield,
    eit_forward,
    eit_leadfield,
    electrode_response,
    solve_response,
)

__all__ = [
    "ConvergenceFailure", "PcgSettings", "ldp", "pcg_solve", "transfer_matrix",
    "assemble_A", "ground_node", "stiffness_blocks", "volume_stiffness",
    "build_dof_map", "dof_sensitivities", "eeg_leadfield", "eit_forward", "eit_leadfield",
    "electrode_response", "solve_response",
]
