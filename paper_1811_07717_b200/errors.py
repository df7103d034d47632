"""Exception types of the lead-field path (headfem/errors.py:10-124).

When the reference package `headfem` is importable the engine raises the
reference's own classes, so a patched-in `headfem` (see `install`) keeps its
error contract (`pytest.raises(headfem.errors.ConvergenceError)` still
matches).  Otherwise the same hierarchy is defined here with the same names,
bases and payloads.
"""
from __future__ import annotations

try:  # pragma: no cover - depends on the environment
    from headfem.errors import (  # type: ignore
        AssemblyError,
        ComputationError,
        ConvergenceError,
        CurrentPatternError,
        DofError,
        ElectrodeError,
        EmptyMeshError,
        FormatError,
        HeadfemError,
        LocationError,
        ParameterError,
        SetupError,
        SingularPreconditionerError,
        SingularSystemError,
        TopologyError,
    )
    FROM_REFERENCE = True
except ImportError:
    FROM_REFERENCE = False

    class HeadfemError(Exception):
        """Base class (errors.py:10)."""

    class SetupError(HeadfemError):
        """Invalid input data or configuration (CLI exit code 2)."""

    class ComputationError(HeadfemError):
        """Numerical or runtime failure (CLI exit code 3)."""

    class FormatError(SetupError):
        """Malformed input data (errors.py:24)."""

    class TopologyError(SetupError):
        """A surface is not closed or not consistently oriented (errors.py:28)."""

    class EmptyMeshError(ComputationError):
        """Mesh generation produced no elements (errors.py:34)."""

    class ParameterError(SetupError):
        """A numeric parameter is outside its admissible range."""

    class AssemblyError(ComputationError):
        """System assembly produced an invalid (non-SPD) operator."""

    class ElectrodeError(SetupError):
        """An electrode definition covers no boundary area."""

    class LocationError(SetupError):
        """A point could not be located inside the mesh."""

    class SingularPreconditionerError(ComputationError):
        """The lumped diagonal preconditioner has a zero entry."""

    class ConvergenceError(ComputationError):
        """Iterative solve did not reach the tolerance; carries the best iterate
        (`best_x`, `residual`, `iterations`) and, from a multi-column solve, the
        failing `column` (errors.py:66-80)."""

        def __init__(self, message, best_x=None, residual=None, iterations=None, column=None):
            super().__init__(message)
            self.best_x = best_x
            self.residual = residual
            self.iterations = iterations
            self.column = column

    class SingularSystemError(ComputationError):
        """A dense electrode-level system is singular."""

    class CurrentPatternError(SetupError):
        """Injected currents do not sum to zero."""

    class DofError(SetupError):
        """A conductivity DOF has an empty element support."""


__all__ = [
    "HeadfemError", "SetupError", "ComputationError", "ParameterError", "AssemblyError",
    "ElectrodeError", "LocationError", "FormatError", "TopologyError", "EmptyMeshError", "SingularPreconditionerError", "ConvergenceError",
    "SingularSystemError", "CurrentPatternError", "DofError", "FROM_REFERENCE",
]
