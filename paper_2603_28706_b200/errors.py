"""Exception types of the reference's failure surface
(constitutive.py:56-57, solver/multigrid.py:46-52, slab.py:50-68).

When pdflow itself is importable (the drop-in setting: the reference's own
time marcher, Newton driver or harness calls this package), its classes ARE
the ones raised here, so ``march``'s ``except SlabSolveError``
(slab.py:256-258) converts a device-solver failure into ``MarchError`` and
pdflow callers catching ``SingularPatchError`` / ``ConstitutiveDomainError``
see libpdst's failures.  Otherwise look-alike classes with the same
constructors and attributes are defined.  ``PDFLOW_EXCEPTIONS`` says which.
"""

from __future__ import annotations

try:  # pragma: no cover - depends on the environment
    from pdflow.constitutive import ConstitutiveDomainError
    from pdflow.slab import SlabSolveError
    from pdflow.solver.multigrid import SingularPatchError

    PDFLOW_EXCEPTIONS = True
except ImportError:
    PDFLOW_EXCEPTIONS = False

    class ConstitutiveDomainError(ValueError):
        """Operation evaluated outside its admissible parameter regime."""

    class SingularPatchError(RuntimeError):
        """A local Vanka patch matrix was numerically singular."""

        def __init__(self, level: int, patch: int):
            super().__init__(f"singular patch matrix (level {level}, patch {patch})")
            self.level = level
            self.patch = patch

    class SlabSolveError(RuntimeError):
        """A slab solve failed; kind is one of line_search, max_iterations, krylov."""

        def __init__(self, kind: str, message: str, diagnostics=None):
            super().__init__(f"{kind}: {message}")
            self.kind = kind
            self.diagnostics = diagnostics


class PdstCudaError(RuntimeError):
    """CUDA runtime failure inside libpdst."""


__all__ = ["ConstitutiveDomainError", "SingularPatchError", "SlabSolveError", "PdstCudaError", "PDFLOW_EXCEPTIONS"]
