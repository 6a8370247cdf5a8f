"""Exception types mirroring the reference's failure surface
(constitutive.py:56-57, solver/multigrid.py:46-52, slab.py:50-68)."""


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
