"""Host-side problem description mirroring the reference's data model.

These light dataclasses carry the same attribute names the reference exposes
(mesh.py:50-148, forms.py:60-302, constitutive.py:60-160, slab.py:71-141), so
the GPU operators in :mod:`operators` accept either these objects or the
reference's own ``SlabContext`` (duck typing).  Nothing here computes on the
hot path; it only describes the problem.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .errors import ConstitutiveDomainError
from .radau import TimeBasis, TimeMatrices, gauss_radau, temporal_matrices

DIRICHLET = "dirichlet"
NEUMANN = "neumann"
SIDES = ("bottom", "right", "top", "left")
PIC, EXN, MODN = "pic", "exn", "modn"


@dataclass(frozen=True)
class ModelParams:
    """(p, delta, nu, nu_inf) with the validation of constitutive.py:73-81."""

    p: float
    delta: float
    nu: float
    nu_inf: float = 0.0

    def __post_init__(self):
        if not 1.0 < self.p <= 2.0:
            raise ConstitutiveDomainError(f"exponent p must lie in (1, 2], got {self.p}")
        if self.delta < 0.0:
            raise ConstitutiveDomainError(f"delta must be >= 0, got {self.delta}")
        if self.nu <= 0.0:
            raise ConstitutiveDomainError(f"nu must be > 0, got {self.nu}")
        if self.nu_inf < 0.0:
            raise ConstitutiveDomainError(f"nu_inf must be >= 0, got {self.nu_inf}")


@dataclass(frozen=True)
class TangentVariant:
    kind: str
    sigma_max: float = math.inf

    def __post_init__(self):
        if self.kind not in (PIC, EXN, MODN):
            raise ValueError(f"unknown tangent kind {self.kind!r}")
        if self.kind == MODN and self.sigma_max < 0.0:
            raise ValueError("sigma_max must be >= 0")


def picard() -> TangentVariant:
    return TangentVariant(PIC)


def exact_newton() -> TangentVariant:
    return TangentVariant(EXN)


def modified_newton(sigma_max: float) -> TangentVariant:
    return TangentVariant(MODN, sigma_max)


@dataclass(frozen=True)
class QuadMesh:
    """Uniform nx-by-ny quad mesh; boundary_tags per boundary face in side
    order bottom, right, top, left (None = all Dirichlet)."""

    nx: int
    ny: int
    x0: float = 0.0
    y0: float = 0.0
    x1: float = 1.0
    y1: float = 1.0
    level: int = 0
    boundary_tags: np.ndarray | None = None

    def __post_init__(self):
        if self.nx < 1 or self.ny < 1:
            raise ValueError("cell counts must be >= 1")
        if self.x1 <= self.x0 or self.y1 <= self.y0:
            raise ValueError("degenerate domain extents")

    @property
    def hx(self):
        return (self.x1 - self.x0) / self.nx

    @property
    def hy(self):
        return (self.y1 - self.y0) / self.ny

    @property
    def ncells(self):
        return self.nx * self.ny


def tag_sides(mesh: QuadMesh, neumann_sides=()) -> QuadMesh:
    tags = []
    for side in SIDES:
        n = mesh.nx if side in ("bottom", "top") else mesh.ny
        tags += [NEUMANN if side in neumann_sides else DIRICHLET] * n
    return QuadMesh(mesh.nx, mesh.ny, mesh.x0, mesh.y0, mesh.x1, mesh.y1, mesh.level, np.array(tags, dtype=object))


def dirichlet_flags(mesh) -> np.ndarray:
    """uint8 tags per boundary face: 1 Dirichlet, 0 Neumann, 2 partition cut
    (integer tag arrays pass through); untagged = all Dirichlet (forms.py:144-145)."""
    nbf = 2 * (mesh.nx + mesh.ny)
    tags = getattr(mesh, "boundary_tags", None)
    if tags is None:
        return np.ones(nbf, dtype=np.uint8)
    arr = np.asarray(tags)
    if arr.dtype.kind in "iu":
        return arr.astype(np.uint8)
    return np.array([str(t) == DIRICHLET for t in tags], dtype=np.uint8)


PRESSURE_SPACES = ("p1disc", "q1")


@dataclass
class Discretization:
    """Q2 velocity with the reference's P1disc pressure (femspace.py:109-160),
    or -- pressure="q1" -- the Taylor-Hood pair Q2/Q1 (continuous bilinear
    pressure on the (nx+1)(ny+1) vertices, row-major (y, x); BASELINE
    north_star (1), no reference counterpart)."""

    mesh: QuadMesh
    pressure: str = "p1disc"

    def __post_init__(self):
        if self.pressure not in PRESSURE_SPACES:
            raise ValueError(f"unknown pressure space {self.pressure!r} (one of {PRESSURE_SPACES})")

    @property
    def n_velocity(self):
        return 2 * (2 * self.mesh.nx + 1) * (2 * self.mesh.ny + 1)

    @property
    def n_pressure(self):
        if self.pressure == "q1":
            return (self.mesh.nx + 1) * (self.mesh.ny + 1)
        return 3 * self.mesh.ncells

    @property
    def ndof(self):
        return self.n_velocity + self.n_pressure

    @property
    def all_dirichlet(self):
        return bool((dirichlet_flags(self.mesh) == 1).all())


@dataclass
class DiscretizationConfig:
    gamma1: float = 1.0e3
    gamma2: float = 1.0e3
    gamma_cip: float = 1.0
    g_hat: np.ndarray | None = None
    enable_viscous: bool = True
    enable_convection: bool = True
    enable_pressure: bool = True

    def __post_init__(self):
        if self.gamma1 <= 0.0 or self.gamma2 <= 0.0:
            raise ValueError("Nitsche penalties gamma1, gamma2 must be positive")
        if self.gamma_cip < 0.0:
            raise ValueError("gamma_cip must be >= 0")


@dataclass
class ProblemData:
    f: object = None  # f(x, y, t) -> (..., 2); None means zero forcing
    g_d: object = None
    v0: object = None


@dataclass
class SlabContext:
    disc: Discretization
    params: ModelParams
    config: DiscretizationConfig
    data: ProblemData
    basis: TimeBasis
    tmat: TimeMatrices
    t_start: float
    tau: float
    v_minus: np.ndarray

    def __post_init__(self):
        if self.tau <= 0.0:
            raise ValueError("tau must be positive")

    @property
    def node_times(self):
        return self.t_start + self.tau * self.basis.nodes

    @property
    def n_nodes(self):
        return self.basis.k + 1

    @property
    def ndof(self):
        return self.n_nodes * self.disc.ndof


def make_context(nx, ny, k, params: ModelParams, tau, *, extents=(0.0, 0.0, 1.0, 1.0), neumann_sides=(),
                 config: DiscretizationConfig | None = None, f=None, t_start=0.0, v_minus=None,
                 pressure: str = "p1disc") -> SlabContext:
    """Convenience constructor for a slab context on a uniform mesh
    (pressure="q1": the Taylor-Hood pair)."""
    mesh = tag_sides(QuadMesh(nx, ny, *extents), neumann_sides)
    disc = Discretization(mesh, pressure)
    basis = gauss_radau(k)
    tmat = temporal_matrices(basis)
    if v_minus is None:
        v_minus = np.zeros(disc.n_velocity)
    return SlabContext(disc, params, config or DiscretizationConfig(), ProblemData(f=f), basis, tmat, t_start, tau,
                       np.asarray(v_minus, dtype=float))
