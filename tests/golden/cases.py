"""Golden-case definitions shared by the fixture generator (run once, in the
build container, against the reference) and the tests (run anywhere).

Each case names a mesh, a time degree, a linearization and discretization
options; inputs come from ``paper_2603_28706_b200.synth`` with a fixed seed
so the fixture stores only what the reference computed plus the inputs
needed to recompute them.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

from paper_2603_28706_b200.synth import SynthConfig, CONFIGS


def forcing_a(x, y, t):
    """A smooth body force used by the f != 0 residual case; returns (..., 2)."""
    return np.stack([np.sin(2.0 * x + 1.0) * np.cos(y) + t, x * y - 0.5 * t * np.cos(3.0 * y)], axis=-1)


FORCINGS = {"zero": None, "a": forcing_a}


def ghat_field(X, Y):
    """Velocity field whose Q2 interpolant is used as the Nitsche lifting g_hat."""
    return np.stack([0.3 * np.sin(np.pi * X) * np.cos(0.5 * Y) + 0.1, -0.2 * X * Y + 0.05 * np.cos(2 * X)], axis=-1)


@dataclass(frozen=True)
class Case:
    name: str
    cfg: SynthConfig
    variant: str = "modn"
    sigma_max: float | None = None  # None -> nu (harness.py:49-58)
    neumann_sides: tuple = ()  # subset of ("bottom", "right", "top", "left")
    ghat: bool = False
    forcing: str = "zero"
    t_start: float = 0.0
    patches: bool = False  # also build STMG patches / Vanka / V-cycle
    surrogate: bool = True
    min_cells: int = 4
    coarse_mode: str = "galerkin"  # MgConfig.coarse_mode (multigrid.py:302-324)


def _cfg(name, nx, ny, k, p=1.5, delta=1e-2, nu=1.0, nu_inf=1e-3, modes=4, seed=1, **kw):
    return SynthConfig(name, nx, ny, k, p, delta, nu, nu_inf, modes, seed, **kw)


CASES = [
    Case("cfg1", CONFIGS["cfg1"], patches=True),
    Case("cfg1_exact", replace(CONFIGS["cfg1"], name="cfg1_exact"), patches=True, surrogate=False),
    Case("cfg1_pic", replace(CONFIGS["cfg1"], name="cfg1_pic"), variant="pic"),
    Case("cfg1_exn", replace(CONFIGS["cfg1"], name="cfg1_exn"), variant="exn"),
    Case("n1_k0_pic", _cfg("n1_k0_pic", 1, 1, 0, seed=11), variant="pic"),
    Case("n1_k1_exn", _cfg("n1_k1_exn", 1, 1, 1, seed=12), variant="exn"),
    Case("n2_k1_modn", _cfg("n2_k1_modn", 2, 2, 1, seed=13, p=1.3, delta=1e-3, nu_inf=0.0)),
    Case("rect_k2_exn", _cfg("rect_k2_exn", 3, 2, 2, seed=14, extents=(0.0, -0.5, 2.0, 1.0)), variant="exn", t_start=0.3),
    Case("n4_k0_modn", _cfg("n4_k0_modn", 4, 4, 0, seed=15), sigma_max=0.05),
    Case("n4_k2_pic", _cfg("n4_k2_pic", 4, 4, 2, seed=16, p=1.1, delta=1e-4, nu_inf=1e-4), variant="pic"),
    Case("n4_ghat_exn", _cfg("n4_ghat_exn", 4, 4, 1, seed=17), variant="exn", ghat=True),
    Case("n4_neumann", _cfg("n4_neumann", 4, 4, 1, seed=18), neumann_sides=("right",)),
    Case("n4_forcing", _cfg("n4_forcing", 4, 4, 1, seed=19), forcing="a", t_start=0.25),
    Case("n5x3_mixed", _cfg("n5x3_mixed", 5, 3, 1, seed=20, gamma1=1e3, gamma2=5e2, gamma_cip=0.5),
         variant="exn", neumann_sides=("top", "left"), ghat=True, forcing="a"),
    # Patch / Vanka / V-cycle cases (levels: 6 -> 3, 8 -> 4).
    Case("p6_k0_exn", _cfg("p6_k0_exn", 6, 6, 0, seed=21), variant="exn", patches=True),
    Case("p6_k1_modn", _cfg("p6_k1_modn", 6, 6, 1, seed=22), patches=True),
    Case("p6_k2_pic_exact", _cfg("p6_k2_pic_exact", 6, 6, 2, seed=23, p=1.3, delta=1e-3), variant="pic",
         patches=True, surrogate=False),
    Case("p6_neumann_ghat", _cfg("p6_neumann_ghat", 6, 6, 1, seed=24), variant="exn", patches=True,
         neumann_sides=("bottom",), ghat=True),
    Case("p8_k1_exn_rect", _cfg("p8_k1_exn_rect", 8, 4, 1, seed=25, extents=(0.0, 0.0, 2.0, 1.0)), variant="exn",
         patches=True, min_cells=2),
    # coarse_mode="rediscretize": coarse levels re-linearized at the injected state
    Case("p6_k1_modn_redisc", _cfg("p6_k1_modn_redisc", 6, 6, 1, seed=26), patches=True, coarse_mode="rediscretize"),
    Case("p8_ghat_redisc", _cfg("p8_ghat_redisc", 8, 8, 1, seed=27), variant="exn", patches=True, min_cells=2,
         neumann_sides=("bottom",), ghat=True, coarse_mode="rediscretize"),
    Case("p8_k2_pic_redisc", _cfg("p8_k2_pic_redisc", 8, 8, 2, seed=28, p=1.3, delta=1e-3), variant="pic",
         patches=True, min_cells=2, surrogate=False, coarse_mode="rediscretize"),
]

CASE_BY_NAME = {c.name: c for c in CASES}

TRANSFER_PAIRS = [(1, 1), (2, 2), (3, 3), (4, 2), (4, 4)]  # coarse (nx, ny); fine is 2x


@dataclass(frozen=True)
class SolverCase:
    """FGMRES / Newton fixtures (f1).

    fgmres: the slab case's Jacobian at the synthetic state, rhs = its
    residual, STMG preconditioner (or none) and the mass norm.
    newton: the first slab of the reference's benchmark problem
    (bench/harness.py:91-115: unit square, manufactured forcing, v0 = 0,
    default discretization), with a Neumann right side, solved by
    nonlinear_solve_slab with an STMG factory.  Runs that end in the
    reference's SlabSolveError are fixtures too (partial statistics + kind)."""

    name: str
    kind: str  # "fgmres" or "newton"
    case: Case | None = None  # fgmres
    tol: float = 1e-8
    restart: int = 60
    max_iters: int = 300
    params: tuple = (1.5, 1e-2, 1.0, 1e-3)  # newton: (p, delta, nu, nu_inf)
    variant: str = "modn"
    nx: int = 8
    k: int = 1
    tau: float = 0.1
    min_cells: int = 4
    rebuild_rho: float = 0.9
    abs_tol: float = 1e-12
    rel_tol: float = 1e-10


SOLVER_CASES = [
    # a Neumann side removes the constant-pressure null space of the all-Dirichlet slab
    SolverCase("fg_p8_modn", "fgmres", Case("fg_p8_modn", _cfg("fg_p8_modn", 8, 8, 1, seed=31, gamma1=1e3,
                                                                gamma2=1e3), neumann_sides=("right",)),
               tol=1e-6, restart=20, max_iters=80),
    SolverCase("fg_p8_exn_noprec", "fgmres", Case("fg_p8_exn_noprec", _cfg("fg_p8_exn_noprec", 8, 8, 0, seed=32),
                                                  variant="exn", neumann_sides=("top",)),
               tol=1e-6, restart=30, max_iters=90),
    # single-level STMG (exact coarse solve), rebuilt every step: converges at abs_tol 1e-6
    SolverCase("nw_h8_modn_conv", "newton", min_cells=8, rebuild_rho=0.0, abs_tol=1e-6),
    SolverCase("nw_h8_exn_conv", "newton", variant="exn", params=(1.3, 1e-3, 1.0, 0.0), min_cells=8,
               rebuild_rho=0.0, abs_tol=1e-6),
    SolverCase("nw_h8_pic_k0", "newton", variant="pic", k=0, min_cells=8, rebuild_rho=0.0, abs_tol=1e-6),
    # default tolerances: the reference stops with SlabSolveError("krylov") after 3 steps
    SolverCase("nw_h8_modn_fail", "newton", min_cells=8, rebuild_rho=0.0),
]
SOLVER_BY_NAME = {c.name: c for c in SOLVER_CASES}
