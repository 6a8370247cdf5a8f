"""Nonlinear slab solves (Picard / exact / modified Newton) on the GPU.

Drop-in counterpart of ``pdflow.solver.newton`` (newton.py:33-298): same
``NewtonConfig``, ``NewtonStepStats``, ``SlabStats``, ``nonlinear_solve_slab``
and ``make_slab_solver``; same Eisenstat-Walker forcing (choice 2 with the
power safeguard and cap, newton.py:140-148), Armijo backtracking on
phi = 1/2 |R|_M^2 (newton.py:230-251), preconditioner rebuild policy
(multigrid.py:343-350), convergence tests and SlabSolveError kinds.  The state
``U``, residuals and Newton updates stay on the device: the residual
(``pdst_residual``), the Jacobian (``pdst_linearize`` + apply), the STMG
V-cycle, FGMRES (``krylov.fgmres``) and the mass norm are libpdst calls; only
scalars (norms, forcing terms, step lengths) come back to the host.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import SlabSolveError
from .krylov import KrylovConfig, fgmres
from .operators import MassNorm, SlabDevice, SlabJacobian, slab_residual
from .problem import PIC
from .stmg import MgConfig, StmgFactory

__all__ = ["NewtonConfig", "NewtonStepStats", "SlabStats", "nonlinear_solve_slab", "make_slab_solver",
           "rebuild_policy", "StmgFactory", "MgConfig", "KrylovConfig"]


@dataclass
class NewtonConfig:
    """Termination, globalization and forcing parameters (newton.py:33-56)."""

    variant: object
    abs_tol: float = 1.0e-12
    rel_tol: float = 1.0e-10
    max_nonlinear: int = 50
    armijo_c1: float = 1.0e-4
    armijo_backtrack: float = 0.5
    armijo_lambda_min: float = 2.0**-10
    forcing_eta0: float = 1.0e-2
    forcing_exponent: float = 2.0
    forcing_gamma: float = 0.9
    forcing_cap: float = 0.9
    forcing_safeguard: float = 0.1
    picard_fixed_tol: float = 1.0e-4

    def __post_init__(self):
        if self.abs_tol <= 0.0 or self.rel_tol <= 0.0:
            raise ValueError("tolerances must be positive")
        if not 0.0 < self.armijo_c1 < 1.0:
            raise ValueError("armijo_c1 must lie in (0, 1)")


@dataclass
class NewtonStepStats:
    n_l: int
    lam: float
    eta: float
    res_before: float
    res_after: float
    lin_res: float
    rebuilt: bool


@dataclass
class SlabStats:
    steps: list = field(default_factory=list)
    initial_res: float = 0.0
    final_res: float = 0.0
    converged: bool = False
    failure: str | None = None

    @property
    def n_nl(self) -> int:
        return len(self.steps)

    @property
    def n_l_total(self) -> int:
        return sum(s.n_l for s in self.steps)

    @property
    def rebuilds(self) -> int:
        return sum(1 for s in self.steps if s.rebuilt)


def rebuild_policy(residual_ratio: float, last_n_l: int, previous_n_l: int, rho: float, factor: float) -> bool:
    """Rebuild on a stalling residual or a Krylov blow-up (multigrid.py:343-350)."""
    if residual_ratio > rho:
        return True
    if previous_n_l > 0 and last_n_l > factor * previous_n_l:
        return True
    return False


def _forcing(newton: NewtonConfig, m: int, rnorm: float, rnorm_prev: float, eta_prev: float) -> float:
    if m == 0:
        return newton.forcing_eta0
    eta = newton.forcing_gamma * (rnorm / rnorm_prev) ** newton.forcing_exponent
    guard = newton.forcing_gamma * eta_prev**newton.forcing_exponent
    if guard > newton.forcing_safeguard:
        eta = max(eta, guard)
    return min(eta, newton.forcing_cap)


def _all_dirichlet(ctx) -> bool:
    from .problem import dirichlet_flags

    return bool((dirichlet_flags(ctx.disc.mesh) == 1).all())


def _normalize_pressure(ctx, U):
    """Zero the area-weighted mean of the constant pressure mode per Radau
    node when no Neumann face exists (newton.py:151-165).  Uniform mesh: all
    cell areas are equal, so the weighted mean is the plain mean."""
    if not _all_dirichlet(ctx):
        return U
    mv = ctx.disc.n_velocity
    out = U.clone()
    p0 = out[:, mv::3]
    p0 -= p0.mean(dim=1, keepdim=True)
    return out


def nonlinear_solve_slab(ctx, U0, newton: NewtonConfig, krylov: KrylovConfig | None = None,
                         precond_factory: StmgFactory | None = None, device=0):
    """Solve R_n(U) = 0 on one slab (newton.py:168-284).  U0 may be numpy
    (result returned as numpy) or a device tensor."""
    import torch

    krylov = krylov or KrylovConfig()
    host_io = not isinstance(U0, torch.Tensor)
    dev_t = torch.device("cuda", device)
    U = torch.as_tensor(np.ascontiguousarray(U0, dtype=np.float64), device=dev_t) if host_io else \
        U0.to(torch.float64).clone()
    sd = SlabDevice(ctx, device)            # residuals and norms
    jd = SlabDevice(ctx, device)            # the Newton Jacobian (re-linearized in place)
    norm = MassNorm(ctx, dev=sd)
    is_picard = newton.variant.kind == PIC

    def residual(V):
        return slab_residual(ctx, V, dev=sd)

    def out(V):
        return V.cpu().numpy() if host_io else V

    R = residual(U)
    rnorm = norm.norm(R)
    stats = SlabStats(initial_res=rnorm)
    r0 = rnorm
    precond = None
    eta_prev = newton.forcing_eta0
    rnorm_prev = rnorm
    prev_n_l = 0
    try:
        for m in range(newton.max_nonlinear):
            if rnorm <= newton.abs_tol or rnorm <= newton.rel_tol * r0:
                stats.converged = True
                stats.final_res = rnorm
                return out(_normalize_pressure(ctx, U)), stats
            jac = SlabJacobian(ctx, U, newton.variant, dev=jd)
            rebuilt = False
            if precond_factory is not None:
                ratio = rnorm / rnorm_prev if m > 0 else 0.0
                last_n_l = stats.steps[-1].n_l if stats.steps else 0
                if precond is None or rebuild_policy(ratio, last_n_l, prev_n_l, precond_factory.mg.rebuild_rho,
                                                     precond_factory.mg.rebuild_factor):
                    precond = precond_factory.build(ctx, U, newton.variant)
                    rebuilt = True
                prev_n_l = stats.steps[-1].n_l if stats.steps else 0
            eta = newton.picard_fixed_tol if is_picard else _forcing(newton, m, rnorm, rnorm_prev, eta_prev)
            result = fgmres(jac.matvec, R.reshape(-1), eta, krylov,
                            precond=precond.apply if precond is not None else None, mass=norm)
            if not result.converged:
                stats.failure = "krylov"
                stats.final_res = rnorm
                raise SlabSolveError("krylov", f"FGMRES stalled at |r|={result.residual_norm:.3e} "
                                               f"(target {result.target:.3e})", stats)
            dU = result.x.reshape(U.shape)
            phi = 0.5 * rnorm**2
            lam = 1.0
            if is_picard:
                U = U + dU
                R_new = residual(U)
                rnorm_new = norm.norm(R_new)
            else:
                while True:
                    U_try = U + lam * dU
                    R_new = residual(U_try)
                    rnorm_new = norm.norm(R_new)
                    if 0.5 * rnorm_new**2 <= (1.0 - newton.armijo_c1 * lam) * phi:
                        U = U_try
                        break
                    lam *= newton.armijo_backtrack
                    if lam < newton.armijo_lambda_min:
                        stats.failure = "line_search"
                        stats.final_res = rnorm
                        raise SlabSolveError("line_search",
                                             f"no sufficient decrease above lambda={lam:.2e} at |R|={rnorm:.3e}",
                                             stats)
            stats.steps.append(NewtonStepStats(n_l=result.iterations, lam=lam, eta=eta, res_before=rnorm,
                                               res_after=rnorm_new, lin_res=result.residual_norm, rebuilt=rebuilt))
            rnorm_prev = rnorm
            rnorm = rnorm_new
            eta_prev = eta
            R = R_new
        if rnorm <= newton.abs_tol or rnorm <= newton.rel_tol * r0:
            stats.converged = True
            stats.final_res = rnorm
            return out(_normalize_pressure(ctx, U)), stats
        stats.failure = "max_iterations"
        stats.final_res = rnorm
        raise SlabSolveError("max_iterations", f"|R|={rnorm:.3e} after {newton.max_nonlinear} iterations (target "
                                               f"abs {newton.abs_tol:.1e} / rel {newton.rel_tol * r0:.1e})", stats)
    finally:
        torch.cuda.synchronize(dev_t)


def make_slab_solver(newton: NewtonConfig, krylov: KrylovConfig | None = None,
                     precond_factory: StmgFactory | None = None, device=0):
    """``solve(ctx, U0) -> (U, stats)`` for time marching (newton.py:287-298)."""

    def solve(ctx, U0):
        return nonlinear_solve_slab(ctx, U0, newton, krylov, precond_factory, device=device)

    return solve
