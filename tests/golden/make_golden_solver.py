"""Generate FGMRES / Newton fixtures by running the
REFERENCE's own solvers (pdflow.solver.krylov.fgmres,
pdflow.solver.newton.nonlinear_solve_slab) in this build container.
Run once:  python tests/golden/make_golden_solver.py [names...]
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np
import scipy

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import build_ctx  # noqa: E402  (puts the reference on sys.path)

from pdflow import constitutive as law  # noqa: E402
from pdflow.bench.manufactured import ManufacturedCase  # noqa: E402
from pdflow.forms import Discretization, DiscretizationConfig  # noqa: E402
from pdflow.mesh import DIRICHLET, NEUMANN, boundary_tag_assign, uniform_mesh  # noqa: E402
from pdflow.slab import SlabJacobian, SlabProblem, SlabSolveError, initial_guess, slab_residual  # noqa: E402
from pdflow.timebasis import gauss_radau  # noqa: E402
from pdflow.solver.krylov import KrylovConfig, fgmres  # noqa: E402
from pdflow.solver.multigrid import MgConfig, MgGeometry, StmgPreconditioner  # noqa: E402
from pdflow.solver.newton import MassNorm, NewtonConfig, StmgFactory, nonlinear_solve_slab  # noqa: E402

from cases import SOLVER_CASES  # noqa: E402
from paper_2603_28706_b200.operators import forcing_at_qp  # noqa: E402


def gen_fgmres(sc):
    ctx, variant, syn, _ = build_ctx(sc.case)
    mg = MgConfig(min_cells=sc.min_cells)
    geom = MgGeometry.from_fine(ctx.disc, min_cells=sc.min_cells)
    kc = KrylovConfig(restart=sc.restart, max_iters=sc.max_iters)
    jac = SlabJacobian(ctx, syn.U, variant)
    rhs = slab_residual(ctx, syn.U).reshape(-1)
    pre = StmgPreconditioner(geom, ctx, syn.U, variant, mg) if "noprec" not in sc.name else None
    res = fgmres(jac.matvec, rhs, sc.tol, kc, precond=pre.apply if pre else None, mass=MassNorm(ctx))
    print(sc.name, "iters", res.iterations, "res", res.residual_norm, "target", res.target)
    return dict(U0=syn.U, v_minus=syn.v_minus, nodes=ctx.basis.nodes, weights=ctx.basis.weights, K_t=ctx.tmat.K_t,
                m_t=ctx.tmat.m_t, tags=np.array([t == "dirichlet" for t in ctx.disc.mesh.boundary_tags]),
                rhs=rhs, x=res.x, iterations=res.iterations, converged=res.converged,
                residual_norm=res.residual_norm, target=res.target)


def newton_ctx(sc):
    params = law.ModelParams(*sc.params)
    mesh = boundary_tag_assign(uniform_mesh(sc.nx, sc.nx), lambda f: NEUMANN if f.side == "right" else DIRICHLET)
    disc = Discretization(mesh)
    case = ManufacturedCase(params)
    prob = SlabProblem(disc=disc, params=params, config=DiscretizationConfig(), data=case.problem_data(),
                       basis=gauss_radau(sc.k))
    return prob.context(0.0, sc.tau, np.zeros(disc.n_velocity)), params


def gen_newton(sc):
    ctx, params = newton_ctx(sc)
    U0 = initial_guess(ctx)
    variant = {"pic": law.picard(), "exn": law.exact_newton(), "modn": law.modified_newton(params.nu)}[sc.variant]
    mg = MgConfig(min_cells=sc.min_cells, rebuild_rho=sc.rebuild_rho)
    nc = NewtonConfig(variant=variant, abs_tol=sc.abs_tol, rel_tol=sc.rel_tol)
    failure, U = "", None
    try:
        U, stats = nonlinear_solve_slab(ctx, U0, nc, KrylovConfig(restart=sc.restart, max_iters=sc.max_iters),
                                        StmgFactory(MgGeometry.from_fine(ctx.disc, min_cells=sc.min_cells), mg))
    except SlabSolveError as err:
        failure, stats = err.kind, err.diagnostics
    st = stats.steps
    print(sc.name, "steps", len(st), "n_l", [s.n_l for s in st], "lam", [s.lam for s in st],
          "res", stats.initial_res, "->", stats.final_res, "failure", failure)
    c = ctx.config
    out = dict(U0=U0, v_minus=ctx.v_minus, t_start=ctx.t_start, tau=ctx.tau, nodes=ctx.basis.nodes,
               weights=ctx.basis.weights, K_t=ctx.tmat.K_t, m_t=ctx.tmat.m_t,
               gammas=np.array([c.gamma1, c.gamma2, c.gamma_cip]), fq=forcing_at_qp(ctx),
               n_l=np.array([s.n_l for s in st]), lam=np.array([s.lam for s in st]),
               eta=np.array([s.eta for s in st]), res_before=np.array([s.res_before for s in st]),
               res_after=np.array([s.res_after for s in st]), lin_res=np.array([s.lin_res for s in st]),
               rebuilt=np.array([s.rebuilt for s in st]), initial_res=stats.initial_res, final_res=stats.final_res,
               failure=failure)
    if U is not None:
        out["U"] = U
    return out


def gen(sc):
    t = time.time()
    out = gen_fgmres(sc) if sc.kind == "fgmres" else gen_newton(sc)
    out.update(numpy_version=np.__version__, scipy_version=scipy.__version__)
    np.savez_compressed(os.path.join(HERE, f"{sc.name}.npz"), **out)
    print(f"  {time.time() - t:.1f} s")


if __name__ == "__main__":
    names = sys.argv[1:]
    for sc in SOLVER_CASES:
        if not names or sc.name in names:
            gen(sc)
