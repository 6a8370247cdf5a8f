"""Is the weak V-cycle preconditioning of the cfg5 solve (profiles/solve_cfg5_r01.json)
reference behaviour?  Runs the REFERENCE (pdflow, build container only) on a
32^2 analogue of BASELINE configs[4] (p=1.2, delta=1e-4, nu_inf=0, DG(1),
tau=0.01, the synth.py modal state, modified Newton): the first Newton
system J dU = R at the synthetic state, solved by pdflow's own FGMRES in the
M-norm (rtol 1e-2, restart 30) with its StmgPreconditioner (Galerkin, 2+2
sweeps, omega=0.7, surrogate patches at rep_fraction 1.0) on 2..5 levels, and
without a preconditioner.  usage: PYTHONPATH=/root/reference/pkg/src python
scripts/check_vcycle_reference.py [n]"""
import dataclasses
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, "/root/reference/pkg/src")

from pdflow import constitutive as law  # noqa: E402
from pdflow.forms import Discretization, DiscretizationConfig, ProblemData  # noqa: E402
from pdflow.mesh import DIRICHLET, boundary_tag_assign, uniform_mesh  # noqa: E402
from pdflow.slab import SlabContext, SlabJacobian, slab_residual  # noqa: E402
from pdflow.solver.krylov import KrylovConfig, fgmres  # noqa: E402
from pdflow.solver.multigrid import MgConfig, MgGeometry, StmgPreconditioner  # noqa: E402
from pdflow.solver.newton import MassNorm  # noqa: E402
from pdflow.timebasis import gauss_radau, temporal_matrices  # noqa: E402

from paper_2603_28706_b200.synth import CONFIGS, make_slab_inputs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
cfg = dataclasses.replace(CONFIGS["cfg5"], nx=n, ny=n)
mesh = boundary_tag_assign(uniform_mesh(n, n), lambda f: DIRICHLET)
disc = Discretization(mesh)
basis = gauss_radau(cfg.k)
syn = make_slab_inputs(cfg, nodes=basis.nodes)
ctx = SlabContext(disc=disc, params=law.ModelParams(cfg.p, cfg.delta, cfg.nu, cfg.nu_inf),
                  config=DiscretizationConfig(gamma1=cfg.gamma1, gamma2=cfg.gamma2, gamma_cip=cfg.gamma_cip),
                  data=ProblemData(f=lambda x, y, t: np.zeros(np.shape(x) + (2,)), g_d=None, v0=None),
                  basis=basis, tmat=temporal_matrices(basis), t_start=0.0, tau=cfg.tau, v_minus=syn.v_minus)
variant = law.modified_newton(cfg.nu)
R = slab_residual(ctx, syn.U).reshape(-1)
jac = SlabJacobian(ctx, syn.U, variant)
norm = MassNorm(ctx)
kc = KrylovConfig(restart=30, max_iters=60)
print(f"reference pdflow, {n}x{n} cfg5 recipe (p={cfg.p}, delta={cfg.delta}, nu_inf={cfg.nu_inf}), |R|_M = {norm.norm(R):.4e}")
res = fgmres(jac.matvec, R, 1e-2, kc, precond=None, mass=norm)
print(f"  no preconditioner: {res.iterations} FGMRES iterations, converged={res.converged}, |r| {res.residual_norm:.3e}")
for levels in (2, 3, 4, 5):
    min_cells = n >> (levels - 1)
    mg = MgConfig(rep_fraction=1.0, min_cells=min_cells, omega=cfg.omega)
    geom = MgGeometry.from_fine(disc, min_cells=min_cells)
    t0 = time.time()
    pre = StmgPreconditioner(geom, ctx, syn.U, variant, mg)
    res = fgmres(jac.matvec, R, 1e-2, kc, precond=pre.apply, mass=norm)
    print(f"  STMG {geom.num_levels} levels (coarsest {n >> (levels - 1)}^2): {res.iterations} FGMRES iterations, "
          f"converged={res.converged}, |r| {res.residual_norm:.3e}  ({time.time() - t0:.1f} s)")
