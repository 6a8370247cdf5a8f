"""The product's counterpart of scripts/check_vcycle_reference.py (GPU):
the same 32^2 cfg5-recipe Newton system through this package's FGMRES and
StmgPreconditioner (dense coarsest solve like the reference)."""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_28706_b200 import problem as pb  # noqa: E402
from paper_2603_28706_b200.krylov import KrylovConfig, fgmres  # noqa: E402
from paper_2603_28706_b200.operators import MassNorm, SlabJacobian, slab_residual  # noqa: E402
from paper_2603_28706_b200.stmg import MgConfig, StmgPreconditioner  # noqa: E402
from paper_2603_28706_b200.synth import CONFIGS, make_slab_inputs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
cfg = dataclasses.replace(CONFIGS["cfg5"], nx=n, ny=n)
params = pb.ModelParams(cfg.p, cfg.delta, cfg.nu, cfg.nu_inf)
conf = pb.DiscretizationConfig(cfg.gamma1, cfg.gamma2, cfg.gamma_cip)
syn = make_slab_inputs(cfg)
ctx = pb.make_context(n, n, cfg.k, params, cfg.tau, config=conf, v_minus=syn.v_minus)
var = pb.modified_newton(cfg.nu)
U = torch.as_tensor(syn.U, device="cuda")
R = slab_residual(ctx, U).reshape(-1)
jac = SlabJacobian(ctx, U, var)
norm = MassNorm(ctx, dev=jac.dev)
kc = KrylovConfig(restart=30, max_iters=60)
print(f"product (GPU), {n}x{n} cfg5 recipe, |R|_M = {norm.norm(R):.4e}")
res = fgmres(jac.matvec, R, 1e-2, kc, precond=None, mass=norm)
print(f"  no preconditioner: {res.iterations} FGMRES iterations, converged={res.converged}, |r| {res.residual_norm:.3e}")
for levels in (2, 3, 4, 5):
    mc = n >> (levels - 1)
    pre = StmgPreconditioner(None, ctx, U, var, MgConfig(rep_fraction=1.0, min_cells=mc, omega=cfg.omega), jac=jac)
    res = fgmres(jac.matvec, R, 1e-2, kc, precond=pre.apply, mass=norm)
    print(f"  STMG {pre.num_levels} levels (coarsest {mc}^2): {res.iterations} FGMRES iterations, "
          f"converged={res.converged}, |r| {res.residual_norm:.3e}")
