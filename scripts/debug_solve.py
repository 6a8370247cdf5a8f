"""Small-mesh probe of the FGMRES + STMG Newton step with the synth recipe."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dataclasses
import numpy as np, torch
from paper_2603_28706_b200 import problem as pb
from paper_2603_28706_b200.krylov import KrylovConfig, fgmres
from paper_2603_28706_b200.operators import MassNorm, SlabJacobian, slab_residual
from paper_2603_28706_b200.stmg import MgConfig, StmgPreconditioner
from paper_2603_28706_b200.synth import CONFIGS, make_slab_inputs

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
cfg = dataclasses.replace(CONFIGS["cfg2"], nx=n, ny=n)
params = pb.ModelParams(cfg.p, cfg.delta, cfg.nu, cfg.nu_inf)
conf = pb.DiscretizationConfig(cfg.gamma1, cfg.gamma2, cfg.gamma_cip)
syn = make_slab_inputs(cfg)
ctx = pb.make_context(cfg.nx, cfg.ny, cfg.k, params, cfg.tau, config=conf, v_minus=syn.v_minus)
var = pb.modified_newton(cfg.nu)
U = torch.as_tensor(syn.U, device="cuda")
R = slab_residual(ctx, U)
norm = MassNorm(ctx)
jac = SlabJacobian(ctx, U, var)
print("R finite", bool(torch.isfinite(R).all()), "|R|_M", norm.norm(R))
for mc, cs in ((n // 4, "dense"), (n // 4, "fgmres"), (n, "fgmres")):
    try:
        pre = StmgPreconditioner(None, ctx, U, var, MgConfig(min_cells=mc, rep_fraction=1.0, coarse_solver=cs))
    except Exception as e:
        print("build failed", mc, cs, e); continue
    z = pre.apply(R.reshape(-1))
    Jz = jac.matvec(z)
    print(f"min_cells={mc} {cs} levels={pre.num_levels}: z finite {bool(torch.isfinite(z).all())} |z| {float(z.norm()):.3e} "
          f"|R - J z|_M / |R|_M = {norm.norm(R.reshape(-1) - Jz) / norm.norm(R):.3e}")
    res = fgmres(jac.matvec, R.reshape(-1), 1e-2, KrylovConfig(restart=30, max_iters=30), precond=pre.apply, mass=norm)
    print("   fgmres", res.iterations, res.converged, res.residual_norm, res.target)
res = fgmres(jac.matvec, R.reshape(-1), 1e-2, KrylovConfig(restart=30, max_iters=30), precond=None, mass=norm)
print("no precond fgmres", res.iterations, res.converged, res.residual_norm, res.target)
