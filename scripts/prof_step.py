"""Small driver for ncu: cfg2 setup + a few (apply + Vanka sweep) steps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_28706_b200 import problem as pb
from paper_2603_28706_b200.operators import SlabJacobian
from paper_2603_28706_b200.smoother import VankaLevel
from paper_2603_28706_b200.synth import CONFIGS, make_slab_inputs

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = CONFIGS[name]
params = pb.ModelParams(cfg.p, cfg.delta, cfg.nu, cfg.nu_inf)
conf = pb.DiscretizationConfig(cfg.gamma1, cfg.gamma2, cfg.gamma_cip)
syn = make_slab_inputs(cfg)
ctx = pb.make_context(cfg.nx, cfg.ny, cfg.k, params, cfg.tau, config=conf, v_minus=syn.v_minus)
U = torch.as_tensor(syn.U, device="cuda"); x = torch.as_tensor(syn.x, device="cuda")
d = torch.as_tensor(syn.d0, device="cuda"); y = torch.empty_like(x)
v = pb.modified_newton(cfg.nu)
jac = SlabJacobian(ctx, U, v)
lvl = VankaLevel(ctx, U, v, surrogate=True, rep_fraction=cfg.rep_fraction, jac=jac)
for _ in range(steps):
    jac.matvec(x, out=y)
    lvl.smooth(d, x, 1, cfg.omega, inplace=True)
torch.cuda.synchronize()
print("ok", float(y.norm()), float(d.norm()))
