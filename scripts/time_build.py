"""Preconditioner build at a config (for an ncu launch list of its kernels)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_28706_b200 import problem as pb
from paper_2603_28706_b200.operators import SlabJacobian
from paper_2603_28706_b200.smoother import VankaLevel
from paper_2603_28706_b200.synth import CONFIGS, make_slab_inputs

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = CONFIGS[name]
params = pb.ModelParams(cfg.p, cfg.delta, cfg.nu, cfg.nu_inf)
conf = pb.DiscretizationConfig(cfg.gamma1, cfg.gamma2, cfg.gamma_cip)
syn = make_slab_inputs(cfg)
ctx = pb.make_context(cfg.nx, cfg.ny, cfg.k, params, cfg.tau, config=conf, v_minus=syn.v_minus)
U = torch.as_tensor(syn.U, device="cuda")
jac = SlabJacobian(ctx, U, pb.modified_newton(cfg.nu))
for _ in range(2):
    VankaLevel(ctx, U, pb.modified_newton(cfg.nu), surrogate=True, rep_fraction=cfg.rep_fraction, jac=jac)
torch.cuda.synchronize()
print("ok")
