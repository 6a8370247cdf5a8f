"""Per-kernel-class device time of one single-domain V-cycle (libpdst profiler).
usage: prof_vcycle.py CONFIG LEVELS"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import torch
from paper_2603_28706_b200 import _lib as L
from paper_2603_28706_b200 import problem as pb
from paper_2603_28706_b200.stmg import MgConfig, StmgPreconditioner
from paper_2603_28706_b200.synth import CONFIGS, make_slab_inputs

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
levels = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = CONFIGS[name]
params = pb.ModelParams(cfg.p, cfg.delta, cfg.nu, cfg.nu_inf)
conf = pb.DiscretizationConfig(cfg.gamma1, cfg.gamma2, cfg.gamma_cip)
syn = make_slab_inputs(cfg)
ctx = pb.make_context(cfg.nx, cfg.ny, cfg.k, params, cfg.tau, config=conf, v_minus=syn.v_minus)
mg = MgConfig(omega=cfg.omega, rep_fraction=cfg.rep_fraction, min_cells=max(1, cfg.nx >> (levels - 1)),
              coarse_solver="fgmres", coarse_sweeps=2, coarse_iters=30, coarse_rtol=1e-6)
U = torch.as_tensor(syn.U, device="cuda")
pre = StmgPreconditioner(None, ctx, U, pb.modified_newton(cfg.nu), mg)
r = torch.as_tensor(syn.x, device="cuda")
z = torch.empty_like(r)
for _ in range(2):
    pre.apply(r, out=z)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); pre.apply(r, out=z); b.record(); torch.cuda.synchronize()
print(f"{name}: V-cycle {a.elapsed_time(b):.2f} ms ({pre.num_levels} levels)")
h = pre.dev.h
L.lib().pdst_profile(h, 1)
pre.apply(r, out=z)
torch.cuda.synchronize()
names = ["jacobian", "vanka_gemv", "vanka_scatter", "residual", "transfer", "level_apply", "defect_apply"]
for k, n in enumerate(names):
    ms, cnt = C.c_double(), C.c_int64()
    L.lib().pdst_profile_read(h, k, C.byref(ms), C.byref(cnt))
    print(f"  {n:14s} {ms.value:8.2f} ms  {cnt.value:5d} launches")
L.lib().pdst_profile(h, 0)
