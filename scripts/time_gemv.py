"""Device time of one Vanka sweep's kernels at cfg2 (libpdst profiler, L2 flushed)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import torch
from paper_2603_28706_b200 import _lib as L, problem as pb
from paper_2603_28706_b200.operators import SlabJacobian
from paper_2603_28706_b200.smoother import VankaLevel
from paper_2603_28706_b200.synth import CONFIGS, make_slab_inputs
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
params = pb.ModelParams(cfg.p, cfg.delta, cfg.nu, cfg.nu_inf)
conf = pb.DiscretizationConfig(cfg.gamma1, cfg.gamma2, cfg.gamma_cip)
syn = make_slab_inputs(cfg)
ctx = pb.make_context(cfg.nx, cfg.ny, cfg.k, params, cfg.tau, config=conf, v_minus=syn.v_minus)
U = torch.as_tensor(syn.U, device="cuda"); x = torch.as_tensor(syn.x, device="cuda")
d = torch.as_tensor(syn.d0, device="cuda")
v = pb.modified_newton(cfg.nu)
jac = SlabJacobian(ctx, U, v)
lvl = VankaLevel(ctx, U, v, surrogate=True, rep_fraction=cfg.rep_fraction, jac=jac)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(5): lvl.smooth(d, x, 1, cfg.omega, inplace=True)
L.lib().pdst_profile(jac.dev.h, 1)
for _ in range(20):
    flush.fill_(1); lvl.smooth(d, x, 1, cfg.omega, inplace=True)
torch.cuda.synchronize()
for kid, name in ((0, "apply"), (1, "gemv"), (2, "scatter")):
    ms, cnt = C.c_double(), C.c_int64()
    L.lib().pdst_profile_read(jac.dev.h, kid, C.byref(ms), C.byref(cnt))
    print(f"{name}: {ms.value / max(cnt.value, 1) * 1e3:.1f} us")
