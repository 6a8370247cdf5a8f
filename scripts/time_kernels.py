"""Quick device timing of the slab kernels at a config (CUDA events)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2603_28706_b200 import problem as pb
from paper_2603_28706_b200.operators import SlabJacobian, slab_residual
from paper_2603_28706_b200.synth import CONFIGS, make_slab_inputs

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = CONFIGS[name]
params = pb.ModelParams(cfg.p, cfg.delta, cfg.nu, cfg.nu_inf)
conf = pb.DiscretizationConfig(cfg.gamma1, cfg.gamma2, cfg.gamma_cip)
t0 = time.time(); syn = make_slab_inputs(cfg); print("synth", time.time() - t0)
ctx = pb.make_context(cfg.nx, cfg.ny, cfg.k, params, cfg.tau, config=conf, v_minus=syn.v_minus)
U = torch.as_tensor(syn.U, device="cuda"); x = torch.as_tensor(syn.x, device="cuda")
jac = SlabJacobian(ctx, U, pb.modified_newton(cfg.nu))
y = torch.empty_like(x)
for _ in range(5): jac.matvec(x, out=y)
torch.cuda.synchronize()
n = 50
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(n): jac.matvec(x, out=y)
e1.record(); torch.cuda.synchronize()
t = e0.elapsed_time(e1) / n * 1e-3
N = x.numel()
print(f"{name}: apply {t*1e6:.1f} us  {N/t/1e9:.2f} GDoF/s  N_dof={N}")
# cold L2: flush (256 MiB write) before every timed apply
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for _ in range(20):
    flush.fill_(1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); jac.matvec(x, out=y); b.record()
    torch.cuda.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
ts.sort()
print(f"{name}: apply cold-L2 median {ts[len(ts)//2]:.1f} us  min {ts[0]:.1f} us")
r = torch.as_tensor(syn.d0, device="cuda")
ts = []
for _ in range(20):
    flush.fill_(1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); jac.defect(x, r, out=y); b.record()
    torch.cuda.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
ts.sort()
print(f"{name}: defect cold-L2 median {ts[len(ts)//2]:.1f} us  min {ts[0]:.1f} us")
R = slab_residual(ctx, U); torch.cuda.synchronize()
e0.record()
for _ in range(n): slab_residual(ctx, U, dev=jac.dev)
e1.record(); torch.cuda.synchronize()
print(f"{name}: residual {e0.elapsed_time(e1)/n*1e3:.1f} us (incl. host forcing/launch)")
