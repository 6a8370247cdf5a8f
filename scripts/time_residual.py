"""Device time of the slab residual (pdst_residual, device pointers) at a config."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_28706_b200 import _lib as L
from paper_2603_28706_b200 import problem as pb
from paper_2603_28706_b200.operators import SlabDevice
from paper_2603_28706_b200.synth import CONFIGS, make_slab_inputs

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = CONFIGS[name]
params = pb.ModelParams(cfg.p, cfg.delta, cfg.nu, cfg.nu_inf)
conf = pb.DiscretizationConfig(cfg.gamma1, cfg.gamma2, cfg.gamma_cip)
syn = make_slab_inputs(cfg)
ctx = pb.make_context(cfg.nx, cfg.ny, cfg.k, params, cfg.tau, config=conf, v_minus=syn.v_minus)
dev = SlabDevice(ctx)
U = torch.as_tensor(syn.U, device="cuda").reshape(-1)
vm = torch.as_tensor(syn.v_minus, device="cuda")
R = torch.empty_like(U)
w = dev.where(U, vm, R)
call = lambda: L.check(L.lib().pdst_residual(dev.h, L.vptr(U), L.vptr(vm), None, None, L.vptr(R), w))
for _ in range(3): call()
torch.cuda.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for _ in range(20):
    flush.fill_(1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); call(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
ts.sort()
N = U.numel()
print(f"{name}: residual cold-L2 median {ts[len(ts)//2]:.1f} us ({N / ts[len(ts)//2] / 1e3:.2f} GDoF/s)")
