"""Soak test of the Jacobian apply / defect over many mesh sizes (ragged tiles, one tile, several waves) and
k = 0..2: defect == r - J x bitwise, and 12 repeated launches without host synchronization reproduce the first
result bit for bit (the epilogue runs under the tile pass behind completion counters).  B200: 101 cases, 0 bad."""
import sys, os, random
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2603_28706_b200 import problem as pb
from paper_2603_28706_b200.operators import SlabJacobian
from paper_2603_28706_b200.synth import SynthConfig, make_slab_inputs
random.seed(7)
bad = 0; n = 0
sizes = [(1,1),(16,16),(17,16),(16,17),(33,47),(160,15),(15,160),(148*1,16),(200,200),(256,130),(64,320)] + [(random.randint(1,220), random.randint(1,220)) for _ in range(24)]
for (nx, ny) in sizes:
    for k in (0, 1, 2):
        if k == 2 and nx * ny > 30000: continue
        cfg = SynthConfig("soak", nx, ny, k, 1.3, 1.0e-3, 1.0, 0.0, 4, 11 + nx + 7 * ny)
        syn = make_slab_inputs(cfg)
        params = pb.ModelParams(cfg.p, cfg.delta, cfg.nu, cfg.nu_inf)
        ctx = pb.make_context(nx, ny, k, params, cfg.tau, config=pb.DiscretizationConfig(cfg.gamma1, cfg.gamma2, cfg.gamma_cip), v_minus=syn.v_minus)
        U = torch.as_tensor(syn.U, device="cuda"); x = torch.as_tensor(syn.x, device="cuda"); r = torch.as_tensor(syn.d0, device="cuda")
        jac = SlabJacobian(ctx, U, pb.modified_newton(cfg.nu))
        y0 = jac.matvec(x).clone(); d0 = jac.defect(x, r).clone()
        torch.cuda.synchronize()
        if not torch.equal(d0, r - y0): bad += 1; print("defect != r - Jx", nx, ny, k)
        y = torch.empty_like(x); d = torch.empty_like(x)
        acc = torch.zeros((), dtype=torch.int64, device="cuda")
        for _ in range(12):
            y.zero_(); d.zero_()
            jac.matvec(x, out=y); jac.defect(x, r, out=d)
            acc += (y != y0).any().long() + (d != d0).any().long()
        if int(acc.item()): bad += 1; print("nondeterministic", nx, ny, k, int(acc.item()))
        n += 1
        del jac
print("soak:", n, "cases,", bad, "bad")
