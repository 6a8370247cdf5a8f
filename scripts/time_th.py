"""Device time of the Taylor-Hood Q2/Q1 Jacobian apply (pressure_space = 1) next to the P1disc one at a
BASELINE config's mesh and parameters (CUDA events, cold L2)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2603_28706_b200 import problem as pb
from paper_2603_28706_b200.operators import SlabJacobian
from paper_2603_28706_b200.radau import gauss_radau, temporal_matrices
from paper_2603_28706_b200.synth import CONFIGS, make_slab_inputs

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = CONFIGS[name]
syn = make_slab_inputs(cfg)
params = pb.ModelParams(cfg.p, cfg.delta, cfg.nu, cfg.nu_inf)
conf = pb.DiscretizationConfig(cfg.gamma1, cfg.gamma2, cfg.gamma_cip)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda"); rd = torch.zeros_like(flush)
for space in ("p1disc", "q1"):
    mesh = pb.QuadMesh(cfg.nx, cfg.ny, 0.0, 0.0, 1.0, 1.0)
    disc = pb.Discretization(mesh, space) if space == "q1" else pb.Discretization(mesh)
    b = gauss_radau(cfg.k); tm = temporal_matrices(b)
    mv, nd = disc.n_velocity, disc.ndof
    rng = np.random.default_rng(1)
    U = np.zeros((cfg.k + 1, nd)); U[:, :mv] = syn.U[:, :mv]; U[:, mv:] = rng.uniform(-1, 1, (cfg.k + 1, nd - mv))
    ctx = pb.SlabContext(disc, params, conf, pb.ProblemData(f=None), b, tm, 0.0, cfg.tau, syn.v_minus)
    Ud = torch.as_tensor(U, device="cuda"); x = torch.as_tensor(rng.uniform(-1, 1, (cfg.k + 1) * nd), device="cuda")
    jac = SlabJacobian(ctx, Ud, pb.modified_newton(cfg.nu)); y = torch.empty_like(x)
    for _ in range(3): jac.matvec(x, out=y)
    ts = []
    for _ in range(15):
        flush.fill_(1); rd.sum()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); jac.matvec(x, out=y); e.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(e) * 1e3)
    ts.sort()
    print(f"{name} {space}: N_dof {x.numel()}, apply cold-L2 median {ts[len(ts)//2]:.1f} us ({x.numel() / ts[len(ts)//2] / 1e3:.2f} GDoF/s)")
