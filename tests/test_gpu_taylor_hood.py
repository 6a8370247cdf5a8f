"""Taylor-Hood Q2/Q1 on the GPU (pressure_space = 1, csrc/pdst_th.cu; BASELINE
north_star (1)) against the self-checked restatement
oracle/th_oracle.py (the reference has no Taylor-Hood pair, so the oracle is
pinned by tests/test_th_oracle.py instead of reference vectors), plus
properties at the cfg2 size:

* Jacobian apply, slab residual (incl. a g_hat lifting, forcing, Neumann
  sides) and the block mass / mass norm at relative 1e-12;
* the pressure coupling tested both ways: <G u, q> = <u, G' q>, with the
  Jacobian's own velocity-pressure blocks;
* all-Dirichlet: the per-node constant pressure is in the kernel of J;
* linearity; exact Newton = d(residual) with frozen lagged weights;
* the P1disc-only entry points (Vanka, multigrid) refuse Taylor-Hood handles.
"""

import numpy as np
import pytest

from helpers import assert_close, orc
from oracle import th_oracle as th

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _case(nx, ny, k, variant="exn", neumann=(), ghat=False, forcing=False, seed=0):
    import dataclasses

    from cases import forcing_a

    from paper_2603_28706_b200 import problem as pb
    from paper_2603_28706_b200.radau import gauss_radau, temporal_matrices

    rng = np.random.default_rng(seed + 100 * nx + ny)
    ext = (0.0, 0.0, 1.3, 1.0)
    mesh = pb.tag_sides(pb.QuadMesh(nx, ny, *ext), neumann)
    disc = pb.Discretization(mesh, "q1")
    mv, nd = disc.n_velocity, disc.ndof
    gh = 0.2 * np.sin(np.arange(mv) * 0.37) if ghat else None
    conf = pb.DiscretizationConfig(40.0, 30.0, 0.8, gh)
    params = pb.ModelParams(1.35, 2e-3, 1.0, 1e-3)
    b = gauss_radau(k)
    tm = temporal_matrices(b)
    f = forcing_a if forcing else None
    vm = rng.uniform(-1, 1, mv)
    ctx = pb.SlabContext(disc, params, conf, pb.ProblemData(f=f), b, tm, 0.1, 0.02, vm)
    U = rng.uniform(-1, 1, (k + 1, nd))
    x = rng.uniform(-1, 1, (k + 1) * nd)
    tags = pb.dirichlet_flags(mesh).astype(bool)
    grid = orc.Grid(nx, ny, ext, tags, 40.0, 30.0, 0.8, gh)
    slab = orc.Slab(grid, orc.Params(1.35, 2e-3, 1.0, 1e-3), k, b.nodes, b.weights, tm.K_t, tm.m_t, 0.02, 0.1, vm, f)
    var = {"pic": pb.picard(), "exn": pb.exact_newton(), "modn": pb.modified_newton(0.6)}[variant]
    ovar = {"pic": orc.Variant("pic"), "exn": orc.Variant("exn"), "modn": orc.Variant("modn", 0.6)}[variant]
    return ctx, U, x, var, slab, ovar


@pytest.mark.parametrize("nx,ny,k,variant,neumann,ghat", [
    (4, 4, 1, "exn", (), False), (9, 7, 2, "modn", ("top",), True), (20, 20, 1, "pic", ("left", "bottom"), False),
    (33, 17, 0, "modn", (), True), (18, 24, 3, "exn", ("right",), False)])
def test_apply_residual_mass_vs_oracle(nx, ny, k, variant, neumann, ghat):
    from paper_2603_28706_b200.operators import MassNorm, SlabJacobian, slab_residual

    ctx, U, x, var, slab, ovar = _case(nx, ny, k, variant, neumann, ghat, forcing=True)
    jac = SlabJacobian(ctx, U, var)
    assert_close(jac.matvec(x), th.th_slab_matvec(slab, U, ovar, x), TOL, "TH apply")
    assert_close(slab_residual(ctx, U), th.th_slab_residual(slab, U).reshape(-1), TOL, "TH residual")
    m = MassNorm(ctx, dev=jac.dev)
    ref = th.th_mass_apply(slab, x)
    assert_close(m.apply(x), ref, TOL, "TH mass")
    assert abs(m.norm(x) - np.sqrt(x @ ref)) <= TOL * np.sqrt(x @ ref)


def test_properties_at_cfg2_size():
    import torch

    from paper_2603_28706_b200 import problem as pb
    from paper_2603_28706_b200.operators import SlabJacobian, slab_residual
    from paper_2603_28706_b200.synth import CONFIGS, make_slab_inputs

    cfg = CONFIGS["cfg2"]
    syn = make_slab_inputs(cfg)
    params = pb.ModelParams(cfg.p, cfg.delta, cfg.nu, cfg.nu_inf)
    conf = pb.DiscretizationConfig(cfg.gamma1, cfg.gamma2, cfg.gamma_cip)
    ctx = pb.make_context(cfg.nx, cfg.ny, cfg.k, params, cfg.tau, config=conf, v_minus=syn.v_minus, pressure="q1")
    mv, nd = ctx.disc.n_velocity, ctx.disc.ndof
    k1 = cfg.k + 1
    rng = np.random.default_rng(9)
    U = np.zeros((k1, nd))
    U[:, :mv] = syn.U[:, :mv]
    U[:, mv:] = rng.uniform(-1, 1, (k1, nd - mv))
    dev = torch.device("cuda", 0)
    Ut = torch.as_tensor(U, device=dev)
    jac = SlabJacobian(ctx, Ut, pb.exact_newton())
    x = torch.as_tensor(rng.uniform(-1, 1, k1 * nd), device=dev)
    z = torch.as_tensor(rng.uniform(-1, 1, k1 * nd), device=dev)
    Jx, Jz = jac.matvec(x), jac.matvec(z)
    J = jac.matvec(0.25 * x - 2.0 * z)
    assert float(torch.linalg.vector_norm(J - (0.25 * Jx - 2.0 * Jz)) / torch.linalg.vector_norm(J)) <= 1e-13
    # the coupling both ways: velocity-only and pressure-only directions
    xv, zp = x.clone().view(k1, nd), z.clone().view(k1, nd)
    xv[:, mv:] = 0.0
    zp[:, :mv] = 0.0
    yv = jac.matvec(xv.reshape(-1)).view(k1, nd)  # pressure rows: tau w G u
    yp = jac.matvec(zp.reshape(-1)).view(k1, nd)  # velocity rows: tau w G' q
    for mu in range(k1):
        a = float(yv[mu, mv:] @ zp[mu, mv:])
        b = float(xv[mu, :mv] @ yp[mu, :mv])
        assert abs(a - b) <= 1e-12 * (abs(a) + abs(b)), (mu, a, b)
    # all-Dirichlet: constant pressure per node -> zero
    one = torch.zeros(k1, nd, dtype=torch.float64, device=dev)
    one[:, mv:] = 1.0
    y1 = jac.matvec(one.reshape(-1))
    assert float(y1.abs().max()) <= 1e-12 * float(yp.abs().max())
    # exact Newton = -d(residual) along x with the lagged weights frozen (slab.py:144-159)
    eps = 1e-6
    xs = x.view(k1, nd)
    Rp = slab_residual(ctx, Ut + eps * xs, advect=Ut, dev=jac.dev)
    Rm = slab_residual(ctx, Ut - eps * xs, advect=Ut, dev=jac.dev)
    fd = -(Rp - Rm).reshape(-1) / (2 * eps)
    assert float(torch.linalg.vector_norm(fd - Jx) / torch.linalg.vector_norm(Jx)) <= 1e-6


def test_p1disc_only_entry_points_refuse():
    from paper_2603_28706_b200.smoother import VankaLevel
    from paper_2603_28706_b200.stmg import MgConfig, StmgPreconditioner

    ctx, U, x, var, slab, ovar = _case(8, 8, 1)
    with pytest.raises(NotImplementedError):
        VankaLevel(ctx, U, var)
    with pytest.raises(NotImplementedError):
        StmgPreconditioner(None, ctx, U, var, MgConfig(min_cells=2))
