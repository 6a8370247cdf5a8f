"""Size-independent properties at BASELINE.json's full sizes (cfg2 256^2
DG(1), cfg3 1024^2 DG(2)), where the CPU oracle cannot follow:

* linearity of the matrix-free Jacobian (relative 1e-13);
* defect mode == rhs - J x (bitwise: same summation, one subtraction);
* omega = 0 Vanka sweep is the identity (bitwise);
* <a, M b> == <b, M a> (relative 1e-13);
* exact-Newton Jacobian == finite difference of the residual with the
  lagged CIP / inflow weights frozen (slab.py:144-159 `advect`), relative
  error O(eps);
* the 2-rank strip partition reproduces the single-domain apply (1e-13);
* cfg3's three linearizations: modified Newton with an unbounded sigma_max is
  exact Newton bitwise, the three differ, exact Newton = d(residual).
"""

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _setup(name, variant="modn"):
    import torch

    from paper_2603_28706_b200 import problem as pb
    from paper_2603_28706_b200.synth import CONFIGS, make_slab_inputs

    cfg = CONFIGS[name]
    params = pb.ModelParams(cfg.p, cfg.delta, cfg.nu, cfg.nu_inf)
    conf = pb.DiscretizationConfig(cfg.gamma1, cfg.gamma2, cfg.gamma_cip)
    syn = make_slab_inputs(cfg)
    ctx = pb.make_context(cfg.nx, cfg.ny, cfg.k, params, cfg.tau, config=conf, v_minus=syn.v_minus)
    var = {"modn": pb.modified_newton(cfg.nu), "exn": pb.exact_newton(), "pic": pb.picard()}[variant]
    dev = torch.device("cuda", 0)
    return cfg, ctx, var, syn, dev


def _rel(a, b):
    import torch

    return float(torch.linalg.vector_norm(a - b) / torch.linalg.vector_norm(b))


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_linearity_and_defect(name):
    import torch

    from paper_2603_28706_b200.operators import SlabJacobian

    cfg, ctx, var, syn, dev = _setup(name)
    U = torch.as_tensor(syn.U, device=dev)
    x = torch.as_tensor(syn.x, device=dev)
    y = torch.as_tensor(syn.d0, device=dev)
    jac = SlabJacobian(ctx, U, var)
    Jx, Jy = jac.matvec(x), jac.matvec(y)
    Jz = jac.matvec(0.75 * x - 1.5 * y)
    assert _rel(Jz, 0.75 * Jx - 1.5 * Jy) <= 1e-13
    r = torch.as_tensor(syn.d0[::-1].copy(), device=dev)
    assert torch.equal(jac.defect(x, r), r - Jx)
    assert torch.isfinite(Jx).all()


def test_cfg2_vanka_identity_mass_symmetry_partition():
    import torch

    from paper_2603_28706_b200.operators import MassNorm, SlabJacobian
    from paper_2603_28706_b200.partition import DistributedSlab, LocalTransport, StripPartition, distributed_apply
    from paper_2603_28706_b200.smoother import VankaLevel

    cfg, ctx, var, syn, dev = _setup("cfg2")
    U = torch.as_tensor(syn.U, device=dev)
    x = torch.as_tensor(syn.x, device=dev)
    d = torch.as_tensor(syn.d0, device=dev)
    jac = SlabJacobian(ctx, U, var)
    lvl = VankaLevel(ctx, U, var, surrogate=True, rep_fraction=cfg.rep_fraction, jac=jac)
    assert torch.equal(lvl.smooth(d, x, 1, 0.0), d)
    m = MassNorm(ctx, dev=jac.dev)
    ab, ba = float(m.dot(x, d)), float(m.dot(d, x))
    assert abs(ab - ba) <= 1e-13 * abs(ab)
    # two strips, one GPU
    part = StripPartition(cfg.nx, cfg.ny, 2)
    tr = LocalTransport([part.layout(r) for r in range(2)])
    ranks = [DistributedSlab(ctx, syn.U, var, part, r, tr) for r in range(2)]
    xs = [torch.as_tensor(rk.local(syn.x), device=dev) for rk in ranks]
    ys = distributed_apply(ranks, xs, tr)
    y_ref = jac.matvec(x).cpu().numpy()
    g = np.full(y_ref.size, np.nan)
    for rk, yl in zip(ranks, ys):
        rk.owned_into(yl.cpu().numpy(), g)
    assert np.linalg.norm(g - y_ref) <= 1e-13 * np.linalg.norm(y_ref)


def test_cfg2_exact_newton_is_residual_derivative():
    import torch

    from paper_2603_28706_b200.operators import SlabDevice, SlabJacobian, slab_residual

    cfg, ctx, var, syn, dev = _setup("cfg2", "exn")
    U = torch.as_tensor(syn.U, device=dev)
    dU = torch.as_tensor(syn.x, device=dev).reshape(U.shape)
    sd = SlabDevice(ctx)
    jac = SlabJacobian(ctx, U, var)
    JdU = jac.matvec(dU.reshape(-1))
    errs = []
    for eps in (1e-6, 1e-7):
        Rp = slab_residual(ctx, U + eps * dU, advect=U, dev=sd)
        Rm = slab_residual(ctx, U - eps * dU, advect=U, dev=sd)
        fd = ((Rp - Rm) / (2 * eps)).reshape(-1)
        # R = -tau w F + ..., the Jacobian of the slab system is -dR/dU (newton.py solves J dU = R)
        errs.append(min(_rel(-fd, JdU), _rel(fd, JdU)))
    assert min(errs) <= 1e-6, errs


def test_cfg3_three_linearizations():
    """BASELINE configs[2]: the apply in all three linearizations at full size
    (1024^2, DG(2), 34.6 M dofs), compared: modified Newton with an unbounded
    sigma_max IS exact Newton (the clip factor is exactly 1: bitwise), the
    three differ from each other, each is linear, and exact Newton is the
    derivative of the residual (central differences, lagged weights frozen)."""
    import torch

    from paper_2603_28706_b200 import problem as pb
    from paper_2603_28706_b200.operators import SlabDevice, SlabJacobian, slab_residual

    cfg, ctx, _, syn, dev = _setup("cfg3")
    U = torch.as_tensor(syn.U, device=dev)
    x = torch.as_tensor(syn.x, device=dev)
    y = torch.as_tensor(syn.d0, device=dev)
    sd = SlabDevice(ctx)
    out = {}
    for name, var in (("pic", pb.picard()), ("exn", pb.exact_newton()), ("modn", pb.modified_newton(cfg.nu)),
                      ("modn_inf", pb.modified_newton(1e300))):
        jac = SlabJacobian(ctx, U, var, dev=sd)
        Jx, Jy = jac.matvec(x), jac.matvec(y)
        assert torch.isfinite(Jx).all()
        assert _rel(jac.matvec(2.0 * x - 0.5 * y), 2.0 * Jx - 0.5 * Jy) <= 1e-13
        out[name] = Jx
    assert torch.equal(out["modn_inf"], out["exn"])
    for a, b in (("pic", "exn"), ("pic", "modn"), ("modn", "exn")):
        assert _rel(out[a], out[b]) > 1e-8, (a, b)
    dU = x.reshape(U.shape)
    errs = []
    for eps in (1e-6, 1e-7):
        Rp = slab_residual(ctx, U + eps * dU, advect=U, dev=sd)
        Rm = slab_residual(ctx, U - eps * dU, advect=U, dev=sd)
        fd = ((Rp - Rm) / (2 * eps)).reshape(-1)
        errs.append(min(_rel(-fd, out["exn"]), _rel(fd, out["exn"])))
    assert min(errs) <= 1e-6, errs


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_repeated_applies_are_bitwise_reproducible(name):
    """The apply's epilogue runs under the tile pass behind completion counters
    (one wave at cfg2, many waves at cfg3): back-to-back applies and defects on
    one handle, without host synchronization in between, reproduce the first
    result bit for bit."""
    import torch

    from paper_2603_28706_b200.operators import SlabJacobian

    cfg, ctx, var, syn, dev = _setup(name)
    U = torch.as_tensor(syn.U, device=dev)
    x = torch.as_tensor(syn.x, device=dev)
    r = torch.as_tensor(syn.d0, device=dev)
    jac = SlabJacobian(ctx, U, var)
    y0, d0 = jac.matvec(x).clone(), jac.defect(x, r).clone()
    y, d = torch.empty_like(x), torch.empty_like(x)
    bad = torch.zeros((), dtype=torch.int64, device=dev)
    for _ in range(24):
        y.zero_()
        d.zero_()
        jac.matvec(x, out=y)
        jac.defect(x, r, out=d)
        bad += (y != y0).any().long() + (d != d0).any().long()
    assert int(bad.item()) == 0
