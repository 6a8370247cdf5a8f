"""GPU parity of the slab Jacobian, residual and mass reductions (through the
C ABI) against the reference golden vectors and the pinned oracle.

Tolerance (north_star): relative 1e-12 in both the L2 and the Linf norm;
integer maps bit-exact."""

import numpy as np
import pytest

from helpers import (CASES, assert_close, load, oracle_slab, orc, product_ctx, product_variant, variant_of)

pytestmark = pytest.mark.gpu
TOL = 1e-12


@pytest.mark.parametrize("case", CASES, ids=lambda c: c.name)
def test_golden_apply_residual(case):
    from paper_2603_28706_b200.operators import MassNorm, SlabJacobian, slab_residual

    fx = load(case.name)
    ctx = product_ctx(case, fx)
    jac = SlabJacobian(ctx, fx["U"], product_variant(case))
    assert_close(jac.matvec(fx["x"]), fx["y"], TOL, "jacobian vs reference")
    assert_close(jac.apply(fx["x"].reshape(fx["U"].shape)).reshape(-1), fx["y"], TOL, "apply")
    assert_close(slab_residual(ctx, fx["U"]), fx["R"], TOL, "residual vs reference")
    mn = MassNorm(ctx)
    assert_close(mn.apply(fx["x"]), fx["mass_x"], TOL, "mass apply")
    assert abs(mn.norm(fx["x"]) - float(fx["mnorm_x"])) <= TOL * float(fx["mnorm_x"])
    # defect form used by the Vanka sweep
    r = np.linspace(-1, 1, fx["x"].size)
    assert_close(jac.defect(fx["x"], r), r - fx["y"], TOL, "defect")


@pytest.mark.parametrize("case", CASES[:6], ids=lambda c: c.name)
def test_integer_maps_bit_exact(case):
    import ctypes as C

    from paper_2603_28706_b200 import _lib as L
    from paper_2603_28706_b200.operators import SlabDevice

    fx = load(case.name)
    dev = SlabDevice(product_ctx(case, fx))
    nc = case.cfg.nx * case.cfg.ny
    cn = np.empty((nc, 9), dtype=np.int64)
    ids = np.empty((nc, 21 * (case.cfg.k + 1)), dtype=np.int64)
    L.check(L.lib().pdst_cell_maps(dev.h, C.c_void_p(cn.ctypes.data), C.c_void_p(ids.ctypes.data)))
    assert np.array_equal(cn, fx["cell_nodes"])
    g = orc.Grid(case.cfg.nx, case.cfg.ny)
    assert np.array_equal(ids, g.patch_ids(case.cfg.k + 1))


def _sized_case(nx, ny, k, variant):
    from cases import Case, _cfg
    from paper_2603_28706_b200.radau import gauss_radau, temporal_matrices
    from paper_2603_28706_b200.synth import make_slab_inputs

    case = Case(f"s{nx}x{ny}", _cfg(f"s{nx}x{ny}", nx, ny, k, seed=nx * 1000 + ny, p=1.3, delta=1e-3, nu_inf=0.0,
                                     modes=8, extents=(0.0, 0.0, 1.5, 1.0)),
                variant=variant, neumann_sides=("top",), forcing="a", t_start=0.1)
    b = gauss_radau(k)
    tm = temporal_matrices(b)
    syn = make_slab_inputs(case.cfg, nodes=b.nodes)
    tags = np.ones(2 * (nx + ny), dtype=bool)
    tags[nx + ny: 2 * nx + ny] = False
    fx = dict(nodes=b.nodes, weights=b.weights, K_t=tm.K_t, m_t=tm.m_t, M_t=tm.M_t, v_minus=syn.v_minus, tags=tags)
    return case, fx, syn


SIZES = [(16, 16, 1), (31, 17, 0), (33, 40, 2), (45, 30, 3), (64, 64, 1)]


@pytest.mark.parametrize("nx,ny,k", SIZES)
@pytest.mark.parametrize("variant", ["pic", "exn", "modn"])
def test_oracle_parity_sizes(nx, ny, k, variant):
    """Multi-tile meshes (tile = 15x15 cells) with ragged edges, k = 0..3."""
    from paper_2603_28706_b200.operators import SlabJacobian, slab_residual

    case, fx, syn = _sized_case(nx, ny, k, variant)
    ctx = product_ctx(case, fx)
    s = oracle_slab(case, fx)
    y_ref = orc.SlabJacobianOracle(s, syn.U, variant_of(case)).matvec(syn.x)
    y = SlabJacobian(ctx, syn.U, product_variant(case)).matvec(syn.x)
    assert_close(y, y_ref, TOL, "jacobian vs oracle")
    assert_close(slab_residual(ctx, syn.U), orc.slab_residual(s, syn.U), TOL, "residual vs oracle")


def test_device_tensors_roundtrip():
    import torch

    from paper_2603_28706_b200.operators import SlabJacobian

    case = CASES[0]
    fx = load(case.name)
    ctx = product_ctx(case, fx)
    jac = SlabJacobian(ctx, torch.as_tensor(fx["U"], device="cuda"), product_variant(case))
    y = jac.matvec(torch.as_tensor(fx["x"], device="cuda"))
    torch.cuda.synchronize()
    assert_close(y.cpu().numpy(), fx["y"], TOL, "device-pointer apply")


def test_domain_errors():
    from paper_2603_28706_b200 import problem as pb
    from paper_2603_28706_b200.errors import ConstitutiveDomainError
    from paper_2603_28706_b200.operators import SlabJacobian, slab_residual

    ctx = pb.make_context(4, 4, 1, pb.ModelParams(1.5, 0.0, 1.0, 0.0), 0.01)
    U = np.zeros((2, ctx.disc.ndof))
    with pytest.raises(ConstitutiveDomainError):
        SlabJacobian(ctx, U, pb.picard())
    with pytest.raises(ConstitutiveDomainError):
        slab_residual(ctx, U)


def test_buffer_size_errors():
    """Short, mistyped or strided vectors are rejected before the C ABI sees
    their pointers (apply, defect, residual, mass, Vanka, V-cycle)."""
    import torch

    from paper_2603_28706_b200 import problem as pb
    from paper_2603_28706_b200.operators import MassNorm, SlabJacobian, slab_residual
    from paper_2603_28706_b200.smoother import VankaLevel

    ctx = pb.make_context(4, 4, 1, pb.ModelParams(1.5, 1e-2, 1.0, 0.0), 0.01)
    n = 2 * ctx.disc.ndof
    U = np.zeros((2, ctx.disc.ndof))
    jac = SlabJacobian(ctx, U, pb.modified_newton(1.0))
    x = np.ones(n)
    for bad in (np.ones(n - 1), np.ones(n, dtype=np.float32).astype(np.float64)[:-1]):
        with pytest.raises(ValueError):
            jac.matvec(bad)
    with pytest.raises(ValueError):
        jac.matvec(x, out=np.zeros(n, dtype=np.float32))
    with pytest.raises(ValueError):
        jac.matvec(x, out=np.zeros(n + 1))
    with pytest.raises(ValueError):
        jac.defect(x, np.ones(n - 2))
    with pytest.raises(ValueError):
        jac.matvec(torch.ones(2 * n, dtype=torch.float64, device="cuda")[::2])
    with pytest.raises(ValueError):
        slab_residual(ctx, np.zeros(n - 1))
    with pytest.raises(ValueError):
        MassNorm(ctx, dev=jac.dev).dot(x, np.ones(n - 1))
    lvl = VankaLevel(ctx, U, pb.modified_newton(1.0), jac=jac)
    with pytest.raises(ValueError):
        lvl.smooth(x, np.ones(n - 1), 1, 0.7)
    # the right sizes still work
    assert np.isfinite(jac.matvec(x)).all()
    assert np.isfinite(lvl.smooth(x, x, 1, 0.7)).all()


def test_apply_repeats_and_graph_replay():
    """The apply's epilogue polls per-node completion counters that the last
    epilogue CTA re-arms: back-to-back applies / defects on one handle and a
    captured-and-replayed launch sequence give the same bits as the first call
    (multi-tile mesh, so tile-line partials and both counters are in play)."""
    import torch

    from paper_2603_28706_b200 import problem as pb
    from paper_2603_28706_b200.operators import SlabJacobian
    from paper_2603_28706_b200.synth import SynthConfig, make_slab_inputs

    cfg = SynthConfig("graph", 40, 24, 1, 1.3, 1.0e-3, 1.0, 0.0, 4, 3)
    syn = make_slab_inputs(cfg)
    params = pb.ModelParams(cfg.p, cfg.delta, cfg.nu, cfg.nu_inf)
    ctx = pb.make_context(cfg.nx, cfg.ny, cfg.k, params, cfg.tau,
                          config=pb.DiscretizationConfig(cfg.gamma1, cfg.gamma2, cfg.gamma_cip), v_minus=syn.v_minus)
    U = torch.as_tensor(syn.U, device="cuda")
    x = torch.as_tensor(syn.x, device="cuda")
    r = torch.as_tensor(syn.d0, device="cuda")
    jac = SlabJacobian(ctx, U, pb.modified_newton(cfg.nu))
    y0 = jac.matvec(x).clone()
    d0 = jac.defect(x, r).clone()
    y, d = torch.empty_like(x), torch.empty_like(x)
    for _ in range(5):
        jac.matvec(x, out=y)
        jac.defect(x, r, out=d)
    torch.cuda.synchronize()
    assert torch.equal(y, y0) and torch.equal(d, d0)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        jac.matvec(x, out=y)  # warm-up on the side stream
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            jac.matvec(x, out=y)
            jac.defect(x, r, out=d)
        for _ in range(3):
            y.zero_()
            d.zero_()
            g.replay()
        torch.cuda.synchronize()
    assert torch.equal(y, y0) and torch.equal(d, d0)
