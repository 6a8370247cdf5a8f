"""GPU parity of the strip-partitioned hot path: P virtual
ranks on one GPU, each with its own local mesh (cut-tagged sides, ghost rows)
and its own libpdst handle, exchanging through LocalTransport.  The owned
entries of the distributed Jacobian apply, slab residual and Vanka step must
match the single-domain results.  Tolerance: relative 1e-13 (the local
kernels sum the same terms; only the tile decomposition differs)."""

import numpy as np
import pytest

from helpers import assert_close, product_ctx, product_variant

pytestmark = pytest.mark.gpu
TOL = 1e-13


def _ranks(ctx, U, variant, P, build_patches=False, surrogate=True):
    from paper_2603_28706_b200.partition import DistributedSlab, LocalTransport, StripPartition

    m = ctx.disc.mesh
    part = StripPartition(m.nx, m.ny, P)
    lays = [part.layout(r) for r in range(P)]
    tr = LocalTransport(lays)
    ranks = [DistributedSlab(ctx, U, variant, part, r, tr, surrogate=surrogate) for r in range(P)]
    if build_patches:
        for rk in ranks:
            rk.build_patches()
    return ranks, tr


def _scatter_with_garbage(ranks, xg, seed):
    """Local vectors whose ghost entries are garbage (the exchange must fix them)."""
    rng = np.random.default_rng(seed)
    out = []
    for rk in ranks:
        xl = rk.local(xg)
        own = np.zeros_like(xg)
        rk.owned_into(np.ones_like(xl), own)
        mask = rk.local(own) > 0
        xl[~mask] = 1e3 * rng.standard_normal((~mask).sum())
        out.append(xl)
    return out


def _gather(ranks, xs, n):
    g = np.full(n, np.nan)
    for rk, x in zip(ranks, xs):
        rk.owned_into(np.asarray(x), g)
    assert not np.isnan(g).any()
    return g


@pytest.mark.parametrize("nx,ny,k,P", [(12, 9, 1, 2), (20, 14, 2, 3), (17, 24, 0, 4), (33, 40, 1, 5)])
@pytest.mark.parametrize("variant", ["exn", "modn"])
def test_distributed_apply_and_residual(nx, ny, k, P, variant):
    from test_gpu_operator import _sized_case

    from paper_2603_28706_b200.operators import SlabJacobian, slab_residual
    from paper_2603_28706_b200.partition import distributed_apply

    case, fx, syn = _sized_case(nx, ny, k, variant)
    ctx = product_ctx(case, fx)
    var = product_variant(case)
    y_ref = SlabJacobian(ctx, syn.U, var).matvec(syn.x)
    ranks, tr = _ranks(ctx, syn.U, var, P)
    xs = _scatter_with_garbage(ranks, syn.x, 1)
    ys = distributed_apply(ranks, xs, tr)
    assert_close(_gather(ranks, ys, y_ref.size), y_ref, TOL, "distributed apply")
    R_ref = slab_residual(ctx, syn.U).reshape(-1)
    Rs = [slab_residual(rk.ctx, np.stack([rk.lay.to_local(syn.U[mu]) for mu in range(rk.k1)])).reshape(-1)
          for rk in ranks]
    assert_close(_gather(ranks, Rs, R_ref.size), R_ref, TOL, "distributed residual")


@pytest.mark.parametrize("nx,ny,k,P,surrogate", [(12, 9, 1, 2, True), (20, 14, 2, 3, False), (18, 16, 1, 4, True)])
def test_distributed_vanka_step(nx, ny, k, P, surrogate):
    from test_gpu_operator import _sized_case

    from paper_2603_28706_b200.partition import distributed_vanka_step
    from paper_2603_28706_b200.smoother import VankaLevel, vanka_smooth

    case, fx, syn = _sized_case(nx, ny, k, "exn")
    ctx = product_ctx(case, fx)
    var = product_variant(case)
    lvl = VankaLevel(ctx, syn.U, var, surrogate=surrogate, rep_fraction=0.5)
    ref1 = vanka_smooth(lvl, syn.d0, syn.x, 1, 0.7)
    ref2 = vanka_smooth(lvl, syn.d0, syn.x, 2, 0.7)
    ranks, tr = _ranks(ctx, syn.U, var, P, build_patches=True, surrogate=surrogate)
    ds = _scatter_with_garbage(ranks, syn.d0, 2)
    rs = [rk.local(syn.x) for rk in ranks]
    distributed_vanka_step(ranks, ds, rs, 0.7, tr)
    assert_close(_gather(ranks, ds, ref1.size), ref1, TOL, "distributed vanka 1 step")
    distributed_vanka_step(ranks, ds, rs, 0.7, tr)
    assert_close(_gather(ranks, ds, ref2.size), ref2, TOL, "distributed vanka 2 steps")


@pytest.mark.parametrize("nx,ny,k,P", [(12, 9, 1, 2), (18, 16, 1, 4)])
def test_fused_apply_and_vanka_step(nx, ny, k, P):
    """The bench's distributed step with the x / d halos grouped equals the
    separate distributed apply and Vanka step bitwise."""
    import torch

    from test_gpu_operator import _sized_case

    from paper_2603_28706_b200.partition import (distributed_apply, distributed_apply_and_vanka_step,
                                                 distributed_vanka_step)

    case, fx, syn = _sized_case(nx, ny, k, "modn")
    ctx = product_ctx(case, fx)
    ranks, tr = _ranks(ctx, syn.U, product_variant(case), P, build_patches=True)
    xs = [torch.as_tensor(x, device="cuda") for x in _scatter_with_garbage(ranks, syn.x, 3)]
    ds = [torch.as_tensor(x, device="cuda") for x in _scatter_with_garbage(ranks, syn.d0, 4)]
    rs = [torch.as_tensor(rk.local(syn.x), device="cuda") for rk in ranks]
    xs2, ds2 = [x.clone() for x in xs], [d.clone() for d in ds]
    ys = distributed_apply(ranks, xs, tr)
    distributed_vanka_step(ranks, ds, rs, 0.7, tr)
    ys2 = distributed_apply_and_vanka_step(ranks, xs2, ds2, rs, 0.7, tr)
    for a, b in zip(ys, ys2):
        assert torch.equal(a, b)
    for a, b in zip(ds, ds2):
        assert torch.equal(a, b)


@pytest.mark.parametrize("nx,ny,k,P,surrogate", [(12, 9, 1, 2, True), (20, 14, 2, 3, False), (18, 16, 1, 4, True),
                                                 (17, 24, 0, 4, True), (33, 40, 3, 5, True)])
def test_libpdst_strip_step(nx, ny, k, P, surrogate):
    """The data plane inside libpdst (pdst_strips_step_local: halo pack /
    unpack kernels, owned-row fused Vanka update with the increment row sent
    up, reverse-add): owned entries of y = J x and of 1 / 2 Vanka steps equal
    the single domain (1e-13), ghost entries garbage on input."""
    import torch

    from test_gpu_operator import _sized_case

    from paper_2603_28706_b200.operators import SlabJacobian
    from paper_2603_28706_b200.partition import strip_step
    from paper_2603_28706_b200.smoother import VankaLevel, vanka_smooth

    case, fx, syn = _sized_case(nx, ny, k, "exn")
    ctx = product_ctx(case, fx)
    var = product_variant(case)
    jac = SlabJacobian(ctx, syn.U, var)
    lvl = VankaLevel(ctx, syn.U, var, surrogate=surrogate, rep_fraction=0.5, jac=jac)
    y_ref = jac.matvec(syn.x)
    ref1 = vanka_smooth(lvl, syn.d0, syn.x, 1, 0.7)
    ref2 = vanka_smooth(lvl, syn.d0, syn.x, 2, 0.7)
    ranks, tr = _ranks(ctx, syn.U, var, P, build_patches=True, surrogate=surrogate)
    for rk in ranks:
        rk.strip_setup()
    xs = [torch.as_tensor(x, device="cuda") for x in _scatter_with_garbage(ranks, syn.x, 5)]
    ds = [torch.as_tensor(x, device="cuda") for x in _scatter_with_garbage(ranks, syn.d0, 6)]
    rs = [torch.as_tensor(x, device="cuda") for x in _scatter_with_garbage(ranks, syn.x, 7)]
    ys = strip_step(ranks, xs, ds, rs, 0.7)
    n = y_ref.size
    assert_close(_gather(ranks, [y.cpu().numpy() for y in ys], n), y_ref, TOL, "strip apply")
    assert_close(_gather(ranks, [d.cpu().numpy() for d in ds], n), ref1, TOL, "strip vanka 1 step")
    strip_step(ranks, xs, ds, rs, 0.7)
    assert_close(_gather(ranks, [d.cpu().numpy() for d in ds], n), ref2, TOL, "strip vanka 2 steps")
