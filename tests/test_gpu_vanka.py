"""GPU parity of the Vanka patches (exact and surrogate) and sweeps against
the reference golden vectors and the oracle.  Tolerance: relative 1e-12
(L2 and Linf); patch index sets bit-exact."""

import numpy as np
import pytest

from helpers import CASES, assert_close, load, oracle_slab, orc, product_ctx, product_variant, rel_err, variant_of

pytestmark = pytest.mark.gpu
TOL = 1e-12
PATCH_CASES = [c for c in CASES if c.patches]


@pytest.mark.parametrize("case", PATCH_CASES, ids=lambda c: c.name)
def test_golden_patches_and_sweeps(case):
    from paper_2603_28706_b200.smoother import VankaLevel, vanka_smooth

    fx = load(case.name)
    ctx = product_ctx(case, fx)
    lvl = VankaLevel(ctx, fx["U"], product_variant(case), surrogate=case.surrogate,
                     rep_fraction=case.cfg.rep_fraction)
    assert np.array_equal(lvl.patch_ids(), fx["patch_ids"])
    mats = lvl.patch_matrices()
    worst = max(rel_err(mats[c], fx["patch_mats"][c])[0] for c in range(mats.shape[0]))
    assert worst <= TOL, f"worst per-patch rel err {worst:.3e}"
    om = case.cfg.omega
    assert_close(vanka_smooth(lvl, fx["d0"], fx["x"], 1, om), fx["vanka_d"], TOL, "vanka 1 step")
    assert_close(vanka_smooth(lvl, fx["d0"], fx["x"], 2, om), fx["vanka_d2"], TOL, "vanka 2 steps")
    assert_close(vanka_smooth(lvl, 0 * fx["x"], fx["x"], 1, om), fx["vanka_zero"], TOL, "vanka from zero")


# (15, 13): odd cell count, so the dof count per Radau node is odd and the
# second node plane is not 16-byte aligned (the scatter's scalar path)
@pytest.mark.parametrize("nx,ny,k,surrogate", [(20, 17, 1, True), (16, 31, 2, False), (24, 24, 0, True),
                                               (17, 12, 3, True), (15, 13, 1, True), (15, 13, 1, False)])
def test_oracle_parity_vanka_sizes(nx, ny, k, surrogate):
    from test_gpu_operator import _sized_case

    from paper_2603_28706_b200.smoother import VankaLevel, vanka_smooth

    case, fx, syn = _sized_case(nx, ny, k, "exn")
    ctx = product_ctx(case, fx)
    s = oracle_slab(case, fx)
    pre = orc.StmgOracle(s, syn.U, variant_of(case), surrogate=surrogate, rep_fraction=0.5, min_cells=max(nx, ny))
    fine = pre.levels[-1]
    lvl = VankaLevel(ctx, syn.U, product_variant(case), surrogate=surrogate, rep_fraction=0.5)
    mats = lvl.patch_matrices()
    worst = max(rel_err(mats[c], fine.mats[c])[0] for c in range(mats.shape[0]))
    assert worst <= TOL, f"worst per-patch rel err {worst:.3e}"
    assert_close(vanka_smooth(lvl, syn.d0, syn.x, 2, 0.7), orc.vanka(fine, syn.d0, syn.x, 2, 0.7), TOL, "vanka")


def test_vanka_identities():
    """omega = 0 is the identity; k = 0 surrogate == exact patches bitwise."""
    from paper_2603_28706_b200.smoother import VankaLevel, vanka_smooth

    case = [c for c in CASES if c.name == "p6_k0_exn"][0]
    fx = load(case.name)
    ctx = product_ctx(case, fx)
    a = VankaLevel(ctx, fx["U"], product_variant(case), surrogate=True)
    b = VankaLevel(ctx, fx["U"], product_variant(case), surrogate=False)
    assert np.array_equal(a.patch_matrices(), b.patch_matrices())
    d = vanka_smooth(a, fx["d0"], fx["x"], 3, 0.0)
    assert np.array_equal(d, fx["d0"])


def test_singular_patch_reported():
    from paper_2603_28706_b200 import problem as pb
    from paper_2603_28706_b200.errors import SingularPatchError
    from paper_2603_28706_b200.smoother import VankaLevel

    # Stokes-limit with viscosity switched off and no convection: the velocity
    # blocks reduce to the tiny time-mass part only when tau is huge... use
    # disabled viscous + convection + pressure so each patch is K_t (x) M on
    # velocity and an all-zero pressure block -> exactly singular.
    conf = pb.DiscretizationConfig(40.0, 40.0, 1.0, None, False, False, False)
    ctx = pb.make_context(3, 3, 0, pb.ModelParams(1.5, 1e-2, 1.0, 0.0), 0.01, config=conf)
    U = np.zeros((1, ctx.disc.ndof))
    with pytest.raises(SingularPatchError) as ei:
        VankaLevel(ctx, U, pb.picard())
    assert ei.value.patch == 0


def test_async_host_calls_match_sync():
    """PDST_HOST_ASYNC (page-locked numpy buffers, copies on their own streams,
    calls return at once): a pipelined sequence of applies and in-place Vanka
    sweeps on the same host buffers gives bitwise the synchronous results, and
    unpinned memory is rejected."""
    import torch

    from paper_2603_28706_b200 import problem as pb
    from paper_2603_28706_b200.operators import SlabJacobian
    from paper_2603_28706_b200.smoother import VankaLevel
    from paper_2603_28706_b200.synth import CONFIGS, make_slab_inputs

    cfg = CONFIGS["cfg1"]
    params = pb.ModelParams(cfg.p, cfg.delta, cfg.nu, cfg.nu_inf)
    conf = pb.DiscretizationConfig(cfg.gamma1, cfg.gamma2, cfg.gamma_cip)
    syn = make_slab_inputs(cfg)
    ctx = pb.make_context(cfg.nx, cfg.ny, cfg.k, params, cfg.tau, config=conf, v_minus=syn.v_minus)
    var = pb.modified_newton(cfg.nu)
    jac = SlabJacobian(ctx, syn.U, var)
    lvl = VankaLevel(ctx, syn.U, var, surrogate=True, rep_fraction=cfg.rep_fraction, jac=jac)

    def pinned(a):
        t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
        t.numpy()[...] = a
        return t.numpy()

    xh, rh, dh, yh = pinned(syn.x), pinned(syn.x), pinned(syn.d0), pinned(np.zeros_like(syn.x))
    ys, d = [], syn.d0.copy()
    for i in range(3):
        ys.append(jac.matvec(syn.x * (i + 1)))
        d = lvl.smooth(d, syn.x, 1, cfg.omega)
    outs = []
    for i in range(3):
        xh[...] = syn.x * (i + 1)
        jac.matvec(xh, out=yh, asynchronous=True)
        lvl.smooth(dh, rh, 1, cfg.omega, inplace=True, asynchronous=True)
        jac.dev.sync()
        outs.append(yh.copy())
    for a, b in zip(outs, ys):
        assert np.array_equal(a, b)
    assert np.array_equal(dh, d)
    # back to back without syncs in between: the d round trip stays ordered
    d2 = d.copy()
    for _ in range(4):
        d2 = lvl.smooth(d2, syn.x, 1, cfg.omega)
    for _ in range(4):
        jac.matvec(xh, out=yh, asynchronous=True)
        lvl.smooth(dh, rh, 1, cfg.omega, inplace=True, asynchronous=True)
    jac.dev.sync()
    assert np.array_equal(dh, d2)
    assert np.array_equal(yh, ys[2])
    with pytest.raises(ValueError):
        jac.matvec(syn.x.copy(), out=np.zeros_like(syn.x), asynchronous=True)


# The exact kernels bench.py times: the persistent TMA-ring patch GEMVs
# (pdst_timediag.cu k_vanka_gemv_diag_tma / k_vanka_gemv_exact_tma).  Their
# grids are 2 CTAs per SM, so meshes of <= 24^2 cells never give a CTA a
# second patch group; these sizes make every CTA run >= 3.5 groups, so the
# mbarrier ring wraps (parity flips, bulk copies re-issued after
# fence.proxy.async) several times.  (nx, ny, k, surrogate, pb): pb = patches
# per group of the launched instantiation (tma_pb<NB>, xtma_pb<D>).
RING_CASES = [
    (64, 64, 1, True, 4),    # DG(1) surrogate: one complex 21x21 block, 3-stage ring
    (96, 96, 1, True, 4),    # 7.8 groups per CTA
    (72, 72, 2, True, 4),    # DG(2) surrogate: NB = 2 (complex + real block), 2-stage ring
    (64, 64, 3, True, 4),    # DG(3) surrogate: two complex blocks
    (64, 64, 0, True, 4),    # DG(0): one real block
    (48, 48, 1, False, 2),   # exact D = 42 (the coarse levels' kernel)
    (32, 32, 3, False, 1),   # exact D = 84
]


@pytest.mark.parametrize("nx,ny,k,surrogate,pb", RING_CASES)
def test_oracle_parity_vanka_ring_wraps(nx, ny, k, surrogate, pb):
    import torch

    from test_gpu_operator import _sized_case

    from paper_2603_28706_b200.smoother import VankaLevel, vanka_smooth

    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    groups = (nx * ny + pb - 1) // pb
    assert groups / (2 * nsm) >= 1.7, "case too small to wrap the ring"
    case, fx, syn = _sized_case(nx, ny, k, "modn")
    ctx = product_ctx(case, fx)
    s = oracle_slab(case, fx)
    pre = orc.StmgOracle(s, syn.U, variant_of(case), surrogate=surrogate, rep_fraction=1.0, min_cells=max(nx, ny))
    fine = pre.levels[-1]
    lvl = VankaLevel(ctx, syn.U, product_variant(case), surrogate=surrogate, rep_fraction=1.0)
    for steps in (1, 2):
        assert_close(vanka_smooth(lvl, syn.d0, syn.x, steps, 0.7), orc.vanka(fine, syn.d0, syn.x, steps, 0.7), TOL,
                     f"vanka {steps} step(s)")
    z = np.zeros_like(syn.x)
    assert_close(vanka_smooth(lvl, z, syn.x, 1, 0.7), orc.vanka(fine, z, syn.x, 1, 0.7), TOL, "vanka from zero")
    # device-resident vectors take the same kernels
    dd = torch.as_tensor(syn.d0, device="cuda")
    rr = torch.as_tensor(syn.x, device="cuda")
    assert_close(vanka_smooth(lvl, dd, rr, 2, 0.7).cpu().numpy(), orc.vanka(fine, syn.d0, syn.x, 2, 0.7), TOL,
                 "vanka device 2 steps")
