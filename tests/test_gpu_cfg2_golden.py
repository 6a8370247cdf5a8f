"""The bench workload itself against the REFERENCE: cfg2 (256x256, DG(1),
modified Newton, surrogate patches at the last Radau point, omega = 0.7) —
the Jacobian apply and the Vanka sweeps bench.py times, i.e. the persistent
TMA-ring patch GEMV with ~55 patch groups per CTA — compared with pdflow's own
outputs frozen by tests/golden/make_golden_cfg2.py (norms, a 64-row seeded
Gaussian sketch, 48,593 sampled entries incl. every boundary-strip and
tile-line dof of both Radau nodes, and 8 whole patch matrices).

Tolerance: relative 1e-12 (north_star); the sketch rows are compared
normwise at 1e-12 of |S y|.
"""

import os

import numpy as np
import pytest

from helpers import GOLDEN

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
TOL = 1e-12


def _fixture():
    return dict(np.load(os.path.join(GOLDEN, "cfg2_frozen.npz")))


def _check(name, y, fx):
    from make_golden_cfg2 import sketch

    y = np.asarray(y)
    for norm, val in (("l2", np.linalg.norm(y)), ("l1", np.abs(y).sum()), ("linf", np.abs(y).max())):
        ref = float(fx[f"{name}_{norm}"])
        assert abs(val - ref) <= TOL * ref, f"{name} {norm}: {val!r} vs {ref!r}"
    s = sketch(y, int(fx["sketch_seed"]), int(fx["n_sketch"]))
    e = np.linalg.norm(s - fx[f"{name}_sketch"]) / np.linalg.norm(fx[f"{name}_sketch"])
    assert e <= TOL, f"{name} sketch rel err {e:.3e}"
    smp = y[fx["idx"]]
    ref = fx[f"{name}_sample"]
    e2 = np.linalg.norm(smp - ref) / np.linalg.norm(ref)
    ei = np.abs(smp - ref).max() / np.abs(ref).max()
    assert e2 <= TOL and ei <= TOL, f"{name} samples: rel L2 {e2:.3e}, rel Linf {ei:.3e}"


def test_cfg2_bench_path_matches_reference():
    import torch

    from paper_2603_28706_b200 import problem as pb
    from paper_2603_28706_b200.operators import SlabJacobian
    from paper_2603_28706_b200.smoother import VankaLevel, vanka_smooth
    from paper_2603_28706_b200.synth import CONFIGS, make_slab_inputs

    fx = _fixture()
    cfg = CONFIGS["cfg2"]
    params = pb.ModelParams(cfg.p, cfg.delta, cfg.nu, cfg.nu_inf)
    conf = pb.DiscretizationConfig(cfg.gamma1, cfg.gamma2, cfg.gamma_cip)
    syn = make_slab_inputs(cfg)
    ctx = pb.make_context(cfg.nx, cfg.ny, cfg.k, params, cfg.tau, config=conf, v_minus=syn.v_minus)
    var = pb.modified_newton(cfg.nu)
    dev = torch.device("cuda", 0)
    U, x, d0 = (torch.as_tensor(a, device=dev) for a in (syn.U, syn.x, syn.d0))
    jac = SlabJacobian(ctx, U, var)
    lvl = VankaLevel(ctx, U, var, surrogate=True, rep_fraction=cfg.rep_fraction, jac=jac)
    _check("y", jac.matvec(x).cpu().numpy(), fx)
    _check("v1", vanka_smooth(lvl, d0, x, 1, cfg.omega).cpu().numpy(), fx)
    _check("v2", vanka_smooth(lvl, d0, x, 2, cfg.omega).cpu().numpy(), fx)
    _check("v0", vanka_smooth(lvl, torch.zeros_like(x), x, 1, cfg.omega).cpu().numpy(), fx)
    # in place, the way bench.py calls it (defect apply -> GEMV -> scatter on d itself)
    d = d0.clone()
    lvl.smooth(d, x, 1, cfg.omega, inplace=True)
    _check("v1", d.cpu().numpy(), fx)
    # host buffers through the C ABI (the e2e leg's path)
    _check("y", jac.matvec(syn.x), fx)
    _check("v1", vanka_smooth(lvl, syn.d0, syn.x, 1, cfg.omega), fx)
    mats = lvl.patch_matrices()
    for c, m_ref in zip(fx["patch_pick"], fx["patch_mat_pick"]):
        e = np.linalg.norm(mats[c] - m_ref) / np.linalg.norm(m_ref)
        assert e <= TOL, f"patch {c} rel err {e:.3e}"
