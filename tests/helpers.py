"""Shared test helpers: golden fixture loading and oracle construction."""

from __future__ import annotations

import math
import os
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, GOLDEN):
    if p not in sys.path:
        sys.path.insert(0, p)

from cases import CASE_BY_NAME, CASES, FORCINGS, SOLVER_BY_NAME, SOLVER_CASES  # noqa: E402
from oracle import pdst_oracle as orc  # noqa: E402


def load(name):
    return dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))


def variant_of(case):
    if case.variant == "pic":
        return orc.Variant("pic")
    if case.variant == "exn":
        return orc.Variant("exn")
    return orc.Variant("modn", case.cfg.nu if case.sigma_max is None else case.sigma_max)


def oracle_slab(case, fx):
    cfg = case.cfg
    grid = orc.Grid(cfg.nx, cfg.ny, cfg.extents, fx["tags"], cfg.gamma1, cfg.gamma2, cfg.gamma_cip,
                    fx.get("g_hat"))
    params = orc.Params(cfg.p, cfg.delta, cfg.nu, cfg.nu_inf)
    return orc.Slab(grid, params, cfg.k, fx["nodes"], fx["weights"], fx["K_t"], fx["m_t"], cfg.tau,
                    case.t_start, fx["v_minus"], FORCINGS[case.forcing])


def rel_err(a, b):
    """(relative L2, relative Linf) of a against reference b."""
    a, b = np.asarray(a).ravel(), np.asarray(b).ravel()
    nb2 = np.linalg.norm(b)
    nbi = np.abs(b).max() if b.size else 0.0
    e2 = np.linalg.norm(a - b) / (nb2 if nb2 > 0 else 1.0)
    ei = np.abs(a - b).max() / (nbi if nbi > 0 else 1.0) if b.size else 0.0
    return e2, ei


def assert_close(a, b, tol=1e-12, what=""):
    e2, ei = rel_err(a, b)
    assert e2 <= tol and ei <= tol, f"{what}: rel L2 {e2:.3e}, rel Linf {ei:.3e} > {tol:.0e}"


def product_ctx(case, fx):
    """The product's own SlabContext for a golden case (K_t etc. from the fixture)."""
    from paper_2603_28706_b200 import problem as pb
    from paper_2603_28706_b200.radau import TimeBasis, TimeMatrices

    cfg = case.cfg
    mesh = pb.tag_sides(pb.QuadMesh(cfg.nx, cfg.ny, *cfg.extents), case.neumann_sides)
    disc = pb.Discretization(mesh)
    config = pb.DiscretizationConfig(cfg.gamma1, cfg.gamma2, cfg.gamma_cip, fx.get("g_hat"))
    params = pb.ModelParams(cfg.p, cfg.delta, cfg.nu, cfg.nu_inf)
    basis = TimeBasis(cfg.k, fx["nodes"], fx["weights"])
    tmat = TimeMatrices(fx["M_t"], fx["K_t"], fx["m_t"])
    return pb.SlabContext(disc, params, config, pb.ProblemData(f=FORCINGS[case.forcing]), basis, tmat,
                          case.t_start, cfg.tau, fx["v_minus"])


def product_variant(case):
    from paper_2603_28706_b200 import problem as pb

    if case.variant == "pic":
        return pb.picard()
    if case.variant == "exn":
        return pb.exact_newton()
    return pb.modified_newton(case.cfg.nu if case.sigma_max is None else case.sigma_max)


def cuda_available():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


class FixedForcing:
    """f(x, y, t) replaying forcing values frozen at the quadrature points
    (fixture `fq`, shape (k+1, nc, 16, 2)); t selects the Radau node."""

    def __init__(self, fq, times):
        self.fq = np.asarray(fq)
        self.times = np.asarray(times, dtype=float)

    def __call__(self, x, y, t):
        mu = int(np.argmin(np.abs(self.times - t)))
        assert abs(self.times[mu] - t) < 1e-12 and np.shape(x) == self.fq.shape[1:3]
        return self.fq[mu]


def solver_ctx(sc, fx):
    """Product SlabContext of a SOLVER_CASES entry (fixture fx)."""
    from paper_2603_28706_b200 import problem as pb
    from paper_2603_28706_b200.radau import TimeBasis, TimeMatrices

    if sc.kind == "fgmres":
        fx = dict(fx, M_t=np.diag(fx["weights"]))
        return product_ctx(sc.case, fx)
    mesh = pb.tag_sides(pb.QuadMesh(sc.nx, sc.nx), ("right",))
    disc = pb.Discretization(mesh)
    g = fx["gammas"]
    config = pb.DiscretizationConfig(float(g[0]), float(g[1]), float(g[2]))
    params = pb.ModelParams(*sc.params)
    basis = TimeBasis(sc.k, fx["nodes"], fx["weights"])
    tmat = TimeMatrices(np.diag(fx["weights"]), fx["K_t"], fx["m_t"])
    t0, tau = float(fx["t_start"]), float(fx["tau"])
    f = FixedForcing(fx["fq"], t0 + tau * np.asarray(fx["nodes"]))
    return pb.SlabContext(disc, params, config, pb.ProblemData(f=f), basis, tmat, t0, tau, fx["v_minus"])


def solver_variant(name, nu):
    from paper_2603_28706_b200 import problem as pb

    return {"pic": pb.picard(), "exn": pb.exact_newton(), "modn": pb.modified_newton(nu)}[name]
