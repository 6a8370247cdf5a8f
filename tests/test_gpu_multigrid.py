"""GPU parity of the multigrid pieces: Galerkin coarse operators (as level
matvecs), coarse patches, coarse Vanka, transfers and the full V-cycle,
against the reference golden vectors and the oracle.

Tolerances: relative 1e-12 (L2 and Linf) for operators, patches and sweeps.
The V-cycle ends in a dense solve of the pinned, nearly singular coarsest
system: the numpy oracle and the reference already differ by up to 2e-11
there (tests/test_oracle_golden.py), so the V-cycle is checked to 1e-9."""

import numpy as np
import pytest

from helpers import CASES, assert_close, load, oracle_slab, orc, product_ctx, product_variant, rel_err, variant_of

pytestmark = pytest.mark.gpu
TOL = 1e-12
VCYCLE_TOL = 1e-9
PATCH_CASES = [c for c in CASES if c.patches]


def _precond(case, fx):
    from paper_2603_28706_b200.stmg import MgConfig, StmgPreconditioner

    ctx = product_ctx(case, fx)
    mg = MgConfig(omega=case.cfg.omega, surrogate=case.surrogate, rep_fraction=case.cfg.rep_fraction,
                  min_cells=case.min_cells, coarse_mode=case.coarse_mode)
    return StmgPreconditioner(None, ctx, fx["U"], product_variant(case), mg)


@pytest.mark.parametrize("case", PATCH_CASES, ids=lambda c: c.name)
def test_golden_hierarchy(case):
    fx = load(case.name)
    pre = _precond(case, fx)
    assert pre.num_levels == len(fx["levels_nx"])
    for ell in range(pre.num_levels):
        assert pre.level_shape(ell)[:2] == (int(fx["levels_nx"][ell]), int(fx["levels_ny"][ell]))
    fine = pre.patch_matrices(pre.num_levels - 1)
    worst = max(rel_err(fine[c], fx["patch_mats"][c])[0] for c in range(fine.shape[0]))
    assert worst <= TOL, f"fine patches {worst:.3e}"
    om = case.cfg.omega
    for ell in range(pre.num_levels - 1):
        assert_close(pre.level_matvec(ell, fx[f"L{ell}_x"]), fx[f"L{ell}_Ax"], TOL, f"Galerkin matvec L{ell}")
        pm = pre.patch_matrices(ell)
        ref = fx[f"L{ell}_patch_mats"]
        worst = max(rel_err(pm[c], ref[c])[0] for c in range(pm.shape[0]))
        assert worst <= TOL, f"coarse patches L{ell}: {worst:.3e}"
        x = fx[f"L{ell}_x"]
        assert_close(pre.vanka(ell, 0 * x, x, 1, om), fx[f"L{ell}_vanka"], TOL, f"coarse vanka L{ell}")
    assert_close(pre.apply(fx["x"]), fx["vcycle"], VCYCLE_TOL, "V-cycle")


@pytest.mark.parametrize("nc,k", [((4, 4), 1), ((3, 3), 0), ((4, 2), 2), ((8, 6), 1)])
def test_transfers_vs_oracle(nc, k):
    """Restriction = exact transpose of prolongation; weights bit-exact."""
    from dataclasses import replace

    from cases import Case, _cfg
    from paper_2603_28706_b200.stmg import MgConfig, StmgPreconditioner
    from paper_2603_28706_b200.radau import gauss_radau, temporal_matrices
    from paper_2603_28706_b200.synth import make_slab_inputs

    cx, cy = nc
    case = Case("tr", _cfg("tr", 2 * cx, 2 * cy, k, seed=5), variant="exn", min_cells=min(cx, cy))
    b = gauss_radau(k)
    tm = temporal_matrices(b)
    syn = make_slab_inputs(case.cfg, nodes=b.nodes)
    fx = dict(nodes=b.nodes, weights=b.weights, K_t=tm.K_t, m_t=tm.m_t, M_t=tm.M_t, v_minus=syn.v_minus,
              tags=np.ones(2 * (3 * cx + 3 * cy), dtype=bool)[: 2 * (2 * cx + 2 * cy)], U=syn.U)
    ctx = product_ctx(case, fx)
    pre = StmgPreconditioner(None, ctx, syn.U, product_variant(case),
                             MgConfig(min_cells=min(cx, cy), surrogate=False))
    assert pre.num_levels == 2
    P, _, _, _ = orc.transfer(orc.Grid(cx, cy), orc.Grid(2 * cx, 2 * cy))
    k1 = k + 1
    rng = np.random.default_rng(7)
    rf = rng.uniform(-1, 1, size=k1 * P.shape[0])
    ec = rng.uniform(-1, 1, size=k1 * P.shape[1])
    r_ref = (P.T @ rf.reshape(k1, -1).T).T.reshape(-1)
    e_ref = (P @ ec.reshape(k1, -1).T).T.reshape(-1)
    assert_close(pre.restrict(1, rf), r_ref, 1e-14, "restrict")
    assert_close(pre.prolong(1, ec), e_ref, 1e-14, "prolong")
    # prolongation of unit vectors reproduces the stencil weights bit-exactly
    Pd = P.toarray()
    for col in rng.choice(P.shape[1], size=min(24, P.shape[1]), replace=False):
        e = np.zeros(k1 * P.shape[1])
        e[col] = 1.0
        out = pre.prolong(1, e)[: P.shape[0]]
        assert np.array_equal(out, Pd[:, col])


@pytest.mark.parametrize("coarse_mode", ["galerkin", "rediscretize"])
def test_vcycle_matches_oracle_sizes(coarse_mode):
    """V-cycle on a 3-level hierarchy (16x16 -> 8 -> 4), k = 1, surrogate
    patches; Galerkin or rediscretized coarse operators (multigrid.py:302-324)."""
    from test_gpu_operator import _sized_case

    from paper_2603_28706_b200.stmg import MgConfig, StmgPreconditioner

    case, fx, syn = _sized_case(16, 16, 1, "modn")
    ctx = product_ctx(case, fx)
    s = oracle_slab(case, fx)
    ref = orc.StmgOracle(s, syn.U, variant_of(case), omega=0.7, surrogate=True, rep_fraction=0.5, min_cells=4,
                         coarse_mode=coarse_mode)
    pre = StmgPreconditioner(None, ctx, syn.U, product_variant(case),
                             MgConfig(rep_fraction=0.5, min_cells=4, coarse_mode=coarse_mode))
    assert pre.num_levels == 3 == len(ref.levels)
    for ell in range(2):
        x = np.linspace(-1, 1, pre.level_shape(ell)[2])
        assert_close(pre.level_matvec(ell, x), ref.levels[ell].matvec(x), TOL, f"{coarse_mode} L{ell}")
        assert_close(pre.vanka(ell, 0 * x, x, 2, 0.7), orc.vanka(ref.levels[ell], 0 * x, x, 2, 0.7), TOL,
                     f"{coarse_mode} vanka L{ell}")
    assert_close(pre.apply(syn.x), ref.apply(syn.x.copy()), VCYCLE_TOL, "V-cycle")


def test_rediscretize_fgmres_coarse_solve():
    """Rediscretized hierarchy whose coarsest level is solved by the coarse
    FGMRES (the child handle takes the parent's coarse-solver settings)."""
    from test_gpu_operator import _sized_case

    from paper_2603_28706_b200.stmg import MgConfig, StmgPreconditioner

    case, fx, syn = _sized_case(16, 16, 1, "exn")
    ctx = product_ctx(case, fx)
    s = oracle_slab(case, fx)
    ref = orc.StmgOracle(s, syn.U, variant_of(case), omega=0.7, surrogate=True, rep_fraction=0.5, min_cells=4,
                         coarse_mode="rediscretize")
    ref.coarse_fgmres = (2, 20, 1e-10)
    mg = MgConfig(rep_fraction=0.5, min_cells=4, coarse_mode="rediscretize", coarse_solver="fgmres", coarse_sweeps=2,
                  coarse_iters=20, coarse_rtol=1e-10)
    pre = StmgPreconditioner(None, ctx, syn.U, product_variant(case), mg)
    assert_close(pre.apply(syn.x), ref.apply(syn.x.copy()), 1e-8, "V-cycle with coarse FGMRES")


@pytest.mark.parametrize("solver,sweeps", [("vanka", 0), ("vanka", 12), ("auto", 12)])
def test_vcycle_iterative_coarse_solve(solver, sweeps):
    """MgConfig(coarse_solver=...): the coarsest level solved by Vanka steps
    from zero — against the oracle V-cycle with the same coarse
    sweeps; "auto" on a small hierarchy keeps the dense LU."""
    from test_gpu_operator import _sized_case

    from paper_2603_28706_b200.stmg import MgConfig, StmgPreconditioner

    case, fx, syn = _sized_case(16, 16, 1, "modn")
    ctx = product_ctx(case, fx)
    s = oracle_slab(case, fx)
    ref = orc.StmgOracle(s, syn.U, variant_of(case), omega=0.7, surrogate=True, rep_fraction=0.5, min_cells=4)
    if solver == "vanka":
        ref.coarse_sweeps, ref.coarse_omega = sweeps, 0.6
    mg = MgConfig(rep_fraction=0.5, min_cells=4, coarse_solver=solver, coarse_sweeps=sweeps, coarse_omega=0.6)
    pre = StmgPreconditioner(None, ctx, syn.U, product_variant(case), mg)
    assert pre.num_levels == 3
    assert_close(pre.apply(syn.x), ref.apply(syn.x.copy()), VCYCLE_TOL, f"V-cycle coarse={solver}/{sweeps}")


@pytest.mark.parametrize("iters,rtol", [(3, 0.0), (25, 1e-6)])
def test_vcycle_coarse_fgmres(iters, rtol):
    """MgConfig(coarse_solver="fgmres"): coarsest level by FGMRES right-preconditioned
    with 2 Vanka steps (CGS2, Givens) — against the oracle's restatement."""
    from test_gpu_operator import _sized_case

    from paper_2603_28706_b200.stmg import MgConfig, StmgPreconditioner

    case, fx, syn = _sized_case(16, 16, 1, "modn")
    ctx = product_ctx(case, fx)
    s = oracle_slab(case, fx)
    ref = orc.StmgOracle(s, syn.U, variant_of(case), omega=0.7, surrogate=True, rep_fraction=0.5, min_cells=4)
    ref.coarse_fgmres, ref.coarse_omega = (2, iters, rtol), 0.7
    mg = MgConfig(rep_fraction=0.5, min_cells=4, coarse_solver="fgmres", coarse_sweeps=2, coarse_iters=iters,
                  coarse_rtol=rtol)
    pre = StmgPreconditioner(None, ctx, syn.U, product_variant(case), mg)
    assert_close(pre.apply(syn.x), ref.apply(syn.x.copy()), 1e-8, f"V-cycle coarse fgmres {iters}/{rtol}")
