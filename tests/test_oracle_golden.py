"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  Floating outputs: normwise 1e-12 (L2 and
Linf, relative); integer maps: bit-exact."""

import numpy as np
import pytest
import scipy.sparse as sp

from helpers import CASES, assert_close, load, oracle_slab, orc, variant_of
from cases import TRANSFER_PAIRS

TOL = 1e-12
# The coarsest-level dense LU of the pinned, nearly singular all-Dirichlet
# system amplifies rounding: measured 2e-11 between two correct
# implementations (numpy oracle vs reference) on p6_k2_pic_exact.
VCYCLE_TOL = 1e-9


@pytest.mark.parametrize("case", CASES, ids=lambda c: c.name)
def test_apply_residual_mass(case):
    fx = load(case.name)
    s = oracle_slab(case, fx)
    jac = orc.SlabJacobianOracle(s, fx["U"], variant_of(case))
    assert_close(jac.matvec(fx["x"]), fx["y"], TOL, "jacobian")
    assert_close(orc.slab_residual(s, fx["U"]), fx["R"], TOL, "residual")
    assert_close(orc.mass_apply(s, fx["x"]), fx["mass_x"], TOL, "mass")
    assert abs(orc.mass_norm(s, fx["x"]) - float(fx["mnorm_x"])) <= TOL * float(fx["mnorm_x"])
    assert np.array_equal(s.grid.cell_nodes, fx["cell_nodes"])
    assert np.array_equal(s.grid.cell_patch_dofs, fx["cell_patch_dofs"])


@pytest.mark.parametrize("case", [c for c in CASES if c.patches], ids=lambda c: c.name)
def test_patches_vanka_vcycle(case):
    fx = load(case.name)
    s = oracle_slab(case, fx)
    pre = orc.StmgOracle(s, fx["U"], variant_of(case), omega=case.cfg.omega, surrogate=case.surrogate,
                         rep_fraction=case.cfg.rep_fraction, min_cells=case.min_cells, coarse_mode=case.coarse_mode)
    fine = pre.levels[-1]
    assert [g.nx for g in pre.grids] == list(fx["levels_nx"])
    assert np.array_equal(fine.ids, fx["patch_ids"])
    assert_close(fine.mats, fx["patch_mats"], TOL, "patch matrices")
    assert_close(orc.vanka(fine, fx["d0"], fx["x"], 1, case.cfg.omega), fx["vanka_d"], TOL, "vanka 1")
    assert_close(orc.vanka(fine, fx["d0"], fx["x"], 2, case.cfg.omega), fx["vanka_d2"], TOL, "vanka 2")
    assert_close(orc.vanka(fine, 0 * fx["x"], fx["x"], 1, case.cfg.omega), fx["vanka_zero"], TOL, "vanka d0=0")
    for ell in range(len(pre.levels) - 1):
        lv = pre.levels[ell]
        assert_close(lv.matvec(fx[f"L{ell}_x"]), fx[f"L{ell}_Ax"], TOL, f"galerkin L{ell}")
        assert_close(lv.mats, fx[f"L{ell}_patch_mats"], TOL, f"coarse patches L{ell}")
        assert_close(orc.vanka(lv, 0 * fx[f"L{ell}_x"], fx[f"L{ell}_x"], 1, case.cfg.omega), fx[f"L{ell}_vanka"],
                     TOL, f"coarse vanka L{ell}")
    assert_close(pre.apply(fx["x"].copy()), fx["vcycle"], VCYCLE_TOL, "vcycle")


@pytest.mark.parametrize("pair", TRANSFER_PAIRS, ids=lambda p: f"{p[0]}x{p[1]}")
def test_transfers_bit_exact(pair):
    fx = load("transfers")
    cx, cy = pair
    tag = f"{cx}x{cy}"
    P, _, _, inj = orc.transfer(orc.Grid(cx, cy), orc.Grid(2 * cx, 2 * cy))
    Pg = sp.coo_matrix((fx[f"{tag}_P_val"], (fx[f"{tag}_P_row"], fx[f"{tag}_P_col"])),
                       shape=tuple(fx[f"{tag}_P_shape"])).tocsr()
    assert (P != Pg).nnz == 0
    assert np.array_equal(inj, fx[f"{tag}_inject_v"])
    assert np.array_equal(P.T @ fx[f"{tag}_xf"], fx[f"{tag}_restrict"])
    assert np.array_equal(P @ fx[f"{tag}_xc"], fx[f"{tag}_prolong"])


def test_radau_known_answers():
    from paper_2603_28706_b200.radau import gauss_radau, temporal_matrices

    b = gauss_radau(1)
    np.testing.assert_allclose(b.nodes, [1 / 3, 1.0], rtol=0, atol=1e-15)
    np.testing.assert_allclose(b.weights, [0.75, 0.25], rtol=0, atol=1e-15)
    tm = temporal_matrices(b)
    np.testing.assert_allclose(tm.K_t, [[9 / 8, 3 / 8], [-9 / 8, 5 / 8]], rtol=0, atol=1e-14)
    np.testing.assert_allclose(tm.m_t, [1.5, -0.5], rtol=0, atol=1e-14)
    for case in CASES:
        fx = load(case.name)
        bk = gauss_radau(case.cfg.k)
        tk = temporal_matrices(bk)
        np.testing.assert_allclose(bk.nodes, fx["nodes"], rtol=0, atol=1e-15)
        np.testing.assert_allclose(bk.weights, fx["weights"], rtol=0, atol=1e-15)
        np.testing.assert_allclose(tk.K_t, fx["K_t"], rtol=0, atol=1e-13)


def test_dof_count_known_answer():
    g = orc.Grid(512, 512)
    assert g.nd == 2_887_682
