"""Self-checks of the Taylor-Hood Q2/Q1 restatement (oracle/th_oracle.py).
The reference has no Taylor-Hood space, so nothing pins it;
these checks pin it instead:

* the pressure operator integrates exactly: for a quadratic velocity field v
  (exactly represented by Q2) on an all-Dirichlet mesh, (G v)_q =
  -(psi_q, div v) + <psi_q, v.n> = (grad psi_q, v), computed independently
  by a 6-point Gauss rule per cell;
* the velocity-pressure blocks of the slab Jacobian are each other's
  transposes (b(w, q) tested both ways), per Radau node;
* all-Dirichlet: the per-node constant pressure is in the kernel of J;
* exact Newton: J = -dR/dU (central differences with the lagged CIP / inflow
  weights frozen, slab.py:144-159), incl. a g_hat lifting and Neumann sides;
* the velocity-velocity part equals the P1disc oracle's with its pressure
  terms switched off.
"""

import numpy as np
import pytest

from helpers import orc
from oracle import th_oracle as th


def _slab(nx, ny, k, seed, neumann=(), ghat=False, p=1.4, delta=1e-2, nu_inf=1e-3):
    from paper_2603_28706_b200.radau import gauss_radau, temporal_matrices

    tags = np.ones(2 * (nx + ny), dtype=bool)
    offs = {"bottom": (0, nx), "right": (nx, ny), "top": (nx + ny, nx), "left": (2 * nx + ny, ny)}
    for s in neumann:
        o, n = offs[s]
        tags[o:o + n] = False
    rng = np.random.default_rng(seed)
    g0 = orc.Grid(nx, ny, (0.0, 0.0, 1.2, 1.0), tags, 40.0, 30.0, 0.7)
    gh = None
    if ghat:
        gh = 0.3 * rng.standard_normal(g0.mv)
    g = orc.Grid(nx, ny, (0.0, 0.0, 1.2, 1.0), tags, 40.0, 30.0, 0.7, gh)
    b = gauss_radau(k)
    tm = temporal_matrices(b)
    slab = orc.Slab(g, orc.Params(p, delta, 1.0, nu_inf), k, b.nodes, b.weights, tm.K_t, tm.m_t, 0.02, 0.1,
                    rng.standard_normal(g.mv), None)
    mv, mp, nd = th.th_sizes(g)
    U = rng.standard_normal((k + 1, nd))
    return slab, U, rng


def test_pressure_operator_integrates_exactly():
    nx, ny = 5, 4
    g = orc.Grid(nx, ny, (0.0, 0.0, 1.2, 1.0))
    X, Y = [a.ravel() for a in np.meshgrid(np.linspace(0, 1.2, 2 * nx + 1), np.linspace(0, 1.0, 2 * ny + 1))]

    def field(x, y):
        return np.stack([0.5 + x * x - 0.3 * x * y, y * y + 0.7 * x - 0.2], axis=-1)

    v = field(X, Y).reshape(-1)
    Gv = th.pressure_operator(g) @ v
    # independent: (grad psi_q, v) with a 6-point Gauss rule per cell
    s, w = np.polynomial.legendre.leggauss(6)
    s, w = 0.5 * (s + 1.0), 0.5 * w
    ref = np.zeros((nx + 1) * (ny + 1))
    hx, hy = 1.2 / nx, 1.0 / ny
    for cj in range(ny):
        for ci in range(nx):
            for a, (sx, wx) in enumerate(zip(s, w)):
                for sy, wy in zip(s, w):
                    x, y = (ci + sx) * hx, (cj + sy) * hy
                    vv = field(np.array(x), np.array(y))
                    for jy in range(2):
                        for jx in range(2):
                            lx, ly = (1 - sx, sx)[jx], (1 - sy, sy)[jy]
                            dlx, dly = (-1.0, 1.0)[jx] / hx, (-1.0, 1.0)[jy] / hy
                            ref[(cj + jy) * (nx + 1) + ci + jx] += wx * wy * hx * hy * (dlx * ly * vv[0] + lx * dly * vv[1])
    assert np.allclose(Gv, ref, rtol=0, atol=1e-13 * np.abs(ref).max())


@pytest.mark.parametrize("k,neumann", [(1, ()), (0, ("top",)), (2, ("left", "bottom"))])
def test_pressure_blocks_are_transposes_and_nullspace(k, neumann):
    slab, U, _ = _slab(3, 2, k, 5 + k, neumann)
    A = th.th_jacobian_matrix(slab, U, orc.Variant("exn"))
    mv, mp, nd = th.th_sizes(slab.grid)
    for mu in range(k + 1):
        v = slice(mu * nd, mu * nd + mv)
        p = slice(mu * nd + mv, (mu + 1) * nd)
        assert np.allclose(A[v, p], A[p, v].T, rtol=0, atol=1e-14 * np.abs(A).max())
        assert not A[p, p].any()  # no pressure-pressure block
    if not neumann:
        for mu in range(k + 1):
            e = np.zeros(A.shape[1])
            e[mu * nd + mv:(mu + 1) * nd] = 1.0
            assert np.abs(A @ e).max() <= 1e-13 * np.abs(A).max()


@pytest.mark.parametrize("k,neumann,ghat", [(1, (), False), (1, ("right",), True), (2, ("top",), False),
                                            (0, (), True)])
def test_exact_newton_is_the_residual_derivative(k, neumann, ghat):
    slab, U, rng = _slab(4, 3, k, 11 + k, neumann, ghat)
    x = rng.standard_normal(U.size)
    J = th.th_slab_matvec(slab, U, orc.Variant("exn"), x)
    eps = 1e-6
    Rp = th.th_slab_residual(slab, U + eps * x.reshape(U.shape), advect=U)
    Rm = th.th_slab_residual(slab, U - eps * x.reshape(U.shape), advect=U)
    fd = -(Rp - Rm).reshape(-1) / (2 * eps)
    assert np.linalg.norm(fd - J) <= 1e-7 * np.linalg.norm(J)


def test_velocity_part_is_the_p1disc_operator_without_pressure():
    slab, U, rng = _slab(4, 4, 1, 3)
    g = slab.grid
    mv, mp, nd = th.th_sizes(g)
    x = rng.standard_normal(U.size)
    x.reshape(U.shape)[:, mv:] = 0.0
    J = th.th_slab_matvec(slab, U, orc.Variant("modn", 0.5), x)
    from dataclasses import replace

    gv = replace(g, enable_pressure=False)
    Up = np.zeros((2, gv.nd))
    Up[:, :mv] = U[:, :mv]
    xp = np.zeros((2, gv.nd))
    xp[:, :mv] = x.reshape(U.shape)[:, :mv]
    ref = orc.SlabJacobianOracle(replace(slab, grid=gv), Up, orc.Variant("modn", 0.5)).apply(xp)
    assert np.array_equal(J.reshape(U.shape)[:, :mv], ref[:, :mv])
