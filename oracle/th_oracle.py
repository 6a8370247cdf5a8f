"""CPU restatement of the slab operators with a Taylor-Hood Q2/Q1 space pair
-- TEST INFRASTRUCTURE ONLY (same import rules as ``pdst_oracle``).

BASELINE.json's north_star asks for "Q_k/Q_{k-1} Taylor-Hood cells"; the
reference implements only Q2/P1disc (femspace.py:1-12, 98-106, 146-160;
Taylor-Hood is a non-goal at SPEC.md:346).  This module restates the
reference's forms with the pressure space swapped for continuous bilinear
Q1 on the cell vertices: nothing in the reference pins it,
so the GPU kernels are checked against it together with size-independent
self-checks (tests/test_th_oracle.py, tests/test_gpu_taylor_hood.py).

Every pressure term of the reference's Jacobian and residual is linear in the
pressure (or, for the pressure rows, in the velocity) and is the bilinear form
    b(w, q) = - (q, div w) + < q, w . n >_{Gamma_D}
(forms.py:589-603 volume, 615-635 Dirichlet sides; residual :467-471,
:500-503; Nitsche vector :408-409).  So, with the pressure terms switched off
in the reference's own forms (DiscretizationConfig.enable_pressure = False,
forms.py:75-77) for the velocity-velocity part,
    J_TH x = J_vel x_v + [G' x_p ; G x_v],
    F_TH(u) = F_vel(v) - [G' pi ; G v] + [0 ; N(g_hat)],
with G the pressure-test operator (rows: Q1 vertices, columns: velocity dofs)
of b and N(g_hat) = <g_hat . n, q>_{Gamma_D}.  The slab composition
(slab.py:162-205) is unchanged: tau w_mu scales the spatial blocks, the time
mass acts on the velocity only.

Vector layout per Radau node: the reference's velocity block (Mv, node-major
interleaved), then (nx+1)(ny+1) vertex pressures, row-major (y, x).
Pressure mass (for the mass norm): consistent Q1, hx hy M1_y (x) M1_x with
M1 = [[1/3, 1/6], [1/6, 1/3]].
"""

from __future__ import annotations

from dataclasses import replace

import numpy as np
import scipy.sparse as sp

from . import pdst_oracle as orc

__all__ = ["ThGrid", "th_sizes", "pressure_operator", "th_slab_matvec", "th_slab_residual", "th_mass_apply",
           "th_jacobian_matrix"]


def th_sizes(g: orc.Grid):
    """(Mv, Mp, nd) of the Taylor-Hood pair on g."""
    mp = (g.nx + 1) * (g.ny + 1)
    return g.mv, mp, g.mv + mp


def _q1(s):
    s = np.asarray(s, float)
    return np.stack([1.0 - s, s], axis=-1)  # (..., 2): l_0, l_1


def _dq1(s):
    s = np.asarray(s, float)
    return np.stack([-np.ones_like(s), np.ones_like(s)], axis=-1)


def cell_vertices(g: orc.Grid) -> np.ndarray:
    """(nc, 4) vertex indices of each cell, local order 2 jy + ix."""
    c = np.arange(g.ncells)
    ci, cj = c % g.nx, c // g.nx
    out = np.empty((g.ncells, 4), dtype=np.int64)
    for jy in range(2):
        for ix in range(2):
            out[:, 2 * jy + ix] = (cj + jy) * (g.nx + 1) + ci + ix
    return out


def pressure_operator(g: orc.Grid) -> sp.csr_matrix:
    """G: Mp x Mv, (G v)_q = -(psi_q, div v) + <psi_q, v . n>_{Gamma_D}."""
    B, G1 = g.B, g.G  # (q, i) Q2 values / derivatives at the Gauss points
    s, w = g.s, g.w1
    L = _q1(s)  # (q, 2)
    W = np.outer(w, w) * (g.hx * g.hy)  # (qx, qy)
    # volume: -(psi_j, d_x phi_a) for comp 0 and -(psi_j, d_y phi_a) for comp 1
    # psi_j(qx, qy) = L[qx, jx] L[qy, jy]; phi_a = B[qx, ix] B[qy, iy] (a = 3 iy + ix)
    loc = np.zeros((4, 9, 2))
    for jy in range(2):
        for jx in range(2):
            psi = np.outer(L[:, jx], L[:, jy])  # (qx, qy)
            for iy in range(3):
                for ix in range(3):
                    dx = np.outer(G1[:, ix], B[:, iy]) / g.hx
                    dy = np.outer(B[:, ix], G1[:, iy]) / g.hy
                    loc[2 * jy + jx, 3 * iy + ix, 0] = -np.sum(W * psi * dx)
                    loc[2 * jy + jx, 3 * iy + ix, 1] = -np.sum(W * psi * dy)
    cv, cn = cell_vertices(g), g.cell_nodes
    rows, cols, vals = [], [], []
    for j in range(4):
        for a in range(9):
            for d in range(2):
                rows.append(cv[:, j])
                cols.append(2 * cn[:, a] + d)
                vals.append(np.full(g.ncells, loc[j, a, d]))
    # Dirichlet sides: + <psi_j, phi_a n_d>
    for side in orc.SIDES:
        dm = g.side_mask(side)
        if not dm.any():
            continue
        cells = g.side_cells(side)[dm]
        n = np.array(orc.NORMALS[side])
        h = g.hx if side in ("bottom", "top") else g.hy
        xh, yh = orc.side_points(side, s)
        N = orc._face_tables(g, xh, yh)[0]  # (9, q)
        Pq = np.einsum("qj,qi->jiq", _q1(yh), _q1(xh)).reshape(4, -1)  # (4, q), j = 2 jy + jx
        wf = w * h
        fl = np.einsum("q,jq,aq->ja", wf, Pq, N)  # (4, 9)
        for j in range(4):
            for a in range(9):
                for d in range(2):
                    if n[d] == 0.0:
                        continue
                    rows.append(cv[cells, j])
                    cols.append(2 * cn[cells, a] + d)
                    vals.append(np.full(cells.size, fl[j, a] * n[d]))
    mp = (g.nx + 1) * (g.ny + 1)
    return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(mp, g.mv)).tocsr()


def ghat_vector(g: orc.Grid, ghat) -> np.ndarray:
    """N(g_hat)_q = <g_hat . n, psi_q>_{Gamma_D} (forms.py:408-409 with Q1 tests)."""
    mp = (g.nx + 1) * (g.ny + 1)
    out = np.zeros(mp)
    if ghat is None:
        return out
    cv = cell_vertices(g)
    for side in orc.SIDES:
        dm = g.side_mask(side)
        if not dm.any():
            continue
        cells = g.side_cells(side)[dm]
        n = np.array(orc.NORMALS[side])
        h = g.hx if side in ("bottom", "top") else g.hy
        xh, yh = orc.side_points(side, g.s)
        N = orc._face_tables(g, xh, yh)[0]
        Pq = np.einsum("qj,qi->jiq", _q1(yh), _q1(xh)).reshape(4, -1)
        gf = np.einsum("aq,fad->fqd", N, np.asarray(ghat).reshape(-1, 2)[g.cell_nodes[cells]])
        gn = gf @ n
        np.add.at(out, cv[cells], np.einsum("q,fq,jq->fj", g.w1 * h, gn, Pq))
    return out


def _vel_grid(g: orc.Grid) -> orc.Grid:
    return replace(g, enable_pressure=False)


def th_slab_matvec(slab: orc.Slab, U, variant, x):
    """J_TH x (slab.py:193-205 with the TH pressure): U (k1, nd_TH), x flat."""
    g = slab.grid
    mv, mp, nd = th_sizes(g)
    k1 = slab.k1
    gv = _vel_grid(g)
    sv = replace(slab, grid=gv)
    # the velocity-velocity part through the reference restatement (pressure off, P1disc-sized zero pressure)
    Up = np.zeros((k1, gv.nd))
    Up[:, :mv] = U[:, :mv]
    X = x.reshape(k1, nd)
    Xp = np.zeros((k1, gv.nd))
    Xp[:, :mv] = X[:, :mv]
    Yv = orc.SlabJacobianOracle(sv, Up, variant).apply(Xp)
    Gm = pressure_operator(g)
    out = np.zeros((k1, nd))
    for mu in range(k1):
        tw = slab.tau_w[mu]
        out[mu, :mv] = Yv[mu, :mv] + tw * (Gm.T @ X[mu, mv:])
        out[mu, mv:] = tw * (Gm @ X[mu, :mv])
    return out.reshape(-1)


def th_slab_residual(slab: orc.Slab, U, advect=None):
    """R_TH (slab.py:162-173, forms.py:435-516 with the TH pressure)."""
    g = slab.grid
    mv, mp, nd = th_sizes(g)
    k1 = slab.k1
    gv = _vel_grid(g)
    sv = replace(slab, grid=gv)
    Up = np.zeros((k1, gv.nd))
    Up[:, :mv] = U[:, :mv]
    adv = None
    if advect is not None:
        adv = np.zeros((k1, gv.nd))
        adv[:, :mv] = np.asarray(advect).reshape(k1, nd)[:, :mv]
    Rv = orc.slab_residual(sv, Up, adv)
    Gm = pressure_operator(g)
    Ng = ghat_vector(g, g.g_hat)
    R = np.zeros((k1, nd))
    for mu in range(k1):
        tw = slab.tau_w[mu]
        R[mu, :mv] = Rv[mu, :mv] - tw * (Gm.T @ U[mu, mv:])
        R[mu, mv:] = tw * (Ng - Gm @ U[mu, :mv])
    return R


def th_mass_apply(slab: orc.Slab, x):
    """Block mass (newton.py:96-121) with the consistent Q1 pressure mass."""
    g = slab.grid
    mv, mp, nd = th_sizes(g)
    X = x.reshape(slab.k1, nd)
    m1 = np.array([[1.0 / 3.0, 1.0 / 6.0], [1.0 / 6.0, 1.0 / 3.0]])
    Mp = g.hx * g.hy * sp.kron(_q1_line_mass(g.ny, m1), _q1_line_mass(g.nx, m1), format="csr")
    out = np.empty_like(X)
    out[:, :mv] = slab.tau_w[:, None] * orc.mass_apply_v(g, X[:, :mv])
    out[:, mv:] = slab.tau_w[:, None] * (Mp @ X[:, mv:].T).T
    return out.reshape(x.shape)


def _q1_line_mass(n, m1):
    M = np.zeros((n + 1, n + 1))
    for c in range(n):
        M[c:c + 2, c:c + 2] += m1
    return sp.csr_matrix(M)


def th_jacobian_matrix(slab: orc.Slab, U, variant) -> np.ndarray:
    """Dense slab Jacobian by columns of th_slab_matvec (small meshes)."""
    n = slab.k1 * th_sizes(slab.grid)[2]
    A = np.empty((n, n))
    e = np.zeros(n)
    for j in range(n):
        e[j] = 1.0
        A[:, j] = th_slab_matvec(slab, U, variant, e)
        e[j] = 0.0
    return A


class ThGrid:
    """Convenience: vertex coordinates of a grid's Q1 pressure nodes, row-major (y, x)."""

    def __init__(self, g: orc.Grid):
        x0, y0, x1, y1 = g.extents
        xs = np.linspace(x0, x1, g.nx + 1)
        ys = np.linspace(y0, y1, g.ny + 1)
        self.X, self.Y = np.meshgrid(xs, ys)
