"""CPU oracle for the pdflow slab hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this module, and only as
the checker or the timed CPU baseline.  The product path
(``paper_2603_28706_b200``) never imports it.

This is a numpy restatement of the reference algorithm (arXiv 2603.28706,
package ``pdflow``), written cell-locally:

* every operator is a per-cell "local action" (volume + the cell's boundary
  sides) plus a per-interior-face local action (CIP), scattered with
  ``np.add.at``;
* element and face matrices are obtained by applying those local actions to
  unit vectors, and the global sparse Jacobian is their COO sum;
* patch matrices are extracted from the global matrices exactly as R_K A R_K'.

Parity pin: every public function is checked against golden vectors written
by running the reference itself (``tests/golden/make_golden.py``), see
``tests/test_oracle_golden.py``.

Reference citations (file:line in /root/reference/pkg/src/pdflow):
  tangent coefficients        constitutive.py:296-337
  shape / quadrature tables   femspace.py:46-106, forms.py:183-283
  dof maps                    femspace.py:127-155, forms.py:192-196
  velocity mass               femspace.py:199-211, pressure mass :214-217
  Jacobian action             forms.py:527-652, slab.py:176-205
  residual                    forms.py:343-516, slab.py:144-173
  assembled Jacobian          forms.py:655-763 (here: probed element matrices)
  patches / Vanka             solver/multigrid.py:251-340
  transfers                   solver/multigrid.py:90-154, 523-543
  Galerkin coarse operators   solver/multigrid.py:302-324, 459-470
  coarse solve / V-cycle      solver/multigrid.py:494-578
  mass norm                   solver/newton.py:96-121
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

# ---------------------------------------------------------------------------
# 1-D tables (femspace.py:46-75)
# ---------------------------------------------------------------------------


def gauss01(q: int = 4):
    x, w = np.polynomial.legendre.leggauss(q)
    return (x + 1.0) / 2.0, w / 2.0


def lag(x):
    x = np.asarray(x, dtype=float)
    return np.stack([(1.0 - x) * (1.0 - 2.0 * x), 4.0 * x * (1.0 - x), x * (2.0 * x - 1.0)], axis=-1)


def dlag(x):
    x = np.asarray(x, dtype=float)
    return np.stack([4.0 * x - 3.0, 4.0 - 8.0 * x, 4.0 * x - 1.0], axis=-1)


SIDES = ("bottom", "right", "top", "left")
NORMALS = {"bottom": (0.0, -1.0), "right": (1.0, 0.0), "top": (0.0, 1.0), "left": (-1.0, 0.0)}


def side_points(side, s):
    """Reference-cell coordinates (xh, yh) of the face points of a side."""
    one, zero = np.ones_like(s), np.zeros_like(s)
    return {"bottom": (s, zero), "right": (one, s), "top": (s, one), "left": (zero, s)}[side]


# ---------------------------------------------------------------------------
# Model / variant (constitutive.py:60-160, 323-337)
# ---------------------------------------------------------------------------


class OracleDomainError(ValueError):
    pass


@dataclass(frozen=True)
class Params:
    p: float
    delta: float
    nu: float
    nu_inf: float = 0.0


@dataclass(frozen=True)
class Variant:
    kind: str  # pic | exn | modn
    sigma_max: float = math.inf


def eta_of(params: Params, a_sq):
    return params.nu_inf + params.nu * (params.delta ** 2 + a_sq) ** ((params.p - 2.0) / 2.0)


def beta_of(params: Params, a_sq):
    return params.nu * (params.p - 2.0) * (params.delta ** 2 + a_sq) ** ((params.p - 4.0) / 2.0)


def tangent_eta_gamma(variant: Variant, params: Params, a_sq):
    """(eta, gamma) with T(B) = eta B + gamma (A:B) A (constitutive.py:323-337)."""
    if params.delta <= 0.0:
        raise OracleDomainError("derivative operations require delta > 0")
    dsq = params.delta ** 2 + a_sq
    mu = params.nu * dsq ** ((params.p - 2.0) / 2.0)
    eta = params.nu_inf + mu
    if variant.kind == "pic":
        return eta, np.zeros_like(eta)
    gamma = (params.p - 2.0) * mu / dsq
    if variant.kind == "modn":
        sigma = params.nu * (params.delta ** 2 + a_sq) ** ((params.p - 2.0) / 2.0) * np.sqrt(a_sq)
        with np.errstate(divide="ignore", invalid="ignore"):
            s = np.minimum(1.0, variant.sigma_max / np.where(sigma > 0.0, sigma, np.inf))
        gamma = s * gamma
    return eta, gamma


def sym3(gx, gy):
    """Symmetric gradient (a11, a22, a12) from component gradients.

    gx[..., d] = d/dx u_d, gy[..., d] = d/dy u_d."""
    return gx[..., 0], gy[..., 1], 0.5 * (gy[..., 0] + gx[..., 1])


def nsq3(a):
    return a[0] * a[0] + a[1] * a[1] + 2.0 * a[2] * a[2]


def dot3(a, b):
    return a[0] * b[0] + a[1] * b[1] + 2.0 * a[2] * b[2]


def neg_part(x):
    return 0.5 * (np.abs(x) - x)


# ---------------------------------------------------------------------------
# Geometry (mesh.py:50-148, femspace.py:109-155, forms.py:135-283)
# ---------------------------------------------------------------------------


@dataclass
class Grid:
    """Uniform nx-by-ny Q2/P1disc discretization with tags per boundary face
    (True = Dirichlet) in side order bottom, right, top, left."""

    nx: int
    ny: int
    extents: tuple = (0.0, 0.0, 1.0, 1.0)
    dirichlet: np.ndarray | None = None
    gamma1: float = 1.0e3
    gamma2: float = 1.0e3
    gamma_cip: float = 1.0
    g_hat: np.ndarray | None = None
    enable_viscous: bool = True
    enable_convection: bool = True
    enable_pressure: bool = True

    def __post_init__(self):
        x0, y0, x1, y1 = self.extents
        self.hx = (x1 - x0) / self.nx
        self.hy = (y1 - y0) / self.ny
        if self.dirichlet is None:
            self.dirichlet = np.ones(2 * (self.nx + self.ny), dtype=bool)
        self.dirichlet = np.asarray(self.dirichlet, dtype=bool)
        self.ncells = self.nx * self.ny
        self.nnx, self.nny = 2 * self.nx + 1, 2 * self.ny + 1
        self.nnodes = self.nnx * self.nny
        self.mv = 2 * self.nnodes
        self.mp = 3 * self.ncells
        self.nd = self.mv + self.mp
        self.s, self.w1 = gauss01(4)
        self.B, self.G = lag(self.s), dlag(self.s)  # (q, i)

    # -- integer maps (bit-exact targets) --------------------------------
    @property
    def cell_nodes(self) -> np.ndarray:
        c = np.arange(self.ncells)
        ci, cj = c % self.nx, c // self.nx
        jy, ix = np.divmod(np.arange(9), 3)
        return ((2 * cj[:, None] + jy[None, :]) * self.nnx + 2 * ci[:, None] + ix[None, :]).astype(np.int64)

    @property
    def cell_vdofs(self) -> np.ndarray:
        return (2 * self.cell_nodes[:, :, None] + np.arange(2)).reshape(-1, 18)

    @property
    def cell_patch_dofs(self) -> np.ndarray:
        pd = self.mv + 3 * np.arange(self.ncells)[:, None] + np.arange(3)[None, :]
        return np.hstack([self.cell_vdofs, pd]).astype(np.int64)

    def patch_ids(self, k1: int) -> np.ndarray:
        sp_ids = self.cell_patch_dofs
        return np.concatenate([sp_ids + mu * self.nd for mu in range(k1)], axis=1)

    def side_cells(self, side):
        if side == "bottom":
            return np.arange(self.nx)
        if side == "top":
            return (self.ny - 1) * self.nx + np.arange(self.nx)
        if side == "right":
            return np.arange(self.ny) * self.nx + self.nx - 1
        return np.arange(self.ny) * self.nx

    def side_mask(self, side):
        off = {"bottom": 0, "right": self.nx, "top": self.nx + self.ny, "left": 2 * self.nx + self.ny}[side]
        n = self.nx if side in ("bottom", "top") else self.ny
        return self.dirichlet[off:off + n]

    @property
    def all_dirichlet(self) -> bool:
        return bool(self.dirichlet.all())

    def cell_qpoints(self):
        """Physical quadrature coordinates (nc, 4, 4) each for x and y; axes (cell, qx, qy)."""
        x0, y0, _, _ = self.extents
        c = np.arange(self.ncells)
        ox = x0 + (c % self.nx) * self.hx
        oy = y0 + (c // self.nx) * self.hy
        X = ox[:, None, None] + self.s[None, :, None] * self.hx + 0.0 * self.s[None, None, :]
        Y = oy[:, None, None] + 0.0 * self.s[None, :, None] + self.s[None, None, :] * self.hy
        return X, Y

    # -- mass (femspace.py:199-217) --------------------------------------
    def mass1(self):
        return np.einsum("q,qi,qj->ij", self.w1, self.B, self.B)

    def local_mass(self):
        """9x9 node mass of one cell, node order a = 3 jy + ix."""
        m = self.mass1()
        return self.hx * self.hy * np.einsum("jJ,iI->jiJI", m, m).reshape(9, 9)

    def mass_v(self) -> sp.csr_matrix:
        cn = self.cell_nodes
        loc = self.local_mass()
        rows = np.repeat(cn, 9, axis=1).ravel()
        cols = np.tile(cn, (1, 9)).ravel()
        m = sp.coo_matrix((np.tile(loc.ravel(), self.ncells), (rows, cols)), shape=(self.nnodes,) * 2).tocsr()
        return sp.kron(m, sp.identity(2, format="csr"), format="csr")

    def mass_p_diag(self) -> np.ndarray:
        return np.tile(self.hx * self.hy * np.array([1.0, 1.0 / 12.0, 1.0 / 12.0]), self.ncells)

    # -- field gathers ------------------------------------------------------
    def local_v(self, vflat):
        """(nc, 3, 3, 2) nodal velocity per cell, axes (cell, jy, ix, comp)."""
        return vflat.reshape(-1, 2)[self.cell_nodes].reshape(self.ncells, 3, 3, 2)

    def local_p(self, pflat):
        return pflat.reshape(-1, 3)


# ---------------------------------------------------------------------------
# Pointwise evaluation helpers on a set of reference points
# ---------------------------------------------------------------------------


def _face_tables(grid: Grid, xh, yh):
    """(9, nq) values and (9, nq) x/y physical derivatives of the Q2 shapes at
    reference points (xh, yh), node order a = 3 jy + ix."""
    Lx, Ly, dLx, dLy = lag(xh), lag(yh), dlag(xh), dlag(yh)  # (nq, 3)
    N = np.einsum("qj,qi->jiq", Ly, Lx).reshape(9, -1)
    Nx = np.einsum("qj,qi->jiq", Ly, dLx).reshape(9, -1) / grid.hx
    Ny = np.einsum("qj,qi->jiq", dLy, Lx).reshape(9, -1) / grid.hy
    return N, Nx, Ny


def _p_table(xh, yh):
    return np.stack([np.ones_like(xh), xh - 0.5, yh - 0.5])  # (3, nq)


# ---------------------------------------------------------------------------
# Linearization state (forms.py:527-578)
# ---------------------------------------------------------------------------


@dataclass
class NodeLin:
    """Frozen per-node coefficients; arrays keep (cell, qx, qy) axes."""

    grid: Grid
    params: Params
    variant: Variant
    vstate: np.ndarray  # (Mv,)
    advect: np.ndarray  # (Mv,) lagged field for inflow / CIP weights
    vq: np.ndarray = field(repr=False, default=None)
    a3: tuple = field(repr=False, default=None)
    eta: np.ndarray = field(repr=False, default=None)
    gamma: np.ndarray = field(repr=False, default=None)


def volume_eval(grid: Grid, X):
    """Values and component gradients at the 4x4 volume points.

    X: (..., 3, 3, 2) with axes (jy, ix, comp). Returns val, gx, gy each (..., 4, 4, 2)
    with axes (qx, qy, comp)."""
    B, G = grid.B, grid.G
    val = np.einsum("xi,yj,...jid->...xyd", B, B, X)
    gx = np.einsum("xi,yj,...jid->...xyd", G, B, X) / grid.hx
    gy = np.einsum("xi,yj,...jid->...xyd", B, G, X) / grid.hy
    return val, gx, gy


def volume_test(grid: Grid, Fx, Fy, Fv):
    """sum_q [Fx dx N_a + Fy dy N_a + Fv N_a] with the volume weights.

    F*: (..., 4, 4, 2) axes (qx, qy, comp) already multiplied by the weights.
    Returns (..., 3, 3, 2) axes (jy, ix, comp)."""
    B, G = grid.B, grid.G
    out = np.einsum("xi,yj,...xyd->...jid", G, B, Fx) / grid.hx
    out = out + np.einsum("xi,yj,...xyd->...jid", B, G, Fy) / grid.hy
    out = out + np.einsum("xi,yj,...xyd->...jid", B, B, Fv)
    return out


def vol_weights(grid: Grid):
    return np.outer(grid.w1, grid.w1) * (grid.hx * grid.hy)  # (qx, qy)


def linearize(grid: Grid, params: Params, variant: Variant, vstate, advect=None) -> NodeLin:
    if params.delta <= 0.0:
        raise OracleDomainError("jacobian requires delta > 0")
    lin = NodeLin(grid, params, variant, np.asarray(vstate, float),
                  np.asarray(vstate if advect is None else advect, float))
    val, gx, gy = volume_eval(grid, grid.local_v(lin.vstate))
    lin.vq = val
    lin.a3 = sym3(gx, gy)
    lin.eta, lin.gamma = tangent_eta_gamma(variant, params, nsq3(lin.a3))
    return lin


# ---------------------------------------------------------------------------
# Per-cell local actions
# ---------------------------------------------------------------------------


def _lifting_face(grid: Grid, params: Params, side, cells):
    """(eta_d, beta_d, dgh3) at the face points of a side (forms.py:343-356)."""
    xh, yh = side_points(side, grid.s)
    nq = xh.size
    if grid.g_hat is None:
        z = np.zeros((cells.size, nq))
        dg = (z, z, z)
    else:
        N, Nx, Ny = _face_tables(grid, xh, yh)
        loc = grid.g_hat.reshape(-1, 2)[grid.cell_nodes[cells]]  # (nf, 9, 2)
        gx = np.einsum("aq,fad->fqd", Nx, loc)
        gy = np.einsum("aq,fad->fqd", Ny, loc)
        dg = sym3(gx, gy)
    a_sq = nsq3(dg)
    return eta_of(params, a_sq), beta_of(params, a_sq), dg


def _bs_test(Nx, Ny, n, eta_d, beta_d, dg, uf, wf):
    """Rows of <u, DS(Dg)[D phi] n> for face field uf (nf, nq, 2) -> (nf, 9, 2)
    (forms.py:359-371)."""
    gan = Nx * n[0] + Ny * n[1]  # (9, nq)
    gdotu = np.einsum("aq,fq->faq", Nx, uf[..., 0]) + np.einsum("aq,fq->faq", Ny, uf[..., 1])
    term = 0.5 * eta_d[:, None, :, None] * (gan[None, :, :, None] * uf[:, None, :, :]
                                            + gdotu[..., None] * np.asarray(n)[None, None, None, :])
    dgn = np.stack([dg[0] * n[0] + dg[2] * n[1], dg[2] * n[0] + dg[1] * n[1]], axis=-1)
    dgn_u = np.einsum("fqd,fqd->fq", dgn, uf)
    dgga = np.stack([dg[0][:, None, :] * Nx[None] + dg[2][:, None, :] * Ny[None],
                     dg[2][:, None, :] * Nx[None] + dg[1][:, None, :] * Ny[None]], axis=-1)  # (nf, 9, nq, 2)
    term = term + (beta_d * dgn_u)[:, None, :, None] * dgga
    return np.einsum("q,faqd->fad", wf, term)


def jacobian_local(lin: NodeLin, X, P):
    """Cell-local J x contributions.

    X: (nc, nb, 3, 3, 2) direction velocities, P: (nc, nb, 3) pressures.
    Returns yv (nc, nb, 3, 3, 2), yp (nc, nb, 3) — volume and boundary sides,
    forms.py:589-637."""
    g = lin.grid
    W = vol_weights(g)
    du, dgx, dgy = volume_eval(g, X)
    yv = np.zeros(X.shape)
    yp = np.zeros(P.shape)
    eta, gam = lin.eta[:, None], lin.gamma[:, None]
    A = tuple(a[:, None] for a in lin.a3)
    vq = lin.vq[:, None]
    Fx = np.zeros(du.shape)
    Fy = np.zeros(du.shape)
    if g.enable_viscous:
        Bt = sym3(dgx, dgy)
        ab = dot3(A, Bt)
        T = tuple(eta * b + gam * ab * a for b, a in zip(Bt, A))
        Fx[..., 0] += T[0]
        Fx[..., 1] += T[2]
        Fy[..., 0] += T[2]
        Fy[..., 1] += T[1]
    if g.enable_convection:
        # -(du_d v_e + v_d du_e) tested with d_e phi
        Fx -= du * vq[..., 0:1] + vq * du[..., 0:1]
        Fy -= du * vq[..., 1:2] + vq * du[..., 1:2]
    if g.enable_pressure:
        xh, yh = g.s[:, None] + 0 * g.s[None, :], 0 * g.s[:, None] + g.s[None, :]
        psi = np.stack([np.ones_like(xh), xh - 0.5, yh - 0.5])  # (3, qx, qy)
        dpq = np.einsum("jxy,cbj->cbxy", psi, P)
        Fx[..., 0] -= dpq
        Fy[..., 1] -= dpq
        divu = dgx[..., 0] + dgy[..., 1]
        yp -= np.einsum("xy,jxy,cbxy->cbj", W, psi, divu)
    yv += volume_test(g, Fx * W[..., None], Fy * W[..., None], np.zeros_like(Fx))

    nb = X.shape[1]
    for side in SIDES:
        cells = g.side_cells(side)
        dm = g.side_mask(side).astype(float)
        n = np.array(NORMALS[side])
        h = g.hx if side in ("bottom", "top") else g.hy
        xh, yh = side_points(side, g.s)
        N, Nx, Ny = _face_tables(g, xh, yh)
        PS = _p_table(xh, yh)
        wf = g.w1 * h
        Xf = X[cells].reshape(cells.size, nb, 9, 2)
        uf = np.einsum("aq,fbad->fbqd", N, Xf)
        ugx = np.einsum("aq,fbad->fbqd", Nx, Xf)
        ugy = np.einsum("aq,fbad->fbqd", Ny, Xf)
        un = uf @ n
        Sloc = lin.vstate.reshape(-1, 2)[g.cell_nodes[cells]]
        vf = np.einsum("aq,fad->fqd", N, Sloc)[:, None]
        vn = vf @ n
        advf = np.einsum("aq,fad->fqd", N, lin.advect.reshape(-1, 2)[g.cell_nodes[cells]])
        wneg = neg_part(advf @ n)[:, None]
        bc = np.zeros((cells.size, nb, 9, 2))
        bp = np.zeros((cells.size, nb, 3))
        if g.enable_convection:
            bc += np.einsum("q,fbqd,aq->fbad", wf, vn[..., None] * uf + un[..., None] * vf, N)
        if dm.any():
            db = np.zeros_like(bc)
            dbp = np.zeros_like(bp)
            if g.enable_viscous:
                sgx = np.einsum("aq,fad->fqd", Nx, Sloc)
                sgy = np.einsum("aq,fad->fqd", Ny, Sloc)
                af = sym3(sgx, sgy)
                eta_f, gam_f = tangent_eta_gamma(lin.variant, lin.params, nsq3(af))
                Bf = sym3(ugx, ugy)
                afb = tuple(a[:, None] for a in af)
                ab = dot3(afb, Bf)
                T = tuple(eta_f[:, None] * b + gam_f[:, None] * ab * a for b, a in zip(Bf, afb))
                Tn = np.stack([T[0] * n[0] + T[2] * n[1], T[2] * n[0] + T[1] * n[1]], axis=-1)
                db -= np.einsum("q,fbqd,aq->fbad", wf, Tn, N)
                eta_d, beta_d, dg = _lifting_face(g, lin.params, side, cells)
                for b in range(nb):
                    db[:, b] -= _bs_test(Nx, Ny, n, eta_d, beta_d, dg, uf[:, b], wf)
                pen = (g.gamma1 / h) * eta_d[:, None, :, None] * uf + (g.gamma2 / h) * un[..., None] * n
                db += np.einsum("q,fbqd,aq->fbad", wf, pen, N)
            if g.enable_convection:
                db -= np.einsum("q,fbqd,aq->fbad", wf, wneg[..., None] * uf, N)
            if g.enable_pressure:
                dpf = np.einsum("jq,fbj->fbq", PS, P[cells])
                db += np.einsum("q,fbq,aq->fba", wf, dpf, N)[..., None] * n
                dbp += np.einsum("q,fbq,jq->fbj", wf, un, PS)
            bc += db * dm[:, None, None, None]
            bp += dbp * dm[:, None, None]
        yv[cells] += bc.reshape(cells.size, nb, 3, 3, 2)
        yp[cells] += bp
    return yv, yp


def _cip_geometry(g: Grid):
    """[(cells_L, cells_R, n, h, NL, NnL, NnR)] for vertical then horizontal faces
    (forms.py:251-283)."""
    out = []
    if g.nx > 1:
        jj, ii = np.meshgrid(np.arange(g.ny), np.arange(g.nx - 1), indexing="ij")
        cl = (jj * g.nx + ii).ravel()
        n = np.array([1.0, 0.0])
        NL, NxL, NyL = _face_tables(g, *side_points("right", g.s))
        _, NxR, NyR = _face_tables(g, *side_points("left", g.s))
        out.append((cl, cl + 1, n, g.hy, NL, NxL, NxR))
    if g.ny > 1:
        jj, ii = np.meshgrid(np.arange(g.ny - 1), np.arange(g.nx), indexing="ij")
        cl = (jj * g.nx + ii).ravel()
        n = np.array([0.0, 1.0])
        NL, NxL, NyL = _face_tables(g, *side_points("top", g.s))
        _, NxR, NyR = _face_tables(g, *side_points("bottom", g.s))
        out.append((cl, cl + g.nx, n, g.hx, NL, NyL, NyR))
    return out


def cip_weights(lin: NodeLin):
    """|v_hat . n| from the left/lower cell's lagged trace, per face group."""
    g = lin.grid
    res = []
    if not (g.enable_convection and g.gamma_cip > 0.0):
        return res
    for cl, cr, n, h, NL, NnL, NnR in _cip_geometry(g):
        loc = lin.advect.reshape(-1, 2)[g.cell_nodes[cl]]
        res.append(np.abs(np.einsum("aq,fad,d->fq", NL, loc, n)))
    return res


def cip_local(lin: NodeLin, XL, XR, group: int, wts):
    """Face-local CIP action; XL, XR (nf, nb, 9, 2) -> contributions to L and R
    (forms.py:639-650)."""
    g = lin.grid
    cl, cr, n, h, NL, NnL, NnR = _cip_geometry(g)[group]
    wf = g.w1 * h
    jump = np.einsum("aq,fbad->fbqd", NnL, XL) - np.einsum("aq,fbad->fbqd", NnR, XR)
    coef = g.gamma_cip * h * h
    core = coef * wf[None, None, :, None] * wts[:, None, :, None] * jump
    yl = np.einsum("fbqd,aq->fbad", core, NnL)
    yr = -np.einsum("fbqd,aq->fbad", core, NnR)
    return yl, yr


def spatial_jacobian_apply(lin: NodeLin, x):
    """J_mu x for one node (forms.py:581-652); x flat (nd,)."""
    g = lin.grid
    X = g.local_v(x[:g.mv])[:, None]
    P = g.local_p(x[g.mv:])[:, None]
    yv, yp = jacobian_local(lin, X, P)
    out_v = np.zeros((g.nnodes, 2))
    np.add.at(out_v, g.cell_nodes, yv[:, 0].reshape(g.ncells, 9, 2))
    wts = cip_weights(lin)
    for grp, w in enumerate(wts):
        cl, cr = _cip_geometry(g)[grp][:2]
        Xv = g.local_v(x[:g.mv]).reshape(g.ncells, 9, 2)
        yl, yr = cip_local(lin, Xv[cl][:, None], Xv[cr][:, None], grp, w)
        np.add.at(out_v, g.cell_nodes[cl], yl[:, 0])
        np.add.at(out_v, g.cell_nodes[cr], yr[:, 0])
    return np.concatenate([out_v.reshape(-1), yp[:, 0].reshape(-1)])


# ---------------------------------------------------------------------------
# Slab operators (slab.py:144-205)
# ---------------------------------------------------------------------------


@dataclass
class Slab:
    grid: Grid
    params: Params
    k: int
    nodes: np.ndarray
    weights: np.ndarray
    K_t: np.ndarray
    m_t: np.ndarray
    tau: float
    t_start: float = 0.0
    v_minus: np.ndarray | None = None
    forcing: object = None  # f(x, y, t) -> (..., 2) or None

    @property
    def k1(self):
        return self.k + 1

    @property
    def ndof(self):
        return self.k1 * self.grid.nd

    @property
    def tau_w(self):
        return self.tau * self.weights

    def node_times(self):
        return self.t_start + self.tau * self.nodes


def mass_apply_v(grid: Grid, V):
    """M_x V for velocity blocks V (..., Mv) using cell-local Kronecker masses."""
    V = np.atleast_2d(V)
    m = grid.mass1()
    out = np.zeros((V.shape[0], grid.nnodes, 2))
    for r in range(V.shape[0]):
        loc = grid.local_v(V[r])
        y = grid.hx * grid.hy * np.einsum("jJ,iI,cJId->cjid", m, m, loc)
        np.add.at(out[r], grid.cell_nodes, y.reshape(grid.ncells, 9, 2))
    return out.reshape(V.shape[0], -1)


class SlabJacobianOracle:
    """out_mu = tau w_mu J_mu x_mu + sum_nu K_t[mu,nu] M x_nu (slab.py:193-205)."""

    def __init__(self, slab: Slab, U, variant: Variant):
        self.slab = slab
        g = slab.grid
        self.lins = [linearize(g, slab.params, variant, U[mu, :g.mv]) for mu in range(slab.k1)]

    def apply(self, dU):
        s, g = self.slab, self.slab.grid
        out = np.empty_like(dU)
        for mu, lin in enumerate(self.lins):
            out[mu] = s.tau_w[mu] * spatial_jacobian_apply(lin, dU[mu])
        out[:, :g.mv] += mass_apply_v(g, s.K_t @ dU[:, :g.mv])
        return out

    def matvec(self, x):
        return self.apply(x.reshape(self.slab.k1, -1)).reshape(-1)


def spatial_residual(slab: Slab, vstate, pstate, t, advect=None):
    """F_mu = <f,w> + B(g_hat, w) - A(u)(w) (forms.py:435-516)."""
    g, params = slab.grid, slab.params
    if params.delta <= 0.0:
        raise OracleDomainError("spatial residual requires delta > 0")
    adv = vstate if advect is None else advect
    W = vol_weights(g)
    Xs = g.local_v(vstate)
    vq, gx, gy = volume_eval(g, Xs)
    a3 = sym3(gx, gy)
    Fx = np.zeros(vq.shape)
    Fy = np.zeros(vq.shape)
    Fv = np.zeros(vq.shape)
    if slab.forcing is not None:
        QX, QY = g.cell_qpoints()
        Fv += np.asarray(slab.forcing(QX, QY, t), dtype=float)
    if g.enable_viscous:
        eta = eta_of(params, nsq3(a3))
        S = tuple(eta * a for a in a3)
        Fx[..., 0] -= S[0]
        Fx[..., 1] -= S[2]
        Fy[..., 0] -= S[2]
        Fy[..., 1] -= S[1]
    if g.enable_convection:
        Fx += vq * vq[..., 0:1]
        Fy += vq * vq[..., 1:2]
    rp = np.zeros((g.ncells, 3))
    if g.enable_pressure:
        xh, yh = g.s[:, None] + 0 * g.s[None, :], 0 * g.s[:, None] + g.s[None, :]
        psi = np.stack([np.ones_like(xh), xh - 0.5, yh - 0.5])
        pq = np.einsum("jxy,cj->cxy", psi, g.local_p(pstate))
        Fx[..., 0] += pq
        Fy[..., 1] += pq
        rp += np.einsum("xy,jxy,cxy->cj", W, psi, gx[..., 0] + gy[..., 1])
    yv = volume_test(g, Fx * W[..., None], Fy * W[..., None], Fv * W[..., None])
    rv = np.zeros((g.nnodes, 2))
    np.add.at(rv, g.cell_nodes, yv.reshape(g.ncells, 9, 2))

    for side in SIDES:
        cells = g.side_cells(side)
        dm = g.side_mask(side).astype(float)
        n = np.array(NORMALS[side])
        h = g.hx if side in ("bottom", "top") else g.hy
        xh, yh = side_points(side, g.s)
        N, Nx, Ny = _face_tables(g, xh, yh)
        PS = _p_table(xh, yh)
        wf = g.w1 * h
        loc = vstate.reshape(-1, 2)[g.cell_nodes[cells]]
        vf = np.einsum("aq,fad->fqd", N, loc)
        vn = vf @ n
        advf = np.einsum("aq,fad->fqd", N, adv.reshape(-1, 2)[g.cell_nodes[cells]])
        aneg = neg_part(advf @ n)
        bc = np.zeros((cells.size, 9, 2))
        bp = np.zeros((cells.size, 3))
        if g.enable_convection:
            bc -= np.einsum("q,fqd,aq->fad", wf, vn[..., None] * vf, N)
        if dm.any():
            db = np.zeros_like(bc)
            dbp = np.zeros_like(bp)
            eta_d, beta_d, dg = _lifting_face(g, params, side, cells)
            if g.enable_viscous:
                af = sym3(np.einsum("aq,fad->fqd", Nx, loc), np.einsum("aq,fad->fqd", Ny, loc))
                ef = eta_of(params, nsq3(af))
                Sn = np.stack([ef * (af[0] * n[0] + af[2] * n[1]), ef * (af[2] * n[0] + af[1] * n[1])], axis=-1)
                db += np.einsum("q,fqd,aq->fad", wf, Sn, N)
                db += _bs_test(Nx, Ny, n, eta_d, beta_d, dg, vf, wf)
                pen = (g.gamma1 / h) * eta_d[..., None] * vf + (g.gamma2 / h) * vn[..., None] * n
                db -= np.einsum("q,fqd,aq->fad", wf, pen, N)
            if g.enable_convection:
                db += np.einsum("q,fqd,aq->fad", wf, aneg[..., None] * vf, N)
            if g.enable_pressure:
                pf = np.einsum("jq,fj->fq", PS, g.local_p(pstate)[cells])
                db -= np.einsum("q,fq,aq->fa", wf, pf, N)[..., None] * n
                dbp -= np.einsum("q,fq,jq->fj", wf, vn, PS)
            bc += db * dm[:, None, None]
            bp += dbp * dm[:, None]
        np.add.at(rv, g.cell_nodes[cells], bc)
        np.add.at(rp, cells, bp)

    if g.enable_convection and g.gamma_cip > 0.0:
        Xv = Xs.reshape(g.ncells, 9, 2)
        Av = g.local_v(adv).reshape(g.ncells, 9, 2)
        for cl, cr, n, h, NL, NnL, NnR in _cip_geometry(g):
            wts = np.abs(np.einsum("aq,fad,d->fq", NL, Av[cl], n))
            wf = g.w1 * h
            jump = np.einsum("aq,fad->fqd", NnL, Xv[cl]) - np.einsum("aq,fad->fqd", NnR, Xv[cr])
            core = g.gamma_cip * h * h * wf[None, :, None] * wts[..., None] * jump
            np.add.at(rv, g.cell_nodes[cl], -np.einsum("fqd,aq->fad", core, NnL))
            np.add.at(rv, g.cell_nodes[cr], np.einsum("fqd,aq->fad", core, NnR))

    res = np.concatenate([rv.reshape(-1), rp.reshape(-1)])
    if g.g_hat is not None:
        res += nitsche_vector(slab, g.g_hat)
    return res


def nitsche_vector(slab: Slab, gv):
    """B_gamma(g, .) over Dirichlet faces (forms.py:374-412)."""
    g, params = slab.grid, slab.params
    rv = np.zeros((g.nnodes, 2))
    rp = np.zeros((g.ncells, 3))
    for side in SIDES:
        dm = g.side_mask(side).astype(float)
        if not dm.any():
            continue
        cells = g.side_cells(side)
        n = np.array(NORMALS[side])
        h = g.hx if side in ("bottom", "top") else g.hy
        xh, yh = side_points(side, g.s)
        N, Nx, Ny = _face_tables(g, xh, yh)
        PS = _p_table(xh, yh)
        wf = g.w1 * h
        vf = np.einsum("aq,fad->fqd", N, gv.reshape(-1, 2)[g.cell_nodes[cells]])
        vn = vf @ n
        bc = np.zeros((cells.size, 9, 2))
        bp = np.zeros((cells.size, 3))
        eta_d, beta_d, dg = _lifting_face(g, params, side, cells)
        if g.enable_viscous:
            bc -= _bs_test(Nx, Ny, n, eta_d, beta_d, dg, vf, wf)
            pen = (g.gamma1 / h) * eta_d[..., None] * vf + (g.gamma2 / h) * vn[..., None] * n
            bc += np.einsum("q,fqd,aq->fad", wf, pen, N)
        if g.enable_convection:
            bc -= np.einsum("q,fqd,aq->fad", wf, neg_part(vn)[..., None] * vf, N)
        if g.enable_pressure:
            bp += np.einsum("q,fq,jq->fj", wf, vn, PS)
        np.add.at(rv, g.cell_nodes[cells], bc * dm[:, None, None])
        np.add.at(rp, cells, bp * dm[:, None])
    return np.concatenate([rv.reshape(-1), rp.reshape(-1)])


def slab_residual(slab: Slab, U, advect=None):
    """R = tau w F(U) - [(K_t x M) V - (m_t x M) v_minus; 0] (slab.py:162-173)."""
    g = slab.grid
    times = slab.node_times()
    R = np.empty_like(U)
    for mu in range(slab.k1):
        adv = None if advect is None else advect[mu, :g.mv]
        R[mu] = slab.tau_w[mu] * spatial_residual(slab, U[mu, :g.mv], U[mu, g.mv:], float(times[mu]), adv)
    W = slab.K_t @ U[:, :g.mv] - np.outer(slab.m_t, slab.v_minus)
    R[:, :g.mv] -= mass_apply_v(g, W)
    return R


# ---------------------------------------------------------------------------
# Assembled matrices by probing the local actions (forms.py:655-763)
# ---------------------------------------------------------------------------


def spatial_jacobian_matrix(lin: NodeLin) -> sp.csr_matrix:
    """Global sparse J_mu from element (21x21) and CIP face (36x36) matrices."""
    g = lin.grid
    nc = g.ncells
    I21 = np.eye(21)
    X = np.broadcast_to(I21[:, :18].reshape(21, 3, 3, 2), (nc, 21, 3, 3, 2)).copy()
    P = np.broadcast_to(I21[:, 18:], (nc, 21, 3)).copy()
    yv, yp = jacobian_local(lin, X, P)  # (nc, 21 cols, ...)
    E = np.concatenate([yv.reshape(nc, 21, 18), yp], axis=2)  # E[c, col, row]
    dofs = g.cell_patch_dofs
    rows = [np.broadcast_to(dofs[:, None, :], (nc, 21, 21)).ravel()]
    cols = [np.broadcast_to(dofs[:, :, None], (nc, 21, 21)).ravel()]
    vals = [E.ravel()]
    wts = cip_weights(lin)
    I18 = np.eye(18).reshape(18, 9, 2)
    for grp, w in enumerate(wts):
        cl, cr = _cip_geometry(g)[grp][:2]
        nf = cl.size
        Z = np.zeros((nf, 18, 9, 2))
        U18 = np.broadcast_to(I18, (nf, 18, 9, 2))
        for side_in, (XL, XR) in enumerate(((U18, Z), (Z, U18))):
            yl, yr = cip_local(lin, XL, XR, grp, w)
            cdofs = g.cell_vdofs[cl] if side_in == 0 else g.cell_vdofs[cr]
            for yy, rdofs in ((yl, g.cell_vdofs[cl]), (yr, g.cell_vdofs[cr])):
                rows.append(np.broadcast_to(rdofs[:, None, :], (nf, 18, 18)).ravel())
                cols.append(np.broadcast_to(cdofs[:, :, None], (nf, 18, 18)).ravel())
                vals.append(yy.reshape(nf, 18, 18).ravel())
    mat = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(g.nd, g.nd))
    return mat.tocsr()


# ---------------------------------------------------------------------------
# Patches and Vanka (solver/multigrid.py:251-340)
# ---------------------------------------------------------------------------


def extract_blocks(A: sp.csr_matrix, ids: np.ndarray) -> np.ndarray:
    A = A.tocsr()
    out = np.empty((ids.shape[0], ids.shape[1], ids.shape[1]))
    for c in range(ids.shape[0]):
        out[c] = A[ids[c]][:, ids[c]].toarray()
    return out


@dataclass
class LevelOp:
    """One level: grid, spatial node blocks (csr), velocity mass, slab data."""

    grid: Grid
    j_nodes: list
    mass_v: sp.csr_matrix
    K_t: np.ndarray
    tau_w: np.ndarray
    matvec: object = None
    ids: np.ndarray | None = None
    mats: np.ndarray | None = None
    invs: np.ndarray | None = None

    @property
    def k1(self):
        return self.tau_w.size


def sparse_matvec(lv: LevelOp):
    g = lv.grid

    def mv(x):
        X = x.reshape(lv.k1, g.nd)
        out = np.empty_like(X)
        for mu in range(lv.k1):
            out[mu] = lv.tau_w[mu] * (lv.j_nodes[mu] @ X[mu])
        out[:, :g.mv] += (lv.mass_v @ (lv.K_t @ X[:, :g.mv]).T).T
        return out.reshape(-1)

    return mv


def patch_matrices(lv: LevelOp, blocks: list):
    g = lv.grid
    k1 = lv.k1
    sp_ids = g.cell_patch_dofs
    mass = extract_blocks(lv.mass_v, g.cell_vdofs)
    nodeb = [extract_blocks(b, sp_ids) for b in blocks]
    D = 21 * k1
    A = np.zeros((g.ncells, D, D))
    for mu in range(k1):
        for nu in range(k1):
            A[:, 21 * mu:21 * mu + 18, 21 * nu:21 * nu + 18] += lv.K_t[mu, nu] * mass
        A[:, 21 * mu:21 * mu + 21, 21 * mu:21 * mu + 21] += lv.tau_w[mu] * nodeb[mu]
    return g.patch_ids(k1), A


def vanka(lv: LevelOp, d, r, steps, omega):
    out = np.array(d, dtype=float)
    for _ in range(steps):
        defect = r - lv.matvec(out)
        upd = np.einsum("pij,pj->pi", lv.invs, defect[lv.ids])
        np.add.at(out, lv.ids, omega * upd)
    return out


# ---------------------------------------------------------------------------
# Transfers (solver/multigrid.py:90-154)
# ---------------------------------------------------------------------------


def transfer(gc: Grid, gf: Grid):
    """(P, P_v, P_p, inject_v) for nested meshes, fine = 2x coarse."""
    if gf.nx != 2 * gc.nx or gf.ny != 2 * gc.ny:
        raise ValueError("transfer requires a mesh refined exactly once")
    IX, IY = np.meshgrid(np.arange(gf.nnx), np.arange(gf.nny))
    cx = np.clip(IX // 4, 0, gc.nx - 1).ravel()
    cy = np.clip(IY // 4, 0, gc.ny - 1).ravel()
    lx = lag(IX.ravel() / 4.0 - cx)
    ly = lag(IY.ravel() / 4.0 - cy)
    rows, cols, vals = [], [], []
    fine_idx = np.arange(gf.nnodes)
    for jy in range(3):
        for jx in range(3):
            rows.append(fine_idx)
            cols.append((2 * cy + jy) * gc.nnx + 2 * cx + jx)
            vals.append(ly[:, jy] * lx[:, jx])
    pn = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                       shape=(gf.nnodes, gc.nnodes)).tocsr()
    pn.eliminate_zeros()
    P_v = sp.kron(pn, sp.identity(2, format="csr"), format="csr")
    c = np.arange(gc.ncells)
    ci, cj = c % gc.nx, c // gc.nx
    r_, c_, v_ = [], [], []
    for oy in (0, 1):
        for ox in (0, 1):
            child = (2 * cj + oy) * gf.nx + 2 * ci + ox
            bf, bc = 3 * child, 3 * c
            for rr, cc, vv in ((bf, bc, 1.0), (bf, bc + 1, (2 * ox - 1) / 4.0), (bf, bc + 2, (2 * oy - 1) / 4.0),
                               (bf + 1, bc + 1, 0.5), (bf + 2, bc + 2, 0.5)):
                r_.append(rr)
                c_.append(cc)
                v_.append(np.full(gc.ncells, vv))
    P_p = sp.coo_matrix((np.concatenate(v_), (np.concatenate(r_), np.concatenate(c_))),
                        shape=(gf.mp, gc.mp)).tocsr()
    P = sp.block_diag([P_v, P_p], format="csr")
    CX, CY = np.meshgrid(np.arange(gc.nnx), np.arange(gc.nny))
    fnode = (2 * CY * gf.nnx + 2 * CX).ravel()
    inject_v = np.stack([2 * fnode, 2 * fnode + 1], axis=1).ravel()
    return P, P_v, P_p, inject_v


def coarse_grid(g: Grid) -> Grid:
    """Coarse grid inheriting the first tag of every fine side (multigrid.py:171-182)."""
    nx, ny = g.nx // 2, g.ny // 2
    first = {s: g.side_mask(s)[0] for s in SIDES}
    tags = np.concatenate([np.full(nx, first["bottom"]), np.full(ny, first["right"]),
                           np.full(nx, first["top"]), np.full(ny, first["left"])])
    return Grid(nx, ny, g.extents, tags, g.gamma1, g.gamma2, g.gamma_cip, None,
                g.enable_viscous, g.enable_convection, g.enable_pressure)


def hierarchy(g: Grid, min_cells: int):
    grids = [g]
    m = g
    while m.nx > min_cells and m.nx % 2 == 0 and m.ny > min_cells and m.ny % 2 == 0:
        m = coarse_grid(m)
        grids.append(m)
    return grids[::-1]


# ---------------------------------------------------------------------------
# STMG V-cycle (solver/multigrid.py:386-578)
# ---------------------------------------------------------------------------


class StmgOracle:
    def __init__(self, slab: Slab, U, variant: Variant, omega=0.7, pre=2, post=2, surrogate=True,
                 rep_fraction=0.5, min_cells=4, coarse_mode="galerkin"):
        self.slab = slab
        self.omega, self.pre, self.post = omega, pre, post
        grids = hierarchy(slab.grid, min_cells)
        self.grids = grids
        self.transfers = [transfer(grids[i], grids[i + 1]) for i in range(len(grids) - 1)]
        jac = SlabJacobianOracle(slab, U, variant)
        self.jac = jac
        j_fine = [spatial_jacobian_matrix(lin) for lin in jac.lins]
        L = len(grids)
        levels = [None] * L
        levels[-1] = LevelOp(grids[-1], j_fine, grids[-1].mass_v(), slab.K_t, slab.tau_w, jac.matvec)
        # rediscretize (multigrid.py:302-324, 406-431): node states injected level
        # by level (pressure 0, unused by the Jacobian), g_hat injected alike
        states = [np.asarray(U[mu][:slab.grid.mv], float) for mu in range(slab.k1)]
        ghat = slab.grid.g_hat
        for ell in range(L - 2, -1, -1):
            P, P_v, _, inject_v = self.transfers[ell]
            if coarse_mode == "galerkin":
                blocks = [(P.T @ jb @ P).tocsr() for jb in levels[ell + 1].j_nodes]
                mass_c = (P_v.T @ levels[ell + 1].mass_v @ P_v).tocsr()
            elif coarse_mode == "rediscretize":
                states = [st[inject_v] for st in states]
                if ghat is not None:
                    ghat = np.asarray(ghat)[inject_v]
                    grids[ell] = replace(grids[ell], g_hat=ghat)
                blocks = [spatial_jacobian_matrix(linearize(grids[ell], slab.params, variant, st)) for st in states]
                mass_c = grids[ell].mass_v()
            else:
                raise ValueError(coarse_mode)
            levels[ell] = LevelOp(grids[ell], blocks, mass_c, slab.K_t, slab.tau_w)
            levels[ell].matvec = sparse_matvec(levels[ell])
        for ell, lv in enumerate(levels):
            if ell == L - 1 and surrogate:
                if slab.k1 > 1:
                    from_nodes = _lagrange_at(slab.nodes, rep_fraction)
                    rep = from_nodes @ U
                else:
                    rep = U[0]
                rep_lin = linearize(slab.grid, slab.params, variant, rep[:slab.grid.mv])
                rep_block = spatial_jacobian_matrix(rep_lin)
                lv.ids, lv.mats = patch_matrices(lv, [rep_block] * slab.k1)
            else:
                lv.ids, lv.mats = patch_matrices(lv, lv.j_nodes)
            lv.invs = np.linalg.inv(lv.mats)
        self.levels = levels
        self.coarse_lu = None  # built on first use (the dense coarse LU is O(N^2) memory)
        self.coarse_sweeps = None  # set (with coarse_omega) for the iterative coarse solve
        self.coarse_omega = omega
        self.coarse_fgmres = None  # (sweeps, iters, rtol): coarse FGMRES with Vanka preconditioning

    def _coarse(self):
        lv = self.levels[0]
        g = lv.grid
        k1, nd, mv = lv.k1, g.nd, g.mv
        A = np.zeros((k1 * nd, k1 * nd))
        Md = lv.mass_v.toarray()
        for mu in range(k1):
            for nu in range(k1):
                A[mu * nd:mu * nd + mv, nu * nd:nu * nd + mv] += lv.K_t[mu, nu] * Md
            A[mu * nd:(mu + 1) * nd, mu * nd:(mu + 1) * nd] += lv.tau_w[mu] * lv.j_nodes[mu].toarray()
        if g.all_dirichlet:
            scale = np.mean(np.abs(A.diagonal()))
            mpd = g.mass_p_diag()
            for mu in range(k1):
                z = np.zeros(k1 * nd)
                zp = np.zeros(g.mp)
                zp[0::3] = mpd[0::3]
                z[mu * nd + mv:(mu + 1) * nd] = zp
                z /= np.linalg.norm(z)
                A += scale * np.outer(z, z)
        self.coarse_lu = sla.lu_factor(A)

    def vcycle(self, ell, b):
        if ell == 0:
            if self.coarse_fgmres is not None:
                return self._coarse_fgmres(b, *self.coarse_fgmres)
            if self.coarse_sweeps is not None:
                # iterative coarse solve (the product's MgConfig(coarse_solver="vanka"),
                # no reference counterpart): Vanka steps from zero on the coarsest level
                return vanka(self.levels[0], np.zeros_like(b), b, self.coarse_sweeps, self.coarse_omega)
            if self.coarse_lu is None:
                self._coarse()
            return sla.lu_solve(self.coarse_lu, b)
        lv = self.levels[ell]
        d = vanka(lv, np.zeros_like(b), b, self.pre, self.omega)
        r = b - lv.matvec(d)
        P = self.transfers[ell - 1][0]
        k1 = lv.k1
        rc = (P.T @ r.reshape(k1, -1).T).T.reshape(-1)
        e = self.vcycle(ell - 1, rc)
        d = d + (P @ e.reshape(k1, -1).T).T.reshape(-1)
        return vanka(lv, d, b, self.post, self.omega)

    def _coarse_fgmres(self, b, sweeps, iters, rtol):
        """Restatement of the product's coarsest-level FGMRES (csrc/pdst_mg.cu
        coarse_fgmres): right preconditioning by `sweeps` Vanka steps from zero,
        Euclidean, classical Gram-Schmidt twice, Givens rotations."""
        lv = self.levels[0]
        beta = float(np.sqrt(b @ b))
        if not beta > 0.0:
            return np.zeros_like(b)
        V = [b / beta]
        Z = []
        H = np.zeros((iters + 1, iters))
        cs, sn = np.zeros(iters), np.zeros(iters)
        g = np.zeros(iters + 1)
        g[0] = beta
        k = 0
        for j in range(iters):
            z = vanka(lv, np.zeros_like(b), V[j], sweeps, self.coarse_omega)
            Z.append(z)
            w = lv.matvec(z)
            Vm = np.array(V)
            for _ in range(2):
                hc = Vm @ w
                w = w - Vm.T @ hc
                H[: j + 1, j] += hc
            hn = float(np.sqrt(w @ w))
            H[j + 1, j] = hn
            if hn > 0.0:
                V.append(w / hn)
            for i in range(j):
                a, c = H[i, j], H[i + 1, j]
                H[i, j], H[i + 1, j] = cs[i] * a + sn[i] * c, -sn[i] * a + cs[i] * c
            a, c = H[j, j], H[j + 1, j]
            r = float(np.hypot(a, c))
            cs[j], sn[j] = (a / r, c / r) if r > 0.0 else (1.0, 0.0)
            H[j, j], H[j + 1, j] = r, 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            k = j + 1
            if abs(g[j + 1]) <= rtol * beta or not hn > 0.0:
                break
        y = np.zeros(k)
        for i in range(k - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1:k] @ y[i + 1:]) / H[i, i] if H[i, i] != 0.0 else 0.0
        return np.array(Z[:k]).T @ y

    def apply(self, r):
        z = self.vcycle(len(self.levels) - 1, r)
        g = self.slab.grid
        if g.all_dirichlet:
            mpd = g.mass_p_diag()
            area = mpd[0::3].sum()
            Z = z.reshape(self.slab.k1, g.nd)
            for mu in range(self.slab.k1):
                p = Z[mu, g.mv:]
                p[0::3] -= float(np.dot(mpd[0::3], p[0::3])) / area
        return z


def _lagrange_at(nodes, that):
    out = np.ones(nodes.size)
    for mu in range(nodes.size):
        val = 1.0
        for nu in range(nodes.size):
            if nu != mu:
                val = val * (that - nodes[nu]) / (nodes[mu] - nodes[nu])
        out[mu] = val
    return out


# ---------------------------------------------------------------------------
# Mass norm (solver/newton.py:96-121)
# ---------------------------------------------------------------------------


def mass_apply(slab: Slab, x):
    g = slab.grid
    X = x.reshape(slab.k1, g.nd)
    out = np.empty_like(X)
    out[:, :g.mv] = slab.tau_w[:, None] * mass_apply_v(g, X[:, :g.mv])
    out[:, g.mv:] = slab.tau_w[:, None] * (g.mass_p_diag() * X[:, g.mv:])
    return out.reshape(x.shape)


def mass_norm(slab: Slab, x):
    return float(np.sqrt(np.dot(x.reshape(-1), mass_apply(slab, x.reshape(-1)))))
