"""Space-time multigrid preconditioner on the GPU.

Drop-in counterparts of (file:line into /root/reference/pkg/src/pdflow):
  MgConfig                                  solver/multigrid.py:55-73
  MgGeometry.from_fine (hierarchy rule)     solver/multigrid.py:164-191
  StmgPreconditioner(.apply, levels)        solver/multigrid.py:386-578
  StmgFactory(.mg, .build)                  solver/newton.py:129-137

Everything below the Python objects — Galerkin coarse operators, exact and
surrogate patches, the coarsest dense solve, Vanka sweeps, transfers and the
V-cycle — runs in libpdst on the device.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .operators import SlabJacobian, _f64, _is_torch

__all__ = ["MgConfig", "MgGeometry", "MgLevel", "PatchSet", "StmgPreconditioner", "StmgFactory", "mg_vcycle"]

_COARSE = {"dense": 0, "vanka": 1, "auto": 2, "fgmres": 3}  # pdst_set_coarse_solver kinds


@dataclass
class MgConfig:
    """Smoothing, surrogate and rebuild parameters (multigrid.py:55-73)."""

    pre_smooth: int = 2
    post_smooth: int = 2
    omega: float = 0.7
    surrogate: bool = True
    rep_fraction: float = 0.5
    rebuild_rho: float = 0.9
    rebuild_factor: float = 2.0
    coarse_mode: str = "galerkin"
    min_cells: int = 4
    # coarsest-level solve (no reference counterpart beyond "dense", the
    # reference's LU of the pinned slab system, multigrid.py:494-520):
    #   "vanka"  coarse_sweeps Vanka steps from zero with coarse_omega (default omega);
    #   "fgmres" FGMRES right-preconditioned by coarse_sweeps Vanka steps, at most
    #            coarse_iters iterations or relative residual coarse_rtol;
    #   "auto"   dense up to 4096 dofs, else "fgmres".
    # a 5-level hierarchy of a 2048^2 mesh ends at 128^2
    # (362,500 dofs), beyond the dense LU.
    coarse_solver: str = "dense"
    coarse_sweeps: int | None = None  # default 30 ("vanka") / 2 ("fgmres", "auto")
    coarse_omega: float | None = None
    coarse_iters: int = 30
    coarse_rtol: float = 1.0e-6

    def __post_init__(self):
        if not 0.0 < self.omega <= 1.0:
            raise ValueError("omega must lie in (0, 1]")
        if self.coarse_solver not in _COARSE:
            raise ValueError(f"unknown coarse solver {self.coarse_solver!r}")
        if self.coarse_sweeps is not None and self.coarse_sweeps < 0:
            raise ValueError("coarse_sweeps must be >= 0")
        if not 1 <= self.coarse_iters <= 1000 or not self.coarse_rtol >= 0.0:
            raise ValueError("coarse_iters must lie in [1, 1000] and coarse_rtol be >= 0")
        if self.coarse_omega is not None and not 0.0 < self.coarse_omega <= 1.0:
            raise ValueError("coarse_omega must lie in (0, 1]")
        if self.coarse_mode not in ("galerkin", "rediscretize"):
            raise ValueError(f"unknown coarse mode {self.coarse_mode!r}")


def _mg_get(mg, name, default):
    """Read an MgConfig field, falling back to the default for fields a
    pdflow ``MgConfig`` (multigrid.py:55-73) does not carry."""
    v = getattr(mg, name, default)
    return default if v is None and default is not None else v


class MgGeometry:
    """State-independent level list (multigrid.py:157-195): ``discs`` coarsest
    first, the finest being the slab's own Discretization object.

    ``from_fine`` applies the reference's coarsening rule (halve while both
    cell counts exceed min_cells and are even; coarse boundary faces inherit
    the fine side tags).  The transfers themselves live in libpdst (exact
    dyadic stencils); ``transfers[i]`` records the (coarse, fine) cell counts
    of the level pair i -> i+1."""

    def __init__(self, discs, transfers=None):
        self.discs = list(discs)
        self.transfers = transfers if transfers is not None else [
            ((a.mesh.nx, a.mesh.ny), (b.mesh.nx, b.mesh.ny)) for a, b in zip(self.discs[:-1], self.discs[1:])]

    @classmethod
    def from_fine(cls, fine, min_cells: int = 4) -> "MgGeometry":
        from .problem import SIDES, Discretization, QuadMesh

        discs = [fine]
        m = fine.mesh
        while m.nx > min_cells and m.nx % 2 == 0 and m.ny > min_cells and m.ny % 2 == 0:
            tags = getattr(m, "boundary_tags", None)
            ctags = None
            if tags is not None:
                offs = {"bottom": 0, "right": m.nx, "top": m.nx + m.ny, "left": 2 * m.nx + m.ny}
                ctags = []
                for side in SIDES:
                    n = m.nx // 2 if side in ("bottom", "top") else m.ny // 2
                    ctags += [tags[offs[side]]] * n
                ctags = np.array(ctags, dtype=object)
            cm = QuadMesh(m.nx // 2, m.ny // 2, m.x0, m.y0, m.x1, m.y1, max(getattr(m, "level", 0) - 1, 0), ctags)
            discs.append(Discretization(cm))
            m = cm
        discs.reverse()
        return cls(discs)

    @property
    def num_levels(self) -> int:
        return len(self.discs)


class PatchSet:
    """Device-resident patches of one level (multigrid.py:198-209).

    ``ids`` is the reference's index set (cell_patch_dofs + mu nd, node-major,
    int64, bit-exact); ``matrices`` reads the composed patch matrices back
    from libpdst (where they are retained).  The factorized inverses stay on
    the device (stored transposed, or temporally diagonalized for surrogate
    patches) and have no host copy."""

    def __init__(self, owner, level):
        self._owner = owner
        self.level = level

    @property
    def ids(self):
        nx, ny, _ = self._owner.level_shape(self.level)
        return _patch_ids(nx, ny, self._owner.k1)

    @property
    def matrices(self):
        return self._owner.patch_matrices(self.level)


def _patch_ids(nx, ny, k1):
    """cell_patch_dofs of forms.py:192-196 replicated over the Radau nodes (multigrid.py:273-275)."""
    row = 2 * nx + 1
    nd = 2 * row * (2 * ny + 1) + 3 * nx * ny
    mv = 2 * row * (2 * ny + 1)
    c = np.arange(nx * ny)
    ci, cj = c % nx, c // nx
    a = np.arange(9)
    node = (2 * cj[:, None] + a[None, :] // 3) * row + (2 * ci[:, None] + a[None, :] % 3)
    vd = np.stack([2 * node, 2 * node + 1], axis=-1).reshape(-1, 18)
    pd = mv + 3 * c[:, None] + np.arange(3)[None, :]
    sp = np.concatenate([vd, pd], axis=1).astype(np.int64)
    return np.concatenate([sp + mu * nd for mu in range(k1)], axis=1)


class MgLevel:
    """One level of the device hierarchy with the attributes of the
    reference's MgLevel (multigrid.py:212-231): ``matvec`` (the matrix-free
    slab Jacobian on the finest level, the Galerkin level operator below),
    ``patches``, ``K_t``, ``tau_w``; ``vanka_smooth(level, ...)`` runs the
    level's sweeps in libpdst."""

    def __init__(self, owner, index, disc):
        self._owner = owner
        self.index = index
        self.disc = disc
        self.K_t = np.asarray(owner.ctx.tmat.K_t, dtype=float)
        self.tau_w = owner.ctx.tau * np.asarray(owner.ctx.basis.weights, dtype=float)
        self.patches = PatchSet(owner, index)

    @property
    def n_nodes(self):
        return self.tau_w.size

    @property
    def slab_dim(self):
        return self._owner.level_shape(self.index)[2]

    def matvec(self, x):
        if self.index == self._owner.num_levels - 1:
            return self._owner.jac.matvec(x)
        return self._owner.level_matvec(self.index, x)

    def smooth(self, d, r, steps, omega):
        return self._owner.vanka(self.index, d, r, steps, omega)


class StmgPreconditioner:
    """One state-bound V-cycle: Galerkin hierarchy, patches and coarsest solve
    (multigrid.py:386-578), with the reference's positional signature
    ``StmgPreconditioner(geometry, ctx, U, variant, mg, reuse_fine_patches=None)``.

    ``geometry`` is a pdflow ``MgGeometry`` or this module's (or None: the
    levels follow ``mg.min_cells``); as in the reference its finest
    Discretization must be ``ctx.disc`` (multigrid.py:404-405).  ``mg`` may be
    a pdflow ``MgConfig``: the fields it lacks (``coarse_solver``, ...) take
    this module's defaults.  ``reuse_fine_patches`` is accepted for signature
    compatibility; the reference never passes it (newton.py:136-137)."""

    def __init__(self, geometry, ctx, U, variant, mg=None, reuse_fine_patches=None, *, device=0,
                 jac: SlabJacobian | None = None):
        if geometry is not None and geometry.discs[-1] is not ctx.disc:
            raise ValueError("hierarchy finest level must match the slab discretization")
        if reuse_fine_patches is not None:
            raise NotImplementedError("reuse_fine_patches: the finest patches live in the previous handle "
                                      "(the reference never passes this argument, newton.py:136-137)")
        self.geometry = geometry
        self.mg = mg = mg if mg is not None else MgConfig()
        omega = float(_mg_get(mg, "omega", 0.7))
        if not 0.0 < omega <= 1.0:
            raise ValueError("omega must lie in (0, 1]")
        coarse_mode = _mg_get(mg, "coarse_mode", "galerkin")
        if coarse_mode not in ("galerkin", "rediscretize"):
            raise ValueError(f"unknown coarse mode {coarse_mode!r}")
        coarse_solver = _mg_get(mg, "coarse_solver", "dense")
        if coarse_solver not in _COARSE:
            raise ValueError(f"unknown coarse solver {coarse_solver!r}")
        self.ctx = ctx
        self.jac = jac or SlabJacobian(ctx, U, variant, device=device)
        self.dev = self.jac.dev
        nl = C.c_int(0)
        if geometry is not None:
            L.check(L.lib().pdst_hierarchy_depth(self.dev.h, int(geometry.num_levels), C.byref(nl)),
                    "pdst_hierarchy_depth")
        else:
            L.check(L.lib().pdst_hierarchy(self.dev.h, int(_mg_get(mg, "min_cells", 4)), C.byref(nl)),
                    "pdst_hierarchy")
        self.num_levels = nl.value
        if geometry is not None:
            for ell, d in enumerate(geometry.discs):
                if self.level_shape(ell)[:2] != (d.mesh.nx, d.mesh.ny):
                    raise ValueError(f"level {ell}: geometry mesh {d.mesh.nx}x{d.mesh.ny} is not the "
                                     f"device hierarchy's {self.level_shape(ell)[:2]}")
        cw = _mg_get(mg, "coarse_omega", None)
        cw = omega if cw is None else float(cw)
        sw = _mg_get(mg, "coarse_sweeps", None)
        sw = (30 if coarse_solver == "vanka" else 2) if sw is None else int(sw)
        L.check(L.lib().pdst_set_coarse_solver(self.dev.h, _COARSE[coarse_solver], sw, cw,
                                               int(_mg_get(mg, "coarse_iters", 30)),
                                               float(_mg_get(mg, "coarse_rtol", 1.0e-6))), "pdst_set_coarse_solver")
        # coarse operators: Galerkin P' J P, or each coarse level re-linearized on
        # its own mesh at the injected state (multigrid.py:302-324, 406-431)
        L.check(L.lib().pdst_set_coarse_mode(self.dev.h, 1 if coarse_mode == "rediscretize" else 0),
                "pdst_set_coarse_mode")
        self.omega = omega
        self.pre_smooth = int(_mg_get(mg, "pre_smooth", 2))
        self.post_smooth = int(_mg_get(mg, "post_smooth", 2))
        bl, bp = C.c_int(-1), C.c_int64(-1)
        rc = L.lib().pdst_patches_build(self.dev.h, int(bool(_mg_get(mg, "surrogate", True))),
                                        float(_mg_get(mg, "rep_fraction", 0.5)), C.byref(bl), C.byref(bp))
        # one level (min_cells >= the mesh): the V-cycle is the coarsest dense
        # solve of the whole slab system, as in the reference (multigrid.py:545-547)
        L.check(rc, "pdst_patches_build", level=bl.value, patch=bp.value)
        self.k1 = self.dev.k1
        discs = geometry.discs if geometry is not None else [None] * self.num_levels
        self.levels = [MgLevel(self, ell, discs[ell] if discs[ell] is not None else
                               _level_disc(ctx.disc, *self.level_shape(ell)[:2])) for ell in range(self.num_levels)]

    # -- level introspection ---------------------------------------------------
    def level_shape(self, level):
        nx, ny, nd = C.c_int32(), C.c_int32(), C.c_int64()
        L.check(L.lib().pdst_level_sizes(self.dev.h, level, C.byref(nx), C.byref(ny), C.byref(nd)))
        return nx.value, ny.value, nd.value

    def patch_matrices(self, level):
        nx, ny, _ = self.level_shape(level)
        D = 21 * self.k1
        out = np.empty((nx * ny, D, D))
        L.check(L.lib().pdst_patch_matrices(self.dev.h, level, L.vptr(out)), "pdst_patch_matrices")
        return out

    def _call(self, fn, level, x, in_len, out_len, name):
        xc = _f64(x).reshape(-1)
        y = self.dev.empty_like(xc, shape=(out_len,))
        w = self.dev.where(xc, y)
        L.check(fn(self.dev.h, level, L.vptr(xc, in_len, "x"), L.vptr(y), w), name)
        return y

    def level_matvec(self, level, x):
        n = self.level_shape(level)[2]
        return self._call(L.lib().pdst_level_apply, level, x, n, n, "pdst_level_apply")

    def restrict(self, fine_level, r):
        return self._call(L.lib().pdst_restrict, fine_level, r, self.level_shape(fine_level)[2],
                          self.level_shape(fine_level - 1)[2], "pdst_restrict")

    def prolong(self, fine_level, e):
        return self._call(L.lib().pdst_prolong, fine_level, e, self.level_shape(fine_level - 1)[2],
                          self.level_shape(fine_level)[2], "pdst_prolong")

    def vanka(self, level, d, r, steps, omega):
        rc_ = _f64(r).reshape(-1)
        out = d.clone() if _is_torch(d) else np.array(d, dtype=np.float64, copy=True).reshape(-1)
        w = self.dev.where(out, rc_)
        n = self.level_shape(level)[2]
        L.check(L.lib().pdst_vanka(self.dev.h, level, L.vptr(out, n, "d"), L.vptr(rc_, n, "r"), int(steps), float(omega), w),
                "pdst_vanka")
        return out

    # -- the preconditioner ------------------------------------------------------
    def apply(self, r, out=None):
        """z = V-cycle(r), projected off the mean-pressure modes when all-Dirichlet."""
        rc_ = _f64(r).reshape(-1)
        z = self.dev.empty_like(rc_) if out is None else out
        w = self.dev.where(rc_, z)
        n = self.dev.ndof
        L.check(L.lib().pdst_vcycle(self.dev.h, L.vptr(rc_, n, "r"), L.vptr(z, n, "out"), self.pre_smooth,
                                    self.post_smooth, self.omega, w), "pdst_vcycle")
        return z


def mg_vcycle(precond: StmgPreconditioner, rhs):
    return precond.apply(rhs)


def _level_disc(fine, nx, ny):
    """Discretization of a coarse level (sizes only) when no geometry is given."""
    if fine.mesh.nx == nx and fine.mesh.ny == ny:
        return fine
    from .problem import Discretization, QuadMesh

    m = fine.mesh
    return Discretization(QuadMesh(nx, ny, m.x0, m.y0, m.x1, m.y1))


class StmgFactory:
    """Builds state-bound preconditioners over a fixed geometry
    (solver/newton.py:129-137): ``StmgFactory(geometry, mg)``, ``.mg``
    (``rebuild_rho`` / ``rebuild_factor`` are read by the Newton driver) and
    ``.build(ctx, U, variant)``.  ``geometry`` may be None (levels from
    ``mg.min_cells``); ``mg`` may be a pdflow MgConfig."""

    def __init__(self, geometry=None, mg=None, *, device=0):
        if mg is None and isinstance(geometry, MgConfig):  # StmgFactory(mg) shorthand
            geometry, mg = None, geometry
        self.geometry = geometry
        self.mg = mg if mg is not None else MgConfig()
        self.device = device

    def build(self, ctx, U, variant) -> StmgPreconditioner:
        geometry = self.geometry
        if geometry is not None and geometry.discs[-1] is not ctx.disc:
            # a geometry built for another Discretization object of the same
            # mesh (our own contexts are rebuilt per slab): same levels
            if _same_mesh(geometry.discs[-1], ctx.disc):
                geometry = MgGeometry(list(geometry.discs[:-1]) + [ctx.disc])
        return StmgPreconditioner(geometry, ctx, U, variant, self.mg, device=self.device)


def _same_mesh(a, b):
    ma, mb = a.mesh, b.mesh
    return (ma.nx, ma.ny, ma.x0, ma.y0, ma.x1, ma.y1) == (mb.nx, mb.ny, mb.x0, mb.y0, mb.x1, mb.y1)
