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

__all__ = ["MgConfig", "StmgPreconditioner", "StmgFactory", "mg_vcycle"]

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
        if self.coarse_mode == "rediscretize":
            raise NotImplementedError("coarse_mode='rediscretize' is not ported (galerkin is the default)")


class StmgPreconditioner:
    """One state-bound V-cycle: Galerkin hierarchy, patches and coarsest solve."""

    def __init__(self, ctx, U, variant, mg: MgConfig | None = None, device=0, jac: SlabJacobian | None = None):
        self.mg = mg or MgConfig()
        self.ctx = ctx
        self.jac = jac or SlabJacobian(ctx, U, variant, device=device)
        self.dev = self.jac.dev
        nl = C.c_int(0)
        L.check(L.lib().pdst_hierarchy(self.dev.h, int(self.mg.min_cells), C.byref(nl)), "pdst_hierarchy")
        mg = self.mg
        cw = mg.coarse_omega if mg.coarse_omega is not None else mg.omega
        sw = mg.coarse_sweeps if mg.coarse_sweeps is not None else (30 if mg.coarse_solver == "vanka" else 2)
        L.check(L.lib().pdst_set_coarse_solver(self.dev.h, _COARSE[mg.coarse_solver], int(sw), float(cw),
                                               int(mg.coarse_iters), float(mg.coarse_rtol)), "pdst_set_coarse_solver")
        self.num_levels = nl.value
        bl, bp = C.c_int(-1), C.c_int64(-1)
        rc = L.lib().pdst_patches_build(self.dev.h, int(self.mg.surrogate), float(self.mg.rep_fraction),
                                        C.byref(bl), C.byref(bp))
        # one level (min_cells >= the mesh): the V-cycle is the coarsest dense
        # solve of the whole slab system, as in the reference (multigrid.py:545-547)
        L.check(rc, "pdst_patches_build", level=bl.value, patch=bp.value)
        self.k1 = self.dev.k1

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
        L.check(L.lib().pdst_vcycle(self.dev.h, L.vptr(rc_, n, "r"), L.vptr(z, n, "out"), int(self.mg.pre_smooth),
                                    int(self.mg.post_smooth), float(self.mg.omega), w), "pdst_vcycle")
        return z


def mg_vcycle(precond: StmgPreconditioner, rhs):
    return precond.apply(rhs)


class StmgFactory:
    """Builds state-bound preconditioners (solver/newton.py:129-137)."""

    def __init__(self, mg: MgConfig | None = None, geometry=None, device=0):
        self.mg = mg or MgConfig()
        self.geometry = geometry
        self.device = device

    def build(self, ctx, U, variant) -> StmgPreconditioner:
        return StmgPreconditioner(ctx, U, variant, self.mg, device=self.device)
