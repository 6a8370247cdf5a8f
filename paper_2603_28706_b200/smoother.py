"""Space-time Vanka smoother on the GPU.

Drop-in counterparts of (file:line into /root/reference/pkg/src/pdflow):
  build_patches / PatchSet (exact and surrogate)   solver/multigrid.py:198-299, 475-488
  vanka_smooth(level, d, r, steps, omega)          solver/multigrid.py:327-340

The patch matrices, their inverses and every sweep live in libpdst; the only
host work is argument handling.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .operators import SlabJacobian, _f64, _is_torch

__all__ = ["VankaLevel", "vanka_smooth"]


class VankaLevel:
    """Finest-level Vanka data bound to one Newton state: the slab Jacobian
    (level matvec) and the factorized cell patches.

    surrogate=True freezes the spatial blocks at the blended state of
    ``rep_fraction`` (exact temporal factors); surrogate=False uses the exact
    per-node blocks, as ``StmgPreconditioner`` does (multigrid.py:475-488)."""

    def __init__(self, ctx, U, variant, surrogate=True, rep_fraction=0.5, device=0, jac: SlabJacobian | None = None):
        self.ctx = ctx
        self.jac = jac or SlabJacobian(ctx, U, variant, device=device)
        self.dev = self.jac.dev
        self.surrogate = bool(surrogate)
        self.rep_fraction = float(rep_fraction)
        self.index = 0  # finest level (the only one until pdst_hierarchy adds coarse levels)
        bl, bp = C.c_int(-1), C.c_int64(-1)
        rc = L.lib().pdst_patches_build(self.dev.h, int(self.surrogate), self.rep_fraction, C.byref(bl), C.byref(bp))
        L.check(rc, "pdst_patches_build", level=bl.value, patch=bp.value)
        self.k1 = self.dev.k1
        self.D = 21 * self.k1

    @property
    def matvec(self):
        return self.jac.matvec

    @property
    def ncells(self):
        m = self.ctx.disc.mesh
        return m.nx * m.ny

    def patch_matrices(self) -> np.ndarray:
        out = np.empty((self.ncells, self.D, self.D))
        L.check(L.lib().pdst_patch_matrices(self.dev.h, self.index, L.vptr(out)), "pdst_patch_matrices")
        return out

    def patch_info(self):
        """(D, diagonalized complex blocks per patch, bytes streamed per patch per sweep)."""
        D, nb, by = C.c_int32(), C.c_int32(), C.c_int64()
        L.check(L.lib().pdst_patch_info(self.dev.h, self.index, C.byref(D), C.byref(nb), C.byref(by)), "pdst_patch_info")
        return D.value, nb.value, by.value

    def patch_ids(self) -> np.ndarray:
        nc = self.ncells
        cn = np.empty((nc, 9), dtype=np.int64)
        ids = np.empty((nc, self.D), dtype=np.int64)
        L.check(L.lib().pdst_cell_maps(self.dev.h, L.vptr(cn), L.vptr(ids)), "pdst_cell_maps")
        return ids

    def smooth(self, d, r, steps, omega, inplace=False, asynchronous=False):
        """d <- d + omega sum_K R_K' A_K^-1 R_K (r - A d), `steps` times.
        Returns a new array unless inplace (a device tensor, or a C-contiguous
        writable float64 host array -- e.g. pinned -- updated through the C ABI).
        asynchronous=True (inplace, page-locked host d and r): returns at once,
        `self.dev.sync()` before reading d or reusing r."""
        if asynchronous and not inplace:
            raise TypeError("asynchronous smoothing is in place")
        rc_ = _f64(r)
        if _is_torch(d):
            out = d if inplace else d.clone()
        elif inplace:
            if not (isinstance(d, np.ndarray) and d.dtype == np.float64 and d.flags.c_contiguous and d.flags.writeable):
                raise TypeError("inplace smoothing needs a C-contiguous writable float64 array")
            out = d
        else:
            out = np.array(d, dtype=np.float64, copy=True)
        w = self.dev.where(out, rc_, asynchronous=asynchronous)
        n = self.dev.ndof
        L.check(L.lib().pdst_vanka(self.dev.h, self.index, L.vptr(out, n, "d"), L.vptr(rc_, n, "r"), int(steps),
                                   float(omega), w),
                "pdst_vanka")
        return out


    def increment(self, defect, row_lo, row_hi, omega):
        """omega sum_K R_K' A_K^-1 R_K defect over the patches of cell rows [row_lo, row_hi)."""
        dc = _f64(defect)
        inc = self.dev.empty_like(dc)
        w = self.dev.where(dc, inc)
        L.check(L.lib().pdst_vanka_increment(self.dev.h, self.index, L.vptr(dc, self.dev.ndof, "defect"), L.vptr(inc), int(row_lo),
                                             int(row_hi), float(omega), w), "pdst_vanka_increment")
        return inc


def vanka_smooth(level, d, r, steps: int, omega: float):
    """Damped additive Schwarz sweeps d <- d + omega sum_K R_K' A_K^-1 R_K (r - A d)
    (solver/multigrid.py:327-340) on a device level: a ``VankaLevel`` or one of
    ``StmgPreconditioner.levels`` (``stmg.MgLevel``).  Returns a new array, as
    the reference does (multigrid.py:334)."""
    smooth = getattr(level, "smooth", None)
    if smooth is None:
        raise TypeError("vanka_smooth needs a device level (VankaLevel or StmgPreconditioner.levels[i]); "
                        f"got {type(level).__name__} whose patches live on the host")
    return smooth(d, r, steps, omega)
