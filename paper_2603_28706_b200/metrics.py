"""Space-time error norms of a slab trajectory on the GPU (drop-in for
``pdflow.bench.metrics.error_norms``, bench/metrics.py:35-85; eoc as
bench/metrics.py:88-101).

e_phi = || Phi_delta(Dv) - Phi_delta(Dv_h) ||_L2(L2) (the natural distance,
Phi_delta(A) = (delta^2 + |A|^2)^((p-2)/4) A) and e_div = || div v_h ||_L2(L2),
with one Gauss order beyond the assembly rule in space (5^2 points per cell)
and k+2 Gauss points per slab in time, against the manufactured solution.
Each slab's squared contributions come from one kernel pass
(``pdst_error_norms``); the host sums the slabs in order and takes the roots.
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _lib as L

__all__ = ["error_norms", "eoc"]


def error_norms(disc, basis, partition, traj, case, spatial_order: int | None = None,
                temporal_points: int | None = None, device=0) -> tuple[float, float]:
    """(e_phi, e_div) of the slab trajectory traj[n] ((k+1, ndof) per interval
    of `partition`) against the ManufacturedCase `case` (reference or ours)."""
    if type(case).__name__ != "ManufacturedCase":
        raise NotImplementedError("device error norms are implemented for the manufactured solution only")
    from .operators import SlabDevice
    from .problem import DiscretizationConfig, ProblemData, SlabContext, temporal_matrices

    q = spatial_order or 5  # disc.quad.q + 1 with the 4-point assembly rule
    ntp = temporal_points or (basis.k + 2)
    ctx = SlabContext(disc, case.params, DiscretizationConfig(), ProblemData(), basis, temporal_matrices(basis), 0.0,
                      1.0, np.zeros(disc.n_velocity))
    dev = SlabDevice(ctx, device)
    try:
        e_phi_sq = e_div_sq = 0.0
        sq = np.zeros(2)
        for (t0, t1), U in zip(partition.intervals(), traj):
            Uc = np.ascontiguousarray(U, dtype=np.float64)
            if Uc.size != dev.k1 * disc.ndof:
                raise ValueError("slab state has the wrong size")
            L.check(L.lib().pdst_error_norms(dev.h, L.vptr(Uc), float(t0), float(t1), int(q), int(ntp),
                                             sq.ctypes.data_as(C.c_void_p), L.HOST), "pdst_error_norms")
            e_phi_sq += float(sq[0])
            e_div_sq += float(sq[1])
        return math.sqrt(e_phi_sq), math.sqrt(e_div_sq)
    finally:
        dev.close()


def eoc(errors) -> list:
    """Experimental orders log2(e_i / e_{i+1}) under mesh halving; None where undefined."""
    errors = list(errors)
    return [None if a <= 0.0 or b <= 0.0 else math.log2(a / b) for a, b in zip(errors[:-1], errors[1:])]
