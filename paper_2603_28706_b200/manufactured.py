"""Manufactured-solution benchmark problem (drop-in for
``pdflow.bench.manufactured.ManufacturedCase``, bench/manufactured.py:30-167).

The prescribed velocity s(t) (a(x) b(y), -b(x) a(y)) with a = sin^2(pi x),
b = sin(2 pi x) / 2, s = sin t is divergence free and vanishes on the
boundary and at t = 0; the pressure is s b(x) b(y).  The analytic fields are
evaluated here on the host (numpy, as the reference does); the body force
that the slab residual consumes at every volume point is evaluated on the
device (``pdst_manufactured_forcing``) whenever the residual is computed
through ``operators.slab_residual`` with this case's ``forcing`` as the
problem's ``f`` and matching model parameters.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .problem import ModelParams, ProblemData

__all__ = ["ManufacturedCase"]

_PI = np.pi


def _fields(x):
    """a, a', a'', b, b', b'' of one coordinate."""
    s1, s2, c2 = np.sin(_PI * x), np.sin(2.0 * _PI * x), np.cos(2.0 * _PI * x)
    return s1 * s1, _PI * s2, 2.0 * _PI**2 * c2, 0.5 * s2, _PI * c2, -2.0 * _PI**2 * s2


@dataclass(frozen=True)
class ManufacturedCase:
    params: ModelParams

    def velocity(self, x, y, t):
        ax, _, _, bx, _, _ = _fields(x)
        ay, _, _, by, _, _ = _fields(y)
        s = np.sin(t)
        return np.stack(np.broadcast_arrays(s * ax * by, -s * bx * ay), axis=-1)

    def velocity_dt(self, x, y, t):
        ax, _, _, bx, _, _ = _fields(x)
        ay, _, _, by, _, _ = _fields(y)
        c = np.cos(t)
        return np.stack(np.broadcast_arrays(c * ax * by, -c * bx * ay), axis=-1)

    def velocity_grad(self, x, y, t):
        """grad[..., d, k] = d v_d / d x_k."""
        ax, dax, _, bx, dbx, _ = _fields(x)
        ay, day, _, by, dby, _ = _fields(y)
        s = np.sin(t)
        g00, g01, g10, g11 = np.broadcast_arrays(s * dax * by, s * ax * dby, -s * dbx * ay, -s * bx * day)
        return np.stack([np.stack([g00, g01], -1), np.stack([g10, g11], -1)], -2)

    def sym_grad(self, x, y, t):
        """(..., 3) components (a11, a22, a12)."""
        g = self.velocity_grad(x, y, t)
        return np.stack([g[..., 0, 0], g[..., 1, 1], 0.5 * (g[..., 0, 1] + g[..., 1, 0])], axis=-1)

    def pressure(self, x, y, t):
        return np.sin(t) * _fields(x)[3] * _fields(y)[3]

    def pressure_grad(self, x, y, t):
        _, _, _, bx, dbx, _ = _fields(x)
        _, _, _, by, dby, _ = _fields(y)
        s = np.sin(t)
        return np.stack(np.broadcast_arrays(s * dbx * by, s * bx * dby), axis=-1)

    def forcing(self, x, y, t):
        """f = dv/dt + (v . grad) v - div S(Dv) + grad(pi), hand-differentiated."""
        prm = self.params
        ax, dax, ddax, bx, dbx, ddbx = _fields(x)
        ay, day, dday, by, dby, ddby = _fields(y)
        s = np.sin(t)
        v0, v1 = s * ax * by, -s * bx * ay
        g00, g01, g10, g11 = s * dax * by, s * ax * dby, -s * dbx * ay, -s * bx * day
        h000, h001, h011 = s * ddax * by, s * dax * dby, s * ax * ddby
        h100, h101, h111 = -s * ddbx * ay, -s * dbx * day, -s * bx * dday
        a11, a22, a12 = g00, g11, 0.5 * (g01 + g10)
        da11 = (h000, h001)
        da22 = (h101, h111)
        da12 = (0.5 * (h001 + h100), 0.5 * (h011 + h101))
        a_sq = a11**2 + a22**2 + 2.0 * a12**2
        dasq = [2.0 * (a11 * da11[k] + a22 * da22[k] + 2.0 * a12 * da12[k]) for k in range(2)]
        dsq = prm.delta**2 + a_sq
        eta = prm.nu_inf + prm.nu * dsq ** ((prm.p - 2.0) / 2.0)
        dfac = prm.nu * ((prm.p - 2.0) / 2.0) * dsq ** ((prm.p - 4.0) / 2.0)
        ds0 = dfac * dasq[0] * a11 + dfac * dasq[1] * a12 + eta * (da11[0] + da12[1])
        ds1 = dfac * dasq[0] * a12 + dfac * dasq[1] * a22 + eta * (da12[0] + da22[1])
        c = np.cos(t)
        f0 = c * ax * by + (v0 * g00 + v1 * g01) - ds0 + s * dbx * by
        f1 = -c * bx * ay + (v0 * g10 + v1 * g11) - ds1 + s * bx * dby
        return np.stack(np.broadcast_arrays(f0, f1), axis=-1)

    def dirichlet(self, x, y, t):
        return np.zeros(np.broadcast(x, y).shape + (2,))

    def initial_velocity(self, x, y):
        return self.velocity(x, y, 0.0)

    def problem_data(self) -> ProblemData:
        return ProblemData(f=self.forcing, g_d=self.dirichlet, v0=self.initial_velocity)


def device_forcing_case(ctx):
    """The ManufacturedCase whose forcing is ctx.data.f, if the device kernel
    can evaluate it (same model parameters), else None."""
    f = getattr(ctx.data, "f", None)
    case = getattr(f, "__self__", None)
    if not isinstance(case, ManufacturedCase) or getattr(f, "__func__", None) is not ManufacturedCase.forcing:
        return None
    a, b = case.params, ctx.params
    if (a.p, a.delta, a.nu, a.nu_inf) != (b.p, b.delta, b.nu, b.nu_inf):
        return None
    return case
