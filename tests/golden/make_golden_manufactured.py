"""Generate the manufactured-solution fixtures by running the
REFERENCE (pdflow.bench.manufactured.ManufacturedCase.forcing and
pdflow.bench.metrics.error_norms) in this build container.
Run once:  python tests/golden/make_golden_manufactured.py
"""

from __future__ import annotations

import os
import sys

import numpy as np
import scipy

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import build_ctx  # noqa: E402,F401  (puts the reference on sys.path)

from pdflow import constitutive as law  # noqa: E402
from pdflow.bench.manufactured import ManufacturedCase  # noqa: E402
from pdflow.bench.metrics import error_norms  # noqa: E402
from pdflow.femspace import interpolate_velocity, tensor_gauss  # noqa: E402
from pdflow.forms import Discretization  # noqa: E402
from pdflow.mesh import uniform_mesh  # noqa: E402
from pdflow.timebasis import TimePartition, gauss_radau  # noqa: E402

# name: nx, ny, k, (p, delta, nu, nu_inf), t_start, tau, slabs
CASES = {
    "mf_a": (5, 4, 1, (1.4, 1.0e-2, 1.0, 1.0e-3), 0.3, 0.1, 2),
    "mf_b": (6, 6, 2, (1.2, 1.0e-3, 0.5, 0.0), 0.0, 0.05, 2),
    "mf_c": (4, 7, 0, (1.8, 0.0, 1.0, 1.0e-2), 0.7, 0.2, 3),  # delta = 0: Phi zero-limit branch
}


def gen(name):
    nx, ny, k, prm, t0, tau, nsl = CASES[name]
    params = law.ModelParams(*prm)
    case = ManufacturedCase(params)
    disc = Discretization(uniform_mesh(nx, ny))
    basis = gauss_radau(k)
    mesh = disc.mesh
    pts = mesh.cell_origins[:, None, :] + tensor_gauss(4).points[None, :, :] * np.array([mesh.hx, mesh.hy])
    f = None
    if prm[1] > 0.0:  # the strong-form forcing needs delta > 0 where Dv vanishes
        times = t0 + tau * np.asarray(basis.nodes)
        f = np.stack([case.forcing(pts[..., 0], pts[..., 1], float(t)) for t in times])  # (k+1, nc, 16, 2)
    # a trajectory: the interpolated exact velocity at the Radau nodes plus
    # seeded perturbations (so both error norms are nonzero)
    rng = np.random.default_rng(20260420 + nx)
    part = TimePartition(t0 + tau * np.arange(nsl + 1))
    traj = []
    for (a, b) in part.intervals():
        U = np.zeros((k + 1, disc.ndof))
        for mu in range(k + 1):
            t = a + (b - a) * basis.nodes[mu]
            U[mu, : disc.n_velocity] = interpolate_velocity(disc.velocity, case.velocity, float(t))
            U[mu, : disc.n_velocity] += 1e-2 * rng.standard_normal(disc.n_velocity)
            U[mu, disc.n_velocity:] = rng.uniform(-1, 1, disc.ndof - disc.n_velocity)
        traj.append(U)
    e_phi, e_div = error_norms(disc, basis, part, traj, case)
    e_phi3, e_div3 = error_norms(disc, basis, part, traj, case, spatial_order=3, temporal_points=2)
    out = dict(nx=nx, ny=ny, k=k, params=np.array(prm), t0=t0, tau=tau, times=part.t, traj=np.stack(traj),
               e_phi=e_phi, e_div=e_div, e_phi_q3t2=e_phi3, e_div_q3t2=e_div3, nodes=basis.nodes,
               numpy=np.__version__, scipy=scipy.__version__)
    if f is not None:
        out["f_qp"] = f
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, "e_phi", e_phi, "e_div", e_div, "f" if f is not None else "")


if __name__ == "__main__":
    for n in sys.argv[1:] or CASES:
        gen(n)
