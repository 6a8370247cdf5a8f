"""Freeze the REFERENCE's own outputs at the bench workload (BASELINE
configs[1], cfg2: 256x256, DG(1), modified Newton, surrogate patches at the
last Radau point, omega = 0.7) so the GPU tests can compare the exact code
path ``bench.py`` times -- the persistent TMA-ring patch GEMV with ~55 patch
groups per CTA -- against pdflow itself.

Run once in the build container (about 7 minutes, pdflow is single-threaded):
    python tests/golden/make_golden_cfg2.py

The full vectors (1.4 M doubles each) are too large to commit, so the fixture
stores, per output: its L2 / L1 / Linf norms, a 64-row seeded Gaussian
sketch S y (S regenerated from SKETCH_SEED by the test), and the values at
24,576 sampled indices (uniform random plus every boundary-strip dof of both
Radau nodes' first node rows, where the apply's epilogue and side products
write).  The fine level is built from the reference's own pieces
(SlabJacobian, SpatialLinearization.assemble, build_patches, vanka_smooth,
multigrid.py:261-340 / 475-488) exactly as StmgPreconditioner.__init__ does
for its finest level; the full preconditioner is not constructed because its
coarsest-level dense LU (multigrid.py:494-520) would be a 1.4 M^2 matrix at
min_cells = 256.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np
import scipy

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

SKETCH_SEED = 777
N_SKETCH = 64
N_SAMPLE = 16384


def sketch(y, seed=SKETCH_SEED, rows=N_SKETCH, chunk=1 << 18):
    """S y with S ~ N(0,1)^{rows x n} drawn chunk by chunk (bounded memory)."""
    rng = np.random.default_rng(seed)
    out = np.zeros(rows)
    for a in range(0, y.size, chunk):
        b = min(y.size, a + chunk)
        out += rng.standard_normal((rows, b - a)) @ y[a:b]
    return out


def sample_indices(nx, ny, k1):
    nn = (2 * nx + 1) * (2 * ny + 1)
    nd = 2 * nn + 3 * nx * ny
    rng = np.random.default_rng(4242)
    idx = set(rng.choice(k1 * nd, size=N_SAMPLE, replace=False).tolist())
    row = 2 * nx + 1
    for mu in range(k1):
        for j in (0, 1, 2, 2 * ny - 2, 2 * ny - 1, 2 * ny):  # bottom / top node rows
            for i in range(row):
                for c in range(2):
                    idx.add(mu * nd + 2 * (j * row + i) + c)
        for j in range(2 * ny + 1):  # left / right node columns
            for i in (0, 1, 2, 2 * nx - 2, 2 * nx - 1, 2 * nx):
                for c in range(2):
                    idx.add(mu * nd + 2 * (j * row + i) + c)
        for t in (16, 17, 127, 128, 255):  # tile-line node rows / columns (16x16-cell tiles)
            for i in range(row):
                idx.add(mu * nd + 2 * ((2 * t) * row + i))
            for j in range(2 * ny + 1):
                idx.add(mu * nd + 2 * (j * row + 2 * t) + 1)
    return np.array(sorted(idx), dtype=np.int64)


def summary(prefix, y, idx):
    return {f"{prefix}_l2": np.array(np.linalg.norm(y)), f"{prefix}_l1": np.array(np.abs(y).sum()),
            f"{prefix}_linf": np.array(np.abs(y).max()), f"{prefix}_sketch": sketch(y),
            f"{prefix}_sample": y[idx]}


def main():
    from pdflow import constitutive as law
    from pdflow.forms import Discretization, DiscretizationConfig, ProblemData, SpatialLinearization
    from pdflow.mesh import DIRICHLET, boundary_tag_assign, uniform_mesh
    from pdflow.slab import SlabContext, SlabJacobian
    from pdflow.solver.multigrid import MgLevel, build_patches, vanka_smooth
    from pdflow.timebasis import gauss_radau, temporal_matrices

    from paper_2603_28706_b200.synth import CONFIGS, make_slab_inputs

    cfg = CONFIGS["cfg2"]
    mesh = boundary_tag_assign(uniform_mesh(cfg.nx, cfg.ny, (0.0, 0.0, 1.0, 1.0)), lambda f: DIRICHLET)
    disc = Discretization(mesh)
    config = DiscretizationConfig(gamma1=cfg.gamma1, gamma2=cfg.gamma2, gamma_cip=cfg.gamma_cip, g_hat=None)
    params = law.ModelParams(cfg.p, cfg.delta, cfg.nu, cfg.nu_inf)
    basis = gauss_radau(cfg.k)
    tmat = temporal_matrices(basis)
    syn = make_slab_inputs(cfg, nodes=basis.nodes)
    ctx = SlabContext(disc=disc, params=params, config=config,
                      data=ProblemData(f=lambda x, y, t: np.zeros(np.shape(x) + (2,)), g_d=None, v0=None),
                      basis=basis, tmat=tmat, t_start=0.0, tau=cfg.tau, v_minus=syn.v_minus)
    variant = law.modified_newton(cfg.nu)
    k1 = cfg.k + 1
    idx = sample_indices(cfg.nx, cfg.ny, k1)
    out = dict(numpy_version=np.__version__, scipy_version=scipy.__version__, idx=idx,
               sketch_seed=np.array(SKETCH_SEED), n_sketch=np.array(N_SKETCH))

    t0 = time.time()
    jac = SlabJacobian(ctx, syn.U, variant)
    out.update(summary("y", jac.matvec(syn.x), idx))
    print(f"apply done {time.time() - t0:.1f} s", flush=True)

    # the finest level exactly as StmgPreconditioner.__init__ builds it (multigrid.py:417-431, 475-486)
    lvl = MgLevel(index=0, disc=disc, j_nodes=None, mass_v=disc.mass_v, K_t=tmat.K_t,
                  tau_w=cfg.tau * basis.weights, matvec=jac.matvec)
    rep_state = ctx.state_at(syn.U, cfg.rep_fraction)
    rep_block = SpatialLinearization(disc, rep_state, variant, ctx.params, ctx.config).assemble()
    lvl.patches = build_patches(lvl, [rep_block] * k1)
    print(f"patches done {time.time() - t0:.1f} s", flush=True)
    # a few whole patch inverses (the diagonalized device inverse must equal them)
    pick = np.array([0, 1, 255, 256, 32767, 32896, 65279, 65535])
    out["patch_pick"] = pick
    out["patch_inv_pick"] = lvl.patches.inverses[pick]
    out["patch_mat_pick"] = lvl.patches.matrices[pick]

    om = cfg.omega
    out.update(summary("v1", vanka_smooth(lvl, syn.d0, syn.x, 1, om), idx))
    out.update(summary("v2", vanka_smooth(lvl, syn.d0, syn.x, 2, om), idx))
    out.update(summary("v0", vanka_smooth(lvl, np.zeros_like(syn.x), syn.x, 1, om), idx))
    print(f"sweeps done {time.time() - t0:.1f} s", flush=True)
    np.savez_compressed(os.path.join(HERE, "cfg2_frozen.npz"), **out)


if __name__ == "__main__":
    main()
