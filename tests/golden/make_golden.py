"""Generate the golden fixtures by running the REFERENCE (pdflow) in this
build container.  Run once:  python tests/golden/make_golden.py

The reference is imported read-only from /root/reference/pkg/src; it does not
exist on the GPU box, so its outputs are frozen here as compressed .npz files
next to this script.  numpy/scipy versions are recorded in every file.
"""

from __future__ import annotations

import os
import sys

import numpy as np
import scipy

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))
sys.path.insert(0, "/root/reference/pkg/src")

from pdflow import constitutive as law  # noqa: E402
from pdflow.femspace import interpolate_velocity  # noqa: E402
from pdflow.forms import Discretization, DiscretizationConfig, ProblemData  # noqa: E402
from pdflow.mesh import DIRICHLET, NEUMANN, boundary_tag_assign, uniform_mesh  # noqa: E402
from pdflow.slab import SlabContext, SlabJacobian, slab_residual  # noqa: E402
from pdflow.solver.multigrid import (  # noqa: E402
    MgConfig,
    MgGeometry,
    StmgPreconditioner,
    transfer_build,
    vanka_smooth,
)
from pdflow.solver.newton import MassNorm  # noqa: E402
from pdflow.timebasis import gauss_radau, temporal_matrices  # noqa: E402

from cases import CASES, FORCINGS, TRANSFER_PAIRS, ghat_field  # noqa: E402
from paper_2603_28706_b200.synth import make_slab_inputs, q2_node_coords  # noqa: E402


def _zero_f(x, y, t):
    return np.zeros(np.shape(x) + (2,))


def build_ctx(case):
    cfg = case.cfg
    x0, y0, x1, y1 = cfg.extents
    mesh = uniform_mesh(cfg.nx, cfg.ny, (x0, y0, x1, y1))

    def rule(face):
        return NEUMANN if face.side in case.neumann_sides else DIRICHLET

    mesh = boundary_tag_assign(mesh, rule)
    disc = Discretization(mesh)
    g_hat = None
    if case.ghat:
        X, Y = q2_node_coords(cfg.nx, cfg.ny, cfg.extents)
        g_hat = ghat_field(X, Y).reshape(-1).copy()
    config = DiscretizationConfig(gamma1=cfg.gamma1, gamma2=cfg.gamma2, gamma_cip=cfg.gamma_cip, g_hat=g_hat)
    params = law.ModelParams(cfg.p, cfg.delta, cfg.nu, cfg.nu_inf)
    f = FORCINGS[case.forcing] or _zero_f
    data = ProblemData(f=f, g_d=None, v0=None)
    basis = gauss_radau(cfg.k)
    tmat = temporal_matrices(basis)
    syn = make_slab_inputs(cfg, nodes=basis.nodes)
    ctx = SlabContext(disc=disc, params=params, config=config, data=data, basis=basis, tmat=tmat,
                      t_start=case.t_start, tau=cfg.tau, v_minus=syn.v_minus)
    if case.variant == "pic":
        variant = law.picard()
    elif case.variant == "exn":
        variant = law.exact_newton()
    else:
        variant = law.modified_newton(cfg.nu if case.sigma_max is None else case.sigma_max)
    return ctx, variant, syn, g_hat


def gen_case(case):
    ctx, variant, syn, g_hat = build_ctx(case)
    cfg = case.cfg
    out = dict(
        numpy_version=np.__version__, scipy_version=scipy.__version__,
        nodes=ctx.basis.nodes, weights=ctx.basis.weights, K_t=ctx.tmat.K_t, m_t=ctx.tmat.m_t,
        M_t=ctx.tmat.M_t, U=syn.U, x=syn.x, d0=syn.d0, v_minus=syn.v_minus,
        tags=np.array([t == DIRICHLET for t in ctx.disc.mesh.boundary_tags]),
    )
    if g_hat is not None:
        out["g_hat"] = g_hat
    jac = SlabJacobian(ctx, syn.U, variant)
    out["y"] = jac.matvec(syn.x)
    out["R"] = slab_residual(ctx, syn.U)
    mn = MassNorm(ctx)
    out["mass_x"] = mn.apply(syn.x)
    out["mnorm_x"] = np.array(mn.norm(syn.x))
    out["cell_patch_dofs"] = ctx.disc.cell_patch_dofs
    out["cell_nodes"] = ctx.disc.cell_nodes
    out["mass_v_diag"] = ctx.disc.mass_v.diagonal()
    if case.patches:
        mg = MgConfig(rep_fraction=cfg.rep_fraction, surrogate=case.surrogate, min_cells=case.min_cells,
                      omega=cfg.omega, coarse_mode=case.coarse_mode)
        geom = MgGeometry.from_fine(ctx.disc, min_cells=mg.min_cells)
        pre = StmgPreconditioner(geom, ctx, syn.U, variant, mg)
        fine = pre.levels[-1]
        out["levels_nx"] = np.array([lv.disc.mesh.nx for lv in pre.levels])
        out["levels_ny"] = np.array([lv.disc.mesh.ny for lv in pre.levels])
        out["patch_ids"] = fine.patches.ids
        out["patch_mats"] = fine.patches.matrices
        out["vanka_d"] = vanka_smooth(fine, syn.d0, syn.x, 1, mg.omega)
        out["vanka_d2"] = vanka_smooth(fine, syn.d0, syn.x, 2, mg.omega)
        out["vanka_zero"] = vanka_smooth(fine, np.zeros_like(syn.x), syn.x, 1, mg.omega)
        out["vcycle"] = pre.apply(syn.x.copy())
        for ell in range(len(pre.levels) - 1):
            lv = pre.levels[ell]
            rng = np.random.default_rng(1000 + ell)
            xc = rng.uniform(-1.0, 1.0, size=lv.slab_dim)
            out[f"L{ell}_x"] = xc
            out[f"L{ell}_Ax"] = lv.matvec(xc)
            out[f"L{ell}_patch_mats"] = lv.patches.matrices
            out[f"L{ell}_vanka"] = vanka_smooth(lv, np.zeros_like(xc), xc, 1, mg.omega)
    np.savez_compressed(os.path.join(HERE, f"{case.name}.npz"), **out)
    print(case.name, "N_dof", syn.x.size, "|y|", np.linalg.norm(out["y"]))


def gen_transfers():
    out = dict(numpy_version=np.__version__, scipy_version=scipy.__version__)
    for (cx, cy) in TRANSFER_PAIRS:
        mc = boundary_tag_assign(uniform_mesh(cx, cy), lambda f: DIRICHLET)
        mf = boundary_tag_assign(uniform_mesh(2 * cx, 2 * cy), lambda f: DIRICHLET)
        tr = transfer_build(Discretization(mc), Discretization(mf))
        tag = f"{cx}x{cy}"
        P = tr.P.tocoo()
        out[f"{tag}_P_row"] = P.row
        out[f"{tag}_P_col"] = P.col
        out[f"{tag}_P_val"] = P.data
        out[f"{tag}_P_shape"] = np.array(P.shape)
        out[f"{tag}_inject_v"] = tr.inject_v
        rng = np.random.default_rng(cx * 100 + cy)
        xf = rng.uniform(-1, 1, size=P.shape[0])
        xc = rng.uniform(-1, 1, size=P.shape[1])
        out[f"{tag}_xf"] = xf
        out[f"{tag}_xc"] = xc
        out[f"{tag}_restrict"] = tr.P.T @ xf
        out[f"{tag}_prolong"] = tr.P @ xc
    np.savez_compressed(os.path.join(HERE, "transfers.npz"), **out)


def main(names=None):
    for case in CASES:
        if names and case.name not in names:
            continue
        gen_case(case)
    if not names or "transfers" in names:
        gen_transfers()


if __name__ == "__main__":
    main(sys.argv[1:])
