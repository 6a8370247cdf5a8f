"""GPU parity of the strip-partitioned V-cycle (SURVEY.md §8e with rows a15-a17):
P virtual ranks on one GPU, each with its own libpdst handle holding the
hierarchy of its local mesh (strip + 2^L ghost rows, `pdst_hierarchy_depth`),
exchanging through LocalTransport.  The owned entries of the distributed
V-cycle must match the single-domain `StmgPreconditioner.apply` with the same
coarsest-level FGMRES.  Tolerance: relative 1e-9 — the local kernels sum the
same terms, but the coarsest FGMRES's allreduced inner products round
differently from the single-domain fixed reduction tree, and FGMRES amplifies
that (the V-cycle parity against the reference itself is pinned at 1e-9 too)."""

import numpy as np
import pytest

from helpers import assert_close, product_ctx, product_variant

pytestmark = pytest.mark.gpu
TOL = 1e-9


def _case(nx, ny, k, neumann):
    from cases import Case, _cfg
    from paper_2603_28706_b200.radau import gauss_radau, temporal_matrices
    from paper_2603_28706_b200.synth import make_slab_inputs

    case = Case(f"d{nx}x{ny}", _cfg(f"d{nx}x{ny}", nx, ny, k, seed=nx * 100 + ny + 7, p=1.3, delta=1e-3, nu_inf=0.0,
                                     modes=8, extents=(0.0, 0.0, 1.5, 1.0)),
                variant="modn", neumann_sides=neumann, forcing="a", t_start=0.1)
    b = gauss_radau(k)
    tm = temporal_matrices(b)
    syn = make_slab_inputs(case.cfg, nodes=b.nodes)
    fx = dict(nodes=b.nodes, weights=b.weights, K_t=tm.K_t, m_t=tm.m_t, M_t=tm.M_t, v_minus=syn.v_minus)
    return case, fx, syn


def _local_with_garbage(rk, xg, seed):
    """A rank's local vector of a global one, ghost entries garbage."""
    import torch

    rng = np.random.default_rng(seed)
    nd = rk.lay.nd
    xl = np.concatenate([rk.lay.to_local(xg[mu * nd:(mu + 1) * nd]) for mu in range(rk.k1)])
    own = rk.masks[0].cpu().numpy() > 0
    xl[~own] = 1e3 * rng.standard_normal((~own).sum())
    return torch.as_tensor(xl, device=rk.device)


def _gather(ranks, zs, n):
    g = np.full(n, np.nan)
    for rk, z in zip(ranks, zs):
        lay, nd, ndl = rk.lay, rk.lay.nd, rk.lay.nd_loc
        zl = z.cpu().numpy()
        for mu in range(rk.k1):
            lay.owned_into_global(zl[mu * ndl:(mu + 1) * ndl], g[mu * nd:(mu + 1) * nd])
    assert not np.isnan(g).any()
    return g


@pytest.mark.parametrize("nx,ny,k,P,min_cells,surrogate,neumann", [
    (16, 32, 1, 2, 4, True, ("top",)),
    (32, 32, 1, 4, 8, True, ()),
    (24, 32, 2, 2, 6, False, ()),
    (16, 48, 0, 3, 4, True, ("right",)),
])
def test_distributed_vcycle_matches_single_domain(nx, ny, k, P, min_cells, surrogate, neumann):
    from paper_2603_28706_b200.dist_mg import DistributedStmg, distributed_vcycle, global_levels
    from paper_2603_28706_b200.partition import LocalTransport, StripPartition
    from paper_2603_28706_b200.stmg import MgConfig, StmgPreconditioner

    case, fx, syn = _case(nx, ny, k, neumann)
    ctx = product_ctx(case, fx)
    var = product_variant(case)
    mg = MgConfig(min_cells=min_cells, coarse_solver="fgmres", coarse_iters=12, coarse_rtol=1e-10,
                  surrogate=surrogate, rep_fraction=1.0)
    z_ref = StmgPreconditioner(None, ctx, syn.U, var, mg).apply(syn.x)
    nl = global_levels(nx, ny, min_cells)
    assert nl >= 3
    part = StripPartition(nx, ny, P, levels=nl)
    ranks = [DistributedStmg(ctx, syn.U, var, part, r, mg) for r in range(P)]
    assert any(rk.lay.c_lo > 0 for rk in ranks)  # some local mesh is cut
    tr = LocalTransport([rk.lay for rk in ranks])
    xs = [_local_with_garbage(rk, syn.x, 10 + r) for r, rk in enumerate(ranks)]
    zs = distributed_vcycle(ranks, xs, tr)
    assert_close(_gather(ranks, zs, z_ref.size), z_ref, TOL, "distributed V-cycle")


def test_distributed_fgmres_with_vcycle():
    """FGMRES on the strip partition preconditioned by the distributed V-cycle
    takes the iterations of the single-domain FGMRES with the same V-cycle."""
    import torch

    from paper_2603_28706_b200.dist_mg import DistributedStmg, distributed_fgmres_mg, global_levels
    from paper_2603_28706_b200.krylov import KrylovConfig, fgmres
    from paper_2603_28706_b200.operators import MassNorm, SlabJacobian
    from paper_2603_28706_b200.partition import LocalTransport, StripPartition
    from paper_2603_28706_b200.stmg import MgConfig, StmgPreconditioner

    nx, ny, k, P = 16, 32, 1, 2
    case, fx, syn = _case(nx, ny, k, ())
    ctx = product_ctx(case, fx)
    var = product_variant(case)
    mg = MgConfig(min_cells=4, coarse_solver="fgmres", coarse_iters=12, coarse_rtol=1e-10, rep_fraction=1.0)
    jac = SlabJacobian(ctx, syn.U, var)
    pre = StmgPreconditioner(None, ctx, syn.U, var, mg, jac=jac)
    b = torch.as_tensor(syn.x, device="cuda")
    cfg = KrylovConfig(restart=20, max_iters=20)
    ref = fgmres(jac.matvec, b, 1e-8, cfg, precond=lambda v, out=None: pre.apply(v, out=out),
                 mass=MassNorm(ctx, dev=jac.dev))
    part = StripPartition(nx, ny, P, levels=global_levels(nx, ny, 4))
    ranks = [DistributedStmg(ctx, syn.U, var, part, r, mg) for r in range(P)]
    tr = LocalTransport([rk.lay for rk in ranks])
    xs = [_local_with_garbage(rk, syn.x, 3) for rk in ranks]
    res = distributed_fgmres_mg(ranks, tr, xs, 1e-8, cfg)
    assert res.iterations == ref.iterations
    x = _gather(ranks, res.x, syn.x.size)
    assert_close(x, ref.x.cpu().numpy(), 1e-8, "distributed FGMRES + V-cycle")


def test_two_process_vcycle_and_fgmres(tmp_path):
    """The same cycle and FGMRES as two processes (TorchDistTransport, DistComm
    over gloo staged through the host) against the single domain."""
    import os
    import socket
    import subprocess
    import sys

    import torch

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    from dist_mg_worker import problem

    from paper_2603_28706_b200.krylov import KrylovConfig, fgmres
    from paper_2603_28706_b200.operators import MassNorm, SlabJacobian
    from paper_2603_28706_b200.stmg import StmgPreconditioner

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = str(s.getsockname()[1])
    s.close()
    outs = [str(tmp_path / f"r{r}.npz") for r in range(2)]
    procs = [subprocess.Popen([sys.executable, os.path.join(here, "dist_mg_worker.py"), str(r), "2", port, outs[r]])
             for r in range(2)]
    assert [p.wait(timeout=600) for p in procs] == [0, 0]
    parts = [np.load(o) for o in outs]
    cfg, ctx, syn, var, mg = problem()
    jac = SlabJacobian(ctx, syn.U, var)
    pre = StmgPreconditioner(None, ctx, syn.U, var, mg, jac=jac)
    z_ref = pre.apply(syn.x)
    assert_close(parts[0]["z"] + parts[1]["z"], z_ref, TOL, "two-process V-cycle")
    ref = fgmres(jac.matvec, torch.as_tensor(syn.x, device="cuda"), 1e-8, KrylovConfig(restart=20, max_iters=20),
                 precond=lambda v, out=None: pre.apply(v, out=out), mass=MassNorm(ctx, dev=jac.dev))
    assert int(parts[0]["iters"]) == int(parts[1]["iters"]) == ref.iterations
    assert_close(parts[0]["x"] + parts[1]["x"], ref.x.cpu().numpy(), 1e-8, "two-process FGMRES + V-cycle")


@pytest.mark.parametrize("P,max_nl", [(2, 3), (4, 2)])
def test_distributed_newton_matches_single_domain(P, max_nl):
    """A slab's modified-Newton solve on P strips (distributed residual, M-norms,
    deep state halos, FGMRES + distributed V-cycle, Armijo line search) takes the
    single-domain solve's steps: same Krylov iteration counts, step lengths,
    failure kind, residual history to 1e-7."""
    import sys

    import os

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from dist_mg_worker import problem

    from paper_2603_28706_b200.dist_mg import distributed_nonlinear_solve, global_levels
    from paper_2603_28706_b200.errors import SlabSolveError
    from paper_2603_28706_b200.krylov import KrylovConfig
    from paper_2603_28706_b200.newton import NewtonConfig, StmgFactory, nonlinear_solve_slab
    from paper_2603_28706_b200.partition import LocalTransport, StripPartition

    cfg, ctx, syn, var, mg = problem()
    if P == 4:  # strips of 8 rows: the 2^L = 8 ghost rows still come from direct neighbours
        import dataclasses

        mg = dataclasses.replace(mg, min_cells=8)
    newton = NewtonConfig(variant=var, max_nonlinear=max_nl)
    krylov = KrylovConfig(restart=20, max_iters=40)

    def run(fn):
        try:
            out, st = fn()
            return out, st, None
        except SlabSolveError as e:
            return None, e.diagnostics, e.kind

    U_ref, st_ref, kind_ref = run(lambda: nonlinear_solve_slab(ctx, syn.U, newton, krylov, StmgFactory(mg)))
    part = StripPartition(cfg.nx, cfg.ny, P, levels=global_levels(cfg.nx, cfg.ny, mg.min_cells))
    tr = LocalTransport([part.layout(r) for r in range(P)])
    Us, st, kind = run(lambda: distributed_nonlinear_solve(ctx, syn.U, newton, krylov, mg, part, list(range(P)), tr))
    assert kind == kind_ref
    assert len(st.steps) == len(st_ref.steps) >= 1
    assert abs(st.initial_res - st_ref.initial_res) <= 1e-10 * st_ref.initial_res
    for a, b in zip(st.steps, st_ref.steps):
        assert a.n_l == b.n_l and a.lam == b.lam and a.rebuilt == b.rebuilt
        assert abs(a.res_after - b.res_after) <= 1e-7 * b.res_before
    if U_ref is not None:
        lays = [part.layout(r) for r in range(P)]
        g = np.full(U_ref.shape, np.nan)
        for lay, u in zip(lays, Us):
            for mu in range(U_ref.shape[0]):
                lay.owned_into_global(u[mu].cpu().numpy(), g[mu])
        assert_close(g.reshape(-1), np.asarray(U_ref).reshape(-1), 1e-9, "distributed Newton state")
