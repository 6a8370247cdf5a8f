"""Space-time multigrid V-cycle on a strip partition.

The single-domain V-cycle (`stmg.StmgPreconditioner.apply`, reference
`StmgPreconditioner.vcycle` solver/multigrid.py:545-578) distributed over the
cell-row strips of `partition.StripPartition(..., levels=L)`:

* Each rank builds the whole L-level hierarchy of its local mesh (its strip
  plus 2^L ghost cell rows per side) with `pdst_hierarchy_depth`: the strips
  are aligned with the coarsest cells, so level f of the local mesh is a row
  range of the global level-f mesh with two ghost rows left on the coarsest
  level.  The Galerkin coarse operators (element form, multigrid.py:302-324)
  and the exact coarse patches of every cell the rank owns are then exactly
  the global ones: they depend only on fine cells inside the local mesh.
* Operators are owner-computes on every level: the x halo (two ghost cell rows)
  before each level matvec, the Vanka defect row and the increment
  reverse-add of the fine strip (`partition.distributed_vanka_step`), now on
  every level's layout.
* Restriction (P' of multigrid.py:523-532) of the owned part of the residual,
  then a reverse-add of the coarse node row on the strip boundary (the same
  plan as the Vanka increment); prolongation (multigrid.py:534-543) after a
  coarse halo exchange.
* Coarsest level: FGMRES right-preconditioned by Vanka steps from zero with
  allreduced Euclidean products — the distributed form of libpdst's
  `coarse_solver="fgmres"` (pdst_mg.cu coarse_fgmres: CGS2, Givens rotations)
  — since the reference's dense LU (multigrid.py:494-520) of a 128^2 coarsest
  level does not exist at cfg5 sizes.
* The mean-pressure projection (multigrid.py:557-572) with an allreduced mean.

Every vector a rank holds is its local (ghosted) level vector; only owned
entries are meaningful after each operation.  `ranks` arguments are lists of
`DistributedStmg` (several ranks in one process with `LocalTransport`, or one
rank per process with `TorchDistTransport`)."""

from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _lib as L
from .partition import StripPartition, local_context, owned_mask

__all__ = ["global_levels", "DistributedStmg", "distributed_vcycle", "LocalComm", "distributed_fgmres_mg",
           "distributed_nonlinear_solve"]

_VANKA = 1  # pdst_set_coarse_solver kind without a dense setup (the local coarsest level is never solved alone)


def global_levels(nx: int, ny: int, min_cells: int) -> int:
    """Levels of the global hierarchy (multigrid.py:164-191, pdst_hierarchy)."""
    n = 1
    while nx > min_cells and nx % 2 == 0 and ny > min_cells and ny % 2 == 0:
        nx, ny, n = nx // 2, ny // 2, n + 1
    return n


class LocalComm:
    """Sum over the ranks held in this process (the LocalTransport counterpart of
    `partition.DistComm`): allreduce of a list of per-rank tensors."""

    def allreduce_list(self, ts):
        s = ts[0].clone()
        for t in ts[1:]:
            s += t
        for t in ts:
            t.copy_(s)
        return ts


class _DistCommList:
    """Adapter: one rank per process, a list of one tensor."""

    def __init__(self, comm):
        self.comm = comm

    def allreduce_list(self, ts):
        (t,) = ts
        self.comm.allreduce_(t)
        return ts


class DistributedStmg:
    """One rank's local hierarchy, patches and level layouts."""

    def __init__(self, ctx, U, variant, part: StripPartition, rank: int, mg=None, device=0, U_is_local=False):
        import torch

        from .operators import SlabJacobian
        from .problem import dirichlet_flags
        from .stmg import MgConfig

        self.mg = mg or MgConfig()
        m = ctx.disc.mesh
        nl = global_levels(m.nx, m.ny, self.mg.min_cells)
        if part.levels != nl:
            raise ValueError(f"partition aligned for {part.levels} levels, the hierarchy has {nl}")
        tags = np.asarray(dirichlet_flags(m))
        nx, ny = m.nx, m.ny
        for side, sl in ((1, slice(nx, nx + ny)), (3, slice(2 * nx + ny, 2 * nx + 2 * ny))):
            if nl > 1 and np.any(tags[sl] != tags[sl][0]):
                # coarse faces take the tag of their side's first fine face (multigrid.py:174-182)
                raise NotImplementedError("distributed multigrid needs one boundary tag per left/right side")
        self.all_dirichlet = bool(np.all(tags == 1))
        self.part, self.rank, self.levels = part, rank, nl
        self.lay = part.layout(rank)
        self.lays = [self.lay.level(f) for f in range(nl)]  # f = 0 finest
        self.k1 = ctx.basis.k + 1
        self.ctx = local_context(ctx, self.lay)
        Ul = U if U_is_local else np.stack([self.lay.to_local(np.asarray(U[mu])) for mu in range(self.k1)])
        self.jac = SlabJacobian(self.ctx, Ul, variant, device=device)
        self.dev = self.jac.dev
        lib = L.lib()
        n = C.c_int(0)
        L.check(lib.pdst_hierarchy_depth(self.dev.h, nl, C.byref(n)), "pdst_hierarchy_depth")
        L.check(lib.pdst_set_coarse_solver(self.dev.h, _VANKA, 0, float(self.mg.omega), 1, 0.0),
                "pdst_set_coarse_solver")
        bl, bp = C.c_int(-1), C.c_int64(-1)
        rc = lib.pdst_patches_build(self.dev.h, int(self.mg.surrogate), float(self.mg.rep_fraction), C.byref(bl),
                                    C.byref(bp))
        L.check(rc, "pdst_patches_build", level=bl.value, patch=bp.value)
        self.device = torch.device("cuda", self.dev.device)
        self.masks = [owned_mask(l, self.k1, self.device) for l in self.lays]
        self.sizes = [self.k1 * l.nd_loc for l in self.lays]
        mg = self.mg
        self.coarse_sweeps = mg.coarse_sweeps if mg.coarse_sweeps is not None else 2
        self.coarse_omega = mg.coarse_omega if mg.coarse_omega is not None else mg.omega

    # -- local kernels (C level index: 0 = coarsest, L-1 = finest) -----------------
    def _idx(self, f):
        return self.levels - 1 - f

    def zeros(self, f):
        import torch

        return torch.zeros(self.sizes[f], dtype=torch.float64, device=self.device)

    def defect(self, f, d, r):
        if f == 0:
            return self.jac.defect(d, r)
        y = self.empty(f)
        L.check(L.lib().pdst_level_apply(self.dev.h, self._idx(f), L.vptr(d), L.vptr(y), self.dev.where(d, y)),
                "pdst_level_apply")
        return r - y

    def matvec(self, f, x):
        if f == 0:
            return self.jac.matvec(x)
        y = self.empty(f)
        L.check(L.lib().pdst_level_apply(self.dev.h, self._idx(f), L.vptr(x), L.vptr(y), self.dev.where(x, y)),
                "pdst_level_apply")
        return y

    def empty(self, f):
        import torch

        return torch.empty(self.sizes[f], dtype=torch.float64, device=self.device)

    def increment(self, f, defect, omega):
        lay = self.lays[f]
        inc = self.empty(f)
        L.check(L.lib().pdst_vanka_increment(self.dev.h, self._idx(f), L.vptr(defect), L.vptr(inc), lay.a - lay.c_lo,
                                             lay.b - lay.c_lo, float(omega), self.dev.where(defect, inc)),
                "pdst_vanka_increment")
        return inc

    def restrict(self, f, r):
        out = self.empty(f + 1)
        L.check(L.lib().pdst_restrict(self.dev.h, self._idx(f), L.vptr(r), L.vptr(out), self.dev.where(r, out)),
                "pdst_restrict")
        return out

    def prolong(self, f, e):
        out = self.empty(f)
        L.check(L.lib().pdst_prolong(self.dev.h, self._idx(f), L.vptr(e), L.vptr(out), self.dev.where(e, out)),
                "pdst_prolong")
        return out


# ---------------------------------------------------------------------------
# The distributed cycle (lists of ranks; every step is collective)
# ---------------------------------------------------------------------------


def _vanka_steps(ranks, f, ds, rs, steps, omega, transport, zero_start=False):
    """`steps` additive Vanka steps on level f (multigrid.py:327-340), owner computes.
    zero_start: the iterates ds are zero (the V-cycle's and the coarse solver's
    smoothing from a zero guess), so the first step's defect r - A 0 is r itself:
    no halo exchange of d and no operator apply for it (as libpdst's vanka_level)."""
    k1 = ranks[0].k1
    for s in range(steps):
        if zero_start and s == 0:
            defects = [r.clone() for r in rs]
        else:
            transport.exchange(ds, "halo_recv", k1, level=f)
            defects = [rk.defect(f, d, r) for rk, d, r in zip(ranks, ds, rs)]
        transport.exchange(defects, "defect_recv", k1, level=f)
        incs = [rk.increment(f, df, omega) for rk, df in zip(ranks, defects)]
        transport.exchange(incs, "inc_recv", k1, add=True, level=f)
        for d, inc in zip(ds, incs):
            d += inc
    return ds


def _dots(ranks, comm, A_list, w_list):
    """Global A_r' w_r (owned entries only: the operands have zero ghosts)."""
    vals = [A @ w for A, w in zip(A_list, w_list)]
    comm.allreduce_list(vals)
    return vals[0]


def _coarse_fgmres(ranks, bs, transport, comm):
    """Distributed restatement of libpdst's coarsest-level FGMRES (pdst_mg.cu
    coarse_fgmres): right preconditioning by Vanka steps from zero, CGS2,
    Givens rotations, stop after coarse_iters or at relative residual coarse_rtol."""
    import torch

    f = ranks[0].levels - 1
    k1 = ranks[0].k1
    mg = ranks[0].mg
    m = int(mg.coarse_iters)
    masks = [rk.masks[f] for rk in ranks]
    b = [bb * mk for bb, mk in zip(bs, masks)]
    beta = math.sqrt(float(_dots(ranks, comm, [x.view(1, -1) for x in b], b)[0]))
    zs = [rk.zeros(f) for rk in ranks]
    if not beta > 0.0:
        return zs
    V = [torch.zeros((m + 1, rk.sizes[f]), dtype=torch.float64, device=rk.device) for rk in ranks]
    Z = [torch.zeros((m, rk.sizes[f]), dtype=torch.float64, device=rk.device) for rk in ranks]
    for Vr, br in zip(V, b):
        Vr[0] = br / beta
    H = np.zeros((m + 1, m))
    cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
    g[0] = beta
    k = 0
    for j in range(m):
        zj = [rk.zeros(f) for rk in ranks]
        _vanka_steps(ranks, f, zj, [Vr[j] for Vr in V], ranks[0].coarse_sweeps, ranks[0].coarse_omega, transport,
                     zero_start=True)
        for Zr, z, mk in zip(Z, zj, masks):
            Zr[j] = z * mk
        transport.exchange(zj, "halo_recv", k1, level=f)
        w = [rk.matvec(f, z) * mk for rk, z, mk in zip(ranks, zj, masks)]
        for _ in range(2):  # CGS2
            c = _dots(ranks, comm, [Vr[: j + 1] for Vr in V], w)
            for wr, Vr in zip(w, V):
                wr -= Vr[: j + 1].T @ c
            H[: j + 1, j] += c.cpu().numpy()
        hn = math.sqrt(float(_dots(ranks, comm, [x.view(1, -1) for x in w], w)[0]))
        H[j + 1, j] = hn
        if hn > 0.0:
            for Vr, wr in zip(V, w):
                Vr[j + 1] = wr / hn
        for i in range(j):
            a, c_ = H[i, j], H[i + 1, j]
            H[i, j] = cs[i] * a + sn[i] * c_
            H[i + 1, j] = -sn[i] * a + cs[i] * c_
        a, c_ = H[j, j], H[j + 1, j]
        r = math.hypot(a, c_)
        cs[j] = a / r if r > 0.0 else 1.0
        sn[j] = c_ / r if r > 0.0 else 0.0
        H[j, j], H[j + 1, j] = r, 0.0
        g[j + 1] = -sn[j] * g[j]
        g[j] = cs[j] * g[j]
        k = j + 1
        if abs(g[j + 1]) <= mg.coarse_rtol * beta or not hn > 0.0:
            break
    y = np.zeros(k)
    for i in range(k - 1, -1, -1):
        s = g[i] - H[i, i + 1:k] @ y[i + 1:k]
        y[i] = s / H[i, i] if H[i, i] != 0.0 else 0.0
    for zr, Zr in zip(zs, Z):
        zr += Zr[:k].T @ torch.as_tensor(y, device=zr.device)
    return zs


def _cycle(ranks, f, bs, transport, comm, pre, post, omega):
    k1 = ranks[0].k1
    if f == ranks[0].levels - 1:
        return _coarse_fgmres(ranks, bs, transport, comm)
    zs = [rk.zeros(f) for rk in ranks]
    _vanka_steps(ranks, f, zs, bs, pre, omega, transport, zero_start=True)
    transport.exchange(zs, "halo_recv", k1, level=f)
    res = [rk.defect(f, z, b) * rk.masks[f] for rk, z, b in zip(ranks, zs, bs)]
    rc = [rk.restrict(f, r) for rk, r in zip(ranks, res)]
    transport.exchange(rc, "inc_recv", k1, add=True, level=f + 1)  # the strip-boundary coarse row
    rc = [r * rk.masks[f + 1] for rk, r in zip(ranks, rc)]
    zc = _cycle(ranks, f + 1, rc, transport, comm, pre, post, omega)
    transport.exchange(zc, "halo_recv", k1, level=f + 1)
    for rk, z, e in zip(ranks, zs, zc):
        z += rk.prolong(f, e)
    _vanka_steps(ranks, f, zs, bs, post, omega, transport)
    return zs


def distributed_vcycle(ranks, rs, transport, comm=None, pre=None, post=None, omega=None):
    """z_r = V-cycle(r) on every rank (StmgPreconditioner.apply, multigrid.py:545-578).

    rs: the ranks' local finest-level vectors (device tensors; ghost entries
    ignored).  comm: `LocalComm` for ranks in this process (default when
    len(ranks) > 1), or a `partition.DistComm`.  Returns local vectors with
    zero ghost entries, projected off the mean pressure when the global mesh
    is all-Dirichlet."""
    import torch

    mg = ranks[0].mg
    pre = mg.pre_smooth if pre is None else pre
    post = mg.post_smooth if post is None else post
    omega = mg.omega if omega is None else omega
    if comm is None:
        comm = LocalComm()
    elif not hasattr(comm, "allreduce_list"):
        comm = _DistCommList(comm)
    bs = [torch.as_tensor(r, device=rk.device).reshape(-1) for rk, r in zip(ranks, rs)]
    zs = _cycle(ranks, 0, bs, transport, comm, pre, post, omega)
    zs = [z * rk.masks[0] for rk, z in zip(ranks, zs)]
    if ranks[0].all_dirichlet:
        # remove the mean of the constant pressure coefficient per Radau node (k_project_pressure)
        k1 = ranks[0].k1
        sums = []
        for rk, z in zip(ranks, zs):
            lay = rk.lay
            p0 = z.view(k1, lay.nd_loc)[:, lay.prs_slice_local(lay.a, lay.b)][:, 0::3]
            sums.append(p0.sum(dim=1))
        comm.allreduce_list(sums)
        ncells = ranks[0].lay.nx * ranks[0].lay.ny
        for rk, z, s in zip(ranks, zs, sums):
            lay = rk.lay
            zv = z.view(k1, lay.nd_loc)
            pl = lay.prs_slice_local(lay.a, lay.b)
            zv[:, pl.start:pl.stop:3] -= (s / ncells).view(k1, 1)
    return zs


# ---------------------------------------------------------------------------
# FGMRES preconditioned by the distributed V-cycle (the modified-Newton inner
# solve of newton.py:204-222 on a strip partition)
# ---------------------------------------------------------------------------


class _NoComm:
    """The ranks' local vectors are stacked into one vector (all ranks in this
    process): the local products are already global."""

    def allreduce_(self, t):
        return t


def distributed_fgmres_mg(ranks, transport, rhs, tol, config=None, comm=None, x0=None, op_jacs=None):
    """FGMRES in the M-inner product (krylov.fgmres) on the strip partition,
    right-preconditioned by `distributed_vcycle`.

    ranks: the `DistributedStmg` of this process (all ranks with
    LocalTransport, or this process's one rank with TorchDistTransport and a
    `partition.DistComm`).  The ranks' local vectors (ghost entries zero) are
    stacked into one Krylov vector, so every inner product is the owned-entry
    sum — plus one allreduce per Gram-Schmidt pass across processes.  Returns
    the FgmresResult with x as the list of local vectors (ghosts zero).
    op_jacs: the operator's SlabJacobians (default: the ranks' own, i.e. the
    preconditioner's linearization)."""
    import dataclasses

    import torch

    from .krylov import fgmres
    from .operators import MassNorm

    k1 = ranks[0].k1
    sizes = [rk.sizes[0] for rk in ranks]
    offs = np.concatenate([[0], np.cumsum(sizes)]).tolist()
    device = ranks[0].device
    mask = torch.cat([rk.masks[0] for rk in ranks])
    masses = [MassNorm(rk.ctx, dev=rk.dev) for rk in ranks]
    vcomm = LocalComm() if comm is None else _DistCommList(comm)

    def split(v):
        return [v[offs[i]:offs[i + 1]] for i in range(len(ranks))]

    def halo_copy(v):
        parts = [p.clone() for p in split(v)]
        transport.exchange(parts, "halo_recv", k1)
        return parts

    jacs = op_jacs if op_jacs is not None else [rk.jac for rk in ranks]

    def op(v, out=None):
        y = torch.cat([jac.matvec(p) for jac, p in zip(jacs, halo_copy(v))]) * mask
        if out is not None:
            out.copy_(y)
            return out
        return y

    class _Mass:
        dev = ranks[0].dev

        def apply_into(self, v, out):
            for ms, p, o in zip(masses, halo_copy(v), split(out)):
                ms.apply_into(p, o)
            out.mul_(mask)
            return out

    def precond(v, out=None):
        z = torch.cat(distributed_vcycle(ranks, split(v), transport, vcomm))
        if out is not None:
            out.copy_(z)
            return out
        return z

    b = torch.cat([torch.as_tensor(r, device=device).reshape(-1) for r in rhs]) * mask
    x0c = None if x0 is None else torch.cat([torch.as_tensor(x, device=device).reshape(-1) for x in x0]) * mask
    res = fgmres(op, b, tol, config, precond=precond, mass=_Mass(), x0=x0c, comm=comm or _NoComm())
    return dataclasses.replace(res, x=split(res.x))


# ---------------------------------------------------------------------------
# One slab's modified-Newton solve on a strip partition (newton.py:168-284)
# ---------------------------------------------------------------------------


def distributed_nonlinear_solve(ctx, U0, newton, krylov, mg, part: StripPartition, rank_ids, transport, comm=None,
                                device=0):
    """`newton.nonlinear_solve_slab` with FGMRES preconditioned by the
    distributed V-cycle, on the strips `rank_ids` of `part` held by this
    process (all of them with LocalTransport, one with TorchDistTransport and
    a `partition.DistComm`).  Same control flow: Eisenstat-Walker forcing,
    Armijo backtracking, the rebuild policy, the same failure kinds.  The
    state lives as local (ghosted) slabs whose 2^L ghost rows are refreshed
    from the neighbours after every update (`deep_halo_recv`), so each rank's
    residual, linearization and hierarchy see the global state.  Norms are
    M-norms of the owned entries summed over the ranks.  Returns (list of the
    local states, SlabStats)."""
    import torch

    from .errors import SlabSolveError
    from .newton import PIC, NewtonStepStats, SlabStats, _forcing, rebuild_policy
    from .operators import MassNorm, SlabDevice, SlabJacobian, slab_residual
    from .problem import dirichlet_flags

    k1 = ctx.basis.k + 1
    dev = torch.device("cuda", device)
    lays = [part.layout(r) for r in rank_ids]
    lctxs = [local_context(ctx, lay) for lay in lays]
    masks = [owned_mask(lay, k1, dev) for lay in lays]
    U0 = np.asarray(U0, dtype=np.float64)
    Us = [torch.as_tensor(np.stack([lay.to_local(U0[mu]) for mu in range(k1)]), device=dev) for lay in lays]
    sds = [SlabDevice(lc, device) for lc in lctxs]
    jds = [SlabDevice(lc, device) for lc in lctxs]
    masses = [MassNorm(lc, dev=sd) for lc, sd in zip(lctxs, sds)]
    vcomm = LocalComm() if comm is None else _DistCommList(comm)
    is_picard = newton.variant.kind == PIC

    def refresh(U_list):
        transport.exchange([u.view(-1) for u in U_list], "deep_halo_recv", k1)

    def residual(U_list):
        refresh(U_list)
        return [slab_residual(lc, u, dev=sd).reshape(-1) * m for lc, u, sd, m in zip(lctxs, U_list, sds, masks)]

    def mnorm(R_list):
        tmp = [r.clone() for r in R_list]
        transport.exchange(tmp, "halo_recv", k1)
        vals = []
        for ms, t, r, m in zip(masses, tmp, R_list, masks):
            mr = torch.empty_like(t)
            ms.apply_into(t, mr)
            vals.append((r * (mr * m)).sum().reshape(1))
        vcomm.allreduce_list(vals)
        return float(np.sqrt(max(float(vals[0].item()), 0.0)))

    R = residual(Us)
    rnorm = mnorm(R)
    stats = SlabStats(initial_res=rnorm)
    r0 = rnorm
    pre = None
    eta_prev = newton.forcing_eta0
    rnorm_prev = rnorm
    prev_n_l = 0

    def finish():
        if bool((dirichlet_flags(ctx.disc.mesh) == 1).all()):  # zero mean of the constant pressure mode
            sums = []
            for lay, u in zip(lays, Us):
                pl = lay.prs_slice_local(lay.a, lay.b)
                sums.append(u[:, pl.start:pl.stop:3].sum(dim=1))
            vcomm.allreduce_list(sums)
            n = ctx.disc.mesh.nx * ctx.disc.mesh.ny
            out = []
            for lay, u, sm in zip(lays, Us, sums):
                v = u.clone()
                v[:, lay.mv_loc::3] -= (sm / n).view(k1, 1)
                out.append(v)
            return out
        return Us

    for m in range(newton.max_nonlinear):
        if rnorm <= newton.abs_tol or rnorm <= newton.rel_tol * r0:
            stats.converged = True
            stats.final_res = rnorm
            return finish(), stats
        jacs = [SlabJacobian(lc, u, newton.variant, dev=jd) for lc, u, jd in zip(lctxs, Us, jds)]
        ratio = rnorm / rnorm_prev if m > 0 else 0.0
        last_n_l = stats.steps[-1].n_l if stats.steps else 0
        rebuilt = False
        if pre is None or rebuild_policy(ratio, last_n_l, prev_n_l, mg.rebuild_rho, mg.rebuild_factor):
            pre = [DistributedStmg(ctx, u, newton.variant, part, r, mg, device=device, U_is_local=True)
                   for r, u in zip(rank_ids, Us)]
            rebuilt = True
        prev_n_l = stats.steps[-1].n_l if stats.steps else 0
        eta = newton.picard_fixed_tol if is_picard else _forcing(newton, m, rnorm, rnorm_prev, eta_prev)
        result = distributed_fgmres_mg(pre, transport, R, eta, krylov, comm=comm, op_jacs=jacs)
        if not result.converged:
            stats.failure = "krylov"
            stats.final_res = rnorm
            raise SlabSolveError("krylov", f"FGMRES stalled at |r|={result.residual_norm:.3e} "
                                           f"(target {result.target:.3e})", stats)
        dUs = [x.reshape(u.shape) for x, u in zip(result.x, Us)]
        phi = 0.5 * rnorm**2
        lam = 1.0
        if is_picard:
            Us = [u + du for u, du in zip(Us, dUs)]
            R_new = residual(Us)
            rnorm_new = mnorm(R_new)
        else:
            while True:
                U_try = [u + lam * du for u, du in zip(Us, dUs)]
                R_new = residual(U_try)
                rnorm_new = mnorm(R_new)
                if 0.5 * rnorm_new**2 <= (1.0 - newton.armijo_c1 * lam) * phi:
                    Us = U_try
                    break
                lam *= newton.armijo_backtrack
                if lam < newton.armijo_lambda_min:
                    stats.failure = "line_search"
                    stats.final_res = rnorm
                    raise SlabSolveError("line_search",
                                         f"no sufficient decrease above lambda={lam:.2e} at |R|={rnorm:.3e}", stats)
        stats.steps.append(NewtonStepStats(n_l=result.iterations, lam=lam, eta=eta, res_before=rnorm,
                                           res_after=rnorm_new, lin_res=result.residual_norm, rebuilt=rebuilt))
        rnorm_prev = rnorm
        rnorm = rnorm_new
        eta_prev = eta
        R = R_new
    if rnorm <= newton.abs_tol or rnorm <= newton.rel_tol * r0:
        stats.converged = True
        stats.final_res = rnorm
        return finish(), stats
    stats.failure = "max_iterations"
    stats.final_res = rnorm
    raise SlabSolveError("max_iterations", f"|R|={rnorm:.3e} after {newton.max_nonlinear} iterations", stats)
