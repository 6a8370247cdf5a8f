"""Cell-strip partition of the slab hot path across GPUs.

Rank r owns the cell rows [a_r, b_r) of the nx x ny mesh: the Q2 node rows
[2 a_r, 2 b_r) (the last rank also the top row 2 ny) and the P1disc dofs of
its cells.  Its local mesh is the strip plus two ghost cell rows on each side,
[c_lo, c_hi) = [max(0, a-2), min(ny, b+2)); the sides of the local mesh that
are interior faces of the global mesh carry the "cut" tag (2), so the kernels
apply no boundary terms there.  Two ghost rows are what the CIP gradient-jump
faces need: the face below cell a-1 still touches node row 2a, and the face
above cell b still touches node row 2b, which belongs to the Vanka patch of
cell b-1.  With that depth every owned node receives all of its element,
CIP-face and temporal-mass contributions locally and every owned patch matrix
is exact: owner computes, no reverse-add for the operator.

Exchanges (one per operator application, contiguous slices of the node-major
layout, per Radau block):
  * x halo: node rows [2c_lo, 2a) from rank r-1, [2b, 2b+2] from rank r+1,
    plus the pressure of the ghost cells below (cells c_lo..a-1) -- the ghost
    node rows above 2b+2 only feed ghost outputs;
  * Vanka defect halo: node row 2b (owned by r+1) for the patch of cell b-1;
  * Vanka increment reverse-add: the increment of node row 2b computed from
    r's patch of cell b-1 is added by r+1 (and r adds r-1's at row 2a).
Transports: LocalTransport (several ranks' local vectors in one process,
e.g. one GPU) and TorchDistTransport (torch.distributed point-to-point:
NCCL on GPUs, gloo on CPU tensors).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["StripPartition", "RankLayout", "LocalTransport", "TorchDistTransport", "DistributedSlab", "DistComm",
           "distributed_fgmres", "distributed_apply_and_vanka_step"]

CUT = 2


def strip_bounds(ny: int, nranks: int, unit: int = 1):
    """Cell-row ranges [a_r, b_r), as even as possible in multiples of `unit`
    rows (the coarsest multigrid cell), each >= 2 units."""
    if ny % unit:
        raise ValueError(f"{ny} cell rows are not a multiple of the coarsest cell ({unit} rows)")
    nu = ny // unit
    if nu < 2 * nranks:
        raise ValueError(f"{ny} cell rows cannot give {nranks} strips of >= 2 x {unit} rows")
    return [(r * nu // nranks * unit, (r + 1) * nu // nranks * unit) for r in range(nranks)]


def ghost_rows(levels: int) -> int:
    """Ghost cell rows per side of the finest local mesh: 2 on every level of a
    `levels`-level hierarchy (the strip coarsens with the global mesh)."""
    return 2 if levels <= 1 else 2 ** levels


@dataclass(frozen=True)
class RankLayout:
    rank: int
    nranks: int
    nx: int
    ny: int  # global cell rows
    a: int
    b: int  # owned cell rows [a, b)
    c_lo: int
    c_hi: int  # local cell rows [c_lo, c_hi)
    levels: int = 1  # multigrid levels the partition is aligned for
    f: int = 0  # this layout's level (0 = finest)

    def level(self, f: int) -> "RankLayout":
        """The same rank's layout on multigrid level f (every index halved f times)."""
        if not 0 <= f < self.levels or self.f != 0:
            raise ValueError(f"level {f} of a {self.levels}-level partition")
        s = f
        return RankLayout(self.rank, self.nranks, self.nx >> s, self.ny >> s, self.a >> s, self.b >> s,
                          self.c_lo >> s, self.c_hi >> s, self.levels, f)

    @property
    def ny_loc(self):
        return self.c_hi - self.c_lo

    @property
    def nnx(self):
        return 2 * self.nx + 1

    @property
    def mv_loc(self):
        return 2 * self.nnx * (2 * self.ny_loc + 1)

    @property
    def nd_loc(self):
        return self.mv_loc + 3 * self.nx * self.ny_loc

    @property
    def mv(self):
        return 2 * self.nnx * (2 * self.ny + 1)

    @property
    def nd(self):
        return self.mv + 3 * self.nx * self.ny

    @property
    def last(self):
        return self.rank == self.nranks - 1

    # -- node rows (global Y) ----------------------------------------------
    @property
    def owned_node_rows(self):
        return range(2 * self.a, 2 * self.ny + 1 if self.last else 2 * self.b)

    def vel_slice_local(self, Y0: int, Y1: int):
        """Local velocity slice of global node rows [Y0, Y1)."""
        y0, y1 = Y0 - 2 * self.c_lo, Y1 - 2 * self.c_lo
        return slice(2 * y0 * self.nnx, 2 * y1 * self.nnx)

    def prs_slice_local(self, j0: int, j1: int):
        """Local pressure slice of global cell rows [j0, j1)."""
        return slice(self.mv_loc + 3 * (j0 - self.c_lo) * self.nx, self.mv_loc + 3 * (j1 - self.c_lo) * self.nx)

    def vel_slice_global(self, Y0: int, Y1: int):
        return slice(2 * Y0 * self.nnx, 2 * Y1 * self.nnx)

    def prs_slice_global(self, j0: int, j1: int):
        return slice(self.mv + 3 * j0 * self.nx, self.mv + 3 * j1 * self.nx)

    # -- local mesh description --------------------------------------------
    def local_tags(self, global_tags: np.ndarray) -> np.ndarray:
        """uint8 tags of the local mesh's boundary faces (bottom, right, top, left)."""
        nx, ny = self.nx, self.ny
        g = np.asarray(global_tags, dtype=np.uint8)
        bottom = g[0:nx] if self.c_lo == 0 else np.full(nx, CUT, np.uint8)
        right = g[nx + self.c_lo: nx + self.c_hi]
        top = g[nx + ny: 2 * nx + ny] if self.c_hi == ny else np.full(nx, CUT, np.uint8)
        left = g[2 * nx + ny + self.c_lo: 2 * nx + ny + self.c_hi]
        return np.concatenate([bottom, right, top, left]).astype(np.uint8)

    def local_extents(self, extents):
        x0, y0, x1, y1 = extents
        hy = (y1 - y0) / self.ny
        return (x0, y0 + self.c_lo * hy, x1, y0 + self.c_hi * hy)

    # -- global <-> local vectors (per Radau block) ---------------------------
    def to_local(self, xg: np.ndarray) -> np.ndarray:
        """Local block (with ghosts) of a global block vector."""
        out = np.empty(self.nd_loc, dtype=xg.dtype)
        out[: self.mv_loc] = xg[self.vel_slice_global(2 * self.c_lo, 2 * self.c_hi + 1)]
        out[self.mv_loc:] = xg[self.prs_slice_global(self.c_lo, self.c_hi)]
        return out

    def owned_into_global(self, xl: np.ndarray, xg: np.ndarray):
        Y0, Y1 = self.owned_node_rows.start, self.owned_node_rows.stop
        xg[self.vel_slice_global(Y0, Y1)] = xl[self.vel_slice_local(Y0, Y1)]
        xg[self.prs_slice_global(self.a, self.b)] = xl[self.prs_slice_local(self.a, self.b)]

    # -- exchange plans: lists of (peer, my local slice, peer's local slice) ---
    def halo_recv(self):
        """(peer, my ghost slice, peer-owned slice in the peer's local vector) for the x halo."""
        out = []
        if self.rank > 0:
            lo = _layout_of(self, self.rank - 1)
            h = max(self.c_lo, self.a - 2)  # two ghost cell rows feed every owned output
            out.append((self.rank - 1, self.vel_slice_local(2 * h, 2 * self.a), lo.vel_slice_local(2 * h, 2 * self.a)))
            out.append((self.rank - 1, self.prs_slice_local(h, self.a), lo.prs_slice_local(h, self.a)))
        if not self.last:
            hi = _layout_of(self, self.rank + 1)
            top = min(2 * self.b + 3, 2 * self.c_hi + 1)
            out.append((self.rank + 1, self.vel_slice_local(2 * self.b, top), hi.vel_slice_local(2 * self.b, top)))
        return out

    def deep_halo_recv(self):
        """Every ghost row of the local mesh (state / linearization halo of a
        multigrid partition, 2^L rows deep) from the two neighbours, which own
        them when the strips are at least that thick (checked)."""
        out = []
        if self.rank > 0:
            lo = _layout_of(self, self.rank - 1)
            if self.c_lo < lo.a:
                raise ValueError(f"rank {self.rank}: ghost rows from {self.c_lo} reach past rank {self.rank - 1}")
            out.append((self.rank - 1, self.vel_slice_local(2 * self.c_lo, 2 * self.a),
                        lo.vel_slice_local(2 * self.c_lo, 2 * self.a)))
            out.append((self.rank - 1, self.prs_slice_local(self.c_lo, self.a), lo.prs_slice_local(self.c_lo, self.a)))
        if not self.last:
            hi = _layout_of(self, self.rank + 1)
            if not (self.c_hi < hi.b or hi.last):
                raise ValueError(f"rank {self.rank}: ghost rows up to {self.c_hi} reach past rank {self.rank + 1}")
            out.append((self.rank + 1, self.vel_slice_local(2 * self.b, 2 * self.c_hi + 1),
                        hi.vel_slice_local(2 * self.b, 2 * self.c_hi + 1)))
            out.append((self.rank + 1, self.prs_slice_local(self.b, self.c_hi), hi.prs_slice_local(self.b, self.c_hi)))
        return out

    def defect_recv(self):
        """The defect of node row 2b (owned by rank+1)."""
        if self.last:
            return []
        hi = _layout_of(self, self.rank + 1)
        return [(self.rank + 1, self.vel_slice_local(2 * self.b, 2 * self.b + 1),
                 hi.vel_slice_local(2 * self.b, 2 * self.b + 1))]

    def inc_recv(self):
        """Increment of node row 2a computed by rank-1 (from its patch of cell a-1)."""
        if self.rank == 0:
            return []
        lo = _layout_of(self, self.rank - 1)
        return [(self.rank - 1, self.vel_slice_local(2 * self.a, 2 * self.a + 1),
                 lo.vel_slice_local(2 * self.a, 2 * self.a + 1))]


class StripPartition:
    """Cell-row strips of an nx x ny mesh.  levels > 1 aligns the strips with the
    coarsest cells of a `levels`-level hierarchy and deepens the ghost region to
    2^levels rows, so each rank's local mesh coarsens into the global coarse
    mesh's rows with two ghost rows left on the coarsest level."""

    def __init__(self, nx: int, ny: int, nranks: int, levels: int = 1):
        self.nx, self.ny, self.nranks, self.levels = nx, ny, nranks, levels
        self.unit = 2 ** (levels - 1)
        if nx % self.unit:
            raise ValueError(f"nx={nx} cannot be coarsened {levels - 1} times")
        self.bounds = strip_bounds(ny, nranks, self.unit)
        self.ghost = ghost_rows(levels)

    def layout(self, rank: int) -> RankLayout:
        a, b = self.bounds[rank]
        gh = self.ghost
        return RankLayout(rank, self.nranks, self.nx, self.ny, a, b, max(0, a - gh), min(self.ny, b + gh), self.levels)


def _layout_of(lay: RankLayout, rank: int) -> RankLayout:
    fine = StripPartition(lay.nx << lay.f, lay.ny << lay.f, lay.nranks, lay.levels).layout(rank)
    return fine.level(lay.f) if lay.f else fine


# ---------------------------------------------------------------------------
# Transports
# ---------------------------------------------------------------------------


class LocalTransport:
    """All ranks' local vectors in one process (same device or host)."""

    def __init__(self, layouts):
        self.layouts = layouts

    def exchange(self, vectors, plan_name: str, k1: int, add: bool = False, level: int = 0):
        """vectors[r]: rank r's local slab vector (k1 blocks of nd_loc) on
        multigrid level `level` of the partition."""
        lays = [l.level(level) for l in self.layouts] if level else self.layouts
        for r, lay in enumerate(lays):
            for peer, mine, theirs in getattr(lay, plan_name)():
                nd, ndp = lay.nd_loc, lays[peer].nd_loc
                for mu in range(k1):
                    dst = vectors[r][mu * nd + mine.start: mu * nd + mine.stop]
                    src = vectors[peer][mu * ndp + theirs.start: mu * ndp + theirs.stop]
                    if add:
                        dst += src
                    else:
                        dst[...] = src

    def exchange_many(self, items, k1: int, level: int = 0):
        """Several independent exchanges [(vectors, plan_name, add), ...]."""
        _exchange_many_sequential(self, items, k1, level)


def _exchange_many_sequential(transport, items, k1, level=0):
    for vectors, plan_name, add in items:
        transport.exchange(vectors, plan_name, k1, add=add, level=level)


class TorchDistTransport:
    """One rank per process over torch.distributed point-to-point messages.

    For plan entry (peer, mine, theirs) rank r receives into `mine`; the peer
    sends its slice `theirs` — every rank derives both sides from the
    partition, so no metadata is exchanged."""

    def __init__(self, layout: RankLayout, part: StripPartition):
        import torch.distributed as dist

        self.dist = dist
        self.lay = layout
        self.part = part

    def _ops(self, vec, plan_name, k1, level):
        """(P2P ops, received-buffer placements) of one exchange of `vec`."""
        import torch

        if isinstance(vec, (list, tuple)):  # the distributed_* helpers pass one vector per local rank
            (vec,) = vec
        lay = self.lay.level(level) if level else self.lay
        # gloo moves host tensors only: stage device slices through the host
        xdev = vec.device if self.dist.get_backend() == "gloo" else None
        bdev = torch.device("cpu") if xdev is not None and xdev.type == "cuda" else vec.device
        ops, recv_bufs = [], []
        for peer, mine, _ in getattr(lay, plan_name)():
            buf = torch.empty((k1, mine.stop - mine.start), dtype=vec.dtype, device=bdev)
            recv_bufs.append((vec, lay, mine, buf))
            ops.append(self.dist.P2POp(self.dist.irecv, buf, peer))
        # what my neighbours receive from me
        for peer in (lay.rank - 1, lay.rank + 1):
            if peer < 0 or peer >= lay.nranks:
                continue
            pl = self.part.layout(peer)
            pl = pl.level(level) if level else pl
            for src_rank, _, theirs in getattr(pl, plan_name)():
                if src_rank != lay.rank:
                    continue
                v2 = vec.view(k1, lay.nd_loc)
                ops.append(self.dist.P2POp(self.dist.isend, v2[:, theirs].contiguous().to(bdev), peer))
        return ops, recv_bufs

    @staticmethod
    def _place(recv_bufs, k1, add):
        for vec, lay, mine, buf in recv_bufs:
            v2 = vec.view(k1, lay.nd_loc)
            buf = buf.to(vec.device)
            if add:
                v2[:, mine] += buf
            else:
                v2[:, mine] = buf

    def exchange(self, vec, plan_name: str, k1: int, add: bool = False, level: int = 0):
        self.exchange_many([(vec, plan_name, add)], k1, level)

    def exchange_many(self, items, k1: int, level: int = 0):
        """Several independent exchanges [(vec, plan_name, add), ...] in ONE
        grouped send/recv (one NCCL launch and latency instead of one each)."""
        ops, placements = [], []
        for vec, plan_name, add in items:
            o, r = self._ops(vec, plan_name, k1, level)
            ops += o
            placements.append((r, add))
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()
        for r, add in placements:
            self._place(r, k1, add)


# ---------------------------------------------------------------------------
# Distributed operators (one local SlabDevice per rank)
# ---------------------------------------------------------------------------


def local_context(ctx, lay: RankLayout):
    """The reference-style SlabContext of a rank's local mesh (cut tags)."""
    from .problem import Discretization, QuadMesh, SlabContext, dirichlet_flags

    m = ctx.disc.mesh
    ext = lay.local_extents((m.x0, m.y0, m.x1, m.y1))
    tags = lay.local_tags(dirichlet_flags(m))
    mesh = QuadMesh(m.nx, lay.ny_loc, *ext, boundary_tags=_TagArray(tags))
    cfg = ctx.config
    if getattr(cfg, "g_hat", None) is not None:
        from dataclasses import replace

        cfg = replace(cfg, g_hat=lay.to_local(np.concatenate([np.asarray(cfg.g_hat), np.zeros(3 * m.nx * m.ny)]))[
            : lay.mv_loc])
    vm = lay.to_local(np.concatenate([np.asarray(ctx.v_minus), np.zeros(3 * m.nx * m.ny)]))[: lay.mv_loc]
    return SlabContext(Discretization(mesh), ctx.params, cfg, ctx.data, ctx.basis, ctx.tmat, ctx.t_start, ctx.tau, vm)


class _TagArray(np.ndarray):
    """uint8 tag array understood by problem.dirichlet_flags (0/1/2 verbatim)."""

    def __new__(cls, tags):
        return np.asarray(tags, dtype=np.uint8).view(cls)


class DistributedSlab:
    """Slab Jacobian + Vanka sweep of one rank of a strip partition."""

    def __init__(self, ctx, U, variant, part: StripPartition, rank: int, transport, device=0, surrogate=True,
                 rep_fraction=0.5, U_is_local=False):
        from .operators import SlabJacobian
        from .smoother import VankaLevel

        self.lay = part.layout(rank)
        self.k1 = ctx.basis.k + 1
        self.transport = transport
        self.ctx = local_context(ctx, self.lay)
        Ul = U if U_is_local else np.stack([self.lay.to_local(U[mu]) for mu in range(self.k1)])
        self.jac = SlabJacobian(self.ctx, Ul, variant, device=device)
        self.level = None
        self.surrogate, self.rep_fraction = surrogate, rep_fraction
        self.strip = self.nccl = False  # libpdst data plane (strip_setup / attach_nccl)

    def strip_setup(self):
        """Register this rank's strip with its libpdst handle (pdst_strip):
        the in-library data plane (halo pack / unpack kernels, fused owned-row
        Vanka update, NCCL exchanges) of pdst_strip_step."""
        from . import _lib as L

        lay = self.lay
        lower_c_hi = _layout_of(lay, lay.rank - 1).c_hi if lay.rank > 0 else 0
        upper_c_lo = _layout_of(lay, lay.rank + 1).c_lo if not lay.last else lay.ny
        L.check(L.lib().pdst_strip(self.jac.dev.h, lay.rank, lay.nranks, lay.ny, lay.a, lay.b, lay.c_lo, lay.c_hi,
                                   lower_c_hi, upper_c_lo), "pdst_strip")
        self.strip = True

    def attach_nccl(self, group=None):
        """Hand torch.distributed's NCCL communicator (ProcessGroupNCCL's
        ncclComm_t, rank order = partition order) to libpdst (pdst_strip_comm)."""
        import torch
        import torch.distributed as dist

        from . import _lib as L

        pg = group or dist.group.WORLD
        backend = pg._get_backend(torch.device("cuda", self.jac.dev.device))
        ptr = backend._comm_ptr()
        if not ptr:
            raise RuntimeError("the NCCL communicator is not initialized (init_process_group(device_id=...))")
        L.check(L.lib().pdst_strip_comm(self.jac.dev.h, L.C.c_void_p(ptr)), "pdst_strip_comm")
        self.nccl = True

    def build_patches(self):
        from .smoother import VankaLevel

        self.level = VankaLevel(self.ctx, None, None, surrogate=self.surrogate, rep_fraction=self.rep_fraction,
                                jac=self.jac)
        return self.level

    def local(self, xg):
        """Local (ghosted) slab vector of a global slab vector (numpy)."""
        nd = self.lay.nd
        return np.concatenate([self.lay.to_local(xg[mu * nd:(mu + 1) * nd]) for mu in range(self.k1)])

    def owned_into(self, xl, xg):
        nd, ndl = self.lay.nd, self.lay.nd_loc
        for mu in range(self.k1):
            self.lay.owned_into_global(np.asarray(xl[mu * ndl:(mu + 1) * ndl]), xg[mu * nd:(mu + 1) * nd])


def distributed_apply(ranks, xs, transport):
    """y_r = J x on every rank after the x halo exchange (owner computes)."""
    transport.exchange(xs, "halo_recv", ranks[0].k1)
    return [rk.jac.matvec(x) for rk, x in zip(ranks, xs)]


def distributed_vanka_step(ranks, ds, rs, omega, transport):
    """One additive Vanka step on every rank; ds updated in place (local)."""
    k1 = ranks[0].k1
    transport.exchange(ds, "halo_recv", k1)
    defects = [rk.jac.defect(d, r) for rk, d, r in zip(ranks, ds, rs)]
    transport.exchange(defects, "defect_recv", k1)
    incs = []
    for rk, df in zip(ranks, defects):
        lay = rk.lay
        incs.append(rk.level.increment(df, lay.a - lay.c_lo, lay.b - lay.c_lo, omega))
    transport.exchange(incs, "inc_recv", k1, add=True)
    for d, inc in zip(ds, incs):
        d += inc
    return ds


def strip_step(ranks, xs, ds, rs, omega, ys=None):
    """The distributed apply + Vanka step inside libpdst (pdst_strip.cu):
    every exchange a pack kernel, a transfer and an unpack kernel, the Vanka
    update one fused scatter over the owned patches, all on one stream with
    no host synchronization.  ranks: all ranks of the partition in this
    process (virtual ranks on one device, pdst_strips_step_local) or this
    process's one rank with an attached NCCL communicator (pdst_strip_step).
    Returns the ys; ds updated in place."""
    import torch

    from . import _lib as L

    ys = ys if ys is not None else [torch.empty_like(x) for x in xs]
    h0 = ranks[0].jac.dev
    h0.where(xs[0])  # torch's current stream for the whole step
    if len(ranks) == 1 and ranks[0].lay.nranks > 1:
        L.check(L.lib().pdst_strip_step(h0.h, L.vptr(xs[0]), L.vptr(ys[0]), L.vptr(ds[0]), L.vptr(rs[0]),
                                        float(omega)), "pdst_strip_step")
        return ys
    n = len(ranks)
    P = L.C.c_void_p * n
    hs = P(*[rk.jac.dev.h.value for rk in ranks])
    arr = lambda vs: P(*[v.data_ptr() for v in vs])  # noqa: E731
    L.check(L.lib().pdst_strips_step_local(L.C.cast(hs, L.C.c_void_p), n, L.C.cast(arr(xs), L.C.c_void_p),
                                           L.C.cast(arr(ys), L.C.c_void_p), L.C.cast(arr(ds), L.C.c_void_p),
                                           L.C.cast(arr(rs), L.C.c_void_p), float(omega)), "pdst_strips_step_local")
    return ys


def _strip_ready(ranks, transport):
    """The libpdst data plane applies: every rank registered as a strip, and
    either all ranks in this process (LocalTransport) or one rank with its
    NCCL communicator attached."""
    if not all(getattr(rk, "strip", False) for rk in ranks):
        return False
    if isinstance(transport, LocalTransport):
        return True
    return len(ranks) == 1 and getattr(ranks[0], "nccl", False)


def distributed_apply_and_vanka_step(ranks, xs, ds, rs, omega, transport):
    """y = J x and one Vanka step on d (rhs r) on every rank, the two
    independent x / d halos in one grouped exchange.  Returns the ys; ds
    updated in place.  Same results as distributed_apply then
    distributed_vanka_step.  With the ranks registered as strips
    (DistributedSlab.strip_setup, and attach_nccl across processes) the
    whole step runs inside libpdst (strip_step)."""
    if _strip_ready(ranks, transport) and all(hasattr(x, "data_ptr") for x in xs):
        return strip_step(ranks, xs, ds, rs, omega)
    k1 = ranks[0].k1
    transport.exchange_many([(xs, "halo_recv", False), (ds, "halo_recv", False)], k1)
    ys = [rk.jac.matvec(x) for rk, x in zip(ranks, xs)]
    defects = [rk.jac.defect(d, r) for rk, d, r in zip(ranks, ds, rs)]
    transport.exchange(defects, "defect_recv", k1)
    incs = []
    for rk, df in zip(ranks, defects):
        lay = rk.lay
        incs.append(rk.level.increment(df, lay.a - lay.c_lo, lay.b - lay.c_lo, omega))
    transport.exchange(incs, "inc_recv", k1, add=True)
    for d, inc in zip(ds, incs):
        d += inc
    return ys


# ---------------------------------------------------------------------------
# Distributed Krylov (FGMRES in the M-inner product with allreduced dots)
# ---------------------------------------------------------------------------


class DistComm:
    """Sum-allreduce of device (or host) tensors over a torch.distributed group
    (NCCL between GPUs; gloo staged through the host)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.host = dist.get_backend(group) == "gloo"

    def allreduce_(self, t):
        if self.host and t.is_cuda:
            h = t.cpu()
            self.dist.all_reduce(h, group=self.group)
            t.copy_(h)
        else:
            self.dist.all_reduce(t, group=self.group)
        return t


def owned_mask(lay: RankLayout, k1: int, device=None):
    """1 on the dofs rank `lay` owns, 0 on its ghost dofs (local slab vector)."""
    import torch

    m = torch.zeros((k1, lay.nd_loc), dtype=torch.float64, device=device)
    rows = lay.owned_node_rows
    m[:, lay.vel_slice_local(rows.start, rows.stop)] = 1.0
    m[:, lay.prs_slice_local(lay.a, lay.b)] = 1.0
    return m.reshape(-1)


def distributed_fgmres(rank: DistributedSlab, transport, comm: DistComm, rhs, tol, config=None, vanka_steps=0,
                       omega=0.7, x0=None):
    """FGMRES on the strip-partitioned slab system (krylov.fgmres with comm).

    rhs: this rank's local (ghosted) device vector; its ghost entries are
    ignored.  Operator: x halo exchange + owner-computes Jacobian; mass: halo +
    (tau w (x) M); preconditioner (optional): `vanka_steps` distributed Vanka
    steps from zero (patches of the owned cells, increments reverse-added).
    Every Krylov vector keeps zero ghost entries, so local Euclidean products
    are owned-only and one allreduce makes them global.  Returns the
    FgmresResult with x local (ghosts zero)."""
    import torch

    from .krylov import fgmres
    from .operators import MassNorm

    k1 = rank.k1
    dev = rank.jac.dev
    device = torch.device("cuda", dev.device)
    mask = owned_mask(rank.lay, k1, device)
    mass = MassNorm(rank.ctx, dev=dev)
    tmp = torch.empty(k1 * rank.lay.nd_loc, dtype=torch.float64, device=device)

    def op(v, out=None):
        tmp.copy_(v)
        transport.exchange([tmp], "halo_recv", k1)
        y = rank.jac.matvec(tmp, out=out)
        y.mul_(mask)
        return y

    class _Mass:
        def apply_into(self, v, out):
            tmp.copy_(v)
            transport.exchange([tmp], "halo_recv", k1)
            mass.apply_into(tmp, out)
            out.mul_(mask)
            return out

    precond = None
    if vanka_steps > 0:
        if rank.level is None:
            rank.build_patches()

        def precond(v, out=None):
            d = torch.zeros_like(v)
            r = v.clone()
            transport.exchange([r], "halo_recv", k1)
            for _ in range(vanka_steps):
                distributed_vanka_step([rank], [d], [r], omega, transport)
            d.mul_(mask)
            if out is not None:
                out.copy_(d)
                return out
            return d

    op.dev = dev
    b = (rhs if isinstance(rhs, torch.Tensor) else torch.as_tensor(rhs, device=device)).reshape(-1) * mask
    return fgmres(op, b, tol, config, precond=precond, mass=_Mass(), x0=x0, comm=comm)
