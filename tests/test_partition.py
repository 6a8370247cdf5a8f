"""CPU tests of the strip partition: ownership, local <-> global maps and the
halo / defect / increment exchanges, in one process (LocalTransport) and over
torch.distributed gloo with world_size 2 (TorchDistTransport)."""

import os

import numpy as np
import pytest

from paper_2603_28706_b200.partition import LocalTransport, StripPartition, strip_bounds


@pytest.mark.parametrize("nx,ny,P", [(5, 4, 2), (6, 9, 3), (3, 17, 4), (8, 16, 8)])
def test_ownership_is_a_partition(nx, ny, P):
    part = StripPartition(nx, ny, P)
    lay0 = part.layout(0)
    nd = lay0.nd
    seen = np.zeros(nd, dtype=int)
    for r in range(P):
        lay = part.layout(r)
        ids = np.arange(nd, dtype=np.int64)
        loc = lay.to_local(ids)
        tmp = np.full(nd, -1, dtype=np.int64)
        lay.owned_into_global(loc, tmp)
        seen[tmp >= 0] += 1
        assert np.array_equal(tmp[tmp >= 0], np.flatnonzero(tmp >= 0))  # owned entries are the right ids
        # the local mesh is the strip + 2 ghost rows on each side
        assert lay.c_lo == max(0, lay.a - 2) and lay.c_hi == min(ny, lay.b + 2)
    assert (seen == 1).all()


def test_strip_bounds_validation():
    assert strip_bounds(8, 4) == [(0, 2), (2, 4), (4, 6), (6, 8)]
    with pytest.raises(ValueError):
        strip_bounds(7, 4)


@pytest.mark.parametrize("nx,ny,P,k1", [(4, 8, 2, 2), (3, 13, 3, 1), (5, 12, 4, 3)])
def test_local_transport_halo_and_increments(nx, ny, P, k1):
    part = StripPartition(nx, ny, P)
    lays = [part.layout(r) for r in range(P)]
    nd = lays[0].nd
    gid = np.arange(k1 * nd, dtype=float)
    # every rank fills only its OWNED entries with the global ids, ghosts with -1
    vecs = []
    for lay in lays:
        loc = np.concatenate([lay.to_local(gid[mu * nd:(mu + 1) * nd]) for mu in range(k1)])
        mask = np.concatenate([lay.to_local(_owned_mask(lay, nd)) for _ in range(k1)])
        loc[mask == 0] = -1.0
        vecs.append(loc)
    tr = LocalTransport(lays)
    tr.exchange(vecs, "halo_recv", k1)
    for lay, v in zip(lays, vecs):
        ref = np.concatenate([lay.to_local(gid[mu * nd:(mu + 1) * nd]) for mu in range(k1)])
        # everything the operator needs (all local nodes, pressure of cells below the strip) is now valid
        ndl = lay.nd_loc
        for mu in range(k1):
            blk, rb = v[mu * ndl:(mu + 1) * ndl], ref[mu * ndl:(mu + 1) * ndl]
            vel = lay.vel_slice_local(2 * lay.c_lo, min(2 * lay.b + 3, 2 * lay.c_hi + 1))
            assert np.array_equal(blk[vel], rb[vel])
            need = lay.prs_slice_local(lay.c_lo, lay.b)
            assert np.array_equal(blk[need], rb[need])
    # increment reverse-add: rank r-1's contribution lands on rank r's row 2a
    incs = [np.ones(lay.nd_loc * k1) for lay in lays]
    tr.exchange(incs, "inc_recv", k1, add=True)
    for r, (lay, inc) in enumerate(zip(lays, incs)):
        sl = lay.vel_slice_local(2 * lay.a, 2 * lay.a + 1)
        expect = 2.0 if r > 0 else 1.0
        assert np.all(inc[: lay.nd_loc][sl] == expect)


def _owned_mask(lay, nd):
    m = np.zeros(nd)
    lay.owned_into_global(np.ones(lay.nd_loc), m)
    return m


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2603_28706_b200.partition import StripPartition, TorchDistTransport

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nx, ny, k1 = 4, 9, 2
        part = StripPartition(nx, ny, world)
        lay = part.layout(rank)
        nd = lay.nd
        gid = np.arange(k1 * nd, dtype=float)
        loc = np.concatenate([lay.to_local(gid[mu * nd:(mu + 1) * nd]) for mu in range(k1)])
        owned = np.concatenate([lay.to_local(_owned_mask(lay, nd)) for _ in range(k1)])
        ref = loc.copy()
        loc[owned == 0] = -1.0
        t = torch.tensor(loc)
        TorchDistTransport(lay, part).exchange(t, "halo_recv", k1)
        ok = True
        ndl = lay.nd_loc
        for mu in range(k1):
            blk, rb = t.numpy()[mu * ndl:(mu + 1) * ndl], ref[mu * ndl:(mu + 1) * ndl]
            vel = lay.vel_slice_local(2 * lay.c_lo, min(2 * lay.b + 3, 2 * lay.c_hi + 1))
            ok &= np.array_equal(blk[vel], rb[vel])
        inc = torch.ones(k1 * ndl, dtype=torch.float64)
        TorchDistTransport(lay, part).exchange(inc, "inc_recv", k1, add=True)
        sl = lay.vel_slice_local(2 * lay.a, 2 * lay.a + 1)
        ok &= bool((inc.numpy()[:ndl][sl] == (2.0 if rank > 0 else 1.0)).all())
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_exchange():
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}



@pytest.mark.parametrize("nx,ny,P,k1", [(4, 8, 2, 2), (5, 12, 3, 1), (3, 16, 4, 3)])
def test_owned_masks_partition_unity(nx, ny, P, k1):
    """The ranks' owned-dof masks (distributed FGMRES inner products) cover every
    global dof exactly once."""
    import torch

    from paper_2603_28706_b200.partition import StripPartition, owned_mask

    part = StripPartition(nx, ny, P)
    tot = np.zeros(k1 * part.layout(0).nd)
    for r in range(P):
        lay = part.layout(r)
        m = owned_mask(lay, k1).numpy()
        g = np.zeros(lay.nd)
        for mu in range(k1):
            lay.owned_into_global(m[mu * lay.nd_loc:(mu + 1) * lay.nd_loc], g)
            tot[mu * lay.nd:(mu + 1) * lay.nd] += g
            g[:] = 0.0
        assert m.sum() == k1 * (len(lay.owned_node_rows) * lay.nnx * 2 + 3 * nx * (lay.b - lay.a))
    assert np.array_equal(tot, np.ones_like(tot))


@pytest.mark.parametrize("nx,ny,P,levels", [(16, 32, 2, 3), (32, 32, 4, 3), (16, 48, 3, 3), (8, 64, 2, 4)])
def test_multilevel_layouts(nx, ny, P, levels):
    """Strips aligned with the coarsest cells: on every level the owned node rows
    partition the level's node rows, every local mesh keeps >= 2 ghost rows
    towards each neighbour (exactly 2 on the coarsest level), level f+1 is level
    f halved, and every halo / defect / increment slice lies in the peer's owned
    rows (bit-exact index maps: the distributed V-cycle's exchange plans)."""
    from paper_2603_28706_b200.partition import StripPartition, ghost_rows

    part = StripPartition(nx, ny, P, levels=levels)
    assert part.ghost == ghost_rows(levels) == 2 ** levels
    for f in range(levels):
        lays = [part.layout(r).level(f) for r in range(P)]
        nyf = ny >> f
        covered = np.zeros(2 * nyf + 1, int)
        for lay in lays:
            assert lay.ny == nyf and lay.nx == nx >> f and lay.f == f
            covered[list(lay.owned_node_rows)] += 1
            if lay.rank > 0:
                assert lay.a - lay.c_lo >= 2
            if not lay.last:
                assert lay.c_hi - lay.b >= 2
            if f == levels - 1:
                assert lay.rank == 0 or lay.a - lay.c_lo == 2
            if f + 1 < levels:
                nxt = part.layout(lay.rank).level(f + 1)
                assert (nxt.a, nxt.b, nxt.c_lo, nxt.c_hi) == (lay.a // 2, lay.b // 2, lay.c_lo // 2, lay.c_hi // 2)
                assert lay.a % 2 == 0 and lay.c_lo % 2 == 0
            for plan in ("halo_recv", "defect_recv", "inc_recv"):
                for peer, mine, theirs in getattr(lay, plan)():
                    pl = lays[peer]
                    own = pl.owned_node_rows
                    # the peer's slice, in global node rows / cell rows
                    if theirs.start < pl.mv_loc:
                        y0 = theirs.start // (2 * pl.nnx) + 2 * pl.c_lo
                        y1 = theirs.stop // (2 * pl.nnx) + 2 * pl.c_lo
                        if plan == "inc_recv":  # the peer's contribution to my first owned row
                            assert (y0, y1) == (2 * lay.a, 2 * lay.a + 1) and y0 < 2 * pl.c_hi + 1
                        else:
                            assert own.start <= y0 and y1 <= own.stop, (f, plan, lay.rank, peer)
                        assert mine.stop - mine.start == theirs.stop - theirs.start
                    else:
                        j0 = (theirs.start - pl.mv_loc) // (3 * pl.nx) + pl.c_lo
                        j1 = (theirs.stop - pl.mv_loc) // (3 * pl.nx) + pl.c_lo
                        assert pl.a <= j0 and j1 <= pl.b
        assert np.array_equal(covered, np.ones_like(covered))


def test_multilevel_alignment_validation():
    from paper_2603_28706_b200.partition import StripPartition

    with pytest.raises(ValueError):
        StripPartition(16, 30, 2, levels=3)  # 30 rows are not a multiple of 4
    with pytest.raises(ValueError):
        StripPartition(16, 16, 3, levels=3)  # 4 coarse rows cannot give 3 strips of >= 2
    with pytest.raises(ValueError):
        StripPartition(16, 32, 2, levels=3).layout(0).level(3)


def test_gloo_world2_coarse_level_exchange():
    """The TorchDistTransport plans on a coarse level, two processes over gloo:
    the same result as the in-process LocalTransport."""
    import torch.multiprocessing as mp

    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    mp.spawn(_coarse_worker, args=(2, port), nprocs=2, join=True)


def _coarse_worker(rank, world, port):
    import os

    import torch
    import torch.distributed as dist

    from paper_2603_28706_b200.partition import LocalTransport, StripPartition, TorchDistTransport

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        part = StripPartition(8, 32, world, levels=3)
        k1, f = 2, 1
        lays = [part.layout(r).level(f) for r in range(world)]
        gen = torch.Generator().manual_seed(5)
        vecs = [torch.randn(k1 * l.nd_loc, generator=gen, dtype=torch.float64) for l in lays]
        for plan, add in (("halo_recv", False), ("defect_recv", False), ("inc_recv", True)):
            ref = [v.clone() for v in vecs]
            LocalTransport([part.layout(r) for r in range(world)]).exchange(ref, plan, k1, add=add, level=f)
            mine = vecs[rank].clone()
            TorchDistTransport(part.layout(rank), part).exchange(mine, plan, k1, add=add, level=f)
            assert torch.equal(mine, ref[rank]), plan
        # two independent exchanges in one grouped send/recv (finest level)
        lays0 = [part.layout(r) for r in range(world)]
        a = [torch.randn(k1 * l.nd_loc, generator=gen, dtype=torch.float64) for l in lays0]
        b = [torch.randn(k1 * l.nd_loc, generator=gen, dtype=torch.float64) for l in lays0]
        ra, rb = [v.clone() for v in a], [v.clone() for v in b]
        lt = LocalTransport(lays0)
        lt.exchange(ra, "halo_recv", k1)
        lt.exchange(rb, "inc_recv", k1, add=True)
        ma, mb = a[rank].clone(), b[rank].clone()
        TorchDistTransport(part.layout(rank), part).exchange_many([(ma, "halo_recv", False), (mb, "inc_recv", True)], k1)
        assert torch.equal(ma, ra[rank]) and torch.equal(mb, rb[rank])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("nx,ny,P,levels", [(16, 32, 2, 3), (16, 48, 3, 3), (8, 64, 4, 3)])
def test_deep_halo_plan(nx, ny, P, levels):
    """The state halo of a multigrid partition: every ghost row of every local
    mesh comes from the neighbour that owns it, and together with the owned
    rows the local slab is exactly the global slab restricted to the local mesh."""
    from paper_2603_28706_b200.partition import LocalTransport, StripPartition

    part = StripPartition(nx, ny, P, levels=levels)
    lays = [part.layout(r) for r in range(P)]
    rng = np.random.default_rng(1)
    k1 = 2
    xg = rng.standard_normal(k1 * lays[0].nd)
    nd = lays[0].nd
    vecs = []
    for lay in lays:  # owned entries right, ghosts garbage
        own = np.zeros(nd)
        lay.owned_into_global(np.ones(lay.nd_loc), own)
        v = np.concatenate([np.where(lay.to_local(own) > 0, lay.to_local(xg[mu * nd:(mu + 1) * nd]), 1e9)
                            for mu in range(k1)])
        vecs.append(v)
    LocalTransport(lays).exchange(vecs, "deep_halo_recv", k1)
    for lay, v in zip(lays, vecs):
        ref = np.concatenate([lay.to_local(xg[mu * nd:(mu + 1) * nd]) for mu in range(k1)])
        assert np.array_equal(v, ref)


def test_deep_halo_needs_thick_strips():
    from paper_2603_28706_b200.partition import StripPartition

    part = StripPartition(16, 32, 4, levels=3)  # strips of 8 rows, 8 ghost rows: the top one reaches 2 ranks up
    with pytest.raises(ValueError):
        for r in range(4):
            part.layout(r).deep_halo_recv()
