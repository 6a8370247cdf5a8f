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
