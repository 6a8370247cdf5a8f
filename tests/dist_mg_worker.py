"""One rank of the two-process distributed multigrid test (tests/test_gpu_dist_mg.py):
TorchDistTransport + DistComm over gloo, one process per rank.
usage: dist_mg_worker.py RANK WORLD PORT OUT"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def problem():
    import dataclasses

    from paper_2603_28706_b200 import problem as pb
    from paper_2603_28706_b200.stmg import MgConfig
    from paper_2603_28706_b200.synth import CONFIGS, make_slab_inputs

    cfg = dataclasses.replace(CONFIGS["cfg1"], nx=16, ny=32)
    params = pb.ModelParams(cfg.p, cfg.delta, cfg.nu, cfg.nu_inf)
    conf = pb.DiscretizationConfig(cfg.gamma1, cfg.gamma2, cfg.gamma_cip)
    syn = make_slab_inputs(cfg)
    ctx = pb.make_context(cfg.nx, cfg.ny, cfg.k, params, cfg.tau, config=conf, v_minus=syn.v_minus)
    mg = MgConfig(min_cells=4, omega=cfg.omega, coarse_solver="fgmres", coarse_iters=12, coarse_rtol=1e-10,
                  rep_fraction=cfg.rep_fraction)
    return cfg, ctx, syn, pb.modified_newton(cfg.nu), mg


def main():
    rank, ws, port, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=port)
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2603_28706_b200.dist_mg import DistributedStmg, distributed_fgmres_mg, distributed_vcycle, global_levels
    from paper_2603_28706_b200.krylov import KrylovConfig
    from paper_2603_28706_b200.partition import DistComm, StripPartition, TorchDistTransport

    dist.init_process_group("gloo", rank=rank, world_size=ws)
    cfg, ctx, syn, var, mg = problem()
    part = StripPartition(cfg.nx, cfg.ny, ws, levels=global_levels(cfg.nx, cfg.ny, mg.min_cells))
    tr = TorchDistTransport(part.layout(rank), part)
    rk = DistributedStmg(ctx, syn.U, var, part, rank, mg)
    nd = rk.lay.nd
    xl = torch.as_tensor(np.concatenate([rk.lay.to_local(syn.x[mu * nd:(mu + 1) * nd]) for mu in range(rk.k1)]),
                         device="cuda")
    (z,) = distributed_vcycle([rk], [xl], tr, DistComm())
    res = distributed_fgmres_mg([rk], tr, [xl], 1e-8, KrylovConfig(restart=20, max_iters=20), comm=DistComm())
    zg, xg = np.zeros(syn.x.size), np.zeros(syn.x.size)
    ndl = rk.lay.nd_loc
    for mu in range(rk.k1):
        rk.lay.owned_into_global(z.cpu().numpy()[mu * ndl:(mu + 1) * ndl], zg[mu * nd:(mu + 1) * nd])
        rk.lay.owned_into_global(res.x[0].cpu().numpy()[mu * ndl:(mu + 1) * ndl], xg[mu * nd:(mu + 1) * nd])
    np.savez(out, z=zg, x=xg, iters=res.iterations)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
