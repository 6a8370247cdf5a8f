"""One rank of the distributed-FGMRES parity test (tests/test_gpu_dist_krylov.py).
usage: dist_krylov_worker.py RANK WORLD PORT OUT VANKA_STEPS"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def problem():
    import dataclasses

    from paper_2603_28706_b200 import problem as pb
    from paper_2603_28706_b200.synth import CONFIGS, make_slab_inputs

    cfg = dataclasses.replace(CONFIGS["cfg1"], nx=12, ny=16)
    params = pb.ModelParams(cfg.p, cfg.delta, cfg.nu, cfg.nu_inf)
    conf = pb.DiscretizationConfig(cfg.gamma1, cfg.gamma2, cfg.gamma_cip)
    syn = make_slab_inputs(cfg)
    ctx = pb.make_context(cfg.nx, cfg.ny, cfg.k, params, cfg.tau, config=conf, v_minus=syn.v_minus)
    return cfg, ctx, syn, pb.modified_newton(cfg.nu)


def main():
    rank, ws, port, out, steps = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4], int(sys.argv[5])
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=port)
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2603_28706_b200.krylov import KrylovConfig
    from paper_2603_28706_b200.partition import (DistComm, DistributedSlab, StripPartition, TorchDistTransport,
                                                 distributed_fgmres)

    dist.init_process_group("gloo", rank=rank, world_size=ws)
    cfg, ctx, syn, var = problem()
    part = StripPartition(cfg.nx, cfg.ny, ws)
    tr = TorchDistTransport(part.layout(rank), part)
    rk = DistributedSlab(ctx, syn.U, var, part, rank, tr, device=0, surrogate=True, rep_fraction=cfg.rep_fraction)
    b = torch.as_tensor(rk.local(syn.x), device="cuda")
    res = distributed_fgmres(rk, tr, DistComm(), b, 1e-8, KrylovConfig(restart=15, max_iters=40), vanka_steps=steps,
                             omega=cfg.omega)
    xg = np.zeros(syn.x.size)
    rk.owned_into(res.x.cpu().numpy(), xg)
    np.savez(out, x=xg, iters=res.iterations, conv=res.converged, res=res.residual_norm)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
