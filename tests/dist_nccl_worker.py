"""One rank of the 2-GPU NCCL parity test (tests/test_gpu_dist_nccl.py),
launched by torch.distributed.run: the strip-partitioned Jacobian apply and
Vanka step over NCCL point-to-point exchanges between two GPUs.
usage: dist_nccl_worker.py OUT_PREFIX"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def main():
    import numpy as np
    import torch
    import torch.distributed as dist

    from dist_krylov_worker import problem
    from paper_2603_28706_b200.partition import (DistributedSlab, StripPartition, TorchDistTransport,
                                                 distributed_apply_and_vanka_step)

    rank, ws, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    assert dist.get_backend() == "nccl"
    cfg, ctx, syn, var = problem()
    part = StripPartition(cfg.nx, cfg.ny, ws)
    tr = TorchDistTransport(part.layout(rank), part)
    rk = DistributedSlab(ctx, syn.U, var, part, rank, tr, device=local, surrogate=True, rep_fraction=cfg.rep_fraction)
    rk.build_patches()
    dev = torch.device("cuda", local)
    out = {"device": torch.cuda.current_device()}
    for tag in ("py", "lib"):  # torch.distributed exchanges, then libpdst's NCCL data plane
        if tag == "lib":
            rk.strip_setup()
            rk.attach_nccl()
        x = torch.as_tensor(rk.local(syn.x), device=dev)
        r = x.clone()
        d = torch.as_tensor(rk.local(syn.d0), device=dev)
        (y,) = distributed_apply_and_vanka_step([rk], [x], [d], [r], cfg.omega, tr)
        distributed_apply_and_vanka_step([rk], [x], [d], [r], cfg.omega, tr)  # a second step on the updated d
        torch.cuda.synchronize()
        yg, dg = np.zeros(syn.x.size), np.zeros(syn.x.size)
        rk.owned_into(y.cpu().numpy(), yg)
        rk.owned_into(d.cpu().numpy(), dg)
        out[f"y_{tag}"], out[f"d_{tag}"] = yg, dg
    np.savez(f"{sys.argv[1]}{rank}.npz", **out)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
