"""Distributed FGMRES (strip partition, allreduced M-inner products, SURVEY.md
§8e) against the single-domain FGMRES on the same seeded problem: two ranks as
two processes on the one GPU, gloo staged through the host (the kernels do not
wait on each other; NCCL carries the same calls between GPUs)."""

import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("steps", [0, 1])
def test_distributed_fgmres_matches_single_domain(tmp_path, steps):
    import torch

    sys.path.insert(0, HERE)
    from dist_krylov_worker import problem

    from paper_2603_28706_b200.krylov import KrylovConfig, fgmres
    from paper_2603_28706_b200.operators import MassNorm, SlabJacobian
    from paper_2603_28706_b200.smoother import VankaLevel

    port = str(_port())
    outs = [str(tmp_path / f"r{r}.npz") for r in range(2)]
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "dist_krylov_worker.py"), str(r), "2", port,
                               outs[r], str(steps)]) for r in range(2)]
    codes = [p.wait(timeout=600) for p in procs]
    assert codes == [0, 0], codes
    parts = [np.load(o) for o in outs]
    x_dist = parts[0]["x"] + parts[1]["x"]  # owned dofs are disjoint

    cfg, ctx, syn, var = problem()
    U = torch.as_tensor(syn.U, device="cuda")
    jac = SlabJacobian(ctx, U, var)
    pre = None
    if steps:
        lvl = VankaLevel(ctx, U, var, surrogate=True, rep_fraction=cfg.rep_fraction, jac=jac)

        def pre(v):
            return lvl.smooth(torch.zeros_like(v), v, steps, cfg.omega)

    res = fgmres(jac.matvec, torch.as_tensor(syn.x, device="cuda"), 1e-8, KrylovConfig(restart=15, max_iters=40),
                 precond=pre, mass=MassNorm(ctx, dev=jac.dev))
    x = res.x.cpu().numpy()
    assert int(parts[0]["iters"]) == int(parts[1]["iters"]) == res.iterations
    assert bool(parts[0]["conv"]) == res.converged
    err = np.linalg.norm(x_dist - x) / np.linalg.norm(x)
    assert err <= 1e-9, err
