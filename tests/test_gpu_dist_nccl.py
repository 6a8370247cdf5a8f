"""Two GPUs, two processes, NCCL: the strip-partitioned apply + Vanka steps
(partition.TorchDistTransport over NCCL send/recv) equal the single-domain
apply and sweeps (relative 1e-13), and `bench.py --gpus 2` launches two ranks
itself and reports n_gpus = 2.  Skipped when fewer than two GPUs are visible
(the 1-GPU boxes of this pool); the same exchanges are covered on one GPU by
tests/test_gpu_partition.py (virtual ranks) and on CPU by the gloo tests in
tests/test_partition.py."""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def _two_gpus():
    try:
        import torch

        return torch.cuda.device_count() >= 2
    except Exception:
        return False


needs2 = pytest.mark.skipif(not _two_gpus(), reason="needs two CUDA devices")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return str(p)


@needs2
def test_nccl_two_ranks_match_single_domain(tmp_path):
    import torch

    sys.path.insert(0, HERE)
    from dist_krylov_worker import problem

    from paper_2603_28706_b200.operators import SlabJacobian
    from paper_2603_28706_b200.smoother import VankaLevel

    prefix = str(tmp_path / "r")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", _port(), os.path.join(HERE, "dist_nccl_worker.py"), prefix]
    res = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-3000:]
    parts = [np.load(f"{prefix}{r}.npz") for r in range(2)]
    assert int(parts[0]["device"]) != int(parts[1]["device"])
    cases = []
    for tag in ("py", "lib"):  # torch.distributed exchanges; libpdst's NCCL data plane (pdst_strip_step)
        y = parts[0][f"y_{tag}"] + parts[1][f"y_{tag}"]  # owned dofs are disjoint
        d = parts[0][f"d_{tag}"] + parts[1][f"d_{tag}"]
        cases.append((tag, y, d))
    cfg, ctx, syn, var = problem()
    U = torch.as_tensor(syn.U, device="cuda")
    jac = SlabJacobian(ctx, U, var)
    lvl = VankaLevel(ctx, U, var, surrogate=True, rep_fraction=cfg.rep_fraction, jac=jac)
    x = torch.as_tensor(syn.x, device="cuda")
    y_ref = jac.matvec(x).cpu().numpy()
    d_ref = lvl.smooth(torch.as_tensor(syn.d0, device="cuda"), x, 2, cfg.omega).cpu().numpy()
    for tag, y, d in cases:
        for a, b, what in ((y, y_ref, "apply"), (d, d_ref, "2 Vanka steps")):
            e = np.linalg.norm(a - b) / np.linalg.norm(b)
            assert e <= 1e-13, f"{tag} {what}: rel err {e:.3e}"


@needs2
def test_bench_launches_its_own_ranks():
    res = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3",
                          "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True, timeout=1200)
    assert res.returncode == 0, res.stderr[-3000:]
    line = json.loads(res.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["value"] > 0
