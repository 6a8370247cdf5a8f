"""bench.py's launcher contract on a machine without enough GPUs: `--gpus N`
outside torchrun must refuse loudly (exit 2, a message naming N) instead of
silently timing one GPU, and WORLD_SIZE must agree with --gpus."""

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.update(env or {})
    e["CUDA_VISIBLE_DEVICES"] = ""
    return subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, env=e, capture_output=True, text=True,
                          timeout=300)


def test_gpus_n_without_devices_fails_loudly():
    r = _run(["--gpus", "4", "--steps", "3"])
    assert r.returncode == 2
    assert "--gpus 4" in r.stderr and "0 CUDA device" in r.stderr


def test_world_size_must_match_gpus():
    r = _run(["--gpus", "2"], env={"WORLD_SIZE": "4", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2 and "WORLD_SIZE=4" in r.stderr
