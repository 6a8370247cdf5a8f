"""CPU timing of the oracle port — TEST / BASELINE INFRASTRUCTURE ONLY.

Used by bench.py's ``cpu_baseline`` leg (single thread) and by its
``--impl reference`` arm (one worker process per host core).  A "step" is the
same unit as the GPU bench: one slab Jacobian apply plus one Vanka sweep,
here on a bounded sample mesh with the cfg2 parameters (building the sample's
patches is untimed setup, as in the GPU arm).

Run standalone:  python -m oracle.cpu_bench --n 64 --steps 5 [--procs P]
prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


class Sample:
    def __init__(self, n: int, seed_offset: int = 0):
        from dataclasses import replace

        from oracle import pdst_oracle as orc
        from paper_2603_28706_b200.radau import gauss_radau, temporal_matrices
        from paper_2603_28706_b200.synth import CONFIGS, make_slab_inputs

        cfg = replace(CONFIGS["cfg2"], nx=n, ny=n, seed=CONFIGS["cfg2"].seed + seed_offset)
        b = gauss_radau(cfg.k)
        tm = temporal_matrices(b)
        syn = make_slab_inputs(cfg, nodes=b.nodes)
        grid = orc.Grid(n, n, cfg.extents, None, cfg.gamma1, cfg.gamma2, cfg.gamma_cip)
        slab = orc.Slab(grid, orc.Params(cfg.p, cfg.delta, cfg.nu, cfg.nu_inf), cfg.k, b.nodes, b.weights, tm.K_t,
                        tm.m_t, cfg.tau, 0.0, syn.v_minus, None)
        variant = orc.Variant("modn", cfg.nu)
        t0 = time.perf_counter()
        self.pre = orc.StmgOracle(slab, syn.U, variant, omega=cfg.omega, surrogate=True,
                                  rep_fraction=cfg.rep_fraction, min_cells=n)
        self.build_s = time.perf_counter() - t0
        self.jac = self.pre.jac
        self.level = self.pre.levels[-1]
        self.syn = syn
        self.cfg = cfg
        self.orc = orc
        self.n_dof = syn.x.size

    def step(self):
        y = self.jac.matvec(self.syn.x)
        d = self.orc.vanka(self.level, self.syn.d0, self.syn.x, 1, self.cfg.omega)
        return float(y[0] + d[0])

    def timed(self, steps: int):
        t_apply = t_sweep = 0.0
        for _ in range(steps):
            t0 = time.perf_counter()
            self.jac.matvec(self.syn.x)
            t1 = time.perf_counter()
            self.orc.vanka(self.level, self.syn.d0, self.syn.x, 1, self.cfg.omega)
            t2 = time.perf_counter()
            t_apply += t1 - t0
            t_sweep += t2 - t1
        return t_apply / steps, t_sweep / steps


def single_thread(n: int, steps: int) -> dict:
    s = Sample(n)
    s.step()  # warm caches
    ta, ts = s.timed(steps)
    return {"n": n, "n_dof": s.n_dof, "steps": steps, "t_apply_s": ta, "t_sweep_s": ts,
            "gdofs": s.n_dof / (ta + ts) / 1e9, "build_s": s.build_s}


# -- multi-process arm ------------------------------------------------------
_S = None


def _init(n, off):
    global _S
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    _S = Sample(n, off)


def _work(_):
    t0 = time.perf_counter()
    _S.step()
    return time.perf_counter() - t0


def _worker(n, rank, q_in, q_out):
    _init(n, rank)
    q_out.put(("ready", _S.n_dof))
    while True:
        cmd = q_in.get()
        if cmd is None:
            return
        q_out.put(("done", _work(None)))


class Pool:
    """P worker processes, each owning one sample; step() runs one
    apply + sweep on every worker concurrently and returns the wall time."""

    def __init__(self, n: int, procs: int):
        ctx = mp.get_context("fork")
        self.qs = [ctx.Queue() for _ in range(procs)]
        self.out = ctx.Queue()
        self.ps = [ctx.Process(target=_worker, args=(n, r, self.qs[r], self.out), daemon=True) for r in range(procs)]
        for p in self.ps:
            p.start()
        self.n_dof = 0
        for _ in range(procs):
            kind, nd = self.out.get()
            self.n_dof = nd
        self.procs = procs

    def step(self) -> float:
        t0 = time.perf_counter()
        for q in self.qs:
            q.put(1)
        for _ in range(self.procs):
            self.out.get()
        return time.perf_counter() - t0

    def close(self):
        for q in self.qs:
            q.put(None)
        for p in self.ps:
            p.join(timeout=10)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--procs", type=int, default=1)
    a = ap.parse_args()
    if a.procs <= 1:
        print(json.dumps(single_thread(a.n, a.steps)))
    else:
        pool = Pool(a.n, a.procs)
        ts = [pool.step() for _ in range(a.steps)]
        pool.close()
        t = sum(ts) / len(ts)
        print(json.dumps({"n": a.n, "procs": a.procs, "t_step_s": t, "gdofs": a.procs * pool.n_dof / t / 1e9}))


if __name__ == "__main__":
    main()
