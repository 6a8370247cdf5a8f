"""Benchmark of the B200 slab hot path.

Workload (BASELINE.json configs[1], "cfg2"): 256x256 Q2/P1disc, DG(1) with 2
right-Radau points, fp64, p=1.3, delta=1e-3, nu=1, nu_inf=0, modified-Newton
tangent (sigma_max = nu), surrogate Vanka patches frozen at the last Radau
point, omega = 0.7.  N_dof = 1,445,892.

One step = one matrix-free slab Jacobian apply (y = J x) + one Vanka sweep
(d <- d + omega sum_K R_K' A_K^-1 R_K (r - J d)) on device-resident vectors.
metric = GDoF/s = N_dof x ranks / (time per step).  L2 is flushed (256 MiB
write) between timed steps, outside the events.

  python bench.py [--gpus N --steps K --warmup W]      our arm (one JSON line)
  python bench.py --impl reference ...                  CPU reference arm (oracle port)

Multi-GPU (torchrun, N > 1): weak scaling over the strip partition
(partition.py).  The global mesh is nx x (N ny) on [0,1]x[0,N]
(same h as cfg2), rank r owns cell rows [r ny, (r+1) ny) plus two ghost rows per
side; a step is the distributed apply + Vanka step with the three NCCL
point-to-point exchanges (x halo, defect row, increment reverse-add).
``--virtual-ranks P`` runs the same partitioned step with P ranks on one GPU
(LocalTransport) to exercise the path without NCCL.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "GDoF/s of matrix-free space-time Jacobian apply + Vanka sweep; HBM % of peak"
UNIT = "GDoF/s"
CPU_SAMPLE_N = 64


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = sorted(float(r[0]) for r in rows if r[0].replace(".", "").isdigit())
        mx = max(float(r[1]) for r in rows if r[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_baseline_single(steps=6):
    env = dict(os.environ, OPENBLAS_NUM_THREADS="1", OMP_NUM_THREADS="1", MKL_NUM_THREADS="1")
    out = subprocess.run([sys.executable, "-m", "oracle.cpu_bench", "--n", str(CPU_SAMPLE_N), "--steps", str(steps)],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    if out.returncode != 0:
        return {"value": None, "unit": UNIT, "cores": 1, "kind": "port", "sample": "failed: " + out.stderr[-300:]}
    r = json.loads(out.stdout.strip().splitlines()[-1])
    return {"value": r["gdofs"], "unit": UNIT, "cores": 1, "kind": "port",
            "sample": (f"oracle/pdst_oracle.py (numpy restatement of pdflow) on a {CPU_SAMPLE_N}x{CPU_SAMPLE_N} "
                       f"mesh with the cfg2 parameters (N_dof={r['n_dof']}), {steps} x (apply + sweep), 1 thread; "
                       f"apply {r['t_apply_s']:.3f} s, sweep {r['t_sweep_s']:.3f} s"),
            "t_apply_s": r["t_apply_s"], "t_sweep_s": r["t_sweep_s"]}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    procs = max(1, min(os.cpu_count() or 1, 64))
    from oracle.cpu_bench import Pool

    t0 = time.time()
    pool = Pool(CPU_SAMPLE_N, procs)
    build = time.time() - t0
    for _ in range(args.warmup):
        pool.step()
    ts = [pool.step() for _ in range(args.steps)]
    pool.close()
    t = sum(ts) / len(ts)
    value = procs * pool.n_dof / t / 1e9
    sample = (f"{procs} worker processes (all host threads, one numpy oracle each) on {CPU_SAMPLE_N}x{CPU_SAMPLE_N} "
              f"cfg2-parameter samples (N_dof={pool.n_dof} each); step = apply + sweep on every worker; "
              f"wall time per step {t:.3f} s; untimed patch build {build:.1f} s")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded modal state, SURVEY.md §8d)",
            "impl": "reference",
            "config": {"workload": "cfg2 parameters on bounded CPU samples", "sample_mesh": CPU_SAMPLE_N,
                       "parallelism": f"{procs} processes"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_distributed(args):
    """Strip-partitioned step (weak scaling); see the module docstring."""
    import dataclasses

    import numpy as np
    import torch

    from paper_2603_28706_b200 import _lib as L
    from paper_2603_28706_b200 import problem as pb
    from paper_2603_28706_b200.partition import (DistributedSlab, LocalTransport, StripPartition,
                                                 TorchDistTransport, distributed_apply_and_vanka_step)
    from paper_2603_28706_b200.synth import CONFIGS, make_slab_inputs

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    P = ws if ws > 1 else args.virtual_ranks
    base = CONFIGS[args.config]
    # weak scaling (default): cfg's rows per rank; --strong: cfg's mesh in P strips
    cfg = base if args.strong else dataclasses.replace(base, ny=base.ny * P, extents=(0.0, 0.0, 1.0, float(P)))
    params = pb.ModelParams(cfg.p, cfg.delta, cfg.nu, cfg.nu_inf)
    conf = pb.DiscretizationConfig(cfg.gamma1, cfg.gamma2, cfg.gamma_cip)
    syn = make_slab_inputs(cfg)
    ctx = pb.make_context(cfg.nx, cfg.ny, cfg.k, params, cfg.tau, extents=cfg.extents, config=conf,
                          v_minus=syn.v_minus)
    variant = pb.modified_newton(cfg.nu)
    dev = torch.device("cuda", local)
    part = StripPartition(cfg.nx, cfg.ny, P)
    mine = [rank] if ws > 1 else list(range(P))
    if ws > 1:
        transport = TorchDistTransport(part.layout(rank), part)
    else:
        transport = LocalTransport([part.layout(r) for r in range(P)])
    t_setup = time.time()
    ranks = [DistributedSlab(ctx, syn.U, variant, part, r, transport, device=local, rep_fraction=cfg.rep_fraction)
             for r in mine]
    for rk in ranks:
        rk.build_patches()
        rk.strip_setup()  # the data plane inside libpdst (pdst_strip_step / pdst_strips_step_local)
        if ws > 1:
            rk.attach_nccl()  # torch.distributed's NCCL communicator, used by libpdst's exchanges
    torch.cuda.synchronize()
    t_setup = time.time() - t_setup
    xs = [torch.as_tensor(rk.local(syn.x), device=dev) for rk in ranks]
    rs = [x.clone() for x in xs]
    ds = [torch.as_tensor(rk.local(syn.d0), device=dev) for rk in ranks]
    N = syn.x.size
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)

    def step():
        distributed_apply_and_vanka_step(ranks, xs, ds, rs, cfg.omega, transport)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    t_end = time.time() + 1.2
    while time.time() < t_end:
        step()
        torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    n_launch0 = L.lib().pdst_launch_count()
    for i in range(args.steps):
        flush_l2(flush, i)
        ev[i][0].record()
        step()
        ev[i][1].record()
    torch.cuda.synchronize()
    n_launches = L.lib().pdst_launch_count() - n_launch0
    if dist is not None:
        dist.barrier()
    clk = clocks.stop()
    t_step = sum(a.elapsed_time(b) for a, b in ev) / args.steps / 1e3
    if dist is not None:
        tt = torch.tensor([t_step], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step = float(tt.item())
    value = N / t_step / 1e9

    # e2e: owned inputs from pinned host memory, results back to the host, every step
    hx = [torch.empty(x.shape, dtype=torch.float64, pin_memory=True) for x in xs]
    hd = [torch.empty(x.shape, dtype=torch.float64, pin_memory=True) for x in ds]
    for h, x in zip(hx, xs):
        h.copy_(x)
    for h, d in zip(hd, ds):
        h.copy_(d)
    hy = [torch.empty_like(h) for h in hx]

    def step_host():
        for h, x, r in zip(hx, xs, rs):
            x.copy_(h, non_blocking=True)
            r.copy_(h, non_blocking=True)
        for h, d in zip(hd, ds):
            d.copy_(h, non_blocking=True)
        ys = distributed_apply_and_vanka_step(ranks, xs, ds, rs, cfg.omega, transport)
        for h, y in zip(hy, ys):
            h.copy_(y, non_blocking=True)
        for h, d in zip(hd, ds):
            h.copy_(d, non_blocking=True)
        torch.cuda.synchronize()

    for _ in range(2):
        step_host()
    if dist is not None:
        dist.barrier()
    n_e2e = max(3, args.steps)  # the K timed steps (pipeline fill and drain included)
    t0 = time.perf_counter()
    for _ in range(n_e2e):
        step_host()
    t_e2e = (time.perf_counter() - t0) / n_e2e
    if dist is not None:
        tt = torch.tensor([t_e2e], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_e2e = float(tt.item())
    nloc = sum(x.numel() for x in xs)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "strong" if args.strong else "weak",
        "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded 16-mode modal state + 1e-3 noise, SURVEY.md §8d; no dataset)",
        "config": {"workload": f"{base.name} strips: {cfg.nx}x{cfg.ny} global mesh on [0,1]x[0,{cfg.extents[3]:g}], "
                               f"{cfg.ny // P} cell rows per rank + 2 ghost rows per side, DG({cfg.k}), modN, "
                               f"surrogate patches, omega={cfg.omega}",
                   "n_dof": N, "step": "distributed Jacobian apply + Vanka step inside libpdst (pdst_strip_step: "
                                       "x / d halos, defect row and increment reverse-add as pack -> NCCL "
                                       "send/recv (or in-process copy) -> unpack kernels, fused owned-row Vanka "
                                       "update; one stream, no host synchronization)",
                   "l2": "flushed between timed steps (256 MiB write, then a 256 MiB read of another buffer so no dirty lines remain; outside events)",
                   "parallelism": (f"strip partition x{ws} over NCCL send/recv (libpdst, torch's communicator)"
                                   if ws > 1 else f"{P} virtual ranks on one GPU (pdst_strips_step_local)")},
        "gpu_launches": n_launches,
        "setup_s": t_setup,
        "clocks": clk,
        "e2e": {"value": N / t_e2e / 1e9, "unit": UNIT, "h2d_bytes_per_step": 3 * 8 * nloc,
                "d2h_bytes_per_step": 2 * 8 * nloc, "ms_per_step": t_e2e * 1e3,
                "note": "per rank: pinned host x, r, d -> device, partitioned step, y and d -> host; wall clock"},
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def run_ours(args):
    import numpy as np
    import torch

    ws, rank, local = dist_env()
    if ws > 1 or args.virtual_ranks > 1:
        return run_distributed(args)
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2603_28706_b200 import _lib as L
    from paper_2603_28706_b200 import problem as pb
    from paper_2603_28706_b200.operators import SlabJacobian
    from paper_2603_28706_b200.smoother import VankaLevel
    from paper_2603_28706_b200.synth import CONFIGS, make_slab_inputs

    cfg = CONFIGS[args.config]
    params = pb.ModelParams(cfg.p, cfg.delta, cfg.nu, cfg.nu_inf)
    conf = pb.DiscretizationConfig(cfg.gamma1, cfg.gamma2, cfg.gamma_cip)
    syn = make_slab_inputs(cfg)
    ctx = pb.make_context(cfg.nx, cfg.ny, cfg.k, params, cfg.tau, config=conf, v_minus=syn.v_minus)
    variant = pb.modified_newton(cfg.nu)
    dev = torch.device("cuda", local)
    U = torch.as_tensor(syn.U, device=dev)
    x = torch.as_tensor(syn.x, device=dev)
    r = x.clone()
    d0 = torch.as_tensor(syn.d0, device=dev)
    d = d0.clone()
    y = torch.empty_like(x)
    t_setup = time.time()
    jac = SlabJacobian(ctx, U, variant, device=local)
    lvl = VankaLevel(ctx, U, variant, surrogate=True, rep_fraction=cfg.rep_fraction, jac=jac)
    torch.cuda.synchronize()
    t_setup = time.time() - t_setup
    N = x.numel()
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)

    def step():
        jac.matvec(x, out=y)
        lvl.smooth(d, r, 1, cfg.omega, inplace=True)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    # clocks are sampled while the GPU is kept busy around the timed region
    clocks = ClockSampler(local)
    clocks.start()
    t_end = time.time() + 1.2
    while time.time() < t_end:
        step()
        torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    n_launch0 = L.lib().pdst_launch_count()
    for i in range(args.steps):
        flush_l2(flush, i)
        ev[i][0].record()
        step()
        ev[i][1].record()
    torch.cuda.synchronize()
    n_launches = L.lib().pdst_launch_count() - n_launch0
    if ws > 1:
        torch.distributed.barrier()
    t_end = time.time() + 0.4
    while time.time() < t_end:
        step()
        torch.cuda.synchronize()
    clk = clocks.stop()
    t_step = sum(a.elapsed_time(b) for a, b in ev) / args.steps / 1e3  # seconds
    if ws > 1:
        tt = torch.tensor([t_step], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_step = float(tt.item())
    value = ws * N / t_step / 1e9

    # -- per-kernel times (CUDA events inside libpdst, same stream) ---------
    h = jac.dev.h
    L.lib().pdst_profile(h, 1)
    nprof = max(3, min(args.steps, 20))
    for i in range(nprof):
        flush_l2(flush, i)
        step()
    torch.cuda.synchronize()
    kt = {}
    # class 0: the Jacobian apply y = J x; class 6: the sweep's defect apply y = r - J x (same kernels + rhs)
    for kid, name in ((0, "jacobian"), (1, "vanka_gemv"), (2, "vanka_scatter"), (6, "jacobian_defect")):
        ms, cnt = L.C.c_double(), L.C.c_int64()
        L.lib().pdst_profile_read(h, kid, L.C.byref(ms), L.C.byref(cnt))
        kt[name] = (ms.value / max(cnt.value, 1), cnt.value)
    L.lib().pdst_profile(h, 0)
    # the apply as a Krylov loop sees it: back to back on one stream, no flush (x and y stay in L2, the
    # 141 MB coefficient stream does not fit it), PDL overlap between consecutive applies
    nb2b = 50
    for _ in range(3):
        jac.matvec(x, out=y)
    eb0, eb1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    eb0.record()
    for _ in range(nb2b):
        jac.matvec(x, out=y)
    eb1.record()
    torch.cuda.synchronize()
    t_b2b = eb0.elapsed_time(eb1) / nb2b * 1e-3

    nc, k1 = cfg.nx * cfg.ny, cfg.k + 1
    D = 21 * k1
    nd = ctx.disc.ndof
    mv = ctx.disc.n_velocity
    nbf = 2 * (cfg.nx + cfg.ny)
    # algorithmic bytes
    _, nblk, bpp = lvl.patch_info()
    b_gemv = float(nc * bpp) + 8.0 * (N + nc * D)  # patch inverses (diagonalized if nblk) + defect + update
    # x, y, the coefficient stream (108 doubles per cell and Radau node) and the side matrices
    b_apply_ours = 8.0 * (2 * N + 108 * k1 * nc + 441 * k1 * nbf)
    b_apply_ref = 8.0 * k1 * (2 * nd + 112 * nc + 56 * nbf + 4 * (2 * cfg.nx * (cfg.nx - 1)))
    # SURVEY §8d's minimal variant: state only (coefficients recomputed per apply)
    b_apply_min = 8.0 * k1 * (2 * nd + mv)
    peak, peak_kind = _peaks()
    t_gemv = kt["vanka_gemv"][0] * 1e-3
    t_jac = kt["jacobian"][0] * 1e-3
    ach = b_gemv / t_gemv / 1e9
    traffic = traffic_apply = None
    import glob

    # dram bytes per launch, one ncu capture per config (scripts/ncu_traffic.py): the latest round's file,
    # profiles/traffic_rNN.json for cfg2 and profiles/traffic_<config>_rNN.json for the others
    pat = "traffic_r*.json" if args.config == "cfg2" else f"traffic_{args.config}_r*.json"
    tps = sorted(glob.glob(os.path.join(ROOT, "profiles", pat)))
    tp = tps[-1] if tps else ""
    if tp:
        try:
            tr = json.load(open(tp))
            traffic, traffic_apply = tr.get("vanka_gemv"), tr.get("jacobian_apply")
        except Exception:
            traffic = traffic_apply = None

    # -- e2e through the public API with host (pinned) buffers ---------------
    def pinned(a):
        t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
        t.numpy()[...] = a
        return t.numpy()

    xh, rh, dh = pinned(syn.x), pinned(syn.x), pinned(syn.d0)
    yh = pinned(np.zeros_like(syn.x))

    def step_host():
        jac.matvec(xh, out=yh)
        return lvl.smooth(dh, rh, 1, cfg.omega, inplace=True)

    for _ in range(2):
        step_host()
    n_e2e = max(3, args.steps)  # the K timed steps (pipeline fill and drain included)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n_e2e):
        step_host()
    torch.cuda.synchronize()
    t_e2e = (time.perf_counter() - t0) / n_e2e
    if ws > 1:
        tt = torch.tensor([t_e2e], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_e2e = float(tt.item())
    # the same calls with PDST_HOST_ASYNC: each call enqueues its H2D copies on a
    # copy-in stream, its kernels behind them and its D2H on a copy-out stream
    # and returns, so one step's transfers overlap the other calls' kernels and
    # transfers (PCIe is full duplex); d's round trip stays ordered across steps
    def step_host_async():
        jac.matvec(xh, out=yh, asynchronous=True)
        lvl.smooth(dh, rh, 1, cfg.omega, inplace=True, asynchronous=True)

    for _ in range(2):
        step_host_async()
    jac.dev.sync()
    t0 = time.perf_counter()
    for _ in range(n_e2e):
        step_host_async()
    jac.dev.sync()
    t_e2e_async = (time.perf_counter() - t0) / n_e2e
    if ws > 1:
        tt = torch.tensor([t_e2e_async], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_e2e_async = float(tt.item())
    e2e = {"value": ws * N / t_e2e_async / 1e9, "unit": UNIT, "h2d_bytes_per_step": 3 * 8 * N,
           "d2h_bytes_per_step": 2 * 8 * N, "ms_per_step": t_e2e_async * 1e3,
           "sync_value": ws * N / t_e2e / 1e9, "sync_ms_per_step": t_e2e * 1e3,
           "note": "SlabJacobian.matvec(xh, out=yh) + VankaLevel.smooth(dh, rh, inplace) on pinned numpy buffers "
                   "through the C ABI with PDST_HOST_ASYNC (x, r, d in and y, d out every step on copy streams, "
                   "overlapping the other calls' kernels; one pdst_sync after the timed steps), wall clock; "
                   "sync_value: the same calls with synchronous PDST_HOST copies"}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_single(args.cpu_steps)
    extra = measure_residual_and_build(cfg, ctx, syn, jac, lvl, dev, flush, peak)
    others = {}
    if ws == 1 and not args.no_secondary:
        for name in args.secondary.split(","):
            if name and name != args.config:
                others[name] = measure_config_kernels(name, peak)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded 16-mode modal state + 1e-3 noise, SURVEY.md §8d; no dataset)",
        "config": {"workload": f"{cfg.name}: {cfg.nx}x{cfg.ny} Q2/P1disc, DG({cfg.k}), p={cfg.p}, delta={cfg.delta}, "
                               f"nu={cfg.nu}, nu_inf={cfg.nu_inf}, modN(sigma_max=nu), surrogate patches at "
                               f"rep_fraction={cfg.rep_fraction}, omega={cfg.omega}",
                   "n_dof": N, "step": "1 Jacobian apply + 1 Vanka sweep (1 smoothing step)",
                   "l2": "flushed between timed steps (256 MiB write, then a 256 MiB read of another buffer so no dirty lines remain; outside events)",
                   "parallelism": f"replicas x{ws}"},
        "gpu_launches": n_launches,
        # dominant kernel by time: the Jacobian apply (y = J x; the sweep's defect
        # apply, the same kernels with a right-hand side, is kernels.jacobian_defect).  Its
        # algorithmic bytes are SURVEY §8(d)'s B_apply (the reference algorithm's
        # compulsory traffic: x, y and the per-qp / side / CIP coefficient cache).
        "roofline": {"bound": "hbm", "kernel": "jacobian apply (k_jacobian + k_jac_post)",
                     "achieved": b_apply_ref / t_jac / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": b_apply_ref / t_jac / 1e9 / peak, "traffic": traffic_apply, "peak_kind": peak_kind,
                     "algorithmic_bytes": b_apply_ref, "launch_ms": kt["jacobian"][0],
                     "note": "coefficient-stream apply (DESIGN.md §3.1): moves x, y and a per-quadrature-point "
                             "cache of 108 doubles per cell and Radau node (kernels.jacobian_apply.algorithmic_bytes), "
                             "the reference algorithm's cache in our layout; traffic = ncu DRAM bytes per apply"},
        "roofline_gemv": {"bound": "hbm", "kernel": f"vanka_gemv (patch-inverse stream, {nblk} complex 21x21 "
                                                    f"block(s)/patch)",
                          "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak, "traffic": traffic,
                          "peak_kind": peak_kind, "algorithmic_bytes": b_gemv, "launch_ms": kt["vanka_gemv"][0]},
        "kernels": {
            "jacobian_apply": {"ms": kt["jacobian"][0], "gdofs": N / t_jac / 1e9,
                               "algorithmic_bytes": b_apply_ours, "gbs": b_apply_ours / t_jac / 1e9,
                               "frac_hbm": b_apply_ours / t_jac / 1e9 / peak,
                               "reference_cache_bytes": b_apply_ref,
                               "reference_cache_equiv_gbs": b_apply_ref / t_jac / 1e9,
                               "minimal_state_bytes": b_apply_min,
                               "minimal_state_equiv_gbs": b_apply_min / t_jac / 1e9,
                               "back_to_back_ms": t_b2b * 1e3,
                               "back_to_back_frac_hbm": b_apply_ref / t_b2b / 1e9 / peak,
                               "back_to_back_note": f"{nb2b} applies back to back between two events, no L2 flush "
                                                    "(x, y L2-resident as in a Krylov loop; the coefficient stream "
                                                    "exceeds L2); the roofline object above uses the flushed step"},
            "jacobian_defect": {"ms": kt["jacobian_defect"][0],
                                "algorithmic_bytes": b_apply_ref + 8.0 * N,
                                "frac_hbm": (b_apply_ref + 8.0 * N) / max(kt["jacobian_defect"][0], 1e-9) / 1e6 / peak,
                                "note": "the sweep's defect apply r - J d: the apply's kernels plus the right-hand side"},
            "vanka_gemv": {"ms": kt["vanka_gemv"][0]},
            "vanka_scatter": {"ms": kt["vanka_scatter"][0]},
            **extra,
        },
        "apply_gdofs": N / t_jac / 1e9,
        "sweep_gdofs": N / (kt["jacobian_defect"][0] * 1e-3 + t_gemv + kt["vanka_scatter"][0] * 1e-3) / 1e9,
        "setup_s": t_setup,
        "clocks": clk,
        "e2e": e2e,
    }
    if others:
        line["other_configs"] = others
    if cpu is not None:
        line["cpu_baseline"] = cpu
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def measure_residual_and_build(cfg, ctx, syn, jac, lvl, dev, flush, peak, reps=10):
    """Device time of the slab residual (pdst_residual, device pointers, L2
    flushed) with its HBM roofline, and of the preconditioner build
    (pdst_patches_build: surrogate linearization, patch assembly and the
    temporally diagonalized factorization) against the measured FP64 peak.
    Algorithmic traffic of the residual: U and R (k+1) nd each plus v_minus
    (Mv); algorithmic flops of the build: SURVEY §8(d)'s 2 D^3 per patch."""
    import torch

    from paper_2603_28706_b200 import _lib as L

    N = syn.x.size
    U = torch.as_tensor(syn.U, device=dev).reshape(-1)
    vm = torch.as_tensor(syn.v_minus, device=dev)
    R = torch.empty_like(U)
    w = jac.dev.where(U, vm, R)

    def res():
        L.check(L.lib().pdst_residual(jac.dev.h, L.vptr(U), L.vptr(vm), None, None, L.vptr(R), w), "pdst_residual")

    for _ in range(2):
        res()
    ts = []
    for i in range(reps):
        flush_l2(flush, i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        res()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    t_res = sum(ts) / len(ts) * 1e-3
    b_res = 8.0 * (2 * N + ctx.disc.n_velocity)
    # preconditioner build: rebuild the same patches (one synchronous call)
    tb = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        lvl2 = type(lvl)(ctx, None, None, surrogate=True, rep_fraction=cfg.rep_fraction, jac=jac)
        torch.cuda.synchronize()
        tb.append(time.perf_counter() - t0)
        del lvl2
    t_build = min(tb)
    nc, D = cfg.nx * cfg.ny, 21 * (cfg.k + 1)
    flop = 2.0 * nc * D ** 3
    tf = L.C.c_double()
    L.check(L.lib().pdst_fp64_peak(torch.cuda.current_device(), L.C.byref(tf)), "pdst_fp64_peak")
    return {
        "residual": {"ms": t_res * 1e3, "gdofs": N / t_res / 1e9, "algorithmic_bytes": b_res,
                     "gbs": b_res / t_res / 1e9, "frac_hbm": b_res / t_res / 1e9 / peak,
                     "note": "pdst_residual on device pointers, L2 flushed; algorithmic bytes 8 [2 (k+1) nd + Mv] "
                             "(state in, residual out, v_minus); FP64/latency-bound (one pow per volume point)"},
        "patch_build": {"ms": t_build * 1e3, "algorithmic_flop": flop, "tflops": flop / t_build / 1e12,
                        "fp64_peak_tflops": tf.value, "frac_fp64": flop / t_build / 1e12 / tf.value,
                        "note": "pdst_patches_build wall time (surrogate linearization, element and patch assembly, "
                                "temporally diagonalized inverses) against SURVEY 8(d)'s 2 D^3 flop per patch; "
                                "fp64 peak measured in-run (pdst_fp64_peak, DFMA chains)"},
    }


def measure_config_kernels(name, peak, steps=5):
    """Apply and Vanka-GEMV rooflines of another BASELINE config in the same
    run (libpdst's per-launch CUDA events over `steps` apply + sweep steps,
    L2 flushed between steps): the secondary lines of the bench output."""
    import torch

    from paper_2603_28706_b200 import _lib as L
    from paper_2603_28706_b200 import problem as pb
    from paper_2603_28706_b200.operators import SlabJacobian
    from paper_2603_28706_b200.smoother import VankaLevel
    from paper_2603_28706_b200.synth import CONFIGS, make_slab_inputs

    cfg = CONFIGS[name]
    params = pb.ModelParams(cfg.p, cfg.delta, cfg.nu, cfg.nu_inf)
    conf = pb.DiscretizationConfig(cfg.gamma1, cfg.gamma2, cfg.gamma_cip)
    syn = make_slab_inputs(cfg)
    ctx = pb.make_context(cfg.nx, cfg.ny, cfg.k, params, cfg.tau, config=conf, v_minus=syn.v_minus)
    dev = torch.device("cuda", torch.cuda.current_device())
    U = torch.as_tensor(syn.U, device=dev)
    x = torch.as_tensor(syn.x, device=dev)
    d = torch.as_tensor(syn.d0, device=dev)
    y = torch.empty_like(x)
    del syn
    jac = SlabJacobian(ctx, U, pb.modified_newton(cfg.nu))
    lvl = VankaLevel(ctx, U, pb.modified_newton(cfg.nu), surrogate=True, rep_fraction=cfg.rep_fraction, jac=jac)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
    for _ in range(2):
        jac.matvec(x, out=y)
        lvl.smooth(d, x, 1, cfg.omega, inplace=True)
    torch.cuda.synchronize()
    h = jac.dev.h
    L.lib().pdst_profile(h, 1)
    for i in range(steps):
        flush_l2(flush, i)
        jac.matvec(x, out=y)
        lvl.smooth(d, x, 1, cfg.omega, inplace=True)
    torch.cuda.synchronize()
    kt = {}
    for kid, kn in ((0, "jacobian"), (1, "vanka_gemv"), (2, "vanka_scatter"), (6, "jacobian_defect")):
        ms, cnt = L.C.c_double(), L.C.c_int64()
        L.lib().pdst_profile_read(h, kid, L.C.byref(ms), L.C.byref(cnt))
        kt[kn] = ms.value / max(cnt.value, 1)
    L.lib().pdst_profile(h, 0)
    N = x.numel()
    nc, k1 = cfg.nx * cfg.ny, cfg.k + 1
    nd, nbf = ctx.disc.ndof, 2 * (cfg.nx + cfg.ny)
    b_apply_ref = 8.0 * k1 * (2 * nd + 112 * nc + 56 * nbf + 4 * (2 * cfg.nx * (cfg.nx - 1)))
    _, nblk, bpp = lvl.patch_info()
    b_gemv = float(nc * bpp) + 8.0 * (N + nc * 21 * k1)
    t_j, t_g = kt["jacobian"] * 1e-3, kt["vanka_gemv"] * 1e-3
    t_step = t_j + (kt["jacobian_defect"] + kt["vanka_scatter"]) * 1e-3 + t_g  # apply + (defect apply, GEMV, scatter)
    out = {"workload": f"{name}: {cfg.nx}x{cfg.ny} Q2/P1disc, DG({cfg.k}), p={cfg.p}, delta={cfg.delta}, "
                       f"nu_inf={cfg.nu_inf}, modN, surrogate patches", "n_dof": N,
           "apply": {"ms": kt["jacobian"], "gdofs": N / t_j / 1e9, "algorithmic_bytes": b_apply_ref,
                     "achieved_gbs": b_apply_ref / t_j / 1e9, "frac": b_apply_ref / t_j / 1e9 / peak},
           "vanka_gemv": {"ms": kt["vanka_gemv"], "algorithmic_bytes": b_gemv, "achieved_gbs": b_gemv / t_g / 1e9,
                          "frac": b_gemv / t_g / 1e9 / peak},
           "defect_apply_ms": kt["jacobian_defect"],
           "vanka_scatter_ms": kt["vanka_scatter"],
           "step_gdofs_from_kernels": N / t_step / 1e9,
           "note": "same run as the headline line; libpdst per-launch CUDA events, L2 flushed between steps"}
    del jac, lvl, U, x, d, y, flush
    torch.cuda.empty_cache()
    return out


def run_solve(args):
    """BASELINE configs[4] workload: one modified-Newton iteration of the slab
    system, FGMRES preconditioned by the space-time multigrid V-cycle (5
    geometric levels, 2 + 2 Vanka sweeps, iterative coarsest-level solve),
    reporting Krylov iterations and the device time per V-cycle.  Not the
    driver's headline line (that is the default cfg2 step); evidence for
    DESIGN.md §9."""
    import numpy as np
    import torch

    from paper_2603_28706_b200 import problem as pb
    from paper_2603_28706_b200.errors import SlabSolveError
    from paper_2603_28706_b200.krylov import KrylovConfig
    from paper_2603_28706_b200.newton import NewtonConfig, nonlinear_solve_slab
    from paper_2603_28706_b200.stmg import MgConfig, StmgFactory
    from paper_2603_28706_b200.synth import CONFIGS, make_slab_inputs

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1 or args.virtual_ranks > 1:
        return run_solve_distributed(args)
    cfg = CONFIGS[args.config]
    params = pb.ModelParams(cfg.p, cfg.delta, cfg.nu, cfg.nu_inf)
    conf = pb.DiscretizationConfig(cfg.gamma1, cfg.gamma2, cfg.gamma_cip)
    syn = make_slab_inputs(cfg)
    ctx = pb.make_context(cfg.nx, cfg.ny, cfg.k, params, cfg.tau, config=conf, v_minus=syn.v_minus)
    variant = pb.modified_newton(cfg.nu)
    U0 = torch.as_tensor(syn.U, device=torch.device("cuda", local))
    min_cells = max(1, cfg.nx >> (args.levels - 1))
    mg = MgConfig(pre_smooth=2, post_smooth=2, omega=cfg.omega, surrogate=True, rep_fraction=cfg.rep_fraction,
                  min_cells=min_cells, coarse_solver="auto", coarse_sweeps=args.coarse_sweeps)
    vc = {"ms": [], "build_s": []}

    class TimedFactory(StmgFactory):
        def build(self, ctx_, U_, var_):
            torch.cuda.synchronize()
            t0 = time.time()
            pre = super().build(ctx_, U_, var_)
            torch.cuda.synchronize()
            vc["build_s"].append(time.time() - t0)
            vc["levels"] = pre.num_levels
            inner = pre.apply

            def apply(r, out=None):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                z = inner(r, out=out)
                b.record()
                b.synchronize()
                vc["ms"].append(a.elapsed_time(b))
                return z

            pre.apply = apply
            return pre

    newton = NewtonConfig(variant=variant, max_nonlinear=1)
    krylov = KrylovConfig(restart=args.restart, max_iters=args.max_krylov)
    torch.cuda.synchronize()
    t0 = time.time()
    stats, status, msg = None, "converged", ""
    try:
        _, stats = nonlinear_solve_slab(ctx, U0, newton, krylov, TimedFactory(mg), device=local)
    except SlabSolveError as e:
        stats, status, msg = e.diagnostics, e.kind, str(e)
    torch.cuda.synchronize()
    wall = time.time() - t0
    st = stats.steps[0] if stats is not None and stats.steps else None
    N = U0.numel()
    line = {
        "metric": "modified-Newton iteration: FGMRES + space-time multigrid V-cycle (Krylov iterations, ms per "
                  "V-cycle)", "impl": "ours", "n_gpus": 1, "dtype": "f64", "data": "synthetic (synth.py seeded state)",
        "config": {"workload": f"{cfg.name}: {cfg.nx}x{cfg.ny} Q2/P1disc, DG({cfg.k}), p={cfg.p}, delta={cfg.delta}, "
                               f"nu_inf={cfg.nu_inf}; {vc.get('levels')} levels (min_cells={min_cells}), 2+2 Vanka "
                               f"(omega={cfg.omega}, surrogate patches at rep_fraction={cfg.rep_fraction}), coarsest "
                               f"level: dense LU up to 4096 dofs, else FGMRES(<= 30, rtol 1e-6) preconditioned by "
                               f"{2 if args.coarse_sweeps is None else args.coarse_sweeps} Vanka steps, "
                               f"FGMRES(restart={args.restart}, budget {args.max_krylov}) in the M-inner product, "
                               f"Eisenstat-Walker eta0=1e-2",
                   "n_dof": N},
        "krylov_iterations": st.n_l if st else len(vc["ms"]), "newton_status": status, "newton_message": msg,
        "initial_residual": stats.initial_res if stats is not None else None,
        "residual_before": st.res_before if st else None, "residual_after": st.res_after if st else None,
        "linear_residual": st.lin_res if st else None, "line_search_lambda": st.lam if st else None,
        "vcycles": len(vc["ms"]), "ms_per_vcycle": float(np.median(vc["ms"])) if vc["ms"] else None,
        "vcycle_gdofs": N / (np.median(vc["ms"]) * 1e6) if vc["ms"] else None,
        "preconditioner_build_s": vc["build_s"], "newton_iteration_wall_s": wall,
    }
    print(json.dumps(line), flush=True)
    return 0


def run_solve_distributed(args):
    """configs[4] on a strip partition: one modified-Newton iteration of the
    slab system (distributed residual and M-norms, FGMRES preconditioned by the
    distributed V-cycle, coarsest level by FGMRES(coarse_iters) with 2 Vanka
    steps) over N GPUs (torchrun, NCCL) or --virtual-ranks P on one GPU."""
    import numpy as np
    import torch

    from paper_2603_28706_b200 import problem as pb
    from paper_2603_28706_b200.dist_mg import distributed_nonlinear_solve, global_levels
    from paper_2603_28706_b200.errors import SlabSolveError
    from paper_2603_28706_b200.krylov import KrylovConfig
    from paper_2603_28706_b200.newton import NewtonConfig
    from paper_2603_28706_b200.partition import DistComm, LocalTransport, StripPartition, TorchDistTransport
    from paper_2603_28706_b200.stmg import MgConfig
    from paper_2603_28706_b200.synth import CONFIGS, make_slab_inputs

    ws, rank, local = dist_env()
    dist = None
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    P = ws if ws > 1 else args.virtual_ranks
    cfg = CONFIGS[args.config]
    params = pb.ModelParams(cfg.p, cfg.delta, cfg.nu, cfg.nu_inf)
    conf = pb.DiscretizationConfig(cfg.gamma1, cfg.gamma2, cfg.gamma_cip)
    syn = make_slab_inputs(cfg)
    ctx = pb.make_context(cfg.nx, cfg.ny, cfg.k, params, cfg.tau, config=conf, v_minus=syn.v_minus)
    variant = pb.modified_newton(cfg.nu)
    min_cells = max(1, cfg.nx >> (args.levels - 1))
    mg = MgConfig(pre_smooth=2, post_smooth=2, omega=cfg.omega, surrogate=True, rep_fraction=cfg.rep_fraction,
                  min_cells=min_cells, coarse_solver="fgmres", coarse_sweeps=2, coarse_iters=args.coarse_iters,
                  coarse_rtol=1e-6)
    part = StripPartition(cfg.nx, cfg.ny, P, levels=global_levels(cfg.nx, cfg.ny, min_cells))
    mine = [rank] if ws > 1 else list(range(P))
    transport = (TorchDistTransport(part.layout(rank), part) if ws > 1
                 else LocalTransport([part.layout(r) for r in range(P)]))
    comm = DistComm() if ws > 1 else None
    newton = NewtonConfig(variant=variant, max_nonlinear=1)
    krylov = KrylovConfig(restart=args.restart, max_iters=args.max_krylov)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.time()
    status, msg = "converged", ""
    try:
        _, stats = distributed_nonlinear_solve(ctx, syn.U, newton, krylov, mg, part, mine, transport, comm, local)
    except SlabSolveError as e:
        stats, status, msg = e.diagnostics, e.kind, str(e)
    torch.cuda.synchronize()
    wall = time.time() - t0
    if dist:
        t = torch.tensor([wall], device=torch.device("cuda", local))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        wall = float(t.item())
    st = stats.steps[0] if stats is not None and stats.steps else None
    if rank == 0:
        print(json.dumps({
            "metric": "modified-Newton iteration on a strip partition: FGMRES + distributed space-time multigrid "
                      "(Krylov iterations, wall time)", "impl": "ours", "n_gpus": ws,
            "virtual_ranks": P if ws == 1 else None, "dtype": "f64", "data": "synthetic (synth.py seeded state)",
            "scaling": "strong",
            "config": {"workload": f"{cfg.name}: {cfg.nx}x{cfg.ny} Q2/P1disc, DG({cfg.k}); {part.levels} levels, "
                                   f"2+2 Vanka, coarsest FGMRES({args.coarse_iters}) + 2 Vanka steps, "
                                   f"FGMRES(restart={args.restart}, budget {args.max_krylov})",
                       "n_dof": (cfg.k + 1) * part.layout(0).nd, "parallelism": f"strips x{P}"},
            "newton_status": status, "newton_message": msg,
            "initial_residual": stats.initial_res if stats is not None else None,
            # a stalled FGMRES has spent its whole budget (krylov.py:118-139)
            "krylov_iterations": st.n_l if st else (args.max_krylov if status == "krylov" else None),
            "residual_after": st.res_after if st else None,
            "newton_iteration_wall_s": wall}), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def run_vcycle(args):
    """BASELINE configs[4]'s strong-scaling measurement: the space-time multigrid
    V-cycle (2 + 2 Vanka sweeps per level, coarsest level by FGMRES with Vanka
    preconditioning) on a strip partition of ONE global mesh over N GPUs
    (torchrun, NCCL halo exchanges and allreduces) or `--virtual-ranks P` ranks
    on one GPU.  Time per V-cycle = max over ranks of the device time; value =
    global dofs / that time (scaling "strong")."""
    import numpy as np
    import torch

    from paper_2603_28706_b200 import problem as pb
    from paper_2603_28706_b200.dist_mg import DistributedStmg, distributed_vcycle, global_levels
    from paper_2603_28706_b200.partition import DistComm, LocalTransport, StripPartition, TorchDistTransport
    from paper_2603_28706_b200.stmg import MgConfig
    from paper_2603_28706_b200.synth import CONFIGS, make_slab_inputs

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    P = ws if ws > 1 else args.virtual_ranks
    cfg = CONFIGS[args.config]
    params = pb.ModelParams(cfg.p, cfg.delta, cfg.nu, cfg.nu_inf)
    conf = pb.DiscretizationConfig(cfg.gamma1, cfg.gamma2, cfg.gamma_cip)
    syn = make_slab_inputs(cfg)
    ctx = pb.make_context(cfg.nx, cfg.ny, cfg.k, params, cfg.tau, config=conf, v_minus=syn.v_minus)
    variant = pb.modified_newton(cfg.nu)
    min_cells = max(1, cfg.nx >> (args.levels - 1))
    mg = MgConfig(pre_smooth=2, post_smooth=2, omega=cfg.omega, surrogate=True, rep_fraction=cfg.rep_fraction,
                  min_cells=min_cells, coarse_solver="fgmres", coarse_sweeps=2, coarse_iters=args.coarse_iters,
                  coarse_rtol=1e-6)
    nl = global_levels(cfg.nx, cfg.ny, min_cells)
    part = StripPartition(cfg.nx, cfg.ny, P, levels=nl)
    mine = [rank] if ws > 1 else list(range(P))
    transport = (TorchDistTransport(part.layout(rank), part) if ws > 1
                 else LocalTransport([part.layout(r) for r in range(P)]))
    comm = DistComm() if ws > 1 else None
    dev = torch.device("cuda", local)
    t0 = time.time()
    ranks = [DistributedStmg(ctx, syn.U, variant, part, r, mg, device=local) for r in mine]
    torch.cuda.synchronize()
    t_build = time.time() - t0
    nd = part.layout(0).nd
    rs = [torch.as_tensor(np.concatenate([rk.lay.to_local(syn.x[mu * nd:(mu + 1) * nd]) for mu in range(rk.k1)]),
                          device=dev) for rk in ranks]
    del syn

    def cycle():
        return distributed_vcycle(ranks, rs, transport, comm)

    for _ in range(args.warmup):
        cycle()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        cycle()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    if dist:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    N = (cfg.k + 1) * nd
    if rank == 0:
        print(json.dumps({
            "metric": "space-time multigrid V-cycle on a strip partition (GDoF/s = global dofs / ms per V-cycle)",
            "value": N / (ms * 1e6), "unit": "GDoF/s", "n_gpus": ws, "virtual_ranks": P if ws == 1 else None,
            "steps": args.steps, "warmup": args.warmup, "ms_per_vcycle": ms, "higher_is_better": True,
            "scaling": "strong", "dtype": "f64", "data": "synthetic (synth.py seeded state)",
            "config": {"workload": f"{cfg.name}: {cfg.nx}x{cfg.ny} Q2/P1disc, DG({cfg.k}); {nl} levels "
                                   f"(min_cells={min_cells}), 2+2 Vanka (omega={cfg.omega}, surrogate at "
                                   f"rep_fraction={cfg.rep_fraction}), coarsest level FGMRES({args.coarse_iters}) "
                                   f"with 2 Vanka steps, strips aligned to the coarsest cells, "
                                   f"{part.ghost} ghost rows per side",
                       "n_dof": N, "parallelism": f"strips x{P}"},
            "build_s": t_build}), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def relaunch(n):
    """`bench.py --gpus N` outside torchrun: start N ranks (one per GPU) under
    torch.distributed.run on 127.0.0.1 and return their exit status; fails
    loudly when fewer than N GPUs are visible."""
    import socket

    import torch

    have = torch.cuda.device_count()
    if have < n:
        sys.stderr.write(f"bench.py: --gpus {n} requested but only {have} CUDA device(s) are visible\n")
        return 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(n), "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd, cwd=ROOT).returncode


_FLUSH_READ = {}


def flush_l2(flush, i):
    """Cold L2 between timed steps: write a buffer larger than L2 (256 MiB), then read ANOTHER
    256 MiB buffer so the cache is left holding clean lines -- otherwise the first timed kernel
    shares HBM with the write-back of the flush's dirty lines (measured: ~2 us on a 44 us apply).
    Both passes are outside the timed events."""
    flush.fill_(float(i))
    rd = _FLUSH_READ.get(flush.device)
    if rd is None or rd.numel() != flush.numel():
        rd = _FLUSH_READ[flush.device] = flush.new_zeros(flush.shape)
    rd.sum()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--cpu-steps", type=int, default=6)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--virtual-ranks", type=int, default=1)
    ap.add_argument("--solve", action="store_true", help="one Newton iteration with FGMRES + STMG (configs[4])")
    ap.add_argument("--levels", type=int, default=5)
    ap.add_argument("--restart", type=int, default=20)
    ap.add_argument("--max-krylov", type=int, default=60)
    ap.add_argument("--coarse-sweeps", type=int, default=None,
                    help="--solve: Vanka steps per coarsest-level preconditioner application (default 2)")
    ap.add_argument("--vcycle", action="store_true", help="distributed V-cycle timing (configs[4] strong scaling)")
    ap.add_argument("--coarse-iters", type=int, default=30)
    ap.add_argument("--secondary", default="cfg5",
                    help="comma-separated configs whose apply / GEMV rooflines are measured after the headline step")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--strong", action="store_true",
                    help="strong scaling: the config's mesh split into N strips (default: weak, cfg rows per rank)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    ws = int(os.environ.get("WORLD_SIZE", "0") or 0)
    if ws == 0 and args.gpus > 1:
        return relaunch(args.gpus)
    if ws and ws != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}\n")
        return 2
    if args.impl == "reference":
        return run_reference(args)
    if args.solve:
        return run_solve(args)
    if args.vcycle:
        return run_vcycle(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
