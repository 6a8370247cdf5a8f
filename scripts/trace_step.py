"""Device-side timeline of the bench step (apply, defect apply, patch GEMV, scatter) from the
%globaltimer marks of a -DPDST_TRACE build of every translation unit:
  NVCC_DEFS=-DPDST_TRACE scripts/build_variant.sh trace_all 's/XYZZY//'
  PDST_LIB=$PWD/exp/libpdst_trace_all.so python scripts/trace_step.py [cfg2]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2603_28706_b200 import problem as pb, _lib
from paper_2603_28706_b200.operators import SlabJacobian
from paper_2603_28706_b200.smoother import VankaLevel
from paper_2603_28706_b200.synth import CONFIGS, make_slab_inputs

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
params = pb.ModelParams(cfg.p, cfg.delta, cfg.nu, cfg.nu_inf)
conf = pb.DiscretizationConfig(cfg.gamma1, cfg.gamma2, cfg.gamma_cip)
syn = make_slab_inputs(cfg)
ctx = pb.make_context(cfg.nx, cfg.ny, cfg.k, params, cfg.tau, config=conf, v_minus=syn.v_minus)
U = torch.as_tensor(syn.U, device="cuda"); x = torch.as_tensor(syn.x, device="cuda")
d = torch.as_tensor(syn.d0, device="cuda").clone(); r = torch.as_tensor(syn.x, device="cuda").clone()
variant = pb.modified_newton(cfg.nu)
jac = SlabJacobian(ctx, U, variant)
lvl = VankaLevel(ctx, U, variant, surrogate=True, rep_fraction=cfg.rep_fraction, jac=jac)
y = torch.empty_like(x)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda"); rd = torch.zeros_like(flush)
lib = _lib.lib()
buf = np.zeros((8192, 16), dtype=np.uint64)
def step():
    jac.matvec(x, out=y)
    lvl.smooth(d, r, 1, cfg.omega, inplace=True)
for _ in range(5): step()
rows = []
for rep in range(9):
    torch.cuda.synchronize()
    lib.pdst_debug_trace(buf.ctypes.data_as(ctypes.c_void_p), 8192)
    flush.fill_(1); rd.sum()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); step(); b.record()
    torch.cuda.synchronize()
    lib.pdst_debug_trace(buf.ctypes.data_as(ctypes.c_void_p), 8192)
    st = np.frombuffer(buf[8189:8191].tobytes(), dtype=np.uint64)[:32].astype(np.float64)
    t0 = st[0]
    rows.append([(st[4 * k + j] - t0) / 1e3 for k in range(6) for j in range(3)] + [a.elapsed_time(b) * 1e3])
m = np.median(np.array(rows), axis=0)
names = ["apply tile", "apply epilogue", "defect tile", "defect epilogue", "patch GEMV", "scatter"]
print("median over 9 cold steps, us from the apply's first CTA: first start / first past its wait / last end")
for k, n in enumerate(names):
    print(f"  {n:16s} {m[3*k]:8.2f} {m[3*k+1]:8.2f} {m[3*k+2]:8.2f}   (active after wait: {m[3*k+2]-m[3*k+1]:6.2f} us)")
print(f"  step by CUDA events: {m[-1]:.1f} us; device span apply start -> scatter end: {m[17]:.2f} us")
