"""Phase timeline of k_jacobian per CTA (needs a -DPDST_TRACE build via PDST_LIB)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2603_28706_b200 import problem as pb, _lib
from paper_2603_28706_b200.operators import SlabJacobian
from paper_2603_28706_b200.synth import CONFIGS, make_slab_inputs

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
params = pb.ModelParams(cfg.p, cfg.delta, cfg.nu, cfg.nu_inf)
conf = pb.DiscretizationConfig(cfg.gamma1, cfg.gamma2, cfg.gamma_cip)
syn = make_slab_inputs(cfg)
ctx = pb.make_context(cfg.nx, cfg.ny, cfg.k, params, cfg.tau, config=conf, v_minus=syn.v_minus)
U = torch.as_tensor(syn.U, device="cuda"); x = torch.as_tensor(syn.x, device="cuda")
jac = SlabJacobian(ctx, U, pb.modified_newton(cfg.nu))
y = torch.empty_like(x)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(5): jac.matvec(x, out=y)
lib = _lib.lib()
_b0 = np.zeros((8192, 16), dtype=np.uint64)
torch.cuda.synchronize()
lib.pdst_debug_trace(_b0.ctypes.data_as(ctypes.c_void_p), 8192)
flush.fill_(1)
jac.matvec(x, out=y)
torch.cuda.synchronize()
n = ((cfg.nx + 15) // 16) * ((cfg.ny + 15) // 16)
buf = np.zeros((8192, 16), dtype=np.uint64)
lib.pdst_debug_trace(buf.ctypes.data_as(ctypes.c_void_p), 8192)
t = buf[:n].astype(np.float64)
t0 = t[:, 0].min()
names = ["start", "staged"] + [f"mu{m}:{p}" for m in range(cfg.k + 1) for p in ("vol", "cip", "mass+sides", "sync1", "assembled")]
print(f"{n} CTAs; times in us from the first CTA start (min / median / max over CTAs)")
for i, nm in enumerate(names):
    c = (t[:, i] - t0) / 1e3
    print(f"{i:2d} {nm:18s} {c.min():7.1f} {np.median(c):7.1f} {c.max():7.1f}")
d = (t[:, len(names) - 1] - t[:, 0]) / 1e3
print("CTA duration min/median/max", d.min(), np.median(d), d.max())

kt = buf[8191, :8].astype(np.float64)
if kt[1] > 0:
    k0 = kt[0]
    print("kernel marks (us from the first tile CTA start): tile pass end %.2f | side products end %.2f | post released (first warp) %.2f, post end %.2f"
          % ((kt[1] - k0) / 1e3, (kt[3] - k0) / 1e3, (kt[6] - k0) / 1e3, (kt[7] - k0) / 1e3))
# per-role / per-SM-load breakdown (role = (tile // 148) & 1; SM id in column 15)
sm = buf[:n, 15].astype(np.int64)
cnt = np.bincount(sm, minlength=160)
load = cnt[sm]
role = (np.arange(n) // 148) & 1
same = sum(1 for s_ in np.unique(sm) if cnt[s_] == 2 and len(set(role[sm == s_])) == 1)
print("SMs used", (cnt > 0).sum(), "with 2 CTAs", (cnt == 2).sum(), "of which same-role pairs", same, "max CTAs/SM", cnt.max())
for key, sel in (("role0", role == 0), ("role1", role == 1), ("lone", load == 1), ("paired", load == 2)):
    if sel.sum() == 0: continue
    c = (t[sel][:, :len(names)] - t0) / 1e3
    print(key, sel.sum(), " ".join(f"{np.median(c[:, i]):6.1f}" for i in range(len(names))))

# precise cold spans from the kernel marks (globaltimer, 0.26 us resolution): 9 repetitions each
r = torch.as_tensor(syn.d0, device="cuda")
def spans(fn, reps=9):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        lib.pdst_debug_trace(_b0.ctypes.data_as(ctypes.c_void_p), 8192)
        flush.fill_(1)
        fn()
        torch.cuda.synchronize()
        lib.pdst_debug_trace(buf.ctypes.data_as(ctypes.c_void_p), 8192)
        k = buf[8191, :8].astype(np.float64)
        tt = buf[:n].astype(np.float64)
        out.append(((k[1] - k[0]) / 1e3, (k[7] - k[0]) / 1e3, np.median(tt[:, len(names) - 1] - tt[:, 0]) / 1e3))
        ph = np.median(tt[:, :len(names)] - tt[:, :1], axis=0) / 1e3
    a = np.array(out)
    print("   phases (median CTA, last repetition):", " ".join(f"{v:.1f}" for v in ph))
    return np.median(a, axis=0), a.min(axis=0)
for nm, fn in (("apply", lambda: jac.matvec(x, out=y)), ("defect", lambda: jac.defect(x, r, out=y))):
    med, mn = spans(fn)
    print(f"SPAN {nm}: tile pass {med[0]:.2f} us, tile start -> epilogue end {med[1]:.2f} us (min {mn[1]:.2f}), median CTA {med[2]:.2f} us")

# the slowest CTAs of the last repetition
tt = buf[:n].astype(np.float64)
end = (tt[:, len(names) - 1] - tt[:, 0].min()) / 1e3
sm = buf[:n, 15].astype(np.int64)
cnt = np.bincount(sm, minlength=200)
order = np.argsort(-end)
ntx = (cfg.nx + 15) // 16
print("slowest CTAs: (end us, tile x, tile y, sm, CTAs on that sm, started first on sm, staged us)")
for i in order[:16]:
    first = all(tt[i, 0] <= tt[j, 0] for j in np.where(sm == sm[i])[0])
    print(f"  {end[i]:6.2f} {i % ntx:3d} {i // ntx:3d} {sm[i]:4d} {cnt[sm[i]]} {int(first)} {(tt[i,1]-tt[:,0].min())/1e3:6.2f}")
lone = cnt[sm] == 1
print("lone CTAs end: median %.2f max %.2f | paired: median %.2f max %.2f" % (np.median(end[lone]), end[lone].max(), np.median(end[~lone]), end[~lone].max()))
idx = np.arange(n)
print("second CTA per SM (tile >= 148): median %.2f max %.2f; first: median %.2f max %.2f" % (np.median(end[idx >= 148]), end[idx >= 148].max(), np.median(end[idx < 148]), end[idx < 148].max()))
