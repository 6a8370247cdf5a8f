"""GPU slab operators behind the reference's operator interface.

Drop-in counterparts of (file:line into /root/reference/pkg/src/pdflow):
  SlabJacobian(ctx, U, variant).apply / .matvec      slab.py:176-205
  slab_residual(ctx, U, advect=None)                 slab.py:168-173
  MassNorm(ctx).apply / .norm                        solver/newton.py:96-121

Arguments may be numpy arrays (host; copied in/out by libpdst) or CUDA
torch tensors (device; launched asynchronously on torch's current stream).
Every call goes through libpdst.so; there is no CPU path.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .errors import ConstitutiveDomainError

__all__ = ["SlabDevice", "SlabJacobian", "slab_residual", "MassNorm", "forcing_at_qp", "variant_kind"]

_GAUSS_S = np.array([0.06943184420297371, 0.33000947820757187, 0.6699905217924281, 0.9305681557970262])


def variant_kind(variant):
    kind = getattr(variant, "kind", variant)
    if kind not in L.KIND:
        raise ValueError(f"unknown tangent kind {kind!r}")
    sigma = float(getattr(variant, "sigma_max", np.inf))
    return L.KIND[kind], sigma


def _is_torch(a):
    return a is not None and not isinstance(a, np.ndarray) and hasattr(a, "data_ptr")


def _f64(a):
    if a is None or _is_torch(a):
        return a
    return np.ascontiguousarray(a, dtype=np.float64)


def _torch_stream(device):
    import torch

    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def forcing_at_qp(ctx, times=None):
    """Body force f(x, y, t) at the x-major volume points of every cell and
    Radau node, shape (k+1, ncells, 16, 2) — the coordinates of
    forms.py:189-191 (cell origin + Gauss point * cell size).  None when
    ctx.data.f is None."""
    f = getattr(ctx.data, "f", None)
    if f is None:
        return None
    mesh = ctx.disc.mesh
    nx, ny = mesh.nx, mesh.ny
    hx, hy = mesh.hx, mesh.hy
    i, j = np.arange(nx), np.arange(ny)
    ox, oy = np.meshgrid(mesh.x0 + i * hx, mesh.y0 + j * hy)
    ox, oy = ox.ravel(), oy.ravel()
    px = np.repeat(_GAUSS_S, 4)  # q = 4 qx + qy
    py = np.tile(_GAUSS_S, 4)
    X = ox[:, None] + px[None, :] * hx
    Y = oy[:, None] + py[None, :] * hy
    times = ctx.t_start + ctx.tau * np.asarray(ctx.basis.nodes) if times is None else times
    out = np.empty((len(times), nx * ny, 16, 2))
    for mu, t in enumerate(times):
        out[mu] = np.asarray(f(X, Y, float(t)), dtype=float)
    if not out.any():
        return None
    return out


class SlabDevice:
    """Owns one libpdst handle bound to a slab context's mesh, time basis,
    discretization and model parameters."""

    def __init__(self, ctx, device=0):
        self.ctx = ctx
        disc, mesh = ctx.disc, ctx.disc.mesh
        from .problem import dirichlet_flags

        self._dir = dirichlet_flags(mesh)
        k = int(ctx.basis.k)
        self.k1 = k + 1
        self._nodes = np.ascontiguousarray(ctx.basis.nodes, dtype=np.float64)
        self._weights = np.ascontiguousarray(ctx.basis.weights, dtype=np.float64)
        self._K = np.ascontiguousarray(ctx.tmat.K_t, dtype=np.float64)
        self._m = np.ascontiguousarray(ctx.tmat.m_t, dtype=np.float64)
        m = L.Mesh(mesh.nx, mesh.ny, mesh.x0, mesh.y0, mesh.x1, mesh.y1,
                   self._dir.ctypes.data_as(C.POINTER(C.c_uint8)))
        t = L.Time(k, L.dptr(self._nodes), L.dptr(self._weights), L.dptr(self._K), L.dptr(self._m))
        cfg = ctx.config
        d = L.Disc(cfg.gamma1, cfg.gamma2, cfg.gamma_cip, int(cfg.enable_viscous), int(cfg.enable_convection),
                   int(cfg.enable_pressure), 1 if getattr(disc, "pressure", "p1disc") == "q1" else 0)
        pr = ctx.params
        p = L.Params(pr.p, pr.delta, pr.nu, pr.nu_inf)
        h = C.c_void_p()
        self.device = device
        L.check(L.lib().pdst_create(C.byref(m), C.byref(t), C.byref(d), C.byref(p), float(ctx.tau), device, None,
                                    C.byref(h)), "pdst_create")
        self.h = h
        mv, mp, nd, ndof = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        L.check(L.lib().pdst_sizes(h, C.byref(mv), C.byref(mp), C.byref(nd), C.byref(ndof)))
        self.mv, self.mp, self.nd, self.ndof = mv.value, mp.value, nd.value, ndof.value
        if disc.n_velocity != self.mv or disc.ndof != self.nd:
            raise ValueError("discretization is not Q2/P1disc on a structured quad mesh")
        g_hat = getattr(cfg, "g_hat", None)
        if g_hat is not None:
            gh = np.ascontiguousarray(g_hat, dtype=np.float64)
            L.check(L.lib().pdst_set_lifting(h, L.vptr(gh), L.HOST), "pdst_set_lifting")

    def close(self):
        if getattr(self, "h", None):
            L.lib().pdst_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- argument handling ---------------------------------------------------
    def where(self, *arrays, asynchronous=False):
        """PDST_DEVICE for torch CUDA tensors (torch's current stream), else
        PDST_HOST (copied, synchronous) or, with asynchronous=True,
        PDST_HOST_ASYNC (page-locked numpy buffers; call sync() before using them)."""
        dev = [a for a in arrays if _is_torch(a)]
        if dev:
            if len(dev) != len([a for a in arrays if a is not None]):
                raise TypeError("mix of host and device arrays")
            L.check(L.lib().pdst_set_stream(self.h, _torch_stream(dev[0].device)))
            return L.DEVICE
        L.check(L.lib().pdst_set_stream(self.h, None))
        return L.HOST_ASYNC if asynchronous else L.HOST

    def sync(self):
        """Wait for every call of this handle, incl. asynchronous host copies."""
        L.check(L.lib().pdst_sync(self.h), "pdst_sync")

    @staticmethod
    def empty_like(a, shape=None):
        if _is_torch(a):
            import torch

            return torch.empty(shape if shape is not None else a.shape, dtype=torch.float64, device=a.device)
        return np.empty(shape if shape is not None else a.shape)


class SlabJacobian:
    """Matrix-free slab Jacobian J_n(U) on the GPU (slab.py:176-205).

    J x = [tau w_mu J_mu x_mu + sum_nu K_t[mu,nu] M_x x_nu,v]_mu with the
    frozen per-node linearizations of forms.py:527-578."""

    def __init__(self, ctx, U, variant, device=0, dev: SlabDevice | None = None):
        if ctx.params.delta <= 0.0:
            raise ConstitutiveDomainError("jacobian requires delta > 0")
        self.ctx = ctx
        self.variant = variant
        self.dev = dev or SlabDevice(ctx, device)
        kind, sigma = variant_kind(variant)
        Uc = _f64(U)
        w = self.dev.where(Uc)
        L.check(L.lib().pdst_linearize(self.dev.h, L.vptr(Uc, self.dev.ndof, "U"), kind, sigma, w), "pdst_linearize")

    @property
    def shape(self):
        return (self.dev.ndof, self.dev.ndof)

    def matvec(self, x, out=None, asynchronous=False):
        """y = J x.  asynchronous=True (host arrays in page-locked memory, `out`
        given): returns at once; the copies overlap other calls' kernels and
        transfers; `self.dev.sync()` before reading `out` or reusing `x`."""
        xc = _f64(x)
        if asynchronous and (out is None or _is_torch(xc)):
            raise TypeError("asynchronous matvec needs page-locked host x and out")
        y = self.dev.empty_like(xc) if out is None else out
        w = self.dev.where(xc, y, asynchronous=asynchronous)
        n = self.dev.ndof
        L.check(L.lib().pdst_jacobian_apply(self.dev.h, L.vptr(xc, n, "x"), L.vptr(y, n, "out"), w), "pdst_jacobian_apply")
        return y

    def apply(self, dU):
        shape = dU.shape
        return self.matvec(dU.reshape(-1)).reshape(shape)

    def defect(self, x, r, out=None):
        """r - J x (the Vanka defect, solver/multigrid.py:336)."""
        xc, rc = _f64(x), _f64(r)
        y = self.dev.empty_like(xc) if out is None else out
        w = self.dev.where(xc, rc, y)
        n = self.dev.ndof
        L.check(L.lib().pdst_jacobian_defect(self.dev.h, L.vptr(xc, n, "x"), L.vptr(rc, n, "r"), L.vptr(y, n, "out"), w), "pdst_jacobian_defect")
        return y

    __matmul__ = matvec


def slab_residual(ctx, U, advect=None, dev: SlabDevice | None = None, device=0):
    """R_n(U) = tau (diag(w) x I) F(U) - [(K_t x M) V - (m_t x M) v_minus; 0] (slab.py:168-173)."""
    if ctx.params.delta <= 0.0:
        raise ConstitutiveDomainError("spatial residual requires delta > 0")
    own = dev is None
    dev = dev or SlabDevice(ctx, device)
    try:
        from .manufactured import device_forcing_case

        Uc = _f64(U)
        dev_f = device_forcing_case(ctx) is not None
        # the manufactured problem's forcing is evaluated on the device
        # (pdst_manufactured_forcing); any other f(x, y, t) on the host, as the
        # reference does (forms.py:459)
        fq = dev.empty_like(Uc, shape=(dev.k1 * ctx.disc.mesh.nx * ctx.disc.mesh.ny * 32,)) if dev_f else \
            forcing_at_qp(ctx)
        if dev_f:
            L.check(L.lib().pdst_manufactured_forcing(dev.h, float(ctx.t_start), L.vptr(fq), dev.where(fq)),
                    "pdst_manufactured_forcing")
        vm = ctx.v_minus
        adv = _f64(advect)
        if _is_torch(Uc):
            import torch

            fq = None if fq is None else torch.as_tensor(fq, device=Uc.device)
            vm = torch.as_tensor(np.asarray(vm, dtype=np.float64), device=Uc.device) if not _is_torch(vm) else vm
        else:
            fq = None if fq is None else np.ascontiguousarray(fq)
            vm = np.ascontiguousarray(vm, dtype=np.float64)
        R = dev.empty_like(Uc)
        w = dev.where(Uc, vm, fq, adv, R)
        L.check(L.lib().pdst_residual(dev.h, L.vptr(Uc, dev.ndof, "U"), L.vptr(vm, dev.mv, "v_minus"), L.vptr(fq),
                                      L.vptr(adv, None if adv is None else dev.ndof, "advect"), L.vptr(R), w),
                "pdst_residual")
        return R
    finally:
        if own and not _is_torch(U):
            dev.close()


class MassNorm:
    """Block mass-weighted norm (solver/newton.py:96-121) on the GPU."""

    def __init__(self, ctx, dev: SlabDevice | None = None, device=0):
        self.dev = dev or SlabDevice(ctx, device)

    def apply(self, x):
        xc = _f64(x)
        shape = xc.shape
        flat = xc.reshape(-1)
        y = self.dev.empty_like(flat)
        w = self.dev.where(flat, y)
        L.check(L.lib().pdst_mass_apply(self.dev.h, L.vptr(flat, self.dev.ndof, "x"), L.vptr(y), w), "pdst_mass_apply")
        return y.reshape(shape)

    def apply_into(self, x, out):
        """out = M x for device tensors (no allocation; FGMRES basis rows)."""
        w = self.dev.where(x, out)
        L.check(L.lib().pdst_mass_apply(self.dev.h, L.vptr(x, self.dev.ndof, "x"), L.vptr(out, self.dev.ndof, "out"), w), "pdst_mass_apply")
        return out

    def dot(self, a, b):
        ac, bc = _f64(a).reshape(-1), _f64(b).reshape(-1)
        if _is_torch(ac):
            import torch

            out = torch.empty(1, dtype=torch.float64, device=ac.device)
            w = self.dev.where(ac, bc, out)
            L.check(L.lib().pdst_mass_dot(self.dev.h, L.vptr(ac, self.dev.ndof, "a"), L.vptr(bc, self.dev.ndof, "b"), L.vptr(out), w), "pdst_mass_dot")
            return out
        out = np.zeros(1)
        L.check(L.lib().pdst_mass_dot(self.dev.h, L.vptr(ac, self.dev.ndof, "a"), L.vptr(bc, self.dev.ndof, "b"), L.vptr(out), L.HOST), "pdst_mass_dot")
        return float(out[0])

    def norm(self, x):
        v = self.dot(x, x)
        return float(np.sqrt(max(float(v), 0.0)))
