"""Flexible right-preconditioned GMRES in the M-inner product, on the GPU.

Drop-in counterpart of ``pdflow.solver.krylov`` (krylov.py:17-139): same
``KrylovConfig`` / ``FgmresResult`` / ``fgmres(op, rhs, tol, config, precond,
mass, x0)`` signature, restart / budget / breakdown / Givens / lstsq logic and
iteration count semantics.  The Krylov basis ``V``, its mass image ``MV`` and
the flexible directions ``Z`` live in device memory as (m+1, n) blocks.  The
orthogonalization is the reference's modified Gram-Schmidt with one
re-orthogonalization pass (krylov.py:100-108) in block form: per pass one
batched multi-dot ``c = MV' w`` (``pdst_multidot``), the MGS recurrence
``h_i = c_i - sum_{l<i} <MV_i, V_l> h_l`` on the host from the Gram rows of
the basis, and one fused update of ``w`` and ``M w`` (``pdst_multi_axpy``) --
algebraically MGS for any basis.  The small Hessenberg
least-squares problem stays on the host, exactly as the reference does it
(numpy Givens rotations and ``lstsq``).

Vectors may be torch device tensors (the fast path) or numpy arrays (copied
to the device once; the result is returned as numpy).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib as L

__all__ = ["KrylovConfig", "FgmresResult", "fgmres"]


@dataclass
class KrylovConfig:
    """Restart length and total iteration budget (krylov.py:20-29)."""

    restart: int = 60
    max_iters: int = 300

    def __post_init__(self):
        if self.restart <= 0 or self.max_iters <= 0:
            raise ValueError("restart and max_iters must be positive")


@dataclass
class FgmresResult:
    x: object
    iterations: int
    converged: bool
    residual_norm: float
    target: float


def _torch():
    import torch

    return torch


def _owner_dev(*objs):
    """The libpdst handle wrapper (SlabDevice) of the first object that has one."""
    for o in objs:
        if o is None:
            continue
        for cand in (o, getattr(o, "__self__", None)):
            dev = getattr(cand, "dev", None)
            if dev is not None and getattr(dev, "h", None) is not None:
                return dev
    raise ValueError("fgmres on the GPU needs a libpdst-backed operator, preconditioner or mass (MassNorm)")


class _Block:
    """(rows, n) fp64 device block with the libpdst block kernels."""

    def __init__(self, dev, rows, n, device):
        torch = _torch()
        self.dev = dev
        self.t = torch.zeros((rows, n), dtype=torch.float64, device=device)
        self.n = n

    def row(self, i):
        return self.t[i]

    def dots(self, m, w, out):
        """out[:m] = <row_i, w>."""
        L.check(L.lib().pdst_multidot(self.dev.h, L.vptr(self.t), self.n, m, L.vptr(w), self.n, L.vptr(out),
                                      L.DEVICE), "pdst_multidot")

    def sub(self, m, c, w, other=None, w2=None):
        """w -= sum_i c[i] row_i (and w2 -= sum_i c[i] other.row_i)."""
        L.check(L.lib().pdst_multi_axpy(self.dev.h, L.vptr(self.t), L.vptr(other.t) if other is not None else None,
                                        self.n, m, L.vptr(c), L.vptr(w), L.vptr(w2), self.n, L.DEVICE),
                "pdst_multi_axpy")


def fgmres(op, rhs, tol: float, config: KrylovConfig | None = None, precond=None, mass=None, x0=None,
           comm=None) -> FgmresResult:
    """Solve op(x) = rhs to a relative tolerance in the M-weighted norm
    (krylov.py:46-139).  The iteration count is the number of preconditioned
    operator applications.

    comm (partition.DistComm): the vectors are one rank's part of a
    distributed slab vector whose non-owned (ghost) entries are zero; every
    inner product is the local Euclidean product (with M applied through
    `mass`, itself halo-aware) summed over the ranks by comm.allreduce_ —
    one allreduce of a (j+1)-vector per Gram-Schmidt pass."""
    torch = _torch()
    config = config or KrylovConfig()
    dev = _owner_dev(mass, op, precond)
    device = torch.device("cuda", dev.device)
    host_io = not isinstance(rhs, torch.Tensor)
    b = torch.as_tensor(np.ascontiguousarray(rhs, dtype=np.float64).reshape(-1) if host_io else rhs.reshape(-1),
                        device=device).to(torch.float64).contiguous()
    n = b.numel()
    L.check(L.lib().pdst_set_stream(dev.h, L.C.c_void_p(torch.cuda.current_stream(device).cuda_stream)))

    def dev_vec(v):
        return v if isinstance(v, torch.Tensor) else torch.as_tensor(np.ascontiguousarray(v, dtype=np.float64),
                                                                     device=device)

    def apply_op(v, out=None):
        mv = getattr(op, "__self__", None)
        if out is not None and mv is not None and hasattr(mv, "matvec") and getattr(op, "__name__", "") == "matvec":
            return mv.matvec(v, out=out)
        y = dev_vec(op(v)).reshape(-1)
        if out is not None:
            out.copy_(y)
            return out
        return y

    def apply_mass(v, out):
        if mass is None:
            out.copy_(v)
            return out
        if hasattr(mass, "apply_into"):
            return mass.apply_into(v, out)
        out.copy_(dev_vec(mass.apply(v)).reshape(-1))
        return out

    scal = torch.empty(1, dtype=torch.float64, device=device)

    def mdot(a, b_):
        if comm is not None:  # <a, M b> = sum over ranks of the owned a . (M b)
            mb = apply_mass(b_, torch.empty_like(b_)) if mass is not None else b_
            L.check(L.lib().pdst_dot(dev.h, L.vptr(a), L.vptr(mb), n, L.vptr(scal), L.DEVICE), "pdst_dot")
            comm.allreduce_(scal)
        elif mass is None:
            L.check(L.lib().pdst_dot(dev.h, L.vptr(a), L.vptr(b_), n, L.vptr(scal), L.DEVICE), "pdst_dot")
        else:
            L.check(L.lib().pdst_mass_dot(dev.h, L.vptr(a), L.vptr(b_), L.vptr(scal), L.DEVICE), "pdst_mass_dot")
        return float(scal.item())

    def m_norm(v):
        return float(np.sqrt(mdot(v, v)))

    def finish(x, it, conv, rn, tgt):
        return FgmresResult(x.cpu().numpy() if host_io else x, it, conv, rn, tgt)

    x = torch.zeros(n, dtype=torch.float64, device=device) if x0 is None else dev_vec(x0).reshape(-1).clone()
    b_norm = m_norm(b)
    if b_norm == 0.0:
        return finish(torch.zeros_like(b), 0, True, 0.0, 0.0)
    target = tol * b_norm

    def residual(xv):
        mv = getattr(op, "__self__", None)
        if mv is not None and hasattr(mv, "defect") and getattr(op, "__name__", "") == "matvec":
            return mv.defect(xv, b)  # r = b - J x in one kernel
        return b - apply_op(xv)

    pc_out = precond is not None and _accepts_out(precond)
    r = residual(x) if x0 is not None else b.clone()
    res_norm = m_norm(r)
    total_iters = 0
    rest = min(config.restart, config.max_iters)
    V = _Block(dev, rest + 1, n, device)
    MV = _Block(dev, rest + 1, n, device)
    Z = _Block(dev, rest, n, device)
    hdev = torch.empty(rest + 1, dtype=torch.float64, device=device)
    ydev = torch.empty(rest, dtype=torch.float64, device=device)

    while total_iters < config.max_iters:
        if res_norm <= target:
            return finish(x, total_iters, True, res_norm, target)
        m = min(config.restart, config.max_iters - total_iters)
        torch.mul(r, 1.0 / res_norm, out=V.row(0))
        apply_mass(V.row(0), MV.row(0))
        if mass is not None:
            # the reference divides the mass image of the (already normalized)
            # first basis vector by res_norm once more (krylov.py:89); kept so
            # iteration counts and stalls match the reference exactly
            MV.row(0).mul_(1.0 / res_norm)
        H = np.zeros((m + 1, m))
        G = np.zeros((m + 1, m + 1))
        cs = np.zeros(m)
        sn = np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = res_norm
        j_used = 0
        for j in range(m):
            vj = V.row(j)
            if precond is None:
                Z.row(j).copy_(vj)
            elif pc_out:
                precond(vj, out=Z.row(j))
            else:
                Z.row(j).copy_(dev_vec(precond(vj)).reshape(-1))
            w, mw = V.row(j + 1), MV.row(j + 1)
            apply_op(Z.row(j), out=w)
            apply_mass(w, mw)
            # modified Gram-Schmidt with one re-orthogonalization pass, in block
            # form: c = MV' w (one multi-dot), h from the lower-triangular
            # recurrence h_i = c_i - sum_{l<i} G[i,l] h_l with the basis Gram
            # matrix G[i,l] = <MV_i, V_l> (identical to the sequential MGS of
            # krylov.py:103-108 even though the reference's first mass-weighted
            # vector is mis-scaled), then w -= V h, mw -= MV h (one fused update)
            for p in range(2):
                MV.dots(j + 1, w, hdev[: j + 1])
                if comm is not None:
                    comm.allreduce_(hdev[: j + 1])
                c = hdev[: j + 1].cpu().numpy()
                h = np.empty(j + 1)
                for i in range(j + 1):
                    h[i] = c[i] - float(np.dot(G[i, :i], h[:i]))
                H[: j + 1, j] += h
                hdev[: j + 1].copy_(torch.from_numpy(h))
                V.sub(j + 1, hdev[: j + 1], w, MV, mw)
            hh2 = mdot_plain(dev, w, mw, n, scal, comm)
            hh = float(np.sqrt(max(hh2, 0.0)))
            H[j + 1, j] = hh
            total_iters += 1
            j_used = j + 1
            breakdown = hh <= 1e-14 * max(1.0, abs(H[: j + 1, j]).max())
            if not breakdown:
                w.mul_(1.0 / hh)
                mw.mul_(1.0 / hh)
                if j + 1 < m:  # Gram row of the new basis vector: G[j+1, l] = <MV_{j+1}, V_l>
                    V.dots(j + 1, mw, hdev[: j + 1])
                    if comm is not None:
                        comm.allreduce_(hdev[: j + 1])
                    G[j + 1, : j + 1] = hdev[: j + 1].cpu().numpy()
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            denom = np.hypot(H[j, j], H[j + 1, j])
            if denom == 0.0:
                cs[j], sn[j] = 1.0, 0.0
            else:
                cs[j], sn[j] = H[j, j] / denom, H[j + 1, j] / denom
            H[j, j] = cs[j] * H[j, j] + sn[j] * H[j + 1, j]
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            if abs(g[j + 1]) <= target or breakdown:
                break
        k = j_used
        y = np.linalg.lstsq(H[:k, :k], g[:k], rcond=None)[0] if k else np.zeros(0)
        if k:
            ydev[:k].copy_(torch.as_tensor(-y, dtype=torch.float64))
            Z.sub(k, ydev, x)  # x += sum_i y_i Z_i
        r = residual(x)
        res_norm = m_norm(r)
    return finish(x, total_iters, res_norm <= target, res_norm, target)


def _accepts_out(fn):
    import inspect

    try:
        return "out" in inspect.signature(fn).parameters
    except (TypeError, ValueError):
        return False


def mdot_plain(dev, a, b, n, scal, comm=None):
    """Euclidean <a, b> on the device (the Arnoldi norm <w, M w>, krylov.py:109)."""
    L.check(L.lib().pdst_dot(dev.h, L.vptr(a), L.vptr(b), n, L.vptr(scal), L.DEVICE), "pdst_dot")
    if comm is not None:
        comm.allreduce_(scal)
    return float(scal.item())
