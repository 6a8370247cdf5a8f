"""CPU restatement of the reference's FGMRES and Newton driver — TEST
INFRASTRUCTURE ONLY (imported by tests/, never by the product path).

fgmres(...) follows pdflow/solver/krylov.py:46-139 (modified Gram-Schmidt
with one re-orthogonalization pass, Givens rotations, lstsq head solve, true
residual at restarts, and the reference's extra 1/res_norm on the first
mass-weighted basis vector, krylov.py:89); ``orth="gram"`` evaluates the same
MGS recurrence in block form (one multi-dot plus a small triangular solve
with the basis Gram matrix), which is what the device implementation does;
``orth="cgs2"`` (classical Gram-Schmidt twice) is NOT equivalent here because
the reference's first mass-weighted basis vector is mis-scaled.
Pinned against the reference's own runs (tests/golden/fg_*.npz).
"""

from __future__ import annotations

import numpy as np


def fgmres(op, rhs, tol, restart=60, max_iters=300, precond=None, mass=None, x0=None, orth="mgs2"):
    n = rhs.size
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=float)
    M = (lambda v: v) if mass is None else mass

    def m_norm(v):
        return float(np.sqrt(np.dot(v, M(v))))

    b_norm = m_norm(rhs)
    if b_norm == 0.0:
        return np.zeros(n), 0, True, 0.0, 0.0
    target = tol * b_norm
    r = rhs - op(x) if x0 is not None else rhs.copy()
    res_norm = m_norm(r)
    total = 0
    while total < max_iters:
        if res_norm <= target:
            return x, total, True, res_norm, target
        m = min(restart, max_iters - total)
        V = [r / res_norm]
        MV = [M(V[0]) / res_norm] if mass is not None else [V[0]]
        Z = []
        H = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        g[0] = res_norm
        j_used = 0
        for j in range(m):
            z = V[j] if precond is None else precond(V[j])
            Z.append(z)
            w = op(z)
            mw = M(w) if mass is not None else w
            for _ in range(2):
                if orth == "mgs2":
                    for i in range(j + 1):
                        hij = float(np.dot(w, MV[i]))
                        H[i, j] += hij
                        w = w - hij * V[i]
                        mw = w if mass is None else mw - hij * MV[i]
                elif orth == "gram":
                    # MGS as one block product: c = MV' w, then the lower-triangular
                    # solve h_i = c_i - sum_{l<i} <MV_i, V_l> h_l (exactly the
                    # sequential MGS recurrence, also for a non-orthogonal basis)
                    c = np.array([np.dot(w, MV[i]) for i in range(j + 1)])
                    h = np.zeros(j + 1)
                    for i in range(j + 1):
                        h[i] = c[i] - sum(np.dot(MV[i], V[l]) * h[l] for l in range(i))
                    H[: j + 1, j] += h
                    w = w - sum(h[i] * V[i] for i in range(j + 1))
                    mw = w if mass is None else mw - sum(h[i] * MV[i] for i in range(j + 1))
                else:
                    h = np.array([np.dot(w, MV[i]) for i in range(j + 1)])
                    H[: j + 1, j] += h
                    w = w - sum(h[i] * V[i] for i in range(j + 1))
                    mw = w if mass is None else mw - sum(h[i] * MV[i] for i in range(j + 1))
            hh = float(np.sqrt(max(np.dot(w, mw), 0.0)))
            H[j + 1, j] = hh
            total += 1
            j_used = j + 1
            breakdown = hh <= 1e-14 * max(1.0, abs(H[: j + 1, j]).max())
            if not breakdown:
                V.append(w / hh)
                MV.append(V[-1] if mass is None else mw / hh)
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            d = np.hypot(H[j, j], H[j + 1, j])
            cs[j], sn[j] = (1.0, 0.0) if d == 0.0 else (H[j, j] / d, H[j + 1, j] / d)
            H[j, j] = cs[j] * H[j, j] + sn[j] * H[j + 1, j]
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            if abs(g[j + 1]) <= target or breakdown:
                break
        k = j_used
        y = np.linalg.lstsq(H[:k, :k], g[:k], rcond=None)[0] if k else np.zeros(0)
        for i in range(k):
            x = x + y[i] * Z[i]
        r = rhs - op(x)
        res_norm = m_norm(r)
    return x, total, res_norm <= target, res_norm, target
