"""Host-side DG(k) time basis: right Gauss-Radau nodes on (0, 1] and the
temporal matrices (M_t, K_t, m_t).

Restates timebasis.py:67-119 (nodes = mapped roots of the Jacobi polynomial
P_k^(1,0) plus the right endpoint; weights = integrals of the nodal Lagrange
cardinals; K_t[i,j] = int l_j' l_i + l_j(0) l_i(0) by (2k+2)-point
Gauss-Legendre).  These are tiny (k+1)-sized host arrays; they are computed
once here and passed to the device verbatim.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from numpy.polynomial import Polynomial
from scipy.special import roots_jacobi

__all__ = ["TimeBasis", "TimeMatrices", "gauss_radau", "temporal_matrices", "lagrange_weights_at"]

MAX_DEGREE = 6  # timebasis.py:36


@dataclass(frozen=True)
class TimeBasis:
    k: int
    nodes: np.ndarray
    weights: np.ndarray


@dataclass(frozen=True)
class TimeMatrices:
    M_t: np.ndarray
    K_t: np.ndarray
    m_t: np.ndarray


def _cardinals(nodes: np.ndarray):
    out = []
    for mu in range(nodes.size):
        rest = np.delete(nodes, mu)
        poly = Polynomial.fromroots(rest) if rest.size else Polynomial([1.0])
        out.append(poly / poly(nodes[mu]))
    return out


def gauss_radau(k: int) -> TimeBasis:
    """(k+1)-point right Gauss-Radau rule on (0, 1] (timebasis.py:67-82)."""
    if not 0 <= k <= MAX_DEGREE:
        raise ValueError(f"temporal degree k must lie in [0, {MAX_DEGREE}], got {k}")
    if k == 0:
        return TimeBasis(0, np.array([1.0]), np.array([1.0]))
    roots, _ = roots_jacobi(k, 1.0, 0.0)
    nodes = np.append((roots + 1.0) / 2.0, 1.0)
    weights = np.array([c.integ()(1.0) - c.integ()(0.0) for c in _cardinals(nodes)])
    return TimeBasis(k, nodes, weights)


def lagrange_weights_at(nodes: np.ndarray, that: float) -> np.ndarray:
    """Values l_mu(that) of all nodal cardinals (timebasis.py:85-93 order of
    operations: running product over nu != mu)."""
    k1 = nodes.size
    out = np.ones(k1)
    for mu in range(k1):
        val = 1.0
        for nu in range(k1):
            if nu != mu:
                val = val * (that - nodes[nu]) / (nodes[mu] - nodes[nu])
        out[mu] = val
    return out


def temporal_matrices(basis: TimeBasis) -> TimeMatrices:
    """M_t, K_t, m_t by (2k+2)-point Gauss-Legendre (timebasis.py:103-119)."""
    k = basis.k
    gx, gw = np.polynomial.legendre.leggauss(2 * k + 2)
    gx = (gx + 1.0) / 2.0
    gw = gw / 2.0
    vals = np.array([[lagrange_weights_at(basis.nodes, t)[mu] for t in gx] for mu in range(k + 1)])
    ders = np.array([c.deriv()(gx) for c in _cardinals(basis.nodes)])
    at0 = lagrange_weights_at(basis.nodes, 0.0)
    M_t = np.einsum("q,jq,iq->ij", gw, vals, vals)
    K_t = np.einsum("q,jq,iq->ij", gw, ders, vals) + np.outer(at0, at0)
    return TimeMatrices(M_t=M_t, K_t=K_t, m_t=at0)
