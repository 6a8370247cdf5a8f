"""Seeded synthetic slab inputs shared by the oracle harness, the GPU tests
and ``bench.py``.  Nothing here is measured; it only makes
bit-identical numpy inputs from a config name and a seed.

Draw order (fixed, so every consumer sees the same numbers):
  1. mode amplitudes a ~ U[-1,1]^{M x 2}
  2. integer wavenumbers (k_m, l_m) ~ U{1..4}^{M x 2}
  3. per Radau node mu: noise eps_mu ~ noise * N(0,1)^{Mv}, pressure ~ U[-1,1]^{Mp}
  4. direction x ~ U[-1,1]^{N_dof}
  5. Vanka initial guess d0 ~ U[-1,1]^{N_dof}   (the right-hand side is r = x)

State velocity: v(x,y) = sum_m (a_m1 sin(pi k_m x) cos(pi l_m y),
                                 a_m2 cos(pi k_m x) sin(pi l_m y))
interpolated at the Q2 nodes (row-major y, x; interleaved components, the
layout of femspace.py:119-125 / femspace.py:176-182), then
U_mu,v = (1 + that_mu) v + eps_mu so that node states differ in time.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["SynthConfig", "CONFIGS", "SynthSlab", "make_slab_inputs", "q2_node_coords"]


@dataclass(frozen=True)
class SynthConfig:
    name: str
    nx: int
    ny: int
    k: int
    p: float
    delta: float
    nu: float
    nu_inf: float
    modes: int
    seed: int
    tau: float = 0.01
    gamma1: float = 40.0  # BASELINE "10 k^2" with k_space = 2
    gamma2: float = 40.0
    gamma_cip: float = 1.0
    noise: float = 1.0e-3
    variant: str = "modn"  # sigma_max = nu (harness.py:49-58)
    rep_fraction: float = 1.0  # BASELINE: frozen at the last Radau point
    omega: float = 0.7
    extents: tuple = (0.0, 0.0, 1.0, 1.0)


CONFIGS = {
    # BASELINE.json configs[0]: the CPU-runnable oracle case.
    "cfg1": SynthConfig("cfg1", 8, 8, 1, 1.5, 1.0e-2, 1.0, 1.0e-3, 4, 20260101),
    # BASELINE.json configs[1]: the headline single-GPU workload.
    "cfg2": SynthConfig("cfg2", 256, 256, 1, 1.3, 1.0e-3, 1.0, 0.0, 16, 20260102),
    # configs[2] as the oracle-checkable Q2/P1disc + DG(2) proxy.
    "cfg3": SynthConfig("cfg3", 1024, 1024, 2, 1.1, 1.0e-4, 1.0, 1.0e-4, 16, 20260103),
    # configs[4] sizes (2048^2, DG(1)).
    "cfg5": SynthConfig("cfg5", 2048, 2048, 1, 1.2, 1.0e-4, 1.0, 0.0, 16, 20260105),
}


def q2_node_coords(nx: int, ny: int, extents=(0.0, 0.0, 1.0, 1.0)):
    """Q2 node coordinates on the half-cell grid, row-major (y, x)."""
    x0, y0, x1, y1 = extents
    hx, hy = (x1 - x0) / nx, (y1 - y0) / ny
    xs = x0 + 0.5 * hx * np.arange(2 * nx + 1)
    ys = y0 + 0.5 * hy * np.arange(2 * ny + 1)
    xx, yy = np.meshgrid(xs, ys)
    return xx.ravel(), yy.ravel()


@dataclass
class SynthSlab:
    cfg: SynthConfig
    nodes: np.ndarray  # Radau nodes on (0, 1]
    U: np.ndarray  # (k+1, nd) linearization state
    x: np.ndarray  # (k+1)*nd direction
    d0: np.ndarray  # (k+1)*nd Vanka initial guess
    v_minus: np.ndarray  # (Mv,) incoming trace (unperturbed modal field)
    vfield: np.ndarray = field(repr=False, default=None)

    @property
    def r(self) -> np.ndarray:
        return self.x


def make_slab_inputs(cfg: SynthConfig | str, nodes: np.ndarray | None = None, seed: int | None = None) -> SynthSlab:
    """Generate the seeded slab inputs of one config.

    ``nodes`` are the Radau nodes of degree cfg.k (pass the host-computed
    ones); if omitted they are computed by ``radau.gauss_radau``.
    """
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    if nodes is None:
        from .radau import gauss_radau

        nodes = gauss_radau(cfg.k).nodes
    nodes = np.asarray(nodes, dtype=float)
    rng = np.random.default_rng(cfg.seed if seed is None else seed)
    nx, ny, k1 = cfg.nx, cfg.ny, cfg.k + 1
    nnodes = (2 * nx + 1) * (2 * ny + 1)
    mv, mp = 2 * nnodes, 3 * nx * ny
    nd = mv + mp

    amp = rng.uniform(-1.0, 1.0, size=(cfg.modes, 2))
    wav = rng.integers(1, 5, size=(cfg.modes, 2))
    # the node grid is a tensor product, so each mode is an outer product of
    # 1-D factors: elementwise the same operations (and bits) as evaluating
    # amp * sin(pi k X) * cos(pi l Y) on the full (2ny+1) x (2nx+1) grid
    x0, y0, x1, y1 = cfg.extents
    xs = x0 + 0.5 * ((x1 - x0) / nx) * np.arange(2 * nx + 1)
    ys = y0 + 0.5 * ((y1 - y0) / ny) * np.arange(2 * ny + 1)
    v = np.zeros((2 * ny + 1, 2 * nx + 1, 2))
    for m in range(cfg.modes):
        km, lm = wav[m]
        v[:, :, 0] += (amp[m, 0] * np.sin(np.pi * km * xs))[None, :] * np.cos(np.pi * lm * ys)[:, None]
        v[:, :, 1] += (amp[m, 1] * np.cos(np.pi * km * xs))[None, :] * np.sin(np.pi * lm * ys)[:, None]
    vflat = v.reshape(-1)

    U = np.empty((k1, nd))
    for mu in range(k1):
        eps = cfg.noise * rng.standard_normal(mv)
        pi = rng.uniform(-1.0, 1.0, size=mp)
        U[mu, :mv] = (1.0 + nodes[mu]) * vflat + eps
        U[mu, mv:] = pi
    x = rng.uniform(-1.0, 1.0, size=k1 * nd)
    d0 = rng.uniform(-1.0, 1.0, size=k1 * nd)
    return SynthSlab(cfg=cfg, nodes=nodes, U=U, x=x, d0=d0, v_minus=vflat.copy(), vfield=vflat)
