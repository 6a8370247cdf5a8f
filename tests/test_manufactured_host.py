"""Host side of the manufactured-solution problem (no GPU): the package's
ManufacturedCase fields against the reference's own forcing (golden vectors
from tests/golden/make_golden_manufactured.py), and eoc."""

import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
_S = np.array([0.06943184420297371, 0.33000947820757187, 0.6699905217924281, 0.9305681557970262])


def volume_points(nx, ny):
    hx, hy = 1.0 / nx, 1.0 / ny
    ox, oy = np.meshgrid(np.arange(nx) * hx, np.arange(ny) * hy)
    px, py = np.repeat(_S, 4), np.tile(_S, 4)  # q = 4 qx + qy
    return ox.ravel()[:, None] + px[None] * hx, oy.ravel()[:, None] + py[None] * hy


@pytest.mark.parametrize("name", ["mf_a", "mf_b"])
def test_forcing_matches_reference(name):
    from paper_2603_28706_b200.manufactured import ManufacturedCase
    from paper_2603_28706_b200.problem import ModelParams

    g = np.load(os.path.join(GOLD, f"{name}.npz"))
    case = ManufacturedCase(ModelParams(*g["params"]))
    X, Y = volume_points(int(g["nx"]), int(g["ny"]))
    for mu, node in enumerate(g["nodes"]):
        f = case.forcing(X, Y, float(g["t0"]) + float(g["tau"]) * node)
        ref = g["f_qp"][mu]
        assert np.abs(f - ref).max() <= 1e-12 * np.abs(ref).max()


def test_fields_divergence_free_and_boundary():
    from paper_2603_28706_b200.manufactured import ManufacturedCase
    from paper_2603_28706_b200.problem import ModelParams

    case = ManufacturedCase(ModelParams(1.5, 1e-2, 1.0, 0.0))
    rng = np.random.default_rng(1)
    x, y = rng.uniform(0, 1, 50), rng.uniform(0, 1, 50)
    g = case.velocity_grad(x, y, 0.7)
    assert np.abs(g[:, 0, 0] + g[:, 1, 1]).max() < 1e-14
    edge = np.linspace(0, 1, 11)
    for xx, yy in ((edge, 0 * edge), (edge, 0 * edge + 1), (0 * edge, edge), (0 * edge + 1, edge)):
        assert np.abs(case.velocity(xx, yy, 0.7)).max() < 1e-15


def test_eoc():
    from paper_2603_28706_b200.metrics import eoc

    assert eoc([1.0, 0.25, 0.0625, 0.0]) == [2.0, 2.0, None]
