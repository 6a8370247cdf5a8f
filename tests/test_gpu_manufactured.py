"""GPU parity of the manufactured-solution problem: the
device forcing and error norms against the reference's own outputs
(tests/golden/mf_*.npz), and the residual with the device forcing against the
residual with the same forcing evaluated on the host."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _setup(name):
    from paper_2603_28706_b200 import problem as pb
    from paper_2603_28706_b200.manufactured import ManufacturedCase

    g = np.load(os.path.join(GOLD, f"{name}.npz"))
    params = pb.ModelParams(*g["params"])
    case = ManufacturedCase(params)
    ctx = pb.make_context(int(g["nx"]), int(g["ny"]), int(g["k"]), params, float(g["tau"]),
                          f=case.forcing, t_start=float(g["t0"]))
    return g, case, ctx


@pytest.mark.parametrize("name", ["mf_a", "mf_b"])
def test_device_forcing_matches_reference(name):
    from paper_2603_28706_b200 import _lib as L
    from paper_2603_28706_b200.operators import SlabDevice

    g, case, ctx = _setup(name)
    dev = SlabDevice(ctx)
    out = np.zeros(g["f_qp"].shape)
    L.check(L.lib().pdst_manufactured_forcing(dev.h, float(g["t0"]), L.vptr(out), L.HOST))
    ref = g["f_qp"]
    assert np.abs(out - ref).max() <= 1e-12 * np.abs(ref).max()
    dev.close()


@pytest.mark.parametrize("name", ["mf_a", "mf_b", "mf_c"])
def test_error_norms_match_reference(name):
    from paper_2603_28706_b200.metrics import error_norms
    from paper_2603_28706_b200.radau import gauss_radau

    g, case, ctx = _setup(name)

    class Part:
        def intervals(self):
            t = g["times"]
            return [(float(t[i]), float(t[i + 1])) for i in range(len(t) - 1)]

    basis = gauss_radau(int(g["k"]))
    e_phi, e_div = error_norms(ctx.disc, basis, Part(), list(g["traj"]), case)
    assert abs(e_phi - float(g["e_phi"])) <= 1e-12 * float(g["e_phi"])
    assert abs(e_div - float(g["e_div"])) <= 1e-12 * float(g["e_div"])
    e_phi, e_div = error_norms(ctx.disc, basis, Part(), list(g["traj"]), case, spatial_order=3, temporal_points=2)
    assert abs(e_phi - float(g["e_phi_q3t2"])) <= 1e-12 * float(g["e_phi_q3t2"])
    assert abs(e_div - float(g["e_div_q3t2"])) <= 1e-12 * float(g["e_div_q3t2"])


@pytest.mark.parametrize("name", ["mf_a", "mf_b"])
def test_residual_with_device_forcing(name):
    import dataclasses

    from paper_2603_28706_b200.operators import slab_residual
    from paper_2603_28706_b200.problem import ProblemData

    g, case, ctx = _setup(name)
    U = g["traj"][0]
    R_dev = slab_residual(ctx, U)  # ctx.data.f is case.forcing: device path
    ctx_host = dataclasses.replace(ctx, data=ProblemData(f=lambda x, y, t: case.forcing(x, y, t)))
    R_host = slab_residual(ctx_host, U)
    assert np.linalg.norm(R_dev - R_host) <= 1e-12 * np.linalg.norm(R_host)
