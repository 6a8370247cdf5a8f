"""The drop-in seam driven with the REFERENCE's own objects (CPU, build
container only: needs /root/reference).

A pdflow harness builds its preconditioner as ``StmgFactory(setup.geometry,
mg)`` (bench/harness.py:140) and the Newton driver calls
``factory.mg.rebuild_rho`` and ``factory.build(ctx, U, variant).apply(r)``
(newton.py:129-137, 204-220); ``march`` catches ``SlabSolveError``
(slab.py:256-258).  This test runs that sequence with pdflow's SlabContext,
MgGeometry, MgConfig and TangentVariant against this package's mirror, with
libpdst replaced by a recording fake, and checks what crosses the C ABI:
the mesh and its side tags, K_t / m_t / Radau nodes and weights (bitwise),
the Nitsche / CIP gammas, the variant kind and sigma_max, the state U, the
level count and the V-cycle's smoothing parameters.  It runs in a
subprocess with pdflow on PYTHONPATH so the package binds pdflow's
exception classes at import.
"""

import os
import subprocess
import sys

import pytest

REF = "/root/reference/pkg/src"
ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))

pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="pdflow (the reference) is not present here")

SCRIPT = r'''
import ctypes as C
import numpy as np

import pdflow.slab as pslab
from pdflow import constitutive as law
from pdflow.forms import Discretization, DiscretizationConfig, ProblemData
from pdflow.mesh import DIRICHLET, NEUMANN, boundary_tag_assign, uniform_mesh
from pdflow.solver.multigrid import MgConfig as RefMgConfig, MgGeometry as RefMgGeometry, SingularPatchError as RefSPE
from pdflow.timebasis import gauss_radau, temporal_matrices

import paper_2603_28706_b200 as pkg
from paper_2603_28706_b200 import _lib as L
from paper_2603_28706_b200 import errors

# -- 1. pdflow's exception classes are the ones the package raises
assert errors.PDFLOW_EXCEPTIONS
assert errors.SlabSolveError is pslab.SlabSolveError
assert errors.SingularPatchError is RefSPE
assert errors.ConstitutiveDomainError is law.ConstitutiveDomainError
from paper_2603_28706_b200 import newton as pnewton
assert pnewton.SlabSolveError is pslab.SlabSolveError


def fails(ctx, U0):
    raise errors.SlabSolveError("krylov", "device FGMRES stalled", None)


# -- 2. a recording stand-in for libpdst
class Rec:
    def __init__(self):
        self.calls = []
        self.levels = []

    def __getattr__(self, name):
        def fn(*args):
            self.calls.append((name, args))
            impl = type(self).__dict__.get("_" + name)
            return impl(self, *args) if impl is not None else 0
        return fn

    def _pdst_last_error(self, *a):
        return b"fake"

    def _pdst_create(self, m, t, d, p, tau, device, comm, h):
        h._obj.value = 4242
        mesh = m._obj
        self.nx, self.ny = mesh.nx, mesh.ny
        nbf = 2 * (mesh.nx + mesh.ny)
        self.tags = np.array([mesh.dirichlet[i] for i in range(nbf)])
        tm = t._obj
        k1 = tm.k + 1
        self.k1 = k1
        self.nodes = np.array([tm.nodes[i] for i in range(k1)])
        self.weights = np.array([tm.weights[i] for i in range(k1)])
        self.K_t = np.array([tm.K_t[i] for i in range(k1 * k1)]).reshape(k1, k1)
        self.m_t = np.array([tm.m_t[i] for i in range(k1)])
        dd = d._obj
        self.gammas = (dd.gamma1, dd.gamma2, dd.gamma_cip, dd.enable_viscous, dd.enable_convection, dd.enable_pressure)
        pp = p._obj
        self.params = (pp.p, pp.delta, pp.nu, pp.nu_inf)
        self.tau = tau
        return 0

    def _nd(self, nx, ny):
        return 2 * (2 * nx + 1) * (2 * ny + 1) + 3 * nx * ny

    def _pdst_sizes(self, h, mv, mp, nd, ndof):
        mv._obj.value = 2 * (2 * self.nx + 1) * (2 * self.ny + 1)
        mp._obj.value = 3 * self.nx * self.ny
        nd._obj.value = self._nd(self.nx, self.ny)
        ndof._obj.value = self.k1 * self._nd(self.nx, self.ny)
        return 0

    def _pdst_linearize(self, h, U, kind, sigma, where):
        n = self.k1 * self._nd(self.nx, self.ny)
        self.U = np.frombuffer((C.c_double * n).from_address(U.value), dtype=np.float64).copy()
        self.kind, self.sigma = kind, sigma
        return 0

    def _pdst_hierarchy_depth(self, h, depth, nl):
        self.levels = [(self.nx >> (depth - 1 - l), self.ny >> (depth - 1 - l)) for l in range(depth)]
        nl._obj.value = depth
        return 0

    def _pdst_level_sizes(self, h, level, nx, ny, nd):
        a, b = self.levels[level]
        nx._obj.value, ny._obj.value = a, b
        nd._obj.value = self.k1 * self._nd(a, b)
        return 0

    def _pdst_vcycle(self, h, r, z, pre, post, omega, where):
        n = self.k1 * self._nd(self.nx, self.ny)
        (C.c_double * n).from_address(z.value)[:] = [0.5] * n
        self.vcycle = (pre, post, omega, where)
        return 0


fake = Rec()
L._lib = fake

# -- 3. the reference harness's construction (bench/harness.py:100-140)
nx = 8
mesh = boundary_tag_assign(uniform_mesh(nx, nx), lambda f: NEUMANN if f.side == "right" else DIRICHLET)
disc = Discretization(mesh)
config = DiscretizationConfig(gamma1=123.0, gamma2=77.0, gamma_cip=0.25)
params = law.ModelParams(1.4, 2e-3, 0.9, 1e-3)
basis = gauss_radau(2)
tmat = temporal_matrices(basis)
rng = np.random.default_rng(3)
ctx = pslab.SlabContext(disc=disc, params=params, config=config, data=ProblemData(f=None, g_d=None, v0=None),
                        basis=basis, tmat=tmat, t_start=0.2, tau=0.05, v_minus=rng.standard_normal(disc.n_velocity))
mg = RefMgConfig(min_cells=2, rep_fraction=1.0, pre_smooth=3, post_smooth=1, omega=0.6)
geometry = RefMgGeometry.from_fine(disc, min_cells=mg.min_cells)

from paper_2603_28706_b200.stmg import StmgFactory, StmgPreconditioner
from paper_2603_28706_b200.smoother import vanka_smooth

factory = StmgFactory(geometry, mg)
assert factory.mg.rebuild_rho == 0.9 and factory.mg.rebuild_factor == 2.0
variant = law.modified_newton(0.37)
U = rng.standard_normal((3, disc.ndof))
pre = factory.build(ctx, U, variant)
assert isinstance(pre, StmgPreconditioner)

# what crossed the ABI
assert (fake.nx, fake.ny) == (8, 8)
exp_tags = np.array([t == DIRICHLET for t in mesh.boundary_tags], dtype=np.uint8)
assert np.array_equal(fake.tags, exp_tags) and fake.tags.sum() == 3 * nx
for got, ref in ((fake.K_t, tmat.K_t), (fake.m_t, tmat.m_t), (fake.nodes, basis.nodes), (fake.weights, basis.weights)):
    assert np.array_equal(got.view(np.uint64), np.ascontiguousarray(ref, dtype=np.float64).view(np.uint64))
assert fake.gammas == (123.0, 77.0, 0.25, 1, 1, 1)
assert fake.params == (1.4, 2e-3, 0.9, 1e-3) and fake.tau == 0.05
assert fake.kind == L.KIND["modn"] and fake.sigma == 0.37
assert np.array_equal(fake.U, U.reshape(-1))
assert pre.num_levels == geometry.num_levels == 3
assert [lv.disc for lv in pre.levels] == list(geometry.discs)
names = [c[0] for c in fake.calls]
assert "pdst_hierarchy_depth" in names and "pdst_patches_build" in names
sc = [c for c in fake.calls if c[0] == "pdst_set_coarse_solver"][0][1]
assert sc[1] == 0  # dense coarsest solve (the reference's LU), pdflow MgConfig has no coarse_solver
pb_args = [c for c in fake.calls if c[0] == "pdst_patches_build"][0][1]
assert pb_args[1] == 1 and pb_args[2] == 1.0  # surrogate at rep_fraction 1.0

# the preconditioner's apply(flat) -> flat (newton.py:215-220)
z = pre.apply(np.ones(ctx.ndof))
assert z.shape == (ctx.ndof,) and np.all(z == 0.5)
assert fake.vcycle == (3, 1, 0.6, L.HOST)

# vanka_smooth on a level of the device hierarchy (multigrid.py:327)
vanka_smooth(pre.levels[1], np.zeros(pre.levels[1].slab_dim), np.ones(pre.levels[1].slab_dim), 2, 0.6)
va = [c for c in fake.calls if c[0] == "pdst_vanka"][-1][1]
assert va[1] == 1 and va[4] == 2 and va[5] == 0.6
assert np.array_equal(pre.levels[2].patches.ids[:, :21], disc.cell_patch_dofs)
assert np.array_equal(pre.levels[2].patches.ids[:, 21:42], disc.cell_patch_dofs + disc.ndof)

# a pdflow level (patches on the host) is refused, not silently run on the CPU
try:
    vanka_smooth(geometry, None, None, 1, 0.7)
    raise SystemExit("foreign level accepted")
except TypeError:
    pass

# the geometry must be built on the slab's own Discretization (multigrid.py:404-405)
other = RefMgGeometry.from_fine(Discretization(mesh), min_cells=2)
try:
    StmgPreconditioner(other, ctx, U, variant, mg)
    raise SystemExit("geometry identity not checked")
except ValueError:
    pass

# libpdst's error codes surface as pdflow's exceptions
try:
    L.check(L.ESINGULAR, "x", level=1, patch=7)
except RefSPE as e:
    assert (e.level, e.patch) == (1, 7)
try:
    L.check(L.EDOMAIN, "x")
    raise SystemExit("no domain error")
except law.ConstitutiveDomainError:
    pass

# -- 4. march converts a device-solver failure into MarchError (slab.py:256-258)
class P2:
    disc = disc

    def context(self, t0, t1, v_minus):
        return ctx


class Part:
    def intervals(self):
        return [(0.0, 0.05)]


try:
    pslab.march(P2(), Part(), np.zeros(disc.n_velocity), fails)
    raise SystemExit("march did not fail")
except pslab.MarchError as e:
    assert e.index == 0 and e.cause.kind == "krylov"
print("seam ok")
'''


def test_mirror_driven_by_pdflow_objects():
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REF, ROOT]))
    res = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=env, capture_output=True, text=True,
                         timeout=300)
    assert res.returncode == 0 and "seam ok" in res.stdout, res.stdout[-3000:] + res.stderr[-3000:]
