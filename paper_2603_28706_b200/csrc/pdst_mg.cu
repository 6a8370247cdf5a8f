// pdst_mg.cu — integer maps, Vanka patches / sweeps and the multigrid entry
// points of the C ABI (include/pdst.h).
//
// Reference: solver/multigrid.py:164-191 (hierarchy), :261-299 (patches),
// :327-340 (vanka_smooth), :475-488 (surrogate), femspace.py:127-140 and
// forms.py:192-196 (dof maps).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../include/pdst.h"
#include "pdst_handle.h"
#include "pdst_device.cuh"
#include "pdst_coarse.h"
#include "pdst_patch.h"

using namespace pdst;

// PDST_DEBUG_SYNC=1 synchronizes after every launch so a fault names its kernel.
static bool debug_sync() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("PDST_DEBUG_SYNC");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

#define CK(expr)                                                                               \
  do {                                                                                         \
    cudaError_t _e = (expr);                                                                   \
    if (_e == cudaSuccess && debug_sync()) {                                                   \
      _e = cudaDeviceSynchronize();                                                            \
      fprintf(stderr, "[pdst] %s -> %s\n", #expr, cudaGetErrorString(_e));                    \
    }                                                                                          \
    if (_e != cudaSuccess) return set_error(PDST_ECUDA, "%s: %s", #expr, cudaGetErrorString(_e)); \
  } while (0)

namespace {

__global__ void k_cell_maps(int nx, int ny, int nd, int k1, int64_t* cell_nodes, int64_t* patch_ids) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nx * ny) return;
  const int ci = c % nx, cj = c / nx;
  const int nnx = 2 * nx + 1;
  const int64_t mv = 2LL * nnx * (2 * ny + 1);
  const int D = 21 * k1;
  for (int a = 0; a < 9; ++a) {
    const int64_t node = (int64_t)(2 * cj + a / 3) * nnx + 2 * ci + a % 3;
    cell_nodes[(int64_t)c * 9 + a] = node;
    for (int mu = 0; mu < k1; ++mu) {
      patch_ids[(int64_t)c * D + 21 * mu + 2 * a] = 2 * node + (int64_t)mu * nd;
      patch_ids[(int64_t)c * D + 21 * mu + 2 * a + 1] = 2 * node + 1 + (int64_t)mu * nd;
    }
  }
  for (int mu = 0; mu < k1; ++mu)
    for (int j = 0; j < 3; ++j) patch_ids[(int64_t)c * D + 21 * mu + 18 + j] = mv + 3LL * c + j + (int64_t)mu * nd;
}

// Lagrange cardinals at `that` in the operation order of timebasis.py:85-93.
std::vector<double> lagrange_at(const std::vector<double>& nodes, double that) {
  const int k1 = (int)nodes.size();
  std::vector<double> out(k1);
  for (int mu = 0; mu < k1; ++mu) {
    double r = 1.0;
    for (int nu = 0; nu < k1; ++nu)
      if (nu != mu) r = r * (that - nodes[nu]) / (nodes[mu] - nodes[nu]);
    out[mu] = r;
  }
  return out;
}

}  // namespace

namespace pdst {
void destroy_child(pdst_handle* c) { pdst_destroy(c); }
}  // namespace pdst

extern "C" {
static int build_rediscretized(pdst_handle* h, int* bad_level, int64_t* bad_patch);
}

namespace {

Level* finest(pdst_handle* h) {
  if (h->levels.empty()) {
    Level* l = new Level();
    l->g = h->g;  // shares the handle's dirichlet flags (not owned)
    l->dirichlet_host = h->dirichlet_host;
    l->all_dirichlet = true;
    for (auto f : h->dirichlet_host) l->all_dirichlet = l->all_dirichlet && f == 1;
    h->levels.push_back(l);
  }
  return h->levels.back();
}

int check_level(pdst_handle* h, int level) {
  if (level < 0 || level >= (int)h->levels.size()) return set_error(PDST_EINVAL, "level %d out of range", level);
  return PDST_OK;
}

}  // namespace

extern "C" {

int pdst_cell_maps(pdst_handle* h, int64_t* cell_nodes, int64_t* patch_ids) {
  if (h && h->g.th) return set_error(PDST_ENOTSUP, "pdst_cell_maps is Q2/P1disc-only (Taylor-Hood handles: apply, residual, mass)");
  if (!h || !cell_nodes || !patch_ids) return set_error(PDST_EINVAL, "null argument");
  CK(cudaSetDevice(h->device));
  const Geom& g = h->g;
  const int k1 = h->td.k1;
  int64_t* dev = nullptr;
  const size_t n1 = (size_t)g.ncells * 9, n2 = (size_t)g.ncells * 21 * k1;
  CK(cudaMalloc(&dev, (n1 + n2) * sizeof(int64_t)));
  PDST_LAUNCH(k_cell_maps<<<(g.ncells + 127) / 128, 128, 0, h->stream>>>(g.nx, g.ny, g.nd, k1, dev, dev + n1));
  cudaError_t e = cudaMemcpyAsync(cell_nodes, dev, n1 * sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(patch_ids, dev + n1, n2 * sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  cudaFree(dev);
  if (e != cudaSuccess) return set_error(PDST_ECUDA, "cell maps: %s", cudaGetErrorString(e));
  return PDST_OK;
}

static int build_hierarchy(pdst_handle* h, int min_cells, int depth, int* num_levels);

int pdst_hierarchy(pdst_handle* h, int min_cells, int* num_levels) {
  if (h && h->g.th) return set_error(PDST_ENOTSUP, "the multigrid hierarchy is Q2/P1disc-only (Taylor-Hood handles: apply, residual, mass)");
  return build_hierarchy(h, min_cells, 0, num_levels);
}

// A hierarchy of exactly `depth` levels regardless of min_cells: a rank's
// strip of a partitioned mesh coarsens as often as the global mesh does.
int pdst_hierarchy_depth(pdst_handle* h, int depth, int* num_levels) {
  if (h && h->g.th) return set_error(PDST_ENOTSUP, "the multigrid hierarchy is Q2/P1disc-only (Taylor-Hood handles: apply, residual, mass)");
  if (depth < 1) return set_error(PDST_EINVAL, "depth must be >= 1");
  return build_hierarchy(h, 0, depth, num_levels);
}

static int build_hierarchy(pdst_handle* h, int min_cells, int depth, int* num_levels) {
  if (!h) return set_error(PDST_EINVAL, "null handle");
  CK(cudaSetDevice(h->device));
  for (auto* l : h->levels) delete l;
  h->levels.clear();
  h->patches_valid = false;
  h->coarse_valid = false;
  h->min_cells = min_cells;
  // coarsen while nx > min_cells and even, same for ny (multigrid.py:170)
  std::vector<Level*> chain;
  Level* f = new Level();
  f->g = h->g;
  f->dirichlet_host = h->dirichlet_host;
  chain.push_back(f);
  while (true) {
    const Level* m = chain.back();
    const int nx = m->g.nx, ny = m->g.ny;
    if (depth > 0) {
      if ((int)chain.size() == depth) break;
      if (nx % 2 || ny % 2) {
        for (auto* l : chain) delete l;
        return set_error(PDST_EINVAL, "a %dx%d level cannot be coarsened (depth %d)", nx, ny, depth);
      }
    } else if (!(nx > min_cells && nx % 2 == 0 && ny > min_cells && ny % 2 == 0)) {
      break;
    }
    Level* c = new Level();
    const int cnx = nx / 2, cny = ny / 2;
    // coarse faces inherit the tag of the first fine face of their side (multigrid.py:174-182)
    const int off_f[4] = {0, nx, nx + ny, 2 * nx + ny};
    const int cnt_c[4] = {cnx, cny, cnx, cny};
    for (int side = 0; side < 4; ++side)
      for (int i = 0; i < cnt_c[side]; ++i) c->dirichlet_host.push_back(m->dirichlet_host[off_f[side]]);
    if (cudaMalloc(&c->dirichlet, c->dirichlet_host.size()) != cudaSuccess) return set_error(PDST_ECUDA, "cudaMalloc");
    CK(cudaMemcpy(c->dirichlet, c->dirichlet_host.data(), c->dirichlet_host.size(), cudaMemcpyHostToDevice));
    c->g = make_geom(cnx, cny, h->extents[0], h->extents[1], h->extents[2], h->extents[3], c->dirichlet);
    chain.push_back(c);
  }
  for (auto it = chain.rbegin(); it != chain.rend(); ++it) {
    Level* l = *it;
    l->all_dirichlet = true;
    for (auto v : l->dirichlet_host) l->all_dirichlet = l->all_dirichlet && v == 1;
    h->levels.push_back(l);
  }
  if (num_levels) *num_levels = (int)h->levels.size();
  return PDST_OK;
}

int pdst_level_sizes(pdst_handle* h, int level, int32_t* nx, int32_t* ny, int64_t* ndof) {
  if (!h) return set_error(PDST_EINVAL, "null handle");
  finest(h);
  if (int e = check_level(h, level)) return e;
  const Geom& g = h->levels[level]->g;
  if (nx) *nx = g.nx;
  if (ny) *ny = g.ny;
  if (ndof) *ndof = (int64_t)h->td.k1 * g.nd;
  return PDST_OK;
}

// Scratch of a coarse level apply (grown to the largest level used).
static double* level_scratch(pdst_handle* h, int l) {
  return h->lvs.ensure(level_apply_scratch(h->levels[l]->g, h->td.k1));
}

// Level operator descriptor of level l (element form).
static LevelOp level_op(pdst_handle* h, int l) {
  Level* lv = h->levels[l];
  LevelOp op{};
  op.g = lv->g;
  op.ds = h->ds;
  op.fine = l == (int)h->levels.size() - 1;
  op.ecell = lv->ecell.ptr;
  op.fv = lv->efx.ptr;
  op.fh = lv->efy.ptr;
  op.state = h->state.ptr;
  return op;
}

// Build-only / read-back arrays above this many doubles (2 GiB) are released
// after the build (the large meshes of configs 3 and 5).
constexpr size_t kKeepMats = (size_t)1 << 28;

static int invert_level_patches(pdst_handle* h, int l, int* badi, int* bad_level, int64_t* bad_patch) {
  Level* lv = h->levels[l];
  const int k1 = h->td.k1, D = 21 * k1;
  const size_t nc = lv->g.ncells;
  const int init = INT_MAX;
  CK(cudaMemcpyAsync(badi, &init, sizeof(int), cudaMemcpyHostToDevice, h->stream));
  if (lv->diag) {
    CK(patch_invert_diag(lv->g, lv->tdiag, lv->spatial.ptr, lv->binv.ptr, badi,
                         h->stream));
  } else {
    double* invs = lv->invs.ensure(nc * D * D);
    if (!invs) return set_error(PDST_ECUDA, "out of device memory (patch inverses)");
    CK(patch_invert(k1, lv->mats.ptr, invs, (int)nc, badi, h->stream));
  }
  int badh = INT_MAX;
  CK(cudaMemcpyAsync(&badh, badi, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  lv->D = D;
  if (badh != INT_MAX) {
    if (bad_level) *bad_level = l;
    if (bad_patch) *bad_patch = badh;
    return set_error(PDST_ESINGULAR, "singular patch matrix (level %d, patch %d)", l, badh);
  }
  return PDST_OK;
}

int pdst_patches_build(pdst_handle* h, int surrogate, double rep_fraction, int* bad_level, int64_t* bad_patch) {
  if (h && h->g.th) return set_error(PDST_ENOTSUP, "the Vanka patches is Q2/P1disc-only (Taylor-Hood handles: apply, residual, mass)");
  if (!h) return set_error(PDST_EINVAL, "null handle");
  if (!h->linearized) return set_error(PDST_ESTATE, "patches built before pdst_linearize");
  CK(cudaSetDevice(h->device));
  h->patches_valid = false;
  h->coarse_valid = false;
  Level* fl = finest(h);
  const int L = (int)h->levels.size();
  const Geom& g = h->g;
  const int k1 = h->td.k1, D = 21 * k1;
  const size_t nc = g.ncells;
  const bool multilevel = L > 1;
  // a hierarchy with a single level (min_cells >= the mesh): the V-cycle is the
  // dense solve of the whole slab system (multigrid.py:494-547)
  const bool single_solve = L == 1 && h->min_cells > 0;
  double* bad = h->ibuf.ensure(1);
  if (!bad) return set_error(PDST_ECUDA, "out of device memory");
  int* badi = reinterpret_cast<int*>(bad);

  // exact per-node element matrices of the finest level (Galerkin input and exact patches)
  const bool redisc = multilevel && h->coarse_mode == 1;
  const bool need_exact = (multilevel && !redisc) || !surrogate || single_solve;
  if (need_exact) {
    double* ET = fl->ecell.ensure((size_t)k1 * nc * 441);
    if (!ET) return set_error(PDST_ECUDA, "out of device memory (element matrices)");
    const Lin L0 = lin_of(h);
    for (int s = 0; s < k1; ++s)
      CK(element_matrices(g, h->ds, L0, s, h->state.ptr + (size_t)s * g.mv, ET + (size_t)s * nc * 441, h->stream));
  }

  // ---- finest-level patches (surrogate or exact), multigrid.py:475-486 ----
  PatchArgs pa{};
  pa.g = g;
  pa.td = h->td;
  pa.ds = h->ds;
  pa.nslot = surrogate ? 1 : k1;
  if (surrogate) {
    double* ET = h->ET.ensure(nc * 441);
    if (!ET) return set_error(PDST_ECUDA, "out of device memory (element matrices)");
    pa.ET = ET;
    if (k1 > 1) {
      // rep state = sum_mu l_mu(rep_fraction) U_mu (slab.py:105-112), linearized alone
      const std::vector<double> c = lagrange_at(h->nodes, rep_fraction);
      double* sr = h->state_rep.ensure(g.mv);
      double* er = h->eta_rep.ensure(16 * nc);
      double* gr = h->gam_rep.ensure(16 * nc);
      double* efr = h->etaf_rep.ensure((size_t)g.nbf * 4);
      double* gfr = h->gamf_rep.ensure((size_t)g.nbf * 4);
      if (!sr || !er || !gr || !efr || !gfr) return set_error(PDST_ECUDA, "out of device memory");
      CK(blend_velocity(g, k1, c.data(), h->state.ptr, g.mv, sr, h->stream));
      CK(linearize(g, h->model, 1, sr, er, gr, efr, gfr, h->stream));
      Lin Lr = lin_of(h);
      Lr.eta = er;
      Lr.gam = gr;
      Lr.etaf = efr;
      Lr.gamf = gfr;
      CK(element_matrices(g, h->ds, Lr, 0, sr, ET, h->stream));
      pa.state = sr;
    } else {
      // k = 0: the surrogate is node 0 itself (multigrid.py:480)
      CK(element_matrices(g, h->ds, lin_of(h), 0, h->state.ptr, ET, h->stream));
      pa.state = h->state.ptr;
    }
  } else {
    pa.ET = fl->ecell.ptr;
    pa.state = h->state.ptr;
  }
  // Surrogate patches share one spatial block across the Radau nodes: keep it
  // and invert the temporally diagonalized blocks instead of A_K itself.
  fl->diag = surrogate && time_diagonalize(k1, h->td.K_t, h->td.tau_w, fl->tdiag);
  // the full D x D patch matrices are inverted on the exact path; on the
  // diagonalized path nothing needs them (pdst_patch_matrices re-assembles
  // them on request from the retained surrogate element data)
  double* mats = nullptr;
  if (!fl->diag) {
    mats = fl->mats.ensure(nc * D * D);
    if (!mats) return set_error(PDST_ECUDA, "out of device memory (patches)");
  } else {
    fl->mats.release();
  }
  pa.mats = mats;
  pa.spatial = nullptr;
  if (fl->diag) {
    pa.spatial = fl->spatial.ensure(nc * 441);
    if (!pa.spatial || !fl->binv.ensure(nc * fl->tdiag.pstride))
      return set_error(PDST_ECUDA, "out of device memory (diagonalized patches)");
  }
  CK(patch_assemble(pa, h->stream));
  if (int e = invert_level_patches(h, L - 1, badi, bad_level, bad_patch)) return e;

  // ---- coarse levels: Galerkin operators, exact patches (multigrid.py:435-488) ----
  if (redisc) {
    if (int e = build_rediscretized(h, bad_level, bad_patch)) return e;
  }
  for (int l = redisc ? -1 : L - 2; l >= 0; --l) {
    Level* lv = h->levels[l];
    const Geom& gc = lv->g;
    double* ec = lv->ecell.ensure((size_t)k1 * gc.ncells * 441);
    double* fv = lv->efx.ensure((size_t)k1 * std::max(1, (gc.nx - 1) * gc.ny) * 324);
    double* fh = lv->efy.ensure((size_t)k1 * std::max(1, gc.nx * (gc.ny - 1)) * 324);
    if (!ec || !fv || !fh) return set_error(PDST_ECUDA, "out of device memory (coarse operators)");
    CK(galerkin(level_op(h, l + 1), gc, k1, ec, fv, fh, h->stream));
    double* m = lv->mats.ensure((size_t)gc.ncells * D * D);
    if (!m) return set_error(PDST_ECUDA, "out of device memory (coarse patches)");
    lv->diag = false;
    CK(patch_assemble_level(level_op(h, l), h->td, m, h->stream));
    if (int e = invert_level_patches(h, l, badi, bad_level, bad_patch)) return e;
    if ((size_t)gc.ncells * D * D > kKeepMats) lv->mats.release();  // only the inverses are used
    const size_t n = (size_t)k1 * gc.nd;
    if (!lv->w0.ensure(n) || !lv->w1.ensure(n) || !lv->w2.ensure(n) || !lv->w3.ensure(n))
      return set_error(PDST_ECUDA, "out of device memory (level vectors)");
  }
  h->patches_valid = true;
  // build-only element data of the finest level (Galerkin input, surrogate
  // element matrices, the spatial blocks of the diagonalized inverses)
  if ((size_t)k1 * nc * 441 > kKeepMats) {
    fl->ecell.release();
    h->ET.release();
    if (fl->diag) fl->spatial.release();
  }

  // ---- coarsest-level solve (multigrid.py:494-520) ----
  if (redisc) {  // held by the coarsest level's child handle
    h->coarse_valid = true;
    return PDST_OK;
  }
  if (multilevel || single_solve) {
    Level* c0 = h->levels[0];
    const int n = k1 * c0->g.nd;
    // (auto: the single-CTA Gauss-Jordan inverse is O(n^3) on one SM, seconds
    // beyond a few thousand dofs)
    h->coarse_iterative = h->coarse_kind == PDST_COARSE_VANKA || h->coarse_kind == PDST_COARSE_FGMRES ||
                          (h->coarse_kind == PDST_COARSE_AUTO && n > 4096);
    if (h->coarse_iterative) {
      c0->dense.release();
      h->coarse_valid = true;
      return PDST_OK;
    }
    if (n > 16384)
      return set_error(PDST_ENOTSUP, "coarsest level too large for the dense solve (%d dofs); "
                                     "use pdst_set_coarse_solver", n);
    double* A = c0->dense.ensure((size_t)n * n);
    double* scr = c0->ipiv.ensure((size_t)n / 2 + 2);
    if (!A || !scr) return set_error(PDST_ECUDA, "out of device memory (coarse solve)");
    int* piv = reinterpret_cast<int*>(scr + 1);
    CK(cudaMemsetAsync(bad, 0, sizeof(int), h->stream));
    CK(dense_build(level_op(h, 0), h->td, c0->all_dirichlet, A, scr, piv, badi, h->stream));
    int badh = 0;
    CK(cudaMemcpyAsync(&badh, badi, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (badh) return set_error(PDST_ESINGULAR, "singular coarsest-level matrix");
    h->coarse_valid = true;
  }
  return PDST_OK;
}

int pdst_patch_matrices(pdst_handle* h, int level, double* mats) {
  if (!h || !mats) return set_error(PDST_EINVAL, "null argument");
  if (int e = check_level(h, level)) return e;
  Level* l = h->levels[level];
  if (!l->D) return set_error(PDST_ESTATE, "patches not built");
  if (l->child) return pdst_patch_matrices(l->child, 0, mats);
  CK(cudaSetDevice(h->device));
  const size_t n = (size_t)l->g.ncells * l->D * l->D;
  if (!l->mats.ptr && l->diag && level == (int)h->levels.size() - 1 && h->ET.ptr) {
    // diagonalized surrogate patches: assemble the D x D matrices on request
    // from the retained surrogate element matrices (the same kernel and
    // arithmetic as the exact path's assembly)
    DeviceBuffer tmp;
    PatchArgs pa{};
    pa.g = h->g;
    pa.td = h->td;
    pa.ds = h->ds;
    pa.nslot = 1;
    pa.ET = h->ET.ptr;
    pa.state = h->td.k1 > 1 ? h->state_rep.ptr : h->state.ptr;
    pa.mats = tmp.ensure(n);
    if (!pa.mats) return set_error(PDST_ECUDA, "out of device memory (patch read-back)");
    CK(patch_assemble(pa, h->stream));
    CK(cudaMemcpyAsync(mats, pa.mats, n * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return PDST_OK;
  }
  if (!l->mats.ptr) return set_error(PDST_ESTATE, "patch matrices of level %d are not retained at this size", level);
  CK(cudaMemcpyAsync(mats, l->mats.ptr, n * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return PDST_OK;
}

int pdst_patch_info(pdst_handle* h, int level, int32_t* D, int32_t* diag_blocks, int64_t* bytes_per_patch) {
  if (!h) return set_error(PDST_EINVAL, "null handle");
  if (int e = check_level(h, level)) return e;
  Level* l = h->levels[level];
  if (!l->D) return set_error(PDST_ESTATE, "patches not built");
  if (l->child) return pdst_patch_info(l->child, 0, D, diag_blocks, bytes_per_patch);
  if (D) *D = l->D;
  if (diag_blocks) *diag_blocks = l->diag ? l->tdiag.nblk : 0;
  if (bytes_per_patch)
    *bytes_per_patch = l->diag ? (int64_t)l->tdiag.pstride * 8 : (int64_t)l->D * l->D * 8;
  return PDST_OK;
}

// coarse_mode "rediscretize" (multigrid.py:302-324, 406-431): a child handle
// per coarse level, created on the level's mesh (inherited side tags) with the
// slab's time basis, discretization and model, linearized with the same
// tangent at the velocity injected from the next finer level (pressure 0) and
// the injected lifting; its exact patches are the level's patches, its mass
// the level's mass (the coarse mesh's own, multigrid.py:431), and the
// coarsest child solves the coarsest level (dense or iterative, as the
// parent is configured).
static int build_rediscretized(pdst_handle* h, int* bad_level, int64_t* bad_patch) {
  const int L = (int)h->levels.size();
  const int k1 = h->td.k1;
  const double* vf = h->state.ptr;  // (k1, Mv) velocity of the finer level
  size_t sf = h->g.mv;
  Geom gf = h->g;
  const double* ghf = h->has_ghat ? h->ghat.ptr : nullptr;
  std::vector<double> Kt((size_t)k1 * k1), mt(k1);
  for (int i = 0; i < k1; ++i) {
    mt[i] = h->td.m_t[i];
    for (int j = 0; j < k1; ++j) Kt[(size_t)i * k1 + j] = h->td.K_t[i * k1 + j];
  }
  for (int l = L - 2; l >= 0; --l) {
    Level* lv = h->levels[l];
    if (lv->child) {
      destroy_child(lv->child);
      lv->child = nullptr;
    }
    const Geom gc = lv->g;
    pdst_mesh m{gc.nx, gc.ny, h->extents[0], h->extents[1], h->extents[2], h->extents[3], lv->dirichlet_host.data()};
    pdst_time t{k1 - 1, h->nodes.data(), h->weights.data(), Kt.data(), mt.data()};
    pdst_disc d{h->ds.gamma1, h->ds.gamma2, h->ds.gamma_cip, h->ds.viscous, h->ds.convection, h->ds.pressure};
    pdst_params pp{h->model.p, h->model.delta, h->model.nu, h->model.nu_inf};
    pdst_handle* c = nullptr;
    if (int e = pdst_create(&m, &t, &d, &pp, h->tau, h->device, h->stream, &c)) return e;
    lv->child = c;
    double* uc = c->scratch_c.ensure((size_t)k1 * gc.nd);
    if (!uc) return set_error(PDST_ECUDA, "out of device memory (rediscretized level)");
    CK(inject_velocity(gc, gf, k1, vf, sf, uc, gc.nd, true, h->stream));
    if (ghf) {
      double* gh = c->scratch_f.ensure(gc.mv);
      if (!gh) return set_error(PDST_ECUDA, "out of device memory (rediscretized level)");
      CK(inject_velocity(gc, gf, 1, ghf, gf.mv, gh, gc.mv, false, h->stream));
      if (int e = pdst_set_lifting(c, gh, PDST_DEVICE)) return e;
    }
    if (int e = pdst_linearize(c, uc, h->model.kind, h->model.sigma_max, PDST_DEVICE)) return e;
    if (l == 0) {  // the coarsest level: a one-level hierarchy whose V-cycle is the coarse solve
      int nl = 0;
      if (int e = pdst_hierarchy(c, INT_MAX, &nl)) return e;
      if (int e = pdst_set_coarse_solver(c, h->coarse_kind, h->coarse_sweeps, h->coarse_omega, h->coarse_iters,
                                         h->coarse_rtol))
        return e;
    }
    int bl = -1;
    int64_t bp = -1;
    if (int e = pdst_patches_build(c, 0, 0.5, &bl, &bp)) {
      if (e == PDST_ESINGULAR) {
        if (bad_level) *bad_level = l;
        if (bad_patch) *bad_patch = bp;
        return set_error(PDST_ESINGULAR, "singular patch matrix (level %d, patch %lld)", l, (long long)bp);
      }
      return e;
    }
    lv->D = 21 * k1;
    const size_t n = (size_t)k1 * gc.nd;
    if (!lv->w0.ensure(n) || !lv->w1.ensure(n) || !lv->w2.ensure(n) || !lv->w3.ensure(n))
      return set_error(PDST_ECUDA, "out of device memory (level vectors)");
    vf = c->state.ptr;
    sf = gc.mv;
    gf = gc;
    ghf = c->has_ghat ? c->ghat.ptr : nullptr;
  }
  return PDST_OK;
}

// y = r - A_l x on level l (device pointers).
static int level_defect(pdst_handle* h, int l, const double* x, const double* r, double* y) {
  const int L = (int)h->levels.size();
  if (pdst_handle* c = h->levels[l]->child) {  // rediscretized level: its own matrix-free Jacobian
    c->stream = h->stream;
    double* part = c->jpart.ensure_zeroed(jacobian_scratch(c->g, c->td.k1));
    if (!part) return set_error(PDST_ECUDA, "out of device memory");
    CK(PDST_TIMED(h, PK_LEVEL, jacobian_apply(c->g, c->td, c->ds, lin_of(c), x, r, y, part, h->stream)));
    return PDST_OK;
  }
  if (l == L - 1) {
    double* part = h->jpart.ensure_zeroed(jacobian_scratch(h->g, h->td.k1));
    if (!part) return set_error(PDST_ECUDA, "out of device memory");
    CK(PDST_TIMED(h, r ? PK_DEFECT : PK_JACOBIAN,
                  jacobian_apply(h->g, h->td, h->ds, lin_of(h), x, r, y, part, h->stream)));
  } else {
    CK(PDST_TIMED(h, PK_LEVEL, level_apply(level_op(h, l), h->td, x, r, y, level_scratch(h, l), h->stream)));
  }
  return PDST_OK;
}

// `steps` Vanka steps on level l, d updated in place (device pointers).
// zero_start: d is to be taken as zero whatever it holds (the V-cycle's and
// the coarse solvers' smoothing from a zero guess, multigrid.py:545-555): the
// first step's defect r - A 0 is r itself and its update is the increment, so
// that step needs neither the operator apply nor a cleared d (the same values
// as the full step up to the sign of zeros).
static int vanka_level(pdst_handle* h, int l, double* d, const double* r, int steps, double omega,
                       bool zero_start = false) {
  Level* lv = h->levels[l];
  if (lv->child) {  // rediscretized level: the child's exact patches
    lv->child->stream = h->stream;
    return vanka_level(lv->child, 0, d, r, steps, omega, zero_start);
  }
  const Geom& g = lv->g;
  const int k1 = h->td.k1;
  const size_t n = (size_t)k1 * g.nd;
  double* defect = h->defect.ensure(std::max(n, (size_t)k1 * h->g.nd));
  double* upd = h->upd.ensure((size_t)h->g.ncells * 21 * k1);
  if (!defect || !upd) return set_error(PDST_ECUDA, "out of device memory");
  if (zero_start && steps == 0) CK(cudaMemsetAsync(d, 0, n * sizeof(double), h->stream));
  for (int s = 0; s < steps; ++s) {
    const bool from_zero = zero_start && s == 0;
    const double* e_in = defect;
    if (from_zero)
      e_in = r;
    else if (int e = level_defect(h, l, d, r, defect))
      return e;
    if (lv->diag)
      CK(PDST_TIMED(h, PK_VANKA_GEMV, vanka_gemv_diag(g, lv->tdiag, lv->binv.ptr, e_in, upd, h->stream)));
    else
      CK(PDST_TIMED(h, PK_VANKA_GEMV, vanka_gemv(g, k1, lv->invs.ptr, e_in, upd, h->stream)));
    // from zero: d = omega sum_K R_K' upd_K (every dof written), else d += ...
    CK(PDST_TIMED(h, PK_VANKA_SCATTER, vanka_scatter(g, k1, upd, omega, d, h->stream, 0, -1, from_zero)));
  }
  return PDST_OK;
}

int pdst_vanka(pdst_handle* h, int level, double* d, const double* r, int steps, double omega, int where) {
  if (h && h->g.th) return set_error(PDST_ENOTSUP, "the Vanka sweep is Q2/P1disc-only (Taylor-Hood handles: apply, residual, mass)");
  if (!h || !d || !r) return set_error(PDST_EINVAL, "null argument");
  if (where == PDST_HOST_ASYNC) {
    if (int e = check_level(h, level)) return e;
    if (!h->patches_valid) return set_error(PDST_ESTATE, "vanka before pdst_patches_build");
    if (steps < 0) return set_error(PDST_EINVAL, "steps must be >= 0");
    CK(cudaSetDevice(h->device));
    const size_t n = (size_t)h->td.k1 * h->levels[level]->g.nd;
    int err = PDST_OK;
    // r first: it does not wait for anything, while d (in and out) waits for
    // the D2H of the previous call's d, so r's copy overlaps that round trip
    const double* rd = async_in(h, h->as_vr, r, n, &err);
    if (err) return err;
    double* dd = const_cast<double*>(async_in(h, h->as_d, d, n, &err));
    if (err) return err;
    if (int e = vanka_level(h, level, dd, rd, steps, omega)) return e;
    if (int e = async_used(h, h->as_vr)) return e;
    return async_out(h, h->as_d, d, n);
  }
  if (int e = check_where(where)) return e;
  if (int e = check_level(h, level)) return e;
  if (!h->patches_valid) return set_error(PDST_ESTATE, "vanka before pdst_patches_build");
  if (steps < 0) return set_error(PDST_EINVAL, "steps must be >= 0");
  CK(cudaSetDevice(h->device));
  const size_t n = (size_t)h->td.k1 * h->levels[level]->g.nd;
  int err = PDST_OK;
  double* dd = where == PDST_DEVICE ? d : h->scratch_b.ensure(n);
  if (!dd) return set_error(PDST_ECUDA, "out of device memory");
  if (where == PDST_HOST) CK(cudaMemcpyAsync(dd, d, n * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  const double* rd = stage_in(h, h->scratch_c, r, n, where, &err);
  if (err) return err;
  if (int e = vanka_level(h, level, dd, rd, steps, omega)) return e;
  return finish_out(h, d, dd, n, where);
}

int pdst_vanka_increment(pdst_handle* h, int level, const double* defect, double* inc, int row_lo, int row_hi,
                         double omega, int where) {
  if (h && h->g.th) return set_error(PDST_ENOTSUP, "the Vanka sweep is Q2/P1disc-only (Taylor-Hood handles: apply, residual, mass)");
  if (!h || !defect || !inc) return set_error(PDST_EINVAL, "null argument");
  if (int e = check_where(where)) return e;
  if (int e = check_level(h, level)) return e;
  if (!h->patches_valid) return set_error(PDST_ESTATE, "vanka before pdst_patches_build");
  Level* lv = h->levels[level];
  if (row_lo < 0 || row_hi > lv->g.ny || row_lo > row_hi) return set_error(PDST_EINVAL, "bad cell-row range");
  CK(cudaSetDevice(h->device));
  const Geom& g = lv->g;
  const int k1 = h->td.k1;
  const size_t n = (size_t)k1 * g.nd;
  int err = PDST_OK;
  const double* dd = stage_in(h, h->scratch_a, defect, n, where, &err);
  if (err) return err;
  double* od = out_ptr(h->scratch_b, inc, n, where);
  double* upd = h->upd.ensure((size_t)h->g.ncells * 21 * k1);
  if (!od || !upd) return set_error(PDST_ECUDA, "out of device memory");
  if (lv->diag)
    CK(PDST_TIMED(h, PK_VANKA_GEMV, vanka_gemv_diag(g, lv->tdiag, lv->binv.ptr, dd,
                                                     upd, h->stream)));
  else
    CK(PDST_TIMED(h, PK_VANKA_GEMV, vanka_gemv(g, k1, lv->invs.ptr, dd, upd, h->stream)));
  CK(PDST_TIMED(h, PK_VANKA_SCATTER, vanka_scatter(g, k1, upd, omega, od, h->stream, row_lo, row_hi, true)));
  return finish_out(h, inc, od, n, where);
}

int pdst_level_apply(pdst_handle* h, int level, const double* x, double* y, int where) {
  if (!h || !x || !y) return set_error(PDST_EINVAL, "null argument");
  finest(h);
  if (int e = check_level(h, level)) return e;
  if (level == (int)h->levels.size() - 1) return pdst_jacobian_apply(h, x, y, where);
  if (!h->patches_valid) return set_error(PDST_ESTATE, "coarse operators are built by pdst_patches_build");
  if (pdst_handle* c = h->levels[level]->child) {
    c->stream = h->stream;
    return pdst_jacobian_apply(c, x, y, where);
  }
  if (int e = check_where(where)) return e;
  CK(cudaSetDevice(h->device));
  const size_t n = (size_t)h->td.k1 * h->levels[level]->g.nd;
  int err = PDST_OK;
  const double* xd = stage_in(h, h->scratch_a, x, n, where, &err);
  if (err) return err;
  double* yd = out_ptr(h->scratch_b, y, n, where);
  if (!yd) return set_error(PDST_ECUDA, "out of device memory");
  CK(PDST_TIMED(h, PK_LEVEL, level_apply(level_op(h, level), h->td, xd, nullptr, yd, level_scratch(h, level), h->stream)));
  return finish_out(h, y, yd, n, where);
}

static int transfer_common(pdst_handle* h, int fine_level, const double* in, double* out, int where, bool prol) {
  if (!h || !in || !out) return set_error(PDST_EINVAL, "null argument");
  if (int e = check_where(where)) return e;
  if (fine_level < 1 || fine_level >= (int)h->levels.size())
    return set_error(PDST_EINVAL, "fine level %d has no coarser level", fine_level);
  CK(cudaSetDevice(h->device));
  const Geom& gf = h->levels[fine_level]->g;
  const Geom& gc = h->levels[fine_level - 1]->g;
  const int k1 = h->td.k1;
  const size_t nin = (size_t)k1 * (prol ? gc.nd : gf.nd), nout = (size_t)k1 * (prol ? gf.nd : gc.nd);
  int err = PDST_OK;
  const double* id = stage_in(h, h->scratch_a, in, nin, where, &err);
  if (err) return err;
  double* od = out_ptr(h->scratch_b, out, nout, where);
  if (!od) return set_error(PDST_ECUDA, "out of device memory");
  if (prol)
    CK(PDST_TIMED(h, PK_TRANSFER, prolong(gc, gf, k1, id, od, h->stream)));
  else
    CK(PDST_TIMED(h, PK_TRANSFER, restrict_(gc, gf, k1, id, od, h->stream)));
  return finish_out(h, out, od, nout, where);
}

int pdst_restrict(pdst_handle* h, int fine_level, const double* r_fine, double* r_coarse, int where) {
  return transfer_common(h, fine_level, r_fine, r_coarse, where, false);
}

int pdst_prolong(pdst_handle* h, int fine_level, const double* e_coarse, double* e_fine, int where) {
  return transfer_common(h, fine_level, e_coarse, e_fine, where, true);
}

// Coarsest-level FGMRES: z ~ A_0^-1 b with right preconditioning by
// `coarse_sweeps` Vanka steps from zero, Euclidean inner product, classical
// Gram-Schmidt applied twice (multi-dot + fused update), Givens rotations on
// the host; stops after `coarse_iters` iterations or at relative residual
// `coarse_rtol`.  Deterministic (fixed reduction trees).
static int coarse_fgmres(pdst_handle* h, const double* b, double* z) {
  Level* lv = h->levels[0];
  const size_t n = (size_t)h->td.k1 * lv->g.nd;
  const int m = h->coarse_iters;
  double* V = lv->kv.ensure((size_t)(m + 1) * n);
  double* Z = lv->kz.ensure((size_t)m * n);
  double* w = lv->kw.ensure(n);
  const size_t nred = std::max(multidot_scratch(m + 1), (size_t)reduce_partials());
  double* sc = lv->ks.ensure(nred + 2 * (size_t)(m + 2));
  if (!V || !Z || !w || !sc) return set_error(PDST_ECUDA, "out of device memory (coarse FGMRES)");
  double* part = sc;
  double* dvec = sc + nred;  // device coefficients (m + 2)
  auto sync_read = [&](double* host, const double* dev, int cnt) -> int {
    CK(cudaMemcpyAsync(host, dev, (size_t)cnt * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return PDST_OK;
  };
  auto norm2 = [&](const double* v, double* out) -> int {
    CK(dot(v, v, n, part, dvec, h->stream));
    double s2 = 0.0;
    if (int e = sync_read(&s2, dvec, 1)) return e;
    *out = std::sqrt(s2);
    return PDST_OK;
  };
  CK(cudaMemsetAsync(z, 0, n * sizeof(double), h->stream));
  double beta = 0.0;
  if (int e = norm2(b, &beta)) return e;
  if (!(beta > 0.0)) return PDST_OK;
  CK(cudaMemsetAsync(V, 0, n * sizeof(double), h->stream));
  CK(axpy(n, 1.0 / beta, b, V, h->stream));
  std::vector<double> H((size_t)(m + 1) * m, 0.0), cs(m), sn(m), g(m + 1, 0.0), hc(m + 1);
  g[0] = beta;
  int k = 0;
  for (int j = 0; j < m; ++j) {
    double* Vj = V + (size_t)j * n;
    double* Zj = Z + (size_t)j * n;
    if (int e = vanka_level(h, 0, Zj, Vj, h->coarse_sweeps, h->coarse_omega, true)) return e;
    // w = A_0 z_j (the matrix-free Jacobian when level 0 is the handle's own mesh)
    if (int e = level_defect(h, 0, Zj, nullptr, w)) return e;
    for (int pass = 0; pass < 2; ++pass) {  // CGS2
      CK(multidot(V, (int64_t)n, j + 1, w, (int64_t)n, part, dvec, h->stream));
      CK(multi_axpy(V, nullptr, (int64_t)n, j + 1, dvec, w, nullptr, (int64_t)n, h->stream));
      if (int e = sync_read(hc.data(), dvec, j + 1)) return e;
      for (int i = 0; i <= j; ++i) H[(size_t)i * m + j] += hc[i];
    }
    double hn = 0.0;
    if (int e = norm2(w, &hn)) return e;
    H[(size_t)(j + 1) * m + j] = hn;
    if (hn > 0.0) {
      double* Vn = V + (size_t)(j + 1) * n;
      CK(cudaMemsetAsync(Vn, 0, n * sizeof(double), h->stream));
      CK(axpy(n, 1.0 / hn, w, Vn, h->stream));
    }
    for (int i = 0; i < j; ++i) {  // previous rotations on column j
      const double a = H[(size_t)i * m + j], c = H[(size_t)(i + 1) * m + j];
      H[(size_t)i * m + j] = cs[i] * a + sn[i] * c;
      H[(size_t)(i + 1) * m + j] = -sn[i] * a + cs[i] * c;
    }
    const double a = H[(size_t)j * m + j], c = H[(size_t)(j + 1) * m + j];
    const double r = std::hypot(a, c);
    cs[j] = r > 0.0 ? a / r : 1.0;
    sn[j] = r > 0.0 ? c / r : 0.0;
    H[(size_t)j * m + j] = r;
    H[(size_t)(j + 1) * m + j] = 0.0;
    g[j + 1] = -sn[j] * g[j];
    g[j] = cs[j] * g[j];
    k = j + 1;
    if (std::fabs(g[j + 1]) <= h->coarse_rtol * beta || !(hn > 0.0)) break;
  }
  // y = H^-1 g (upper triangular k x k), z = Z y
  std::vector<double> y(k, 0.0);
  for (int i = k - 1; i >= 0; --i) {
    double s = g[i];
    for (int l2 = i + 1; l2 < k; ++l2) s -= H[(size_t)i * m + l2] * y[l2];
    y[i] = H[(size_t)i * m + i] != 0.0 ? s / H[(size_t)i * m + i] : 0.0;
  }
  for (int i = 0; i < k; ++i) y[i] = -y[i];  // multi_axpy subtracts
  CK(cudaMemcpyAsync(dvec, y.data(), (size_t)k * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  CK(multi_axpy(Z, nullptr, (int64_t)n, k, dvec, z, nullptr, (int64_t)n, h->stream));
  CK(cudaStreamSynchronize(h->stream));  // y lives on the host stack
  return PDST_OK;
}

// One V-cycle on level l with zero initial guess: z = V_l b (multigrid.py:545-555).
static int vcycle_level(pdst_handle* h, int l, const double* b, double* z, int pre, int post, double omega) {
  Level* lv = h->levels[l];
  const int k1 = h->td.k1;
  const size_t n = (size_t)k1 * lv->g.nd;
  if (l == 0 && lv->child) {  // rediscretized coarsest level: the child's coarse solve
    lv->child->stream = h->stream;
    return vcycle_level(lv->child, 0, b, z, pre, post, omega);
  }
  if (l == 0) {
    if (h->coarse_iterative) {
      if (h->coarse_kind == PDST_COARSE_VANKA) {  // Vanka steps from zero on the coarsest level
        return vanka_level(h, 0, z, b, h->coarse_sweeps, h->coarse_omega, true);
      }
      return coarse_fgmres(h, b, z);
    }
    CK(dense_solve(lv->dense.ptr, (int)n, b, z, h->stream));
    return PDST_OK;
  }
  Level* lc = h->levels[l - 1];
  const Geom& gc = lc->g;
  double* r = lv == h->levels.back() ? h->scratch_d.ensure(n) : lv->w1.ptr;
  if (!r) return set_error(PDST_ECUDA, "out of device memory");
  if (int e = vanka_level(h, l, z, b, pre, omega, true)) return e;  // (clears z itself when pre == 0)
  if (int e = level_defect(h, l, z, b, r)) return e;
  CK(PDST_TIMED(h, PK_TRANSFER, restrict_(gc, lv->g, k1, r, lc->w0.ptr, h->stream)));
  if (int e = vcycle_level(h, l - 1, lc->w0.ptr, lc->w2.ptr, pre, post, omega)) return e;
  CK(PDST_TIMED(h, PK_TRANSFER, prolong(gc, lv->g, k1, lc->w2.ptr, r, h->stream)));
  CK(axpy(n, 1.0, r, z, h->stream));
  if (int e = vanka_level(h, l, z, b, post, omega)) return e;
  return PDST_OK;
}

int pdst_set_coarse_mode(pdst_handle* h, int mode) {
  if (!h) return set_error(PDST_EINVAL, "null handle");
  if (mode != 0 && mode != 1) return set_error(PDST_EINVAL, "unknown coarse mode %d (0 galerkin, 1 rediscretize)", mode);
  h->coarse_mode = mode;
  h->patches_valid = false;
  h->coarse_valid = false;
  return PDST_OK;
}

int pdst_set_coarse_solver(pdst_handle* h, int kind, int sweeps, double omega, int iters, double rtol) {
  if (!h) return set_error(PDST_EINVAL, "null handle");
  if (kind < PDST_COARSE_DENSE || kind > PDST_COARSE_FGMRES) return set_error(PDST_EINVAL, "unknown coarse solver %d", kind);
  if (sweeps < 0) return set_error(PDST_EINVAL, "coarse sweeps must be >= 0");
  if (!(omega > 0.0 && omega <= 1.0)) return set_error(PDST_EINVAL, "coarse omega must lie in (0, 1]");
  if (iters < 1 || iters > 1000) return set_error(PDST_EINVAL, "coarse FGMRES iterations must lie in [1, 1000]");
  if (!(rtol >= 0.0)) return set_error(PDST_EINVAL, "coarse rtol must be >= 0");
  h->coarse_kind = kind;
  h->coarse_sweeps = sweeps;
  h->coarse_omega = omega;
  h->coarse_iters = iters;
  h->coarse_rtol = rtol;
  h->coarse_valid = false;
  return PDST_OK;
}

int pdst_vcycle(pdst_handle* h, const double* r, double* z, int pre, int post, double omega, int where) {
  if (h && h->g.th) return set_error(PDST_ENOTSUP, "the V-cycle is Q2/P1disc-only (Taylor-Hood handles: apply, residual, mass)");
  if (!h || !r || !z) return set_error(PDST_EINVAL, "null argument");
  if (int e = check_where(where)) return e;
  if (!h->patches_valid || !h->coarse_valid)
    return set_error(PDST_ESTATE, "V-cycle needs pdst_hierarchy and pdst_patches_build");
  CK(cudaSetDevice(h->device));
  const int L = (int)h->levels.size();
  const size_t n = (size_t)h->td.k1 * h->g.nd;
  int err = PDST_OK;
  const double* rd = stage_in(h, h->scratch_c, r, n, where, &err);
  if (err) return err;
  double* zd = out_ptr(h->scratch_b, z, n, where);
  if (!zd) return set_error(PDST_ECUDA, "out of device memory");
  if (int e = vcycle_level(h, L - 1, rd, zd, pre, post, omega)) return e;
  if (h->levels.back()->all_dirichlet) {
    double* pp = h->ppartials.ensure(project_scratch(h->td.k1));
    if (!pp) return set_error(PDST_ECUDA, "out of device memory");
    CK(project_pressure(h->g, h->td.k1, zd, pp, h->stream));
  }
  return finish_out(h, z, zd, n, where);
}

}  // extern "C"
