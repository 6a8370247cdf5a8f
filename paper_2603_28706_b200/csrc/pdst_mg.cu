// pdst_mg.cu — integer maps, Vanka patches / sweeps and the multigrid entry
// points of the C ABI (include/pdst.h).
//
// Reference: solver/multigrid.py:164-191 (hierarchy), :261-299 (patches),
// :327-340 (vanka_smooth), :475-488 (surrogate), femspace.py:127-140 and
// forms.py:192-196 (dof maps).
#include <cuda_runtime.h>

#include <climits>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../include/pdst.h"
#include "pdst_handle.h"
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

Level* finest(pdst_handle* h) {
  if (h->levels.empty()) {
    Level* l = new Level();
    l->g = h->g;  // shares the handle's dirichlet flags (not owned)
    l->dirichlet_host = h->dirichlet_host;
    l->all_dirichlet = true;
    for (auto f : h->dirichlet_host) l->all_dirichlet = l->all_dirichlet && f;
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
  if (!h || !cell_nodes || !patch_ids) return set_error(PDST_EINVAL, "null argument");
  CK(cudaSetDevice(h->device));
  const Geom& g = h->g;
  const int k1 = h->td.k1;
  int64_t* dev = nullptr;
  const size_t n1 = (size_t)g.ncells * 9, n2 = (size_t)g.ncells * 21 * k1;
  CK(cudaMalloc(&dev, (n1 + n2) * sizeof(int64_t)));
  k_cell_maps<<<(g.ncells + 127) / 128, 128, 0, h->stream>>>(g.nx, g.ny, g.nd, k1, dev, dev + n1);
  cudaError_t e = cudaMemcpyAsync(cell_nodes, dev, n1 * sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(patch_ids, dev + n1, n2 * sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  cudaFree(dev);
  if (e != cudaSuccess) return set_error(PDST_ECUDA, "cell maps: %s", cudaGetErrorString(e));
  return PDST_OK;
}

int pdst_hierarchy(pdst_handle* h, int min_cells, int* num_levels) {
  if (!h) return set_error(PDST_EINVAL, "null handle");
  finest(h);
  (void)min_cells;
  if (num_levels) *num_levels = (int)h->levels.size();
  return set_error(PDST_ENOTSUP, "coarse levels not built in this version");
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

int pdst_patches_build(pdst_handle* h, int surrogate, double rep_fraction, int* bad_level, int64_t* bad_patch) {
  if (!h) return set_error(PDST_EINVAL, "null handle");
  if (!h->linearized) return set_error(PDST_ESTATE, "patches built before pdst_linearize");
  CK(cudaSetDevice(h->device));
  Level* fl = finest(h);
  const Geom& g = h->g;
  const int k1 = h->td.k1, D = 21 * k1;
  const size_t nc = g.ncells;
  PatchArgs pa{};
  pa.g = g;
  pa.td = h->td;
  pa.ds = h->ds;
  const bool rep = surrogate && k1 > 1;
  pa.nslot = surrogate ? 1 : k1;
  double* ET = h->ET.ensure((size_t)pa.nslot * nc * 441);
  if (!ET) return set_error(PDST_ECUDA, "out of device memory (element matrices)");
  pa.ET = ET;
  if (rep) {
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
    Lin L = lin_of(h);
    L.eta = er;
    L.gam = gr;
    L.etaf = efr;
    L.gamf = gfr;
    CK(element_matrices(g, h->ds, L, 0, sr, ET, h->stream));
    pa.state = sr;
  } else {
    const Lin L = lin_of(h);
    for (int s = 0; s < pa.nslot; ++s)
      CK(element_matrices(g, h->ds, L, s, h->state.ptr + (size_t)s * g.mv, ET + (size_t)s * nc * 441, h->stream));
    pa.state = h->state.ptr;
  }
  double* mats = fl->mats.ensure(nc * D * D);
  double* bad = h->ibuf.ensure(1);
  if (!mats || !bad) return set_error(PDST_ECUDA, "out of device memory (patches)");
  pa.mats = mats;
  // Surrogate patches share one spatial block across the Radau nodes: keep it
  // and invert the temporally diagonalized blocks instead of A_K itself.
  const char* nd_env = getenv("PDST_NO_TIMEDIAG");
  fl->diag = surrogate && !(nd_env && nd_env[0] == '1') && time_diagonalize(k1, h->td.K_t, h->td.tau_w, fl->tdiag);
  pa.spatial = nullptr;
  if (fl->diag) {
    pa.spatial = fl->spatial.ensure(nc * 441);
    if (!pa.spatial || !fl->binv.ensure(nc * 441 * 2 * fl->tdiag.nblk))
      return set_error(PDST_ECUDA, "out of device memory (diagonalized patches)");
  }
  CK(patch_assemble(pa, h->stream));
  int* badi = reinterpret_cast<int*>(bad);
  const int init = INT_MAX;
  CK(cudaMemcpyAsync(badi, &init, sizeof(int), cudaMemcpyHostToDevice, h->stream));
  if (fl->diag) {
    CK(patch_invert_diag(g, fl->tdiag, pa.spatial, reinterpret_cast<double2*>(fl->binv.ptr), badi, h->stream));
  } else {
    double* invs = fl->invs.ensure(nc * D * D);
    if (!invs) return set_error(PDST_ECUDA, "out of device memory (patch inverses)");
    CK(patch_invert(k1, mats, invs, (int)nc, badi, h->stream));
  }
  int badh = INT_MAX;
  CK(cudaMemcpyAsync(&badh, badi, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  fl->D = D;
  const int L = (int)h->levels.size();
  if (badh != INT_MAX) {
    if (bad_level) *bad_level = L - 1;
    if (bad_patch) *bad_patch = badh;
    h->patches_valid = false;
    return set_error(PDST_ESINGULAR, "singular patch matrix (level %d, patch %d)", L - 1, badh);
  }
  h->patches_valid = true;
  return PDST_OK;
}

int pdst_patch_matrices(pdst_handle* h, int level, double* mats) {
  if (!h || !mats) return set_error(PDST_EINVAL, "null argument");
  if (int e = check_level(h, level)) return e;
  Level* l = h->levels[level];
  if (!l->D) return set_error(PDST_ESTATE, "patches not built");
  CK(cudaSetDevice(h->device));
  const size_t n = (size_t)l->g.ncells * l->D * l->D;
  CK(cudaMemcpyAsync(mats, l->mats.ptr, n * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return PDST_OK;
}

int pdst_patch_info(pdst_handle* h, int level, int32_t* D, int32_t* diag_blocks, int64_t* bytes_per_patch) {
  if (!h) return set_error(PDST_EINVAL, "null handle");
  if (int e = check_level(h, level)) return e;
  Level* l = h->levels[level];
  if (!l->D) return set_error(PDST_ESTATE, "patches not built");
  if (D) *D = l->D;
  if (diag_blocks) *diag_blocks = l->diag ? l->tdiag.nblk : 0;
  if (bytes_per_patch)
    *bytes_per_patch = l->diag ? (int64_t)l->tdiag.nblk * 441 * 16 : (int64_t)l->D * l->D * 8;
  return PDST_OK;
}

int pdst_vanka(pdst_handle* h, int level, double* d, const double* r, int steps, double omega, int where) {
  if (!h || !d || !r) return set_error(PDST_EINVAL, "null argument");
  if (int e = check_where(where)) return e;
  if (int e = check_level(h, level)) return e;
  if (!h->patches_valid) return set_error(PDST_ESTATE, "vanka before pdst_patches_build");
  if (steps < 0) return set_error(PDST_EINVAL, "steps must be >= 0");
  if (level != (int)h->levels.size() - 1) return set_error(PDST_ENOTSUP, "coarse-level Vanka not built");
  CK(cudaSetDevice(h->device));
  Level* l = h->levels[level];
  const Geom& g = l->g;
  const int k1 = h->td.k1;
  const size_t n = (size_t)k1 * g.nd;
  int err = PDST_OK;
  double* dd = where == PDST_DEVICE ? d : h->scratch_b.ensure(n);
  if (!dd) return set_error(PDST_ECUDA, "out of device memory");
  if (where == PDST_HOST) CK(cudaMemcpyAsync(dd, d, n * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  const double* rd = stage_in(h, h->scratch_c, r, n, where, &err);
  if (err) return err;
  double* defect = h->defect.ensure(n);
  double* upd = h->upd.ensure((size_t)g.ncells * 21 * k1);
  if (!defect || !upd) return set_error(PDST_ECUDA, "out of device memory");
  const Lin L = lin_of(h);
  double* part = h->jpart.ensure(jacobian_scratch(g, k1));
  if (!part) return set_error(PDST_ECUDA, "out of device memory");
  for (int s = 0; s < steps; ++s) {
    CK(PDST_TIMED(h, PK_JACOBIAN, jacobian_apply(g, h->td, h->ds, L, h->state.ptr, dd, rd, defect, part, h->stream)));
    if (l->diag)
      CK(PDST_TIMED(h, PK_VANKA_GEMV, vanka_gemv_diag(g, l->tdiag, reinterpret_cast<const double2*>(l->binv.ptr),
                                                       defect, upd, h->stream)));
    else
      CK(PDST_TIMED(h, PK_VANKA_GEMV, vanka_gemv(g, k1, l->invs.ptr, defect, upd, h->stream)));
    CK(PDST_TIMED(h, PK_VANKA_SCATTER, vanka_scatter(g, k1, upd, omega, dd, h->stream)));
  }
  return finish_out(h, d, dd, n, where);
}

int pdst_level_apply(pdst_handle* h, int level, const double* x, double* y, int where) {
  if (!h) return set_error(PDST_EINVAL, "null handle");
  finest(h);
  if (int e = check_level(h, level)) return e;
  if (level == (int)h->levels.size() - 1) return pdst_jacobian_apply(h, x, y, where);
  return set_error(PDST_ENOTSUP, "coarse levels not built in this version");
}

int pdst_restrict(pdst_handle*, int, const double*, double*, int) {
  return set_error(PDST_ENOTSUP, "transfers not built in this version");
}
int pdst_prolong(pdst_handle*, int, const double*, double*, int) {
  return set_error(PDST_ENOTSUP, "transfers not built in this version");
}
int pdst_vcycle(pdst_handle*, const double*, double*, int, int, double, int) {
  return set_error(PDST_ENOTSUP, "V-cycle not built in this version");
}

}  // extern "C"
