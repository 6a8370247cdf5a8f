// pdst_capi.cu — the extern "C" boundary (include/pdst.h): handle lifetime,
// host/device pointer staging, argument validation and error reporting.
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/pdst.h"
#include "pdst_handle.h"

using namespace pdst;

namespace {
thread_local std::string g_last_error;
}  // namespace

int pdst::set_error(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

namespace {
#define fail pdst::set_error

int cuda_fail(cudaError_t e, const char* where) {
  return fail(PDST_ECUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define CK(expr)                                      \
  do {                                                \
    cudaError_t _e = (expr);                          \
    if (_e != cudaSuccess) return cuda_fail(_e, #expr); \
  } while (0)

}  // namespace

// ---------------------------------------------------------------------------
// Handle helpers
// ---------------------------------------------------------------------------
namespace pdst {

double* DeviceBuffer::ensure(size_t n) {
  if (n > cap) {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
    if (cudaMalloc(&ptr, n * sizeof(double)) != cudaSuccess) return nullptr;
    cap = n;
  }
  return ptr;
}

double* DeviceBuffer::ensure_zeroed(size_t n) {
  if (n <= cap) return ptr;
  double* p = ensure(n);
  if (p && cudaMemset(p, 0, n * sizeof(double)) != cudaSuccess) return nullptr;
  return p;
}

void DeviceBuffer::release() {
  if (ptr) cudaFree(ptr);
  ptr = nullptr;
  cap = 0;
}

Geom make_geom(int nx, int ny, double x0, double y0, double x1, double y1, const uint8_t* dirichlet_dev, int th) {
  Geom g{};
  g.nx = nx;
  g.ny = ny;
  g.nnx = 2 * nx + 1;
  g.nny = 2 * ny + 1;
  g.ncells = nx * ny;
  g.mv = 2 * g.nnx * g.nny;
  g.th = th;
  g.nd = g.mv + (th ? (nx + 1) * (ny + 1) : 3 * g.ncells);
  g.nbf = 2 * (nx + ny);
  g.hx = (x1 - x0) / nx;
  g.hy = (y1 - y0) / ny;
  g.ihx = 1.0 / g.hx;
  g.ihy = 1.0 / g.hy;
  g.dirichlet = dirichlet_dev;
  return g;
}

}  // namespace pdst

// Copy a caller array to a device scratch buffer when it lives on the host.
const double* pdst::stage_in(pdst_handle* h, DeviceBuffer& buf, const double* p, size_t n, int where, int* err) {
  if (!p) return nullptr;
  if (where == PDST_DEVICE) return p;
  double* d = buf.ensure(n);
  if (!d) {
    *err = fail(PDST_ECUDA, "out of device memory (%zu doubles)", n);
    return nullptr;
  }
  cudaError_t e = cudaMemcpyAsync(d, p, n * sizeof(double), cudaMemcpyHostToDevice, h->stream);
  if (e != cudaSuccess) {
    *err = cuda_fail(e, "H2D");
    return nullptr;
  }
  return d;
}

double* pdst::out_ptr(DeviceBuffer& buf, double* p, size_t n, int where) {
  return where == PDST_DEVICE ? p : buf.ensure(n);
}

int pdst::finish_out(pdst_handle* h, double* host, const double* dev, size_t n, int where) {
  if (where == PDST_DEVICE) return PDST_OK;
  CK(cudaMemcpyAsync(host, dev, n * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return PDST_OK;
}

static int ensure_async(pdst_handle* h, pdst::AsyncSlot& s) {
  if (!h->copy_in) {
    CK(cudaStreamCreateWithFlags(&h->copy_in, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&h->copy_out, cudaStreamNonBlocking));
  }
  if (!s.in_done) {
    CK(cudaEventCreateWithFlags(&s.in_done, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&s.use_done, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&s.out_done, cudaEventDisableTiming));
  }
  return PDST_OK;
}

static bool pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

const double* pdst::async_in(pdst_handle* h, AsyncSlot& s, const double* p, size_t n, int* err) {
  if (!p) return nullptr;
  if ((*err = ensure_async(h, s))) return nullptr;
  if (!pinned(p)) {
    *err = fail(PDST_EINVAL, "PDST_HOST_ASYNC needs page-locked host memory");
    return nullptr;
  }
  double* d = s.buf.ensure(n);
  if (!d) {
    *err = fail(PDST_ECUDA, "out of device memory (%zu doubles)", n);
    return nullptr;
  }
  cudaError_t e = cudaSuccess;
  // the slot's previous kernels and D2H must be done with it; a D2H into p must have landed
  if (s.used) e = cudaStreamWaitEvent(h->copy_in, s.use_done, 0);
  if (e == cudaSuccess && s.outed) e = cudaStreamWaitEvent(h->copy_in, s.out_done, 0);
  for (auto& po : h->pending_out)
    if (e == cudaSuccess && po.first == p) e = cudaStreamWaitEvent(h->copy_in, po.second, 0);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d, p, n * sizeof(double), cudaMemcpyHostToDevice, h->copy_in);
  if (e == cudaSuccess) e = cudaEventRecord(s.in_done, h->copy_in);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(h->stream, s.in_done, 0);
  if (e != cudaSuccess) {
    *err = cuda_fail(e, "async H2D");
    return nullptr;
  }
  return d;
}

double* pdst::async_out_ptr(pdst_handle* h, AsyncSlot& s, size_t n, int* err) {
  if ((*err = ensure_async(h, s))) return nullptr;
  double* d = s.buf.ensure(n);
  if (!d) {
    *err = fail(PDST_ECUDA, "out of device memory (%zu doubles)", n);
    return nullptr;
  }
  if (s.outed) {  // its previous D2H must have read it before the kernels overwrite it
    cudaError_t e = cudaStreamWaitEvent(h->stream, s.out_done, 0);
    if (e != cudaSuccess) {
      *err = cuda_fail(e, "async order");
      return nullptr;
    }
  }
  return d;
}

int pdst::async_used(pdst_handle* h, AsyncSlot& s) {
  CK(cudaEventRecord(s.use_done, h->stream));
  s.used = true;
  return PDST_OK;
}

int pdst::async_out(pdst_handle* h, AsyncSlot& s, double* p, size_t n) {
  if (!pinned(p)) return fail(PDST_EINVAL, "PDST_HOST_ASYNC needs page-locked host memory");
  if (int e = async_used(h, s)) return e;
  CK(cudaStreamWaitEvent(h->copy_out, s.use_done, 0));
  CK(cudaMemcpyAsync(p, s.buf.ptr, n * sizeof(double), cudaMemcpyDeviceToHost, h->copy_out));
  CK(cudaEventRecord(s.out_done, h->copy_out));
  s.outed = true;
  bool found = false;
  for (auto& po : h->pending_out)
    if (po.first == p) {
      po.second = s.out_done;
      found = true;
    }
  if (!found) h->pending_out.push_back({p, s.out_done});
  return PDST_OK;
}

int pdst_sync(pdst_handle* h) {
  if (!h) return fail(PDST_EINVAL, "null handle");
  CK(cudaSetDevice(h->device));
  CK(cudaStreamSynchronize(h->stream));
  if (h->copy_in) CK(cudaStreamSynchronize(h->copy_in));
  if (h->copy_out) CK(cudaStreamSynchronize(h->copy_out));
  h->pending_out.clear();
  return PDST_OK;
}

int pdst::check_where(int where) {
  if (where != PDST_HOST && where != PDST_DEVICE) return fail(PDST_EINVAL, "where must be PDST_HOST or PDST_DEVICE");
  return PDST_OK;
}

static std::atomic<int64_t> g_launches{0};
void pdst_count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

extern "C" {

const char* pdst_last_error(void) { return g_last_error.c_str(); }
const char* pdst_version(void) { return "pdst-b200 0.1 (sm_100a fp64)"; }
int64_t pdst_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int pdst_create(const pdst_mesh* mesh, const pdst_time* time, const pdst_disc* disc, const pdst_params* params,
                double tau, int device, void* stream, pdst_handle** out) {
  if (!mesh || !time || !disc || !params || !out) return fail(PDST_EINVAL, "null argument");
  *out = nullptr;
  if (mesh->nx < 1 || mesh->ny < 1) return fail(PDST_EINVAL, "cell counts must be >= 1");
  if (!(mesh->x1 > mesh->x0) || !(mesh->y1 > mesh->y0)) return fail(PDST_EINVAL, "degenerate domain extents");
  if (time->k < 0 || time->k + 1 > MAXK1) return fail(PDST_EINVAL, "temporal degree k must lie in [0, 6]");
  if (time->k + 1 > 4) return fail(PDST_ENOTSUP, "kernels are instantiated for k <= 3");
  if (!time->nodes || !time->weights || !time->K_t || !time->m_t) return fail(PDST_EINVAL, "null time arrays");
  if (!(tau > 0.0)) return fail(PDST_EINVAL, "tau must be positive");
  if (disc->gamma1 <= 0.0 || disc->gamma2 <= 0.0)
    return fail(PDST_EINVAL, "Nitsche penalties gamma1, gamma2 must be positive");
  if (disc->gamma_cip < 0.0) return fail(PDST_EINVAL, "gamma_cip must be >= 0");
  if (disc->pressure_space != 0 && disc->pressure_space != 1)
    return fail(PDST_EINVAL, "pressure_space must be 0 (P1disc) or 1 (Taylor-Hood Q1)");
  if (!(params->p > 1.0 && params->p <= 2.0)) return fail(PDST_EDOMAIN, "exponent p must lie in (1, 2]");
  if (params->delta < 0.0) return fail(PDST_EDOMAIN, "delta must be >= 0");
  if (params->nu <= 0.0) return fail(PDST_EDOMAIN, "nu must be > 0");
  if (params->nu_inf < 0.0) return fail(PDST_EDOMAIN, "nu_inf must be >= 0");

  CK(cudaSetDevice(device));
  static bool tables_set[64] = {false};
  if (device >= 0 && device < 64 && !tables_set[device]) {
    CK(set_tables(host_tables()));
    tables_set[device] = true;
  }
  std::unique_ptr<pdst_handle> h(new pdst_handle());
  h->device = device;
  h->stream = static_cast<cudaStream_t>(stream);
  const int nbf = 2 * (mesh->nx + mesh->ny);
  std::vector<uint8_t> dir(nbf, 1);
  if (mesh->dirichlet)
    for (int i = 0; i < nbf; ++i) {
      if (mesh->dirichlet[i] > 2) return fail(PDST_EINVAL, "boundary tag %d of face %d is not 0, 1 or 2", mesh->dirichlet[i], i);
      dir[i] = mesh->dirichlet[i];
    }
  h->dirichlet_host = dir;
  CK(cudaMalloc(&h->dirichlet, nbf));
  CK(cudaMemcpy(h->dirichlet, dir.data(), nbf, cudaMemcpyHostToDevice));
  h->extents[0] = mesh->x0;
  h->extents[1] = mesh->y0;
  h->extents[2] = mesh->x1;
  h->extents[3] = mesh->y1;
  h->g = make_geom(mesh->nx, mesh->ny, mesh->x0, mesh->y0, mesh->x1, mesh->y1, h->dirichlet, disc->pressure_space);
  const int k1 = time->k + 1;
  h->td.k1 = k1;
  h->tau = tau;
  h->nodes.assign(time->nodes, time->nodes + k1);
  h->weights.assign(time->weights, time->weights + k1);
  for (int i = 0; i < k1; ++i) {
    h->td.tau_w[i] = tau * time->weights[i];  // ctx.tau * ctx.basis.weights (slab.py:171)
    h->td.m_t[i] = time->m_t[i];
    for (int j = 0; j < k1; ++j) h->td.K_t[i * k1 + j] = time->K_t[i * k1 + j];
  }
  h->ds.gamma1 = disc->gamma1;
  h->ds.gamma2 = disc->gamma2;
  h->ds.gamma_cip = disc->gamma_cip;
  h->ds.viscous = disc->enable_viscous;
  h->ds.convection = disc->enable_convection;
  h->ds.pressure = disc->enable_pressure;
  if (h->g.th) {  // Taylor-Hood: the velocity kernels run without pressure terms, pdst_th.cu adds them
    h->th_pressure = disc->enable_pressure != 0;
    h->ds.pressure = 0;
  }
  h->model.p = params->p;
  h->model.delta = params->delta;
  h->model.nu = params->nu;
  h->model.nu_inf = params->nu_inf;
  h->model.kind = 0;
  h->model.sigma_max = INFINITY;
  // lifting caches with the zero lifting (forms.py:347-349)
  const Geom& g = h->g;
  double* ed = h->etad.ensure((size_t)g.nbf * 4);
  double* bd = h->betad.ensure((size_t)g.nbf * 4);
  double* dg = h->dg.ensure((size_t)g.nbf * 12);
  if (!ed || !bd || !dg) return fail(PDST_ECUDA, "out of device memory");
  CK(lifting(g, h->model, nullptr, ed, bd, dg, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  *out = h.release();
  return PDST_OK;
}

int pdst_destroy(pdst_handle* h) {
  if (!h) return PDST_OK;
  cudaSetDevice(h->device);
  cudaStreamSynchronize(h->stream);
  delete h;
  return PDST_OK;
}

int pdst_set_stream(pdst_handle* h, void* stream) {
  if (!h) return fail(PDST_EINVAL, "null handle");
  h->stream = static_cast<cudaStream_t>(stream);
  return PDST_OK;
}

int pdst_sizes(const pdst_handle* h, int64_t* mv, int64_t* mp, int64_t* nd, int64_t* ndof) {
  if (!h) return fail(PDST_EINVAL, "null handle");
  if (mv) *mv = h->g.mv;
  if (mp) *mp = 3LL * h->g.ncells;
  if (nd) *nd = h->g.nd;
  if (ndof) *ndof = (int64_t)h->td.k1 * h->g.nd;
  return PDST_OK;
}

int pdst_set_lifting(pdst_handle* h, const double* g_hat, int where) {
  if (!h) return fail(PDST_EINVAL, "null handle");
  if (int e = check_where(where)) return e;
  CK(cudaSetDevice(h->device));
  const Geom& g = h->g;
  const double* gp = nullptr;
  if (g_hat) {
    double* dst = h->ghat.ensure(g.mv);
    if (!dst) return fail(PDST_ECUDA, "out of device memory");
    CK(cudaMemcpyAsync(dst, g_hat, g.mv * sizeof(double),
                       where == PDST_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, h->stream));
    gp = dst;
    h->has_ghat = true;
  } else {
    h->has_ghat = false;
  }
  CK(lifting(g, h->model, gp, h->etad.ptr, h->betad.ptr, h->dg.ptr, h->stream));
  if (where == PDST_HOST) CK(cudaStreamSynchronize(h->stream));
  return PDST_OK;
}

int pdst_linearize(pdst_handle* h, const double* U, int kind, double sigma_max, int where) {
  if (!h || !U) return fail(PDST_EINVAL, "null argument");
  if (int e = check_where(where)) return e;
  if (kind < 0 || kind > 2) return fail(PDST_EINVAL, "unknown tangent kind %d", kind);
  if (kind == PDST_MODIFIED_NEWTON && sigma_max < 0.0) return fail(PDST_EINVAL, "sigma_max must be >= 0");
  if (h->model.delta <= 0.0) return fail(PDST_EDOMAIN, "jacobian requires delta > 0");
  CK(cudaSetDevice(h->device));
  const Geom& g = h->g;
  const int k1 = h->td.k1;
  int err = PDST_OK;
  const double* Ud = stage_in(h, h->scratch_a, U, (size_t)k1 * g.nd, where, &err);
  if (err) return err;
  double* st = h->state.ensure((size_t)k1 * g.mv);
  double* eta = h->eta.ensure((size_t)k1 * 16 * g.ncells);
  double* gam = h->gam.ensure((size_t)k1 * 16 * g.ncells);
  double* etaf = h->etaf.ensure((size_t)k1 * g.nbf * 4);
  double* gamf = h->gamf.ensure((size_t)k1 * g.nbf * 4);
  if (!st || !eta || !gam || !etaf || !gamf) return fail(PDST_ECUDA, "out of device memory");
  CK(copy_velocity_blocks(g, k1, Ud, st, h->stream));
  h->model.kind = kind;
  h->model.sigma_max = sigma_max;
  CK(linearize(g, h->model, k1, st, eta, gam, etaf, gamf, h->stream));
  {
    double* bm = h->bmat.ensure((size_t)k1 * 441 * g.nbf);
    if (!bm) return fail(PDST_ECUDA, "out of device memory");
    Lin L = lin_of(h);
    L.bmat = nullptr;
    CK(boundary_matrices(g, h->ds, L, k1, st, bm, h->stream));
    double* apc = h->apc.ensure(apply_cache_size(g, k1));
    if (!apc) return fail(PDST_ECUDA, "out of device memory");
    CK(apply_cache(g, h->td, h->ds, L, st, apc, h->stream));
  }
  if (h->jpart.ptr && h->jpart.cap >= jacobian_scratch(g, k1))  // (allocated by the first apply)
    CK(jacobian_reset_counters(g, k1, h->jpart.ptr, h->stream));
  h->linearized = true;
  h->patches_valid = false;
  if (where == PDST_HOST) CK(cudaStreamSynchronize(h->stream));
  return PDST_OK;
}

// Taylor-Hood: add the pressure coupling to the velocity apply (pdst_th.cu)
static int th_add(pdst_handle* h, const double* x, double* y) {
  double* cb = h->th_cells.ensure(th_scratch(h->g, h->td.k1));
  if (!cb) return fail(PDST_ECUDA, "out of device memory");
  CK(th_apply(h->g, h->td, h->th_pressure, x, y, cb, h->stream));
  return PDST_OK;
}

static int jac_common(pdst_handle* h, const double* x, const double* r, double* y, int where) {
  if (!h || !x || !y) return fail(PDST_EINVAL, "null argument");
  if (h->g.th && r) return fail(PDST_ENOTSUP, "defect form (the Vanka sweep) is P1disc-only; Taylor-Hood handles "
                                              "support the apply, the residual and the mass products");
  if (where == PDST_HOST_ASYNC) {
    if (!h->linearized) return fail(PDST_ESTATE, "jacobian used before pdst_linearize");
    CK(cudaSetDevice(h->device));
    const size_t n = (size_t)h->td.k1 * h->g.nd;
    int err = PDST_OK;
    const double* xd = async_in(h, h->as_x, x, n, &err);
    if (err) return err;
    const double* rd = async_in(h, h->as_r, r, n, &err);
    if (err) return err;
    double* yd = async_out_ptr(h, h->as_y, n, &err);
    if (err) return err;
    double* part = h->jpart.ensure_zeroed(jacobian_scratch(h->g, h->td.k1));
    if (!part) return fail(PDST_ECUDA, "out of device memory");
    CK(PDST_TIMED(h, rd ? PK_DEFECT : PK_JACOBIAN, jacobian_apply(h->g, h->td, h->ds, lin_of(h), xd, rd, yd, part, h->stream)));
    if (h->g.th)
      if (int e = th_add(h, xd, yd)) return e;
    if (int e = async_used(h, h->as_x)) return e;
    if (r)
      if (int e = async_used(h, h->as_r)) return e;
    return async_out(h, h->as_y, y, n);
  }
  if (int e = check_where(where)) return e;
  if (!h->linearized) return fail(PDST_ESTATE, "jacobian used before pdst_linearize");
  CK(cudaSetDevice(h->device));
  const size_t n = (size_t)h->td.k1 * h->g.nd;
  int err = PDST_OK;
  const double* xd = stage_in(h, h->scratch_a, x, n, where, &err);
  if (err) return err;
  const double* rd = stage_in(h, h->scratch_c, r, n, where, &err);
  if (err) return err;
  double* yd = out_ptr(h->scratch_b, y, n, where);
  if (!yd) return fail(PDST_ECUDA, "out of device memory");
  double* part = h->jpart.ensure_zeroed(jacobian_scratch(h->g, h->td.k1));
  if (!part) return fail(PDST_ECUDA, "out of device memory");
  CK(PDST_TIMED(h, rd ? PK_DEFECT : PK_JACOBIAN,
                jacobian_apply(h->g, h->td, h->ds, lin_of(h), xd, rd, yd, part, h->stream)));
  if (h->g.th)
    if (int e = th_add(h, xd, yd)) return e;
  return finish_out(h, y, yd, n, where);
}

int pdst_jacobian_apply(pdst_handle* h, const double* x, double* y, int where) {
  return jac_common(h, x, nullptr, y, where);
}

int pdst_jacobian_defect(pdst_handle* h, const double* x, const double* r, double* y, int where) {
  if (!r) return fail(PDST_EINVAL, "null rhs");
  return jac_common(h, x, r, y, where);
}

int pdst_residual(pdst_handle* h, const double* U, const double* v_minus, const double* f_qp, const double* advect,
                  double* R, int where) {
  if (!h || !U || !v_minus || !R) return fail(PDST_EINVAL, "null argument");
  if (int e = check_where(where)) return e;
  if (h->model.delta <= 0.0) return fail(PDST_EDOMAIN, "spatial residual requires delta > 0");
  CK(cudaSetDevice(h->device));
  const Geom& g = h->g;
  const int k1 = h->td.k1;
  const size_t n = (size_t)k1 * g.nd;
  int err = PDST_OK;
  const double* Ud = stage_in(h, h->scratch_a, U, n, where, &err);
  if (err) return err;
  const double* vm = stage_in(h, h->scratch_d, v_minus, g.mv, where, &err);
  if (err) return err;
  const double* fq = stage_in(h, h->scratch_f, f_qp, (size_t)k1 * g.ncells * 32, where, &err);
  if (err) return err;
  const double* ad = stage_in(h, h->scratch_c, advect, n, where, &err);
  if (err) return err;
  double* Rd = out_ptr(h->scratch_b, R, n, where);
  if (!Rd) return fail(PDST_ECUDA, "out of device memory");
  Lin L = lin_of(h);
  CK(PDST_TIMED(h, PK_RESIDUAL,
                slab_residual(g, h->td, h->ds, h->model, L, Ud, ad, vm, fq, h->has_ghat ? h->ghat.ptr : nullptr, Rd,
                              h->stream)));
  if (g.th) {  // Taylor-Hood pressure terms (pdst_th.cu)
    double* cb = h->th_cells.ensure(th_scratch(g, k1));
    if (!cb) return fail(PDST_ECUDA, "out of device memory");
    CK(th_residual(g, h->td, h->th_pressure, Ud, h->has_ghat ? h->ghat.ptr : nullptr, Rd, cb, h->stream));
  }
  return finish_out(h, R, Rd, n, where);
}

int pdst_mass_apply(pdst_handle* h, const double* x, double* y, int where) {
  if (!h || !x || !y) return fail(PDST_EINVAL, "null argument");
  if (int e = check_where(where)) return e;
  CK(cudaSetDevice(h->device));
  const size_t n = (size_t)h->td.k1 * h->g.nd;
  int err = PDST_OK;
  const double* xd = stage_in(h, h->scratch_a, x, n, where, &err);
  if (err) return err;
  double* yd = out_ptr(h->scratch_b, y, n, where);
  if (!yd) return fail(PDST_ECUDA, "out of device memory");
  CK(mass_apply(h->g, h->td, xd, yd, h->stream));
  if (h->g.th) CK(th_pressure_mass(h->g, h->td, xd, yd, h->stream));
  return finish_out(h, y, yd, n, where);
}

static int dot_common(pdst_handle* h, const double* a, const double* b, int64_t n_in, double* out, int where,
                      bool mass) {
  if (!h || !a || !b || !out) return fail(PDST_EINVAL, "null argument");
  if (int e = check_where(where)) return e;
  CK(cudaSetDevice(h->device));
  const size_t n = mass ? (size_t)h->td.k1 * h->g.nd : (size_t)n_in;
  int err = PDST_OK;
  const double* ad = stage_in(h, h->scratch_a, a, n, where, &err);
  if (err) return err;
  const double* bd = stage_in(h, h->scratch_c, b, n, where, &err);
  if (err) return err;
  double* part = h->partials.ensure(reduce_partials() + 1);
  if (!part) return fail(PDST_ECUDA, "out of device memory");
  double* res = where == PDST_DEVICE ? out : part + reduce_partials();
  if (mass && h->g.th) {  // Taylor-Hood: <a, M b> with the consistent Q1 pressure mass
    double* mb = h->scratch_d.ensure(n);
    if (!mb) return fail(PDST_ECUDA, "out of device memory");
    CK(mass_apply(h->g, h->td, bd, mb, h->stream));
    CK(th_pressure_mass(h->g, h->td, bd, mb, h->stream));
    CK(dot(ad, mb, n, part, res, h->stream));
  } else if (mass) {
    CK(mass_dot(h->g, h->td, ad, bd, part, res, h->stream));
  } else {
    CK(dot(ad, bd, n, part, res, h->stream));
  }
  return finish_out(h, out, res, 1, where);
}

int pdst_profile(pdst_handle* h, int enable) {
  if (!h) return fail(PDST_EINVAL, "null handle");
  h->prof.drain();
  for (int k = 0; k < Profiler::NK; ++k) {
    h->prof.total_ms[k] = 0.0;
    h->prof.count[k] = 0;
  }
  h->prof.on = enable != 0;
  return PDST_OK;
}

int pdst_profile_read(pdst_handle* h, int kernel, double* total_ms, int64_t* launches) {
  if (!h) return fail(PDST_EINVAL, "null handle");
  if (kernel < 0 || kernel >= Profiler::NK) return fail(PDST_EINVAL, "kernel class %d out of range", kernel);
  CK(cudaSetDevice(h->device));
  h->prof.drain();
  if (total_ms) *total_ms = h->prof.total_ms[kernel];
  if (launches) *launches = h->prof.count[kernel];
  return PDST_OK;
}

int pdst_mass_dot(pdst_handle* h, const double* a, const double* b, double* out, int where) {
  return dot_common(h, a, b, 0, out, where, true);
}

int pdst_multidot(pdst_handle* h, const double* A, int64_t lda, int m, const double* w, int64_t n, double* out,
                  int where) {
  if (!h || !A || !w || !out) return fail(PDST_EINVAL, "null argument");
  if (where != PDST_DEVICE) return fail(PDST_ENOTSUP, "pdst_multidot takes device pointers only");
  if (m < 0 || n < 0 || lda < n) return fail(PDST_EINVAL, "bad sizes (m=%d, n=%lld, lda=%lld)", m, (long long)n,
                                             (long long)lda);
  CK(cudaSetDevice(h->device));
  double* part = h->kpartials.ensure(multidot_scratch(m > 0 ? m : 1));
  if (!part) return fail(PDST_ECUDA, "out of device memory");
  CK(multidot(A, lda, m, w, n, part, out, h->stream));
  return PDST_OK;
}

int pdst_multi_axpy(pdst_handle* h, const double* A, const double* B, int64_t lda, int m, const double* c, double* w,
                    double* w2, int64_t n, int where) {
  if (!h || !A || !c || !w || (B && !w2)) return fail(PDST_EINVAL, "null argument");
  if (where != PDST_DEVICE) return fail(PDST_ENOTSUP, "pdst_multi_axpy takes device pointers only");
  if (m < 0 || n < 0 || lda < n) return fail(PDST_EINVAL, "bad sizes");
  CK(cudaSetDevice(h->device));
  CK(multi_axpy(A, B, lda, m, c, w, w2, n, h->stream));
  return PDST_OK;
}

int pdst_dot(pdst_handle* h, const double* a, const double* b, int64_t n, double* out, int where) {
  if (n < 0) return fail(PDST_EINVAL, "negative length");
  return dot_common(h, a, b, n, out, where, false);
}

}  // extern "C"

namespace pdst {
// 1-D Gauss(4) / Q2 tables (femspace.py:46-75) as the host computes them.
Tables host_tables() {
  Tables t{};
  const double s[4] = {0.06943184420297371, 0.33000947820757187, 0.6699905217924281, 0.9305681557970262};
  const double w[4] = {0.17392742256872679, 0.3260725774312732, 0.3260725774312732, 0.17392742256872679};
  auto L = [](double x, double out[3]) {
    out[0] = (1.0 - x) * (1.0 - 2.0 * x);
    out[1] = 4.0 * x * (1.0 - x);
    out[2] = x * (2.0 * x - 1.0);
  };
  auto dL = [](double x, double out[3]) {
    out[0] = 4.0 * x - 3.0;
    out[1] = 4.0 - 8.0 * x;
    out[2] = 4.0 * x - 1.0;
  };
  for (int q = 0; q < 4; ++q) {
    t.s[q] = s[q];
    t.w[q] = w[q];
    L(s[q], t.B[q]);
    dL(s[q], t.G[q]);
  }
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double acc = 0.0;
      for (int q = 0; q < 4; ++q) acc += w[q] * t.B[q][i] * t.B[q][j];
      t.M1[i][j] = acc;
    }
  L(0.0, t.E[0]);
  L(1.0, t.E[1]);
  dL(0.0, t.dE[0]);
  dL(1.0, t.dE[1]);
  return t;
}
}  // namespace pdst
