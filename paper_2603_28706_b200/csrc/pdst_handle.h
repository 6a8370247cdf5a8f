// pdst_handle.h — the opaque handle behind include/pdst.h.
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "pdst_device.cuh"
#include "pdst_internal.h"
#include "pdst_patch.h"

struct pdst_handle;

namespace pdst {

// Destroys a rediscretized level's handle (pdst_mg.cu).
void destroy_child(pdst_handle* c);

struct DeviceBuffer {
  double* ptr = nullptr;
  size_t cap = 0;
  DeviceBuffer() = default;
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  ~DeviceBuffer() { release(); }
  double* ensure(size_t n);
  // As ensure(), zero-filling a fresh allocation (counters that must start at 0).
  double* ensure_zeroed(size_t n);
  void release();
};

Geom make_geom(int nx, int ny, double x0, double y0, double x1, double y1, const uint8_t* dirichlet_dev, int th = 0);

// One multigrid level.  Level L-1 is the handle's own (finest) mesh whose
// operator is matrix free; coarser levels carry Galerkin element operators.
struct Level {
  Geom g{};
  uint8_t* dirichlet = nullptr;
  std::vector<uint8_t> dirichlet_host;
  bool all_dirichlet = true;
  // Galerkin element representation per node mu (coarse levels only):
  //   ecell [k1][ncells][21][21]       volume + boundary blocks
  //   efx   [k1][ny][nx-1][18][18]     couplings across vertical faces (L,R) as
  //   efy   [k1][ny-1][nx][18][18]     the 2x2 block structure LL, LR, RL, RR
  //                                    stored as 4 x (9x9 node blocks x I2)
  DeviceBuffer ecell, efx, efy;
  // patches
  DeviceBuffer mats, invs;
  int D = 0;
  // surrogate patches in temporally diagonalized form (pdst_timediag.cu)
  bool diag = false;
  TimeDiag tdiag{};
  DeviceBuffer spatial, binv;
  // coarsest level: dense inverse of the (pinned) slab matrix
  DeviceBuffer dense;
  DeviceBuffer ipiv;
  // work vectors (k1 * nd each)
  DeviceBuffer w0, w1, w2, w3;
  // coarsest-level FGMRES: basis V [(m+1) n], preconditioned directions Z [m n],
  // work vector, reduction scratch
  DeviceBuffer kv, kz, kw, ks;
  // coarse_mode "rediscretize" (multigrid.py:302-324, 406-431): the level's
  // operator is the matrix-free Jacobian of its own mesh, linearized at the
  // injected state, held by a child handle (which also owns the level's exact
  // patches and, on the coarsest level, its coarse solve)
  pdst_handle* child = nullptr;
  ~Level() {
    if (child) destroy_child(child);
    if (dirichlet) cudaFree(dirichlet);
  }
};

// Optional CUDA-event timing of every kernel launch (bench / roofline).
struct Profiler {
  static constexpr int NK = 8;
  bool on = false;
  std::vector<cudaEvent_t> pool;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending[NK];
  double total_ms[NK] = {0};
  long long count[NK] = {0};
  cudaEvent_t get() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
  void drain() {
    for (int k = 0; k < NK; ++k) {
      for (auto& pr : pending[k]) {
        float ms = 0.f;
        cudaEventSynchronize(pr.second);
        cudaEventElapsedTime(&ms, pr.first, pr.second);
        total_ms[k] += ms;
        count[k] += 1;
        pool.push_back(pr.first);
        pool.push_back(pr.second);
      }
      pending[k].clear();
    }
  }
  ~Profiler() {
    for (int k = 0; k < NK; ++k)
      for (auto& pr : pending[k]) {
        cudaEventDestroy(pr.first);
        cudaEventDestroy(pr.second);
      }
    for (auto e : pool) cudaEventDestroy(e);
  }
};

}  // namespace pdst

namespace pdst {
// Device staging buffer of one PDST_HOST_ASYNC argument with the events that
// order it: in_done (H2D finished, on the copy-in stream), use_done (the last
// kernel reading / writing it finished, on the compute stream), out_done (its
// D2H finished, on the copy-out stream).
struct AsyncSlot {
  DeviceBuffer buf;
  cudaEvent_t in_done = nullptr, use_done = nullptr, out_done = nullptr;
  bool used = false, outed = false;
  ~AsyncSlot() {
    if (in_done) cudaEventDestroy(in_done);
    if (use_done) cudaEventDestroy(use_done);
    if (out_done) cudaEventDestroy(out_done);
  }
};
}  // namespace pdst

struct pdst_handle {
  int device = 0;
  cudaStream_t stream = nullptr;
  pdst::Geom g{};
  uint8_t* dirichlet = nullptr;
  std::vector<uint8_t> dirichlet_host;
  double extents[4] = {0, 0, 1, 1};
  pdst::TimeData td{};
  pdst::Disc ds{};
  bool th_pressure = false;      // Taylor-Hood handle: pressure coupling enabled (pdst_th.cu)
  pdst::DeviceBuffer th_cells;   // Taylor-Hood per-cell contributions
  pdst::Model model{};
  double tau = 0.0;
  std::vector<double> nodes;
  std::vector<double> weights;  // Radau weights as given (tau_w = tau * weights)

  // linearization caches
  pdst::DeviceBuffer state;  // (k1, Mv)
  pdst::DeviceBuffer eta, gam, etaf, gamf;
  pdst::DeviceBuffer etad, betad, dg;
  pdst::DeviceBuffer bmat;  // boundary-side matrices of the linearization
  pdst::DeviceBuffer apc;   // apply cache of the linearization (the Jacobian apply's coefficient stream)
  pdst::DeviceBuffer ghat;
  bool has_ghat = false;
  bool linearized = false;

  // staging for host pointers
  pdst::DeviceBuffer scratch_a, scratch_b, scratch_c, scratch_d, scratch_f;
  pdst::DeviceBuffer partials;
  pdst::DeviceBuffer kpartials;  // FGMRES multi-dot partial sums
  pdst::DeviceBuffer ppartials;  // mean-pressure projection partial sums
  pdst::DeviceBuffer jpart;  // Jacobian tile-boundary partial sums (+ the tile pass's completion counters)

  // surrogate (representative-state) linearization and patch scratch
  pdst::DeviceBuffer state_rep, eta_rep, gam_rep, etaf_rep, gamf_rep;
  pdst::DeviceBuffer ET, upd, defect, ibuf;
  pdst::DeviceBuffer lvs;  // coarse level apply: element products (level_apply_scratch)

  pdst::Profiler prof;

  // PDST_HOST_ASYNC: copy streams, one slot per (entry point, argument), and
  // the host buffers with a D2H in flight (an H2D from one waits for it)
  cudaStream_t copy_in = nullptr, copy_out = nullptr;
  pdst::AsyncSlot as_x, as_r, as_y, as_d, as_vr;
  std::vector<std::pair<const void*, cudaEvent_t>> pending_out;

  // strip partition (pdst_strip.cu): this handle's mesh is rank `rank`'s
  // local strip, global cell rows [c_lo, c_hi), owned [a, b); the neighbours'
  // local row ranges define what they receive; nccl = the communicator of
  // the ranks (or null for virtual ranks of one process)
  struct StripInfo {
    bool on = false;
    int rank = 0, nranks = 1, ny = 0, a = 0, b = 0, c_lo = 0, c_hi = 0, lower_c_hi = 0, upper_c_lo = 0;
    void* nccl = nullptr;
    pdst::DeviceBuffer buf[4];  // send to lower / upper, receive from lower / upper
  } strip;

  // multigrid
  std::vector<pdst::Level*> levels;  // 0 = coarsest
  int min_cells = 0;
  // coarsest-level solve (pdst_set_coarse_solver): 0 dense (the reference's
  // LU, <= 16384 dofs), 1 `coarse_sweeps` Vanka steps from zero with
  // `coarse_omega`, 2 dense up to 4096 dofs else FGMRES, 3 FGMRES
  // right-preconditioned by `coarse_sweeps` Vanka steps
  int coarse_mode = 0;  // 0 galerkin, 1 rediscretize (pdst_set_coarse_mode)
  int coarse_kind = 0;
  int coarse_sweeps = 30;
  double coarse_omega = 0.7;
  int coarse_iters = 30;        // FGMRES iteration cap (PDST_COARSE_FGMRES)
  double coarse_rtol = 1.0e-6;  // FGMRES relative residual target
  bool coarse_iterative = false;  // resolved at pdst_patches_build
  bool coarse_valid = false;  // Galerkin operators / coarse patches / dense solve built
  bool patches_valid = false;

  ~pdst_handle() {
    if (copy_in) cudaStreamDestroy(copy_in);
    if (copy_out) cudaStreamDestroy(copy_out);
    for (auto* l : levels) delete l;
    if (dirichlet) cudaFree(dirichlet);
  }
};

namespace pdst {
// Record the message returned by pdst_last_error(); returns `code`.
int set_error(int code, const char* fmt, ...);
// Host/device argument staging (where = PDST_HOST copies through the handle).
const double* stage_in(pdst_handle* h, DeviceBuffer& buf, const double* p, size_t n, int where, int* err);
double* out_ptr(DeviceBuffer& buf, double* p, size_t n, int where);
int finish_out(pdst_handle* h, double* host, const double* dev, size_t n, int where);
int check_where(int where);
// PDST_HOST_ASYNC staging (page-locked host buffers; see pdst.h): H2D of p into
// the slot on the copy-in stream, ordered before the next compute-stream work;
// async_used after the kernels that touched the slot; async_out D2H of the slot
// into p on the copy-out stream after them.  The call returns at once.
const double* async_in(pdst_handle* h, AsyncSlot& s, const double* p, size_t n, int* err);
double* async_out_ptr(pdst_handle* h, AsyncSlot& s, size_t n, int* err);
int async_used(pdst_handle* h, AsyncSlot& s);
int async_out(pdst_handle* h, AsyncSlot& s, double* p, size_t n);

// Kernel classes for pdst_profile_read.
enum { PK_JACOBIAN = 0, PK_VANKA_GEMV = 1, PK_VANKA_SCATTER = 2, PK_RESIDUAL = 3, PK_TRANSFER = 4, PK_LEVEL = 5,
       PK_DEFECT = 6 /* the finest Jacobian apply with a right-hand side: y = r - J x */ };

// Launch `expr` (a cudaError_t expression) bracketed by profiling events when enabled.
#define PDST_TIMED(h, kid, expr)                                      \
  ([&]() -> cudaError_t {                                            \
    if (!(h)->prof.on) return (expr);                                \
    cudaEvent_t _a = (h)->prof.get(), _b = (h)->prof.get();          \
    cudaEventRecord(_a, (h)->stream);                                \
    cudaError_t _r = (expr);                                         \
    cudaEventRecord(_b, (h)->stream);                                \
    (h)->prof.pending[(kid)].push_back({_a, _b});                    \
    return _r;                                                       \
  }())

inline Lin lin_of(pdst_handle* h) {
  Lin L{};
  L.eta = h->eta.ptr;
  L.gam = h->gam.ptr;
  L.etaf = h->etaf.ptr;
  L.gamf = h->gamf.ptr;
  L.etad = h->etad.ptr;
  L.betad = h->betad.ptr;
  L.dg = h->dg.ptr;
  L.bmat = h->bmat.ptr;
  L.apc = h->apc.ptr;
  L.has_gamma = h->model.kind != 0;
  return L;
}
}  // namespace pdst
