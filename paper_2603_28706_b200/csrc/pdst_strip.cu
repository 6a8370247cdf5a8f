// pdst_strip.cu — the strip partition's data plane inside libpdst (SURVEY.md
// §8e): halo pack / unpack kernels, the fused owned-rows Vanka
// update, and the distributed apply + Vanka step over NCCL point-to-point
// (one rank per GPU, the communicator torch.distributed created) or over
// the ranks of one process (virtual ranks on one device).
//
// A handle becomes rank `rank` of a strip partition with pdst_strip(): its
// mesh is the rank's local strip, global cell rows [c_lo, c_hi), of which it
// owns [a, b) (partition.py RankLayout).  The exchanges, per Radau block,
// are contiguous slices of the node-major local vector:
//   HALO   from the lower rank: node rows [2h, 2a) and the pressures of
//          cells [h, a), h = max(c_lo, a - 2); from the upper rank: node rows
//          [2b, min(2b + 3, 2 c_hi + 1));
//   DEFECT from the upper rank: node row 2b (the patch of cell b-1 reads it);
//   INC    the increment of node row 2b from this rank's patches, added by
//          the upper rank to its own row 2a (= 2b).
// The sends are the neighbours' receives (their layouts come from the
// neighbours' c_hi / c_lo given to pdst_strip), packed into one buffer per
// neighbour and exchange by a pack kernel; the receives unpacked by one
// kernel (add for INC).  No layout metadata travels.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "../../include/pdst.h"
#include "pdst_device.cuh"
#include "pdst_handle.h"
#include "pdst_patch.h"

using namespace pdst;

namespace {

#define CKS(expr)                                                                              \
  do {                                                                                         \
    cudaError_t _e = (expr);                                                                   \
    if (_e != cudaSuccess) return set_error(PDST_ECUDA, "%s: %s", #expr, cudaGetErrorString(_e)); \
  } while (0)

enum { KIND_HALO = 0, KIND_DEFECT = 1, KIND_INC = 2 };
enum { SIDE_LO = 0, SIDE_UP = 1 };

// A list of (offset, length) slices of one Radau block of the local vector.
struct SegList {
  int n = 0;
  int64_t off[2] = {0, 0}, len[2] = {0, 0};
  int64_t total = 0;  // doubles per Radau block
  void add(int64_t o, int64_t l) {
    if (l <= 0) return;
    off[n] = o;
    len[n] = l;
    total += l;
    ++n;
  }
};

// local offsets of the rank's node rows / cell rows (global indices)
struct Local {
  const pdst_handle* h;
  int64_t vel(int Y0) const { return 2 * (int64_t)(Y0 - 2 * h->strip.c_lo) * h->g.nnx; }
  int64_t vlen(int Y0, int Y1) const { return 2 * (int64_t)(Y1 - Y0) * h->g.nnx; }
  int64_t prs(int j0) const { return h->g.mv + 3 * (int64_t)(j0 - h->strip.c_lo) * h->g.nx; }
  int64_t plen(int j0, int j1) const { return 3 * (int64_t)(j1 - j0) * h->g.nx; }
};

// what this rank RECEIVES from `side` for `kind`
SegList recv_plan(const pdst_handle* h, int kind, int side) {
  const auto& s = h->strip;
  const Local L{h};
  SegList out;
  const bool lo = s.rank > 0, up = s.rank < s.nranks - 1;
  if (kind == KIND_HALO) {
    if (side == SIDE_LO && lo) {
      const int hh = std::max(s.c_lo, s.a - 2);
      out.add(L.vel(2 * hh), L.vlen(2 * hh, 2 * s.a));
      out.add(L.prs(hh), L.plen(hh, s.a));
    }
    if (side == SIDE_UP && up) {
      const int top = std::min(2 * s.b + 3, 2 * s.c_hi + 1);
      out.add(L.vel(2 * s.b), L.vlen(2 * s.b, top));
    }
  } else if (kind == KIND_DEFECT) {
    if (side == SIDE_UP && up) out.add(L.vel(2 * s.b), L.vlen(2 * s.b, 2 * s.b + 1));
  } else {  // INC: the lower rank's increment of my row 2a
    if (side == SIDE_LO && lo) out.add(L.vel(2 * s.a), L.vlen(2 * s.a, 2 * s.a + 1));
  }
  return out;
}

// what this rank SENDS to `side` for `kind` (= that neighbour's receive)
SegList send_plan(const pdst_handle* h, int kind, int side) {
  const auto& s = h->strip;
  const Local L{h};
  SegList out;
  const bool lo = s.rank > 0, up = s.rank < s.nranks - 1;
  if (kind == KIND_HALO) {
    if (side == SIDE_LO && lo) {  // the lower rank's rows [2 b_lo, min(2 b_lo + 3, 2 c_hi_lo + 1)), b_lo = a
      const int top = std::min(2 * s.a + 3, 2 * s.lower_c_hi + 1);
      out.add(L.vel(2 * s.a), L.vlen(2 * s.a, top));
    }
    if (side == SIDE_UP && up) {  // the upper rank's rows [2h, 2 a_up), h = max(c_lo_up, a_up - 2), a_up = b
      const int hh = std::max(s.upper_c_lo, s.b - 2);
      out.add(L.vel(2 * hh), L.vlen(2 * hh, 2 * s.b));
      out.add(L.prs(hh), L.plen(hh, s.b));
    }
  } else if (kind == KIND_DEFECT) {
    if (side == SIDE_LO && lo) out.add(L.vel(2 * s.a), L.vlen(2 * s.a, 2 * s.a + 1));
  } else {  // INC: my increment of node row 2b, to the upper rank (the scatter's side output)
    if (side == SIDE_UP && up) out.add(0, 2 * (int64_t)h->g.nnx);
  }
  return out;
}

// blockIdx.y selects one of up to two vectors (vec, vec2); their packed
// blocks follow each other in buf
__global__ void k_pack(const double* __restrict__ vec0, const double* __restrict__ vec1, int64_t nd, SegList L, int k1,
                       double* __restrict__ buf) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= L.total * k1) return;
  const double* vec = blockIdx.y ? vec1 : vec0;
  buf += blockIdx.y * L.total * k1;
  const int mu = (int)(t / L.total);
  int64_t r = t - mu * L.total;
  const int s = r < L.len[0] ? 0 : 1;
  if (s) r -= L.len[0];
  buf[t] = vec[mu * nd + L.off[s] + r];
}

__global__ void k_unpack(double* __restrict__ vec0, double* __restrict__ vec1, int64_t nd, SegList L, int k1,
                         const double* __restrict__ buf, int add) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= L.total * k1) return;
  double* vec = blockIdx.y ? vec1 : vec0;
  buf += blockIdx.y * L.total * k1;
  const int mu = (int)(t / L.total);
  int64_t r = t - mu * L.total;
  const int s = r < L.len[0] ? 0 : 1;
  if (s) r -= L.len[0];
  double* p = vec + mu * nd + L.off[s] + r;
  *p = add ? *p + buf[t] : buf[t];
}

int pack(pdst_handle* h, const double* vec, const double* vec2, const SegList& L, double* buf) {
  if (!L.total) return PDST_OK;
  const int64_t n = L.total * h->td.k1;
  const dim3 grid((unsigned)((n + 255) / 256), vec2 ? 2 : 1);
  PDST_LAUNCH(k_pack<<<grid, 256, 0, h->stream>>>(vec, vec2, h->g.nd, L, h->td.k1, buf));
  CKS(cudaGetLastError());
  return PDST_OK;
}

int unpack(pdst_handle* h, double* vec, double* vec2, const SegList& L, const double* buf, bool add) {
  if (!L.total) return PDST_OK;
  const int64_t n = L.total * h->td.k1;
  const dim3 grid((unsigned)((n + 255) / 256), vec2 ? 2 : 1);
  PDST_LAUNCH(k_unpack<<<grid, 256, 0, h->stream>>>(vec, vec2, h->g.nd, L, h->td.k1, buf, add ? 1 : 0));
  CKS(cudaGetLastError());
  return PDST_OK;
}

// --- NCCL, resolved in the process's already-loaded libnccl (torch's) ---
struct Nccl {
  bool ok = false;
  int (*send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*group_start)() = nullptr;
  int (*group_end)() = nullptr;
  const char* (*err)(int) = nullptr;
};
constexpr int kNcclFloat64 = 8;  // ncclFloat64 / ncclDouble in nccl.h

const Nccl& nccl() {
  static Nccl n;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (lib) {
      n.send = reinterpret_cast<decltype(n.send)>(dlsym(lib, "ncclSend"));
      n.recv = reinterpret_cast<decltype(n.recv)>(dlsym(lib, "ncclRecv"));
      n.group_start = reinterpret_cast<decltype(n.group_start)>(dlsym(lib, "ncclGroupStart"));
      n.group_end = reinterpret_cast<decltype(n.group_end)>(dlsym(lib, "ncclGroupEnd"));
      n.err = reinterpret_cast<decltype(n.err)>(dlsym(lib, "ncclGetErrorString"));
      n.ok = n.send && n.recv && n.group_start && n.group_end;
    }
  }
  return n;
}

#define NCK(expr)                                                                                      \
  do {                                                                                                 \
    int _r = (expr);                                                                                   \
    if (_r != 0) return set_error(PDST_ENCCL, "%s: %s", #expr, nccl().err ? nccl().err(_r) : "nccl error"); \
  } while (0)

double* buf_of(pdst_handle* h, int which, size_t n) {
  return h->strip.buf[which].ensure(std::max<size_t>(n, 1));
}
enum { B_SEND_LO = 0, B_SEND_UP = 1, B_RECV_LO = 2, B_RECV_UP = 3 };

// One exchange of `kind` over the n ranks hs[0..n-1] of vectors vecs (n == 1
// with NCCL: this rank and its communicator; n > 1: virtual ranks of one
// process on one stream, neighbours' send buffers read directly).
int exchange(pdst_handle* const* hs, int n, double* const* vecs, int kind, double* const* vecs2 = nullptr) {
  const bool add = kind == KIND_INC;
  const int nv = vecs2 ? 2 : 1;  // vectors exchanged together (one pack, transfer and unpack)
  for (int r = 0; r < n; ++r) {
    pdst_handle* h = hs[r];
    const int k1 = h->td.k1;
    for (int side = 0; side < 2; ++side) {
      if (kind == KIND_INC) continue;  // the scatter wrote the INC send buffer
      const SegList L = send_plan(h, kind, side);
      if (!L.total) continue;
      double* b = buf_of(h, side == SIDE_LO ? B_SEND_LO : B_SEND_UP, (size_t)L.total * k1 * nv);
      if (!b) return set_error(PDST_ECUDA, "out of device memory (strip buffers)");
      if (int e = pack(h, vecs[r], vecs2 ? vecs2[r] : nullptr, L, b)) return e;
    }
  }
  if (n == 1 && hs[0]->strip.nccl) {
    pdst_handle* h = hs[0];
    const int k1 = h->td.k1;
    const Nccl& N = nccl();
    const SegList rl = recv_plan(h, kind, SIDE_LO), ru = recv_plan(h, kind, SIDE_UP);
    const SegList sl = send_plan(h, kind, SIDE_LO), su = send_plan(h, kind, SIDE_UP);
    double* brl = buf_of(h, B_RECV_LO, (size_t)rl.total * k1 * nv);
    double* bru = buf_of(h, B_RECV_UP, (size_t)ru.total * k1 * nv);
    if (!brl || !bru) return set_error(PDST_ECUDA, "out of device memory (strip buffers)");
    NCK(N.group_start());
    if (sl.total) NCK(N.send(h->strip.buf[B_SEND_LO].ptr, (size_t)sl.total * k1 * nv, kNcclFloat64, h->strip.rank - 1,
                             h->strip.nccl, h->stream));
    if (su.total) NCK(N.send(h->strip.buf[B_SEND_UP].ptr, (size_t)su.total * k1 * nv, kNcclFloat64, h->strip.rank + 1,
                             h->strip.nccl, h->stream));
    if (rl.total)
      NCK(N.recv(brl, (size_t)rl.total * k1 * nv, kNcclFloat64, h->strip.rank - 1, h->strip.nccl, h->stream));
    if (ru.total)
      NCK(N.recv(bru, (size_t)ru.total * k1 * nv, kNcclFloat64, h->strip.rank + 1, h->strip.nccl, h->stream));
    NCK(N.group_end());
    if (int e = unpack(h, vecs[0], vecs2 ? vecs2[0] : nullptr, rl, brl, add)) return e;
    if (int e = unpack(h, vecs[0], vecs2 ? vecs2[0] : nullptr, ru, bru, add)) return e;
    return PDST_OK;
  }
  // virtual ranks: my receive from the lower rank is its send to its upper
  // side, and vice versa (the sizes agree by construction of the plans)
  for (int r = 0; r < n; ++r) {
    pdst_handle* h = hs[r];
    if (r > 0) {
      const SegList rl = recv_plan(h, kind, SIDE_LO);
      if (rl.total)
        if (int e = unpack(h, vecs[r], vecs2 ? vecs2[r] : nullptr, rl, hs[r - 1]->strip.buf[B_SEND_UP].ptr, add))
          return e;
    }
    if (r + 1 < n) {
      const SegList ru = recv_plan(h, kind, SIDE_UP);
      if (ru.total)
        if (int e = unpack(h, vecs[r], vecs2 ? vecs2[r] : nullptr, ru, hs[r + 1]->strip.buf[B_SEND_LO].ptr, add))
          return e;
    }
  }
  return PDST_OK;
}

int check_strips(pdst_handle* const* hs, int n) {
  if (!hs || n < 1) return set_error(PDST_EINVAL, "no ranks");
  for (int r = 0; r < n; ++r) {
    pdst_handle* h = hs[r];
    if (!h || !h->strip.on) return set_error(PDST_ESTATE, "rank %d: pdst_strip not called", r);
    if (!h->linearized || !h->patches_valid)
      return set_error(PDST_ESTATE, "rank %d: strip step needs pdst_linearize and pdst_patches_build", r);
    if (n > 1 && (h->strip.rank != r || h->strip.nranks != n))
      return set_error(PDST_EINVAL, "virtual ranks must be given in partition order (rank %d)", r);
    if (n > 1 && (h->device != hs[0]->device))
      return set_error(PDST_EINVAL, "virtual ranks must share one device");
  }
  if (n == 1 && hs[0]->strip.nranks > 1 && !hs[0]->strip.nccl)
    return set_error(PDST_ESTATE, "a rank of a multi-rank partition needs pdst_strip_comm (NCCL)");
  return PDST_OK;
}

// y_r = J x_r and one Vanka step on d_r (rhs r_r) on every rank, owner computes.
int strip_step(pdst_handle* const* hs, int n, double* const* xs, double* const* ys, double* const* ds,
               const double* const* rs, double omega) {
  if (int e = check_strips(hs, n)) return e;
  cudaStream_t st = hs[0]->stream;
  CKS(cudaSetDevice(hs[0]->device));
  for (int r = 1; r < n; ++r) hs[r]->stream = st;
  if (int e = exchange(hs, n, xs, KIND_HALO, ds)) return e;  // x and d halos together
  std::vector<double*> defects(n);
  for (int r = 0; r < n; ++r) {
    pdst_handle* h = hs[r];
    const int k1 = h->td.k1;
    const size_t nl = (size_t)k1 * h->g.nd;
    double* part = h->jpart.ensure_zeroed(jacobian_scratch(h->g, k1));
    defects[r] = h->defect.ensure(nl);
    if (!part || !defects[r]) return set_error(PDST_ECUDA, "out of device memory");
    CKS(PDST_TIMED(h, PK_JACOBIAN, jacobian_apply(h->g, h->td, h->ds, lin_of(h), xs[r], nullptr, ys[r], part, st)));
    CKS(PDST_TIMED(h, PK_DEFECT, jacobian_apply(h->g, h->td, h->ds, lin_of(h), ds[r], rs[r], defects[r], part, st)));
  }
  if (int e = exchange(hs, n, defects.data(), KIND_DEFECT)) return e;
  for (int r = 0; r < n; ++r) {
    pdst_handle* h = hs[r];
    const auto& s = h->strip;
    const int k1 = h->td.k1;
    Level* lv = h->levels.back();
    double* upd = h->upd.ensure((size_t)h->g.ncells * 21 * k1);
    if (!upd) return set_error(PDST_ECUDA, "out of device memory");
    if (lv->diag)
      CKS(PDST_TIMED(h, PK_VANKA_GEMV, vanka_gemv_diag(h->g, lv->tdiag, lv->binv.ptr, defects[r], upd, st)));
    else
      CKS(PDST_TIMED(h, PK_VANKA_GEMV, vanka_gemv(h->g, k1, lv->invs.ptr, defects[r], upd, st)));
    // d += omega sum over the OWNED patches; node row 2b's increment also to
    // the INC send buffer (the upper rank adds it to its row 2a)
    const bool up = s.rank < s.nranks - 1;
    double* inc = up ? buf_of(h, B_SEND_UP, 2 * (size_t)h->g.nnx * k1) : nullptr;
    if (up && !inc) return set_error(PDST_ECUDA, "out of device memory (strip buffers)");
    CKS(PDST_TIMED(h, PK_VANKA_SCATTER, vanka_scatter(h->g, k1, upd, omega, ds[r], st, s.a - s.c_lo, s.b - s.c_lo,
                                                      false, inc, up ? 2 * (s.b - s.c_lo) : -1)));
  }
  if (int e = exchange(hs, n, ds, KIND_INC)) return e;
  return PDST_OK;
}

}  // namespace

extern "C" {

int pdst_strip(pdst_handle* h, int rank, int nranks, int ny_global, int a, int b, int c_lo, int c_hi, int lower_c_hi,
               int upper_c_lo) {
  if (h && h->g.th) return set_error(PDST_ENOTSUP, "the strip partition is Q2/P1disc-only (Taylor-Hood handles: apply, residual, mass)");
  if (!h) return set_error(PDST_EINVAL, "null handle");
  if (nranks < 1 || rank < 0 || rank >= nranks) return set_error(PDST_EINVAL, "bad rank %d of %d", rank, nranks);
  if (!(0 <= c_lo && c_lo <= a && a < b && b <= c_hi && c_hi <= ny_global))
    return set_error(PDST_EINVAL, "inconsistent strip rows");
  if (c_hi - c_lo != h->g.ny) return set_error(PDST_EINVAL, "local mesh has %d cell rows, the strip %d", h->g.ny,
                                               c_hi - c_lo);
  if (rank > 0 && (a - c_lo < 2 || lower_c_hi < a + 1))
    return set_error(PDST_EINVAL, "rank %d: needs two ghost cell rows below", rank);
  if (rank < nranks - 1 && (c_hi - b < 2 || upper_c_lo > b - 1 || b < 2))
    return set_error(PDST_EINVAL, "rank %d: needs two ghost cell rows above", rank);
  auto& s = h->strip;
  s.on = true;
  s.rank = rank;
  s.nranks = nranks;
  s.ny = ny_global;
  s.a = a;
  s.b = b;
  s.c_lo = c_lo;
  s.c_hi = c_hi;
  s.lower_c_hi = lower_c_hi;
  s.upper_c_lo = upper_c_lo;
  return PDST_OK;
}

int pdst_strip_comm(pdst_handle* h, void* nccl_comm) {
  if (!h) return set_error(PDST_EINVAL, "null handle");
  if (nccl_comm && !nccl().ok)
    return set_error(PDST_ENCCL, "libnccl.so.2 is not loadable in this process (ncclSend / ncclRecv not found)");
  h->strip.nccl = nccl_comm;
  return PDST_OK;
}

int pdst_strip_halo(pdst_handle* h, double* x) {
  pdst_handle* hs[1] = {h};
  if (!h || !x) return set_error(PDST_EINVAL, "null argument");
  if (!h->strip.on) return set_error(PDST_ESTATE, "pdst_strip not called");
  if (h->strip.nranks > 1 && !h->strip.nccl) return set_error(PDST_ESTATE, "pdst_strip_comm not called");
  CKS(cudaSetDevice(h->device));
  double* v[1] = {x};
  return exchange(hs, 1, v, KIND_HALO);
}

int pdst_strip_step(pdst_handle* h, const double* x, double* y, double* d, const double* r, double omega) {
  if (!h || !x || !y || !d || !r) return set_error(PDST_EINVAL, "null argument");
  pdst_handle* hs[1] = {h};
  double* xs[1] = {const_cast<double*>(x)};
  double* ys[1] = {y};
  double* ds[1] = {d};
  const double* rs[1] = {r};
  return strip_step(hs, 1, xs, ys, ds, rs, omega);
}

int pdst_strips_step_local(pdst_handle* const* hs, int nranks, double* const* xs, double* const* ys,
                           double* const* ds, const double* const* rs, double omega) {
  if (!xs || !ys || !ds || !rs) return set_error(PDST_EINVAL, "null argument");
  for (int q = 0; q < nranks; ++q)
    if (!xs[q] || !ys[q] || !ds[q] || !rs[q]) return set_error(PDST_EINVAL, "null vector of rank %d", q);
  return strip_step(hs, nranks, xs, ys, ds, rs, omega);
}

}  // extern "C"
