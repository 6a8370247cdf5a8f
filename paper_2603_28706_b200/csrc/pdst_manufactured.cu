// pdst_manufactured.cu — the manufactured-solution benchmark problem on the
// device: the closed-form body force at the residual's
// volume points and the space-time error norms of a slab trajectory.
//
// Reference (file:line into /root/reference/pkg/src/pdflow):
//   ManufacturedCase fields / forcing   bench/manufactured.py:30-167
//   error_norms (e_phi, e_div)          bench/metrics.py:35-85
//   phi_scale_field                     constitutive.py:340-351
// The prescribed velocity is s(t) (a(x) b(y), -b(x) a(y)) with
// a = sin^2(pi x), b = sin(2 pi x) / 2, s = sin t; pressure s b(x) b(y).
#include <cmath>
#include <vector>

#include "../../include/pdst.h"
#include "pdst_device.cuh"
#include "pdst_handle.h"
#include "pdst_internal.h"

namespace pdst {
namespace {

constexpr double kPi = 3.141592653589793;

struct Ab {  // a, a', a'', b, b', b'' at one coordinate
  double a, da, dda, b, db, ddb;
};

__device__ __forceinline__ Ab ab_at(double x) {
  const double s1 = sin(kPi * x), s2 = sin(2.0 * kPi * x), c2 = cos(2.0 * kPi * x);
  Ab r;
  r.a = s1 * s1;
  r.da = kPi * s2;
  r.dda = 2.0 * kPi * kPi * c2;
  r.b = 0.5 * s2;
  r.db = kPi * c2;
  r.ddb = -2.0 * kPi * kPi * s2;
  return r;
}

// Strong-form forcing f = dv/dt + (v . grad) v - div S(Dv) + grad pi
// (manufactured.py:121-157), at (x, y, t).
__device__ void mf_forcing(const Model& m, double x, double y, double t, double f[2]) {
  const Ab X = ab_at(x), Y = ab_at(y);
  const double s = sin(t), c = cos(t);
  const double v0 = s * X.a * Y.b, v1 = -s * X.b * Y.a;
  // g[d][k] = d v_d / d x_k
  const double g00 = s * X.da * Y.b, g01 = s * X.a * Y.db;
  const double g10 = -s * X.db * Y.a, g11 = -s * X.b * Y.da;
  // h[d][k][l]
  const double h000 = s * X.dda * Y.b, h001 = s * X.da * Y.db, h011 = s * X.a * Y.ddb;
  const double h100 = -s * X.ddb * Y.a, h101 = -s * X.db * Y.da, h111 = -s * X.b * Y.dda;
  const double conv0 = v0 * g00 + v1 * g01, conv1 = v0 * g10 + v1 * g11;
  const double a11 = g00, a22 = g11, a12 = 0.5 * (g01 + g10);
  // d a / d x_k
  const double da11_0 = h000, da11_1 = h001;
  const double da22_0 = h101, da22_1 = h111;
  const double da12_0 = 0.5 * (h001 + h100), da12_1 = 0.5 * (h011 + h101);
  const double a_sq = a11 * a11 + a22 * a22 + 2.0 * a12 * a12;
  const double dasq0 = 2.0 * (a11 * da11_0 + a22 * da22_0 + 2.0 * a12 * da12_0);
  const double dasq1 = 2.0 * (a11 * da11_1 + a22 * da22_1 + 2.0 * a12 * da12_1);
  const double dsq = m.delta * m.delta + a_sq;
  const double eta = m.nu_inf + m.nu * pow(dsq, (m.p - 2.0) / 2.0);
  const double dfac = m.nu * ((m.p - 2.0) / 2.0) * pow(dsq, (m.p - 4.0) / 2.0);
  const double deta0 = dfac * dasq0, deta1 = dfac * dasq1;
  const double ds0 = deta0 * a11 + deta1 * a12 + eta * (da11_0 + da12_1);
  const double ds1 = deta0 * a12 + deta1 * a22 + eta * (da12_0 + da22_1);
  const double vt0 = c * X.a * Y.b, vt1 = -c * X.b * Y.a;
  const double gp0 = s * X.db * Y.b, gp1 = s * X.b * Y.db;
  f[0] = vt0 + conv0 - ds0 + gp0;
  f[1] = vt1 + conv1 - ds1 + gp1;
}

// Exact symmetric gradient (a11, a22, a12) at (x, y, t) (manufactured.py:113-118).
__device__ void mf_sym_grad(double x, double y, double t, double A[3]) {
  const Ab X = ab_at(x), Y = ab_at(y);
  const double s = sin(t);
  const double g00 = s * X.da * Y.b, g01 = s * X.a * Y.db, g10 = -s * X.db * Y.a, g11 = -s * X.b * Y.da;
  A[0] = g00;
  A[1] = g11;
  A[2] = 0.5 * (g01 + g10);
}

// phi_scale_field (constitutive.py:340-351): (delta^2 + |A|^2)^((p-2)/4), with
// the zero-limit convention at delta = 0.
__device__ __forceinline__ double phi_scale(const Model& m, double a_sq) {
  const double dsq = m.delta * m.delta + a_sq;
  if (m.delta == 0.0) return dsq > 0.0 ? pow(dsq, (m.p - 2.0) / 4.0) : 0.0;
  return pow(dsq, (m.p - 2.0) / 4.0);
}

struct MfTimes {
  int k1;
  double t[MAXK1];
};

// f at the x-major volume points (cell origin + Gauss point * cell size,
// forms.py:189-191) of every cell and Radau node: fqp[mu][cell][q][2].
__global__ void k_mf_forcing(Geom g, Model m, MfTimes tt, double x0, double y0, double* __restrict__ fqp) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;  // cell * 16 + q
  const int mu = blockIdx.y;
  if (i >= (size_t)g.ncells * 16 || mu >= tt.k1) return;
  const int c = (int)(i / 16), q = (int)(i % 16);
  const int ci = c % g.nx, cj = c / g.nx;
  const double ox = x0 + ci * g.hx, oy = y0 + cj * g.hy;
  const double x = ox + c_tab.s[q / 4] * g.hx, y = oy + c_tab.s[q % 4] * g.hy;
  double f[2];
  mf_forcing(m, x, y, tt.t[mu], f);
  double* o = fqp + ((size_t)mu * g.ncells * 16 + i) * 2;
  o[0] = f[0];
  o[1] = f[1];
}

constexpr int MFQ = 8;  // max 1-D spatial / temporal points
struct ErrTabs {
  int q, ntp, k1;
  double s[MFQ], w[MFQ];          // spatial Gauss points / weights on [0, 1]
  double L[MFQ][3], dL[MFQ][3];   // 1-D Q2 values / derivatives at s
  double tg[MFQ], tw[MFQ];        // temporal Gauss points / weights on [0, 1]
  double blend[MFQ][MAXK1];       // Radau Lagrange basis at tg
};

constexpr int EB = 128;

// Per-cell contributions to (e_phi^2, e_div^2) of one slab (metrics.py:60-83),
// block partial sums in a fixed order.
__global__ void __launch_bounds__(EB) k_error_norms(Geom g, Model m, ErrTabs T, double x0, double y0, double t0,
                                                   double tau, const double* __restrict__ U,
                                                   double* __restrict__ partial) {
  __shared__ double red[2][EB];
  const int c = blockIdx.x * EB + threadIdx.x;
  double ep = 0.0, ed = 0.0;
  if (c < g.ncells) {
    const int ci = c % g.nx, cj = c / g.nx;
    const double ox = x0 + ci * g.hx, oy = y0 + cj * g.hy;
    for (int ig = 0; ig < T.ntp; ++ig) {
      const double tcur = t0 + tau * T.tg[ig];
      // blended nodal velocity of the cell
      double loc[9][2];
      for (int a = 0; a < 9; ++a) {
        const size_t node = (size_t)(2 * cj + a / 3) * g.nnx + 2 * ci + a % 3;
        double v0 = 0.0, v1 = 0.0;
        for (int mu = 0; mu < T.k1; ++mu) {
          v0 += T.blend[ig][mu] * U[(size_t)mu * g.nd + 2 * node];
          v1 += T.blend[ig][mu] * U[(size_t)mu * g.nd + 2 * node + 1];
        }
        loc[a][0] = v0;
        loc[a][1] = v1;
      }
      double sp = 0.0, sd = 0.0;
      for (int qx = 0; qx < T.q; ++qx)
        for (int qy = 0; qy < T.q; ++qy) {
          double gh[2][2] = {{0, 0}, {0, 0}};
          for (int a = 0; a < 9; ++a) {
            const int ix = a % 3, jy = a / 3;
            const double gx = T.dL[qx][ix] * T.L[qy][jy] * g.ihx, gy = T.L[qx][ix] * T.dL[qy][jy] * g.ihy;
            gh[0][0] += gx * loc[a][0];
            gh[0][1] += gy * loc[a][0];
            gh[1][0] += gx * loc[a][1];
            gh[1][1] += gy * loc[a][1];
          }
          const double ah0 = gh[0][0], ah1 = gh[1][1], ah2 = 0.5 * (gh[0][1] + gh[1][0]);
          double ae[3];
          mf_sym_grad(ox + T.s[qx] * g.hx, oy + T.s[qy] * g.hy, tcur, ae);
          const double ph = phi_scale(m, ah0 * ah0 + ah1 * ah1 + 2.0 * ah2 * ah2);
          const double pe = phi_scale(m, ae[0] * ae[0] + ae[1] * ae[1] + 2.0 * ae[2] * ae[2]);
          const double d0 = ph * ah0 - pe * ae[0], d1 = ph * ah1 - pe * ae[1], d2 = ph * ah2 - pe * ae[2];
          const double wq = T.w[qx] * T.w[qy] * (g.hx * g.hy);
          sp += wq * (d0 * d0 + d1 * d1 + 2.0 * d2 * d2);
          const double dv = gh[0][0] + gh[1][1];
          sd += wq * dv * dv;
        }
      ep += tau * T.tw[ig] * sp;
      ed += tau * T.tw[ig] * sd;
    }
  }
  red[0][threadIdx.x] = ep;
  red[1][threadIdx.x] = ed;
  __syncthreads();
  for (int s = EB / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      red[0][threadIdx.x] += red[0][threadIdx.x + s];
      red[1][threadIdx.x] += red[1][threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    partial[2 * blockIdx.x] = red[0][0];
    partial[2 * blockIdx.x + 1] = red[1][0];
  }
}

// Gauss-Legendre points / weights on [0, 1] (numpy.polynomial.legendre.leggauss
// mapped as in metrics.py:30-32), by Newton iteration on P_n.
void gauss01(int n, double* x, double* w) {
  for (int i = 0; i < n; ++i) {
    double z = std::cos(kPi * (i + 0.75) / (n + 0.5)), dp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = z;
      for (int k = 2; k <= n; ++k) {
        const double pk = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = pk;
      }
      if (n == 1) {
        p1 = z;
        p0 = 1.0;
      }
      dp = n * (z * p1 - p0) / (z * z - 1.0);
      const double dz = p1 / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-16) break;
    }
    // ascending order on [0, 1]
    x[n - 1 - i] = (z + 1.0) / 2.0;
    w[n - 1 - i] = (2.0 / ((1.0 - z * z) * dp * dp)) / 2.0;
  }
}

// Lagrange cardinals of the Radau nodes at `that` (timebasis.py:85-93).
std::vector<double> cardinals_at(const std::vector<double>& nodes, double that) {
  const size_t n = nodes.size();
  std::vector<double> out(n, 1.0);
  for (size_t mu = 0; mu < n; ++mu) {
    double val = 1.0;
    for (size_t nu = 0; nu < n; ++nu)
      if (nu != mu) val = val * (that - nodes[nu]) / (nodes[mu] - nodes[nu]);
    out[mu] = val;
  }
  return out;
}

}  // namespace
}  // namespace pdst

using namespace pdst;

extern "C" {

int pdst_manufactured_forcing(pdst_handle* h, double t_start, double* fqp, int where) {
  if (h && h->g.th) return set_error(PDST_ENOTSUP, "the manufactured forcing is Q2/P1disc-only (Taylor-Hood handles: apply, residual, mass)");
  if (!h || !fqp) return set_error(PDST_EINVAL, "null argument");
  if (int e = check_where(where)) return e;
  if (cudaSetDevice(h->device) != cudaSuccess) return set_error(PDST_ECUDA, "cudaSetDevice failed");
  const Geom& g = h->g;
  MfTimes tt{};
  tt.k1 = h->td.k1;
  for (int mu = 0; mu < tt.k1; ++mu) tt.t[mu] = t_start + h->tau * h->nodes[mu];
  const size_t n = (size_t)tt.k1 * g.ncells * 32;
  double* out = out_ptr(h->scratch_f, fqp, n, where);
  if (!out) return set_error(PDST_ECUDA, "out of device memory");
  const size_t items = (size_t)g.ncells * 16;
  PDST_LAUNCH(k_mf_forcing<<<dim3((unsigned)((items + 127) / 128), tt.k1), 128, 0, h->stream>>>(
      g, h->model, tt, h->extents[0], h->extents[1], out));
  if (cudaGetLastError() != cudaSuccess) return set_error(PDST_ECUDA, "k_mf_forcing launch failed");
  return finish_out(h, fqp, out, n, where);
}

int pdst_error_norms(pdst_handle* h, const double* U, double t0, double t1, int spatial_points, int temporal_points,
                     double* sq2, int where) {
  if (h && h->g.th) return set_error(PDST_ENOTSUP, "the error norms is Q2/P1disc-only (Taylor-Hood handles: apply, residual, mass)");
  if (!h || !U || !sq2) return set_error(PDST_EINVAL, "null argument");
  if (int e = check_where(where)) return e;
  if (spatial_points < 1 || spatial_points > MFQ || temporal_points < 1 || temporal_points > MFQ)
    return set_error(PDST_EINVAL, "quadrature orders must lie in [1, %d]", MFQ);
  if (!(t1 > t0)) return set_error(PDST_EINVAL, "empty slab interval");
  if (cudaSetDevice(h->device) != cudaSuccess) return set_error(PDST_ECUDA, "cudaSetDevice failed");
  const Geom& g = h->g;
  const int k1 = h->td.k1;
  int err = PDST_OK;
  const double* Ud = stage_in(h, h->scratch_a, U, (size_t)k1 * g.nd, where, &err);
  if (err) return err;
  ErrTabs T{};
  T.q = spatial_points;
  T.ntp = temporal_points;
  T.k1 = k1;
  gauss01(T.q, T.s, T.w);
  gauss01(T.ntp, T.tg, T.tw);
  for (int i = 0; i < T.q; ++i) {
    const double x = T.s[i];
    T.L[i][0] = (1.0 - x) * (1.0 - 2.0 * x);
    T.L[i][1] = 4.0 * x * (1.0 - x);
    T.L[i][2] = x * (2.0 * x - 1.0);
    T.dL[i][0] = 4.0 * x - 3.0;
    T.dL[i][1] = 4.0 - 8.0 * x;
    T.dL[i][2] = 4.0 * x - 1.0;
  }
  for (int ig = 0; ig < T.ntp; ++ig) {
    const std::vector<double> l = cardinals_at(h->nodes, T.tg[ig]);
    for (int mu = 0; mu < k1; ++mu) T.blend[ig][mu] = l[mu];
  }
  const int blocks = (g.ncells + EB - 1) / EB;
  double* part = h->partials.ensure((size_t)2 * blocks);
  if (!part) return set_error(PDST_ECUDA, "out of device memory");
  PDST_LAUNCH(k_error_norms<<<blocks, EB, 0, h->stream>>>(g, h->model, T, h->extents[0], h->extents[1], t0, t1 - t0,
                                                          Ud, part));
  if (cudaGetLastError() != cudaSuccess) return set_error(PDST_ECUDA, "k_error_norms launch failed");
  std::vector<double> hp((size_t)2 * blocks);
  if (cudaMemcpyAsync(hp.data(), part, hp.size() * sizeof(double), cudaMemcpyDeviceToHost, h->stream) != cudaSuccess ||
      cudaStreamSynchronize(h->stream) != cudaSuccess)
    return set_error(PDST_ECUDA, "error-norm readback failed");
  double sp = 0.0, sd = 0.0;
  for (int b = 0; b < blocks; ++b) {
    sp += hp[2 * b];
    sd += hp[2 * b + 1];
  }
  sq2[0] = sp;
  sq2[1] = sd;
  return PDST_OK;
}

}  // extern "C"
