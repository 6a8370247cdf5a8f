// pdst_th.cu — Taylor-Hood Q2/Q1 pressure coupling (BASELINE north_star (1),
// SURVEY.md §9.1; the reference implements only Q2/P1disc, femspace.py:1-12).
//
// Every pressure term of the reference's Jacobian and residual is the
// bilinear form b(w, q) = -(q, div w) + <q, w.n>_{Gamma_D} (forms.py:589-603,
// 615-635, 467-471, 500-503; Nitsche vector 408-409).  A Taylor-Hood handle
// runs the velocity-velocity kernels with their pressure terms off and adds
//   J:  y_v += tau w_mu G' x_p,   y_p  = tau w_mu G x_v,
//   R:  R_v -= tau w_mu G' pi,    R_p  = tau w_mu (N(g_hat) - G v),
// with G the Q1-vertex x Q2-velocity operator of b (oracle/th_oracle.py).
// Two deterministic kernels: k_th_cell evaluates each cell's 18 + 4
// contributions (4x4 Gauss volume points, 4 points per Dirichlet side) into a
// structure-of-arrays buffer, k_th_gather sums the <= 4 cells of every
// velocity node and pressure vertex in a fixed order.  Pressure vertices are
// row-major (y, x), (nx+1)(ny+1) per Radau node after the velocity block.
#include <cuda_runtime.h>

#include "../../include/pdst.h"
#include "pdst_device.cuh"
#include "pdst_handle.h"

namespace pdst {
namespace {

constexpr int THN = 22;  // 18 velocity + 4 vertex-pressure contributions per cell

__device__ __forceinline__ double q1v(int j, double s) { return j ? s : 1.0 - s; }

// side s: bottom (y = 0), right (x = 1), top (y = 1), left (x = 0)
__device__ __forceinline__ bool side_on(const Geom& g, int side, int ci, int cj, int& bf) {
  bf = side_offset(g, side) + ((side == 0 || side == 2) ? ci : cj);
  const bool on = side == 0 ? cj == 0 : side == 1 ? ci == g.nx - 1 : side == 2 ? cj == g.ny - 1 : ci == 0;
  return on && g.dirichlet[bf] == 1;
}

// cb[(mu * THN + i) * nc + c]: i < 18 the velocity row 2a + d of (G' p)_cell,
// i >= 18 the vertex row 2 jy + jx of (G u)_cell - N(g_hat)_cell.
__global__ void k_th_cell(Geom g, int k1, const double* __restrict__ x, const double* __restrict__ ghat,
                          double* __restrict__ cb) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int mu = blockIdx.y;
  if (t >= (size_t)g.ncells) return;
  const int c = (int)t, ci = c % g.nx, cj = c / g.nx;
  const double* xm = x + (size_t)mu * g.nd;
  double u[9][2], p[4];
#pragma unroll
  for (int a = 0; a < 9; ++a) {
    const size_t o = 2 * ((size_t)(2 * cj + a / 3) * g.nnx + 2 * ci + a % 3);
    u[a][0] = xm[o];
    u[a][1] = xm[o + 1];
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) p[j] = xm[g.mv + (size_t)(cj + (j >> 1)) * (g.nx + 1) + ci + (j & 1)];
  double vo[9][2], po[4];
#pragma unroll
  for (int a = 0; a < 9; ++a) vo[a][0] = vo[a][1] = 0.0;
#pragma unroll
  for (int j = 0; j < 4; ++j) po[j] = 0.0;
  const double area = g.hx * g.hy;
  // ---- volume: -(p, div phi_a) and -(div u, psi_j) ----
#pragma unroll
  for (int qx = 0; qx < 4; ++qx) {
#pragma unroll
    for (int qy = 0; qy < 4; ++qy) {
      const double sx = c_tab.s[qx], sy = c_tab.s[qy];
      const double w = c_tab.w[qx] * c_tab.w[qy] * area;
      double pq = 0.0;
#pragma unroll
      for (int j = 0; j < 4; ++j) pq = fma(q1v(j & 1, sx) * q1v(j >> 1, sy), p[j], pq);
      double div = 0.0;
#pragma unroll
      for (int a = 0; a < 9; ++a) {
        const int ix = a % 3, iy = a / 3;
        const double dx = c_tab.G[qx][ix] * c_tab.B[qy][iy] * g.ihx, dy = c_tab.B[qx][ix] * c_tab.G[qy][iy] * g.ihy;
        div = fma(dx, u[a][0], fma(dy, u[a][1], div));
        vo[a][0] = fma(-w * pq, dx, vo[a][0]);
        vo[a][1] = fma(-w * pq, dy, vo[a][1]);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) po[j] = fma(-w * div, q1v(j & 1, sx) * q1v(j >> 1, sy), po[j]);
    }
  }
  // ---- Dirichlet sides: +<p, phi_a . n> and +<(u - g_hat) . n, psi_j> ----
  for (int side = 0; side < 4; ++side) {
    int bf;
    if (!side_on(g, side, ci, cj, bf)) continue;
    const double n0 = side == 1 ? 1.0 : side == 3 ? -1.0 : 0.0, n1 = side == 2 ? 1.0 : side == 0 ? -1.0 : 0.0;
    const double h = (side == 0 || side == 2) ? g.hx : g.hy;
    for (int q = 0; q < 4; ++q) {
      const double s = c_tab.s[q];
      // reference coordinates of the face point
      const double xh = side == 1 ? 1.0 : side == 3 ? 0.0 : s, yh = side == 2 ? 1.0 : side == 0 ? 0.0 : s;
      double phi[9];
#pragma unroll
      for (int a = 0; a < 9; ++a) {
        const int ix = a % 3, iy = a / 3;
        const double lx = side == 1 ? c_tab.E[1][ix] : side == 3 ? c_tab.E[0][ix] : c_tab.B[q][ix];
        const double ly = side == 2 ? c_tab.E[1][iy] : side == 0 ? c_tab.E[0][iy] : c_tab.B[q][iy];
        phi[a] = lx * ly;
      }
      const double wf = c_tab.w[q] * h;
      double pq = 0.0, un = 0.0, gn = 0.0;
#pragma unroll
      for (int j = 0; j < 4; ++j) pq = fma(q1v(j & 1, xh) * q1v(j >> 1, yh), p[j], pq);
#pragma unroll
      for (int a = 0; a < 9; ++a) {
        un = fma(phi[a], u[a][0] * n0 + u[a][1] * n1, un);
        if (ghat) {
          const size_t o = 2 * ((size_t)(2 * cj + a / 3) * g.nnx + 2 * ci + a % 3);
          gn = fma(phi[a], ghat[o] * n0 + ghat[o + 1] * n1, gn);
        }
        vo[a][0] = fma(wf * pq * n0, phi[a], vo[a][0]);
        vo[a][1] = fma(wf * pq * n1, phi[a], vo[a][1]);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) po[j] = fma(wf * (un - gn), q1v(j & 1, xh) * q1v(j >> 1, yh), po[j]);
    }
  }
  const size_t nc = g.ncells;
  double* o = cb + (size_t)mu * THN * nc + c;
#pragma unroll
  for (int a = 0; a < 9; ++a) {
    o[(2 * a) * nc] = vo[a][0];
    o[(2 * a + 1) * nc] = vo[a][1];
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) o[(18 + j) * nc] = po[j];
}

// y_v += sgn tau w_mu sum_cells cb_v (velocity nodes), y_p = sgn tau w_mu
// sum_cells cb_p (vertices; scale 0 writes zeros), cells in (row, column)
// order.
__global__ void k_th_gather(Geom g, TimeData td, const double* __restrict__ cb, double sgn, int on,
                            double* __restrict__ y) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int mu = blockIdx.y;
  const size_t nn = (size_t)g.nnx * g.nny, nv = (size_t)(g.nx + 1) * (g.ny + 1), nc = g.ncells;
  const double sc = on ? sgn * td.tau_w[mu] : 0.0;
  const double* cm = cb + (size_t)mu * THN * nc;
  double* ym = y + (size_t)mu * g.nd;
  if (t < nn) {
    if (!on) return;
    const int X = (int)(t % g.nnx), Y = (int)(t / g.nnx);
    double s0 = 0.0, s1 = 0.0;
    for (int cy = max(0, (Y - 1) / 2); cy <= min(g.ny - 1, Y / 2); ++cy)
      for (int cx = max(0, (X - 1) / 2); cx <= min(g.nx - 1, X / 2); ++cx) {
        const int a = 3 * (Y - 2 * cy) + (X - 2 * cx);
        const size_t c = (size_t)cy * g.nx + cx;
        s0 += cm[(2 * a) * nc + c];
        s1 += cm[(2 * a + 1) * nc + c];
      }
    ym[2 * t] += sc * s0;
    ym[2 * t + 1] += sc * s1;
  } else if (t < nn + nv) {
    const size_t v = t - nn;
    const int i = (int)(v % (g.nx + 1)), j = (int)(v / (g.nx + 1));
    double s = 0.0;
    for (int cy = max(0, j - 1); cy <= min(g.ny - 1, j); ++cy)
      for (int cx = max(0, i - 1); cx <= min(g.nx - 1, i); ++cx)
        s += cm[(18 + 2 * (j - cy) + (i - cx)) * nc + (size_t)cy * g.nx + cx];
    ym[g.mv + v] = sc * s;
  }
}

// y_p = tau w_mu M_p x_p, consistent Q1 mass hx hy M1_y (x) M1_x,
// M1 = [[1/3, 1/6], [1/6, 1/3]] assembled on the vertex lines.
__device__ __forceinline__ double q1line(int i, int ip, int n) {
  if (i == ip) return ((i > 0) + (i < n)) * (1.0 / 3.0);
  return (ip == i - 1 || ip == i + 1) ? 1.0 / 6.0 : 0.0;
}
__global__ void k_th_pmass(Geom g, TimeData td, const double* __restrict__ x, double* __restrict__ y) {
  const size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int mu = blockIdx.y;
  const size_t nv = (size_t)(g.nx + 1) * (g.ny + 1);
  if (v >= nv) return;
  const int i = (int)(v % (g.nx + 1)), j = (int)(v / (g.nx + 1));
  const double* xm = x + (size_t)mu * g.nd + g.mv;
  double s = 0.0;
  for (int jp = max(0, j - 1); jp <= min(g.ny, j + 1); ++jp) {
    double r = 0.0;
    for (int ip = max(0, i - 1); ip <= min(g.nx, i + 1); ++ip) r = fma(q1line(i, ip, g.nx), xm[(size_t)jp * (g.nx + 1) + ip], r);
    s = fma(q1line(j, jp, g.ny), r, s);
  }
  y[(size_t)mu * g.nd + g.mv + v] = td.tau_w[mu] * (g.hx * g.hy * s);
}

}  // namespace

// J: y (velocity rows already J_vel x) += [tau w G' x_p ; tau w G x_v]
cudaError_t th_apply(const Geom& g, const TimeData& td, bool on, const double* x, double* y, double* cb,
                     cudaStream_t st) {
  dim3 gc((unsigned)((g.ncells + 127) / 128), td.k1);
  if (on) PDST_LAUNCH(k_th_cell<<<gc, 128, 0, st>>>(g, td.k1, x, nullptr, cb));
  const size_t n = (size_t)g.nnx * g.nny + (size_t)(g.nx + 1) * (g.ny + 1);
  PDST_LAUNCH(k_th_gather<<<dim3((unsigned)((n + 255) / 256), td.k1), 256, 0, st>>>(g, td, cb, 1.0, on ? 1 : 0, y));
  return cudaGetLastError();
}

// R: R_v -= tau w G' pi, R_p = tau w (N(g_hat) - G v)
cudaError_t th_residual(const Geom& g, const TimeData& td, bool on, const double* U, const double* ghat, double* R,
                        double* cb, cudaStream_t st) {
  dim3 gc((unsigned)((g.ncells + 127) / 128), td.k1);
  if (on) PDST_LAUNCH(k_th_cell<<<gc, 128, 0, st>>>(g, td.k1, U, ghat, cb));
  const size_t n = (size_t)g.nnx * g.nny + (size_t)(g.nx + 1) * (g.ny + 1);
  PDST_LAUNCH(k_th_gather<<<dim3((unsigned)((n + 255) / 256), td.k1), 256, 0, st>>>(g, td, cb, -1.0, on ? 1 : 0, R));
  return cudaGetLastError();
}

cudaError_t th_pressure_mass(const Geom& g, const TimeData& td, const double* x, double* y, cudaStream_t st) {
  const size_t nv = (size_t)(g.nx + 1) * (g.ny + 1);
  PDST_LAUNCH(k_th_pmass<<<dim3((unsigned)((nv + 255) / 256), td.k1), 256, 0, st>>>(g, td, x, y));
  return cudaGetLastError();
}

size_t th_scratch(const Geom& g, int k1) { return (size_t)k1 * THN * g.ncells; }

}  // namespace pdst
