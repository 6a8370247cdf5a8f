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
// On the uniform rectangles of this mesh the volume part of G is ONE 4 x 18
// cell matrix, separable into 1-D Gauss sums (ThTabs), so no quadrature loop
// and no per-cell buffer: k_th_gather gives every velocity node and pressure
// vertex the products of its <= 4 cells directly from x, in a fixed (row,
// column) order.  Only cells with a Dirichlet side carry more — the boundary
// terms, evaluated per boundary cell by k_th_sides into a small buffer that
// the gather adds.  Pressure vertices are row-major (y, x), (nx+1)(ny+1) per
// Radau node after the velocity block.
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

// 1-D Gauss sums of the Q1 x Q2 coupling on the reference interval:
//   D[j][i] = sum_q w_q psi_j(s_q) L_i'(s_q),  M[j][i] = sum_q w_q psi_j(s_q) L_i(s_q),
// psi_0 = 1 - s, psi_1 = s.  The cell matrix of -(psi_J, d_d phi_a):
//   d = 0: -hy D[jx][ix] M[jy][iy],   d = 1: -hx M[jx][ix] D[jy][iy]   (area / h_d).
struct ThTabs {
  double G[4][9][2];  // the cell matrix itself, mesh scales folded in (kernel parameter: constant-bank operands)
};
__device__ __forceinline__ double th_g(const ThTabs& T, const Geom&, int J, int a, int d) { return T.G[J][a][d]; }

// Boundary cells: bottom row, top row, then the left / right cells of the rows
// between (every cell when the mesh is one cell wide or tall).
__host__ __device__ inline size_t th_nbcells(const Geom& g) {
  return g.nx == 1 || g.ny == 1 ? (size_t)g.ncells : (size_t)2 * g.nx + 2 * (g.ny - 2);
}
__device__ inline void th_bcell_of(const Geom& g, size_t t, int& ci, int& cj) {
  if (g.nx == 1 || g.ny == 1) {
    ci = (int)(t % g.nx), cj = (int)(t / g.nx);
  } else if (t < (size_t)g.nx) {
    ci = (int)t, cj = 0;
  } else if (t < (size_t)2 * g.nx) {
    ci = (int)(t - g.nx), cj = g.ny - 1;
  } else {
    const size_t u = t - 2 * (size_t)g.nx;
    cj = 1 + (int)(u / 2), ci = (u & 1) ? g.nx - 1 : 0;
  }
}
__device__ inline int th_bcell_index(const Geom& g, int ci, int cj) {
  if (g.nx == 1 || g.ny == 1) return cj * g.nx + ci;
  if (cj == 0) return ci;
  if (cj == g.ny - 1) return g.nx + ci;
  if (ci == 0) return 2 * g.nx + 2 * (cj - 1);
  if (ci == g.nx - 1) return 2 * g.nx + 2 * (cj - 1) + 1;
  return -1;
}

// Dirichlet-side terms of boundary cell cb: +<p, phi_a . n> and
// +<(u - g_hat) . n, psi_j>, 4 Gauss points per side.
// sb[(mu * THN + i) * ncb + cb]: i < 18 the velocity row 2a + d, i >= 18 the vertex row 2 jy + jx.
__global__ void k_th_sides(Geom g, int k1, const double* __restrict__ x, const double* __restrict__ ghat,
                           double* __restrict__ sb) {
  // PDL-launched behind the velocity apply without a dependency wait: it reads only x (complete since
  // the apply's tile pass passed its own wait) and writes sb, which the previous gather has released
  pdl_trigger();
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int mu = blockIdx.y;
  const size_t ncb = th_nbcells(g);
  if (t >= ncb) {
    pdl_wait();
    return;
  }
  int ci, cj;
  th_bcell_of(g, t, ci, cj);
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
  double* o = sb + (size_t)mu * THN * ncb + t;
#pragma unroll
  for (int a = 0; a < 9; ++a) {
    o[(2 * a) * ncb] = vo[a][0];
    o[(2 * a + 1) * ncb] = vo[a][1];
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) o[(18 + j) * ncb] = po[j];
  // this grid completes only after its predecessor (the velocity apply's epilogue) has: the
  // gather waits for this grid alone and adds to the y that epilogue finishes
  pdl_wait();
}

// y_v += sgn tau w_mu sum_cells (G' x_p)_cell (velocity nodes), y_p = sgn tau
// w_mu sum_cells (G x_v)_cell (vertices; `on` = 0 writes zeros).  One thread
// per pressure vertex (ci, cj), 0 <= ci <= nx, 0 <= cj <= ny: it finishes the
// vertex and the <= 4 velocity nodes (2 ci + {0,1}, 2 cj + {0,1}) from the
// cells (ci - 1 .. ci, cj - 1 .. cj) around it, so every local index below is
// a compile-time constant; each cell's volume part comes from the separable
// cell matrix and, for boundary cells, its side terms from sb; cells in (row,
// column) order.
constexpr int TG_BW = 32, TG_BH = 4;                             // vertices per CTA (x, y)
constexpr int TG_NC = 2 * TG_BW + 3, TG_NR = 2 * TG_BH + 3;      // staged velocity nodes: the block's cells' nodes
__global__ void __launch_bounds__(TG_BW * TG_BH) k_th_gather(Geom g, TimeData td, ThTabs T,
                                                             const double* __restrict__ x,
                                                             const double* __restrict__ sb, double sgn, int on,
                                                             double* __restrict__ y) {
  pdl_trigger();
  __shared__ __align__(16) double us[TG_NR][2 * TG_NC + 2];  // x's velocity nodes (2 ci0 - 2 .., 2 cj0 - 2 ..), components interleaved
  const int nbx = (g.nx + 1 + TG_BW - 1) / TG_BW;
  const int bx = blockIdx.x % nbx, by = blockIdx.x / nbx;
  const int mu = blockIdx.y;
  const int lx = threadIdx.x % TG_BW, ly = threadIdx.x / TG_BW;
  const int ci = bx * TG_BW + lx, cj = by * TG_BH + ly;
  const size_t ncb = th_nbcells(g);
  const double sc = on ? sgn * td.tau_w[mu] : 0.0;
  const double* xm = x + (size_t)mu * g.nd;
  const double* sm = sb + (size_t)mu * THN * ncb;
  double* ym = y + (size_t)mu * g.nd;
  {  // coalesced staging of the node patch (zero outside the mesh); x does not depend on the predecessors
    const int X0 = 2 * bx * TG_BW - 2, Y0 = 2 * by * TG_BH - 2;
    for (int idx = threadIdx.x; idx < TG_NR * 2 * TG_NC; idx += TG_BW * TG_BH) {
      const int r = idx / (2 * TG_NC), c2 = idx - r * (2 * TG_NC);
      const int X = X0 + (c2 >> 1), Y = Y0 + r;
      us[r][c2] = (X >= 0 && X < g.nnx && Y >= 0 && Y < g.nny) ? __ldg(xm + 2 * ((size_t)Y * g.nnx + X) + (c2 & 1)) : 0.0;
    }
  }
  __syncthreads();
  pdl_wait();  // the side terms and, through them, the velocity apply that y already holds
  if (ci > g.nx || cj > g.ny) return;
  const size_t t = (size_t)cj * (g.nx + 1) + ci;
  // the four cells around the vertex: k = 2 dy + dx -> cell (ci - 1 + dx, cj - 1 + dy)
  bool has[4];
  int cbi[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int cx = ci - 1 + (k & 1), cy = cj - 1 + (k >> 1);
    has[k] = cx >= 0 && cx < g.nx && cy >= 0 && cy < g.ny;
    cbi[k] = has[k] ? th_bcell_index(g, cx, cy) : -1;
  }
  double pv = 0.0;  // the vertex row, cells in (row, column) order
  if (on) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (!has[k]) continue;
      const int J = 3 - k;  // the vertex's index in that cell: 2 (cj - cy) + (ci - cx)
      // the cell's node (0, 0) in the staged patch: row 2 ly + 2 dy, column 2 lx + 2 dx
      const int r0 = 2 * ly + 2 * (k >> 1), c0 = 2 * lx + 2 * (k & 1);
      double c = 0.0;
#pragma unroll
      for (int a = 0; a < 9; ++a) {
        const double2 uu = *reinterpret_cast<const double2*>(&us[r0 + a / 3][2 * (c0 + a % 3)]);
        c = fma(th_g(T, g, J, a, 0), uu.x, c);
        c = fma(th_g(T, g, J, a, 1), uu.y, c);
      }
      if (cbi[k] >= 0) c += sm[(size_t)(18 + J) * ncb + cbi[k]];
      pv += c;
    }
  }
  ym[g.mv + t] = sc * pv;
  if (!on) return;
  // pressures of the 3 x 3 vertices around (ci, cj) (0 outside the mesh; never used there)
  double p[3][3];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int vi = ci - 1 + c, vj = cj - 1 + r;
      p[r][c] = (vi >= 0 && vi <= g.nx && vj >= 0 && vj <= g.ny) ? __ldg(xm + g.mv + (size_t)vj * (g.nx + 1) + vi) : 0.0;
    }
  // velocity node (2 ci + ex, 2 cj + ey): the cells containing it among the four, with its local index there
  auto node = [&](int ex, int ey) {
    if ((ex && ci == g.nx) || (ey && cj == g.ny)) return;  // beyond the mesh's last node column / row
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int dx = k & 1, dy = k >> 1;
      if ((ex && !dx) || (ey && !dy)) continue;  // an odd node lies inside the right / upper cells only
      if (!has[k]) continue;
      // local node index in cell k: x position 2 - 2 dx + ex, y position 2 - 2 dy + ey
      const int a = 3 * (2 - 2 * dy + ey) + (2 - 2 * dx + ex);
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int J = 0; J < 4; ++J) {
        const double pj = p[dy + (J >> 1)][dx + (J & 1)];  // vertex (cx + jx, cy + jy)
        c0 = fma(th_g(T, g, J, a, 0), pj, c0);
        c1 = fma(th_g(T, g, J, a, 1), pj, c1);
      }
      if (cbi[k] >= 0) {
        c0 += sm[(size_t)(2 * a) * ncb + cbi[k]];
        c1 += sm[(size_t)(2 * a + 1) * ncb + cbi[k]];
      }
      s0 += c0;
      s1 += c1;
    }
    double* yo = ym + 2 * ((size_t)(2 * cj + ey) * g.nnx + 2 * ci + ex);
    yo[0] += sc * s0;
    yo[1] += sc * s1;
  };
  node(0, 0);
  node(1, 0);
  node(0, 1);
  node(1, 1);
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

static ThTabs th_tabs(const Geom& g) {
  // 4-point Gauss sums, the points / weights / Q2 values of the device tables
  static const Tables tab = host_tables();
  double D[2][3], M[2][3];
  for (int j = 0; j < 2; ++j)
    for (int i = 0; i < 3; ++i) {
      double d = 0.0, m = 0.0;
      for (int q = 0; q < 4; ++q) {
        const double psi = j ? tab.s[q] : 1.0 - tab.s[q];
        d += tab.w[q] * psi * tab.G[q][i];
        m += tab.w[q] * psi * tab.B[q][i];
      }
      D[j][i] = d;
      M[j][i] = m;
    }
  ThTabs T;
  for (int J = 0; J < 4; ++J)
    for (int a = 0; a < 9; ++a) {
      const int jx = J & 1, jy = J >> 1, ix = a % 3, iy = a / 3;
      T.G[J][a][0] = -g.hy * (D[jx][ix] * M[jy][iy]);
      T.G[J][a][1] = -g.hx * (M[jx][ix] * D[jy][iy]);
    }
  return T;
}

static cudaError_t th_coupling(const Geom& g, const TimeData& td, bool on, const double* x, const double* ghat,
                               double sgn, double* y, double* sb, cudaStream_t st) {
  const ThTabs T = th_tabs(g);
  const size_t ncb = th_nbcells(g);
  cudaError_t e = cudaSuccess;
  if (on)
    PDST_LAUNCH(e = launch_pdl(k_th_sides, dim3((unsigned)((ncb + 127) / 128), td.k1), dim3(128), 0, st, g, td.k1, x,
                               ghat, sb));
  if (e != cudaSuccess) return e;
  const unsigned nblk = (unsigned)(((g.nx + 1 + TG_BW - 1) / TG_BW) * ((g.ny + 1 + TG_BH - 1) / TG_BH));
  PDST_LAUNCH(e = launch_pdl(k_th_gather, dim3(nblk, td.k1), dim3(TG_BW * TG_BH), 0, st, g, td, T, x,
                             (const double*)sb, sgn, on ? 1 : 0, y));
  return e;
}

// J: y (velocity rows already J_vel x) += [tau w G' x_p ; tau w G x_v]
cudaError_t th_apply(const Geom& g, const TimeData& td, bool on, const double* x, double* y, double* cb,
                     cudaStream_t st) {
  return th_coupling(g, td, on, x, nullptr, 1.0, y, cb, st);
}

// R: R_v -= tau w G' pi, R_p = tau w (N(g_hat) - G v)
cudaError_t th_residual(const Geom& g, const TimeData& td, bool on, const double* U, const double* ghat, double* R,
                        double* cb, cudaStream_t st) {
  return th_coupling(g, td, on, U, ghat, -1.0, R, cb, st);
}

cudaError_t th_pressure_mass(const Geom& g, const TimeData& td, const double* x, double* y, cudaStream_t st) {
  const size_t nv = (size_t)(g.nx + 1) * (g.ny + 1);
  PDST_LAUNCH(k_th_pmass<<<dim3((unsigned)((nv + 255) / 256), td.k1), 256, 0, st>>>(g, td, x, y));
  return cudaGetLastError();
}

size_t th_scratch(const Geom& g, int k1) { return (size_t)k1 * THN * th_nbcells(g); }  // boundary cells' side terms

}  // namespace pdst
