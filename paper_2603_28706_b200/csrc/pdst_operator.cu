// pdst_operator.cu — linearization, matrix-free slab Jacobian apply and slab
// residual kernels (sm_100a, fp64).
//
// Kernel design:
//   * Jacobian apply (k_apply_cache once per linearization; k_jacobian +
//     k_jac_post per apply): the per-quadrature-point coefficients are a
//     tile-major stream (the reference's linearization cache); one CTA per
//     16 x 16-cell tile, one thread per cell, the direction's Radau planes
//     staged in shared memory with a one-cell ring, volume by sum
//     factorisation, CIP through cached face matrices, temporal mass, fixed-
//     order node assembly; tile-line nodes and the boundary-face side terms
//     are finished by the PDL-launched epilogue;
//   * residual (k_residual): tiles of TX x TY owned cells plus a halo ring of
//     one cell to the left and below (owner computes), the state staged with a
//     two-cell ring, nonlinear stress evaluated per point;
//   * element / boundary-side matrices by probing the cell-local action with
//     unit vectors (the assembled and matrix-free paths agree to rounding).
//
// Reference: forms.py:581-652 (J x), forms.py:435-516 (residual),
// slab.py:162-205 (slab composition), constitutive.py:323-337 (tangent).
#include <cstdlib>

#include "pdst_device.cuh"
#include "pdst_internal.h"

#ifdef PDST_TRACE
__device__ unsigned long long g_steptrace[32];  // step timeline (pdst_device.cuh STEP_MARK)
#endif

namespace pdst {

__constant__ Tables c_tab;

namespace {

constexpr int TX = 15;           // owned cells per tile, x
constexpr int TY = 15;           // owned cells per tile, y
constexpr int CX = TX + 1;       // computed cells (with left halo)
constexpr int CY = TY + 1;
constexpr int NT = CX * CY;      // threads per CTA
constexpr int NC = 2 * (TX + 3) + 1;  // staged node columns
constexpr int NR = 2 * (TY + 3) + 1;  // staged node rows
constexpr int NC2 = (NC + 1) / 2;     // columns per parity half-row
constexpr int RS = 2 * NC2;           // staged row stride
constexpr int PLANE = NR * RS;

// Staged node plane: each row holds the even node columns then the odd ones,
// so threads of consecutive cells (node columns 2tx+{0,1,2}) read
// consecutive doubles (conflict-free 64-bit shared loads).
__host__ __device__ constexpr int pidx(int r, int c) { return r * RS + (c & 1) * NC2 + (c >> 1); }

struct Plane2 {
  const double* p0;  // component 0
  const double* p1;  // component 1
  __device__ double at(int d, int r, int c) const { return (d == 0 ? p0 : p1)[pidx(r, c)]; }
};

// A staged plane pair addressed by its offset in the kernel's dynamic shared
// memory: the accesses stay LDS (a pointer array can be demoted to local
// memory and turn them into generic loads).
extern __shared__ __align__(16) double g_dsmem[];

// Accumulators for the cell's 9-node velocity contributions: registers (the
// element-matrix kernel, the volume phase) or the thread's shared-memory slot
// (structure of arrays over the CTA's threads, stride NT).
struct RegAcc {
  double (*a)[3][2];
  __device__ __forceinline__ void add(int jy, int ix, int d, double v) const { a[jy][ix][d] += v; }
};
struct SmemAcc {
  double* p;
  __device__ __forceinline__ void add(int jy, int ix, int d, double v) const { p[(2 * (3 * jy + ix) + d) * NT] += v; }
};
template <int STRIDE>
struct SmemAccN {
  double* p;
  __device__ __forceinline__ void add(int jy, int ix, int d, double v) const {
    p[(2 * (3 * jy + ix) + d) * STRIDE] += v;
  }
};

// Asynchronous 8-byte global->shared copy (LDGSTS); size 0 zero-fills.
__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  const int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(src), "r"(sz) : "memory");
}
// 16-byte variant (both components of a node); source and destination 16-byte aligned.
__device__ __forceinline__ void cp_async16(void* dst, const double* src, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(src), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }
// Streaming 8-byte load of read-once data (the apply's coefficient cache): not
// allocated in L1, which holds the staged-plane misses and the few spill slots.
__device__ __forceinline__ double ldg_stream(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];\n" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p)); }

// Stage one slab block's velocity into two shared planes (zero outside the domain).
__device__ void stage_velocity(const Geom& g, const double* __restrict__ v, double* pl0, double* pl1, int X0,
                               int Y0) {
  for (int idx = threadIdx.x; idx < NR * NC; idx += blockDim.x) {
    const int r = idx / NC, c = idx - r * NC;
    const int X = X0 + c, Y = Y0 + r;
    double a = 0.0, b = 0.0;
    if (X >= 0 && X < g.nnx && Y >= 0 && Y < g.nny) {
      const size_t o = 2 * ((size_t)Y * g.nnx + X);
      a = __ldg(v + o);
      b = __ldg(v + o + 1);
    }
    pl0[pidx(r, c)] = a;
    pl1[pidx(r, c)] = b;
  }
}

// line[t][d] = sum_n coef[n] F(node (n along axis-normal, t along tangent))
// for the 3x3 node block whose lower-left staged node is (r0, c0).
template <class FA>
__device__ __forceinline__ void line_sums(const FA& F, int r0, int c0, int axis, const double* coef,
                                          double line[3][2]) {
#pragma unroll
  for (int t = 0; t < 3; ++t) {
#pragma unroll
    for (int d = 0; d < 2; ++d) {
      double s = 0.0;
#pragma unroll
      for (int n = 0; n < 3; ++n) {
        const double f = axis == 0 ? F.at(d, r0 + t, c0 + n) : F.at(d, r0 + n, c0 + t);
        s = fma(coef[n], f, s);
      }
      line[t][d] = s;
    }
  }
}

__device__ __forceinline__ void side_info(int side, int& axis, int& e, double& n0, double& n1) {
  // 0 bottom, 1 right, 2 top, 3 left
  axis = (side == 1 || side == 3) ? 0 : 1;
  e = (side == 1 || side == 2) ? 1 : 0;
  n0 = side == 1 ? 1.0 : side == 3 ? -1.0 : 0.0;
  n1 = side == 2 ? 1.0 : side == 0 ? -1.0 : 0.0;
}

// Scatter face accumulators RE (value/tangential tests) and RD (normal
// derivative tests) to the cell's 9 nodes.
template <class ACC>
__device__ __forceinline__ void face_scatter(int axis, int e, const double RE[3][2], const double RD[3][2],
                                             const ACC& acc) {
#pragma unroll
  for (int n = 0; n < 3; ++n) {
    const double en = c_tab.E[e][n], dn = c_tab.dE[e][n];
#pragma unroll
    for (int t = 0; t < 3; ++t) {
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        const double v = en * RE[t][d] + dn * RD[t][d];
        if (axis == 0)
          acc.add(t, n, d, v);
        else
          acc.add(n, t, d, v);
      }
    }
  }
}

// CIP face term (forms.py:639-650 / 415-432), computed ONCE per interior face:
// RD[t][d] = gamma_cip h^2 / hn^2 * sum_q (w_q h) |a_L . n| jump_d(q) B[q][t]
// where jump = d_n u|_L - d_n u|_R (n = +x for axis 0, +y for axis 1) and the
// weight uses the lagged advective trace of the left/lower cell.  The left /
// lower cell adds +dE(1) (x) RD to its nodes, the right / upper cell
// -dE(0) (x) RD (cip_scatter).  (rL, cL) = staged origin of the left block.
template <class FA, class AA>
__device__ __forceinline__ void cip_face(const Geom& g, const Disc& ds, int axis, const FA& F, const AA& A, int rL,
                                         int cL, double RD[3][2], double scale = 1.0) {
  const int rR = axis == 1 ? rL + 2 : rL, cR = axis == 0 ? cL + 2 : cL;
  const double hface = axis == 0 ? g.hy : g.hx;
  const double ihn = axis == 0 ? g.ihx : g.ihy;
  double dl[3][2], dr[3][2];
  line_sums(F, rL, cL, axis, c_tab.dE[1], dl);
  line_sums(F, rR, cR, axis, c_tab.dE[0], dr);
  double tr[3];
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    double v = 0.0;
#pragma unroll
    for (int n = 0; n < 3; ++n)
      v = fma(c_tab.E[1][n], axis == 0 ? A.at(0, rL + t, cL + n) : A.at(1, rL + n, cL + t), v);
    tr[t] = v;
    dl[t][0] -= dr[t][0];
    dl[t][1] -= dr[t][1];
  }
  const double coef = scale * ds.gamma_cip * hface * hface * (ihn * ihn);
#pragma unroll
  for (int t = 0; t < 3; ++t) RD[t][0] = RD[t][1] = 0.0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    double vt = 0.0, j0 = 0.0, j1 = 0.0;
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      const double b = c_tab.B[q][t];
      vt = fma(b, tr[t], vt);
      j0 = fma(b, dl[t][0], j0);
      j1 = fma(b, dl[t][1], j1);
    }
    const double wgt = coef * (c_tab.w[q] * hface) * fabs(vt);
    const double c0v = wgt * j0, c1v = wgt * j1;
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      RD[t][0] = fma(c0v, c_tab.B[q][t], RD[t][0]);
      RD[t][1] = fma(c1v, c_tab.B[q][t], RD[t][1]);
    }
  }
}

// acc(n,t) += sgn * f(n) RD[t] with f = dE(1) for the left/lower cell, -dE(0) for the right/upper one.
template <class ACC>
__device__ __forceinline__ void cip_scatter(int axis, bool left, double sgn, const double RD[3][2], const ACC& acc) {
#pragma unroll
  for (int n = 0; n < 3; ++n) {
    const double f = sgn * (left ? c_tab.dE[1][n] : -c_tab.dE[0][n]);
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      if (axis == 0) {
        acc.add(t, n, 0, f * RD[t][0]);
        acc.add(t, n, 1, f * RD[t][1]);
      } else {
        acc.add(n, t, 0, f * RD[t][0]);
        acc.add(n, t, 1, f * RD[t][1]);
      }
    }
  }
}

// Own CIP faces of a computed cell: the right and upper faces (shared with the
// neighbour through fR/fT), plus the left / lower faces of the halo column /
// row whose left neighbour is outside the tile.
template <class FA, class AA, class ACC>
__device__ __forceinline__ void cip_own(const Geom& g, const Disc& ds, const FA& F, const AA& A, int ci, int cj,
                                        int tx, int ty, int r0, int c0, double sgn, double* fR, double* fT,
                                        const ACC& acc) {
  double RD[3][2];
  if (ci < g.nx - 1) {
    cip_face(g, ds, 0, F, A, r0, c0, RD);
    cip_scatter(0, true, sgn, RD, acc);
#pragma unroll
    for (int k = 0; k < 6; ++k) fR[k * NT + threadIdx.x] = RD[k / 2][k % 2];
  }
  if (cj < g.ny - 1) {
    cip_face(g, ds, 1, F, A, r0, c0, RD);
    cip_scatter(1, true, sgn, RD, acc);
#pragma unroll
    for (int k = 0; k < 6; ++k) fT[k * NT + threadIdx.x] = RD[k / 2][k % 2];
  }
  if (tx == 0 && ci > 0) {
    cip_face(g, ds, 0, F, A, r0, c0 - 2, RD);
    cip_scatter(0, false, sgn, RD, acc);
  }
  if (ty == 0 && cj > 0) {
    cip_face(g, ds, 1, F, A, r0 - 2, c0, RD);
    cip_scatter(1, false, sgn, RD, acc);
  }
}

// All four CIP faces of a cell, own side only (no exchange): the face jump is
// evaluated from the staged neighbour block.  `scale` multiplies the term.
template <class FA, class AA, class ACC>
__device__ __forceinline__ void cip_all(const Geom& g, const Disc& ds, const FA& F, const AA& A, int ci, int cj, int r0,
                                        int c0, double scale, const ACC& acc) {
  double RD[3][2];
  if (ci < g.nx - 1) {
    cip_face(g, ds, 0, F, A, r0, c0, RD, scale);
    cip_scatter(0, true, 1.0, RD, acc);
  }
  if (cj < g.ny - 1) {
    cip_face(g, ds, 1, F, A, r0, c0, RD, scale);
    cip_scatter(1, true, 1.0, RD, acc);
  }
  if (ci > 0) {
    cip_face(g, ds, 0, F, A, r0, c0 - 2, RD, scale);
    cip_scatter(0, false, 1.0, RD, acc);
  }
  if (cj > 0) {
    cip_face(g, ds, 1, F, A, r0 - 2, c0, RD, scale);
    cip_scatter(1, false, 1.0, RD, acc);
  }
}

// After a barrier: the left / lower faces computed by the neighbour thread.
template <class ACC>
__device__ __forceinline__ void cip_received(const Geom& g, int ci, int cj, int tx, int ty, double sgn,
                                             const double* fR, const double* fT, const ACC& acc) {
  double RD[3][2];
  if (tx >= 1 && ci > 0) {
#pragma unroll
    for (int k = 0; k < 6; ++k) RD[k / 2][k % 2] = fR[k * NT + threadIdx.x - 1];
    cip_scatter(0, false, sgn, RD, acc);
  }
  if (ty >= 1 && cj > 0) {
#pragma unroll
    for (int k = 0; k < 6; ++k) RD[k / 2][k % 2] = fT[k * NT + threadIdx.x - CX];
    cip_scatter(1, false, sgn, RD, acc);
  }
}

// Evaluate a staged field on a boundary side at face point q:
// value u[d], gradient ux[d], uy[d].
struct FaceLines {
  double E[3][2], D[3][2];
};

__device__ __forceinline__ void face_point(const FaceLines& L, int axis, int q, double ihtan, double ihnorm, double u[2],
                                           double ux[2], double uy[2]) {
#pragma unroll
  for (int d = 0; d < 2; ++d) {
    double v = 0, dt = 0, dn = 0;
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      v = fma(c_tab.B[q][t], L.E[t][d], v);
      dt = fma(c_tab.G[q][t], L.E[t][d], dt);
      dn = fma(c_tab.B[q][t], L.D[t][d], dn);
    }
    u[d] = v;
    if (axis == 0) {
      ux[d] = dn * ihnorm;
      uy[d] = dt * ihtan;
    } else {
      ux[d] = dt * ihtan;
      uy[d] = dn * ihnorm;
    }
  }
}

// Jacobian boundary-side terms of one cell side (forms.py:605-637).
template <class XA, class SA, class ACC>
__device__ __noinline__ void jac_boundary_side(const Geom& g, const Disc& ds, const Lin& L, int mu, int side, int bf,
                                  const XA& X, const SA& S, int r0, int c0, const double P[3],
                                  const ACC& acc, double accp[3], double tw) {
  int axis, e;
  double n0, n1;
  side_info(side, axis, e, n0, n1);
  const double htan = axis == 0 ? g.hy : g.hx;
  const double ihtan = axis == 0 ? g.ihy : g.ihx;
  const double ihnorm = axis == 0 ? g.ihx : g.ihy;
  const double pen1 = ds.gamma1 / htan, pen2 = ds.gamma2 / htan;
  if (g.dirichlet[bf] == kCutSide) return;  // partition cut: an interior face owned elsewhere
  FaceLines LU, LV;
  line_sums(X, r0, c0, axis, c_tab.E[e], LU.E);
  line_sums(X, r0, c0, axis, c_tab.dE[e], LU.D);
  line_sums(S, r0, c0, axis, c_tab.E[e], LV.E);
  line_sums(S, r0, c0, axis, c_tab.dE[e], LV.D);
  const bool dm = g.dirichlet[bf] == 1;
  double RE[3][2] = {{0, 0}, {0, 0}, {0, 0}}, RD[3][2] = {{0, 0}, {0, 0}, {0, 0}};
  for (int q = 0; q < 4; ++q) {
    const double wq = c_tab.w[q] * htan * tw;
    double u[2], ux[2], uy[2], v[2], vx[2], vy[2];
    face_point(LU, axis, q, ihtan, ihnorm, u, ux, uy);
    face_point(LV, axis, q, ihtan, ihnorm, v, vx, vy);
    const double vn = v[0] * n0 + v[1] * n1;
    const double un = u[0] * n0 + u[1] * n1;
    double Cv[2] = {0, 0}, Cgx[2] = {0, 0}, Cgy[2] = {0, 0};
    if (ds.convection) {
      Cv[0] += vn * u[0] + un * v[0];
      Cv[1] += vn * u[1] + un * v[1];
    }
    if (dm) {
      if (ds.viscous) {
        const double a0 = vx[0], a1 = vy[1], a2 = 0.5 * (vy[0] + vx[1]);
        const double b0 = ux[0], b1 = uy[1], b2 = 0.5 * (uy[0] + ux[1]);
        const size_t fi = ((size_t)mu * g.nbf + bf) * 4 + q;
        const double ef = L.etaf[fi];
        const double gf = L.has_gamma ? L.gamf[fi] : 0.0;
        const double ab = a0 * b0 + a1 * b1 + 2.0 * a2 * b2;
        const double t0 = ef * b0 + gf * ab * a0, t1 = ef * b1 + gf * ab * a1, t2 = ef * b2 + gf * ab * a2;
        Cv[0] -= t0 * n0 + t2 * n1;
        Cv[1] -= t2 * n0 + t1 * n1;
        const size_t li = (size_t)bf * 4 + q;
        const double ed = L.etad[li], bd = L.betad[li];
        const double g0 = L.dg[li * 3 + 0], g1 = L.dg[li * 3 + 1], g2 = L.dg[li * 3 + 2];
        const double dgn0 = g0 * n0 + g2 * n1, dgn1 = g2 * n0 + g1 * n1;
        const double dgnu = dgn0 * u[0] + dgn1 * u[1];
        Cgx[0] -= 0.5 * ed * (n0 * u[0] + u[0] * n0) + bd * dgnu * g0;
        Cgx[1] -= 0.5 * ed * (n0 * u[1] + u[0] * n1) + bd * dgnu * g2;
        Cgy[0] -= 0.5 * ed * (n1 * u[0] + u[1] * n0) + bd * dgnu * g2;
        Cgy[1] -= 0.5 * ed * (n1 * u[1] + u[1] * n1) + bd * dgnu * g1;
        const double p1 = pen1 * ed, p2 = pen2 * un;
        Cv[0] += p1 * u[0] + p2 * n0;
        Cv[1] += p1 * u[1] + p2 * n1;
      }
      if (ds.convection) {
        const double wneg = 0.5 * (fabs(vn) - vn);
        Cv[0] -= wneg * u[0];
        Cv[1] -= wneg * u[1];
      }
      if (ds.pressure) {
        const double xh = axis == 0 ? (double)e : c_tab.s[q];
        const double yh = axis == 0 ? c_tab.s[q] : (double)e;
        const double dp = P[0] + P[1] * (xh - 0.5) + P[2] * (yh - 0.5);
        Cv[0] += dp * n0;
        Cv[1] += dp * n1;
        accp[0] += wq * un;
        accp[1] += wq * un * (xh - 0.5);
        accp[2] += wq * un * (yh - 0.5);
      }
    }
    const double* Ct = axis == 0 ? Cgy : Cgx;
    const double* Cn = axis == 0 ? Cgx : Cgy;
#pragma unroll
    for (int t = 0; t < 3; ++t) {
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        RE[t][d] += wq * (Cv[d] * c_tab.B[q][t] + Ct[d] * (c_tab.G[q][t] * ihtan));
        RD[t][d] += wq * (Cn[d] * (c_tab.B[q][t] * ihnorm));
      }
    }
  }
  face_scatter(axis, e, RE, RD, acc);
}

// Residual boundary-side terms (forms.py:474-507) plus, when a lifting is
// present, the Nitsche vector B_gamma(g_hat, .) of forms.py:374-412.
template <class ACC>
__device__ __forceinline__ void res_boundary_side(const Geom& g, const Disc& ds, const Model& m, const Lin& L, int side, int bf,
                                  const Plane2& S, const Plane2& A, int r0, int c0, const double PI[3],
                                  const double* ghat_nodes /*9x2*/, bool has_ghat, const ACC& acc, double accp[3]) {
  int axis, e;
  double n0, n1;
  side_info(side, axis, e, n0, n1);
  const double htan = axis == 0 ? g.hy : g.hx;
  const double ihtan = axis == 0 ? g.ihy : g.ihx;
  const double ihnorm = axis == 0 ? g.ihx : g.ihy;
  const double pen1 = ds.gamma1 / htan, pen2 = ds.gamma2 / htan;
  if (g.dirichlet[bf] == kCutSide) return;  // partition cut
  FaceLines LV, LA;
  line_sums(S, r0, c0, axis, c_tab.E[e], LV.E);
  line_sums(S, r0, c0, axis, c_tab.dE[e], LV.D);
  line_sums(A, r0, c0, axis, c_tab.E[e], LA.E);
  line_sums(A, r0, c0, axis, c_tab.dE[e], LA.D);
  double GE[3][2] = {{0, 0}, {0, 0}, {0, 0}};
  if (has_ghat) {
#pragma unroll
    for (int t = 0; t < 3; ++t)
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        double s = 0.0;
#pragma unroll
        for (int n = 0; n < 3; ++n) {
          const int a = axis == 0 ? 3 * t + n : 3 * n + t;
          s = fma(c_tab.E[e][n], ghat_nodes[2 * a + d], s);
        }
        GE[t][d] = s;
      }
  }
  const bool dm = g.dirichlet[bf] == 1;
  double RE[3][2] = {{0, 0}, {0, 0}, {0, 0}}, RD[3][2] = {{0, 0}, {0, 0}, {0, 0}};
  for (int q = 0; q < 4; ++q) {
    const double wq = c_tab.w[q] * htan;
    double v[2], vx[2], vy[2], a[2], ax_[2], ay_[2];
    face_point(LV, axis, q, ihtan, ihnorm, v, vx, vy);
    face_point(LA, axis, q, ihtan, ihnorm, a, ax_, ay_);
    const double vn = v[0] * n0 + v[1] * n1;
    double Cv[2] = {0, 0}, Cgx[2] = {0, 0}, Cgy[2] = {0, 0};
    if (ds.convection) {
      Cv[0] -= vn * v[0];
      Cv[1] -= vn * v[1];
    }
    if (dm) {
      const size_t li = (size_t)bf * 4 + q;
      const double ed = L.etad[li], bd = L.betad[li];
      const double g0 = L.dg[li * 3 + 0], g1 = L.dg[li * 3 + 1], g2 = L.dg[li * 3 + 2];
      const double dgn0 = g0 * n0 + g2 * n1, dgn1 = g2 * n0 + g1 * n1;
      if (ds.viscous) {
        const double a0 = vx[0], a1 = vy[1], a2 = 0.5 * (vy[0] + vx[1]);
        const double ef = eta_field(m, a0 * a0 + a1 * a1 + 2.0 * a2 * a2);
        Cv[0] += ef * (a0 * n0 + a2 * n1);
        Cv[1] += ef * (a2 * n0 + a1 * n1);
        const double dgnv = dgn0 * v[0] + dgn1 * v[1];
        Cgx[0] += 0.5 * ed * (n0 * v[0] + v[0] * n0) + bd * dgnv * g0;
        Cgx[1] += 0.5 * ed * (n0 * v[1] + v[0] * n1) + bd * dgnv * g2;
        Cgy[0] += 0.5 * ed * (n1 * v[0] + v[1] * n0) + bd * dgnv * g2;
        Cgy[1] += 0.5 * ed * (n1 * v[1] + v[1] * n1) + bd * dgnv * g1;
        const double p1 = pen1 * ed, p2 = pen2 * vn;
        Cv[0] -= p1 * v[0] + p2 * n0;
        Cv[1] -= p1 * v[1] + p2 * n1;
      }
      const double xh = axis == 0 ? (double)e : c_tab.s[q];
      const double yh = axis == 0 ? c_tab.s[q] : (double)e;
      if (ds.convection) {
        const double an = a[0] * n0 + a[1] * n1;
        const double aneg = 0.5 * (fabs(an) - an);
        Cv[0] += aneg * v[0];
        Cv[1] += aneg * v[1];
      }
      if (ds.pressure) {
        const double pf = PI[0] + PI[1] * (xh - 0.5) + PI[2] * (yh - 0.5);
        Cv[0] -= pf * n0;
        Cv[1] -= pf * n1;
        accp[0] -= wq * vn;
        accp[1] -= wq * vn * (xh - 0.5);
        accp[2] -= wq * vn * (yh - 0.5);
      }
      if (has_ghat) {
        double gv[2];
#pragma unroll
        for (int d = 0; d < 2; ++d) {
          double s = 0.0;
#pragma unroll
          for (int t = 0; t < 3; ++t) s = fma(c_tab.B[q][t], GE[t][d], s);
          gv[d] = s;
        }
        const double gn = gv[0] * n0 + gv[1] * n1;
        if (ds.viscous) {
          const double dgng = dgn0 * gv[0] + dgn1 * gv[1];
          Cgx[0] -= 0.5 * ed * (n0 * gv[0] + gv[0] * n0) + bd * dgng * g0;
          Cgx[1] -= 0.5 * ed * (n0 * gv[1] + gv[0] * n1) + bd * dgng * g2;
          Cgy[0] -= 0.5 * ed * (n1 * gv[0] + gv[1] * n0) + bd * dgng * g2;
          Cgy[1] -= 0.5 * ed * (n1 * gv[1] + gv[1] * n1) + bd * dgng * g1;
          const double p1 = pen1 * ed, p2 = pen2 * gn;
          Cv[0] += p1 * gv[0] + p2 * n0;
          Cv[1] += p1 * gv[1] + p2 * n1;
        }
        if (ds.convection) {
          const double gneg = 0.5 * (fabs(gn) - gn);
          Cv[0] -= gneg * gv[0];
          Cv[1] -= gneg * gv[1];
        }
        if (ds.pressure) {
          accp[0] += wq * gn;
          accp[1] += wq * gn * (xh - 0.5);
          accp[2] += wq * gn * (yh - 0.5);
        }
      }
    }
    const double* Ct = axis == 0 ? Cgy : Cgx;
    const double* Cn = axis == 0 ? Cgx : Cgy;
#pragma unroll
    for (int t = 0; t < 3; ++t) {
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        RE[t][d] += wq * (Cv[d] * c_tab.B[q][t] + Ct[d] * (c_tab.G[q][t] * ihtan));
        RD[t][d] += wq * (Cn[d] * (c_tab.B[q][t] * ihnorm));
      }
    }
  }
  face_scatter(axis, e, RE, RD, acc);
}

// Stage-1 sums along x for one Q2 row jy at Gauss column qx.
template <class FA>
__device__ __forceinline__ void row_sums(const FA& F, int r, int c0, int qx, double sB[2], double sG[2]) {
#pragma unroll
  for (int d = 0; d < 2; ++d) {
    const double f0 = F.at(d, r, c0), f1 = F.at(d, r, c0 + 1), f2 = F.at(d, r, c0 + 2);
    sB[d] = c_tab.B[qx][0] * f0 + c_tab.B[qx][1] * f1 + c_tab.B[qx][2] * f2;
    sG[d] = c_tab.G[qx][0] * f0 + c_tab.G[qx][1] * f1 + c_tab.G[qx][2] * f2;
  }
}

// acc += s * (M1 (x) M1) XT for the cell, XT = sum_nu K_t[mu,nu] F_nu - mfac * Fm.
template <int K1, class ACC, class FA = Plane2>
__device__ __forceinline__ void add_mass(const FA* F, const FA* Fm, double mfac, const double* Krow, int r0,
                                         int c0, double s, const ACC& acc) {
#pragma unroll
  for (int jj = 0; jj < 3; ++jj) {  // source row jy'
    double T1[3][2];
    double xt[3][2];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        double v = 0.0;
#pragma unroll
        for (int nu = 0; nu < K1; ++nu) v = fma(Krow[nu], F[nu].at(d, r0 + jj, c0 + i), v);
        if (Fm) v -= mfac * Fm->at(d, r0 + jj, c0 + i);
        xt[i][d] = v;
      }
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int d = 0; d < 2; ++d)
        T1[i][d] = c_tab.M1[i][0] * xt[0][d] + c_tab.M1[i][1] * xt[1][d] + c_tab.M1[i][2] * xt[2][d];
#pragma unroll
    for (int jy = 0; jy < 3; ++jy) {
      const double m = s * c_tab.M1[jy][jj];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int d = 0; d < 2; ++d) acc.add(jy, i, d, m * T1[i][d]);
    }
  }
}

// Cell-local Jacobian action (volume + the cell's boundary sides), without the
// CIP faces, the temporal mass and the tau w_mu scaling.  XA / SA are field
// accessors (shared-memory planes in the apply, unit vectors / global memory
// in the element-matrix kernel).  forms.py:589-637.
template <class XA, class SA, class ACC>
__device__ __forceinline__ void jac_volume(const Geom& g, const Disc& ds, const Lin& L, int mu, int c,
                                           const XA& XM, const SA& SP, int r0, int c0, const double P[3],
                                           const ACC& acc, double accp[3], double tw = 1.0) {
  const double W = g.hx * g.hy * tw;
  // eta / gamma of the next Gauss column are loaded one column ahead
  const double* pe = L.eta + ((size_t)mu * g.ncells + c) * 16;
  const double* pg = L.gam + ((size_t)mu * g.ncells + c) * 16;
  const bool vis = ds.viscous, hg = L.has_gamma && ds.viscous;
  double en[4], gn[4];
#pragma unroll
  for (int qy = 0; qy < 4; ++qy) {
    en[qy] = vis ? __ldg(pe + qy) : 0.0;
    gn[qy] = hg ? __ldg(pg + qy) : 0.0;
  }
      // ---- volume (forms.py:589-603) ----
  double R[3][3][2];
#pragma unroll
  for (int jy = 0; jy < 3; ++jy)
#pragma unroll
    for (int ix = 0; ix < 3; ++ix) R[jy][ix][0] = R[jy][ix][1] = 0.0;
#pragma unroll 1
      for (int qx = 0; qx < 4; ++qx) {
        double ec[4], gc[4];
#pragma unroll
        for (int qy = 0; qy < 4; ++qy) {
          ec[qy] = en[qy];
          gc[qy] = gn[qy];
        }
        if (qx < 3) {
#pragma unroll
          for (int qy = 0; qy < 4; ++qy) {
            en[qy] = vis ? __ldg(pe + 4 * (qx + 1) + qy) : 0.0;
            gn[qy] = hg ? __ldg(pg + 4 * (qx + 1) + qy) : 0.0;
          }
        }
        double xB[3][2], xG[3][2], sB[3][2], sG[3][2];
#pragma unroll
        for (int jy = 0; jy < 3; ++jy) {
          row_sums(XM, r0 + jy, c0, qx, xB[jy], xG[jy]);
          row_sums(SP, r0 + jy, c0, qx, sB[jy], sG[jy]);
        }
        double Pa[3][2] = {{0, 0}, {0, 0}, {0, 0}}, Qa[3][2] = {{0, 0}, {0, 0}, {0, 0}};
        const double xh = c_tab.s[qx] - 0.5;
#pragma unroll
        for (int qy = 0; qy < 4; ++qy) {
          double u[2], ux[2], uy[2], v[2], vx[2], vy[2];
#pragma unroll
          for (int d = 0; d < 2; ++d) {
            u[d] = c_tab.B[qy][0] * xB[0][d] + c_tab.B[qy][1] * xB[1][d] + c_tab.B[qy][2] * xB[2][d];
            ux[d] = (c_tab.B[qy][0] * xG[0][d] + c_tab.B[qy][1] * xG[1][d] + c_tab.B[qy][2] * xG[2][d]) * g.ihx;
            uy[d] = (c_tab.G[qy][0] * xB[0][d] + c_tab.G[qy][1] * xB[1][d] + c_tab.G[qy][2] * xB[2][d]) * g.ihy;
            v[d] = c_tab.B[qy][0] * sB[0][d] + c_tab.B[qy][1] * sB[1][d] + c_tab.B[qy][2] * sB[2][d];
            vx[d] = (c_tab.B[qy][0] * sG[0][d] + c_tab.B[qy][1] * sG[1][d] + c_tab.B[qy][2] * sG[2][d]) * g.ihx;
            vy[d] = (c_tab.G[qy][0] * sB[0][d] + c_tab.G[qy][1] * sB[1][d] + c_tab.G[qy][2] * sB[2][d]) * g.ihy;
          }
          const int q = 4 * qx + qy;
          const double wq = c_tab.w[qx] * c_tab.w[qy] * W;
          double Fx0 = 0, Fx1 = 0, Fy0 = 0, Fy1 = 0;
          if (ds.viscous) {
            const double eta = ec[qy];
            const double gam = gc[qy];
            const double a0 = vx[0], a1 = vy[1], a2 = 0.5 * (vy[0] + vx[1]);
            const double b0 = ux[0], b1 = uy[1], b2 = 0.5 * (uy[0] + ux[1]);
            const double ab = a0 * b0 + a1 * b1 + 2.0 * a2 * b2;
            Fx0 = eta * b0 + gam * ab * a0;
            Fy1 = eta * b1 + gam * ab * a1;
            Fx1 = Fy0 = eta * b2 + gam * ab * a2;
          }
          if (ds.convection) {
            Fx0 -= u[0] * v[0] + v[0] * u[0];
            Fx1 -= u[1] * v[0] + v[1] * u[0];
            Fy0 -= u[0] * v[1] + v[0] * u[1];
            Fy1 -= u[1] * v[1] + v[1] * u[1];
          }
          if (ds.pressure) {
            const double yh = c_tab.s[qy] - 0.5;
            const double dp = P[0] + P[1] * xh + P[2] * yh;
            Fx0 -= dp;
            Fy1 -= dp;
            const double dv = wq * (ux[0] + uy[1]);
            accp[0] -= dv;
            accp[1] -= dv * xh;
            accp[2] -= dv * yh;
          }
#pragma unroll
          for (int jy = 0; jy < 3; ++jy) {
            Pa[jy][0] = fma(wq * Fx0, c_tab.B[qy][jy], Pa[jy][0]);
            Pa[jy][1] = fma(wq * Fx1, c_tab.B[qy][jy], Pa[jy][1]);
            Qa[jy][0] = fma(wq * Fy0, c_tab.G[qy][jy], Qa[jy][0]);
            Qa[jy][1] = fma(wq * Fy1, c_tab.G[qy][jy], Qa[jy][1]);
          }
        }
#pragma unroll
        for (int jy = 0; jy < 3; ++jy)
#pragma unroll
          for (int ix = 0; ix < 3; ++ix)
#pragma unroll
            for (int d = 0; d < 2; ++d)
              R[jy][ix][d] += (c_tab.G[qx][ix] * g.ihx) * Pa[jy][d] + (c_tab.B[qx][ix] * g.ihy) * Qa[jy][d];
      }
#pragma unroll
  for (int jy = 0; jy < 3; ++jy)
#pragma unroll
    for (int ix = 0; ix < 3; ++ix)
#pragma unroll
      for (int d = 0; d < 2; ++d) acc.add(jy, ix, d, R[jy][ix][d]);
}

// The cell's boundary sides (forms.py:605-637).
template <class XA, class SA, class ACC>
__device__ __forceinline__ void jac_sides(const Geom& g, const Disc& ds, const Lin& L, int mu, int ci, int cj,
                                          const XA& XM, const SA& SP, int r0, int c0, const double P[3],
                                          const ACC& acc, double accp[3], double tw = 1.0) {
      if (ci == 0 || cj == 0 || ci == g.nx - 1 || cj == g.ny - 1) {
        if (cj == 0) jac_boundary_side(g, ds, L, mu, 0, side_offset(g, 0) + ci, XM, SP, r0, c0, P, acc, accp, tw);
        if (ci == g.nx - 1) jac_boundary_side(g, ds, L, mu, 1, side_offset(g, 1) + cj, XM, SP, r0, c0, P, acc, accp, tw);
        if (cj == g.ny - 1) jac_boundary_side(g, ds, L, mu, 2, side_offset(g, 2) + ci, XM, SP, r0, c0, P, acc, accp, tw);
        if (ci == 0) jac_boundary_side(g, ds, L, mu, 3, side_offset(g, 3) + cj, XM, SP, r0, c0, P, acc, accp, tw);
      }
}

// Node assembly from per-cell shared slots and the final write.
__device__ void assemble_and_store(const Geom& g, const double* sacc, int i0, int j0, int mu,
                                   const double* __restrict__ rhs, double* __restrict__ out) {
  const bool lastx = (i0 + TX >= g.nx), lasty = (j0 + TY >= g.ny);
  const int lxe = lastx ? 2 * (g.nx - (i0 - 1)) + 1 : 2 * TX + 2;  // exclusive local node bound
  const int lye = lasty ? 2 * (g.ny - (j0 - 1)) + 1 : 2 * TY + 2;
  const int wx = lxe - 2, wy = lye - 2;  // owned local nodes start at 2
  const int n = wx * wy;
  const size_t base = (size_t)mu * g.nd;
  constexpr int MAXIT = ((2 * TX + 1) * (2 * TY + 1) + NT - 1) / NT;
  double r0v[MAXIT], r1v[MAXIT];
  if (rhs) {
#pragma unroll
    for (int it = 0; it < MAXIT; ++it) {
      const int idx = threadIdx.x + it * NT;
      r0v[it] = r1v[it] = 0.0;
      if (idx < n) {
        const int ly = 2 + idx / wx, lx = 2 + idx % wx;
        const size_t o = base + 2 * ((size_t)(2 * (j0 - 1) + ly) * g.nnx + 2 * (i0 - 1) + lx);
        r0v[it] = __ldg(rhs + o);
        r1v[it] = __ldg(rhs + o + 1);
      }
    }
  }
#pragma unroll
  for (int it = 0; it < MAXIT; ++it) {
    const int idx = threadIdx.x + it * NT;
    if (idx >= n) break;
    const int ly = 2 + idx / wx, lx = 2 + idx % wx;
    double s0 = 0.0, s1 = 0.0;
    const int cxa = (lx & 1) ? (lx - 1) / 2 : lx / 2 - 1;
    const int cxb = lx / 2;
    const int cya = (ly & 1) ? (ly - 1) / 2 : ly / 2 - 1;
    const int cyb = ly / 2;
    for (int cy = cya; cy <= cyb; ++cy) {
      if (cy < 0 || cy >= CY) continue;
      for (int cx = cxa; cx <= cxb; ++cx) {
        if (cx < 0 || cx >= CX) continue;
        const int a = 3 * (ly - 2 * cy) + (lx - 2 * cx);
        const int cell = cy * CX + cx;
        s0 += sacc[(2 * a) * NT + cell];
        s1 += sacc[(2 * a + 1) * NT + cell];
      }
    }
    const int X = 2 * (i0 - 1) + lx, Y = 2 * (j0 - 1) + ly;
    const size_t o = base + 2 * ((size_t)Y * g.nnx + X);
    if (rhs) {
      s0 = r0v[it] - s0;
      s1 = r1v[it] - s1;
    }
    out[o] = s0;
    out[o + 1] = s1;
  }
}

// ---------------------------------------------------------------------------
// Slab Jacobian apply: out = J x  (or rhs - J x when rhs != null)
//
// Tiles of JT x JT cells, one thread per cell, NO redundant halo cells: nodes
// interior to a tile are complete and written directly; nodes on a tile
// boundary shared with a neighbour tile are written as partial sums to `part`
// and combined by k_jac_post in a fixed order (deterministic), which also adds
// the boundary-face side terms.
// ---------------------------------------------------------------------------
// Per-CTA phase timeline of the apply (profiling builds only, -DPDST_TRACE).
#ifdef PDST_TRACE
__device__ unsigned long long g_trace[8192][16];
#define TR(i)                                                                                          \
  do {                                                                                                 \
    if (threadIdx.x == 0) {                                                                            \
      unsigned long long t_;                                                                           \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                           \
      g_trace[blockIdx.y * gridDim.x + blockIdx.x][i] = t_;                                            \
      if ((i) == 0) {                                                                                  \
        unsigned s_;                                                                                   \
        asm volatile("mov.u32 %0, %%smid;" : "=r"(s_));                                                \
        g_trace[blockIdx.y * gridDim.x + blockIdx.x][15] = s_;                                         \
      }                                                                                                \
    }                                                                                                  \
  } while (0)
// kernel-level marks: even slots keep the minimum, odd slots the maximum
__device__ unsigned long long g_ktrace[8] = {~0ull, 0ull, ~0ull, 0ull, ~0ull, 0ull, ~0ull, 0ull};
#define KTR(i)                                                     \
  do {                                                             \
    if (threadIdx.x == 0) {                                        \
      unsigned long long t_;                                       \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));       \
      if ((i) & 1)                                                 \
        atomicMax(&g_ktrace[i], t_);                               \
      else                                                         \
        atomicMin(&g_ktrace[i], t_);                               \
    }                                                              \
  } while (0)
#define KTRT(i)                                                  \
  if ((threadIdx.x & 31) == 0) do {                              \
    unsigned long long t_;                                       \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));       \
    if ((i) & 1)                                                 \
      atomicMax(&g_ktrace[i], t_);                               \
    else                                                         \
      atomicMin(&g_ktrace[i], t_);                               \
  } while (0)
#else
#define TR(i) \
  do {        \
  } while (0)
#define KTRT(i) \
  do {          \
  } while (0)
#define KTR(i) \
  do {         \
  } while (0)
#endif
#ifndef PDST_JT
#define PDST_JT 16
#endif
constexpr int JT = PDST_JT;       // owned cells per tile side
constexpr int JNT = JT * JT;      // threads per CTA
constexpr int JPER = 8 * JT;      // perimeter nodes of a tile's node rectangle
// Staged direction planes of the apply: the tile's nodes with a one-cell ring
// (CIP jumps of the tile's edge cells), even/odd column split as in pidx.
constexpr int JNC = 2 * (JT + 2) + 1;
constexpr int JNC2 = (JNC + 1) / 2;
constexpr int JRS = 2 * JNC2;
constexpr int JPLANE = JNC * JRS;
// The cells' pressure dofs are staged in shared memory: all Radau nodes with
// the planes while two CTAs still fit an SM (DG(0), DG(1)); beyond, one node
// at a time, issued at the start of that node's volume phase.
__host__ __device__ constexpr bool jac_pstage(int k1) { return k1 <= 2; }
__host__ __device__ constexpr int jpidx(int r, int c) { return r * JRS + (c & 1) * JNC2 + (c >> 1); }

// A staged direction plane addressed by its offset in the kernel's dynamic
// shared memory (the accesses stay LDS; a pointer array can be demoted to
// local memory and turn them into generic loads).  A node holds both velocity
// components as one double2, even / odd node columns split per row, so the
// threads of consecutive cells read consecutive 16-byte words: one
// conflict-free LDS.128 per node instead of two LDS.64.
struct PlaneS {
  int o;  // offset of the plane in doubles (a multiple of 2)
  __device__ __forceinline__ double2 at2(int r, int c) const {
    return reinterpret_cast<const double2*>(g_dsmem + o)[jpidx(r, c)];
  }
  __device__ __forceinline__ double at(int d, int r, int c) const {
    const double2 v = at2(r, c);
    return d == 0 ? v.x : v.y;
  }
};

// Issue the asynchronous staging of one velocity block into the apply's plane
// at offset o (zero outside the domain): one 16-byte copy per node when the
// block is 16-byte aligned (even nd, or node 0), else two 8-byte copies.
__device__ __forceinline__ void stage_jac_async(const Geom& g, const double* __restrict__ v, int o, int X0, int Y0) {
  const bool al16 = (reinterpret_cast<size_t>(v) & 15) == 0;
  double2* pl = reinterpret_cast<double2*>(g_dsmem + o);
  // node (r, c) of the staged square per thread, advanced by JNT nodes per step without divisions
  int r = threadIdx.x / JNC, c = threadIdx.x - r * JNC;
  constexpr int DR = JNT / JNC, DC = JNT - DR * JNC;
  if (al16) {
    for (; r < JNC; r += DR) {
      const int X = X0 + c, Y = Y0 + r;
      const bool in = X >= 0 && X < g.nnx && Y >= 0 && Y < g.nny;
      cp_async16(pl + jpidx(r, c), in ? v + 2 * ((size_t)Y * g.nnx + X) : v, in);
      c += DC;
      if (c >= JNC) {
        c -= JNC;
        ++r;
      }
    }
  } else {
    for (; r < JNC; r += DR) {
      const int X = X0 + c, Y = Y0 + r;
      const bool in = X >= 0 && X < g.nnx && Y >= 0 && Y < g.nny;
      const double* src = in ? v + 2 * ((size_t)Y * g.nnx + X) : v;
      double2* dst = pl + jpidx(r, c);
      cp_async8(&dst->x, src, in);
      cp_async8(&dst->y, in ? src + 1 : v, in);
      c += DC;
      if (c >= JNC) {
        c -= JNC;
        ++r;
      }
    }
  }
}

__host__ __device__ inline int jac_tiles_x(const Geom& g) { return (g.nx + JT - 1) / JT; }
__host__ __device__ inline int jac_tiles_y(const Geom& g) { return (g.ny + JT - 1) / JT; }

// Canonical perimeter index of node (lx, ly) of a full T x T tile node rectangle.
template <int T>
__device__ __forceinline__ int perim_t(int lx, int ly) {
  if (ly == 0) return lx;
  if (ly == 2 * T) return 2 * T + 1 + lx;
  if (lx == 0) return 2 * (2 * T + 1) + ly - 1;
  return 2 * (2 * T + 1) + 2 * T - 1 + ly - 1;
}
__device__ __forceinline__ int perim(int lx, int ly) { return perim_t<JT>(lx, ly); }

// ---------------------------------------------------------------------------
// Apply cache (built once per linearization by k_apply_cache, read by every
// apply): the reference's per-quadrature-point linearization cache
// (forms.py:544-578) in the form the apply consumes, tile-major so that a
// warp's 32 cells read one contiguous 256-byte row per slot.
//   apc[((tile * k1 + mu) * APC_SLOTS + s) * JNT + t],  t = cell in tile
//   volume slots s = (qx * 6 + k) * 4 + qy with wq = tau w_mu hx hy w_qx w_qy:
//     k = 0   e   = wq eta
//     k = 1-3 a~  = sqrt(-wq gamma) (a0, a1, a2),  A = sym grad v = [[a0 a2][a2 a1]]
//             (gamma <= 0 for 1 < p <= 2, so wq T(B) = e B - (a~ : B) a~)
//     k = 4-5 wq v (convection)
//   CIP slots 96 + 6 f + e, the cell's right (f = 0) and top (f = 1) faces:
//     the symmetric 3x3 face matrix W[t][t'] = sum_q c_q B[q][t] B[q][t']
//     (e = 00 01 02 11 12 22) with the face weight of cip_face
//     c_q = tau w_mu gamma_cip h^2 / hn^2 (w_q h) |v_L . n|, so the face term
//     is RD = W J with J the jump of the normal derivative at the 3 face
//     nodes.  A cell's left / bottom faces are its neighbours' right / top.
// ---------------------------------------------------------------------------
constexpr int APC_VOL = 96;
constexpr int APC_SLOTS = APC_VOL + 12;
#ifndef PDST_PF_AHEAD
#define PDST_PF_AHEAD 2  // half-columns between the L2 prefetch and the use
#endif

// L2 prefetch of half h (0..7: Gauss column h/2, points 2(h%2), 2(h%2)+1) of
// a node's cache block; h == 8 is the CIP block.
__device__ __forceinline__ void apc_prefetch_l2(const double* __restrict__ cp, int h, bool hasg = true) {
  // a warp's half-column is 12 slot rows x 256 bytes = 24 lines: lane l < 24 prefetches line l
  const int lane = threadIdx.x & 31;
  const int i = lane >> 1;  // slot row 0..11 of the half-column (or of the CIP block)
  const double* w0 = cp - lane + 16 * (lane & 1);
  if (h < 8) {
    const int qx = h >> 1, qy0 = (h & 1) * 2;
    const int j = i / 6, k = i - 6 * j;
    if (lane < 24 && (hasg || k == 0 || k > 3)) prefetch_l2(w0 + (qx * 24 + k * 4 + qy0 + j) * JNT);
  } else if (h == 8) {
    if (lane < 24) prefetch_l2(w0 + (APC_VOL + i) * JNT);
  }
}

// Completion counters of the tile pass, one per Radau node: a tile adds 1
// once all its stores of that node (interior sums, tile-line partials, raw
// strip sums) are done — after a CTA barrier, by one thread, behind a
// device-scope fence — and the epilogue (k_jac_post) of that node polls the
// counter instead of waiting for the whole grid, so node mu's epilogue runs
// under the tile pass of node mu + 1.  The last epilogue CTA to finish sets the
// counters back to zero (every epilogue CTA is past its waits by then, and the
// next apply's tile pass signals only after its own grid-dependency wait), so
// the targets are constants and a captured launch sequence can be replayed.
// No deadlock: the epilogue is launched (PDL) only after every tile CTA has
// started.
__device__ __forceinline__ void tile_signal(unsigned long long* sig) {
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(sig, 1ull);
  }
}
__device__ __forceinline__ void tile_wait(const unsigned long long* sig, unsigned long long target) {
  if (threadIdx.x == 0) {
    unsigned long long v;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(sig) : "memory");
      if (v >= target) break;
      __nanosleep(64);
    }
  }
  __syncthreads();
}

// 1-D tables of the apply with the mesh scales folded in (kernel parameter).
struct JTabs {
  double B[4][3];    // L_i(s_q)
  double Gx[4][3];   // L_i'(s_q) / hx
  double Gy[4][3];   // L_i'(s_q) / hy
  double w[4];       // w_q
  double wyh[4];     // w_q (s_q - 1/2)
  double xh[4];      // s_q - 1/2
  double cJ[5];      // normal-derivative jump across a face from the 5 node
                     // lines of the two cells: L'(1) on the left, -L'(0) on the right
  // 1-D Gauss sums of the pressure coupling (P1disc x Q2 is separable):
  double pAx[3], pAy[3];  // sum_q w_q L_i'(s_q) / h
  double pBx[3], pBy[3];  // sum_q w_q (s_q - 1/2) L_i'(s_q) / h
  double pM0[3];          // sum_q w_q L_i(s_q)
  double pM1[3];          // sum_q w_q (s_q - 1/2) L_i(s_q)
};

// Volume terms (forms.py:589-603) from the apply cache, without the pressure
// coupling (evaluated with the temporal mass); the first writer of the cell's
// slot.  Called by every thread of the CTA (cells outside the mesh stream
// zeros into their own slot) because of the barrier inside.
template <bool HG, class XA>
__device__ __forceinline__ void jac_volume_cached(const JTabs& T, const Disc& ds, const double* __restrict__ cp,
                                                  const XA& XM, int r0, int c0, double2* slot, bool sync_first,
                                                  unsigned long long* sig) {
#pragma unroll 1
  for (int qx = 0; qx < 4; ++qx) {
    double xB[3][2], xG[3][2];
#pragma unroll
    for (int jy = 0; jy < 3; ++jy) {
      const double2 f0 = XM.at2(r0 + jy, c0), f1 = XM.at2(r0 + jy, c0 + 1), f2 = XM.at2(r0 + jy, c0 + 2);
      xB[jy][0] = T.B[qx][0] * f0.x + T.B[qx][1] * f1.x + T.B[qx][2] * f2.x;
      xB[jy][1] = T.B[qx][0] * f0.y + T.B[qx][1] * f1.y + T.B[qx][2] * f2.y;
      xG[jy][0] = T.Gx[qx][0] * f0.x + T.Gx[qx][1] * f1.x + T.Gx[qx][2] * f2.x;
      xG[jy][1] = T.Gx[qx][0] * f0.y + T.Gx[qx][1] * f1.y + T.Gx[qx][2] * f2.y;
    }
    double Pa[3][2] = {{0, 0}, {0, 0}, {0, 0}}, Qa[3][2] = {{0, 0}, {0, 0}, {0, 0}};
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int h = 2 * qx + hh;
      double cv[2][6];
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int k = 0; k < 6; ++k)  // Picard: the a~ slots are zeros, not read
          cv[j][k] = (k >= 1 && k <= 3 && !HG) ? 0.0 : ldg_stream(cp + (qx * 24 + k * 4 + 2 * hh + j) * JNT);
      apc_prefetch_l2(cp, h + PDST_PF_AHEAD, HG);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int qy = 2 * hh + j;
        double u[2], ux[2], uy[2];
#pragma unroll
        for (int d = 0; d < 2; ++d) {
          u[d] = T.B[qy][0] * xB[0][d] + T.B[qy][1] * xB[1][d] + T.B[qy][2] * xB[2][d];
          ux[d] = T.B[qy][0] * xG[0][d] + T.B[qy][1] * xG[1][d] + T.B[qy][2] * xG[2][d];
          uy[d] = T.Gy[qy][0] * xB[0][d] + T.Gy[qy][1] * xB[1][d] + T.Gy[qy][2] * xB[2][d];
        }
        const double ce = cv[j][0], ca0 = cv[j][1], ca1 = cv[j][2], ca2 = cv[j][3], cv0 = cv[j][4], cv1 = cv[j][5];
        // wq T(B) with B = sym grad u (b0, b1, b2 = cc / 2)
        const double b0 = ux[0], b1 = uy[1], cc = uy[0] + ux[1];
        const double t = ca0 * b0 + ca1 * b1 + ca2 * cc;
        double F00 = ce * b0 - t * ca0;
        double F11 = ce * b1 - t * ca1;
        double F01 = ce * (0.5 * cc) - t * ca2;
        // - wq (u (x) v + v (x) u)
        F00 -= 2.0 * u[0] * cv0;
        F11 -= 2.0 * u[1] * cv1;
        F01 -= u[1] * cv0 + u[0] * cv1;
#pragma unroll
        for (int jy = 0; jy < 3; ++jy) {
          Pa[jy][0] = fma(F00, T.B[qy][jy], Pa[jy][0]);
          Pa[jy][1] = fma(F01, T.B[qy][jy], Pa[jy][1]);
          Qa[jy][0] = fma(F01, T.Gy[qy][jy], Qa[jy][0]);
          Qa[jy][1] = fma(F11, T.Gy[qy][jy], Qa[jy][1]);
        }
      }
    }
    // the column's test-function sums go straight to the cell's slot (the
    // first column stores): keeps the loop at 128 registers.  The slots still
    // hold the previous Radau node's sums until every thread has assembled
    // its nodes: that barrier sits here, behind the first column's arithmetic.
    if (qx == 0 && sync_first) {
      __syncthreads();
      tile_signal(sig);  // the previous node's sums of this tile are all stored
    }
#pragma unroll
    for (int jy = 0; jy < 3; ++jy)
#pragma unroll
      for (int ix = 0; ix < 3; ++ix) {
        const double v0 = T.Gx[qx][ix] * Pa[jy][0] + T.B[qx][ix] * Qa[jy][0];
        const double v1 = T.Gx[qx][ix] * Pa[jy][1] + T.B[qx][ix] * Qa[jy][1];
        double2* sp = slot + (3 * jy + ix) * JNT;  // both components: one 16-byte access
        if (qx == 0) {
          *sp = make_double2(v0, v1);
        } else {
          const double2 o = *sp;
          *sp = make_double2(o.x + v0, o.y + v1);
        }
      }
  }
}

// CIP face term (forms.py:639-650) with the cached face matrix W:
// RD = W J, J[t] = jump of the normal derivative at face line t, from the 5
// staged node lines of the left / lower cell at (rL, cL) and its neighbour.
template <class FA>
__device__ __forceinline__ void cip_face_w(const JTabs& T, int axis, const FA& F, int rL, int cL, const double W[6],
                                           double RD[3][2]) {
  double J[3][2];
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    double v0 = 0.0, v1 = 0.0;
#pragma unroll
    for (int m = 0; m < 5; ++m) {
      const double2 f = axis == 0 ? F.at2(rL + t, cL + m) : F.at2(rL + m, cL + t);
      v0 = fma(T.cJ[m], f.x, v0);
      v1 = fma(T.cJ[m], f.y, v1);
    }
    J[t][0] = v0;
    J[t][1] = v1;
  }
#pragma unroll
  for (int d = 0; d < 2; ++d) {
    RD[0][d] = W[0] * J[0][d] + W[1] * J[1][d] + W[2] * J[2][d];
    RD[1][d] = W[1] * J[0][d] + W[3] * J[1][d] + W[4] * J[2][d];
    RD[2][d] = W[2] * J[0][d] + W[4] * J[1][d] + W[5] * J[2][d];
  }
}

// The four CIP faces of a cell (right, top, left, bottom), own side only;
// W[f] = the faces' matrices (left / bottom from the neighbours' cache).
template <class FA, class ACC>
__device__ __forceinline__ void cip_all_w(const JTabs& T, const Geom& g, const FA& F, int ci, int cj, int r0, int c0,
                                          const double (*W)[6], const ACC& acc) {
  double RD[3][2];
  if (ci < g.nx - 1) {
    cip_face_w(T, 0, F, r0, c0, W[0], RD);
    cip_scatter(0, true, 1.0, RD, acc);
  }
  if (cj < g.ny - 1) {
    cip_face_w(T, 1, F, r0, c0, W[1], RD);
    cip_scatter(1, true, 1.0, RD, acc);
  }
  if (ci > 0) {
    cip_face_w(T, 0, F, r0, c0 - 2, W[2], RD);
    cip_scatter(0, false, 1.0, RD, acc);
  }
  if (cj > 0) {
    cip_face_w(T, 1, F, r0 - 2, c0, W[3], RD);
    cip_scatter(1, false, 1.0, RD, acc);
  }
}

// ---------------------------------------------------------------------------
// Apply epilogue (k_side_products + k_jac_post, PDL-launched behind the tile
// pass and released per Radau node by its completion counters): the nodes the
// tile pass cannot finish alone.
//   * tile-line nodes (shared by 2 or 4 tiles): sum of the tiles' partials;
//   * boundary-strip nodes (in a cell with a boundary side) and the pressures
//     of boundary cells: + the side terms tau w_mu B_f x_loc of every boundary
//     face whose cell holds the dof, with the precomputed side matrices B_f
//     (forms.py:605-637 probed once per linearization, k_boundary_matrices).
// The tile pass writes these dofs without the right-hand side; here
// y = rhs - s or y = s with s = (interior sum) + (side terms), summed in a
// fixed order, so apply and defect agree bitwise.  The side products depend
// only on x and run under the tile pass.
// ---------------------------------------------------------------------------
__host__ __device__ inline bool in_strip(const Geom& g, int X, int Y) {
  return X <= 2 || Y <= 2 || X >= g.nnx - 3 || Y >= g.nny - 3;
}
__host__ __device__ inline bool on_tile_line(const Geom& g, int X, int Y) {
  const int ntx = jac_tiles_x(g), nty = jac_tiles_y(g);
  return (X % (2 * JT) == 0 && X > 0 && X / (2 * JT) < ntx) || (Y % (2 * JT) == 0 && Y > 0 && Y / (2 * JT) < nty);
}

// Strip node t -> (X, Y): the rows 0-2 and nny-3..nny-1 in full, then the
// columns 0-2 and nnx-3..nnx-1 of the rows between.
struct StripIdx {
  int nb, nt, ncl, ncr;  // bottom rows, top rows, left cols, right cols
  __host__ __device__ StripIdx(const Geom& g) {
    nb = min(3, g.nny);
    nt = min(3, g.nny - nb);
    ncl = min(3, g.nnx);
    ncr = min(3, g.nnx - ncl);
  }
  __host__ __device__ size_t count(const Geom& g) const {
    return (size_t)(nb + nt) * g.nnx + (size_t)(g.nny - nb - nt) * (ncl + ncr);
  }
  __device__ void node(const Geom& g, size_t t, int& X, int& Y) const {
    const size_t full = (size_t)(nb + nt) * g.nnx;
    if (t < full) {
      const int r = (int)(t / g.nnx);
      Y = r < nb ? r : g.nny - nt + (r - nb);
      X = (int)(t % g.nnx);
    } else {
      const size_t u = t - full;
      const int w = ncl + ncr;
      Y = nb + (int)(u / w);
      const int cc = (int)(u % w);
      X = cc < ncl ? cc : g.nnx - ncr + (cc - ncl);
    }
  }
};

// Boundary cells: bottom row, top row, then the left / right cells of the rows
// between (every cell when the mesh is one cell wide or tall).
__host__ __device__ inline size_t n_bcells(const Geom& g) {
  return g.nx == 1 || g.ny == 1 ? (size_t)g.ncells : (size_t)2 * g.nx + 2 * (g.ny - 2);
}
__device__ inline void bcell_of(const Geom& g, size_t t, int& ci, int& cj) {
  if (g.nx == 1 || g.ny == 1) {
    ci = (int)(t % g.nx);
    cj = (int)(t / g.nx);
  } else if (t < (size_t)g.nx) {
    ci = (int)t;
    cj = 0;
  } else if (t < (size_t)2 * g.nx) {
    ci = (int)(t - g.nx);
    cj = g.ny - 1;
  } else {
    const size_t u = t - 2 * g.nx;
    cj = 1 + (int)(u / 2);
    ci = (u % 2) ? g.nx - 1 : 0;
  }
}
// index of boundary cell (ci, cj), or -1 for an interior cell
__device__ inline int bcell_index(const Geom& g, int ci, int cj) {
  if (g.nx == 1 || g.ny == 1) return cj * g.nx + ci;
  if (cj == 0) return ci;
  if (cj == g.ny - 1) return g.nx + ci;
  if (ci == 0) return 2 * g.nx + 2 * (cj - 1);
  if (ci == g.nx - 1) return 2 * g.nx + 2 * (cj - 1) + 1;
  return -1;
}

// Side products of the boundary cells: sp[mu][r][cb] = sum over the cell's
// boundary faces f (side order, cut faces skipped) of tau w_mu (B_f x_loc)[r],
// B_f the side matrices of forms.py:605-637 probed once per linearization
// (k_boundary_matrices, face-contiguous, column-major [mu][bf][col][row]).  One warp per
// boundary cell, lane r < 21 computes row r; x_loc is loaded once and
// broadcast by shuffles.  Depends only on x: launched with PDL behind the tile
// pass (whose CTAs trigger it after their own wait, so x is complete), its
// short-lived CTAs run on the SMs the tile pass leaves half empty and count
// themselves done in `sdone` (tile_signal) for the epilogue.
__global__ void __launch_bounds__(128, 8) k_side_products(Geom g, TimeData td, const double* __restrict__ bmat,
                                                       const double* __restrict__ x, double* __restrict__ sp,
                                                       unsigned long long* __restrict__ sdone) {
  pdl_trigger();
  const int mu = blockIdx.y, lane = threadIdx.x & 31;
  const size_t ncb = n_bcells(g);
  const size_t cb = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (cb < ncb) {
    int ci, cj;
    bcell_of(g, cb, ci, cj);
    const double* xm = x + (size_t)mu * g.nd;
    double xj = 0.0;
    if (lane < 18) {
      const int n = lane >> 1;
      xj = __ldg(xm + 2 * ((size_t)(2 * cj + n / 3) * g.nnx + 2 * ci + n % 3) + (lane & 1));
    } else if (lane < 21 && !g.th) {  // (Taylor-Hood: no P1disc pressure; pdst_th.cu)
      xj = __ldg(xm + g.mv + 3 * ((size_t)cj * g.nx + ci) + (lane - 18));
    }
    const int r = lane < 21 ? lane : 20;
    const double tw = td.tau_w[mu];
    double acc = 0.0;
    for (int side = 0; side < 4; ++side) {
      const bool on = side == 0 ? cj == 0 : side == 1 ? ci == g.nx - 1 : side == 2 ? cj == g.ny - 1 : ci == 0;
      const int bf = side_offset(g, side) + ((side == 0 || side == 2) ? ci : cj);
      if (!on || g.dirichlet[bf] == kCutSide) continue;
      const double* Br = bmat + ((size_t)mu * g.nbf + bf) * 441 + r;  // row r of column-major B_f
      double s = 0.0;
#pragma unroll
      for (int col = 0; col < 21; ++col) s = fma(__ldg(Br + 21 * col), __shfl_sync(0xffffffffu, xj, col), s);
      acc += tw * s;
    }
    if (lane < 21) sp[((size_t)mu * 21 + lane) * ncb + cb] = acc;
  }
  __syncthreads();
  tile_signal(sdone);
  KTR(3);
}

// Side terms at velocity node (X, Y): sum of the side products of the
// boundary cells containing it, (row, column) order.
__device__ void strip_sides(const Geom& g, const double* __restrict__ sp, int mu, int X, int Y, double b[2]) {
  b[0] = b[1] = 0.0;
  const size_t ncb = n_bcells(g);
  const int jlo = max(0, (Y - 1) / 2), jhi = min(g.ny - 1, Y / 2);
  const int ilo = max(0, (X - 1) / 2), ihi = min(g.nx - 1, X / 2);
  for (int cj = jlo; cj <= jhi; ++cj)
    for (int ci = ilo; ci <= ihi; ++ci) {
      const int cb = bcell_index(g, ci, cj);
      if (cb < 0) continue;
      const int a = 3 * (Y - 2 * cj) + (X - 2 * ci);
      b[0] += __ldcg(sp + ((size_t)mu * 21 + 2 * a) * ncb + cb);
      b[1] += __ldcg(sp + ((size_t)mu * 21 + 2 * a + 1) * ncb + cb);
    }
}

// Sum of the tile partials at tile-line node (X, Y).
__device__ void tile_partials(const Geom& g, const double* part, int mu, int X, int Y, double s[2]) {
  const int ntx = jac_tiles_x(g), nty = jac_tiles_y(g);
  int bxs[2], bys[2], nbx, nby;
  if (X % (2 * JT) == 0 && X > 0 && X / (2 * JT) < ntx) {
    bxs[0] = X / (2 * JT) - 1;
    bxs[1] = X / (2 * JT);
    nbx = 2;
  } else {
    bxs[0] = min(X / (2 * JT), ntx - 1);
    nbx = 1;
  }
  if (Y % (2 * JT) == 0 && Y > 0 && Y / (2 * JT) < nty) {
    bys[0] = Y / (2 * JT) - 1;
    bys[1] = Y / (2 * JT);
    nby = 2;
  } else {
    bys[0] = min(Y / (2 * JT), nty - 1);
    nby = 1;
  }
  const size_t ntiles = (size_t)ntx * nty;
  s[0] = s[1] = 0.0;
  for (int b = 0; b < nby; ++b)
    for (int a = 0; a < nbx; ++a) {
      const int lx = X - 2 * JT * bxs[a], ly = Y - 2 * JT * bys[b];
      const double* pp = part + (((size_t)mu * ntiles + (size_t)bys[b] * ntx + bxs[a]) * JPER + perim(lx, ly)) * 2;
      s[0] += __ldcg(pp);  // written by CTAs still running: not through L1
      s[1] += __ldcg(pp + 1);
    }
}

// Work items per Radau node: strip nodes, then tile-line nodes off the
// strips, then boundary cells (pressure).  Launched with PDL behind the side
// products but WITHOUT a grid-dependency wait (which would also wait for the
// tile pass, the side products' own predecessor): the side products and the
// tile pass's sums of node mu are awaited through their completion counters
// (tile_wait), so node mu's items run while the tile pass works on the later
// nodes.  Every item only sums.
__global__ void __launch_bounds__(128, 8) k_jac_post(Geom g, TimeData td, const double* __restrict__ part,
                                                 const double* __restrict__ sp, const double* __restrict__ rhs,
                                                 double* __restrict__ out,
                                                 const unsigned long long* __restrict__ done,
                                                 unsigned long long target, unsigned long long starget) {
  pdl_trigger();  // a PDL-launched consumer (the Vanka GEMV) may start its own prologue
  STEP_MARK(rhs ? 3 : 1, 0);
  const int mu = blockIdx.y;
  const size_t base = (size_t)mu * g.nd;
  // 1. decode the item (nothing here depends on the other kernels)
  int kind = 0;  // 1 strip node, 2 tile-line node off the strips, 3 boundary cell (pressure)
  int X = 0, Y = 0;
  size_t o = 0, cb = 0;
  {
    const StripIdx si(g);
    const size_t ns = si.count(g);
    const int ntx = jac_tiles_x(g), nty = jac_tiles_y(g);
    const size_t nv = (size_t)(ntx - 1) * g.nny, nh = (size_t)(nty - 1) * g.nnx;
    const size_t ncb = n_bcells(g);
    size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < ns) {
      si.node(g, t, X, Y);
      kind = 1;
    } else if ((t -= ns) < nv + nh) {
      bool skip = false;
      if (t < nv) {
        X = 2 * JT * (int)(t / g.nny + 1);
        Y = (int)(t % g.nny);
      } else {
        const size_t u = t - nv;
        Y = 2 * JT * (int)(u / g.nnx + 1);
        X = (int)(u % g.nnx);
        skip = X % (2 * JT) == 0 && X > 0 && X / (2 * JT) < ntx;  // on a vertical line
      }
      if (!skip && !in_strip(g, X, Y)) kind = 2;
    } else if ((t -= nv + nh) < ncb && !g.th) {
      int ci, cj;
      bcell_of(g, t, ci, cj);
      cb = t;
      o = base + g.mv + 3 * ((size_t)cj * g.nx + ci);
      kind = 3;
    }
    if (kind == 1 || kind == 2) o = base + 2 * ((size_t)Y * g.nnx + X);
  }
  // 2. what does not depend on the tile pass: right-hand side, side products
  double r[3] = {0.0, 0.0, 0.0}, b[3] = {0.0, 0.0, 0.0};
  if (rhs && kind) {
    r[0] = __ldg(rhs + o);
    r[1] = __ldg(rhs + o + 1);
    if (kind == 3) r[2] = __ldg(rhs + o + 2);
  }
  tile_wait(done + 4, starget);  // the side products (all threads pass a barrier)
  if (kind == 1) {
    strip_sides(g, sp, mu, X, Y, b);
  } else if (kind == 3) {
    const size_t ncb = n_bcells(g);
#pragma unroll
    for (int j = 0; j < 3; ++j) b[j] = __ldcg(sp + ((size_t)mu * 21 + 18 + j) * ncb + cb);
  }
  // 3. the tile pass's sums of node mu
  tile_wait(done + mu, target);
  // The last epilogue CTA past its waits re-arms the counters (done[5] counts
  // them): nobody polls any more, and the next apply signals only after this
  // grid has completed.  Off the critical path: the items follow.
  if (threadIdx.x == 0) {
    unsigned long long* cnt = const_cast<unsigned long long*>(done);
    if (atomicAdd(cnt + 5, 1ull) == (unsigned long long)gridDim.x * gridDim.y - 1) {
#pragma unroll
      for (int i = 0; i < 6; ++i) cnt[i] = 0ull;
    }
  }
  KTRT(6);
  if (mu == (int)gridDim.y - 1) STEP_MARK(rhs ? 3 : 1, 1);  // the last node's release
  if (kind == 1 || kind == 2) {
    double s[2];
    if (kind == 2 || on_tile_line(g, X, Y)) {
      tile_partials(g, part, mu, X, Y, s);
    } else {
      s[0] = __ldcg(out + o);
      s[1] = __ldcg(out + o + 1);
    }
    s[0] += b[0];
    s[1] += b[1];
    out[o] = rhs ? r[0] - s[0] : s[0];
    out[o + 1] = rhs ? r[1] - s[1] : s[1];
    KTRT(7);
  } else if (kind == 3) {
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const double s = __ldcg(out + o + j) + b[j];
      out[o + j] = rhs ? r[j] - s : s;
    }
    KTRT(7);
  }
  STEP_MARK(rhs ? 3 : 1, 2);
}

__host__ __device__ inline size_t jac_post_items(const Geom& g) {
  const size_t ncb = n_bcells(g);
  return StripIdx(g).count(g) + (size_t)(jac_tiles_x(g) - 1) * g.nny + (size_t)(jac_tiles_y(g) - 1) * g.nnx + ncb;
}

// One thread per cell, two CTAs (16 warps) per SM: the state is not staged —
// its contribution comes from the apply cache, streamed once per apply — so
// the CTA holds only the direction planes of all Radau nodes and one set of
// per-cell node slots.
template <int K1, bool HG>
__global__ void __launch_bounds__(JNT, 65536 / (JNT * 128)) k_jacobian(Geom g, TimeData td, Disc ds, Lin L,
                                                  const double* __restrict__ x, const double* __restrict__ rhs,
                                                  double* __restrict__ out, double* __restrict__ part,
                                                  unsigned long long* __restrict__ done, const JTabs T) {
  double* sacc = g_dsmem + (size_t)K1 * 2 * JPLANE;  // [18][JNT] per-cell node contributions
  double* spres = sacc + 18 * JNT;                    // [K1][3][JNT] the cells' pressure dofs (K1 <= 2), else [3][JNT]
  constexpr bool PSTAGE = jac_pstage(K1);
  // [K1][2][JPLANE] direction x_nu, all Radau nodes (one-cell ring), in front
  const int bx = blockIdx.x, by = blockIdx.y;
  const int i0 = bx * JT, j0 = by * JT;
  const int X0 = 2 * (i0 - 1), Y0 = 2 * (j0 - 1);
  const int ntx = min(JT, g.nx - i0), nty = min(JT, g.ny - j0);
  PlaneS XP[K1];
#pragma unroll
  for (int nu = 0; nu < K1; ++nu) XP[nu] = PlaneS{nu * 2 * JPLANE};
  const int tx = threadIdx.x % JT, ty = threadIdx.x / JT;
  const int ci = i0 + tx, cj = j0 + ty;
  const bool valid = tx < ntx && ty < nty;
  const int c = cj * g.nx + ci;
  const int r0 = 2 + 2 * ty, c0 = 2 + 2 * tx;  // staged origin of the cell's nodes
  const bool cip = ds.convection && ds.gamma_cip > 0.0;
  const size_t ntiles = (size_t)jac_tiles_x(g) * jac_tiles_y(g);
  const size_t tile = (size_t)by * jac_tiles_x(g) + bx;
  // nodes owned by this cell in the tile: its lower-left 2x2, plus the tile's
  // last row / column of nodes for the last cell column / row
  const bool lastx = tx == ntx - 1, lasty = ty == nty - 1;
  const double* cbase = L.apc + tile * K1 * APC_SLOTS * JNT + threadIdx.x;

  TR(0);
  KTR(0);
  STEP_MARK(rhs ? 2 : 0, 0);
  // HG == false (Picard, or no viscous term): the a~ slots are zeros and never read
  // The direction's node rows towards L2 before the wait as well: L2 is the
  // point of coherence, so lines the predecessor still writes are updated in
  // place, and a cold x (first apply after other work) lands while we wait.
  for (int idx = threadIdx.x; idx < K1 * JNC * 5; idx += JNT) {
    const int nu = idx / (JNC * 5), rem = idx - nu * (JNC * 5);
    const int r = rem / 5, X = X0 + 8 * (rem - 5 * r), Y = Y0 + r;
    if (Y >= 0 && Y < g.nny && X < g.nnx)
      prefetch_l2(x + (size_t)nu * g.nd + 2 * ((size_t)Y * g.nnx + max(X, 0)));
  }
  if (valid)  // the coefficient stream does not depend on the predecessor
    for (int h = 0; h < PDST_PF_AHEAD; ++h) apc_prefetch_l2(cbase, h, HG);
  // launched with PDL: x (and the scratch the predecessor's epilogue may still
  // read) only after the predecessor has completed; then k_side_products may
  // start under this grid (k_jac_post polls both kernels' completion counters)
  pdl_wait();
  STEP_MARK(rhs ? 2 : 0, 1);
  pdl_trigger();
  // node 0's plane in its own group: its volume and CIP (which read only that
  // plane) start while the other planes land; the temporal mass waits for all
  stage_jac_async(g, x, 0, X0, Y0);
  cp_async_commit();
  for (int nu = 1; nu < K1; ++nu) stage_jac_async(g, x + (size_t)nu * g.nd, nu * 2 * JPLANE, X0, Y0);
  // the cell's pressure dofs of every node (read by the own thread with the temporal mass)
  if (PSTAGE && valid && ds.pressure && !g.th)
#pragma unroll
    for (int nu = 0; nu < K1; ++nu)
#pragma unroll
      for (int j = 0; j < 3; ++j)
        cp_async8(spres + (size_t)(nu * 3 + j) * JNT + threadIdx.x, x + (size_t)nu * g.nd + g.mv + 3 * (size_t)c + j, true);
  cp_async_commit();
  cp_async_wait_group<1>();
  __syncthreads();
  TR(1);
  for (int mu = 0; mu < K1; ++mu) {
    const double tw = td.tau_w[mu];
    const double* cp = cbase + (size_t)mu * APC_SLOTS * JNT;
    double2* slot = reinterpret_cast<double2*>(sacc) + threadIdx.x;  // [9 nodes][JNT] (both components)
    const PlaneS XM{mu * 2 * JPLANE};
    double accp[3] = {0.0, 0.0, 0.0};
    if (!PSTAGE && valid && ds.pressure && !g.th) {  // this node's pressure dofs, landed by the mass phase
#pragma unroll
      for (int j = 0; j < 3; ++j)
        cp_async8(spres + (size_t)j * JNT + threadIdx.x, x + (size_t)mu * g.nd + g.mv + 3 * (size_t)c + j, true);
      cp_async_commit();
    }
    // CIP, temporal mass and boundary sides accumulate in registers (the
    // volume's registers are free by then) and reach the slot in one pass
    double ra[3][3][2];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) ra[a][b][0] = ra[a][b][1] = 0.0;
    const RegAcc racc{ra};
    // tau w_mu J_mu x_mu: volume, boundary sides, CIP faces (weights carry tau w_mu)
    if (K1 > 1 || valid) jac_volume_cached<HG>(T, ds, cp, XM, r0, c0, slot, K1 > 1 && mu > 0, done + (mu > 0 ? mu - 1 : 0));
    TR(2 + 5 * mu);
    // The cell's indices are recomputed from the (laundered) thread and block
    // ids here, so that nothing but the stream pointer, the slot and the staged
    // origin stays live across the volume phase (ptxas spilled the tile-edge
    // flags to local memory otherwise and the assembly stalled on the reload).
    int tid_ = threadIdx.x, bx_ = blockIdx.x, by_ = blockIdx.y;
    asm volatile("" : "+r"(tid_), "+r"(bx_), "+r"(by_));
    const int tx = tid_ % JT, ty = tid_ / JT;
    const int i0 = bx_ * JT, j0 = by_ * JT;
    const int ci = i0 + tx, cj = j0 + ty;
    const int c = cj * g.nx + ci;
    const size_t tile = (size_t)by_ * jac_tiles_x(g) + bx_;
    const bool lastx = tx == min(JT, g.nx - i0) - 1, lasty = ty == min(JT, g.ny - j0) - 1;
    double rv[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};  // rhs of the own 2x2 nodes (defect mode)
    double rp[3] = {0, 0, 0};
    if (valid) {
      if (cip) {
        // face matrices: own right / top, the left / bottom neighbours' right / top
        double W[4][6];
        const double* wl = tx > 0 ? cp - 1 : L.apc + ((tile - 1) * K1 + mu) * APC_SLOTS * JNT + ty * JT + JT - 1;
        const double* wb = ty > 0 ? cp - JT : L.apc + ((tile - jac_tiles_x(g)) * K1 + mu) * APC_SLOTS * JNT + (JT - 1) * JT + tx;
#pragma unroll
        for (int e = 0; e < 6; ++e) {
          W[0][e] = __ldg(cp + (APC_VOL + e) * JNT);
          W[1][e] = __ldg(cp + (APC_VOL + 6 + e) * JNT);
          W[2][e] = ci > 0 ? __ldg(wl + (APC_VOL + e) * JNT) : 0.0;
          W[3][e] = cj > 0 ? __ldg(wb + (APC_VOL + 6 + e) * JNT) : 0.0;
        }
        cip_all_w(T, g, XM, ci, cj, r0, c0, W, racc);
      }
      if (mu + 1 < K1)  // the next node's first half-columns towards L2
        for (int h = 0; h < PDST_PF_AHEAD; ++h) apc_prefetch_l2(cp + APC_SLOTS * JNT, h, HG);
      TR(3 + 5 * mu);
    }
    if (valid) {
      // defect mode: the right-hand side of this cell's own nodes (lower-left
      // 2x2) and pressures, loaded behind the face matrices, for the assembly
      if (rhs) {
#pragma unroll
        for (int n = 0; n < 4; ++n) {
          const size_t o = (size_t)mu * g.nd + 2 * ((size_t)(2 * cj + (n >> 1)) * g.nnx + 2 * ci + (n & 1));
          rv[n][0] = __ldg(rhs + o);
          rv[n][1] = __ldg(rhs + o + 1);
        }
        if (!g.th)
#pragma unroll
          for (int j = 0; j < 3; ++j) rp[j] = __ldg(rhs + (size_t)mu * g.nd + g.mv + 3 * (size_t)c + j);
      }
    }
    if (K1 > 1 && mu == 0) {  // the other nodes' planes (staging group 2) for the temporal mass
      cp_async_wait_group<0>();
      __syncthreads();
    }
    if (valid) {
      // + M_K sum_nu K_t[mu,nu] x_nu (slab.py:199-200)
      {
        const double* Krow = td.K_t + mu * K1;
        const double m = g.hx * g.hy;
#pragma unroll
        for (int jj = 0; jj < 3; ++jj) {  // source row jy'
          double xt[3][2];
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            double v0 = 0.0, v1 = 0.0;
#pragma unroll
            for (int nu = 0; nu < K1; ++nu) {
              const double2 f = XP[nu].at2(r0 + jj, c0 + i);
              v0 = fma(Krow[nu], f.x, v0);
              v1 = fma(Krow[nu], f.y, v1);
            }
            xt[i][0] = v0;
            xt[i][1] = v1;
          }
          double T1[3][2];
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int d = 0; d < 2; ++d)
              T1[i][d] = c_tab.M1[i][0] * xt[0][d] + c_tab.M1[i][1] * xt[1][d] + c_tab.M1[i][2] * xt[2][d];
#pragma unroll
          for (int jy = 0; jy < 3; ++jy) {
            const double mm = m * c_tab.M1[jy][jj];
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
              for (int d = 0; d < 2; ++d) ra[jy][i][d] += mm * T1[i][d];
          }
        }
      }
      // Pressure coupling (forms.py:589-603, the -p div w and -q div u terms):
      // P1disc x Q2 on a rectangle is separable, so the 16-point sums collapse
      // to 1-D Gauss sums (JTabs pA/pB/pM) and stay out of the volume loop.
      if (ds.pressure && !g.th) {  // Taylor-Hood: the pressure coupling is pdst_th.cu's
        const double WT = g.hx * g.hy * tw;
        cp_async_wait_group<0>();  // the own thread's copies (this node's; DG(0) has no wait on its second staging group)
        const double* pp = spres + (size_t)(PSTAGE ? mu : 0) * 3 * JNT + threadIdx.x;
        const double P0 = WT * pp[0], P1 = WT * pp[JNT], P2 = WT * pp[2 * JNT];
        // -q div u: rows of x_mu against the 1-D sums
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll
        for (int jy = 0; jy < 3; ++jy) {
          const double2 f0 = XM.at2(r0 + jy, c0), f1 = XM.at2(r0 + jy, c0 + 1), f2 = XM.at2(r0 + jy, c0 + 2);
          const double sA = T.pAx[0] * f0.x + T.pAx[1] * f1.x + T.pAx[2] * f2.x;   // sum_i A_i x0
          const double sB = T.pBx[0] * f0.x + T.pBx[1] * f1.x + T.pBx[2] * f2.x;   // sum_i Bx_i x0
          const double s0 = T.pM0[0] * f0.y + T.pM0[1] * f1.y + T.pM0[2] * f2.y;   // sum_i M0_i x1
          const double s1 = T.pM1[0] * f0.y + T.pM1[1] * f1.y + T.pM1[2] * f2.y;   // sum_i M1_i x1
          a0 += T.pM0[jy] * sA + T.pAy[jy] * s0;
          a1 += T.pM0[jy] * sB + T.pAy[jy] * s1;
          a2 += T.pM1[jy] * sA + T.pBy[jy] * s0;
        }
        accp[0] = -WT * a0;
        accp[1] = -WT * a1;
        accp[2] = -WT * a2;
        // -p div w
#pragma unroll
        for (int jy = 0; jy < 3; ++jy) {
          const double dy = P0 * T.pAy[jy] + P2 * T.pBy[jy], ey = P1 * T.pAy[jy];
#pragma unroll
          for (int ix = 0; ix < 3; ++ix) {
            const double cA = P0 * T.pAx[ix] + P1 * T.pBx[ix], cB = P2 * T.pAx[ix];
            ra[jy][ix][0] -= cA * T.pM0[jy] + cB * T.pM1[jy];
            ra[jy][ix][1] -= T.pM0[ix] * dy + T.pM1[ix] * ey;
          }
        }
      }
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          double2* sp = slot + (3 * a + b) * JNT;
          const double2 o = *sp;
          *sp = make_double2(o.x + ra[a][b][0], o.y + ra[a][b][1]);
        }
      const size_t o = (size_t)mu * g.nd + g.mv + 3 * (size_t)c;
      // boundary cells: raw sum, finished (side terms, rhs) by k_jac_post
      const bool bcell = ci == 0 || cj == 0 || ci == g.nx - 1 || cj == g.ny - 1;
      if (!g.th)
#pragma unroll
        for (int j = 0; j < 3; ++j) out[o + j] = (rhs && !bcell) ? rp[j] - accp[j] : accp[j];
    }
    TR(4 + 5 * mu);
    __syncthreads();
    TR(5 + 5 * mu);
    // node assembly: each cell writes the nodes it owns (lower-left 2x2 of its
    // 3x3 block, plus the right column / top row for the tile's last cells),
    // summing the <= 4 cells that contain a node in a fixed order.
    if (valid) {
      const size_t base = (size_t)mu * g.nd;
      const int me = ty * JT + tx;
      const bool hl = tx > 0, hd = ty > 0;
      // neighbour slots: left, down, down-left cell of this thread's cell
      const double2* sm_ = reinterpret_cast<const double2*>(sacc) + me;
      const double2* sl_ = sm_ - 1;
      const double2* sd_ = sm_ - JT;
      const double2* sld = sm_ - JT - 1;
      auto at = [&](const double2* p, int a, int d) {  // (the two components' loads of a node merge)
        const double2 v = p[a * JNT];
        return d == 0 ? v.x : v.y;
      };
      const bool oal = (reinterpret_cast<size_t>(out + base) & 15) == 0;
      // n = own-node index (lower-left 2x2, rhs preloaded) or -1 (tile edge row / column)
      auto emit = [&](int lx, int ly, double s0, double s1, int n) {
        const bool shx = (lx == 0 && i0 > 0) || (lx == 2 * JT && i0 + JT < g.nx);
        const bool shy = (ly == 0 && j0 > 0) || (ly == 2 * JT && j0 + JT < g.ny);
        if (shx || shy) {
          double* pp = part + (((size_t)mu * ntiles + tile) * JPER + perim(lx, ly)) * 2;
          *reinterpret_cast<double2*>(pp) = make_double2(s0, s1);
        } else {
          const size_t o = base + 2 * ((size_t)(2 * j0 + ly) * g.nnx + 2 * i0 + lx);
          if (rhs && !in_strip(g, 2 * i0 + lx, 2 * j0 + ly)) {  // strip nodes: k_jac_post
            s0 = (n >= 0 ? rv[n][0] : __ldg(rhs + o)) - s0;
            s1 = (n >= 0 ? rv[n][1] : __ldg(rhs + o + 1)) - s1;
          }
          if (oal) {  // both components of the node as one 16-byte store
            *reinterpret_cast<double2*>(out + o) = make_double2(s0, s1);
          } else {  // odd nd and an odd Radau node: the block is only 8-byte aligned
            out[o] = s0;
            out[o + 1] = s1;
          }
        }
      };
      const int lx = 2 * tx, ly = 2 * ty;
      // the cells sharing a node are summed in (row, column) order, lower first
      {  // node (0,0): cells down-left, down, left, self
        double s0 = 0.0, s1 = 0.0;
        if (hl && hd) { s0 += at(sld, 8, 0); s1 += at(sld, 8, 1); }
        if (hd) { s0 += at(sd_, 6, 0); s1 += at(sd_, 6, 1); }
        if (hl) { s0 += at(sl_, 2, 0); s1 += at(sl_, 2, 1); }
        s0 += at(sm_, 0, 0);
        s1 += at(sm_, 0, 1);
        emit(lx, ly, s0, s1, 0);
      }
      {  // (1,0): down, self
        double s0 = 0.0, s1 = 0.0;
        if (hd) { s0 += at(sd_, 7, 0); s1 += at(sd_, 7, 1); }
        s0 += at(sm_, 1, 0);
        s1 += at(sm_, 1, 1);
        emit(lx + 1, ly, s0, s1, 1);
      }
      {  // (0,1): left, self
        double s0 = 0.0, s1 = 0.0;
        if (hl) { s0 += at(sl_, 5, 0); s1 += at(sl_, 5, 1); }
        s0 += at(sm_, 3, 0);
        s1 += at(sm_, 3, 1);
        emit(lx, ly + 1, s0, s1, 2);
      }
      emit(lx + 1, ly + 1, 0.0 + at(sm_, 4, 0), 0.0 + at(sm_, 4, 1), 3);  // (1,1): self only
      if (lastx) {
        double s0 = 0.0, s1 = 0.0;  // (2,0): down, self
        if (hd) { s0 += at(sd_, 8, 0); s1 += at(sd_, 8, 1); }
        s0 += at(sm_, 2, 0);
        s1 += at(sm_, 2, 1);
        emit(lx + 2, ly, s0, s1, -1);
        emit(lx + 2, ly + 1, 0.0 + at(sm_, 5, 0), 0.0 + at(sm_, 5, 1), -1);
      }
      if (lasty) {
        double s0 = 0.0, s1 = 0.0;  // (0,2): left, self
        if (hl) { s0 += at(sl_, 8, 0); s1 += at(sl_, 8, 1); }
        s0 += at(sm_, 6, 0);
        s1 += at(sm_, 6, 1);
        emit(lx, ly + 2, s0, s1, -1);
        emit(lx + 1, ly + 2, 0.0 + at(sm_, 7, 0), 0.0 + at(sm_, 7, 1), -1);
        if (lastx) emit(lx + 2, ly + 2, 0.0 + at(sm_, 8, 0), 0.0 + at(sm_, 8, 1), -1);
      }
    }
    TR(6 + 5 * mu);  // (the barrier before the slots are rewritten is inside the next volume pass)
  }
  __syncthreads();
  tile_signal(done + K1 - 1);
  KTR(1);
  STEP_MARK(rhs ? 2 : 0, 2);
}

// ---------------------------------------------------------------------------
// Slab residual: R = tau w F(U) - [(K_t x M)V - (m_t x M) v_minus; 0]
// ---------------------------------------------------------------------------
template <int K1>
__global__ void __launch_bounds__(NT) k_residual(Geom g, TimeData td, Disc ds, Model m, Lin L,
                                                 const double* __restrict__ U, const double* __restrict__ advect,
                                                 const double* __restrict__ vminus, const double* __restrict__ fqp,
                                                 const double* __restrict__ ghat, double* __restrict__ out) {
  extern __shared__ double smem[];
  double* us = smem;                          // [K1][2][PLANE] state velocities
  double* vm = us + (size_t)K1 * 2 * PLANE;   // [2][PLANE] v_minus
  double* as = vm + 2 * PLANE;                // [2][PLANE] advect (if given)
  double* sacc = as + 2 * PLANE;              // [18][NT]
  double* fR = sacc + 18 * NT;
  double* fT = fR + 6 * NT;
  const bool cip = ds.convection && ds.gamma_cip > 0.0;
  const int i0 = blockIdx.x * TX, j0 = blockIdx.y * TY;
  const int X0 = 2 * (i0 - 2), Y0 = 2 * (j0 - 2);
  for (int nu = 0; nu < K1; ++nu)
    stage_velocity(g, U + (size_t)nu * g.nd, us + (size_t)nu * 2 * PLANE, us + (size_t)nu * 2 * PLANE + PLANE, X0,
                   Y0);
  stage_velocity(g, vminus, vm, vm + PLANE, X0, Y0);
  Plane2 UP[K1];
#pragma unroll
  for (int nu = 0; nu < K1; ++nu) UP[nu] = Plane2{us + nu * 2 * PLANE, us + nu * 2 * PLANE + PLANE};
  const Plane2 VM{vm, vm + PLANE};
  const Plane2 AP{as, as + PLANE};

  const int tx = threadIdx.x % CX, ty = threadIdx.x / CX;
  const int ci = i0 - 1 + tx, cj = j0 - 1 + ty;
  const bool valid = ci >= 0 && ci < g.nx && cj >= 0 && cj < g.ny;
  const bool owned = valid && tx >= 1 && ty >= 1;
  const int c = cj * g.nx + ci;
  const int r0 = 2 + 2 * ty, c0 = 2 + 2 * tx;
  const double W = g.hx * g.hy;

  // small meshes: one Radau node per CTA (grid.z = k+1), so the register-heavy
  // residual (1 CTA per SM) fills the waves more evenly; large ones loop over
  // the nodes with the state staged once
  const int mu_lo = gridDim.z > 1 ? (int)blockIdx.z : 0, mu_hi = gridDim.z > 1 ? (int)blockIdx.z + 1 : K1;
  for (int mu = mu_lo; mu < mu_hi; ++mu) {
    if (advect) stage_velocity(g, advect + (size_t)mu * g.nd, as, as + PLANE, X0, Y0);
    __syncthreads();
    // the node's planes by offset (indexing the plane array with the runtime mu
    // would place it in local memory)
    const Plane2 SP{us + mu * 2 * PLANE, us + mu * 2 * PLANE + PLANE};
    const Plane2 AW = advect ? AP : SP;
    double acc[3][3][2];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    double accp[3] = {0.0, 0.0, 0.0};
    if (valid) {
      double PI[3] = {0.0, 0.0, 0.0};
      if (!g.th) {  // Taylor-Hood: the pressure terms are pdst_th.cu's
        const double* pp = U + (size_t)mu * g.nd + g.mv + 3 * (size_t)c;
        PI[0] = __ldg(pp);
        PI[1] = __ldg(pp + 1);
        PI[2] = __ldg(pp + 2);
      }
#pragma unroll 1
      for (int qx = 0; qx < 4; ++qx) {
        double sB[3][2], sG[3][2];
#pragma unroll
        for (int jy = 0; jy < 3; ++jy) row_sums(SP, r0 + jy, c0, qx, sB[jy], sG[jy]);
        double Pa[3][2] = {{0, 0}, {0, 0}, {0, 0}}, Qa[3][2] = {{0, 0}, {0, 0}, {0, 0}};
        const double xh = c_tab.s[qx] - 0.5;
#pragma unroll
        for (int qy = 0; qy < 4; ++qy) {
          double v[2], vx[2], vy[2];
#pragma unroll
          for (int d = 0; d < 2; ++d) {
            v[d] = c_tab.B[qy][0] * sB[0][d] + c_tab.B[qy][1] * sB[1][d] + c_tab.B[qy][2] * sB[2][d];
            vx[d] = (c_tab.B[qy][0] * sG[0][d] + c_tab.B[qy][1] * sG[1][d] + c_tab.B[qy][2] * sG[2][d]) * g.ihx;
            vy[d] = (c_tab.G[qy][0] * sB[0][d] + c_tab.G[qy][1] * sB[1][d] + c_tab.G[qy][2] * sB[2][d]) * g.ihy;
          }
          const int q = 4 * qx + qy;
          const double wq = c_tab.w[qx] * c_tab.w[qy] * W;
          double Fx0 = 0, Fx1 = 0, Fy0 = 0, Fy1 = 0, Fv0 = 0, Fv1 = 0;
          if (fqp) {
            const size_t fi = (((size_t)mu * g.ncells + c) * 16 + q) * 2;
            Fv0 = __ldg(fqp + fi);
            Fv1 = __ldg(fqp + fi + 1);
          }
          if (ds.viscous) {
            const double a0 = vx[0], a1 = vy[1], a2 = 0.5 * (vy[0] + vx[1]);
            const double eta = eta_field(m, a0 * a0 + a1 * a1 + 2.0 * a2 * a2);
            Fx0 -= eta * a0;
            Fy1 -= eta * a1;
            Fx1 -= eta * a2;
            Fy0 -= eta * a2;
          }
          if (ds.convection) {
            Fx0 += v[0] * v[0];
            Fx1 += v[1] * v[0];
            Fy0 += v[0] * v[1];
            Fy1 += v[1] * v[1];
          }
          if (ds.pressure) {
            const double yh = c_tab.s[qy] - 0.5;
            const double pq = PI[0] + PI[1] * xh + PI[2] * yh;
            Fx0 += pq;
            Fy1 += pq;
            const double dv = wq * (vx[0] + vy[1]);
            accp[0] += dv;
            accp[1] += dv * xh;
            accp[2] += dv * yh;
          }
#pragma unroll
          for (int jy = 0; jy < 3; ++jy) {
            Pa[jy][0] = fma(wq * Fx0, c_tab.B[qy][jy], Pa[jy][0]);
            Pa[jy][1] = fma(wq * Fx1, c_tab.B[qy][jy], Pa[jy][1]);
            Qa[jy][0] = fma(wq * Fy0, c_tab.G[qy][jy] * g.ihy, fma(wq * Fv0, c_tab.B[qy][jy], Qa[jy][0]));
            Qa[jy][1] = fma(wq * Fy1, c_tab.G[qy][jy] * g.ihy, fma(wq * Fv1, c_tab.B[qy][jy], Qa[jy][1]));
          }
        }
#pragma unroll
        for (int jy = 0; jy < 3; ++jy)
#pragma unroll
          for (int ix = 0; ix < 3; ++ix)
#pragma unroll
            for (int d = 0; d < 2; ++d)
              acc[jy][ix][d] += (c_tab.G[qx][ix] * g.ihx) * Pa[jy][d] + c_tab.B[qx][ix] * Qa[jy][d];
      }
      if (cip) cip_own(g, ds, SP, AW, ci, cj, tx, ty, r0, c0, -1.0, fR, fT, RegAcc{acc});
    }
    // the cell's sums to its shared slot; the boundary sides (a noinline
    // call) add into the slot, so the register accumulators never need an
    // address (no local-memory copy of acc)
    double* slot = sacc + threadIdx.x;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        slot[(2 * (3 * a + b)) * NT] = acc[a][b][0];
        slot[(2 * (3 * a + b) + 1) * NT] = acc[a][b][1];
      }
    if (valid && (ci == 0 || cj == 0 || ci == g.nx - 1 || cj == g.ny - 1)) {
      double PI[3] = {0.0, 0.0, 0.0};
      if (!g.th) {  // Taylor-Hood: the pressure terms are pdst_th.cu's
        const double* pp = U + (size_t)mu * g.nd + g.mv + 3 * (size_t)c;
        PI[0] = __ldg(pp);
        PI[1] = __ldg(pp + 1);
        PI[2] = __ldg(pp + 2);
      }
      double gn[18];
#pragma unroll
      for (int a = 0; a < 9; ++a) {
        const size_t node = (size_t)(2 * cj + a / 3) * g.nnx + 2 * ci + a % 3;
        gn[2 * a] = ghat ? ghat[2 * node] : 0.0;
        gn[2 * a + 1] = ghat ? ghat[2 * node + 1] : 0.0;
      }
      const bool gp = ghat != nullptr;
      const SmemAccN<NT> sa{slot};
      if (cj == 0) res_boundary_side(g, ds, m, L, 0, side_offset(g, 0) + ci, SP, AW, r0, c0, PI, gn, gp, sa, accp);
      if (ci == g.nx - 1) res_boundary_side(g, ds, m, L, 1, side_offset(g, 1) + cj, SP, AW, r0, c0, PI, gn, gp, sa, accp);
      if (cj == g.ny - 1) res_boundary_side(g, ds, m, L, 2, side_offset(g, 2) + ci, SP, AW, r0, c0, PI, gn, gp, sa, accp);
      if (ci == 0) res_boundary_side(g, ds, m, L, 3, side_offset(g, 3) + cj, SP, AW, r0, c0, PI, gn, gp, sa, accp);
    }
    __syncthreads();
    if (valid) {
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          acc[a][b][0] = slot[(2 * (3 * a + b)) * NT];
          acc[a][b][1] = slot[(2 * (3 * a + b) + 1) * NT];
        }
      if (cip) cip_received(g, ci, cj, tx, ty, -1.0, fR, fT, RegAcc{acc});
      const double tw = td.tau_w[mu];
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          acc[a][b][0] *= tw;
          acc[a][b][1] *= tw;
        }
      add_mass<K1>(UP, &VM, td.m_t[mu], td.K_t + mu * K1, r0, c0, -W, RegAcc{acc});
      if (owned && !g.th) {
        const size_t o = (size_t)mu * g.nd + g.mv + 3 * (size_t)c;
#pragma unroll
        for (int j = 0; j < 3; ++j) out[o + j] = tw * accp[j];
      }
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          slot[(2 * (3 * a + b)) * NT] = acc[a][b][0];
          slot[(2 * (3 * a + b) + 1) * NT] = acc[a][b][1];
        }
    }
    __syncthreads();
    assemble_and_store(g, sacc, i0, j0, mu, nullptr, out);
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Linearization caches (forms.py:544-571): per cell qp (eta, gamma), per
// boundary face qp (eta_f, gamma_f), lifting coefficients (eta_d, beta_d, Dg).
// ---------------------------------------------------------------------------
__global__ void k_linearize_cells(Geom g, Model m, int k1, const double* __restrict__ state, double* __restrict__ eta,
                                  double* __restrict__ gam) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int mu = blockIdx.y;
  if (c >= g.ncells || mu >= k1) return;
  const int ci = c % g.nx, cj = c / g.nx;
  const double* sv = state + (size_t)mu * g.mv;
  double S[3][3][2];
#pragma unroll
  for (int jy = 0; jy < 3; ++jy)
#pragma unroll
    for (int ix = 0; ix < 3; ++ix) {
      const size_t node = (size_t)(2 * cj + jy) * g.nnx + 2 * ci + ix;
      const double2 v = __ldg(reinterpret_cast<const double2*>(sv) + node);
      S[jy][ix][0] = v.x;
      S[jy][ix][1] = v.y;
    }
  for (int qx = 0; qx < 4; ++qx) {
    double sB[3][2], sG[3][2];
#pragma unroll
    for (int jy = 0; jy < 3; ++jy)
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        sB[jy][d] = c_tab.B[qx][0] * S[jy][0][d] + c_tab.B[qx][1] * S[jy][1][d] + c_tab.B[qx][2] * S[jy][2][d];
        sG[jy][d] = c_tab.G[qx][0] * S[jy][0][d] + c_tab.G[qx][1] * S[jy][1][d] + c_tab.G[qx][2] * S[jy][2][d];
      }
    for (int qy = 0; qy < 4; ++qy) {
      double vx[2], vy[2];
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        vx[d] = (c_tab.B[qy][0] * sG[0][d] + c_tab.B[qy][1] * sG[1][d] + c_tab.B[qy][2] * sG[2][d]) * g.ihx;
        vy[d] = (c_tab.G[qy][0] * sB[0][d] + c_tab.G[qy][1] * sB[1][d] + c_tab.G[qy][2] * sB[2][d]) * g.ihy;
      }
      const double a0 = vx[0], a1 = vy[1], a2 = 0.5 * (vy[0] + vx[1]);
      double e, gm;
      tangent_coeffs(m, a0 * a0 + a1 * a1 + 2.0 * a2 * a2, e, gm);
      const size_t o = ((size_t)mu * g.ncells + c) * 16 + 4 * qx + qy;
      eta[o] = e;
      gam[o] = gm;
    }
  }
}

// Sym gradient of a nodal field on boundary face bf at face point q.
__device__ void face_symgrad(const Geom& g, const double* __restrict__ v, int bf, int q, double& a0, double& a1,
                             double& a2) {
  int side = 0;
  while (side < 3 && bf >= side_offset(g, side + 1)) ++side;
  const int f = bf - side_offset(g, side);
  int ci, cj;
  if (side == 0) { ci = f; cj = 0; }
  else if (side == 1) { ci = g.nx - 1; cj = f; }
  else if (side == 2) { ci = f; cj = g.ny - 1; }
  else { ci = 0; cj = f; }
  const int axis = (side == 1 || side == 3) ? 0 : 1;
  const int e = (side == 1 || side == 2) ? 1 : 0;
  const double ihtan = axis == 0 ? g.ihy : g.ihx, ihnorm = axis == 0 ? g.ihx : g.ihy;
  double ux[2], uy[2];
  for (int d = 0; d < 2; ++d) {
    double dt = 0.0, dn = 0.0;
    for (int t = 0; t < 3; ++t) {
      double le = 0.0, ld = 0.0;
      for (int n = 0; n < 3; ++n) {
        const int jy = axis == 0 ? t : n, ix = axis == 0 ? n : t;
        const double val = v[2 * ((size_t)(2 * cj + jy) * g.nnx + 2 * ci + ix) + d];
        le = fma(c_tab.E[e][n], val, le);
        ld = fma(c_tab.dE[e][n], val, ld);
      }
      dt = fma(c_tab.G[q][t], le, dt);
      dn = fma(c_tab.B[q][t], ld, dn);
    }
    if (axis == 0) {
      ux[d] = dn * ihnorm;
      uy[d] = dt * ihtan;
    } else {
      ux[d] = dt * ihtan;
      uy[d] = dn * ihnorm;
    }
  }
  a0 = ux[0];
  a1 = uy[1];
  a2 = 0.5 * (uy[0] + ux[1]);
}

__global__ void k_linearize_faces(Geom g, Model m, int k1, const double* __restrict__ state, double* __restrict__ etaf,
                                  double* __restrict__ gamf) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;  // bf*4 + q
  const int mu = blockIdx.y;
  if (t >= g.nbf * 4 || mu >= k1) return;
  const int bf = t / 4, q = t % 4;
  double a0, a1, a2;
  face_symgrad(g, state + (size_t)mu * g.mv, bf, q, a0, a1, a2);
  double e, gm;
  tangent_coeffs(m, a0 * a0 + a1 * a1 + 2.0 * a2 * a2, e, gm);
  etaf[(size_t)mu * g.nbf * 4 + t] = e;
  gamf[(size_t)mu * g.nbf * 4 + t] = gm;
}

__global__ void k_lifting(Geom g, Model m, const double* __restrict__ ghat, double* __restrict__ etad,
                          double* __restrict__ betad, double* __restrict__ dg) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= g.nbf * 4) return;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  if (ghat) face_symgrad(g, ghat, t / 4, t % 4, a0, a1, a2);
  const double a_sq = a0 * a0 + a1 * a1 + 2.0 * a2 * a2;
  etad[t] = eta_field(m, a_sq);
  betad[t] = beta_field(m, a_sq);
  dg[3 * t] = a0;
  dg[3 * t + 1] = a1;
  dg[3 * t + 2] = a2;
}

// ---------------------------------------------------------------------------
// Element matrices by applying the cell-local action to unit vectors, so the
// assembled blocks agree with the matrix-free action to rounding (the
// property of forms.py:519-525).  ET[c][j][i] = E_c[i][j] (column-major per
// cell), local dofs i = 2a + d (a = 3 jy + ix) then 18 + pressure j.
// ---------------------------------------------------------------------------
struct UnitAcc {
  int r, c, d;
  __device__ double at(int dd, int rr, int cc) const { return (dd == d && rr == r && cc == c) ? 1.0 : 0.0; }
};

struct GlobAcc {
  const double* v;
  int nnx, X0, Y0;
  __device__ double at(int d, int r, int c) const { return __ldg(v + 2 * ((size_t)(Y0 + r) * nnx + X0 + c) + d); }
};

// Apply cache of the current linearization (layout at APC_SLOTS).  One
// thread per (cell, Radau node); the quantities and their arithmetic follow
// jac_volume (state value / sym gradient at the volume points, cached eta /
// gamma) and cip_face (|v_L . n| on the left / lower trace).
__global__ void __launch_bounds__(JNT) k_apply_cache(Geom g, TimeData td, Disc ds, Lin L, int k1,
                                                     const double* __restrict__ state, double* __restrict__ apc) {
  const int bx = blockIdx.x, by = blockIdx.y, mu = blockIdx.z;
  const size_t tile = (size_t)by * jac_tiles_x(g) + bx;
  const int tx = threadIdx.x % JT, ty = threadIdx.x / JT;
  const int ci = bx * JT + tx, cj = by * JT + ty;
  double* cp = apc + (tile * k1 + mu) * APC_SLOTS * JNT + threadIdx.x;
  if (ci >= g.nx || cj >= g.ny) {
    for (int s = 0; s < APC_SLOTS; ++s) cp[(size_t)s * JNT] = 0.0;
    return;
  }
  const int c = cj * g.nx + ci;
  const double tw = td.tau_w[mu];
  const double W = g.hx * g.hy * tw;
  const double* sv = state + (size_t)mu * g.mv;
  const GlobAcc S{sv, g.nnx, 2 * ci, 2 * cj};
  const bool vis = ds.viscous, hg = L.has_gamma && ds.viscous, conv = ds.convection;
  for (int qx = 0; qx < 4; ++qx) {
    double sB[3][2], sG[3][2];
#pragma unroll
    for (int jy = 0; jy < 3; ++jy) row_sums(S, jy, 0, qx, sB[jy], sG[jy]);
#pragma unroll
    for (int qy = 0; qy < 4; ++qy) {
      double v[2], vx[2], vy[2];
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        v[d] = c_tab.B[qy][0] * sB[0][d] + c_tab.B[qy][1] * sB[1][d] + c_tab.B[qy][2] * sB[2][d];
        vx[d] = (c_tab.B[qy][0] * sG[0][d] + c_tab.B[qy][1] * sG[1][d] + c_tab.B[qy][2] * sG[2][d]) * g.ihx;
        vy[d] = (c_tab.G[qy][0] * sB[0][d] + c_tab.G[qy][1] * sB[1][d] + c_tab.G[qy][2] * sB[2][d]) * g.ihy;
      }
      const size_t o = ((size_t)mu * g.ncells + c) * 16 + 4 * qx + qy;
      const double eta = vis ? L.eta[o] : 0.0;
      const double gam = hg ? L.gam[o] : 0.0;
      const double wq = c_tab.w[qx] * c_tab.w[qy] * W;
      const double sg = sqrt(-(wq * gam));  // gamma <= 0 (p <= 2); NaN propagates
      const double a0 = vx[0], a1 = vy[1], a2 = 0.5 * (vy[0] + vx[1]);
      double* cq = cp + (size_t)qx * 24 * JNT + qy * JNT;
      cq[0 * 4 * JNT] = wq * eta;
      cq[1 * 4 * JNT] = sg * a0;
      cq[2 * 4 * JNT] = sg * a1;
      cq[3 * 4 * JNT] = sg * a2;
      cq[4 * 4 * JNT] = conv ? wq * v[0] : 0.0;
      cq[5 * 4 * JNT] = conv ? wq * v[1] : 0.0;
    }
  }
  // CIP face matrices of the right and top faces (this cell is the left /
  // lower one, whose trace gives the weight); zero where not interior.
  const bool cip = ds.convection && ds.gamma_cip > 0.0;
  for (int f = 0; f < 2; ++f) {
    const int axis = f;
    const bool has = f == 0 ? ci < g.nx - 1 : cj < g.ny - 1;
    double* wp = cp + (size_t)(APC_VOL + 6 * f) * JNT;
    double W[6] = {0, 0, 0, 0, 0, 0};
    if (has && cip) {
      const double hface = axis == 0 ? g.hy : g.hx;
      const double ihn = axis == 0 ? g.ihx : g.ihy;
      double tr[3];
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        double v = 0.0;
#pragma unroll
        for (int n = 0; n < 3; ++n) v = fma(c_tab.E[1][n], axis == 0 ? S.at(0, t, n) : S.at(1, n, t), v);
        tr[t] = v;
      }
      const double coef = tw * ds.gamma_cip * hface * hface * (ihn * ihn);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        double vt = 0.0;
#pragma unroll
        for (int t = 0; t < 3; ++t) vt = fma(c_tab.B[q][t], tr[t], vt);
        const double wq = coef * (c_tab.w[q] * hface) * fabs(vt);
        W[0] += wq * c_tab.B[q][0] * c_tab.B[q][0];
        W[1] += wq * c_tab.B[q][0] * c_tab.B[q][1];
        W[2] += wq * c_tab.B[q][0] * c_tab.B[q][2];
        W[3] += wq * c_tab.B[q][1] * c_tab.B[q][1];
        W[4] += wq * c_tab.B[q][1] * c_tab.B[q][2];
        W[5] += wq * c_tab.B[q][2] * c_tab.B[q][2];
      }
    }
#pragma unroll
    for (int e = 0; e < 6; ++e) wp[e * JNT] = W[e];
  }
}

__global__ void __launch_bounds__(128) k_element_matrices(Geom g, Disc ds, Lin L, int mu, const double* __restrict__ state,
                                                          double* __restrict__ ET) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t c = t / 21;
  const int j = (int)(t % 21);
  if (c >= (size_t)g.ncells) return;
  const int ci = (int)(c % g.nx), cj = (int)(c / g.nx);
  const GlobAcc S{state, g.nnx, 2 * ci, 2 * cj};
  double P[3] = {0.0, 0.0, 0.0};
  UnitAcc X{-1, -1, -1};
  if (j < 18) {
    X.r = (j / 2) / 3;
    X.c = (j / 2) % 3;
    X.d = j % 2;
  } else {
    P[j - 18] = 1.0;
  }
  double acc[3][3][2];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  double accp[3] = {0.0, 0.0, 0.0};
  jac_volume(g, ds, L, mu, (int)c, X, S, 0, 0, P, RegAcc{acc}, accp);
  jac_sides(g, ds, L, mu, ci, cj, X, S, 0, 0, P, RegAcc{acc}, accp);
  double* out = ET + (c * 21 + j) * 21;
#pragma unroll
  for (int a = 0; a < 9; ++a) {
    out[2 * a] = acc[a / 3][a % 3][0];
    out[2 * a + 1] = acc[a / 3][a % 3][1];
  }
  out[18] = accp[0];
  out[19] = accp[1];
  out[20] = accp[2];
}

// Boundary-side matrices of the linearization: column j of side bf is the
// side terms of forms.py:605-637 applied to the local unit vector j.  The apply
// then does one 21x21 mat-vec per boundary side instead of the face evaluation.
__global__ void __launch_bounds__(128) k_boundary_matrices(Geom g, Disc ds, Lin L, int k1,
                                                           const double* __restrict__ state,
                                                           double* __restrict__ bmat) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int mu = blockIdx.y;
  const int bf = (int)(t / 21), j = (int)(t % 21);
  if (bf >= g.nbf || mu >= k1) return;
  int side = 0;
  while (side < 3 && bf >= side_offset(g, side + 1)) ++side;
  const int f = bf - side_offset(g, side);
  int ci, cj;
  if (side == 0) { ci = f; cj = 0; }
  else if (side == 1) { ci = g.nx - 1; cj = f; }
  else if (side == 2) { ci = f; cj = g.ny - 1; }
  else { ci = 0; cj = f; }
  const GlobAcc S{state + (size_t)mu * g.mv, g.nnx, 2 * ci, 2 * cj};
  double P[3] = {0.0, 0.0, 0.0};
  UnitAcc X{-1, -1, -1};
  if (j < 18) {
    X.r = (j / 2) / 3;
    X.c = (j / 2) % 3;
    X.d = j % 2;
  } else {
    P[j - 18] = 1.0;
  }
  double acc[3][3][2];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  double accp[3] = {0.0, 0.0, 0.0};
  jac_boundary_side(g, ds, L, mu, side, bf, X, S, 0, 0, P, RegAcc{acc}, accp, 1.0);
  // column-major [mu][bf][col][row]: this thread's column is contiguous, and the
  // side products' lanes (one row each) read consecutive doubles per column
  double* col = bmat + ((size_t)mu * g.nbf + bf) * 441 + (size_t)j * 21;
  for (int a = 0; a < 9; ++a) {
    col[2 * a] = acc[a / 3][a % 3][0];
    col[2 * a + 1] = acc[a / 3][a % 3][1];
  }
  for (int r = 0; r < 3; ++r) col[18 + r] = accp[r];
}

template <int K1>
size_t jac_smem() {
  return ((size_t)2 * K1 * JPLANE + (size_t)JNT * (18 + (jac_pstage(K1) ? 3 * K1 : 3))) * sizeof(double);
}
template <int K1>
size_t res_smem() {
  return ((size_t)K1 * 2 * PLANE + 4 * PLANE + (size_t)NT * 30) * sizeof(double);
}

template <int K1>
cudaError_t launch_jac(const Geom& g, const TimeData& td, const Disc& ds, const Lin& L, const double* x,
                       const double* rhs, double* out, double* part, cudaStream_t st) {
  static DeviceOnce once;
  const size_t sm = jac_smem<K1>();
  const int dev = current_device();
  if (!once.done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_jacobian<K1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_jacobian<K1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    once.done[dev] = true;
  }
  if (!L.bmat || !L.apc) return cudaErrorInvalidValue;  // built by pdst_linearize
  dim3 grid(jac_tiles_x(g), jac_tiles_y(g));
  cudaError_t e;
  JTabs T;
  {
    static const Tables tab = host_tables();
    for (int q = 0; q < 4; ++q) {
      for (int i = 0; i < 3; ++i) {
        T.B[q][i] = tab.B[q][i];
        T.Gx[q][i] = tab.G[q][i] * g.ihx;
        T.Gy[q][i] = tab.G[q][i] * g.ihy;
      }
      T.w[q] = tab.w[q];
      T.xh[q] = tab.s[q] - 0.5;
      T.wyh[q] = tab.w[q] * (tab.s[q] - 0.5);
    }
    for (int i = 0; i < 3; ++i) {
      double a = 0.0, b = 0.0, m0 = 0.0, m1 = 0.0;
      for (int q = 0; q < 4; ++q) {
        a += tab.w[q] * tab.G[q][i];
        b += tab.w[q] * (tab.s[q] - 0.5) * tab.G[q][i];
        m0 += tab.w[q] * tab.B[q][i];
        m1 += tab.w[q] * (tab.s[q] - 0.5) * tab.B[q][i];
      }
      T.pAx[i] = a * g.ihx;
      T.pAy[i] = a * g.ihy;
      T.pBx[i] = b * g.ihx;
      T.pBy[i] = b * g.ihy;
      T.pM0[i] = m0;
      T.pM1[i] = m1;
    }
    T.cJ[0] = tab.dE[1][0];
    T.cJ[1] = tab.dE[1][1];
    T.cJ[2] = tab.dE[1][2] - tab.dE[0][0];
    T.cJ[3] = -tab.dE[0][1];
    T.cJ[4] = -tab.dE[0][2];
  }
  const size_t ncb = n_bcells(g);
  const size_t ntiles = (size_t)jac_tiles_x(g) * jac_tiles_y(g);
  double* sp = part + (size_t)K1 * ntiles * JPER * 2;
  // completion counters behind the side products (zero in a fresh scratch)
  unsigned long long* done = reinterpret_cast<unsigned long long*>(sp + (size_t)K1 * 21 * ncb);
  const dim3 sgrid((unsigned)((ncb + 3) / 4), K1);
  const unsigned long long target = ntiles, starget = (unsigned long long)sgrid.x * sgrid.y;
  if (L.has_gamma && ds.viscous)
    PDST_LAUNCH(e = launch_pdl(k_jacobian<K1, true>, grid, dim3(JNT), sm, st, g, td, ds, L, x, rhs, out, part, done, T));
  else  // Picard (or no viscous term): the tangent's a~ slots are zeros, not streamed
    PDST_LAUNCH(e = launch_pdl(k_jacobian<K1, false>, grid, dim3(JNT), sm, st, g, td, ds, L, x, rhs, out, part, done, T));
  if (e != cudaSuccess) return e;
  {
    // tile pass -> side products (overlapping it, then waiting for it) -> epilogue
    PDST_LAUNCH(e = launch_pdl(k_side_products, sgrid, dim3(128), 0, st, g, td, (const double*)L.bmat, x, sp, done + 4));
    if (e != cudaSuccess) return e;
  }
  {
    const size_t n = jac_post_items(g);
    dim3 pg((unsigned)((n + 127) / 128), K1);
    PDST_LAUNCH(e = launch_pdl(k_jac_post, pg, dim3(128), 0, st, g, td, (const double*)part, (const double*)sp, rhs, out,
                               (const unsigned long long*)done, target, starget));
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

template <int K1>
cudaError_t launch_res(const Geom& g, const TimeData& td, const Disc& ds, const Model& m, const Lin& L,
                       const double* U, const double* advect, const double* vminus, const double* fqp,
                       const double* ghat, double* out, cudaStream_t st) {
  static DeviceOnce once;
  const size_t sm = res_smem<K1>();
  const int dev = current_device();
  if (!once.done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_residual<K1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    once.nsm[dev] = device_sms(dev);
    once.done[dev] = true;
  }
  const unsigned tiles = (unsigned)(((g.nx + TX - 1) / TX) * ((g.ny + TY - 1) / TY));
  dim3 grid((g.nx + TX - 1) / TX, (g.ny + TY - 1) / TY, tiles < 8u * (unsigned)once.nsm[dev] ? K1 : 1);
  PDST_LAUNCH(k_residual<K1><<<grid, NT, sm, st>>>(g, td, ds, m, L, U, advect, vminus, fqp, ghat, out));
  return cudaGetLastError();
}

}  // namespace

#ifdef PDST_TRACE
extern "C" int pdst_debug_trace(unsigned long long* out, int n) {
  cudaError_t e = cudaMemcpyFromSymbol(out, g_trace, (size_t)n * 16 * sizeof(unsigned long long));
  if (e == cudaSuccess && n >= 8192) {  // the kernel marks ride in the last row, then reset
    e = cudaMemcpyFromSymbol(out + (size_t)8191 * 16, g_ktrace, sizeof(g_ktrace));
    const unsigned long long init[8] = {~0ull, 0ull, ~0ull, 0ull, ~0ull, 0ull, ~0ull, 0ull};
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_ktrace, init, sizeof(init));
    // the step timeline rides in the two rows before, then resets (min slots to ~0, max slots to 0)
    if (e == cudaSuccess) e = cudaMemcpyFromSymbol(out + (size_t)8189 * 16, g_steptrace, sizeof(g_steptrace));
    unsigned long long sinit[32];
    for (int i = 0; i < 32; ++i) sinit[i] = (i % 4 == 2) ? 0ull : ~0ull;
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_steptrace, sinit, sizeof(sinit));
  }
  return (int)e;
}
#endif

cudaError_t set_tables(const Tables& t) { return cudaMemcpyToSymbol(c_tab, &t, sizeof(Tables)); }

size_t jacobian_scratch(const Geom& g, int k1) {
  // tile partials, then the boundary cells' side products, then the completion counters (4 nodes, side products)
  return (size_t)k1 * jac_tiles_x(g) * jac_tiles_y(g) * JPER * 2 + (size_t)k1 * 21 * n_bcells(g) + 8;
}

cudaError_t jacobian_reset_counters(const Geom& g, int k1, double* part, cudaStream_t st) {
  // the 8 trailing words of the scratch (every completed apply leaves them at zero; an apply cut
  // short by a device error would not)
  return cudaMemsetAsync(part + jacobian_scratch(g, k1) - 8, 0, 8 * sizeof(double), st);
}

cudaError_t jacobian_apply(const Geom& g, const TimeData& td, const Disc& ds, const Lin& L, const double* x,
                           const double* rhs, double* out, double* part, cudaStream_t st) {
  switch (td.k1) {
    case 1: return launch_jac<1>(g, td, ds, L, x, rhs, out, part, st);
    case 2: return launch_jac<2>(g, td, ds, L, x, rhs, out, part, st);
    case 3: return launch_jac<3>(g, td, ds, L, x, rhs, out, part, st);
    case 4: return launch_jac<4>(g, td, ds, L, x, rhs, out, part, st);
    default: return cudaErrorNotSupported;
  }
}

cudaError_t slab_residual(const Geom& g, const TimeData& td, const Disc& ds, const Model& m, const Lin& L,
                          const double* U, const double* advect, const double* vminus, const double* fqp,
                          const double* ghat, double* out, cudaStream_t st) {
  switch (td.k1) {
    case 1: return launch_res<1>(g, td, ds, m, L, U, advect, vminus, fqp, ghat, out, st);
    case 2: return launch_res<2>(g, td, ds, m, L, U, advect, vminus, fqp, ghat, out, st);
    case 3: return launch_res<3>(g, td, ds, m, L, U, advect, vminus, fqp, ghat, out, st);
    case 4: return launch_res<4>(g, td, ds, m, L, U, advect, vminus, fqp, ghat, out, st);
    default: return cudaErrorNotSupported;
  }
}

cudaError_t linearize(const Geom& g, const Model& m, int k1, const double* state, double* eta, double* gam,
                      double* etaf, double* gamf, cudaStream_t st) {
  dim3 gc((g.ncells + 127) / 128, k1);
  PDST_LAUNCH(k_linearize_cells<<<gc, 128, 0, st>>>(g, m, k1, state, eta, gam));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  dim3 gf((g.nbf * 4 + 127) / 128, k1);
  PDST_LAUNCH(k_linearize_faces<<<gf, 128, 0, st>>>(g, m, k1, state, etaf, gamf));
  return cudaGetLastError();
}

size_t apply_cache_size(const Geom& g, int k1) {
  return (size_t)jac_tiles_x(g) * jac_tiles_y(g) * k1 * APC_SLOTS * JNT;
}

cudaError_t apply_cache(const Geom& g, const TimeData& td, const Disc& ds, const Lin& L, const double* state,
                        double* apc, cudaStream_t st) {
  dim3 grid(jac_tiles_x(g), jac_tiles_y(g), td.k1);
  PDST_LAUNCH(k_apply_cache<<<grid, JNT, 0, st>>>(g, td, ds, L, td.k1, state, apc));
  return cudaGetLastError();
}

cudaError_t element_matrices(const Geom& g, const Disc& ds, const Lin& L, int mu, const double* state, double* ET,
                             cudaStream_t st) {
  const size_t n = (size_t)g.ncells * 21;
  PDST_LAUNCH(k_element_matrices<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(g, ds, L, mu, state, ET));
  return cudaGetLastError();
}

cudaError_t boundary_matrices(const Geom& g, const Disc& ds, const Lin& L, int k1, const double* state, double* bmat,
                              cudaStream_t st) {
  const size_t n = (size_t)g.nbf * 21;
  PDST_LAUNCH(k_boundary_matrices<<<dim3((unsigned)((n + 127) / 128), k1), 128, 0, st>>>(g, ds, L, k1, state, bmat));
  return cudaGetLastError();
}

cudaError_t lifting(const Geom& g, const Model& m, const double* ghat, double* etad, double* betad, double* dg,
                    cudaStream_t st) {
  PDST_LAUNCH(k_lifting<<<(g.nbf * 4 + 127) / 128, 128, 0, st>>>(g, m, ghat, etad, betad, dg));
  return cudaGetLastError();
}

}  // namespace pdst
