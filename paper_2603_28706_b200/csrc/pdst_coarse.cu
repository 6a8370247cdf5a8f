// pdst_coarse.cu — multigrid levels: grid transfers, Galerkin coarse
// operators in element form, coarse level apply, coarse patches and the
// coarsest-level dense solve (sm_100a, fp64).
//
// Reference (file:line into /root/reference/pkg/src/pdflow):
//   transfer_build (Q2 nodal interpolation, P1disc child rewrite)  solver/multigrid.py:90-154
//   _restrict / _prolong (per Radau node)                           solver/multigrid.py:523-543
//   coarse_operator (Galerkin P' J P per node)                       solver/multigrid.py:302-324
//   coarse mass P_v' M P_v                                           solver/multigrid.py:459-460
//   _sparse_level_matvec                                             solver/multigrid.py:234-248
//   _build_coarse_solver (dense, pressure pinning) / vcycle          solver/multigrid.py:494-578
//
// Element form of a level operator (per Radau node mu):
//   ecell[mu][c][i][j]            21x21 cell block (volume + boundary, plus the
//                                  CIP couplings of fine faces interior to c)
//   fv[mu][fj*(nx-1)+fi][sA][sB][a][b]  vertical face (fi,fj)|(fi+1,fj): 9x9 node
//   fh[mu][fj*nx+fi][sA][sB][a][b]      horizontal face (fi,fj)|(fi,fj+1) blocks,
//                                  identity in the velocity component (I2).
// Because the fine values of a child cell depend only on its parent's 9
// coarse nodes / 3 pressure coefficients, P' J P is exactly the sum of the
// children's P_K' E_K P_K plus the face blocks mapped the same way.  The
// coarse mass is the coarse Q2 mass (exact for nested spaces).
#include <cuda_runtime.h>

#include "pdst_coarse.h"
#include "pdst_device.cuh"

namespace pdst {
namespace {

__device__ __forceinline__ double lag(int i, double x) {
  return i == 0 ? (1.0 - x) * (1.0 - 2.0 * x) : i == 1 ? 4.0 * x * (1.0 - x) : x * (2.0 * x - 1.0);
}

__device__ __forceinline__ double m1g(int X, int Xp, int n) {
  double s = 0.0;
  const int lo = max(0, (max(X, Xp) - 1) / 2);
  for (int c = lo; c <= min(X, Xp) / 2 && c < n; ++c) {
    const int a = X - 2 * c, b = Xp - 2 * c;
    if (a >= 0 && a <= 2 && b >= 0 && b <= 2) s += c_tab.M1[a][b];
  }
  return s;
}

// ---------------------------------------------------------------------------
// Transfers (multigrid.py:90-154): fine node (X, Y) of the half-cell grid lies
// in coarse cell (min(X/4, ncx-1), min(Y/4, ncy-1)) at local coordinate X/4 - cx.
// ---------------------------------------------------------------------------
__global__ void k_prolong(Geom gc, Geom gf, int k1, const double* __restrict__ ec, double* __restrict__ ef) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int mu = blockIdx.y;
  const size_t nnf = (size_t)gf.nnx * gf.nny;
  const double* e = ec + (size_t)mu * gc.nd;
  double* o = ef + (size_t)mu * gf.nd;
  if (t < nnf) {
    const int X = (int)(t % gf.nnx), Y = (int)(t / gf.nnx);
    const int cx = min(X / 4, gc.nx - 1), cy = min(Y / 4, gc.ny - 1);
    const double xi = X / 4.0 - cx, eta = Y / 4.0 - cy;
    double s0 = 0.0, s1 = 0.0;
    for (int jy = 0; jy < 3; ++jy) {
      const double ly = lag(jy, eta);
      if (ly == 0.0) continue;
      for (int jx = 0; jx < 3; ++jx) {
        const double w = ly * lag(jx, xi);
        if (w == 0.0) continue;
        const size_t node = (size_t)(2 * cy + jy) * gc.nnx + 2 * cx + jx;
        s0 += w * e[2 * node];
        s1 += w * e[2 * node + 1];
      }
    }
    o[2 * t] = s0;
    o[2 * t + 1] = s1;
  } else if (t < nnf + (size_t)gf.ncells) {
    const int cf = (int)(t - nnf);
    const int fi = cf % gf.nx, fj = cf / gf.nx;
    const int ox = fi & 1, oy = fj & 1;
    const int c = (fj >> 1) * gc.nx + (fi >> 1);
    const double* pc = e + gc.mv + 3 * (size_t)c;
    double* pf = o + gf.mv + 3 * (size_t)cf;
    pf[0] = pc[0] + (2 * ox - 1) / 4.0 * pc[1] + (2 * oy - 1) / 4.0 * pc[2];
    pf[1] = 0.5 * pc[1];
    pf[2] = 0.5 * pc[2];
  }
}

__global__ void k_restrict(Geom gc, Geom gf, int k1, const double* __restrict__ rf, double* __restrict__ rc) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int mu = blockIdx.y;
  const size_t nnc = (size_t)gc.nnx * gc.nny;
  const double* r = rf + (size_t)mu * gf.nd;
  double* o = rc + (size_t)mu * gc.nd;
  if (t < nnc) {
    const int Xc = (int)(t % gc.nnx), Yc = (int)(t / gc.nnx);
    double s0 = 0.0, s1 = 0.0;
    for (int Y = max(0, 2 * Yc - 4); Y <= min(gf.nny - 1, 2 * Yc + 4); ++Y) {
      const int cy = min(Y / 4, gc.ny - 1), my = Yc - 2 * cy;
      if (my < 0 || my > 2) continue;
      const double wy = lag(my, Y / 4.0 - cy);
      if (wy == 0.0) continue;
      for (int X = max(0, 2 * Xc - 4); X <= min(gf.nnx - 1, 2 * Xc + 4); ++X) {
        const int cx = min(X / 4, gc.nx - 1), mx = Xc - 2 * cx;
        if (mx < 0 || mx > 2) continue;
        const double w = wy * lag(mx, X / 4.0 - cx);
        if (w == 0.0) continue;
        const size_t node = (size_t)Y * gf.nnx + X;
        s0 += w * r[2 * node];
        s1 += w * r[2 * node + 1];
      }
    }
    o[2 * t] = s0;
    o[2 * t + 1] = s1;
  } else if (t < nnc + (size_t)gc.ncells) {
    const int c = (int)(t - nnc);
    const int ci = c % gc.nx, cj = c / gc.nx;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int oy = 0; oy < 2; ++oy)
      for (int ox = 0; ox < 2; ++ox) {
        const size_t cf = (size_t)(2 * cj + oy) * gf.nx + 2 * ci + ox;
        const double* pf = r + gf.mv + 3 * cf;
        s0 += pf[0];
        s1 += (2 * ox - 1) / 4.0 * pf[0] + 0.5 * pf[1];
        s2 += (2 * oy - 1) / 4.0 * pf[0] + 0.5 * pf[2];
      }
    double* pc = o + gc.mv + 3 * (size_t)c;
    pc[0] = s0;
    pc[1] = s1;
    pc[2] = s2;
  }
}

// Local prolongation of child (ox, oy): Pk[i][j] maps the parent's 21 local
// dofs (j) to the child's 21 local dofs (i).
__device__ double ploc(int ox, int oy, int i, int j) {
  if (i < 18 && j < 18) {
    if ((i & 1) != (j & 1)) return 0.0;
    const int af = i >> 1, bc = j >> 1;
    const double xi = (2 * ox + af % 3) / 4.0, eta = (2 * oy + af / 3) / 4.0;
    return lag(bc % 3, xi) * lag(bc / 3, eta);
  }
  if (i >= 18 && j >= 18) {
    const int fi = i - 18, cj = j - 18;
    if (fi == 0) return cj == 0 ? 1.0 : cj == 1 ? (2 * ox - 1) / 4.0 : (2 * oy - 1) / 4.0;
    if (fi == 1) return cj == 1 ? 0.5 : 0.0;
    return cj == 2 ? 0.5 : 0.0;
  }
  return 0.0;
}

// Fine-level CIP face block entry (on the fly from the lagged state):
// coef sum_q (w_q h) |a_L . n| gA_a(q) gB_b(q), g^L = +dE(1) B ihn, g^R = -dE(0) B ihn.
__device__ double cip_block(const Geom& g, const Disc& ds, const double* v, int axis, int fi, int fj, int sA, int a,
                            int sB, int b) {
  const double hface = axis == 0 ? g.hy : g.hx;
  const double ihn = axis == 0 ? g.ihx : g.ihy;
  const double coef = ds.gamma_cip * hface * hface * ihn * ihn;
  const int na = axis == 0 ? a % 3 : a / 3, ta = axis == 0 ? a / 3 : a % 3;
  const int nb = axis == 0 ? b % 3 : b / 3, tb = axis == 0 ? b / 3 : b % 3;
  const double fa = sA == 0 ? c_tab.dE[1][na] : -c_tab.dE[0][na];
  const double fb = sB == 0 ? c_tab.dE[1][nb] : -c_tab.dE[0][nb];
  double s = 0.0;
  for (int q = 0; q < 4; ++q) {
    double tr = 0.0;
    for (int t = 0; t < 3; ++t) {
      const size_t node = axis == 0 ? (size_t)(2 * fj + t) * g.nnx + 2 * fi + 2 : (size_t)(2 * fj + 2) * g.nnx + 2 * fi + t;
      tr = fma(c_tab.B[q][t], v[2 * node + axis], tr);
    }
    s += (c_tab.w[q] * hface) * fabs(tr) * (fa * c_tab.B[q][ta]) * (fb * c_tab.B[q][tb]);
  }
  return coef * s;
}

// cip_block in two steps for the Galerkin kernels, which evaluate all 324 entries of a fine
// face: the point weights (w_q h) |a_L . n| once per (face, q), then the entry from them
// (the same products in the same order).
__device__ double cip_point_weight(const Geom& g, const double* v, int axis, int fi, int fj, int q) {
  const double hface = axis == 0 ? g.hy : g.hx;
  double tr = 0.0;
  for (int t = 0; t < 3; ++t) {
    const size_t node = axis == 0 ? (size_t)(2 * fj + t) * g.nnx + 2 * fi + 2 : (size_t)(2 * fj + 2) * g.nnx + 2 * fi + t;
    tr = fma(c_tab.B[q][t], v[2 * node + axis], tr);
  }
  return (c_tab.w[q] * hface) * fabs(tr);
}
__device__ double cip_block_w(const Geom& g, const Disc& ds, const double* wq, int axis, int sA, int a, int sB, int b) {
  const double hface = axis == 0 ? g.hy : g.hx;
  const double ihn = axis == 0 ? g.ihx : g.ihy;
  const double coef = ds.gamma_cip * hface * hface * ihn * ihn;
  const int na = axis == 0 ? a % 3 : a / 3, ta = axis == 0 ? a / 3 : a % 3;
  const int nb = axis == 0 ? b % 3 : b / 3, tb = axis == 0 ? b / 3 : b % 3;
  const double fa = sA == 0 ? c_tab.dE[1][na] : -c_tab.dE[0][na];
  const double fb = sB == 0 ? c_tab.dE[1][nb] : -c_tab.dE[0][nb];
  double s = 0.0;
  for (int q = 0; q < 4; ++q) s += wq[q] * (fa * c_tab.B[q][ta]) * (fb * c_tab.B[q][tb]);
  return coef * s;
}

// Face block entry of a level (stored for coarse levels, on the fly for the finest).
__device__ __forceinline__ double face_entry(const LevelOp& op, int mu, int axis, int fi, int fj, int sA, int a, int sB,
                                             int b) {
  if (op.fine) {
    if (!(op.ds.convection && op.ds.gamma_cip > 0.0)) return 0.0;
    return cip_block(op.g, op.ds, op.state + (size_t)mu * op.g.mv, axis, fi, fj, sA, a, sB, b);
  }
  const double* F = axis == 0 ? op.fv + ((size_t)mu * (op.g.nx - 1) * op.g.ny + (size_t)fj * (op.g.nx - 1) + fi) * 324
                              : op.fh + ((size_t)mu * op.g.nx * (op.g.ny - 1) + (size_t)fj * op.g.nx + fi) * 324;
  return F[((sA * 2 + sB) * 9 + b) * 9 + a];  // column-major 9x9 node blocks
}

__device__ __forceinline__ double cell_entry(const LevelOp& op, int mu, int c, int i, int j) {
  // column-major on every level (ET[c][j][i]): a thread per row reads coalesced columns
  const size_t base = ((size_t)mu * op.g.ncells + c) * 441;
  return op.ecell[base + (size_t)j * 21 + i];
}

// The four children's local prolongation blocks, the same for every cell:
// evaluated once per device (k_pm_init) instead of once per CTA.
__device__ double g_pm[4 * 441];
__global__ void k_pm_init() {
  for (int idx = threadIdx.x; idx < 4 * 441; idx += blockDim.x) {
    const int k = idx / 441, e = idx % 441;
    g_pm[idx] = ploc(k & 1, k >> 1, e / 21, e % 21);
  }
}

// Galerkin coarse cell block: one CTA (448 threads) per (coarse cell, mu).
// The four children's triple products P_K' E_K P_K run side by side on 196
// threads, each holding a 3 x 3 register tile of one child's product (six
// shared-memory operands per nine DFMA; one output per thread needed two per
// DFMA and was bound by the shared-memory pipe); every entry is still the
// same m-ordered fma chain and the children are summed in the same order.
__global__ void __launch_bounds__(448, 3) k_galerkin_cells(LevelOp f, Geom gc, double* __restrict__ ecell_c) {
  __shared__ double Pm[4][21][22];  // row stride 22: rows 2b and 2b + 1 read side by side fall into disjoint banks
  // Es[4][441] (the children's element blocks, column-major; later their products) and T[4][21][22];
  // the face part below reuses the space as FB[16][9][10] and SB[8][9][18]
  __shared__ __align__(16) double W[4 * 441 + 4 * 21 * 22];
  double* Es = W;
  double(*T)[21][22] = reinterpret_cast<double(*)[21][22]>(W + 4 * 441);
  double(*FB)[9][10] = reinterpret_cast<double(*)[9][10]>(W);
  double(*SB)[9][18] = reinterpret_cast<double(*)[9][18]>(W + 16 * 90);
  const int C = blockIdx.x, mu = blockIdx.y;
  const int t = threadIdx.x;
  const int ci = C % gc.nx, cj = C / gc.nx;
  for (int idx = t; idx < 4 * 441; idx += blockDim.x) {
    const int e = idx % 441;
    Pm[idx / 441][e / 21][e % 21] = g_pm[idx];
  }
  for (int idx = t; idx < 4 * 441; idx += blockDim.x) {
    const int k = idx / 441, e = idx - 441 * k;
    const int K = (2 * cj + (k >> 1)) * f.g.nx + 2 * ci + (k & 1);
    Es[idx] = f.ecell[((size_t)mu * f.g.ncells + K) * 441 + e];
  }
  const int i = t / 21, j = t % 21;
  const int tk = t / 49, tile = t % 49, i0 = 3 * (tile / 7), j0 = 3 * (tile % 7);
  __syncthreads();
  if (t < 196) {  // T_k = E_k P_k  (rows = child dofs, cols = parent dofs)
    double s[3][3] = {};
#pragma unroll 3
    for (int m = 0; m < 21; ++m) {
      double e[3], pr[3];
#pragma unroll
      for (int r = 0; r < 3; ++r) e[r] = Es[tk * 441 + m * 21 + i0 + r];
#pragma unroll
      for (int c = 0; c < 3; ++c) pr[c] = Pm[tk][m][j0 + c];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) s[r][c] = fma(e[r], pr[c], s[r][c]);
    }
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) T[tk][i0 + r][j0 + c] = s[r][c];
  }
  __syncthreads();
  if (t < 196) {  // P_k' T_k, into the child's (now free) element block space, row-major
    double s[3][3] = {};
#pragma unroll 3
    for (int m = 0; m < 21; ++m) {
      double pl[3], tr[3];
#pragma unroll
      for (int r = 0; r < 3; ++r) pl[r] = Pm[tk][m][i0 + r];
#pragma unroll
      for (int c = 0; c < 3; ++c) tr[c] = T[tk][m][j0 + c];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) s[r][c] = fma(pl[r], tr[c], s[r][c]);
    }
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) Es[tk * 441 + (i0 + r) * 21 + j0 + c] = s[r][c];
  }
  __syncthreads();
  double acc = 0.0;
  if (t < 441)
    for (int k = 0; k < 4; ++k) acc += Es[k * 441 + i * 21 + j];
  // finest level: the CIP point weights of the four interior fine faces, once per (face, point)
  __shared__ double Wq[4][4];
  const bool fine_cip = f.fine && f.ds.convection && f.ds.gamma_cip > 0.0;
  if (fine_cip && t < 16) {
    const int fidx = t >> 2, axis = fidx < 2 ? 0 : 1, o = fidx & 1;
    Wq[fidx][t & 3] = cip_point_weight(f.g, f.state + (size_t)mu * f.g.mv, axis, 2 * ci + (axis == 0 ? 0 : o),
                                       2 * cj + (axis == 0 ? o : 0), t & 3);
  }
  __syncthreads();
  // fine faces interior to C: vertical (children (0,oy)|(1,oy)), horizontal ((ox,0)|(ox,1)).
  // All 16 (face, side, side) node blocks are evaluated first, by all threads, then summed
  // without further barriers.
  for (int idx = t; idx < 16 * 81; idx += blockDim.x) {
    const int blk = idx / 81, e = idx - 81 * blk;
    const int fidx = blk >> 2, sA = (blk >> 1) & 1, sB = blk & 1;
    const int axis = fidx < 2 ? 0 : 1, o = fidx & 1;
    const int fi = 2 * ci + (axis == 0 ? 0 : o), fj = 2 * cj + (axis == 0 ? o : 0);
    FB[blk][e / 9][e % 9] = !f.fine      ? face_entry(f, mu, axis, fi, fj, sA, e / 9, sB, e % 9)
                            : fine_cip ? cip_block_w(f.g, f.ds, Wq[fidx], axis, sA, e / 9, sB, e % 9)
                                       : 0.0;
  }
  __syncthreads();
  // sum_{a,b} P_kA[2a+d][i] F[a][b] P_kB[2b+d][j] per block, factored: the inner sums
  // SB[a][j] = sum_b F[a][b] P_kB[2b+d][j] do not depend on i, so they are formed once per
  // (block, a, j) — 8 blocks at a time — and every (i, j) pair then needs 9 terms per block
  // instead of 90 (same products and order as the unfactored double loop).
  for (int half = 0; half < 2; ++half) {
    for (int idx = t; idx < 8 * 9 * 18; idx += blockDim.x) {
      const int bl = idx / 162, a = (idx / 18) % 9, jv = idx % 18, d = jv & 1;
      const int blk = 8 * half + bl, fidx = blk >> 2, sB = blk & 1;
      const int axis = fidx < 2 ? 0 : 1, o = fidx & 1;
      const int kl = axis == 0 ? (o * 2 + 0) : (0 * 2 + o), kr = axis == 0 ? (o * 2 + 1) : (1 * 2 + o);
      const int kB = sB == 0 ? kl : kr;
      double sb = 0.0;
      for (int b = 0; b < 9; ++b) sb = fma(FB[blk][a][b], Pm[kB][2 * b + d][jv], sb);
      SB[bl][a][jv] = sb;
    }
    __syncthreads();
    if (t < 441 && i < 18 && j < 18 && (i & 1) == (j & 1)) {
      const int d = i & 1;  // I2: component d of i and j must agree
      for (int bl = 0; bl < 8; ++bl) {
        const int blk = 8 * half + bl, fidx = blk >> 2, sA = (blk >> 1) & 1;
        const int axis = fidx < 2 ? 0 : 1, o = fidx & 1;
        const int kl = axis == 0 ? (o * 2 + 0) : (0 * 2 + o), kr = axis == 0 ? (o * 2 + 1) : (1 * 2 + o);
        const int kA = sA == 0 ? kl : kr;  // child index k = ox + 2 oy of the left/lower (sA = 0) or right/upper cell
        double sacc = 0.0;
        for (int a = 0; a < 9; ++a) {
          const double pa = Pm[kA][2 * a + d][i];
          if (pa == 0.0) continue;
          sacc = fma(pa, SB[bl][a][j], sacc);
        }
        acc += sacc;
      }
    }
    __syncthreads();
  }
  if (t < 441) ecell_c[((size_t)mu * gc.ncells + C) * 441 + (size_t)j * 21 + i] = acc;  // column-major
}

// Galerkin coarse face blocks from the two fine faces lying on the coarse face.
// One CTA (324 threads: sA, sB, a, b) per (coarse face, mu); axis via blockIdx.z.
__global__ void __launch_bounds__(324, 4) k_galerkin_faces(LevelOp f, Geom gc, double* __restrict__ fv_c,
                                                        double* __restrict__ fh_c) {
  __shared__ double Pn[4][9][9];  // node-level prolongation of child k: Pn[k][a_fine][b_coarse]
  __shared__ double F[2][2][9][9];
  __shared__ double SBf[2][2][9][9];
  __shared__ double wq[4];  // finest level: the fine face's CIP point weights
  const bool fine_cip = f.fine && f.ds.convection && f.ds.gamma_cip > 0.0;
  const int axis = blockIdx.z, mu = blockIdx.y;
  const int nfx = axis == 0 ? gc.nx - 1 : gc.nx;
  const int nface = axis == 0 ? (gc.nx - 1) * gc.ny : gc.nx * (gc.ny - 1);
  const int fc = blockIdx.x;
  if (fc >= nface) return;
  const int fi = fc % nfx, fj = fc / nfx;
  const int t = threadIdx.x;
  for (int idx = t; idx < 4 * 81; idx += blockDim.x) {
    const int k = idx / 81, e = idx % 81;
    Pn[k][e / 9][e % 9] = g_pm[k * 441 + (2 * (e / 9)) * 21 + 2 * (e % 9)];  // (k_pm_init ran with the cell kernel)
  }
  const int sA = t / 162, sB = (t / 81) % 2, a = (t / 9) % 9, b = t % 9;
  double acc = 0.0;
  for (int o = 0; o < 2; ++o) {
    // fine face: vertical between (2fi+1, 2fj+o) and (2fi+2, 2fj+o); horizontal between (2fi+o, 2fj+1) and (2fi+o, 2fj+2)
    const int ffi = axis == 0 ? 2 * fi + 1 : 2 * fi + o, ffj = axis == 0 ? 2 * fj + o : 2 * fj + 1;
    const int kl = axis == 0 ? (1 + 2 * o) : (o + 2 * 1);  // child index in the left/lower coarse cell
    const int kr = axis == 0 ? (0 + 2 * o) : (o + 2 * 0);  // child index in the right/upper coarse cell
    if (fine_cip && t < 4) wq[t] = cip_point_weight(f.g, f.state + (size_t)mu * f.g.mv, axis, ffi, ffj, t);
    __syncthreads();
    if (t < 324)
      F[sA][sB][a][b] = !f.fine      ? face_entry(f, mu, axis, ffi, ffj, sA, a, sB, b)
                        : fine_cip ? cip_block_w(f.g, f.ds, wq, axis, sA, a, sB, b)
                                   : 0.0;
    __syncthreads();
    // factored: SBf[sA][sB][p][b] = sum_q F[sA][sB][p][q] Pn[kB][q][b] once per (p, b), thread (a, b) playing (p, b)
    if (t < 324) {
      const int kB = sB == 0 ? kl : kr;
      double sb = 0.0;
      for (int q = 0; q < 9; ++q) sb = fma(F[sA][sB][a][q], Pn[kB][q][b], sb);
      SBf[sA][sB][a][b] = sb;
    }
    __syncthreads();
    if (t < 324) {
      const int kA = sA == 0 ? kl : kr;
      double s = 0.0;
      for (int p = 0; p < 9; ++p) {
        const double pa = Pn[kA][p][a];
        if (pa == 0.0) continue;
        s = fma(pa, SBf[sA][sB][p][b], s);
      }
      acc += s;
    }
  }
  if (t < 324) {
    double* dst = axis == 0 ? fv_c + ((size_t)mu * nface + fc) * 324 : fh_c + ((size_t)mu * nface + fc) * 324;
    dst[((sA * 2 + sB) * 9 + b) * 9 + a] = acc;  // column-major node blocks
  }
}

// Coarse level apply (multigrid.py:234-248), two PDL-chained kernels:
// y_mu = tau w_mu J_mu x_mu + sum_nu K_t[mu,nu] M x_nu; rhs != null gives
// y = rhs - A x.
//  1. k_level_products: per cell c and local row i, the cell's whole share
//        cp[mu][c][i] = sum_j E_c[i][j] x_c[j]
//                     + sum over c's faces f (right, top, left, bottom) of
//                       sum_sB,b F_f[s(c)][sB][a][b] x_sB[b][d]   (i = 2a + d < 18)
//     one thread per row; the column-major element / face blocks make each
//     warp-wide column load one contiguous segment; every block entry is read
//     once (a face block's two row halves by its two cells); x_c staged in
//     shared memory.
//     The share is tau w_mu (that) + the cell's temporal mass share
//     hx hy (M1 (x) M1)(K_t x) (the assembled Q2 mass is the sum of them).
//  2. k_level_gather: every dof sums the <= 4 cell shares containing it in a
//     fixed order and finishes (deterministic).
constexpr int LP_CELLS = 12;  // cells per CTA (12 x 21 = 252 threads)
constexpr int LP_NT = 252;

__global__ void __launch_bounds__(LP_NT, 4) k_level_products(LevelOp op, TimeData td, const double* __restrict__ x,
                                                             double* __restrict__ cp) {
  pdl_trigger();  // the gather may launch; it waits for this grid
  const Geom& g = op.g;
  const int mu = blockIdx.y;
  const double* xm = x + (size_t)mu * g.nd;
  __shared__ double xs[LP_CELLS][21];
  __shared__ double xt[LP_CELLS][18];  // sum_nu K_t[mu,nu] x_nu at the cell's velocity dofs
  const int t = threadIdx.x;
  const int p = t / 21, i = t % 21;
  const int c = blockIdx.x * LP_CELLS + p;
  const bool ok = p < LP_CELLS && c < g.ncells;
  const int cx = ok ? c % g.nx : 0, cy = ok ? c / g.nx : 0;
  auto xnode = [&](int cell_x, int cell_y, int b, int d) {
    return xm[2 * ((size_t)(2 * cell_y + b / 3) * g.nnx + 2 * cell_x + b % 3) + d];
  };
  if (ok) {
    xs[p][i] = i < 18 ? xnode(cx, cy, i >> 1, i & 1) : xm[g.mv + 3 * (size_t)c + i - 18];
    if (i < 18) {
      const int b = i >> 1;
      const size_t o = 2 * ((size_t)(2 * cy + b / 3) * g.nnx + 2 * cx + b % 3) + (i & 1);
      double v = 0.0;
      for (int nu = 0; nu < td.k1; ++nu) v = fma(td.K_t[mu * td.k1 + nu], x[(size_t)nu * g.nd + o], v);
      xt[p][i] = v;
    }
  }
  __syncthreads();
  if (!ok) return;
  const double* E = op.ecell + ((size_t)mu * g.ncells + c) * 441 + i;  // column j at E[21 j]
  double s = 0.0;
#pragma unroll 7
  for (int j = 0; j < 21; ++j) s = fma(__ldg(E + 21 * j), xs[p][j], s);
  if (i < 18) {
    const int a = i >> 1, d = i & 1;
    // faces of c: right (c = left cell of a vertical face), top, left, bottom
#pragma unroll 1
    for (int k = 0; k < 4; ++k) {
      const int axis = k & 1;
      const bool own_first = k < 2;  // c is the left / lower cell
      const int fi = axis == 0 ? (own_first ? cx : cx - 1) : cx;
      const int fj = axis == 0 ? cy : (own_first ? cy : cy - 1);
      const int nfx = axis == 0 ? g.nx - 1 : g.nx, nfy = axis == 0 ? g.ny : g.ny - 1;
      if (fi < 0 || fj < 0 || fi >= nfx || fj >= nfy) continue;
      const int sA = own_first ? 0 : 1;
      const int ox = axis == 0 ? (own_first ? 1 : -1) : 0, oy = axis == 1 ? (own_first ? 1 : -1) : 0;
      const size_t f = (size_t)fj * nfx + fi;
      const size_t nf = (size_t)nfx * nfy;
      const double* F = (axis == 0 ? op.fv : op.fh) + ((size_t)mu * nf + f) * 324 + (size_t)sA * 162 + a;
#pragma unroll
      for (int sB = 0; sB < 2; ++sB) {
        const bool own = (sB == sA);
        const int bxc = own ? cx : cx + ox, byc = own ? cy : cy + oy;
#pragma unroll
        for (int b = 0; b < 9; ++b) {
          const double xv = own ? xs[p][2 * b + d] : xnode(bxc, byc, b, d);
          s = fma(__ldg(F + sB * 81 + b * 9), xv, s);  // F[sA][sB][b][a], column-major node block
        }
      }
    }
  }
  double out = td.tau_w[mu] * s;
  if (i < 18) {  // + the cell's temporal mass share hx hy (M1 (x) M1) (K_t x)
    const int a = i >> 1, d = i & 1, ay = a / 3, ax = a % 3;
    double m = 0.0;
#pragma unroll
    for (int b = 0; b < 9; ++b) m = fma(c_tab.M1[ay][b / 3] * c_tab.M1[ax][b % 3], xt[p][2 * b + d], m);
    out = fma(g.hx * g.hy, m, out);
  }
  cp[((size_t)mu * g.ncells + c) * 21 + i] = out;
}

__global__ void k_level_gather(LevelOp op, const double* __restrict__ cp, const double* __restrict__ rhs,
                               double* __restrict__ y) {
  const Geom& g = op.g;
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int mu = blockIdx.y;
  const size_t nn = (size_t)g.nnx * g.nny;
  pdl_wait();
  if (t < nn) {
    const int X = (int)(t % g.nnx), Y = (int)(t / g.nnx);
    const size_t o0 = (size_t)mu * g.nd + 2 * t;
    double j0 = 0.0, j1 = 0.0;
    for (int cy = max(0, (Y - 1) / 2); cy <= min(g.ny - 1, Y / 2); ++cy)
      for (int cx = max(0, (X - 1) / 2); cx <= min(g.nx - 1, X / 2); ++cx) {
        const int c = cy * g.nx + cx;
        const int a = 3 * (Y - 2 * cy) + (X - 2 * cx);
        const double* q = cp + ((size_t)mu * g.ncells + c) * 21 + 2 * a;
        j0 += q[0];
        j1 += q[1];
      }
    y[o0] = rhs ? rhs[o0] - j0 : j0;
    y[o0 + 1] = rhs ? rhs[o0 + 1] - j1 : j1;
  } else if (t < nn + (size_t)g.ncells) {
    const size_t c = t - nn;
    const double* q = cp + ((size_t)mu * g.ncells + c) * 21 + 18;
    for (int r = 0; r < 3; ++r) {
      const size_t o = (size_t)mu * g.nd + g.mv + 3 * c + r;
      y[o] = rhs ? rhs[o] - q[r] : q[r];
    }
  }
}

__device__ __forceinline__ int ceil_half(int v) { return v <= 0 ? -((-v) / 2) : (v + 1) / 2; }
__device__ __forceinline__ int floor_half(int v) { return v >= 0 ? v / 2 : -((-v + 1) / 2); }

// (R_K J_mu R_K')_{ij} of a level in element form, for every Radau node at once
// (the cells and faces an entry gathers from do not depend on mu).
template <int K1>
__device__ __forceinline__ void level_spatial_entries(const LevelOp& op, int K, int i, int j, double* val) {
  const Geom& g = op.g;
#pragma unroll
  for (int mu = 0; mu < K1; ++mu) val[mu] = 0.0;
  if (i >= 18 || j >= 18) {
#pragma unroll
    for (int mu = 0; mu < K1; ++mu) val[mu] = cell_entry(op, mu, K, i, j);
    return;
  }
  const int ki = K % g.nx, kj = K / g.nx;
  const int ia = i >> 1, d = i & 1, jb = j >> 1, e = j & 1;
  const int XA = 2 * ki + ia % 3, YA = 2 * kj + ia / 3;
  const int XB = 2 * ki + jb % 3, YB = 2 * kj + jb / 3;
  const int xmin = min(XA, XB), xmax = max(XA, XB), ymin = min(YA, YB), ymax = max(YA, YB);
  for (int cy = max(0, ceil_half(ymax - 2)); cy <= min(g.ny - 1, floor_half(ymin)); ++cy)
    for (int cx = max(0, ceil_half(xmax - 2)); cx <= min(g.nx - 1, floor_half(xmin)); ++cx) {
      const int c = cy * g.nx + cx;
      const int al = 3 * (YA - 2 * cy) + (XA - 2 * cx), bl = 3 * (YB - 2 * cy) + (XB - 2 * cx);
#pragma unroll
      for (int mu = 0; mu < K1; ++mu) val[mu] += cell_entry(op, mu, c, 2 * al + d, 2 * bl + e);
    }
  if (d != e) return;
  for (int axis = 0; axis < 2; ++axis) {
    const int nfx = axis == 0 ? g.nx - 1 : g.nx, nfy = axis == 0 ? g.ny : g.ny - 1;
    const int xr = axis == 0 ? 4 : 2, yr = axis == 0 ? 2 : 4;
    for (int fj = max(0, ceil_half(ymax - yr)); fj <= min(nfy - 1, floor_half(ymin)); ++fj)
      for (int fi = max(0, ceil_half(xmax - xr)); fi <= min(nfx - 1, floor_half(xmin)); ++fi) {
        // the face's cells: (fi, fj) and its right / upper neighbour
        for (int sA = 0; sA < 2; ++sA) {
          const int ax = XA - 2 * (fi + (axis == 0 ? sA : 0)), ay = YA - 2 * (fj + (axis == 1 ? sA : 0));
          if (ax < 0 || ax > 2 || ay < 0 || ay > 2) continue;
          for (int sB = 0; sB < 2; ++sB) {
            const int bx = XB - 2 * (fi + (axis == 0 ? sB : 0)), by = YB - 2 * (fj + (axis == 1 ? sB : 0));
            if (bx < 0 || bx > 2 || by < 0 || by > 2) continue;
#pragma unroll
            for (int mu = 0; mu < K1; ++mu) val[mu] += face_entry(op, mu, axis, fi, fj, sA, 3 * ay + ax, sB, 3 * by + bx);
          }
        }
      }
  }
}

// Exact coarse patches: A_K = sum K_t (x) R_K M R_K' + tau w_mu R_K J_mu R_K'.
// The spatial entries are evaluated column-major (consecutive threads =
// consecutive rows i: the element and face blocks are stored column-major, so
// their loads coalesce), staged in shared memory, and written row-major.
template <int K1>
__global__ void __launch_bounds__(448, 3) k_patch_level(LevelOp op, TimeData td, double* __restrict__ mats) {
  __shared__ double sJ[K1][441];  // [mu][i * 21 + j]
  const int K = blockIdx.x;
  const int t = threadIdx.x;
  const Geom& g = op.g;
  const int k1 = td.k1, D = 21 * k1;
  if (t < 441) {
    const int ci_ = t % 21, cj_ = t / 21;
    double val[K1];
    level_spatial_entries<K1>(op, K, ci_, cj_, val);
#pragma unroll
    for (int mu = 0; mu < K1; ++mu) sJ[mu][ci_ * 21 + cj_] = val[mu];
  }
  __syncthreads();
  if (t >= 441) return;
  const int i = t / 21, j = t % 21;
  double M = 0.0;
  if (i < 18 && j < 18 && (i & 1) == (j & 1)) {
    const int ki = K % g.nx, kj = K / g.nx;
    const int ia = i >> 1, jb = j >> 1;
    M = g.hx * g.hy * (m1g(2 * kj + ia / 3, 2 * kj + jb / 3, g.ny) * m1g(2 * ki + ia % 3, 2 * ki + jb % 3, g.nx));
  }
  double* A = mats + (size_t)K * D * D;
  for (int mu = 0; mu < k1; ++mu) {
    const double J = sJ[mu][t];
    for (int nu = 0; nu < k1; ++nu) {
      double v = (i < 18 && j < 18) ? td.K_t[mu * k1 + nu] * M : 0.0;
      if (mu == nu) v += td.tau_w[mu] * J;
      A[(size_t)(21 * mu + i) * D + 21 * nu + j] = v;
    }
  }
}

// Dense coarsest-level slab matrix (multigrid.py:494-520), one thread per row.
__global__ void k_dense_assemble(LevelOp op, TimeData td, double* __restrict__ A, int n) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  const Geom& g = op.g;
  const int mu = row / g.nd, r = row % g.nd;
  double* Ar = A + (size_t)row * n;
  for (int c = 0; c < n; ++c) Ar[c] = 0.0;
  const double tw = td.tau_w[mu];
  if (r >= g.mv) {
    const int c = (r - g.mv) / 3, pr = (r - g.mv) % 3;
    const int cx = c % g.nx, cy = c / g.nx;
    for (int jj = 0; jj < 21; ++jj) {
      const int col = jj < 18 ? 2 * ((2 * cy + (jj >> 1) / 3) * g.nnx + 2 * cx + (jj >> 1) % 3) + (jj & 1)
                              : g.mv + 3 * c + jj - 18;
      Ar[(size_t)mu * g.nd + col] += tw * cell_entry(op, mu, c, 18 + pr, jj);
    }
    return;
  }
  const int node = r >> 1, d = r & 1;
  const int X = node % g.nnx, Y = node / g.nnx;
  for (int cy = max(0, (Y - 1) / 2); cy <= min(g.ny - 1, Y / 2); ++cy)
    for (int cx = max(0, (X - 1) / 2); cx <= min(g.nx - 1, X / 2); ++cx) {
      const int c = cy * g.nx + cx;
      const int a = 3 * (Y - 2 * cy) + (X - 2 * cx);
      for (int jj = 0; jj < 21; ++jj) {
        const int col = jj < 18 ? 2 * ((2 * cy + (jj >> 1) / 3) * g.nnx + 2 * cx + (jj >> 1) % 3) + (jj & 1)
                                : g.mv + 3 * c + jj - 18;
        Ar[(size_t)mu * g.nd + col] += tw * cell_entry(op, mu, c, 2 * a + d, jj);
      }
    }
  for (int axis = 0; axis < 2; ++axis) {
    const int nfx = axis == 0 ? g.nx - 1 : g.nx, nfy = axis == 0 ? g.ny : g.ny - 1;
    const int xr = axis == 0 ? 4 : 2, yr = axis == 0 ? 2 : 4;
    for (int fj = max(0, (Y - yr + 1) / 2); fj <= min(nfy - 1, Y / 2); ++fj)
      for (int fi = max(0, (X - xr + 1) / 2); fi <= min(nfx - 1, X / 2); ++fi) {
        const int cl = fj * g.nx + fi, cr = axis == 0 ? cl + 1 : cl + g.nx;
        for (int sA = 0; sA < 2; ++sA) {
          const int cA = sA == 0 ? cl : cr;
          const int ax = X - 2 * (cA % g.nx), ay = Y - 2 * (cA / g.nx);
          if (ax < 0 || ax > 2 || ay < 0 || ay > 2) continue;
          for (int sB = 0; sB < 2; ++sB) {
            const int cB = sB == 0 ? cl : cr;
            for (int bb = 0; bb < 9; ++bb) {
              const int nb = (2 * (cB / g.nx) + bb / 3) * g.nnx + 2 * (cB % g.nx) + bb % 3;
              Ar[(size_t)mu * g.nd + 2 * nb + d] += tw * face_entry(op, mu, axis, fi, fj, sA, 3 * ay + ax, sB, bb);
            }
          }
        }
      }
  }
  // K_t (x) M on velocity
  for (int Yp = max(0, Y - 2); Yp <= min(g.nny - 1, Y + 2); ++Yp) {
    const double my = m1g(Y, Yp, g.ny);
    if (my == 0.0) continue;
    for (int Xp = max(0, X - 2); Xp <= min(g.nnx - 1, X + 2); ++Xp) {
      const double mx = m1g(X, Xp, g.nx);
      if (mx == 0.0) continue;
      const double m = g.hx * g.hy * (my * mx);
      for (int nu = 0; nu < td.k1; ++nu)
        Ar[(size_t)nu * g.nd + 2 * (Yp * g.nnx + Xp) + d] += td.K_t[mu * td.k1 + nu] * m;
    }
  }
}

// Add scale * z z' with z the normalized per-node constant-pressure mode
// (multigrid.py:509-519); one thread per (row, col) pair of the pressure blocks.
__global__ void k_dense_pin(Geom g, int k1, double* __restrict__ A, int n, double scale) {
  const int nc = g.ncells;
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t per = (size_t)nc * nc;
  if (t >= per * k1) return;
  const int mu = (int)(t / per);
  const int a = (int)((t % per) / nc), b = (int)(t % nc);
  // z entries: area on every p0 dof, normalized: 1/sqrt(nc)
  const double za = 1.0 / sqrt((double)nc);
  const size_t ra = (size_t)mu * g.nd + g.mv + 3 * (size_t)a, rb = (size_t)mu * g.nd + g.mv + 3 * (size_t)b;
  A[ra * n + rb] += scale * (za * za);
}

__global__ void k_diag_abs_sum(const double* __restrict__ A, int n, double* __restrict__ out) {
  __shared__ double sh[1024];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += fabs(A[(size_t)i * n + i]);
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if (threadIdx.x < off) sh[threadIdx.x] += sh[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0] / n;
}

// Dense in-place Gauss-Jordan with partial pivoting, one CTA (coarsest level).
__global__ void __launch_bounds__(1024) k_dense_invert(double* __restrict__ A, int n, int* __restrict__ piv,
                                                       int* __restrict__ bad) {
  __shared__ double sv[1024];
  __shared__ int si[1024];
  __shared__ double pinv_s;
  for (int k = 0; k < n; ++k) {
    double best = -1.0;
    int bi = n;
    for (int i = k + threadIdx.x; i < n; i += blockDim.x) {
      const double v = fabs(A[(size_t)i * n + k]);
      if (v > best || (v == best && i < bi)) {
        best = v;
        bi = i;
      }
    }
    sv[threadIdx.x] = best;
    si[threadIdx.x] = bi;
    __syncthreads();
    for (int off = blockDim.x / 2; off > 0; off >>= 1) {
      if (threadIdx.x < off) {
        const double ov = sv[threadIdx.x + off];
        const int oi = si[threadIdx.x + off];
        if (ov > sv[threadIdx.x] || (ov == sv[threadIdx.x] && oi < si[threadIdx.x])) {
          sv[threadIdx.x] = ov;
          si[threadIdx.x] = oi;
        }
      }
      __syncthreads();
    }
    const int p = si[0];
    if (!(sv[0] > 0.0)) {
      if (threadIdx.x == 0) *bad = 1;
      return;
    }
    if (threadIdx.x == 0) piv[k] = p;
    if (p != k)
      for (int j = threadIdx.x; j < n; j += blockDim.x) {
        const double tmp = A[(size_t)k * n + j];
        A[(size_t)k * n + j] = A[(size_t)p * n + j];
        A[(size_t)p * n + j] = tmp;
      }
    __syncthreads();
    if (threadIdx.x == 0) pinv_s = 1.0 / A[(size_t)k * n + k];
    __syncthreads();
    const double pinv = pinv_s;
    for (int j = threadIdx.x; j < n; j += blockDim.x)
      A[(size_t)k * n + j] = (j == k ? 1.0 : A[(size_t)k * n + j]) * pinv;
    __syncthreads();
    for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
      const int i = idx / n, j = idx - i * n;
      if (i == k || j == k) continue;
      A[(size_t)i * n + j] -= A[(size_t)i * n + k] * A[(size_t)k * n + j];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x)
      if (i != k) A[(size_t)i * n + k] = -A[(size_t)i * n + k] * pinv;
    __syncthreads();
  }
  for (int k = n - 1; k >= 0; --k) {
    const int p = piv[k];
    if (p != k)
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double tmp = A[(size_t)i * n + k];
        A[(size_t)i * n + k] = A[(size_t)i * n + p];
        A[(size_t)i * n + p] = tmp;
      }
    __syncthreads();
  }
}

// y = Ainv b (coarsest-level solve), one warp per row.
__global__ void k_dense_gemv(const double* __restrict__ Ainv, int n, const double* __restrict__ b,
                             double* __restrict__ y) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= n) return;
  const double* r = Ainv + (size_t)warp * n;
  double s = 0.0;
  for (int j = lane; j < n; j += 32) s = fma(r[j], b[j], s);
  for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
  if (lane == 0) y[warp] = s;
}

// Remove the mass-weighted mean of the constant pressure mode per node
// (multigrid.py:557-572).  Two passes over the cells with a fixed reduction
// tree (PP_PARTS partial sums per node, summed in order by every CTA of the
// second pass), so the result does not depend on scheduling.
constexpr int PP_PARTS = 592, PP_NT = 256;
__device__ __forceinline__ double pp_block_sum(double v, double* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int off = PP_NT / 2; off > 0; off >>= 1) {
    if ((int)threadIdx.x < off) sh[threadIdx.x] += sh[threadIdx.x + off];
    __syncthreads();
  }
  const double r = sh[0];
  __syncthreads();
  return r;
}
__global__ void __launch_bounds__(PP_NT) k_project_partial(Geom g, const double* __restrict__ z,
                                                          double* __restrict__ partial) {
  __shared__ double sh[PP_NT];
  const int mu = blockIdx.y;
  const double* p = z + (size_t)mu * g.nd + g.mv;
  const double area_c = g.hx * g.hy;
  const size_t chunk = ((size_t)g.ncells + PP_PARTS - 1) / PP_PARTS;
  const size_t c0 = (size_t)blockIdx.x * chunk, c1 = min(c0 + chunk, (size_t)g.ncells);
  double s = 0.0;
  for (size_t c = c0 + threadIdx.x; c < c1; c += PP_NT) s = fma(area_c, p[3 * c], s);
  s = pp_block_sum(s, sh);
  if (threadIdx.x == 0) partial[(size_t)mu * PP_PARTS + blockIdx.x] = s;
}
__global__ void __launch_bounds__(PP_NT) k_project_apply(Geom g, const double* __restrict__ partial,
                                                        double* __restrict__ z) {
  __shared__ double sh[PP_NT];
  const int mu = blockIdx.y;
  double* p = z + (size_t)mu * g.nd + g.mv;
  double s = 0.0;
  for (int i = threadIdx.x; i < PP_PARTS; i += PP_NT) s += partial[(size_t)mu * PP_PARTS + i];
  s = pp_block_sum(s, sh);
  const double mean = s / ((g.hx * g.hy) * g.ncells);
  const size_t c = (size_t)blockIdx.x * PP_NT + threadIdx.x;
  if (c < (size_t)g.ncells) p[3 * c] -= mean;
}

__global__ void k_axpy(size_t n, double a, const double* __restrict__ x, double* __restrict__ y) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] += a * x[i];
}

}  // namespace

cudaError_t prolong(const Geom& gc, const Geom& gf, int k1, const double* ec, double* ef, cudaStream_t st) {
  const size_t n = (size_t)gf.nnx * gf.nny + gf.ncells;
  PDST_LAUNCH(k_prolong<<<dim3((unsigned)((n + 255) / 256), k1), 256, 0, st>>>(gc, gf, k1, ec, ef));
  return cudaGetLastError();
}

cudaError_t restrict_(const Geom& gc, const Geom& gf, int k1, const double* rf, double* rc, cudaStream_t st) {
  const size_t n = (size_t)gc.nnx * gc.nny + gc.ncells;
  PDST_LAUNCH(k_restrict<<<dim3((unsigned)((n + 255) / 256), k1), 256, 0, st>>>(gc, gf, k1, rf, rc));
  return cudaGetLastError();
}

cudaError_t galerkin(const LevelOp& fine, const Geom& gc, int k1, double* ecell_c, double* fv_c, double* fh_c,
                     cudaStream_t st) {
  {
    static DeviceOnce once;
    const int dev = current_device();
    if (!once.done[dev]) {
      PDST_LAUNCH(k_pm_init<<<1, 448, 0, st>>>());
      cudaError_t e0 = cudaStreamSynchronize(st);  // once: other streams' builds may follow at once
      if (e0 != cudaSuccess) return e0;
      once.done[dev] = true;
    }
  }
  PDST_LAUNCH(k_galerkin_cells<<<dim3(gc.ncells, k1), 448, 0, st>>>(fine, gc, ecell_c));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int nf = max((gc.nx - 1) * gc.ny, gc.nx * (gc.ny - 1));
  if (nf > 0) PDST_LAUNCH(k_galerkin_faces<<<dim3(nf, k1, 2), 324, 0, st>>>(fine, gc, fv_c, fh_c));
  return cudaGetLastError();
}

size_t level_apply_scratch(const Geom& g, int k1) { return (size_t)k1 * 21 * (size_t)g.ncells; }

cudaError_t level_apply(const LevelOp& op, const TimeData& td, const double* x, const double* rhs, double* y,
                        double* scratch, cudaStream_t st) {
  if (!scratch) return cudaErrorMemoryAllocation;
  const Geom& g = op.g;
  const int ncb = (g.ncells + LP_CELLS - 1) / LP_CELLS;
  PDST_LAUNCH(k_level_products<<<dim3((unsigned)ncb, td.k1), LP_NT, 0, st>>>(op, td, x, scratch));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const size_t n = (size_t)g.nnx * g.nny + g.ncells;
  PDST_LAUNCH(e = launch_pdl(k_level_gather, dim3((unsigned)((n + 127) / 128), td.k1), dim3(128), 0, st, op,
                             (const double*)scratch, rhs, y));
  return e;
}

cudaError_t patch_assemble_level(const LevelOp& op, const TimeData& td, double* mats, cudaStream_t st) {
  switch (td.k1) {  // exact patches exist up to D = 84 (pdst_patch.cu launch_invert)
    case 1: PDST_LAUNCH(k_patch_level<1><<<op.g.ncells, 448, 0, st>>>(op, td, mats)); break;
    case 2: PDST_LAUNCH(k_patch_level<2><<<op.g.ncells, 448, 0, st>>>(op, td, mats)); break;
    case 3: PDST_LAUNCH(k_patch_level<3><<<op.g.ncells, 448, 0, st>>>(op, td, mats)); break;
    case 4: PDST_LAUNCH(k_patch_level<4><<<op.g.ncells, 448, 0, st>>>(op, td, mats)); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t dense_build(const LevelOp& op, const TimeData& td, bool pin, double* A, double* scratch, int* piv,
                        int* bad, cudaStream_t st) {
  const int n = td.k1 * op.g.nd;
  PDST_LAUNCH(k_dense_assemble<<<(n + 127) / 128, 128, 0, st>>>(op, td, A, n));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (pin) {
    PDST_LAUNCH(k_diag_abs_sum<<<1, 1024, 0, st>>>(A, n, scratch));
    double scale = 0.0;
    e = cudaMemcpyAsync(&scale, scratch, sizeof(double), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return e;
    const size_t tot = (size_t)op.g.ncells * op.g.ncells * td.k1;
    PDST_LAUNCH(k_dense_pin<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(op.g, td.k1, A, n, scale));
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  PDST_LAUNCH(k_dense_invert<<<1, 1024, 0, st>>>(A, n, piv, bad));
  return cudaGetLastError();
}

cudaError_t dense_solve(const double* Ainv, int n, const double* b, double* y, cudaStream_t st) {
  PDST_LAUNCH(k_dense_gemv<<<(n * 32 + 255) / 256, 256, 0, st>>>(Ainv, n, b, y));
  return cudaGetLastError();
}

size_t project_scratch(int k1) { return (size_t)k1 * PP_PARTS; }

cudaError_t project_pressure(const Geom& g, int k1, double* z, double* partial, cudaStream_t st) {
  PDST_LAUNCH(k_project_partial<<<dim3(PP_PARTS, k1), PP_NT, 0, st>>>(g, z, partial));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  PDST_LAUNCH(k_project_apply<<<dim3((unsigned)((g.ncells + PP_NT - 1) / PP_NT), k1), PP_NT, 0, st>>>(g, partial, z));
  return cudaGetLastError();
}

cudaError_t axpy(size_t n, double a, const double* x, double* y, cudaStream_t st) {
  PDST_LAUNCH(k_axpy<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, a, x, y));
  return cudaGetLastError();
}

namespace {
__global__ void k_inject(Geom gc, Geom gf, const double* __restrict__ vf, size_t sf, double* __restrict__ vc,
                         size_t sc, int zero_pressure) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int mu = blockIdx.y;
  const size_t nn = (size_t)gc.nnx * gc.nny;
  if (t < nn) {
    const int i = (int)(t % gc.nnx), j = (int)(t / gc.nnx);
    const size_t f = 2 * ((size_t)(2 * j) * gf.nnx + 2 * i);
    vc[mu * sc + 2 * t] = vf[mu * sf + f];
    vc[mu * sc + 2 * t + 1] = vf[mu * sf + f + 1];
  } else if (zero_pressure && t < nn + 3 * (size_t)gc.ncells) {
    vc[mu * sc + gc.mv + (t - nn)] = 0.0;
  }
}
}  // namespace

cudaError_t inject_velocity(const Geom& gc, const Geom& gf, int k1, const double* vf, size_t sf, double* vc,
                            size_t sc, bool zero_pressure, cudaStream_t st) {
  const size_t n = (size_t)gc.nnx * gc.nny + (zero_pressure ? 3 * (size_t)gc.ncells : 0);
  PDST_LAUNCH(k_inject<<<dim3((unsigned)((n + 255) / 256), k1), 256, 0, st>>>(gc, gf, vf, sf, vc, sc,
                                                                              zero_pressure ? 1 : 0));
  return cudaGetLastError();
}

}  // namespace pdst
