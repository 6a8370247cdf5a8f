// pdst_patch.cu — Vanka patch matrices, batched patch inversion and the
// additive Vanka sweep (sm_100a, fp64).
//
// Reference: solver/multigrid.py:251-299 (patch extraction + np.linalg.inv),
// :327-340 (vanka_smooth), :475-488 (surrogate finest patches).
//
// Patch of cell K = the 21 spatial dofs of K (18 velocity a-major comp-minor,
// 3 pressure) replicated over the k+1 Radau nodes, D = 21 (k+1):
//   A_K[(mu,i),(nu,j)] = K_t[mu,nu] (R_K M R_K')_{ij}  (velocity i, j)
//                      + delta_{mu nu} tau w_mu (R_K J_mu R_K')_{ij}.
// R_K J R_K' is formed WITHOUT a global matrix: entry (A, B) sums the element
// matrices of every cell that contains both nodes (up to 4 cells of the 3x3
// neighbourhood) plus the CIP couplings of every interior face whose two
// cells contain both nodes (up to 12 faces), evaluated on the fly from the
// lagged state trace.  The mass block uses the assembled 1-D Q2 mass
// (M = hx hy M1y (x) M1x (x) I2).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "pdst_device.cuh"
#include "pdst_patch.h"

namespace pdst {
namespace {

__device__ __forceinline__ double m1g(int X, int Xp, int n) {
  double s = 0.0;
  const int lo = max(0, (max(X, Xp) - 1) / 2);
  for (int c = lo; c <= min(X, Xp) / 2 && c < n; ++c) {
    const int a = X - 2 * c, b = Xp - 2 * c;
    if (a >= 0 && a <= 2 && b >= 0 && b <= 2) s += c_tab.M1[a][b];
  }
  return s;
}

__device__ __forceinline__ int ceil_half(int v) { return v <= 0 ? -((-v) / 2) : (v + 1) / 2; }
__device__ __forceinline__ int floor_half(int v) { return v >= 0 ? v / 2 : -((-v + 1) / 2); }

// Jump of the normal derivative of the global Q2 basis function at node
// coordinate Xn (normal direction) across the face whose left cell starts at
// node 2f, times B[q][t] (tangential factor applied by the caller).
__device__ __forceinline__ double jump_factor(int Xn, int f) {
  double v = 0.0;
  const int l = Xn - 2 * f;          // position in the left cell
  if (l >= 0 && l <= 2) v += c_tab.dE[1][l];
  const int r = Xn - 2 * f - 2;      // position in the right cell
  if (r >= 0 && r <= 2) v -= c_tab.dE[0][r];
  return v;
}

// CIP face weights of the faces that can couple two nodes of patch K, one
// table per slot, computed once per patch (CTA) instead of once per entry:
//   vertical faces (normal +x) between cells (fi, fj) and (fi+1, fj), fi =
//   ki-2..ki+1, fj = kj-1..kj+1:  cwv[s][fi - ki + 2][fj - kj + 1][q]
//   horizontal faces (normal +y) between (fi, fj) and (fi, fj+1), fj =
//   kj-2..kj+1, fi = ki-1..ki+1:  cwh[s][fj - kj + 2][fi - ki + 1][q]
// with the value (w_q h) |v_L . n| of the lagged left / lower trace at face
// point q (0 for faces outside the mesh; never read for them).
constexpr int CW_FACE = 4 * 3 * 4;  // 48 values per orientation and slot

__device__ void cip_weights(const PatchArgs& a, int K, double* cwv, double* cwh) {
  const Geom& g = a.g;
  const int ki = K % g.nx, kj = K / g.nx;
  for (int idx = threadIdx.x; idx < a.nslot * 2 * CW_FACE; idx += blockDim.x) {
    const int s = idx / (2 * CW_FACE), r = idx % (2 * CW_FACE), hor = r / CW_FACE, u = r % CW_FACE;
    const int o1 = u / 12, o2 = (u / 4) % 3, q = u % 4;
    const double* v = a.state + (size_t)s * g.mv;
    double val = 0.0;
    if (!hor) {
      const int fi = ki - 2 + o1, fj = kj - 1 + o2;
      if (fi >= 0 && fi <= g.nx - 2 && fj >= 0 && fj <= g.ny - 1) {
        const double h = g.hy;
        double tr = 0.0;
        for (int t = 0; t < 3; ++t)
          tr = fma(c_tab.B[q][t], v[2 * ((size_t)(2 * fj + t) * g.nnx + 2 * fi + 2)], tr);
        val = (c_tab.w[q] * h) * fabs(tr);
      }
      cwv[s * CW_FACE + u] = val;
    } else {
      const int fj = kj - 2 + o1, fi = ki - 1 + o2;
      if (fi >= 0 && fi <= g.nx - 1 && fj >= 0 && fj <= g.ny - 2) {
        const double h = g.hx;
        double tr = 0.0;
        for (int t = 0; t < 3; ++t)
          tr = fma(c_tab.B[q][t], v[2 * ((size_t)(2 * fj + 2) * g.nnx + 2 * fi + t) + 1], tr);
        val = (c_tab.w[q] * h) * fabs(tr);
      }
      cwh[s * CW_FACE + u] = val;
    }
  }
}

// Per-patch tables of the CIP couplings, filled once per CTA: the jump factors
// of the patch's three node columns / rows against the four faces per
// direction that can see them, the faces' validity and the tangential basis
// values — so an entry's face loop is table lookups in a fixed order instead of
// index arithmetic, constant-bank gathers and branches per face.
struct PatchTabs {
  double jx[4][3];      // jump_factor(2 ki + xn, ki - 2 + f)   vertical faces
  double jy[4][3];      // jump_factor(2 kj + yn, kj - 2 + f)   horizontal faces
  double B[4][3];       // c_tab.B
  unsigned char vv[4][3];  // vertical face (ki - 2 + f, kj - 1 + g) inside the mesh
  unsigned char vh[4][3];  // horizontal face (ki - 1 + g, kj - 2 + f) inside the mesh
};

__device__ void patch_tabs(const Geom& g, int K, PatchTabs& T) {
  const int ki = K % g.nx, kj = K / g.nx;
  const int t = threadIdx.x;
  if (t < 12) {
    const int f = t / 3, n = t % 3;
    T.jx[f][n] = jump_factor(2 * ki + n, ki - 2 + f);
    T.jy[f][n] = jump_factor(2 * kj + n, kj - 2 + f);
    T.B[f][n] = c_tab.B[f][n];
    const int fi = ki - 2 + f, fj = kj - 1 + n;  // vertical face, its cell row
    T.vv[f][n] = fi >= 0 && fi <= g.nx - 2 && fj >= 0 && fj <= g.ny - 1;
    const int hj = kj - 2 + f, hi = ki - 1 + n;  // horizontal face, its cell column
    T.vh[f][n] = hj >= 0 && hj <= g.ny - 2 && hi >= 0 && hi <= g.nx - 1;
  }
}

// Spatial block entry (R_K J R_K')_{ij} of element slot s in two parts (cwv /
// cwh: the patch's face weights, cip_weights; T: patch_tabs).  The faces are
// visited in (row, column) order and skipped where a jump factor vanishes.
// Part 1 (independent of the face weights): the element matrices of every
// cell containing both dofs.
__device__ double spatial_entry_cells(const PatchArgs& a, int s, int K, int i, int j) {
  const Geom& g = a.g;
  const int ki = K % g.nx, kj = K / g.nx;
  const double* ET = a.ET + (size_t)s * g.ncells * 441;
  if (i >= 18 || j >= 18) return ET[((size_t)K * 21 + j) * 21 + i];  // pressure couplings are cell-local
  const int ia = i >> 1, d = i & 1, jb = j >> 1, e = j & 1;
  const int XA = 2 * ki + ia % 3, YA = 2 * kj + ia / 3;
  const int XB = 2 * ki + jb % 3, YB = 2 * kj + jb / 3;
  const int xmin = min(XA, XB), xmax = max(XA, XB), ymin = min(YA, YB), ymax = max(YA, YB);
  double val = 0.0;
  for (int cy = max(0, ceil_half(ymax - 2)); cy <= min(g.ny - 1, floor_half(ymin)); ++cy)
    for (int cx = max(0, ceil_half(xmax - 2)); cx <= min(g.nx - 1, floor_half(xmin)); ++cx) {
      const int c = cy * g.nx + cx;
      const int al = 3 * (YA - 2 * cy) + (XA - 2 * cx), bl = 3 * (YB - 2 * cy) + (XB - 2 * cx);
      val += ET[((size_t)c * 21 + 2 * bl + e) * 21 + 2 * al + d];
    }
  return val;
}

// Part 2: + the CIP couplings of the faces that see both nodes (added to val = part 1).
__device__ double spatial_entry_faces(const PatchArgs& a, int s, int i, int j, double val, const double* cwv,
                                      const double* cwh, const PatchTabs& T) {
  const Geom& g = a.g;
  if (i >= 18 || j >= 18) return val;
  const int ia = i >> 1, d = i & 1, jb = j >> 1, e = j & 1;
  const int xa = ia % 3, ya = ia / 3, xb = jb % 3, yb = jb / 3;  // node positions in the patch cell
  if (d != e || !(a.ds.convection && a.ds.gamma_cip > 0.0)) return val;
  // vertical faces (normal +x) between (fi, fj) and (fi+1, fj): fj = kj - 1 + gr, fi = ki - 2 + f
  {
    const double h = g.hy, coef = a.ds.gamma_cip * h * h / (g.hx * g.hx);
#pragma unroll
    for (int gr = 0; gr < 3; ++gr) {
      const int ta = ya + 2 - 2 * gr, tb = yb + 2 - 2 * gr;  // the nodes' rows in cell row fj
      if (ta < 0 || ta > 2 || tb < 0 || tb > 2) continue;
#pragma unroll
      for (int f = 0; f < 4; ++f) {
        if (!T.vv[f][gr]) continue;
        const double ja = T.jx[f][xa], jb2 = T.jx[f][xb];
        if (ja == 0.0 || jb2 == 0.0) continue;
        const double* cw = cwv + s * CW_FACE + (f * 3 + gr) * 4;
        double sum = 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q) sum += cw[q] * (ja * T.B[q][ta]) * (jb2 * T.B[q][tb]);
        val += coef * sum;
      }
    }
  }
  // horizontal faces (normal +y) between (fi, fj) and (fi, fj+1): fj = kj - 2 + f, fi = ki - 1 + gc
  {
    const double h = g.hx, coef = a.ds.gamma_cip * h * h / (g.hy * g.hy);
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      const double ja = T.jy[f][ya], jb2 = T.jy[f][yb];
      if (ja == 0.0 || jb2 == 0.0) continue;
#pragma unroll
      for (int gc = 0; gc < 3; ++gc) {
        const int ta = xa + 2 - 2 * gc, tb = xb + 2 - 2 * gc;  // the nodes' columns in cell column fi
        if (ta < 0 || ta > 2 || tb < 0 || tb > 2) continue;
        if (!T.vh[f][gc]) continue;
        const double* cw = cwh + s * CW_FACE + (f * 3 + gc) * 4;
        double sum = 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q) sum += cw[q] * (ja * T.B[q][ta]) * (jb2 * T.B[q][tb]);
        val += coef * sum;
      }
    }
  }
  return val;
}

__global__ void __launch_bounds__(448, 3) k_patch_fine(PatchArgs a) {
  const int K = blockIdx.x;
  const int t = threadIdx.x;
  __shared__ double cwv[MAXK1 * CW_FACE], cwh[MAXK1 * CW_FACE];
  __shared__ PatchTabs tabs;
  __shared__ double sJ[MAXK1][441];  // the slots' spatial blocks, [i][j]
  const bool cip = a.ds.convection && a.ds.gamma_cip > 0.0;
  // Entries are evaluated column-major (consecutive threads = consecutive rows
  // i: the element matrices are stored [cell][j][i], so their loads coalesce)
  // and the cell sums are issued before the barrier on the face weights.
  const int ci_ = t % 21, cj_ = t / 21;
  double Js[MAXK1];
  if (t < 441)
    for (int s = 0; s < a.nslot; ++s) Js[s] = spatial_entry_cells(a, s, K, ci_, cj_);
  if (cip) {
    cip_weights(a, K, cwv, cwh);
    patch_tabs(a.g, K, tabs);
  }
  __syncthreads();
  if (t < 441)
    for (int s = 0; s < a.nslot; ++s) sJ[s][ci_ * 21 + cj_] = spatial_entry_faces(a, s, ci_, cj_, Js[s], cwv, cwh, tabs);
  __syncthreads();
  if (t >= 441) return;
  // output, row-major: consecutive threads = consecutive columns j
  const Geom& g = a.g;
  const int i = t / 21, j = t % 21;
  const int k1 = a.td.k1, D = 21 * k1;
  if (a.spatial) a.spatial[(size_t)K * 441 + t] = sJ[0][t];
  if (!a.mats) return;  // diagonalized path at scale: the spatial block is all the inverse needs
  double M = 0.0;
  if (i < 18 && j < 18 && (i & 1) == (j & 1)) {
    const int ki = K % g.nx, kj = K / g.nx;
    const int ia = i >> 1, jb = j >> 1;
    M = g.hx * g.hy * (m1g(2 * kj + ia / 3, 2 * kj + jb / 3, g.ny) * m1g(2 * ki + ia % 3, 2 * ki + jb % 3, g.nx));
  }
  double* A = a.mats + (size_t)K * D * D;
  for (int mu = 0; mu < k1; ++mu) {
    const double J = sJ[a.nslot == 1 ? 0 : mu][t];
    for (int nu = 0; nu < k1; ++nu) {
      double v = (i < 18 && j < 18) ? a.td.K_t[mu * k1 + nu] * M : 0.0;
      if (mu == nu) v += a.td.tau_w[mu] * J;
      A[(size_t)(21 * mu + i) * D + 21 * nu + j] = v;
    }
  }
}

// In-place Gauss-Jordan inversion with partial (row) pivoting, one warp per
// patch, matrix in shared memory (row stride D+1).  An exactly zero pivot
// column marks the patch singular (LAPACK getrf info > 0, the condition under
// which np.linalg.inv raises).  Output is stored transposed: invT[K][j][i].
template <int D>
__host__ __device__ constexpr int inv_wpb() { return D > 63 ? 2 : 4; }

template <int D>
__global__ void __launch_bounds__(128) k_invert(const double* __restrict__ mats, double* __restrict__ invT, int npatch,
                                                int* __restrict__ bad) {
  constexpr int WPB = inv_wpb<D>();
  constexpr int LD = D + 1;
  extern __shared__ double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = blockIdx.x * WPB + warp;
  double* A = sm + (size_t)warp * (D * LD + D);
  double* col = A + D * LD;
  __shared__ int perm[WPB][D];
  if (K >= npatch) return;
  const double* src = mats + (size_t)K * D * D;
  for (int idx = lane; idx < D * D; idx += 32) A[(idx / D) * LD + idx % D] = src[idx];
  __syncwarp();
  bool singular = false;
  for (int k = 0; k < D; ++k) {
    double best = -1.0;
    int bi = D;
    for (int i = k + lane; i < D; i += 32) {
      const double v = fabs(A[i * LD + k]);
      if (v > best || (v == best && i < bi)) {
        best = v;
        bi = i;
      }
    }
    for (int off = 16; off > 0; off >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (ov > best || (ov == best && oi < bi)) {
        best = ov;
        bi = oi;
      }
    }
    if (!(best > 0.0)) {
      singular = true;
      break;
    }
    if (lane == 0) perm[warp][k] = bi;
    if (bi != k)
      for (int jj = lane; jj < D; jj += 32) {
        const double tmp = A[k * LD + jj];
        A[k * LD + jj] = A[bi * LD + jj];
        A[bi * LD + jj] = tmp;
      }
    __syncwarp();
    const double pivinv = 1.0 / A[k * LD + k];
    __syncwarp();
    for (int jj = lane; jj < D; jj += 32) A[k * LD + jj] = (jj == k ? 1.0 : A[k * LD + jj]) * pivinv;
    for (int i = lane; i < D; i += 32) col[i] = A[i * LD + k];
    __syncwarp();
    // a lane takes whole columns: the pivot-row entry stays in a register, no index division,
    // conflict-free column accesses (same arithmetic per entry as an entry-wise sweep)
    for (int jj = lane; jj < D; jj += 32) {
      const double pk = A[k * LD + jj];
      const bool pc = jj == k;
#pragma unroll 6
      for (int i = 0; i < D; ++i) {
        if (i == k) continue;
        const double base = pc ? 0.0 : A[i * LD + jj];
        A[i * LD + jj] = base - col[i] * pk;
      }
    }
    __syncwarp();
  }
  if (singular) {
    if (lane == 0) atomicMin(bad, K);
    return;
  }
  // unscramble the columns in reverse pivot order
  for (int k = D - 1; k >= 0; --k) {
    const int p = perm[warp][k];
    if (p != k)
      for (int i = lane; i < D; i += 32) {
        const double tmp = A[i * LD + k];
        A[i * LD + k] = A[i * LD + p];
        A[i * LD + p] = tmp;
      }
    __syncwarp();
  }
  double* dst = invT + (size_t)K * D * D;
  for (int idx = lane; idx < D * D; idx += 32) {
    const int jj = idx / D, i = idx - jj * D;
    dst[idx] = A[i * LD + jj];
  }
}

// The same inversion for D <= 42 with the matrix in REGISTERS: lane l holds
// rows l and l + 32 (D = 42: lanes 0-9 two rows), no physical row swaps (the
// pivot row is the unused row with the largest |entry|, ties to the lower
// row; lane / slot p_k that pivoted column k ends up holding row k of the
// inverse with entry j standing for column p_j, undone on the store as in
// k_invert_diag).  Per step the pivot row goes through shared memory, where
// lane j scales entry j by 1 / pivot, and every lane eliminates its rows with
// it: D DFMA per row and step, D / 2 16-byte shared loads per warp and step -
// the shared-memory kernel above moves three words per DFMA and is bound by
// that.  Same operations per entry (scaled pivot row, fma(-f, P_j, R_j)).
template <int D>
__global__ void __launch_bounds__(128, D > 32 ? 2 : 4) k_invert_rows(const double* __restrict__ mats,
                                                                   double* __restrict__ invT, int npatch,
                                                                   int* __restrict__ bad) {
  constexpr int WPB = 4, NS = (D + 31) / 32, DP = (D + 1) & ~1;
  __shared__ __align__(16) double prow[WPB][DP];
  __shared__ int piv[WPB][D];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = blockIdx.x * WPB + warp;
  if (K >= npatch) return;
  const double* src = mats + (size_t)K * D * D;
  double R[NS][D];
  bool used[NS];
  int mycol[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const int r = lane + 32 * s;
    used[s] = r >= D;
    mycol[s] = -1;
#pragma unroll
    for (int j = 0; j < D; ++j) R[s][j] = r < D ? __ldg(src + (size_t)r * D + j) : 0.0;
  }
  if (lane == 0 && DP > D) prow[warp][DP - 1] = 0.0;
  bool singular = false;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    double best = -1.0;
    int bi = 64;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const double v = fabs(R[s][k]);
      if (!used[s] && v > best) {
        best = v;
        bi = lane + 32 * s;
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (ov > best || (ov == best && oi < bi)) {
        best = ov;
        bi = oi;
      }
    }
    if (!(best > 0.0)) {
      singular = true;
      break;
    }
    const int pl = bi & 31, ps = bi >> 5;
    double pv = R[0][k];
    if (NS > 1 && ps) pv = R[NS - 1][k];
    const double pinv = 1.0 / __shfl_sync(0xffffffffu, pv, pl);
    if (lane == pl) {  // the pivot row goes to shared memory as it is
#pragma unroll
      for (int s = 0; s < NS; ++s)
        if (ps == s) {
#pragma unroll
          for (int j = 0; j < D; ++j) prow[warp][j] = R[s][j];
          used[s] = true;
          mycol[s] = k;
        }
      piv[warp][k] = bi;
    }
    __syncwarp();
#pragma unroll
    for (int s = 0; s < NS; ++s) {  // lane j scales entry j
      const int j = lane + 32 * s;
      if (j < D) prow[warp][j] = (j == k ? 1.0 : prow[warp][j]) * pinv;
    }
    __syncwarp();
    double f[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) f[s] = R[s][k];
#pragma unroll
    for (int j2 = 0; j2 < DP / 2; ++j2) {
      if (NS > 1 && j2 % 3 == 0) asm volatile("" ::: "memory");  // keep the row loads from piling up in registers
      const double2 a = reinterpret_cast<const double2*>(prow[warp])[j2];
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        R[s][2 * j2] = fma(-f[s], a.x, 2 * j2 == k ? 0.0 : R[s][2 * j2]);
        if (2 * j2 + 1 < D) R[s][2 * j2 + 1] = fma(-f[s], a.y, 2 * j2 + 1 == k ? 0.0 : R[s][2 * j2 + 1]);
      }
    }
    if (lane == pl) {  // the pivot lane takes its scaled row back (its own elimination result is discarded)
#pragma unroll
      for (int s = 0; s < NS; ++s)
        if (ps == s) {
#pragma unroll
          for (int j = 0; j < D; ++j) R[s][j] = prow[warp][j];
        }
    }
    __syncwarp();
  }
  if (singular) {
    if (lane == 0) atomicMin(bad, K);
    return;
  }
  double* dst = invT + (size_t)K * D * D;
#pragma unroll
  for (int s = 0; s < NS; ++s)
    if (lane + 32 * s < D) {
#pragma unroll
      for (int j = 0; j < D; ++j) dst[(size_t)piv[warp][j] * D + mycol[s]] = R[s][j];
    }
}

// Slab dof of local patch position l of cell K.
__device__ __forceinline__ size_t patch_dof(const Geom& g, int K, int l) {
  const int mu = l / 21, s = l % 21;
  const size_t base = (size_t)mu * g.nd;
  if (s >= 18) return base + g.mv + 3 * (size_t)K + (s - 18);
  const int a = s >> 1, d = s & 1;
  const int ki = K % g.nx, kj = K / g.nx;
  return base + 2 * ((size_t)(2 * kj + a / 3) * g.nnx + 2 * ki + a % 3) + d;
}

// upd_K = A_K^{-1} defect[ids_K]; threads (patch, row) read invT columns coalesced.
template <int D>
__global__ void __launch_bounds__(256) k_vanka_gemv(Geom g, const double* __restrict__ invT,
                                                    const double* __restrict__ defect, double* __restrict__ upd) {
  constexpr int PB = 256 / D;
  __shared__ double loc[PB][D];
  const int p = threadIdx.x / D, i = threadIdx.x % D;
  const int K = blockIdx.x * PB + p;
  const bool active = p < PB && K < g.ncells;
  if (active) loc[p][i] = __ldg(defect + patch_dof(g, K, i));
  __syncthreads();
  if (!active) return;
  const double* col = invT + (size_t)K * D * D + i;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int jj = 0;
#pragma unroll 4
  for (; jj + 3 < D; jj += 4) {
    s0 = fma(__ldg(col + (size_t)jj * D), loc[p][jj], s0);
    s1 = fma(__ldg(col + (size_t)(jj + 1) * D), loc[p][jj + 1], s1);
    s2 = fma(__ldg(col + (size_t)(jj + 2) * D), loc[p][jj + 2], s2);
    s3 = fma(__ldg(col + (size_t)(jj + 3) * D), loc[p][jj + 3], s3);
  }
  for (; jj < D; ++jj) s0 = fma(__ldg(col + (size_t)jj * D), loc[p][jj], s0);
  upd[(size_t)i * g.ncells + K] = (s0 + s1) + (s2 + s3);  // structure of arrays [D][ncells]
}

// d += omega * sum_K R_K' upd_K, one thread per (cell, Radau node): the cell
// writes the nodes it owns (lower-left 2x2 of its 3x3 block, plus the last
// row / column of the mesh) summing the <= 4 patches containing each node in a
// fixed order (down-left, down, left, self), both velocity components of a
// node as one 16-byte pair when the node plane is 16-byte aligned (VEC), and
// the cell's 3 pressure dofs.  upd is structure of arrays [21 k1][ncells], so
// every read is coalesced; all loads are issued before the first store.
// Only patches of cell rows [row_lo, row_hi) contribute; inc_only writes the
// increment instead of adding it (distributed sweeps combine increments).
// inc_row (optional): omega * (sum of the contributing patches) of node row
// inc_Y is also written there, [mu][2 nnx] (the increment a strip partition's
// upper neighbour adds to its own row, csrc/pdst_strip.cu).
template <bool VEC>
__global__ void __launch_bounds__(256, 4) k_vanka_scatter(Geom g, int k1, const double* __restrict__ upd, double omega,
                                                       double* __restrict__ d, int row_lo, int row_hi,
                                                       int inc_only, double* __restrict__ inc_row, int inc_Y) {
  STEP_MARK(5, 0);
  pdl_wait();  // PDL-launched behind the GEMV that writes upd
  STEP_MARK(5, 1);
  const size_t c = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int mu = blockIdx.y;
  if (c >= (size_t)g.ncells) return;
  const int ci = (int)(c % g.nx), cj = (int)(c / g.nx);
  const size_t nc = g.ncells;
  const double* u = upd + (size_t)21 * mu * nc;  // u[(2a + comp) * nc + cell]
  double* dm = d + (size_t)mu * g.nd;
  const bool me = cj >= row_lo && cj < row_hi;
  const bool hd = cj > 0 && cj - 1 >= row_lo && cj - 1 < row_hi;
  const bool lastx = ci == g.nx - 1, lasty = cj == g.ny - 1;
  // neighbour cells (clamped to self when absent; their values are masked to 0)
  const size_t cl = ci > 0 ? c - 1 : c, cd = cj > 0 ? c - g.nx : c, cld = (ci > 0 && cj > 0) ? c - g.nx - 1 : c;
  const double ml = (ci > 0 && me) ? 1.0 : 0.0, md = hd ? 1.0 : 0.0, mld = (hd && ci > 0) ? 1.0 : 0.0;
  const double ms = me ? 1.0 : 0.0;
  auto U = [&](size_t cell, int a, int dd) { return __ldg(u + (size_t)(2 * a + dd) * nc + cell); };
  auto node = [&](int r, int cc) { return dm + 2 * ((size_t)(2 * cj + r) * g.nnx + 2 * ci + cc); };
  auto load2 = [&](const double* p, double* v) {
    if (VEC) {
      const double2 t = *reinterpret_cast<const double2*>(p);
      v[0] = t.x, v[1] = t.y;
    } else {
      v[0] = p[0], v[1] = p[1];
    }
  };
  auto store2 = [&](double* p, const double* o, const double* sv) {
    const double v0 = inc_only ? omega * sv[0] : o[0] + omega * sv[0];
    const double v1 = inc_only ? omega * sv[1] : o[1] + omega * sv[1];
    if (inc_row) {
      const size_t node = (size_t)(p - dm) / 2;  // node index in the Radau plane
      if ((int)(node / g.nnx) == inc_Y) {
        double* q = inc_row + (size_t)mu * 2 * g.nnx + 2 * (node % g.nnx);
        q[0] = omega * sv[0];
        q[1] = omega * sv[1];
      }
    }
    if (VEC) {
      *reinterpret_cast<double2*>(p) = make_double2(v0, v1);
    } else {
      p[0] = v0, p[1] = v1;
    }
  };
  double pv[3], po[3] = {0.0, 0.0, 0.0};
  double* op = dm + g.mv + 3 * c;
  {  // the 4 nodes every cell owns: local nodes 0, 1, 3, 4 (all loads first)
    double s[4][2], o[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
    for (int dd = 0; dd < 2; ++dd) {
      s[0][dd] = ((0.0 + mld * U(cld, 8, dd)) + md * U(cd, 6, dd)) + ml * U(cl, 2, dd) + ms * U(c, 0, dd);
      s[1][dd] = (0.0 + md * U(cd, 7, dd)) + ms * U(c, 1, dd);
      s[2][dd] = (0.0 + ml * U(cl, 5, dd)) + ms * U(c, 3, dd);
      s[3][dd] = 0.0 + ms * U(c, 4, dd);
    }
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      pv[j] = __ldg(upd + (size_t)(21 * mu + 18 + j) * nc + c);
      if (!inc_only) po[j] = op[j];
    }
    if (!inc_only) {
      load2(node(0, 0), o[0]);
      load2(node(0, 1), o[1]);
      load2(node(1, 0), o[2]);
      load2(node(1, 1), o[3]);
    }
    store2(node(0, 0), o[0], s[0]);
    store2(node(0, 1), o[1], s[1]);
    store2(node(1, 0), o[2], s[2]);
    store2(node(1, 1), o[3], s[3]);
  }
  // the mesh's last node column / row: local nodes 2, 5 / 6, 7 / 8
  if (lastx || lasty) {
    double s[2], o[2] = {0.0, 0.0};
    auto one = [&](int r, int cc, int a, int na, size_t ncell, double m) {
#pragma unroll
      for (int dd = 0; dd < 2; ++dd) s[dd] = na >= 0 ? (0.0 + m * U(ncell, na, dd)) + ms * U(c, a, dd) : 0.0 + ms * U(c, a, dd);
      if (!inc_only) load2(node(r, cc), o);
      store2(node(r, cc), o, s);
    };
    if (lastx) {
      one(0, 2, 2, 8, cd, md);  // (2,0): down, self
      one(1, 2, 5, -1, c, 0.0);
    }
    if (lasty) {
      one(2, 0, 6, 8, cl, ml);  // (0,2): left, self
      one(2, 1, 7, -1, c, 0.0);
      if (lastx) one(2, 2, 8, -1, c, 0.0);
    }
  }
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const double v = me ? omega * pv[j] : 0.0;
    op[j] = inc_only ? v : po[j] + v;
  }
  STEP_MARK(5, 2);
}

template <int D>
cudaError_t launch_invert(const double* mats, double* invT, int np, int* bad, cudaStream_t st) {
  if constexpr (D <= 42) {
    PDST_LAUNCH(k_invert_rows<D><<<(np + 3) / 4, 128, 0, st>>>(mats, invT, np, bad));
    return cudaGetLastError();
  }
  constexpr int WPB = inv_wpb<D>();
  const size_t smem = (size_t)WPB * (D * (D + 1) + D) * sizeof(double);
  static DeviceOnce once;
  const int dev = current_device();
  if (!once.done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_invert<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    once.done[dev] = true;
  }
  PDST_LAUNCH(k_invert<D><<<(np + WPB - 1) / WPB, 32 * WPB, smem, st>>>(mats, invT, np, bad));
  return cudaGetLastError();
}

template <int D>
cudaError_t launch_gemv(const Geom& g, const double* invT, const double* defect, double* upd, cudaStream_t st) {
  constexpr int PB = 256 / D;
  PDST_LAUNCH(k_vanka_gemv<D><<<(g.ncells + PB - 1) / PB, 256, 0, st>>>(g, invT, defect, upd));
  return cudaGetLastError();
}

}  // namespace

cudaError_t patch_assemble(const PatchArgs& a, cudaStream_t st) {
  PDST_LAUNCH(k_patch_fine<<<a.g.ncells, 448, 0, st>>>(a));
  return cudaGetLastError();
}

cudaError_t patch_invert(int k1, const double* mats, double* invT, int npatch, int* bad, cudaStream_t st) {
  switch (k1) {
    case 1: return launch_invert<21>(mats, invT, npatch, bad, st);
    case 2: return launch_invert<42>(mats, invT, npatch, bad, st);
    case 3: return launch_invert<63>(mats, invT, npatch, bad, st);
    case 4: return launch_invert<84>(mats, invT, npatch, bad, st);
    default: return cudaErrorNotSupported;
  }
}

cudaError_t vanka_gemv(const Geom& g, int k1, const double* invT, const double* defect, double* upd, cudaStream_t st) {
  cudaError_t e = cudaSuccess;
  if (vanka_gemv_exact_tma(g, k1, invT, defect, upd, st, &e)) return e;
  switch (k1) {
    case 1: return launch_gemv<21>(g, invT, defect, upd, st);
    case 2: return launch_gemv<42>(g, invT, defect, upd, st);
    case 3: return launch_gemv<63>(g, invT, defect, upd, st);
    case 4: return launch_gemv<84>(g, invT, defect, upd, st);
    default: return cudaErrorNotSupported;
  }
}

cudaError_t vanka_scatter(const Geom& g, int k1, const double* upd, double omega, double* d, cudaStream_t st,
                          int row_lo, int row_hi, bool inc_only, double* inc_row, int inc_Y) {
  if (row_hi < 0) row_hi = g.ny;
  dim3 grid((unsigned)((g.ncells + 255) / 256), k1);
  // node pairs (2 node, 2 node + 1) are 16-byte aligned in every Radau plane
  const bool vec = (g.nd % 2 == 0 || k1 == 1) && ((uintptr_t)d % 16 == 0);
  cudaError_t e;
  auto kern = vec ? k_vanka_scatter<true> : k_vanka_scatter<false>;
  PDST_LAUNCH(e = launch_pdl(kern, grid, dim3(256), 0, st, g, k1, upd, omega, d, row_lo, row_hi, inc_only ? 1 : 0,
                             inc_row, inc_Y));
  return e;
}

}  // namespace pdst
