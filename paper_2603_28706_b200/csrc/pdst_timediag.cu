// pdst_timediag.cu — temporally diagonalized surrogate Vanka patches.
//
// A surrogate patch (solver/multigrid.py:475-488) uses ONE spatial block for
// every Radau node, so
//   A_K = K_t (x) Mhat + W (x) Jhat,   W = diag(tau w_mu),
// with Mhat the 21x21 patch mass (zero pressure rows/cols) and Jhat the
// 21x21 surrogate spatial block.  With S = W^-1 K_t = V diag(lam) V^-1,
//   A_K^-1 = (V (x) I) blockdiag_i[(lam_i Mhat + Jhat)^-1] (V^-1 W^-1 (x) I).
// The Radau eigenvalues of S come in complex-conjugate pairs (plus one real
// eigenvalue for odd k+1), so each patch stores one complex 21x21 inverse per
// pair and one real 21x21 inverse per real eigenvalue: 882 doubles instead of
// 42^2 = 1764 for DG(1), 882 + 442 (one pad) instead of 63^2 = 3969 for DG(2),
// 442 instead of 441 for DG(0).  The Vanka sweep streams those bytes.  Mathematically identical to
// np.linalg.inv(A_K) @ e (multigrid.py:290-291, 338); rounding differs.
#include <cuda_runtime.h>

#include <cmath>
#include <complex>

#include <algorithm>

#include "pdst_device.cuh"
#include "pdst_patch.h"

namespace pdst {

using cplx = std::complex<double>;

namespace {

// Complex Gauss-Jordan inverse of an n x n matrix (n <= 7), partial pivoting.
bool cinv(int n, cplx* A /* row-major, in/out */) {
  int perm[MAXK1];
  for (int k = 0; k < n; ++k) {
    int p = k;
    double best = std::abs(A[k * n + k]);
    for (int i = k + 1; i < n; ++i)
      if (std::abs(A[i * n + k]) > best) {
        best = std::abs(A[i * n + k]);
        p = i;
      }
    if (!(best > 0.0)) return false;
    perm[k] = p;
    if (p != k)
      for (int j = 0; j < n; ++j) std::swap(A[k * n + j], A[p * n + j]);
    const cplx pinv = 1.0 / A[k * n + k];
    A[k * n + k] = 1.0;
    for (int j = 0; j < n; ++j) A[k * n + j] *= pinv;
    for (int i = 0; i < n; ++i) {
      if (i == k) continue;
      const cplx f = A[i * n + k];
      A[i * n + k] = 0.0;
      for (int j = 0; j < n; ++j) A[i * n + j] -= f * A[k * n + j];
    }
  }
  for (int k = n - 1; k >= 0; --k)
    if (perm[k] != k)
      for (int i = 0; i < n; ++i) std::swap(A[i * n + k], A[i * n + perm[k]]);
  return true;
}

// Eigenvalues of a real n x n matrix via Durand-Kerner on the characteristic
// polynomial (Faddeev-LeVerrier), n <= 7, after scaling to unit magnitude.
bool eigenvalues(int n, const double* S, cplx* lam) {
  double scale = 0.0;
  for (int i = 0; i < n * n; ++i) scale = std::max(scale, std::fabs(S[i]));
  if (!(scale > 0.0)) return false;
  double A[MAXK1 * MAXK1], M[MAXK1 * MAXK1], AM[MAXK1 * MAXK1], c[MAXK1 + 1];
  for (int i = 0; i < n * n; ++i) A[i] = S[i] / scale;
  // Faddeev-LeVerrier: p(x) = x^n + c1 x^(n-1) + ... + cn
  for (int i = 0; i < n * n; ++i) M[i] = 0.0;
  c[0] = 1.0;
  for (int k = 1; k <= n; ++k) {
    // M = A M_prev + c_{k-1} I
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        double s = 0.0;
        for (int l = 0; l < n; ++l) s += A[i * n + l] * M[l * n + j];
        AM[i * n + j] = s + (i == j ? c[k - 1] : 0.0);
      }
    for (int i = 0; i < n * n; ++i) M[i] = AM[i];
    double tr = 0.0;
    for (int i = 0; i < n; ++i)
      for (int l = 0; l < n; ++l) tr += A[i * n + l] * M[l * n + i];
    c[k] = -tr / k;
  }
  auto poly = [&](cplx x) {
    cplx v = 1.0;
    for (int k = 1; k <= n; ++k) v = v * x + c[k];
    return v;
  };
  cplx z[MAXK1];
  const cplx seed(0.4, 0.9);
  z[0] = 1.0;
  for (int i = 0; i < n; ++i) z[i] = std::pow(seed, i + 1) * 1.5;
  for (int it = 0; it < 500; ++it) {
    double delta = 0.0;
    for (int i = 0; i < n; ++i) {
      cplx den = 1.0;
      for (int j = 0; j < n; ++j)
        if (j != i) den *= (z[i] - z[j]);
      if (std::abs(den) == 0.0) return false;
      const cplx dz = poly(z[i]) / den;
      z[i] -= dz;
      delta = std::max(delta, std::abs(dz));
    }
    if (delta < 1e-17) break;
  }
  for (int i = 0; i < n; ++i) lam[i] = z[i] * scale;
  return true;
}

}  // namespace

bool time_diagonalize(int k1, const double* K_t, const double* tau_w, TimeDiag& out) {
  out = TimeDiag{};
  out.k1 = k1;
  if (k1 < 1 || k1 > 4) return false;
  double S[MAXK1 * MAXK1];
  for (int i = 0; i < k1; ++i) {
    out.itw[i] = 1.0 / tau_w[i];
    for (int j = 0; j < k1; ++j) S[i * k1 + j] = K_t[i * k1 + j] / tau_w[i];
  }
  cplx lam[MAXK1];
  if (k1 == 1) {
    lam[0] = S[0];
  } else if (!eigenvalues(k1, S, lam)) {
    return false;
  }
  // Newton-polish each eigenvalue on det(S - lam I) via inverse iteration
  cplx V[MAXK1 * MAXK1];
  double snorm = 0.0;
  for (int i = 0; i < k1 * k1; ++i) snorm = std::max(snorm, std::fabs(S[i]));
  for (int b = 0; b < k1; ++b) {
    // snap near-real eigenvalues to the real axis
    if (std::fabs(lam[b].imag()) < 1e-12 * std::abs(lam[b])) lam[b] = cplx(lam[b].real(), 0.0);
    cplx v[MAXK1];
    for (int i = 0; i < k1; ++i) v[i] = cplx(1.0 + 0.1 * i, 0.05 * i);
    for (int it = 0; it < 4; ++it) {
      cplx A[MAXK1 * MAXK1];
      const cplx shift = lam[b] + cplx(1e-11 * snorm, 0.0);
      for (int i = 0; i < k1; ++i)
        for (int j = 0; j < k1; ++j) A[i * k1 + j] = S[i * k1 + j] - (i == j ? shift : 0.0);
      if (!cinv(k1, A)) return false;
      cplx w[MAXK1];
      double nrm = 0.0;
      for (int i = 0; i < k1; ++i) {
        w[i] = 0.0;
        for (int j = 0; j < k1; ++j) w[i] += A[i * k1 + j] * v[j];
        nrm = std::max(nrm, std::abs(w[i]));
      }
      for (int i = 0; i < k1; ++i) v[i] = w[i] / nrm;
      // Rayleigh-type refinement of lam
      cplx num = 0.0, den = 0.0;
      for (int i = 0; i < k1; ++i) {
        cplx sv = 0.0;
        for (int j = 0; j < k1; ++j) sv += S[i * k1 + j] * v[j];
        num += std::conj(v[i]) * sv;
        den += std::conj(v[i]) * v[i];
      }
      if (lam[b].imag() != 0.0) lam[b] = num / den;
      else lam[b] = cplx((num / den).real(), 0.0);
    }
    if (lam[b].imag() == 0.0)
      for (int i = 0; i < k1; ++i) v[i] = cplx(v[i].real(), 0.0);
    for (int i = 0; i < k1; ++i) V[i * k1 + b] = v[i];
  }
  // enforce exact conjugate pairs: for each lam with Im > 0 find its partner
  bool used[MAXK1] = {false};
  int keep[MAXK1], nk = 0, partner[MAXK1];
  for (int b = 0; b < k1; ++b) partner[b] = -1;
  for (int b = 0; b < k1; ++b) {
    if (used[b]) continue;
    used[b] = true;
    if (lam[b].imag() == 0.0) {
      keep[nk++] = b;
      continue;
    }
    int best = -1;
    double bd = 1e300;
    for (int c = 0; c < k1; ++c)
      if (!used[c]) {
        const double d = std::abs(lam[c] - std::conj(lam[b]));
        if (d < bd) {
          bd = d;
          best = c;
        }
      }
    if (best < 0 || bd > 1e-8 * std::abs(lam[b])) return false;
    used[best] = true;
    const int pos = lam[b].imag() > 0.0 ? b : best, neg = pos == b ? best : b;
    lam[neg] = std::conj(lam[pos]);
    for (int i = 0; i < k1; ++i) V[i * k1 + neg] = std::conj(V[i * k1 + pos]);
    keep[nk++] = pos;
    partner[pos] = neg;
  }
  cplx Vi[MAXK1 * MAXK1];
  for (int i = 0; i < k1 * k1; ++i) Vi[i] = V[i];
  if (!cinv(k1, Vi)) return false;
  // residual check |S V - V Lam| and conditioning
  double res = 0.0, vn = 0.0, vin = 0.0;
  for (int i = 0; i < k1; ++i)
    for (int b = 0; b < k1; ++b) {
      cplx sv = 0.0;
      for (int j = 0; j < k1; ++j) sv += S[i * k1 + j] * V[j * k1 + b];
      res = std::max(res, std::abs(sv - lam[b] * V[i * k1 + b]));
      vn = std::max(vn, std::abs(V[i * k1 + b]));
      vin = std::max(vin, std::abs(Vi[i * k1 + b]));
    }
  if (!(res <= 1e-12 * snorm * vn) || !(vn * vin < 1e6)) return false;
  out.nblk = nk;
  int off = 0;
  for (int s = 0; s < nk; ++s) {
    const int b = keep[s];
    out.pair[s] = partner[b] >= 0 ? 1 : 0;
    out.boff[s] = off;
    off += out.pair[s] ? 882 : 442;
    out.lam_re[s] = lam[b].real();
    out.lam_im[s] = lam[b].imag();
    for (int mu = 0; mu < k1; ++mu) {
      out.V_re[mu * MAXK1 + s] = V[mu * k1 + b].real();
      out.V_im[mu * MAXK1 + s] = V[mu * k1 + b].imag();
      out.Vi_re[s * MAXK1 + mu] = Vi[b * k1 + mu].real();
      out.Vi_im[s * MAXK1 + mu] = Vi[b * k1 + mu].imag();
    }
  }
  out.pstride = off;
  return true;
}

namespace {

__device__ __forceinline__ double m1g_d(int X, int Xp, int n) {
  double s = 0.0;
  const int lo = max(0, (max(X, Xp) - 1) / 2);
  for (int c = lo; c <= min(X, Xp) / 2 && c < n; ++c) {
    const int a = X - 2 * c, b = Xp - 2 * c;
    if (a >= 0 && a <= 2 && b >= 0 && b <= 2) s += c_tab.M1[a][b];
  }
  return s;
}

__device__ __forceinline__ double cabs1(double2 z) { return fabs(z.x) + fabs(z.y); }

// One warp per (patch, stored eigen-block): C = lam Mhat + Jhat (21x21
// complex), lane r < 21 holding row r in REGISTERS, Gauss-Jordan by exchange
// steps with partial pivoting (the pivot row is chosen among the rows not yet
// used by the largest |Re| + |Im| as izamax / dcabs1 in zgetrf, ties to the
// lower row) and no physical row swaps: the pivot row goes through shared
// memory, where lane j scales its entry j by 1 / pivot (one complex product
// per lane instead of 21 on the pivot lane alone), the pivot lane reads the
// scaled row back and the other lanes eliminate with it (4 DFMA per entry).
// The in-place Gauss-Jordan with row swaps, operation for operation, up to
// the fused roundings; after all steps lane p_k holds row k of the inverse with its
// column k' standing for column p_k' (tableau exchange), undone on the store.
// Output transposed: binvT[K][b][col][row].
__global__ void __launch_bounds__(128, 3) k_invert_diag(Geom g, TimeDiag td, const double* __restrict__ spatial,
                                                     double* __restrict__ binvT, int* __restrict__ bad) {
  constexpr int N = 21, WPB = 4;
  __shared__ double2 prow[WPB][N];  // the current pivot row
  __shared__ int piv[WPB][N];       // piv[k] = lane that pivoted column k
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int task = blockIdx.x * WPB + warp;
  if (task >= g.ncells * td.nblk) return;
  const int K = task / td.nblk, b = task % td.nblk;
  const int ki = K % g.nx, kj = K / g.nx;
  const double lr = td.lam_re[b], li = td.lam_im[b];
  const bool row = lane < N;
  // the patch's assembled 1-D mass factors between its three node columns /
  // rows, once per warp (they only differ from the interior values next to
  // the mesh boundary): m1[0..8] x direction, m1[9..17] y direction
  __shared__ double m1[WPB][18];
  if (lane < 9)
    m1[warp][lane] = m1g_d(2 * ki + lane / 3, 2 * ki + lane % 3, g.nx);
  else if (lane < 18)
    m1[warp][lane] = m1g_d(2 * kj + (lane - 9) / 3, 2 * kj + (lane - 9) % 3, g.ny);
  __syncwarp();
  double2 R[N];
#pragma unroll
  for (int j = 0; j < N; ++j) {
    double m = 0.0, jv = 0.0;
    if (row) {
      if (lane < 18 && j < 18 && (lane & 1) == (j & 1)) {
        const int ia = lane >> 1, jb = j >> 1;
        m = g.hx * g.hy * (m1[warp][9 + 3 * (ia / 3) + jb / 3] * m1[warp][3 * (ia % 3) + jb % 3]);
      }
      jv = spatial[(size_t)K * 441 + lane * N + j];
    }
    R[j] = make_double2(fma(lr, m, jv), li * m);
  }
  bool used = !row;
  int mycol = -1;
  bool singular = false;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    double best = used ? -1.0 : cabs1(R[k]);
    int bi = used ? 32 : lane;
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
    // 1 / pivot on every lane (the pivot value broadcast by shuffle)
    const double px = __shfl_sync(0xffffffffu, R[k].x, bi), py = __shfl_sync(0xffffffffu, R[k].y, bi);
    const double den = px * px + py * py;
    const double2 pinv = make_double2(px / den, -py / den);
    if (lane == bi) {  // the pivot row goes to shared memory as it is
#pragma unroll
      for (int j = 0; j < N; ++j) prow[warp][j] = R[j];
      piv[warp][k] = lane;
      used = true;
      mycol = k;
    }
    __syncwarp();
    if (row) {  // lane j scales entry j: P[k] <- 1 / pivot, P[j] <- P[j] / pivot
      const double2 a = (lane == k) ? make_double2(1.0, 0.0) : prow[warp][lane];
      prow[warp][lane] = make_double2(a.x * pinv.x - a.y * pinv.y, a.x * pinv.y + a.y * pinv.x);
    }
    __syncwarp();
    if (lane == bi) {  // the pivot lane takes its scaled row back
#pragma unroll
      for (int j = 0; j < N; ++j) R[j] = prow[warp][j];
    } else if (row) {  // the others eliminate column k: R[j] -= f P[j], R[k] = -f P[k]
      const double2 f = R[k];
#pragma unroll
      for (int j = 0; j < N; ++j) {
        const double2 base = (j == k) ? make_double2(0.0, 0.0) : R[j];
        const double2 a = prow[warp][j];
        R[j] = make_double2(fma(f.y, a.y, fma(-f.x, a.x, base.x)), fma(-f.y, a.x, fma(-f.x, a.y, base.y)));
      }
    }
    __syncwarp();
  }
  if (singular) {
    if (lane == 0) atomicMin(bad, K);
    return;
  }
  // lane p_k holds row k = mycol of the inverse; its entry j is column piv[j]
  double* base = binvT + (size_t)K * td.pstride + td.boff[b];
  if (row) {
    if (td.pair[b]) {
      double2* dst = reinterpret_cast<double2*>(base);
#pragma unroll
      for (int j = 0; j < N; ++j) dst[piv[warp][j] * N + mycol] = R[j];
    } else {  // real eigenvalue: the inverse is real (every imaginary part is an exact 0)
#pragma unroll
      for (int j = 0; j < N; ++j) base[piv[warp][j] * N + mycol] = R[j].x;
      if (lane == 0) base[N * N] = 0.0;  // pad
    }
  }
}

__device__ __forceinline__ size_t patch_dof_d(const Geom& g, int K, int l) {
  const int mu = l / 21, s = l % 21;
  const size_t base = (size_t)mu * g.nd;
  if (s >= 18) return base + g.mv + 3 * (size_t)K + (s - 18);
  const int a = s >> 1, d = s & 1;
  const int ki = K % g.nx, kj = K / g.nx;
  return base + 2 * ((size_t)(2 * kj + a / 3) * g.nnx + 2 * ki + a % 3) + d;
}

// ---------------------------------------------------------------------------
// The same GEMV as a persistent, TMA-fed pipeline: one CTA per SM streams the
// patch inverses of groups of PB patches through an S-stage shared-memory ring
// with bulk copies (cp.async.bulk, completion counted in bytes on an
// mbarrier), so S-1 groups are always in flight regardless of what the warps
// are doing; the warps gather the next group's defect while multiplying the
// current one out of shared memory.  Same arithmetic (and summation order) as
// the row-per-thread GEMV it replaces (88 -> 84 us at cfg2).
//   upd_K = A_K^-1 e_K via the temporal diagonalization; threads (patch, row r).
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// Pipeline shape per stored block count: PB patches per group, STAGES groups
// in flight per CTA, 2 CTAs per SM; threads (patch p, block b, row r).
template <int NB>
__host__ __device__ constexpr int tma_pb() { return NB == 1 ? 4 : NB == 2 ? 4 : 2; }
template <int NB>
__host__ __device__ constexpr int tma_stages() { return NB == 1 ? 3 : 2; }
constexpr int TMA_CTAS_PER_SM = 2;
template <int NB>
__host__ __device__ constexpr size_t tma_smem_max() { return (size_t)tma_stages<NB>() * tma_pb<NB>() * NB * 882 * 8; }

template <int K1, int NB>
__global__ void __launch_bounds__(tma_pb<NB>() * NB * 21, TMA_CTAS_PER_SM) k_vanka_gemv_diag_tma(Geom g, TimeDiag td,
                                                                           const double* __restrict__ binvT,
                                                                           const double* __restrict__ defect,
                                                                           double* __restrict__ upd, int ngroups) {
  constexpr int PB = tma_pb<NB>(), STAGES = tma_stages<NB>();
  const unsigned PBYTES = (unsigned)td.pstride * 8u;
  extern __shared__ __align__(128) unsigned char tma_ring[];
  __shared__ double2 gs[2][PB][NB][21];               // eigen-transformed defects, double buffered
  __shared__ double2 hs[NB > 1 ? 2 : 1][PB][NB][21];  // per-block products (NB > 1), double buffered
  __shared__ __align__(8) uint64_t full[STAGES];
  const int p = threadIdx.x / (21 * NB), b = (threadIdx.x / 21) % NB, r = threadIdx.x % 21;
  auto stage_ptr = [&](int st) { return reinterpret_cast<double*>(tma_ring + (size_t)st * PB * PBYTES); };
  auto issue = [&](int gi, int st) {  // one thread: arm the stage's barrier and start its copies
    const int K0 = gi * PB, cnt = min(PB, g.ncells - K0);
    mbar_expect_tx(&full[st], (unsigned)cnt * PBYTES);
    for (int q = 0; q < cnt; ++q)
      bulk_g2s(stage_ptr(st) + (size_t)q * td.pstride, binvT + (size_t)(K0 + q) * td.pstride, PBYTES, &full[st]);
  };
  // defect of this thread's (patch, row) in group gi (the loads, issued early)
  auto load_defect = [&](int gi, double f[K1]) {
    const int K = gi * PB + p;
    if (gi < ngroups && K < g.ncells) {
#pragma unroll
      for (int mu = 0; mu < K1; ++mu) f[mu] = __ldg(defect + patch_dof_d(g, K, 21 * mu + r));
    }
  };
  auto transform = [&](const double f[K1], int buf) {  // this thread's block b
    double gr = 0.0, gi2 = 0.0;
#pragma unroll
    for (int mu = 0; mu < K1; ++mu) {
      gr = fma(td.Vi_re[b * MAXK1 + mu], f[mu] * td.itw[mu], gr);
      gi2 = fma(td.Vi_im[b * MAXK1 + mu], f[mu] * td.itw[mu], gi2);
    }
    gs[buf][p][b][r] = make_double2(gr, gi2);
  };
  // the mu output of (patch, row) from all blocks' products, blocks in order
  auto emit = [&](int K, const double* hr, const double* hi, int mu) {
    double sacc = 0.0;
#pragma unroll
    for (int bb = 0; bb < NB; ++bb) {
      const double re = td.V_re[mu * MAXK1 + bb] * hr[bb] - td.V_im[mu * MAXK1 + bb] * hi[bb];
      sacc += td.pair[bb] ? 2.0 * re : re;
    }
    upd[(size_t)(21 * mu + r) * g.ncells + K] = sacc;
  };
  pdl_trigger();
  STEP_MARK(4, 0);
  if (threadIdx.x == 0) {
    for (int st = 0; st < STAGES; ++st) mbar_init(&full[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    for (int st = 0; st < STAGES; ++st) {
      const int gi = blockIdx.x + st * gridDim.x;
      if (gi < ngroups) issue(gi, st);
    }
  }
  // launched with PDL: the inverse stream above does not depend on the
  // defect; everything below does (and upd may still be read by a predecessor)
  pdl_wait();
  STEP_MARK(4, 1);
  {
    double f[K1] = {};
    load_defect(blockIdx.x, f);
    transform(f, 0);
  }
  __syncthreads();
  int it = 0;
  for (int gi = blockIdx.x; gi < ngroups; gi += gridDim.x, ++it) {
    const int st = it % STAGES, buf = it & 1;
    const unsigned parity = (unsigned)(it / STAGES) & 1u;
    const int K = gi * PB + p;
    double fn[K1] = {};
    load_defect(gi + gridDim.x, fn);  // next group's defect, consumed after this group's product
    mbar_wait(&full[st], parity);
    if (K < g.ncells) {
      const double* blk = stage_ptr(st) + (size_t)p * td.pstride + td.boff[b];
      double hr, hi;
      if (td.pair[b]) {
        const double2* col = reinterpret_cast<const double2*>(blk) + r;
        double ar = 0.0, ai = 0.0, br = 0.0, bi = 0.0;
#pragma unroll 7
        for (int j = 0; j < 21; ++j) {
          const double2 m = col[21 * j];
          const double2 v = gs[buf][p][b][j];
          ar = fma(m.x, v.x, ar);
          br = fma(m.y, v.y, br);
          ai = fma(m.x, v.y, ai);
          bi = fma(m.y, v.x, bi);
        }
        hr = ar - br;
        hi = ai + bi;
      } else {  // real block, real transformed defect: half the bytes, same sums
        const double* col = blk + r;
        double ar = 0.0;
#pragma unroll 7
        for (int j = 0; j < 21; ++j) ar = fma(col[21 * j], gs[buf][p][b][j].x, ar);
        hr = ar;
        hi = 0.0;
      }
      if constexpr (NB == 1) {
#pragma unroll
        for (int mu = 0; mu < K1; ++mu) emit(K, &hr, &hi, mu);
      } else {
        hs[buf][p][b][r] = make_double2(hr, hi);
      }
    }
    transform(fn, buf ^ 1);
    __syncthreads();  // stage st is free, gs[buf ^ 1] and hs[buf] are complete
    if constexpr (NB > 1) {
      if (K < g.ncells) {
        double hrs[NB], his[NB];
#pragma unroll
        for (int bb = 0; bb < NB; ++bb) {
          const double2 h2 = hs[buf][p][bb][r];
          hrs[bb] = h2.x;
          his[bb] = h2.y;
        }
        for (int mu = b; mu < K1; mu += NB) emit(K, hrs, his, mu);
      }
    }
    if (threadIdx.x == 0) {
      const int gn = gi + STAGES * gridDim.x;
      if (gn < ngroups) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic reads before the async writes
        issue(gn, st);
      }
    }
  }
  STEP_MARK(4, 2);
}

template <int K1, int NB>
cudaError_t launch_gemv_tma(const Geom& g, const TimeDiag& td, const double* binvT, const double* defect,
                            double* upd, cudaStream_t st) {
  static DeviceOnce once;
  const size_t smax = tma_smem_max<NB>();
  const int dev = current_device();
  if (!once.done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_vanka_gemv_diag_tma<K1, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smax);
    if (e != cudaSuccess) return e;
    once.nsm[dev] = device_sms(dev);
    once.done[dev] = true;
  }
  const int nsm = once.nsm[dev];
  constexpr int PB = tma_pb<NB>();
  const size_t sm = (size_t)tma_stages<NB>() * PB * td.pstride * sizeof(double);
  const int ngroups = (g.ncells + PB - 1) / PB;
  const int grid = std::min(ngroups, TMA_CTAS_PER_SM * nsm);
  cudaError_t e;
  PDST_LAUNCH(e = launch_pdl(k_vanka_gemv_diag_tma<K1, NB>, dim3(grid), dim3(PB * NB * 21), sm, st, g, td, binvT, defect,
                             upd, ngroups));
  return e;
}

// Exact (non-surrogate) patch inverses through the same kind of pipeline:
// D x D column-major inverses (D even: 16-byte bulk copies) streamed by
// thread 0 into an S-stage ring, threads (patch p, row i) form
// sum_j invT[j][i] e_j against the gathered defect in shared memory (same
// 4-accumulator order as k_vanka_gemv), next group's defect gathered under the
// current product.  Coarse multigrid levels use these patches.
template <int D>
__host__ __device__ constexpr int xtma_pb() { return D <= 42 ? 2 : 1; }
constexpr int XTMA_STAGES = 3;

template <int D>
__global__ void __launch_bounds__(xtma_pb<D>() * D, 2) k_vanka_gemv_exact_tma(Geom g, const double* __restrict__ invT,
                                                                           const double* __restrict__ defect,
                                                                           double* __restrict__ upd, int ngroups) {
  constexpr int PB = xtma_pb<D>();
  constexpr unsigned PBYTES = (unsigned)D * D * 8u;
  static_assert(PBYTES % 16 == 0, "bulk copies move 16-byte multiples");
  extern __shared__ __align__(128) unsigned char xring[];
  __shared__ double es[2][PB][D];
  __shared__ __align__(8) uint64_t full[XTMA_STAGES];
  const int p = threadIdx.x / D, i = threadIdx.x % D;
  auto stage_ptr = [&](int st) { return reinterpret_cast<double*>(xring + (size_t)st * PB * PBYTES); };
  auto issue = [&](int gi, int st) {
    const int K0 = gi * PB, cnt = min(PB, g.ncells - K0);
    mbar_expect_tx(&full[st], (unsigned)cnt * PBYTES);
    bulk_g2s(stage_ptr(st), invT + (size_t)K0 * D * D, (unsigned)cnt * PBYTES, &full[st]);
  };
  auto load_defect = [&](int gi) {
    const int K = gi * PB + p;
    return (gi < ngroups && K < g.ncells) ? __ldg(defect + patch_dof_d(g, K, i)) : 0.0;
  };
  pdl_trigger();
  if (threadIdx.x == 0) {
    for (int st = 0; st < XTMA_STAGES; ++st) mbar_init(&full[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    for (int st = 0; st < XTMA_STAGES; ++st) {
      const int gi = blockIdx.x + st * gridDim.x;
      if (gi < ngroups) issue(gi, st);
    }
  }
  pdl_wait();
  es[0][p][i] = load_defect(blockIdx.x);
  __syncthreads();
  int it = 0;
  for (int gi = blockIdx.x; gi < ngroups; gi += gridDim.x, ++it) {
    const int st = it % XTMA_STAGES, buf = it & 1;
    const unsigned parity = (unsigned)(it / XTMA_STAGES) & 1u;
    const int K = gi * PB + p;
    const double en = load_defect(gi + gridDim.x);
    mbar_wait(&full[st], parity);
    if (K < g.ncells) {
      const double* col = stage_ptr(st) + (size_t)p * D * D + i;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int jj = 0;
#pragma unroll 4
      for (; jj + 3 < D; jj += 4) {
        s0 = fma(col[(size_t)jj * D], es[buf][p][jj], s0);
        s1 = fma(col[(size_t)(jj + 1) * D], es[buf][p][jj + 1], s1);
        s2 = fma(col[(size_t)(jj + 2) * D], es[buf][p][jj + 2], s2);
        s3 = fma(col[(size_t)(jj + 3) * D], es[buf][p][jj + 3], s3);
      }
      for (; jj < D; ++jj) s0 = fma(col[(size_t)jj * D], es[buf][p][jj], s0);
      upd[(size_t)i * g.ncells + K] = (s0 + s1) + (s2 + s3);  // structure of arrays [D][ncells]
    }
    es[buf ^ 1][p][i] = en;
    __syncthreads();  // stage st is free, es[buf ^ 1] is complete
    if (threadIdx.x == 0) {
      const int gn = gi + XTMA_STAGES * gridDim.x;
      if (gn < ngroups) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        issue(gn, st);
      }
    }
  }
}

template <int D>
cudaError_t launch_gemv_exact_tma(const Geom& g, const double* invT, const double* defect, double* upd,
                                  cudaStream_t st) {
  static DeviceOnce once;
  constexpr int PB = xtma_pb<D>();
  const size_t sm = (size_t)XTMA_STAGES * PB * D * D * sizeof(double);
  const int dev = current_device();
  if (!once.done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_vanka_gemv_exact_tma<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sm);
    if (e != cudaSuccess) return e;
    once.nsm[dev] = device_sms(dev);
    // persistent: exactly the CTAs that are resident at once
    int per_sm = 1;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_vanka_gemv_exact_tma<D>, PB * D, sm);
    if (e != cudaSuccess) return e;
    once.per_sm[dev] = std::max(1, per_sm);
    once.done[dev] = true;
  }
  const int nsm = once.nsm[dev], per_sm = once.per_sm[dev];
  const int ngroups = (g.ncells + PB - 1) / PB;
  const int grid = std::min(ngroups, per_sm * nsm);
  cudaError_t e;
  PDST_LAUNCH(e = launch_pdl(k_vanka_gemv_exact_tma<D>, dim3(grid), dim3(PB * D), sm, st, g, invT, defect, upd,
                             ngroups));
  return e;
}

}  // namespace

cudaError_t patch_invert_diag(const Geom& g, const TimeDiag& td, const double* spatial, double* binvT, int* bad,
                              cudaStream_t st) {
  const int tasks = g.ncells * td.nblk;
  PDST_LAUNCH(k_invert_diag<<<(tasks + 3) / 4, 128, 0, st>>>(g, td, spatial, binvT, bad));
  return cudaGetLastError();
}

cudaError_t vanka_gemv_diag(const Geom& g, const TimeDiag& td, const double* binvT, const double* defect,
                            double* upd, cudaStream_t st) {
  switch (td.k1 * 10 + td.nblk) {
    case 11: return launch_gemv_tma<1, 1>(g, td, binvT, defect, upd, st);
    case 21: return launch_gemv_tma<2, 1>(g, td, binvT, defect, upd, st);
    case 22: return launch_gemv_tma<2, 2>(g, td, binvT, defect, upd, st);
    case 32: return launch_gemv_tma<3, 2>(g, td, binvT, defect, upd, st);
    case 33: return launch_gemv_tma<3, 3>(g, td, binvT, defect, upd, st);
    case 42: return launch_gemv_tma<4, 2>(g, td, binvT, defect, upd, st);
    case 43: return launch_gemv_tma<4, 3>(g, td, binvT, defect, upd, st);
    case 44: return launch_gemv_tma<4, 4>(g, td, binvT, defect, upd, st);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace pdst

namespace pdst {
// Exact-patch GEMV through the TMA pipeline for even D (k+1 = 2, 4); false
// when the caller must use the row-per-thread kernel (odd D: 8-byte rows).
bool vanka_gemv_exact_tma(const Geom& g, int k1, const double* invT, const double* defect, double* upd,
                          cudaStream_t st, cudaError_t* err) {
  switch (k1) {
    case 2: *err = launch_gemv_exact_tma<42>(g, invT, defect, upd, st); return true;
    case 4: *err = launch_gemv_exact_tma<84>(g, invT, defect, upd, st); return true;
    default: return false;
  }
}
}  // namespace pdst
