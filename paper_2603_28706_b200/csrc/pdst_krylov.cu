// pdst_krylov.cu — the N-vector work of FGMRES in the M-inner product
// (krylov.py:93-126): batched dot products of one vector against a block of
// basis vectors, and the fused block update w -= V c, mw -= MV c.
//
// The reference's modified Gram-Schmidt (2(j+1) dependent dot/axpy pairs per
// pass) runs in block form: ONE multi-dot c = MV' w, a (j+1)-term triangular
// recurrence with the basis Gram matrix on the host, ONE fused update
// (krylov.py; exactly the MGS recurrence even for a non-orthogonal basis).
//
// Both kernels stream the basis block once (HBM bound) and use fixed
// reduction trees, so results do not depend on scheduling.
#include "pdst_device.cuh"
#include "pdst_internal.h"

namespace pdst {
namespace {

constexpr int KB = 256;        // threads per block
constexpr int KPARTS = 592;    // 4 x 148 SMs
constexpr int KROWS = 8;       // basis rows per register group

// partial[p][i] = sum over this block's slice of A[i][e] * w[e].
__global__ void __launch_bounds__(KB) k_multidot_partial(const double* __restrict__ A, int64_t lda, int m,
                                                         const double* __restrict__ w, int64_t n,
                                                         double* __restrict__ partial) {
  __shared__ double red[KB / 32][KROWS];
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t e0 = (int64_t)blockIdx.x * chunk, e1 = min(n, e0 + chunk);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int i0 = 0; i0 < m; i0 += KROWS) {
    double s[KROWS];
#pragma unroll
    for (int r = 0; r < KROWS; ++r) s[r] = 0.0;
    for (int64_t e = e0 + threadIdx.x; e < e1; e += KB) {
      const double we = __ldg(w + e);
#pragma unroll
      for (int r = 0; r < KROWS; ++r)
        if (i0 + r < m) s[r] = fma(__ldg(A + (int64_t)(i0 + r) * lda + e), we, s[r]);
    }
#pragma unroll
    for (int r = 0; r < KROWS; ++r) {
      double v = s[r];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) red[wid][r] = v;
    }
    __syncthreads();
    if (threadIdx.x < KROWS && i0 + threadIdx.x < m) {
      double v = 0.0;
      for (int q = 0; q < KB / 32; ++q) v += red[q][threadIdx.x];
      partial[(size_t)blockIdx.x * m + i0 + threadIdx.x] = v;
    }
    __syncthreads();
  }
}

// out[i] = sum_p partial[p][i] (one warp per row, fixed order).
__global__ void k_multidot_finish(const double* __restrict__ partial, int parts, int m, double* __restrict__ out) {
  const int i = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= m) return;
  double v = 0.0;
  for (int p = lane; p < parts; p += 32) v += partial[(size_t)p * m + i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) out[i] = v;
}

// w[e] -= sum_i c[i] A[i][e]  (and w2[e] -= sum_i c[i] B[i][e] when B != null).
__global__ void __launch_bounds__(KB) k_multi_axpy(const double* __restrict__ A, const double* __restrict__ B,
                                                   int64_t lda, int m, const double* __restrict__ c,
                                                   double* __restrict__ w, double* __restrict__ w2, int64_t n) {
  extern __shared__ double cs[];
  for (int i = threadIdx.x; i < m; i += blockDim.x) cs[i] = c[i];
  __syncthreads();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0, t = 0.0;
    for (int i = 0; i < m; ++i) {
      s = fma(cs[i], __ldg(A + (int64_t)i * lda + e), s);
      if (B) t = fma(cs[i], __ldg(B + (int64_t)i * lda + e), t);
    }
    w[e] -= s;
    if (B) w2[e] -= t;
  }
}

}  // namespace

size_t multidot_scratch(int m) { return (size_t)KPARTS * (size_t)m; }

cudaError_t multidot(const double* A, int64_t lda, int m, const double* w, int64_t n, double* partial, double* out,
                     cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  PDST_LAUNCH(k_multidot_partial<<<KPARTS, KB, 0, st>>>(A, lda, m, w, n, partial));
  PDST_LAUNCH(k_multidot_finish<<<(m + 7) / 8, 256, 0, st>>>(partial, KPARTS, m, out));
  return cudaGetLastError();
}

cudaError_t multi_axpy(const double* A, const double* B, int64_t lda, int m, const double* c, double* w, double* w2,
                       int64_t n, cudaStream_t st) {
  if (m <= 0 || n <= 0) return cudaSuccess;
  int64_t blocks = (n + KB - 1) / KB;
  if (blocks > 148 * 16) blocks = 148 * 16;
  PDST_LAUNCH(k_multi_axpy<<<(unsigned)blocks, KB, (size_t)m * sizeof(double), st>>>(A, B, lda, m, c, w, w2, n));
  return cudaGetLastError();
}

}  // namespace pdst
