// pdst_vector.cu — slab vector utilities: block-mass apply and mass-weighted
// dot products (the reductions FGMRES and Newton call, newton.py:96-121,
// krylov.py:67-68/102/106), velocity-block copies and temporal blends.
//
// The consistent Q2 mass on a uniform mesh is hx*hy*(M1y (x) M1x) on the node
// grid, where M1 is the assembled 1-D quadratic mass; every reduction is a
// fixed two-level tree (deterministic).
#include "pdst_device.cuh"
#include "pdst_internal.h"
#include "pdst_handle.h"
#include "../../include/pdst.h"

namespace pdst {
namespace {

constexpr int RB = 256;       // reduction block
constexpr int RPARTS = 1184;  // 8 x 148 SMs

// Assembled 1-D Q2 mass entry between nodes X and Xp on an n-cell line.
__device__ __forceinline__ double m1g(int X, int Xp, int n) {
  double s = 0.0;
  const int lo = max(0, (max(X, Xp) - 2 + 1) / 2);
  for (int c = lo; c <= min(X, Xp) / 2 && c < n; ++c) {
    const int a = X - 2 * c, b = Xp - 2 * c;
    if (a >= 0 && a <= 2 && b >= 0 && b <= 2) s += c_tab.M1[a][b];
  }
  return s;
}

__global__ void k_mass_apply(Geom g, TimeData td, const double* __restrict__ x, double* __restrict__ y) {
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int mu = blockIdx.y;
  const size_t nn = (size_t)g.nnx * g.nny;
  const double tw = td.tau_w[mu];
  const double* xm = x + (size_t)mu * g.nd;
  double* ym = y + (size_t)mu * g.nd;
  if (tid < nn) {
    const int X = (int)(tid % g.nnx), Y = (int)(tid / g.nnx);
    double s0 = 0.0, s1 = 0.0;
    for (int Yp = max(0, Y - 2); Yp <= min(g.nny - 1, Y + 2); ++Yp) {
      const double my = m1g(Y, Yp, g.ny);
      if (my == 0.0) continue;
      double r0 = 0.0, r1 = 0.0;
      for (int Xp = max(0, X - 2); Xp <= min(g.nnx - 1, X + 2); ++Xp) {
        const double mx = m1g(X, Xp, g.nx);
        const size_t o = 2 * ((size_t)Yp * g.nnx + Xp);
        r0 = fma(mx, xm[o], r0);
        r1 = fma(mx, xm[o + 1], r1);
      }
      s0 = fma(my, r0, s0);
      s1 = fma(my, r1, s1);
    }
    const double h = g.hx * g.hy;
    ym[2 * tid] = tw * (h * s0);
    ym[2 * tid + 1] = tw * (h * s1);
  } else if (tid < nn + (size_t)g.ncells && !g.th) {  // Taylor-Hood pressure mass: pdst_th.cu
    const size_t c = tid - nn;
    const double h = g.hx * g.hy;
    const size_t o = g.mv + 3 * c;
    ym[o] = tw * (h * xm[o]);
    ym[o + 1] = tw * (h * (1.0 / 12.0) * xm[o + 1]);
    ym[o + 2] = tw * (h * (1.0 / 12.0) * xm[o + 2]);
  }
}

__device__ double block_sum(double v, double* sh) {
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    t = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
    for (int off = 16; off > 0; off >>= 1) t += __shfl_down_sync(0xffffffffu, t, off);
  }
  __syncthreads();
  return t;
}

// Per-cell a_K' M_K b_K over all nodes mu (with tau w_mu), plus pressure.
__global__ void k_mass_dot_partial(Geom g, TimeData td, const double* __restrict__ a, const double* __restrict__ b,
                                   double* __restrict__ partials) {
  __shared__ double sh[32];
  double acc = 0.0;
  const size_t total = (size_t)td.k1 * g.ncells;
  const double h = g.hx * g.hy;
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (size_t)gridDim.x * blockDim.x) {
    const int mu = (int)(t / g.ncells);
    const int c = (int)(t % g.ncells);
    const int ci = c % g.nx, cj = c / g.nx;
    const double* am = a + (size_t)mu * g.nd;
    const double* bm = b + (size_t)mu * g.nd;
    double cell = 0.0;
    for (int d = 0; d < 2; ++d) {
      double B[3][3];
      for (int jy = 0; jy < 3; ++jy)
        for (int ix = 0; ix < 3; ++ix)
          B[jy][ix] = bm[2 * ((size_t)(2 * cj + jy) * g.nnx + 2 * ci + ix) + d];
      for (int jy = 0; jy < 3; ++jy)
        for (int ix = 0; ix < 3; ++ix) {
          double mb = 0.0;
          for (int jj = 0; jj < 3; ++jj)
            for (int ii = 0; ii < 3; ++ii) mb = fma(c_tab.M1[jy][jj] * c_tab.M1[ix][ii], B[jj][ii], mb);
          cell = fma(am[2 * ((size_t)(2 * cj + jy) * g.nnx + 2 * ci + ix) + d], mb, cell);
        }
    }
    const size_t o = g.mv + 3 * (size_t)c;
    const double pp = g.th ? 0.0 : am[o] * bm[o] + (1.0 / 12.0) * (am[o + 1] * bm[o + 1] + am[o + 2] * bm[o + 2]);
    acc += td.tau_w[mu] * h * (cell + pp);
  }
  const double s = block_sum(acc, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__global__ void k_dot_partial(const double* __restrict__ a, const double* __restrict__ b, size_t n,
                              double* __restrict__ partials) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    acc = fma(a[i], b[i], acc);
  const double s = block_sum(acc, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__global__ void k_finish(const double* __restrict__ partials, int n, double* __restrict__ result) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += partials[i];
  const double s = block_sum(acc, sh);
  if (threadIdx.x == 0) *result = s;
}

__global__ void k_copy_velocity(Geom g, int k1, const double* __restrict__ U, double* __restrict__ V) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int mu = blockIdx.y;
  if (i < (size_t)g.mv && mu < k1) V[(size_t)mu * g.mv + i] = U[(size_t)mu * g.nd + i];
}

struct Coef7 {
  double c[MAXK1];
};

__global__ void k_blend(Geom g, int k1, Coef7 cf, const double* __restrict__ U, size_t stride, double* __restrict__ V) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (size_t)g.mv) return;
  double s = 0.0;
  for (int mu = 0; mu < k1; ++mu) s = fma(cf.c[mu], U[(size_t)mu * stride + i], s);
  V[i] = s;
}

}  // namespace

int reduce_partials() { return RPARTS; }

cudaError_t mass_apply(const Geom& g, const TimeData& td, const double* x, double* y, cudaStream_t st) {
  const size_t n = (size_t)g.nnx * g.nny + g.ncells;
  dim3 grid((unsigned)((n + 255) / 256), td.k1);
  PDST_LAUNCH(k_mass_apply<<<grid, 256, 0, st>>>(g, td, x, y));
  return cudaGetLastError();
}

cudaError_t mass_dot(const Geom& g, const TimeData& td, const double* a, const double* b, double* partials,
                     double* result, cudaStream_t st) {
  PDST_LAUNCH(k_mass_dot_partial<<<RPARTS, RB, 0, st>>>(g, td, a, b, partials));
  PDST_LAUNCH(k_finish<<<1, 1024, 0, st>>>(partials, RPARTS, result));
  return cudaGetLastError();
}

cudaError_t dot(const double* a, const double* b, size_t n, double* partials, double* result, cudaStream_t st) {
  PDST_LAUNCH(k_dot_partial<<<RPARTS, RB, 0, st>>>(a, b, n, partials));
  PDST_LAUNCH(k_finish<<<1, 1024, 0, st>>>(partials, RPARTS, result));
  return cudaGetLastError();
}

cudaError_t copy_velocity_blocks(const Geom& g, int k1, const double* U, double* V, cudaStream_t st) {
  dim3 grid((unsigned)((g.mv + 255) / 256), k1);
  PDST_LAUNCH(k_copy_velocity<<<grid, 256, 0, st>>>(g, k1, U, V));
  return cudaGetLastError();
}

cudaError_t blend_velocity(const Geom& g, int k1, const double* coef, const double* U, size_t stride, double* V,
                           cudaStream_t st) {
  Coef7 cf{};
  for (int i = 0; i < k1 && i < MAXK1; ++i) cf.c[i] = coef[i];
  PDST_LAUNCH(k_blend<<<(unsigned)((g.mv + 255) / 256), 256, 0, st>>>(g, k1, cf, U, stride, V));
  return cudaGetLastError();
}

}  // namespace pdst

// ---------------------------------------------------------------------------
// FP64 peak of the device (the roofline denominator of the FP64-bound kernels:
// patch factorization, residual): independent DFMA chains, CUDA-event timed.
// ---------------------------------------------------------------------------
namespace pdst {
namespace {
__global__ void k_dfma_peak(double* out, int iters, double s) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], s, 1e-9);
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += a[i];
  if (r == 12345.678) out[threadIdx.x] = r;  // never true: keeps the chains live
}
}  // namespace
}  // namespace pdst

extern "C" int pdst_fp64_peak(int device, double* tflops) {
  if (!tflops) return pdst::set_error(PDST_EINVAL, "null argument");
  if (cudaSetDevice(device) != cudaSuccess) return pdst::set_error(PDST_ECUDA, "cudaSetDevice(%d) failed", device);
  const int sms = pdst::device_sms(device);
  double* out = nullptr;
  if (cudaMalloc(&out, 1 << 16) != cudaSuccess) return pdst::set_error(PDST_ECUDA, "out of device memory");
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = sms * 8, threads = 256, iters = 20000;
  pdst::k_dfma_peak<<<blocks, threads>>>(out, 100, 0.999);  // warm-up
  cudaEventRecord(a);
  pdst::k_dfma_peak<<<blocks, threads>>>(out, iters, 0.999);
  cudaEventRecord(b);
  cudaError_t e = cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  if (e != cudaSuccess) return pdst::set_error(PDST_ECUDA, "%s", cudaGetErrorString(e));
  *tflops = 2.0 * 8 * iters * (double)blocks * threads / (ms * 1e-3) / 1e12;
  return PDST_OK;
}
