// FP64 pipe microbenchmark (B200): dependent-issue latency of DFMA and the
// per-warp issue interval with K independent chains and W warps per SM.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bench_tools/fp64_lat bench_tools/fp64_lat.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int K>
__global__ void chains(double* out, long long* cyc, double a, double b, int iters) {
  double v[K];
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = threadIdx.x * 1e-3 + k;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int k = 0; k < K; ++k) v[k] = fma(v[k], a, b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) s += v[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int K>
void run(int warps) {
  double* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 8); cudaMalloc(&cyc, 148 * 8);
  const int iters = 2000;
  chains<K><<<148, warps * 32>>>(out, cyc, 0.999, 1e-3, iters);
  chains<K><<<148, warps * 32>>>(out, cyc, 0.999, 1e-3, iters);
  long long h[148]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double c = (double)h[0] / (iters * 8.0 * K);
  printf("K=%d chains, %2d warps/SM: %.2f cycles per DFMA per warp (=> %.2f cyc between dependent ops), SM rate %.1f lanes/clk\n", K, warps,
         c, c * K, warps * 32.0 / c);
  cudaFree(out); cudaFree(cyc);
}
int main() {
  for (int w : {1, 4, 8, 16}) { run<1>(w); run<2>(w); run<4>(w); run<8>(w); run<16>(w); }
  return 0;
}
