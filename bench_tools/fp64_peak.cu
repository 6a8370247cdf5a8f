// FP64 peak microbenchmark on the B200 ("FP64 peak is not in
// MEASURED_PEAKS; measure it with a DFMA loop"): DFMA vector pipe and
// DMMA.8x8x4 tensor-core throughput, CUDA-event timed, printed as JSON.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters, double s) {
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
  if (r == 12345.678) out[threadIdx.x] = r;
}

__global__ void k_dmma(double* out, int iters) {
  double av = 1.0 + threadIdx.x * 1e-6, bv = 0.5;
  double d[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[i][0]), "+d"(d[i][1]) : "d"(av), "d"(bv));
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += d[i][0] + d[i][1];
  if (r == 12345.678) out[threadIdx.x] = r;
}

int main() {
  double* out;
  cudaMalloc(&out, 1 << 20);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 20000;
  float ms;
  // DFMA: 8 chains x iters x 2 flop per thread
  const int blocks = sms * 8, threads = 256;
  k_dfma<<<blocks, threads>>>(out, 100, 0.999);
  cudaEventRecord(a);
  k_dfma<<<blocks, threads>>>(out, iters, 0.999);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  const double fl_dfma = 2.0 * 8 * iters * (double)blocks * threads;
  // DMMA: per warp 8 x iters x (8*8*4*2) flop
  k_dmma<<<blocks, threads>>>(out, 100);
  float ms2;
  cudaEventRecord(a);
  k_dmma<<<blocks, threads>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms2, a, b);
  const double fl_dmma = 8.0 * iters * 512.0 * (double)blocks * threads / 32;
  printf("{\"fp64_dfma_tflops\": %.2f, \"fp64_dmma_tflops\": %.2f, \"sms\": %d, \"dfma_ms\": %.3f, \"dmma_ms\": %.3f}\n",
         fl_dfma / ms / 1e9, fl_dmma / ms2 / 1e9, sms, ms, ms2);
  return 0;
}
