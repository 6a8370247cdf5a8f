// Does the SM scheduler share issue slots fairly between two co-resident CTAs
// (vs the warps of one 512-thread CTA)?  Every warp runs the same FP64 + LDS
// loop and records when it finishes.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bench_tools/sched_fair bench_tools/sched_fair.cu
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
extern __shared__ double sm[];
__global__ void work(double* out, unsigned long long* t_end, unsigned long long* t_start, unsigned* smid, int iters) {
  const int warp = threadIdx.x >> 5;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  double v[6];
  for (int k = 0; k < 6; ++k) v[k] = threadIdx.x * 1e-3 + k;
  sm[threadIdx.x] = v[0];
  __syncthreads();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
#pragma unroll
      for (int k = 0; k < 6; ++k) v[k] = fma(v[k], 0.999, 1e-3);
      v[r] += sm[(threadIdx.x + 32 * r + i) & (blockDim.x - 1)];
    }
  }
  double s = 0;
  for (int k = 0; k < 6; ++k) s += v[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if ((threadIdx.x & 31) == 0) {
    const int w = blockIdx.x * (blockDim.x >> 5) + warp;
    t_end[w] = t1;
    t_start[w] = t0;
    unsigned s_;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s_));
    smid[w] = s_;
  }
}
void run(int grid, int block, size_t smem, const char* name) {
  const int nw = grid * block / 32;
  double* out; unsigned long long *te, *ts; unsigned* sid;
  cudaMalloc(&out, (size_t)grid * block * 8); cudaMalloc(&te, nw * 8); cudaMalloc(&ts, nw * 8); cudaMalloc(&sid, nw * 4);
  cudaFuncSetAttribute(work, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int rep = 0; rep < 2; ++rep) work<<<grid, block, smem>>>(out, te, ts, sid, 3000);
  cudaDeviceSynchronize();
  std::vector<unsigned long long> e(nw), s(nw); std::vector<unsigned> id(nw);
  cudaMemcpy(e.data(), te, nw * 8, cudaMemcpyDeviceToHost); cudaMemcpy(s.data(), ts, nw * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(id.data(), sid, nw * 4, cudaMemcpyDeviceToHost);
  unsigned long long t0 = *std::min_element(s.begin(), s.end());
  // per-CTA (or per half of a 512-thread CTA) mean end time, split by "first 8 warps on the SM" / "second 8"
  const int wpc = block / 32;
  double first = 0, second = 0, mx = 0; int nf = 0, ns = 0;
  for (int c = 0; c < grid; ++c)
    for (int w = 0; w < wpc; ++w) {
      const double t = (e[c * wpc + w] - t0) / 1e3;
      mx = std::max(mx, t);
      bool isSecond = (block == 512) ? (w >= 8) : (c >= 148);
      if (isSecond) { second += t; ++ns; } else { first += t; ++nf; }
    }
  printf("%s: first 8 warps of an SM end at %.2f us (mean), second 8 at %.2f us, last warp %.2f us\n", name, first / nf, ns ? second / ns : 0.0, mx);
}
int main() {
  run(296, 256, 90 * 1024, "2 CTAs x 256 threads per SM");
  run(148, 512, 180 * 1024, "1 CTA x 512 threads per SM");
  run(148, 256, 90 * 1024, "1 CTA x 256 threads per SM");
  return 0;
}
