// pdst_mg.cu — integer maps, multigrid hierarchy, patches, Vanka, transfers
// and the V-cycle entry points of the C ABI.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/pdst.h"
#include "pdst_handle.h"

using namespace pdst;

namespace {

__global__ void k_cell_maps(int nx, int ny, int nd, int k1, int64_t* cell_nodes, int64_t* patch_ids) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nx * ny) return;
  const int ci = c % nx, cj = c / nx;
  const int nnx = 2 * nx + 1;
  const int64_t mv = 2LL * nnx * (2 * ny + 1);
  const int D = 21 * k1;
  for (int a = 0; a < 9; ++a) {
    const int64_t node = (int64_t)(2 * cj + a / 3) * nnx + 2 * ci + a % 3;
    cell_nodes[(int64_t)c * 9 + a] = node;
    for (int mu = 0; mu < k1; ++mu) {
      patch_ids[(int64_t)c * D + 21 * mu + 2 * a] = 2 * node + (int64_t)mu * nd;
      patch_ids[(int64_t)c * D + 21 * mu + 2 * a + 1] = 2 * node + 1 + (int64_t)mu * nd;
    }
  }
  for (int mu = 0; mu < k1; ++mu)
    for (int j = 0; j < 3; ++j) patch_ids[(int64_t)c * D + 21 * mu + 18 + j] = mv + 3LL * c + j + (int64_t)mu * nd;
}

}  // namespace


extern "C" {

int pdst_cell_maps(pdst_handle* h, int64_t* cell_nodes, int64_t* patch_ids) {
  if (!h || !cell_nodes || !patch_ids) return PDST_EINVAL;
  cudaSetDevice(h->device);
  const Geom& g = h->g;
  const int k1 = h->td.k1;
  int64_t* dev = nullptr;
  const size_t n1 = (size_t)g.ncells * 9, n2 = (size_t)g.ncells * 21 * k1;
  if (cudaMalloc(&dev, (n1 + n2) * sizeof(int64_t)) != cudaSuccess) return PDST_ECUDA;
  k_cell_maps<<<(g.ncells + 127) / 128, 128, 0, h->stream>>>(g.nx, g.ny, g.nd, k1, dev, dev + n1);
  cudaError_t e = cudaMemcpyAsync(cell_nodes, dev, n1 * sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(patch_ids, dev + n1, n2 * sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  cudaFree(dev);
  return e == cudaSuccess ? PDST_OK : PDST_ECUDA;
}

int pdst_hierarchy(pdst_handle*, int, int*) { return PDST_ENOTSUP; }
int pdst_level_sizes(pdst_handle*, int, int32_t*, int32_t*, int64_t*) { return PDST_ENOTSUP; }
int pdst_patches_build(pdst_handle*, int, double, int*, int64_t*) { return PDST_ENOTSUP; }
int pdst_patch_matrices(pdst_handle*, int, double*) { return PDST_ENOTSUP; }
int pdst_vanka(pdst_handle*, int, double*, const double*, int, double, int) { return PDST_ENOTSUP; }
int pdst_level_apply(pdst_handle*, int, const double*, double*, int) { return PDST_ENOTSUP; }
int pdst_restrict(pdst_handle*, int, const double*, double*, int) { return PDST_ENOTSUP; }
int pdst_prolong(pdst_handle*, int, const double*, double*, int) { return PDST_ENOTSUP; }
int pdst_vcycle(pdst_handle*, const double*, double*, int, int, double, int) { return PDST_ENOTSUP; }

}  // extern "C"
