// pdst_patch.h — patch / Vanka launchers.
#pragma once

#include <cuda_runtime.h>

#include "pdst_device.cuh"

namespace pdst {

struct PatchArgs {
  Geom g;
  TimeData td;
  Disc ds;
  const double* ET;     // [nslot][ncells][21][21] element matrices (column-major per cell)
  int nslot;            // k1 (exact patches) or 1 (surrogate)
  const double* state;  // [nslot][Mv] lagged velocity per slot (CIP weights)
  double* mats;         // [ncells][D][D] row-major output
};

cudaError_t patch_assemble(const PatchArgs& a, cudaStream_t st);
cudaError_t patch_invert(int k1, const double* mats, double* invT, int npatch, int* bad, cudaStream_t st);
cudaError_t vanka_gemv(const Geom& g, int k1, const double* invT, const double* defect, double* upd, cudaStream_t st);
cudaError_t vanka_scatter(const Geom& g, int k1, const double* upd, double omega, double* d, cudaStream_t st);

}  // namespace pdst
