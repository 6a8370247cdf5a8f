// pdst_handle.h — the opaque handle behind include/pdst.h.
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "pdst_device.cuh"
#include "pdst_internal.h"

namespace pdst {

struct DeviceBuffer {
  double* ptr = nullptr;
  size_t cap = 0;
  DeviceBuffer() = default;
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  ~DeviceBuffer() { release(); }
  double* ensure(size_t n);
  void release();
};

Geom make_geom(int nx, int ny, double x0, double y0, double x1, double y1, const uint8_t* dirichlet_dev);

// One multigrid level.  Level L-1 is the handle's own (finest) mesh whose
// operator is matrix free; coarser levels carry Galerkin element operators.
struct Level {
  Geom g{};
  uint8_t* dirichlet = nullptr;
  std::vector<uint8_t> dirichlet_host;
  bool all_dirichlet = true;
  // Galerkin element representation per node mu (coarse levels only):
  //   ecell [k1][ncells][21][21]       volume + boundary blocks
  //   efx   [k1][ny][nx-1][18][18]     couplings across vertical faces (L,R) as
  //   efy   [k1][ny-1][nx][18][18]     the 2x2 block structure LL, LR, RL, RR
  //                                    stored as 4 x (9x9 node blocks x I2)
  DeviceBuffer ecell, efx, efy;
  // patches
  DeviceBuffer mats, invs;
  int D = 0;
  // work vectors (k1 * nd each)
  DeviceBuffer w0, w1, w2, w3;
  ~Level() {
    if (dirichlet) cudaFree(dirichlet);
  }
};

}  // namespace pdst

struct pdst_handle {
  int device = 0;
  cudaStream_t stream = nullptr;
  pdst::Geom g{};
  uint8_t* dirichlet = nullptr;
  std::vector<uint8_t> dirichlet_host;
  double extents[4] = {0, 0, 1, 1};
  pdst::TimeData td{};
  pdst::Disc ds{};
  pdst::Model model{};
  double tau = 0.0;
  std::vector<double> nodes;

  // linearization caches
  pdst::DeviceBuffer state;  // (k1, Mv)
  pdst::DeviceBuffer eta, gam, etaf, gamf;
  pdst::DeviceBuffer etad, betad, dg;
  pdst::DeviceBuffer ghat;
  bool has_ghat = false;
  bool linearized = false;

  // staging for host pointers
  pdst::DeviceBuffer scratch_a, scratch_b, scratch_c, scratch_d, scratch_f;
  pdst::DeviceBuffer partials;

  // multigrid
  std::vector<pdst::Level*> levels;  // 0 = coarsest
  bool patches_valid = false;

  ~pdst_handle() {
    for (auto* l : levels) delete l;
    if (dirichlet) cudaFree(dirichlet);
  }
};
