// pdst_coarse.h — multigrid level operators (element form), transfers, coarsest solve.
#pragma once

#include <cuda_runtime.h>

#include "pdst_device.cuh"

namespace pdst {

// A level operator in element form (see pdst_coarse.cu).  fine == true: the
// finest level, ecell holds the column-major element matrices ET of every Radau
// node and the CIP face blocks are evaluated on the fly from `state`.
struct LevelOp {
  Geom g;
  Disc ds;
  int fine;
  const double* ecell;  // [k1][ncells][441]
  const double* fv;     // [k1][(nx-1) ny][324]   (coarse levels)
  const double* fh;     // [k1][nx (ny-1)][324]
  const double* state;  // [k1][Mv] lagged velocity (finest level)
};

cudaError_t prolong(const Geom& gc, const Geom& gf, int k1, const double* ec, double* ef, cudaStream_t st);
cudaError_t restrict_(const Geom& gc, const Geom& gf, int k1, const double* rf, double* rc, cudaStream_t st);
cudaError_t galerkin(const LevelOp& fine, const Geom& gc, int k1, double* ecell_c, double* fv_c, double* fh_c,
                     cudaStream_t st);
// y = A x (rhs == null) or rhs - A x on a coarse level; scratch holds
// level_apply_scratch() doubles (the element products).
size_t level_apply_scratch(const Geom& g, int k1);
cudaError_t level_apply(const LevelOp& op, const TimeData& td, const double* x, const double* rhs, double* y,
                        double* scratch, cudaStream_t st);
cudaError_t patch_assemble_level(const LevelOp& op, const TimeData& td, double* mats, cudaStream_t st);
// Dense coarsest slab matrix, optional pressure pinning, in-place inverse.
// scratch: >= 1 double; piv: >= n ints; bad: 1 int (set to 1 when singular).
cudaError_t dense_build(const LevelOp& op, const TimeData& td, bool pin, double* A, double* scratch, int* piv,
                        int* bad, cudaStream_t st);
cudaError_t dense_solve(const double* Ainv, int n, const double* b, double* y, cudaStream_t st);
// `partial`: project_scratch(k1) doubles of scratch.
size_t project_scratch(int k1);
cudaError_t project_pressure(const Geom& g, int k1, double* z, double* partial, cudaStream_t st);
cudaError_t axpy(size_t n, double a, const double* x, double* y, cudaStream_t st);
// Node injection (multigrid.py:146-153 inject_v, used by coarse_mode
// "rediscretize", :406-418): coarse node (i, j) <- fine node (2i, 2j), both
// components, per block mu; blocks of stride sf (fine) / sc (coarse) doubles.
// With zero_pressure the coarse blocks' pressure dofs are set to 0.
cudaError_t inject_velocity(const Geom& gc, const Geom& gf, int k1, const double* vf, size_t sf, double* vc,
                            size_t sc, bool zero_pressure, cudaStream_t st);

}  // namespace pdst
