// pdst_internal.h — host-side launch wrappers shared by the C-ABI layer.
#pragma once

#include <cuda_runtime.h>

#include "pdst_device.cuh"

namespace pdst {

cudaError_t set_tables(const Tables& t);
Tables host_tables();

// y = J x (rhs == null) or y = rhs - J x; `part` holds jacobian_scratch() doubles, zero when
// first used (its tail holds the apply's completion counters, which every apply leaves at zero).
size_t jacobian_scratch(const Geom& g, int k1);
// Re-zero the completion counters at the tail of `part` (called per linearization).
cudaError_t jacobian_reset_counters(const Geom& g, int k1, double* part, cudaStream_t st);
// Requires the linearization's boundary matrices (L.bmat) and apply cache (L.apc).
cudaError_t jacobian_apply(const Geom& g, const TimeData& td, const Disc& ds, const Lin& L, const double* x,
                           const double* rhs, double* out, double* part, cudaStream_t st);

// Apply cache of the linearization L at velocity state (k1, Mv): the
// per-quadrature-point coefficients the Jacobian apply streams
// (apply_cache_size() doubles).
size_t apply_cache_size(const Geom& g, int k1);
cudaError_t apply_cache(const Geom& g, const TimeData& td, const Disc& ds, const Lin& L, const double* state,
                        double* apc, cudaStream_t st);

cudaError_t slab_residual(const Geom& g, const TimeData& td, const Disc& ds, const Model& m, const Lin& L,
                          const double* U, const double* advect, const double* vminus, const double* fqp,
                          const double* ghat, double* out, cudaStream_t st);

cudaError_t linearize(const Geom& g, const Model& m, int k1, const double* state, double* eta, double* gam,
                      double* etaf, double* gamf, cudaStream_t st);

// Element matrices (volume + boundary sides, no CIP / mass / tau w) of node
// slot mu of the linearization L at velocity state (Mv), column-major per cell.
cudaError_t element_matrices(const Geom& g, const Disc& ds, const Lin& L, int mu, const double* state, double* ET,
                             cudaStream_t st);

// Boundary-side matrices [k1][nbf][col][row] of the current linearization (L.bmat ignored).
cudaError_t boundary_matrices(const Geom& g, const Disc& ds, const Lin& L, int k1, const double* state, double* bmat,
                              cudaStream_t st);

cudaError_t lifting(const Geom& g, const Model& m, const double* ghat, double* etad, double* betad, double* dg,
                    cudaStream_t st);

// Mass-weighted slab products (newton.py:96-121): y = (tau w (x) M) x and
// the dot <a, M b>; `partials` must hold at least reduce_partials() doubles.
cudaError_t mass_apply(const Geom& g, const TimeData& td, const double* x, double* y, cudaStream_t st);
int reduce_partials();
cudaError_t mass_dot(const Geom& g, const TimeData& td, const double* a, const double* b, double* partials,
                     double* result, cudaStream_t st);
cudaError_t dot(const double* a, const double* b, size_t n, double* partials, double* result, cudaStream_t st);

// Taylor-Hood Q2/Q1 pressure coupling (pdst_th.cu); cb holds th_scratch() doubles.
size_t th_scratch(const Geom& g, int k1);
cudaError_t th_apply(const Geom& g, const TimeData& td, bool on, const double* x, double* y, double* cb,
                     cudaStream_t st);
cudaError_t th_residual(const Geom& g, const TimeData& td, bool on, const double* U, const double* ghat, double* R,
                        double* cb, cudaStream_t st);
cudaError_t th_pressure_mass(const Geom& g, const TimeData& td, const double* x, double* y, cudaStream_t st);

// Strip the velocity components of a slab state into a dense (k1, Mv) copy.
cudaError_t copy_velocity_blocks(const Geom& g, int k1, const double* U, double* V, cudaStream_t st);
// V = sum_mu c[mu] U_mu (velocity part of blocks of length `stride`)
cudaError_t blend_velocity(const Geom& g, int k1, const double* coef, const double* U, size_t stride, double* V,
                           cudaStream_t st);

// FGMRES block kernels (pdst_krylov.cu): out[i] = <A_i, w> (i < m, rows lda
// apart; `partial` holds multidot_scratch(m) doubles) and w -= A^T c,
// w2 -= B^T c.
size_t multidot_scratch(int m);
cudaError_t multidot(const double* A, int64_t lda, int m, const double* w, int64_t n, double* partial, double* out,
                     cudaStream_t st);
cudaError_t multi_axpy(const double* A, const double* B, int64_t lda, int m, const double* c, double* w, double* w2,
                       int64_t n, cudaStream_t st);

}  // namespace pdst
