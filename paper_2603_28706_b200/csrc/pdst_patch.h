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
  double* spatial;      // optional [ncells][21][21] surrogate spatial block R_K J_rep R_K' (row-major)
};

// Temporal diagonalization of a surrogate patch:
//   A_K = K_t (x) Mhat + diag(tau w) (x) Jhat,  S = diag(tau w)^-1 K_t = V diag(lam) V^-1,
//   A_K^-1 e = (V (x) I) blockdiag[(lam_i Mhat + Jhat)^-1] (V^-1 diag(tau w)^-1 (x) I) e.
// Only one member of each complex-conjugate pair is stored (nblk blocks).
struct TimeDiag {
  int k1;
  int nblk;                    // stored eigen-blocks
  int pair[MAXK1];             // 1 if block b is one of a conjugate pair (weight 2 Re), 0 if real
  double lam_re[MAXK1], lam_im[MAXK1];
  double V_re[MAXK1 * MAXK1], V_im[MAXK1 * MAXK1];        // V[mu][b] for stored blocks b (column b)
  double Vi_re[MAXK1 * MAXK1], Vi_im[MAXK1 * MAXK1];      // Vinv[b][mu] rows for stored blocks
  double itw[MAXK1];           // 1 / (tau w_mu)
  // per-patch storage: block b at boff[b] doubles into the patch, a conjugate
  // pair's complex inverse as 441 double2, a real eigenvalue's (real) inverse
  // as 441 doubles padded to 442 (16-byte multiple for the bulk copies)
  int boff[MAXK1];
  int pstride;                 // doubles per patch
};

// Host: diagonalize S = diag(tau w)^-1 K_t (k1 <= 4). Returns false when S is
// defective / ill-conditioned (the caller keeps the full real inverses).
bool time_diagonalize(int k1, const double* K_t, const double* tau_w, TimeDiag& out);

cudaError_t patch_invert_diag(const Geom& g, const TimeDiag& td, const double* spatial, double* binvT, int* bad,
                              cudaStream_t st);
cudaError_t vanka_gemv_diag(const Geom& g, const TimeDiag& td, const double* binvT, const double* defect,
                            double* upd, cudaStream_t st);

bool vanka_gemv_exact_tma(const Geom& g, int k1, const double* invT, const double* defect, double* upd,
                          cudaStream_t st, cudaError_t* err);

cudaError_t patch_assemble(const PatchArgs& a, cudaStream_t st);
cudaError_t patch_invert(int k1, const double* mats, double* invT, int npatch, int* bad, cudaStream_t st);
cudaError_t vanka_gemv(const Geom& g, int k1, const double* invT, const double* defect, double* upd, cudaStream_t st);
cudaError_t vanka_scatter(const Geom& g, int k1, const double* upd, double omega, double* d, cudaStream_t st,
                          int row_lo = 0, int row_hi = -1, bool inc_only = false, double* inc_row = nullptr,
                          int inc_Y = -1);

}  // namespace pdst
