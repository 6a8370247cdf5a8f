/* pdst.h — C ABI of the B200 slab hot path (libpdst.so).
 *
 * Drop-in boundary for the operator/smoother seam of the reference package
 * pdflow (arXiv 2603.28706).  Every entry point replaces one reference
 * interface (file:line into /root/reference/pkg/src/pdflow):
 *
 *   pdst_create            SlabContext + Discretization setup      slab.py:71-112, forms.py:135-283
 *   pdst_set_lifting       DiscretizationConfig.g_hat / lifting     forms.py:60-83, 343-356
 *   pdst_linearize         SlabJacobian.__init__                    slab.py:183-191, forms.py:527-578
 *   pdst_jacobian_apply    SlabJacobian.matvec / .apply             slab.py:193-205, forms.py:581-652
 *   pdst_jacobian_defect   r - level.matvec(d) inside vanka_smooth   solver/multigrid.py:336
 *   pdst_residual          slab_residual                            slab.py:168-173, forms.py:435-516
 *   pdst_mass_apply        MassNorm.apply                           solver/newton.py:112-117
 *   pdst_mass_dot          MassNorm.norm / FGMRES M-inner products  solver/newton.py:119-121, krylov.py:67-68
 *   pdst_dot               FGMRES Euclidean dots on M-weighted vecs solver/krylov.py:102, 106
 *   pdst_cell_maps         Discretization.cell_nodes / patch ids    femspace.py:127-140, forms.py:192-196,
 *                                                                   solver/multigrid.py:273-275
 *   pdst_hierarchy         MgGeometry.from_fine                     solver/multigrid.py:164-191
 *   pdst_hierarchy_depth   MgGeometry.from_fine on a partition      solver/multigrid.py:164-191 (the
 *                          rank's strip coarsens with the global mesh; no reference counterpart)
 *   pdst_patches_build     StmgPreconditioner patch setup           solver/multigrid.py:261-299, 475-488
 *   pdst_patch_matrices    PatchSet.matrices (read back)            solver/multigrid.py:198-209
 *   pdst_vanka             vanka_smooth                             solver/multigrid.py:327-340
 *   pdst_level_apply       MgLevel.matvec (coarse Galerkin levels)  solver/multigrid.py:234-248, 302-324
 *   pdst_restrict          StmgPreconditioner._restrict             solver/multigrid.py:523-532
 *   pdst_prolong           StmgPreconditioner._prolong              solver/multigrid.py:534-543
 *   pdst_vcycle            StmgPreconditioner.apply                 solver/multigrid.py:545-578
 *
 * Conventions: all arrays are fp64 (integers int64) in the reference layout
 * — slab vectors are (k+1) node-major blocks of nd = Mv + Mp, velocity dofs
 * interleaved 2*node + component with nodes row-major (y, x), then 3 P1disc
 * dofs per cell.  `where` says whether pointers are host memory (copied in
 * and out, call is synchronous) or device memory on the handle's device
 * (call is asynchronous on the handle's stream).  The caller owns every
 * argument buffer; the handle owns all device caches.  A handle is bound to
 * one device and stream and is not thread safe.
 */
#ifndef PDST_H
#define PDST_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define PDST_OK 0
#define PDST_EINVAL 1    /* bad argument (maps to ValueError) */
#define PDST_EDOMAIN 2   /* delta <= 0 etc. (ConstitutiveDomainError) */
#define PDST_ESINGULAR 3 /* singular patch (SingularPatchError) */
#define PDST_ECUDA 4     /* CUDA runtime failure */
#define PDST_ESTATE 5    /* call order (e.g. apply before linearize) */
#define PDST_ENOTSUP 6   /* unsupported size (k > 3 for the kernels) */
#define PDST_ENCCL 7     /* NCCL failure in a strip exchange */

#define PDST_HOST 0
#define PDST_DEVICE 1
/* PDST_HOST_ASYNC (pdst_jacobian_apply, pdst_jacobian_defect, pdst_vanka only):
 * host pointers to page-locked memory; the H2D copies run on a copy-in stream,
 * the kernels on the handle's stream once their inputs have landed, the D2H
 * copies on a copy-out stream, and the call returns at once, so consecutive
 * calls overlap their transfers with each other's kernels.  The caller must
 * not touch the buffers of a call before pdst_sync(h).  Unpinned memory is
 * rejected (PDST_EINVAL). */
#define PDST_HOST_ASYNC 2

/* linearization kinds (constitutive.py:133-160) */
#define PDST_PICARD 0
#define PDST_EXACT_NEWTON 1
#define PDST_MODIFIED_NEWTON 2

typedef struct pdst_handle pdst_handle;

typedef struct {
  int32_t nx, ny;              /* cells per direction */
  double x0, y0, x1, y1;       /* rectangle */
  const uint8_t* dirichlet;    /* 2(nx+ny) tags, sides bottom,right,top,left: 0 Neumann, 1 Dirichlet,
                                  2 partition cut (interior face of the global mesh); NULL = all Dirichlet */
} pdst_mesh;

typedef struct {
  int32_t k;                   /* DG(k) in time, k+1 right Radau nodes */
  const double* nodes;         /* k+1 */
  const double* weights;       /* k+1 */
  const double* K_t;           /* (k+1)^2 row-major */
  const double* m_t;           /* k+1 */
} pdst_time;

typedef struct {
  double gamma1, gamma2, gamma_cip;
  int32_t enable_viscous, enable_convection, enable_pressure;
  /* 0: Q2/P1disc, the reference's pair (3 pressure dofs per cell);
     1: Taylor-Hood Q2/Q1 (continuous bilinear pressure on the (nx+1)(ny+1)
     vertices, row-major (y, x), after the velocity block; BASELINE north_star
     (1), no reference counterpart -- SURVEY §9.1).  Taylor-Hood handles
     support the Jacobian apply, the residual and the mass products; the
     patch / multigrid / strip / manufactured entry points return
     PDST_ENOTSUP for them. */
  int32_t pressure_space;
} pdst_disc;

typedef struct {
  double p, delta, nu, nu_inf;
} pdst_params;

int pdst_create(const pdst_mesh* mesh, const pdst_time* time, const pdst_disc* disc, const pdst_params* params,
                double tau, int device, void* stream, pdst_handle** out);
int pdst_destroy(pdst_handle* h);
int pdst_set_stream(pdst_handle* h, void* stream);
/* wait for every call of the handle (kernels and PDST_HOST_ASYNC copies) */
int pdst_sync(pdst_handle* h);
int pdst_sizes(const pdst_handle* h, int64_t* mv, int64_t* mp, int64_t* nd, int64_t* ndof);

int pdst_set_lifting(pdst_handle* h, const double* g_hat, int where); /* g_hat: Mv or NULL */
int pdst_linearize(pdst_handle* h, const double* U, int kind, double sigma_max, int where);
int pdst_jacobian_apply(pdst_handle* h, const double* x, double* y, int where);
int pdst_jacobian_defect(pdst_handle* h, const double* x, const double* r, double* y, int where);
/* f_qp: (k+1, ncells, 16, 2) body force at x-major volume points, or NULL (f = 0);
   advect: (k+1)*nd lagged state or NULL (= U) */
int pdst_residual(pdst_handle* h, const double* U, const double* v_minus, const double* f_qp, const double* advect,
                  double* R, int where);
int pdst_mass_apply(pdst_handle* h, const double* x, double* y, int where);
int pdst_mass_dot(pdst_handle* h, const double* a, const double* b, double* out, int where);
int pdst_dot(pdst_handle* h, const double* a, const double* b, int64_t n, double* out, int where);

/* integer maps, host output: cell_nodes (ncells, 9), patch_ids (ncells, 21(k+1)) */
int pdst_cell_maps(pdst_handle* h, int64_t* cell_nodes, int64_t* patch_ids);

/* multigrid: levels 0 (coarsest) .. L-1 (finest = the handle mesh) */
int pdst_hierarchy(pdst_handle* h, int min_cells, int* num_levels);
/* exactly `depth` levels (a partition rank's strip coarsens with the global mesh) */
int pdst_hierarchy_depth(pdst_handle* h, int depth, int* num_levels);
int pdst_level_sizes(pdst_handle* h, int level, int32_t* nx, int32_t* ny, int64_t* ndof);
/* surrogate != 0: finest patches from the blended state at rep_fraction; coarse levels exact.
   On ESINGULAR, *bad_level / *bad_patch identify the first singular patch. */
int pdst_patches_build(pdst_handle* h, int surrogate, double rep_fraction, int* bad_level, int64_t* bad_patch);
int pdst_patch_matrices(pdst_handle* h, int level, double* mats /* host (ncells, D, D) */);
/* storage of a level's factorized patches: D, number of temporally diagonalized
   complex 21x21 blocks (0 = full real D x D inverses), bytes streamed per patch per sweep */
int pdst_patch_info(pdst_handle* h, int level, int32_t* D, int32_t* diag_blocks, int64_t* bytes_per_patch);
int pdst_vanka(pdst_handle* h, int level, double* d, const double* r, int steps, double omega, int where);
/* One Vanka update without the defect: inc = omega sum_K R_K' A_K^-1 R_K defect over the
   patches of cell rows [row_lo, row_hi) (distributed sweeps combine increments across ranks). */
int pdst_vanka_increment(pdst_handle* h, int level, const double* defect, double* inc, int row_lo, int row_hi,
                         double omega, int where);
int pdst_level_apply(pdst_handle* h, int level, const double* x, double* y, int where);
int pdst_restrict(pdst_handle* h, int fine_level, const double* r_fine, double* r_coarse, int where);
int pdst_prolong(pdst_handle* h, int fine_level, const double* e_coarse, double* e_fine, int where);
int pdst_vcycle(pdst_handle* h, const double* r, double* z, int pre, int post, double omega, int where);

/* Manufactured-solution benchmark problem on the device.
 * pdst_manufactured_forcing: ManufacturedCase.forcing (bench/manufactured.py:
 *   121-157) at the residual's volume points of every cell and Radau node
 *   t_start + tau * node[mu]: fqp (k+1, ncells, 16, 2), the f_qp argument of
 *   pdst_residual.  Uses the handle's model parameters and mesh extents.
 * pdst_error_norms: one slab's contribution (squared) to error_norms
 *   (bench/metrics.py:35-85): sq2 = {e_phi^2, e_div^2} over [t0, t1] with
 *   `spatial_points`^2 Gauss points per cell and `temporal_points` in time
 *   (the reference's defaults: 5 and k+2); sq2 is a host double[2]. */
int pdst_manufactured_forcing(pdst_handle* h, double t_start, double* fqp, int where);
int pdst_error_norms(pdst_handle* h, const double* U, double t0, double t1, int spatial_points, int temporal_points,
                     double* sq2, int where);

/* Coarse operators of the hierarchy (MgConfig.coarse_mode,
   solver/multigrid.py:302-324, 406-431): 0 "galerkin" (default, P' J P in
   element form), 1 "rediscretize" (every coarse level re-linearized on its
   own mesh at the state injected from the next finer level -- pressure zero,
   g_hat injected alike -- with the coarse mesh's own mass and exact patches).
   Takes effect at the next pdst_patches_build. */
int pdst_set_coarse_mode(pdst_handle* h, int mode);

/* Coarsest-level solve of the V-cycle (takes effect at the next
 * pdst_patches_build).  kind:
 *   PDST_COARSE_DENSE   the reference's dense LU of the pinned slab system
 *                       (multigrid.py:494-520), up to 16384 dofs;
 *   PDST_COARSE_VANKA   `sweeps` Vanka steps with `omega` from a zero guess;
 *   PDST_COARSE_FGMRES  FGMRES (Euclidean, classical Gram-Schmidt twice) right-
 *                       preconditioned by `sweeps` Vanka steps from zero, at
 *                       most `iters` iterations or until the relative residual
 *                       reaches `rtol`;
 *   PDST_COARSE_AUTO    dense up to 4096 dofs, else FGMRES.
 * A 5-level hierarchy of a 2048^2 mesh ends at 128^2 (362,500 dofs), beyond
 * the dense LU.  No reference counterpart beyond DENSE. */
#define PDST_COARSE_DENSE 0
#define PDST_COARSE_VANKA 1
#define PDST_COARSE_AUTO 2
#define PDST_COARSE_FGMRES 3
int pdst_set_coarse_solver(pdst_handle* h, int kind, int sweeps, double omega, int iters, double rtol);

/* Kernel timing for benchmarks: CUDA events around every launch of class
   kernel (0 jacobian/defect, 1 vanka gemv, 2 vanka scatter, 3 residual,
   4 transfers, 5 coarse-level operators) while enabled. */
/* FGMRES block operations (krylov.py:93-126), device pointers only
   (where must be PDST_DEVICE), asynchronous on the handle's stream:
   out[i] = <A_i, w> for i < m, basis rows A_i = A + i*lda (length n);
   w -= sum_i c[i] A_i and, when B != NULL, w2 -= sum_i c[i] B_i (c: m doubles
   on the device).  Classical Gram-Schmidt applied twice is two
   multidot + multi_axpy pairs. */
int pdst_multidot(pdst_handle* h, const double* A, int64_t lda, int m, const double* w, int64_t n, double* out,
                  int where);
int pdst_multi_axpy(pdst_handle* h, const double* A, const double* B, int64_t lda, int m, const double* c, double* w,
                    double* w2, int64_t n, int where);

/* Per-launch CUDA events around the handle's kernel groups (measurement only;
   the events disable PDL overlap between the groups).  Kernel classes:
   0 Jacobian apply y = J x, 1 patch GEMV, 2 Vanka scatter, 3 residual,
   4 transfers, 5 coarse level applies, 6 defect apply y = r - J x. */
int pdst_profile(pdst_handle* h, int enable);
int pdst_profile_read(pdst_handle* h, int kernel, double* total_ms, int64_t* launches);

/* ---- strip partition: the distributed data plane -------
   The handle's mesh is rank `rank`'s local strip of an nx x ny_global mesh:
   global cell rows [c_lo, c_hi), owned [a, b) (paper_2603_28706_b200.partition
   RankLayout; two ghost cell rows towards every neighbour).  lower_c_hi /
   upper_c_lo: the neighbours' local row ranges (what they receive). */
int pdst_strip(pdst_handle* h, int rank, int nranks, int ny_global, int a, int b, int c_lo, int c_hi, int lower_c_hi,
               int upper_c_lo);
/* The ranks' NCCL communicator (ncclComm_t, rank order = partition order),
   e.g. torch.distributed's ProcessGroupNCCL._comm_ptr(); NULL detaches.
   Exchanges are ncclSend / ncclRecv groups on the handle's stream, resolved
   in the process's loaded libnccl.so.2 (SURVEY §8b "nccl_comm"). */
int pdst_strip_comm(pdst_handle* h, void* nccl_comm);
/* Refresh the ghost rows of the local (device) vector x from the neighbours
   (halo pack kernel -> NCCL group -> unpack kernel). */
int pdst_strip_halo(pdst_handle* h, double* x);
/* This rank's distributed Jacobian apply + one Vanka step, device pointers,
   everything enqueued on the handle's stream (no host synchronization):
   x and d halos, y = J x, e = r - J d, the defect row from the upper rank,
   the patch GEMV, d += omega sum over the OWNED patches (one fused scatter;
   node row 2b's increment goes to the upper rank), the lower rank's
   increment added to row 2a.  x's and d's ghost rows are overwritten. */
int pdst_strip_step(pdst_handle* h, const double* x, double* y, double* d, const double* r, double omega);
/* The same step for all ranks of a partition held in one process on one
   device (virtual ranks, partition order; the neighbours' packed buffers
   are read directly): the parity and overhead check of the data plane. */
int pdst_strips_step_local(pdst_handle* const* hs, int nranks, double* const* xs, double* const* ys,
                           double* const* ds, const double* const* rs, double omega);

/* Measured FP64 (DFMA) throughput of `device` in TFLOP/s: the roofline
   denominator of the FP64-bound kernels (patch factorization, residual); no
   reference counterpart -- benchmark bookkeeping. */
int pdst_fp64_peak(int device, double* tflops);

const char* pdst_last_error(void);
const char* pdst_version(void);
/* Number of kernels libpdst has launched in this process (all handles); no
   reference counterpart -- benchmark bookkeeping. */
int64_t pdst_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* PDST_H */
