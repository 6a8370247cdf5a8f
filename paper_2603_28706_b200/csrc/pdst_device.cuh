// pdst_device.cuh — device-side tables, kernel parameter blocks and the
// per-cell Q2/P1disc element math shared by the slab Jacobian, residual and
// patch kernels (sm_100a, fp64).
//
// Mathematics follows the reference pdflow package (file:line into
// /root/reference/pkg/src/pdflow):
//   tangent coefficients  constitutive.py:323-337
//   Jacobian action       forms.py:581-652, slab.py:193-201
//   residual              forms.py:435-516, slab.py:162-173
//   tables                femspace.py:46-106 (x-major volume points q = 4 qx + qy,
//                         local node a = 3 jy + ix, interleaved components)
//
// Layout conventions (global memory):
//   slab vectors  (k+1) blocks of nd = Mv + Mp doubles, Mv = 2 (2nx+1)(2ny+1);
//                 velocity dof of node (X, Y) component d at 2 (Y (2nx+1) + X) + d;
//                 pressure dof j of cell c at Mv + 3 c + j
//   qp caches     [mu][cell][q] (16 volume points of a cell contiguous)
//   face caches   [mu][bface][q], bface = side offset + index along the side,
//                 side order bottom, right, top, left
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

// Process-wide count of libpdst kernel launches (pdst_launch_count; the
// bench's gpu_launches).  Every launch site goes through PDST_LAUNCH.
void pdst_count_launch();
// Programmatic dependent launch (PDL): a kernel launched with launch_pdl may
// start while its stream predecessor is still running once every CTA of the
// predecessor has called pdl_trigger(); pdl_wait() then blocks until the
// predecessor has completed and its writes are visible (a no-op for a normal
// launch).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

#define PDST_LAUNCH(...)   \
  do {                     \
    __VA_ARGS__;           \
    pdst_count_launch();   \
  } while (0)

// Step timeline of profiling builds (-DPDST_TRACE): g_steptrace[4 k + j] for
// kernel class k (0 apply tile pass, 1 apply epilogue, 2 defect tile pass,
// 3 defect epilogue, 4 patch GEMV, 5 Vanka scatter), j = 0 first start (min),
// 1 first past its dependency wait (min), 2 last end (max); %globaltimer ns.
#ifdef PDST_TRACE
extern __device__ unsigned long long g_steptrace[32];
#define STEP_MARK(k, j)                                               \
  do {                                                                \
    if (threadIdx.x == 0) {                                           \
      unsigned long long t_;                                          \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));          \
      if ((j) == 2)                                                   \
        atomicMax(&g_steptrace[4 * (k) + (j)], t_);                   \
      else                                                            \
        atomicMin(&g_steptrace[4 * (k) + (j)], t_);                   \
    }                                                                 \
  } while (0)
#else
#define STEP_MARK(k, j) \
  do {                  \
  } while (0)
#endif

namespace pdst {

// One-time setup of a launch site, kept PER DEVICE: the dynamic shared-memory
// opt-in (cudaFuncSetAttribute) and the SM / occupancy figures belong to a
// device context, so handles on several devices in one process each
// configure their own.
constexpr int kMaxDevices = 64;
struct DeviceOnce {
  bool done[kMaxDevices] = {};
  int nsm[kMaxDevices] = {};
  int per_sm[kMaxDevices] = {};
};
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d < kMaxDevices ? d : kMaxDevices - 1;
}
inline int device_sms(int dev) {
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

constexpr int MAXK1 = 7;

// 1-D Gauss(4) on [0,1] and Q2 Lagrange tables, filled from the host.
struct Tables {
  double s[4];      // Gauss points
  double w[4];      // Gauss weights
  double B[4][3];   // L_i(s_q)
  double G[4][3];   // L_i'(s_q)
  double M1[3][3];  // 1-D mass sum_q w_q L_i L_j
  double E[2][3];   // L_i(0), L_i(1)
  double dE[2][3];  // L_i'(0), L_i'(1)
};

extern __constant__ Tables c_tab;

// Boundary-face tags: 0 Neumann, 1 Dirichlet, 2 partition cut (an interior
// face of the global mesh at the edge of a rank's local mesh: no side terms).
constexpr uint8_t kCutSide = 2;

struct Geom {
  int nx, ny;    // cells
  int nnx, nny;  // Q2 nodes per direction
  int ncells;
  int mv, nd;    // velocity dofs, dofs per node block
  int nbf;       // boundary faces 2 (nx + ny)
  double hx, hy;
  double ihx, ihy;           // 1/hx, 1/hy (the reference's grad_scale, femspace.py:142-143)
  const uint8_t* dirichlet;  // nbf tags (device): 0 Neumann, 1 Dirichlet, 2 cut
  int th;                    // pressure space: 0 the reference's P1disc (3 per cell), 1 Taylor-Hood Q1
                             // ((nx+1)(ny+1) vertex values after the velocity block, pdst_th.cu)
};

struct TimeData {
  int k1;
  double tau_w[MAXK1];
  double K_t[MAXK1 * MAXK1];
  double m_t[MAXK1];
};

struct Disc {
  double gamma1, gamma2, gamma_cip;
  int viscous, convection, pressure;
};

struct Model {
  double p, delta, nu, nu_inf;
  int kind;  // 0 pic, 1 exn, 2 modn
  double sigma_max;
};

// Frozen linearization (per node mu).
struct Lin {
  const double* eta;    // [k1][nc][16]
  const double* gam;    // [k1][nc][16]
  const double* etaf;   // [k1][nbf][4]
  const double* gamf;   // [k1][nbf][4]
  const double* etad;   // [nbf][4]  lifting viscosity (state independent)
  const double* betad;  // [nbf][4]
  const double* dg;     // [nbf][4][3] sym grad of the lifting
  const double* bmat;   // [k1][nbf][21 cols][21 rows] boundary-side matrices (column-major), or null
  const double* apc;    // apply cache (pdst_operator.cu, APC_SLOTS), or null
  int has_gamma;        // 0 for Picard (gamma == 0)
};

__host__ __device__ inline int side_offset(const Geom& g, int side) {
  // bottom, right, top, left
  return side == 0 ? 0 : side == 1 ? g.nx : side == 2 ? g.nx + g.ny : 2 * g.nx + g.ny;
}

// x^e for x >= 0 through exp(e log x): 2-3x cheaper than pow(), relative error a few 1e-15.
__device__ __forceinline__ double powr(double x, double e) { return e == 0.0 ? 1.0 : exp(e * log(x)); }

// (eta, gamma) of T(B) = eta B + gamma (A:B) A at squared norm a_sq.
// constitutive.py:323-337 (gamma scaled by the clip factor of :311-320 for modn).
__device__ inline void tangent_coeffs(const Model& m, double a_sq, double& eta, double& gam) {
  const double dsq = m.delta * m.delta + a_sq;
  const double mu = m.nu * powr(dsq, (m.p - 2.0) / 2.0);
  eta = m.nu_inf + mu;
  if (m.kind == 0) {
    gam = 0.0;
    return;
  }
  double g = (m.p - 2.0) * mu / dsq;
  if (m.kind == 2) {
    const double sigma = mu * sqrt(a_sq);
    // s = min(1, sigma_max / (sigma > 0 ? sigma : inf)); NaN propagates like np.minimum.
    const double r = m.sigma_max / (sigma > 0.0 ? sigma : __longlong_as_double(0x7ff0000000000000LL));
    const double s = (r > 1.0) ? 1.0 : r;
    g = s * g;
  }
  gam = g;
}

__device__ inline double eta_field(const Model& m, double a_sq) {
  return m.nu_inf + m.nu * powr(m.delta * m.delta + a_sq, (m.p - 2.0) / 2.0);
}

__device__ inline double beta_field(const Model& m, double a_sq) {
  return m.nu * (m.p - 2.0) * powr(m.delta * m.delta + a_sq, (m.p - 4.0) / 2.0);
}

}  // namespace pdst
