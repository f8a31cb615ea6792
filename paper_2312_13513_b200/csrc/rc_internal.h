// rc_internal.h -- private definitions of the B200 (sm_100a) reactive-cell library.
// Nothing here is shared with oracle/ (the CPU oracle is independent test code).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/rc.h"

#define RC_MAX_NS 32
#define RC_MAX_NE 8
#define RC_RU 8314.46261815324  // J/kmol/K (R12)

// ---------------------------------------------------------------------------
// Device-resident species tables.  One contiguous fp64 buffer; each kernel
// stages the segment it needs into shared memory with one bulk TMA copy
// (cp.async.bulk), "constant memory for storing constant
// coefficients" re-done the Blackwell way.
// ---------------------------------------------------------------------------
struct ThermoSeg {        // doubles, offsets relative to the segment start
  // [0] Tmin  [1] Tmax  [2] Tmid (if uniform) [3] uniform flag (1.0 / 0.0)
  // [4 .. 4+6ns)      hlo[k][j]: j<5: (R/W_k) a_{j+1}^lo/(j+1); j=5: (R/W_k) a6^lo
  // [.. + 6ns)        hhi[k][j]
  // [.. + ns)         invW[k]
  // [.. + ns)         Tmid[k]
  __host__ __device__ static constexpr int hlo(int) { return 4; }
  __host__ __device__ static constexpr int hhi(int ns) { return 4 + 6 * ns; }
  __host__ __device__ static constexpr int invW(int ns) { return 4 + 12 * ns; }
  __host__ __device__ static constexpr int tmid(int ns) { return 4 + 13 * ns; }
  __host__ __device__ static constexpr int size(int ns) { return (4 + 14 * ns + 1) & ~1; }  // even -> 16-byte multiple
};

struct TransportSeg {
  // visc[ns][5] cond[ns][5] diff[np][6] (5 fit coefficients + pad: 16-byte aligned pairs)
  // W[nse] invW[nse] and the factorised Wilke matrices M0, M1, M2 [ns][nse] (nse = ns rounded
  // up to even, rows 16-byte aligned): with c1_kj = (W_j/W_k)^(1/4), c2_kj = 1/sqrt(8(1+W_k/W_j)),
  // M0 = c2, M1 = 2 c2 c1, M2 = c2 c1^2, so that sum_j X_j Phi_kj = A_k + s_k (B_k + s_k C_k)
  // with A = M0 X, B = M1 (X/s), C = M2 (X/s^2) and s_k = sqrt(mu_k)
  __host__ __device__ static constexpr int nse(int ns) { return (ns + 1) & ~1; }
  __host__ __device__ static constexpr int visc(int) { return 0; }
  __host__ __device__ static constexpr int cond(int ns) { return 5 * ns; }
  __host__ __device__ static constexpr int diff(int ns) { return 10 * ns; }
  __host__ __device__ static constexpr int W(int ns) { return 10 * ns + 6 * (ns * (ns + 1) / 2); }
  __host__ __device__ static constexpr int invW(int ns) { return W(ns) + nse(ns); }
  __host__ __device__ static constexpr int M(int ns, int q) { return W(ns) + 2 * nse(ns) + q * ns * nse(ns); }
  __host__ __device__ static constexpr int size(int ns) { return M(ns, 3); }
};

struct rc_mech {
  int ns, ne, device;
  bool uniform_tmid;
  double Tmin, Tmax;
  std::vector<double> W, P, thermo_host, transport_host;
  std::vector<double> nasa_lo, nasa_hi, T_mid;  // [ns][7], [ns]: raw NASA-7 (the kinetics table's g_k)
  std::vector<uint8_t> inert;
  double *d_thermo = nullptr;     // ThermoSeg
  double *d_transport = nullptr;  // TransportSeg
  double *d_P = nullptr;          // [ns][ns] element projection (R6)
  double *d_EF = nullptr;         // [2][ne][ns]: F = (E E^T)^-1 E, then E (P = I - E^T F; low-rank epilogue)
  std::vector<double> EF_host;    // the same on the host (the epilogue's kernel-parameter constants)
};

struct rc_mlp {
  int n_nets, d_in, h1, h2, h3, precision, ns, device;
  int gnets;                      // nets the hidden-layer GEMMs run: n_nets, or 1 (RC_MLP_SHARED)
  int flags;                      // rc_mlp_desc.flags (RC_MLP_LAYERWISE)
  int kpad1;                      // padded K of layer 1 (64 bf16 / 32 fp32)
  double lambda_bc, dt;
  int inv_lambda;                 // 1/lambda as an integer power
  std::vector<int> species_of_net;
  bool species_identity = false;  // species_of_net[i] == i for every output (the epilogue's factored projection)
  std::vector<float> b4_host;              // [n_nets] (the epilogue's kernel-parameter constants)
  std::vector<double> ymean_host, ystd_host;
  std::vector<float> xmean_host, xinvstd_host;  // [d_in] (the prologue's kernel-parameter constants)
  // device buffers
  void *d_W1 = nullptr, *d_W2 = nullptr, *d_W3 = nullptr;   // [nets][N][K] bf16 or fp32(tf32-rounded)
  void *d_W1lo = nullptr, *d_W2lo = nullptr, *d_W3lo = nullptr;  // RC_TF32X3: tf32(W - W_hi)
  float *d_b1 = nullptr, *d_b2 = nullptr, *d_b3 = nullptr;  // [nets][N]
  void *d_b2k = nullptr, *d_b3k = nullptr;  // bf16: b2, b3 as K = 16 MMA operands [nets][N][16] = (hi, lo, 0...)
  float *d_w4 = nullptr;                                    // [n_nets][h3] (shared: the output layer)
  float *d_b4 = nullptr;                                    // [nets]
  float *d_xmean = nullptr, *d_xinvstd = nullptr;           // [d_in]
  double *d_ymean = nullptr, *d_ystd = nullptr;             // [nets]
  int *d_species = nullptr;                                 // [nets]
};

// ---------------------------------------------------------------------------
// errors / bookkeeping
// ---------------------------------------------------------------------------
int rc_fail(int code, const char *fmt, ...);
// SMs of the current device, and the resident CTAs of `kernel` at (threads, dynamic smem) over the
// whole device (occupancy x SMs; persistent grids are sized with it).  Cached per device/kernel/config.
int rc_sm_count();
// layer-3 overlap counters (mlp_l2_sm100.cu; rc_overlap_read)
int l2_overlap_read(long long *out, int reset);
int rc_resident_blocks(const void *kernel, int threads, size_t smem);
void rc_count_launch(int n = 1);
void rc_reset_launches();
// per-stage CUDA-event timing (rc_profile_*); no-op unless enabled
struct ProfScope {
  int stage;
  cudaStream_t s;
  int slot;
  ProfScope(int stage, cudaStream_t s);
  ~ProfScope();
};

#define RC_CUDA_TRY(x)                                                                    \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess) return rc_fail(RC_ECUDA, "%s: %s", #x, cudaGetErrorString(e_)); \
  } while (0)
#define RC_LAUNCH_CHECK()                                                                           \
  do {                                                                                              \
    cudaError_t e_ = cudaGetLastError();                                                            \
    if (e_ != cudaSuccess) return rc_fail(RC_ECUDA, "launch failed: %s", cudaGetErrorString(e_));   \
    rc_count_launch();                                                                              \
  } while (0)

// ---------------------------------------------------------------------------
// Kernel launchers (defined in the .cu files)
// ---------------------------------------------------------------------------
struct CellsDev {
  int64_t n, ld;
  int mode;
  double *h, *T;
  const double *p, *Y;
  double *cp, *rho, *mu, *lambda, *D, *wdot, *qdot;
  float *o;
  double *red;
  int64_t *diag;
  const double *tau_mix;  // PaSR mixing time (NULL = laminar)
};

int launch_thermo(const rc_mech *m, const CellsDev &c, cudaStream_t s);
int launch_transport(const rc_mech *m, const CellsDev &c, cudaStream_t s);

struct ChemWs;  // defined in mlp_sm100.cu
size_t chem_workspace_bytes(const rc_mech *m, const rc_mlp *n, int64_t ncells);
size_t chem_workspace_min_bytes(const rc_mlp *n, int64_t ncells);  // the smallest chunk (256 cells)
int launch_chem(const rc_mech *m, const rc_mlp *n, const CellsDev &c, void *ws, size_t ws_bytes, cudaStream_t s);
// detailed kinetics (kinetics.cu): one 48-double record per reaction + eff [nr][ns] + NASA g table
struct rc_kin {
  int nr, ns, device;
  double *d_tab = nullptr;   // KinSeg
  double *d_qpart = nullptr; // per-block qdot partials (deterministic sum)
  size_t tab_doubles = 0;
};
int launch_kinetics(const rc_mech *m, const rc_kin *k, const CellsDev &c, cudaStream_t s);
int launch_qdot_finalize(const double *qpart, int n, double *red, cudaStream_t s);

int launch_combine_reductions(const double *rp, const int64_t *dp, int k, double *red, int64_t *diag, cudaStream_t s);
int mlp_upload(rc_mlp *n, const rc_mlp_desc *d);
