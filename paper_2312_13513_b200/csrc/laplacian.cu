// laplacian.cu -- downstream consumer of the cell-local update (DESIGN.md
// reading R22): implicit Laplacian assembly of PAPER.md Algorithm 1 (lines 137-158) for the species
// and energy equations, with the coefficients this path produces (gamma = rho D_k for species k,
// lambda / cp for the energy equation), on a periodic Cartesian mesh or a z-slab of one (the
// multi-GPU block, halo planes exchanged by the caller over NCCL P2P); ldu storage
// and the ldu -> CSR conversion that feeds the linear solver.
//
// HBM-bound ("discretization typically display a memory-bound characteristic").  The
// paper's kernel runs one thread per face and accumulates the diagonal with atomicAdd (Algorithm 1
// lines 5-6, RC_LAP_ATOMIC here); the default RC_LAP_GATHER runs one thread per cell, writes the
// cell's three "+" faces and gathers its diagonal from all six faces (the "-" faces recomputed from
// the neighbours' coefficients with the owner's operand order, so every face value is bitwise the
// one its owner stores): no atomics, no zeroing pass, deterministic.
#include "ptx.cuh"
#include "rc_internal.h"

namespace {

struct LapGeo {
  int nx, ny, nz;
  int64_t n, plane;
  double S[3];  // |S_f| / |d_f| per direction
};

// coefficient gamma of system s at cell c of this block (c in [0, n)) or of a halo plane
// (h = 0: below, 1: above; p = in-plane index) from the property outputs
struct Gamma {
  const double *rho, *lam, *cp, *D;
  int64_t ld;
  int ns;
  const double *halo[2];  // [(ns + 3)][plane]: rho, lambda, cp, D_0..D_{ns-1}
  int64_t plane;
  __device__ __forceinline__ double cell(int s, int64_t c) const {
    return s < ns ? rho[c] * D[s * ld + c] : lam[c] / cp[c];
  }
  __device__ __forceinline__ double halo_cell(int h, int s, int64_t p) const {
    const double *b = halo[h];
    return s < ns ? b[p] * b[(3 + s) * plane + p] : b[plane + p] / b[2 * plane + p];
  }
};

// grid (ceil(nx / 256), ny, nz): thread (i, j, k) without integer division; the coefficients of the
// 7-point stencil are formed per system from the neighbours' properties (rho, lambda/cp read once)
__global__ void __launch_bounds__(256, 4) lap_gather_kernel(LapGeo g, Gamma G, int nsys, double *upper, double *diag) {
  const bool halo = G.halo[0] != nullptr;
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y, k = blockIdx.z;
  if (i >= g.nx) return;
  const int64_t c = i + (int64_t)g.nx * (j + (int64_t)g.ny * k);
  const int64_t p = c - (int64_t)k * g.plane;  // in-plane index
  const bool top = k + 1 == g.nz, bot = k == 0;
  // stencil: 0 = c, 1 = x+, 2 = x-, 3 = y+, 4 = y-, 5 = z+, 6 = z- (z: wrap or halo plane)
  const int64_t nb[7] = {c,
                         c + (i + 1 == g.nx ? 1 - g.nx : 1),
                         c + (i == 0 ? g.nx - 1 : -1),
                         c + (j + 1 == g.ny ? (int64_t)(1 - g.ny) * g.nx : g.nx),
                         c + (j == 0 ? (int64_t)(g.ny - 1) * g.nx : -g.nx),
                         top ? c + g.plane - g.n : c + g.plane,
                         bot ? c - g.plane + g.n : c - g.plane};
  const bool hz[7] = {false, false, false, false, false, top && halo, bot && halo};
  double rho[7];  // rho of the 7 stencil cells (lambda / cp is formed for the energy system at the end)
#pragma unroll
  for (int q = 0; q < 7; ++q) rho[q] = hz[q] ? G.halo[q == 5 ? 1 : 0][p] : G.rho[nb[q]];
  double *up = upper + c, *dg = diag + c;
  auto emit = [&](const double (&gm)[7]) {
    // owner's operand order: gamma_f = (gamma_owner + gamma_neighbour) / 2
    const double axp = 0.5 * __dadd_rn(gm[0], gm[1]) * g.S[0], axm = 0.5 * __dadd_rn(gm[2], gm[0]) * g.S[0];
    const double ayp = 0.5 * __dadd_rn(gm[0], gm[3]) * g.S[1], aym = 0.5 * __dadd_rn(gm[4], gm[0]) * g.S[1];
    const double azp = 0.5 * __dadd_rn(gm[0], gm[5]) * g.S[2], azm = 0.5 * __dadd_rn(gm[6], gm[0]) * g.S[2];
    up[0] = axp;
    up[g.n] = ayp;
    up[2 * g.n] = azp;
    dg[0] = -(((axp + axm) + (ayp + aym)) + (azp + azm));
    up += 3 * g.n;
    dg += g.n;
  };
  // species systems: per stencil cell a pointer to its D_s (block or halo plane), advanced by its
  // stride each system; the loads of system s + 1 are issued before system s is finished (two systems
  // of loads in flight per thread: the pass is bound by L2/HBM latency, ncu long_scoreboard)
  const int nspec = nsys - 1 < G.ns ? nsys - 1 : G.ns;
  const double *dp[7];
  int64_t ds[7];
#pragma unroll
  for (int q = 0; q < 7; ++q) {
    dp[q] = hz[q] ? G.halo[q == 5 ? 1 : 0] + 3 * g.plane + p : G.D + nb[q];
    ds[q] = hz[q] ? g.plane : G.ld;
  }
  double cur[7], nxt[7];
#pragma unroll
  for (int q = 0; q < 7; ++q) cur[q] = nspec > 0 ? *dp[q] : 0.0;
#pragma unroll 1
  for (int s = 0; s < nspec; ++s) {
    if (s + 1 < nspec)
#pragma unroll
      for (int q = 0; q < 7; ++q) nxt[q] = dp[q][(s + 1) * ds[q]];
    double gm[7];
#pragma unroll
    for (int q = 0; q < 7; ++q) gm[q] = __dmul_rn(rho[q], cur[q]);  // rounded: no FMA into the face sums
    emit(gm);
#pragma unroll
    for (int q = 0; q < 7; ++q) cur[q] = nxt[q];
  }
  if (nsys > nspec) {  // energy: gamma = lambda / cp
    double gm[7];
#pragma unroll
    for (int q = 0; q < 7; ++q) {
      if (hz[q]) {
        const double *b = G.halo[q == 5 ? 1 : 0];
        gm[q] = b[g.plane + p] / b[2 * g.plane + p];
      } else {
        gm[q] = G.lam[nb[q]] / G.cp[nb[q]];
      }
    }
    emit(gm);
  }
}

// PAPER.md Algorithm 1 as written: one thread per face, diagonal by atomicAdd (diag zeroed first)
__global__ void __launch_bounds__(256) lap_atomic_kernel(LapGeo g, Gamma G, int nsys, double *upper, double *diag) {
  const bool halo = G.halo[0] != nullptr;
  const int64_t nf = 3 * g.n + (halo ? g.plane : 0);  // + the faces from the plane below onto plane 0
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < nf; f += (int64_t)gridDim.x * blockDim.x) {
    if (f >= 3 * g.n) {  // face (halo below, plane-0 cell p): owned by the rank below
      const int64_t p = f - 3 * g.n;
      for (int s = 0; s < nsys; ++s)
        atomicAdd(&diag[(size_t)s * g.n + p], -(0.5 * (G.halo_cell(0, s, p) + G.cell(s, p)) * g.S[2]));
      continue;
    }
    const int d = (int)(f / g.n);
    const int64_t c = f - d * g.n;
    const int i = (int)(c % g.nx), j = (int)((c / g.nx) % g.ny), k = (int)(c / g.plane);
    int64_t nb;
    bool in_halo = false;
    if (d == 0) nb = c + (i + 1 == g.nx ? 1 - g.nx : 1);
    else if (d == 1) nb = c + (j + 1 == g.ny ? (int64_t)(1 - g.ny) * g.nx : g.nx);
    else {
      in_halo = halo && k + 1 == g.nz;
      nb = k + 1 < g.nz ? c + g.plane : c + g.plane - g.n;
    }
    for (int s = 0; s < nsys; ++s) {
      const double gN = in_halo ? G.halo_cell(1, s, c - (int64_t)(g.nz - 1) * g.plane) : G.cell(s, nb);
      const double a = 0.5 * (G.cell(s, c) + gN) * g.S[d];            // gamma_f delta_f S_f
      upper[(size_t)s * 3 * g.n + f] = a;
      atomicAdd(&diag[(size_t)s * g.n + c], -a);                       // diag[owner] -= upper
      if (!in_halo) atomicAdd(&diag[(size_t)s * g.n + nb], -a);        // diag[neighbour] -= lower
    }
  }
}

// ldu -> CSR: row c holds the diagonal and the six faces of cell c, columns ascending
__global__ void __launch_bounds__(256) ldu_to_csr_kernel(LapGeo g, int nsys, const double *upper, const double *diag,
                                                         int64_t *row_ptr, int32_t *col, double *val) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y, k = blockIdx.z;
  const int i0 = i - lane;                                  // first row of the warp
  if (i0 >= g.nx) return;                                   // whole warp past the end of the x row
  const bool act = i < g.nx;
  const int nrow = g.nx - i0 < 32 ? g.nx - i0 : 32;         // active rows of the warp (contiguous)
  const int ic = act ? i : i0;                              // inactive lanes mirror row i0 (never stored)
  const int64_t c = ic + (int64_t)g.nx * (j + (int64_t)g.ny * k);
  const int64_t c0 = i0 + (int64_t)g.nx * (j + (int64_t)g.ny * k);
  const int64_t nbr[7] = {c,
                          c + (ic + 1 == g.nx ? 1 - g.nx : 1),
                          c + (ic == 0 ? g.nx - 1 : -1),
                          c + (j + 1 == g.ny ? (int64_t)(1 - g.ny) * g.nx : g.nx),
                          c + (j == 0 ? (int64_t)(g.ny - 1) * g.nx : -g.nx),
                          k + 1 == g.nz ? c + g.plane - g.n : c + g.plane,
                          k == 0 ? c - g.plane + g.n : c - g.plane};
  // value slots: diag, upper of the + faces (owner c), upper of the - faces (owner = neighbour)
  const int64_t slot[7] = {-1, c, nbr[2], g.n + c, g.n + nbr[4], 2 * g.n + c, 2 * g.n + nbr[6]};
  int ord[7] = {0, 1, 2, 3, 4, 5, 6};
#pragma unroll
  for (int a = 1; a < 7; ++a)  // insertion sort by column (7 entries)
#pragma unroll
    for (int b = a; b > 0; --b)
      if (nbr[ord[b]] < nbr[ord[b - 1]]) {
        const int t = ord[b]; ord[b] = ord[b - 1]; ord[b - 1] = t;
      }
  if (act) {
    row_ptr[c] = 7 * c;
    if (c == g.n - 1) row_ptr[g.n] = 7 * g.n;
  }
  // the warp's rows are 7 nrow contiguous entries: staged in shared memory and written as 16-byte
  // vectors (a row-per-thread store of 7 entries scatters each store instruction over 56-byte strides)
  __shared__ __align__(16) double stg[8][32 * 7];
  int32_t *sc = reinterpret_cast<int32_t *>(stg[w]);
#pragma unroll
  for (int e = 0; e < 7; ++e) sc[lane * 7 + e] = (int32_t)nbr[ord[e]];
  __syncwarp();
  for (int q = lane; q < nrow * 7; q += 32) col[7 * c0 + q] = sc[q];
  __syncwarp();
  // per entry: its source (diag or upper) and the stride to the next system; the next system's seven
  // values are loaded before this one is staged (the pass is latency-bound, ncu long_scoreboard)
  const double *src[7];
  int64_t sstr[7];
#pragma unroll
  for (int e = 0; e < 7; ++e) {
    const int64_t sl = slot[ord[e]];
    src[e] = sl < 0 ? diag + c : upper + sl;
    sstr[e] = sl < 0 ? g.n : 3 * g.n;
  }
  double cur[7], nxt[7];
#pragma unroll
  for (int e = 0; e < 7; ++e) cur[e] = nsys > 0 ? src[e][0] : 0.0;
  for (int s = 0; s < nsys; ++s) {
    if (s + 1 < nsys)
#pragma unroll
      for (int e = 0; e < 7; ++e) nxt[e] = src[e][(s + 1) * sstr[e]];
#pragma unroll
    for (int e = 0; e < 7; ++e) stg[w][lane * 7 + e] = cur[e];
    __syncwarp();
    double *dst = val + (size_t)s * 7 * g.n + 7 * c0;
    if (nrow == 32 && ((uintptr_t)dst & 15u) == 0) {
      for (int q = lane; q < 112; q += 32) reinterpret_cast<double2 *>(dst)[q] = reinterpret_cast<const double2 *>(stg[w])[q];
    } else {
      for (int q = lane; q < nrow * 7; q += 32) dst[q] = stg[w][q];
    }
    __syncwarp();
#pragma unroll
    for (int e = 0; e < 7; ++e) cur[e] = nxt[e];
  }
}

// the bottom / top planes of this block's inputs -> [(ns + 3)][plane] (rho, lambda, cp, D_k): the
// halo the neighbouring ranks need
__global__ void __launch_bounds__(256) pack_planes_kernel(LapGeo g, Gamma G, double *bottom, double *top) {
  const int nf = 3 + G.ns;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nf * g.plane; e += (int64_t)gridDim.x * blockDim.x) {
    const int f = (int)(e / g.plane);
    const int64_t p = e - f * g.plane;
    const double *src = f == 0 ? G.rho : f == 1 ? G.lam : f == 2 ? G.cp : G.D + (size_t)(f - 3) * G.ld;
    if (bottom) bottom[e] = src[p];
    if (top) top[e] = src[(int64_t)(g.nz - 1) * g.plane + p];
  }
}

bool aligned8(const void *p) { return ((uintptr_t)p & 7u) == 0; }

int geo_of(const rc_mesh *mesh, int64_t n, LapGeo &g) {
  if (!mesh) return rc_fail(RC_EINVAL, "NULL mesh");
  if (mesh->nx < 1 || mesh->ny < 1 || mesh->nz < 1 || !(mesh->dx > 0 && mesh->dy > 0 && mesh->dz > 0))
    return rc_fail(RC_EINVAL, "mesh: need nx, ny, nz >= 1 and positive spacings");
  if (mesh->ny > 65535 || mesh->nz > 65535) return rc_fail(RC_EUNSUPPORTED, "mesh: ny, nz <= 65535 (grid dimensions)");
  g.nx = mesh->nx; g.ny = mesh->ny; g.nz = mesh->nz;
  g.plane = (int64_t)g.nx * g.ny;
  g.n = g.plane * g.nz;
  if (n >= 0 && n != g.n) return rc_fail(RC_EINVAL, "mesh has %lld cells, rc_cells.n = %lld", (long long)g.n, (long long)n);
  g.S[0] = mesh->dy * mesh->dz / mesh->dx;
  g.S[1] = mesh->dx * mesh->dz / mesh->dy;
  g.S[2] = mesh->dx * mesh->dy / mesh->dz;
  return RC_OK;
}

int64_t grid_for(int64_t work) {
  int64_t b = (work + 255) / 256, cap = (int64_t)rc_sm_count() * 8;
  return b < 1 ? 1 : b > cap ? cap : b;
}

}  // namespace

extern "C" int rc_laplacian(const rc_mech *m, const rc_mesh *mesh, const rc_cells *c, const double *halo_lo,
                            const double *halo_hi, double *upper, double *diag, int mode, void *stream) {
  rc_reset_launches();
  if (!m || !c) return rc_fail(RC_EINVAL, "NULL mech or cells");
  LapGeo g;
  int rc = geo_of(mesh, c->n, g);
  if (rc) return rc;
  if (c->ld < c->n) return rc_fail(RC_EINVAL, "ld < n");
  if (!c->rho || !c->lambda || !c->cp || !c->D || !upper || !diag)
    return rc_fail(RC_EINVAL, "rc_laplacian needs rho, lambda, cp, D, upper and diag");
  if ((halo_lo == nullptr) != (halo_hi == nullptr)) return rc_fail(RC_EINVAL, "halo_lo and halo_hi: both or neither");
  if (mode != RC_LAP_GATHER && mode != RC_LAP_ATOMIC) return rc_fail(RC_EINVAL, "unknown assembly mode %d", mode);
  const void *ptrs[] = {c->rho, c->lambda, c->cp, c->D, halo_lo, halo_hi, upper, diag};
  for (const void *p : ptrs)
    if (p && !aligned8(p)) return rc_fail(RC_EALIGN, "rc_laplacian arrays must be 8-byte aligned");
  Gamma G{c->rho, c->lambda, c->cp, c->D, c->ld, m->ns, {halo_lo, halo_hi}, g.plane};
  const int nsys = m->ns + 1;
  cudaStream_t s = (cudaStream_t)stream;
  if (g.n == 0) return RC_OK;
  ProfScope prof(RC_STAGE_LAPLACIAN, s);
  if (mode == RC_LAP_GATHER) {
    lap_gather_kernel<<<dim3((g.nx + 255) / 256, g.ny, g.nz), 256, 0, s>>>(g, G, nsys, upper, diag);
    RC_LAUNCH_CHECK();
  } else {
    RC_CUDA_TRY(cudaMemsetAsync(diag, 0, (size_t)nsys * g.n * sizeof(double), s));
    lap_atomic_kernel<<<(unsigned)grid_for(3 * g.n + g.plane), 256, 0, s>>>(g, G, nsys, upper, diag);
    RC_LAUNCH_CHECK();
  }
  return RC_OK;
}

extern "C" int rc_ldu_to_csr(const rc_mesh *mesh, int nsys, const double *upper, const double *diag, int64_t *row_ptr,
                             int32_t *col, double *val, void *stream) {
  rc_reset_launches();
  LapGeo g;
  int rc = geo_of(mesh, -1, g);
  if (rc) return rc;
  if (g.nx < 3 || g.ny < 3 || g.nz < 3) return rc_fail(RC_EUNSUPPORTED, "CSR needs nx, ny, nz >= 3 (7 distinct columns)");
  if (g.n > INT32_MAX) return rc_fail(RC_EUNSUPPORTED, "CSR column indices are int32");
  if (nsys < 1 || !upper || !diag || !row_ptr || !col || !val) return rc_fail(RC_EINVAL, "rc_ldu_to_csr: bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  ProfScope prof(RC_STAGE_CSR, s);
  ldu_to_csr_kernel<<<dim3((g.nx + 255) / 256, g.ny, g.nz), 256, 0, s>>>(g, nsys, upper, diag, row_ptr, col, val);
  RC_LAUNCH_CHECK();
  return RC_OK;
}

extern "C" int rc_pack_planes(const rc_mech *m, const rc_mesh *mesh, const rc_cells *c, double *bottom, double *top,
                              void *stream) {
  rc_reset_launches();
  if (!m || !c) return rc_fail(RC_EINVAL, "NULL mech or cells");
  LapGeo g;
  int rc = geo_of(mesh, c->n, g);
  if (rc) return rc;
  if (!c->rho || !c->lambda || !c->cp || !c->D) return rc_fail(RC_EINVAL, "rc_pack_planes needs rho, lambda, cp, D");
  Gamma G{c->rho, c->lambda, c->cp, c->D, c->ld, m->ns, {nullptr, nullptr}, g.plane};
  cudaStream_t s = (cudaStream_t)stream;
  pack_planes_kernel<<<(unsigned)grid_for((3 + m->ns) * g.plane), 256, 0, s>>>(g, G, bottom, top);
  RC_LAUNCH_CHECK();
  return RC_OK;
}
