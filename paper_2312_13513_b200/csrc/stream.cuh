// stream.cuh -- TMA-staged streaming of component-major (SoA) cell tiles for the
// cell-local kernels (thermo, transport, chemistry prologue and epilogue).
//
// PAPER.md:180 ("coalesce the same component": SoA fields) and PAPER.md:181
// (shared memory for the per-cell mass/mole fractions), re-done the sm_100a way:
// a CTA owns a ring of `stages` shared-memory stages; a stage holds one tile of
// TILE consecutive cells as rows, one per SoA component (T, p, Y_k, raw net
// outputs, ...): n8 fp64 rows (TILE x 8 B) then n4 fp32 rows (TILE x 4 B), each
// filled by ONE cp.async.bulk whose completion is counted on the stage's
// mbarrier.  One thread keeps stages - 1 tiles in flight ahead of the tile being
// computed, so the HBM stream never waits for the per-cell arithmetic and no
// register holds a load in flight (the one-thread-per-cell kernels of round 1
// were long-scoreboard bound: 38-43% of their stalls, profiles/ncu_r02a.json).
//
// Rules the callers follow (include/rc.h): every row pointer is 16-byte aligned
// at cell 0 and TILE is a multiple of 4, so every copy starts 16-byte aligned;
// a ragged last tile copies its byte count rounded up to 16, i.e. at most one
// fp64 / three fp32 elements past the last cell, which stay inside the row
// because ld is even (fp64 rows) or the row is padded to a multiple of 4 cells
// (fp32 rows: the chunk capacity is a multiple of 256).
#pragma once
#include "ptx.cuh"

namespace rcs {

// STAGES > 0: the stage count as a compile-time constant (must equal `stages`); a power of two lets
// the consumers derive stage and phase from the tile counter with a mask and a shift (one register)
template <int TILE, int STAGES = 0>
struct Ring {
  static_assert(TILE % 4 == 0, "16-byte aligned rows");
  static constexpr bool POW2 = STAGES > 0 && (STAGES & (STAGES - 1)) == 0;
  uint8_t *buf;     // [stages][n8 x TILE x 8 B | n4 x TILE x 4 B]
  uint64_t *full;   // [stages] mbarriers, count 1
  int n8, n4, stages;

  __host__ __device__ static size_t stage_bytes(int n8, int n4) { return (size_t)TILE * (8 * n8 + 4 * n4); }
  __host__ __device__ static size_t smem_bytes(int n8, int n4, int stages) { return stages * stage_bytes(n8, n4); }

  __device__ __forceinline__ double *row8(int s, int r) const {
    return reinterpret_cast<double *>(buf + s * stage_bytes(n8, n4)) + (size_t)r * TILE;
  }
  __device__ __forceinline__ float *row4(int s, int r) const {
    return reinterpret_cast<float *>(buf + s * stage_bytes(n8, n4) + (size_t)TILE * 8 * n8) + (size_t)r * TILE;
  }

  // one thread, before the CTA's first __syncthreads; `full` holds 2 x stages barriers when the
  // warp-specialised runner is used (full[s], then empty[s] = full[stages + s], one arrival per
  // consumer warp)
  __device__ __forceinline__ void init(int consumer_warps = 0) const {
    for (int s = 0; s < stages; ++s) rcx::mbar_init(&full[s], 1);
    if (consumer_warps)
      for (int s = 0; s < stages; ++s) rcx::mbar_init(&full[stages + s], consumer_warps);
    rcx::fence_mbar_init();
  }

  // One thread: copy tile t (cells [t*TILE, min(n, (t+1)*TILE))) into stage s.
  // src8(r) / src4(r): address of cell 0 of fp64 row r / fp32 row r.
  template <class F8, class F4>
  __device__ __forceinline__ void issue(int s, int64_t t, int64_t n, F8 &&src8, F4 &&src4) const {
    const int64_t c0 = t * TILE;
    const uint32_t rem = (uint32_t)(n - c0 < TILE ? n - c0 : TILE);
    const uint32_t b8 = (rem * 8u + 15u) & ~15u, b4 = (rem * 4u + 15u) & ~15u;
    rcx::mbar_arrive_expect_tx(&full[s], n8 * b8 + n4 * b4);
    for (int r = 0; r < n8; ++r) rcx::bulk_g2s(row8(s, r), src8(r) + c0, b8, &full[s]);
    for (int r = 0; r < n4; ++r) rcx::bulk_g2s(row4(s, r), src4(r) + c0, b4, &full[s]);
  }

  // Static round-robin tile schedule over a persistent grid: body(s, t) computes tile t
  // from stage s.  Every thread of the CTA calls run(); blockDim.x == TILE.
  template <class F8, class F4, class Body>
  __device__ __forceinline__ void run(int64_t n, F8 &&src8, F4 &&src4, Body &&body) const {
    const int64_t ntiles = (n + TILE - 1) / TILE;
    if (threadIdx.x == 0)
      for (int s = 0; s < stages; ++s) {
        const int64_t t = blockIdx.x + (int64_t)s * gridDim.x;
        if (t < ntiles) issue(s, t, n, src8, src4);
      }
    // stage index and phase carried incrementally (a runtime `it % stages` is an integer division
    // per tile in every thread)
    int s = 0;
    uint32_t ph = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      rcx::mbar_wait(&full[s], ph);
      body(s, t);
      __syncthreads();  // every thread has read stage s
      const int64_t tn = t + (int64_t)stages * gridDim.x;
      if (threadIdx.x == 0 && tn < ntiles) issue(s, tn, n, src8, src4);
      if (++s == stages) { s = 0; ph ^= 1u; }
    }
  }

  // Warp-specialised schedule: warp 0 is the producer (one elected lane issues the copies of the
  // next tile as soon as its stage is released), warps 1..blockDim/32-1 are consumers, one cell
  // per consumer thread (TILE == blockDim.x - 32).  A consumer warp releases a stage with one
  // arrival on its empty barrier after reading it, so warps drift by up to `stages` tiles and no
  // CTA-wide barrier waits for the slowest cell (Newton iteration counts differ per cell).
  // body(s, t, j): thread j (0..TILE-1) of tile t in stage s.  Returns after the last tile; every
  // thread of the CTA calls it.
  template <class F8, class F4, class Body>
  __device__ __forceinline__ void run_ws(int64_t n, F8 &&src8, F4 &&src4, Body &&body) const {
    const int64_t ntiles = (n + TILE - 1) / TILE;
    uint64_t *empty = full + stages;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
      if ((threadIdx.x & 31) == 0) {
        int s = 0;
        uint32_t ph = 1;  // the first pass over the stages waits for nothing
        bool first = true;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
          if (!first) rcx::mbar_wait_sleep(&empty[s], ph);
          issue(s, t, n, src8, src4);
          if (++s == stages) { s = 0; ph ^= 1u; first = false; }
        }
      }
      __syncwarp();
      return;
    }
    const int j = threadIdx.x - 32;
    int s = 0, it = 0;
    uint32_t ph = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      if constexpr (POW2) {
        s = it & (STAGES - 1);
        ph = (uint32_t)(it / STAGES) & 1u;
        ++it;
      }
      rcx::mbar_wait(&full[s], ph);
      body(s, t, j);
      __syncwarp();
      if ((threadIdx.x & 31) == 0) rcx::mbar_arrive(&empty[s]);
      if constexpr (!POW2)
        if (++s == stages) { s = 0; ph ^= 1u; }
    }
  }

  // run_ws with an early release: body(s, t, j, release) copies what it needs out of stage s and
  // then calls release() -- once, from every lane of the warp (no lane may return before it) -- so
  // the producer refills the stage while the warp is still computing; one or two stages then keep
  // the HBM stream going for kernels whose per-cell arithmetic dwarfs the copy.
  template <class F8, class F4, class Body>
  __device__ __forceinline__ void run_ws_release(int64_t n, F8 &&src8, F4 &&src4, Body &&body) const {
    const int64_t ntiles = (n + TILE - 1) / TILE;
    uint64_t *empty = full + stages;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
      if ((threadIdx.x & 31) == 0) {
        int s = 0;
        uint32_t ph = 1;  // the first pass over the stages waits for nothing
        bool first = true;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
          if (!first) rcx::mbar_wait_sleep(&empty[s], ph);
          issue(s, t, n, src8, src4);
          if (++s == stages) { s = 0; ph ^= 1u; first = false; }
        }
      }
      __syncwarp();
      return;
    }
    const int j = threadIdx.x - 32;
    int s = 0;
    uint32_t ph = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      rcx::mbar_wait(&full[s], ph);
      auto release = [&]() {
        __syncwarp();
        if ((threadIdx.x & 31) == 0) rcx::mbar_arrive(&empty[s]);
      };
      body(s, t, j, release);
      if (++s == stages) { s = 0; ph ^= 1u; }
    }
  }
};

}  // namespace rcs
