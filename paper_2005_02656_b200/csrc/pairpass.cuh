// pairpass.cuh -- device helpers shared by the neighbour search (search.cu) and the
// pair passes (cellpass.cu): unit stencils in shared memory, work claiming and warp
// reductions.
//
// Neighbour lists.  A pair-pass UNIT (stencil.cuh) stages the
// particles of its union stencil as one flat sequence (slots in order, each slot a
// contiguous cell range).  Target t's row holds the FLAT INDICES of its neighbours
// in that sequence, ascending (fixed row stride, 16-bit entries unless a unit
// stencil exceeds 65,535 particles): a pass reads a neighbour's staged data at
// shared index entry - (group start) with no table lookup, and the host decodes
// entries to global ids with the cell tables (sph_get_neighbors).
#pragma once

#include "stencil.cuh"

namespace sphb {

constexpr int kCT = 256;          // search CTA threads
constexpr int kNW = kCT / 32;
constexpr int kTgtU = 416;        // targets per sub-block (a whole 2x2x1 unit, <= 9x9x5 at config 5)
constexpr int kSlots = kKMax;     // slot tables: every stencil the grid chooser admits
#ifndef SPH_CELL_CHUNK
#define SPH_CELL_CHUNK 4
#endif
constexpr int kCellChunk = SPH_CELL_CHUNK;  // consecutive cells per claim (L2 reuse of shared stencils)
constexpr int kSearchCap = 4096;  // staged candidates per group (float4): a unit stencil in one group
constexpr int kSearchTiles = kSearchCap / 32;
constexpr int kSearchWords = kSearchTiles / 32;  // tile bitmask words
constexpr int kDensCap = 4096;    // density: staged particles per group, 4 fp64 fields
constexpr int kIadCap = 4096;     // IAD: the same fields
constexpr int kMomCap = 1312;     // momentum: staged 144-byte records per group (a 48-cell unit in 3 groups)
#ifndef SPH_MOM_THREADS
#define SPH_MOM_THREADS 512
#endif
constexpr int kCTM = SPH_MOM_THREADS;  // momentum CTA: 16 warps, one CTA per SM (A/B builds override)
#ifndef SPH_DENS_THREADS
#define SPH_DENS_THREADS 1024
#endif
constexpr int kCTD = SPH_DENS_THREADS;  // density / IAD CTA: 32 warps, one CTA per SM (A/B builds override)
constexpr int kNWM = kCTM / 32;
constexpr int kNWD = kCTD / 32;
constexpr uint32_t kSent = 0xffffffffu;  // past-the-end row entry
static_assert(kSearchCap % 32 == 0 && kDensCap % 32 == 0 && kIadCap % 32 == 0 && kMomCap % 32 == 0,
              "staging groups are whole tiles");
static_assert(kSlots >= kKMax, "slot tables must hold the largest admitted stencil");

// Per-unit stencil tables.  cum[k] is the flat index of slot k's first particle.
struct CellSm {
  uint32_t t_start[kSlots];     // first sorted index of slot k's cell
  uint32_t cum[kSlots + 1];     // exclusive prefix of the slot counts
  signed char t_sh[kSlots][3];  // periodic image shift of slot k (in periods)
  uint32_t next[2];             // dynamic target counters, by group parity
  Stencil st;
  int c3[3];
  uint32_t sc, ec, total;
  int kself;
};

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double wmax(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Sum NV (power of two) per-lane values over the warp by transpose-reduce: each
// exchange step halves the values a lane keeps, so the cost is NV-1+log2(32/NV)
// shuffles instead of NV*5.  On return v[0] of lane k*(32/NV) holds the sum of
// value k (lanes in between hold the same sums).
template <int NV>
__device__ __forceinline__ void warp_multi_sum(double (&v)[NV]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int cnt = NV, off = 16; cnt > 1; cnt >>= 1, off >>= 1) {
    const bool upper = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < cnt / 2; ++i) {
      const double send = upper ? v[i] : v[i + cnt / 2];
      const double keep = upper ? v[i + cnt / 2] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
#pragma unroll
  for (int off = 16 / NV; off > 0; off >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], off);
}

// transpose-reduce over each 16-lane half: value k of a half ends in its lane 4k (NV = 4)
template <int NV>
__device__ __forceinline__ void half_multi_sum(double (&v)[NV]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int cnt = NV, off = 8; cnt > 1; cnt >>= 1, off >>= 1) {
    const bool upper = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < cnt / 2; ++i) {
      const double send = upper ? v[i] : v[i + cnt / 2];
      const double keep = upper ? v[i + cnt / 2] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
#pragma unroll
  for (int off = 8 / NV; off > 0; off >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], off);
}
__device__ __forceinline__ double half_max(double v) {
#pragma unroll
  for (int o = 8; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ double min_img(double d, double L) {
  if (d > 0.5 * L) d -= L;
  else if (d < -0.5 * L) d += L;
  return d;
}

// Warp 0: per-slot tables of S.st and their prefix (flat staging index of each slot).
// Lane 0 has set S.st / S.sc / S.ec.
__device__ __forceinline__ void slot_tables(const Grid& g, const uint32_t* __restrict__ cstart,
                                            const uint32_t* __restrict__ cend, CellSm& S) {
  const int lane = threadIdx.x;
  const int K = S.st.K;
  uint32_t carry = 0;
  for (int b = 0; b < K; b += 32) {
    const int k = b + lane;
    uint32_t cnt = 0;
    if (k < K) {
      int sh[3];
      const int64_t cell = slot_cell(g, S.st, k, sh);
      const uint32_t s0 = cstart[cell];
      cnt = cend[cell] - s0;
      S.t_start[k] = s0;
      S.t_sh[k][0] = (signed char)sh[0];
      S.t_sh[k][1] = (signed char)sh[1];
      S.t_sh[k][2] = (signed char)sh[2];
    }
    uint32_t x = cnt;  // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (k < K) S.cum[k] = carry + x - cnt;
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
  if (lane == 0) {
    S.cum[K] = carry;
    S.total = carry;
  }
}

// Unit records (one thread per unit, once per step before the search): the union
// stencil of the unit's cells and its target range, so a CTA prologue is one 48-byte
// load instead of a serial chain of dependent cell-table loads.
__device__ __forceinline__ void pack_unit(const Stencil& u, uint32_t sc, uint32_t ec, uint32_t cf,
                                          int4* rec) {
  rec[0] = make_int4(u.lo[0], u.lo[1], u.lo[2], u.K);
  rec[1] = make_int4(u.cnt[0], u.cnt[1], u.cnt[2], u.wrap[0] | (u.wrap[1] << 2) | (u.wrap[2] << 4));
  rec[2] = make_int4((int)sc, (int)ec, (int)cf, 0);
}
__device__ __forceinline__ void unpack_unit(const int4* __restrict__ rec, Stencil& u, uint32_t& sc,
                                            uint32_t& ec, uint32_t* cf = nullptr) {
  const int4 a = rec[0], b = rec[1], c = rec[2];
  if (cf) *cf = (uint32_t)c.z;
  u.lo[0] = a.x; u.lo[1] = a.y; u.lo[2] = a.z; u.K = a.w;
  u.cnt[0] = b.x; u.cnt[1] = b.y; u.cnt[2] = b.z;
  u.wrap[0] = b.w & 3; u.wrap[1] = (b.w >> 2) & 3; u.wrap[2] = (b.w >> 4) & 3;
  sc = (uint32_t)c.x;
  ec = (uint32_t)c.y;
}

// CTA prologue for pair-pass unit u (warp 0, one CTA barrier): the unit's target
// range (its cells are consecutive in the cell list and in particle order), the
// union stencil of its cells, and the slot tables.
__device__ __forceinline__ void unit_setup(const Grid& g, uint32_t u, const int4* __restrict__ urec,
                                           const uint32_t* __restrict__ cstart,
                                           const uint32_t* __restrict__ cend, CellSm& S) {
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) {
      uint32_t sc, ec, cf;
      unpack_unit(urec + 3 * (size_t)u, S.st, sc, ec, &cf);
      S.sc = sc;
      S.ec = ec;
      S.kself = -1;
      cell_coords(g, cf, S.c3);  // first cell of the unit
    }
    __syncwarp();
    slot_tables(g, cstart, cend, S);
  }
  __syncthreads();
}

// The units a pair-pass launch processes: indices [*lo (0 if null), *hi) into `order`
// (the identity if null) -- all units, or the interior / boundary split of the
// multi-GPU overlap (cellpass.cu unit_range).
struct URange {
  const uint32_t* order;
  const uint32_t* lo;
  const uint32_t* hi;
};

// Dynamic claims of work chunks from a global counter, the next claim issued one
// chunk ahead (its atomic's latency overlaps the current chunk).
struct ChunkClaim {
  uint32_t* work;
  uint32_t step, nxt;
  __device__ __forceinline__ uint32_t first(uint32_t* s_chunk) {
    if (threadIdx.x == 0) *s_chunk = atomicAdd(work, step);
    __syncthreads();
    const uint32_t v = *s_chunk;
    __syncthreads();
    if (threadIdx.x == 0) nxt = atomicAdd(work, step);  // lands while this chunk runs
    return v;
  }
  __device__ __forceinline__ uint32_t next(uint32_t* s_chunk) {
    if (threadIdx.x == 0) *s_chunk = nxt;
    __syncthreads();
    const uint32_t v = *s_chunk;
    __syncthreads();
    if (threadIdx.x == 0) nxt = atomicAdd(work, step);
    return v;
  }
};

// slot of flat index f: the largest k < K with cum[k] <= f (skips empty slots)
__device__ __forceinline__ int slot_of(const CellSm& S, uint32_t f) {
  int lo = 0, hi = S.st.K - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (S.cum[mid] <= f) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ void shifts_of(const Grid& g, const CellSm& S, int slot, double sh[3]) {
  sh[0] = S.t_sh[slot][0] * g.L[0];
  sh[1] = S.t_sh[slot][1] * g.L[1];
  sh[2] = S.t_sh[slot][2] * g.L[2];
}

}  // namespace sphb
