// stencil.cuh -- the per-cell candidate stencil shared by the search and the
// pair passes (host + device, so sph_get_neighbors can decode rows on the host).
//
// A search cell c with largest smoothing length h_max(c) needs, per dimension,
// the cells within R_d = ceil(2 h_max (1 + 2^-20) / edge_d) of c (all cells of
// the dimension when 2R+1 >= nc).  Slots enumerate that box z-major, then y,
// then x.  A pair pass stages the stencil of a unit of cells (below) as one flat
// sequence, slot by slot; a neighbour-row entry is the flat index in it, so rows
// sorted by entry are in staging order.
#pragma once

#include <cstring>

#include "sph_internal.cuh"

namespace sphb {

constexpr int kKMax = 1024;       // max slots per stencil (R <= 4 in every dim)

struct Stencil {
  int lo[3];    // first cell coordinate per dim (may be < 0 or run past nc when periodic)
  int cnt[3];   // cells per dim
  int wrap[3];  // 0 open/none, 1 periodic with shifted slots, 2 periodic "all cells" (per-pair min image)
  int K;
};

__host__ __device__ __forceinline__ void cell_coords(const Grid& g, int64_t c, int c3[3]) {
  c3[0] = (int)(c % g.nc[0]);
  c3[1] = (int)((c / g.nc[0]) % g.nc[1]);
  c3[2] = (int)(c / ((int64_t)g.nc[0] * g.nc[1]));
}

__host__ __device__ __forceinline__ int stencil_radius(const Grid& g, int d, double reach) {
  return (int)ceil(reach * g.inv[d]);
}

__host__ __device__ __forceinline__ void make_stencil(const Grid& g, const int c3[3], double reach,
                                                      Stencil& s) {
  for (int d = 0; d < 3; ++d) {
    int R = stencil_radius(g, d, reach);
    if (2 * R + 1 >= g.nc[d]) {
      s.lo[d] = 0;
      s.cnt[d] = g.nc[d];
      s.wrap[d] = g.periodic[d] ? 2 : 0;
    } else if (g.periodic[d]) {
      s.lo[d] = c3[d] - R;
      s.cnt[d] = 2 * R + 1;
      s.wrap[d] = 1;
    } else {
      int l = c3[d] - R < 0 ? 0 : c3[d] - R;
      int u = c3[d] + R > g.nc[d] - 1 ? g.nc[d] - 1 : c3[d] + R;
      s.lo[d] = l;
      s.cnt[d] = u - l + 1;
      s.wrap[d] = 0;
    }
  }
  s.K = s.cnt[0] * s.cnt[1] * s.cnt[2];
}

// slot -> cell id; sh[d] in {-1, 0, +1}: add sh[d] * L[d] to a candidate of that
// cell to bring it next to the target cell (wrap == 1 dims only).
__host__ __device__ __forceinline__ int64_t slot_cell(const Grid& g, const Stencil& s, int k,
                                                      int sh[3]) {
  int i[3] = {k % s.cnt[0], (k / s.cnt[0]) % s.cnt[1], k / (s.cnt[0] * s.cnt[1])};
  int cc[3];
  for (int d = 0; d < 3; ++d) {
    int q = s.lo[d] + i[d];
    sh[d] = 0;
    if (q < 0) {
      q += g.nc[d];
      sh[d] = -1;
    } else if (q >= g.nc[d]) {
      q -= g.nc[d];
      sh[d] = 1;
    }
    cc[d] = q;
  }
  return cc[0] + (int64_t)g.nc[0] * (cc[1] + (int64_t)g.nc[1] * cc[2]);
}

__host__ __device__ __forceinline__ int self_slot(const Stencil& s, const int c3[3]) {
  return (c3[0] - s.lo[0]) + s.cnt[0] * ((c3[1] - s.lo[1]) + s.cnt[1] * (c3[2] - s.lo[2]));
}

__host__ __device__ __forceinline__ uint32_t compact3_hd(uint64_t v) {
  v &= 0x1249249249249249ull;
  v = (v ^ (v >> 2)) & 0x10c30c30c30c30c3ull;
  v = (v ^ (v >> 4)) & 0x100f00f00f00f00full;
  v = (v ^ (v >> 8)) & 0x1f0000ff0000ffull;
  v = (v ^ (v >> 16)) & 0x1f00000000ffffull;
  v = (v ^ (v >> 32)) & 0x1fffffull;
  return (uint32_t)v;
}

// linear cell id of a sort key (Morton code of the cell above the sub-cell and id bits)
__host__ __device__ __forceinline__ int64_t key_cell_hd(const Grid& g, uint64_t key) {
  uint64_t m = g.kshift >= 64 ? 0 : key >> g.kshift;
  int64_t cx = compact3_hd(m), cy = compact3_hd(m >> 1), cz = compact3_hd(m >> 2);
  return cx + (int64_t)g.nc[0] * (cy + (int64_t)g.nc[1] * cz);
}

__host__ __device__ __forceinline__ double reach_of(double hmax) {
  return 2.0 * hmax * (1.0 + 0x1p-20);
}
// stencil reach of a cell: 2 h_max of its own particles (gather), or of every
// particle that may reach into it (symmetric relation: the global h_max)
__host__ __device__ __forceinline__ double cell_reach(const Grid& g, double cell_hmax) {
  return reach_of(cell_hmax > g.hsym ? cell_hmax : g.hsym);
}

// ---------------------------------------------------------------- pair-pass units
// The pair passes give one CTA a UNIT of cells: the cells whose Morton codes agree
// above the lowest g.ubits bits (ubits = 2: an aligned 2x2x1 block; 0: one cell).
// Particles are sorted by cell Morton code, so a unit's targets are one contiguous
// range, and the unit stages the UNION of its cells' stencils once: 4x4x3 = 48 cells
// for four 27-cell stencils, i.e. 12 staged cells per target cell instead of 27.
// The search stages the same unit stencil and writes neighbour rows as flat
// indices into it, so rows are sorted in the passes' staging order.
__host__ __device__ __forceinline__ void unit_base(const Grid& g, const int c3[3], int b3[3]) {
  for (int d = 0; d < 3; ++d) b3[d] = g.ubits > d ? (c3[d] & ~1) : c3[d];
}

// Union (bounding box) of the stencils of the unit's non-empty cells; c3 is any
// cell of the unit.  Depends only on those cells' ranges and h_max, so the search
// (per cell) and the passes (per unit) build the same box on every rank.
__host__ __device__ __forceinline__ void make_unit_stencil(const Grid& g, const int c3[3],
                                                           const uint32_t* cstart, const uint32_t* cend,
                                                           const unsigned long long* chmax, Stencil& u) {
  int b3[3];
  unit_base(g, c3, b3);
  int lo[3] = {0, 0, 0}, hi[3] = {-1, -1, -1};
  bool any = false;
  const int w0 = g.ubits > 0 ? 2 : 1, w1 = g.ubits > 1 ? 2 : 1, w2 = g.ubits > 2 ? 2 : 1;
  for (int dz = 0; dz < w2; ++dz)
    for (int dy = 0; dy < w1; ++dy)
      for (int dx = 0; dx < w0; ++dx) {
        const int q[3] = {b3[0] + dx, b3[1] + dy, b3[2] + dz};
        if (q[0] >= g.nc[0] || q[1] >= g.nc[1] || q[2] >= g.nc[2]) continue;
        const int64_t cell = q[0] + (int64_t)g.nc[0] * (q[1] + (int64_t)g.nc[1] * q[2]);
        const bool self = q[0] == c3[0] && q[1] == c3[1] && q[2] == c3[2];
        if (!self && cstart[cell] >= cend[cell]) continue;  // empty cell: no stencil
        const unsigned long long hb = chmax[cell];
        double hm;
#ifdef __CUDA_ARCH__
        hm = __longlong_as_double((long long)hb);
#else
        memcpy(&hm, &hb, sizeof(double));
#endif
        Stencil s;
        make_stencil(g, q, cell_reach(g, hm), s);
        for (int d = 0; d < 3; ++d) {
          const int l = s.lo[d], h = s.lo[d] + s.cnt[d] - 1;
          lo[d] = any ? (l < lo[d] ? l : lo[d]) : l;
          hi[d] = any ? (h > hi[d] ? h : hi[d]) : h;
          u.wrap[d] = s.wrap[d];
        }
        any = true;
      }
  u.K = 1;
  for (int d = 0; d < 3; ++d) {
    u.lo[d] = lo[d];
    u.cnt[d] = hi[d] - lo[d] + 1;
    u.K *= u.cnt[d];
  }
}

}  // namespace sphb
