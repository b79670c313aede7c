// stencil.cuh -- the per-cell candidate stencil shared by the search and the
// pair passes (host + device, so sph_get_neighbors can decode rows on the host).
//
// A search cell c with largest smoothing length h_max(c) needs, per dimension,
// the cells within R_d = ceil(2 h_max (1 + 2^-20) / edge_d) of c (all cells of
// the dimension when 2R+1 >= nc).  Slots enumerate that box z-major, then y,
// then x; a neighbour-row entry is packed as (slot << 20) | local index in the
// slot's cell, so rows sorted by the packed value are sorted by slot, then by
// particle order -- exactly the order in which candidates are staged.
#pragma once

#include "sph_internal.cuh"

namespace sphb {

constexpr int kKMax = 1024;       // max slots per stencil (R <= 4 in every dim)
constexpr int kLocalBits = 20;    // local index bits of a packed row entry
constexpr uint32_t kLocalMask = (1u << kLocalBits) - 1u;

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

}  // namespace sphb
