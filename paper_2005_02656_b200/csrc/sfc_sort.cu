// sfc_sort.cu -- a1-a3: bounding box, Morton (SFC) keys, LSD radix sort,
// in-place permutation of the particle state, cell-range tables.
//
// PAPER.md P:162 / P:201: "particles are kept in memory in an order that matches
// the octree ... depth-first-search ordering sequence (similar to a Morton
// ordering)".  Here the order is the Morton code of the search cell (high bits)
// followed by the particle id (low bits, reading R25): every search cell is one
// contiguous range of the sorted order, and the order is canonical (independent
// of the input order and of the rank count).
#include "sph_internal.cuh"

namespace sphb {

// ------------------------------------------------------------------ bbox (a1)
// out[0..2] = min x,y,z; out[3..5] = max x,y,z; out[6] = max h; out[7] = sum h;
// out[8] = max id.
constexpr int kRedThreads = 256;
constexpr int kBB = 9;

__device__ __forceinline__ double warp_min(double v) {
  for (int o = 16; o; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(kRedThreads) k_bbox(const double* __restrict__ x,
                                                      const double* __restrict__ y,
                                                      const double* __restrict__ z,
                                                      const double* __restrict__ h,
                                                      const double* __restrict__ m,
                                                      const int64_t* __restrict__ id, int64_t n,
                                                      double* __restrict__ part,
                                                      unsigned long long* __restrict__ bad_id) {
  double v[kBB] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY, 0.0, 0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double xi = x[i], yi = y[i], zi = z[i], hi = h[i], mi = m[i];
    // positions finite, h and m finite and positive; the smallest offending id is
    // reported (sph_diag.first_bad_id) and the step fails with SPH_ERR_NUMERIC
    if (!(isfinite(xi) && isfinite(yi) && isfinite(zi) && hi > 0.0 && hi < INFINITY && mi > 0.0 &&
          mi < INFINITY))
      atomicMin(bad_id, (unsigned long long)id[i]);
    v[0] = fmin(v[0], xi); v[1] = fmin(v[1], yi); v[2] = fmin(v[2], zi);
    v[3] = fmax(v[3], xi); v[4] = fmax(v[4], yi); v[5] = fmax(v[5], zi);
    v[6] = fmax(v[6], hi); v[7] += hi;
    v[8] = fmax(v[8], (double)id[i]);
  }
  __shared__ double sh[kBB][kRedThreads / 32];
  int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = 0; k < kBB; ++k) {
    double r = k < 3 ? warp_min(v[k]) : (k == 7 ? warp_sum(v[k]) : warp_max(v[k]));
    if (lane == 0) sh[k][w] = r;
  }
  __syncthreads();
  if (threadIdx.x < kBB) {
    int k = threadIdx.x;
    double r = sh[k][0];
    for (int q = 1; q < kRedThreads / 32; ++q)
      r = k < 3 ? fmin(r, sh[k][q]) : (k == 7 ? r + sh[k][q] : fmax(r, sh[k][q]));
    part[(int64_t)blockIdx.x * kBB + k] = r;
  }
}

// one warp per reduced value: lanes stride over the block partials, then a fixed
// shuffle tree (deterministic order; a single thread looping over ~600 partials cost
// ~0.1 ms of dependent L2 loads per step)
__global__ void k_bbox_final(const double* __restrict__ part, int nblk, double* __restrict__ out) {
  const int k = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (k >= kBB) return;
  double r = k < 3 ? INFINITY : (k == 7 ? 0.0 : -INFINITY);
  for (int b = lane; b < nblk; b += 32) {
    const double q = part[(int64_t)b * kBB + k];
    r = k < 3 ? fmin(r, q) : (k == 7 ? r + q : fmax(r, q));
  }
  r = k < 3 ? warp_min(r) : (k == 7 ? warp_sum(r) : warp_max(r));
  if (lane == 0) out[k] = r;
}

int launch_bbox(sph_ctx* c) {
  int64_t n = c->P.n;
  int nb = grid_blocks(c, n, kRedThreads, 4);
  k_bbox<<<nb, kRedThreads, 0, c->stream>>>(c->P.x, c->P.y, c->P.z, c->P.h, c->P.m, c->P.id, n,
                                              c->s.red, c->s.bad_id);
  k_bbox_final<<<1, 32 * kBB, 0, c->stream>>>(c->s.red, nb, c->s.bbox);
  return 2;
}

// ------------------------------------------------------------------ keys (a1)

__device__ __forceinline__ int cell_coord(const Grid& g, int d, double v) {
  double q = (v - g.lo[d]) * g.inv[d];
  int c = (int)floor(q);
  c = c < 0 ? 0 : c;
  c = c > g.nc[d] - 1 ? g.nc[d] - 1 : c;
  return c;
}

__device__ __forceinline__ uint64_t spread3(uint64_t v) {  // 21 bits -> every 3rd bit
  v &= 0x1fffffull;
  v = (v | (v << 32)) & 0x1f00000000ffffull;
  v = (v | (v << 16)) & 0x1f0000ff0000ffull;
  v = (v | (v << 8)) & 0x100f00f00f00f00full;
  v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}

__global__ void k_keys(const double* __restrict__ x, const double* __restrict__ y,
                       const double* __restrict__ z, const int64_t* __restrict__ id, int64_t n,
                       Grid g, uint64_t* __restrict__ keys, uint32_t* __restrict__ idx,
                       int64_t i0) {  // idx[i] = i0 + i: absolute index for the sort
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    // cell Morton code (high bits), then the Morton code of the 2^sbits-per-dim
    // sub-cell (so a cell's particles are Z-ordered: staged 32-particle tiles are
    // compact blocks the search can cull), then the id (canonical tie-break, R25)
    const double v3[3] = {x[i], y[i], z[i]};
    uint64_t cc[3], sc[3];
    const double sub = (double)(1 << g.sbits);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const double q = (v3[d] - g.lo[d]) * g.inv[d];
      const int c = cell_coord(g, d, v3[d]);
      int s = (int)floor((q - (double)c) * sub);
      s = s < 0 ? 0 : (s > (1 << g.sbits) - 1 ? (1 << g.sbits) - 1 : s);
      cc[d] = (uint64_t)c;
      sc[d] = (uint64_t)s;
    }
    uint64_t morton = spread3(cc[0]) | (spread3(cc[1]) << 1) | (spread3(cc[2]) << 2);
    morton = (morton << (3 * g.sbits)) | spread3(sc[0]) | (spread3(sc[1]) << 1) | (spread3(sc[2]) << 2);
    uint64_t idm = g.idbits >= 64 ? ~0ull : ((1ull << g.idbits) - 1);
    keys[i] = (g.idbits >= 64 ? 0 : (morton << g.idbits)) | ((uint64_t)id[i] & idm);
    idx[i] = (uint32_t)(i0 + i);
  }
}

int launch_keys(sph_ctx* c) { return launch_keys_range(c, 0, c->P.n); }

int launch_keys_range(sph_ctx* c, int64_t i0, int64_t n) {
  if (n <= 0) return 0;
  k_keys<<<grid_blocks(c, n, 256, 8), 256, 0, c->stream>>>(c->P.x + i0, c->P.y + i0, c->P.z + i0,
                                                          c->P.id + i0, n, c->grid, c->s.keys + i0,
                                                          c->s.idx + i0, i0);
  return 1;
}

// ------------------------------------------------------------------ radix sort (a2)
// LSD, 8-bit digits.  Per pass: per-block digit histograms -> exclusive scan in
// digit-major order -> stable scatter (per-warp ordered segments, match_any ranks).
constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_ITEMS = 16;
constexpr int RS_WSEG = 32 * RS_ITEMS;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;

__global__ void __launch_bounds__(RS_THREADS) k_rs_hist(const uint64_t* __restrict__ keys,
                                                        int64_t n, int shift,
                                                        uint32_t* __restrict__ hist, int nblk) {
  __shared__ uint32_t hs[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) hs[i] = 0;
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * RS_TILE;
  for (int k = threadIdx.x; k < RS_TILE; k += RS_THREADS) {
    int64_t i = base + k;
    if (i < n) atomicAdd(&hs[(keys[i] >> shift) & 255u], 1u);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < 256; d += blockDim.x) hist[(int64_t)d * nblk + blockIdx.x] = hs[d];
}

// exclusive scan of uint32 (n <= 2^32 total): tiles of SC_TILE
constexpr int SC_THREADS = 1024;
constexpr int SC_ITEMS = 8;
constexpr int SC_TILE = SC_THREADS * SC_ITEMS;

__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* sh, uint32_t* total) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t incl = v;
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) sh[w] = incl;
  __syncthreads();
  if (w == 0) {
    uint32_t s = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0;
    uint32_t si = s;
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t t = __shfl_up_sync(0xffffffffu, si, o);
      if (lane >= o) si += t;
    }
    sh[lane] = si - s;
    if (lane == 31) sh[32] = si;
  }
  __syncthreads();
  uint32_t r = sh[w] + incl - v;
  if (total) *total = sh[32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(SC_THREADS) k_scan_reduce(const uint32_t* __restrict__ in,
                                                            int64_t n, uint32_t* __restrict__ sums) {
  __shared__ uint32_t sh[33];
  int64_t base = (int64_t)blockIdx.x * SC_TILE + (int64_t)threadIdx.x * SC_ITEMS;
  uint32_t s = 0;
  for (int k = 0; k < SC_ITEMS; ++k)
    if (base + k < n) s += in[base + k];
  uint32_t tot;
  block_excl_scan(s, sh, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(SC_THREADS) k_scan_sums(uint32_t* sums, int nb) {
  __shared__ uint32_t sh[33];
  uint32_t carry = 0;
  for (int base = 0; base < nb; base += SC_THREADS) {
    int i = base + threadIdx.x;
    uint32_t v = i < nb ? sums[i] : 0;
    uint32_t tot;
    uint32_t e = block_excl_scan(v, sh, &tot);
    if (i < nb) sums[i] = carry + e;
    carry += tot;
  }
}

__global__ void __launch_bounds__(SC_THREADS) k_scan_down(const uint32_t* __restrict__ in,
                                                          uint32_t* __restrict__ out, int64_t n,
                                                          const uint32_t* __restrict__ sums) {
  __shared__ uint32_t sh[33];
  int64_t base = (int64_t)blockIdx.x * SC_TILE + (int64_t)threadIdx.x * SC_ITEMS;
  uint32_t v[SC_ITEMS];
  uint32_t s = 0;
  for (int k = 0; k < SC_ITEMS; ++k) {
    v[k] = base + k < n ? in[base + k] : 0;
    s += v[k];
  }
  uint32_t run = block_excl_scan(s, sh, nullptr) + sums[blockIdx.x];
  for (int k = 0; k < SC_ITEMS; ++k) {
    if (base + k < n) out[base + k] = run;
    run += v[k];
  }
}

static int scan_excl(sph_ctx* c, const uint32_t* in, uint32_t* out, int64_t n) {
  int nb = (int)((n + SC_TILE - 1) / SC_TILE);
  k_scan_reduce<<<nb, SC_THREADS, 0, c->stream>>>(in, n, c->s.scan_tmp);
  k_scan_sums<<<1, SC_THREADS, 0, c->stream>>>(c->s.scan_tmp, nb);
  k_scan_down<<<nb, SC_THREADS, 0, c->stream>>>(in, out, n, c->s.scan_tmp);
  return 3;
}

__global__ void __launch_bounds__(RS_THREADS) k_rs_scatter(const uint64_t* __restrict__ kin,
                                                           const uint32_t* __restrict__ vin,
                                                           uint64_t* __restrict__ kout,
                                                           uint32_t* __restrict__ vout, int64_t n,
                                                           int shift,
                                                           const uint32_t* __restrict__ hscan,
                                                           int nblk) {
  __shared__ uint32_t wc[RS_WARPS][256];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < RS_WARPS * 256; i += blockDim.x) (&wc[0][0])[i] = 0;
  __syncthreads();
  const int64_t wbase = (int64_t)blockIdx.x * RS_TILE + (int64_t)w * RS_WSEG;
  uint32_t dig[RS_ITEMS];
#pragma unroll
  for (int r = 0; r < RS_ITEMS; ++r) {
    int64_t i = wbase + r * 32 + lane;
    dig[r] = i < n ? (uint32_t)((kin[i] >> shift) & 255u) : 256u;
    if (i < n) atomicAdd(&wc[w][dig[r]], 1u);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < 256; d += blockDim.x) {
    uint32_t run = hscan[(int64_t)d * nblk + blockIdx.x];
    for (int q = 0; q < RS_WARPS; ++q) {
      uint32_t t = wc[q][d];
      wc[q][d] = run;
      run += t;
    }
  }
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int r = 0; r < RS_ITEMS; ++r) {
    int64_t i = wbase + r * 32 + lane;
    bool valid = i < n;
    unsigned vm = __ballot_sync(0xffffffffu, valid);
    if (valid) {
      unsigned peers = __match_any_sync(vm, dig[r]);
      uint32_t rank = __popc(peers & lt);
      uint32_t basepos = wc[w][dig[r]];
      uint32_t pos = basepos + rank;
      kout[pos] = kin[i];
      vout[pos] = vin[i];
      __syncwarp(vm);
      if (rank == 0) wc[w][dig[r]] = basepos + __popc(peers);
    }
    __syncwarp();
  }
}

int launch_sort(sph_ctx* c, int nbits, const uint32_t** perm_out) {
  int64_t n = c->P.n;
  int nblk = (int)((n + RS_TILE - 1) / RS_TILE);
  int passes = (nbits + 7) / 8;
  uint64_t* kin = c->s.keys;
  uint64_t* kout = c->s.keys_alt;
  uint32_t* vin = c->s.idx;
  uint32_t* vout = c->s.idx_alt;
  int launched = 0;
  for (int p = 0; p < passes; ++p) {
    int shift = 8 * p;
    k_rs_hist<<<nblk, RS_THREADS, 0, c->stream>>>(kin, n, shift, c->s.hist, nblk);
    launched += 1 + scan_excl(c, c->s.hist, c->s.hist, (int64_t)256 * nblk);
    k_rs_scatter<<<nblk, RS_THREADS, 0, c->stream>>>(kin, vin, kout, vout, n, shift, c->s.hist,
                                                     nblk);
    launched += 1;
    std::swap(kin, kout);
    std::swap(vin, vout);
  }
  // sorted keys must end in s.keys (the cell kernel reads them there)
  if (kin != c->s.keys) {
    std::swap(c->s.keys, c->s.keys_alt);
    std::swap(c->s.idx, c->s.idx_alt);
  }
  *perm_out = c->s.idx;
  return launched;
}

// ------------------------------------------------------------------ permute (a2)
struct Fields13 {
  double* f[13];
};

__global__ void k_gather(Fields13 src, const int64_t* __restrict__ id_src,
                         const uint32_t* __restrict__ perm, int64_t n, double* __restrict__ dst,
                         int64_t stride, int64_t* __restrict__ id_dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t j = perm[i];
#pragma unroll
    for (int k = 0; k < 13; ++k) dst[k * stride + i] = src.f[k][j];
    id_dst[i] = id_src[j];
  }
}

__global__ void k_scatter_back(Fields13 dst, int64_t* __restrict__ id_dst,
                               const double* __restrict__ src, int64_t stride,
                               const int64_t* __restrict__ id_src, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int k = 0; k < 13; ++k) dst.f[k][i] = src[k * stride + i];
    id_dst[i] = id_src[i];
  }
}

int launch_permute(sph_ctx* c, const uint32_t* perm) {
  sph_particles& P = c->P;
  Fields13 f = {{P.x, P.y, P.z, P.vx, P.vy, P.vz, P.h, P.m, P.u, P.vhx, P.vhy, P.vhz, P.du_prev}};
  int nb = grid_blocks(c, P.n, 256, 8);
  k_gather<<<nb, 256, 0, c->stream>>>(f, P.id, perm, P.n, c->s.gather, c->cap, c->s.gather_id);
  k_scatter_back<<<nb, 256, 0, c->stream>>>(f, P.id, c->s.gather, c->cap, c->s.gather_id, P.n);
  return 2;
}

// ------------------------------------------------------------------ cell tables (a3)
__device__ __forceinline__ uint32_t compact3(uint64_t v) {  // inverse of spread3
  v &= 0x1249249249249249ull;
  v = (v ^ (v >> 2)) & 0x10c30c30c30c30c3ull;
  v = (v ^ (v >> 4)) & 0x100f00f00f00f00full;
  v = (v ^ (v >> 8)) & 0x1f0000ff0000ffull;
  v = (v ^ (v >> 16)) & 0x1f00000000ffffull;
  v = (v ^ (v >> 32)) & 0x1fffffull;
  return (uint32_t)v;
}

__device__ __forceinline__ int64_t key_cell(const Grid& g, uint64_t key) {
  uint64_t m = g.kshift >= 64 ? 0 : key >> g.kshift;
  int64_t cx = compact3(m), cy = compact3(m >> 1), cz = compact3(m >> 2);
  return cx + (int64_t)g.nc[0] * (cy + (int64_t)g.nc[1] * cz);
}

__global__ void k_cells(const uint64_t* __restrict__ keys, int64_t n, Grid g,
                        uint32_t* __restrict__ cstart, uint32_t* __restrict__ cend,
                        uint32_t* __restrict__ flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = key_cell(g, keys[i]);
    const bool head = i == 0 || key_cell(g, keys[i - 1]) != c;
    if (head) cstart[c] = (uint32_t)i;
    if (i == n - 1 || key_cell(g, keys[i + 1]) != c) cend[c] = (uint32_t)(i + 1);
    flag[i] = head ? 1u : 0u;
  }
}

// non-empty cells in Morton order (deterministic: rank = exclusive scan of heads)
__global__ void k_cell_list(const uint64_t* __restrict__ keys, int64_t n, Grid g,
                            const uint32_t* __restrict__ flag, const uint32_t* __restrict__ rank,
                            uint32_t* __restrict__ list, uint32_t* __restrict__ nlist) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (flag[i]) list[rank[i]] = (uint32_t)key_cell(g, keys[i]);
    if (i == n - 1) *nlist = rank[i] + flag[i];
  }
}

// max h per non-empty cell (one warp per cell): sets the cell's stencil radius
__global__ void k_cell_hmax(const uint32_t* __restrict__ list, const uint32_t* __restrict__ nlist,
                            const uint32_t* __restrict__ cstart, const uint32_t* __restrict__ cend,
                            const double* __restrict__ h, unsigned long long* __restrict__ chmax) {
  const int lane = threadIdx.x & 31;
  const uint32_t nl = *nlist;
  for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nl;
       w += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t c = list[w];
    double m = 0.0;
    for (uint32_t i = cstart[c] + lane; i < cend[c]; i += 32) m = fmax(m, h[i]);
    m = warp_max(m);
    if (lane == 0) chmax[c] = (unsigned long long)__double_as_longlong(m);
  }
}

// first particle of each pair-pass unit (the cells sharing Morton code >> ubits)
__global__ void k_unit_flags(const uint64_t* __restrict__ keys, int64_t n, Grid g,
                             uint32_t* __restrict__ flag) {
  const int sh = g.kshift + g.ubits;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t u = sh >= 64 ? 0 : keys[i] >> sh;
    flag[i] = (i == 0 || (sh >= 64 ? 0 : keys[i - 1] >> sh) != u) ? 1u : 0u;
  }
}

// unit list: index into the cell list of each unit's first cell, plus the end
// sentinel list[nunit] = ncell_list (a unit spans cells list[u] .. list[u+1]-1)
__global__ void k_unit_list(int64_t n, const uint32_t* __restrict__ uflag,
                            const uint32_t* __restrict__ urank, const uint32_t* __restrict__ cflag,
                            const uint32_t* __restrict__ crank, uint32_t* __restrict__ list,
                            uint32_t* __restrict__ nlist) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (uflag[i]) list[urank[i]] = crank[i];  // the unit's first particle heads its first cell
    if (i == n - 1) {
      const uint32_t nu = urank[i] + uflag[i];
      *nlist = nu;
      list[nu] = crank[i] + cflag[i];
    }
  }
}

// cell ranges of the halo segment [i0, i0 + n) (sorted; cells disjoint from owned ones)
__global__ void k_cells_range(const uint64_t* __restrict__ keys, int64_t i0, int64_t n, Grid g,
                              uint32_t* __restrict__ cstart, uint32_t* __restrict__ cend) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + k;
    const int64_t c = key_cell(g, keys[i]);
    if (k == 0 || key_cell(g, keys[i - 1]) != c) cstart[c] = (uint32_t)i;
    if (k == n - 1 || key_cell(g, keys[i + 1]) != c) cend[c] = (uint32_t)(i + 1);
  }
}

int launch_cells_halo(sph_ctx* c, int64_t i0, int64_t n) {
  if (n <= 0) return 0;
  k_cells_range<<<grid_blocks(c, n, 256, 8), 256, 0, c->stream>>>(c->s.keys, i0, n, c->grid,
                                                                 c->s.cell_start, c->s.cell_end);
  return 1;
}

int scan_u32(sph_ctx* c, const uint32_t* in, uint32_t* out, int64_t n) {
  return n > 0 ? scan_excl(c, in, out, n) : 0;
}

int launch_cells(sph_ctx* c) {
  const int64_t n = c->P.n;
  cudaMemsetAsync(c->s.cell_start, 0, sizeof(uint32_t) * c->grid.ncell, c->stream);
  cudaMemsetAsync(c->s.cell_end, 0, sizeof(uint32_t) * c->grid.ncell, c->stream);
  if (n == 0) {  // a rank may own no particle
    cudaMemsetAsync(c->s.ncell_list, 0, sizeof(uint32_t), c->stream);
    cudaMemsetAsync(c->s.nunit_list, 0, sizeof(uint32_t), c->stream);
    return 0;
  }
  const int nb = grid_blocks(c, n, 256, 8);
  k_cells<<<nb, 256, 0, c->stream>>>(c->s.keys, n, c->grid, c->s.cell_start, c->s.cell_end,
                                     c->s.cell_flag);
  int k = 1 + scan_excl(c, c->s.cell_flag, c->s.cell_rank, n);
  k_cell_list<<<nb, 256, 0, c->stream>>>(c->s.keys, n, c->grid, c->s.cell_flag, c->s.cell_rank,
                                         c->s.cell_list, c->s.ncell_list);
  k_cell_hmax<<<grid_blocks(c, n, 256, 8), 256, 0, c->stream>>>(
      c->s.cell_list, c->s.ncell_list, c->s.cell_start, c->s.cell_end, c->P.h, c->s.cell_hmax);
  // pair-pass units (stencil.cuh): heads where the unit key changes, scanned into a list
  k_unit_flags<<<nb, 256, 0, c->stream>>>(c->s.keys, n, c->grid, c->s.unit_flag);
  k += scan_excl(c, c->s.unit_flag, c->s.unit_rank, n);
  k_unit_list<<<nb, 256, 0, c->stream>>>(n, c->s.unit_flag, c->s.unit_rank, c->s.cell_flag,
                                         c->s.cell_rank, c->s.unit_list, c->s.nunit_list);
  return k + 4;
}

}  // namespace sphb
