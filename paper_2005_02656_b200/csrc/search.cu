// search.cu -- a5 neighbour search N(a) = {b != a : r_ab^2 < (2 h_a)^2} (P:103,
// P:149 / Eq. 6 support, reading R10; symmetric variant r < 2 max(h_a, h_b), R24).
//
// One CTA per pair-pass UNIT (stencil.cuh): the unit's union stencil is staged in
// shared memory as fp32 coordinates relative to the unit's base-cell corner
// (periodic images shifted at staging time), cut into 32-candidate tiles with fp32
// bounding boxes.  LANE PER TARGET: a warp takes 32 consecutive (Z-ordered, so
// compact) targets, culls the tiles no member can reach with one box-to-box test,
// and streams the surviving tiles' candidates from shared memory as broadcasts --
// every lane tests the same candidate against its own target: one fp32 subtraction
// against the band's lower edge whose SIGN BIT is the hit (funnel-shifted into a
// 32-bit tile mask) and a running min |r^2 - lo| that flags the rare ambiguous tile --
// ~9 instructions per test, no per-hit bookkeeping.  The lane appends the segment
// (mask, tile) to its target's row region (one 8-byte store per non-empty tile).  k_expand_rows then rewrites every
// row in place as flat staging indices (pairpass.cuh), a warp per row through shared
// memory, so the row stores are coalesced (per-bit stores from the lane-per-target
// loop touched 32 rows per instruction and doubled the search time).
//
// Exactness: fp32 test with an error band, the exact fp64 test in
// the oracle's association (__dmul_rn/__dadd_rn, minimum image) for candidates
// inside the band, so lists are bit-exact.
#include <algorithm>

#include "pairpass.cuh"

namespace sphb {

#ifndef SPH_SEARCH_THREADS
#define SPH_SEARCH_THREADS 320
#endif
constexpr int kCTS = SPH_SEARCH_THREADS;  // search CTA: 10 warps = one 32-target block each per round
constexpr int kNWS = kCTS / 32;

struct TgtW {  // per-target search data (fp32 band + own flat index; the rare exact test
  float f[6];   // re-reads the fp64 position) -- x, y, z (unit-relative), band lo, hi, width
  uint32_t self;
};

__device__ __forceinline__ bool exact_hit(const Grid& g, const double* __restrict__ x,
                                          const double* __restrict__ y, const double* __restrict__ z,
                                          uint32_t j, uint32_t t, const double* pos, double lim) {
  // r^2 in the oracle's association, no FMA, minimum image (Eq. 6; R10)
  if (j == t) return false;
  double ex = __dsub_rn(x[j], pos[0]), ey = __dsub_rn(y[j], pos[1]), ez = __dsub_rn(z[j], pos[2]);
  if (g.periodic[0]) ex = min_img(ex, g.L[0]);
  if (g.periodic[1]) ey = min_img(ey, g.L[1]);
  if (g.periodic[2]) ez = min_img(ez, g.L[2]);
  return __dadd_rn(__dadd_rn(__dmul_rn(ex, ex), __dmul_rn(ey, ey)), __dmul_rn(ez, ez)) < lim;
}

__device__ __forceinline__ float wrap1(float d, float L) {
  return d > 0.5f * L ? d - L : (d < -0.5f * L ? d + L : d);
}

// fp32 band [lo, hi) around lim = (2h)^2 for a staged-coordinate bound M (DESIGN.md
// §6): r2_32 < lo implies r2 < lim, r2_32 >= hi implies r2 >= lim
__device__ __forceinline__ float2 band32(double hh, double M) {
  const double th = 2.0 * hh, lim = __dmul_rn(th, th);
  const double mh = M / hh;
  const double delta = 0x1p-20 * (2.0 + 2.0 * mh + 0x1p-20 * mh * mh);
  if (!(delta < 0.25)) return make_float2(-1.0f, INFINITY);
  return make_float2((float)(lim * (1.0 - delta)), (float)(lim * (1.0 + delta)));
}

// Unit records (one thread per unit, once per step before the search).  Multi-GPU
// (iflag != null): a unit is INTERIOR when no slot of its stencil holds halo particles
// (halos sit behind the n_owned owned particles), i.e. its pair passes read nothing a
// halo exchange delivers -- they run while the exchange is in flight (sph_api.cu).
__global__ void k_unit_prep(Grid g, const uint32_t* __restrict__ clist, const uint32_t* __restrict__ ulist,
                            const uint32_t* __restrict__ nulist, const uint32_t* __restrict__ cstart,
                            const uint32_t* __restrict__ cend, const unsigned long long* __restrict__ chmax,
                            int4* __restrict__ urec, int64_t n_owned, uint32_t* __restrict__ iflag) {
  const uint32_t nu = *nulist;
  for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < nu; u += gridDim.x * blockDim.x) {
    const uint32_t i0 = ulist[u], i1 = ulist[u + 1];
    const uint32_t cf = clist[i0], cl = clist[i1 - 1];
    int c3[3];
    cell_coords(g, cf, c3);
    Stencil st;
    make_unit_stencil(g, c3, cstart, cend, chmax, st);
    pack_unit(st, cstart[cf], cend[cl], cf, urec + 3 * (size_t)u);
    if (iflag) {
      bool interior = true;
      for (int k = 0; k < st.K && interior; ++k) {
        int sh[3];
        const int64_t cell = slot_cell(g, st, k, sh);
        if (cend[cell] > cstart[cell] && (int64_t)cstart[cell] >= n_owned) interior = false;
      }
      iflag[u] = interior ? 1u : 0u;
    }
  }
}

// unit order for the overlapped passes: interior units first, then boundary units, each
// in Morton order (iexcl = exclusive scan of iflag over the unit indices)
__global__ void k_unit_order(const uint32_t* __restrict__ nulist, const uint32_t* __restrict__ iflag,
                             const uint32_t* __restrict__ iexcl, uint32_t* __restrict__ order,
                             uint32_t* __restrict__ bounds) {
  const uint32_t nu = *nulist;
  const uint32_t nint = nu ? iexcl[nu - 1] + iflag[nu - 1] : 0u;
  for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < nu; u += gridDim.x * blockDim.x)
    order[iflag[u] ? iexcl[u] : nint + (u - iexcl[u])] = u;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    bounds[0] = 0;
    bounds[1] = nint;
    bounds[2] = nu;
  }
}

int launch_unit_order(sph_ctx* c) {
  int k = scan_u32(c, c->s.unit_iflag, c->s.unit_iexcl, c->P.n);
  k_unit_order<<<grid_blocks(c, c->P.n, 256, 4), 256, 0, c->stream>>>(c->s.nunit_list, c->s.unit_iflag,
                                                                      c->s.unit_iexcl, c->s.unit_order,
                                                                      c->s.unit_bounds);
  return k + 1;
}

// W2: a periodic dim whose stencil spans every cell (per-pair minimum image in fp32).
// SYM: symmetric relation -- each staged candidate carries its own band, and the exact
// test uses the larger of the two limits (the oracle's (2 max h)^2).
template <bool W2, bool SYM, typename E>
__global__ void __launch_bounds__(kCTS, 2) k_search(const double* __restrict__ x,
                                                 const double* __restrict__ y,
                                                 const double* __restrict__ z,
                                                 const double* __restrict__ h, Grid g,
                                                 const uint32_t* __restrict__ cstart,
                                                 const uint32_t* __restrict__ cend,
                                                 const int4* __restrict__ urec,
                                                 const uint32_t* __restrict__ nulist,
                                                 uint32_t* __restrict__ work, E* __restrict__ nbr,
                                                 uint32_t* __restrict__ ncount, uint32_t* __restrict__ nseg,
                                                 int maxn, unsigned int* __restrict__ maxima) {
  extern __shared__ float4 cand[];  // kSearchCap + 32 (last tile padded with sentinels)
  float2* const candb = reinterpret_cast<float2*>(cand + kSearchCap + 32);  // SYM: per-candidate band
  __shared__ CellSm S;
  // per staged HALF tile (16 candidates): fp32 bounding box; .w of thi: SYM largest band
  __shared__ float4 tlo[2 * kSearchTiles], thi[2 * kSearchTiles];
  __shared__ uint32_t tcnt[kTgtU], tseg[kTgtU];            // per target: neighbours / segments so far
  __shared__ TgtW TW[kTgtU];
  __shared__ uint32_t s_chunk;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned int mxcnt = 0, mxseg = 0, wide = 0;
  const uint32_t segcap = (uint32_t)((size_t)maxn * sizeof(E) / sizeof(uint2));  // segments a row region holds
  const uint32_t nun = *nulist;
  const uint32_t uchunk = (uint32_t)kCellChunk >> g.ubits ? (uint32_t)kCellChunk >> g.ubits : 1u;
  ChunkClaim claim{work, uchunk, 0u};
  for (uint32_t cfirst = claim.first(&s_chunk); cfirst < nun; cfirst = claim.next(&s_chunk)) {
    for (uint32_t ci = cfirst; ci < min(nun, cfirst + uchunk); ++ci) {
      unit_setup(g, ci, urec, cstart, cend, S);
      const Stencil st = S.st;
      if (sizeof(E) < 4 && S.total > 0xffffu) {  // 16-bit rows cannot index this unit stencil:
        wide = 1;                                 // the host reruns the search with 32-bit rows
        continue;
      }
      int b3[3];
      unit_base(g, S.c3, b3);
      double org[3], M = 0.0;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const double edge = g.inv[d] > 0.0 ? 1.0 / g.inv[d] : 0.0;
        org[d] = g.lo[d] + b3[d] * edge;
        // bound on |staged or target coordinate - org| (stencil cells + 1 cell of slack)
        const double Md = st.wrap[d] == 2
                              ? g.L[d]
                              : (double)(max(b3[d] - st.lo[d], st.lo[d] + st.cnt[d] - b3[d]) + 1) * edge;
        M = fmax(M, Md);
      }
      for (uint32_t t0 = S.sc; t0 < S.ec; t0 += kTgtU) {
        const uint32_t t1 = min(S.ec, t0 + kTgtU);
        for (uint32_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
          tcnt[t - t0] = 0;
          tseg[t - t0] = 0;
          const double ha = h[t];
          const float2 bd = band32(ha, M);
          const double px = x[t], py = y[t], pz = z[t];
          TgtW& w = TW[t - t0];
          w.f[0] = (float)(px - org[0]);
          w.f[1] = (float)(py - org[1]);
          w.f[2] = (float)(pz - org[2]);
          w.f[3] = bd.x;
          w.f[4] = bd.y;
          // |d| (the fused fl(r2 - lo) below) of a candidate inside [lo, hi) is below this:
          // hi - lo plus 2^-20 hi for the three roundings of the fused chain (<= 3u max(lo, r2)
          // on each side of the test)
          w.f[5] = bd.y < INFINITY ? (bd.y - bd.x) * (1.0f + 0x1p-20f) + 0x1p-20f * bd.y + 0x1p-126f : INFINITY;
          // own flat staging index (the unit slot of the target's cell): never its own neighbour
          w.self = 0xffffffffu;
          for (int dz = 0; dz < (g.ubits > 2 ? 2 : 1); ++dz)
            for (int dy = 0; dy < (g.ubits > 1 ? 2 : 1); ++dy)
              for (int dx = 0; dx < (g.ubits > 0 ? 2 : 1); ++dx) {
                const int q0 = b3[0] + dx, q1 = b3[1] + dy, q2 = b3[2] + dz;
                if (q0 >= g.nc[0] || q1 >= g.nc[1] || q2 >= g.nc[2]) continue;
                const int64_t cell = q0 + (int64_t)g.nc[0] * (q1 + (int64_t)g.nc[1] * q2);
                const uint32_t cs0 = cstart[cell];
                if (t >= cs0 && t < cend[cell]) {
                  const int us = (q0 - st.lo[0]) + st.cnt[0] * ((q1 - st.lo[1]) + st.cnt[1] * (q2 - st.lo[2]));
                  w.self = S.cum[us] + (t - cs0);
                }
              }
        }
        __syncthreads();
        for (uint32_t gb = 0; gb < S.total; gb += kSearchCap) {
          const int total = (int)(min(S.total, gb + kSearchCap) - gb);
          for (int q = threadIdx.x; q < total; q += blockDim.x) {  // flat staging, all threads
            const uint32_t f = gb + q;
            const int slot = slot_of(S, f);
            const uint32_t j = S.t_start[slot] + (f - S.cum[slot]);
            double sh[3];
            shifts_of(g, S, slot, sh);
            float4 v;
            v.x = (float)((x[j] + sh[0]) - org[0]);
            v.y = (float)((y[j] + sh[1]) - org[1]);
            v.z = (float)((z[j] + sh[2]) - org[2]);
            v.w = 0.0f;
            cand[q] = v;
            if constexpr (SYM) candb[q] = band32(h[j], M);
          }
          // pad the last tile with far-away sentinels (never a hit, never ambiguous)
          const int ntile = (total + 31) / 32;
          for (int q = total + threadIdx.x; q < 32 * ntile; q += blockDim.x) {
            cand[q] = make_float4(INFINITY, INFINITY, INFINITY, 0.0f);
            if constexpr (SYM) candb[q] = make_float2(-1.0f, -1.0f);
          }
          __syncthreads();
          // half-tile bounding boxes (staged candidates are Z-ordered within each cell, so
          // 16 consecutive candidates are a compact block); one warp per tile
          for (int q = warp; q < ntile; q += kNWS) {
            const float4 v = cand[32 * q + lane];
            const bool ok = v.x != INFINITY;
            float lx = ok ? v.x : INFINITY, ly = ok ? v.y : INFINITY, lz = ok ? v.z : INFINITY;
            float hx = ok ? v.x : -INFINITY, hy = ok ? v.y : -INFINITY, hz = ok ? v.z : -INFINITY;
            float hb = -1.0f;  // SYM: largest candidate band of the tile
            if constexpr (SYM) hb = ok ? candb[32 * q + lane].y : -1.0f;
#pragma unroll
            for (int o = 8; o; o >>= 1) {  // within each 16-lane half
              if constexpr (SYM) hb = fmaxf(hb, __shfl_xor_sync(0xffffffffu, hb, o));
              lx = fminf(lx, __shfl_xor_sync(0xffffffffu, lx, o));
              ly = fminf(ly, __shfl_xor_sync(0xffffffffu, ly, o));
              lz = fminf(lz, __shfl_xor_sync(0xffffffffu, lz, o));
              hx = fmaxf(hx, __shfl_xor_sync(0xffffffffu, hx, o));
              hy = fmaxf(hy, __shfl_xor_sync(0xffffffffu, hy, o));
              hz = fmaxf(hz, __shfl_xor_sync(0xffffffffu, hz, o));
            }
            if ((lane & 15) == 0) {
              tlo[2 * q + (lane >> 4)] = make_float4(lx, ly, lz, 0.f);
              thi[2 * q + (lane >> 4)] = make_float4(hx, hy, hz, hb);
            }
          }
          __syncthreads();
          // lane per target: 32 consecutive targets per warp
          for (uint32_t tb = t0 + 32u * warp; tb < t1; tb += 32u * kNWS) {
            const uint32_t t = tb + lane;
            const bool act = t < t1;
            const TgtW& T = TW[act ? t - t0 : 0];
            const float ax = T.f[0], ay = T.f[1], az = T.f[2];
            const float lo = act ? T.f[3] : -1.0f, hi = act ? T.f[4] : -1.0f;
            const float wband = act ? T.f[5] : -1.0f;
            const uint32_t selff = T.self - gb;  // >= ntile*32 (wraps) when not in this group
            const uint32_t selfq = selff >> 5, selfbit = 1u << (selff & 31u);
            uint32_t ncn = act ? tcnt[t - t0] : 0u, nsg = act ? tseg[t - t0] : 0u;
            uint2* const row = reinterpret_cast<uint2*>(nbr + (size_t)(act ? t : 0) * maxn);
            // the block's bounding box and largest band (box-to-box culling)
            float blx = act ? ax : INFINITY, bly = act ? ay : INFINITY, blz = act ? az : INFINITY;
            float bhx = act ? ax : -INFINITY, bhy = act ? ay : -INFINITY, bhz = act ? az : -INFINITY;
            float bhi = hi;
#pragma unroll
            for (int o = 16; o; o >>= 1) {
              blx = fminf(blx, __shfl_xor_sync(0xffffffffu, blx, o));
              bly = fminf(bly, __shfl_xor_sync(0xffffffffu, bly, o));
              blz = fminf(blz, __shfl_xor_sync(0xffffffffu, blz, o));
              bhx = fmaxf(bhx, __shfl_xor_sync(0xffffffffu, bhx, o));
              bhy = fmaxf(bhy, __shfl_xor_sync(0xffffffffu, bhy, o));
              bhz = fmaxf(bhz, __shfl_xor_sync(0xffffffffu, bhz, o));
              bhi = fmaxf(bhi, __shfl_xor_sync(0xffffffffu, bhi, o));
            }
            // Tiles any member can reach.  Box gap per dim in the prefilter's own fp32
            // expression: rounding is monotone, so the gap never exceeds |c - a| of a
            // member pair, box d2 <= r2_32, and box d2 >= every hi excludes hits and
            // ambiguous candidates alike (lists stay exact).
            // half tiles any member can reach (one bit per 16 candidates)
            uint32_t need[2 * kSearchWords];
#pragma unroll
            for (int w = 0; w < 2 * kSearchWords; ++w) {
              const int q = 32 * w + lane;  // half-tile index
              bool nd = false;
              if (q < 2 * ntile) {
                if constexpr (W2) {
                  nd = true;
                } else {
                  const float4 L = tlo[q], H = thi[q];
                  const float bx = fmaxf(fmaxf(L.x - bhx, blx - H.x), 0.f);
                  const float by = fmaxf(fmaxf(L.y - bhy, bly - H.y), 0.f);
                  const float bz = fmaxf(fmaxf(L.z - bhz, blz - H.z), 0.f);
                  nd = fmaf(bz, bz, fmaf(by, by, bx * bx)) < fmaxf(bhi, SYM ? H.w : -1.0f);
                }
              }
              need[w] = __ballot_sync(0xffffffffu, nd);
            }
#pragma unroll 1
            for (int w = 0; w < 2 * kSearchWords; ++w) {
              // tiles of this word (16 per word) with any half needed: bit pairs (lo, hi)
              const uint32_t hw = need[w];
              uint32_t nm = (hw | (hw >> 1)) & 0x55555555u;
              while (nm) {
                const int b2 = __ffs(nm) - 1;  // even bit: the tile's low half
                nm &= nm - 1;
                const int q = 16 * w + (b2 >> 1);
                const bool need_lo = (hw >> b2) & 1u, need_hi = (hw >> (b2 + 1)) & 1u;
                const float4* cq = cand + 32 * q;
                uint32_t in = 0u;
                // rare: exact fp64 test of candidate b (the oracle's r^2 < (2h)^2, R10)
                auto exact = [&](uint32_t b) -> bool {
                  const uint32_t f = gb + 32u * q + b;
                  const int kq = slot_of(S, f);
                  const uint32_t j = S.t_start[kq] + (f - S.cum[kq]);
                  const double tha = 2.0 * h[t];
                  double lim = __dmul_rn(tha, tha);
                  if constexpr (SYM) {
                    const double thb = 2.0 * h[j];
                    lim = fmax(lim, __dmul_rn(thb, thb));
                  }
                  const double pos[3] = {x[t], y[t], z[t]};
                  return exact_hit(g, x, y, z, j, t, pos, lim);
                };
                auto r2of = [&](int k) -> float {
                  const float4 c = cq[k];
                  float dx = c.x - ax, dy = c.y - ay, dz = c.z - az;
                  if constexpr (W2) {
                    if (st.wrap[0] == 2) dx = wrap1(dx, (float)g.L[0]);
                    if (st.wrap[1] == 2) dy = wrap1(dy, (float)g.L[1]);
                    if (st.wrap[2] == 2) dz = wrap1(dz, (float)g.L[2]);
                  }
                  return fmaf(dz, dz, fmaf(dy, dy, dx * dx));
                };
                // r2 - lo in one fused chain (three FFMA, no separate subtract)
                auto dof = [&](int k) -> float {
                  const float4 c = cq[k];
                  float dx = c.x - ax, dy = c.y - ay, dz = c.z - az;
                  if constexpr (W2) {
                    if (st.wrap[0] == 2) dx = wrap1(dx, (float)g.L[0]);
                    if (st.wrap[1] == 2) dy = wrap1(dy, (float)g.L[1]);
                    if (st.wrap[2] == 2) dz = wrap1(dz, (float)g.L[2]);
                  }
                  return fmaf(dz, dz, fmaf(dy, dy, fmaf(dx, dx, -lo)));
                };
                if constexpr (!SYM) {
                  // hit iff d = r2 - lo < 0: the sign bit, funnel-shifted in (candidate 31
                  // first, so bit k ends at position k); a candidate inside [lo, hi) has
                  // |d| < wband, caught by the running minimum
                  // (a half tile no member can reach is skipped: its 16 bits stay 0)
                  float mn = INFINITY;
                  if (need_hi) {
#pragma unroll
                    for (int k = 31; k >= 16; --k) {
                      const float d = dof(k);
                      in = __funnelshift_l(__float_as_uint(d), in, 1);
                      mn = fminf(mn, fabsf(d));
                    }
                  }
                  in <<= need_hi ? 0 : 16;
                  if (need_lo) {
#pragma unroll
                    for (int k = 15; k >= 0; --k) {
                      const float d = dof(k);
                      in = __funnelshift_l(__float_as_uint(d), in, 1);
                      mn = fminf(mn, fabsf(d));
                    }
                  } else {
                    in <<= 16;
                  }
                  if (!act) in = 0u;
                  const bool slow = mn < wband;
                  if (__any_sync(0xffffffffu, slow) && slow) {
                    for (int k = 0; k < 32; ++k)
                      if (fabsf(dof(k)) < wband) in = exact((uint32_t)k) ? in | (1u << k) : in & ~(1u << k);
                  }
                } else {  // symmetric relation: either side's support, per-candidate band
                  uint32_t near = 0u;
#pragma unroll
                  for (int k = 0; k < 32; ++k) {
                    const float r = r2of(k);
                    const float2 cb = candb[32 * q + k];
                    if (r < fmaxf(lo, cb.x)) in |= 1u << k;
                    if (r < fmaxf(hi, cb.y)) near |= 1u << k;
                  }
                  if (!act) in = near = 0u;  // a padding lane must not pick up candidate bands
                  uint32_t amb = near & ~in;
                  if (__any_sync(0xffffffffu, amb != 0u)) {
                    while (amb) {
                      const uint32_t b = __ffs(amb) - 1;
                      amb &= amb - 1;
                      if (exact(b)) in |= 1u << b;
                    }
                  }
                }
                if ((uint32_t)q == selfq) in &= ~selfbit;
                // append the segment (mask, first flat index of the tile); a row region
                // that would overflow is counted, not written (the host grows it, R23)
                if (in) {
                  if (nsg < segcap) row[nsg] = make_uint2(in, gb + 32u * (uint32_t)q);
                  ++nsg;
                  ncn += __popc(in);
                }
              }
            }
            if (act) {
              tcnt[t - t0] = ncn;
              tseg[t - t0] = nsg;
            }
          }
          __syncthreads();
        }
        for (uint32_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
          const uint32_t nc = tcnt[t - t0], ns = tseg[t - t0];
          ncount[t] = nc;
          nseg[t] = ns;
          mxcnt = max(mxcnt, nc);
          mxseg = max(mxseg, ns);
        }
        __syncthreads();
      }
    }
  }
  // largest neighbour count (row capacity, diagnostics) and segment count of the launch;
  // a unit too large for 16-bit rows
  for (int o = 16; o; o >>= 1) {
    mxcnt = max(mxcnt, __shfl_xor_sync(0xffffffffu, mxcnt, o));
    mxseg = max(mxseg, __shfl_xor_sync(0xffffffffu, mxseg, o));
  }
  if (lane == 0 && mxcnt) atomicMax(&maxima[0], mxcnt);
  if (lane == 0 && mxseg > segcap) atomicOr(&maxima[2], 1u);
  if (wide && threadIdx.x == 0) atomicOr(&maxima[1], 1u);
}

// Rows in place: segments (mask, first flat index) -> ascending flat indices.  A warp
// per row: its segments and their exclusive prefix (a warp scan) are staged in shared
// memory (all of them before any entry is written back), then the warp writes each
// segment with ONE LANE PER BIT (lane b stores the entry of bit b at prefix +
// popc(mask below b)): consecutive shared-memory addresses, no bank conflicts, and
// the instruction count is per segment, not per entry of the longest segment (a lane
// per segment walking its own bits ran max-popcount iterations at ~31 % lane use).
// The row goes back to HBM in 16-byte stores.  Rows longer than the stride are left
// alone (the host grows the stride and reruns the search before anything reads them).
constexpr int kExpWarps = 8;
template <typename E>
__global__ void __launch_bounds__(32 * kExpWarps) k_expand_rows(unsigned char* __restrict__ rows, int64_t n,
                                                              const uint32_t* __restrict__ nseg,
                                                              const uint32_t* __restrict__ ncount, int maxn) {
  extern __shared__ uint4 xsm[];
  const uint32_t lane = threadIdx.x & 31, lt = (1u << lane) - 1u;
  const int warp = threadIdx.x >> 5;
  const size_t rbytes = (size_t)maxn * sizeof(E);  // a multiple of 16 (stride rounded to 32 entries)
  const uint32_t segcap = (uint32_t)(rbytes / sizeof(uint2));
  uint4* const sseg = xsm + (size_t)warp * (segcap + rbytes / 16);  // (mask, base, prefix, -) per segment
  E* const sout = reinterpret_cast<E*>(sseg + segcap);
  const int nw = blockDim.x >> 5;  // kExpWarps, fewer for long rows (shared-memory budget)
  const int64_t stride = (int64_t)gridDim.x * nw;
  int64_t t = (int64_t)blockIdx.x * nw + warp;
  uint32_t ns = t < n ? nseg[t] : 0u, nc = t < n ? ncount[t] : 0u;
  for (; t < n; t += stride) {
    const uint32_t cns = ns, cnc = nc;
    if (t + stride < n) {  // the next row's counts land while this one is rewritten
      ns = nseg[t + stride];
      nc = ncount[t + stride];
    }
    if (cnc > (uint32_t)maxn || cns > segcap) continue;
    unsigned char* const row = rows + (size_t)t * rbytes;
    const uint2* const gseg = reinterpret_cast<const uint2*>(row);
    uint32_t carry = 0;
    for (uint32_t k0 = 0; k0 < cns; k0 += 32) {
      const uint32_t k = k0 + lane;
      const uint2 sg = k < cns ? gseg[k] : make_uint2(0u, 0u);
      const uint32_t pc = __popc(sg.x);
      uint32_t v = pc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= (uint32_t)o) v += u;
      }
      if (k < cns) sseg[k] = make_uint4(sg.x, sg.y, carry + v - pc, 0u);
      carry += __shfl_sync(0xffffffffu, v, 31);
    }
    __syncwarp();  // every segment was read: the row region may be overwritten
#pragma unroll 4
    for (uint32_t j = 0; j < cns; ++j) {
      const uint4 sg = sseg[j];  // broadcast
      if (sg.x & (1u << lane)) sout[sg.z + __popc(sg.x & lt)] = (E)(sg.y + lane);
    }
    __syncwarp();
    const uint32_t nv = (uint32_t)((cnc * sizeof(E) + 15) / 16);
    uint4* const dst = reinterpret_cast<uint4*>(row);
    const uint4* const src = reinterpret_cast<const uint4*>(sout);
    for (uint32_t k = lane; k < nv; k += 32) dst[k] = src[k];
    __syncwarp();
  }
}

static bool any_wrap2_s(const sph_ctx* c) {
  const Grid& g = c->grid;
  for (int d = 0; d < 3; ++d)
    if (g.periodic[d] && 2 * stencil_radius(g, d, reach_of(c->hmax)) + 1 >= g.nc[d]) return true;
  return false;
}

template <typename E>
static void search_t(sph_ctx* c, int gs, size_t smem, bool w2, bool sym) {
  auto kern = w2 ? (sym ? k_search<true, true, E> : k_search<true, false, E>)
                 : (sym ? k_search<false, true, E> : k_search<false, false, E>);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<gs, kCTS, smem, c->stream>>>(c->P.x, c->P.y, c->P.z, c->P.h, c->grid, c->s.cell_start,
                                      c->s.cell_end, c->s.unit_rec, c->s.nunit_list, c->s.work + 0,
                                      reinterpret_cast<E*>(c->s.nbr), c->s.ncount, c->s.nseg, c->maxn_cap,
                                      c->s.nbr_max);
}

template <typename E>
static bool expand_t(sph_ctx* c) {
  const size_t rbytes = (size_t)c->maxn_cap * sizeof(E);
  const size_t per_warp = rbytes / sizeof(uint2) * sizeof(uint4) + rbytes;
  const size_t budget = 200 * 1024;  // dynamic shared memory per block
  const int nw = (int)std::min<size_t>(kExpWarps, budget / per_warp);
  if (nw < 1) return false;  // a row stride beyond ~4,000 16-bit entries
  const size_t smem = (size_t)nw * per_warp;
  cudaFuncSetAttribute(k_expand_rows<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  // one wave of resident blocks (a grid-stride loop): num_sms x 8 left a partial second
  // wave when registers allow only 6 blocks per SM
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_expand_rows<E>, 32 * nw, smem) != cudaSuccess ||
      per_sm < 1) {
    cudaGetLastError();
    per_sm = 1;
  }
  const int64_t blocks = std::min<int64_t>((c->P.n + nw - 1) / nw, (int64_t)c->num_sms * per_sm);
  k_expand_rows<E><<<(int)std::max<int64_t>(blocks, 1), 32 * nw, smem, c->stream>>>(
      c->s.nbr, c->P.n, c->s.nseg, c->s.ncount, c->maxn_cap);
  return true;
}

// segments -> rows in place (after the capacity check of the search's maxima)
int launch_expand_rows(sph_ctx* c) {
  const bool ok = c->wide_rows ? expand_t<uint32_t>(c) : expand_t<uint16_t>(c);
  return ok ? 1 : -1;
}

// unit records (union stencils + target ranges) for the search and the three passes
int launch_unit_prep(sph_ctx* c) {
  const int64_t cells = c->grid.ncell < c->P.n ? c->grid.ncell : c->P.n;
  const int gprep = (int)std::min<int64_t>(std::max<int64_t>(cells, 1), (int64_t)c->num_sms * 8);
  if (c->s.unit_iflag)  // flags past the unit count must read 0 for the scan
    cudaMemsetAsync(c->s.unit_iflag, 0, sizeof(uint32_t) * c->P.n, c->stream);
  k_unit_prep<<<gprep, 128, 0, c->stream>>>(c->grid, c->s.cell_list, c->s.unit_list, c->s.nunit_list,
                                            c->s.cell_start, c->s.cell_end, c->s.cell_hmax, c->s.unit_rec,
                                            c->P.n, c->s.unit_iflag);
  return 1 + (c->s.unit_iflag ? launch_unit_order(c) : 0);
}

// the search proper into rows of the current type / stride (maxima[0]: largest count,
// maxima[1]: a unit stencil too large for 16-bit rows)
int launch_search(sph_ctx* c) {
  const bool sym = c->phys.sym != 0;
  const size_t smem = (kSearchCap + 32) * sizeof(float4) + (sym ? (kSearchCap + 32) * sizeof(float2) : 0);
  cudaMemsetAsync(c->s.work + 0, 0, sizeof(uint32_t), c->stream);
  cudaMemsetAsync(c->s.nbr_max, 0, 3 * sizeof(unsigned int), c->stream);
  const int64_t cells = c->grid.ncell < c->P.n ? c->grid.ncell : c->P.n;
  const int gs = (int)std::min<int64_t>(std::max<int64_t>(cells, 1), (int64_t)c->num_sms * 2);
  if (c->wide_rows) search_t<uint32_t>(c, gs, smem, any_wrap2_s(c), sym);
  else search_t<uint16_t>(c, gs, smem, any_wrap2_s(c), sym);
  return 1;
}

}  // namespace sphb
