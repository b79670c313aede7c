// cellpass.cu -- a5 neighbour search, a6 density + Omega + EOS, a8 IAD and
// a10-a11 momentum + energy + AV + dt, each as ONE CTA PER SEARCH CELL.
//
// Why: the per-target gathers of the warp-per-target kernels are latency bound
// (ncu, profiles/r1_ncu_v1_1m.md: long-scoreboard stalls, 16 warps/SM).  Here a
// CTA owns a cell of ~72 targets, stages the source particles of the cell's
// stencil into shared memory with coalesced loads (each cell is a contiguous
// range of the Morton order), and lets one warp per target walk the target's
// neighbour row with lanes striding over entries.  Every source particle is
// read from L2/HBM once per target CELL instead of once per pair.
//
// Neighbour rows hold packed entries (slot << 20 | local) -> the shared-memory
// index of a neighbour is slot_off[slot] + local: no search, no global gather.
//
// The search tests r^2 < (2 h_a)^2 first in fp32 on cell-relative coordinates
// with an error band derived below; candidates inside the band are decided by
// the exact fp64 test in the oracle's association, so lists stay bit-exact.
#include "stencil.cuh"

namespace sphb {

constexpr int kCT = 256;            // threads per CTA
constexpr int kNW = kCT / 32;       // warps per CTA
constexpr int kTgtMax = 256;        // targets per sub-block (per-target state in smem)
constexpr int kMaxUnits = 160;      // staged (slot, local range) pieces per group
constexpr int kSearchCap = 2048;    // staged candidates per group (float4 = 32 KB)
constexpr int kDensCap = 2048;      // staged particles per group, 4 fp64 fields (64 KB)
constexpr int kMomCap = 576;        // staged particles per group, 17 fp64 fields (78 KB)
constexpr int kMomFields = 17;

struct GroupSm {
  int nu, total, k, l;
  uint32_t pend;
  int u_slot[kMaxUnits];
  uint32_t u_g[kMaxUnits];
  int u_base[kMaxUnits];
  int u_len[kMaxUnits];
  int u_l0[kMaxUnits];
};

struct CellSm {
  uint32_t t_start[kKMax];
  uint32_t t_cnt[kKMax];
  int slot_off[kKMax];
  signed char t_sh[kKMax][3];
  GroupSm G;
  Stencil st;
  int c3[3];
  uint32_t sc, ec;
  int kself;
};

__device__ __forceinline__ double min_img(double d, int periodic, double L) {
  if (periodic) {
    if (d > 0.5 * L) d -= L;
    else if (d < -0.5 * L) d += L;
  }
  return d;
}

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

__device__ __forceinline__ double sinc_poly(const Phys& ph, double t) {
  double p = ph.poly[kPolyTerms - 1];
#pragma unroll
  for (int k = kPolyTerms - 2; k >= 0; --k) p = fma(p, t, ph.poly[k]);
  return p;
}
__device__ __forceinline__ double sinc_dpoly(const Phys& ph, double t) {
  double p = ph.dpoly[kPolyTerms - 2];
#pragma unroll
  for (int k = kPolyTerms - 3; k >= 0; --k) p = fma(p, t, ph.dpoly[k]);
  return p;
}
__device__ __forceinline__ double ipow(double s, int n) {  // "inline x*x*x..."
  if (n == 6) {
    double s2 = s * s;
    double s4 = s2 * s2;
    return s4 * s2;
  }
  double r = 1.0;
  for (int k = 0; k < n; ++k) r *= s;
  return r;
}

// CTA prologue for cell c: stencil + per-slot (start, count, shift) tables.
__device__ void cell_setup(const Grid& g, uint32_t c, const uint32_t* __restrict__ cstart,
                           const uint32_t* __restrict__ cend,
                           const unsigned long long* __restrict__ chmax, CellSm& S) {
  if (threadIdx.x == 0) {
    cell_coords(g, c, S.c3);
    S.sc = cstart[c];
    S.ec = cend[c];
    make_stencil(g, S.c3, reach_of(__longlong_as_double((long long)chmax[c])), S.st);
    S.kself = self_slot(S.st, S.c3);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < S.st.K; k += blockDim.x) {
    int sh[3];
    int64_t cell = slot_cell(g, S.st, k, sh);
    uint32_t s0 = cstart[cell];
    S.t_start[k] = s0;
    S.t_cnt[k] = cend[cell] - s0;
    S.t_sh[k][0] = (signed char)sh[0];
    S.t_sh[k][1] = (signed char)sh[1];
    S.t_sh[k][2] = (signed char)sh[2];
  }
  __syncthreads();
}

// thread 0: next group of staged pieces from the (k, l) cursor, at most `cap` particles
__device__ void build_group(CellSm& S, int cap) {
  GroupSm& G = S.G;
  int k = G.k, l = G.l, nu = 0, total = 0;
  const int K = S.st.K;
  while (k < K && nu < kMaxUnits && total < cap) {
    int cnt = (int)S.t_cnt[k];
    if (l >= cnt) {
      ++k;
      l = 0;
      continue;
    }
    int take = min(cnt - l, cap - total);
    G.u_slot[nu] = k;
    G.u_g[nu] = S.t_start[k] + l;
    G.u_base[nu] = total;
    G.u_len[nu] = take;
    G.u_l0[nu] = l;
    S.slot_off[k] = total - l;
    ++nu;
    total += take;
    l += take;
    if (l >= cnt) {
      ++k;
      l = 0;
    }
  }
  while (k < K && S.t_cnt[k] == 0) ++k;  // tighten the end marker
  G.nu = nu;
  G.total = total;
  G.k = k;
  G.l = l;
  G.pend = k >= K ? 0xffffffffu : (((uint32_t)k << kLocalBits) | (uint32_t)l);
}

// ------------------------------------------------------------------ a5 search
__global__ void __launch_bounds__(kCT) k_search(const double* __restrict__ x,
                                                const double* __restrict__ y,
                                                const double* __restrict__ z,
                                                const double* __restrict__ h, Grid g,
                                                const uint32_t* __restrict__ cstart,
                                                const uint32_t* __restrict__ cend,
                                                const unsigned long long* __restrict__ chmax,
                                                const uint32_t* __restrict__ clist,
                                                const uint32_t* __restrict__ nclist,
                                                uint32_t* __restrict__ nbr,
                                                uint32_t* __restrict__ ncount, int maxn,
                                                unsigned int* __restrict__ maxcount) {
  extern __shared__ float4 cand[];  // kSearchCap staged candidates
  __shared__ CellSm S;
  __shared__ uint32_t tcount[kTgtMax];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const uint32_t ncl = *nclist;
  for (uint32_t ci = blockIdx.x; ci < ncl; ci += gridDim.x) {
    cell_setup(g, clist[ci], cstart, cend, chmax, S);
    const Stencil st = S.st;
    double org[3], M = 0.0;
    for (int d = 0; d < 3; ++d) {
      double edge = g.inv[d] > 0.0 ? 1.0 / g.inv[d] : 0.0;
      org[d] = g.lo[d] + S.c3[d] * edge;
      // bound on |staged coordinate - org| (cells of the stencil +1 cell of slack)
      double Md = st.wrap[d] == 2 ? g.L[d]
                                  : (double)(max(S.c3[d] - st.lo[d], st.lo[d] + st.cnt[d] - S.c3[d]) + 1) * edge;
      M = fmax(M, Md);
    }
    const float L32[3] = {(float)g.L[0], (float)g.L[1], (float)g.L[2]};
    for (uint32_t t0 = S.sc; t0 < S.ec; t0 += kTgtMax) {
      const uint32_t t1 = min(S.ec, t0 + kTgtMax);
      for (uint32_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) tcount[t - t0] = 0;
      if (threadIdx.x == 0) {
        S.G.k = 0;
        S.G.l = 0;
      }
      __syncthreads();
      for (;;) {
        if (threadIdx.x == 0) build_group(S, kSearchCap);
        __syncthreads();
        const int nu = S.G.nu, total = S.G.total;
        if (nu == 0) break;
        for (int u = warp; u < nu; u += kNW) {
          const int slot = S.G.u_slot[u], base = S.G.u_base[u], len = S.G.u_len[u], l0 = S.G.u_l0[u];
          const uint32_t g0 = S.G.u_g[u];
          const double sx = S.t_sh[slot][0] * g.L[0], sy = S.t_sh[slot][1] * g.L[1],
                       sz = S.t_sh[slot][2] * g.L[2];
          for (int i = lane; i < len; i += 32) {
            const uint32_t j = g0 + i;
            float4 v;
            v.x = (float)((x[j] + sx) - org[0]);
            v.y = (float)((y[j] + sy) - org[1]);
            v.z = (float)((z[j] + sz) - org[2]);
            v.w = __uint_as_float(((uint32_t)slot << kLocalBits) | (uint32_t)(l0 + i));
            cand[base + i] = v;
          }
        }
        __syncthreads();
        for (uint32_t t = t0 + warp; t < t1; t += kNW) {
          const double xa = x[t], ya = y[t], za = z[t];
          const double tha = 2.0 * h[t];
          const double lim = __dmul_rn(tha, tha);
          // fp32 error band: |r2_32 - r2| <= delta * lim with
          // delta = 2^-20 (2 + 2 M/h + 2^-20 (M/h)^2), M >= |coordinates|.
          const double mh = M / h[t];
          const double delta = 0x1p-20 * (2.0 + 2.0 * mh + 0x1p-20 * mh * mh);
          float lo32 = -1.0f, hi32 = INFINITY;
          if (delta < 0.25) {
            lo32 = (float)(lim * (1.0 - delta));
            hi32 = (float)(lim * (1.0 + delta));
          }
          const float ax = (float)(xa - org[0]), ay = (float)(ya - org[1]), az = (float)(za - org[2]);
          const uint32_t self_pk = ((uint32_t)S.kself << kLocalBits) | (t - S.sc);
          uint32_t count = tcount[t - t0];
          uint32_t* row = nbr + (size_t)t * maxn;
          for (int q0 = 0; q0 < total; q0 += 32) {
            const int q = q0 + lane;
            bool hit = false;
            uint32_t pk = 0;
            if (q < total) {
              const float4 cd = cand[q];
              float dx = cd.x - ax, dy = cd.y - ay, dz = cd.z - az;
              if (st.wrap[0] == 2) dx = dx > 0.5f * L32[0] ? dx - L32[0] : (dx < -0.5f * L32[0] ? dx + L32[0] : dx);
              if (st.wrap[1] == 2) dy = dy > 0.5f * L32[1] ? dy - L32[1] : (dy < -0.5f * L32[1] ? dy + L32[1] : dy);
              if (st.wrap[2] == 2) dz = dz > 0.5f * L32[2] ? dz - L32[2] : (dz < -0.5f * L32[2] ? dz + L32[2] : dz);
              const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
              pk = __float_as_uint(cd.w);
              if (r2 < lo32) {
                hit = pk != self_pk;
              } else if (r2 < hi32) {  // inside the band: the exact fp64 test (oracle's association)
                const uint32_t j = S.t_start[pk >> kLocalBits] + (pk & kLocalMask);
                if (j != t) {
                  double ex = min_img(__dsub_rn(x[j], xa), g.periodic[0], g.L[0]);
                  double ey = min_img(__dsub_rn(y[j], ya), g.periodic[1], g.L[1]);
                  double ez = min_img(__dsub_rn(z[j], za), g.periodic[2], g.L[2]);
                  double r2e = __dadd_rn(__dadd_rn(__dmul_rn(ex, ex), __dmul_rn(ey, ey)), __dmul_rn(ez, ez));
                  hit = r2e < lim;
                }
              }
            }
            const unsigned b = __ballot_sync(0xffffffffu, hit);
            if (hit) {
              const uint32_t p = count + __popc(b & lt);
              if (p < (uint32_t)maxn) row[p] = pk;
            }
            count += __popc(b);
          }
          if (lane == 0) tcount[t - t0] = count;
        }
        __syncthreads();
      }
      for (uint32_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
        const uint32_t cn = tcount[t - t0];
        ncount[t] = cn;
        if (cn > (uint32_t)maxn) atomicMax(maxcount, cn);
      }
      __syncthreads();
    }
  }
}

// Walk target t's row from its cursor over the entries of the current group;
// calls body(smem index) for each entry owned by this lane.
template <class Body>
__device__ __forceinline__ uint32_t walk_group(const uint32_t* __restrict__ row, uint32_t cur,
                                               uint32_t n, uint32_t pend, const int* slot_off,
                                               Body&& body) {
  const int lane = threadIdx.x & 31;
  while (cur < n) {
    const uint32_t p = cur + lane;
    const uint32_t e = p < n ? row[p] : 0xffffffffu;
    const bool in = e < pend;
    const unsigned b = __ballot_sync(0xffffffffu, in);
    if (in) body(slot_off[e >> kLocalBits] + (int)(e & kLocalMask));
    const int m = __popc(b);
    cur += m;
    if (m < 32) break;
  }
  return cur;
}

// ------------------------------------------------------------------ a6 density + Omega + EOS
__global__ void __launch_bounds__(kCT) k_density_c(
    const double* __restrict__ x, const double* __restrict__ y, const double* __restrict__ z,
    const double* __restrict__ h, const double* __restrict__ m, const double* __restrict__ u,
    Grid g, const uint32_t* __restrict__ cstart, const uint32_t* __restrict__ cend,
    const unsigned long long* __restrict__ chmax, const uint32_t* __restrict__ clist,
    const uint32_t* __restrict__ nclist, const uint32_t* __restrict__ nbr,
    const uint32_t* __restrict__ ncount, int maxn, Phys ph, double* __restrict__ rho,
    double* __restrict__ omega, double* __restrict__ p, double* __restrict__ cs,
    double* __restrict__ wB, double* __restrict__ ih2, double* __restrict__ vol,
    double* __restrict__ rinv, double* __restrict__ X, double* __restrict__ mX,
    unsigned long long* __restrict__ cnt) {
  extern __shared__ double dsm[];
  double* sx = dsm;
  double* sy = sx + kDensCap;
  double* sz = sy + kDensCap;
  double* sm = sz + kDensCap;
  __shared__ CellSm S;
  __shared__ uint32_t cur[kTgtMax];
  __shared__ double acc[kTgtMax][2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t ncl = *nclist;
  for (uint32_t ci = blockIdx.x; ci < ncl; ci += gridDim.x) {
    cell_setup(g, clist[ci], cstart, cend, chmax, S);
    for (uint32_t t0 = S.sc; t0 < S.ec; t0 += kTgtMax) {
      const uint32_t t1 = min(S.ec, t0 + kTgtMax);
      for (uint32_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
        cur[t - t0] = 0;
        acc[t - t0][0] = 0.0;
        acc[t - t0][1] = 0.0;
      }
      if (threadIdx.x == 0) {
        S.G.k = 0;
        S.G.l = 0;
      }
      __syncthreads();
      for (;;) {
        if (threadIdx.x == 0) build_group(S, kDensCap);
        __syncthreads();
        const int nu = S.G.nu;
        if (nu == 0) break;
        for (int uu = warp; uu < nu; uu += kNW) {
          const int base = S.G.u_base[uu], len = S.G.u_len[uu];
          const uint32_t g0 = S.G.u_g[uu];
          for (int i = lane; i < len; i += 32) {
            sx[base + i] = x[g0 + i];
            sy[base + i] = y[g0 + i];
            sz[base + i] = z[g0 + i];
            sm[base + i] = m[g0 + i];
          }
        }
        __syncthreads();
        const uint32_t pend = S.G.pend;
        for (uint32_t t = t0 + warp; t < t1; t += kNW) {
          const double xa = x[t], ya = y[t], za = z[t];
          const double ih = 1.0 / h[t];
          const double ih2a = ih * ih;
          double sr = 0.0, sd = 0.0;
          const uint32_t c2 = walk_group(nbr + (size_t)t * maxn, cur[t - t0], ncount[t], pend, S.slot_off,
                                         [&](int q) {
            const double dx = min_img(sx[q] - xa, ph.periodic[0], ph.L[0]);
            const double dy = min_img(sy[q] - ya, ph.periodic[1], ph.L[1]);
            const double dz = min_img(sz[q] - za, ph.periodic[2], ph.L[2]);
            const double tt = (dx * dx + dy * dy + dz * dz) * ih2a;
            const double P = sinc_poly(ph, tt);
            const double Pn1 = ipow(P, ph.n - 1);
            const double dP = sinc_dpoly(ph, tt);
            const double mj = sm[q];
            sr += mj * (Pn1 * P);
            sd += mj * (Pn1 * (3.0 * P + 2.0 * ph.n * tt * dP));  // 3 S + v S'(v)
          });
          sr = wsum(sr);
          sd = wsum(sd);
          if (lane == 0) {
            cur[t - t0] = c2;
            acc[t - t0][0] += sr;
            acc[t - t0][1] += sd;
          }
        }
        __syncthreads();
      }
      for (uint32_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
        const double ha = h[t], ma = m[t];
        const double ih = 1.0 / ha;
        const double ih2a = ih * ih;
        const double wBa = ph.B * ih * ih2a;                         // B / h^3
        const double r = wBa * (ma + acc[t - t0][0]);                // Eq. 1 incl. self (R11)
        const double dsum = -wBa * ih * (3.0 * ma + acc[t - t0][1]);  // sum m dW/dh
        double om = ph.omega_mode ? 1.0 : 1.0 + ha / (3.0 * r) * dsum;  // R8
        if (om < 0.1) {
          om = 0.1;
          atomicAdd(&cnt[CNT_OMEGA], 1ull);
        }
        double P_, c_;
        if (ph.eos == SPH_EOS_LINEAR) {
          P_ = ph.c0 * ph.c0 * (r - ph.rho0);
          c_ = ph.c0;
        } else {
          P_ = (ph.gamma - 1.0) * r * u[t];
          c_ = sqrt(ph.gamma * P_ / r);
        }
        const double Xt = P_ / (om * r * r);  // R1
        rho[t] = r;
        omega[t] = om;
        p[t] = P_;
        cs[t] = c_;
        wB[t] = wBa;
        ih2[t] = ih2a;
        vol[t] = ma / r;
        rinv[t] = 1.0 / r;
        X[t] = Xt;
        mX[t] = ma * Xt;
      }
      __syncthreads();
    }
  }
}

// ------------------------------------------------------------------ a8 IAD
__global__ void __launch_bounds__(kCT) k_iad_c(
    const double* __restrict__ x, const double* __restrict__ y, const double* __restrict__ z,
    Grid g, const uint32_t* __restrict__ cstart, const uint32_t* __restrict__ cend,
    const unsigned long long* __restrict__ chmax, const uint32_t* __restrict__ clist,
    const uint32_t* __restrict__ nclist, const uint32_t* __restrict__ nbr,
    const uint32_t* __restrict__ ncount, int maxn, Phys ph, const double* __restrict__ wB,
    const double* __restrict__ ih2, const double* __restrict__ vol, double* __restrict__ c11,
    double* __restrict__ c12, double* __restrict__ c13, double* __restrict__ c22,
    double* __restrict__ c23, double* __restrict__ c33, double* __restrict__ ct,
    int64_t ct_stride, unsigned long long* __restrict__ cnt) {
  extern __shared__ double dsm[];
  double* sx = dsm;
  double* sy = sx + kDensCap;
  double* sz = sy + kDensCap;
  double* sv = sz + kDensCap;
  __shared__ CellSm S;
  __shared__ uint32_t cur[kTgtMax];
  __shared__ double acc[kTgtMax][6];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t ncl = *nclist;
  for (uint32_t ci = blockIdx.x; ci < ncl; ci += gridDim.x) {
    cell_setup(g, clist[ci], cstart, cend, chmax, S);
    for (uint32_t t0 = S.sc; t0 < S.ec; t0 += kTgtMax) {
      const uint32_t t1 = min(S.ec, t0 + kTgtMax);
      for (uint32_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
        cur[t - t0] = 0;
        for (int k = 0; k < 6; ++k) acc[t - t0][k] = 0.0;
      }
      if (threadIdx.x == 0) {
        S.G.k = 0;
        S.G.l = 0;
      }
      __syncthreads();
      for (;;) {
        if (threadIdx.x == 0) build_group(S, kDensCap);
        __syncthreads();
        const int nu = S.G.nu;
        if (nu == 0) break;
        for (int uu = warp; uu < nu; uu += kNW) {
          const int base = S.G.u_base[uu], len = S.G.u_len[uu];
          const uint32_t g0 = S.G.u_g[uu];
          for (int i = lane; i < len; i += 32) {
            sx[base + i] = x[g0 + i];
            sy[base + i] = y[g0 + i];
            sz[base + i] = z[g0 + i];
            sv[base + i] = vol[g0 + i];
          }
        }
        __syncthreads();
        const uint32_t pend = S.G.pend;
        for (uint32_t t = t0 + warp; t < t1; t += kNW) {
          const double xa = x[t], ya = y[t], za = z[t], ih2a = ih2[t];
          double t11 = 0, t12 = 0, t13 = 0, t22 = 0, t23 = 0, t33 = 0;
          const uint32_t c2 = walk_group(nbr + (size_t)t * maxn, cur[t - t0], ncount[t], pend, S.slot_off,
                                         [&](int q) {
            const double dx = min_img(sx[q] - xa, ph.periodic[0], ph.L[0]);
            const double dy = min_img(sy[q] - ya, ph.periodic[1], ph.L[1]);
            const double dz = min_img(sz[q] - za, ph.periodic[2], ph.L[2]);
            const double tt = (dx * dx + dy * dy + dz * dz) * ih2a;
            const double w = sv[q] * ipow(sinc_poly(ph, tt), ph.n);  // (m_b/rho_b) S
            const double wx = w * dx, wy = w * dy;
            t11 += wx * dx;
            t12 += wx * dy;
            t13 += wx * dz;
            t22 += wy * dy;
            t23 += wy * dz;
            t33 += w * dz * dz;
          });
          t11 = wsum(t11); t12 = wsum(t12); t13 = wsum(t13);
          t22 = wsum(t22); t23 = wsum(t23); t33 = wsum(t33);
          if (lane == 0) {
            cur[t - t0] = c2;
            acc[t - t0][0] += t11; acc[t - t0][1] += t12; acc[t - t0][2] += t13;
            acc[t - t0][3] += t22; acc[t - t0][4] += t23; acc[t - t0][5] += t33;
          }
        }
        __syncthreads();
      }
      for (uint32_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
        const double s = wB[t];
        const double* A = acc[t - t0];
        const double a11 = A[0] * s, a12 = A[1] * s, a13 = A[2] * s, a22 = A[3] * s,
                     a23 = A[4] * s, a33 = A[5] * s;
        const double det = a11 * (a22 * a33 - a23 * a23) - a12 * (a12 * a33 - a23 * a13) +
                           a13 * (a12 * a23 - a22 * a13);
        const double id = 1.0 / det;
        double i11 = (a22 * a33 - a23 * a23) * id;
        double i12 = (a13 * a23 - a12 * a33) * id;
        double i13 = (a12 * a23 - a13 * a22) * id;
        double i22 = (a11 * a33 - a13 * a13) * id;
        double i23 = (a12 * a13 - a11 * a23) * id;
        double i33 = (a11 * a22 - a12 * a12) * id;
        const double nt = sqrt(a11 * a11 + a22 * a22 + a33 * a33 + 2.0 * (a12 * a12 + a13 * a13 + a23 * a23));
        const double ni = sqrt(i11 * i11 + i22 * i22 + i33 * i33 + 2.0 * (i12 * i12 + i13 * i13 + i23 * i23));
        if (!(det > 0.0) || !(nt * ni <= 1e12)) {  // reading R29
          const double tr = a11 + a22 + a33;
          const double q = tr > 0.0 ? 3.0 / tr : 0.0;
          i11 = q; i22 = q; i33 = q;
          i12 = 0.0; i13 = 0.0; i23 = 0.0;
          atomicAdd(&cnt[CNT_IAD_SINGULAR], 1ull);
        }
        c11[t] = i11; c12[t] = i12; c13[t] = i13;
        c22[t] = i22; c23[t] = i23; c33[t] = i33;
        // C~ = (B/h^3) C, staged by the momentum pass (A_ab(h_b) = C~_b Delta S_b)
        ct[0 * ct_stride + t] = s * i11; ct[1 * ct_stride + t] = s * i12; ct[2 * ct_stride + t] = s * i13;
        ct[3 * ct_stride + t] = s * i22; ct[4 * ct_stride + t] = s * i23; ct[5 * ct_stride + t] = s * i33;
      }
      __syncthreads();
    }
  }
}

// ------------------------------------------------------------------ a10-a11 momentum + energy + AV + dt
struct MomSrc {  // per-particle arrays staged for the source side of a pair
  const double *x, *y, *z, *vx, *vy, *vz, *m, *ih2, *c, *mX, *mr;
  const double* ct;  // 6 x stride: C~ = (B/h^3) C
  int64_t ct_stride;
};
struct MomTgt {
  const double *h, *wB, *rinv, *X, *c11, *c12, *c13, *c22, *c23, *c33;
};
struct MomOut {
  double *ax, *ay, *az, *du, *vsig;
};

__global__ void __launch_bounds__(kCT, 2) k_momentum_c(
    MomSrc src, MomTgt tg, MomOut out, Grid g, const uint32_t* __restrict__ cstart,
    const uint32_t* __restrict__ cend, const unsigned long long* __restrict__ chmax,
    const uint32_t* __restrict__ clist, const uint32_t* __restrict__ nclist,
    const uint32_t* __restrict__ nbr, const uint32_t* __restrict__ ncount, int maxn, Phys ph,
    double* __restrict__ dts, unsigned long long* __restrict__ cnt) {
  extern __shared__ double dsm[];
  double* F[kMomFields];
#pragma unroll
  for (int k = 0; k < kMomFields; ++k) F[k] = dsm + k * kMomCap;
  __shared__ CellSm S;
  __shared__ uint32_t cur[kTgtMax];
  __shared__ double acc[kTgtMax][5];
  __shared__ double shdt[kNW];
  __shared__ unsigned long long shco;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t ncl = *nclist;
  double dtmin = INFINITY;
  unsigned long long ncoinc = 0;
  for (uint32_t ci = blockIdx.x; ci < ncl; ci += gridDim.x) {
    cell_setup(g, clist[ci], cstart, cend, chmax, S);
    for (uint32_t t0 = S.sc; t0 < S.ec; t0 += kTgtMax) {
      const uint32_t t1 = min(S.ec, t0 + kTgtMax);
      for (uint32_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
        cur[t - t0] = 0;
        acc[t - t0][0] = 0.0;
        acc[t - t0][1] = 0.0;
        acc[t - t0][2] = 0.0;
        acc[t - t0][3] = 0.0;
        acc[t - t0][4] = -1.0;
      }
      if (threadIdx.x == 0) {
        S.G.k = 0;
        S.G.l = 0;
      }
      __syncthreads();
      for (;;) {
        if (threadIdx.x == 0) build_group(S, kMomCap);
        __syncthreads();
        const int nu = S.G.nu;
        if (nu == 0) break;
        for (int uu = warp; uu < nu; uu += kNW) {
          const int base = S.G.u_base[uu], len = S.G.u_len[uu];
          const uint32_t g0 = S.G.u_g[uu];
          for (int i = lane; i < len; i += 32) {
            const uint32_t j = g0 + i;
            const int q = base + i;
            F[0][q] = src.x[j];
            F[1][q] = src.y[j];
            F[2][q] = src.z[j];
            F[3][q] = src.vx[j];
            F[4][q] = src.vy[j];
            F[5][q] = src.vz[j];
            F[6][q] = src.m[j];
            F[7][q] = src.ih2[j];
            F[8][q] = src.c[j];
            F[9][q] = src.mX[j];
            F[10][q] = src.mr[j];
#pragma unroll
            for (int k = 0; k < 6; ++k) F[11 + k][q] = src.ct[k * src.ct_stride + j];
          }
        }
        __syncthreads();
        const uint32_t pend = S.G.pend;
        for (uint32_t t = t0 + warp; t < t1; t += kNW) {
          const double xa = src.x[t], ya = src.y[t], za = src.z[t];
          const double vxa = src.vx[t], vya = src.vy[t], vza = src.vz[t];
          const double ih2a = src.ih2[t], wBa = tg.wB[t], rinva = tg.rinv[t], Xa = tg.X[t],
                       ca = src.c[t];
          const double a11 = tg.c11[t], a12 = tg.c12[t], a13 = tg.c13[t], a22 = tg.c22[t],
                       a23 = tg.c23[t], a33 = tg.c33[t];
          double fx = 0.0, fy = 0.0, fz = 0.0, fu = 0.0, vs = -1.0;
          const uint32_t c2 = walk_group(nbr + (size_t)t * maxn, cur[t - t0], ncount[t], pend, S.slot_off,
                                         [&](int q) {
            const double dx = min_img(F[0][q] - xa, ph.periodic[0], ph.L[0]);  // Delta_ab = x_b - x_a
            const double dy = min_img(F[1][q] - ya, ph.periodic[1], ph.L[1]);
            const double dz = min_img(F[2][q] - za, ph.periodic[2], ph.L[2]);
            const double r2 = dx * dx + dy * dy + dz * dz;
            if (r2 == 0.0) {  // coincident pair: skipped, counted
              ++ncoinc;
              return;
            }
            const double ta = r2 * ih2a;
            const double Sa = ipow(sinc_poly(ph, ta), ph.n);
            const double Wa = wBa * Sa;
            const double tb = r2 * F[7][q];
            double Sb = 0.0;  // b's support may not reach a (variable h)
            if (tb < 4.0) Sb = (tb == ta) ? Sa : ipow(sinc_poly(ph, tb), ph.n);
            // R5: A_ab(h_a) = C_a Delta W_ab(h_a);  R4: A_ab(h_b) = C~_b Delta S_b
            const double Aax = (a11 * dx + a12 * dy + a13 * dz) * Wa;
            const double Aay = (a12 * dx + a22 * dy + a23 * dz) * Wa;
            const double Aaz = (a13 * dx + a23 * dy + a33 * dz) * Wa;
            const double Abx = (F[11][q] * dx + F[12][q] * dy + F[13][q] * dz) * Sb;
            const double Aby = (F[12][q] * dx + F[14][q] * dy + F[15][q] * dz) * Sb;
            const double Abz = (F[13][q] * dx + F[15][q] * dy + F[16][q] * dz) * Sb;
            const double mb = F[6][q], mXb = F[9][q], mrb = F[10][q], cb = F[8][q];
            const double vabx = vxa - F[3][q], vaby = vya - F[4][q], vabz = vza - F[5][q];
            const double vdotx = -(vabx * dx + vaby * dy + vabz * dz);  // v_ab . x_ab
            double Pi = 0.0, w = 0.0;
            if (vdotx < 0.0) {  // Eq. 5
              w = vdotx * rsqrt(r2);
              Pi = -0.5 * ph.alpha * (ca + cb - 3.0 * w) * w;
            }
            vs = fmax(vs, ca + cb - 3.0 * w);  // v_sig
            // g = 1/2 m_b Pi' (A_a / rho_a + A_b / rho_b)   (Eq. 4 pair term)
            const double hp = 0.5 * Pi;
            const double mra = mb * rinva;
            const double gx = hp * (mra * Aax + mrb * Abx);
            const double gy = hp * (mra * Aay + mrb * Aby);
            const double gz = hp * (mra * Aaz + mrb * Abz);
            const double mXa = mb * Xa;
            fx += -(mXa * Aax + mXb * Abx) - gx;  // Eq. 2 with R2
            fy += -(mXa * Aay + mXb * Aby) - gy;
            fz += -(mXa * Aaz + mXb * Abz) - gz;
            fu += mXa * (vabx * Aax + vaby * Aay + vabz * Aaz) +
                  0.5 * (vabx * gx + vaby * gy + vabz * gz);  // Eq. 3 with R1, R3
          });
          fx = wsum(fx);
          fy = wsum(fy);
          fz = wsum(fz);
          fu = wsum(fu);
          vs = wmax(vs);
          if (lane == 0) {
            cur[t - t0] = c2;
            acc[t - t0][0] += fx;
            acc[t - t0][1] += fy;
            acc[t - t0][2] += fz;
            acc[t - t0][3] += fu;
            acc[t - t0][4] = fmax(acc[t - t0][4], vs);
          }
        }
        __syncthreads();
      }
      for (uint32_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
        double vsig = acc[t - t0][4];
        if (vsig < 0.0) vsig = 2.0 * src.c[t];  // no interacting neighbour
        out.ax[t] = acc[t - t0][0];
        out.ay[t] = acc[t - t0][1];
        out.az[t] = acc[t - t0][2];
        out.du[t] = acc[t - t0][3];
        out.vsig[t] = vsig;
        const double dta = ph.courant * tg.h[t] / vsig;  // R19
        if (!(dta > 0.0)) atomicAdd(&cnt[CNT_NONFINITE], 1ull);
        dtmin = fmin(dtmin, dta);
      }
      __syncthreads();
    }
  }
  // block min dt -> one atomicMin per block (positive doubles order like uint64)
  dtmin = wmax(-dtmin) * -1.0;
  if (threadIdx.x == 0) shco = 0;
  __syncthreads();
  if (ncoinc) atomicAdd(&shco, ncoinc);
  if (lane == 0) shdt[warp] = dtmin;
  __syncthreads();
  if (threadIdx.x == 0) {
    double mn = shdt[0];
    for (int q = 1; q < kNW; ++q) mn = fmin(mn, shdt[q]);
    if (mn > 0.0)
      atomicMin((unsigned long long*)&dts[DT_RAW_BITS], (unsigned long long)__double_as_longlong(mn));
    if (shco) atomicAdd(&cnt[CNT_COINCIDENT], shco);
  }
}

// ------------------------------------------------------------------ launchers
static int cell_grid(const sph_ctx* c, int per_sm) {
  int64_t cells = c->grid.ncell < c->P.n ? c->grid.ncell : c->P.n;
  int64_t mx = (int64_t)c->num_sms * per_sm;
  return (int)(cells < mx ? (cells > 0 ? cells : 1) : mx);
}

int launch_neighbors(sph_ctx* c) {
  static bool attr = false;
  const size_t smem = kSearchCap * sizeof(float4);
  if (!attr) {
    cudaFuncSetAttribute(k_search, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  k_search<<<cell_grid(c, 4), kCT, smem, c->stream>>>(
      c->P.x, c->P.y, c->P.z, c->P.h, c->grid, c->s.cell_start, c->s.cell_end, c->s.cell_hmax,
      c->s.cell_list, c->s.ncell_list, c->s.nbr, c->s.ncount, c->maxn, c->s.nbr_maxcount);
  return 1;
}

int launch_density(sph_ctx* c) {
  static bool attr = false;
  const size_t smem = 4 * kDensCap * sizeof(double);
  if (!attr) {
    cudaFuncSetAttribute(k_density_c, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  sph_particles& P = c->P;
  k_density_c<<<cell_grid(c, 2), kCT, smem, c->stream>>>(
      P.x, P.y, P.z, P.h, P.m, P.u, c->grid, c->s.cell_start, c->s.cell_end, c->s.cell_hmax,
      c->s.cell_list, c->s.ncell_list, c->s.nbr, c->s.ncount, c->maxn, c->phys, P.rho, P.omega,
      P.p, P.c, c->s.wB, c->s.ih2, c->s.vol, c->s.rinv, c->s.X, c->s.mX, c->s.cnt);
  return 1;
}

int launch_iad(sph_ctx* c) {
  static bool attr = false;
  const size_t smem = 4 * kDensCap * sizeof(double);
  if (!attr) {
    cudaFuncSetAttribute(k_iad_c, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  sph_particles& P = c->P;
  k_iad_c<<<cell_grid(c, 2), kCT, smem, c->stream>>>(
      P.x, P.y, P.z, c->grid, c->s.cell_start, c->s.cell_end, c->s.cell_hmax, c->s.cell_list,
      c->s.ncell_list, c->s.nbr, c->s.ncount, c->maxn, c->phys, c->s.wB, c->s.ih2, c->s.vol,
      P.c11, P.c12, P.c13, P.c22, P.c23, P.c33, c->s.ct, c->cap, c->s.cnt);
  return 1;
}

int launch_momentum(sph_ctx* c) {
  static bool attr = false;
  const size_t smem = (size_t)kMomFields * kMomCap * sizeof(double);
  if (!attr) {
    cudaFuncSetAttribute(k_momentum_c, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  sph_particles& P = c->P;
  MomSrc src = {P.x, P.y, P.z, P.vx, P.vy, P.vz, P.m, c->s.ih2, P.c, c->s.mX, c->s.vol, c->s.ct, c->cap};
  MomTgt tg = {P.h, c->s.wB, c->s.rinv, c->s.X, P.c11, P.c12, P.c13, P.c22, P.c23, P.c33};
  MomOut out = {P.ax, P.ay, P.az, P.du, P.vsig};
  k_momentum_c<<<cell_grid(c, 2), kCT, smem, c->stream>>>(
      src, tg, out, c->grid, c->s.cell_start, c->s.cell_end, c->s.cell_hmax, c->s.cell_list,
      c->s.ncell_list, c->s.nbr, c->s.ncount, c->maxn, c->phys, c->s.dts, c->s.cnt);
  return 1;
}

}  // namespace sphb
