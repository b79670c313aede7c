// cellpass.cu -- a6 density + Omega + EOS, a8 IAD and a10-a11 momentum + energy +
// AV + dt, each as ONE CTA PER PAIR-PASS UNIT (stencil.cuh; the search is in
// search.cu, shared helpers in pairpass.cuh).
//
// A CTA owns a unit of 2x2x1 search cells (~290 targets at the paper's 300
// neighbours), stages the source particles of the unit's union stencil into shared
// memory in groups -- coalesced loads (density, IAD) or TMA bulk copies of
// per-particle records (momentum); periodic images are shifted at staging time, so
// no pair needs a minimum image -- and a warp (density, IAD) or half-warp
// (momentum) per target walks the target's neighbour row, lanes striding over
// entries.  Row entries are flat staging indices of the unit stencil (16-bit unless
// a unit stencil exceeds 65,535 particles): the shared-memory index of a neighbour
// is entry - (group start), and "entry < group end" selects a target's segment of
// the group.  Row chunks are prefetched ahead, across target boundaries.
#include "pairpass.cuh"

namespace sphb {

__device__ __forceinline__ int qidx(const uint32_t* cum, uint32_t gb, uint32_t e) {
  (void)cum;
  return (int)(e - gb);  // row entries are flat staging indices of the unit stencil
}

__constant__ double c_poly[kPolyTerms];   // sinc(pi sqrt(t)/2) = sum c_poly[k] t^k
__constant__ double c_dpoly[kPolyTerms];  // derivative in t
__constant__ double c_dpoly4[kPolyTerms]; // 4 x the derivative (exact scaling; density at n = 6)

void set_poly_constants(const double* poly, const double* dpoly) {
  double d4[kPolyTerms];
  for (int k = 0; k < kPolyTerms; ++k) d4[k] = 4.0 * dpoly[k];
  cudaMemcpyToSymbol(c_poly, poly, sizeof(double) * kPolyTerms);
  cudaMemcpyToSymbol(c_dpoly, dpoly, sizeof(double) * kPolyTerms);
  cudaMemcpyToSymbol(c_dpoly4, d4, sizeof(double) * kPolyTerms);
}

__device__ __forceinline__ double sinc_poly(double t) {  // Horner
  double p = c_poly[kPolyTerms - 1];
#pragma unroll
  for (int k = kPolyTerms - 2; k >= 0; --k) p = fma(p, t, c_poly[k]);
  return p;
}
__device__ __forceinline__ double sinc_dpoly(double t) {
  double p = c_dpoly[kPolyTerms - 2];
#pragma unroll
  for (int k = kPolyTerms - 3; k >= 0; --k) p = fma(p, t, c_dpoly[k]);
  return p;
}
__device__ __forceinline__ double sinc_dpoly4(double t) {
  double p = c_dpoly4[kPolyTerms - 2];
#pragma unroll
  for (int k = kPolyTerms - 3; k >= 0; --k) p = fma(p, t, c_dpoly4[k]);
  return p;
}
// Even/odd split P(t) = E(t^2) + t O(t^2): two independent Horner chains of depth 4
// in u = t^2 (dependency depth 6 instead of 9) for the momentum pass, where four
// warps per SMSP cannot hide a single chain's DFMA latency (ncu "wait").  Every DFMA
// takes its coefficient as a constant operand, so no register holds a coefficient
// (an Estrin tree pairs two constants per DFMA and kept ten of them in registers).
__device__ __forceinline__ double sinc_poly_e(double t) {
  const double u = t * t;
  constexpr int te = (kPolyTerms - 1) & ~1, to = (kPolyTerms - 2) | 1;  // top even / odd index
  double e = c_poly[te], o = c_poly[to];
#pragma unroll
  for (int k = te - 2; k >= 0; k -= 2) e = fma(e, u, c_poly[k]);
#pragma unroll
  for (int k = to - 2; k >= 1; k -= 2) o = fma(o, u, c_poly[k]);
  return fma(o, t, e);
}
// "inline x*x*x*x..."; N > 0 fixes the exponent at compile time
template <int N>
__device__ __forceinline__ double ipow(double s, int n) {
  if constexpr (N == 6) {
    double s2 = s * s;
    double s4 = s2 * s2;
    return s4 * s2;
  } else if constexpr (N == 5) {
    double s2 = s * s;
    return s2 * s2 * s;
  } else if constexpr (N > 0) {
    double r = s;
#pragma unroll
    for (int k = 1; k < N; ++k) r *= s;
    return r;
  } else {
    double r = 1.0;
    for (int k = 0; k < n; ++k) r *= s;
    return r;
  }
}

// Kernel value S_n at t = v^2 = r^2/h^2 < 4 in the selected evaluation mode (sph.h
// SPH_KERNEL_*): the polynomial (Horner, or Estrin when EST), the paper's table
// (reading R12: floor index, linear interpolation in v), or sin(x)/x directly.
template <int KM, int N, bool EST>
__device__ __forceinline__ double kern_S(double t, int n, const double* __restrict__ tab, int K) {
  if constexpr (KM == SPH_KERNEL_TABLE) {
    const double q = sqrt(t) * (0.5 * (double)(K - 1));
    int i = (int)q;  // floor (q >= 0)
    i = i > K - 2 ? K - 2 : i;
    const double a = __ldg(tab + i), b = __ldg(tab + i + 1);
    return fma(b - a, q - (double)i, a);
  } else if constexpr (KM == SPH_KERNEL_SIN) {
    const double x = 1.5707963267948966 * sqrt(t);  // pi v / 2
    return ipow<N>(x > 0.0 ? sin(x) / x : 1.0, n);
  } else {
    return ipow<N>(EST ? sinc_poly_e(t) : sinc_poly(t), n);
  }
}

// Warp-level walk over the entries of target rows that fall in the current
// group [.., pend).  Targets are handed out dynamically (shared counter, reset by
// the group loop) so warps reach the group barrier together.  Row chunks (32
// entries) stream through a 3-deep register ring (ncu: with one chunk of
// prefetch the row load was the top stall), and the first three chunks of the
// warp's next target are issued before the current target's work.
template <typename E>
__device__ __forceinline__ uint32_t row_chunk(const E* row, uint32_t pos, uint32_t n) {
  return pos < n ? (uint32_t)row[pos] : kSent;
}

template <int NW, typename E, class Body, class Finish>
__device__ __forceinline__ void walk_targets(uint32_t t0, uint32_t t1, const E* __restrict__ nbr,
                                             int maxn, const uint32_t* s_n, uint32_t* s_cur,
                                             uint32_t pend, const uint32_t* cum, uint32_t gb,
                                             uint32_t* s_next, Body&& body, Finish&& finish) {
  const int lane = threadIdx.x & 31;
  uint32_t t = 0;
  if (lane == 0) t = t0 + atomicAdd(s_next, 1u);
  t = __shfl_sync(0xffffffffu, t, 0);
  uint32_t f0 = kSent, f1 = kSent, f2 = kSent;
  if (t < t1) {
    const uint32_t c0 = s_cur[t - t0] + lane, nn = s_n[t - t0];
    const E* r = nbr + (size_t)t * maxn;
    f0 = row_chunk(r, c0, nn);
    f1 = row_chunk(r, c0 + 32, nn);
    f2 = row_chunk(r, c0 + 64, nn);
  }
  while (t < t1) {
    const uint32_t i = t - t0;
    const uint32_t n = s_n[i];
    const E* row = nbr + (size_t)t * maxn;
    uint32_t cur = s_cur[i];
    uint32_t e0 = f0, e1 = f1, e2 = f2;
    // claim the next target and prefetch its first three chunks
    uint32_t tn = 0;
    if (lane == 0) tn = t0 + atomicAdd(s_next, 1u);
    tn = __shfl_sync(0xffffffffu, tn, 0);
    if (tn < t1) {
      const uint32_t cn = s_cur[tn - t0] + lane, nn = s_n[tn - t0];
      const E* r = nbr + (size_t)tn * maxn;
      f0 = row_chunk(r, cn, nn);
      f1 = row_chunk(r, cn + 32, nn);
      f2 = row_chunk(r, cn + 64, nn);
    }
    body.begin(i);
    for (;;) {
      const bool in = e0 < pend;
      const unsigned b = __ballot_sync(0xffffffffu, in);
      const int m = __popc(b);
      const uint32_t e3 = m == 32 ? row_chunk(row, cur + 96 + lane, n) : kSent;
      if (in) body(qidx(cum, gb, e0));
      cur += m;
      if (m < 32) break;
      e0 = e1;
      e1 = e2;
      e2 = e3;
    }
    finish(i, cur);
    t = tn;
  }
}

// Same walk with 16 lanes per target (two targets per warp, one per half-warp):
// the per-(target, group) setup and reduction is shared by two targets and the
// unused lanes at the end of a segment drop from up to 31 to up to 15.  Both
// halves step together; a half whose segment ended idles until the other is done.
// Row chunks stream through a 2-deep ring consumed in place (unrolled by two): a
// shifted ring (e0 = e1; e1 = e2 <- load) made every step wait for the load it had
// just issued (ncu: long_sb on the ring move), and a momentum step is long enough
// that two chunks of prefetch cover the load latency.
#ifndef SPH_MOM_RING
#define SPH_MOM_RING 2
#endif
constexpr int kMomRing = SPH_MOM_RING;  // row chunks in flight per half-warp (momentum)
template <typename E, class Body, class Finish>
__device__ __forceinline__ void walk_targets_half(uint32_t t0, uint32_t t1,
                                                  const E* __restrict__ nbr, int maxn,
                                                  const uint32_t* s_n, uint32_t* s_cur,
                                                  uint32_t pend, const uint32_t* cum, uint32_t gb,
                                                  uint32_t* s_next, Body&& body, Finish&& finish) {
  (void)cum;
  uint32_t par = 0;  // body.fetch / body.begin: double-buffered per-half prefetch slot
  const int lane = threadIdx.x & 31, l16 = lane & 15;
  const unsigned hmask = (threadIdx.x & 16) ? 0xffff0000u : 0x0000ffffu;
  auto claim = [&]() {
    uint32_t v = 0;
    if (l16 == 0) v = t0 + atomicAdd(s_next, 1u);
    return __shfl_sync(0xffffffffu, v, lane & 16);
  };
  uint32_t t = claim();
  uint32_t f0 = kSent, f1 = kSent, f2 = kSent;
  if (t < t1) {
    const uint32_t c0 = s_cur[t - t0] + l16, nn = s_n[t - t0];
    const E* r = nbr + (size_t)t * maxn;
    f0 = row_chunk(r, c0, nn);
    f1 = row_chunk(r, c0 + 16, nn);
    if constexpr (kMomRing > 2) f2 = row_chunk(r, c0 + 32, nn);
  }
  body.fetch(t, par, t < t1);
  while (__any_sync(0xffffffffu, t < t1)) {
    const bool act = t < t1;
    const uint32_t i = act ? t - t0 : 0;
    const uint32_t n = act ? s_n[i] : 0;
    uint32_t cur = act ? s_cur[i] : 0;
    uint32_t off = cur + l16 + 16 * kMomRing;  // row position of the next chunk to load (kMomRing ahead)
    const E* rp = nbr + (size_t)(act ? t : 0) * maxn + off;
    uint32_t e0 = f0, e1 = f1, e2 = f2;
    const uint32_t tn = claim();
    f0 = f1 = f2 = kSent;
    if (tn < t1) {
      const uint32_t cn = s_cur[tn - t0] + l16, nn = s_n[tn - t0];
      const E* r = nbr + (size_t)tn * maxn;
      f0 = row_chunk(r, cn, nn);
      f1 = row_chunk(r, cn + 16, nn);
      if constexpr (kMomRing > 2) f2 = row_chunk(r, cn + 32, nn);
    }
    body.fetch(tn, par ^ 1u, tn < t1);  // the next target's record lands while this one runs
    // (skipping a target with no entry in the group, as the full-warp walk does, hung
    // this walk on the GPU: not done here)
    const bool has = act;
    body.begin(par, has);  // every lane (the prefetch wait is a warp-wide barrier)
    par ^= 1u;
    bool live = has;
#define SPH_HALF_STEP(R)                                                       \
  {                                                                            \
    const uint32_t e = R;                                                      \
    const bool in = live && e < pend;                                          \
    const int m = __popc(__ballot_sync(0xffffffffu, in) & hmask);              \
    const bool more = live && m == 16;                                         \
    const int qi = (int)(e - gb);                                              \
    R = (more && off < n) ? (uint32_t)*rp : kSent;                                       \
    rp += 16;                                                                  \
    off += 16;                                                                 \
    if (in) body(qi);                                                          \
    cur += m;                                                                  \
    live = more;                                                               \
    if (!__any_sync(0xffffffffu, live)) break;                                 \
  }
    for (;;) {
      SPH_HALF_STEP(e0)
      SPH_HALF_STEP(e1)
      if constexpr (kMomRing > 2) SPH_HALF_STEP(e2)
    }
#undef SPH_HALF_STEP
    finish(has, i, cur);
    t = tn;
  }
}

// Lean full-warp walk (density, IAD): the ring of RING row chunks is consumed in
// place -- each step refills the register it just used with the chunk RING steps
// ahead (a shifted ring makes every move wait for the latest load) -- through a
// running row pointer, and the body runs on every lane with a validity flag instead
// of a divergent branch (ncu: per-step bookkeeping was as large as the pair math).
// RING row chunks in flight per warp (4: density -0.1 ms, IAD -0.2 to -0.5 ms vs 3,
// profiles/r2_ab14_*; IAD stays at its 64-register cap without spills)
#ifndef SPH_DENS_RING
#define SPH_DENS_RING 4
#endif
#ifndef SPH_IAD_RING
#define SPH_IAD_RING 4
#endif
template <int RING, typename E, class Body, class Finish>
__device__ __forceinline__ void walk_targets_fast(uint32_t t0, uint32_t t1,
                                                  const E* __restrict__ nbr, int maxn,
                                                  const uint32_t* s_n, const uint32_t* s_cur,
                                                  uint32_t pend, const uint32_t* cum, uint32_t gb,
                                                  uint32_t* s_next, Body&& body, Finish&& finish) {
  const uint32_t lane = threadIdx.x & 31;
  auto claim = [&]() {
    uint32_t v = 0;
    if (lane == 0) v = t0 + atomicAdd(s_next, 1u);
    return __shfl_sync(0xffffffffu, v, 0);
  };
  uint32_t t = claim();
  uint32_t f0 = kSent, f1 = kSent, f2 = kSent, f3 = kSent;
  if (t < t1) {
    const uint32_t c0 = s_cur[t - t0] + lane, nn = s_n[t - t0];
    const E* r = nbr + (size_t)t * maxn;
    f0 = row_chunk(r, c0, nn);
    f1 = row_chunk(r, c0 + 32, nn);
    f2 = row_chunk(r, c0 + 64, nn);
    if constexpr (RING > 3) f3 = row_chunk(r, c0 + 96, nn);
  }
  while (t < t1) {
    const uint32_t i = t - t0, n = s_n[i];
    uint32_t cur = s_cur[i];
    const uint32_t lim = n - cur;  // valid positions: offset < lim from cur
    const E* rp = nbr + (size_t)t * maxn + cur + lane + 32 * RING;
    uint32_t off = lane + 32 * RING;
    uint32_t e0 = f0, e1 = f1, e2 = f2, e3 = f3;
    const uint32_t tn = claim();
    if (tn < t1) {  // the next target's first RING chunks
      const uint32_t cn = s_cur[tn - t0] + lane, nn = s_n[tn - t0];
      const E* r = nbr + (size_t)tn * maxn;
      f0 = row_chunk(r, cn, nn);
      f1 = row_chunk(r, cn + 32, nn);
      f2 = row_chunk(r, cn + 64, nn);
      if constexpr (RING > 3) f3 = row_chunk(r, cn + 96, nn);
    }
    // no entry of this target in the group (rows ascend: its first entry is past it):
    // nothing to add, skip the set-up and the reduction (variable h: most visits of a
    // small-h target in a big unit stencil are empty)
    if (__shfl_sync(0xffffffffu, e0, 0) >= pend) {
      t = tn;
      continue;
    }
    body.begin(i);
#define SPH_FAST_STEP(R)                                                             \
  {                                                                                  \
    const uint32_t e = R;                                                            \
    const bool in = e < pend;                                                        \
    const int m = __popc(__ballot_sync(0xffffffffu, in));                            \
    const int qi = in ? (int)(e - gb) : 0; /* e dies here: the refill can reuse R */ \
    R = (m == 32 && off < lim) ? (uint32_t)*rp : kSent;                                        \
    rp += 32;                                                                        \
    off += 32;                                                                       \
    body(qi, in);                                                                    \
    cur += m;                                                                        \
    if (m < 32) break;                                                               \
  }
    for (;;) {
      SPH_FAST_STEP(e0)
      SPH_FAST_STEP(e1)
      SPH_FAST_STEP(e2)
      if constexpr (RING > 3) SPH_FAST_STEP(e3)
    }
#undef SPH_FAST_STEP
    finish(i, cur);
    t = tn;
  }
}

// stage (x, y) and (z, f) of the current group as double2 pairs: one 16-byte LDS
// per pair of fields, bank conflicts only within 8-lane quarters (ncu: the
// 8-byte SoA layout cost ~3x the ideal shared-memory wavefronts)
__device__ __forceinline__ void stage2x2(const Grid& g, const CellSm& S, uint32_t gb, uint32_t ge,
                                         const double* __restrict__ x, const double* __restrict__ y,
                                         const double* __restrict__ z, const double* __restrict__ f,
                                         double2* s01, double2* s23) {
  for (uint32_t q = threadIdx.x; q < ge - gb; q += blockDim.x) {  // flat: every thread equal work
    const uint32_t fi = gb + q;
    const int k = slot_of(S, fi);
    const uint32_t j = S.t_start[k] + (fi - S.cum[k]);
    double sh[3];
    shifts_of(g, S, k, sh);
    s01[q] = make_double2(x[j] + sh[0], y[j] + sh[1]);
    s23[q] = make_double2(z[j] + sh[2], f[j]);
  }
}

// The pass kernels' W2 flag selects the GENERAL variant, which checks the rare cases at
// run time: periodic dims whose stencil spans every cell (per-pair minimum image) and
// the symmetric neighbour relation (extra pairs with W(r, h_a) = 0).  The default
// variant (W2 = false) carries neither test in its pair loop.
//
// minimum image only for periodic dims where the stencil spans every cell
template <bool W2>
__device__ __forceinline__ void delta3(const Stencil& st, const Grid& g, double& dx, double& dy,
                                       double& dz) {
  if constexpr (W2) {
    if (st.wrap[0] == 2) dx = min_img(dx, g.L[0]);
    if (st.wrap[1] == 2) dy = min_img(dy, g.L[1]);
    if (st.wrap[2] == 2) dz = min_img(dz, g.L[2]);
  }
}

// ------------------------------------------------------------------ a6 density + Omega + EOS
// n = 6 with the polynomial: the grad-h summand 3 S + v S'(v) = 3 P^5 (P + 4 t P') is
// accumulated divided by 3 (one FMA on 4 P', whose coefficients are exact multiples)
template <int KM, int N>
__host__ __device__ constexpr bool fold3() { return KM == SPH_KERNEL_POLY && N == 6; }
struct DensBody {
  const double2 *s01, *s23;
  const double *tx, *ty, *tz, *tih2;
  const Stencil* st;
  const Grid* g;
  double xa, ya, za, ih2a, sr, sd;
  __device__ __forceinline__ void begin(uint32_t i) {
    xa = tx[i];
    ya = ty[i];
    za = tz[i];
    ih2a = tih2[i];
    sr = 0.0;
    sd = 0.0;
  }
};

template <int N, bool W2, int KM, typename E>
__global__ void __launch_bounds__(kCTD, 1) k_density_c(
    const double* __restrict__ x, const double* __restrict__ y, const double* __restrict__ z,
    const double* __restrict__ h, const double* __restrict__ m, const double* __restrict__ u,
    Grid g, const uint32_t* __restrict__ cstart, const uint32_t* __restrict__ cend,
    const unsigned long long* __restrict__ chmax, const uint32_t* __restrict__ clist,
    const uint32_t* __restrict__ nclist, const int4* __restrict__ urec, URange ur, uint32_t* __restrict__ work, const E* __restrict__ nbr,
    const uint32_t* __restrict__ ncount, int maxn, Phys ph, double* __restrict__ rho,
    double* __restrict__ omega, double* __restrict__ p, double* __restrict__ cs,
    double* __restrict__ wB, double* __restrict__ ih2, double* __restrict__ vol,
    double* __restrict__ rinv, double* __restrict__ X, double* __restrict__ mX,
    unsigned long long* __restrict__ cnt) {
  extern __shared__ double dsm[];
  double2* s01 = reinterpret_cast<double2*>(dsm);
  double2* s23 = s01 + kDensCap;
  __shared__ CellSm S;
  __shared__ uint32_t s_n[kTgtU], s_cur[kTgtU];
  __shared__ double tx[kTgtU], ty[kTgtU], tz[kTgtU], tih2[kTgtU], acc0[kTgtU], acc1[kTgtU];
  const int lane = threadIdx.x & 31;
  __shared__ uint32_t s_chunk;
  const int n = N > 0 ? N : ph.n;
  // cells in chunks of kCellChunk consecutive (Morton-order) cells claimed from a
  // counter: consecutive cells share most of their stencil, so a CTA's next staging
  // finds its sources in L2 (a grid stride left the re-reads to HBM)
  const uint32_t ulo = ur.lo ? *ur.lo : 0u, nun = *ur.hi;
  const uint32_t uchunk = (uint32_t)kCellChunk >> g.ubits ? (uint32_t)kCellChunk >> g.ubits : 1u;
  ChunkClaim claim{work, uchunk, 0u};
  for (uint32_t cfirst = ulo + claim.first(&s_chunk); cfirst < nun; cfirst = ulo + claim.next(&s_chunk)) {
    for (uint32_t ck = cfirst; ck < min(nun, cfirst + uchunk); ++ck) {
      unit_setup(g, ur.order ? ur.order[ck] : ck, urec, cstart, cend, S);
      const Stencil st = S.st;
      for (uint32_t t0 = S.sc; t0 < S.ec; t0 += kTgtU) {
        const uint32_t t1 = min(S.ec, t0 + kTgtU);
        for (uint32_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
          const uint32_t i = t - t0;
          s_n[i] = ncount[t];
          s_cur[i] = 0;
          tx[i] = x[t];
          ty[i] = y[t];
          tz[i] = z[t];
          const double ih = 1.0 / h[t];
          tih2[i] = ih * ih;
          acc0[i] = 0.0;
          acc1[i] = 0.0;
        }
        if (threadIdx.x == 0) S.next[0] = 0;
        __syncthreads();
        for (uint32_t gb = 0, gi = 0; gb < S.total; gb += kDensCap, ++gi) {
          const uint32_t ge = min(S.total, gb + kDensCap), pend = ge;
          if (threadIdx.x == 0) S.next[(gi + 1) & 1] = 0;
          stage2x2(g, S, gb, ge, x, y, z, m, s01, s23);
          __syncthreads();
          struct B : DensBody {
            int n, K, sym;
            const double* tab;
            // ok == false: padding lane of the walk; its terms are discarded by selects
            // (not multiplied by 0: a far padding pair may overflow the polynomial)
            __device__ __forceinline__ void operator()(int q, bool ok) {
              const double2 p01 = s01[q], p23 = s23[q];
              double dx = p01.x - xa, dy = p01.y - ya, dz = p23.x - za;
              delta3<W2>(*st, *g, dx, dy, dz);
              const double tt = (dx * dx + dy * dy + dz * dz) * ih2a;
              if (W2 && sym) ok = ok && tt < 4.0;  // symmetric extra pair: W(r, h_a) = 0
              const double P = sinc_poly(tt);
              const double Pn1 = ipow<N - 1 < 0 ? 0 : N - 1>(P, n - 1);
              const double mj = p23.y;
              double a, b;
              if constexpr (fold3<KM, N>()) {  // b / 3 = P^5 (P + 4 t P'): 2n = 12 = 3 x 4, 4 P' exact
                a = Pn1 * P;
                b = Pn1 * fma(tt, sinc_dpoly4(tt), P);
              } else if constexpr (KM == SPH_KERNEL_POLY) {
                const double dP = sinc_dpoly(tt);
                a = Pn1 * P;
                b = Pn1 * (3.0 * P + (2.0 * n) * tt * dP);  // 3 S + v S'(v)
              } else {  // S from the selected mode; v S'(v) from the exact polynomial (R12)
                const double dP = sinc_dpoly(tt);
                const double S_ = kern_S<KM, N, false>(tt, n, tab, K);
                a = S_;
                b = fma(3.0, S_, Pn1 * (2.0 * n) * tt * dP);
              }
              sr = fma(mj, ok ? a : 0.0, sr);
              sd = fma(mj, ok ? b : 0.0, sd);
            }
          } body;
          body.s01 = s01; body.s23 = s23;
          body.tx = tx; body.ty = ty; body.tz = tz; body.tih2 = tih2;
          body.st = &st; body.g = &g; body.n = n; body.K = ph.tableK; body.tab = ph.table;
          body.sym = ph.sym;
          walk_targets_fast<SPH_DENS_RING>(t0, t1, nbr, maxn, s_n, s_cur, pend, S.cum, gb, &S.next[gi & 1], body,
                            [&](uint32_t i, uint32_t c2) {
                              double v[2] = {body.sr, body.sd};
                              warp_multi_sum<2>(v);
                              if (lane == 0) {
                                s_cur[i] = c2;
                                acc0[i] += v[0];
                              }
                              if (lane == 16) acc1[i] += v[0];
                            });
          __syncthreads();
        }
        for (uint32_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
          const uint32_t i = t - t0;
          const double ha = h[t], ma = m[t];
          const double ih = 1.0 / ha;
          const double ih2a = ih * ih;
          const double wBa = ph.B * ih * ih2a;               // B / h^3
          const double r = wBa * (ma + acc0[i]);             // Eq. 1 incl. self (R11)
          // sum m dW/dh (acc1 holds sum m (3 S + v S') / 3 when fold3)
          const double dsum = fold3<KM, N>() ? -wBa * ih * (3.0 * (ma + acc1[i])) : -wBa * ih * (3.0 * ma + acc1[i]);
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
}

struct MomSrc {  // per-particle arrays staged for the source side of a pair
  const double *x, *y, *z, *vx, *vy, *vz, *m, *ih2, *c, *mX, *mr;
  const double* ct;  // 6 x stride: C~ = (B/h^3) C
  int64_t ct_stride;
};
constexpr int kMomPairs = 9;  // 144-byte momentum source record: 9 double2 (layout below)
// The IAD epilogue writes the records of its targets (owned particles) straight from
// the values it has just computed (C~) or staged (x, 1/h^2): the separate record pass
// then covers halos only.  Build with -DSPH_SEPARATE_RECORDS for the A/B baseline.
#ifdef SPH_SEPARATE_RECORDS
constexpr bool kIadRecords = false;
#else
constexpr bool kIadRecords = true;
#endif

// ------------------------------------------------------------------ a8 IAD
template <int N, bool W2, int KM, typename E>
__global__ void __launch_bounds__(kCTD, 1) k_iad_c(
    const double* __restrict__ x, const double* __restrict__ y, const double* __restrict__ z,
    Grid g, const uint32_t* __restrict__ cstart, const uint32_t* __restrict__ cend,
    const unsigned long long* __restrict__ chmax, const uint32_t* __restrict__ clist,
    const uint32_t* __restrict__ nclist, const int4* __restrict__ urec, URange ur, uint32_t* __restrict__ work, const E* __restrict__ nbr,
    const uint32_t* __restrict__ ncount, int maxn, Phys ph, const double* __restrict__ wB,
    const double* __restrict__ ih2, const double* __restrict__ vol, double* __restrict__ c11,
    double* __restrict__ c12, double* __restrict__ c13, double* __restrict__ c22,
    double* __restrict__ c23, double* __restrict__ c33, double* __restrict__ ct,
    int64_t ct_stride, unsigned long long* __restrict__ cnt, MomSrc rs, double2* __restrict__ mrec) {
  extern __shared__ double dsm[];
  double2* s01 = reinterpret_cast<double2*>(dsm);
  double2* s23 = s01 + kIadCap;
  __shared__ CellSm S;
  __shared__ uint32_t s_n[kTgtU], s_cur[kTgtU];
  __shared__ double tx[kTgtU], ty[kTgtU], tz[kTgtU], tih2[kTgtU];
  __shared__ double acc[6][kTgtU];
  const int lane = threadIdx.x & 31;
  __shared__ uint32_t s_chunk;
  const int n = N > 0 ? N : ph.n;
  // cells in chunks of kCellChunk consecutive (Morton-order) cells claimed from a
  // counter: consecutive cells share most of their stencil, so a CTA's next staging
  // finds its sources in L2 (a grid stride left the re-reads to HBM)
  const uint32_t ulo = ur.lo ? *ur.lo : 0u, nun = *ur.hi;
  const uint32_t uchunk = (uint32_t)kCellChunk >> g.ubits ? (uint32_t)kCellChunk >> g.ubits : 1u;
  ChunkClaim claim{work, uchunk, 0u};
  for (uint32_t cfirst = ulo + claim.first(&s_chunk); cfirst < nun; cfirst = ulo + claim.next(&s_chunk)) {
    for (uint32_t ck = cfirst; ck < min(nun, cfirst + uchunk); ++ck) {
      unit_setup(g, ur.order ? ur.order[ck] : ck, urec, cstart, cend, S);
      const Stencil st = S.st;
      for (uint32_t t0 = S.sc; t0 < S.ec; t0 += kTgtU) {
        const uint32_t t1 = min(S.ec, t0 + kTgtU);
        for (uint32_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
          const uint32_t i = t - t0;
          s_n[i] = ncount[t];
          s_cur[i] = 0;
          tx[i] = x[t];
          ty[i] = y[t];
          tz[i] = z[t];
          tih2[i] = ih2[t];
          for (int k = 0; k < 6; ++k) acc[k][i] = 0.0;
        }
        if (threadIdx.x == 0) S.next[0] = 0;
        __syncthreads();
        for (uint32_t gb = 0, gi = 0; gb < S.total; gb += kIadCap, ++gi) {
          const uint32_t ge = min(S.total, gb + kIadCap), pend = ge;
          if (threadIdx.x == 0) S.next[(gi + 1) & 1] = 0;
          stage2x2(g, S, gb, ge, x, y, z, vol, s01, s23);
          __syncthreads();
          struct B {
            const double2 *s01, *s23;
            const double *tx, *ty, *tz, *tih2;
            const Stencil* st;
            const Grid* g;
            int n, K, sym;
            const double* tab;
            double xa, ya, za, ih2a, t11, t12, t13, t22, t23, t33;
            __device__ __forceinline__ void begin(uint32_t i) {
              xa = tx[i];
              ya = ty[i];
              za = tz[i];
              ih2a = tih2[i];
              t11 = t12 = t13 = t22 = t23 = t33 = 0.0;
            }
            __device__ __forceinline__ void operator()(int q, bool ok) {  // ok: see density
              const double2 p01 = s01[q], p23 = s23[q];
              double dx = p01.x - xa, dy = p01.y - ya, dz = p23.x - za;
              delta3<W2>(*st, *g, dx, dy, dz);
              const double tt = (dx * dx + dy * dy + dz * dz) * ih2a;
              if (W2 && sym) ok = ok && tt < 4.0;  // symmetric extra pair: W(r, h_a) = 0
              const double S_ = kern_S<KM, N, false>(tt, n, tab, K);
              const double w = p23.y * (ok ? S_ : 0.0);  // (m_b/rho_b) S
              const double wx = w * dx, wy = w * dy;
              t11 = fma(wx, dx, t11);
              t12 = fma(wx, dy, t12);
              t13 = fma(wx, dz, t13);
              t22 = fma(wy, dy, t22);
              t23 = fma(wy, dz, t23);
              t33 = fma(w * dz, dz, t33);
            }
          } body;
          body.s01 = s01; body.s23 = s23;
          body.tx = tx; body.ty = ty; body.tz = tz; body.tih2 = tih2;
          body.st = &st; body.g = &g; body.n = n; body.K = ph.tableK; body.tab = ph.table;
          body.sym = ph.sym;
          walk_targets_fast<SPH_IAD_RING>(t0, t1, nbr, maxn, s_n, s_cur, pend, S.cum, gb, &S.next[gi & 1], body,
                            [&](uint32_t i, uint32_t c2) {
                              double v[8] = {body.t11, body.t12, body.t13, body.t22,
                                             body.t23, body.t33, 0.0, 0.0};
                              warp_multi_sum<8>(v);
                              if ((lane & 3) == 0 && lane < 24) acc[lane >> 2][i] += v[0];
                              if (lane == 0) s_cur[i] = c2;
                            });
          __syncthreads();
        }
        for (uint32_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
          const uint32_t i = t - t0;
          const double s = wB[t];
          // the record's per-particle fields, loaded first: their latency overlaps the
          // inverse below (the ct stores would otherwise order them after it)
          double rvx = 0.0, rvy = 0.0, rvz = 0.0, rm = 1.0, rc = 0.0, rmX = 0.0, rmr = 0.0;
          if (mrec) {
            rvx = rs.vx[t]; rvy = rs.vy[t]; rvz = rs.vz[t]; rm = rs.m[t];
            rc = rs.c[t]; rmX = rs.mX[t]; rmr = rs.mr[t];
          }
          const double a11 = acc[0][i] * s, a12 = acc[1][i] * s, a13 = acc[2][i] * s,
                       a22 = acc[3][i] * s, a23 = acc[4][i] * s, a33 = acc[5][i] * s;
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
          if (mrec) {  // the target's momentum source record (k_mom_records' layout), staged
            double2* r = s01 + (size_t)i * kMomPairs;  // staging buffer is free after the groups
            r[0] = make_double2(tx[i], ty[i]);
            r[1] = make_double2(tz[i], rvx);
            r[2] = make_double2(rvy, rvz);
            r[3] = make_double2(rm, tih2[i]);
            r[4] = make_double2(rc, rmX);
            r[5] = make_double2(rmr, s * i11);
            r[6] = make_double2(s * i12, s * i13);
            r[7] = make_double2(s * i22, s * i23);
            r[8] = make_double2(s * i33, 1.0 / rm);
          }
        }
        if (mrec) {  // the sub-block's records leave in coalesced 16-byte stores
          __syncthreads();
          const uint32_t nr = (t1 - t0) * kMomPairs;
          double2* const out = mrec + (size_t)t0 * kMomPairs;
          for (uint32_t e = threadIdx.x; e < nr; e += blockDim.x) out[e] = s01[e];
        }
        __syncthreads();
      }
      }
  }
}

// ------------------------------------------------------------------ a10-a11 momentum + energy + AV + dt
// ---- TMA bulk copies (cp.async.bulk) completing on an mbarrier (sm_90+; SASS UBLKCP)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(
                   smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t ok = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok)
                 : "r"(smem_u32(bar)), "r"(phase)
                 : "memory");
  } while (!ok);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
// cp.async (LDGSTS): 16 bytes global -> shared, L2 only (.cg), grouped per thread
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_prev() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

struct MomTgt {
  const double *h, *wB, *rinv, *X, *c11, *c12, *c13, *c22, *c23, *c33;
};
struct MomOut {
  double *ax, *ay, *az, *du, *vsig;
};
// staged field slots (SoA, kMomCap doubles each)
// staged source fields as double2 pairs (one 144-byte record per particle):
//   0 (x, y)  1 (z, vx)  2 (vy, vz)  3 (m, 1/h^2)  4 (c, m X)  5 (m/rho, C~11)
//   6 (C~12, C~13)  7 (C~22, C~23)  8 (C~33, 1/m)
// The TARGET side of a pair reads the target's own record too: X_a = (m X) (1/m),
// 1/rho_a = (m/rho) (1/m), and A_ab(h_a) = C_a Delta W(r, h_a) = C~_a Delta S(r/h_a)
// (C~ = (B/h^3) C), so no per-target table is staged.  (kMomPairs = 9 is defined
// above the IAD kernel, whose epilogue writes the owned particles' records.)

// Momentum source records: the kMomPairs double2 a pair reads from its source, one
// contiguous 144-byte record per particle, built once per step by the IAD epilogue
// (owned) and k_mom_records (halo).  A staging group is then a handful of bulk copies (one per stencil slot).
constexpr int kRecThreads = 256;  // k_mom_records block: records transposed through smem
__global__ void __launch_bounds__(kRecThreads) k_mom_records(MomSrc src, int64_t i0, int64_t n,
                                                              double2* __restrict__ rec) {
  // each thread assembles one record in shared memory, then the block writes its
  // kRecThreads consecutive records as one contiguous, fully coalesced range
  // (per-thread 144-byte-strided stores wrote each L2 sector piecemeal: 3.0 ms at 25M)
  __shared__ double2 buf[kRecThreads * kMomPairs];
  for (int64_t b0 = (int64_t)blockIdx.x * kRecThreads; b0 < n; b0 += (int64_t)gridDim.x * kRecThreads) {
    const int64_t j = i0 + b0 + threadIdx.x;  // records [i0, i0 + n)
    if (b0 + threadIdx.x < n) {
      const int64_t cs = src.ct_stride;
      double2* r = buf + threadIdx.x * kMomPairs;
      r[0] = make_double2(src.x[j], src.y[j]);
      r[1] = make_double2(src.z[j], src.vx[j]);
      r[2] = make_double2(src.vy[j], src.vz[j]);
      r[3] = make_double2(src.m[j], src.ih2[j]);
      r[4] = make_double2(src.c[j], src.mX[j]);
      r[5] = make_double2(src.mr[j], src.ct[j]);
      r[6] = make_double2(src.ct[cs + j], src.ct[2 * cs + j]);
      r[7] = make_double2(src.ct[3 * cs + j], src.ct[4 * cs + j]);
      r[8] = make_double2(src.ct[5 * cs + j], 1.0 / src.m[j]);  // 1/m: the target side derives X, 1/rho
    }
    __syncthreads();
    const int64_t cnt = min((int64_t)kRecThreads, n - b0) * kMomPairs;
    double2* out = rec + (i0 + b0) * kMomPairs;
    for (int64_t e = threadIdx.x; e < cnt; e += kRecThreads) out[e] = buf[e];
    __syncthreads();
  }
}

template <int N, bool W2, int KM, typename E>
__global__ void __launch_bounds__(kCTM, 1) k_momentum_c(
    MomSrc src, MomTgt tg, MomOut out, Grid g, const uint32_t* __restrict__ cstart,
    const uint32_t* __restrict__ cend, const unsigned long long* __restrict__ chmax,
    const uint32_t* __restrict__ clist, const uint32_t* __restrict__ nclist,
    const int4* __restrict__ urec, URange ur, uint32_t* __restrict__ work,
    const E* __restrict__ nbr, const uint32_t* __restrict__ ncount, int maxn, Phys ph,
    double* __restrict__ dts, unsigned long long* __restrict__ cnt, const double2* __restrict__ mrec) {
  extern __shared__ double dsm[];  // kMomCap staged source records
  double2* const F2 = reinterpret_cast<double2*>(dsm);
  __shared__ double2 tslot[kNWM * 2][2][kMomPairs];  // per half-warp: the current / next target's record
  __shared__ CellSm S;
  __shared__ uint32_t s_n[kTgtU], s_cur[kTgtU];
  __shared__ double acc[5][kTgtU];
  __shared__ double shdt[kNWM];
  __shared__ unsigned long long shco;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ uint32_t s_chunk;
  const int n = N > 0 ? N : ph.n;
  double dtmin = INFINITY;
  uint32_t ncoinc = 0;
  __shared__ __align__(8) uint64_t mbar;  // staging: bulk copies complete on it
  __shared__ int s_wrap;
  uint32_t mphase = 0;
  if (threadIdx.x == 0) mbar_init(&mbar, 1);
  __syncthreads();
  // cells in chunks of kCellChunk consecutive (Morton-order) cells claimed from a
  // counter: consecutive cells share most of their stencil, so a CTA's next staging
  // finds its sources in L2 (a grid stride left the re-reads to HBM)
  const uint32_t ulo = ur.lo ? *ur.lo : 0u, nun = *ur.hi;
  const uint32_t uchunk = (uint32_t)kCellChunk >> g.ubits ? (uint32_t)kCellChunk >> g.ubits : 1u;
  ChunkClaim claim{work, uchunk, 0u};
  for (uint32_t cfirst = ulo + claim.first(&s_chunk); cfirst < nun; cfirst = ulo + claim.next(&s_chunk)) {
    for (uint32_t ck = cfirst; ck < min(nun, cfirst + uchunk); ++ck) {
      unit_setup(g, ur.order ? ur.order[ck] : ck, urec, cstart, cend, S);
      const Stencil st = S.st;
      for (uint32_t t0 = S.sc; t0 < S.ec; t0 += kTgtU) {
        const uint32_t t1 = min(S.ec, t0 + kTgtU);
        for (uint32_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
          const uint32_t i = t - t0;
          s_n[i] = ncount[t];
          s_cur[i] = 0;
          acc[0][i] = 0.0;
          acc[1][i] = 0.0;
          acc[2][i] = 0.0;
          acc[3][i] = 0.0;
          acc[4][i] = -1.0;
        }
        if (threadIdx.x == 0) S.next[0] = 0;
        __syncthreads();
        for (uint32_t gb = 0, gi = 0; gb < S.total; gb += kMomCap, ++gi) {
          const uint32_t ge = min(S.total, gb + kMomCap), pend = ge;
          if (threadIdx.x == 0) S.next[(gi + 1) & 1] = 0;
          // stage [gb, ge): warp 0 issues one bulk copy of consecutive records per slot
          // (the slot's cell is a contiguous range), all complete on one mbarrier
          if (warp == 0) {
            if (lane == 0) {
              fence_proxy_async();  // the buffer's previous group was read through the generic proxy
              mbar_expect_tx(&mbar, (ge - gb) * (uint32_t)sizeof(double2) * kMomPairs);
            }
            __syncwarp();
            const int k0 = slot_of(S, gb), k1 = slot_of(S, ge - 1);
            int wr = 0;
            for (int k = k0 + lane; k <= k1; k += 32) {
              const uint32_t f0 = max(S.cum[k], gb), f1 = min(S.cum[k + 1], ge);
              if (f1 > f0) {
                bulk_g2s(F2 + (size_t)(f0 - gb) * kMomPairs,
                         mrec + (size_t)(S.t_start[k] + (f0 - S.cum[k])) * kMomPairs,
                         (f1 - f0) * (uint32_t)sizeof(double2) * kMomPairs, &mbar);
                wr |= S.t_sh[k][0] | S.t_sh[k][1] | S.t_sh[k][2];
              }
            }
            wr = __any_sync(0xffffffffu, wr != 0);
            if (lane == 0) s_wrap = wr;
          }
          mbar_wait(&mbar, mphase);
          mphase ^= 1;
          __syncthreads();  // s_wrap
          if (s_wrap) {  // periodic images: shift the staged positions of wrapped slots
            for (uint32_t qq = threadIdx.x; qq < ge - gb; qq += blockDim.x) {
              const int k = slot_of(S, gb + qq);
              if (S.t_sh[k][0] | S.t_sh[k][1] | S.t_sh[k][2]) {
                double sh[3];
                shifts_of(g, S, k, sh);
                double2* q = F2 + (size_t)qq * kMomPairs;
                q[0].x += sh[0];
                q[0].y += sh[1];
                q[1].x += sh[2];
              }
            }
            __syncthreads();
          }
          struct B {
            const double2* F2;
            const double2* __restrict__ mrec;
            double2 (*slot)[kMomPairs];  // this half-warp's two prefetch slots
            const Stencil* st;
            const Grid* g;
            double alpha;
            int n, K, sym;
            const double* tab;
            uint32_t* ncoinc;
            double xa, ya, za, vxa, vya, vza, ih2a, rinva, Xa, ca, a11, a12, a13, a22, a23, a33;
            double fx, fy, fz, fu, vs;
            // target t's record -> prefetch slot p (cp.async, 16 bytes per lane, 9 lanes);
            // every call commits one group (empty when !valid), so begin's "all but the
            // newest group" wait always means "this target's record has landed"
            __device__ __forceinline__ void fetch(uint32_t t, uint32_t p, bool valid) {
              const uint32_t l16 = threadIdx.x & 15;
              if (valid && l16 < (uint32_t)kMomPairs) cp_async16(&slot[p][l16], mrec + (size_t)t * kMomPairs + l16);
              cp_async_commit();
            }
            __device__ __forceinline__ void begin(uint32_t p, bool has) {
              cp_async_wait_prev();
              __syncwarp();  // (a half-warp mask here with the other half diverged hung the pass)
              fx = fy = fz = fu = 0.0;
              vs = -1.0;
              if (!has) return;
              const double2* r = slot[p];
              const double2 r0 = r[0], r1 = r[1], r2 = r[2], r3 = r[3], r4 = r[4], r5 = r[5], r6 = r[6],
                            r7 = r[7], r8 = r[8];
              xa = r0.x; ya = r0.y; za = r1.x; vxa = r1.y; vya = r2.x; vza = r2.y;
              ih2a = r3.y; ca = r4.x;
              Xa = r4.y * r8.y;     // (m X) / m
              rinva = r5.x * r8.y;  // (m / rho) / m
              a11 = r5.y; a12 = r6.x; a13 = r6.y; a22 = r7.x; a23 = r7.y; a33 = r8.x;  // C~_a
            }
            // pair (a, b = staged entry qi): accumulate the Eq. 2 / Eq. 3 terms and v_sig
            __device__ __forceinline__ void operator()(int qi) {
              const double2* q = F2 + (size_t)qi * kMomPairs;
              const double2 p0 = q[0], p1 = q[1], p3 = q[3];
              double dx = p0.x - xa, dy = p0.y - ya, dz = p1.x - za;
              delta3<W2>(*st, *g, dx, dy, dz);  // Delta_ab = x_b - x_a
              const double r2 = dx * dx + dy * dy + dz * dz;
              // coincident pair: Delta = 0 zeroes every term below; it is only
              // kept out of v_sig and counted (no branch)
              const bool coinc = r2 == 0.0;
              *ncoinc += coinc;
              const double ta = r2 * ih2a;
              // symmetric extra pair (r >= 2 h_a): W(r, h_a) = 0, only the h_b terms remain
              const double Sa = (W2 && sym && !(ta < 4.0)) ? 0.0 : kern_S<KM, N, true>(ta, n, tab, K);
              const double Wa = Sa;  // with u = C~_a Delta: A_ab(h_a) = Wa u
              const double tb = r2 * p3.y;
              // W(r, h_b): evaluated unconditionally (a branch on h_b != h_a cost more than
              // the second polynomial, A/B measured), zero outside its support
              const double Sb0 = kern_S<KM, N, true>(tb, n, tab, K);
              const double Sb = tb < 4.0 ? Sb0 : 0.0;
              // R5: A_ab(h_a) = C~_a Delta S_a = Wa u;  R4: A_ab(h_b) = C~_b Delta S_b = Sb w
              const double ux = a11 * dx + a12 * dy + a13 * dz;
              const double uy = a12 * dx + a22 * dy + a23 * dz;
              const double uz = a13 * dx + a23 * dy + a33 * dz;
              const double2 p5 = q[5], p6 = q[6], p7 = q[7], p8 = q[8];
              const double b11 = p5.y, b12 = p6.x, b13 = p6.y, b22 = p7.x, b23 = p7.y, b33 = p8.x;
              const double wx = b11 * dx + b12 * dy + b13 * dz;
              const double wy = b12 * dx + b22 * dy + b23 * dz;
              const double wz = b13 * dx + b23 * dy + b33 * dz;
              const double2 p2 = q[2], p4 = q[4];
              const double mb = p3.x, mXb = p4.y, mrb = p5.x, cb = p4.x;
              const double vabx = vxa - p1.y, vaby = vya - p2.x, vabz = vza - p2.y;
              const double vdotx = -(vabx * dx + vaby * dy + vabz * dz);  // v_ab . x_ab
              // Eq. 5: w_ab = v_ab . x_ab / |x_ab|, Pi' only when approaching
#ifdef SPH_MOM_AV_ALWAYS  // A/B build: branch-free w (r2 = 0 only for Delta = 0, where vdotx = 0)
              const double w = fmin(vdotx, 0.0) * rsqrt(fmax(r2, 1e-300));
#else
              const double w = vdotx < 0.0 ? vdotx * rsqrt(r2) : 0.0;
#endif
              const double vsab = ca + cb - 3.0 * w;  // v_sig; w == min(w, 0)
              const double hp = -0.25 * alpha * vsab * w;  // Pi'/2, Eq. 5
              // Eq. 2 with R2 and Eq. 4: a += -m_b (X_a A_a + X_b A_b) - g,
              //   g = (Pi'/2) (m_b/rho_a A_a + m_b/rho_b A_b), folded onto u and w
              vs = (!coinc && vsab > vs) ? vsab : vs;  // a coincident pair stays out of v_sig
              // accumulated straight into the sums (two FMA per component, no product
              // temporaries): ka = m_b W_a (X_a + (Pi'/2) / rho_a), kb = (m_b X_b + (Pi'/2) m_b/rho_b) S_b
              const double mbW = mb * Wa;
              const double ka = mbW * fma(hp, rinva, Xa);
              const double kb = fma(hp, mrb, mXb) * Sb;
              fx = fma(-ka, ux, fma(-kb, wx, fx));
              fy = fma(-ka, uy, fma(-kb, wy, fy));
              fz = fma(-ka, uz, fma(-kb, wz, fz));
              // Eq. 3 with R1, R3: du += m_b X_a v_ab.A_a + (1/2) v_ab.g
              const double vu = vabx * ux + vaby * uy + vabz * uz;
              const double vw = vabx * wx + vaby * wy + vabz * wz;
              const double hh = 0.5 * hp;
              fu = fma(mbW * fma(hh, rinva, Xa), vu, fma(hh * mrb * Sb, vw, fu));
            }
          } body;
          body.F2 = F2; body.mrec = mrec; body.slot = tslot[threadIdx.x >> 4];
          body.st = &st; body.g = &g; body.alpha = ph.alpha; body.n = n;
          body.K = ph.tableK; body.tab = ph.table; body.sym = ph.sym;
          body.ncoinc = &ncoinc;
          walk_targets_half(t0, t1, nbr, maxn, s_n, s_cur, pend, S.cum, gb, &S.next[gi & 1], body,
                            [&](bool act, uint32_t i, uint32_t c2) {
                              double v[4] = {body.fx, body.fy, body.fz, body.fu};
                              half_multi_sum<4>(v);
                              const double e = half_max(body.vs);
                              const int l16 = lane & 15;
                              if (act) {
                                if ((l16 & 3) == 0) acc[l16 >> 2][i] += v[0];
                                if (l16 == 0) {
                                  s_cur[i] = c2;
                                  acc[4][i] = fmax(acc[4][i], e);
                                }
                              }
                            });
          __syncthreads();
        }
        for (uint32_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
          const uint32_t i = t - t0;
          double vsig = acc[4][i];
          if (vsig < 0.0) vsig = 2.0 * src.c[t];  // no interacting neighbour
          out.ax[t] = acc[0][i];
          out.ay[t] = acc[1][i];
          out.az[t] = acc[2][i];
          out.du[t] = acc[3][i];
          out.vsig[t] = vsig;
          const double dta = ph.courant * tg.h[t] / vsig;  // R19
          if (!(dta > 0.0)) atomicAdd(&cnt[CNT_NONFINITE], 1ull);
          dtmin = fmin(dtmin, dta);
        }
        __syncthreads();
      }
      }
  }
  // block min dt -> one atomicMin per block (positive doubles order like uint64)
  dtmin = -wmax(-dtmin);
  if (threadIdx.x == 0) shco = 0;
  __syncthreads();
  if (ncoinc) atomicAdd(&shco, (unsigned long long)ncoinc);
  if (lane == 0) shdt[warp] = dtmin;
  __syncthreads();
  if (threadIdx.x == 0) {
    double mn = shdt[0];
    for (int q = 1; q < kNWM; ++q) mn = fmin(mn, shdt[q]);
    if (mn > 0.0)
      atomicMin((unsigned long long*)&dts[DT_RAW_BITS], (unsigned long long)__double_as_longlong(mn));
    if (shco) atomicAdd(&cnt[CNT_COINCIDENT], shco);
  }
}

// ------------------------------------------------------------------ launchers
// Which units a pass launch covers (c->unit_sel): all, or -- multi-GPU, communication
// overlapped (§8(f) NEXT-3) -- the INTERIOR units (stencil without halo cells, runnable
// while a halo exchange is in flight) or the BOUNDARY units (launched after it lands).
static URange unit_range(const sph_ctx* c) {
  if (c->unit_sel == 0 || !c->s.unit_order) return URange{nullptr, nullptr, c->s.nunit_list};
  return c->unit_sel == 1 ? URange{c->s.unit_order, nullptr, c->s.unit_bounds + 1}
                          : URange{c->s.unit_order, c->s.unit_bounds + 1, c->s.unit_bounds + 2};
}
// a claim counter per (pass, unit selection): the two launches of a pass may overlap
static int unit_work(const sph_ctx* c, int pass) { return c->unit_sel == 2 ? pass + 3 : pass; }

static int cell_grid(const sph_ctx* c, int per_sm) {
  int64_t cells = c->grid.ncell < c->P.n ? c->grid.ncell : c->P.n;
  int64_t mx = (int64_t)c->num_sms * per_sm;
  return (int)(cells < mx ? (cells > 0 ? cells : 1) : mx);
}

static bool any_wrap2(const sph_ctx* c) {
  // a periodic dim whose stencil spans every cell (tiny periodic extents): per-pair minimum image
  const Grid& g = c->grid;
  for (int d = 0; d < 3; ++d)
    if (g.periodic[d] && 2 * stencil_radius(g, d, reach_of(c->hmax)) + 1 >= g.nc[d]) return true;
  return false;
}

template <class K>
static void set_smem(K kern, size_t bytes) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <int N, bool W2, int KM, typename E>
static void density_t(sph_ctx* c) {
  const size_t smem = 4 * kDensCap * sizeof(double);
  set_smem(k_density_c<N, W2, KM, E>, smem);
  sph_particles& P = c->P;
  cudaMemsetAsync(c->s.work + unit_work(c, 1), 0, sizeof(uint32_t), c->stream);
  k_density_c<N, W2, KM, E><<<cell_grid(c, 1), kCTD, smem, c->stream>>>(
      P.x, P.y, P.z, P.h, P.m, P.u, c->grid, c->s.cell_start, c->s.cell_end, c->s.cell_hmax,
      c->s.cell_list, c->s.ncell_list, c->s.unit_rec, unit_range(c), c->s.work + unit_work(c, 1), reinterpret_cast<const E*>(c->s.nbr), c->s.ncount, c->maxn_cap, c->phys, P.rho, P.omega,
      P.p, P.c, c->s.wB, c->s.ih2, c->s.vol, c->s.rinv, c->s.X, c->s.mX, c->s.cnt);
}

// row type x kernel-mode x exponent x wrap dispatch of a pair pass
#define SPH_DISPATCH_E(fn, E)                                                         \
  do {                                                                                \
    const bool w2 = any_wrap2(c) || c->phys.sym; /* the general (rare-case) variant */ \
    const bool n6 = c->phys.n == 6;                                                   \
    switch (c->phys.kmode) {                                                          \
      case SPH_KERNEL_TABLE:                                                          \
        n6 ? (w2 ? fn<6, true, 1, E>(c) : fn<6, false, 1, E>(c))                      \
           : (w2 ? fn<0, true, 1, E>(c) : fn<0, false, 1, E>(c));                     \
        break;                                                                        \
      case SPH_KERNEL_SIN:                                                            \
        n6 ? (w2 ? fn<6, true, 2, E>(c) : fn<6, false, 2, E>(c))                      \
           : (w2 ? fn<0, true, 2, E>(c) : fn<0, false, 2, E>(c));                     \
        break;                                                                        \
      default:                                                                        \
        n6 ? (w2 ? fn<6, true, 0, E>(c) : fn<6, false, 0, E>(c))                      \
           : (w2 ? fn<0, true, 0, E>(c) : fn<0, false, 0, E>(c));                     \
    }                                                                                 \
  } while (0)
#define SPH_DISPATCH(fn)                                                              \
  do {                                                                                \
    if (c->wide_rows) SPH_DISPATCH_E(fn, uint32_t);                                   \
    else SPH_DISPATCH_E(fn, uint16_t);                                                \
  } while (0)

int launch_density(sph_ctx* c) {
  SPH_DISPATCH(density_t);
  return 1;
}

template <int N, bool W2, int KM, typename E>
static void iad_t(sph_ctx* c) {
  const size_t smem = 4 * kIadCap * sizeof(double);
  set_smem(k_iad_c<N, W2, KM, E>, smem);
  sph_particles& P = c->P;
  cudaMemsetAsync(c->s.work + unit_work(c, 2), 0, sizeof(uint32_t), c->stream);
  k_iad_c<N, W2, KM, E><<<cell_grid(c, 1), kCTD, smem, c->stream>>>(
      P.x, P.y, P.z, c->grid, c->s.cell_start, c->s.cell_end, c->s.cell_hmax, c->s.cell_list,
      c->s.ncell_list, c->s.unit_rec, unit_range(c), c->s.work + unit_work(c, 2), reinterpret_cast<const E*>(c->s.nbr), c->s.ncount, c->maxn_cap, c->phys, c->s.wB, c->s.ih2, c->s.vol,
      P.c11, P.c12, P.c13, P.c22, P.c23, P.c33, c->s.ct, c->cap, c->s.cnt,
      MomSrc{P.x, P.y, P.z, P.vx, P.vy, P.vz, P.m, c->s.ih2, P.c, c->s.mX, c->s.vol, c->s.ct, c->cap},
      kIadRecords ? reinterpret_cast<double2*>(c->s.mrec) : nullptr);
}

int launch_iad(sph_ctx* c) {
  SPH_DISPATCH(iad_t);
  return 1;
}

template <int N, bool W2, int KM, typename E>
static void momentum_t(sph_ctx* c) {
  const size_t smem = (size_t)2 * kMomPairs * kMomCap * sizeof(double);
  set_smem(k_momentum_c<N, W2, KM, E>, smem);
  sph_particles& P = c->P;
  MomSrc src = {P.x, P.y, P.z, P.vx, P.vy, P.vz, P.m, c->s.ih2, P.c, c->s.mX, c->s.vol, c->s.ct, c->cap};
  MomTgt tg = {P.h, c->s.wB, c->s.rinv, c->s.X, P.c11, P.c12, P.c13, P.c22, P.c23, P.c33};
  MomOut out = {P.ax, P.ay, P.az, P.du, P.vsig};
  cudaMemsetAsync(c->s.work + unit_work(c, 3), 0, sizeof(uint32_t), c->stream);
  k_momentum_c<N, W2, KM, E><<<cell_grid(c, 1), kCTM, smem, c->stream>>>(
      src, tg, out, c->grid, c->s.cell_start, c->s.cell_end, c->s.cell_hmax, c->s.cell_list,
      c->s.ncell_list, c->s.unit_rec, unit_range(c), c->s.work + unit_work(c, 3), reinterpret_cast<const E*>(c->s.nbr), c->s.ncount, c->maxn_cap, c->phys, c->s.dts, c->s.cnt,
      reinterpret_cast<const double2*>(c->s.mrec));
}

int launch_momentum(sph_ctx* c) {
  SPH_DISPATCH(momentum_t);
  return 1;
}

int launch_mom_records_range(sph_ctx* c, int64_t i0, int64_t n, cudaStream_t st) {
  if (n <= 0) return 0;
  sph_particles& P = c->P;
  MomSrc src = {P.x, P.y, P.z, P.vx, P.vy, P.vz, P.m, c->s.ih2, P.c, c->s.mX, c->s.vol, c->s.ct, c->cap};
  k_mom_records<<<grid_blocks(c, n, kRecThreads, 6), kRecThreads, 0, st>>>(src, i0, n,
                                                                          reinterpret_cast<double2*>(c->s.mrec));
  return 1;
}

int launch_mom_records_owned(sph_ctx* c) {  // multi-GPU: halo records come with exchange #3
  return kIadRecords ? 0 : launch_mom_records_range(c, 0, c->P.n, c->stream);
}

int launch_mom_records(sph_ctx* c) {  // the sources the IAD epilogue did not write
  return kIadRecords ? launch_mom_records_range(c, c->P.n, c->n_halo, c->stream)
                     : launch_mom_records_range(c, 0, c->P.n + c->n_halo, c->stream);
}

}  // namespace sphb
