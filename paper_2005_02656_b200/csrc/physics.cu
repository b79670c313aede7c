// physics.cu -- a5 neighbour search, a6 density + Omega + EOS, a8 IAD,
// a10-a11 momentum + energy + AV + dt, a12-a13 update + h, a15 diagnostics.
//
// Execution model: ONE WARP PER TARGET PARTICLE; the 32 lanes stride over the
// target's candidates (search) or neighbour row (pair passes).  Target data is
// warp-uniform (broadcast loads, registers); neighbour rows are read with
// coalesced 128-byte loads; neighbours of one target come in runs of
// consecutive indices (cells are contiguous in the Morton order), so the SoA
// gathers are mostly coalesced too.  Per-target sums are finished with a
// shuffle tree, so no atomics touch particle data (results are deterministic).
//
// Kernel evaluation (Eq. 6): S(v) = [sinc(pi v/2)]^n is evaluated
// as P(t)^n with t = v^2 = r^2/h^2 and P the Maclaurin polynomial of
// sinc(pi sqrt(t)/2) (13 terms, truncation < 8e-16 absolute on t in [0,4]).
// No sqrt, sin or division per pair -- the B200 counterpart of the paper's
// lookup table + integer pow, and more accurate than that table.
#include "sph_internal.cuh"

namespace sphb {

constexpr int kWarpThreads = 256;  // 8 warps = 8 targets in flight per block

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
// "inline x*x*x*x..."
__device__ __forceinline__ double ipow(double s, int n) {
  if (n == 6) {
    double s2 = s * s;
    double s4 = s2 * s2;
    return s4 * s2;
  }
  double r = 1.0;
  for (int k = 0; k < n; ++k) r *= s;
  return r;
}

// minimum image on periodic dims -- same branch formula as the oracle
__device__ __forceinline__ double min_image(double d, int periodic, double L) {
  if (periodic) {
    if (d > 0.5 * L) d -= L;
    else if (d < -0.5 * L) d += L;
  }
  return d;
}

__device__ __forceinline__ int cell_coord(const Grid& g, int d, double v) {
  double q = (v - g.lo[d]) * g.inv[d];
  int c = (int)floor(q);
  c = c < 0 ? 0 : c;
  c = c > g.nc[d] - 1 ? g.nc[d] - 1 : c;
  return c;
}

// ------------------------------------------------------------------ a5 neighbours
// N(a) = {b != a : r_ab^2 < (2 h_a)^2}; r^2 evaluated with _rn intrinsics in the
// oracle's association ((dx dx + dy dy) + dz dz), no FMA, so the set is bit-exact.
// Candidate cells: per dim, the cells within R = ceil(2 h_a (1 + 2^-20) / edge)
// of the target's cell (all cells when 2R+1 >= nc) -- conservative by construction.
__global__ void __launch_bounds__(kWarpThreads) k_neighbors(
    const double* __restrict__ x, const double* __restrict__ y, const double* __restrict__ z,
    const double* __restrict__ h, int64_t n, Grid g, const uint32_t* __restrict__ cstart,
    const uint32_t* __restrict__ cend, uint32_t* __restrict__ nbr, uint32_t* __restrict__ ncount,
    int maxn, unsigned int* __restrict__ maxcount) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t a = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; a < n; a += nw) {
    const double xa = x[a], ya = y[a], za = z[a];
    const double tha = 2.0 * h[a];
    const double lim = __dmul_rn(tha, tha);
    const double reach = tha * (1.0 + 0x1p-20);
    int lo[3], cnt[3];
    const double pos[3] = {xa, ya, za};
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      int ca = cell_coord(g, d, pos[d]);
      int R = (int)ceil(reach * g.inv[d]);
      if (2 * R + 1 >= g.nc[d]) {
        lo[d] = 0;
        cnt[d] = g.nc[d];
      } else if (g.periodic[d]) {
        lo[d] = ca - R;
        cnt[d] = 2 * R + 1;
      } else {
        int l = ca - R < 0 ? 0 : ca - R;
        int u = ca + R > g.nc[d] - 1 ? g.nc[d] - 1 : ca + R;
        lo[d] = l;
        cnt[d] = u - l + 1;
      }
    }
    uint32_t count = 0;
    uint32_t* row = nbr + (size_t)a * maxn;
    for (int iz = 0; iz < cnt[2]; ++iz) {
      int cz = lo[2] + iz;
      cz = cz < 0 ? cz + g.nc[2] : (cz >= g.nc[2] ? cz - g.nc[2] : cz);
      for (int iy = 0; iy < cnt[1]; ++iy) {
        int cy = lo[1] + iy;
        cy = cy < 0 ? cy + g.nc[1] : (cy >= g.nc[1] ? cy - g.nc[1] : cy);
        for (int ix = 0; ix < cnt[0]; ++ix) {
          int cx = lo[0] + ix;
          cx = cx < 0 ? cx + g.nc[0] : (cx >= g.nc[0] ? cx - g.nc[0] : cx);
          int64_t c = cx + (int64_t)g.nc[0] * (cy + (int64_t)g.nc[1] * cz);
          const uint32_t s = cstart[c], e = cend[c];
          for (uint32_t base = s; base < e; base += 32) {
            const uint32_t j = base + lane;
            bool hit = false;
            if (j < e && (int64_t)j != a) {
              double dx = min_image(__dsub_rn(x[j], xa), g.periodic[0], g.L[0]);
              double dy = min_image(__dsub_rn(y[j], ya), g.periodic[1], g.L[1]);
              double dz = min_image(__dsub_rn(z[j], za), g.periodic[2], g.L[2]);
              double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                                    __dmul_rn(dz, dz));
              hit = r2 < lim;
            }
            const unsigned b = __ballot_sync(0xffffffffu, hit);
            if (hit) {
              uint32_t p = count + __popc(b & lt);
              if (p < (uint32_t)maxn) row[p] = j;
            }
            count += __popc(b);
          }
        }
      }
    }
    if (lane == 0) {
      ncount[a] = count;
      if (count > (uint32_t)maxn) atomicMax(maxcount, count);
    }
  }
}

int launch_neighbors(sph_ctx* c) {
  int nb = grid_blocks(c, c->P.n * 32, kWarpThreads, 8);
  k_neighbors<<<nb, kWarpThreads, 0, c->stream>>>(c->P.x, c->P.y, c->P.z, c->P.h, c->P.n, c->grid,
                                                  c->s.cell_start, c->s.cell_end, c->s.nbr,
                                                  c->s.ncount, c->maxn, c->s.nbr_maxcount);
  return 1;
}

// ------------------------------------------------------------------ a6 density + Omega + EOS
__global__ void __launch_bounds__(kWarpThreads) k_density(
    const double* __restrict__ x, const double* __restrict__ y, const double* __restrict__ z,
    const double* __restrict__ h, const double* __restrict__ m, const double* __restrict__ u,
    int64_t n, const uint32_t* __restrict__ nbr, const uint32_t* __restrict__ ncount, int maxn,
    Phys ph, double* __restrict__ rho, double* __restrict__ omega, double* __restrict__ p,
    double* __restrict__ cs, double* __restrict__ wB, double* __restrict__ ih2,
    double* __restrict__ vol, double* __restrict__ rinv, double* __restrict__ X,
    unsigned long long* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t a = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; a < n; a += nw) {
    const double xa = x[a], ya = y[a], za = z[a], ha = h[a];
    const double ih = 1.0 / ha;
    const double ih2a = ih * ih;
    const uint32_t cn = ncount[a];
    const uint32_t* row = nbr + (size_t)a * maxn;
    double sr = 0.0, sd = 0.0;
    for (uint32_t k = lane; k < cn; k += 32) {
      const uint32_t j = row[k];
      double dx = min_image(x[j] - xa, ph.periodic[0], ph.L[0]);
      double dy = min_image(y[j] - ya, ph.periodic[1], ph.L[1]);
      double dz = min_image(z[j] - za, ph.periodic[2], ph.L[2]);
      double t = (dx * dx + dy * dy + dz * dz) * ih2a;
      double P = sinc_poly(ph, t);
      double Pn1 = ipow(P, ph.n - 1);
      double dP = sinc_dpoly(ph, t);
      double mj = m[j];
      sr += mj * (Pn1 * P);
      // 3 S + v S'(v) = P^(n-1) (3 P + 2 n t P'(t))
      sd += mj * (Pn1 * (3.0 * P + 2.0 * ph.n * t * dP));
    }
    sr = wsum(sr);
    sd = wsum(sd);
    if (lane == 0) {
      const double ma = m[a];
      const double wBa = ph.B * ih * ih2a;            // B / h^3
      const double r = wBa * (ma + sr);               // Eq. 1 with self term (R11)
      const double dsum = -wBa * ih * (3.0 * ma + sd);  // sum_b m_b dW_ab/dh_a
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
        P_ = (ph.gamma - 1.0) * r * u[a];
        c_ = sqrt(ph.gamma * P_ / r);
      }
      rho[a] = r;
      omega[a] = om;
      p[a] = P_;
      cs[a] = c_;
      wB[a] = wBa;
      ih2[a] = ih2a;
      vol[a] = ma / r;
      rinv[a] = 1.0 / r;
      X[a] = P_ / (om * r * r);  // R1: P / (Omega rho^2)
    }
  }
}

int launch_density(sph_ctx* c) {
  sph_particles& P = c->P;
  int nb = grid_blocks(c, P.n * 32, kWarpThreads, 8);
  k_density<<<nb, kWarpThreads, 0, c->stream>>>(
      P.x, P.y, P.z, P.h, P.m, P.u, P.n, c->s.nbr, c->s.ncount, c->maxn, c->phys, P.rho, P.omega,
      P.p, P.c, c->s.wB, c->s.ih2, c->s.vol, c->s.rinv, c->s.X, c->s.cnt);
  return 1;
}

// ------------------------------------------------------------------ a8 IAD
__global__ void __launch_bounds__(kWarpThreads) k_iad(
    const double* __restrict__ x, const double* __restrict__ y, const double* __restrict__ z,
    int64_t n, const uint32_t* __restrict__ nbr, const uint32_t* __restrict__ ncount, int maxn,
    Phys ph, const double* __restrict__ wB, const double* __restrict__ ih2,
    const double* __restrict__ vol, double* __restrict__ c11, double* __restrict__ c12,
    double* __restrict__ c13, double* __restrict__ c22, double* __restrict__ c23,
    double* __restrict__ c33, unsigned long long* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t a = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; a < n; a += nw) {
    const double xa = x[a], ya = y[a], za = z[a], ih2a = ih2[a];
    const uint32_t cn = ncount[a];
    const uint32_t* row = nbr + (size_t)a * maxn;
    double t11 = 0, t12 = 0, t13 = 0, t22 = 0, t23 = 0, t33 = 0;
    for (uint32_t k = lane; k < cn; k += 32) {
      const uint32_t j = row[k];
      double dx = min_image(x[j] - xa, ph.periodic[0], ph.L[0]);
      double dy = min_image(y[j] - ya, ph.periodic[1], ph.L[1]);
      double dz = min_image(z[j] - za, ph.periodic[2], ph.L[2]);
      double t = (dx * dx + dy * dy + dz * dz) * ih2a;
      double w = vol[j] * ipow(sinc_poly(ph, t), ph.n);  // (m_b/rho_b) S  (B/h^3 applied below)
      double wx = w * dx, wy = w * dy;
      t11 += wx * dx;
      t12 += wx * dy;
      t13 += wx * dz;
      t22 += wy * dy;
      t23 += wy * dz;
      t33 += w * dz * dz;
    }
    t11 = wsum(t11); t12 = wsum(t12); t13 = wsum(t13);
    t22 = wsum(t22); t23 = wsum(t23); t33 = wsum(t33);
    if (lane == 0) {
      const double s = wB[a];
      t11 *= s; t12 *= s; t13 *= s; t22 *= s; t23 *= s; t33 *= s;
      double det = t11 * (t22 * t33 - t23 * t23) - t12 * (t12 * t33 - t23 * t13) +
                   t13 * (t12 * t23 - t22 * t13);
      double id = 1.0 / det;
      double i11 = (t22 * t33 - t23 * t23) * id;
      double i12 = (t13 * t23 - t12 * t33) * id;
      double i13 = (t12 * t23 - t13 * t22) * id;
      double i22 = (t11 * t33 - t13 * t13) * id;
      double i23 = (t12 * t13 - t11 * t23) * id;
      double i33 = (t11 * t22 - t12 * t12) * id;
      double nt = sqrt(t11 * t11 + t22 * t22 + t33 * t33 + 2.0 * (t12 * t12 + t13 * t13 + t23 * t23));
      double ni = sqrt(i11 * i11 + i22 * i22 + i33 * i33 + 2.0 * (i12 * i12 + i13 * i13 + i23 * i23));
      if (!(det > 0.0) || !(nt * ni <= 1e12)) {  // reading R29
        double tr = t11 + t22 + t33;
        double q = tr > 0.0 ? 3.0 / tr : 0.0;
        i11 = q; i22 = q; i33 = q;
        i12 = 0.0; i13 = 0.0; i23 = 0.0;
        atomicAdd(&cnt[CNT_IAD_SINGULAR], 1ull);
      }
      c11[a] = i11; c12[a] = i12; c13[a] = i13;
      c22[a] = i22; c23[a] = i23; c33[a] = i33;
    }
  }
}

int launch_iad(sph_ctx* c) {
  sph_particles& P = c->P;
  int nb = grid_blocks(c, P.n * 32, kWarpThreads, 8);
  k_iad<<<nb, kWarpThreads, 0, c->stream>>>(P.x, P.y, P.z, P.n, c->s.nbr, c->s.ncount, c->maxn,
                                            c->phys, c->s.wB, c->s.ih2, c->s.vol, P.c11, P.c12,
                                            P.c13, P.c22, P.c23, P.c33, c->s.cnt);
  return 1;
}

// ------------------------------------------------------------------ a10-a11 momentum + energy + dt
struct MomIn {
  const double *x, *y, *z, *vx, *vy, *vz, *h, *m, *c;
  const double *c11, *c12, *c13, *c22, *c23, *c33;
  const double *wB, *ih2, *rinv, *X;
};
struct MomOut {
  double *ax, *ay, *az, *du, *vsig;
};

__global__ void __launch_bounds__(kWarpThreads) k_momentum(MomIn in, MomOut out, int64_t n,
                                                           const uint32_t* __restrict__ nbr,
                                                           const uint32_t* __restrict__ ncount,
                                                           int maxn, Phys ph,
                                                           double* __restrict__ dts,
                                                           unsigned long long* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double dtmin = INFINITY;
  unsigned long long ncoinc = 0;
  for (int64_t a = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; a < n; a += nw) {
    const double xa = in.x[a], ya = in.y[a], za = in.z[a];
    const double vxa = in.vx[a], vya = in.vy[a], vza = in.vz[a];
    const double ih2a = in.ih2[a], wBa = in.wB[a], rinva = in.rinv[a], Xa = in.X[a], ca = in.c[a];
    const double a11 = in.c11[a], a12 = in.c12[a], a13 = in.c13[a], a22 = in.c22[a],
                 a23 = in.c23[a], a33 = in.c33[a];
    const uint32_t cn = ncount[a];
    const uint32_t* row = nbr + (size_t)a * maxn;
    double fx = 0.0, fy = 0.0, fz = 0.0, fu = 0.0, vs = -1.0;
    for (uint32_t k = lane; k < cn; k += 32) {
      const uint32_t j = row[k];
      const double dx = min_image(in.x[j] - xa, ph.periodic[0], ph.L[0]);  // Delta_ab = x_b - x_a
      const double dy = min_image(in.y[j] - ya, ph.periodic[1], ph.L[1]);
      const double dz = min_image(in.z[j] - za, ph.periodic[2], ph.L[2]);
      const double r2 = dx * dx + dy * dy + dz * dz;
      if (r2 == 0.0) {  // coincident pair: skipped, counted
        ++ncoinc;
        continue;
      }
      const double ta = r2 * ih2a;
      const double Sa = ipow(sinc_poly(ph, ta), ph.n);
      const double Wa = wBa * Sa;
      const double tb = r2 * in.ih2[j];
      double Sb = 0.0;  // b's support may not reach a (variable h)
      if (tb < 4.0) Sb = (tb == ta) ? Sa : ipow(sinc_poly(ph, tb), ph.n);
      const double Wb = in.wB[j] * Sb;
      // R5: A_ab(h_a) = C_a Delta W_ab(h_a);  R4: A_ab(h_b) = C_b Delta W_ab(h_b)
      const double Aax = (a11 * dx + a12 * dy + a13 * dz) * Wa;
      const double Aay = (a12 * dx + a22 * dy + a23 * dz) * Wa;
      const double Aaz = (a13 * dx + a23 * dy + a33 * dz) * Wa;
      const double b11 = in.c11[j], b12 = in.c12[j], b13 = in.c13[j], b22 = in.c22[j],
                   b23 = in.c23[j], b33 = in.c33[j];
      const double Abx = (b11 * dx + b12 * dy + b13 * dz) * Wb;
      const double Aby = (b12 * dx + b22 * dy + b23 * dz) * Wb;
      const double Abz = (b13 * dx + b23 * dy + b33 * dz) * Wb;
      const double mb = in.m[j], Xb = in.X[j], rinvb = in.rinv[j], cb = in.c[j];
      const double vabx = vxa - in.vx[j], vaby = vya - in.vy[j], vabz = vza - in.vz[j];
      const double vdotx = -(vabx * dx + vaby * dy + vabz * dz);  // v_ab . x_ab
      double Pi = 0.0, w = 0.0;
      if (vdotx < 0.0) {  // Eq. 5
        w = vdotx * rsqrt(r2);  // w_ab = v_ab . x_ab / |x_ab|
        Pi = -0.5 * ph.alpha * (ca + cb - 3.0 * w) * w;
      }
      vs = fmax(vs, ca + cb - 3.0 * w);  // v_sig; w == min(w, 0) here
      // Eq. 4 pair term g = 1/2 m_b Pi' (A_a / rho_a + A_b / rho_b)
      const double hp = 0.5 * mb * Pi;
      const double gx = hp * (Aax * rinva + Abx * rinvb);
      const double gy = hp * (Aay * rinva + Aby * rinvb);
      const double gz = hp * (Aaz * rinva + Abz * rinvb);
      // Eq. 2 with R2 (AV subtracted)
      fx += -mb * (Xa * Aax + Xb * Abx) - gx;
      fy += -mb * (Xa * Aay + Xb * Aby) - gy;
      fz += -mb * (Xa * Aaz + Xb * Abz) - gz;
      // Eq. 3 with R1, R3
      fu += mb * Xa * (vabx * Aax + vaby * Aay + vabz * Aaz) + 0.5 * (vabx * gx + vaby * gy + vabz * gz);
    }
    fx = wsum(fx);
    fy = wsum(fy);
    fz = wsum(fz);
    fu = wsum(fu);
    vs = wmax(vs);
    if (lane == 0) {
      if (vs < 0.0) vs = 2.0 * ca;  // no interacting neighbour
      out.ax[a] = fx;
      out.ay[a] = fy;
      out.az[a] = fz;
      out.du[a] = fu;
      out.vsig[a] = vs;
      double dta = ph.courant * in.h[a] / vs;  // R19
      if (!(dta > 0.0) || dta == INFINITY) {
        if (!(dta > 0.0)) atomicAdd(&cnt[CNT_NONFINITE], 1ull);
      }
      dtmin = fmin(dtmin, dta);
    }
  }
  // block min of dt -> one atomicMin per block on the bit pattern (dt > 0: ordered as uint64)
  __shared__ double sh[kWarpThreads / 32];
  __shared__ unsigned long long shc;
  if (threadIdx.x == 0) shc = 0;
  __syncthreads();
  if (ncoinc) atomicAdd(&shc, ncoinc);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = dtmin;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = sh[0];
    for (int q = 1; q < kWarpThreads / 32; ++q) m = fmin(m, sh[q]);
    if (m > 0.0) atomicMin((unsigned long long*)&dts[DT_RAW_BITS], (unsigned long long)__double_as_longlong(m));
    if (shc) atomicAdd(&cnt[CNT_COINCIDENT], shc);
  }
}

int launch_momentum(sph_ctx* c) {
  sph_particles& P = c->P;
  MomIn in = {P.x, P.y, P.z, P.vx, P.vy, P.vz, P.h, P.m, P.c, P.c11, P.c12, P.c13, P.c22, P.c23,
              P.c33, c->s.wB, c->s.ih2, c->s.rinv, c->s.X};
  MomOut out = {P.ax, P.ay, P.az, P.du, P.vsig};
  int nb = grid_blocks(c, P.n * 32, kWarpThreads, 8);
  k_momentum<<<nb, kWarpThreads, 0, c->stream>>>(in, out, P.n, c->s.nbr, c->s.ncount, c->maxn,
                                                 c->phys, c->s.dts, c->s.cnt);
  return 1;
}

// dt = min(raw, growth * dt_prev) except on the first step; dt_prev := dt on the first step
__global__ void k_dt_finalize(double* dts, int first, double growth) {
  double raw = __longlong_as_double((long long)*(unsigned long long*)&dts[DT_RAW_BITS]);
  double prev = first ? raw : dts[DT_COMMITTED];
  double dt = raw;
  if (!first && growth * prev < dt) dt = growth * prev;
  dts[DT_CUR] = dt;
  dts[DT_PREV] = first ? dt : prev;
}

int launch_dt_finalize(sph_ctx* c) {
  k_dt_finalize<<<1, 1, 0, c->stream>>>(c->s.dts, c->first ? 1 : 0, c->phys.dt_growth);
  return 1;
}

// ------------------------------------------------------------------ a12-a13 update + h
struct UpdState {
  double *x, *y, *z, *vx, *vy, *vz, *vhx, *vhy, *vhz, *u, *du_prev, *h;
  const double *ax, *ay, *az, *du;
};

__global__ void k_update(UpdState s, int64_t n, const uint32_t* __restrict__ ncount, Phys ph,
                         int first, double* __restrict__ dts, unsigned long long* __restrict__ cnt) {
  const double dt = dts[DT_CUR], dtp = dts[DT_PREV];
  const double q = dt / dtp;
  unsigned long long nfl = 0, nhc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double* X[3] = {s.x, s.y, s.z};
    double* V[3] = {s.vx, s.vy, s.vz};
    double* VH[3] = {s.vhx, s.vhy, s.vhz};
    const double* A[3] = {s.ax, s.ay, s.az};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double ak = A[k][i];
      double vb = first ? V[k][i] - 0.5 * ak * dt : VH[k][i];
      vb = vb + ak * (dtp + dt) * 0.5;  // kick to t + dt/2 (R17)
      double xn = X[k][i] + dt * vb;    // drift
      if (ph.periodic[k]) {
        if (xn >= ph.box_hi[k]) xn -= ph.L[k];
        else if (xn < ph.box_lo[k]) xn += ph.L[k];
      }
      X[k][i] = xn;
      VH[k][i] = vb;
      V[k][i] = vb + 0.5 * ak * dt;
    }
    // variable-step AB2 (R18)
    const double dui = s.du[i];
    const double dp = first ? dui : s.du_prev[i];
    double un = s.u[i] + dt * ((1.0 + 0.5 * q) * dui - 0.5 * q * dp);
    if (un < ph.u_floor) {
      un = ph.u_floor;
      ++nfl;
    }
    s.u[i] = un;
    s.du_prev[i] = dui;
    // h update (R20)
    const uint32_t nn = ncount[i];
    double hn = s.h[i] * 0.5 * (1.0 + cbrt(ph.n_target / (double)(nn > 1 ? nn : 1)));
    if (hn < ph.h_min) {
      hn = ph.h_min;
      ++nhc;
    }
    if (ph.h_max > 0.0 && hn > ph.h_max) {
      hn = ph.h_max;
      ++nhc;
    }
    s.h[i] = hn;
  }
  if (nfl) atomicAdd(&cnt[CNT_U_FLOOR], nfl);
  if (nhc) atomicAdd(&cnt[CNT_H_CLAMP], nhc);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    dts[DT_COMMITTED] = dt;
    dts[DT_TIME] += dt;
  }
}

int launch_update(sph_ctx* c) {
  sph_particles& P = c->P;
  UpdState s = {P.x, P.y, P.z, P.vx, P.vy, P.vz, P.vhx, P.vhy, P.vhz, P.u, P.du_prev, P.h,
                P.ax, P.ay, P.az, P.du};
  k_update<<<grid_blocks(c, P.n, 256, 8), 256, 0, c->stream>>>(s, P.n, c->s.ncount, c->phys,
                                                               c->first ? 1 : 0, c->s.dts, c->s.cnt);
  return 1;
}

// ------------------------------------------------------------------ a15 diagnostics
__global__ void k_diag(const double* __restrict__ m, const double* __restrict__ x,
                       const double* __restrict__ y, const double* __restrict__ z,
                       const double* __restrict__ vx, const double* __restrict__ vy,
                       const double* __restrict__ vz, const double* __restrict__ u,
                       const uint32_t* __restrict__ ncount, int64_t n, double* __restrict__ part) {
  double v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double mi = m[i], X = x[i], Y = y[i], Z = z[i], VX = vx[i], VY = vy[i], VZ = vz[i];
    v[0] += mi * VX;
    v[1] += mi * VY;
    v[2] += mi * VZ;
    v[3] += mi * (Y * VZ - Z * VY);
    v[4] += mi * (Z * VX - X * VZ);
    v[5] += mi * (X * VY - Y * VX);
    v[6] += mi * (u[i] + 0.5 * (VX * VX + VY * VY + VZ * VZ));
    v[7] += (double)ncount[i];
  }
  __shared__ double sh[8][8];
  int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = 0; k < 8; ++k) {
    double r = wsum(v[k]);
    if (lane == 0) sh[k][w] = r;
  }
  __syncthreads();
  if (threadIdx.x < 8) {
    double r = 0.0;
    for (int q = 0; q < 8; ++q) r += sh[threadIdx.x][q];
    part[(int64_t)blockIdx.x * 8 + threadIdx.x] = r;
  }
}

__global__ void k_diag_final(const double* __restrict__ part, int nblk, double* __restrict__ out) {
  int k = threadIdx.x;
  if (k >= 8) return;
  double r = 0.0;
  for (int b = 0; b < nblk; ++b) r += part[(int64_t)b * 8 + k];
  out[k] = r;
}

int launch_diag(sph_ctx* c) {
  sph_particles& P = c->P;
  int nb = grid_blocks(c, P.n, 256, 4);
  k_diag<<<nb, 256, 0, c->stream>>>(P.m, P.x, P.y, P.z, P.vx, P.vy, P.vz, P.u, c->s.ncount, P.n,
                                    c->s.red);
  k_diag_final<<<1, 32, 0, c->stream>>>(c->s.red, nb, c->s.diag);
  return 2;
}

}  // namespace sphb
