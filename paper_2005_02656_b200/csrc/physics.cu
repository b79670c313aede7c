// physics.cu -- a11 dt finalisation, a12-a13 update + h, a15 diagnostics.
// (The pair passes a5/a6/a8/a10 live in cellpass.cu.)
#include "sph_internal.cuh"

namespace sphb {


__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// dt = min(raw, growth * dt_prev) except on the first step; dt_prev := dt on the first step
// A non-finite or non-positive dt sets DT_BAD: k_update then leaves the state
// untouched and the next sph_find_neighbors / sph_diagnostics returns SPH_ERR_NUMERIC,
// whether or not the caller asked for dt on the host.
__global__ void k_dt_finalize(double* dts, int first, double growth, int nonempty, unsigned long long* cnt) {
  double raw = __longlong_as_double((long long)*(unsigned long long*)&dts[DT_RAW_BITS]);
  double prev = first ? raw : dts[DT_COMMITTED];
  double dt = raw;
  if (!first && growth * prev < dt) dt = growth * prev;
  dts[DT_CUR] = dt;
  dts[DT_PREV] = first ? dt : prev;
  const bool bad = nonempty && !(dt > 0.0 && dt < INFINITY);  // no particle anywhere: dt = inf
  dts[DT_BAD] = bad ? 1.0 : 0.0;
  if (bad) atomicAdd(&cnt[CNT_NONFINITE], 1ull);
  // re-arm the atomic-min slot for the next momentum pass (+inf)
  *(unsigned long long*)&dts[DT_RAW_BITS] = 0x7ff0000000000000ull;
}

int launch_dt_finalize(sph_ctx* c, bool nonempty) {
  k_dt_finalize<<<1, 1, 0, c->stream>>>(c->s.dts, c->first ? 1 : 0, c->phys.dt_growth, nonempty ? 1 : 0,
                                        c->s.cnt);
  return 1;
}

// ------------------------------------------------------------------ a12-a13 update + h
struct UpdState {
  double *x, *y, *z, *vx, *vy, *vz, *vhx, *vhy, *vhz, *u, *du_prev, *h;
  const double *ax, *ay, *az, *du;
};

__global__ void k_update(UpdState s, int64_t n, const uint32_t* __restrict__ ncount, Phys ph,
                         int first, double* __restrict__ dts, unsigned long long* __restrict__ cnt,
                         const int64_t* __restrict__ id, unsigned long long* __restrict__ bad_id) {
  if (dts[DT_BAD] != 0.0) return;  // invalid dt: keep the state, the error surfaces next call
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
        // reading R30: the wrapped value stays in [lo, hi) against rounding
        if (xn < ph.box_lo[k]) xn = ph.box_lo[k];
        if (xn >= ph.box_hi[k]) xn = nextafter(ph.box_hi[k], ph.box_lo[k]);
      }
      if (!isfinite(xn) || !isfinite(vb)) atomicMin(bad_id, (unsigned long long)id[i]);
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
    if (!isfinite(un) || !(hn > 0.0 && hn < INFINITY)) atomicMin(bad_id, (unsigned long long)id[i]);
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
                                                               c->first ? 1 : 0, c->s.dts, c->s.cnt,
                                                               P.id, c->s.bad_id);
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
