/* oracle/sph_oracle.c -- plain, slow, fp64 CPU oracle of the SPH-EXA hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see sph_oracle.h).  Written from PAPER.md §4.1
 * (Eqs. 1-6) with the readings R1-R29 listed in DESIGN.md §3; each
 * function cites the passage it follows.  No blocking, fusion or reordering:
 * every per-particle quantity is the plain sum of its definition, taken over
 * the neighbour row in ascending order.  OpenMP only splits the outer loop over
 * target particles, so results do not depend on the thread count.
 *
 * Parity pins: tests/test_oracle_*.py (closed forms, brute force, invariants).
 */
#include "sph_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ------------------------------------------------------------------------ */
/* O2 kernel -- Eq. 6: W = B_n/h^3 * [sinc(pi v / 2)]^n, 0<=v<2.  */
/* ------------------------------------------------------------------------ */

static double sinc(double x) { return x == 0.0 ? 1.0 : sin(x) / x; }

/* "inline x*x*x*x..." for integer exponents; generic pow otherwise */
static double powi_or_pow(double s, double n) {
  if (n == 6.0) {
    double s2 = s * s;
    double s4 = s2 * s2;
    return s4 * s2;
  }
  if (n == floor(n) && n >= 0.0 && n <= 9.0) {
    double r = 1.0;
    for (int k = 0; k < (int)n; ++k) r *= s;
    return r;
  }
  return pow(s, n);
}

static double S_direct(double n, double v) {
  if (!(v < 2.0)) return 0.0;
  return powi_or_pow(sinc(0.5 * M_PI * v), n);
}

void orc_table_build(double n, int K, double* table) {
  /* reading R12: K samples of S_n on [0,2] including both endpoints */
  for (int k = 0; k < K; ++k) table[k] = S_direct(n, 2.0 * (double)k / (double)(K - 1));
}

double orc_S(const orc_params* p, double v) {
  if (!(v < 2.0)) return 0.0;
  if (p->table_K > 0) {
    /* P:248 "linear interpolation with the relative distance" (R12) */
    double delta = 2.0 / (double)(p->table_K - 1);
    double q = v / delta;
    int64_t i = (int64_t)floor(q);
    if (i > p->table_K - 2) i = p->table_K - 2;
    return p->table[i] + (p->table[i + 1] - p->table[i]) * (q - (double)i);
  }
  return S_direct(p->n, v);
}

double orc_vdS(const orc_params* p, double v) {
  /* v dS/dv = n sinc^(n-1) (cos x - sinc x), x = pi v / 2 (differentiate Eq. 6;
   * the (pi/2) v / x factor is exactly 1).  Direct in both kernel modes.       */
  if (!(v < 2.0) || v == 0.0) return 0.0;
  double x = 0.5 * M_PI * v;
  double s = sinc(x);
  return p->n * powi_or_pow(s, p->n - 1.0) * (cos(x) - s);
}

double orc_W(const orc_params* p, double r, double h) {
  return p->Bn * orc_S(p, r / h) / (h * h * h);
}

double orc_dWdh(const orc_params* p, double r, double h) {
  /* d/dh [B S(r/h) / h^3] = -B (3 S + v S'(v)) / h^4 */
  double v = r / h;
  return -p->Bn * (3.0 * orc_S(p, v) + orc_vdS(p, v)) / (h * h * h * h);
}

double orc_norm(double n) {
  /* B_n = 1 / (4 pi int_0^2 S(v) v^2 dv)  ("B_n a normalization constant", Eq. 6);
   * composite Simpson, 200000 intervals on a smooth integrand.                 */
  const int M = 200000;
  const double hstep = 2.0 / M;
  double acc = 0.0;
  for (int i = 0; i <= M; ++i) {
    double v = hstep * i;
    double f = S_direct(n, v) * v * v;
    double wgt = (i == 0 || i == M) ? 1.0 : ((i & 1) ? 4.0 : 2.0);
    acc += wgt * f;
  }
  double I = acc * hstep / 3.0;
  return 1.0 / (4.0 * M_PI * I);
}

/* ------------------------------------------------------------------------ */
/* O1 neighbours                                                              */
/* ------------------------------------------------------------------------ */

/* minimum image on periodic dims (periodic z: P:268) */
static void min_image(const orc_params* p, double d[3]) {
  for (int k = 0; k < 3; ++k) {
    if (!p->periodic[k]) continue;
    double L = p->box_hi[k] - p->box_lo[k];
    if (d[k] > 0.5 * L) d[k] -= L;
    else if (d[k] < -0.5 * L) d[k] += L;
  }
}

static void delta_ab(const orc_params* p, const double* x, const double* y, const double* z,
                     int64_t a, int64_t b, double d[3]) {
  /* Delta_ab = x_b - x_a */
  d[0] = x[b] - x[a];
  d[1] = y[b] - y[a];
  d[2] = z[b] - z[a];
  min_image(p, d);
}

static double r2_of(const double d[3]) {
  /* left to right, no FMA (built with -ffp-contract=off) */
  return (d[0] * d[0] + d[1] * d[1]) + d[2] * d[2];
}

/* b is a neighbour of a iff b != a and r^2 < (2 h_a)^2: "v = |x_a - x_b| / h_a"
 * and compact support v <= 2 (Eq. 6), strict (R10).  Symmetric mode:
 * r^2 < (2 max(h_a, h_b))^2, so b in N(a) iff a in N(b); the kernel terms of the
 * extra pairs (r >= 2 h_a) that carry W(r, h_a) vanish by compact support.     */
static int is_neighbor(const orc_params* p, const double* x, const double* y, const double* z,
                       const double* h, int64_t a, int64_t b) {
  if (a == b) return 0;
  double d[3];
  delta_ab(p, x, y, z, a, b, d);
  double tha = 2.0 * h[a];
  if (p->symmetric && h[b] > h[a]) tha = 2.0 * h[b];
  return r2_of(d) < tha * tha;
}

static int cmp_i64(const void* A, const void* B) {
  int64_t a = *(const int64_t*)A, b = *(const int64_t*)B;
  return (a > b) - (a < b);
}

typedef struct {
  int nc[3];
  double lo[3], inv[3];
  int64_t* start; /* ncell+1 */
  int64_t* items; /* N, particles grouped by cell */
} grid_t;

static int64_t cell_coord(const grid_t* g, int k, double v) {
  int64_t c = (int64_t)floor((v - g->lo[k]) * g->inv[k]);
  if (c < 0) c = 0;
  if (c > g->nc[k] - 1) c = g->nc[k] - 1;
  return c;
}

static void grid_build(const orc_params* p, int64_t N, const double* x, const double* y,
                       const double* z, const double* h, grid_t* g) {
  const double* X[3] = {x, y, z};
  double hmax = 0.0;
  for (int64_t i = 0; i < N; ++i) if (h[i] > hmax) hmax = h[i];
  /* cells at least 2 h_max (1 + 2^-20) wide: rounding never drops a pair */
  double cs = 2.0 * hmax * (1.0 + ldexp(1.0, -20));
  for (int k = 0; k < 3; ++k) {
    double lo, ext;
    if (p->periodic[k]) {
      lo = p->box_lo[k];
      ext = p->box_hi[k] - p->box_lo[k];
    } else {
      double mn = X[k][0], mx = X[k][0];
      for (int64_t i = 1; i < N; ++i) {
        if (X[k][i] < mn) mn = X[k][i];
        if (X[k][i] > mx) mx = X[k][i];
      }
      lo = mn;
      ext = mx - mn;
    }
    int nc = (int)floor(ext / cs);
    if (nc < 1) nc = 1;
    if (nc > 1024) nc = 1024;
    g->nc[k] = nc;
    g->lo[k] = lo;
    g->inv[k] = ext > 0.0 ? (double)nc / ext : 0.0;
  }
  int64_t ncell = (int64_t)g->nc[0] * g->nc[1] * g->nc[2];
  g->start = (int64_t*)calloc((size_t)ncell + 1, sizeof(int64_t));
  g->items = (int64_t*)malloc((size_t)(N > 0 ? N : 1) * sizeof(int64_t));
  int64_t* cid = (int64_t*)malloc((size_t)(N > 0 ? N : 1) * sizeof(int64_t));
  for (int64_t i = 0; i < N; ++i) {
    int64_t cx = cell_coord(g, 0, x[i]), cy = cell_coord(g, 1, y[i]), cz = cell_coord(g, 2, z[i]);
    cid[i] = cx + g->nc[0] * (cy + (int64_t)g->nc[1] * cz);
    g->start[cid[i] + 1]++;
  }
  for (int64_t c = 0; c < ncell; ++c) g->start[c + 1] += g->start[c];
  int64_t* fill = (int64_t*)malloc((size_t)ncell * sizeof(int64_t) + 1);
  memcpy(fill, g->start, (size_t)ncell * sizeof(int64_t));
  for (int64_t i = 0; i < N; ++i) g->items[fill[cid[i]]++] = i;
  free(fill);
  free(cid);
}

/* the cells along dim k within one cell of c (wrapping if periodic), each once */
static int stencil_1d(const orc_params* p, const grid_t* g, int k, int64_t c, int64_t out[3]) {
  int nc = g->nc[k];
  if (nc <= 3) {
    for (int i = 0; i < nc; ++i) out[i] = i;
    return nc;
  }
  int n = 0;
  for (int64_t d = -1; d <= 1; ++d) {
    int64_t q = c + d;
    if (p->periodic[k]) {
      q = (q + nc) % nc;
    } else if (q < 0 || q >= nc) {
      continue;
    }
    out[n++] = q;
  }
  return n;
}

typedef struct {
  const orc_params* p;
  const double *x, *y, *z, *h;
  const grid_t* g;
} search_t;

static int64_t search_one(const search_t* s, int method, int64_t N, int64_t a, int64_t* out) {
  int64_t n = 0;
  if (method == 0) {
    for (int64_t b = 0; b < N; ++b)
      if (is_neighbor(s->p, s->x, s->y, s->z, s->h, a, b)) {
        if (out) out[n] = b;
        ++n;
      }
    return n;
  }
  const grid_t* g = s->g;
  int64_t cs[3][3];
  int ns[3];
  int64_t ca[3] = {cell_coord(g, 0, s->x[a]), cell_coord(g, 1, s->y[a]), cell_coord(g, 2, s->z[a])};
  for (int k = 0; k < 3; ++k) ns[k] = stencil_1d(s->p, g, k, ca[k], cs[k]);
  for (int iz = 0; iz < ns[2]; ++iz)
    for (int iy = 0; iy < ns[1]; ++iy)
      for (int ix = 0; ix < ns[0]; ++ix) {
        int64_t c = cs[0][ix] + g->nc[0] * (cs[1][iy] + (int64_t)g->nc[1] * cs[2][iz]);
        for (int64_t q = g->start[c]; q < g->start[c + 1]; ++q) {
          int64_t b = g->items[q];
          if (is_neighbor(s->p, s->x, s->y, s->z, s->h, a, b)) {
            if (out) out[n] = b;
            ++n;
          }
        }
      }
  if (out) qsort(out, (size_t)n, sizeof(int64_t), cmp_i64);
  return n;
}

int64_t orc_neighbors(const orc_params* p, int method, int64_t N, const double* x,
                      const double* y, const double* z, const double* h, int64_t* offsets,
                      int64_t* nbr, int64_t cap) {
  grid_t g;
  memset(&g, 0, sizeof g);
  if (method == 1) grid_build(p, N, x, y, z, h, &g);
  search_t s = {p, x, y, z, h, &g};
  offsets[0] = 0;
#pragma omp parallel for schedule(static)
  for (int64_t a = 0; a < N; ++a) offsets[a + 1] = search_one(&s, method, N, a, NULL);
  for (int64_t a = 0; a < N; ++a) offsets[a + 1] += offsets[a];
  int64_t total = offsets[N];
  if (total <= cap && nbr) {
#pragma omp parallel for schedule(static)
    for (int64_t a = 0; a < N; ++a) search_one(&s, method, N, a, nbr + offsets[a]);
  }
  free(g.start);
  free(g.items);
  return total;
}

/* ------------------------------------------------------------------------ */
/* O3-O5 density, grad-h Omega, EOS                                           */
/* ------------------------------------------------------------------------ */

void orc_density(const orc_params* p, int64_t N, const double* x, const double* y,
                 const double* z, const double* h, const double* m, const double* u,
                 const int64_t* offsets, const int64_t* nbr, double* rho, double* omega,
                 double* P, double* c, double* omega_scale, orc_counters* cnt) {
  int64_t clamped = 0;
#pragma omp parallel for schedule(static) reduction(+ : clamped)
  for (int64_t a = 0; a < N; ++a) {
    double ha = h[a];
    /* Eq. 1: rho_a = sum_b m_b W_ab(h_a), self term included (R11) */
    double r_a = m[a] * orc_W(p, 0.0, ha);
    double dsum = m[a] * orc_dWdh(p, 0.0, ha);
    double dabs = fabs(dsum);
    for (int64_t k = offsets[a]; k < offsets[a + 1]; ++k) {
      int64_t b = nbr[k];
      double d[3];
      delta_ab(p, x, y, z, a, b, d);
      double r = sqrt(r2_of(d));
      r_a += m[b] * orc_W(p, r, ha);
      double t = m[b] * orc_dWdh(p, r, ha);
      dsum += t;
      dabs += fabs(t);
    }
    rho[a] = r_a;
    /* grad-h terms (closure R8): Omega = 1 + h/(3 rho) sum_b m_b dW/dh */
    double om = p->omega_mode ? 1.0 : 1.0 + ha / (3.0 * r_a) * dsum;
    if (om < 0.1) {
      om = 0.1;
      clamped++;
    }
    omega[a] = om;
    if (omega_scale) omega_scale[a] = 1.0 + ha / (3.0 * r_a) * dabs;
    /* EOS (symbols only in P:125; R13) */
    if (p->eos == ORC_EOS_LINEAR) {
      P[a] = p->c0 * p->c0 * (r_a - p->rho0);
      c[a] = p->c0;
    } else {
      P[a] = (p->gamma - 1.0) * r_a * u[a];
      c[a] = sqrt(p->gamma * P[a] / r_a);
    }
  }
  if (cnt) cnt->omega_clamped += clamped;
}

/* ------------------------------------------------------------------------ */
/* O6 IAD ([IAD]): tau_a = sum_b (m_b/rho_b) W_ab(h_a) D D^T, C = tau^-1 */
/* ------------------------------------------------------------------------ */

void orc_iad(const orc_params* p, int64_t N, const double* x, const double* y, const double* z,
             const double* h, const double* m, const double* rho, const int64_t* offsets,
             const int64_t* nbr, double* c11, double* c12, double* c13, double* c22, double* c23,
             double* c33, orc_counters* cnt) {
  int64_t singular = 0;
#pragma omp parallel for schedule(static) reduction(+ : singular)
  for (int64_t a = 0; a < N; ++a) {
    double t11 = 0, t12 = 0, t13 = 0, t22 = 0, t23 = 0, t33 = 0;
    for (int64_t k = offsets[a]; k < offsets[a + 1]; ++k) {
      int64_t b = nbr[k];
      double d[3];
      delta_ab(p, x, y, z, a, b, d);
      double r = sqrt(r2_of(d));
      double w = (m[b] / rho[b]) * orc_W(p, r, h[a]);
      t11 += w * d[0] * d[0];
      t12 += w * d[0] * d[1];
      t13 += w * d[0] * d[2];
      t22 += w * d[1] * d[1];
      t23 += w * d[1] * d[2];
      t33 += w * d[2] * d[2];
    }
    /* cofactor inverse of the symmetric 3x3 tau */
    double det = t11 * (t22 * t33 - t23 * t23) - t12 * (t12 * t33 - t23 * t13) +
                 t13 * (t12 * t23 - t22 * t13);
    double i11 = (t22 * t33 - t23 * t23) / det;
    double i12 = (t13 * t23 - t12 * t33) / det;
    double i13 = (t12 * t23 - t13 * t22) / det;
    double i22 = (t11 * t33 - t13 * t13) / det;
    double i23 = (t12 * t13 - t11 * t23) / det;
    double i33 = (t11 * t22 - t12 * t12) / det;
    double nt = sqrt(t11 * t11 + t22 * t22 + t33 * t33 + 2.0 * (t12 * t12 + t13 * t13 + t23 * t23));
    double ni = sqrt(i11 * i11 + i22 * i22 + i33 * i33 + 2.0 * (i12 * i12 + i13 * i13 + i23 * i23));
    /* reading R29: singular / ill-conditioned tau (det <= 0 or cond_F > 1e12)
     * -> isotropic C = 3/trace(tau) I (0 when trace is 0), counted      */
    if (!(det > 0.0) || !(nt * ni <= 1e12)) {
      double tr = t11 + t22 + t33;
      double s = tr > 0.0 ? 3.0 / tr : 0.0;
      i11 = s; i22 = s; i33 = s;
      i12 = 0.0; i13 = 0.0; i23 = 0.0;
      singular++;
    }
    c11[a] = i11; c12[a] = i12; c13[a] = i13;
    c22[a] = i22; c23[a] = i23; c33[a] = i33;
  }
  if (cnt) cnt->iad_singular += singular;
}

/* ------------------------------------------------------------------------ */
/* O7 momentum + energy + artificial viscosity (Eqs. 2-5)          */
/* ------------------------------------------------------------------------ */

void orc_momentum_energy(const orc_params* p, int64_t N, const double* x, const double* y,
                         const double* z, const double* vx, const double* vy, const double* vz,
                         const double* h, const double* m, const double* rho, const double* omega,
                         const double* P, const double* c, const double* c11, const double* c12,
                         const double* c13, const double* c22, const double* c23,
                         const double* c33, const int64_t* offsets, const int64_t* nbr,
                         double* ax, double* ay, double* az, double* du, double* vsig,
                         double* scale_a, double* scale_du, orc_counters* cnt) {
  int64_t coincident = 0;
#pragma omp parallel for schedule(static) reduction(+ : coincident)
  for (int64_t a = 0; a < N; ++a) {
    /* R1: P_a / (Omega_a rho_a^2) in both Eq. 2 and Eq. 3 */
    double Xa = P[a] / (omega[a] * rho[a] * rho[a]);
    double acc[3] = {0, 0, 0}, dua = 0.0, vs = 0.0;
    double sa[3] = {0, 0, 0}, sdu = 0.0;
    int any = 0;
    for (int64_t k = offsets[a]; k < offsets[a + 1]; ++k) {
      int64_t b = nbr[k];
      double d[3];
      delta_ab(p, x, y, z, a, b, d); /* Delta_ab = x_b - x_a */
      double r2 = r2_of(d);
      if (r2 == 0.0) { /* coincident pair: skipped, counted */
        coincident++;
        continue;
      }
      double r = sqrt(r2);
      double Wa = orc_W(p, r, h[a]);
      double Wb = orc_W(p, r, h[b]);
      /* R5: A_ab(h_a) = C_a Delta_ab W_ab(h_a);  R4: A_ab(h_b) = C_b Delta_ab W_ab(h_b) */
      double Aa[3], Ab[3], Ta[3], Tb[3];
      Aa[0] = (c11[a] * d[0] + c12[a] * d[1] + c13[a] * d[2]) * Wa;
      Aa[1] = (c12[a] * d[0] + c22[a] * d[1] + c23[a] * d[2]) * Wa;
      Aa[2] = (c13[a] * d[0] + c23[a] * d[1] + c33[a] * d[2]) * Wa;
      Ab[0] = (c11[b] * d[0] + c12[b] * d[1] + c13[b] * d[2]) * Wb;
      Ab[1] = (c12[b] * d[0] + c22[b] * d[1] + c23[b] * d[2]) * Wb;
      Ab[2] = (c13[b] * d[0] + c23[b] * d[1] + c33[b] * d[2]) * Wb;
      /* magnitudes for the R27 tolerance scale */
      Ta[0] = (fabs(c11[a] * d[0]) + fabs(c12[a] * d[1]) + fabs(c13[a] * d[2])) * Wa;
      Ta[1] = (fabs(c12[a] * d[0]) + fabs(c22[a] * d[1]) + fabs(c23[a] * d[2])) * Wa;
      Ta[2] = (fabs(c13[a] * d[0]) + fabs(c23[a] * d[1]) + fabs(c33[a] * d[2])) * Wa;
      Tb[0] = (fabs(c11[b] * d[0]) + fabs(c12[b] * d[1]) + fabs(c13[b] * d[2])) * Wb;
      Tb[1] = (fabs(c12[b] * d[0]) + fabs(c22[b] * d[1]) + fabs(c23[b] * d[2])) * Wb;
      Tb[2] = (fabs(c13[b] * d[0]) + fabs(c23[b] * d[1]) + fabs(c33[b] * d[2])) * Wb;
      double Xb = P[b] / (omega[b] * rho[b] * rho[b]);
      /* v_ab = v_a - v_b, x_ab = x_a - x_b = -Delta_ab */
      double vab[3] = {vx[a] - vx[b], vy[a] - vy[b], vz[a] - vz[b]};
      double xab[3] = {-d[0], -d[1], -d[2]};
      double vdotx = vab[0] * xab[0] + vab[1] * xab[1] + vab[2] * xab[2];
      double w = vdotx / r; /* w_ab = v_ab . x_ab / |x_ab| */
      /* Eq. 5, v_sig = c_a + c_b - 3 w_ab */
      double Pi = 0.0;
      if (vdotx < 0.0) Pi = -0.5 * p->alpha * (c[a] + c[b] - 3.0 * w) * w;
      double vsab = c[a] + c[b] - 3.0 * (w < 0.0 ? w : 0.0);
      if (!any || vsab > vs) vs = vsab;
      any = 1;
      /* Eq. 4 pair term g_ab = 1/2 m_b Pi'_ab (A_ab(h_a)/rho_a + A_ab(h_b)/rho_b) */
      double g[3];
      for (int i = 0; i < 3; ++i) g[i] = 0.5 * m[b] * Pi * (Aa[i] / rho[a] + Ab[i] / rho[b]);
      /* Eq. 2 with R2 (AV subtracted) */
      for (int i = 0; i < 3; ++i) acc[i] += -m[b] * (Xa * Aa[i] + Xb * Ab[i]) - g[i];
      /* Eq. 3 with R1 (rho_a^2) and R3 (pairwise AV heating) */
      double vA = vab[0] * Aa[0] + vab[1] * Aa[1] + vab[2] * Aa[2];
      double vg = vab[0] * g[0] + vab[1] * g[1] + vab[2] * g[2];
      dua += m[b] * Xa * vA + 0.5 * vg;
      /* R27 scale: sum over pairs of |each summand| with an AV bound that covers
       * a round-off decided branch (R28)                                      */
      double wt = (fabs(vab[0] * xab[0]) + fabs(vab[1] * xab[1]) + fabs(vab[2] * xab[2])) / r;
      double Pt = 0.5 * p->alpha * (c[a] + c[b] + 3.0 * wt) * wt;
      double gt[3];
      for (int i = 0; i < 3; ++i) {
        gt[i] = 0.5 * m[b] * Pt * (Ta[i] / rho[a] + Tb[i] / rho[b]);
        sa[i] += m[b] * (fabs(Xa) * Ta[i] + fabs(Xb) * Tb[i]) + gt[i];
      }
      sdu += m[b] * fabs(Xa) * (fabs(vab[0]) * Ta[0] + fabs(vab[1]) * Ta[1] + fabs(vab[2]) * Ta[2]) +
             0.5 * (fabs(vab[0]) * gt[0] + fabs(vab[1]) * gt[1] + fabs(vab[2]) * gt[2]);
    }
    if (!any) vs = 2.0 * c[a]; /* no interacting neighbour */
    ax[a] = acc[0];
    ay[a] = acc[1];
    az[a] = acc[2];
    du[a] = dua;
    vsig[a] = vs;
    if (scale_a) {
      scale_a[a] = sa[0];
      scale_a[N + a] = sa[1];
      scale_a[2 * N + a] = sa[2];
    }
    if (scale_du) scale_du[a] = sdu;
  }
  if (cnt) cnt->coincident_pairs += coincident;
}

/* ------------------------------------------------------------------------ */
/* O8 dt = min(C_cour min_a h_a / vsig_a, growth dt_prev)  (R19)       */
/* ------------------------------------------------------------------------ */

double orc_timestep(const orc_params* p, int64_t N, const double* h, const double* vsig,
                    double dt_prev, int first) {
  double dt = INFINITY;
  for (int64_t a = 0; a < N; ++a) {
    double t = p->courant * h[a] / vsig[a];
    if (t < dt) dt = t;
  }
  if (!first && p->dt_growth * dt_prev < dt) dt = p->dt_growth * dt_prev;
  return dt;
}

/* ------------------------------------------------------------------------ */
/* O9 update: Press/Stormer on mid-step velocities (R17), AB2 u (R18)  */
/* ------------------------------------------------------------------------ */

void orc_update(const orc_params* p, int64_t N, double dt, double dt_prev, int first,
                double* x, double* y, double* z, double* vx, double* vy, double* vz,
                double* vhx, double* vhy, double* vhz, const double* ax, const double* ay,
                const double* az, double* u, const double* du, double* du_prev,
                orc_counters* cnt) {
  if (first) dt_prev = dt;
  double q = dt / dt_prev;
  int64_t floored = 0;
#pragma omp parallel for schedule(static) reduction(+ : floored)
  for (int64_t a = 0; a < N; ++a) {
    double* X[3] = {x, y, z};
    double* V[3] = {vx, vy, vz};
    double* VH[3] = {vhx, vhy, vhz};
    const double* A[3] = {ax, ay, az};
    for (int k = 0; k < 3; ++k) {
      /* first step: vbar := v - a dt / 2 (so the kick below gives v + a dt / 2) */
      double vb = first ? V[k][a] - 0.5 * A[k][a] * dt : VH[k][a];
      vb = vb + A[k][a] * (dt_prev + dt) * 0.5; /* kick to t + dt/2 */
      double xn = X[k][a] + dt * vb;            /* drift */
      if (p->periodic[k]) {
        double L = p->box_hi[k] - p->box_lo[k];
        if (xn >= p->box_hi[k]) xn -= L;
        else if (xn < p->box_lo[k]) xn += L;
        /* reading R30: the wrapped coordinate stays in [lo, hi) when the wrap rounds
         * onto an end (x = -1e-15 in [0, 100) wraps to 100.0 exactly)                */
        if (xn < p->box_lo[k]) xn = p->box_lo[k];
        if (xn >= p->box_hi[k]) xn = nextafter(p->box_hi[k], p->box_lo[k]);
      }
      X[k][a] = xn;
      VH[k][a] = vb;
      V[k][a] = vb + 0.5 * A[k][a] * dt; /* synchronised velocity */
    }
    /* variable-step AB2, Euler bootstrap (du_prev := du on the first step) */
    double dp = first ? du[a] : du_prev[a];
    double un = u[a] + dt * ((1.0 + 0.5 * q) * du[a] - 0.5 * q * dp);
    if (un < p->u_floor) {
      un = p->u_floor;
      floored++;
    }
    u[a] = un;
    du_prev[a] = du[a];
  }
  if (cnt) cnt->u_floored += floored;
}

/* ------------------------------------------------------------------------ */
/* O10 h <- h (1 + (n_target / max(n,1))^(1/3)) / 2   (R20)     */
/* ------------------------------------------------------------------------ */

void orc_update_h(const orc_params* p, int64_t N, double* h, const int64_t* offsets,
                  orc_counters* cnt) {
  int64_t clamped = 0;
#pragma omp parallel for schedule(static) reduction(+ : clamped)
  for (int64_t a = 0; a < N; ++a) {
    int64_t n = offsets[a + 1] - offsets[a];
    double nn = (double)(n > 1 ? n : 1);
    double hn = h[a] * 0.5 * (1.0 + cbrt(p->n_target / nn));
    if (hn < p->h_min) {
      hn = p->h_min;
      clamped++;
    }
    if (p->h_max > 0.0 && hn > p->h_max) {
      hn = p->h_max;
      clamped++;
    }
    h[a] = hn;
  }
  if (cnt) cnt->h_clamped += clamped;
}

/* ------------------------------------------------------------------------ */
/* O11 conserved quantities, fixed-order pairwise sums                */
/* ------------------------------------------------------------------------ */

static double pairwise(const double* v, int64_t n) {
  if (n <= 8) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += v[i];
    return s;
  }
  int64_t h = n / 2;
  return pairwise(v, h) + pairwise(v + h, n - h);
}

void orc_diagnostics(int64_t N, const double* m, const double* x, const double* y,
                     const double* z, const double* vx, const double* vy, const double* vz,
                     const double* u, double* out) {
  double* t = (double*)malloc((size_t)(N > 0 ? N : 1) * sizeof(double));
  for (int q = 0; q < 7; ++q) {
    for (int64_t a = 0; a < N; ++a) {
      double v;
      switch (q) {
        case 0: v = m[a] * vx[a]; break;
        case 1: v = m[a] * vy[a]; break;
        case 2: v = m[a] * vz[a]; break;
        case 3: v = m[a] * (y[a] * vz[a] - z[a] * vy[a]); break;
        case 4: v = m[a] * (z[a] * vx[a] - x[a] * vz[a]); break;
        case 5: v = m[a] * (x[a] * vy[a] - y[a] * vx[a]); break;
        default:
          v = m[a] * (u[a] + 0.5 * (vx[a] * vx[a] + vy[a] * vy[a] + vz[a] * vz[a]));
      }
      t[a] = v;
    }
    out[q] = pairwise(t, N);
  }
  free(t);
}
