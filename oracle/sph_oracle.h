/* oracle/sph_oracle.h -- plain, slow, fp64 CPU oracle of the SPH-EXA hot path
 * (Cavelan et al., arXiv 2005.02656, §4.1).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  It
 * shares no code, header, table or constant generator with the CUDA path
 * (paper_2005_02656_b200/csrc) and neither side includes the other.
 *
 * Conventions: all arrays are HOST arrays of length N (SoA, fp64 unless
 * noted), indexed by particle position 0..N-1.  Neighbour lists are CSR:
 * offsets[N+1] (int64) and nbr[offsets[N]] (int64 particle positions, each
 * row sorted ascending).  Every pair sum runs in that ascending order.
 * Build: gcc -O2 -fopenmp -ffp-contract=off -fno-fast-math (no FMA contraction,
 * so r^2 is evaluated exactly as written -- the neighbour test is bit-exact).
 */
#ifndef SPH_ORACLE_H
#define SPH_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_EOS_LINEAR = 0, ORC_EOS_IDEAL = 1 };

typedef struct {
  double n;            /* sinc exponent (reading R9: 6)                        */
  double Bn;           /* normalisation; orc_norm(n)                          */
  int    table_K;      /* 0: direct sin; K>0: K-sample table (R12)      */
  const double* table; /* K samples from orc_table_build (owned by caller)     */
  double alpha;        /* AV strength (R7: 1.0)                                */
  int    eos;          /* ORC_EOS_LINEAR (R13) | ORC_EOS_IDEAL                  */
  double c0, rho0, gamma;
  int    omega_mode;   /* 0: grad-h closure (R8); 1: Omega == 1                */
  double courant;      /* 0.3 (R19)                                            */
  double dt_growth;    /* 1.1 (R19)                                            */
  double n_target;     /* 300 (R20)                                     */
  double h_min, h_max; /* h clamp after update; h_max <= 0 means none          */
  double u_floor;      /* u clamp after update                                 */
  double box_lo[3], box_hi[3];
  int    periodic[3];  /* square patch: {0,0,1}                        */
  int    symmetric;    /* 0: N(a) = {r < 2 h_a} (gather, R10); 1: r < 2 max(h_a, h_b)
                          (pairwise-antisymmetric forces, exact
                          conservation for variable h; closes reading R24)      */
} orc_params;

typedef struct {
  int64_t omega_clamped, iad_singular, coincident_pairs, u_floored, h_clamped;
} orc_counters;

/* ---- kernel, Eq. 6 ---- */
double  orc_norm(double n);                                  /* B_n, 3D        */
void    orc_table_build(double n, int K, double* table);     /* T_k = S(2k/(K-1)) */
double  orc_S(const orc_params* p, double v);                /* [sinc(pi v/2)]^n, v<2 */
double  orc_vdS(const orc_params* p, double v);              /* v * dS/dv       */
double  orc_W(const orc_params* p, double r, double h);      /* B S(r/h)/h^3    */
double  orc_dWdh(const orc_params* p, double r, double h);   /* dW/dh           */

/* ---- O1 neighbours: {b != a : r_ab^2 < (2 h_a)^2}, min image on periodic dims.
 * method 0 = brute force O(N^2), 1 = uniform grid.  Returns the number of
 * pairs; fills nbr only when that number <= cap (call again with room). ---- */
int64_t orc_neighbors(const orc_params* p, int method, int64_t N,
                      const double* x, const double* y, const double* z, const double* h,
                      int64_t* offsets, int64_t* nbr, int64_t cap);

/* ---- O3-O5 density + Omega + EOS (Eq. 1) ---- */
void orc_density(const orc_params* p, int64_t N,
                 const double* x, const double* y, const double* z, const double* h,
                 const double* m, const double* u, const int64_t* offsets, const int64_t* nbr,
                 double* rho, double* omega, double* P, double* c, double* omega_scale,
                 orc_counters* cnt);

/* ---- O6 IAD: tau, C = tau^-1 -- C6 = {c11,c12,c13,c22,c23,c33} each [N] ---- */
void orc_iad(const orc_params* p, int64_t N,
             const double* x, const double* y, const double* z, const double* h,
             const double* m, const double* rho, const int64_t* offsets, const int64_t* nbr,
             double* c11, double* c12, double* c13, double* c22, double* c23, double* c33,
             orc_counters* cnt);

/* ---- O7 momentum + energy + AV (Eqs. 2-5, readings R1-R5).
 * scale_a[3N] (component-major) and scale_du[N] hold sum_b |summand| (R27). ---- */
void orc_momentum_energy(const orc_params* p, int64_t N,
                         const double* x, const double* y, const double* z,
                         const double* vx, const double* vy, const double* vz,
                         const double* h, const double* m, const double* rho,
                         const double* omega, const double* P, const double* c,
                         const double* c11, const double* c12, const double* c13,
                         const double* c22, const double* c23, const double* c33,
                         const int64_t* offsets, const int64_t* nbr,
                         double* ax, double* ay, double* az, double* du, double* vsig,
                         double* scale_a, double* scale_du, orc_counters* cnt);

/* ---- O8 global min dt (R19) ---- */
double orc_timestep(const orc_params* p, int64_t N, const double* h, const double* vsig,
                    double dt_prev, int first);

/* ---- O9 update: Press/Stormer x,v (R17) + variable-step AB2 u (R18) ---- */
void orc_update(const orc_params* p, int64_t N, double dt, double dt_prev, int first,
                double* x, double* y, double* z, double* vx, double* vy, double* vz,
                double* vhx, double* vhy, double* vhz,
                const double* ax, const double* ay, const double* az,
                double* u, const double* du, double* du_prev, orc_counters* cnt);

/* ---- O10 smoothing length (R20) ---- */
void orc_update_h(const orc_params* p, int64_t N, double* h, const int64_t* offsets,
                  orc_counters* cnt);

/* ---- O11 conserved sums: out = {px,py,pz, Lx,Ly,Lz, E} ---- */
void orc_diagnostics(int64_t N, const double* m, const double* x, const double* y,
                     const double* z, const double* vx, const double* vy, const double* vz,
                     const double* u, double* out);

#ifdef __cplusplus
}
#endif
#endif
