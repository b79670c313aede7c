/* include/sph.h -- C ABI of the B200-native SPH-EXA timestep (arXiv 2005.02656).
 *
 * One call per step of the paper's per-timestep loop (Fig. 1 caption
 * P:103, Fig. 2 prose P:180-182, §4.1):
 *
 *   sph_find_neighbors   SFC (Morton) sort + cell tables + neighbour lists   (a1-a5)
 *   sph_density          rho (Eq. 1), grad-h Omega, EOS       (a6)
 *   sph_iad              IAD matrix C = tau^-1 ([IAD])                 (a8)
 *   sph_momentum_energy  Eqs. 2-5 + per-particle v_sig + global min dt (a10-a11)
 *   sph_advance          Press/Stormer x,v + AB2 u + smoothing-length update (a12-a13)
 *   sph_step             all of the above, in that order                      (a1-a13)
 *
 * Physics readings (R1-R29) are listed in DESIGN.md §3.
 *
 * Memory & ownership.
 *  - Particle arrays are DEVICE pointers owned by the caller (PyTorch), SoA,
 *    fp64 unless noted, each at least `capacity` elements.  The library borrows
 *    them between sph_attach and sph_destroy and never frees them.
 *  - sph_find_neighbors / sph_step PERMUTE the state arrays in place into
 *    Morton-cell order ("kept in memory in an order that matches
 *    the octree"); `id` travels with the particles so the caller can map back.
 *  - All scratch (sort buffers, cell tables, neighbour lists, per-particle
 *    auxiliaries) is owned by the library, allocated in sph_init for `capacity`
 *    particles, freed in sph_destroy.
 *  - Calls are stream-ordered on params.stream (a cudaStream_t, NULL = legacy
 *    default stream).  sph_find_neighbors synchronises the stream once (grid
 *    geometry and neighbour-list overflow check); sph_momentum_energy and
 *    sph_step synchronise only when dt_out != NULL.
 *
 * Errors.  No call aborts or exits.  Every call returns an sph_status; a
 * non-OK status is sticky on the context (later calls return it too) and
 * sph_error_string() describes it.  Numerical guards (Omega clamp, singular
 * IAD matrix, coincident pairs, u floor, h clamp) are counted, not fatal, and
 * reported by sph_diagnostics.
 */
#ifndef SPH_B200_H
#define SPH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPH_ABI_VERSION 6

typedef struct sph_ctx sph_ctx;

typedef enum {
  SPH_OK = 0,
  SPH_ERR_NUMERIC = 1,   /* non-finite dt / state (SPEC exit code 1)               */
  SPH_ERR_CONFIG = 2,    /* invalid parameter (SPEC exit code 2)                    */
  SPH_ERR_CAPACITY = 3,  /* n > capacity, or a neighbour row > max_neighbors       */
  SPH_ERR_CUDA = 4,      /* CUDA runtime error (message has the CUDA string)        */
  SPH_ERR_COMM = 5,      /* NCCL error                                              */
  SPH_ERR_STATE = 6      /* call out of order (find -> density -> iad -> momentum)  */
} sph_status;

enum { SPH_EOS_LINEAR = 0, SPH_EOS_IDEAL = 1 };

/* How the kernel value S_n(v) = [sinc(pi v / 2)]^n of Eq. 6 is evaluated in the
 * pair passes.  Every mode is exact to its own
 * definition; the grad-h derivative term of Omega uses the exact polynomial in all
 * modes (the oracle evaluates it directly in all modes, reading R12).             */
enum {
  SPH_KERNEL_POLY = 0,   /* default: degree-8 polynomial of sinc in t = v^2 on [0,4] (no sqrt;
                          |error| <= 5e-14 on sinc, 3e-13 on sinc^6)                      */
  SPH_KERNEL_TABLE = 1,  /* the paper's table: table_size samples of S_n on [0, 2] incl. both
                            ends, index floor(v (K-1)/2), linear interpolation (R12)  */
  SPH_KERNEL_SIN = 2     /* direct: sin(x)/x, x = pi v / 2, raised to n                      */
};

typedef struct {
  int    abi_version;     /* must equal SPH_ABI_VERSION                                  */
  double sinc_n;          /* kernel exponent n of Eq. 6; integer 3..9 (reading R9: 6)     */
  double alpha_av;        /* AV alpha of Eq. 5 (R7: 1.0); beta = 3 via v_sig      */
  int    eos;             /* SPH_EOS_LINEAR: P = c0^2 (rho - rho0), c = c0 (R13)          */
                          /* SPH_EOS_IDEAL:  P = (gamma-1) rho u, c = sqrt(gamma P / rho) */
  double c0, rho0, gamma;
  int    omega_mode;      /* 0: grad-h Omega (R8); 1: Omega == 1                          */
  double courant;         /* dt = courant min_a h_a / vsig_a (R19: 0.3)                   */
  double dt_growth;       /* dt <= dt_growth * dt_prev (R19: 1.1)                         */
  double n_target;        /* neighbour target of the h update (300)                */
  double h_min, h_max;    /* h clamp after the update; h_max <= 0: no upper clamp        */
  double u_floor;         /* u clamp after the update                                     */
  int    max_neighbors;   /* hard limit on neighbours per particle: more -> SPH_ERR_CAPACITY.  */
                          /* 0: no limit -- the library sizes the rows (384 entries, grown */
                          /* on demand; never truncated, R23)                              */
  double cell_factor;     /* search-cell edge = cell_factor * 2 * mean(h) (0: 1.0)        */
  double box_lo[3], box_hi[3]; /* periodic dims: the period is box_hi - box_lo            */
  int    periodic[3];     /* square patch: {0,0,1}                               */
  int    rank, nranks;    /* multi-GPU: this rank / number of ranks (1 for one GPU; <= 64) */
  const void* nccl_unique_id; /* 128-byte ncclUniqueId (rank 0's), NULL when nranks == 1  */
  void*  stream;          /* cudaStream_t                                                 */
  int    kernel_mode;     /* SPH_KERNEL_* (0: polynomial)                                 */
  int    table_size;      /* samples K of SPH_KERNEL_TABLE (0: 20,000 as in P:248); >= 2  */
  int    symmetric;       /* 0: N(a) = {b : r < 2 h_a} (gather, R10);                     */
                          /* 1: r < 2 max(h_a, h_b) -- b in N(a) iff a in N(b), pair forces */
                          /* antisymmetric, exact conservation for variable h (closes R24) */
  int    redecomp_every;  /* multi-GPU: recompute the key-prefix histogram + splitters    */
                          /* every k-th step only (the top tree changes slowly;    */
                          /* SURVEY 8(f) NEXT-3); migration still runs every step against */
                          /* the kept splitters.  0 or 1: every step.  Ignored on 1 GPU.  */
} sph_params;

typedef struct {          /* caller-owned DEVICE buffers, each >= capacity elements       */
  int64_t n;              /* particles currently held (in)                                */
  int64_t capacity;
  int64_t* id;            /* global particle id (travels with the sort)                   */
  double *x, *y, *z, *vx, *vy, *vz, *h, *m, *u;   /* state (in/out)                       */
  double *rho, *omega, *p, *c;                   /* sph_density (out)                     */
  double *c11, *c12, *c13, *c22, *c23, *c33;     /* sph_iad (out)                         */
  double *ax, *ay, *az, *du, *vsig;              /* sph_momentum_energy (out)             */
  double *vhx, *vhy, *vhz, *du_prev;             /* integrator history: mid-step velocity  */
                                                 /* v-bar and previous du (in/out)        */
} sph_particles;

typedef struct {
  int64_t n_owned, n_halo, nbr_total, nbr_max;
  int64_t omega_clamped, iad_singular, coincident_pairs, u_floored, h_clamped;
  int64_t steps;
  int64_t first_bad_id;   /* smallest id with a non-finite / non-positive x, h, m or update,
                             -1 if none; the call that found it returned SPH_ERR_NUMERIC     */
  double  dt, dt_prev, time;
  double  momentum[3], ang_momentum[3], energy;   /* sum m v, sum m x x v, sum m (u + v^2/2) */
  int     grid[3];                                /* search cells per dimension             */
} sph_diag;

/* per-phase device time, accumulated while profiling is on (sph_set_profiling) */
enum {
  SPH_PH_BBOX = 0, SPH_PH_KEYS, SPH_PH_SORT, SPH_PH_PERMUTE, SPH_PH_CELLS, SPH_PH_NEIGHBORS,
  SPH_PH_DENSITY, SPH_PH_IAD, SPH_PH_MOMENTUM, SPH_PH_UPDATE, SPH_PH_HALO,
  SPH_PH_RECORDS,  /* momentum source records (144 B/particle) built before the momentum pass */
  SPH_PH_COUNT
};

int         sph_abi_version(void);
/* The polynomial SPH_KERNEL_POLY evaluates in place of sinc(pi v / 2) of Eq. 6 (the
 * paper's lookup table): P(t) = sum_k coef[k] t^k, t = v^2 in
 * [0, 4].  Writes min(cap, n) coefficients to the HOST array coef (may be NULL when
 * cap = 0) and returns n.  Pure host computation: no context or device needed. */
int         sph_poly_coefficients(double* coef, int cap);
/* Create a context: validates params, computes B_n, allocates scratch for `capacity`
 * particles.  *out is NULL on error (the status says why). */
sph_status  sph_init(const sph_params* params, int64_t capacity, sph_ctx** out);
/* Borrow the caller's particle buffers (DEVICE pointers).  Resets the integrator
 * (the next sph_advance is a first step: v-bar := v - a dt/2, du_prev := du). */
sph_status  sph_attach(sph_ctx* ctx, const sph_particles* particles);
/* a1-a5: bbox, Morton keys, radix sort, in-place permutation, cell tables, neighbour
 * lists N(a) = {b != a : |x_a - x_b|^2 < (2 h_a)^2} (Eq. 6 support; R10). */
sph_status  sph_find_neighbors(sph_ctx* ctx);
/* Host copy of the lists as CSR over the CURRENT particle order: offsets[n+1] and the
 * neighbours' global ids (rows in the device order).  Needs cap >= total pairs; returns
 * SPH_ERR_CAPACITY (and offsets) otherwise.  Synchronises. */
sph_status  sph_get_neighbors(sph_ctx* ctx, int64_t* offsets, int64_t* ids, int64_t cap);
sph_status  sph_density(sph_ctx* ctx);                          /* a6            */
sph_status  sph_iad(sph_ctx* ctx);                              /* a8            */
/* a10-a11; when dt_out != NULL the new dt is copied to the host (synchronises). */
sph_status  sph_momentum_energy(sph_ctx* ctx, double* dt_out);
sph_status  sph_advance(sph_ctx* ctx);                          /* a12-a13       */
sph_status  sph_step(sph_ctx* ctx, double* dt_out);             /* a1-a13        */
/* Copy the state fields (id, x..u, vhx..du_prev) between HOST arrays laid out like
 * sph_particles (host pointers; pinned for speed) and the attached device buffers.
 * sph_upload also sets n.  Both are stream-ordered; sph_download synchronises. */
sph_status  sph_upload(sph_ctx* ctx, const sph_particles* host);
sph_status  sph_download(sph_ctx* ctx, sph_particles* host);
/* Particles currently owned by this rank (== the attached arrays' valid prefix; it changes
 * when particles migrate between ranks) and halo particles held during the current step. */
sph_status  sph_local_count(const sph_ctx* ctx, int64_t* n_owned, int64_t* n_halo);
/* Device memory the library holds for this context (scratch, neighbour rows, multi-GPU
 * buffers), in bytes; the caller's particle arrays are not included. */
sph_status  sph_memory_bytes(const sph_ctx* ctx, int64_t* bytes);
/* Conserved sums and counters ("tracking total momentum and energy"), summed over all
 * ranks when nranks > 1 (n_owned is then the global particle count).  Synchronises. */
sph_status  sph_diagnostics(sph_ctx* ctx, sph_diag* out);
/* Phase timing: on != 0 records CUDA events around every phase; ms_out[SPH_PH_COUNT]
 * receives the accumulated milliseconds and launch counts since the last reset. */
sph_status  sph_set_profiling(sph_ctx* ctx, int on);
sph_status  sph_phase_times(sph_ctx* ctx, double* ms_out, int64_t* launches_out, int reset);
const char* sph_error_string(const sph_ctx* ctx);
sph_status  sph_destroy(sph_ctx* ctx);
/* Multi-GPU bootstrap: write rank 0's 128-byte ncclUniqueId to out (host memory, size >= 128).
 * The caller broadcasts it (e.g. torch.distributed) and passes it as params.nccl_unique_id
 * to sph_init on every rank (one process per GPU).  SPH_ERR_CONFIG if built without NCCL. */
sph_status  sph_nccl_unique_id(void* out, int size);
/* In-process transport (testing and single-GPU runs of the multi-rank path): create a hub
 * for `nranks` ranks and write its 128-byte id to out (host memory, size >= 128).  Passing
 * that id as params.nccl_unique_id makes every sph_init of the same process join the hub
 * instead of NCCL; each rank is then driven by its own host thread (the collectives are
 * blocking rendezvous of those threads; data moves by device-to-device copies).  The
 * decomposition, migration, halo plan and the three exchanges run exactly as over NCCL,
 * so G ranks on one GPU reproduce the NCCL run.  SPH_ERR_CONFIG on bad arguments. */
sph_status  sph_local_comm_id(int nranks, void* out, int size);
/* Host-side decomposition helpers (no GPU needed; used by the library and by CPU tests).
 * splitters: rank r owns key-prefix bins [split[r], split[r+1]) of a global histogram
 * hist[nbins], split[G+1] at equal particle counts (the paper's global tree + bucket rule,
 * P:194-197).  owner: the rank owning a bin. */
int         sph_decomp_splitters(const int64_t* hist, int64_t nbins, int G, int64_t* split);
int         sph_decomp_owner(const int64_t* split, int G, int64_t bin);
/* Utility (not a step of the method): measured FP64 DFMA throughput of this GPU in
 * TFLOP/s (FMA = 2 flops), the roofline denominator of the FP64-bound pair passes.
 * Launches on `stream` (a cudaStream_t) and synchronises it. */
sph_status  sph_measure_fp64_peak(void* stream, double* tflops);

#ifdef __cplusplus
}
#endif
#endif
