// sph_internal.cuh -- shared definitions of the CUDA path (sm_100a).
//
// Layout in HBM: every per-particle quantity is its own fp64
// array (SoA) in Morton-cell order; neighbour lists are rows of flat staging
// indices into the target's unit stencil (16-bit, or 32-bit when a unit stencil
// exceeds 65,535 particles), fixed stride `maxn_cap` (pairpass.cuh); the search grid
// is a dense table of cell ranges
// [cell_start, cell_end) into the sorted order.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/sph.h"

namespace sphb {

#ifndef SPH_POLY_TERMS
#define SPH_POLY_TERMS 9
#endif
constexpr int kPolyTerms = SPH_POLY_TERMS;  // degree-8 polynomial of sinc(pi sqrt(t) / 2) in t = v^2 on [0, 4]
constexpr int kCounters = 8;     // device event counters (see enum below)
enum { CNT_OMEGA = 0, CNT_IAD_SINGULAR, CNT_COINCIDENT, CNT_U_FLOOR, CNT_H_CLAMP, CNT_NONFINITE };

// Search grid (a3).  Identical formula on every rank (derived from the global bbox).
struct Grid {
  double lo[3];     // origin of cell 0 per dim
  double inv[3];    // cells per unit length (nc / extent); 0 when nc == 1 and extent == 0
  double L[3];      // period of periodic dims (box_hi - box_lo)
  int nc[3];        // cells per dim
  int periodic[3];
  int cbits;        // Morton bits per dim
  int idbits;       // id bits at the bottom of the sort key
  int sbits;        // sub-cell Morton bits per dim between the cell code and the id
  int kshift;       // idbits + 3 sbits: key >> kshift = Morton code of the cell
  double hsym;      // symmetric relation: global h_max (every stencil reaches 2 max h); else 0
  int ubits;        // pair-pass units: the cells sharing Morton code >> ubits (stencil.cuh)
  int64_t ncell;
};

// Physics constants by value (kernel parameter space = constant bank).
struct Phys {
  double B;                 // B_n of Eq. 6
  double poly[kPolyTerms];  // P(t) = sum_k poly[k] t^k = sinc(pi sqrt(t) / 2)
  double dpoly[kPolyTerms]; // P'(t)
  int n;                    // integer kernel exponent
  int kmode;                // SPH_KERNEL_* (sph.h)
  int sym;                  // symmetric neighbour relation (sph_params.symmetric)
  int tableK;               // samples of the SPH_KERNEL_TABLE table
  const double* table;      // device table T_k = S_n(2k/(K-1)) (SPH_KERNEL_TABLE), else null
  int eos, omega_mode;
  double alpha, c0, rho0, gamma, courant, dt_growth, n_target, h_min, h_max, u_floor;
  double L[3];
  int periodic[3];
  double box_lo[3], box_hi[3];
};

// Device-side scalars of the integrator: written by kernels, read by kernels.
enum { DT_RAW_BITS = 0, DT_CUR = 1, DT_PREV = 2, DT_COMMITTED = 3, DT_TIME = 4, DT_BAD = 5, DT_SLOTS = 8 };

struct Scratch {
  // sort
  double* ktable = nullptr;      // SPH_KERNEL_TABLE samples
  uint64_t* keys = nullptr;
  uint64_t* keys_alt = nullptr;
  uint32_t* idx = nullptr;
  uint32_t* idx_alt = nullptr;
  uint32_t* hist = nullptr;      // 256 * nblk
  uint32_t* scan_tmp = nullptr;  // block sums for the scan
  double* gather = nullptr;      // 13 * cap doubles (permutation staging)
  int64_t* gather_id = nullptr;  // cap
  // cells
  uint32_t* cell_start = nullptr;
  uint32_t* cell_end = nullptr;
  unsigned long long* cell_hmax = nullptr;  // bit pattern of max h in the cell (h > 0)
  uint32_t* cell_flag = nullptr;            // cap: 1 at the first particle of a cell
  uint32_t* cell_rank = nullptr;            // cap: exclusive scan of cell_flag
  uint32_t* cell_list = nullptr;            // non-empty cells in Morton order
  uint32_t* ncell_list = nullptr;           // device scalar
  uint32_t* unit_flag = nullptr;            // cap: 1 at the first particle of a unit
  uint32_t* unit_rank = nullptr;            // cap: exclusive scan of unit_flag
  uint32_t* unit_list = nullptr;            // cap + 1: index into cell_list of each unit's first cell
  uint32_t* nunit_list = nullptr;           // device scalar
  int4* unit_rec = nullptr;                 // 3 x cap: per unit, its union stencil + target range
  // multi-GPU overlap: units ordered interior first (stencil without halo cells), then boundary
  uint32_t* unit_iflag = nullptr;           // cap: 1 for an interior unit (scan input)
  uint32_t* unit_iexcl = nullptr;           // cap: exclusive scan of unit_iflag
  uint32_t* unit_order = nullptr;           // cap: unit ids, interior then boundary
  uint32_t* unit_bounds = nullptr;          // {0, interior count, unit count}
  int64_t max_cells = 0;
  // neighbours
  unsigned char* nbr = nullptr;  // cap * maxn_cap row entries (uint16_t, or uint32_t when wide_rows)
  uint32_t* ncount = nullptr;    // cap: neighbours per target
  uint32_t* nseg = nullptr;      // cap: search segments per target (before the in-place expansion)
  unsigned int* nbr_max = nullptr;  // [0] largest count, [1] a unit too large for 16 bits, [2] segment overflow
  uint32_t* work = nullptr;              // 8 claim counters: search, density, iad, momentum (+ boundary launches)
  // per-particle auxiliaries written by density, read by iad / momentum
  double* wB = nullptr;    // B / h^3
  double* ih2 = nullptr;   // 1 / h^2
  double* vol = nullptr;   // m / rho
  double* rinv = nullptr;  // 1 / rho
  double* X = nullptr;     // P / (Omega rho^2)   (reading R1)
  double* mX = nullptr;    // m P / (Omega rho^2)
  double* ct = nullptr;    // 6 x cap: (B/h^3) C, written by IAD (and exchanged as halo #3)
  double* mrec = nullptr;  // 18 x cap: momentum source records (144 B each), bulk-copied into smem
  // reductions
  double* red = nullptr;   // block partials
  double* bbox = nullptr;  // 8 doubles (device)
  double* dts = nullptr;   // DT_SLOTS
  unsigned long long* cnt = nullptr;  // kCounters
  unsigned long long* bad_id = nullptr;  // smallest id with a non-finite / non-positive state (~0: none)
  double* diag = nullptr;  // 8
};

struct PhaseEv {
  int ph;
  cudaEvent_t a, b;
};

struct Dist;  // multi-GPU state (sph_dist.cuh)

}  // namespace sphb

struct sph_ctx {
  sph_params prm;
  cudaStream_t stream = nullptr;
  int64_t cap = 0;
  int maxn = 0;             // user limit on neighbours per particle (0: none)
  int maxn_cap = 384;       // row stride (grows on demand up to the user limit)
  bool wide_rows = false;   // 32-bit row entries
  int maxn_cap_alloc = 0;   // the stride / width the row buffer was allocated for
  bool wide_rows_alloc = false;
  size_t mem_bytes = 0;     // device memory the library allocated (sph_memory_bytes)
  sph_particles P{};
  bool attached = false;
  int stage = 0;            // 0 none, 1 neighbours, 2 density, 3 iad, 4 momentum
  bool first = true;        // next advance is the integrator's first step
  int64_t steps = 0;
  sphb::Grid grid{};
  sphb::Phys phys{};
  sphb::Scratch s;
  int nblk_red = 0;
  int num_sms = 148;
  int64_t nbr_total = 0;
  double hmax = 0.0;        // global max h of the current step (grid geometry)
  int64_t nbr_max = 0;
  sph_status status = SPH_OK;
  int64_t first_bad_id = -1;  // sph_diag.first_bad_id
  int unit_sel = 0;           // pass launches: 0 all units, 1 interior, 2 boundary (multi-GPU overlap)
  int64_t n_global = 0;       // particles over all ranks in the current step
  std::string err;
  // profiling
  bool prof = false;
  std::vector<sphb::PhaseEv> pending;
  double phase_ms[SPH_PH_COUNT] = {0};
  int64_t phase_launches[SPH_PH_COUNT] = {0};
  int64_t launches = 0;
  // multi-GPU (nranks > 1): owned particles are [0, P.n), halos [P.n, P.n + n_halo)
  sphb::Dist* dist = nullptr;
  int64_t n_halo = 0;
  std::string dist_err;
};

namespace sphb {

// ---- launchers (each returns the number of kernels it launched) ----
int launch_bbox(sph_ctx* c);
int launch_keys(sph_ctx* c);
int launch_keys_range(sph_ctx* c, int64_t i0, int64_t n);
int launch_cells_halo(sph_ctx* c, int64_t i0, int64_t n);
int scan_u32(sph_ctx* c, const uint32_t* in, uint32_t* out, int64_t n);
int launch_sort(sph_ctx* c, int nbits, const uint32_t** perm_out);
int launch_permute(sph_ctx* c, const uint32_t* perm);
int launch_cells(sph_ctx* c);
int launch_unit_prep(sph_ctx* c);
int launch_search(sph_ctx* c);
int launch_expand_rows(sph_ctx* c);
int launch_density(sph_ctx* c);
int launch_iad(sph_ctx* c);
int launch_momentum(sph_ctx* c);
int launch_mom_records(sph_ctx* c);
int launch_mom_records_owned(sph_ctx* c);
int launch_mom_records_range(sph_ctx* c, int64_t i0, int64_t n, cudaStream_t st);
int launch_unit_order(sph_ctx* c);
int launch_dt_finalize(sph_ctx* c, bool nonempty);
int launch_update(sph_ctx* c);
int launch_diag(sph_ctx* c);
void set_poly_constants(const double* poly, const double* dpoly);

inline int grid_blocks(const sph_ctx* c, int64_t work_items, int threads, int per_sm) {
  int64_t b = (work_items + threads - 1) / threads;
  int64_t mx = (int64_t)c->num_sms * per_sm;
  if (b > mx) b = mx;
  if (b < 1) b = 1;
  return (int)b;
}

}  // namespace sphb
