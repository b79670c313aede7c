// sph_api.cu -- the extern "C" boundary declared in include/sph.h: validation,
// scratch ownership, phase sequencing, grid geometry, error state, profiling.
// Every step of the method runs in the kernels of sfc_sort.cu / physics.cu.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>

#include "sph_dist.cuh"
#include "stencil.cuh"

using namespace sphb;

namespace {

sph_status fail(sph_ctx* c, sph_status st, const std::string& msg) {
  if (c->status == SPH_OK) {
    c->status = st;
    c->err = msg;
  }
  return c->status;
}

#define CK(call)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return fail(c, SPH_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));       \
  } while (0)

#define CKL()                                                                                 \
  do {                                                                                        \
    cudaError_t e_ = cudaGetLastError();                                                      \
    if (e_ != cudaSuccess)                                                                    \
      return fail(c, SPH_ERR_CUDA, std::string("kernel launch (sph_api.cu:") +               \
                                       std::to_string(__LINE__) + "): " + cudaGetErrorString(e_)); \
  } while (0)

// ---- B_n of Eq. 6: 1 / (4 pi int_0^2 [sinc(pi v/2)]^n v^2 dv).
// Composite 8-point Gauss-Legendre in long double (independent of the oracle's
// Simpson rule).
long double sinc_pow_ld(long double v, int n) {
  if (v >= 2.0L) return 0.0L;
  long double x = 0.5L * 3.141592653589793238462643383279502884L * v;
  long double s = x == 0.0L ? 1.0L : std::sin(x) / x;
  long double r = 1.0L;
  for (int k = 0; k < n; ++k) r *= s;
  return r;
}

double kernel_norm(int n) {
  static const long double gx[8] = {-0.960289856497536231683560868569473L, -0.796666477413626739591553936475830L,
                                    -0.525532409916328985817739049189246L, -0.183434642495649804939476142360184L,
                                    0.183434642495649804939476142360184L,  0.525532409916328985817739049189246L,
                                    0.796666477413626739591553936475830L,  0.960289856497536231683560868569473L};
  static const long double gw[8] = {0.101228536290376259152531354309962L, 0.222381034453374470544355994426241L,
                                    0.313706645877887287337962201986601L, 0.362683783378361982965150449277196L,
                                    0.362683783378361982965150449277196L, 0.313706645877887287337962201986601L,
                                    0.222381034453374470544355994426241L, 0.101228536290376259152531354309962L};
  const int panels = 4000;
  long double acc = 0.0L, hw = 1.0L / panels;  // panel half-width (2 / panels / 2)
  for (int p = 0; p < panels; ++p) {
    long double mid = (2.0L * p + 1.0L) * hw;
    for (int k = 0; k < 8; ++k) {
      long double v = mid + hw * gx[k];
      acc += gw[k] * hw * sinc_pow_ld(v, n) * v * v;
    }
  }
  return (double)(1.0L / (4.0L * 3.141592653589793238462643383279502884L * acc));
}

// Coefficients (monomials in t) of the polynomial of degree kPolyTerms - 1 = 8
// interpolating P(t) = sinc(pi sqrt(t) / 2) at the 9 Chebyshev nodes of t in [0, 4]
// (v = sqrt(t) in [0, 2], the support of Eq. 6), in long double: near-minimax, evaluated
// in double max |P - sinc| 5.0e-14, |P^6 - sinc^6| 3.0e-13, |P' - sinc'| 2.0e-12 on
// [0, 4] -- 300x inside the 1e-10 parity tolerance (degree 9: 5.8e-16, one more DFMA per
// evaluation, 1.9 ms per 27M step; degree 7: 4e-11 on S^6, too close to it); dpoly =
// P'(t) of the same polynomial.
void sinc_coeffs(double* poly, double* dpoly) {
  const int N = kPolyTerms;
  const long double pi = 3.141592653589793238462643383279502884L;
  long double f[kPolyTerms], a[kPolyTerms];
  for (int j = 0; j < N; ++j) {  // samples at the nodes s_j = cos(pi (j + 1/2) / N), t = 2 (s + 1)
    const long double sj = std::cos(pi * (j + 0.5L) / N), t = 2.0L * (sj + 1.0L);
    const long double x = 0.5L * pi * std::sqrt(t);
    f[j] = x == 0.0L ? 1.0L : std::sin(x) / x;
  }
  for (int k = 0; k < N; ++k) {  // Chebyshev coefficients of the interpolant
    long double acc = 0.0L;
    for (int j = 0; j < N; ++j) acc += f[j] * std::cos(pi * k * (j + 0.5L) / N);
    a[k] = (k == 0 ? 1.0L : 2.0L) * acc / N;
  }
  // sum_k a_k T_k(s) -> monomials in s (T_{k+1} = 2 s T_k - T_{k-1}) -> monomials in t
  long double Tm[kPolyTerms] = {0}, Tk[kPolyTerms] = {0}, ps[kPolyTerms] = {0};
  Tm[0] = 1.0L;  // T_0
  Tk[1] = 1.0L;  // T_1
  ps[0] += a[0];
  for (int i = 0; i < N; ++i) ps[i] += a[1] * Tk[i];
  for (int k = 2; k < N; ++k) {
    long double Tn[kPolyTerms] = {0};
    for (int i = 0; i < N; ++i) Tn[i] = (i > 0 ? 2.0L * Tk[i - 1] : 0.0L) - Tm[i];
    for (int i = 0; i < N; ++i) {
      Tm[i] = Tk[i];
      Tk[i] = Tn[i];
      ps[i] += a[k] * Tn[i];
    }
  }
  long double pt[kPolyTerms] = {0};  // s = t/2 - 1: s^i = sum_j C(i,j) (t/2)^j (-1)^(i-j)
  for (int i = 0; i < N; ++i) {
    long double binom = 1.0L;
    for (int j = 0; j <= i; ++j) {
      if (j > 0) binom = binom * (i - j + 1) / j;
      pt[j] += ps[i] * binom * std::pow(0.5L, j) * (((i - j) & 1) ? -1.0L : 1.0L);
    }
  }
  for (int k = 0; k < N; ++k) poly[k] = (double)pt[k];
  for (int k = 0; k < N - 1; ++k) dpoly[k] = (double)((k + 1) * pt[k + 1]);
  dpoly[N - 1] = 0.0;
}

int bits_for(uint64_t v) {  // number of bits to hold values 0..v
  int b = 0;
  while (b < 64 && (v >> b)) ++b;
  return b;
}

struct Phase {
  sph_ctx* c;
  int ph;
  cudaEvent_t a = nullptr, b = nullptr;
  Phase(sph_ctx* c_, int ph_) : c(c_), ph(ph_) {
    if (c->prof) {
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, c->stream);
    }
  }
  void done(int launches) {
    c->launches += launches;
    c->phase_launches[ph] += launches;
    if (c->prof) {
      cudaEventRecord(b, c->stream);
      c->pending.push_back({ph, a, b});
      a = b = nullptr;
    }
  }
  ~Phase() {
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
  }
};

template <class T>
sph_status dalloc(sph_ctx* c, T** p, size_t count) {
  CK(cudaMalloc((void**)p, sizeof(T) * (count ? count : 1)));
  c->mem_bytes += sizeof(T) * (count ? count : 1);
  return SPH_OK;
}

sph_status choose_grid(sph_ctx* c, const double* bb, int64_t n) {
  const sph_params& q = c->prm;
  Grid& g = c->grid;
  const double hmean = bb[7] / (double)n;
  c->hmax = bb[6];
  if (!(hmean > 0.0) || !std::isfinite(hmean) || !std::isfinite(bb[6]))
    return fail(c, SPH_ERR_NUMERIC, "non-finite or non-positive smoothing lengths");
  for (int d = 0; d < 3; ++d) {
    if (!std::isfinite(bb[d]) || !std::isfinite(bb[3 + d]))
      return fail(c, SPH_ERR_NUMERIC, "non-finite particle positions");
    if (q.periodic[d] && (bb[d] < q.box_lo[d] || bb[3 + d] >= q.box_hi[d]))
      return fail(c, SPH_ERR_CONFIG, "particle outside the periodic box in dim " + std::to_string(d));
  }
  double edge = q.cell_factor * 2.0 * hmean;
  for (int attempt = 0; attempt < 200; ++attempt) {
    int64_t ncell = 1;
    for (int d = 0; d < 3; ++d) {
      double lo = q.periodic[d] ? q.box_lo[d] : bb[d];
      double ext = q.periodic[d] ? q.box_hi[d] - q.box_lo[d] : bb[3 + d] - bb[d];
      double ncd = std::floor(ext / edge);
      int nc = ncd < 1.0 ? 1 : (ncd > 2097151.0 ? 2097151 : (int)ncd);
      g.lo[d] = lo;
      g.nc[d] = nc;
      g.inv[d] = ext > 0.0 ? (double)nc / ext : 0.0;
      g.L[d] = q.box_hi[d] - q.box_lo[d];
      g.periodic[d] = q.periodic[d];
      ncell *= nc;
    }
    g.ncell = ncell;
    // the largest stencil (cell holding h_max) must fit kKMax slots
    int64_t K = 1;
    for (int d = 0; d < 3; ++d)
      K *= std::min<int64_t>(2 * stencil_radius(g, d, reach_of(bb[6])) + 1, g.nc[d]);
    if (ncell <= c->s.max_cells && K <= kKMax) break;
    edge *= 1.25;
  }
  if (g.ncell > c->s.max_cells) return fail(c, SPH_ERR_CAPACITY, "search grid too large");
  int mx = std::max(g.nc[0], std::max(g.nc[1], g.nc[2]));
  g.cbits = bits_for((uint64_t)(mx - 1));
  g.idbits = bits_for((uint64_t)bb[8]);
  if (3 * g.cbits + g.idbits > 64)
    return fail(c, SPH_ERR_CONFIG, "Morton key + id exceed 64 bits");
  // sub-cell order when bits remain; one bit stays free for the migration sentinel (multi-GPU)
  g.sbits = std::max(0, std::min(3, (63 - 3 * g.cbits - g.idbits) / 3));
  g.kshift = g.idbits + 3 * g.sbits;
  g.hsym = c->phys.sym ? bb[6] : 0.0;
  // pair-pass units (stencil.cuh): 2x2x1 cell blocks unless a periodic dim is so short
  // that stencils wrap onto themselves, or the unit stencil would exceed kKMax slots
  {
    static const int want = [] {
      const char* e = getenv("SPH_UNIT_BITS");  // A/B runs only
      const int v = e ? atoi(e) : 2;
      return v < 0 ? 0 : (v > 2 ? 2 : v);
    }();
    int ub = want;
    for (int d = 0; d < 3; ++d)
      if (g.periodic[d] && 2 * stencil_radius(g, d, reach_of(bb[6])) + 1 >= g.nc[d]) ub = 0;
    for (; ub > 0; --ub) {
      int64_t K = 1;
      for (int d = 0; d < 3; ++d)
        K *= std::min<int64_t>(2 * stencil_radius(g, d, reach_of(bb[6])) + 1 + (ub > d ? 1 : 0),
                               g.nc[d]);
      if (K <= kKMax) break;
    }
    g.ubits = ub;
  }
  return SPH_OK;
}

sph_status drain_profile(sph_ctx* c) {
  for (auto& e : c->pending) {
    float ms = 0.f;
    cudaEventSynchronize(e.b);
    cudaEventElapsedTime(&ms, e.a, e.b);
    c->phase_ms[e.ph] += ms;
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  c->pending.clear();
  return SPH_OK;
}

}  // namespace

extern "C" {

int sph_abi_version(void) { return SPH_ABI_VERSION; }

int sph_poly_coefficients(double* coef, int cap) {
  double p[kPolyTerms], d[kPolyTerms];
  sinc_coeffs(p, d);
  for (int k = 0; k < kPolyTerms && k < cap && coef; ++k) coef[k] = p[k];
  return kPolyTerms;
}

const char* sph_error_string(const sph_ctx* c) {
  if (!c) return "null context";
  return c->status == SPH_OK ? "ok" : c->err.c_str();
}

sph_status sph_init(const sph_params* prm, int64_t capacity, sph_ctx** out) {
  if (!out) return SPH_ERR_CONFIG;
  *out = nullptr;
  if (!prm || prm->abi_version != SPH_ABI_VERSION) return SPH_ERR_CONFIG;
  double nexp = prm->sinc_n;
  if (!(nexp >= 3.0 && nexp <= 9.0 && nexp == std::floor(nexp))) return SPH_ERR_CONFIG;
  if (capacity < 1 || capacity > 0xffffffffLL) return SPH_ERR_CONFIG;
  if (prm->nranks < 1 || prm->rank < 0 || prm->rank >= prm->nranks) return SPH_ERR_CONFIG;
  if (prm->nranks > 1 && !prm->nccl_unique_id) return SPH_ERR_CONFIG;
  if (prm->nranks > 64) return SPH_ERR_CONFIG;  // halo peer masks are 64-bit
  for (int d = 0; d < 3; ++d)
    if (prm->periodic[d] && !(prm->box_hi[d] > prm->box_lo[d])) return SPH_ERR_CONFIG;
  if (prm->eos != SPH_EOS_LINEAR && prm->eos != SPH_EOS_IDEAL) return SPH_ERR_CONFIG;
  if (prm->kernel_mode < SPH_KERNEL_POLY || prm->kernel_mode > SPH_KERNEL_SIN) return SPH_ERR_CONFIG;
  if (prm->kernel_mode == SPH_KERNEL_TABLE && prm->table_size != 0 && prm->table_size < 2)
    return SPH_ERR_CONFIG;

  sph_ctx* c = new sph_ctx();
  c->prm = *prm;
  if (c->prm.max_neighbors < 0) c->prm.max_neighbors = 0;
  if (!(c->prm.cell_factor > 0.0)) c->prm.cell_factor = 1.0;
  c->maxn = c->prm.max_neighbors;
  c->maxn_cap = c->maxn > 0 ? c->maxn : 384;  // 300 neighbours + headroom; grows on demand
  c->cap = capacity;
  c->stream = (cudaStream_t)prm->stream;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, dev);

  Phys& ph = c->phys;
  ph.n = (int)nexp;
  ph.B = kernel_norm(ph.n);
  sinc_coeffs(ph.poly, ph.dpoly);
  set_poly_constants(ph.poly, ph.dpoly);
  ph.kmode = prm->kernel_mode;
  ph.sym = prm->symmetric ? 1 : 0;
  ph.tableK = prm->table_size > 0 ? prm->table_size : 20000;
  ph.table = nullptr;
  ph.eos = prm->eos;
  ph.omega_mode = prm->omega_mode;
  ph.alpha = prm->alpha_av;
  ph.c0 = prm->c0;
  ph.rho0 = prm->rho0;
  ph.gamma = prm->gamma;
  ph.courant = prm->courant;
  ph.dt_growth = prm->dt_growth;
  ph.n_target = prm->n_target;
  ph.h_min = prm->h_min;
  ph.h_max = prm->h_max;
  ph.u_floor = prm->u_floor;
  for (int d = 0; d < 3; ++d) {
    ph.periodic[d] = prm->periodic[d];
    ph.box_lo[d] = prm->box_lo[d];
    ph.box_hi[d] = prm->box_hi[d];
    ph.L[d] = prm->box_hi[d] - prm->box_lo[d];
  }

  Scratch& s = c->s;
  const int64_t cap = capacity;
  const int64_t nblk_rs = (cap + 4095) / 4096;
  s.max_cells = std::max<int64_t>(1 << 16, 2 * cap);
  sph_status st = SPH_OK;
#define AL(p, n)                               \
  if ((st = dalloc(c, &(p), (size_t)(n))) != SPH_OK) { \
    sph_ctx* cc = c;                           \
    *out = cc;                                 \
    return st;                                 \
  }
  AL(s.keys, cap);
  AL(s.keys_alt, cap);
  AL(s.idx, cap);
  AL(s.idx_alt, cap);
  AL(s.hist, 256 * nblk_rs);
  AL(s.scan_tmp, (256 * nblk_rs + cap) / 8192 + 1024);
  AL(s.gather, 13 * cap);
  AL(s.gather_id, cap);
  AL(s.cell_start, s.max_cells);
  AL(s.cell_end, s.max_cells);
  AL(s.cell_hmax, s.max_cells);
  AL(s.cell_flag, cap);
  AL(s.cell_rank, cap);
  AL(s.cell_list, cap);
  AL(s.ncell_list, 1);
  AL(s.unit_flag, cap);
  AL(s.unit_rank, cap);
  AL(s.unit_list, cap + 1);
  AL(s.unit_rec, 3 * cap);
  if (prm->nranks > 1) {
    AL(s.unit_iflag, cap);
    AL(s.unit_iexcl, cap);
    AL(s.unit_order, cap);
    AL(s.unit_bounds, 4);
  }
  AL(s.nunit_list, 1);
  AL(s.mX, cap);
  AL(s.ct, 6 * cap);
  AL(s.mrec, 18 * cap);
  AL(s.nbr, cap * (int64_t)c->maxn_cap * (int64_t)sizeof(uint16_t));
  c->maxn_cap_alloc = c->maxn_cap;
  AL(s.ncount, cap);
  AL(s.nseg, cap);
  AL(s.nbr_max, 3);
  AL(s.work, 8);
  AL(s.wB, cap);
  AL(s.ih2, cap);
  AL(s.vol, cap);
  if (ph.kmode == SPH_KERNEL_TABLE) {  // the paper's table: K samples on [0, 2] incl. ends
    AL(s.ktable, ph.tableK);
    std::vector<double> tab(ph.tableK);
    for (int k = 0; k < ph.tableK; ++k) {
      const long double v = 2.0L * (long double)k / (long double)(ph.tableK - 1);
      tab[k] = v < 2.0L ? (double)sinc_pow_ld(v, ph.n) : 0.0;
    }
    if (cudaMemcpy(s.ktable, tab.data(), sizeof(double) * ph.tableK, cudaMemcpyHostToDevice) != cudaSuccess) {
      *out = c;
      return SPH_ERR_CUDA;
    }
    ph.table = s.ktable;
  }
  AL(s.rinv, cap);
  AL(s.X, cap);
  AL(s.red, (int64_t)c->num_sms * 64 * 9);
  AL(s.bbox, 16);
  AL(s.dts, DT_SLOTS);
  AL(s.cnt, kCounters);
  AL(s.bad_id, 1);
  AL(s.diag, 8);
#undef AL
  cudaMemsetAsync(s.cnt, 0, sizeof(unsigned long long) * kCounters, c->stream);
  cudaMemsetAsync(s.bad_id, 0xff, sizeof(unsigned long long), c->stream);
  cudaMemsetAsync(s.dts, 0, sizeof(double) * DT_SLOTS, c->stream);
  cudaMemsetAsync(s.ncount, 0, sizeof(uint32_t) * cap, c->stream);
  {
    double inf = INFINITY;
    unsigned long long bits;
    memcpy(&bits, &inf, 8);
    cudaMemcpyAsync(s.dts + DT_RAW_BITS, &bits, 8, cudaMemcpyHostToDevice, c->stream);
    cudaStreamSynchronize(c->stream);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fail(c, SPH_ERR_CUDA, cudaGetErrorString(e));
    *out = c;
    return SPH_ERR_CUDA;
  }
  if (prm->nranks > 1 && !dist_init(c, prm)) {  // NCCL communicator + exchange buffers
    fail(c, SPH_ERR_COMM, c->dist_err);
    *out = c;
    return SPH_ERR_COMM;
  }
  *out = c;
  return SPH_OK;
}

sph_status sph_attach(sph_ctx* c, const sph_particles* p) {
  if (!c || !p) return SPH_ERR_CONFIG;
  if (c->status != SPH_OK) return c->status;
  if (p->n < 0 || p->n > c->cap || p->capacity < p->n)
    return fail(c, SPH_ERR_CAPACITY, "n exceeds the context capacity");
  // multi-GPU: migration and halo unpack write up to the context capacity (sph_init)
  if (c->dist && p->capacity < c->cap)
    return fail(c, SPH_ERR_CAPACITY, "multi-GPU: particle arrays must hold the sph_init capacity");
  const void* ptrs[] = {p->id, p->x, p->y, p->z, p->vx, p->vy, p->vz, p->h, p->m, p->u, p->rho,
                        p->omega, p->p, p->c, p->c11, p->c12, p->c13, p->c22, p->c23, p->c33,
                        p->ax, p->ay, p->az, p->du, p->vsig, p->vhx, p->vhy, p->vhz, p->du_prev};
  for (const void* q : ptrs)
    if (!q) return fail(c, SPH_ERR_CONFIG, "null particle array");
  c->P = *p;
  c->first_bad_id = -1;
  CK(cudaMemsetAsync(c->s.bad_id, 0xff, sizeof(unsigned long long), c->stream));
  c->attached = true;
  c->first = true;
  c->stage = 0;
  c->steps = 0;
  return SPH_OK;
}

// Multi-GPU a1-a2 + a14 with ONE sort: keys of the owned set -> global key-prefix
// histogram -> splitters -> owner of every particle from its key;
// leavers are shipped to their owners, stayers close their holes, arrivals
// are appended, and a single radix sort puts the new owned set in canonical
// (cell, sub-cell, id) order.
static sph_status sort_migrate(sph_ctx* c) {
  const int nbits = 3 * c->grid.cbits + c->grid.kshift;
  const int64_t n = c->P.n;
  {
    Phase ph(c, SPH_PH_KEYS);
    int k = launch_keys(c);
    CKL();
    ph.done(k);
  }
  int64_t nleave = 0, nrecv = 0;
  {
    Phase ph(c, SPH_PH_HALO);
    if (!dist_splitters(c) || !dist_migrate(c, &nleave, &nrecv)) return fail(c, SPH_ERR_COMM, c->dist_err);
    c->P.n = n - nleave + nrecv;
    // keys of the moved stayers and the arrivals (all keys: simpler than tracking holes)
    int k = (nleave || nrecv) ? launch_keys(c) : 0;
    CKL();
    ph.done(k);
  }
  if (c->P.n == 0) return SPH_OK;
  const uint32_t* perm = nullptr;
  {
    Phase ph(c, SPH_PH_SORT);
    int k = launch_sort(c, nbits, &perm);
    CKL();
    ph.done(k);
  }
  {
    Phase ph(c, SPH_PH_PERMUTE);
    int k = launch_permute(c, perm);
    CKL();
    ph.done(k);
  }
  return SPH_OK;
}

static sph_status sort_owned(sph_ctx* c) {  // a1-a2 on [0, P.n): keys, radix sort, permutation
  if (c->P.n == 0) return SPH_OK;
  const int nbits = 3 * c->grid.cbits + c->grid.kshift;
  {
    Phase ph(c, SPH_PH_KEYS);
    int k = launch_keys(c);
    CKL();
    ph.done(k);
  }
  const uint32_t* perm = nullptr;
  {
    Phase ph(c, SPH_PH_SORT);
    int k = launch_sort(c, nbits, &perm);
    CKL();
    ph.done(k);
  }
  {
    Phase ph(c, SPH_PH_PERMUTE);
    int k = launch_permute(c, perm);
    CKL();
    ph.done(k);
  }
  return SPH_OK;
}

sph_status sph_find_neighbors(sph_ctx* c) {
  if (!c) return SPH_ERR_CONFIG;
  if (c->status != SPH_OK) return c->status;
  if (!c->attached) return fail(c, SPH_ERR_STATE, "no particles attached");
  const bool multi = c->dist != nullptr;
  c->stage = 0;
  c->n_halo = 0;
  if (!multi && c->P.n == 0) {
    c->nbr_total = c->nbr_max = 0;
    CK(cudaMemsetAsync(c->s.ncell_list, 0, sizeof(uint32_t), c->stream));
    CK(cudaMemsetAsync(c->s.nunit_list, 0, sizeof(uint32_t), c->stream));
    c->stage = 1;
    return SPH_OK;
  }
  double bb[16];
  {
    Phase ph(c, SPH_PH_BBOX);
    int k = launch_bbox(c);
    CKL();
    ph.done(k);
  }
  int64_t n_total = c->P.n;
  // S:90 / S:274: a non-finite or non-positive input (k_bbox) or an invalid dt / update of
  // the previous step (k_dt_finalize, k_update) stops here, read with the bbox (no extra sync)
  unsigned long long bad[2] = {~0ull, 0ull};
  bool bad_any = false;
  if (multi) {  // global domain size + h statistics (P:194 allreduce); the flag is global too
    if (!dist_global_bbox(c, bb, &bad_any)) return fail(c, SPH_ERR_COMM, c->dist_err);
    n_total = dist_n_total(c);
  }
  if (!multi) CK(cudaMemcpyAsync(bb, c->s.bbox, 9 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(&bad[0], c->s.bad_id, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(&bad[1], c->s.cnt + CNT_NONFINITE, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                     c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (bad[0] != ~0ull) c->first_bad_id = (int64_t)bad[0];
  if (bad_any || bad[0] != ~0ull || bad[1])
    return fail(c, SPH_ERR_NUMERIC,
                bad[0] != ~0ull ? "non-finite or non-positive state (x, h, m) of particle id " +
                                      std::to_string(bad[0]) + " (sph_diag.first_bad_id)"
                                : (bad[1] ? std::string("non-finite or non-positive dt in the previous step")
                                          : std::string("non-finite state on another rank")));
  c->n_global = n_total;
  if (n_total == 0) {
    c->stage = 1;
    return SPH_OK;
  }
  if (choose_grid(c, bb, n_total) != SPH_OK) return c->status;
  if (!multi) {
    if (sort_owned(c) != SPH_OK) return c->status;
  } else if (sort_migrate(c) != SPH_OK) {
    return c->status;
  }
  {
    Phase ph(c, SPH_PH_CELLS);
    int k = launch_cells(c);
    CKL();
    ph.done(k);
  }
  if (multi) {  // a4: halo identification + exchange #1
    Phase ph(c, SPH_PH_HALO);
    if (!dist_halo_plan_and_exchange1(c)) return fail(c, SPH_ERR_COMM, c->dist_err);
    c->n_halo = dist_n_halo(c);
    int k = launch_keys_range(c, c->P.n, c->n_halo);
    k += launch_cells_halo(c, c->P.n, c->n_halo);
    CKL();
    ph.done(k);
  }
  unsigned int mx[3] = {0, 0, 0};
  if (c->P.n) {
    Phase ph(c, SPH_PH_NEIGHBORS);
    int k = launch_unit_prep(c) + launch_search(c);
    CKL();
    ph.done(k);
  }
  CK(cudaMemcpyAsync(mx, c->s.nbr_max, sizeof(mx), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  // Rows never truncate (R23): a unit stencil too large for 16-bit entries, or a row
  // longer than the stride, reallocates the rows and reruns the search (rare: the h
  // update keeps counts near n_target); max_neighbors > 0 is a hard limit instead.
  while (c->P.n && (mx[1] || mx[2] || mx[0] > (unsigned)c->maxn_cap)) {
    if (c->maxn > 0 && mx[0] > (unsigned)c->maxn)
      return fail(c, SPH_ERR_CAPACITY, "a particle has " + std::to_string(mx[0]) +
                                           " neighbours > max_neighbors = " + std::to_string(c->maxn));
    if (getenv("SPH_DEBUG_ROWS"))
      fprintf(stderr, "sph: rows grow (max count %u, wide %u, segment overflow %u, stride %d)\n", mx[0], mx[1],
              mx[2], c->maxn_cap);
    if (mx[1]) c->wide_rows = true;
    if (mx[0] > (unsigned)c->maxn_cap) c->maxn_cap = (int)(((mx[0] + mx[0] / 8) + 31) / 32 * 32);
    else if (mx[2]) c->maxn_cap *= 2;  // the segments did not fit the row region
    const size_t old_bytes = (size_t)c->cap * c->maxn_cap_alloc * (c->wide_rows_alloc ? 4 : 2);
    CK(cudaFree(c->s.nbr));
    c->s.nbr = nullptr;
    c->mem_bytes -= old_bytes;
    const size_t bytes = (size_t)c->cap * c->maxn_cap * (c->wide_rows ? 4 : 2);
    if (cudaMalloc((void**)&c->s.nbr, bytes) != cudaSuccess) {
      cudaGetLastError();
      return fail(c, SPH_ERR_CAPACITY, "neighbour rows: cannot allocate " + std::to_string(bytes) + " bytes");
    }
    c->mem_bytes += bytes;
    c->maxn_cap_alloc = c->maxn_cap;
    c->wide_rows_alloc = c->wide_rows;
    Phase ph(c, SPH_PH_NEIGHBORS);
    int k = launch_search(c);
    CKL();
    ph.done(k);
    CK(cudaMemcpyAsync(mx, c->s.nbr_max, sizeof(mx), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  }
  c->nbr_max = mx[0];
  if (c->P.n) {  // segments -> flat-index rows, in place
    Phase ph(c, SPH_PH_NEIGHBORS);
    int k = launch_expand_rows(c);
    if (k < 0)
      return fail(c, SPH_ERR_CAPACITY, "neighbour rows of " + std::to_string(c->maxn_cap) +
                                           " entries exceed the row-expansion buffer");
    CKL();
    ph.done(k);
  }
  c->stage = 1;
  return SPH_OK;
}

sph_status sph_get_neighbors(sph_ctx* c, int64_t* offsets, int64_t* ids, int64_t cap) {
  if (!c || !offsets) return SPH_ERR_CONFIG;
  if (c->status != SPH_OK) return c->status;
  if (c->stage < 1) return fail(c, SPH_ERR_STATE, "sph_get_neighbors before sph_find_neighbors");
  const int64_t n = c->P.n;
  std::vector<uint32_t> cnt(n > 0 ? n : 1);
  const int64_t nl = n + c->n_halo;  // neighbours may be halo particles
  std::vector<int64_t> id(nl > 0 ? nl : 1);
  CK(cudaStreamSynchronize(c->stream));
  if (n) {
    CK(cudaMemcpy(cnt.data(), c->s.ncount, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(id.data(), c->P.id, sizeof(int64_t) * nl, cudaMemcpyDeviceToHost));
  }
  offsets[0] = 0;
  for (int64_t i = 0; i < n; ++i) offsets[i + 1] = offsets[i] + cnt[i];
  if (offsets[n] > cap) return SPH_ERR_CAPACITY;  // not sticky: caller retries with room
  if (!ids) return SPH_OK;
  // rows hold flat indices into unit stencils: decode with the cell tables
  const Grid& g = c->grid;
  std::vector<uint64_t> keys(n);
  std::vector<uint32_t> cs(g.ncell), ce(g.ncell);
  std::vector<unsigned long long> chm(g.ncell);
  CK(cudaMemcpy(keys.data(), c->s.keys, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(cs.data(), c->s.cell_start, sizeof(uint32_t) * g.ncell, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(ce.data(), c->s.cell_end, sizeof(uint32_t) * g.ncell, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(chm.data(), c->s.cell_hmax, sizeof(unsigned long long) * g.ncell,
                cudaMemcpyDeviceToHost));
  const int64_t chunk = 1 << 14;
  const size_t esz = c->wide_rows ? 4 : 2;
  std::vector<unsigned char> rows((size_t)chunk * c->maxn_cap * esz);
  std::vector<int64_t> ucum, ucell;
  int ub3[3] = {-1, -1, -1};
  Stencil st;
  for (int64_t r0 = 0; r0 < n; r0 += chunk) {
    int64_t nr = std::min(chunk, n - r0);
    CK(cudaMemcpy(rows.data(), c->s.nbr + (size_t)r0 * c->maxn_cap * esz,
                  esz * nr * c->maxn_cap, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < nr; ++i) {
      const int64_t cell = key_cell_hd(g, keys[r0 + i]);
      int c3[3];
      cell_coords(g, cell, c3);
      // rows hold flat indices into the target's unit stencil (slots in order, each
      // slot its cell's range): rebuild the slot prefix when the unit changes
      int b3[3];
      unit_base(g, c3, b3);
      if (b3[0] != ub3[0] || b3[1] != ub3[1] || b3[2] != ub3[2]) {
        memcpy(ub3, b3, sizeof(b3));
        make_unit_stencil(g, c3, cs.data(), ce.data(), chm.data(), st);
        ucum.assign(st.K + 1, 0);
        ucell.assign(st.K, 0);
        for (int k = 0; k < st.K; ++k) {
          int sh[3];
          ucell[k] = slot_cell(g, st, k, sh);
          ucum[k + 1] = ucum[k] + (ce[ucell[k]] - cs[ucell[k]]);
        }
      }
      for (uint32_t k = 0; k < cnt[r0 + i]; ++k) {
        const size_t at = (size_t)i * c->maxn_cap + k;
        const int64_t e = c->wide_rows ? (int64_t)((const uint32_t*)rows.data())[at]
                                       : (int64_t)((const uint16_t*)rows.data())[at];
        if (e >= ucum[st.K]) return fail(c, SPH_ERR_STATE, "neighbour row entry outside its unit stencil");
        const int slot = (int)(std::upper_bound(ucum.begin(), ucum.end(), e) - ucum.begin()) - 1;
        ids[offsets[r0 + i] + k] = id[cs[ucell[slot]] + (e - ucum[slot])];
      }
    }
  }
  return SPH_OK;
}

sph_status sph_density(sph_ctx* c) {
  if (!c) return SPH_ERR_CONFIG;
  if (c->status != SPH_OK) return c->status;
  if (c->stage < 1) return fail(c, SPH_ERR_STATE, "sph_density before sph_find_neighbors");
  if (c->P.n) {
    Phase ph(c, SPH_PH_DENSITY);
    int k = launch_density(c);
    CKL();
    ph.done(k);
  }
  if (c->dist) {  // a7: halo exchange #2 (R21), in flight during the interior IAD units
    Phase ph(c, SPH_PH_HALO);
    if (!dist_exchange2(c)) return fail(c, SPH_ERR_COMM, c->dist_err);
    ph.done(0);
  }
  c->stage = 2;
  return SPH_OK;
}

sph_status sph_iad(sph_ctx* c) {
  if (!c) return SPH_ERR_CONFIG;
  if (c->status != SPH_OK) return c->status;
  if (c->stage < 2) return fail(c, SPH_ERR_STATE, "sph_iad before sph_density");
  if (c->dist) {  // interior units while exchange #2 is in flight, then the boundary units
    Phase ph(c, SPH_PH_IAD);
    int k = 0;
    c->unit_sel = 1;
    if (c->P.n) k += launch_iad(c);
    c->unit_sel = 0;
    if (!dist_wait_halo(c)) return fail(c, SPH_ERR_COMM, c->dist_err);
    c->unit_sel = 2;
    if (c->P.n) k += launch_iad(c);
    c->unit_sel = 0;
    CKL();
    ph.done(k);
  } else if (c->P.n) {
    Phase ph(c, SPH_PH_IAD);
    int k = launch_iad(c);
    CKL();
    ph.done(k);
  }
  if (c->dist) {  // a9: halo exchange #3 (R21), in flight during the interior momentum units
    Phase ph(c, SPH_PH_HALO);
    if (!dist_exchange3(c)) return fail(c, SPH_ERR_COMM, c->dist_err);
    ph.done(0);
  }
  c->stage = 3;
  return SPH_OK;
}

sph_status sph_momentum_energy(sph_ctx* c, double* dt_out) {
  if (!c) return SPH_ERR_CONFIG;
  if (c->status != SPH_OK) return c->status;
  if (c->stage < 3) return fail(c, SPH_ERR_STATE, "sph_momentum_energy before sph_iad");
  if (c->P.n) {  // source records not written by the IAD epilogue (multi-GPU halos: with exchange #3)
    Phase ph(c, SPH_PH_RECORDS);
    int k = c->dist ? launch_mom_records_owned(c) : launch_mom_records(c);
    CKL();
    ph.done(k);
  }
  {
    Phase ph(c, SPH_PH_MOMENTUM);
    int k = 0;
    if (c->dist) {  // interior units while exchange #3 is in flight, then the boundary units
      c->unit_sel = 1;
      if (c->P.n) k += launch_momentum(c);
      c->unit_sel = 0;
      if (!dist_wait_halo(c)) return fail(c, SPH_ERR_COMM, c->dist_err);
      c->unit_sel = 2;
      if (c->P.n) k += launch_momentum(c);
      c->unit_sel = 0;
    } else if (c->P.n) {
      k = launch_momentum(c);
    }
    if (c->dist && !dist_allreduce_dt(c)) return fail(c, SPH_ERR_COMM, c->dist_err);  // a11
    k += launch_dt_finalize(c, c->n_global > 0);
    CKL();
    ph.done(k);
  }
  c->stage = 4;
  if (dt_out) {
    double dts[DT_SLOTS];
    CK(cudaMemcpyAsync(dts, c->s.dts, sizeof(dts), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    *dt_out = dts[DT_CUR];
    if (!std::isfinite(dts[DT_CUR]) || !(dts[DT_CUR] > 0.0))
      return fail(c, SPH_ERR_NUMERIC, "non-finite or non-positive dt");
  }
  return SPH_OK;
}

sph_status sph_advance(sph_ctx* c) {
  if (!c) return SPH_ERR_CONFIG;
  if (c->status != SPH_OK) return c->status;
  if (c->stage < 4) return fail(c, SPH_ERR_STATE, "sph_advance before sph_momentum_energy");
  if (c->P.n) {
    Phase ph(c, SPH_PH_UPDATE);
    int k = launch_update(c);
    CKL();
    ph.done(k);
  }
  c->first = false;
  c->steps++;
  c->stage = 0;
  return SPH_OK;
}

sph_status sph_step(sph_ctx* c, double* dt_out) {
  sph_status st;
  if ((st = sph_find_neighbors(c)) != SPH_OK) return st;
  if ((st = sph_density(c)) != SPH_OK) return st;
  if ((st = sph_iad(c)) != SPH_OK) return st;
  if ((st = sph_momentum_energy(c, dt_out)) != SPH_OK) return st;
  return sph_advance(c);
}

static sph_status copy_state(sph_ctx* c, const sph_particles* host, bool up) {
  const sph_particles& P = c->P;
  const int64_t n = up ? host->n : P.n;
  if (up && (n < 0 || n > c->cap || n > P.capacity))
    return fail(c, SPH_ERR_CAPACITY, "upload: n exceeds capacity");
  double* const dev[13] = {P.x, P.y, P.z, P.vx, P.vy, P.vz, P.h, P.m, P.u, P.vhx, P.vhy, P.vhz, P.du_prev};
  double* const hst[13] = {host->x, host->y, host->z, host->vx, host->vy, host->vz, host->h,
                           host->m, host->u, host->vhx, host->vhy, host->vhz, host->du_prev};
  auto kind = up ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
  for (int k = 0; k < 13; ++k) {
    if (!hst[k]) continue;
    CK(cudaMemcpyAsync(up ? (void*)dev[k] : (void*)hst[k], up ? (const void*)hst[k] : (const void*)dev[k],
                       sizeof(double) * n, kind, c->stream));
  }
  if (host->id)
    CK(cudaMemcpyAsync(up ? (void*)P.id : (void*)host->id, up ? (const void*)host->id : (const void*)P.id,
                       sizeof(int64_t) * n, kind, c->stream));
  return SPH_OK;
}

sph_status sph_upload(sph_ctx* c, const sph_particles* host) {
  if (!c || !host) return SPH_ERR_CONFIG;
  if (c->status != SPH_OK) return c->status;
  if (!c->attached) return fail(c, SPH_ERR_STATE, "no particles attached");
  sph_status st = copy_state(c, host, true);
  if (st != SPH_OK) return st;
  c->P.n = host->n;
  c->stage = 0;
  return SPH_OK;
}

sph_status sph_download(sph_ctx* c, sph_particles* host) {
  if (!c || !host) return SPH_ERR_CONFIG;
  if (c->status != SPH_OK) return c->status;
  if (!c->attached) return fail(c, SPH_ERR_STATE, "no particles attached");
  sph_status st = copy_state(c, host, false);
  if (st != SPH_OK) return st;
  host->n = c->P.n;
  CK(cudaStreamSynchronize(c->stream));
  return SPH_OK;
}

sph_status sph_diagnostics(sph_ctx* c, sph_diag* out) {
  if (!c || !out) return SPH_ERR_CONFIG;
  memset(out, 0, sizeof(*out));
  if (c->status != SPH_OK) {  // sticky error: report what the host knows (which particle, when)
    out->first_bad_id = c->first_bad_id;
    out->steps = c->steps;
    return c->status;
  }
  double d[8] = {0};
  unsigned long long badid = ~0ull;
  if (c->attached && c->P.n) {
    launch_diag(c);
    CKL();
  } else {
    CK(cudaMemsetAsync(c->s.diag, 0, sizeof(d), c->stream));
  }
  int64_t n_owned = c->P.n;
  if (c->dist) {  // a15: optional global sums
    if (!dist_allreduce_diag(c, c->s.diag, c->s.cnt)) return fail(c, SPH_ERR_COMM, c->dist_err);
    n_owned = dist_n_total(c);
  }
  CK(cudaMemcpyAsync(d, c->s.diag, sizeof(d), cudaMemcpyDeviceToHost, c->stream));
  unsigned long long cnt[kCounters];
  double dts[DT_SLOTS];
  CK(cudaMemcpyAsync(cnt, c->dist ? dist_counters(c) : c->s.cnt, sizeof(cnt), cudaMemcpyDeviceToHost,
                     c->stream));
  CK(cudaMemcpyAsync(dts, c->s.dts, sizeof(dts), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(&badid, c->s.bad_id, sizeof(badid), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (badid != ~0ull) c->first_bad_id = (int64_t)badid;
  out->first_bad_id = c->first_bad_id;
  out->n_owned = n_owned;
  out->n_halo = c->n_halo;
  out->nbr_total = (int64_t)d[7];
  out->nbr_max = c->nbr_max;
  out->omega_clamped = (int64_t)cnt[CNT_OMEGA];
  out->iad_singular = (int64_t)cnt[CNT_IAD_SINGULAR];
  out->coincident_pairs = (int64_t)cnt[CNT_COINCIDENT];
  out->u_floored = (int64_t)cnt[CNT_U_FLOOR];
  out->h_clamped = (int64_t)cnt[CNT_H_CLAMP];
  out->steps = c->steps;
  out->dt = dts[DT_CUR];
  out->dt_prev = dts[DT_COMMITTED];
  out->time = dts[DT_TIME];
  for (int k = 0; k < 3; ++k) {
    out->momentum[k] = d[k];
    out->ang_momentum[k] = d[3 + k];
    out->grid[k] = c->grid.nc[k];
  }
  out->energy = d[6];
  if (cnt[CNT_NONFINITE]) return fail(c, SPH_ERR_NUMERIC, "non-finite dt encountered");
  if (badid != ~0ull)
    return fail(c, SPH_ERR_NUMERIC, "non-finite state of particle id " + std::to_string(badid));
  return SPH_OK;
}

sph_status sph_memory_bytes(const sph_ctx* c, int64_t* bytes) {
  if (!c || !bytes) return SPH_ERR_CONFIG;
  *bytes = (int64_t)c->mem_bytes + (c->dist ? dist_memory_bytes(c) : 0);
  return SPH_OK;
}

sph_status sph_local_count(const sph_ctx* c, int64_t* n_owned, int64_t* n_halo) {
  if (!c) return SPH_ERR_CONFIG;
  if (n_owned) *n_owned = c->P.n;
  if (n_halo) *n_halo = c->n_halo;
  return SPH_OK;
}

sph_status sph_set_profiling(sph_ctx* c, int on) {
  if (!c) return SPH_ERR_CONFIG;
  c->prof = on != 0;
  return SPH_OK;
}

sph_status sph_phase_times(sph_ctx* c, double* ms_out, int64_t* launches_out, int reset) {
  if (!c) return SPH_ERR_CONFIG;
  drain_profile(c);
  for (int k = 0; k < SPH_PH_COUNT; ++k) {
    if (ms_out) ms_out[k] = c->phase_ms[k];
    if (launches_out) launches_out[k] = c->phase_launches[k];
    if (reset) {
      c->phase_ms[k] = 0.0;
      c->phase_launches[k] = 0;
    }
  }
  return SPH_OK;
}

sph_status sph_destroy(sph_ctx* c) {
  if (!c) return SPH_OK;
  drain_profile(c);
  cudaStreamSynchronize(c->stream);
  dist_destroy(c);
  Scratch& s = c->s;
  void* ptrs[] = {s.keys, s.keys_alt, s.idx, s.idx_alt, s.hist, s.scan_tmp, s.gather, s.gather_id,
                  s.cell_start, s.cell_end, s.cell_hmax, s.cell_flag, s.cell_rank, s.cell_list,
                  s.ncell_list, s.unit_flag, s.unit_rank, s.unit_list, s.nunit_list, s.unit_rec, s.unit_iflag, s.unit_iexcl, s.unit_order, s.unit_bounds, s.nbr, s.ncount, s.nseg, s.nbr_max, s.work, s.wB, s.ih2, s.vol, s.rinv, s.X,
                  s.mX, s.ct, s.mrec, s.red, s.bbox, s.dts, s.cnt, s.bad_id, s.diag, s.ktable};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  delete c;
  return SPH_OK;
}

}  // extern "C"
