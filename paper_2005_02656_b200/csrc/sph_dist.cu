// sph_dist.cu -- multi-GPU SFC domain decomposition (§4.3-4.4, P:191-222;
// SURVEY §8(e)): global bbox/h allreduce, key-prefix histogram allreduce ->
// splitters at equal counts (the paper's global top tree), migration of
// particles that left the rank's key range, halo identification, and the
// three halo exchanges per step (reading R21) over NCCL send/recv.
//
// Local layout on every rank during a step: [owned, sorted by key | halo, sorted
// by key].  Every search cell belongs to exactly one rank and halos are whole
// cells, so a target's stencil slots and the within-cell order are the same as
// on one GPU: per-particle results are bit-identical for any rank count.
#include <algorithm>
#include <numeric>
#include <string>
#include <vector>

#include "stencil.cuh"
#include "sph_dist.cuh"
#ifdef SPH_WITH_NCCL
#include <nccl.h>
#endif

namespace sphb {

// ------------------------------------------------------------------ host logic (testable on CPU)
// Splitters: rank r owns key-prefix bins [split[r], split[r+1]); split[r] is the
// first bin whose inclusive prefix count exceeds floor(r * total / G).
void compute_splitters(const int64_t* hist, int64_t nbins, int G, int64_t* split) {
  int64_t total = 0;
  for (int64_t b = 0; b < nbins; ++b) total += hist[b];
  split[0] = 0;
  int64_t acc = 0, b = 0;
  for (int r = 1; r < G; ++r) {
    const int64_t target = (int64_t)((__int128)total * r / G);
    while (b < nbins && acc + hist[b] <= target) acc += hist[b++];
    split[r] = b;
  }
  split[G] = nbins;
  for (int r = 1; r <= G; ++r) split[r] = std::max(split[r], split[r - 1]);
}

int owner_of_bin(const int64_t* split, int G, int64_t bin) {
  int lo = 0, hi = G;  // largest r with split[r] <= bin
  while (hi - lo > 1) {
    int mid = (lo + hi) / 2;
    if (split[mid] <= bin) lo = mid;
    else hi = mid;
  }
  return lo;
}

// every collective goes through the rank's transport (comm.cuh: NCCL, or the in-process
// hub that runs G ranks as threads of one process on one GPU)
#define COMM(call)                                                                          \
  do {                                                                                      \
    if (!(c->dist->comm->call)) return false;                                               \
  } while (0)
#define CUK(call)                                                                           \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      c->dist_err = std::string(#call) + ": " + cudaGetErrorString(e_);                     \
      return false;                                                                         \
    }                                                                                       \
  } while (0)

// ------------------------------------------------------------------ kernels
__device__ __forceinline__ uint64_t spread3d(uint64_t v) {
  v &= 0x1fffffull;
  v = (v | (v << 32)) & 0x1f00000000ffffull;
  v = (v | (v << 16)) & 0x1f0000ff0000ffull;
  v = (v | (v << 8)) & 0x100f00f00f00f00full;
  v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}

__device__ __forceinline__ int64_t key_bin(const Grid& g, uint64_t key, int shift) {
  const uint64_t m = g.kshift >= 64 ? 0 : key >> g.kshift;
  return (int64_t)(m >> shift);
}

// Key-prefix histogram.  Particles are still in the previous step's (cell) order, so
// a warp's 32 consecutive keys fall into one or two bins: one atomic per distinct
// bin of the warp (match_any) instead of 32 atomics on the same address (which
// serialised to ~9 ms per step at 25M particles, profiled per rank).
__global__ void k_bin_hist(const uint64_t* __restrict__ keys, int64_t n, Grid g, int shift,
                           unsigned long long* __restrict__ hist) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); i0 < n; i0 += stride) {
    const int64_t i = i0 + lane;
    const bool ok = i < n;
    const unsigned long long bin = ok ? (unsigned long long)key_bin(g, keys[i], shift) : ~0ull;
    const unsigned grp = __match_any_sync(0xffffffffu, bin);
    if (ok && lane == __ffs(grp) - 1) atomicAdd(&hist[bin], (unsigned long long)__popc(grp));
  }
}

__device__ __forceinline__ int owner_dev(const int64_t* split, int G, int64_t bin) {
  int lo = 0, hi = G;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (split[mid] <= bin) lo = mid;
    else hi = mid;
  }
  return lo;
}

struct FieldSet {
  uint64_t* f[16];
  int nf;
};

// a14: owner of every owned particle from its (unsorted) key; leavers per owner
__global__ void k_owner_count(const uint64_t* __restrict__ keys, int64_t n, Grid g, int shift,
                              const int64_t* __restrict__ split, int G, int me,
                              uint32_t* __restrict__ dest, unsigned long long* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int o = owner_dev(split, G, key_bin(g, keys[i], shift));
    dest[i] = (uint32_t)o;
    if (o != me) atomicAdd(&cnt[o], 1ull);
  }
}
// Leavers: per-owner send lists, and the compaction pairs -- leavers below n_keep
// ("holes") and stayers at or above n_keep ("movers") are equally many; each mover
// fills one hole.  Any order and pairing will do: the owned set is sorted next.
__global__ void k_owner_fill(int64_t n, int64_t n_keep, const uint32_t* __restrict__ dest, int me,
                             const int64_t* __restrict__ soff, unsigned long long* __restrict__ fill,
                             uint32_t* __restrict__ send_idx, unsigned long long* __restrict__ hm,
                             uint32_t* __restrict__ holes, uint32_t* __restrict__ movers) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t o = dest[i];
    if ((int)o != me) {
      const unsigned long long slot = atomicAdd(&fill[o], 1ull);
      send_idx[soff[o] + (int64_t)slot] = (uint32_t)i;
      if (i < n_keep) holes[atomicAdd(&hm[0], 1ull)] = (uint32_t)i;
    } else if (i >= n_keep) {
      movers[atomicAdd(&hm[1], 1ull)] = (uint32_t)i;
    }
  }
}
__global__ void k_fill_holes_dev(FieldSet fs, const uint32_t* __restrict__ holes,
                                 const uint32_t* __restrict__ movers,
                                 const unsigned long long* __restrict__ hm) {
  const int64_t k = (int64_t)hm[0];  // == hm[1]
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < k;
       t += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t h = holes[t], m = movers[t];
    for (int f = 0; f < fs.nf; ++f) fs.f[f][h] = fs.f[f][m];
  }
}

// per owned non-empty cell: bit r set if rank r owns a cell within the halo box
__global__ void k_halo_mask(const uint32_t* __restrict__ clist, const uint32_t* __restrict__ ncl,
                            Grid g, int Rx, int Ry, int Rz, const int64_t* __restrict__ split, int G,
                            int rank, int shift, unsigned long long* __restrict__ mask) {
  const uint32_t nl = *ncl;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nl; i += gridDim.x * blockDim.x) {
    int c3[3];
    cell_coords(g, clist[i], c3);
    const int R[3] = {Rx, Ry, Rz};
    int lo[3], cnt[3];
    for (int d = 0; d < 3; ++d) {
      if (2 * R[d] + 1 >= g.nc[d]) {
        lo[d] = 0;
        cnt[d] = g.nc[d];
      } else if (g.periodic[d]) {
        lo[d] = c3[d] - R[d];
        cnt[d] = 2 * R[d] + 1;
      } else {
        const int l = max(0, c3[d] - R[d]), u = min(g.nc[d] - 1, c3[d] + R[d]);
        lo[d] = l;
        cnt[d] = u - l + 1;
      }
    }
    unsigned long long m = 0;
    for (int iz = 0; iz < cnt[2]; ++iz)
      for (int iy = 0; iy < cnt[1]; ++iy)
        for (int ix = 0; ix < cnt[0]; ++ix) {
          int q[3] = {lo[0] + ix, lo[1] + iy, lo[2] + iz};
          for (int d = 0; d < 3; ++d) q[d] = q[d] < 0 ? q[d] + g.nc[d] : (q[d] >= g.nc[d] ? q[d] - g.nc[d] : q[d]);
          const uint64_t mort = spread3d(q[0]) | (spread3d(q[1]) << 1) | (spread3d(q[2]) << 2);
          const int o = owner_dev(split, G, (int64_t)(mort >> shift));
          if (o != rank) m |= 1ull << o;
        }
    mask[i] = m;
  }
}

// per-peer halo totals in one pass (block-aggregated atomics; G <= 64)
__global__ void k_peer_totals(const uint32_t* __restrict__ clist, const uint32_t* __restrict__ ncl,
                              const uint32_t* __restrict__ cstart, const uint32_t* __restrict__ cend,
                              const unsigned long long* __restrict__ mask, int G,
                              unsigned long long* __restrict__ tot) {
  __shared__ unsigned long long bt[64];
  for (int r = threadIdx.x; r < G; r += blockDim.x) bt[r] = 0;
  __syncthreads();
  const uint32_t nl = *ncl;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nl; i += gridDim.x * blockDim.x) {
    unsigned long long m = mask[i];
    if (!m) continue;
    const uint32_t c = clist[i];
    const unsigned long long cnt = cend[c] - cstart[c];
    while (m) {
      const int r = __ffsll((long long)m) - 1;
      m &= m - 1;
      atomicAdd(&bt[r], cnt);
    }
  }
  __syncthreads();
  for (int r = threadIdx.x; r < G; r += blockDim.x)
    if (bt[r]) atomicAdd(&tot[r], bt[r]);
}

// particles each owned cell sends to peer r (0 when the bit is clear)
__global__ void k_peer_counts(const uint32_t* __restrict__ clist, const uint32_t* __restrict__ ncl,
                              const uint32_t* __restrict__ cstart, const uint32_t* __restrict__ cend,
                              const unsigned long long* __restrict__ mask, int r,
                              uint32_t* __restrict__ cnt) {
  const uint32_t nl = *ncl;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nl; i += gridDim.x * blockDim.x) {
    const uint32_t c = clist[i];
    cnt[i] = (mask[i] >> r) & 1ull ? cend[c] - cstart[c] : 0u;
  }
}

__global__ void k_fill_send(const uint32_t* __restrict__ clist, const uint32_t* __restrict__ ncl,
                            const uint32_t* __restrict__ cstart, const uint32_t* __restrict__ cend,
                            const unsigned long long* __restrict__ mask, int r,
                            const uint32_t* __restrict__ off, uint32_t* __restrict__ out) {
  const uint32_t nl = *ncl;
  const int lane = threadIdx.x & 31;
  for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < nl;
       i += (gridDim.x * blockDim.x) >> 5) {
    if (!((mask[i] >> r) & 1ull)) continue;
    const uint32_t c = clist[i], s = cstart[c], e = cend[c], o = off[i];
    for (uint32_t k = lane; k < e - s; k += 32) out[o + k] = s + k;
  }
}



// sendbuf layout per peer: nf blocks of cnt_r elements
__global__ void k_pack(FieldSet fs, const uint32_t* __restrict__ idx, int64_t n, int64_t base,
                       uint64_t* __restrict__ buf) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t j = idx[k];
    for (int f = 0; f < fs.nf; ++f) buf[base * fs.nf + f * n + k] = fs.f[f][j];
  }
}
__global__ void k_unpack(FieldSet fs, const uint64_t* __restrict__ buf, int64_t n, int64_t base,
                         int64_t dst0) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    for (int f = 0; f < fs.nf; ++f) fs.f[f][dst0 + k] = buf[base * fs.nf + f * n + k];
}
__global__ void k_bbox_pack(const double* __restrict__ bb, int64_t n, const unsigned long long* __restrict__ bad_id,
                            const unsigned long long* __restrict__ cnt, double* __restrict__ mx,
                            double* __restrict__ sm) {
  // MAX of {-min x,y,z, max x,y,z, max h, max id, bad state flag}; SUM of {sum h, n}
  mx[0] = -bb[0]; mx[1] = -bb[1]; mx[2] = -bb[2];
  mx[3] = bb[3]; mx[4] = bb[4]; mx[5] = bb[5];
  mx[6] = bb[6]; mx[7] = bb[8];
  mx[8] = (*bad_id != ~0ull || cnt[CNT_NONFINITE]) ? 1.0 : 0.0;
  sm[0] = n ? bb[7] : 0.0;
  sm[1] = (double)n;
}

// ------------------------------------------------------------------ orchestration
static FieldSet state_fields(sph_ctx* c, bool with_hist) {
  sph_particles& P = c->P;
  FieldSet fs{};
  uint64_t** f = fs.f;
  int k = 0;
  for (double* p : {P.x, P.y, P.z, P.vx, P.vy, P.vz, P.h, P.m, P.u}) f[k++] = (uint64_t*)p;
  if (with_hist)
    for (double* p : {P.vhx, P.vhy, P.vhz, P.du_prev}) f[k++] = (uint64_t*)p;
  f[k++] = (uint64_t*)P.id;
  fs.nf = k;
  return fs;
}

// Pack on the compute stream, transfer on `xs` (the compute stream, or the comm stream
// of an overlapped exchange, which first waits for the packing).
static bool exchange(sph_ctx* c, const FieldSet& fs, cudaStream_t xs) {
  // send the per-peer index lists (send_idx at soff), receive in rank order
  Dist& D = *c->dist;
  const int G = D.G, me = D.rank;
  const int F = fs.nf;
  int64_t sbase = 0, rbase = 0;
  for (int r = 0; r < G; ++r) {
    if (D.scnt[r] && r != me) {
      k_pack<<<grid_blocks(c, D.scnt[r], 256, 4), 256, 0, c->stream>>>(fs, D.send_idx + D.soff[r],
                                                                       D.scnt[r], sbase, D.sendbuf);
      c->launches++;
    }
    if (r != me) sbase += D.scnt[r];
  }
  CUK(cudaGetLastError());
  if (xs != c->stream) {
    CUK(cudaEventRecord(D.ev_pack, c->stream));
    CUK(cudaStreamWaitEvent(xs, D.ev_pack, 0));
  }
  std::vector<Xfer> sends, recvs;
  sbase = 0;
  for (int r = 0; r < G; ++r) {
    if (r == me) continue;
    if (D.scnt[r]) sends.push_back({r, D.sendbuf + sbase * F, (size_t)D.scnt[r] * F * sizeof(uint64_t)});
    if (D.rcnt[r]) recvs.push_back({r, D.recvbuf + rbase * F, (size_t)D.rcnt[r] * F * sizeof(uint64_t)});
    sbase += D.scnt[r];
    rbase += D.rcnt[r];
  }
  COMM(exchange(sends, recvs, xs, c->dist_err));
  return true;
}

static bool unpack_all(sph_ctx* c, const FieldSet& fs, int64_t dst0, cudaStream_t us) {
  Dist& D = *c->dist;
  int64_t rbase = 0;
  for (int r = 0; r < D.G; ++r) {
    if (r == D.rank) continue;
    if (D.rcnt[r]) {
      k_unpack<<<grid_blocks(c, D.rcnt[r], 256, 4), 256, 0, us>>>(fs, D.recvbuf, D.rcnt[r], rbase,
                                                                 dst0 + rbase);
      c->launches++;
    }
    rbase += D.rcnt[r];
  }
  CUK(cudaGetLastError());
  return true;
}

// all-gather the per-peer send counts, derive receive counts
// All-gather every rank's row [send counts to each peer..., base count] and derive this
// rank's receive counts.  `need(send_total, recv_total, base)` is then evaluated for EVERY
// rank from the same matrix, so a capacity failure is a collective decision: all ranks
// fail together instead of one rank leaving the others blocked in the next collective.
template <class Need>
static bool swap_counts(sph_ctx* c, int64_t base, Need&& need) {
  Dist& D = *c->dist;
  const int G = D.G, W = G + 1;
  std::vector<int64_t> row(W);
  for (int r = 0; r < G; ++r) row[r] = D.scnt[r];
  row[G] = base;
  CUK(cudaMemcpyAsync(D.cnt_d, row.data(), sizeof(int64_t) * W, cudaMemcpyHostToDevice, c->stream));
  COMM(allgather(D.cnt_d, D.cnt_all_d, W, DType::I64, c->stream, c->dist_err));
  std::vector<int64_t> all((size_t)G * W);
  CUK(cudaMemcpyAsync(all.data(), D.cnt_all_d, sizeof(int64_t) * G * W, cudaMemcpyDeviceToHost, c->stream));
  CUK(cudaStreamSynchronize(c->stream));
  for (int s = 0; s < G; ++s) D.rcnt[s] = s == D.rank ? 0 : all[(size_t)s * W + D.rank];
  D.moved_total = 0;
  for (int s = 0; s < G; ++s) {
    int64_t sent = 0, recv = 0;
    for (int r = 0; r < G; ++r) {
      if (r == s) continue;
      sent += all[(size_t)s * W + r];
      recv += all[(size_t)r * W + s];
    }
    D.moved_total += sent;
    if (!need(sent, recv, all[(size_t)s * W + G])) {
      c->dist_err = "rank " + std::to_string(s) + " would exceed its particle capacity (sends " +
                    std::to_string(sent) + ", receives " + std::to_string(recv) +
                    "); raise the capacity passed to sph_init";
      return false;
    }
  }
  return true;
}

bool dist_global_bbox(sph_ctx* c, double* bb_out, bool* bad_any) {
  Dist& D = *c->dist;
  k_bbox_pack<<<1, 1, 0, c->stream>>>(c->s.bbox, c->P.n, c->s.bad_id, c->s.cnt, D.red_d, D.red_d + 9);
  COMM(allreduce(D.red_d, D.red_d, 9, DType::F64, ROp::Max, c->stream, c->dist_err));
  COMM(allreduce(D.red_d + 9, D.red_d + 9, 2, DType::F64, ROp::Sum, c->stream, c->dist_err));
  double v[11];
  CUK(cudaMemcpyAsync(v, D.red_d, sizeof(v), cudaMemcpyDeviceToHost, c->stream));
  CUK(cudaStreamSynchronize(c->stream));
  bb_out[0] = -v[0]; bb_out[1] = -v[1]; bb_out[2] = -v[2];
  bb_out[3] = v[3]; bb_out[4] = v[4]; bb_out[5] = v[5];
  bb_out[6] = v[6]; bb_out[7] = v[9]; bb_out[8] = v[7];
  *bad_any = v[8] != 0.0;
  D.n_total = (int64_t)v[10];
  return true;
}

// splitters from the global key-prefix histogram; ranges of the sorted owned array
bool dist_splitters(sph_ctx* c) {
  Dist& D = *c->dist;
  const Grid& g = c->grid;
  const int mbits = 3 * g.cbits;
  // bins are whole pair-pass units (shift >= ubits): a unit never straddles two ranks,
  // so every rank stages the same unit stencils as one GPU does (bit-identical sums)
  int shift = mbits > kBinBits ? mbits - kBinBits : 0;
  if (shift < g.ubits) shift = g.ubits < mbits ? g.ubits : mbits;
  // lazy re-decomposition: keep the splitters for `every` steps while the bin
  // space is unchanged; migration below still moves every particle to its owner
  const bool keep = D.have_split && D.every > 1 && (D.decomp_calls % D.every) != 0 && shift == D.shift &&
                    ((int64_t)1 << (mbits - shift)) == D.nbins;
  ++D.decomp_calls;
  if (keep) return true;
  D.shift = shift;
  D.have_split = true;
  D.nbins = (int64_t)1 << (mbits - D.shift);
  CUK(cudaMemsetAsync(D.hist_d, 0, sizeof(unsigned long long) * D.nbins, c->stream));
  if (c->P.n) {
    k_bin_hist<<<grid_blocks(c, c->P.n, 256, 8), 256, 0, c->stream>>>(c->s.keys, c->P.n, g, D.shift, D.hist_d);
    c->launches++;
  }
  COMM(allreduce(D.hist_d, D.hist_d, D.nbins, DType::U64, ROp::Sum, c->stream, c->dist_err));
  std::vector<int64_t> hist(D.nbins);
  CUK(cudaMemcpyAsync(hist.data(), D.hist_d, sizeof(int64_t) * D.nbins, cudaMemcpyDeviceToHost, c->stream));
  CUK(cudaStreamSynchronize(c->stream));
  compute_splitters(hist.data(), D.nbins, D.G, D.split.data());
  CUK(cudaMemcpyAsync(D.split_d, D.split.data(), sizeof(int64_t) * (D.G + 1), cudaMemcpyHostToDevice, c->stream));
  return true;
}

// a14: ship particles outside this rank's key range to their owners.  Keys
// of the owned set are current (unsorted).  After the leavers are packed, stayers
// from the tail fill their holes and arrivals land behind: the new owned set is
// [0, n - nleave + nrecv), unsorted -- sort_migrate sorts it once.
bool dist_migrate(sph_ctx* c, int64_t* nleave, int64_t* nrecv) {
  Dist& D = *c->dist;
  const int G = D.G;
  const int64_t n = c->P.n;
  *nleave = *nrecv = 0;
  CUK(cudaMemsetAsync(D.tot_d, 0, sizeof(int64_t) * G, c->stream));
  if (n) {
    k_owner_count<<<grid_blocks(c, n, 256, 8), 256, 0, c->stream>>>(
        c->s.keys, n, c->grid, D.shift, D.split_d, G, D.rank, D.pcnt_d, (unsigned long long*)D.tot_d);
    c->launches++;
  }
  std::vector<int64_t> tot(G);
  CUK(cudaMemcpyAsync(tot.data(), D.tot_d, sizeof(int64_t) * G, cudaMemcpyDeviceToHost, c->stream));
  CUK(cudaStreamSynchronize(c->stream));
  int64_t off = 0;
  for (int r = 0; r < G; ++r) {
    D.soff[r] = off;
    D.scnt[r] = r == D.rank ? 0 : tot[r];
    off += D.scnt[r];
  }
  const int64_t cap = c->cap, xcap = D.xcap;
  if (!swap_counts(c, n, [&](int64_t sent, int64_t recv, int64_t nb) {
        return nb - sent + recv <= cap && sent <= xcap && recv <= xcap;
      }))
    return false;
  if (D.moved_total == 0) return true;
  for (int r = 0; r < G; ++r) {
    *nleave += D.scnt[r];
    *nrecv += D.rcnt[r];
  }
  const int64_t n_keep = n - *nleave;
  uint32_t* holes = c->s.cell_flag;   // scratch until launch_cells rebuilds the cell tables
  uint32_t* movers = c->s.cell_rank;
  if (*nleave) {
    CUK(cudaMemcpyAsync(D.off_d, D.soff.data(), sizeof(int64_t) * G, cudaMemcpyHostToDevice, c->stream));
    CUK(cudaMemsetAsync(D.cnt_d, 0, sizeof(int64_t) * (G + 1), c->stream));
    CUK(cudaMemsetAsync(D.hm_d, 0, sizeof(unsigned long long) * 2, c->stream));
    k_owner_fill<<<grid_blocks(c, n, 256, 8), 256, 0, c->stream>>>(
        n, n_keep, D.pcnt_d, D.rank, D.off_d, (unsigned long long*)D.cnt_d, D.send_idx, D.hm_d, holes,
        movers);
    c->launches++;
  }
  FieldSet fs = state_fields(c, true);
  if (!exchange(c, fs, c->stream)) return false;  // packs the leavers (stream order: before the moves)
  if (*nleave) {
    // holes below n_keep == stayers at or above n_keep (both equal nleave minus the
    // leavers already at or above n_keep); the host does not need the count
    k_fill_holes_dev<<<grid_blocks(c, *nleave, 256, 8), 256, 0, c->stream>>>(fs, holes, movers, D.hm_d);
    c->launches++;
  }
  return unpack_all(c, fs, n_keep, c->stream);
}

// halo plan (who needs which of my cells) + exchange #1 (x, v, h, m, u, id)
bool dist_halo_plan_and_exchange1(sph_ctx* c) {
  Dist& D = *c->dist;
  const Grid& g = c->grid;
  const int G = D.G;
  const double reach = reach_of(c->hmax);
  const int Rx = stencil_radius(g, 0, reach), Ry = stencil_radius(g, 1, reach), Rz = stencil_radius(g, 2, reach);
  const int64_t n = c->P.n;
  const int nbc = grid_blocks(c, n, 256, 8);
  k_halo_mask<<<nbc, 256, 0, c->stream>>>(c->s.cell_list, c->s.ncell_list, g, Rx, Ry, Rz, D.split_d, G,
                                          D.rank, D.shift, D.mask_d);
  c->launches++;
  // pass 1: per-peer totals only (nothing written yet), then a collective capacity check
  CUK(cudaMemsetAsync(D.tot_d, 0, sizeof(int64_t) * G, c->stream));
  k_peer_totals<<<nbc, 256, 0, c->stream>>>(c->s.cell_list, c->s.ncell_list, c->s.cell_start, c->s.cell_end,
                                            D.mask_d, G, (unsigned long long*)D.tot_d);
  c->launches++;
  std::vector<int64_t> tot(G, 0);
  uint32_t ncl = 0;
  CUK(cudaMemcpyAsync(tot.data(), D.tot_d, sizeof(int64_t) * G, cudaMemcpyDeviceToHost, c->stream));
  CUK(cudaMemcpyAsync(&ncl, c->s.ncell_list, sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
  CUK(cudaStreamSynchronize(c->stream));
  int64_t total = 0;
  for (int r = 0; r < G; ++r) {
    D.soff[r] = total;
    D.scnt[r] = r == D.rank ? 0 : tot[r];
    total += D.scnt[r];
  }
  const int64_t cap = c->cap, xcap = D.xcap;
  if (!swap_counts(c, n, [&](int64_t sent, int64_t recv, int64_t nb) {
        return sent <= xcap && recv <= xcap && nb + recv <= cap;
      }))
    return false;
  // pass 2: fill the per-peer send lists (cells in Morton order -> key-sorted halos)
  const int nbl = grid_blocks(c, ncl, 256, 8);
  for (int r = 0; r < G; ++r) {
    if (r == D.rank || D.scnt[r] == 0) continue;
    k_peer_counts<<<nbl, 256, 0, c->stream>>>(c->s.cell_list, c->s.ncell_list, c->s.cell_start, c->s.cell_end,
                                              D.mask_d, r, D.pcnt_d);
    scan_u32(c, D.pcnt_d, D.poff_d, ncl);
    k_fill_send<<<nbl, 256, 0, c->stream>>>(c->s.cell_list, c->s.ncell_list, c->s.cell_start, c->s.cell_end,
                                            D.mask_d, r, D.poff_d, D.send_idx + D.soff[r]);
    c->launches += 4;
  }
  D.n_halo = 0;
  for (int r = 0; r < G; ++r) D.n_halo += D.rcnt[r];
  FieldSet fs = state_fields(c, false);
  if (!exchange(c, fs, c->stream)) return false;
  return unpack_all(c, fs, n, c->stream);
}

// Exchanges #2 and #3 (R21) overlap the interior units' passes (SURVEY 8(f) NEXT-3,
// P:388): packed on the compute stream, sent / received / unpacked on the comm stream,
// and an event the compute stream waits on before the boundary units (dist_wait_halo).
bool dist_exchange2(sph_ctx* c) {  // after density: quantities IAD / momentum read at sources
  Dist& D = *c->dist;
  FieldSet fs{};
  fs.f[0] = (uint64_t*)c->s.vol;
  fs.f[1] = (uint64_t*)c->s.ih2;
  fs.f[2] = (uint64_t*)c->P.c;
  fs.f[3] = (uint64_t*)c->s.mX;
  fs.nf = 4;
  if (!exchange(c, fs, D.cstream) || !unpack_all(c, fs, c->P.n, D.cstream)) return false;
  CUK(cudaEventRecord(D.ev_halo, D.cstream));
  return true;
}

bool dist_exchange3(sph_ctx* c) {  // after IAD: C~ = (B/h^3) C of the sources, then their records
  Dist& D = *c->dist;
  FieldSet fs{};
  for (int k = 0; k < 6; ++k) fs.f[k] = (uint64_t*)(c->s.ct + (size_t)k * c->cap);
  fs.nf = 6;
  if (!exchange(c, fs, D.cstream) || !unpack_all(c, fs, c->P.n, D.cstream)) return false;
  c->launches += launch_mom_records_range(c, c->P.n, c->n_halo, D.cstream);  // halo sources
  CUK(cudaGetLastError());
  CUK(cudaEventRecord(D.ev_halo, D.cstream));
  return true;
}

bool dist_wait_halo(sph_ctx* c) {  // the compute stream waits for the last async exchange
  CUK(cudaStreamWaitEvent(c->stream, c->dist->ev_halo, 0));
  return true;
}

bool dist_allreduce_dt(sph_ctx* c) {
  COMM(allreduce(c->s.dts + DT_RAW_BITS, c->s.dts + DT_RAW_BITS, 1, DType::U64, ROp::Min, c->stream,
                 c->dist_err));
  return true;
}

bool dist_allreduce_diag(sph_ctx* c, double* d_dev, unsigned long long* cnt_dev) {
  Dist& D = *c->dist;
  COMM(allreduce(d_dev, d_dev, 8, DType::F64, ROp::Sum, c->stream, c->dist_err));
  COMM(allreduce(cnt_dev, D.cntred_d, kCounters, DType::U64, ROp::Sum, c->stream, c->dist_err));
  return true;
}

bool dist_init(sph_ctx* c, const sph_params* prm) {
  Dist* D = new Dist();
  c->dist = D;
  D->G = prm->nranks;
  D->rank = prm->rank;
  D->every = prm->redecomp_every > 1 ? prm->redecomp_every : 1;
  D->split.assign(D->G + 1, 0);
  D->soff.assign(D->G, 0);
  D->scnt.assign(D->G, 0);
  D->rcnt.assign(D->G, 0);
  D->comm = comm_create(prm->nccl_unique_id, D->G, D->rank, c->dist_err);
  if (!D->comm) return false;
  CUK(cudaStreamCreateWithFlags(&D->cstream, cudaStreamNonBlocking));
  CUK(cudaEventCreateWithFlags(&D->ev_pack, cudaEventDisableTiming));
  CUK(cudaEventCreateWithFlags(&D->ev_halo, cudaEventDisableTiming));
  D->xcap = c->cap;
  const int64_t cap = c->cap;
  CUK(cudaMalloc(&D->hist_d, sizeof(unsigned long long) << kBinBits));
  CUK(cudaMalloc(&D->split_d, sizeof(int64_t) * (D->G + 1)));
  CUK(cudaMalloc(&D->off_d, sizeof(int64_t) * (D->G + 1)));
  CUK(cudaMalloc(&D->cnt_d, sizeof(int64_t) * (D->G + 1)));
  CUK(cudaMalloc(&D->cnt_all_d, sizeof(int64_t) * D->G * (D->G + 1)));
  CUK(cudaMalloc(&D->tot_d, sizeof(int64_t) * D->G));
  CUK(cudaMalloc(&D->red_d, sizeof(double) * 16));
  CUK(cudaMalloc(&D->cntred_d, sizeof(unsigned long long) * kCounters));
  CUK(cudaMalloc(&D->hm_d, sizeof(unsigned long long) * 2));
  CUK(cudaMalloc(&D->mask_d, sizeof(unsigned long long) * cap));
  CUK(cudaMalloc(&D->pcnt_d, sizeof(uint32_t) * cap));
  CUK(cudaMalloc(&D->poff_d, sizeof(uint32_t) * cap));
  CUK(cudaMalloc(&D->send_idx, sizeof(uint32_t) * D->xcap));
  CUK(cudaMalloc(&D->sendbuf, sizeof(uint64_t) * 14 * D->xcap));
  CUK(cudaMalloc(&D->recvbuf, sizeof(uint64_t) * 14 * D->xcap));
  return true;
}

int64_t dist_memory_bytes(const sph_ctx* c) {
  const Dist& D = *c->dist;
  const int64_t cap = c->cap, G = D.G;
  return (int64_t)(sizeof(unsigned long long) << kBinBits) + 8 * (4 * (G + 1) + G * (G + 1) + G + 16 + kCounters + 2) +
         cap * (8 + 4 + 4) + D.xcap * (4 + 2 * 8 * 14);
}

void dist_destroy(sph_ctx* c) {
  Dist* D = c->dist;
  if (!D) return;
  delete D->comm;
  if (D->cstream) cudaStreamSynchronize(D->cstream), cudaStreamDestroy(D->cstream);
  if (D->ev_pack) cudaEventDestroy(D->ev_pack);
  if (D->ev_halo) cudaEventDestroy(D->ev_halo);
  void* ptrs[] = {D->hist_d, D->split_d, D->off_d, D->cnt_d, D->cnt_all_d, D->tot_d, D->red_d,
                  D->mask_d, D->pcnt_d, D->poff_d, D->send_idx, D->sendbuf, D->recvbuf, D->cntred_d,
                  D->hm_d};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  delete D;
  c->dist = nullptr;
}



}  // namespace sphb

extern "C" sph_status sph_local_comm_id(int nranks, void* out, int size) {
  if (!out || size < sphb::kCommIdBytes || nranks < 1 || nranks > 64) return SPH_ERR_CONFIG;
  return sphb::local_hub_create(nranks, out) ? SPH_OK : SPH_ERR_CONFIG;
}

extern "C" sph_status sph_nccl_unique_id(void* out, int size) {
#ifdef SPH_WITH_NCCL
  if (!out || size < (int)sizeof(ncclUniqueId)) return SPH_ERR_CONFIG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return SPH_ERR_COMM;
  memcpy(out, &id, sizeof(id));
  return SPH_OK;
#else
  (void)out;
  (void)size;
  return SPH_ERR_CONFIG;
#endif
}

// host-side decomposition helpers, exported for CPU tests (no GPU needed)
extern "C" int sph_decomp_splitters(const int64_t* hist, int64_t nbins, int G, int64_t* split) {
  if (!hist || !split || G < 1 || nbins < 1) return SPH_ERR_CONFIG;
  sphb::compute_splitters(hist, nbins, G, split);
  return SPH_OK;
}
extern "C" int sph_decomp_owner(const int64_t* split, int G, int64_t bin) {
  return sphb::owner_of_bin(split, G, bin);
}
