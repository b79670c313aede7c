// sph_dist.cuh -- state of the multi-GPU decomposition (see sph_dist.cu).
#pragma once

#include <vector>

#include "comm.cuh"
#include "sph_internal.cuh"

namespace sphb {

constexpr int kBinBits = 16;  // key-prefix histogram: 2^16 bins (top Morton bits)

struct Dist {
  int G = 1, rank = 0;
  Comm* comm = nullptr;     // NCCL or the in-process hub (comm.cuh)
  cudaStream_t cstream = nullptr;   // overlapped halo exchanges #2 / #3
  cudaEvent_t ev_pack = nullptr, ev_halo = nullptr;
  int shift = 0;            // bin = Morton(cell) >> shift
  int every = 1;            // recompute splitters every k-th step (sph_params.redecomp_every)
  int64_t decomp_calls = 0; // dist_splitters calls so far
  bool have_split = false;
  int64_t nbins = 1;
  int64_t n_total = 0;      // particles over all ranks
  int64_t n_halo = 0;
  int64_t xcap = 0;         // capacity of send lists / buffers (particles)
  int64_t moved_total = 0;  // particles exchanged by the last swap, all ranks
  std::vector<int64_t> split;  // G + 1 bin boundaries
  std::vector<int64_t> soff, scnt, rcnt;
  unsigned long long* hist_d = nullptr;
  int64_t *split_d = nullptr, *off_d = nullptr, *cnt_d = nullptr, *cnt_all_d = nullptr, *tot_d = nullptr;
  double* red_d = nullptr;
  unsigned long long* mask_d = nullptr;
  uint32_t *pcnt_d = nullptr, *poff_d = nullptr, *send_idx = nullptr;
  uint64_t *sendbuf = nullptr, *recvbuf = nullptr;
  unsigned long long* cntred_d = nullptr;  // all-reduced event counters
  unsigned long long* hm_d = nullptr;      // migration: hole / mover counters
};

void compute_splitters(const int64_t* hist, int64_t nbins, int G, int64_t* split);
int owner_of_bin(const int64_t* split, int G, int64_t bin);

bool dist_init(sph_ctx* c, const sph_params* prm);
inline int64_t dist_n_total(const sph_ctx* c) { return c->dist->n_total; }
inline int64_t dist_n_halo(const sph_ctx* c) { return c->dist->n_halo; }
inline unsigned long long* dist_counters(const sph_ctx* c) { return c->dist->cntred_d; }
void dist_destroy(sph_ctx* c);
int64_t dist_memory_bytes(const sph_ctx* c);
bool dist_global_bbox(sph_ctx* c, double* bb_out, bool* bad_any);
bool dist_splitters(sph_ctx* c);
bool dist_migrate(sph_ctx* c, int64_t* nleave, int64_t* nrecv);
bool dist_halo_plan_and_exchange1(sph_ctx* c);
bool dist_exchange2(sph_ctx* c);
bool dist_exchange3(sph_ctx* c);
bool dist_wait_halo(sph_ctx* c);
bool dist_allreduce_dt(sph_ctx* c);
bool dist_allreduce_diag(sph_ctx* c, double* d_dev, unsigned long long* cnt_dev);

}  // namespace sphb
