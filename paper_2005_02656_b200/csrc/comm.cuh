// comm.cuh -- the collectives the multi-GPU decomposition needs (sph_dist.cu):
// allreduce (sum / max / min), allgather and grouped point-to-point transfers.
//
// Two transports behind one interface:
//  * NcclComm   -- one process per GPU, NCCL over NVLink / NVSwitch (the product path);
//  * LocalComm  -- G ranks as G host threads of ONE process (sharing one or more devices),
//                  each rank its own sph_ctx: collectives meet at an in-process hub and
//                  move data with device-to-device copies.  It runs the whole decomposition
//                  data path (splitters, migration, halo plan, pack/unpack, three exchanges,
//                  dt / diagnostics reductions) on a single GPU, so the driver's 1-GPU test
//                  box exercises it; results are identical to the NCCL transport's because
//                  every reduction it performs is exact (max / min / integer sums) or, for
//                  the fp64 sums, summed in rank order on every rank.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

namespace sphb {

enum class DType { F64, U64, I64 };
enum class ROp { Sum, Max, Min };

struct Xfer {  // one send or receive of a grouped point-to-point exchange
  int peer;
  void* ptr;
  size_t bytes;
};

struct Comm {
  virtual ~Comm() {}
  // every call is collective over the G ranks and stream-ordered on `s`; on return the
  // result is enqueued on `s` (NCCL) or already complete (local).  false + err on failure.
  virtual bool allreduce(const void* send, void* recv, size_t count, DType t, ROp op,
                         cudaStream_t s, std::string& err) = 0;
  virtual bool allgather(const void* send, void* recv, size_t count, DType t, cudaStream_t s,
                         std::string& err) = 0;
  virtual bool exchange(const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs,
                        cudaStream_t s, std::string& err) = 0;
};

constexpr int kCommIdBytes = 128;  // == sizeof(ncclUniqueId)

// Create the transport for rank `rank` of `G` from a 128-byte id: a local hub id
// (sph_local_comm_id) or an NCCL unique id.  nullptr + err on failure.
Comm* comm_create(const void* id, int G, int rank, std::string& err);
bool comm_id_is_local(const void* id);
// a new in-process hub for G ranks; writes its id (kCommIdBytes)
bool local_hub_create(int G, void* id_out);

}  // namespace sphb
