// comm.cu -- the two transports of comm.cuh.
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>

#include "comm.cuh"
#ifdef SPH_WITH_NCCL
#include <nccl.h>
#endif

namespace sphb {

namespace {

size_t dsize(DType) { return 8; }

const char kLocalMagic[8] = {'S', 'P', 'H', 'L', 'O', 'C', 'A', 'L'};

// ------------------------------------------------------------------ in-process hub
struct Hub {
  int G = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  int64_t gen = 0;
  bool broken = false;
  std::vector<const void*> slot;          // per rank: its send buffer of the current collective
  std::vector<std::vector<Xfer>> sends;   // per rank: its sends of the current exchange

  // generation barrier; false after a timeout (a rank died or never came): every later
  // collective on this hub fails instead of hanging
  bool barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (broken) return false;
    const int64_t g = gen;
    if (++arrived == G) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    const bool ok = cv.wait_for(lk, std::chrono::seconds(600), [&] { return gen != g || broken; });
    if (!ok || broken) {
      broken = true;
      cv.notify_all();
      return false;
    }
    return true;
  }
};

std::mutex g_reg_mu;
std::map<uint64_t, std::shared_ptr<Hub>> g_reg;
uint64_t g_next_key = 1;

template <class T>
void reduce_into(T* acc, const T* v, size_t n, ROp op) {
  for (size_t i = 0; i < n; ++i) {
    if (op == ROp::Sum) acc[i] += v[i];
    else if (op == ROp::Max) acc[i] = v[i] > acc[i] ? v[i] : acc[i];
    else acc[i] = v[i] < acc[i] ? v[i] : acc[i];
  }
}

#define LCK(call)                                                              \
  do {                                                                         \
    cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess) {                                                   \
      err = std::string("local comm: ") + #call + ": " + cudaGetErrorString(e_); \
      return false;                                                            \
    }                                                                          \
  } while (0)

class LocalComm : public Comm {
 public:
  LocalComm(std::shared_ptr<Hub> hub, int rank) : hub_(std::move(hub)), rank_(rank) {}
  ~LocalComm() override {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    for (auto it = g_reg.begin(); it != g_reg.end(); ++it)
      if (it->second == hub_ && hub_.use_count() <= 2) {
        g_reg.erase(it);
        break;
      }
  }

  bool allreduce(const void* send, void* recv, size_t count, DType t, ROp op, cudaStream_t s,
                 std::string& err) override {
    const size_t bytes = count * dsize(t);
    LCK(cudaStreamSynchronize(s));  // the send buffer is complete
    hub_->slot[rank_] = send;
    if (!hub_->barrier()) return fail(err);
    std::vector<unsigned char> acc(bytes ? bytes : 1), tmp(bytes ? bytes : 1);
    for (int r = 0; r < hub_->G; ++r) {  // rank order on every rank: identical fp64 sums
      LCK(cudaMemcpyAsync(r == 0 ? acc.data() : tmp.data(), hub_->slot[r], bytes,
                          cudaMemcpyDeviceToHost, s));
      LCK(cudaStreamSynchronize(s));
      if (r == 0) continue;
      if (t == DType::F64)
        reduce_into((double*)acc.data(), (const double*)tmp.data(), count, op);
      else if (t == DType::U64)
        reduce_into((uint64_t*)acc.data(), (const uint64_t*)tmp.data(), count, op);
      else
        reduce_into((int64_t*)acc.data(), (const int64_t*)tmp.data(), count, op);
    }
    if (!hub_->barrier()) return fail(err);  // every rank has read every input
    LCK(cudaMemcpyAsync(recv, acc.data(), bytes, cudaMemcpyHostToDevice, s));
    LCK(cudaStreamSynchronize(s));
    return true;
  }

  bool allgather(const void* send, void* recv, size_t count, DType t, cudaStream_t s,
                 std::string& err) override {
    const size_t bytes = count * dsize(t);
    LCK(cudaStreamSynchronize(s));
    hub_->slot[rank_] = send;
    if (!hub_->barrier()) return fail(err);
    std::vector<unsigned char> all(bytes * hub_->G + 1);
    for (int r = 0; r < hub_->G; ++r)
      LCK(cudaMemcpyAsync(all.data() + bytes * r, hub_->slot[r], bytes, cudaMemcpyDeviceToHost, s));
    LCK(cudaStreamSynchronize(s));
    if (!hub_->barrier()) return fail(err);
    LCK(cudaMemcpyAsync(recv, all.data(), bytes * hub_->G, cudaMemcpyHostToDevice, s));
    LCK(cudaStreamSynchronize(s));
    return true;
  }

  bool exchange(const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs, cudaStream_t s,
                std::string& err) override {
    LCK(cudaStreamSynchronize(s));  // packed send buffers are complete
    hub_->sends[rank_] = sends;
    if (!hub_->barrier()) return fail(err);
    for (const Xfer& r : recvs) {
      const Xfer* src = nullptr;
      for (const Xfer& x : hub_->sends[r.peer])
        if (x.peer == rank_) src = &x;
      if (!src || src->bytes != r.bytes) {
        err = "local comm: unmatched send/recv between ranks " + std::to_string(r.peer) + " and " +
              std::to_string(rank_);
        hub_->barrier();
        return false;
      }
      LCK(cudaMemcpyAsync(r.ptr, src->ptr, r.bytes, cudaMemcpyDefault, s));
    }
    LCK(cudaStreamSynchronize(s));
    if (!hub_->barrier()) return fail(err);  // every receive done: senders may reuse buffers
    return true;
  }

 private:
  bool fail(std::string& err) {
    err = "local comm: a rank did not reach the collective (timeout or earlier failure)";
    return false;
  }
  std::shared_ptr<Hub> hub_;
  int rank_;
};

#ifdef SPH_WITH_NCCL
ncclDataType_t nt(DType t) {
  return t == DType::F64 ? ncclFloat64 : (t == DType::U64 ? ncclUint64 : ncclInt64);
}
ncclRedOp_t nop(ROp o) { return o == ROp::Sum ? ncclSum : (o == ROp::Max ? ncclMax : ncclMin); }

#define NCK(call)                                                         \
  do {                                                                    \
    ncclResult_t r_ = (call);                                             \
    if (r_ != ncclSuccess) {                                              \
      err = std::string(#call) + ": " + ncclGetErrorString(r_);           \
      return false;                                                       \
    }                                                                     \
  } while (0)

class NcclComm : public Comm {
 public:
  ncclComm_t comm = nullptr;
  ~NcclComm() override {
    if (comm) ncclCommDestroy(comm);
  }
  bool allreduce(const void* send, void* recv, size_t count, DType t, ROp op, cudaStream_t s,
                 std::string& err) override {
    NCK(ncclAllReduce(send, recv, count, nt(t), nop(op), comm, s));
    return true;
  }
  bool allgather(const void* send, void* recv, size_t count, DType t, cudaStream_t s,
                 std::string& err) override {
    NCK(ncclAllGather(send, recv, count, nt(t), comm, s));
    return true;
  }
  bool exchange(const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs, cudaStream_t s,
                std::string& err) override {
    NCK(ncclGroupStart());
    for (const Xfer& x : sends) NCK(ncclSend(x.ptr, x.bytes, ncclUint8, x.peer, comm, s));
    for (const Xfer& x : recvs) NCK(ncclRecv(x.ptr, x.bytes, ncclUint8, x.peer, comm, s));
    NCK(ncclGroupEnd());
    return true;
  }
};
#endif

}  // namespace

bool comm_id_is_local(const void* id) { return id && memcmp(id, kLocalMagic, 8) == 0; }

bool local_hub_create(int G, void* id_out) {
  if (G < 1 || !id_out) return false;
  auto hub = std::make_shared<Hub>();
  hub->G = G;
  hub->slot.assign(G, nullptr);
  hub->sends.assign(G, {});
  uint64_t key;
  {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    key = g_next_key++;
    g_reg[key] = hub;
  }
  memset(id_out, 0, kCommIdBytes);
  memcpy(id_out, kLocalMagic, 8);
  memcpy((char*)id_out + 8, &key, 8);
  memcpy((char*)id_out + 16, &G, sizeof(int));
  return true;
}

Comm* comm_create(const void* id, int G, int rank, std::string& err) {
  if (comm_id_is_local(id)) {
    uint64_t key;
    int hg;
    memcpy(&key, (const char*)id + 8, 8);
    memcpy(&hg, (const char*)id + 16, sizeof(int));
    std::shared_ptr<Hub> hub;
    {
      std::lock_guard<std::mutex> lk(g_reg_mu);
      auto it = g_reg.find(key);
      if (it != g_reg.end()) hub = it->second;
    }
    if (!hub || hg != G) {
      err = "local comm: unknown hub id or rank count mismatch";
      return nullptr;
    }
    return new LocalComm(hub, rank);
  }
#ifdef SPH_WITH_NCCL
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  NcclComm* c = new NcclComm();
  ncclResult_t r = ncclCommInitRank(&c->comm, G, uid, rank);
  if (r != ncclSuccess) {
    err = std::string("ncclCommInitRank: ") + ncclGetErrorString(r);
    c->comm = nullptr;
    delete c;
    return nullptr;
  }
  return c;
#else
  err = "built without NCCL (only the in-process transport is available)";
  return nullptr;
#endif
}

}  // namespace sphb
