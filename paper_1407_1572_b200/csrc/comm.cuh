// Rank-to-rank transport of the subtree-sharded factorization.
//
// One process per GPU; every rank replays the same host-side schedule, so each
// collective below is entered by all ranks in the same order with sizes every
// rank computes identically.  Two transports:
//   NcclComm  -- NCCL over NVLink/NVSwitch (libnccl resolved at run time with
//                dlopen: the process usually has torch's copy loaded already).
//   LocalComm -- V virtual ranks as host threads of one process on one GPU,
//                each with its own stream and device state; the collectives
//                are device-to-device copies behind a host barrier.  Used to
//                check the sharded schedule on a single GPU (kernels of
//                different virtual ranks never wait on one another).
#pragma once
#include <condition_variable>
#include <memory>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace ifmm {

struct Msg {
  int peer;
  void* ptr;
  size_t bytes;
};

class Comm {
 public:
  virtual ~Comm() {}
  int rank() const { return rank_; }
  int size() const { return size_; }
  // Every rank contributes `bytes` at dsend; drecv (size() * bytes, rank-major)
  // receives all contributions.  Device buffers, ordered on `s`; the data is
  // complete in drecv when the call returns and `s` is synchronised.
  virtual void allgather(const void* dsend, void* drecv, size_t bytes, cudaStream_t s) = 0;
  // Grouped point-to-point transfer: every send is matched by the peer's recv
  // of the same size (messages between a pair are matched in list order).
  // Ordered on `s` like allgather.
  virtual void exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t s) = 0;
  // bytes moved through this communicator (sent by this rank)
  double bytes_sent = 0, bytes_meta = 0;
  long long calls = 0;

 protected:
  int rank_ = 0, size_ = 1;
};

// -------------------------------------------------------------- NCCL
struct NcclApi;  // dlopen'd entry points
class NcclComm : public Comm {
 public:
  // id: 128-byte ncclUniqueId produced by nccl_unique_id() on one rank and
  // shared with the others (the Python side broadcasts it with torch.distributed)
  NcclComm(const void* id, int nranks, int rank);
  ~NcclComm() override;
  void allgather(const void* dsend, void* drecv, size_t bytes, cudaStream_t s) override;
  void exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t s) override;

 private:
  void* comm_ = nullptr;
  const NcclApi* api_ = nullptr;
};
void nccl_unique_id(void* out128);
int nccl_version();

// -------------------------------------------------------------- host-staged
// Collectives through caller-supplied host callbacks (e.g. torch.distributed
// over gloo): device buffers are staged through pinned host memory.  Slow, but
// it runs the real multi-process control flow -- one process per rank, the
// same schedule and messages as NCCL -- on any number of processes sharing
// one GPU (the kernels of different ranks never wait on one another).
typedef int (*HostAllgatherFn)(void* ctx, const void* send, void* recv, int64_t bytes);
typedef int (*HostExchangeFn)(void* ctx, int nsend, const int32_t* send_peer, void* const* send_buf,
                              const int64_t* send_bytes, int nrecv, const int32_t* recv_peer, void* const* recv_buf,
                              const int64_t* recv_bytes);
class HostComm : public Comm {
 public:
  HostComm(int nranks, int rank, HostAllgatherFn ag, HostExchangeFn ex, void* ctx)
      : ag_(ag), ex_(ex), ctx_(ctx) {
    rank_ = rank;
    size_ = nranks;
  }
  void allgather(const void* dsend, void* drecv, size_t bytes, cudaStream_t s) override;
  void exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t s) override;

 private:
  HostAllgatherFn ag_;
  HostExchangeFn ex_;
  void* ctx_;
  Staging st_;
};

// -------------------------------------------------------------- threads
struct LocalWorld {
  explicit LocalWorld(int n) : size(n), posted_ptr(n), posted_sends(n) {}
  int size;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  bool abort = false;
  std::vector<const void*> posted_ptr;
  std::vector<std::vector<Msg>> posted_sends;
  // barrier; throws if another virtual rank failed (so no thread waits forever)
  void barrier();
  void fail();
};

class LocalComm : public Comm {
 public:
  LocalComm(std::shared_ptr<LocalWorld> w, int rank) : w_(std::move(w)) {
    rank_ = rank;
    size_ = w_->size;
  }
  void allgather(const void* dsend, void* drecv, size_t bytes, cudaStream_t s) override;
  void exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t s) override;
  LocalWorld& world() { return *w_; }

 private:
  std::shared_ptr<LocalWorld> w_;
};

// -------------------------------------------------------------- partition
// Subtree partition: level-2 clusters are dealt to ranks in contiguous Morton
// ranges (2 ranks: halves, 4: quadrants, 8: pairs of level-2 cells in 2-D), and
// every cluster of level k >= 2 belongs to the owner of its level-2 ancestor,
// so parent/child work (parent near field, basis row insertion) stays local.
// A rank holds the blocks and bases of every cluster within one cell of its
// own ones (the read/write set of its eliminations); at level 2 every rank
// holds everything (the top-level system is inverted on every rank).
struct Partition {
  int nranks = 1, rank = 0, dim = 2, depth = 0;
  std::vector<std::vector<int>> owner;                   // [k][i]
  std::vector<std::vector<std::vector<uint8_t>>> held;   // [k][s][i]
  bool mine(int k, int i) const { return owner[k][i] == rank; }
  bool holds(int s, int k, int i) const { return held[k][s][i] != 0; }
};
// Routing rule of one halo item (a block (a, b), or the basis of a when b < 0)
// written at level k by a pivot of rank `writer`: the writer sends it to every
// other rank storing it -- to(s) is called for each -- and a non-writer that
// stores it receives it from the writer (returns true).  Every rank evaluates
// the same rule on the same replicated metadata, so sends and receives match.
template <class SendTo>
bool halo_route(const Partition& P, int k, int writer, int me, int a, int b, SendTo to) {
  auto stored = [&](int s) { return P.holds(s, k, a) || (b >= 0 && P.holds(s, k, b)); };
  if (me == writer) {
    for (int s = 0; s < P.nranks; s++)
      if (s != me && stored(s)) to(s);
    return false;
  }
  return stored(me);
}
// Host-only plan check: halo items per peer of one colour batch of `level`
// with the initial block pattern (neighbour P2P pairs, interaction-list M2L
// pairs, bases of the pivots' neighbours), routed by halo_route.
void halo_plan_counts(const Partition& P, int level, int colour, std::vector<int>& send, std::vector<int>& recv);
// grid coordinates of every cluster of every level (g[k][i*dim + d])
Partition make_partition(int dim, int depth, int nranks, int rank, const std::vector<std::vector<int>>& grid);
// the same without a tree (Morton decode of the cluster index): C-ABI test hook
Partition make_partition_geometric(int dim, int depth, int nranks, int rank);

}  // namespace ifmm
