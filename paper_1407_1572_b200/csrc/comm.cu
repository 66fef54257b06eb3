// Transports and the subtree partition of the sharded factorization
// (comm.cuh).  NCCL is resolved with dlopen so the library has no link-time
// NCCL dependency and shares the process's copy with torch.distributed.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>

#include "comm.cuh"

namespace ifmm {

// -------------------------------------------------------------- NCCL
struct NcclApi {
  decltype(&ncclGetVersion) GetVersion = nullptr;
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclAllGather) AllGather = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
};

static const NcclApi& nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    // prefer a copy the process already has (torch's), then IFMM_NCCL_LIB, then the system one
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h && getenv("IFMM_NCCL_LIB")) h = dlopen(getenv("IFMM_NCCL_LIB"), RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
#define IFMM_NCCL_SYM(name) api.name = reinterpret_cast<decltype(api.name)>(dlsym(h, "nccl" #name))
    IFMM_NCCL_SYM(GetVersion);
    IFMM_NCCL_SYM(GetUniqueId);
    IFMM_NCCL_SYM(CommInitRank);
    IFMM_NCCL_SYM(CommDestroy);
    IFMM_NCCL_SYM(AllGather);
    IFMM_NCCL_SYM(Send);
    IFMM_NCCL_SYM(Recv);
    IFMM_NCCL_SYM(GroupStart);
    IFMM_NCCL_SYM(GroupEnd);
    IFMM_NCCL_SYM(GetErrorString);
#undef IFMM_NCCL_SYM
    if (!api.GetUniqueId || !api.CommInitRank || !api.AllGather || !api.Send || !api.Recv || !api.GroupStart ||
        !api.GroupEnd || !api.CommDestroy)
      err = "libnccl.so.2 lacks a required symbol";
  });
  if (!err.empty()) throw Error(IFMM_CUDA, err);
  return api;
}

static void nccl_check(const NcclApi& a, ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  char buf[256];
  snprintf(buf, sizeof buf, "NCCL %s failed: %s", what, a.GetErrorString ? a.GetErrorString(r) : "?");
  throw Error(IFMM_CUDA, buf);
}

void nccl_unique_id(void* out128) {
  const NcclApi& a = nccl_api();
  ncclUniqueId id;
  nccl_check(a, a.GetUniqueId(&id), "GetUniqueId");
  memcpy(out128, &id, sizeof id);
}

int nccl_version() {
  const NcclApi& a = nccl_api();
  int v = 0;
  if (a.GetVersion) a.GetVersion(&v);
  return v;
}

NcclComm::NcclComm(const void* id, int nranks, int rank) {
  api_ = &nccl_api();
  rank_ = rank;
  size_ = nranks;
  ncclUniqueId u;
  memcpy(&u, id, sizeof u);
  ncclComm_t c = nullptr;
  nccl_check(*api_, api_->CommInitRank(&c, nranks, u, rank), "CommInitRank");
  comm_ = c;
}

NcclComm::~NcclComm() {
  if (comm_) api_->CommDestroy(static_cast<ncclComm_t>(comm_));
}

void NcclComm::allgather(const void* dsend, void* drecv, size_t bytes, cudaStream_t s) {
  calls++;
  bytes_meta += double(bytes) * (size_ - 1);
  nccl_check(*api_, api_->AllGather(dsend, drecv, bytes, ncclChar, static_cast<ncclComm_t>(comm_), s), "AllGather");
}

void NcclComm::exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t s) {
  calls++;
  ncclComm_t c = static_cast<ncclComm_t>(comm_);
  nccl_check(*api_, api_->GroupStart(), "GroupStart");
  for (const Msg& m : sends)
    if (m.bytes) {
      bytes_sent += double(m.bytes);
      nccl_check(*api_, api_->Send(m.ptr, m.bytes, ncclChar, m.peer, c, s), "Send");
    }
  for (const Msg& m : recvs)
    if (m.bytes) nccl_check(*api_, api_->Recv(m.ptr, m.bytes, ncclChar, m.peer, c, s), "Recv");
  nccl_check(*api_, api_->GroupEnd(), "GroupEnd");
}

// -------------------------------------------------------------- host-staged
void HostComm::allgather(const void* dsend, void* drecv, size_t bytes, cudaStream_t s) {
  calls++;
  bytes_meta += double(bytes) * (size_ - 1);
  st_.reset();
  char* hs = static_cast<char*>(st_.get(std::max<size_t>(1, bytes)));
  char* hr = static_cast<char*>(st_.get(std::max<size_t>(1, bytes * size_)));
  if (bytes) CK(cudaMemcpyAsync(hs, dsend, bytes, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (ag_(ctx_, hs, hr, int64_t(bytes)) != 0) throw Error(IFMM_CUDA, "host all-gather callback failed");
  if (bytes) CK(cudaMemcpyAsync(drecv, hr, bytes * size_, cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));
}

void HostComm::exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t s) {
  calls++;
  st_.reset();
  std::vector<int32_t> sp, rp;
  std::vector<void*> sb, rb;
  std::vector<int64_t> sn, rn;
  for (const Msg& m : sends) {
    void* h = st_.get(std::max<size_t>(1, m.bytes));
    if (m.bytes) CK(cudaMemcpyAsync(h, m.ptr, m.bytes, cudaMemcpyDeviceToHost, s));
    sp.push_back(m.peer);
    sb.push_back(h);
    sn.push_back(int64_t(m.bytes));
    bytes_sent += double(m.bytes);
  }
  for (const Msg& m : recvs) {
    rp.push_back(m.peer);
    rb.push_back(st_.get(std::max<size_t>(1, m.bytes)));
    rn.push_back(int64_t(m.bytes));
  }
  CK(cudaStreamSynchronize(s));
  if (ex_(ctx_, int(sp.size()), sp.data(), sb.data(), sn.data(), int(rp.size()), rp.data(), rb.data(), rn.data()) != 0)
    throw Error(IFMM_CUDA, "host exchange callback failed");
  for (size_t q = 0; q < recvs.size(); q++)
    if (recvs[q].bytes) CK(cudaMemcpyAsync(recvs[q].ptr, rb[q], recvs[q].bytes, cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));
}

// -------------------------------------------------------------- threads
void LocalWorld::barrier() {
  std::unique_lock<std::mutex> lk(mu);
  if (abort) throw Error(IFMM_CUDA, "another virtual rank failed");
  const long long g = gen;
  if (++arrived == size) {
    arrived = 0;
    gen++;
    cv.notify_all();
    return;
  }
  cv.wait(lk, [&] { return gen != g || abort; });
  if (gen == g) throw Error(IFMM_CUDA, "another virtual rank failed");
}

void LocalWorld::fail() {
  std::lock_guard<std::mutex> lk(mu);
  abort = true;
  cv.notify_all();
}

void LocalComm::allgather(const void* dsend, void* drecv, size_t bytes, cudaStream_t s) {
  calls++;
  bytes_meta += double(bytes) * (size_ - 1);
  CK(cudaStreamSynchronize(s));  // the contribution is complete before peers read it
  w_->posted_ptr[rank_] = dsend;
  w_->barrier();
  for (int p = 0; p < size_; p++)
    if (bytes)
      CK(cudaMemcpyAsync(static_cast<char*>(drecv) + size_t(p) * bytes, w_->posted_ptr[p], bytes,
                         cudaMemcpyDeviceToDevice, s));
  CK(cudaStreamSynchronize(s));
  w_->barrier();  // peers may reuse their buffers after everyone has read them
}

void LocalComm::exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t s) {
  calls++;
  CK(cudaStreamSynchronize(s));
  w_->posted_sends[rank_] = sends;
  w_->barrier();
  std::vector<size_t> used(size_, 0);  // per source: messages to me consumed so far
  std::string bad;
  for (const Msg& r : recvs) {
    const std::vector<Msg>& ps = w_->posted_sends[r.peer];
    size_t seen = 0;
    const Msg* m = nullptr;
    for (const Msg& c : ps)
      if (c.peer == rank_ && seen++ == used[r.peer]) {
        m = &c;
        break;
      }
    used[r.peer]++;
    if (!m || m->bytes != r.bytes) {
      char buf[160];
      snprintf(buf, sizeof buf, "exchange mismatch: rank %d expects %zu bytes from %d, peer sends %zu", rank_, r.bytes,
               r.peer, m ? m->bytes : size_t(0));
      bad = buf;
      break;
    }
    if (r.bytes) CK(cudaMemcpyAsync(r.ptr, m->ptr, r.bytes, cudaMemcpyDeviceToDevice, s));
  }
  if (bad.empty())
    for (int p = 0; p < size_; p++) {  // every message sent to me must have been received
      size_t cnt = 0;
      for (const Msg& c : w_->posted_sends[p]) cnt += c.peer == rank_;
      if (p != rank_ && cnt != used[p]) {
        char buf[160];
        snprintf(buf, sizeof buf, "exchange mismatch: rank %d sends %zu messages to %d, which expects %zu", p, cnt,
                 rank_, used[p]);
        bad = buf;
      }
    }
  for (const Msg& m : sends) bytes_sent += double(m.bytes);
  CK(cudaStreamSynchronize(s));
  if (!bad.empty()) {
    w_->fail();
    throw Error(IFMM_INVALID, bad);
  }
  w_->barrier();
}

// -------------------------------------------------------------- partition
Partition make_partition(int dim, int depth, int nranks, int rank, const std::vector<std::vector<int>>& grid) {
  Partition P;
  P.nranks = nranks;
  P.rank = rank;
  P.dim = dim;
  P.depth = depth;
  const int nc2 = 1 << (2 * dim);
  if (nranks < 1 || nranks > nc2) {
    char buf[128];
    snprintf(buf, sizeof buf, "subtree partition needs 1 <= ranks <= %d (level-2 clusters), got %d", nc2, nranks);
    invalid(buf);
  }
  if (rank < 0 || rank >= nranks) invalid("rank out of range");
  P.owner.assign(depth + 1, {});
  P.held.assign(depth + 1, {});
  for (int k = 2; k <= depth; k++) {
    const int nc = 1 << (dim * k);
    std::vector<int>& ow = P.owner[k];
    ow.resize(nc);
    for (int i = 0; i < nc; i++) ow[i] = int((int64_t(i >> (dim * (k - 2))) * nranks) / nc2);
    P.held[k].assign(nranks, std::vector<uint8_t>(nc, 0));
    const std::vector<int>& g = grid[k];
    const int side = 1 << k;
    // cluster index of grid coordinates (Morton, axis 0 least significant)
    auto index = [&](const int* c) {
      int64_t m = 0;
      for (int b = 0; b < k; b++)
        for (int ax = 0; ax < dim; ax++) m |= int64_t((c[ax] >> b) & 1) << (b * dim + ax);
      return int(m);
    };
    for (int i = 0; i < nc; i++) {
      if (k == 2) {
        for (int s = 0; s < nranks; s++) P.held[k][s][i] = 1;
        continue;
      }
      int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0}, c[3] = {0, 0, 0};
      for (int d = 0; d < dim; d++) {
        lo[d] = std::max(0, g[i * dim + d] - 1);
        hi[d] = std::min(side - 1, g[i * dim + d] + 1);
      }
      for (c[0] = lo[0]; c[0] <= hi[0]; c[0]++)
        for (c[1] = lo[1]; c[1] <= hi[1]; c[1]++)
          for (c[2] = lo[2]; c[2] <= hi[2]; c[2]++) P.held[k][ow[index(c)]][i] = 1;
    }
  }
  return P;
}

Partition make_partition_geometric(int dim, int depth, int nranks, int rank) {
  if (dim < 1 || dim > 3 || depth < 2 || depth > (dim == 3 ? 9 : 14)) invalid("bad dim / depth");
  std::vector<std::vector<int>> grid(depth + 1);
  for (int k = 2; k <= depth; k++) {
    const int nc = 1 << (dim * k);
    grid[k].assign(size_t(nc) * dim, 0);
    for (int i = 0; i < nc; i++)
      for (int b = 0; b < k; b++)
        for (int ax = 0; ax < dim; ax++) grid[k][size_t(i) * dim + ax] |= ((i >> (b * dim + ax)) & 1) << b;
  }
  return make_partition(dim, depth, nranks, rank, grid);
}

void halo_plan_counts(const Partition& P, int level, int colour, std::vector<int>& send, std::vector<int>& recv) {
  const int dim = P.dim, k = level, side = 1 << k, nc = 1 << (dim * k);
  send.assign(P.nranks, 0);
  recv.assign(P.nranks, 0);
  auto grid = [&](int i, int* g) {
    for (int d = 0; d < dim; d++) g[d] = 0;
    for (int b = 0; b < k; b++)
      for (int ax = 0; ax < dim; ax++) g[ax] |= ((i >> (b * dim + ax)) & 1) << b;
  };
  auto index = [&](const int* c) {
    int m = 0;
    for (int b = 0; b < k; b++)
      for (int ax = 0; ax < dim; ax++) m |= ((c[ax] >> b) & 1) << (b * dim + ax);
    return m;
  };
  auto cheb = [&](int i, int j) {
    int gi[3], gj[3], d = 0;
    grid(i, gi);
    grid(j, gj);
    for (int ax = 0; ax < dim; ax++) d = std::max(d, std::abs(gi[ax] - gj[ax]));
    return d;
  };
  auto parent_adjacent = [&](int i, int j) { return cheb(i >> dim, j >> dim) <= 1; };
  for (int i = 0; i < nc; i++) {
    int g[3] = {0, 0, 0};
    grid(i, g);
    int col = 0, mul = 1;
    for (int d = 0; d < dim; d++) {
      col += (g[d] % 3) * mul;
      mul *= 3;
    }
    if (col != colour) continue;
    std::vector<int> xp;
    int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0}, c[3] = {0, 0, 0};
    for (int d = 0; d < dim; d++) {
      lo[d] = std::max(0, g[d] - 1);
      hi[d] = std::min(side - 1, g[d] + 1);
    }
    for (c[0] = lo[0]; c[0] <= hi[0]; c[0]++)
      for (c[1] = lo[1]; c[1] <= hi[1]; c[1]++)
        for (c[2] = lo[2]; c[2] <= hi[2]; c[2]++) {
          const int j = index(c);
          if (j != i) xp.push_back(j);
        }
    std::sort(xp.begin(), xp.end());
    const int w = P.owner[k][i];
    auto route = [&](int a, int b) {
      if (halo_route(P, k, w, P.rank, a, b, [&](int s) { send[s]++; })) recv[w]++;
    };
    for (size_t u = 0; u < xp.size(); u++)
      for (size_t v = u; v < xp.size(); v++) {
        route(xp[u], xp[v]);                                          // P2P Schur targets
        if (cheb(xp[u], xp[v]) > 1 && (k <= 1 || parent_adjacent(xp[u], xp[v]))) route(xp[u], xp[v]);  // M2L
      }
    for (int x : xp) route(x, -1);  // augmented bases
  }
}

}  // namespace ifmm
