// C ABI (include/ifmm_b200.h): exception -> status translation, handle
// management, accessors and test hooks for the batched kernels.
#include <cstring>
#include <string>

#include "../../include/ifmm_b200.h"
#include "comm.cuh"
#include "core.cuh"
#include "lu.cuh"
#include "compress.cuh"
#include "cta_la.cuh"

using ifmm::AcaOut;
using ifmm::Arena;
using ifmm::CtaShared;
using ifmm::Error;
using ifmm::FactorH;
using ifmm::GemmBatch;
using ifmm::InitLevel;
using ifmm::KernelParams;
using ifmm::LevelStatsH;
using ifmm::MatDesc;
using ifmm::RecordH;
using ifmm::SingularPivot;
using ifmm::Staging;
using ifmm::StoreH;
using ifmm::Topo;
using ifmm::TreeH;
using ifmm::invalid;
using ifmm::ensure_device;
using ifmm::default_stream;
using ifmm::upload;

struct ifmm_tree { TreeH* h; };
struct ifmm_store { StoreH* h; };
struct ifmm_factor { FactorH* h; };
struct ifmm_comm { std::shared_ptr<ifmm::Comm> h; };

namespace ifmm {
void matvec_release(StoreH* S);
}

static thread_local std::string g_err;
static thread_local int g_sing_level = -1, g_sing_index = -1;
static thread_local double g_sing_cond = 0.0;

template <class F>
static int guard(F&& f) {
  try {
    f();
    return IFMM_OK;
  } catch (const SingularPivot& e) {
    g_err = e.what();
    g_sing_level = e.level;
    g_sing_index = e.index;
    g_sing_cond = e.cond;
    return IFMM_SINGULAR_PIVOT;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return IFMM_OOM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return IFMM_CUDA;
  }
}

extern "C" {

const char* ifmm_last_error(void) { return g_err.c_str(); }

int ifmm_last_singular(int* level, int* index, double* cond) {
  if (level) *level = g_sing_level;
  if (index) *index = g_sing_index;
  if (cond) *cond = g_sing_cond;
  return IFMM_OK;
}

int ifmm_version(void) { return 1; }

int ifmm_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int ifmm_set_device(int device) {
  return guard([&] { CK(cudaSetDevice(device)); });
}

// ---------------------------------------------------------------- tree
int ifmm_tree_build(const double* points, int64_t n, int dim, int depth, int ptr_kind, ifmm_tree** out) {
  return guard([&] {
    if (!out) invalid("null output handle");
    TreeH* h = ifmm::tree_build(points, n, dim, depth, ptr_kind == IFMM_PTR_DEVICE);
    *out = new ifmm_tree{h};
  });
}

int ifmm_release_cached_memory(void) {
  return guard([&] {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    ifmm::slab_cache_flush(dev);
  });
}

int ifmm_tree_build_sparse(const double* points, int64_t n, int dim, int depth, int ptr_kind, ifmm_tree** out) {
  return guard([&] {
    if (!out) invalid("null output handle");
    TreeH* h = ifmm::tree_build(points, n, dim, depth, ptr_kind == IFMM_PTR_DEVICE, true);
    *out = new ifmm_tree{h};
  });
}

int ifmm_tree_info(const ifmm_tree* t, int64_t* n, int* dim, int* depth) {
  return guard([&] {
    if (!t) invalid("null tree");
    if (n) *n = t->h->N;
    if (dim) *dim = t->h->dim;
    if (depth) *depth = t->h->depth;
  });
}

int ifmm_tree_permutation(const ifmm_tree* t, int64_t* perm) {
  return guard([&] { memcpy(perm, t->h->perm.data(), sizeof(int64_t) * t->h->perm.size()); });
}

int ifmm_tree_leaf_offsets(const ifmm_tree* t, int64_t* off) {
  return guard([&] { memcpy(off, t->h->leaf_off.data(), sizeof(int64_t) * t->h->leaf_off.size()); });
}

int ifmm_tree_lists(const ifmm_tree* t, int level, int32_t* nbr_off, int32_t* nbr, int32_t* il_off, int32_t* il,
                    int64_t* sizes) {
  return guard([&] {
    if (level < 1 || level > t->h->depth) invalid("level out of range");
    const Topo& T = t->h->lv[level];
    if (sizes) {
      sizes[0] = int64_t(T.nbr.size());
      sizes[1] = int64_t(T.il.size());
    }
    if (nbr_off) memcpy(nbr_off, T.nbr_off.data(), sizeof(int) * T.nbr_off.size());
    if (nbr) memcpy(nbr, T.nbr.data(), sizeof(int) * T.nbr.size());
    if (il_off) memcpy(il_off, T.il_off.data(), sizeof(int) * T.il_off.size());
    if (il) memcpy(il, T.il.data(), sizeof(int) * T.il.size());
  });
}

int ifmm_tree_colours(const ifmm_tree* t, int level, int32_t* colours) {
  return guard([&] {
    if (level < 1 || level > t->h->depth) invalid("level out of range");
    const Topo& T = t->h->lv[level];
    memcpy(colours, T.colour.data(), sizeof(int) * T.colour.size());
  });
}

void ifmm_tree_free(ifmm_tree* t) {
  if (!t) return;
  delete t->h;
  delete t;
}

// ---------------------------------------------------------------- store
int ifmm_store_init(ifmm_tree* t, int kernel_id, double a, double scale, double shift, int p, double tol,
                    const int32_t* probe_table, int probe_maxm, ifmm_store** out) {
  return guard([&] {
    if (!t || !out) invalid("null handle");
    if (!probe_table || probe_maxm < 1) invalid("ACA probe table required");
    KernelParams kp{kernel_id, a, scale, shift};
    StoreH* h = ifmm::store_init(t->h, kp, p, tol, probe_table, probe_maxm);
    *out = new ifmm_store{h};
  });
}

int ifmm_store_max_init_rank(const ifmm_store* s, int* r) {
  return guard([&] { *r = s->h->max_init_rank; });
}

int ifmm_store_dims(const ifmm_store* s, int level, int32_t* n, int32_t* r) {
  return guard([&] {
    if (level < 2 || level > s->h->tree->depth) invalid("level out of range");
    const InitLevel& L = s->h->lv[level];
    if (n) memcpy(n, L.n.data(), sizeof(int) * L.nc);
    if (r) memcpy(r, L.r0.data(), sizeof(int) * L.nc);
  });
}

int ifmm_store_basis(const ifmm_store* s, int level, int index, double* out) {
  return guard([&] {
    if (level < 2 || level > s->h->tree->depth) invalid("level out of range");
    const InitLevel& L = s->h->lv[level];
    if (index < 0 || index >= L.nc) invalid("index out of range");
    CK(cudaMemcpy(out, L.U[index], sizeof(double) * L.n[index] * L.r0[index], cudaMemcpyDeviceToHost));
  });
}

int ifmm_store_m2l(const ifmm_store* s, int level, int i, int j, double* out) {
  return guard([&] {
    if (level < 2 || level > s->h->tree->depth) invalid("level out of range");
    const InitLevel& L = s->h->lv[level];
    const Topo& T = s->h->tree->lv[level];
    for (int q = T.il_off[i]; q < T.il_off[i + 1]; q++)
      if (T.il[q] == j) {
        CK(cudaMemcpy(out, L.m2l[q], sizeof(double) * L.r0[i] * L.r0[j], cudaMemcpyDeviceToHost));
        return;
      }
    invalid("(i, j) is not an interaction-list pair");
  });
}

int ifmm_store_p2p(const ifmm_store* s, int i, int j, double* out) {
  return guard([&] {
    const StoreH* S = s->h;
    const int K = S->tree->depth;
    const Topo& T = S->tree->lv[K];
    const InitLevel& L = S->lv[K];
    if (i < 0 || j < 0 || i >= T.nc || j >= T.nc) invalid("index out of range");
    const int a = std::min(i, j), b = std::max(i, j), sl = T.slot(a, b);
    const double* blk = sl >= 0 ? S->leaf_p2p[size_t(a) * T.win() + sl] : nullptr;
    bool nb = false;
    for (int q = T.nbr_off[i]; q < T.nbr_off[i + 1]; q++) nb |= T.nbr[q] == j;
    if (!nb || !blk) invalid("(i, j) is not a leaf neighbour pair");
    const int na = L.n[a], nbb = L.n[b];
    std::vector<double> h(size_t(na) * nbb);
    CK(cudaMemcpy(h.data(), blk, sizeof(double) * h.size(), cudaMemcpyDeviceToHost));
    if (i == a) {
      memcpy(out, h.data(), sizeof(double) * h.size());
    } else {  // stored once as (a, b): return the transpose, n_i x n_j column-major
      for (int c = 0; c < na; c++)
        for (int r = 0; r < nbb; r++) out[r + size_t(c) * nbb] = h[c + size_t(r) * na];
    }
  });
}

int ifmm_store_bytes(const ifmm_store* s, double* out3) {
  return guard([&] {
    const StoreH* S = s->h;
    const int K = S->tree->depth;
    double p2p = 0, m2l = 0, bas = 0;
    {
      const Topo& T = S->tree->lv[K];
      const InitLevel& L = S->lv[K];
      for (int i = 0; i < T.nc; i++)
        for (int q = T.nbr_off[i]; q < T.nbr_off[i + 1]; q++)
          if (T.nbr[q] >= i) p2p += 8.0 * L.n[i] * L.n[T.nbr[q]];
    }
    for (int k = 2; k <= K; k++) {
      const Topo& T = S->tree->lv[k];
      const InitLevel& L = S->lv[k];
      for (int i = 0; i < T.nc; i++) {
        bas += 8.0 * L.n[i] * L.r0[i];
        for (int q = T.il_off[i]; q < T.il_off[i + 1]; q++) m2l += 8.0 * L.r0[i] * L.r0[T.il[q]];
      }
    }
    out3[0] = p2p;
    out3[1] = m2l;
    out3[2] = bas;
  });
}

int ifmm_extended_layout(const ifmm_store* s, int64_t* count, int32_t* sym, int32_t* level, int32_t* index,
                         int32_t* dim) {
  return guard([&] {
    const std::vector<ifmm::ExtSlot> v = ifmm::extended_layout(s->h);
    if (count) *count = int64_t(v.size());
    if (!sym) return;
    for (size_t q = 0; q < v.size(); q++) {
      sym[q] = v[q].sym;
      level[q] = v[q].level;
      index[q] = v[q].index;
      dim[q] = v[q].dim;
    }
  });
}

int ifmm_extended_dense(ifmm_store* s, int64_t cap, int64_t* dim, double* out) {
  return guard([&] {
    ensure_device();
    const int64_t m = ifmm::extended_dense(s->h, cap, out);
    if (dim) *dim = m;
  });
}

int ifmm_store_set_basis(ifmm_store* s, int level, int index, const double* in) {
  return guard([&] {
    if (level < 2 || level > s->h->tree->depth) invalid("level out of range");
    const InitLevel& L = s->h->lv[level];
    if (index < 0 || index >= L.nc) invalid("index out of range");
    CK(cudaMemcpy(L.U[index], in, sizeof(double) * L.n[index] * L.r0[index], cudaMemcpyHostToDevice));
  });
}

int ifmm_store_set_m2l(ifmm_store* s, int level, int i, int j, const double* in) {
  return guard([&] {
    if (level < 2 || level > s->h->tree->depth) invalid("level out of range");
    const InitLevel& L = s->h->lv[level];
    const Topo& T = s->h->tree->lv[level];
    if (i < 0 || i >= L.nc) invalid("index out of range");
    for (int q = T.il_off[i]; q < T.il_off[i + 1]; q++)
      if (T.il[q] == j) {
        CK(cudaMemcpy(L.m2l[q], in, sizeof(double) * L.r0[i] * L.r0[j], cudaMemcpyHostToDevice));
        return;
      }
    invalid("(i, j) is not an interaction-list pair");
  });
}

int ifmm_store_set_p2p(ifmm_store* s, int i, int j, const double* in) {
  return guard([&] {
    const StoreH* S = s->h;
    const int K = S->tree->depth;
    const Topo& T = S->tree->lv[K];
    const InitLevel& L = S->lv[K];
    if (i < 0 || j < 0 || i >= T.nc || j >= T.nc) invalid("index out of range");
    const int a = std::min(i, j), b = std::max(i, j), sl = T.slot(a, b);
    double* blk = sl >= 0 ? S->leaf_p2p[size_t(a) * T.win() + sl] : nullptr;
    bool nb = false;
    for (int q = T.nbr_off[i]; q < T.nbr_off[i + 1]; q++) nb |= T.nbr[q] == j;
    if (!nb || !blk) invalid("(i, j) is not a leaf neighbour pair");
    const int na = L.n[a], nbb = L.n[b];
    if (i == a) {
      CK(cudaMemcpy(blk, in, sizeof(double) * size_t(na) * nbb, cudaMemcpyHostToDevice));
    } else {  // stored once as (a, b): in is n_i x n_j = n_b x n_a, store its transpose
      std::vector<double> h(size_t(na) * nbb);
      for (int c = 0; c < nbb; c++)
        for (int r = 0; r < na; r++) h[r + size_t(c) * na] = in[c + size_t(r) * nbb];
      CK(cudaMemcpy(blk, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice));
    }
  });
}

int ifmm_matvec(ifmm_store* s, const double* x, double* y, int64_t nrhs, int ptr_kind) {
  return guard([&] { ifmm::matvec(s->h, x, y, nrhs, ptr_kind == IFMM_PTR_DEVICE); });
}

void ifmm_store_free(ifmm_store* s) {
  if (!s) return;
  matvec_release(s->h);
  delete s->h;
  delete s;
}

// ---------------------------------------------------------------- factor / solve
int ifmm_factorize(ifmm_store* s, double tol, int flags, double cond_limit, ifmm_factor** out) {
  return guard([&] {
    if (!s || !out) invalid("null handle");
    FactorH* h = ifmm::factorize(s->h, tol, flags, cond_limit);
    *out = new ifmm_factor{h};
  });
}

int ifmm_factorize_rank_control(ifmm_store* s, double tol, int flags, double cond_limit, double rank_tol,
                                ifmm_factor** out) {
  return guard([&] {
    if (!s || !out) invalid("null handle");
    if (!(rank_tol > 0.0) || !(rank_tol < 1.0)) invalid("rank_tol must lie in (0, 1)");
    FactorH* h = ifmm::factorize(s->h, tol, flags, cond_limit, rank_tol);
    *out = new ifmm_factor{h};
  });
}

int ifmm_factor_rank_control(const ifmm_factor* f, int64_t* out2) {
  return guard([&] {
    out2[0] = f->h->rc_before;
    out2[1] = f->h->rc_after;
  });
}

int ifmm_factor_info(const ifmm_factor* f, int* r_m, int* top_dim, int64_t* n_records, double* ms) {
  return guard([&] {
    if (r_m) *r_m = f->h->r_m;
    if (top_dim) *top_dim = f->h->top_dim;
    if (n_records) *n_records = int64_t(f->h->recs.size());
    if (ms) *ms = f->h->ms_total;
  });
}

int ifmm_factor_level_stats(const ifmm_factor* f, int level, int32_t* out4) {
  return guard([&] {
    if (level < 2 || level >= int(f->h->stats.size())) invalid("level out of range");
    const LevelStatsH& s = f->h->stats[level];
    out4[0] = s.clusters;
    out4[1] = s.max_rank;
    out4[2] = s.compressed;
    out4[3] = s.dense_kept;
  });
}

int ifmm_factor_level_cond(const ifmm_factor* f, int level, double* max_cond) {
  return guard([&] {
    if (level < 2 || level >= int(f->h->stats.size())) invalid("level out of range");
    *max_cond = f->h->stats[level].max_cond;
  });
}

int ifmm_factor_singular(const ifmm_factor* f, int64_t cap, int32_t* level, int32_t* index, double* cond,
                         int64_t* count) {
  return guard([&] {
    const auto& v = f->h->singular;
    if (count) *count = int64_t(v.size());
    for (int64_t q = 0; q < std::min<int64_t>(cap, int64_t(v.size())); q++) {
      if (level) level[q] = v[q].level;
      if (index) index[q] = v[q].index;
      if (cond) cond[q] = v[q].cond;
    }
  });
}

int ifmm_factor_record(const ifmm_factor* f, int64_t idx, int32_t* info7, int32_t* xp, int32_t* yp) {
  return guard([&] {
    const FactorH& F = *f->h;
    if (idx < 0 || idx >= int64_t(F.recs.size())) invalid("record index out of range");
    const RecordH& R = F.recs[size_t(idx)];
    const auto& X = F.rec_xp[size_t(idx)];
    const auto& Y = F.rec_yp[size_t(idx)];
    if (info7) {
      const int32_t v[7] = {R.level, R.index, R.n, R.r, R.w, int32_t(X.size()), int32_t(Y.size())};
      memcpy(info7, v, sizeof v);
    }
    if (xp) std::copy(X.begin(), X.end(), xp);
    if (yp) std::copy(Y.begin(), Y.end(), yp);
  });
}

int ifmm_factor_record_lu(const ifmm_factor* f, int64_t idx, double* lu, int32_t* perm) {
  return guard([&] {
    const FactorH& F = *f->h;
    if (idx < 0 || idx >= int64_t(F.recs.size())) invalid("record index out of range");
    const RecordH& R = F.recs[size_t(idx)];
    const size_t m = size_t(R.n + R.r);
    CK(cudaStreamSynchronize(F.stream));
    if (lu && m) CK(cudaMemcpy(lu, R.lu, sizeof(double) * m * m, cudaMemcpyDeviceToHost));
    if (perm && m) CK(cudaMemcpy(perm, R.perm, sizeof(int) * m, cudaMemcpyDeviceToHost));
  });
}

int ifmm_factor_top(const ifmm_factor* f, double* lu, int32_t* perm, int64_t* offsets) {
  return guard([&] {
    const FactorH& F = *f->h;
    const size_t M = size_t(F.top_dim);
    CK(cudaStreamSynchronize(F.stream));
    if (lu && M) CK(cudaMemcpy(lu, F.top_lu, sizeof(double) * M * M, cudaMemcpyDeviceToHost));
    if (perm && M) CK(cudaMemcpy(perm, F.top_perm, sizeof(int) * M, cudaMemcpyDeviceToHost));
    if (offsets) std::copy(F.top_off.begin(), F.top_off.end(), offsets);
  });
}

int ifmm_factor_records(const ifmm_factor* f, int32_t* out5) {
  return guard([&] {
    size_t u = 0;
    for (const RecordH& r : f->h->recs) {
      out5[u++] = r.level;
      out5[u++] = r.index;
      out5[u++] = r.n;
      out5[u++] = r.r;
      out5[u++] = r.w;
    }
  });
}

int ifmm_factor_work(const ifmm_factor* f, double* out6) {
  return guard([&] {
    out6[0] = f->h->fl_exec;
    out6[1] = f->h->fl_schur;
    out6[2] = f->h->fl_ref;
    out6[3] = f->h->solve_bytes;
    out6[4] = f->h->fl_lu;
    out6[5] = f->h->fl_x;
  });
}

int ifmm_factor_timing(const ifmm_factor* f, double* ms7, int64_t* launches7) {
  return guard([&] {
    for (int p = 0; p < ifmm::PH_COUNT; p++) {
      if (ms7) ms7[p] = f->h->phase_ms[p];
      if (launches7) launches7[p] = f->h->phase_launches[p];
    }
  });
}

int ifmm_factor_timing_level(const ifmm_factor* f, int level, double* ms9) {
  return guard([&] {
    for (int p = 0; p < ifmm::PH_COUNT; p++)
      ms9[p] = (level >= 0 && size_t(level) < f->h->phase_lvl_ms.size()) ? f->h->phase_lvl_ms[level][p] : 0.0;
    const bool h = level >= 0 && size_t(level) < f->h->host_lvl_ms.size();
    ms9[7] = h ? f->h->host_lvl_ms[level][0] : 0.0;
    ms9[8] = h ? f->h->host_lvl_ms[level][1] : 0.0;
  });
}

int64_t ifmm_launch_count(void) { return ifmm::launch_counter().load(); }

// ---------------------------------------------------------------- sharded
int ifmm_comm_nccl_unique_id(uint8_t* out128) {
  return guard([&] {
    if (!out128) invalid("null output");
    ifmm::nccl_unique_id(out128);
  });
}

int ifmm_comm_nccl_version(int* version) {
  return guard([&] { *version = ifmm::nccl_version(); });
}

int ifmm_comm_nccl_init(const uint8_t* id128, int nranks, int rank, ifmm_comm** out) {
  return guard([&] {
    if (!id128 || !out) invalid("null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) invalid("bad rank / nranks");
    ensure_device();
    *out = new ifmm_comm{std::make_shared<ifmm::NcclComm>(id128, nranks, rank)};
  });
}

int ifmm_comm_host_init(int nranks, int rank, ifmm_host_allgather_fn allgather, ifmm_host_exchange_fn exchange,
                        void* ctx, ifmm_comm** out) {
  return guard([&] {
    if (!allgather || !exchange || !out) invalid("null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) invalid("bad rank / nranks");
    ensure_device();
    *out = new ifmm_comm{std::make_shared<ifmm::HostComm>(nranks, rank, allgather, exchange, ctx)};
  });
}

void ifmm_comm_free(ifmm_comm* c) { delete c; }

int ifmm_comm_selftest(ifmm_comm* c, int64_t n, int32_t* ok) {
  return guard([&] {
    if (!c || n < 1) invalid("bad argument");
    ifmm::Comm& C = *c->h;
    const int me = C.rank(), P = C.size();
    cudaStream_t s = default_stream();
    Arena ws(size_t(16) << 20);
    std::vector<double> h(static_cast<size_t>(n));
    for (int64_t u = 0; u < n; u++) h[u] = 1000.0 * me + double(u);
    double* a = ws.alloc_n<double>(size_t(n));
    double* g = ws.alloc_n<double>(size_t(n) * P);
    double* r = ws.alloc_n<double>(size_t(n));
    CK(cudaMemcpyAsync(a, h.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s));
    C.allgather(a, g, sizeof(double) * n, s);
    const int to = (me + 1) % P, from = (me + P - 1) % P;
    C.exchange({ifmm::Msg{to, a, sizeof(double) * n}}, {ifmm::Msg{from, r, sizeof(double) * n}}, s);
    std::vector<double> hg(static_cast<size_t>(n) * P), hr(static_cast<size_t>(n));
    CK(cudaMemcpyAsync(hg.data(), g, sizeof(double) * hg.size(), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(hr.data(), r, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    bool good = true;
    for (int q = 0; q < P; q++)
      for (int64_t u = 0; u < n; u++) good &= hg[size_t(q) * n + u] == 1000.0 * q + double(u);
    for (int64_t u = 0; u < n; u++) good &= hr[u] == 1000.0 * from + double(u);
    *ok = good ? 1 : 0;
  });
}

int ifmm_factorize_sharded(ifmm_store* s, ifmm_comm* c, double tol, int flags, double cond_limit,
                           ifmm_factor** out) {
  return guard([&] {
    if (!s || !c || !out) invalid("null handle");
    FactorH* h = ifmm::factorize_sharded(s->h, c->h, tol, flags, cond_limit);
    *out = new ifmm_factor{h};
  });
}

int ifmm_factorize_sharded_rank_control(ifmm_store* s, ifmm_comm* c, double tol, int flags, double cond_limit,
                                        double rank_tol, ifmm_factor** out) {
  return guard([&] {
    if (!s || !c || !out) invalid("null handle");
    if (!(rank_tol > 0.0) || !(rank_tol < 1.0)) invalid("rank_tol must lie in (0, 1)");
    FactorH* h = ifmm::factorize_sharded(s->h, c->h, tol, flags, cond_limit, rank_tol);
    *out = new ifmm_factor{h};
  });
}

int ifmm_factorize_emulated_rank_control(ifmm_store* s, int nranks, double tol, int flags, double cond_limit,
                                         double rank_tol, ifmm_factor** out) {
  return guard([&] {
    if (!s || !out) invalid("null handle");
    if (!(rank_tol > 0.0) || !(rank_tol < 1.0)) invalid("rank_tol must lie in (0, 1)");
    std::vector<FactorH*> v;
    ifmm::factorize_emulated(s->h, nranks, tol, flags, cond_limit, v, rank_tol);
    for (int r = 0; r < nranks; r++) out[r] = new ifmm_factor{v[r]};
  });
}

int ifmm_factorize_emulated(ifmm_store* s, int nranks, double tol, int flags, double cond_limit,
                            ifmm_factor** out) {
  return guard([&] {
    if (!s || !out) invalid("null handle");
    std::vector<FactorH*> v;
    ifmm::factorize_emulated(s->h, nranks, tol, flags, cond_limit, v);
    for (int r = 0; r < nranks; r++) out[r] = new ifmm_factor{v[r]};
  });
}

int ifmm_solve_emulated(ifmm_factor** f, int nranks, const double* rhs, double* x, int64_t nrhs, int ptr_kind) {
  return guard([&] {
    if (!f || nranks < 1) invalid("null handle");
    std::vector<FactorH*> v;
    std::vector<double*> xs;
    const int64_t n = f[0]->h->tree->N;
    for (int r = 0; r < nranks; r++) {
      v.push_back(f[r]->h);
      xs.push_back(x + size_t(r) * n * nrhs);
    }
    ifmm::solve_emulated(v, rhs, xs, nrhs, ptr_kind == IFMM_PTR_DEVICE);
  });
}

int ifmm_factor_shard_info(const ifmm_factor* f, int32_t* rank_nranks, double* out4) {
  return guard([&] {
    const FactorH* h = f->h;
    const bool d = h->comm && h->comm->size() > 1;
    if (rank_nranks) {
      rank_nranks[0] = d ? h->comm->rank() : 0;
      rank_nranks[1] = d ? h->comm->size() : 1;
    }
    if (out4) {
      out4[0] = h->halo_bytes;
      out4[1] = h->meta_bytes;
      out4[2] = double(h->exchanges);
      out4[3] = h->phase_ms[ifmm::PH_COMM];
    }
  });
}

int ifmm_partition_halo_counts(int dim, int depth, int level, int nranks, int rank, int colour, int32_t* send,
                               int32_t* recv) {
  return guard([&] {
    if (level < 2 || level > depth) invalid("level out of range");
    const ifmm::Partition P = ifmm::make_partition_geometric(dim, depth, nranks, rank);
    std::vector<int> s, r;
    ifmm::halo_plan_counts(P, level, colour, s, r);
    for (int q = 0; q < nranks; q++) {
      send[q] = s[q];
      recv[q] = r[q];
    }
  });
}

int ifmm_partition(int dim, int depth, int level, int nranks, int32_t* owner, uint8_t* held) {
  return guard([&] {
    if (level < 2 || level > depth) invalid("level out of range");
    const ifmm::Partition P = ifmm::make_partition_geometric(dim, depth, nranks, 0);
    const int nc = 1 << (dim * level);
    for (int i = 0; i < nc; i++) {
      if (owner) owner[i] = P.owner[level][i];
      if (held)
        for (int s = 0; s < nranks; s++) held[size_t(s) * nc + i] = P.held[level][s][i];
    }
  });
}

int ifmm_solve(ifmm_factor* f, const double* rhs, double* x, int64_t nrhs, int ptr_kind) {
  return guard([&] { ifmm::solve(f->h, rhs, x, nrhs, ptr_kind == IFMM_PTR_DEVICE); });
}

int ifmm_solve_refined(ifmm_factor* f, ifmm_store* s, const double* rhs, double* x, int64_t nrhs, int ptr_kind,
                       int max_iters, double target, double* hist, int* iters_done) {
  return guard([&] {
    if (!f || !s) invalid("null handle");
    if (s->h != f->h->store) invalid("store does not belong to this factorization");
    ifmm::solve_refined(f->h, s->h, rhs, x, nrhs, ptr_kind == IFMM_PTR_DEVICE, max_iters, target, hist, iters_done);
  });
}

void ifmm_factor_free(ifmm_factor* f) {
  if (!f) return;
  delete f->h;
  delete f;
}

}  // extern "C"

// ---------------------------------------------------------------- test hooks
// The small-matrix routines run either CTA-wide (256 threads) or on one warp,
// as the compression kernels use them; ifmm_test_set_group selects which.
static int g_test_warp = 0;
template <class G>
__global__ void test_jacobi_kernel(double* a, int m, int n, double* v, double* sig, int* ord) {
  __shared__ CtaShared sh;
  ifmm::g_jacobi(G::make_for_test(sh), a, m, n, m, v, n, sig, ord);
}

template <class G>
__global__ void test_qr_kernel(double* a, int m, int k, double* q, double* r, double* vv) {
  __shared__ CtaShared sh;
  ifmm::g_qr(G::make_for_test(sh), a, m, k, m, r, q, m, vv);
}

template <class G>
__global__ void test_aca_kernel(const double* f, int m, int n, double tol, const int* probes, int kmax, double* uc,
                                double* vc, double* scratch, int* out) {
  __shared__ CtaShared sh;
  double* rr = scratch;
  double* cc = rr + n;
  double* dots = cc + m;
  int* usedr = reinterpret_cast<int*>(dots + kmax);
  int* usedc = usedr + m;
  AcaOut o = ifmm::g_aca(G::make_for_test(sh), f, m, 0, m, n, tol, probes, min(10, m), uc, vc, kmax, rr, cc, usedr,
                         usedc, dots);
  if (threadIdx.x == 0) {
    out[0] = o.k;
    out[1] = o.converged;
  }
}

#define TEST_LAUNCH(kern, ...)                                            \
  do {                                                                    \
    if (g_test_warp) kern<ifmm::WarpGroup><<<1, 32>>>(__VA_ARGS__);       \
    else kern<ifmm::CtaGroup><<<1, 256>>>(__VA_ARGS__);                   \
  } while (0)

extern "C" {

int ifmm_test_set_group(int warp) {
  g_test_warp = warp != 0;
  return IFMM_OK;
}

// Batched LU (the pivot factorization): a[] holds `count` column-major
// matrices back to back, overwritten by their L\U factors; perm[] (sum of m)
// receives each row permutation, info[] the zero-pivot flags, inv_norm1[] the
// dlacn2 estimate of ||A^-1||_1 that the pivot-condition test uses.
int ifmm_test_lu(double* a, const int32_t* m, int count, int32_t* perm, int32_t* info, double* inv_norm1) {
  return guard([&] {
    ensure_device();
    cudaStream_t s = default_stream();
    Arena ws(size_t(64) << 20);
    Staging st;
    std::vector<MatDesc> md(count);
    size_t tot = 0, totm = 0;
    int maxm = 0;
    for (int c = 0; c < count; c++) {
      tot += size_t(m[c]) * m[c];
      totm += size_t(m[c]);
      maxm = std::max(maxm, int(m[c]));
    }
    double* d = ws.alloc_n<double>(tot);
    int* dp = ws.alloc_n<int>(std::max<size_t>(1, totm));
    CK(cudaMemcpy(d, a, sizeof(double) * tot, cudaMemcpyHostToDevice));
    size_t off = 0, offm = 0;
    for (int c = 0; c < count; c++) {
      md[c] = MatDesc{d + off, m[c], m[c], dp + offm, c};
      off += size_t(m[c]) * m[c];
      offm += size_t(m[c]);
    }
    const MatDesc* dmd = upload(ws, md, s, st);
    int* dinfo = ws.alloc_n<int>(count);
    double* dn = ws.alloc_n<double>(count);
    ifmm::batched_lu(md, dmd, dinfo, ws, st, s);
    const ifmm::LuDiag dg = ifmm::launch_lu_diag_inv(md, dmd, ws, st, s, 0.0);
    ifmm::launch_lu_inv_norm1(dmd, count, maxm, dg, dn, s);
    CK(cudaStreamSynchronize(s));
    CK(cudaMemcpy(a, d, sizeof(double) * tot, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(perm, dp, sizeof(int) * totm, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(info, dinfo, sizeof(int) * count, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(inv_norm1, dn, sizeof(double) * count, cudaMemcpyDeviceToHost));
  });
}

// X = S^-1 [[C, 0], [0, -I_r]] for one factored pivot (lu, perm from
// ifmm_test_lu): xtop (n x w) and xbot (r x w), w = wl + r.
int ifmm_test_lu_solve_x(const double* lu, const int32_t* perm, int n, int r, const double* c, int wl, double* xtop,
                         double* xbot) {
  return guard([&] {
    ensure_device();
    cudaStream_t s = default_stream();
    Arena ws(size_t(64) << 20);
    Staging st;
    const int m = n + r, w = wl + r;
    double* dlu = ws.alloc_n<double>(size_t(m) * m);
    int* dp = ws.alloc_n<int>(m);
    double* dc = ws.alloc_n<double>(size_t(std::max(1, n)) * std::max(1, wl));
    double* dt = ws.alloc_n<double>(size_t(std::max(1, n)) * w);
    double* db = ws.alloc_n<double>(size_t(std::max(1, r)) * w);
    CK(cudaMemcpy(dlu, lu, sizeof(double) * m * m, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dp, perm, sizeof(int) * m, cudaMemcpyHostToDevice));
    if (n * wl > 0) CK(cudaMemcpy(dc, c, sizeof(double) * n * wl, cudaMemcpyHostToDevice));
    std::vector<MatDesc> md{MatDesc{dlu, m, m, dp, 0}};
    const MatDesc* dmd = upload(ws, md, s, st);
    const ifmm::LuDiag dg = ifmm::launch_lu_diag_inv(md, dmd, ws, st, s, 0.0);  // refine every block
    std::vector<ifmm::XSolveDesc> xd{ifmm::XSolveDesc{dlu, dp, dc, dt, db, dg.dinv, dg.flags, dg.pflag, m, n, r, wl, w, 0}};
    ifmm::launch_lu_solve_x(xd, ws, st, s);
    CK(cudaStreamSynchronize(s));
    CK(cudaMemcpy(xtop, dt, sizeof(double) * n * w, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(xbot, db, sizeof(double) * r * w, cudaMemcpyDeviceToHost));
  });
}

int ifmm_test_gemm(int transA, int transB, int M, int N, int K, double alpha, const double* A, int lda,
                   const double* B, int ldb, double beta, double* C, int ldc, int transC) {
  return guard([&] {
    ensure_device();
    cudaStream_t s = default_stream();
    Arena ws(size_t(64) << 20);
    Staging st;
    size_t na = size_t(lda) * (transA ? M : K), nb = size_t(ldb) * (transB ? K : N),
           nc = size_t(ldc) * (transC ? M : N);
    double *dA = ws.alloc_n<double>(na), *dB = ws.alloc_n<double>(nb), *dC = ws.alloc_n<double>(nc);
    CK(cudaMemcpy(dA, A, sizeof(double) * na, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B, sizeof(double) * nb, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dC, C, sizeof(double) * nc, cudaMemcpyHostToDevice));
    GemmBatch gb;
    gb.add(dA, lda, dB, ldb, dC, ldc, M, N, K, alpha, beta, transC != 0);
    ifmm::launch_grouped_gemm(gb, transA != 0, transB != 0, ws, st, s);
    CK(cudaStreamSynchronize(s));
    CK(cudaMemcpy(C, dC, sizeof(double) * nc, cudaMemcpyDeviceToHost));
  });
}

int ifmm_test_jacobi(double* a, int m, int n, double* v, double* sig) {
  return guard([&] {
    ensure_device();
    Arena ws(size_t(16) << 20);
    double *da = ws.alloc_n<double>(size_t(m) * n), *dv = ws.alloc_n<double>(size_t(n) * n),
           *ds = ws.alloc_n<double>(n);
    int* dord = ws.alloc_n<int>(n);
    CK(cudaMemcpy(da, a, sizeof(double) * m * n, cudaMemcpyHostToDevice));
    TEST_LAUNCH(test_jacobi_kernel, da, m, n, dv, ds, dord);
    CK_LAUNCH();
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(a, da, sizeof(double) * m * n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(v, dv, sizeof(double) * n * n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(sig, ds, sizeof(double) * n, cudaMemcpyDeviceToHost));
  });
}

int ifmm_test_qr(const double* a, int m, int k, double* q, double* r) {
  return guard([&] {
    ensure_device();
    Arena ws(size_t(16) << 20);
    double *da = ws.alloc_n<double>(size_t(m) * k), *dq = ws.alloc_n<double>(size_t(m) * k),
           *dr = ws.alloc_n<double>(size_t(k) * k), *dvv = ws.alloc_n<double>(k);
    CK(cudaMemcpy(da, a, sizeof(double) * m * k, cudaMemcpyHostToDevice));
    TEST_LAUNCH(test_qr_kernel, da, m, k, dq, dr, dvv);
    CK_LAUNCH();
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(q, dq, sizeof(double) * m * k, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(r, dr, sizeof(double) * k * k, cudaMemcpyDeviceToHost));
  });
}

int ifmm_test_aca(const double* f, int m, int n, double tol, const int32_t* probes, int kmax, double* left,
                  double* right, int32_t* rank, int32_t* incompressible) {
  return guard([&] {
    ensure_device();
    Arena ws(size_t(16) << 20);
    double* df = ws.alloc_n<double>(size_t(m) * n);
    double *du = ws.alloc_n<double>(size_t(m) * kmax), *dv = ws.alloc_n<double>(size_t(n) * kmax);
    double* scr = ws.alloc_n<double>(size_t(2) * (m + n) + kmax + 16);
    int* dp = ws.alloc_n<int>(ifmm::ACA_PROBE_STRIDE);
    int* dout = ws.alloc_n<int>(2);
    CK(cudaMemcpy(df, f, sizeof(double) * m * n, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dp, probes, sizeof(int) * ifmm::ACA_PROBE_STRIDE, cudaMemcpyHostToDevice));
    TEST_LAUNCH(test_aca_kernel, df, m, n, tol, dp, kmax, du, dv, scr, dout);
    CK_LAUNCH();
    CK(cudaDeviceSynchronize());
    int o[2];
    CK(cudaMemcpy(o, dout, 8, cudaMemcpyDeviceToHost));
    *rank = o[0];
    *incompressible = (!o[1] && (o[0] >= std::min(m, n) || o[0] >= kmax) && tol > 0) ? 1 : 0;
    CK(cudaMemcpy(left, du, sizeof(double) * m * o[0], cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(right, dv, sizeof(double) * n * o[0], cudaMemcpyDeviceToHost));
  });
}

int ifmm_test_recompress(const double* f, int m, int n, double tol, const int32_t* probes, int gram, double* left,
                         double* right, double* sv, int32_t* rank, int32_t* status) {
  return guard([&] {
    ensure_device();
    if (m < 1 || n < 1) invalid("fill must be non-empty");
    cudaStream_t s = default_stream();
    Arena ws(size_t(16) << 20);
    Staging st;
    const int kf = std::max(1, std::min(96, std::min(m, n)));
    double* df = ws.alloc_n<double>(size_t(m) * n);
    double* dout = ws.alloc_n<double>(size_t(m + n + 1) * kf);
    const size_t PS = ifmm::ACA_PROBE_STRIDE;
    int* dp = ws.alloc_n<int>(size_t(m + 1) * PS);  // probe table: row m only
    auto* dstate = ws.alloc_n<ifmm::FillState>(1);
    std::vector<int> tab(size_t(m + 1) * PS, 0);
    for (size_t t = 0; t < PS; t++) tab[size_t(m) * PS + t] = probes[t];
    CK(cudaMemcpy(df, f, sizeof(double) * m * n, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dp, tab.data(), sizeof(int) * tab.size(), cudaMemcpyHostToDevice));
    ifmm::test_recompress_one(df, m, n, tol, dp, m, gram, dout, dstate, ws, st, s);
    CK(cudaStreamSynchronize(s));
    ifmm::FillState S;
    CK(cudaMemcpy(&S, dstate, sizeof S, cudaMemcpyDeviceToHost));
    *rank = S.r;
    *status = S.status;
    CK(cudaMemcpy(left, dout, sizeof(double) * size_t(m) * S.r, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(right, dout + size_t(m) * kf, sizeof(double) * size_t(n) * S.r, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(sv, dout + size_t(m + n) * kf, sizeof(double) * S.r, cudaMemcpyDeviceToHost));
  });
}

}  // extern "C"
