// IFMM factorization on the GPU (ifmm/solver.py:106-546), B200 design:
//
// * Levels kappa..2; inside a level the clusters are 9-coloured by
//   (gx mod 3, gy mod 3).  Same-colour clusters are >= 3 cells apart, so their
//   3x3 neighbourhoods -- every block an elimination reads or writes, every
//   basis its fill compression augments -- are disjoint.  One colour is one
//   batch: its eliminations run concurrently and the result equals the
//   sequential sweep in (colour, Morton) order (the oracle's "colour9" order).
// * The extended system is stored once per symmetric pair: P2P(i<=j),
//   M2L(i<=j), XY(i,j) = M2P_ij = P2L_ji^T.  Capacity layout: every rank
//   dimension is allocated at its bound n_i, so basis growth needs no copies.
// * Per batch: gather S_i=[[P2P_ii,U_i],[U_i^T,0]] and C_i (pivot-row
//   couplings) -> batched Gauss-Jordan inverse (partial pivoting, exact 1-norm
//   rcond) -> X = S^-1 C (grouped DMMA GEMM, X_top written straight into the
//   solve record) -> symmetric Schur update T = C^T X on the block upper
//   triangle, fused into the owners' blocks (grouped DMMA GEMM, transposed
//   epilogue where the owner stores the pair the other way round) ->
//   fill-in compression, one CTA per pivot, fills in the reference order
//   (ACA + QR/SVD recompression, new directions, basis augmentation, M2L
//   absorption).
// * The level-2 M2L system is inverted densely.
// * Sharded (comm.cuh): with a communicator every rank replays the
//   whole host schedule (partners, presence, fill lists, ranks -- replicated
//   metadata) but runs the device work of its own subtrees' pivots only.  A
//   rank stores the blocks touching clusters within one cell of its own;
//   after each colour batch the writer of a block ships it to every other
//   rank that stores it (and the batch's fill outcomes / new ranks are
//   all-gathered), so every stored copy is current before it is read.
#include <algorithm>
#include <climits>
#include <unordered_map>
#include <thread>
#include <chrono>
#include <cmath>

#include "core.cuh"
#include "comm.cuh"
#include "lu.cuh"
#include "compress.cuh"
#include "consolidate.cuh"
#include "cta_la.cuh"

namespace ifmm {

// ------------------------------------------------------------------ work level
struct WorkLevel {
  int k = 0, nc = 0, win = 0;
  const Topo* T = nullptr;
  std::vector<int> n, r, rcap, r0;
  std::vector<double*> U;
  std::vector<double*> p2p, m2l, xy;  // nc*win
  std::vector<int> m2l_ld;            // leading dimension of each allocated M2L block
  std::vector<uint8_t> pp, pm, px;
  std::vector<uint8_t> dead;
  // Pairs beyond the 7^d window (dense couplings that chained past +-3 cells)
  // get table entries appended after the window part: ordered pair -> index,
  // and per-cluster adjacency for the partner scan.
  std::unordered_map<uint64_t, int> ovf;
  std::vector<std::vector<int>> ovf_adj;
  int* d_rank = nullptr;
  Arena* arena = nullptr;  // zero-initialised blocks
  // rank-growth control: rows of the parent's basis belonging to a consolidated
  // cluster (r' x r0_parent, ld prow_ld), replacing [R_i ; 0] at the transition
  std::vector<double*> prow;
  std::vector<int> prow_ld;
};

struct BlkRef {
  double* p;
  int ld;
  bool trans;
};

// CUDA-event phase timing on the factorization stream (IFMM_FLAG_TIMING).
struct PhaseTimer {
  bool on = false;
  cudaStream_t s = nullptr;
  struct Span {
    cudaEvent_t a, b;
    int ph;
    long long launches;
  };
  std::vector<Span> spans;
  std::vector<cudaEvent_t> pool;
  int cur = -1;
  cudaEvent_t ev0 = nullptr;
  long long l0 = 0;
  cudaEvent_t get() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    return e;
  }
  void begin(int ph) {
    if (!on) return;
    end();
    ev0 = get();
    CK(cudaEventRecord(ev0, s));
    cur = ph;
    l0 = launch_counter().load();
  }
  void end() {
    if (!on || cur < 0) return;
    cudaEvent_t e = get();
    CK(cudaEventRecord(e, s));
    spans.push_back({ev0, e, cur, launch_counter().load() - l0});
    cur = -1;
  }
  void collect(FactorH* F, int level) {  // call after a stream synchronisation
    if (!on) return;
    end();
    if (F->phase_lvl_ms.size() <= size_t(level)) F->phase_lvl_ms.resize(level + 1, std::array<double, 8>{});
    for (Span& sp : spans) {
      float ms = 0.f;
      CK(cudaEventSynchronize(sp.b));
      CK(cudaEventElapsedTime(&ms, sp.a, sp.b));
      F->phase_ms[sp.ph] += ms;
      F->phase_lvl_ms[level][sp.ph] += ms;
      F->phase_launches[sp.ph] += sp.launches;
      pool.push_back(sp.a);
      pool.push_back(sp.b);
    }
    spans.clear();
  }
  ~PhaseTimer() {
    for (auto& sp : spans) {
      cudaEventDestroy(sp.a);
      cudaEventDestroy(sp.b);
    }
    for (auto e : pool) cudaEventDestroy(e);
  }
};

class Factorizer {
 public:
  Factorizer(StoreH* S, FactorWork* work, cudaStream_t s, std::shared_ptr<Comm> comm, double tol, int flags,
             double cond_limit, double rank_tol = 0.0)
      : S_(S),
        t_(S->tree),
        tol_(tol),
        flags_(flags),
        cond_limit_(cond_limit),
        rank_tol_(rank_tol),
        s_(s),
        ws_(work->ws),
        st_(work->st),
        lvl_arena_(work->lvl),
        work_(work),
        comm_(std::move(comm)) {}
  FactorH* run();

 private:
  StoreH* S_;
  TreeH* t_;
  double tol_;
  int flags_;
  double cond_limit_;  // PIVOT_CONDITION_LIMIT (ifmm/solver.py:50), 1e12 by default
  double rank_tol_;    // > 0: rank-growth control (consolidate.cu) at this relative tolerance
  cudaStream_t s_ = nullptr;
  std::unique_ptr<FactorH> F_;
  Arena& ws_;
  Staging& st_;
  Arena* lvl_arena_;  // [2], alternating between levels
  FactorWork* work_;
  std::shared_ptr<Comm> comm_;          // null: one GPU
  std::shared_ptr<Partition> part_;     // subtree partition (sharded runs)
  int rank_ = 0, nranks_ = 1;
  PhaseTimer tm_;
  WorkLevel cur_, prev_;
  // debug (IFMM_HOST_PROF): host ms per section of eliminate_batch, per level
  double hsec_[16] = {0};
  std::chrono::steady_clock::time_point hmark_;
  void hmark(int sec) {
    const auto now = std::chrono::steady_clock::now();
    hsec_[sec] += std::chrono::duration<double, std::milli>(now - hmark_).count();
    hmark_ = now;
  }
  // per-record host metadata for pos resolution at level end
  struct SlotRef { int kind, j, dim; };  // kind 0: x_j, 1: y_j
  std::vector<std::vector<SlotRef>> rec_slots_;

  // ownership (sharded runs; everything is mine / held on one GPU)
  bool mine(const WorkLevel& W, int i) const { return nranks_ == 1 || part_->owner[W.k][i] == rank_; }
  int owner(const WorkLevel& W, int i) const { return nranks_ == 1 ? 0 : part_->owner[W.k][i]; }
  bool holds(const WorkLevel& W, int s, int i) const { return nranks_ == 1 || part_->held[W.k][s][i]; }
  bool holds1(const WorkLevel& W, int i) const { return holds(W, rank_, i); }
  bool holds2(const WorkLevel& W, int a, int b) const { return holds(W, rank_, a) || holds(W, rank_, b); }
  bool holds2s(const WorkLevel& W, int s, int a, int b) const { return holds(W, s, a) || holds(W, s, b); }
  // level arenas hand out zeroed memory (slabs are cleared on creation/reset)
  double* zalloc(WorkLevel& W, size_t n) { return W.arena->alloc_n<double>(std::max<size_t>(1, n)); }
  // Table index of the ordered pair (a, b): its window slot, else its overflow
  // entry (created on demand when `create`), else -1.
  int64_t pidx(WorkLevel& W, int a, int b, bool create) {
    const int sl = W.T->slot(a, b);
    if (sl >= 0) return int64_t(a) * W.win + sl;
    const uint64_t key = (uint64_t(uint32_t(a)) << 32) | uint32_t(b);
    auto it = W.ovf.find(key);
    if (it != W.ovf.end()) return it->second;
    if (!create) return -1;
    const int64_t ix = int64_t(W.p2p.size());
    W.ovf.emplace(key, int(ix));
    W.p2p.push_back(nullptr);
    W.m2l.push_back(nullptr);
    W.m2l_ld.push_back(0);
    W.xy.push_back(nullptr);
    W.pp.push_back(0);
    W.pm.push_back(0);
    W.px.push_back(0);
    if (W.ovf_adj.empty()) W.ovf_adj.resize(W.nc);
    W.ovf_adj[a].push_back(b);
    if (a != b) W.ovf_adj[b].push_back(a);
    return ix;
  }
  BlkRef p2p_ref(WorkLevel& W, int i, int j, bool alloc) {
    int a = std::min(i, j), b = std::max(i, j);
    const int64_t ix = pidx(W, a, b, alloc);
    if (ix < 0) return {nullptr, W.n[a], i > j};
    double*& p = W.p2p[size_t(ix)];
    if (!p && alloc && holds2(W, a, b)) p = zalloc(W, size_t(W.n[a]) * W.n[b]);
    return {p, W.n[a], i > j};
  }
  BlkRef m2l_ref(WorkLevel& W, int i, int j, bool alloc) {
    int a = std::min(i, j), b = std::max(i, j);
    const int64_t ix = pidx(W, a, b, alloc);
    if (ix < 0) return {nullptr, W.rcap[a], i > j};
    double*& p = W.m2l[size_t(ix)];
    if (!p && alloc && holds2(W, a, b)) {  // live endpoints: capacity layout (ranks may grow)
      p = zalloc(W, size_t(W.rcap[a]) * W.rcap[b]);
      W.m2l_ld[size_t(ix)] = W.rcap[a];
    }
    return {p, p ? W.m2l_ld[size_t(ix)] : W.rcap[a], i > j};
  }
  BlkRef xy_ref(WorkLevel& W, int i, int j, bool alloc) {
    const int64_t ix = pidx(W, i, j, alloc);
    if (ix < 0) return {nullptr, W.n[i], false};
    double*& p = W.xy[size_t(ix)];
    // hybrid blocks are only created with j already eliminated: its rank is final
    if (!p && alloc && holds2(W, i, j)) p = zalloc(W, size_t(W.n[i]) * std::max(1, W.r[j]));
    return {p, W.n[i], false};
  }
  bool get_pres(const std::vector<uint8_t>& v, WorkLevel& W, int i, int j) {
    const int64_t ix = pidx(W, i, j, false);
    return ix >= 0 && v[size_t(ix)];
  }
  void set_pres(std::vector<uint8_t>& v, WorkLevel& W, int i, int j, uint8_t val) {
    const int64_t ix = pidx(W, i, j, val != 0);
    if (ix >= 0) v[size_t(ix)] = val;
  }
  bool pp_present(WorkLevel& W, int i, int j) { return get_pres(W.pp, W, std::min(i, j), std::max(i, j)); }
  void set_pp(WorkLevel& W, int i, int j, uint8_t v) { set_pres(W.pp, W, std::min(i, j), std::max(i, j), v); }
  void set_pm(WorkLevel& W, int i, int j, uint8_t v) { set_pres(W.pm, W, std::min(i, j), std::max(i, j), v); }
  bool pm_present(WorkLevel& W, int i, int j) { return get_pres(W.pm, W, std::min(i, j), std::max(i, j)); }
  bool px_present(WorkLevel& W, int i, int j) { return get_pres(W.px, W, i, j); }
  void set_px(WorkLevel& W, int i, int j, uint8_t v) { set_pres(W.px, W, i, j, v); }
  // Schur target of kind 0 (P2P), 1 (hybrid x-y) or 2 (M2L): created (storage
  // where held, presence flag) with a single table lookup
  BlkRef schur_target(WorkLevel& W, int kind, int i, int j) {
    const int a = kind == 1 ? i : std::min(i, j), b = kind == 1 ? j : std::max(i, j);
    const size_t ix = size_t(pidx(W, a, b, true));
    const bool held = holds2(W, a, b);
    if (kind == 0) {
      W.pp[ix] = 1;
      double*& p = W.p2p[ix];
      if (!p && held) p = zalloc(W, size_t(W.n[a]) * W.n[b]);
      return {p, W.n[a], i > j};
    }
    if (kind == 1) {
      W.px[ix] = 1;
      double*& p = W.xy[ix];
      if (!p && held) p = zalloc(W, size_t(W.n[i]) * std::max(1, W.r[j]));  // j eliminated: final rank
      return {p, W.n[i], false};
    }
    W.pm[ix] = 1;
    double*& p = W.m2l[ix];
    if (!p && held) {
      // Schur targets of kind 2 couple y / z slots: both clusters are
      // eliminated (or being eliminated), their ranks final -- no capacity
      p = zalloc(W, size_t(std::max(1, W.r[a])) * std::max(1, W.r[b]));
      W.m2l_ld[ix] = std::max(1, W.r[a]);
    }
    return {p, p ? W.m2l_ld[ix] : W.rcap[a], i > j};
  }

  // IFMM_HOST_PROF: host ms between marks of the level start
  std::chrono::steady_clock::time_point hp_t_;
  void hprof_mark(const char* what) {
    static const bool on = getenv("IFMM_HOST_PROF") != nullptr;
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    if (what) fprintf(stderr, "  host %s: %.2f ms\n", what, std::chrono::duration<double, std::milli>(now - hp_t_).count());
    hp_t_ = now;
  }
  void init_level_alloc(WorkLevel& W, int k) {
    hprof_mark(nullptr);
    W.k = k;
    W.T = &t_->lv[k];
    W.nc = W.T->nc;
    W.win = W.T->win();
    W.arena = &lvl_arena_[k & 1];
    W.arena->set_zero_stream(s_);
    static const bool hp = getenv("IFMM_HOST_PROF") != nullptr;
    if (hp) fprintf(stderr, "level %d arena: zeroing %.2f GB (reserved %.2f GB)\n", k, W.arena->in_use() / 1e9,
                    W.arena->reserved() / 1e9);
    W.arena->reset();
    hprof_mark("arena reset");
    W.p2p.assign(size_t(W.nc) * W.win, nullptr);
    W.m2l.assign(size_t(W.nc) * W.win, nullptr);
    W.m2l_ld.assign(size_t(W.nc) * W.win, 0);
    W.xy.assign(size_t(W.nc) * W.win, nullptr);
    W.pp.assign(size_t(W.nc) * W.win, 0);
    W.pm.assign(size_t(W.nc) * W.win, 0);
    W.px.assign(size_t(W.nc) * W.win, 0);
    W.ovf.clear();
    W.ovf_adj.clear();
    W.dead.assign(W.nc, 0);
    W.U.assign(W.nc, nullptr);
    W.prow.assign(W.nc, nullptr);
    W.prow_ld.assign(W.nc, 0);
    W.d_rank = W.arena->alloc_n<int>(W.nc);
    hprof_mark("tables");
  }
  std::vector<int> mark_;
  int stamp_ = 0;
  // x-partners (live, coupled through P2P) and y-partners (eliminated, coupled
  // through M2P = P2L^T) of i, sorted (ifmm/solver.py:220-229); scans the 7x7 window
  // Without a dense-kept well-separated fill at this level every coupling is
  // between neighbours (distance-2 fills are always interaction-list pairs and
  // are compressed), so the 3^d neighbour list replaces the 7^d window scan.
  void partners(WorkLevel& W, int i, std::vector<int>& xp, std::vector<int>& yp) {
    const Topo& T = *W.T;
    xp.clear();
    yp.clear();
    const bool near = F_->stats[W.k].dense_kept == 0;
    const int t0 = near ? T.nbr_off[i] : T.wc_off[i], t1 = near ? T.nbr_off[i + 1] : T.wc_off[i + 1];
    const int* lst = near ? T.nbr.data() : T.wc.data();
    for (int t = t0; t < t1; t++) {
      const int j = lst[t];
      if (j == i) continue;
      if (!W.dead[j] && pp_present(W, i, j)) xp.push_back(j);
      if (px_present(W, i, j)) yp.push_back(j);
    }
    if (!near && !W.ovf_adj.empty() && !W.ovf_adj[i].empty()) {  // couplings beyond the window
      std::vector<int> o(W.ovf_adj[i]);
      std::sort(o.begin(), o.end());
      o.erase(std::unique(o.begin(), o.end()), o.end());
      for (int j : o) {
        if (j == i || W.T->slot(i, j) >= 0) continue;
        if (!W.dead[j] && pp_present(W, i, j)) xp.push_back(j);
        if (px_present(W, i, j)) yp.push_back(j);
      }
      std::sort(xp.begin(), xp.end());
      std::sort(yp.begin(), yp.end());
    }
  }
  void start_leaf_level();
  void start_parent_level(WorkLevel& C, int k);
  void eliminate_batch(std::vector<int>& piv, int colour, std::vector<int>& deferred);
  void consolidate_pivots(const std::vector<int>& piv);
  // pivots consolidated in the current batch -> their M2L partners (the blocks the
  // rotation rewrote; sharded runs ship them with the batch's halo)
  std::unordered_map<int, std::vector<int>> cons_parts_;
  void finish_level(int rec_begin);
  void factor_top();
  // sharded runs: one block (or the new columns of a basis) a batch or a
  // transition wrote, shipped from its writer to every other rank storing it
  enum HaloKind : int { HALO_P2P = 0, HALO_XY = 1, HALO_M2L = 2, HALO_U = 3 };
  struct HaloItem {
    int kind, a, b, c0;  // P2P / M2L: (a <= b); XY: (x-cluster a, eliminated b); U: cluster a, columns c0..r_a
  };
  struct HaloRef {
    double* p;
    int ld, rows, cols;
  };
  HaloRef halo_ref(WorkLevel& W, const HaloItem& it);
  void halo_exchange(WorkLevel& W, const std::vector<std::vector<HaloItem>>& send,
                     const std::vector<std::vector<HaloItem>>& recv, CopyBatch* local);
  // solve-vector slots of every pivot of the level (all ranks): (batch, owner, cluster, slots)
  struct LevelPivot {
    int batch, owner, i;
    std::vector<SlotRef> slots;
  };
  std::vector<LevelPivot> lvl_piv_;
};

void Factorizer::start_leaf_level() {
  const int K = t_->depth;
  WorkLevel& W = cur_;
  init_level_alloc(W, K);
  const InitLevel& L = S_->lv[K];
  W.n = L.n;
  W.r0 = L.r0;
  W.r = L.r0;
  W.rcap = L.n;
  CopyBatch cb;
  cb.d.reserve(size_t(W.nc) * 20);
  for (int i = 0; i < W.nc; i++) {
    if (!holds1(W, i)) continue;
    W.U[i] = zalloc(W, size_t(W.n[i]) * W.rcap[i]);
    cb.add(L.U[i], W.n[i], W.U[i], W.n[i], W.n[i], W.r0[i]);
  }
  hprof_mark("leaf U");
  const Topo& T = *W.T;
  for (int i = 0; i < W.nc; i++) {
    for (int q = T.nbr_off[i]; q < T.nbr_off[i + 1]; q++) {
      int j = T.nbr[q];
      if (j < i) continue;
      BlkRef b = p2p_ref(W, i, j, true);
      if (b.p) cb.add(S_->leaf_p2p[size_t(i) * W.win + T.slot(i, j)], W.n[i], b.p, b.ld, W.n[i], W.n[j]);
      set_pp(W, i, j, 1);
    }
    for (int q = T.il_off[i]; q < T.il_off[i + 1]; q++) {
      int j = T.il[q];
      if (j < i) continue;
      BlkRef b = m2l_ref(W, i, j, true);
      if (b.p) cb.add(L.m2l[q], std::max(1, W.r0[i]), b.p, b.ld, W.r0[i], W.r0[j]);
      set_pm(W, i, j, 1);
    }
  }
  CK(cudaMemcpyAsync(W.d_rank, W.r.data(), sizeof(int) * W.nc, cudaMemcpyHostToDevice, s_));
  hprof_mark("leaf descriptors");
  launch_copies(cb, ws_, st_, s_);
  hprof_mark("leaf upload+launch");
}

void Factorizer::start_parent_level(WorkLevel& C, int k) {
  // C: finished child level k+1 ; build level k
  WorkLevel& W = cur_;
  init_level_alloc(W, k);
  const int dim = t_->dim, nch = 1 << dim;
  const InitLevel& L = S_->lv[k];
  W.r0 = L.r0;
  W.r = L.r0;
  W.n.assign(W.nc, 0);
  std::vector<std::vector<int>> off(W.nc, std::vector<int>(nch + 1, 0));
  for (int i = 0; i < W.nc; i++) {
    for (int c = 0; c < nch; c++) off[i][c + 1] = off[i][c] + C.r[(i << dim) + c];
    W.n[i] = off[i][nch];
  }
  W.rcap = W.n;
  CopyBatch cb;
  cb.d.reserve(size_t(W.nc) * (4 + 9 * (1 << (2 * dim))));
  // rank-growth control, sharded: the rotated parent rows of consolidated
  // children exist on their owner only -- the other ranks storing a parent's
  // basis receive it from the parent's owner in the transition's halo exchange
  const bool u_from_owner = nranks_ > 1 && rank_tol_ > 0.0;
  for (int i = 0; i < W.nc; i++) {
    if (!holds1(W, i)) continue;
    W.U[i] = zalloc(W, size_t(W.n[i]) * W.rcap[i]);
    if (u_from_owner && !mine(W, i)) continue;
    const int n0 = int(L.child_off[size_t(i) * (nch + 1) + nch]);
    for (int c = 0; c < nch; c++) {
      const int ch = (i << dim) + c;
      const int64_t ro = L.child_off[size_t(i) * (nch + 1) + c];
      if (C.prow[ch])  // consolidated child: its rotated rows T^T [R ; 0]
        cb.add(C.prow[ch], C.prow_ld[ch], W.U[i] + off[i][c], W.n[i], C.r[ch], W.r0[i]);
      else
        cb.add(L.U[i] + ro, std::max(1, n0), W.U[i] + off[i][c], W.n[i], S_->lv[k + 1].r0[ch], W.r0[i]);
    }
  }
  // parent near field from the children's M2L blocks (ifmm/solver.py:163-192).
  // Sharded: a rank assembles P2P(i, j) when it owns i or j (it stores every
  // child block of its own children); pairs it stores but owns neither end of
  // come from the owner of min(i, j) -- the transition's halo exchange.
  std::vector<std::vector<HaloItem>> send(nranks_), recv(nranks_);
  const Topo& T = *W.T;
  for (int i = 0; i < W.nc; i++) {
    for (int q = T.nbr_off[i]; q < T.nbr_off[i + 1]; q++) {
      int j = T.nbr[q];
      if (j < i) continue;
      // present child M2L blocks of the pair (one table lookup each)
      int nblk = 0;
      int64_t bix[64];
      int bab[64];
      for (int a = 0; a < nch; a++)
        for (int b = 0; b < nch; b++) {
          const int ca = (i << dim) + a, cbb = (j << dim) + b;
          const int64_t ix = pidx(C, std::min(ca, cbb), std::max(ca, cbb), false);
          if (ix >= 0 && C.pm[size_t(ix)]) {
            bix[nblk] = ix;
            bab[nblk++] = a * nch + b;
          }
        }
      if (nblk == 0) continue;
      set_pp(W, i, j, 1);
      BlkRef P = p2p_ref(W, i, j, true);
      const bool build = mine(W, i) || mine(W, j);
      if (nranks_ > 1) {
        const HaloItem it{HALO_P2P, i, j, 0};
        if (owner(W, i) == rank_) {
          for (int s = 0; s < nranks_; s++)
            if (s != rank_ && holds2s(W, s, i, j) && owner(W, i) != s && owner(W, j) != s) send[s].push_back(it);
        } else if (!build && P.p) {
          recv[owner(W, i)].push_back(it);
        }
      }
      if (!build || !P.p) continue;
      for (int u = 0; u < nblk; u++) {
        const int a = bab[u] / nch, b = bab[u] % nch;
        const int ca = (i << dim) + a, cbb = (j << dim) + b;
        const double* mp = C.m2l[size_t(bix[u])];
        if (!mp) {
          if (nranks_ > 1) invalid("sharded transition: a child M2L block is not stored on the assembling rank");
          continue;
        }
        // stored once as (min, max), leading dimension per block
        cb.add(mp, C.m2l_ld[size_t(bix[u])], P.p + off[i][a] + size_t(off[j][b]) * P.ld, P.ld, C.r[ca], C.r[cbb],
               ca > cbb);
      }
    }
    for (int q = T.il_off[i]; q < T.il_off[i + 1]; q++) {
      int j = T.il[q];
      if (j < i) continue;
      BlkRef b = m2l_ref(W, i, j, true);
      if (b.p) cb.add(L.m2l[q], std::max(1, W.r0[i]), b.p, b.ld, W.r0[i], W.r0[j]);
      set_pm(W, i, j, 1);
    }
  }
  if (u_from_owner)
    for (int i = 0; i < W.nc; i++) {
      if (W.n[i] <= 0 || W.r[i] <= 0) continue;
      const HaloItem it{HALO_U, i, 0, 0};
      if (mine(W, i)) {
        for (int s = 0; s < nranks_; s++)
          if (s != rank_ && holds(W, s, i)) send[s].push_back(it);
      } else if (holds1(W, i)) {
        recv[owner(W, i)].push_back(it);
      }
    }
  CK(cudaMemcpyAsync(W.d_rank, W.r.data(), sizeof(int) * W.nc, cudaMemcpyHostToDevice, s_));
  hprof_mark("parent descriptors");
  launch_copies(cb, ws_, st_, s_);
  hprof_mark("parent upload+launch");
  if (nranks_ > 1) {
    tm_.begin(PH_COMM);
    halo_exchange(W, send, recv, nullptr);
  }
}

// Rank-growth control for the pivots of one colour batch (consolidate.cu): their
// bases are final (every neighbour of an earlier colour has been eliminated, the
// remaining ones cannot touch them before they are gone), so each pivot's
// coupling row -- its M2L blocks and its rows of the parent's basis -- is
// re-truncated at rank_tol_ and the basis, the blocks and the parent rows are
// rotated onto the kept directions before S_i and C_i are gathered.
void Factorizer::consolidate_pivots(const std::vector<int>& piv) {
  WorkLevel& W = cur_;
  const Topo& T = *W.T;
  const int k = W.k, dim = t_->dim, nch = 1 << dim;
  const bool dist = nranks_ > 1;
  const InitLevel* Lp = k > 2 ? &S_->lv[k - 1] : nullptr;
  // Every rank lists every pivot's coupling row (replicated metadata: presence
  // flags and ranks); the device work runs for its own pivots only.
  struct Part { int l; BlkRef b; };
  struct Item { int i, r, W, r0p, cd; bool own; double *row, *row2; std::vector<Part> parts; };
  std::vector<Item> items;
  std::vector<ConsDesc> cd;
  cons_parts_.clear();
  int shape_maxr = 1;
  for (int i : piv) {
    const int r = W.r[i];
    if (r <= 0 || W.n[i] <= 0) continue;
    Item it{i, r, 0, 0, -1, mine(W, i), nullptr, nullptr, {}};
    bool self = false;
    auto visit = [&](int l) {
      if (!pm_present(W, i, l)) return;
      if (l == i) { self = true; return; }
      if (W.r[l] <= 0) return;
      BlkRef b{nullptr, 0, false};
      if (it.own) {
        b = m2l_ref(W, i, l, false);
        if (!b.p) invalid("rank-growth control: an M2L block of an own pivot is not stored on this rank");
      }
      it.parts.push_back({l, b});
      it.W += W.r[l];
    };
    for (int t = T.wc_off[i]; t < T.wc_off[i + 1]; t++) visit(T.wc[t]);
    if (!W.ovf_adj.empty()) {
      std::vector<int> o(W.ovf_adj[i]);
      std::sort(o.begin(), o.end());
      o.erase(std::unique(o.begin(), o.end()), o.end());
      for (int l : o)
        if (W.T->slot(i, l) < 0) visit(l);
    }
    if (self) continue;  // only a cluster without a self block is live
    const int par = i >> dim;
    it.r0p = Lp ? Lp->r0[par] : 0;
    it.W += it.r0p;
    if (it.W == 0) continue;
    shape_maxr = std::max(shape_maxr, r);
    if (it.own) {
      it.row = ws_.alloc_n<double>(size_t(r) * it.W);
      it.row2 = ws_.alloc_n<double>(size_t(r) * it.W);
      it.cd = int(cd.size());
      cd.push_back(ConsDesc{i, W.n[i], r, it.W, W.U[i], it.row, it.row2, nullptr, nullptr, nullptr, nullptr});
    }
    std::vector<int>& cp = cons_parts_[i];
    for (const Part& q : it.parts) cp.push_back(q.l);
    items.push_back(std::move(it));
  }
  if (items.empty()) return;
  // Two pivots of the batch can share an M2L block (interaction-list pairs three
  // cells apart have the same colour): every pivot computes its rotation from
  // the block as it was, and the block becomes T_i^T M T_l -- the smaller
  // cluster's rotated row segment T_i^T M times T_l, one more grouped GEMM over
  // the shared pairs.  Sharded: when the two pivots have different owners,
  // owner(l) sends T_l to owner(i), i < l, which forms the block (it reaches the
  // other ranks storing it with the batch's halo).
  std::unordered_map<int, int> item_of;
  for (size_t u = 0; u < items.size(); u++) item_of[items[u].i] = int(u);
  tm_.begin(PH_COMPRESS);
  CopyBatch gather, scatter;
  struct Shared { int u, v; size_t off; const Part* q; const double* Tl; };
  std::vector<Shared> shared;
  struct Cross { int u, v; };  // canonical order on every rank: (smaller pivot's item, partner order)
  std::vector<Cross> cross;
  for (size_t u = 0; u < items.size(); u++) {
    Item& it = items[u];
    size_t off = 0;
    for (const Part& q : it.parts) {
      auto f = item_of.find(q.l);
      const bool both = f != item_of.end();
      if (both && it.i < q.l && dist && owner(W, it.i) != owner(W, q.l)) cross.push_back({int(u), f->second});
      if (it.own) {
        gather.add(q.b.p, q.b.ld, it.row + off * it.r, it.r, it.r, W.r[q.l], q.b.trans);
        if (both) {
          if (it.i < q.l) shared.push_back({int(u), f->second, off, &q, nullptr});  // formed once, by the smaller cluster's owner
        } else if (q.b.trans) {
          // stored (l, i) when i > l: dst (r_l x r) = (row2 block)^T
          scatter.add(it.row2 + off * it.r, it.r, q.b.p, q.b.ld, W.r[q.l], it.r, true);
        } else {
          scatter.add(it.row2 + off * it.r, it.r, q.b.p, q.b.ld, it.r, W.r[q.l]);
        }
      }
      off += W.r[q.l];
    }
    if (it.own && it.r0p > 0) {
      const int par = it.i >> dim, c = it.i - (par << dim);
      const int64_t ro = Lp->child_off[size_t(par) * (nch + 1) + c];
      const int n0 = int(Lp->child_off[size_t(par) * (nch + 1) + nch]);
      const int r0i = W.r0[it.i];
      gather.add(Lp->U[par] + ro, std::max(1, n0), it.row + off * it.r, it.r, r0i, it.r0p);
      if (it.r > r0i) gather.zero(it.row + off * it.r + r0i, it.r, it.r - r0i, it.r0p);
      W.prow[it.i] = zalloc(W, size_t(it.r) * it.r0p);
      W.prow_ld[it.i] = it.r;
      scatter.add(it.row2 + off * it.r, it.r, W.prow[it.i], it.r, it.r, it.r0p);
    }
  }
  int* d_new = ws_.alloc_n<int>(std::max<size_t>(1, cd.size()));
  launch_copies(gather, ws_, st_, s_);
  launch_consolidate(cd, rank_tol_, W.d_rank, d_new, ws_, st_, s_, shape_maxr);
  for (const ConsDesc& D : cd) scatter.add(D.U2, D.n, W.U[D.cluster], D.n, D.n, D.r);
  // rotations of the other side of cross-owner pairs
  std::unordered_map<int64_t, const double*> t_remote;  // (u, v) -> T_l received
  if (!cross.empty()) {
    std::vector<Msg> sm, rm;
    for (const Cross& c : cross) {
      const Item& a = items[c.u];   // smaller cluster: forms the block
      const Item& b2 = items[c.v];  // larger cluster: its owner sends T
      const size_t bytes = sizeof(double) * size_t(b2.r) * b2.r;
      if (b2.own) sm.push_back(Msg{owner(W, a.i), cd[b2.cd].T, bytes});
      if (a.own) {
        double* buf = ws_.alloc_n<double>(size_t(b2.r) * b2.r);
        rm.push_back(Msg{owner(W, b2.i), buf, bytes});
        t_remote[(int64_t(c.u) << 32) | uint32_t(c.v)] = buf;
      }
    }
    comm_->exchange(sm, rm, s_);
    F_->exchanges++;
  }
  if (!shared.empty()) {
    // block (l, i) = T_l^T (T_i^T M)^T, written over the stored (i, l), i < l
    GemmBatch two;
    for (Shared& sh : shared) {
      const Item& a = items[sh.u];
      const Item& b2 = items[sh.v];
      auto f = t_remote.find((int64_t(sh.u) << 32) | uint32_t(sh.v));
      const double* Tl = f != t_remote.end() ? f->second : (b2.own ? cd[b2.cd].T : nullptr);
      if (!Tl) invalid("rank-growth control: missing rotation of a shared block");
      double* tmp = ws_.alloc_n<double>(size_t(b2.r) * a.r);
      two.add(Tl, b2.r, a.row2 + sh.off * a.r, a.r, tmp, b2.r, b2.r, a.r, b2.r, 1.0, 0.0);
      scatter.add(tmp, b2.r, sh.q->b.p, sh.q->b.ld, a.r, b2.r, true);
    }
    launch_grouped_gemm(two, true, true, ws_, st_, s_);
  }
  launch_copies(scatter, ws_, st_, s_);
  std::vector<int> own_new(std::max<size_t>(1, cd.size()), 0);
  if (!cd.empty()) CK(cudaMemcpyAsync(own_new.data(), d_new, sizeof(int) * cd.size(), cudaMemcpyDeviceToHost, s_));
  CK(cudaStreamSynchronize(s_));
  std::vector<int> rn(items.size(), -1);
  for (size_t u = 0; u < items.size(); u++)
    if (items[u].own) rn[u] = own_new[items[u].cd];
  if (dist) {
    // new ranks of every pivot on every rank (the batch's host schedule needs them)
    int* d_send = upload(ws_, rn, s_, st_);
    int* d_recv = ws_.alloc_n<int>(rn.size() * nranks_);
    comm_->allgather(d_send, d_recv, rn.size() * sizeof(int), s_);
    std::vector<int> all(rn.size() * nranks_);
    CK(cudaMemcpyAsync(all.data(), d_recv, sizeof(int) * all.size(), cudaMemcpyDeviceToHost, s_));
    CK(cudaStreamSynchronize(s_));
    for (size_t u = 0; u < items.size(); u++) rn[u] = all[size_t(owner(W, items[u].i)) * rn.size() + u];
    F_->meta_bytes += double(rn.size() * sizeof(int)) * (nranks_ - 1);
  }
  tm_.end();
  for (size_t u = 0; u < items.size(); u++) {
    if (rn[u] <= 0 || rn[u] > items[u].r) invalid("rank-growth control: inconsistent consolidated rank");
    if (items[u].own) {
      F_->rc_before += items[u].r;
      F_->rc_after += rn[u];
    }
    W.r[items[u].i] = rn[u];
  }
  if (dist) CK(cudaMemcpyAsync(W.d_rank, W.r.data(), sizeof(int) * W.nc, cudaMemcpyHostToDevice, s_));
}

void Factorizer::eliminate_batch(std::vector<int>& piv, int colour, std::vector<int>& deferred) {
  const auto t_batch0 = std::chrono::steady_clock::now();
  hmark_ = t_batch0;
  WorkLevel& W = cur_;
  const Topo& T = *W.T;
  const int k = W.k;
  const bool dist = nranks_ > 1;
  // Independence guard: a batch may only contain eliminations whose touched
  // sets {i} u partners(i) are pairwise disjoint (true for the 9-colouring as
  // long as every partner is a neighbour; an incompressible well-separated
  // fill kept dense can break it).  Conflicting pivots are deferred to a
  // follow-up batch of the same colour, preserving their relative order.
  std::vector<std::vector<int>> gxp, gyp;  // partners of the kept pivots (reused below)
  {
    std::vector<int> keep;
    deferred.clear();
    if (mark_.size() != size_t(W.nc)) mark_.assign(W.nc, -1);
    ++stamp_;
    std::vector<int> xp, yp;
    for (int i : piv) {
      partners(W, i, xp, yp);
      bool clash = mark_[i] == stamp_;
      for (int j : xp) clash |= mark_[j] == stamp_;
      for (int j : yp) clash |= mark_[j] == stamp_;
      if (clash) {
        deferred.push_back(i);
        continue;
      }
      mark_[i] = stamp_;
      for (int j : xp) mark_[j] = stamp_;
      for (int j : yp) mark_[j] = stamp_;
      keep.push_back(i);
      gxp.push_back(xp);
      gyp.push_back(yp);
    }
    piv.swap(keep);
  }
  const int np = int(piv.size());
  hmark(0);
  CK(cudaStreamSynchronize(s_));  // staging buffers of earlier uploads are free after this
  if (work_->side.s) CK(cudaStreamSynchronize(work_->side.s));
  if (work_->ahead.s) CK(cudaStreamSynchronize(work_->ahead.s));
  ws_.reset();
  st_.reset();
  hmark(1);
  if (rank_tol_ > 0.0) consolidate_pivots(piv);
  struct PivInfo {
    int i, n, r, m, w;
    bool own;
    std::vector<int> xp, yp;
    std::vector<int> soff;  // slot column offsets (size nslots+1)
    double *S, *C, *Xt, *Xb;
    int* perm;
    int rec;
    const double* dinv = nullptr;
    const unsigned char* pflag = nullptr;
  };
  // Every rank walks all pivots of the batch (metadata); device work is done
  // for its own pivots only (all of them on one GPU).  The batch's fills are
  // determined by the partner sets: hybrid (p in yp u {i}, q in xp, q in
  // IL(p)) then P2P (xp pairs in each other's IL), in the reference order.
  std::vector<PivInfo> P(np);
  std::vector<int> own;  // indices into P
  struct FillHost { int kind, p, q, piv, dev; };  // dev: index among this rank's fills, or -1
  std::vector<FillHost> fh;
  std::vector<int> fill_off(np + 1, 0);  // fills of pivot t: fh[fill_off[t] .. fill_off[t+1])
  const int batch_id = int(F_->batches.size());
  int n_own_fills = 0, gmaxm = 0, shape_mx = 0;
  for (int t = 0; t < np; t++) {
    PivInfo& I = P[t];
    const int i = piv[t];
    I.i = i;
    I.n = W.n[i];
    I.r = W.r[i];
    I.m = I.n + I.r;
    I.own = mine(W, i);
    I.rec = -1;
    I.xp.swap(gxp[t]);
    I.yp.swap(gyp[t]);
    I.soff.assign(1, 0);
    for (int j : I.xp) I.soff.push_back(I.soff.back() + W.n[j]);
    for (int j : I.yp) I.soff.push_back(I.soff.back() + W.r[j]);
    I.soff.push_back(I.soff.back() + I.r);
    I.w = I.soff.back();
    gmaxm = std::max(gmaxm, I.m);
    if (dist) {
      LevelPivot lp{batch_id, owner(W, i), i, {}};
      for (int j : I.xp) lp.slots.push_back({0, j, W.n[j]});
      for (int j : I.yp) lp.slots.push_back({1, j, W.r[j]});
      lp.slots.push_back({1, i, I.r});
      lvl_piv_.push_back(std::move(lp));
    }
    fill_off[t] = int(fh.size());
    std::vector<int> ps(I.yp);
    ps.push_back(I.i);
    std::sort(ps.begin(), ps.end());
    auto note = [&](int kind, int p, int q) {
      fh.push_back({kind, p, q, t, I.own ? n_own_fills++ : -1});
      const int rows = kind == FILL_HYBRID ? W.r[p] : W.n[p];
      shape_mx = std::max(shape_mx, std::max(std::max(W.n[p], W.n[q]), rows));
    };
    for (int p : ps)
      for (int q : I.xp)
        if (T.in_il(p, q)) note(FILL_HYBRID, p, q);
    for (size_t u = 0; u < I.xp.size(); u++)
      for (size_t v = u + 1; v < I.xp.size(); v++)
        if (T.in_il(I.xp[u], I.xp[v])) note(FILL_P2P, I.xp[u], I.xp[v]);
    if (dist) {
      // checked for every pivot on every rank (each rank holds every pivot's
      // partner lists), so all ranks throw together instead of the owner alone
      // leaving its peers blocked in the next exchange
      const int o = owner(W, i);
      bool ok = holds(W, o, i);
      for (int j : I.xp) ok &= holds(W, o, j);
      for (int j : I.yp) ok &= holds(W, o, j);
      if (!ok)
        invalid("sharded factorization: a pivot couples to a cluster more than one cell away (a dense "
                "well-separated fill); factorize this system on one GPU");
    }
    if (!I.own) continue;
    own.push_back(t);
  }
  fill_off[np] = int(fh.size());
  // Pivot LU by size class (register panels up to 256 / 768 rows, shared-memory
  // panels beyond) when a large batch mixes sizes: clustered inputs put
  // few-point and thousand-point cells in one batch, and one launch chain sized
  // for the largest matrix would drag thousands of finished small ones through
  // every step (C4 leaf level: 1.15 s of LU).  Batches of similar sizes, and the
  // small batches of the coarse levels (where a second chain only adds latency),
  // stay one class.  Own pivots are taken in class order (stable); the decision
  // and each class's panel width follow the whole batch (all ranks), so the
  // factors of a pivot do not depend on the sharding.
  int class_cnt[3] = {0, 0, 0};
  auto size_class = [](int m) { return m <= 256 ? 0 : m <= 768 ? 1 : 2; };
  for (int t = 0; t < np; t++) class_cnt[size_class(P[t].m)]++;
  const bool lu_split = (class_cnt[0] >= 512 && class_cnt[1] + class_cnt[2] > 0) ||
                        (class_cnt[0] + class_cnt[1] >= 512 && class_cnt[2] > 0);
  auto lu_class = [&](int m) { return lu_split ? size_class(m) : 0; };
  int class_maxm[3] = {0, 0, 0};
  for (int t = 0; t < np; t++) class_maxm[lu_class(P[t].m)] = std::max(class_maxm[lu_class(P[t].m)], P[t].m);
  if (lu_split) {
    std::stable_sort(own.begin(), own.end(), [&](int a, int b) { return lu_class(P[a].m) < lu_class(P[b].m); });
    // the device fill states follow the order the own pivots are processed in
    int dev = 0;
    for (int t : own)
      for (int f = fill_off[t]; f < fill_off[t + 1]; f++) fh[f].dev = dev++;
  }
  const int no = int(own.size());
  // per-batch device results of this rank's pivots / fills
  double* d_nS = ws_.alloc_n<double>(std::max(1, no));
  double* d_nSi = ws_.alloc_n<double>(std::max(1, no));
  int* d_info = ws_.alloc_n<int>(std::max(1, no));
  const size_t nfill = size_t(n_own_fills);
  FillState* d_state = ws_.alloc_n<FillState>(std::max<size_t>(1, nfill));
  int* d_stats = ws_.alloc_n<int>(4);
  CK(cudaMemsetAsync(d_stats, 0, 16, s_));
  static const bool dbg = getenv("IFMM_DEBUG") != nullptr;
  hmark(11);
  // Own pivots are processed in one chunk per batch (host descriptor work for
  // a chunk is launched before the next one is built; measured at C3, smaller
  // chunks cost more in launch tails than they gain in overlap).  Pivots of a
  // batch are independent, and kernel shapes come from the whole batch (np,
  // gmaxm, shape_mx, fh.size()), so the arithmetic does not depend on chunking.
  const int nchunks = 1;
  bool est_pending = false;
  for (int ch = 0; ch < nchunks && no > 0; ch++) {
    const int u0 = int(int64_t(no) * ch / nchunks), u1 = int(int64_t(no) * (ch + 1) / nchunks);
    const int nc_ = u1 - u0;
    CopyBatch cb;
    std::vector<MatDesc> md;
    std::vector<XSolveDesc> xd;
    for (int u = u0; u < u1; u++) {
      PivInfo& I = P[own[u]];
      const int i = I.i;
      // S (factored in place) and the coupling panel C stay with the solve record
      I.S = F_->arena.alloc_n<double>(size_t(std::max(1, I.m)) * I.m);
      I.perm = F_->arena.alloc_n<int>(std::max(1, I.m));
      I.C = F_->arena.alloc_n<double>(size_t(std::max(1, I.n)) * I.w);
      I.Xt = ws_.alloc_n<double>(size_t(std::max(1, I.n)) * I.w);
      I.Xb = ws_.alloc_n<double>(size_t(std::max(1, I.r)) * I.w);
      md.push_back(MatDesc{I.S, I.m, I.m, I.perm, i});
      // gather S
      BlkRef Pii = p2p_ref(W, i, i, true);
      cb.add(Pii.p, Pii.ld, I.S, I.m, I.n, I.n);
      cb.add(W.U[i], I.n, I.S + size_t(I.n) * I.m, I.m, I.n, I.r);
      cb.add(W.U[i], I.n, I.S + I.n, I.m, I.r, I.n, true);
      cb.zero(I.S + I.n + size_t(I.n) * I.m, I.m, I.r, I.r);
      // gather C_top (n x w)
      int s = 0;
      for (int j : I.xp) {
        BlkRef b = p2p_ref(W, i, j, false);
        cb.add(b.p, b.ld, I.C + size_t(I.soff[s]) * I.n, I.n, I.n, W.n[j], b.trans);
        s++;
      }
      for (int j : I.yp) {
        BlkRef b = xy_ref(W, i, j, false);
        cb.add(b.p, b.ld, I.C + size_t(I.soff[s]) * I.n, I.n, I.n, W.r[j]);
        s++;
      }
      cb.zero(I.C + size_t(I.soff[s]) * I.n, I.n, I.n, I.r);
      xd.push_back(XSolveDesc{I.S, I.perm, I.C, I.Xt, I.Xb, nullptr, nullptr, nullptr, I.m, I.n, I.r, I.w - I.r, I.w, 0});
    }
    hmark(12);
    tm_.begin(PH_GATHER);
    launch_copies(cb, ws_, st_, s_);
    hmark(2);
    {
      const MatDesc* dmd = upload(ws_, md, s_, st_);
      int maxm = 0;
      for (auto& d : md) maxm = std::max(maxm, d.m);
      tm_.begin(PH_GJ);
      launch_norm1(dmd, nc_, maxm, d_nS + u0, s_);
      // panel width from the whole batch (across chunks and ranks): same arithmetic as one launch
      for (size_t q0 = 0; q0 < md.size();) {
        const int c = lu_class(md[q0].m);
        size_t q1 = q0;
        while (q1 < md.size() && lu_class(md[q1].m) == c) q1++;
        std::vector<MatDesc> sub(md.begin() + q0, md.begin() + q1);
        batched_lu(sub, dmd + q0, d_info + u0 + q0, ws_, st_, s_, class_maxm[c], &work_->ahead);
        q0 = q1;
      }
      // larger pivots keep their inverted diagonal blocks (written straight into the records'
      // arena) for the single-rhs sweeps (solve.cu)
      const LuDiag dg = launch_lu_diag_inv(md, dmd, ws_, st_, s_, tol_, &F_->arena, SOLVE_BLK_MIN_M);
      for (int u = u0; u < u1; u++) {
        PivInfo& I = P[own[u]];
        I.pflag = dg.pflag + (u - u0);
        I.dinv = I.m >= SOLVE_BLK_MIN_M ? dg.dinv + dg.h_off[u - u0] : nullptr;
      }
      // the condition estimates only gate the batch's read-back: run them on
      // the side stream, overlapped with the X solve, Schur update and fill
      // compression (which read the factors but never write them)
      SideStream& sd = work_->side;
      sd.ensure();
      CK(cudaEventRecord(sd.fork, s_));
      CK(cudaStreamWaitEvent(sd.s, sd.fork, 0));
      launch_lu_inv_norm1(dmd, nc_, maxm, dg, d_nSi + u0, sd.s);
      for (size_t q = 0; q < xd.size(); q++) {
        xd[q].dinv = dg.dinv + dg.h_off[q];
        xd[q].dflag = dg.flags + 2 * dg.h_foff[q];
        xd[q].pflag = dg.pflag + q;
      }
      CK(cudaEventRecord(sd.join, sd.s));
      est_pending = true;
    }
    hmark(3);
    // records + X = S^-1 C (getrs on the coupling panel)
    for (int u = u0; u < u1; u++) {
      PivInfo& I = P[own[u]];
      RecordH R{};
      R.level = k;
      R.index = I.i;
      R.n = I.n;
      R.r = I.r;
      R.w = I.w;
      R.lu = I.S;
      R.perm = I.perm;
      R.c = I.C;
      R.pos = nullptr;  // set by finish_level (one block per level)
      R.dinv = I.dinv;
      R.pflag = I.pflag;
      I.rec = int(F_->recs.size());
      F_->recs.push_back(R);
      std::vector<SlotRef> sl;
      for (int j : I.xp) sl.push_back({0, j, W.n[j]});
      for (int j : I.yp) sl.push_back({1, j, W.r[j]});
      sl.push_back({1, I.i, I.r});
      rec_slots_.push_back(sl);
      F_->rec_xp.push_back(I.xp);
      F_->rec_yp.push_back(I.yp);
      {
        const double m = I.m, n = I.n, w = I.w, h = I.w - I.r;
        F_->fl_exec += 2.0 / 3.0 * m * m * m + 2.0 * m * m * w;
        F_->fl_lu += 2.0 / 3.0 * m * m * m;
        F_->fl_x += 2.0 * m * m * w;
        F_->fl_ref += 2.0 / 3.0 * m * m * m + 2.0 * m * m * w + 2.0 * h * n * w;
        F_->solve_bytes += 8.0 * (2.0 * m * m + 2.0 * n * h);
      }
    }
    hmark(8);
    tm_.begin(PH_XGEMM);
    launch_lu_solve_x(xd, ws_, st_, s_);
    tm_.end();
    hmark(9);
    // symmetric Schur update on the block upper triangle: target -= C_a^T X_b,
    // one concatenated product per pivot (IFMM_SCHUR_GROUPED: one GEMM per block)
    SchurBatch sbat;
    for (int u = u0; u < u1; u++) {
      PivInfo& I = P[own[u]];
      const int nx = int(I.xp.size()), ny = int(I.yp.size());
      const int ns = nx + ny + 1;
      const int pv = sbat.begin_pivot(I.C, I.Xt, I.n, I.soff);
      auto slot_cluster = [&](int s) { return s < nx ? I.xp[s] : (s < nx + ny ? I.yp[s - nx] : I.i); };
      for (int a = 0; a < ns; a++)
        for (int b = a; b < ns; b++) {
          const bool ax = a < nx, bx = b < nx;
          const int ja = slot_cluster(a), jb = slot_cluster(b);
          const int da = I.soff[a + 1] - I.soff[a], db = I.soff[b + 1] - I.soff[b];
          if (a == ns - 1 && b == ns - 1) {
            BlkRef M = m2l_ref(W, I.i, I.i, true);
            cb.add(I.Xb + size_t(I.soff[b]) * I.r, I.r, M.p, M.ld, I.r, I.r, false, 1.0, true);
            set_pres(W.pm, W, I.i, I.i, 1);
            continue;
          }
          const BlkRef tgt = schur_target(W, (ax && bx) ? 0 : (ax ? 1 : 2), ja, jb);
          if (da == 0 || db == 0) continue;
          F_->fl_schur += 2.0 * I.n * da * db;
          sbat.set_target(pv, a, b, tgt.p, tgt.ld, tgt.trans);
        }
      sbat.finish_pivot(pv);
    }
    hmark(10);
    tm_.begin(PH_SCHUR);
    launch_schur(sbat, ws_, st_, s_);
    tm_.begin(PH_GATHER);
    launch_copies(cb, ws_, st_, s_);
    tm_.end();
    hmark(4);
    // fill-in compression of the chunk's fills (chains are per cluster, and
    // the chunk's clusters are disjoint from every other pivot's)
    CompressBatch cbz;
    cbz.chain_off.assign(1, 0);
    cbz.p2p_off.assign(1, 0);
    int dev0 = -1;
    for (int u = u0; u < u1; u++) {
      const int t = own[u];
      PivInfo& I = P[t];
      std::vector<std::vector<int>> byq(I.xp.size());
      for (int f = fill_off[t]; f < fill_off[t + 1]; f++) {
        const FillHost& h = fh[f];
        if (dev0 < 0) dev0 = h.dev;
        BlkRef M = m2l_ref(W, h.p, h.q, true);
        FillDesc D{};
        D.kind = h.kind;
        D.p = h.p;
        D.q = h.q;
        if (h.kind == FILL_HYBRID) {
          BlkRef F = xy_ref(W, h.q, h.p, false);
          D.F = F.p;
          D.ldF = W.n[h.q];
          D.transF = 1;
          D.rows = W.r[h.p];
        } else {
          BlkRef F = p2p_ref(W, h.p, h.q, false);
          D.F = F.p;
          D.ldF = F.ld;
          D.transF = 0;
          D.rows = W.n[h.p];
        }
        D.cols = W.n[h.q];
        D.n_p = W.n[h.p];
        D.n_q = W.n[h.q];
        D.Up = W.U[h.p];
        D.Uq = W.U[h.q];
        D.M = M.p;
        D.ldM = M.ld;
        D.transM = M.trans ? 1 : 0;
        D.Kf = std::max(1, std::min(96, std::min(D.rows, D.cols)));
        D.kfull = std::max(1, std::min(D.rows, D.cols));
        D.out = ws_.alloc_n<double>(size_t(D.rows + D.cols + 1) * D.Kf);
        const int fi = int(cbz.fills.size());
        cbz.fills.push_back(D);
        if (h.kind == FILL_HYBRID) {
          const size_t x = size_t(std::find(I.xp.begin(), I.xp.end(), h.q) - I.xp.begin());
          byq[x].push_back(fi);
        } else {
          cbz.p2p.push_back(fi);
        }
      }
      for (size_t x = 0; x < I.xp.size(); x++)
        if (!byq[x].empty()) {
          cbz.chain.insert(cbz.chain.end(), byq[x].begin(), byq[x].end());
          cbz.chain_off.push_back(int(cbz.chain.size()));
          cbz.chain_q.push_back(I.xp[x]);
        }
      cbz.p2p_off.push_back(int(cbz.p2p.size()));
    }
    cbz.rank_host = W.r.data();
    cbz.shape_mx = shape_mx;  // worker shapes from the whole batch (across chunks and ranks)
    cbz.shape_nf = int(fh.size());
    cbz.full_rank_ok = t_->sparse ? 1 : 0;
    hmark(5);
    tm_.begin(PH_COMPRESS);
    if (!cbz.fills.empty())
      run_compression(cbz, tol_, S_->d_probe, S_->probe_maxm, W.d_rank, d_state + dev0, d_stats, ws_, st_, s_,
                      dbg ? 1 : 0);
    tm_.end();
    hmark(6);
  }
  // the other ranks' pivots: Schur targets and fill M2L blocks exist here too
  // (presence flags; storage where this rank holds them)
  for (int t = 0; t < np; t++) {
    PivInfo& I = P[t];
    if (I.own) continue;
    const int nx = int(I.xp.size()), ny = int(I.yp.size());
    const int ns = nx + ny + 1;
    auto slot_cluster = [&](int s) { return s < nx ? I.xp[s] : (s < nx + ny ? I.yp[s - nx] : I.i); };
    for (int a = 0; a < ns; a++)
      for (int b = a; b < ns; b++) {
        const int ja = slot_cluster(a), jb = slot_cluster(b);
        if (a == ns - 1 && b == ns - 1) {
          m2l_ref(W, I.i, I.i, true);
          set_pres(W.pm, W, I.i, I.i, 1);
        } else {
          schur_target(W, (a < nx && b < nx) ? 0 : (a < nx ? 1 : 2), ja, jb);
        }
      }
    for (int f = fill_off[t]; f < fill_off[t + 1]; f++) m2l_ref(W, fh[f].p, fh[f].q, true);
  }
  // read back: pivot conditioning, ranks, fill outcomes, counters
  if (est_pending) CK(cudaStreamWaitEvent(s_, work_->side.join, 0));
  const auto t_sync0 = std::chrono::steady_clock::now();
  std::vector<double> nS(no), nSi(no);
  std::vector<int> info(no), stats(4);
  std::vector<FillState> state(nfill);
  std::vector<int> r_before;
  if (dist) r_before = W.r;
  if (no) {
    CK(cudaMemcpyAsync(nS.data(), d_nS, sizeof(double) * no, cudaMemcpyDeviceToHost, s_));
    CK(cudaMemcpyAsync(nSi.data(), d_nSi, sizeof(double) * no, cudaMemcpyDeviceToHost, s_));
    CK(cudaMemcpyAsync(info.data(), d_info, sizeof(int) * no, cudaMemcpyDeviceToHost, s_));
  }
  if (nfill) CK(cudaMemcpyAsync(state.data(), d_state, sizeof(FillState) * nfill, cudaMemcpyDeviceToHost, s_));
  CK(cudaMemcpyAsync(stats.data(), d_stats, 16, cudaMemcpyDeviceToHost, s_));
  CK(cudaMemcpyAsync(W.r.data(), W.d_rank, sizeof(int) * W.nc, cudaMemcpyDeviceToHost, s_));
  CK(cudaStreamSynchronize(s_));
  const auto t_sync1 = std::chrono::steady_clock::now();
  hmark(13);
  if (F_->host_lvl_ms.size() <= size_t(k)) F_->host_lvl_ms.resize(k + 1, std::array<double, 2>{});
  F_->host_lvl_ms[k][0] += std::chrono::duration<double, std::milli>(t_sync0 - t_batch0).count();
  F_->host_lvl_ms[k][1] += std::chrono::duration<double, std::milli>(t_sync1 - t_sync0).count();
  tm_.collect(F_.get(), k);
  if (getenv("IFMM_COND_LOG")) {
    double mx = 0, sum = 0;
    int imx = -1, mmx = 0;
    for (int u = 0; u < no; u++) {
      double c = nS[u] * nSi[u];
      sum += std::log10(std::max(c, 1.0));
      if (c > mx) { mx = c; imx = P[own[u]].i; mmx = P[own[u]].m; }
    }
    fprintf(stderr, "cond level=%d colour=%d pivots=%d max=%.3e (cluster %d, m=%d) geo-mean=%.3e\n", k, colour, no, mx,
            imx, mmx, std::pow(10.0, no ? sum / no : 0.0));
  }
  // first numerically singular own pivot (batch position), if any
  int err_pos = INT_MAX, err_index = -1;
  double err_cond = 0;
  const bool record_only = (flags_ & IFMM_FLAG_RECORD_SINGULAR) != 0;
  for (int u = 0; u < no; u++) {
    const PivInfo& I = P[own[u]];
    if (I.m == 0) continue;  // an empty cluster (clustered inputs): nothing to eliminate
    double rc = (info[u] != 0) ? 0.0 : 1.0 / (nS[u] * nSi[u]);
    const double cond = 1.0 / std::max(rc, 1e-300);
    F_->stats[k].max_cond = std::max(F_->stats[k].max_cond, std::isfinite(cond) ? cond : INFINITY);
    if (!std::isfinite(rc) || rc <= 1.0 / cond_limit_) {
      if (record_only) {
        F_->singular.push_back(SingularH{k, I.i, cond});
        continue;
      }
      if (err_pos == INT_MAX) {
        err_pos = own[u];
        err_index = I.i;
        err_cond = cond;
      }
    }
  }
  // fill outcomes in global fill order (-1: another rank's fill)
  std::vector<int> gstat(fh.size(), -1);
  for (size_t f = 0; f < fh.size(); f++)
    if (fh[f].dev >= 0) gstat[f] = state[fh[f].dev].status;
  if (dist) {
    // all-gather: first failure, counters, ranks, fill outcomes of every rank
    tm_.begin(PH_COMM);
    const size_t L = 8 + size_t(W.nc) + fh.size();
    std::vector<int> mine_meta(L, 0);
    mine_meta[0] = err_pos;
    mine_meta[1] = err_index;
    memcpy(&mine_meta[2], &err_cond, sizeof(double));
    mine_meta[4] = stats[0];
    mine_meta[5] = stats[1];
    mine_meta[6] = stats[2];
    std::copy(W.r.begin(), W.r.end(), mine_meta.begin() + 8);
    std::copy(gstat.begin(), gstat.end(), mine_meta.begin() + 8 + W.nc);
    int* d_send = upload(ws_, mine_meta, s_, st_);
    int* d_recv = ws_.alloc_n<int>(L * nranks_);
    comm_->allgather(d_send, d_recv, L * sizeof(int), s_);
    std::vector<int> all(L * nranks_);
    CK(cudaMemcpyAsync(all.data(), d_recv, sizeof(int) * all.size(), cudaMemcpyDeviceToHost, s_));
    CK(cudaStreamSynchronize(s_));
    stats.assign(4, 0);
    err_pos = INT_MAX;
    for (int q = 0; q < nranks_; q++) {
      const int* m = &all[size_t(q) * L];
      if (m[0] < err_pos) {
        err_pos = m[0];
        err_index = m[1];
        memcpy(&err_cond, &m[2], sizeof(double));
      }
      stats[0] += m[4];
      stats[1] += m[5];
      stats[2] = std::max(stats[2], m[6]);
      for (int c = 0; c < W.nc; c++) W.r[c] = std::max(W.r[c], m[8 + c]);  // ranks only grow
    }
    for (size_t f = 0; f < fh.size(); f++) gstat[f] = all[size_t(owner(W, P[fh[f].piv].i)) * L + 8 + W.nc + f];
    CK(cudaMemcpyAsync(W.d_rank, W.r.data(), sizeof(int) * W.nc, cudaMemcpyHostToDevice, s_));
    F_->meta_bytes += double(L * sizeof(int)) * (nranks_ - 1);
  }
  if (err_pos != INT_MAX) {
    char buf[256];
    snprintf(buf, sizeof buf, "pivot for cluster %d at level %d is numerically singular (condition estimate %.2e)",
             err_index, k, err_cond);
    throw SingularPivot(k, err_index, err_cond, buf);
  }
  LevelStatsH& LS = F_->stats[k];
  LS.compressed += stats[0];
  LS.dense_kept += stats[1];
  LS.max_rank = std::max(LS.max_rank, stats[2]);
  CopyBatch zero_dropped;  // sharded: stored copies of fills another rank dropped
  for (size_t f = 0; f < fh.size(); f++) {
    const FillHost& h = fh[f];
    if (dbg && h.dev >= 0)
      fprintf(stderr, "fill k=%d kind=%d p=%d q=%d status=%d aca=%d rank=%d rank_p=%d\n", k, h.kind, h.p, h.q,
              state[h.dev].status, state[h.dev].k, state[h.dev].r, W.r[h.p]);
    if (gstat[f] != 0) continue;
    if (h.kind == FILL_HYBRID) {
      set_px(W, h.q, h.p, 0);
      if (h.dev < 0) {
        BlkRef F = xy_ref(W, h.q, h.p, false);
        if (F.p) zero_dropped.zero(F.p, F.ld, W.n[h.q], W.r[h.p]);
      }
    } else {
      set_pp(W, h.p, h.q, 0);
      if (h.dev < 0) {
        BlkRef F = p2p_ref(W, h.p, h.q, false);
        if (F.p) zero_dropped.zero(F.p, F.ld, W.n[std::min(h.p, h.q)], W.n[std::max(h.p, h.q)]);
      }
    }
  }
  for (int t = 0; t < np; t++) W.dead[P[t].i] = 1;
  if (dist) {
    // halo: every block / basis the batch wrote goes from the pivot's owner
    // to each other rank storing it (canonical order: pivot, then kind)
    std::vector<std::vector<HaloItem>> send(nranks_), recv(nranks_);
    std::vector<HaloItem> items;
    for (int t = 0; t < np; t++) {
      const PivInfo& I = P[t];
      auto cpit = cons_parts_.find(I.i);  // rank-growth control: the M2L blocks the pivot's rotation rewrote
      if (!I.own) {  // every item of a pivot lies among {i} u partners: none stored here -> none received
        bool any = holds1(W, I.i);
        for (int j : I.xp) any = any || holds1(W, j);
        for (int j : I.yp) any = any || holds1(W, j);
        if (cpit != cons_parts_.end())
          for (int l : cpit->second) any = any || holds1(W, l);
        if (!any) continue;
      }
      items.clear();
      for (size_t a = 0; a < I.xp.size(); a++)
        for (size_t b = a; b < I.xp.size(); b++) {
          const int ja = std::min(I.xp[a], I.xp[b]), jb = std::max(I.xp[a], I.xp[b]);
          if (pp_present(W, ja, jb)) items.push_back({HALO_P2P, ja, jb, 0});
        }
      std::vector<int> ys(I.yp);
      ys.push_back(I.i);
      for (int x : I.xp)
        for (int y : ys)
          if (px_present(W, x, y)) items.push_back({HALO_XY, x, y, 0});
      for (size_t a = 0; a < ys.size(); a++)
        for (size_t b = a; b < ys.size(); b++) {
          const int ja = std::min(ys[a], ys[b]), jb = std::max(ys[a], ys[b]);
          if (pm_present(W, ja, jb)) items.push_back({HALO_M2L, ja, jb, 0});
        }
      for (int f = fill_off[t]; f < fill_off[t + 1]; f++)  // M2L absorption targets
        items.push_back({HALO_M2L, std::min(fh[f].p, fh[f].q), std::max(fh[f].p, fh[f].q), 0});
      for (int x : I.xp)
        if (W.r[x] > r_before[x]) items.push_back({HALO_U, x, 0, r_before[x]});
      if (cpit != cons_parts_.end())
        for (int l : cpit->second) {
          // a block shared with another consolidated pivot was formed by the smaller cluster's owner
          if (l < I.i && cons_parts_.count(l)) continue;
          items.push_back({HALO_M2L, std::min(I.i, l), std::max(I.i, l), 0});
        }
      const int q = owner(W, I.i);
      for (const HaloItem& it : items)
        if (halo_route(*part_, k, q, rank_, it.a, it.kind == HALO_U ? -1 : it.b,
                       [&](int s) { send[s].push_back(it); }))
          recv[q].push_back(it);
    }
    tm_.begin(PH_COMM);
    halo_exchange(W, send, recv, &zero_dropped);
    tm_.end();
  }
  hmark(7);
  (void)colour;
}

Factorizer::HaloRef Factorizer::halo_ref(WorkLevel& W, const HaloItem& it) {
  switch (it.kind) {
    case HALO_P2P: {
      BlkRef b = p2p_ref(W, it.a, it.b, false);
      return {b.p, b.ld, W.n[it.a], W.n[it.b]};
    }
    case HALO_XY: {
      BlkRef b = xy_ref(W, it.a, it.b, false);
      return {b.p, b.ld, W.n[it.a], W.r[it.b]};
    }
    case HALO_M2L: {
      BlkRef b = m2l_ref(W, it.a, it.b, false);
      return {b.p, b.ld, W.r[it.a], W.r[it.b]};
    }
    default: {
      double* u = W.U[it.a];
      return {u ? u + size_t(it.c0) * W.n[it.a] : nullptr, W.n[it.a], W.n[it.a], W.r[it.a] - it.c0};
    }
  }
}

void Factorizer::halo_exchange(WorkLevel& W, const std::vector<std::vector<HaloItem>>& send,
                               const std::vector<std::vector<HaloItem>>& recv, CopyBatch* local) {
  CopyBatch pack, unpack;
  std::vector<Msg> sm, rm;
  auto stage = [&](const std::vector<HaloItem>& items, int peer, bool out) {
    size_t tot = 0;
    for (const HaloItem& it : items) {
      const HaloRef r = halo_ref(W, it);
      if (r.rows > 0 && r.cols > 0) tot += size_t(r.rows) * r.cols;
    }
    if (tot == 0) return;
    double* buf = ws_.alloc_n<double>(tot);
    size_t off = 0;
    for (const HaloItem& it : items) {
      const HaloRef r = halo_ref(W, it);
      if (r.rows <= 0 || r.cols <= 0) continue;
      if (!r.p) {
        char m[160];
        snprintf(m, sizeof m, "sharded factorization: halo block (kind %d, %d, %d) of level %d is not stored on rank %d",
                 it.kind, it.a, it.b, W.k, rank_);
        invalid(m);
      }
      if (out) pack.add(r.p, r.ld, buf + off, r.rows, r.rows, r.cols);
      else unpack.add(buf + off, r.rows, r.p, r.ld, r.rows, r.cols);
      off += size_t(r.rows) * r.cols;
    }
    (out ? sm : rm).push_back(Msg{peer, buf, tot * sizeof(double)});
    if (out) F_->halo_bytes += double(tot) * sizeof(double);
  };
  for (int s = 0; s < nranks_; s++) {
    if (s == rank_) continue;
    stage(send[s], s, true);
    stage(recv[s], s, false);
  }
  launch_copies(pack, ws_, st_, s_);
  comm_->exchange(sm, rm, s_);
  F_->exchanges++;
  if (local) launch_copies(*local, ws_, st_, s_);
  launch_copies(unpack, ws_, st_, s_);
}

void Factorizer::finish_level(int rec_begin) {
  WorkLevel& W = cur_;
  const int k = W.k;
  // level vector layout: x slots at lvl_base[k] (prefix of n), y slots at lvl_base[k-1] (prefix of final r)
  std::vector<int64_t> xoff(W.nc + 1, 0), yoff(W.nc + 1, 0);
  for (int i = 0; i < W.nc; i++) {
    xoff[i + 1] = xoff[i] + W.n[i];
    yoff[i + 1] = yoff[i] + W.r[i];
  }
  const int64_t xb = F_->lvl_base[k];
  const int64_t yb = xb + xoff[W.nc];
  F_->lvl_base[k - 1] = yb;
  F_->vec_size = yb + yoff[W.nc];
  // partner positions: each record's pos array is the concatenation of its
  // slots' ranges [base, base + dim); ship one (base, dim, out) triple per slot
  // and expand on the device into one block for the level
  std::vector<PosRun> runs;
  std::vector<int64_t> posoff;
  int64_t total = 0;
  for (size_t rr = rec_begin; rr < F_->recs.size(); rr++) {
    RecordH& R = F_->recs[rr];
    R.xoff = xb + xoff[R.index];
    posoff.push_back(total);
    for (const SlotRef& sr : rec_slots_[rr]) {
      if (sr.dim <= 0) continue;
      const int64_t base = sr.kind == 0 ? xb + xoff[sr.j] : yb + yoff[sr.j];
      runs.push_back(PosRun{base, total, sr.dim, 0});
      total += sr.dim;
    }
  }
  if (total > 0) {
    int* d = F_->arena.alloc_n<int>(size_t(total));
    const PosRun* druns = upload(ws_, runs, s_, st_);
    launch_pos_expand(druns, int(runs.size()), d, s_);
    for (size_t rr = rec_begin, u = 0; rr < F_->recs.size(); rr++, u++) F_->recs[rr].pos = d + posoff[u];
  }
  if (nranks_ > 1) {
    // sharded solve: the solve-vector runs each rank writes per batch -- the
    // forward sweep writes a pivot's partner slots (its pos runs), the
    // backward sweep its own x slots; pivots are in batch order, owners vary
    std::vector<std::vector<std::vector<int64_t>>> fw, bw;  // [batch][rank] -> pairs
    int b0 = -1;
    for (const LevelPivot& lp : lvl_piv_) {
      if (b0 < 0) b0 = lp.batch;
      const size_t bi = size_t(lp.batch - b0);
      if (fw.size() <= bi) {
        fw.resize(bi + 1, std::vector<std::vector<int64_t>>(nranks_));
        bw.resize(bi + 1, std::vector<std::vector<int64_t>>(nranks_));
      }
      for (const SlotRef& sr : lp.slots) {
        if (sr.dim <= 0) continue;
        fw[bi][lp.owner].push_back(sr.kind == 0 ? xb + xoff[sr.j] : yb + yoff[sr.j]);
        fw[bi][lp.owner].push_back(sr.dim);
      }
      if (W.n[lp.i] > 0) {
        bw[bi][lp.owner].push_back(xb + xoff[lp.i]);
        bw[bi][lp.owner].push_back(W.n[lp.i]);
      }
    }
    for (size_t bi = 0; bi < fw.size(); bi++) {
      BatchH& B = F_->batches[size_t(b0) + bi];
      B.fwd_off.assign(1, 0);
      B.bwd_off.assign(1, 0);
      for (int q = 0; q < nranks_; q++) {
        B.fwd_runs.insert(B.fwd_runs.end(), fw[bi][q].begin(), fw[bi][q].end());
        B.bwd_runs.insert(B.bwd_runs.end(), bw[bi][q].begin(), bw[bi][q].end());
        B.fwd_off.push_back(int(B.fwd_runs.size() / 2));
        B.bwd_off.push_back(int(B.bwd_runs.size() / 2));
      }
    }
    lvl_piv_.clear();
  }
  CK(cudaStreamSynchronize(s_));
  st_.reset();
}

void Factorizer::factor_top() {
  WorkLevel& W = cur_;  // level 2, fully eliminated
  std::vector<int64_t> off(W.nc + 1, 0);
  for (int i = 0; i < W.nc; i++) off[i + 1] = off[i] + W.r[i];
  const int M = int(off[W.nc]);
  F_->top_dim = M;
  F_->top_off = off;
  ws_.reset();
  st_.reset();
  F_->top_lu = F_->arena.alloc_n<double>(size_t(std::max(1, M)) * std::max(1, M));
  F_->top_perm = F_->arena.alloc_n<int>(std::max(1, M));
  CK(cudaMemsetAsync(F_->top_lu, 0, sizeof(double) * std::max(1, M) * std::max(1, M), s_));
  CopyBatch cb;
  for (int i = 0; i < W.nc; i++)
    for (int j = 0; j < W.nc; j++) {
      if (W.T->slot(i, j) < 0 && W.T->slot(j, i) < 0) continue;
      if (W.T->slot(std::min(i, j), std::max(i, j)) < 0) continue;
      if (!pm_present(W, i, j)) continue;
      BlkRef b = m2l_ref(W, i, j, false);
      if (!b.p) continue;
      cb.add(b.p, b.ld, F_->top_lu + off[i] + size_t(off[j]) * M, M, W.r[i], W.r[j], b.trans);
    }
  launch_copies(cb, ws_, st_, s_);
  F_->fl_exec += 2.0 / 3.0 * double(M) * M * M;
  F_->fl_ref += 2.0 / 3.0 * double(M) * M * M;
  F_->solve_bytes += 8.0 * double(M) * M;
  int info = 0;
  if (M > 0) {
    // dense LU of the level-2 system (ifmm/solver.py:528-546: lu_factor)
    std::vector<MatDesc> md(1);
    md[0] = MatDesc{F_->top_lu, M, M, F_->top_perm, -1};
    const MatDesc* dmd = upload(ws_, md, s_, st_);
    int* d_info = ws_.alloc_n<int>(1);
    tm_.begin(PH_TOP);
    batched_lu(md, dmd, d_info, ws_, st_, s_, 0, &work_->ahead);
    CK(cudaMemcpyAsync(&info, d_info, sizeof(int), cudaMemcpyDeviceToHost, s_));
  }
  CK(cudaStreamSynchronize(s_));
  tm_.collect(F_.get(), 1);
  if (info != 0) {
    // scipy's lu_factor only warns on an exactly singular top system and the
    // solve then returns inf/nan; here the factorization fails loudly instead
    char buf[160];
    snprintf(buf, sizeof buf, "the level-2 top system is exactly singular (zero pivot in column %d)", info - 1);
    throw SingularPivot(1, info - 1, INFINITY, buf);
  }
}

FactorH* Factorizer::run() {
  auto t0 = std::chrono::steady_clock::now();
  // exact mode keeps identity bases and adds fills to the far blocks as they are:
  // a rotated basis would break that
  if (rank_tol_ > 0.0 && !(tol_ > 0.0)) invalid("rank_tol needs a compression tolerance tol > 0 (exact mode keeps identity bases)");
  if (getenv("IFMM_HOST_PROF")) fprintf(stderr, "host factorize begin\n");
  tm_.on = (flags_ & IFMM_FLAG_TIMING) != 0;
  tm_.s = s_;
  F_.reset(new FactorH);
  F_->store = S_;
  F_->tree = t_;
  F_->tol = tol_;
  F_->stream = s_;
  const int K = t_->depth;
  if (comm_ && comm_->size() > 1) {
    rank_ = comm_->rank();
    nranks_ = comm_->size();
    std::vector<std::vector<int>> grid(K + 1);
    for (int k = 2; k <= K; k++) grid[k] = t_->lv[k].grid;
    part_ = std::make_shared<Partition>(make_partition(t_->dim, K, nranks_, rank_, grid));
    F_->comm = comm_;
    F_->part = part_;
  }
  F_->stats.assign(K + 1, LevelStatsH{});
  F_->lvl_base.assign(K + 1, 0);
  F_->lvl_base[K] = 0;
  F_->r_m = S_->max_init_rank;
  const int ncol = [&] { int c = 1; for (int d = 0; d < t_->dim; d++) c *= 3; return c; }();
  static const bool hprof = getenv("IFMM_HOST_PROF") != nullptr;  // debug: host time outside the batches
  auto since = [](std::chrono::steady_clock::time_point a) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a).count();
  };
  for (int k = K; k >= 2; k--) {
    const auto tl0 = std::chrono::steady_clock::now();
    if (k == K) {
      tm_.begin(PH_TRANSITION);
      start_leaf_level();
    } else {
      prev_ = std::move(cur_);
      cur_ = WorkLevel{};
      tm_.begin(PH_TRANSITION);
      start_parent_level(prev_, k);
      CK(cudaStreamSynchronize(s_));
      tm_.collect(F_.get(), k);
      prev_ = WorkLevel{};
    }
    if (hprof) fprintf(stderr, "host level %d: start %.1f ms\n", k, since(tl0));
    F_->stats[k].clusters = cur_.nc;
    const int rec_begin = int(F_->recs.size());
    for (int c = 0; c < ncol; c++) {
      std::vector<int> piv;
      for (int i = 0; i < cur_.nc; i++)
        if (cur_.T->colour[i] == c) piv.push_back(i);
      std::vector<int> deferred;
      while (!piv.empty()) {
        const int r0 = int(F_->recs.size());
        eliminate_batch(piv, c, deferred);
        F_->batches.push_back(BatchH{k, c, r0, int(F_->recs.size()), nullptr, 0, 0, 0});
        if (!deferred.empty()) F_->deferred_batches++;
        piv.swap(deferred);
      }
    }
    const auto tf0 = std::chrono::steady_clock::now();
    finish_level(rec_begin);
    if (hprof) {
      fprintf(stderr, "host level %d: finish %.1f ms, level total %.1f ms\n", k, since(tf0), since(tl0));
      fprintf(stderr, "  batches: guard %.1f sync %.1f meta %.1f gatherdesc %.1f gatherlaunch %.1f gj %.1f records %.1f "
              "xlaunch %.1f schurloop %.1f schurlaunch %.1f fills %.1f compress %.1f wait %.1f post %.1f\n",
              hsec_[0], hsec_[1], hsec_[11], hsec_[12], hsec_[2], hsec_[3], hsec_[8], hsec_[9], hsec_[10], hsec_[4],
              hsec_[5], hsec_[6], hsec_[13], hsec_[7]);
    }
    for (double& h : hsec_) h = 0.0;
    F_->r_m = std::max(F_->r_m, F_->stats[k].max_rank);
  }
  const auto tt0 = std::chrono::steady_clock::now();
  factor_top();
  if (hprof) fprintf(stderr, "host top %.1f ms\n", since(tt0));
  const auto tr0 = std::chrono::steady_clock::now();
  // device copies of the batch record tables
  for (BatchH& b : F_->batches) {
    std::vector<RecordH> v(F_->recs.begin() + b.rec0, F_->recs.begin() + b.rec1);
    RecordH* d = F_->arena.alloc_n<RecordH>(v.size());
    CK(cudaMemcpyAsync(d, v.data(), sizeof(RecordH) * v.size(), cudaMemcpyHostToDevice, s_));
    b.d_recs = d;
    for (auto& r : v) {
      b.maxn = std::max(b.maxn, r.n);
      b.maxw = std::max(b.maxw, r.w);
      b.maxm = std::max(b.maxm, r.n + r.r);
    }
  }
  F_->g_off.resize(F_->recs.size() + 1, 0);
  for (size_t r = 0; r < F_->recs.size(); r++) F_->g_off[r + 1] = F_->g_off[r] + F_->recs[r].n;
  F_->g_size = F_->g_off.back();
  F_->d_g_off = F_->arena.alloc_n<int64_t>(F_->g_off.size());
  CK(cudaMemcpyAsync(F_->d_g_off, F_->g_off.data(), sizeof(int64_t) * F_->g_off.size(), cudaMemcpyHostToDevice, s_));
  CK(cudaStreamSynchronize(s_));
  if (hprof) fprintf(stderr, "host record tables %.1f ms\n", since(tr0));
  const auto tc0 = std::chrono::steady_clock::now();
  cur_ = WorkLevel{};
  if (hprof) fprintf(stderr, "host release %.1f ms\n", since(tc0));
  // level arenas stay allocated with the store (zeroed again on next reset)
  F_->fl_exec += F_->fl_schur;
  F_->ms_total = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return F_.release();
}

FactorH::~FactorH() {
  if (own_stream && stream) cudaStreamDestroy(stream);
}

FactorH* factorize(StoreH* S, double tol, int flags, double cond_limit, double rank_tol) {
  ensure_device();
  std::lock_guard<std::mutex> lock(S->work->mu);  // one factorization per store at a time
  Factorizer f(S, S->work.get(), S->stream, nullptr, tol < 0 ? S->tol : tol, flags, cond_limit > 0 ? cond_limit : 1e12,
               rank_tol > 0 ? rank_tol : 0.0);
  return f.run();
}

FactorH* factorize_sharded(StoreH* S, std::shared_ptr<Comm> comm, double tol, int flags, double cond_limit,
                           double rank_tol) {
  ensure_device();
  if (!comm) invalid("null communicator");
  std::lock_guard<std::mutex> lock(S->work->mu);
  Factorizer f(S, S->work.get(), S->stream, std::move(comm), tol < 0 ? S->tol : tol, flags,
               cond_limit > 0 ? cond_limit : 1e12, rank_tol > 0 ? rank_tol : 0.0);
  return f.run();
}

// Virtual ranks as threads on one GPU: each has its own workspaces, stream and
// records; the store (initial operators, read-only here) is shared.
void factorize_emulated(StoreH* S, int nranks, double tol, int flags, double cond_limit, std::vector<FactorH*>& out,
                        double rank_tol) {
  ensure_device();
  if (nranks < 1) invalid("nranks must be >= 1");
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(S->work->mu);
  auto world = std::make_shared<LocalWorld>(nranks);
  std::vector<std::unique_ptr<FactorH>> res(nranks);
  std::vector<std::exception_ptr> errs(nranks);
  std::vector<std::thread> th;
  for (int r = 0; r < nranks; r++)
    th.emplace_back([&, r] {
      try {
        CK(cudaSetDevice(dev));
        std::unique_ptr<FactorWork> work(new FactorWork);
        cudaStream_t s;
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        std::shared_ptr<Comm> c = std::make_shared<LocalComm>(world, r);
        std::unique_ptr<FactorH> F;
        try {
          Factorizer f(S, work.get(), s, c, tol < 0 ? S->tol : tol, flags, cond_limit > 0 ? cond_limit : 1e12,
                       rank_tol > 0 ? rank_tol : 0.0);
          F.reset(f.run());
        } catch (...) {
          cudaStreamSynchronize(s);
          cudaStreamDestroy(s);
          throw;
        }
        F->own_stream = true;
        F->own_work = std::move(work);  // its level arenas return to the slab cache with the factorization
        res[r] = std::move(F);
      } catch (...) {
        errs[r] = std::current_exception();
        world->fail();
      }
    });
  for (auto& t : th) t.join();
  // a real failure (e.g. SingularPivot, raised on every rank) wins over the
  // "another virtual rank failed" aborts it caused
  std::exception_ptr first;
  for (int r = 0; r < nranks && !first; r++)
    if (errs[r]) {
      try {
        std::rethrow_exception(errs[r]);
      } catch (const Error& e) {
        if (std::string(e.what()) != "another virtual rank failed") first = errs[r];
      } catch (...) {
        first = errs[r];
      }
    }
  for (int r = 0; r < nranks && !first; r++)
    if (errs[r]) first = errs[r];
  if (first) std::rethrow_exception(first);
  out.clear();
  for (auto& f : res) out.push_back(f.release());
}

}  // namespace ifmm
