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
#include <algorithm>
#include <chrono>
#include <cmath>

#include "core.cuh"
#include "cta_la.cuh"

namespace ifmm {

// ------------------------------------------------------------------ compression kernel
enum FillKind : int { FILL_HYBRID = 0, FILL_P2P = 1 };

struct FillDesc {
  int kind, p, q;
  double* F;     // fill block
  int ldF, transF;
  int n_p, n_q;
  double* Up;    // n_p x cap (ld n_p)
  double* Uq;    // n_q x cap (ld n_q)
  double* M;     // M2L(p,q) storage
  int ldM, transM;
};

struct PivotWork {
  int f0, f1;
  double* scratch;
  int MX, K;
};

struct CompressParams {
  double tol;          // ACA / truncation tolerance
  const int* probes;   // (maxm+1) x 10 probe table
  int probe_maxm;
  int* rank;           // level ranks (device)
  int* status;         // per fill: 0 compressed, 1 kept dense
  int* stats;          // [compressed, dense_kept, max_rank]
  int debug;
};

__device__ inline void fill_zero(const FillDesc& D, int rows, int cols) {
  for (int e = threadIdx.x; e < rows * cols; e += blockDim.x) {
    const int a = e % rows, b = e / rows;
    if (D.transF) D.F[b + (size_t)a * D.ldF] = 0.0;
    else D.F[a + (size_t)b * D.ldF] = 0.0;
  }
}

// M2L(p,q) += X E^T  (X: rows x r, ld ldx ; E: cols x r, ld lde)
__device__ inline void m2l_add_product(const FillDesc& D, const double* X, int ldx, const double* E, int lde, int rows,
                                       int cols, int r) {
  for (int e = threadIdx.x; e < rows * cols; e += blockDim.x) {
    const int a = e % rows, b = e / rows;
    double v = 0.0;
    for (int t = 0; t < r; t++) v = fma(X[a + (size_t)t * ldx], E[b + (size_t)t * lde], v);
    if (D.transM) D.M[b + (size_t)a * D.ldM] += v;
    else D.M[a + (size_t)b * D.ldM] += v;
  }
}

// New orthonormal directions of X (nU x r, in H) outside U (nU x rU), weighted
// by `wsig` (per-column scale, or null for identity), appended to U.
// Follows ifmm/solver.py:334-358 using the identity sv(M)=sv(res*diag(sig)).
// Returns number of appended columns.
__device__ int new_dirs_append(double* H, int nU, int r, double* U, int rU, const double* wsig, double cutoff,
                               double* E, double* sig2, int* ord2, CtaShared& sh) {
  const int cap = nU - rU;
  if (cap <= 0 || r == 0) return 0;
  cta_project_out(H, nU, nU, r, U, nU, rU, E);
  cta_project_out(H, nU, nU, r, U, nU, rU, E);
  if (wsig)
    for (int e = threadIdx.x; e < nU * r; e += blockDim.x) H[e] *= wsig[e / nU];
  __syncthreads();
  cta_jacobi(H, nU, r, nU, nullptr, 0, sig2, ord2, sh);
  int w = 0;
  for (int t = 0; t < r; t++) w += (sig2[ord2[t]] > cutoff);
  w = min(w, cap);
  double* W = U + (size_t)rU * nU;
  for (int e = threadIdx.x; e < nU * w; e += blockDim.x) {
    const int i = e % nU, c = e / nU;
    const int col = ord2[c];
    W[i + (size_t)c * nU] = H[i + (size_t)col * nU] / sig2[col];
  }
  __syncthreads();
  if (w > 0) cta_project_out(W, nU, nU, w, U, nU, rU, E);
  return w;
}

__global__ void __launch_bounds__(256) compress_kernel(const FillDesc* __restrict__ fills,
                                                       const PivotWork* __restrict__ work, CompressParams P) {
  __shared__ CtaShared sh;
  const PivotWork Wk = work[blockIdx.x];
  const int MX = Wk.MX, K = Wk.K;
  double* s = Wk.scratch;
  double* Uc = s; s += (size_t)MX * K;
  double* Vc = s; s += (size_t)MX * K;
  double* left = s; s += (size_t)MX * K;
  double* right = s; s += (size_t)MX * K;
  double* H = s; s += (size_t)MX * K;
  double* E1 = s; s += (size_t)MX * K;
  double* E2 = s; s += (size_t)MX * K;
  double* Rl = s; s += (size_t)K * K;
  double* Rr = s; s += (size_t)K * K;
  double* core = s; s += (size_t)K * K;
  double* Jv = s; s += (size_t)K * K;
  double* rr = s; s += MX;
  double* cc = s; s += MX;
  double* sig = s; s += MX + K;
  double* sig2 = s; s += MX + K;
  double* dots = s; s += K;
  double* vv = s; s += K;
  int* usedr = reinterpret_cast<int*>(s); s += MX;
  int* usedc = reinterpret_cast<int*>(s); s += MX;
  int* ord = reinterpret_cast<int*>(s); s += MX + K;
  int* ord2 = reinterpret_cast<int*>(s); s += MX + K;
  const double tol = P.tol;
  for (int f = Wk.f0; f < Wk.f1; f++) {
    const FillDesc D = fills[f];
    const int rows = D.kind == FILL_HYBRID ? P.rank[D.p] : D.n_p;
    const int cols = D.n_q;
    if (rows == 0 || cols == 0) {
      if (threadIdx.x == 0) {
        P.status[f] = 0;
        atomicAdd(&P.stats[0], 1);
      }
      __syncthreads();
      continue;
    }
    if (tol == 0.0) {
      // exact mode: bases are identities, the redirected fill is F itself
      double mx = 0.0;
      for (int e = threadIdx.x; e < rows * cols; e += blockDim.x) {
        const int a = e % rows, b = e / rows;
        mx = fmax(mx, fabs(Fat(D.F, D.ldF, D.transF, a, b)));
      }
      mx = block_sum(mx > 0.0 ? 1.0 : 0.0, sh.red);
      for (int e = threadIdx.x; e < rows * cols; e += blockDim.x) {
        const int a = e % rows, b = e / rows;
        const double v = Fat(D.F, D.ldF, D.transF, a, b);
        if (D.transM) D.M[b + (size_t)a * D.ldM] += v;
        else D.M[a + (size_t)b * D.ldM] += v;
      }
      __syncthreads();
      fill_zero(D, rows, cols);
      if (threadIdx.x == 0) {
        P.status[f] = 0;
        atomicAdd(&P.stats[0], 1);
        atomicMax(&P.stats[2], mx > 0.0 ? min(rows, cols) : 0);
      }
      __syncthreads();
      continue;
    }
    const int mrow = rows < P.probe_maxm ? rows : P.probe_maxm;
    const int* probes = P.probes + (size_t)mrow * 10;
    const int nprobe = min(10, rows);
    AcaOut ao = cta_aca(D.F, D.ldF, D.transF, rows, cols, tol, probes, nprobe, Uc, Vc, K, rr, cc, usedr, usedc, dots,
                        sh);
    const int k = ao.k;
    const int full = min(rows, cols);
    if (!ao.converged && (k >= full || k >= K)) {
      if (threadIdx.x == 0) {
        P.status[f] = 1;
        atomicAdd(&P.stats[1], 1);
      }
      __syncthreads();
      continue;
    }
    int r = 0;
    if (k > 0) {
      // recompression: QR of both factors, SVD of the core (ifmm/lowrank.py:164-171)
      cta_qr(Uc, rows, k, rows, Rl, left, rows, vv, sh);   // left <- Ql (rows x k)
      cta_qr(Vc, cols, k, cols, Rr, right, cols, vv, sh);  // right <- Qr (cols x k)
      cta_gemm(k, k, k, 1.0, Rl, k, false, Rr, k, true, 0.0, core, k);
      cta_jacobi(core, k, k, k, Jv, k, sig, ord, sh);
      r = trunc_rank_dev(sig, ord, k, tol);
      // Uc <- Ql * core(:, ord[:r]) ; Vc <- Qr * Jv(:, ord[:r])
      for (int e = threadIdx.x; e < rows * r; e += blockDim.x) {
        const int i = e % rows, c = e / rows;
        const int col = ord[c];
        double acc = 0.0;
        for (int t = 0; t < k; t++) acc = fma(left[i + (size_t)t * rows], core[t + (size_t)col * k], acc);
        Uc[i + (size_t)c * rows] = acc;
      }
      for (int e = threadIdx.x; e < cols * r; e += blockDim.x) {
        const int i = e % cols, c = e / cols;
        const int col = ord[c];
        double acc = 0.0;
        for (int t = 0; t < k; t++) acc = fma(right[i + (size_t)t * cols], Jv[t + (size_t)col * k], acc);
        Vc[i + (size_t)c * cols] = acc;
      }
      for (int c = threadIdx.x; c < r; c += blockDim.x) dots[c] = sig[ord[c]];
      __syncthreads();
    }
    // A = Uc (rows x r), B = Vc (cols x r, orthonormal), dots = singular values
    double fro = 0.0;
    for (int e = threadIdx.x; e < rows * r; e += blockDim.x) fro += Uc[e] * Uc[e];
    fro = sqrt(block_sum(fro, sh.red));
    const double cutoff = tol * fro;
    if (threadIdx.x == 0) {
      P.status[f] = (k << 8) | (r << 20);  // low byte 0: compressed; ranks kept for diagnostics
      atomicAdd(&P.stats[0], 1);
      atomicMax(&P.stats[2], r);
    }
    if (r > 0) {
      // q side: directions of B weighted by A
      int rq = P.rank[D.q];
      for (int e = threadIdx.x; e < cols * r; e += blockDim.x) H[e] = Vc[e];
      __syncthreads();
      int wq = new_dirs_append(H, cols, r, D.Uq, rq, dots, cutoff, E1, sig2, ord2, sh);
      rq += wq;
      __syncthreads();
      if (threadIdx.x == 0) P.rank[D.q] = rq;
      int rp = D.kind == FILL_HYBRID ? rows : P.rank[D.p];
      if (D.kind == FILL_P2P) {
        for (int e = threadIdx.x; e < rows * r; e += blockDim.x) H[e] = Uc[e];
        __syncthreads();
        int wp = new_dirs_append(H, rows, r, D.Up, rp, nullptr, cutoff, E1, sig2, ord2, sh);
        rp += wp;
        __syncthreads();
        if (threadIdx.x == 0) P.rank[D.p] = rp;
        if (P.debug && threadIdx.x == 0) printf("aug p=%d +%d -> %d\n", D.p, wp, rp);
      }
      if (P.debug && threadIdx.x == 0)
        printf("augq fill=%d kind=%d p=%d q=%d r=%d +%d -> %d fro=%.6e\n", f, D.kind, D.p, D.q, r, wq, rq, fro);
      __syncthreads();
      // E2 = Uq^T B (rq x r)
      cta_gemm(rq, r, cols, 1.0, D.Uq, cols, true, Vc, cols, false, 0.0, E2, rq);
      if (D.kind == FILL_HYBRID) {
        // delta = A E2^T (rows x rq)
        m2l_add_product(D, Uc, rows, E2, rq, rows, rq, r);
      } else {
        // delta = (Up^T A)(Uq^T B)^T  (rp x rq)
        cta_gemm(rp, r, rows, 1.0, D.Up, rows, true, Uc, rows, false, 0.0, H, rp);
        m2l_add_product(D, H, rp, E2, rq, rp, rq, r);
      }
      __syncthreads();
    }
    fill_zero(D, rows, cols);
    __syncthreads();
  }
}

// ------------------------------------------------------------------ work level
struct WorkLevel {
  int k = 0, nc = 0, win = 0;
  const Topo* T = nullptr;
  std::vector<int> n, r, rcap, r0;
  std::vector<double*> U;
  std::vector<double*> p2p, m2l, xy;  // nc*win
  std::vector<uint8_t> pp, pm, px;
  std::vector<uint8_t> dead;
  int* d_rank = nullptr;
  Arena* arena = nullptr;  // zero-initialised blocks
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
  void collect(FactorH* F) {  // call after a stream synchronisation
    if (!on) return;
    end();
    for (Span& sp : spans) {
      float ms = 0.f;
      CK(cudaEventSynchronize(sp.b));
      CK(cudaEventElapsedTime(&ms, sp.a, sp.b));
      F->phase_ms[sp.ph] += ms;
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
  Factorizer(StoreH* S, double tol, int flags, double cond_limit)
      : S_(S), t_(S->tree), tol_(tol), flags_(flags), cond_limit_(cond_limit) {}
  FactorH* run();

 private:
  StoreH* S_;
  TreeH* t_;
  double tol_;
  int flags_;
  double cond_limit_;  // PIVOT_CONDITION_LIMIT (ifmm/solver.py:50), 1e12 by default
  cudaStream_t s_ = nullptr;
  std::unique_ptr<FactorH> F_;
  Arena ws_{size_t(256) << 20};
  Staging st_;
  PhaseTimer tm_;
  Arena lvl_arena_[2] = {Arena(size_t(512) << 20), Arena(size_t(512) << 20)};
  WorkLevel cur_, prev_;
  // per-record host metadata for pos resolution at level end
  struct SlotRef { int kind, j, dim; };  // kind 0: x_j, 1: y_j
  std::vector<std::vector<SlotRef>> rec_slots_;

  // level arenas hand out zeroed memory (slabs are cleared on creation/reset)
  double* zalloc(WorkLevel& W, size_t n) { return W.arena->alloc_n<double>(std::max<size_t>(1, n)); }
  BlkRef p2p_ref(WorkLevel& W, int i, int j, bool alloc) {
    int a = std::min(i, j), b = std::max(i, j);
    int sl = W.T->slot(a, b);
    if (sl < 0) invalid("near-field block beyond the 7x7 window (dense fill too far)");
    double*& p = W.p2p[size_t(a) * W.win + sl];
    if (!p && alloc) p = zalloc(W, size_t(W.n[a]) * W.n[b]);
    return {p, W.n[a], i > j};
  }
  BlkRef m2l_ref(WorkLevel& W, int i, int j, bool alloc) {
    int a = std::min(i, j), b = std::max(i, j);
    int sl = W.T->slot(a, b);
    if (sl < 0) invalid("M2L block beyond the 7x7 window");
    double*& p = W.m2l[size_t(a) * W.win + sl];
    if (!p && alloc) p = zalloc(W, size_t(W.rcap[a]) * W.rcap[b]);
    return {p, W.rcap[a], i > j};
  }
  BlkRef xy_ref(WorkLevel& W, int i, int j, bool alloc) {
    int sl = W.T->slot(i, j);
    if (sl < 0) invalid("hybrid block beyond the 7x7 window");
    double*& p = W.xy[size_t(i) * W.win + sl];
    if (!p && alloc) p = zalloc(W, size_t(W.n[i]) * W.rcap[j]);
    return {p, W.n[i], false};
  }
  uint8_t& pres(std::vector<uint8_t>& v, WorkLevel& W, int i, int j) {
    return v[size_t(i) * W.win + W.T->slot(i, j)];
  }
  bool pp_present(WorkLevel& W, int i, int j) { int a = std::min(i, j), b = std::max(i, j); return pres(W.pp, W, a, b); }
  void set_pp(WorkLevel& W, int i, int j, uint8_t v) { int a = std::min(i, j), b = std::max(i, j); pres(W.pp, W, a, b) = v; }
  void set_pm(WorkLevel& W, int i, int j, uint8_t v) { int a = std::min(i, j), b = std::max(i, j); pres(W.pm, W, a, b) = v; }
  bool pm_present(WorkLevel& W, int i, int j) { int a = std::min(i, j), b = std::max(i, j); return pres(W.pm, W, a, b); }

  void init_level_alloc(WorkLevel& W, int k) {
    W.k = k;
    W.T = &t_->lv[k];
    W.nc = W.T->nc;
    W.win = W.T->win();
    W.arena = &lvl_arena_[k & 1];
    W.arena->set_zero_stream(s_);
    W.arena->reset();
    W.p2p.assign(size_t(W.nc) * W.win, nullptr);
    W.m2l.assign(size_t(W.nc) * W.win, nullptr);
    W.xy.assign(size_t(W.nc) * W.win, nullptr);
    W.pp.assign(size_t(W.nc) * W.win, 0);
    W.pm.assign(size_t(W.nc) * W.win, 0);
    W.px.assign(size_t(W.nc) * W.win, 0);
    W.dead.assign(W.nc, 0);
    W.U.assign(W.nc, nullptr);
    W.d_rank = W.arena->alloc_n<int>(W.nc);
  }
  void start_leaf_level();
  void start_parent_level(WorkLevel& C, int k);
  void eliminate_batch(std::vector<int>& piv, int colour);
  void finish_level(int rec_begin);
  void factor_top();
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
  for (int i = 0; i < W.nc; i++) {
    W.U[i] = zalloc(W, size_t(W.n[i]) * W.rcap[i]);
    cb.add(L.U[i], W.n[i], W.U[i], W.n[i], W.n[i], W.r0[i]);
  }
  const Topo& T = *W.T;
  for (int i = 0; i < W.nc; i++) {
    for (int q = T.nbr_off[i]; q < T.nbr_off[i + 1]; q++) {
      int j = T.nbr[q];
      if (j < i) continue;
      BlkRef b = p2p_ref(W, i, j, true);
      cb.add(S_->leaf_p2p[size_t(i) * W.win + T.slot(i, j)], W.n[i], b.p, b.ld, W.n[i], W.n[j]);
      set_pp(W, i, j, 1);
    }
    for (int q = T.il_off[i]; q < T.il_off[i + 1]; q++) {
      int j = T.il[q];
      if (j < i) continue;
      BlkRef b = m2l_ref(W, i, j, true);
      cb.add(L.m2l[q], std::max(1, W.r0[i]), b.p, b.ld, W.r0[i], W.r0[j]);
      set_pm(W, i, j, 1);
    }
  }
  CK(cudaMemcpyAsync(W.d_rank, W.r.data(), sizeof(int) * W.nc, cudaMemcpyHostToDevice, s_));
  launch_copies(cb, ws_, st_, s_);
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
  for (int i = 0; i < W.nc; i++) {
    W.U[i] = zalloc(W, size_t(W.n[i]) * W.rcap[i]);
    const int n0 = int(L.child_off[size_t(i) * (nch + 1) + nch]);
    for (int c = 0; c < nch; c++) {
      const int ch = (i << dim) + c;
      const int64_t ro = L.child_off[size_t(i) * (nch + 1) + c];
      cb.add(L.U[i] + ro, std::max(1, n0), W.U[i] + off[i][c], W.n[i], S_->lv[k + 1].r0[ch], W.r0[i]);
    }
  }
  const Topo& T = *W.T;
  for (int i = 0; i < W.nc; i++) {
    for (int q = T.nbr_off[i]; q < T.nbr_off[i + 1]; q++) {
      int j = T.nbr[q];
      if (j < i) continue;
      bool any = false;
      for (int a = 0; a < nch; a++)
        for (int b = 0; b < nch; b++) any |= pm_present(C, (i << dim) + a, (j << dim) + b);
      if (!any) continue;
      BlkRef P = p2p_ref(W, i, j, true);
      for (int a = 0; a < nch; a++)
        for (int b = 0; b < nch; b++) {
          const int ca = (i << dim) + a, cbb = (j << dim) + b;
          if (!pm_present(C, ca, cbb)) continue;
          BlkRef M = m2l_ref(C, ca, cbb, false);
          if (!M.p) continue;
          cb.add(M.p, M.ld, P.p + off[i][a] + size_t(off[j][b]) * P.ld, P.ld, C.r[ca], C.r[cbb], M.trans);
        }
      set_pp(W, i, j, 1);
    }
    for (int q = T.il_off[i]; q < T.il_off[i + 1]; q++) {
      int j = T.il[q];
      if (j < i) continue;
      BlkRef b = m2l_ref(W, i, j, true);
      cb.add(L.m2l[q], std::max(1, W.r0[i]), b.p, b.ld, W.r0[i], W.r0[j]);
      set_pm(W, i, j, 1);
    }
  }
  CK(cudaMemcpyAsync(W.d_rank, W.r.data(), sizeof(int) * W.nc, cudaMemcpyHostToDevice, s_));
  launch_copies(cb, ws_, st_, s_);
}

void Factorizer::eliminate_batch(std::vector<int>& piv, int colour) {
  WorkLevel& W = cur_;
  const Topo& T = *W.T;
  const int k = W.k;
  const int np = int(piv.size());
  CK(cudaStreamSynchronize(s_));  // staging buffers of earlier uploads are free after this
  ws_.reset();
  st_.reset();
  struct PivInfo {
    int i, n, r, m, w;
    std::vector<int> xp, yp;
    std::vector<int> soff;  // slot column offsets (size nslots+1)
    double *S, *C, *Xb;
    int rec;
  };
  std::vector<PivInfo> P(np);
  CopyBatch cb;
  std::vector<MatDesc> md(np);
  for (int t = 0; t < np; t++) {
    PivInfo& I = P[t];
    const int i = piv[t];
    I.i = i;
    I.n = W.n[i];
    I.r = W.r[i];
    I.m = I.n + I.r;
    // partners: scan the 7x7 window of i
    std::vector<int> cand;
    {
      // enumerate window members of i
      const int dim = T.dim;
      int lo[3], hi[3];
      for (int d = 0; d < dim; d++) {
        lo[d] = std::max(0, T.grid[i * dim + d] - 3);
        hi[d] = std::min((1 << k) - 1, T.grid[i * dim + d] + 3);
      }
      int g[3];
      for (g[0] = lo[0]; g[0] <= hi[0]; g[0]++)
        for (g[1] = (dim > 1 ? lo[1] : 0); g[1] <= (dim > 1 ? hi[1] : 0); g[1]++)
          for (g[2] = (dim > 2 ? lo[2] : 0); g[2] <= (dim > 2 ? hi[2] : 0); g[2]++) {
            int64_t c = 0;
            for (int b = 0; b < k; b++)
              for (int ax = 0; ax < dim; ax++) c |= int64_t((g[ax] >> b) & 1) << (b * dim + ax);
            cand.push_back(int(c));
          }
      std::sort(cand.begin(), cand.end());
    }
    for (int j : cand) {
      if (j == i) continue;
      if (!W.dead[j] && pp_present(W, i, j)) I.xp.push_back(j);
      if (pres(W.px, W, i, j)) I.yp.push_back(j);
    }
    I.soff.assign(1, 0);
    for (int j : I.xp) I.soff.push_back(I.soff.back() + W.n[j]);
    for (int j : I.yp) I.soff.push_back(I.soff.back() + W.r[j]);
    I.soff.push_back(I.soff.back() + I.r);
    I.w = I.soff.back();
    I.S = ws_.alloc_n<double>(size_t(I.m) * I.m);
    I.C = ws_.alloc_n<double>(size_t(std::max(1, I.n)) * I.w);
    I.Xb = ws_.alloc_n<double>(size_t(std::max(1, I.r)) * I.w);
    int* ipiv = ws_.alloc_n<int>(I.m);
    md[t] = MatDesc{I.S, I.m, I.m, ipiv, i};
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
  }
  tm_.begin(PH_GATHER);
  launch_copies(cb, ws_, st_, s_);
  static const char* dump_dir = getenv("IFMM_DUMP_SINGULAR");
  std::vector<double*> Sbak;
  if (dump_dir)
    for (int t = 0; t < np; t++) {
      Sbak.push_back(ws_.alloc_n<double>(size_t(P[t].m) * P[t].m));
      CK(cudaMemcpyAsync(Sbak.back(), P[t].S, sizeof(double) * P[t].m * P[t].m, cudaMemcpyDeviceToDevice, s_));
    }
  const MatDesc* dmd = upload(ws_, md, s_, st_);
  double* d_nS = ws_.alloc_n<double>(np);
  double* d_nSi = ws_.alloc_n<double>(np);
  int* d_info = ws_.alloc_n<int>(np);
  tm_.begin(PH_GJ);
  launch_norm1(dmd, np, d_nS, s_);
  batched_gj_inverse(md, dmd, d_info, ws_, st_, s_);
  {
    int maxm = 0;
    for (auto& d : md) maxm = std::max(maxm, d.m);
    launch_norm1_estimate(dmd, np, maxm, d_nSi, s_);
  }
  // records + X = S^-1 C
  GemmBatch gb;
  for (int t = 0; t < np; t++) {
    PivInfo& I = P[t];
    RecordH R{};
    R.level = k;
    R.index = I.i;
    R.n = I.n;
    R.r = I.r;
    R.w = I.w;
    R.sinv = F_->arena.alloc_n<double>(size_t(std::max(1, I.n)) * std::max(1, I.n));
    R.xtop = F_->arena.alloc_n<double>(size_t(std::max(1, I.n)) * I.w);
    R.pos = F_->arena.alloc_n<int>(I.w);
    I.rec = int(F_->recs.size());
    F_->recs.push_back(R);
    std::vector<SlotRef> sl;
    for (int j : I.xp) sl.push_back({0, j, W.n[j]});
    for (int j : I.yp) sl.push_back({1, j, W.r[j]});
    sl.push_back({1, I.i, I.r});
    rec_slots_.push_back(sl);
    const int wl = I.w - I.r;
    {
      const double m = I.m, n = I.n, w = I.w, h = wl;
      F_->fl_exec += 2.0 * m * m * m + 2.0 * m * n * h;
      F_->fl_ref += 2.0 / 3.0 * m * m * m + 2.0 * m * m * w + 2.0 * h * n * w;
      F_->solve_bytes += 8.0 * (n * n + 2.0 * n * w);
    }
    cb.add(I.S, I.m, R.sinv, I.n, I.n, I.n);
    cb.add(I.S + size_t(I.n) * I.m, I.m, R.xtop + size_t(wl) * I.n, I.n, I.n, I.r, false, -1.0);
    cb.add(I.S + I.n + size_t(I.n) * I.m, I.m, I.Xb + size_t(wl) * I.r, I.r, I.r, I.r, false, -1.0);
    gb.add(I.S, I.m, I.C, I.n, R.xtop, I.n, I.n, wl, I.n, 1.0, 0.0);
    gb.add(I.S + I.n, I.m, I.C, I.n, I.Xb, I.r, I.r, wl, I.n, 1.0, 0.0);
  }
  tm_.begin(PH_GATHER);
  launch_copies(cb, ws_, st_, s_);
  tm_.begin(PH_XGEMM);
  launch_grouped_gemm(gb, false, false, ws_, st_, s_);
  tm_.end();
  // symmetric Schur update on the block upper triangle: target -= C_a^T X_b
  for (int t = 0; t < np; t++) {
    PivInfo& I = P[t];
    const RecordH& R = F_->recs[I.rec];
    const int nx = int(I.xp.size()), ny = int(I.yp.size());
    const int ns = nx + ny + 1;
    auto slot_cluster = [&](int s) { return s < nx ? I.xp[s] : (s < nx + ny ? I.yp[s - nx] : I.i); };
    for (int a = 0; a < ns; a++)
      for (int b = a; b < ns; b++) {
        const bool ax = a < nx, bx = b < nx;
        const int ja = slot_cluster(a), jb = slot_cluster(b);
        const int da = I.soff[a + 1] - I.soff[a], db = I.soff[b + 1] - I.soff[b];
        if (a == ns - 1 && b == ns - 1) {
          BlkRef M = m2l_ref(W, I.i, I.i, true);
          cb.add(I.Xb + size_t(I.soff[b]) * I.r, I.r, M.p, M.ld, I.r, I.r, false, 1.0, true);
          pres(W.pm, W, I.i, I.i) = 1;
          continue;
        }
        BlkRef tgt;
        if (ax && bx) {
          tgt = p2p_ref(W, ja, jb, true);
          set_pp(W, ja, jb, 1);
        } else if (ax && !bx) {
          tgt = xy_ref(W, ja, jb, true);
          pres(W.px, W, ja, jb) = 1;
        } else {
          tgt = m2l_ref(W, ja, jb, true);
          set_pm(W, ja, jb, 1);
        }
        if (da == 0 || db == 0) continue;
        F_->fl_schur += 2.0 * I.n * da * db;
        gb.add(I.C + size_t(I.soff[a]) * I.n, I.n, R.xtop + size_t(I.soff[b]) * I.n, I.n, tgt.p, tgt.ld, da, db, I.n,
               -1.0, 1.0, tgt.trans);
      }
  }
  tm_.begin(PH_SCHUR);
  launch_grouped_gemm(gb, true, false, ws_, st_, s_);
  tm_.begin(PH_GATHER);
  launch_copies(cb, ws_, st_, s_);
  tm_.end();
  // fill-in compression lists (reference order: hybrid pairs sorted, then P2P pairs sorted)
  std::vector<FillDesc> fd;
  std::vector<PivotWork> pw(np);
  struct FillHost { int kind, p, q; };
  std::vector<FillHost> fh;
  for (int t = 0; t < np; t++) {
    PivInfo& I = P[t];
    pw[t].f0 = int(fd.size());
    std::vector<int> ps(I.yp);
    ps.push_back(I.i);
    std::sort(ps.begin(), ps.end());
    int MX = 1, K = 1;
    for (int p : ps)
      for (int q : I.xp) {
        if (!T.in_il(p, q)) continue;
        BlkRef F = xy_ref(W, q, p, false);
        BlkRef M = m2l_ref(W, p, q, true);
        FillDesc D{FILL_HYBRID, p, q, F.p, W.n[q], 1, W.n[p], W.n[q], W.U[p], W.U[q], M.p, M.ld, M.trans ? 1 : 0};
        fd.push_back(D);
        fh.push_back({FILL_HYBRID, p, q});
        MX = std::max(MX, std::max(W.n[p], W.n[q]));
        K = std::max(K, std::min(W.n[p], W.n[q]));
      }
    for (size_t a = 0; a < I.xp.size(); a++)
      for (size_t b = a + 1; b < I.xp.size(); b++) {
        int p = I.xp[a], q = I.xp[b];
        if (!T.in_il(p, q)) continue;
        BlkRef F = p2p_ref(W, p, q, false);
        BlkRef M = m2l_ref(W, p, q, true);
        FillDesc D{FILL_P2P, p, q, F.p, F.ld, 0, W.n[p], W.n[q], W.U[p], W.U[q], M.p, M.ld, M.trans ? 1 : 0};
        fd.push_back(D);
        fh.push_back({FILL_P2P, p, q});
        MX = std::max(MX, std::max(W.n[p], W.n[q]));
        K = std::max(K, std::min(W.n[p], W.n[q]));
      }
    pw[t].f1 = int(fd.size());
    K = std::min(K, 96);
    pw[t].MX = MX;
    pw[t].K = K;
    const size_t per = 7 * size_t(MX) * K + 4 * size_t(K) * K + 2 * MX + 2 * (MX + K) + 2 * K + 4 * (MX + K) + 64;
    pw[t].scratch = pw[t].f1 > pw[t].f0 ? ws_.alloc_n<double>(per) : nullptr;
  }
  int* d_status = ws_.alloc_n<int>(std::max<size_t>(1, fd.size()));
  int* d_stats = ws_.alloc_n<int>(4);
  CK(cudaMemsetAsync(d_stats, 0, 16, s_));
  if (!fd.empty()) {
    tm_.begin(PH_COMPRESS);
    const FillDesc* dfd = upload(ws_, fd, s_, st_);
    const PivotWork* dpw = upload(ws_, pw, s_, st_);
    CompressParams cp{tol_, S_->d_probe, S_->probe_maxm, W.d_rank, d_status, d_stats,
                      getenv("IFMM_DEBUG") != nullptr ? 1 : 0};
    compress_kernel<<<np, 256, 0, s_>>>(dfd, dpw, cp);
    CK_LAUNCH();
  }
  tm_.end();
  // read back: pivot conditioning, ranks, fill outcomes, counters
  std::vector<double> nS(np), nSi(np);
  std::vector<int> info(np), status(fd.size()), stats(4);
  CK(cudaMemcpyAsync(nS.data(), d_nS, sizeof(double) * np, cudaMemcpyDeviceToHost, s_));
  CK(cudaMemcpyAsync(nSi.data(), d_nSi, sizeof(double) * np, cudaMemcpyDeviceToHost, s_));
  CK(cudaMemcpyAsync(info.data(), d_info, sizeof(int) * np, cudaMemcpyDeviceToHost, s_));
  if (!fd.empty()) CK(cudaMemcpyAsync(status.data(), d_status, sizeof(int) * fd.size(), cudaMemcpyDeviceToHost, s_));
  CK(cudaMemcpyAsync(stats.data(), d_stats, 16, cudaMemcpyDeviceToHost, s_));
  CK(cudaMemcpyAsync(W.r.data(), W.d_rank, sizeof(int) * W.nc, cudaMemcpyDeviceToHost, s_));
  CK(cudaStreamSynchronize(s_));
  tm_.collect(F_.get());
  for (int t = 0; t < np; t++) {
    double rc = (info[t] != 0) ? 0.0 : 1.0 / (nS[t] * nSi[t]);
    if (!std::isfinite(rc) || rc <= 1.0 / cond_limit_) {
      double cond = 1.0 / std::max(rc, 1e-300);
      if (dump_dir) {
        std::vector<double> h(size_t(P[t].m) * P[t].m);
        CK(cudaMemcpy(h.data(), Sbak[t], sizeof(double) * h.size(), cudaMemcpyDeviceToHost));
        std::string fn = std::string(dump_dir) + "/S_" + std::to_string(k) + "_" + std::to_string(P[t].i) + ".bin";
        FILE* fp = fopen(fn.c_str(), "wb");
        if (fp) {
          int hdr[2] = {P[t].n, P[t].r};
          fwrite(hdr, sizeof hdr, 1, fp);
          fwrite(h.data(), sizeof(double), h.size(), fp);
          fclose(fp);
        }
      }
      char buf[256];
      snprintf(buf, sizeof buf, "pivot for cluster %d at level %d is numerically singular (condition estimate %.2e)",
               P[t].i, k, cond);
      throw SingularPivot(k, P[t].i, cond, buf);
    }
  }
  LevelStatsH& LS = F_->stats[k];
  LS.compressed += stats[0];
  LS.dense_kept += stats[1];
  LS.max_rank = std::max(LS.max_rank, stats[2]);
  static const bool dbg = getenv("IFMM_DEBUG") != nullptr;
  for (size_t f = 0; f < fh.size(); f++) {
    if (dbg)
      fprintf(stderr, "fill k=%d kind=%d p=%d q=%d status=%d aca=%d rank=%d rank_p=%d\n", k, fh[f].kind, fh[f].p,
              fh[f].q, status[f] & 0xff, (status[f] >> 8) & 0xfff, status[f] >> 20, W.r[fh[f].p]);
    if ((status[f] & 0xff) != 0) continue;
    const FillHost& h = fh[f];
    if (h.kind == FILL_HYBRID) pres(W.px, W, h.q, h.p) = 0;
    else set_pp(W, h.p, h.q, 0);
  }
  for (int t = 0; t < np; t++) W.dead[P[t].i] = 1;
  (void)colour;
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
  std::vector<int> posall;
  std::vector<int64_t> posoff;
  for (size_t rr = rec_begin; rr < F_->recs.size(); rr++) {
    RecordH& R = F_->recs[rr];
    R.xoff = xb + xoff[R.index];
    posoff.push_back(int64_t(posall.size()));
    for (const SlotRef& sr : rec_slots_[rr]) {
      int64_t base = sr.kind == 0 ? xb + xoff[sr.j] : yb + yoff[sr.j];
      for (int u = 0; u < sr.dim; u++) posall.push_back(int(base + u));
    }
  }
  if (!posall.empty()) {
    void* h = st_.get(sizeof(int) * posall.size());
    memcpy(h, posall.data(), sizeof(int) * posall.size());
    // records' pos arrays are separate allocations: copy each
    for (size_t rr = rec_begin, u = 0; rr < F_->recs.size(); rr++, u++) {
      RecordH& R = F_->recs[rr];
      CK(cudaMemcpyAsync(R.pos, static_cast<int*>(h) + posoff[u], sizeof(int) * R.w, cudaMemcpyHostToDevice, s_));
    }
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
  ws_.reset();
  st_.reset();
  F_->top_inv = F_->arena.alloc_n<double>(size_t(std::max(1, M)) * std::max(1, M));
  CK(cudaMemsetAsync(F_->top_inv, 0, sizeof(double) * std::max(1, M) * std::max(1, M), s_));
  CopyBatch cb;
  for (int i = 0; i < W.nc; i++)
    for (int j = 0; j < W.nc; j++) {
      if (W.T->slot(i, j) < 0 && W.T->slot(j, i) < 0) continue;
      if (W.T->slot(std::min(i, j), std::max(i, j)) < 0) continue;
      if (!pm_present(W, i, j)) continue;
      BlkRef b = m2l_ref(W, i, j, false);
      if (!b.p) continue;
      cb.add(b.p, b.ld, F_->top_inv + off[i] + size_t(off[j]) * M, M, W.r[i], W.r[j], b.trans);
    }
  launch_copies(cb, ws_, st_, s_);
  F_->fl_exec += 2.0 * double(M) * M * M;
  F_->fl_ref += 2.0 / 3.0 * double(M) * M * M;
  F_->solve_bytes += 8.0 * double(M) * M;
  if (M > 0) {
    std::vector<MatDesc> md(1);
    md[0] = MatDesc{F_->top_inv, M, M, ws_.alloc_n<int>(M), -1};
    const MatDesc* dmd = upload(ws_, md, s_, st_);
    int* d_info = ws_.alloc_n<int>(1);
    tm_.begin(PH_TOP);
    batched_gj_inverse(md, dmd, d_info, ws_, st_, s_);
  }
  CK(cudaStreamSynchronize(s_));
  tm_.collect(F_.get());
}

FactorH* Factorizer::run() {
  auto t0 = std::chrono::steady_clock::now();
  s_ = S_->stream;
  tm_.on = (flags_ & IFMM_FLAG_TIMING) != 0;
  tm_.s = s_;
  F_.reset(new FactorH);
  F_->store = S_;
  F_->tree = t_;
  F_->tol = tol_;
  F_->stream = s_;
  const int K = t_->depth;
  F_->stats.assign(K + 1, LevelStatsH{});
  F_->lvl_base.assign(K + 1, 0);
  F_->lvl_base[K] = 0;
  F_->r_m = S_->max_init_rank;
  const int ncol = [&] { int c = 1; for (int d = 0; d < t_->dim; d++) c *= 3; return c; }();
  for (int k = K; k >= 2; k--) {
    if (k == K) {
      tm_.begin(PH_TRANSITION);
      start_leaf_level();
    } else {
      prev_ = std::move(cur_);
      cur_ = WorkLevel{};
      tm_.begin(PH_TRANSITION);
      start_parent_level(prev_, k);
      CK(cudaStreamSynchronize(s_));
      tm_.collect(F_.get());
      prev_ = WorkLevel{};
    }
    F_->stats[k].clusters = cur_.nc;
    const int rec_begin = int(F_->recs.size());
    for (int c = 0; c < ncol; c++) {
      std::vector<int> piv;
      for (int i = 0; i < cur_.nc; i++)
        if (cur_.T->colour[i] == c) piv.push_back(i);
      if (piv.empty()) continue;
      const int r0 = int(F_->recs.size());
      eliminate_batch(piv, c);
      F_->batches.push_back(BatchH{k, c, r0, int(F_->recs.size()), nullptr, 0, 0});
    }
    finish_level(rec_begin);
    F_->r_m = std::max(F_->r_m, F_->stats[k].max_rank);
  }
  factor_top();
  // device copies of the batch record tables
  for (BatchH& b : F_->batches) {
    std::vector<RecordH> v(F_->recs.begin() + b.rec0, F_->recs.begin() + b.rec1);
    RecordH* d = F_->arena.alloc_n<RecordH>(v.size());
    CK(cudaMemcpyAsync(d, v.data(), sizeof(RecordH) * v.size(), cudaMemcpyHostToDevice, s_));
    b.d_recs = d;
    for (auto& r : v) {
      b.maxn = std::max(b.maxn, r.n);
      b.maxw = std::max(b.maxw, r.w);
    }
  }
  F_->g_off.resize(F_->recs.size() + 1, 0);
  for (size_t r = 0; r < F_->recs.size(); r++) F_->g_off[r + 1] = F_->g_off[r] + F_->recs[r].n;
  F_->g_size = F_->g_off.back();
  F_->d_g_off = F_->arena.alloc_n<int64_t>(F_->g_off.size());
  CK(cudaMemcpyAsync(F_->d_g_off, F_->g_off.data(), sizeof(int64_t) * F_->g_off.size(), cudaMemcpyHostToDevice, s_));
  CK(cudaStreamSynchronize(s_));
  cur_ = WorkLevel{};
  lvl_arena_[0].release();
  lvl_arena_[1].release();
  F_->fl_exec += F_->fl_schur;
  F_->ms_total = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return F_.release();
}

FactorH* factorize(StoreH* S, double tol, int flags, double cond_limit) {
  ensure_device();
  Factorizer f(S, tol < 0 ? S->tol : tol, flags, cond_limit > 0 ? cond_limit : 1e12);
  return f.run();
}

}  // namespace ifmm
