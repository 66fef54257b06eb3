// Host-side handles of the B200 IFMM: tree, initial operator store,
// factorization.  Device memory is owned by per-handle arenas.
#pragma once
#include <algorithm>
#include <array>
#include <memory>
#include <mutex>

#include "batched.cuh"
#include "common.cuh"
#include "kfun.cuh"

namespace ifmm {

constexpr int WIN1 = 7;  // relative grid offsets -3..3 per axis cover nbr + IL + fills

struct Topo {
  int k = 0, nc = 0, dim = 2;
  std::vector<int> grid;             // nc*dim
  std::vector<int> nbr_off, nbr;     // CSR, sorted, self included (ifmm/geometry.py:229-244)
  std::vector<int> il_off, il;       // CSR, sorted (ifmm/geometry.py:245-262)
  std::vector<int> colour;           // sum_d (g_d mod 3) 3^d
  int win() const { int w = 1; for (int d = 0; d < dim; d++) w *= WIN1; return w; }
  // window slot of j relative to i, or -1 if farther than 3 cells on an axis
  int slot(int i, int j) const {
    int s = 0, mul = 1;
    for (int d = 0; d < dim; d++) {
      int dd = grid[j * dim + d] - grid[i * dim + d];
      if (dd < -3 || dd > 3) return -1;
      s += (dd + 3) * mul;
      mul *= WIN1;
    }
    return s;
  }
  // per cluster: bit s set iff the window slot s holds an interaction-list
  // member (built by prepare(), so in_il is a bit test instead of a scan)
  std::vector<uint64_t> il_mask;
  // per cluster: the clusters of its 7^dim window, sorted (CSR)
  std::vector<int> wc_off, wc;
  void prepare() {
    if (!wc_off.empty() || nc == 0) return;
    if (win() <= 64) il_mask.assign(nc, 0);  // 3-D windows (343 slots) keep the scan
    for (int i = 0; i < nc && !il_mask.empty(); i++)
      for (int t = il_off[i]; t < il_off[i + 1]; t++) {
        const int sl = slot(i, il[t]);
        if (sl >= 0) il_mask[i] |= uint64_t(1) << sl;
      }
    wc_off.assign(nc + 1, 0);
    wc.clear();
    std::vector<int> cand;
    for (int i = 0; i < nc; i++) {
      int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
      for (int d = 0; d < dim; d++) {
        lo[d] = std::max(0, grid[i * dim + d] - 3);
        hi[d] = std::min((1 << k) - 1, grid[i * dim + d] + 3);
      }
      cand.clear();
      int g[3];
      for (g[0] = lo[0]; g[0] <= hi[0]; g[0]++)
        for (g[1] = lo[1]; g[1] <= hi[1]; g[1]++)
          for (g[2] = lo[2]; g[2] <= hi[2]; g[2]++) {
            int64_t c = 0;
            for (int b = 0; b < k; b++)
              for (int ax = 0; ax < dim; ax++) c |= int64_t((g[ax] >> b) & 1) << (b * dim + ax);
            cand.push_back(int(c));
          }
      std::sort(cand.begin(), cand.end());
      wc.insert(wc.end(), cand.begin(), cand.end());
      wc_off[i + 1] = int(wc.size());
    }
  }
  bool in_il(int i, int j) const {
    if (!il_mask.empty()) {
      const int sl = slot(i, j);
      return sl >= 0 && ((il_mask[i] >> sl) & 1);
    }
    for (int t = il_off[i]; t < il_off[i + 1]; t++)
      if (il[t] == j) return true;
    return false;
  }
};

struct TreeH {
  int N = 0, dim = 2, depth = 0;
  bool sparse = false;                // built with allow_empty: leaf cells may hold no points
  std::vector<Topo> lv;               // index k = 1..depth (0 unused)
  std::vector<int64_t> perm;          // permuted position -> original index
  std::vector<int64_t> leaf_off;      // 4^depth + 1
  double* d_pts = nullptr;            // Morton-permuted, N x dim row-major
  int64_t* d_perm = nullptr;
  int64_t* d_leaf_off = nullptr;
  Arena arena{size_t(64) << 20};
  int nclusters(int k) const { return 1 << (dim * k); }
  int64_t range_lo(int k, int i) const { return leaf_off[size_t(i) << (dim * (depth - k))]; }
  int64_t range_hi(int k, int i) const { return leaf_off[size_t(i + 1) << (dim * (depth - k))]; }
};

// Initial (un-eliminated) operators, compact: exactly the reference's
// OperatorStore after init_operators (ifmm/operators.py:164-274).
struct InitLevel {
  int k = 0, nc = 0;
  std::vector<int> n, r0;              // particle dim, initial rank
  std::vector<double*> U;              // n x r0 (ld n)
  std::vector<int64_t> m2l_off;        // CSR over IL of each cluster (both orientations)
  std::vector<double*> m2l;            // r0_i x r0_j (ld r0_i)
  std::vector<int64_t> child_off;      // non-leaf: prefix of child r0 (nc*(2^d+1))
};

// Device workspaces of factorize(), kept with the store so that repeated
// factorizations (factor-once/solve-many is per factorization; benchmarks and
// parameter sweeps refactorize) do not pay cudaMalloc/cudaFree every call.
// A second stream for work that only needs to finish by the end of a colour
// batch (the pivot condition estimates), forked from / joined to the
// factorization stream with events.
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  void ensure() {
    if (s) return;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
  }
  ~SideStream() {
    if (s) {
      cudaStreamDestroy(s);
      cudaEventDestroy(fork);
      cudaEventDestroy(join);
    }
  }
};

struct FactorWork {
  std::mutex mu;
  SideStream side;     // condition estimates
  SideStream ahead;    // LU panel look-ahead
  Arena ws{size_t(256) << 20};
  Staging st;
  Arena lvl[2] = {Arena(size_t(2) << 30), Arena(size_t(2) << 30)};
};

struct StoreH {
  std::unique_ptr<FactorWork> work{new FactorWork};
  TreeH* tree = nullptr;
  KernelParams kp{};
  int p = 8;
  double tol = 1e-14;
  int max_init_rank = 0;
  std::vector<InitLevel> lv;           // index k
  std::vector<double*> leaf_p2p;       // nc_leaf * win: (i,j) for j in nbr(i), j >= i (ld n_i)
  std::vector<int> probe_tab;          // ACA probe rows: row m -> 10 ints
  int probe_maxm = 0;
  int* d_probe = nullptr;
  Arena arena{size_t(512) << 20};
  cudaStream_t stream = nullptr;
};

struct LevelStatsH {
  int clusters = 0, max_rank = 0, compressed = 0, dense_kept = 0;
  double max_cond = 0;  // largest pivot condition estimate ||S||_1 est||S^-1||_1 (this rank's pivots)
};
// A pivot whose condition estimate exceeded the limit (IFMM_FLAG_RECORD_SINGULAR)
struct SingularH {
  int level, index;
  double cond;
};

// Solve record of one elimination (the reference's _Record, ifmm/solver.py:63-74):
// the LU factors of S_i with their row permutation, and the coupling panel C
// (P2P_ij of the live neighbours | M2P_ij of the eliminated partners) the
// sweeps multiply with; partner positions in the solve vector.
struct RecordH {
  int level, index, n, r, w;
  double* lu;        // m x m (ld m), m = n + r: L (unit) and U of P S
  int* perm;         // m: row l of P S is row perm[l] of S
  double* c;         // n x w (ld n); columns [w - r, w) are zero
  int* pos;          // w absolute positions in the solve vector
  int64_t xoff;      // absolute position of x_i
  // larger pivots: inverted 64 x 64 diagonal blocks of L and U (per block: L_kk^-1, U_kk^-1,
  // column-major), kept with the record so the single-rhs sweeps replace the substitution
  // chains by block mat-vecs; *pflag != 0: a block is too ill-conditioned for that (lu.cu)
  const double* dinv;
  const unsigned char* pflag;
};

struct BatchH {
  int level, colour, rec0, rec1;
  const RecordH* d_recs;  // device copy of records[rec0..rec1)
  int maxn, maxw, maxm;
  // sharded solve: solve-vector runs (base, length) each rank writes in the
  // forward / backward sweep of this batch, rank-major with offsets
  std::vector<int64_t> fwd_runs, bwd_runs;  // pairs
  std::vector<int> fwd_off, bwd_off;        // nranks + 1, in pairs
};

class Comm;
struct Partition;

struct FactorH {
  StoreH* store = nullptr;
  TreeH* tree = nullptr;
  double tol = 0;
  int r_m = 0;
  std::vector<LevelStatsH> stats;      // index k
  std::vector<RecordH> recs;
  std::vector<BatchH> batches;
  int64_t vec_size = 0;                // solve vector length
  std::vector<int64_t> lvl_base;       // index k: base of level-k x slots; lvl_base[1] = top
  int top_dim = 0;
  double* top_lu = nullptr;            // LU of the level-2 system (M x M)
  int* top_perm = nullptr;
  int64_t g_size = 0;                  // sum of record n (per rhs)
  std::vector<int64_t> g_off;          // per record
  int64_t* d_g_off = nullptr;
  Arena arena{size_t(4) << 30};        // records, top factors
  cudaStream_t stream = nullptr;
  // timing of the last factorization (ms) and work accounting
  double ms_total = 0;
  double fl_exec = 0, fl_schur = 0, fl_ref = 0, solve_bytes = 0, fl_lu = 0, fl_x = 0;
  // per-phase device time (ms, CUDA events on the factorization stream) when
  // factorize() ran with IFMM_FLAG_TIMING: see PhaseId
  double phase_ms[8] = {0};
  long long phase_launches[8] = {0};
  int deferred_batches = 0;  // colour batches split by the independence guard
  std::vector<SingularH> singular;  // IFMM_FLAG_RECORD_SINGULAR: pivots over the limit, in elimination order
  // per record (host): the x / y partners of the elimination (the reference's
  // _Record.x_partners / y_partners, ifmm/solver.py:63-74)
  std::vector<std::vector<int>> rec_xp, rec_yp;
  std::vector<int64_t> top_off;  // offsets of the level-2 clusters in the top system
  std::vector<std::array<double, 8>> phase_lvl_ms;  // [level][phase]
  std::vector<std::array<double, 2>> host_lvl_ms;   // [level]: host busy until the final sync, time blocked in it
  // sharded factorization (null / 1 rank otherwise): the communicator the
  // solve reuses, this rank's partition, private workspaces and stream of an
  // emulated rank (LocalComm), traffic counters
  std::shared_ptr<Comm> comm;
  std::shared_ptr<Partition> part;
  std::unique_ptr<FactorWork> own_work;
  bool own_stream = false;
  double halo_bytes = 0, meta_bytes = 0;
  long long exchanges = 0;
  long long rc_before = 0, rc_after = 0;  // rank-growth control: sum of pivot ranks before / after
  ~FactorH();
};

enum PhaseId : int {
  PH_GATHER = 0,     // S / C gathers, record copies
  PH_GJ = 1,         // batched LU of the pivots (+ norms, condition estimates)
  PH_XGEMM = 2,      // X = S^-1 C (LU solves on the coupling panel)
  PH_SCHUR = 3,      // symmetric Schur update GEMMs
  PH_COMPRESS = 4,   // fill-in compression
  PH_TRANSITION = 5, // level start (parent near field, bases)
  PH_TOP = 6,        // top-level LU
  PH_COUNT = 7,
  PH_COMM = 7,       // sharded runs: metadata all-gathers + halo pack/exchange/unpack
};
constexpr int IFMM_FLAG_TIMING = 1;
// Record pivots whose condition estimate exceeds the limit and go on, instead
// of raising SingularPivotError at the first one (the reference raises).
constexpr int IFMM_FLAG_RECORD_SINGULAR = 2;

// One unknown slot of the extended system (extended.cu): kind 0 x, 1 y, 2 z
struct ExtSlot {
  int sym, level, index, dim;
};

// ------------------------------------------------------------ entry points
// allow_empty: leaf cells without points are accepted (extension for clustered inputs; the
// reference raises, ifmm/geometry.py:191-195)
TreeH* tree_build(const double* pts, int64_t n, int dim, int depth, bool device_ptr, bool allow_empty = false);
StoreH* store_init(TreeH* t, const KernelParams& kp, int p, double tol, const int* probe_tab, int probe_maxm);
void matvec(StoreH* s, const double* x, double* y, int64_t nrhs, bool device_ptr);
// extended system of the initial store (extended.cu): slot table, and the dense
// matrix (m x m, column-major, into host_out; null: size only) -> m
std::vector<ExtSlot> extended_layout(const StoreH* s);
int64_t extended_dense(StoreH* s, int64_t cap, double* host_out);
// rank_tol > 0: rank-growth control (consolidate.cu) -- an extension, off in the reference-parity path
FactorH* factorize(StoreH* s, double tol, int flags, double cond_limit, double rank_tol = 0.0);
// collective over `comm` (one call per rank, same store contents on every rank)
FactorH* factorize_sharded(StoreH* s, std::shared_ptr<Comm> comm, double tol, int flags, double cond_limit,
                           double rank_tol = 0.0);
// `nranks` virtual ranks as threads on the current GPU (LocalComm): out[r] is rank r's factorization
void factorize_emulated(StoreH* s, int nranks, double tol, int flags, double cond_limit, std::vector<FactorH*>& out,
                        double rank_tol = 0.0);
// solve on every virtual rank of an emulated factorization; x[r] is rank r's solution
void solve_emulated(const std::vector<FactorH*>& f, const double* rhs, const std::vector<double*>& x, int64_t nrhs,
                    bool device_ptr);
void solve(FactorH* f, const double* rhs, double* x, int64_t nrhs, bool device_ptr);
void solve_refined(FactorH* F, StoreH* S, const double* rhs, double* x, int64_t nrhs, bool device_ptr, int iters,
                   double target, double* hist, int* done);

// ------------------------------------------------------------ shared helpers
cudaStream_t default_stream();
void ensure_device();

}  // namespace ifmm
