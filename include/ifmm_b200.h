/*
 * ifmm_b200.h -- C ABI of the B200-native IFMM factorize/solve library
 * (libifmm_b200.so, sm_100a).  Plain pointers and sizes only.
 *
 * The reference (`/root/reference/pkg/src/ifmm`, Python) has no FFI of its own:
 * its boundary is the Python module API.  Each entry point below replaces one
 * reference call (file:line cited); the Python mirror `paper_1407_1572_b200`
 * binds them with ctypes and keeps the reference's names,
 * argument meaning and exceptions.
 *
 * Conventions
 *   - every function returns an IFMM_* status; on failure ifmm_last_error()
 *     holds a message (thread-local).  IFMM_SINGULAR_PIVOT additionally sets
 *     ifmm_last_singular(level, index, cond)   (SingularPivotError,
 *     ifmm/solver.py:53-60, raised at :214-218).
 *   - point arrays are (n, dim) row-major doubles; right-hand sides and
 *     solutions are (n, nrhs) row-major doubles, in ORIGINAL point order.
 *   - ptr_kind = IFMM_PTR_HOST (pageable/pinned host memory; the library does
 *     the host<->device copies) or IFMM_PTR_DEVICE (CUDA device pointers).
 *   - there is no CPU fallback: without a CUDA device every compute entry
 *     point returns IFMM_NO_DEVICE.
 */
#ifndef IFMM_B200_H
#define IFMM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  IFMM_OK = 0,
  IFMM_INVALID = 1,        /* ValueError */
  IFMM_SINGULAR_PIVOT = 2, /* SingularPivotError */
  IFMM_CUDA = 3,           /* RuntimeError */
  IFMM_OOM = 4,            /* MemoryError */
  IFMM_NO_DEVICE = 5       /* RuntimeError: no CUDA device, no fallback */
};

enum { IFMM_PTR_HOST = 0, IFMM_PTR_DEVICE = 1 };
/* IFMM_FLAG_RECORD_SINGULAR: pivots whose condition estimate exceeds the limit
 * are recorded (ifmm_factor_singular) and the factorization goes on; without it
 * the first one raises IFMM_SINGULAR_PIVOT, as the reference does */
enum { IFMM_FLAG_TIMING = 1, IFMM_FLAG_RECORD_SINGULAR = 2 };

/* kernel ids: the reference registry ifmm/kernels.py:160-170 plus the two
 * BASELINE kernels inv_r = scale/r and log_r = scale*(ln r + shift) */
enum {
  IFMM_K_LOG = 0, IFMM_K_LAPLACE3D = 1, IFMM_K_BIHARMONIC = 2, IFMM_K_BESSEL_Y0 = 3,
  IFMM_K_INVERSE_QUADRIC = 4, IFMM_K_INVERSE_MULTIQUADRIC = 5, IFMM_K_HELMHOLTZ3D = 6,
  IFMM_K_GAUSSIAN = 7, IFMM_K_MULTIQUADRIC = 8, IFMM_K_INV_R = 9, IFMM_K_LOG_R = 10
};

typedef struct ifmm_tree ifmm_tree;
typedef struct ifmm_store ifmm_store;
typedef struct ifmm_factor ifmm_factor;
typedef struct ifmm_comm ifmm_comm;

const char* ifmm_last_error(void);
int ifmm_last_singular(int* level, int* index, double* cond);
int ifmm_version(void);
int ifmm_device_count(void);
/* select the CUDA device used by subsequent calls on this thread */
int ifmm_set_device(int device);

/* Device slabs of freed stores / factorizations are cached for reuse (cudaMalloc and
 * cudaFree of multi-GB slabs are slow and synchronise); this returns the cached ones of
 * the current device to the driver.  The cache also flushes itself when an allocation
 * would otherwise fail. */
int ifmm_release_cached_memory(void);

/* ---- tree: PointSet checks + build_tree + compute_lists
 *      (ifmm/geometry.py:47-61, :174-226, :229-262) */
int ifmm_tree_build(const double* points, int64_t n, int dim, int depth, int ptr_kind, ifmm_tree** out);
/* Extension for clustered inputs (BASELINE config 4's Gaussian mixture): the same
 * uniform tree, but leaf cells without points are accepted -- the reference
 * raises on them (ifmm/geometry.py:191-195).  Empty clusters carry no unknowns
 * and are skipped by the elimination. */
int ifmm_tree_build_sparse(const double* points, int64_t n, int dim, int depth, int ptr_kind, ifmm_tree** out);
int ifmm_tree_info(const ifmm_tree* t, int64_t* n, int* dim, int* depth);
/* permuted position -> original index (ClusterTree.point_permutation) */
int ifmm_tree_permutation(const ifmm_tree* t, int64_t* perm);
/* leaf point ranges: 2^(dim*depth)+1 offsets into the permuted points */
int ifmm_tree_leaf_offsets(const ifmm_tree* t, int64_t* off);
/* neighbour / interaction lists of `level` as CSR; call with null arrays to
 * get sizes[0] = #nbr entries, sizes[1] = #il entries */
int ifmm_tree_lists(const ifmm_tree* t, int level, int32_t* nbr_off, int32_t* nbr, int32_t* il_off, int32_t* il,
                    int64_t* sizes);
/* elimination colour of every cluster of `level` (sum_d (g_d mod 3) 3^d) */
int ifmm_tree_colours(const ifmm_tree* t, int level, int32_t* colours);
void ifmm_tree_free(ifmm_tree* t);

/* ---- operators: init_operators(tree, kernel, p, tol) (ifmm/operators.py:164-274)
 * probe_table: (probe_maxm+1) x 22 int32, row m for an m-row fill: the 10 ACA
 * probe rows of ifmm/lowrank.py:196-197 (np.random.default_rng(0).choice), then
 * that generator's PCG64 state after the draw (6 x 64-bit little-endian:
 * state hi, state lo, increment hi, increment lo, has_uint32, uinteger), which
 * the random restart rows of ifmm/lowrank.py:224-226 continue. */
int ifmm_store_init(ifmm_tree* t, int kernel_id, double a, double scale, double shift, int p, double tol,
                    const int32_t* probe_table, int probe_maxm, ifmm_store** out);
int ifmm_store_max_init_rank(const ifmm_store* s, int* r);
/* particle dims and initial ranks of every cluster of `level` (>= 2) */
int ifmm_store_dims(const ifmm_store* s, int level, int32_t* n, int32_t* r);
/* basis U (n x r, column-major) of cluster `index` (OperatorStore.l2p) */
int ifmm_store_basis(const ifmm_store* s, int level, int index, double* out);
/* M2L block (r_i x r_j, column-major) of interaction-list pair (i, j) */
int ifmm_store_m2l(const ifmm_store* s, int level, int i, int j, double* out);
/* leaf near-field block P2P(i, j) (n_i x n_j, column-major) of neighbour pair
 * (i, j) (OperatorStore.p2p, ifmm/operators.py:180-194; stored once per pair) */
int ifmm_store_p2p(const ifmm_store* s, int i, int j, double* out);
/* test hook: overwrite the store's initial operators with blocks
 * built elsewhere -- e.g. the reference's own OperatorStore (ifmm/operators.py:42-137)
 * -- so the elimination can be checked on bit-identical inputs.  Same shapes and
 * layouts as the getters above (basis n x r, M2L r_i x r_j, leaf P2P n_i x n_j,
 * column-major); the ranks must equal the store's. */
int ifmm_store_set_basis(ifmm_store* s, int level, int index, const double* in);
int ifmm_store_set_m2l(ifmm_store* s, int level, int i, int j, const double* in);
int ifmm_store_set_p2p(ifmm_store* s, int i, int j, const double* in);
/* bytes of the assembled operators as stored: out3[0] leaf near field P2P
 * (each neighbour pair once), out3[1] M2L blocks (both orientations of every
 * interaction-list pair), out3[2] bases U (levels >= 2) -- the algorithmic
 * traffic of assembly (written once) and of fmm_matvec (read once) */
int ifmm_store_bytes(const ifmm_store* s, double* out3);
/* extended sparse system of the initial store (verification / export path,
 * ifmm/operators.py:338-364 extended_layout, :367-445 assemble_extended_dense).
 * Slot table: *count slots of (sym 0 x / 1 y / 2 z, level, index, dim) in the
 * reference's order; call with null arrays for the count. */
int ifmm_extended_layout(const ifmm_store* s, int64_t* count, int32_t* sym, int32_t* level, int32_t* index,
                         int32_t* dim);
/* the dense extended matrix (dim x dim, COLUMN-major) scattered on the device
 * into host `out`; out = null returns only *dim.  IFMM_INVALID if dim > cap
 * ("extended dimension m exceeds cap c", as the reference's ValueError). */
int ifmm_extended_dense(ifmm_store* s, int64_t cap, int64_t* dim, double* out);
/* fmm_matvec (ifmm/operators.py:282-330): y = A~ x, x/y (n, nrhs) */
int ifmm_matvec(ifmm_store* s, const double* x, double* y, int64_t nrhs, int ptr_kind);
void ifmm_store_free(ifmm_store* s);

/* ---- factorize(store, tree, tol) (ifmm/solver.py:106-153); tol < 0 -> store tol.
 * cond_limit: PIVOT_CONDITION_LIMIT (ifmm/solver.py:50); <= 0 -> 1e12 (reference).
 * The store's initial operators are left intact (matvec stays valid). */
int ifmm_factorize(ifmm_store* s, double tol, int flags, double cond_limit, ifmm_factor** out);
/* Extension (SURVEY 8f item 3, rank-growth control; the reference's unused
 * _maybe_consolidate, ifmm/solver.py:437-492): right before a cluster is
 * eliminated, its coupling row (its M2L blocks and its rows of the parent's
 * basis) is re-truncated jointly at rank_tol (relative to the row's largest
 * singular value, 0 < rank_tol < 1) and its basis rotated onto the kept
 * directions.  Smaller pivots and parents; not the reference's arithmetic, so
 * ifmm_factorize stays the parity path. */
int ifmm_factorize_rank_control(ifmm_store* s, double tol, int flags, double cond_limit, double rank_tol,
                                ifmm_factor** out);
/* out2 = sum of the pivots' basis ranks before / after their consolidation (0, 0 without rank control) */
int ifmm_factor_rank_control(const ifmm_factor* f, int64_t* out2);
/* r_m, top-level dimension, number of eliminations, factorization wall ms */
int ifmm_factor_info(const ifmm_factor* f, int* r_m, int* top_dim, int64_t* n_records, double* ms);
/* LevelStats of `level`: clusters, max_rank, fillins_compressed, fillins_dense_kept */
int ifmm_factor_level_stats(const ifmm_factor* f, int level, int32_t* out4);
/* largest pivot condition estimate ||S||_1 * est(||S^-1||_1) of `level` (the
 * quantity the reference compares with PIVOT_CONDITION_LIMIT, ifmm/solver.py:214-218) */
int ifmm_factor_level_cond(const ifmm_factor* f, int level, double* max_cond);
/* IFMM_FLAG_RECORD_SINGULAR: *count pivots exceeded the limit; the first `cap`
 * are written as (level, index, cond) in elimination order (arrays may be null) */
int ifmm_factor_singular(const ifmm_factor* f, int64_t cap, int32_t* level, int32_t* index, double* cond,
                         int64_t* count);
/* record idx (elimination order) -- the reference's _Record (ifmm/solver.py:63-74):
 * info7 = level, index, n, r, w, #x partners, #y partners; xp / yp (may be null)
 * receive the partner cluster indices */
int ifmm_factor_record(const ifmm_factor* f, int64_t idx, int32_t* info7, int32_t* xp, int32_t* yp);
/* its pivot factors: lu ((n+r) x (n+r), column-major, L unit lower + U) and perm
 * (row l of P S is row perm[l] of S) -- the reference keeps scipy lu_factor's (lu, piv) */
int ifmm_factor_record_lu(const ifmm_factor* f, int64_t idx, double* lu, int32_t* perm);
/* the level-2 top system's LU (top_dim^2, column-major) + perm, and the offsets
 * of the level-2 clusters in it (4^2 + 1 in 2-D) -- IfmmFactorization.top_lu /
 * top_offsets (ifmm/solver.py:85-98, 528-546) */
int ifmm_factor_top(const ifmm_factor* f, double* lu, int32_t* perm, int64_t* offsets);
/* per elimination (in order): level, index, n, r, w */
int ifmm_factor_records(const ifmm_factor* f, int32_t* out5);
/* work accounting: out[0] executed FP64 flops (pivot LU, X = S^-1 C, symmetric
 * Schur update, top LU), out[1] of which in the Schur update, out[2]
 * reference-equivalent flops (sum 2/3 m^3 + 2 m^2 w + 2 h n w
 * + 2/3 M_top^3), out[3] bytes one solve sweep streams per right-hand side,
 * out[4] pivot LU flops (sum 2/3 m^3), out[5] X = S^-1 C flops (sum 2 m^2 w) */
int ifmm_factor_work(const ifmm_factor* f, double* out6);
/* per-phase device time in ms and kernel launches, recorded with CUDA events
 * on the factorization stream when ifmm_factorize ran with IFMM_FLAG_TIMING:
 * 0 gathers/copies, 1 pivot LU (+ norms), 2 X = S^-1 C, 3 Schur update,
 * 4 fill-in compression, 5 level transitions, 6 top-level LU */
int ifmm_factor_timing(const ifmm_factor* f, double* ms7, int64_t* launches7);
/* the same per level (level 1 = top-level inverse); ms9[7] = host time spent
 * preparing the level's batches before their final sync, ms9[8] = time the
 * host was blocked in those syncs (wall clock, recorded on every run) */
int ifmm_factor_timing_level(const ifmm_factor* f, int level, double* ms9);
/* total kernel launches issued by the library since load */
int64_t ifmm_launch_count(void);
/* solve(fact, rhs) (ifmm/solver.py:549-626) for nrhs >= 1 columns */
int ifmm_solve(ifmm_factor* f, const double* rhs, double* x, int64_t nrhs, int ptr_kind);
/* solve + iterative refinement with the store's compressed FMM operator
 * (an extension; the reference solves once): x <- x + solve(b - A~ x) until
 * ||b - A~ x|| / ||b|| <= target or max_iters refinement steps.  hist
 * (max_iters + 1 doubles, may be null) receives the residual after each step. */
int ifmm_solve_refined(ifmm_factor* f, ifmm_store* s, const double* rhs, double* x, int64_t nrhs, int ptr_kind,
                       int max_iters, double target, double* hist, int* iters_done);
void ifmm_factor_free(ifmm_factor* f);

/* ---- subtree-sharded factorize / solve over several GPUs (the
 * reference is single-process and has no counterpart: this extends
 * factorize(store, tree, tol) ifmm/solver.py:106-153 and solve ifmm/solver.py:549).
 * One process per GPU.  Level-2 subtrees are dealt to ranks in contiguous
 * Morton ranges; every rank replays the host schedule, computes its own
 * subtrees' eliminations and ships the blocks it wrote to the ranks storing
 * them (NCCL send/recv over NVLink after every colour batch).  Every call
 * below marked "collective" must be made by all ranks in the same order. */
/* 128-byte NCCL unique id (call on one rank, share it, e.g. via torch.distributed) */
int ifmm_comm_nccl_unique_id(uint8_t* out128);
int ifmm_comm_nccl_version(int* version);
/* collective: communicator over the current CUDA device of every rank */
int ifmm_comm_nccl_init(const uint8_t* id128, int nranks, int rank, ifmm_comm** out);
/* host-staged transport: the collectives call back into the caller (e.g.
 * torch.distributed over gloo) with pinned host buffers; every rank must make
 * the same sequence of calls.  allgather: recv (nranks * bytes, rank-major)
 * receives every rank's `bytes` from send.  exchange: nsend sends / nrecv
 * receives (peer, buffer, bytes); messages between a pair match in list order.
 * Callbacks return 0 on success.  Runs the real multi-process schedule on
 * processes that share one GPU. */
typedef int (*ifmm_host_allgather_fn)(void* ctx, const void* send, void* recv, int64_t bytes);
typedef int (*ifmm_host_exchange_fn)(void* ctx, int nsend, const int32_t* send_peer, void* const* send_buf,
                                     const int64_t* send_bytes, int nrecv, const int32_t* recv_peer,
                                     void* const* recv_buf, const int64_t* recv_bytes);
int ifmm_comm_host_init(int nranks, int rank, ifmm_host_allgather_fn allgather, ifmm_host_exchange_fn exchange,
                        void* ctx, ifmm_comm** out);
void ifmm_comm_free(ifmm_comm* c);
/* collective transport check: all-gather of n doubles and a ring send/recv
 * (a 1-rank communicator sends to itself); ok = 1 if all data arrived */
int ifmm_comm_selftest(ifmm_comm* c, int64_t n, int32_t* ok);
/* collective: sharded factorization; ifmm_solve on the result is collective
 * too and returns the full solution on every rank.  nranks <= 4^2 (2-D). */
int ifmm_factorize_sharded(ifmm_store* s, ifmm_comm* c, double tol, int flags, double cond_limit,
                           ifmm_factor** out);
/* the same schedule with `nranks` virtual ranks as threads on this GPU
 * (device-to-device copies instead of NCCL): out[nranks] factor handles */
int ifmm_factorize_emulated(ifmm_store* s, int nranks, double tol, int flags, double cond_limit,
                            ifmm_factor** out);
/* the sharded / emulated factorizations with rank-growth control (see
 * ifmm_factorize_rank_control): the rotated M2L blocks travel with each colour
 * batch's halo, the rotation of a block shared by pivots of two ranks and the
 * new ranks in two small extra exchanges per batch */
int ifmm_factorize_sharded_rank_control(ifmm_store* s, ifmm_comm* c, double tol, int flags, double cond_limit,
                                        double rank_tol, ifmm_factor** out);
int ifmm_factorize_emulated_rank_control(ifmm_store* s, int nranks, double tol, int flags, double cond_limit,
                                         double rank_tol, ifmm_factor** out);
/* solve on every virtual rank; x: nranks consecutive (n, nrhs) solutions */
int ifmm_solve_emulated(ifmm_factor** f, int nranks, const double* rhs, double* x, int64_t nrhs, int ptr_kind);
/* rank_nranks[2]; out4: halo bytes sent, metadata bytes sent, exchanges,
 * device ms in communication phases (with IFMM_FLAG_TIMING) */
int ifmm_factor_shard_info(const ifmm_factor* f, int32_t* rank_nranks, double* out4);
/* host-only: owner rank of every cluster of `level` and held[s * nc + i] = 1 if
 * rank s stores cluster i's blocks (its own clusters and their neighbours) */
int ifmm_partition(int dim, int depth, int level, int nranks, int32_t* owner, uint8_t* held);
/* host-only plan check: halo items rank `rank` sends to / receives from each
 * peer for colour batch `colour` of `level` with the initial block pattern,
 * routed by the factorization's own rule (comm.cuh halo_route) */
int ifmm_partition_halo_counts(int dim, int depth, int level, int nranks, int rank, int colour, int32_t* send,
                               int32_t* recv);

/* ---- test hooks for the batched kernels (host arrays in/out) */
/* run the Jacobi / QR / ACA hooks on one warp (1) or a 256-thread CTA (0) */
int ifmm_test_set_group(int warp);
/* in-place batched LU (partial pivoting) of `count` column-major matrices of sizes m[c],
   packed; perm (sum m[c]): row l of P A is row perm[l] of A; info: 0 or 1 + first zero
   pivot column; inv_norm1: dlacn2 estimate of ||A^-1||_1 (the pivot-condition test) */
int ifmm_test_lu(double* a, const int32_t* m, int count, int32_t* perm, int32_t* info, double* inv_norm1);
/* X = S^-1 [[C, 0], [0, -I_r]] for one factored pivot of size n + r (lu, perm from
   ifmm_test_lu; C n x wl column-major): xtop n x (wl + r), xbot r x (wl + r) */
int ifmm_test_lu_solve_x(const double* lu, const int32_t* perm, int n, int r, const double* c, int wl,
                         double* xtop, double* xbot);
/* C = alpha op(A) op(B) + beta C, column-major, one problem */
int ifmm_test_gemm(int transA, int transB, int M, int N, int K, double alpha, const double* A, int lda,
                   const double* B, int ldb, double beta, double* C, int ldc, int transC);
/* one-sided Jacobi: A (m x n) -> orthogonal columns, V (n x n), sig (n) */
int ifmm_test_jacobi(double* a, int m, int n, double* v, double* sig);
/* Householder QR: A (m x k) -> Q (m x k), R (k x k) */
int ifmm_test_qr(const double* a, int m, int k, double* q, double* r);
/* ACA of F (m x n): returns rank, left (m x rank), right (n x rank); probes = one
 * 22-int row of the probe table (see ifmm_store_init) */
int ifmm_test_aca(const double* f, int m, int n, double tol, const int32_t* probes, int kmax, double* left,
                  double* right, int32_t* rank, int32_t* incompressible);
/* fill compression K1 on one m x n fill (ACA + recompression, ifmm/lowrank.py:137-263):
 * gram = 1 via the cross Gram matrices (Householder fallback), 0 via Householder QRs;
 * F ~= left (m x rank) right^T (n x rank), sv = kept singular values, status 1 = kept dense */
int ifmm_test_recompress(const double* f, int m, int n, double tol, const int32_t* probes, int gram, double* left,
                         double* right, double* sv, int32_t* rank, int32_t* status);

#ifdef __cplusplus
}
#endif
#endif
