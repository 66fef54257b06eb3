// Batched block utilities (copy / transpose / scale-accumulate / zero, 1-norms)
// and the batched Gauss-Jordan inversion with partial pivoting used for the
// IFMM pivot blocks S_i = [[P2P_ii, U_i], [U_i^T, 0]].
#pragma once
#include "common.cuh"
#include "gemm.cuh"

namespace ifmm {

// dst(i,j) = [accumulate ? dst(i,j) : 0] + alpha * (trans ? src(j,i) : src(i,j))
// src == nullptr writes zeros (or leaves dst unchanged if accumulate).
struct CopyDesc {
  const double* src;
  double* dst;
  int rows, cols;
  int lds, ldd;
  int trans;
  int accumulate;
  double alpha;
};

struct CopyBatch {
  std::vector<CopyDesc> d;
  void add(const double* src, int lds, double* dst, int ldd, int rows, int cols, bool trans = false,
           double alpha = 1.0, bool accumulate = false) {
    if (rows <= 0 || cols <= 0) return;
    d.push_back(CopyDesc{src, dst, rows, cols, lds, ldd, trans ? 1 : 0, accumulate ? 1 : 0, alpha});
  }
  void zero(double* dst, int ldd, int rows, int cols) { add(nullptr, 0, dst, ldd, rows, cols); }
  void clear() { d.clear(); }
};
void launch_copies(CopyBatch& b, Arena& ws, Staging& st, cudaStream_t s);

// pos[out + u] = base + u for u < dim (solve partner positions)
struct PosRun {
  int64_t base, out;
  int dim, pad;
};
void launch_pos_expand(const PosRun* d_runs, int n, int* pos, cudaStream_t s);

// Matrix descriptor for batched dense kernels (column-major).
struct MatDesc {
  double* A;
  int m;
  int lda;
  int* ipiv;  // length m (GJ)
  int tag;    // caller-defined (pivot id)
};

// 1-norm (max column abs sum) of every matrix -> out[p]
void launch_norm1(const MatDesc* d_desc, int n, int maxm, double* out, cudaStream_t s);
// dlacn2 (Hager/Higham) estimate of the 1-norm of every matrix -> out[p]; out
// holds the exact norm on entry and is only replaced where
// exact * normA[p] >= limit (the estimate is <= the exact norm)
void launch_norm1_estimate(const MatDesc* d_desc, int n, int maxm, double* out, const double* normA, double limit,
                           cudaStream_t s);

// In-place inversion of every matrix by blocked Gauss-Jordan elimination with
// partial pivoting.  `info[p]` = 0, or 1 + first column with an exact zero
// pivot.  Host-side descriptors `h` (same content as d_desc) drive the GEMM
// trailing updates.  With `side` (a high-priority stream and two events) the
// panel of step j+1 runs concurrently with the bulk of step j's update.
struct GjSide {
  cudaStream_t s = nullptr;
  cudaEvent_t e_cols = nullptr, e_panel = nullptr;
  void ensure() {
    if (s) return;
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, hi));
    CK(cudaEventCreateWithFlags(&e_cols, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&e_panel, cudaEventDisableTiming));
  }
  ~GjSide() {
    if (e_cols) cudaEventDestroy(e_cols);
    if (e_panel) cudaEventDestroy(e_panel);
    if (s) cudaStreamDestroy(s);
  }
};
// shape_n / shape_maxm (sharded runs): count and largest size of the whole
// colour batch across ranks -- the blocking scheme is chosen from them, so
// each matrix is inverted with the same arithmetic as on one GPU
void batched_gj_inverse(const std::vector<MatDesc>& h, const MatDesc* d_desc, int* d_info, Arena& ws,
                        Staging& st, cudaStream_t s, const GjSide* side = nullptr, int shape_n = 0,
                        int shape_maxm = 0);

}  // namespace ifmm
