// Batched block utilities (copy / transpose / scale-accumulate / zero, 1-norms)
// and the descriptor of the batched dense kernels (lu.cuh).
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
  int* ipiv;  // length m: row permutation of the LU (lu.cuh)
  int tag;    // caller-defined (pivot id)
};

// 1-norm (max column abs sum) of every matrix -> out[p]
void launch_norm1(const MatDesc* d_desc, int n, int maxm, double* out, cudaStream_t s);
}  // namespace ifmm
