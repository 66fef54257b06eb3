// Solve with the factored IFMM (ifmm/solver.py:549-626), level-wise and
// batch-parallel: for every colour batch one CTA per eliminated cluster.
//   forward : g_i = Sinv_nn b_i ; v[pos] -= X_top^T b_i     (z rows start at 0)
//   top     : y = T^-1 v_top
//   backward: x_i = g_i - X_top v[pos]     (batches and levels in reverse)
// Using X_top = (S^-1 C)_top for both sweeps (S symmetric) means a record is
// only Sinv_nn (n x n) + X_top (n x w): the solve streams each record twice.
// Vectors are (positions x nrhs) row-major; a level's y slots alias the next
// level's x slots.
#include <algorithm>
#include <cmath>

#include "core.cuh"

namespace ifmm {

void launch_permute(const double* in, double* out, const int64_t* perm, int64_t n, int nrhs, bool inverse,
                    cudaStream_t s);

__global__ void __launch_bounds__(256) solve_fwd_kernel(const RecordH* __restrict__ recs, int rec0,
                                                        const int64_t* __restrict__ g_off, double* V, double* G,
                                                        int nrhs) {
  extern __shared__ double sb[];  // n x nrhs
  const RecordH R = recs[blockIdx.x];
  const int n = R.n, w = R.w;
  double* g = G + g_off[rec0 + blockIdx.x] * nrhs;
  for (int e = threadIdx.x; e < n * nrhs; e += blockDim.x) sb[e] = V[R.xoff * nrhs + e];
  __syncthreads();
  // g = Sinv b : thread per (row t, rhs q), coalesced down the columns of Sinv
  for (int e = threadIdx.x; e < n * nrhs; e += blockDim.x) {
    const int t = e % n, q = e / n;
    double s = 0.0;
    for (int c = 0; c < n; c++) s = fma(R.sinv[t + (size_t)c * n], sb[c * nrhs + q], s);
    g[(size_t)t * nrhs + q] = s;
  }
  // v[pos] -= X_top^T b : warp per column
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int e = warp; e < w * nrhs; e += nw) {
    const int c = e / nrhs, q = e % nrhs;
    const double* x = R.xtop + (size_t)c * n;
    double s = 0.0;
    for (int t = lane; t < n; t += 32) s = fma(x[t], sb[t * nrhs + q], s);
    s = warp_sum(s);
    if (lane == 0) V[(int64_t)R.pos[c] * nrhs + q] -= s;
  }
}

__global__ void __launch_bounds__(256) solve_bwd_kernel(const RecordH* __restrict__ recs, int rec0,
                                                        const int64_t* __restrict__ g_off, double* V,
                                                        const double* G, int nrhs) {
  extern __shared__ double sv[];  // w x nrhs gathered partner values
  const RecordH R = recs[blockIdx.x];
  const int n = R.n, w = R.w;
  const double* g = G + g_off[rec0 + blockIdx.x] * nrhs;
  for (int e = threadIdx.x; e < w * nrhs; e += blockDim.x) {
    const int c = e / nrhs, q = e % nrhs;
    sv[e] = V[(int64_t)R.pos[c] * nrhs + q];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < n * nrhs; e += blockDim.x) {
    const int t = e % n, q = e / n;
    double s = g[(size_t)t * nrhs + q];
    for (int c = 0; c < w; c++) s = fma(-R.xtop[t + (size_t)c * n], sv[c * nrhs + q], s);
    V[(R.xoff + t) * nrhs + q] = s;
  }
}

// ------------------------------------------------------------------ refinement
__global__ void resid_kernel(const double* __restrict__ b, double* __restrict__ r, int64_t n, double* sums) {
  // r = b - r ; sums[0] += |r|^2, sums[1] += |b|^2
  __shared__ double red[32];
  double s0 = 0.0, s1 = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = b[i] - r[i];
    r[i] = v;
    s0 += v * v;
    s1 += b[i] * b[i];
  }
  s0 = block_sum(s0, red);
  s1 = block_sum(s1, red);
  if (threadIdx.x == 0) {
    atomicAdd(&sums[0], s0);
    atomicAdd(&sums[1], s1);
  }
}

__global__ void axpy_kernel(double* __restrict__ x, const double* __restrict__ dx, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] += dx[i];
}

void matvec(StoreH* S, const double* x, double* y, int64_t nrhs, bool device_ptr);

// Iterative refinement with the compressed FMM operator of the store:
// x <- x + IFMM^-1 (b - A~ x).  Each step divides the residual by the
// factorization's relative error; hist[j] = ||b - A~ x_j|| / ||b||.
void solve_refined(FactorH* F, StoreH* S, const double* rhs, double* x, int64_t nrhs, bool device_ptr, int iters,
                   double target, double* hist, int* done) {
  const int64_t n = int64_t(F->tree->N) * nrhs;
  cudaStream_t s = F->stream;
  Arena ws(size_t(64) << 20);
  double *db, *dx;
  if (device_ptr) {
    db = const_cast<double*>(rhs);
    dx = x;
  } else {
    db = ws.alloc_n<double>(n);
    dx = ws.alloc_n<double>(n);
    CK(cudaMemcpyAsync(db, rhs, sizeof(double) * n, cudaMemcpyHostToDevice, s));
  }
  double* r = ws.alloc_n<double>(n);
  double* d = ws.alloc_n<double>(n);
  double* sums = ws.alloc_n<double>(2);
  const int grid = int(std::min<int64_t>((n + 255) / 256, 148 * 8));
  solve(F, db, dx, nrhs, true);
  int it = 0;
  for (;; it++) {
    matvec(S, dx, r, nrhs, true);
    CK(cudaMemsetAsync(sums, 0, 16, s));
    resid_kernel<<<grid, 256, 0, s>>>(db, r, n, sums);
    CK_LAUNCH();
    double h[2];
    CK(cudaMemcpyAsync(h, sums, 16, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const double rel = h[1] > 0 ? std::sqrt(h[0] / h[1]) : 0.0;
    if (hist) hist[it] = rel;
    if (it >= iters || rel <= target) break;
    solve(F, r, d, nrhs, true);
    axpy_kernel<<<grid, 256, 0, s>>>(dx, d, n);
    CK_LAUNCH();
  }
  if (done) *done = it;
  if (!device_ptr) CK(cudaMemcpyAsync(x, dx, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
}

void solve(FactorH* F, const double* rhs, double* x, int64_t nrhs, bool device_ptr) {
  TreeH* t = F->tree;
  const int64_t N = t->N;
  if (nrhs < 1) invalid("nrhs must be >= 1");
  const int nr = int(nrhs);
  cudaStream_t s = F->stream;
  Arena ws(size_t(64) << 20);
  double *din, *dout;
  if (device_ptr) {
    din = const_cast<double*>(rhs);
    dout = x;
  } else {
    din = ws.alloc_n<double>(N * nr);
    dout = ws.alloc_n<double>(N * nr);
    CK(cudaMemcpyAsync(din, rhs, sizeof(double) * N * nr, cudaMemcpyHostToDevice, s));
  }
  double* V = ws.alloc_n<double>(std::max<int64_t>(1, F->vec_size) * nr);
  double* G = ws.alloc_n<double>(std::max<int64_t>(1, F->g_size) * nr);
  CK(cudaMemsetAsync(V, 0, sizeof(double) * std::max<int64_t>(1, F->vec_size) * nr, s));
  launch_permute(din, V + F->lvl_base[t->depth] * nr, t->d_perm, N, nr, false, s);
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(solve_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(solve_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  for (const BatchH& b : F->batches) {
    const size_t smem = sizeof(double) * size_t(b.maxn) * nr;
    if (smem > 200 * 1024) invalid("solve: too many right-hand sides for one pass");
    solve_fwd_kernel<<<b.rec1 - b.rec0, 256, smem, s>>>(b.d_recs, b.rec0, F->d_g_off, V, G, nr);
    CK_LAUNCH();
  }
  // top: y = T^-1 b on the level-1 slots (viewed column-major as nrhs x M)
  if (F->top_dim > 0) {
    const int M = F->top_dim;
    double* vt = V + F->lvl_base[1] * nr;
    double* tmp = ws.alloc_n<double>(size_t(M) * nr);
    CK(cudaMemcpyAsync(tmp, vt, sizeof(double) * M * nr, cudaMemcpyDeviceToDevice, s));
    GemmBatch gb;
    Staging st;
    gb.add(tmp, nr, F->top_inv, M, vt, nr, nr, M, M, 1.0, 0.0);
    launch_grouped_gemm(gb, false, true, ws, st, s);
    CK(cudaStreamSynchronize(s));
  }
  for (auto it = F->batches.rbegin(); it != F->batches.rend(); ++it) {
    const BatchH& b = *it;
    const size_t smem = sizeof(double) * size_t(b.maxw) * nr;
    if (smem > 200 * 1024) invalid("solve: too many right-hand sides for one pass");
    solve_bwd_kernel<<<b.rec1 - b.rec0, 256, smem, s>>>(b.d_recs, b.rec0, F->d_g_off, V, G, nr);
    CK_LAUNCH();
  }
  launch_permute(V + F->lvl_base[t->depth] * nr, dout, t->d_perm, N, nr, true, s);
  if (!device_ptr) CK(cudaMemcpyAsync(x, dout, sizeof(double) * N * nr, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
}

}  // namespace ifmm
