// Uniform 2^d tree on the GPU: cell index, Morton code (x bit least
// significant), STABLE radix sort (ties keep input order, which fixes the row
// order inside every leaf exactly as numpy's stable argsort does), leaf
// offsets, permuted points and the duplicate-point check.  Neighbour /
// interaction lists and the 3^d colouring are integer metadata built on the
// host.  Follows ifmm/geometry.py:47-61 (PointSet checks), :124-140 (Morton),
// :174-226 (build_tree), :229-262 (compute_lists).
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cmath>

#include "core.cuh"

namespace ifmm {

static cudaStream_t g_stream = nullptr;
cudaStream_t default_stream() {
  if (!g_stream) CK(cudaStreamCreateWithFlags(&g_stream, cudaStreamNonBlocking));
  return g_stream;
}

void ensure_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    throw Error(IFMM_NO_DEVICE, "no CUDA device available: the B200 IFMM has no CPU fallback");
  }
}

__host__ __device__ inline int64_t morton_enc(const int* g, int dim, int bits) {
  int64_t c = 0;
  for (int b = 0; b < bits; b++)
    for (int ax = 0; ax < dim; ax++) c |= int64_t((g[ax] >> b) & 1) << (b * dim + ax);
  return c;
}
__host__ __device__ inline void morton_dec(int64_t c, int dim, int bits, int* g) {
  for (int ax = 0; ax < dim; ax++) g[ax] = 0;
  for (int b = 0; b < bits; b++)
    for (int ax = 0; ax < dim; ax++) g[ax] |= int((c >> (b * dim + ax)) & 1) << b;
}

__global__ void check_box_kernel(const double* pts, int64_t n, int dim, int* bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * dim; i += (int64_t)gridDim.x * blockDim.x) {
    double v = pts[i];
    if (!(fabs(v) <= 1.0)) atomicOr(bad, 1);
  }
}

__global__ void codes_kernel(const double* pts, int64_t n, int dim, int depth, int64_t* codes, int64_t* idx) {
  const int side = 1 << depth;
  const double inv_w = double(side) / 2.0;  // 1 / cell width, a power of two
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int g[3];
    for (int d = 0; d < dim; d++) {
      // floor((x + 1) / w): the add rounds like numpy, the scaling is exact
      double c = floor(__dmul_rn(__dadd_rn(pts[i * dim + d], 1.0), inv_w));
      int ci = int(c);
      ci = ci < 0 ? 0 : (ci > side - 1 ? side - 1 : ci);
      g[d] = ci;
    }
    codes[i] = morton_enc(g, dim, depth);
    idx[i] = i;
  }
}

__global__ void leaf_count_kernel(const int64_t* codes_sorted, int64_t n, int* counts) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&counts[codes_sorted[i]], 1);
}

__global__ void gather_pts_kernel(const double* in, const int64_t* perm, int64_t n, int dim, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * dim; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = i / dim;
    int d = int(i % dim);
    out[i] = in[perm[p] * dim + d];
  }
}

// Duplicate pairs (distance <= 1e-14, ifmm/geometry.py:57-61): each point is
// compared with the points of its own and the neighbouring leaves; the
// lexicographically smallest (orig_i, orig_j) pair wins (atomicMin on i*N+j).
__global__ void dup_kernel(const double* pts, const int64_t* perm, const int64_t* leaf_off, const int64_t* codes,
                           int64_t n, int dim, int depth, unsigned long long* best) {
  const int side = 1 << depth;
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < n; a += (int64_t)gridDim.x * blockDim.x) {
    int g[3], h[3];
    morton_dec(codes[a], dim, depth, g);
    const int64_t oa = perm[a];
    int nsh = 1;
    for (int d = 0; d < dim; d++) nsh *= 3;
    for (int s = 0; s < nsh; s++) {
      int t = s;
      bool ok = true;
      for (int d = 0; d < dim; d++) {
        h[d] = g[d] + (t % 3) - 1;
        t /= 3;
        if (h[d] < 0 || h[d] >= side) ok = false;
      }
      if (!ok) continue;
      int64_t leaf = morton_enc(h, dim, depth);
      for (int64_t b = leaf_off[leaf]; b < leaf_off[leaf + 1]; b++) {
        const int64_t ob = perm[b];
        if (ob <= oa) continue;
        double acc = 0.0;
        for (int d = 0; d < dim; d++) {
          double df = pts[a * dim + d] - pts[b * dim + d];
          acc += df * df;
        }
        if (sqrt(acc) <= 1e-14) atomicMin(best, (unsigned long long)(oa * n + ob));
      }
    }
  }
}

static void build_lists(TreeH* t) {
  const int dim = t->dim;
  t->lv.assign(t->depth + 1, Topo{});
  int nsh = 1;
  for (int d = 0; d < dim; d++) nsh *= 3;
  for (int k = 1; k <= t->depth; k++) {
    Topo& T = t->lv[k];
    T.k = k;
    T.dim = dim;
    T.nc = 1 << (dim * k);
    T.grid.resize(size_t(T.nc) * dim);
    T.colour.resize(T.nc);
    for (int i = 0; i < T.nc; i++) {
      int g[3];
      morton_dec(i, dim, k, g);
      int col = 0, mul = 1;
      for (int d = 0; d < dim; d++) {
        T.grid[size_t(i) * dim + d] = g[d];
        col += (g[d] % 3) * mul;
        mul *= 3;
      }
      T.colour[i] = col;
    }
    const int side = 1 << k;
    T.nbr_off.assign(1, 0);
    for (int i = 0; i < T.nc; i++) {
      std::vector<int> nb;
      for (int s = 0; s < nsh; s++) {
        int h[3], tt = s;
        bool ok = true;
        for (int d = 0; d < dim; d++) {
          h[d] = T.grid[size_t(i) * dim + d] + (tt % 3) - 1;
          tt /= 3;
          if (h[d] < 0 || h[d] >= side) ok = false;
        }
        if (ok) nb.push_back(int(morton_enc(h, dim, k)));
      }
      std::sort(nb.begin(), nb.end());
      T.nbr.insert(T.nbr.end(), nb.begin(), nb.end());
      T.nbr_off.push_back(int(T.nbr.size()));
    }
  }
  const int nch = 1 << dim;
  for (int k = 1; k <= t->depth; k++) {
    Topo& T = t->lv[k];
    T.il_off.assign(1, 0);
    for (int i = 0; i < T.nc; i++) {
      if (k > 1) {
        const Topo& P = t->lv[k - 1];
        const int pi = i >> dim;
        std::vector<int> cand;
        for (int q = P.nbr_off[pi]; q < P.nbr_off[pi + 1]; q++)
          for (int c = 0; c < nch; c++) {
            int j = (P.nbr[q] << dim) + c;
            bool isn = false;
            for (int u = T.nbr_off[i]; u < T.nbr_off[i + 1]; u++) isn |= (T.nbr[u] == j);
            if (!isn) cand.push_back(j);
          }
        std::sort(cand.begin(), cand.end());
        T.il.insert(T.il.end(), cand.begin(), cand.end());
      }
      T.il_off.push_back(int(T.il.size()));
    }
    T.prepare();  // window lists + interaction-list masks for the factorization
  }
}

TreeH* tree_build(const double* pts_in, int64_t n, int dim, int depth, bool device_ptr, bool allow_empty) {
  ensure_device();
  if (dim < 1 || dim > 3) invalid("dim must be 1, 2 or 3, got " + std::to_string(dim));
  if (n <= 0) invalid("points must have shape (n, dim) with n >= 1");
  std::unique_ptr<TreeH> t(new TreeH);
  t->N = int(n);
  t->dim = dim;
  t->depth = depth;
  cudaStream_t s = default_stream();
  Arena tmp(size_t(64) << 20);
  double* d_in = nullptr;
  if (device_ptr) {
    d_in = const_cast<double*>(pts_in);
  } else {
    d_in = tmp.alloc_n<double>(size_t(n) * dim);
    CK(cudaMemcpyAsync(d_in, pts_in, sizeof(double) * n * dim, cudaMemcpyHostToDevice, s));
  }
  int* d_flag = tmp.alloc_n<int>(4);
  CK(cudaMemsetAsync(d_flag, 0, 16, s));
  const int grid = int(std::min<int64_t>((n * dim + 255) / 256, 148 * 32));
  check_box_kernel<<<grid, 256, 0, s>>>(d_in, n, dim, d_flag);
  CK_LAUNCH();
  int h_flag = 0;
  CK(cudaMemcpyAsync(&h_flag, d_flag, 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (h_flag) invalid("point outside the reference box [-1, 1]^d");
  // duplicate check needs a tree: do it at a safe depth if the requested one is invalid
  if (depth < 2) invalid("depth must be >= 2 (interaction lists start at level 2)");
  if (depth * dim > 62) invalid("depth too large");
  int64_t *d_codes = tmp.alloc_n<int64_t>(n), *d_codes2 = tmp.alloc_n<int64_t>(n);
  int64_t* d_idx = tmp.alloc_n<int64_t>(n);
  t->d_perm = t->arena.alloc_n<int64_t>(n);
  codes_kernel<<<std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, s>>>(d_in, n, dim, depth, d_codes, d_idx);
  CK_LAUNCH();
  size_t tmp_bytes = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, d_codes, d_codes2, d_idx, t->d_perm, n, 0, dim * depth, s));
  void* d_tmp = tmp.alloc(tmp_bytes);
  CK(cub::DeviceRadixSort::SortPairs(d_tmp, tmp_bytes, d_codes, d_codes2, d_idx, t->d_perm, n, 0, dim * depth, s));
  const int64_t nleaf = int64_t(1) << (dim * depth);
  int* d_cnt = tmp.alloc_n<int>(nleaf);
  CK(cudaMemsetAsync(d_cnt, 0, sizeof(int) * nleaf, s));
  leaf_count_kernel<<<std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, s>>>(d_codes2, n, d_cnt);
  CK_LAUNCH();
  std::vector<int> cnt(nleaf);
  CK(cudaMemcpyAsync(cnt.data(), d_cnt, sizeof(int) * nleaf, cudaMemcpyDeviceToHost, s));
  t->perm.resize(n);
  CK(cudaMemcpyAsync(t->perm.data(), t->d_perm, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, s));
  t->d_pts = t->arena.alloc_n<double>(size_t(n) * dim);
  gather_pts_kernel<<<grid, 256, 0, s>>>(d_in, t->d_perm, n, dim, t->d_pts);
  CK_LAUNCH();
  CK(cudaStreamSynchronize(s));
  t->leaf_off.assign(nleaf + 1, 0);
  for (int64_t c = 0; c < nleaf; c++) t->leaf_off[c + 1] = t->leaf_off[c] + cnt[c];
  t->d_leaf_off = t->arena.alloc_n<int64_t>(nleaf + 1);
  CK(cudaMemcpyAsync(t->d_leaf_off, t->leaf_off.data(), sizeof(int64_t) * (nleaf + 1), cudaMemcpyHostToDevice, s));
  // duplicates (reference raises these before the empty-leaf check)
  unsigned long long* d_best = reinterpret_cast<unsigned long long*>(tmp.alloc(8));
  CK(cudaMemsetAsync(d_best, 0xff, 8, s));
  if (n > 1) {
    dup_kernel<<<std::min<int64_t>((n + 127) / 128, 148 * 16), 128, 0, s>>>(t->d_pts, t->d_perm, t->d_leaf_off,
                                                                            d_codes2, n, dim, depth, d_best);
    CK_LAUNCH();
  }
  unsigned long long best = 0;
  CK(cudaMemcpyAsync(&best, d_best, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (best != ~0ull) {
    long long i = (long long)(best / (unsigned long long)n), j = (long long)(best % (unsigned long long)n);
    invalid("duplicate points at indices " + std::to_string(i) + " and " + std::to_string(j));
  }
  for (int64_t c = 0; c < nleaf && !allow_empty; c++)
    if (cnt[c] == 0)  // uniform trees only, as the reference (ifmm/geometry.py:191-195)
      invalid("leaf cell " + std::to_string(c) + " is empty at depth " + std::to_string(depth));
  t->sparse = allow_empty;
  build_lists(t.get());
  return t.release();
}

}  // namespace ifmm
