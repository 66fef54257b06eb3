// FMM matvec with the initial (compressed) operators, ifmm/operators.py:282-330:
// upward y = U^T x (non-leaf x = stacked child y), downward
// z = sum_IL M2L y + parent L2L slice, leaf out = U z + sum_nbr P2P x.
// HBM-bound: one CTA per cluster per level; vectors are (rows x nrhs)
// row-major so a multi-rhs apply streams every operator block once.
#include <algorithm>
#include <map>
#include <mutex>

#include "core.cuh"

namespace ifmm {

struct MvLevelDev {
  const double** U = nullptr;
  int* n = nullptr;
  int* r = nullptr;
  int64_t* yoff = nullptr;      // prefix of r0 (level-k y/z buffers)
  int64_t* xoff = nullptr;      // prefix of n (x buffer at this level)
  const double** m2l = nullptr;
  int* il_off = nullptr;
  int* il = nullptr;
  int64_t* child_off = nullptr;  // nc * (2^d+1)
  const double** p2p = nullptr;  // leaf only: nc * win
  int64_t ysize = 0;
};

struct MvCache {
  std::vector<MvLevelDev> lv;
  Arena arena{size_t(16) << 20};
};


__global__ void __launch_bounds__(256) mv_up_kernel(MvLevelDev L, const double* xin, double* yout, int nrhs) {
  const int i = blockIdx.x;
  const double* U = L.U[i];
  const int n = L.n[i], r = L.r[i];
  const double* x = xin + L.xoff[i] * nrhs;
  double* y = yout + L.yoff[i] * nrhs;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int e = warp; e < r * nrhs; e += nw) {
    const int c = e / nrhs, q = e % nrhs;
    double s = 0.0;
    for (int t = lane; t < n; t += 32) s = fma(U[t + (size_t)c * n], x[(size_t)t * nrhs + q], s);
    s = warp_sum(s);
    if (lane == 0) y[(size_t)c * nrhs + q] = s;
  }
}

__global__ void __launch_bounds__(256) mv_down_kernel(MvLevelDev L, MvLevelDev P, int has_parent, int dim,
                                                      const double* y, double* z, const double* zpar, int nrhs) {
  const int i = blockIdx.x;
  const int r = L.r[i];
  double* zi = z + L.yoff[i] * nrhs;
  for (int e = threadIdx.x; e < r * nrhs; e += blockDim.x) {
    const int c = e / nrhs, q = e % nrhs;
    double s = 0.0;
    for (int u = L.il_off[i]; u < L.il_off[i + 1]; u++) {
      const int j = L.il[u];
      const int rj = L.r[j];
      const double* M = L.m2l[u];
      const double* yj = y + L.yoff[j] * nrhs;
      for (int t = 0; t < rj; t++) s = fma(M[c + (size_t)t * r], yj[(size_t)t * nrhs + q], s);
    }
    if (has_parent) {
      const int pi = i >> dim, cpos = i & ((1 << dim) - 1);
      const double* Up = P.U[pi];
      const int np = P.n[pi], rp = P.r[pi];
      const int64_t ro = P.child_off[(size_t)pi * ((1 << dim) + 1) + cpos];
      const double* zp = zpar + P.yoff[pi] * nrhs;
      for (int t = 0; t < rp; t++) s = fma(Up[ro + c + (size_t)t * np], zp[(size_t)t * nrhs + q], s);
    }
    zi[(size_t)c * nrhs + q] = s;
  }
}

__global__ void __launch_bounds__(256) mv_leaf_kernel(MvLevelDev L, const int* nbr_off, const int* nbr,
                                                      const int* grid, int dim, int win, const double* x,
                                                      const double* z, double* out, int nrhs) {
  const int i = blockIdx.x;
  const int n = L.n[i], r = L.r[i];
  const double* U = L.U[i];
  const double* zi = z + L.yoff[i] * nrhs;
  for (int e = threadIdx.x; e < n * nrhs; e += blockDim.x) {
    const int a = e / nrhs, q = e % nrhs;
    double s = 0.0;
    for (int t = 0; t < r; t++) s = fma(U[a + (size_t)t * n], zi[(size_t)t * nrhs + q], s);
    for (int u = nbr_off[i]; u < nbr_off[i + 1]; u++) {
      const int j = nbr[u];
      const int nj = L.n[j];
      const double* xj = x + L.xoff[j] * nrhs;
      // window slot of j relative to i (and i relative to j)
      int sij = 0, sji = 0, mul = 1;
      for (int d = 0; d < dim; d++) {
        int dd = grid[j * dim + d] - grid[i * dim + d];
        sij += (dd + 3) * mul;
        sji += (-dd + 3) * mul;
        mul *= 7;
      }
      if (j >= i) {
        const double* B = L.p2p[(size_t)i * win + sij];
        for (int b = 0; b < nj; b++) s = fma(B[a + (size_t)b * n], xj[(size_t)b * nrhs + q], s);
      } else {
        const double* B = L.p2p[(size_t)j * win + sji];
        for (int b = 0; b < nj; b++) s = fma(B[b + (size_t)a * nj], xj[(size_t)b * nrhs + q], s);
      }
    }
    out[(L.xoff[i] + a) * nrhs + q] = s;
  }
}

__global__ void permute_rows_kernel(const double* in, double* out, const int64_t* perm, int64_t n, int nrhs, int inverse) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * nrhs; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = e / nrhs;
    const int q = int(e % nrhs);
    if (!inverse) out[e] = in[perm[p] * nrhs + q];
    else out[perm[p] * nrhs + q] = in[e];
  }
}

void launch_permute(const double* in, double* out, const int64_t* perm, int64_t n, int nrhs, bool inverse, cudaStream_t s) {
  const int64_t tot = n * nrhs;
  permute_rows_kernel<<<int(std::min<int64_t>((tot + 255) / 256, 148 * 32)), 256, 0, s>>>(in, out, perm, n, nrhs,
                                                                                        inverse ? 1 : 0);
  CK_LAUNCH();
}

template <class T>
static T* up(Arena& a, const std::vector<T>& v, cudaStream_t s) {
  T* d = a.alloc_n<T>(std::max<size_t>(1, v.size()));
  if (!v.empty()) CK(cudaMemcpyAsync(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, s));
  return d;
}

static MvCache* build_cache(StoreH* S) {
  TreeH* t = S->tree;
  const int K = t->depth, dim = t->dim;
  cudaStream_t s = S->stream;
  MvCache* C = new MvCache;
  C->lv.resize(K + 1);
  for (int k = 2; k <= K; k++) {
    const InitLevel& L = S->lv[k];
    const Topo& T = t->lv[k];
    MvLevelDev& D = C->lv[k];
    std::vector<const double*> U(L.U.begin(), L.U.end());
    std::vector<int64_t> yoff(L.nc + 1, 0), xoff(L.nc + 1, 0);
    for (int i = 0; i < L.nc; i++) {
      yoff[i + 1] = yoff[i] + L.r0[i];
      xoff[i + 1] = xoff[i] + L.n[i];
    }
    D.ysize = yoff[L.nc];
    std::vector<const double*> m2l(L.m2l.begin(), L.m2l.end());
    std::vector<int> ilo(T.il_off.begin(), T.il_off.end());
    D.U = up(C->arena, U, s);
    D.n = up(C->arena, L.n, s);
    D.r = up(C->arena, L.r0, s);
    D.yoff = up(C->arena, yoff, s);
    D.xoff = up(C->arena, xoff, s);
    D.m2l = up(C->arena, m2l, s);
    D.il_off = up(C->arena, ilo, s);
    D.il = up(C->arena, T.il, s);
    if (k < K) D.child_off = up(C->arena, L.child_off, s);
    if (k == K) {
      std::vector<const double*> pp(S->leaf_p2p.begin(), S->leaf_p2p.end());
      D.p2p = up(C->arena, pp, s);
    }
  }
  CK(cudaStreamSynchronize(s));
  return C;
}

// one cache per store (kept alive with the store via a static registry)
static std::mutex g_mv_mu;
static std::map<StoreH*, std::unique_ptr<MvCache>> g_mv;

void matvec_release(StoreH* S) {
  std::lock_guard<std::mutex> g(g_mv_mu);
  g_mv.erase(S);
}

void matvec(StoreH* S, const double* x_in, double* y_out, int64_t nrhs, bool device_ptr) {
  TreeH* t = S->tree;
  const int K = t->depth, dim = t->dim;
  const int64_t N = t->N;
  if (nrhs < 1) invalid("nrhs must be >= 1");
  MvCache* C;
  {
    std::lock_guard<std::mutex> g(g_mv_mu);
    auto it = g_mv.find(S);
    if (it == g_mv.end()) it = g_mv.emplace(S, std::unique_ptr<MvCache>(build_cache(S))).first;
    C = it->second.get();
  }
  cudaStream_t s = S->stream;
  Arena ws(size_t(64) << 20);
  const int nr = int(nrhs);
  double* dx = nullptr;
  double* dy = nullptr;
  if (device_ptr) {
    dx = const_cast<double*>(x_in);
    dy = y_out;
  } else {
    dx = ws.alloc_n<double>(N * nr);
    dy = ws.alloc_n<double>(N * nr);
    CK(cudaMemcpyAsync(dx, x_in, sizeof(double) * N * nr, cudaMemcpyHostToDevice, s));
  }
  double* xp = ws.alloc_n<double>(N * nr);
  double* outp = ws.alloc_n<double>(N * nr);
  launch_permute(dx, xp, t->d_perm, N, nr, false, s);
  std::vector<double*> Y(K + 2, nullptr), Z(K + 2, nullptr);
  for (int k = 2; k <= K; k++) {
    Y[k] = ws.alloc_n<double>(std::max<int64_t>(1, C->lv[k].ysize) * nr);
    Z[k] = ws.alloc_n<double>(std::max<int64_t>(1, C->lv[k].ysize) * nr);
  }
  for (int k = K; k >= 2; k--) {
    const double* in = (k == K) ? xp : Y[k + 1];
    mv_up_kernel<<<t->lv[k].nc, 256, 0, s>>>(C->lv[k], in, Y[k], nr);
    CK_LAUNCH();
  }
  for (int k = 2; k <= K; k++) {
    mv_down_kernel<<<t->lv[k].nc, 256, 0, s>>>(C->lv[k], k > 2 ? C->lv[k - 1] : C->lv[k], k > 2 ? 1 : 0, dim, Y[k],
                                               Z[k], k > 2 ? Z[k - 1] : nullptr, nr);
    CK_LAUNCH();
  }
  {
    const Topo& T = t->lv[K];
    int* d_no = up(ws, T.nbr_off, s);
    int* d_nb = up(ws, T.nbr, s);
    int* d_g = up(ws, T.grid, s);
    mv_leaf_kernel<<<T.nc, 256, 0, s>>>(C->lv[K], d_no, d_nb, d_g, dim, T.win(), xp, Z[K], outp, nr);
    CK_LAUNCH();
  }
  launch_permute(outp, dy, t->d_perm, N, nr, true, s);
  if (!device_ptr) CK(cudaMemcpyAsync(y_out, dy, sizeof(double) * N * nr, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
}

}  // namespace ifmm
