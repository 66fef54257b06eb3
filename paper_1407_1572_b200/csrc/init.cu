// Assembly of the initial extended system on the GPU (ifmm/operators.py:145-274):
//  * leaf near-field P2P blocks (unit diagonal on self blocks), one orientation;
//  * Chebyshev bases level by level: far-field row K(nodes_i, nodes_IL) ->
//    Householder R -> one-sided Jacobi -> truncated left singular vectors;
//    candidate B U_keep -> Jacobi -> orthonormal basis (1e-14 cut); raw rows
//    U^T B feed the parent through the child transfer matrices;
//  * M2L_ij = raw_i K(nodes_i, nodes_j) raw_j^T for interaction-list pairs;
//  * exact mode (tol == 0): identity bases and dense far blocks.
#include <algorithm>
#include <cmath>

#include "compress.cuh"
#include "core.cuh"
#include "cta_la.cuh"

namespace ifmm {

// ---------------------------------------------------------------- near field
struct KBlockDesc {
  int64_t lo_i, lo_j;
  int ni, nj;
  double* out;  // ni x nj, ld ni
  int diag;     // write unit diagonal (self block)
};

__global__ void __launch_bounds__(256) kblock_kernel(const KBlockDesc* __restrict__ desc, const double* pts, int dim,
                                                     KernelParams kp) {
  const KBlockDesc D = desc[blockIdx.x];
  const int tot = D.ni * D.nj;
  for (int e = threadIdx.x + blockIdx.y * blockDim.x; e < tot; e += blockDim.x * gridDim.y) {
    const int a = e % D.ni, b = e / D.ni;
    double v;
    if (D.diag && a == b) {
      v = 1.0;
    } else {
      const double r = dist_rn(pts + (D.lo_i + a) * dim, pts + (D.lo_j + b) * dim, dim);
      v = keval(kp, r);
    }
    D.out[a + (size_t)b * D.ni] = v;
  }
}

static void launch_kblocks(std::vector<KBlockDesc>& v, const double* pts, int dim, const KernelParams& kp, Arena& ws,
                           Staging& st, cudaStream_t s) {
  if (v.empty()) return;
  const KBlockDesc* d = upload(ws, v, s, st);
  int64_t maxe = 0;
  for (auto& x : v) maxe = std::max<int64_t>(maxe, int64_t(x.ni) * x.nj);
  int gy = int(std::min<int64_t>(64, std::max<int64_t>(1, maxe / 4096)));
  for (size_t off = 0; off < v.size(); off += 65535u * 1024u) {
    unsigned g = unsigned(std::min<size_t>(v.size() - off, 65535u * 1024u));
    kblock_kernel<<<dim3(g, gy), 256, 0, s>>>(d + off, pts, dim, kp);
    CK_LAUNCH();
  }
  v.clear();
}

// ---------------------------------------------------------------- Chebyshev helpers
struct ChebConst {
  int p, nd, dim;
  double n1[16];
};

__device__ inline void node_coord(const ChebConst& C, const double* center, double half, int a, double* out) {
  // tensor grid, first coordinate slowest (ifmm/lowrank.py:77-82)
  int idx[3];
  int t = a;
  for (int d = C.dim - 1; d >= 0; d--) {
    idx[d] = t % C.p;
    t /= C.p;
  }
  for (int d = 0; d < C.dim; d++) out[d] = center[d] + half * C.n1[idx[d]];
}

__device__ inline void cluster_center(int level, const int* grid, int dim, double* c, double* half) {
  const double w = 2.0 / double(1 << level);
  for (int d = 0; d < dim; d++) c[d] = -1.0 + (double(grid[d]) + 0.5) * w;
  *half = w / 2.0;
}

// Lagrange cardinal functions at x (ifmm/lowrank.py:61-74), product form.
__device__ inline double lagrange1(const ChebConst& C, double x, int j) {
  double L = 1.0;
  for (int m = 0; m < C.p; m++)
    if (m != j) L = __dmul_rn(L, __ddiv_rn(__dsub_rn(x, C.n1[m]), __dsub_rn(C.n1[j], C.n1[m])));
  return L;
}

// Interpolation matrix entry: point x (dim) in box (center, half), node a.
__device__ inline double tinterp_entry(const ChebConst& C, const double* x, const double* center, double half, int a) {
  int idx[3];
  int t = a;
  for (int d = C.dim - 1; d >= 0; d--) {
    idx[d] = t % C.p;
    t /= C.p;
  }
  double v = 1.0;
  for (int d = 0; d < C.dim; d++) {
    double L = lagrange1(C, __ddiv_rn(__dsub_rn(x[d], center[d]), half), idx[d]);
    v = d == 0 ? L : __dmul_rn(v, L);
  }
  return v;
}

struct BasisDesc {
  int level, idx;
  int n;                 // particle dim
  int64_t lo;            // leaf: first permuted point
  const int* il;         // interaction list (device)
  int nil;
  const double* child_raw[8];  // non-leaf: child raw rows (r_c x nd, ld r_c)
  int child_r[8];
  double* U;             // out: n x min(n,nd) capacity, ld n
  double* raw;           // out: r x nd, ld r (capacity min(n, nd) x nd)
  int* rank;             // out
  double* scratch;
};

// One CTA per cluster.
__global__ void __launch_bounds__(256) cheb_basis_kernel(const BasisDesc* __restrict__ desc, ChebConst C,
                                                         KernelParams kp, const double* pts, const int* grid_all,
                                                         const double* transfers, double tol) {
  __shared__ CtaShared sh;
  const BasisDesc D = desc[blockIdx.x];
  const int nd = C.nd, dim = C.dim;
  double ci[3], half;
  cluster_center(D.level, grid_all + D.idx * dim, dim, ci, &half);
  const int M = D.nil * nd;
  const int rcap = min(D.n, nd);
  // scratch carve
  double* rowT = D.scratch;                  // M x nd
  double* R = rowT + (size_t)max(M, 1) * nd;   // nd x nd
  double* X = R + nd * nd;                   // nd x nd
  double* B = X + nd * nd;                   // n x nd
  double* cand = B + (size_t)D.n * nd;       // n x nd
  double* sig = cand + (size_t)D.n * nd;     // nd
  double* vv = sig + nd;                     // nd
  int* ord = reinterpret_cast<int*>(vv + nd);  // nd ints
  // far-field row, transposed: rowT[(jj*nd + b), a] = K(node_i[a], node_j[b])
  for (int e = threadIdx.x; e < M * nd; e += blockDim.x) {
    const int rr = e % M, a = e / M;
    const int jj = rr / nd, b = rr % nd;
    const int j = D.il[jj];
    double cj[3], hj, xa[3], xb[3];
    cluster_center(D.level, grid_all + j * dim, dim, cj, &hj);
    node_coord(C, ci, half, a, xa);
    node_coord(C, cj, hj, b, xb);
    rowT[rr + (size_t)a * M] = keval(kp, dist_rn(xa, xb, dim));
  }
  __syncthreads();
  int keep = 0;
  if (M > 0) {
    cta_qr(rowT, M, nd, M, R, nullptr, 0, vv, sh);
    // X = R^T ; Jacobi on X -> X V = U S, U = left singular vectors of the row
    for (int e = threadIdx.x; e < nd * nd; e += blockDim.x) {
      const int i = e % nd, j = e / nd;
      X[i + j * nd] = R[j + i * nd];
    }
    __syncthreads();
    cta_jacobi(X, nd, nd, nd, nullptr, 0, sig, ord, sh);
    const double s0 = sig[ord[0]];
    int cnt = 0;
    for (int t = 0; t < nd; t++) cnt += (sig[t] >= s0 * tol);
    keep = min(min(cnt, D.n), nd);
    if (s0 == 0.0) keep = 0;
  }
  // interpolation matrix B (n x nd)
  const int nch = 1 << dim;
  if (D.child_raw[0] == nullptr) {  // leaf
    for (int e = threadIdx.x; e < D.n * nd; e += blockDim.x) {
      const int i = e % D.n, a = e / D.n;
      B[i + (size_t)a * D.n] = tinterp_entry(C, pts + (D.lo + i) * dim, ci, half, a);
    }
  } else {  // stacked child raw rows times transfer matrices
    int off = 0;
    for (int c = 0; c < nch; c++) {
      const int rc = D.child_r[c];
      const double* Tc = transfers + (size_t)c * nd * nd;  // nd x nd, ld nd (rows child nodes)
      const double* Rc = D.child_raw[c];                    // rc x nd, ld min(n_c, nd) -> stored ld rc
      for (int e = threadIdx.x; e < rc * nd; e += blockDim.x) {
        const int i = e % rc, a = e / rc;
        double s = 0.0;
        for (int t = 0; t < nd; t++) s = fma(Rc[i + (size_t)t * rc], Tc[t + (size_t)a * nd], s);
        B[off + i + (size_t)a * D.n] = s;
      }
      off += rc;
    }
  }
  __syncthreads();
  // cand = B U_keep, U_keep = normalized X columns in decreasing order
  for (int e = threadIdx.x; e < D.n * keep; e += blockDim.x) {
    const int i = e % D.n, c = e / D.n;
    const int col = ord[c];
    const double inv = 1.0 / sig[col];
    double s = 0.0;
    for (int t = 0; t < nd; t++) s = fma(B[i + (size_t)t * D.n], X[t + col * nd] * inv, s);
    cand[i + (size_t)c * D.n] = s;
  }
  __syncthreads();
  int r = 0;
  if (keep > 0) {
    cta_jacobi(cand, D.n, keep, D.n, nullptr, 0, sig, ord, sh);
    const double s0 = sig[ord[0]];
    for (int t = 0; t < keep; t++) r += (s0 > 0.0 && sig[t] >= s0 * 1e-14);
  }
  r = min(r, rcap);
  for (int e = threadIdx.x; e < D.n * r; e += blockDim.x) {
    const int i = e % D.n, c = e / D.n;
    const int col = ord[c];
    D.U[i + (size_t)c * D.n] = cand[i + (size_t)col * D.n] / sig[col];
  }
  __syncthreads();
  // raw = U^T B  (r x nd, ld r)
  for (int e = threadIdx.x; e < r * nd; e += blockDim.x) {
    const int c = e % r, a = e / r;
    double s = 0.0;
    for (int t = 0; t < D.n; t++) s = fma(D.U[t + (size_t)c * D.n], B[t + (size_t)a * D.n], s);
    D.raw[c + (size_t)a * r] = s;
  }
  if (threadIdx.x == 0) *D.rank = r;
}

struct M2LDesc {
  int level, i, j;
  const double* raw_i;  // ri x nd (ld ri)
  const double* raw_j;  // rj x nd (ld rj)
  int ri, rj;
  double* out_ij;       // ri x rj (ld ri)
  double* out_ji;       // rj x ri (ld rj)
};

__global__ void __launch_bounds__(256) cheb_m2l_kernel(const M2LDesc* __restrict__ desc, ChebConst C, KernelParams kp,
                                                       const int* grid_all) {
  extern __shared__ double sm[];
  const M2LDesc D = desc[blockIdx.x];
  const int nd = C.nd, dim = C.dim;
  double* Kb = sm;             // nd x nd
  double* T = Kb + nd * nd;    // ri x nd
  double ci[3], cj[3], hi, hj;
  cluster_center(D.level, grid_all + D.i * dim, dim, ci, &hi);
  cluster_center(D.level, grid_all + D.j * dim, dim, cj, &hj);
  for (int e = threadIdx.x; e < nd * nd; e += blockDim.x) {
    const int a = e % nd, b = e / nd;
    double xa[3], xb[3];
    node_coord(C, ci, hi, a, xa);
    node_coord(C, cj, hj, b, xb);
    Kb[a + b * nd] = keval(kp, dist_rn(xa, xb, dim));
  }
  __syncthreads();
  for (int e = threadIdx.x; e < D.ri * nd; e += blockDim.x) {
    const int a = e % D.ri, b = e / D.ri;
    double s = 0.0;
    for (int t = 0; t < nd; t++) s = fma(D.raw_i[a + (size_t)t * D.ri], Kb[t + b * nd], s);
    T[a + (size_t)b * D.ri] = s;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < D.ri * D.rj; e += blockDim.x) {
    const int a = e % D.ri, b = e / D.ri;
    double s = 0.0;
    for (int t = 0; t < nd; t++) s = fma(T[a + (size_t)t * D.ri], D.raw_j[b + (size_t)t * D.rj], s);
    D.out_ij[a + (size_t)b * D.ri] = s;
    D.out_ji[b + (size_t)a * D.rj] = s;
  }
}

// host replica of ifmm/operators.py:145-161 (child transfer matrices)
static std::vector<double> child_transfers(int dim, int p, const std::vector<double>& n1) {
  int nd = 1;
  for (int d = 0; d < dim; d++) nd *= p;
  std::vector<double> out(size_t(1 << dim) * nd * nd);
  auto lag = [&](double x, int j) {
    double L = 1.0;
    for (int m = 0; m < p; m++)
      if (m != j) L = L * ((x - n1[m]) / (n1[j] - n1[m]));
    return L;
  };
  for (int c = 0; c < (1 << dim); c++) {
    for (int a = 0; a < nd; a++) {      // child node (row)
      int ia[3], t = a;
      for (int d = dim - 1; d >= 0; d--) { ia[d] = t % p; t /= p; }
      double x[3];
      for (int d = 0; d < dim; d++) {
        double off = double((c >> d) & 1) - 0.5;
        x[d] = off + 0.5 * n1[ia[d]];
      }
      for (int b = 0; b < nd; b++) {    // parent node (col)
        int ib[3], tt = b;
        for (int d = dim - 1; d >= 0; d--) { ib[d] = tt % p; tt /= p; }
        double v = 1.0;
        for (int d = 0; d < dim; d++) {
          double L = lag((x[d] - 0.0) / 1.0, ib[d]);
          v = d == 0 ? L : v * L;
        }
        out[size_t(c) * nd * nd + a + size_t(b) * nd] = v;
      }
    }
  }
  return out;
}

StoreH* store_init(TreeH* t, const KernelParams& kp, int p, double tol, const int* probe_tab, int probe_maxm) {
  ensure_device();
  if (kp.id < 0 || kp.id >= K_COUNT) invalid("unknown kernel id");
  if (tol < 0) invalid("tol must be >= 0");
  if (tol > 0 && (p < 2 || p > 9)) invalid("Chebyshev order p must be in [2, 9]");
  std::unique_ptr<StoreH> S(new StoreH);
  S->tree = t;
  S->kp = kp;
  S->p = p;
  S->tol = tol;
  S->stream = default_stream();
  cudaStream_t s = S->stream;
  Arena ws(size_t(256) << 20);
  Staging st;
  const int dim = t->dim, K = t->depth;
  S->probe_tab.assign(probe_tab, probe_tab + size_t(probe_maxm + 1) * ACA_PROBE_STRIDE);
  S->probe_maxm = probe_maxm;
  S->d_probe = S->arena.alloc_n<int>(S->probe_tab.size());
  CK(cudaMemcpyAsync(S->d_probe, S->probe_tab.data(), sizeof(int) * S->probe_tab.size(), cudaMemcpyHostToDevice, s));
  S->lv.assign(K + 1, InitLevel{});
  // device topology (grid coords and IL CSR per level)
  std::vector<int*> d_grid(K + 1, nullptr), d_il(K + 1, nullptr);
  for (int k = 1; k <= K; k++) {
    d_grid[k] = upload(ws, t->lv[k].grid, s, st);
    d_il[k] = upload(ws, t->lv[k].il, s, st);
  }
  std::vector<KBlockDesc> kb;
  if (tol == 0.0) {
    // exact mode: identity bases, dense kernel far blocks (ifmm/operators.py:197-216)
    for (int k = K; k >= 2; k--) {
      InitLevel& L = S->lv[k];
      const Topo& T = t->lv[k];
      L.k = k;
      L.nc = T.nc;
      L.n.resize(T.nc);
      L.r0.resize(T.nc);
      L.U.resize(T.nc);
      CopyBatch eye;
      for (int i = 0; i < T.nc; i++) {
        int n = int(t->range_hi(k, i) - t->range_lo(k, i));
        L.n[i] = L.r0[i] = n;
        L.U[i] = S->arena.alloc_n<double>(size_t(n) * n);
        S->max_init_rank = std::max(S->max_init_rank, 0);
      }
      // identity via zero + diagonal kernel
      for (int i = 0; i < T.nc; i++) CK(cudaMemsetAsync(L.U[i], 0, sizeof(double) * L.n[i] * L.n[i], s));
      std::vector<double> one(1, 1.0);
      double* d_one = upload(ws, one, s, st);
      for (int i = 0; i < T.nc; i++) eye.add(d_one, 0, L.U[i], L.n[i] + 1, 1, L.n[i]);
      launch_copies(eye, ws, st, s);
      L.m2l_off.assign(1, 0);
      for (int i = 0; i < T.nc; i++) {
        for (int q = T.il_off[i]; q < T.il_off[i + 1]; q++) {
          int j = T.il[q];
          double* blk = S->arena.alloc_n<double>(size_t(L.n[i]) * L.n[j]);
          L.m2l.push_back(blk);
          kb.push_back(KBlockDesc{t->range_lo(k, i), t->range_lo(k, j), L.n[i], L.n[j], blk, 0});
        }
        L.m2l_off.push_back(int64_t(L.m2l.size()));
      }
      launch_kblocks(kb, t->d_pts, dim, kp, ws, st, s);
    }
  } else {
    ChebConst C{};
    C.p = p;
    C.dim = dim;
    C.nd = 1;
    for (int d = 0; d < dim; d++) C.nd *= p;
    std::vector<double> n1(p);
    for (int j = 0; j < p; j++) n1[j] = -std::cos((2.0 * j + 1.0) * M_PI / (2.0 * p));
    for (int j = 0; j < p; j++) C.n1[j] = n1[j];
    const int nd = C.nd;
    std::vector<double> tr = child_transfers(dim, p, n1);
    double* d_tr = upload(ws, tr, s, st);
    std::vector<std::vector<double*>> raw(K + 2);
    std::vector<std::vector<int>> rnk(K + 2);
    Arena raw_arena[2] = {Arena(size_t(128) << 20), Arena(size_t(128) << 20)};
    CK(cudaFuncSetAttribute(cheb_m2l_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    for (int k = K; k >= 2; k--) {
      InitLevel& L = S->lv[k];
      const Topo& T = t->lv[k];
      L.k = k;
      L.nc = T.nc;
      L.n.resize(T.nc);
      L.r0.resize(T.nc);
      L.U.resize(T.nc);
      raw[k].resize(T.nc);
      Arena& ra = raw_arena[k & 1];
      ra.reset();
      for (int i = 0; i < T.nc; i++) {
        if (k == K) L.n[i] = int(t->leaf_off[i + 1] - t->leaf_off[i]);
        else {
          int n = 0;
          for (int c = 0; c < (1 << dim); c++) n += rnk[k + 1][(i << dim) + c];
          L.n[i] = n;
        }
        const int cap = std::min(L.n[i], nd);
        L.U[i] = S->arena.alloc_n<double>(size_t(std::max(1, L.n[i])) * std::max(1, cap));
        raw[k][i] = ra.alloc_n<double>(size_t(std::max(1, cap)) * nd);
      }
      int* d_rank = ws.alloc_n<int>(T.nc);
      // chunk the clusters to bound scratch
      size_t per_max = 0;
      for (int i = 0; i < T.nc; i++) {
        int nil = T.il_off[i + 1] - T.il_off[i];
        size_t per = size_t(std::max(1, nil * nd)) * nd + 2 * nd * nd + 2 * size_t(L.n[i]) * nd + 3 * nd + 64;
        per_max = std::max(per_max, per);
      }
      int chunk = int(std::max<size_t>(1, std::min<size_t>(T.nc, (size_t(2) << 30) / (per_max * 8))));
      for (int c0 = 0; c0 < T.nc; c0 += chunk) {
        int c1 = std::min(T.nc, c0 + chunk);
        std::vector<BasisDesc> bd(c1 - c0);
        double* scr = ws.alloc_n<double>(per_max * (c1 - c0));
        for (int i = c0; i < c1; i++) {
          BasisDesc& D = bd[i - c0];
          memset(&D, 0, sizeof D);
          D.level = k;
          D.idx = i;
          D.n = L.n[i];
          D.lo = t->leaf_off[size_t(i) << (dim * (K - k))];
          D.il = d_il[k] + T.il_off[i];
          D.nil = T.il_off[i + 1] - T.il_off[i];
          if (k < K)
            for (int c = 0; c < (1 << dim); c++) {
              D.child_raw[c] = raw[k + 1][(i << dim) + c];
              D.child_r[c] = rnk[k + 1][(i << dim) + c];
            }
          D.U = L.U[i];
          D.raw = raw[k][i];
          D.rank = d_rank + i;
          D.scratch = scr + per_max * (i - c0);
        }
        const BasisDesc* dbd = upload(ws, bd, s, st);
        cheb_basis_kernel<<<c1 - c0, 256, 0, s>>>(dbd, C, kp, t->d_pts, d_grid[k], d_tr, tol);
        CK_LAUNCH();
        CK(cudaStreamSynchronize(s));
        st.reset();
      }
      rnk[k].resize(T.nc);
      CK(cudaMemcpyAsync(rnk[k].data(), d_rank, sizeof(int) * T.nc, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      for (int i = 0; i < T.nc; i++) {
        L.r0[i] = rnk[k][i];
        S->max_init_rank = std::max(S->max_init_rank, L.r0[i]);
      }
      // M2L on interaction-list pairs (both orientations stored)
      L.m2l_off.assign(1, 0);
      std::vector<int64_t> pos(T.il.size());
      for (int i = 0; i < T.nc; i++) {
        for (int q = T.il_off[i]; q < T.il_off[i + 1]; q++) {
          int j = T.il[q];
          L.m2l.push_back(S->arena.alloc_n<double>(size_t(std::max(1, L.r0[i])) * std::max(1, L.r0[j])));
        }
        L.m2l_off.push_back(int64_t(L.m2l.size()));
      }
      std::vector<M2LDesc> md;
      for (int i = 0; i < T.nc; i++)
        for (int q = T.il_off[i]; q < T.il_off[i + 1]; q++) {
          int j = T.il[q];
          if (j < i) continue;
          int qj = -1;
          for (int u = T.il_off[j]; u < T.il_off[j + 1]; u++)
            if (T.il[u] == i) qj = u;
          md.push_back(M2LDesc{k, i, j, raw[k][i], raw[k][j], L.r0[i], L.r0[j], L.m2l[q], L.m2l[qj]});
        }
      if (!md.empty()) {
        const M2LDesc* dmd = upload(ws, md, s, st);
        size_t smem = size_t(nd) * nd * 8 + size_t(nd) * nd * 8;
        cheb_m2l_kernel<<<unsigned(md.size()), 256, smem, s>>>(dmd, C, kp, d_grid[k]);
        CK_LAUNCH();
      }
      CK(cudaStreamSynchronize(s));
      st.reset();
    }
  }
  // leaf near field, one orientation (j >= i)
  {
    const Topo& T = t->lv[K];
    const int W = T.win();
    S->leaf_p2p.assign(size_t(T.nc) * W, nullptr);
    for (int i = 0; i < T.nc; i++) {
      const int ni = int(t->leaf_off[i + 1] - t->leaf_off[i]);
      for (int q = T.nbr_off[i]; q < T.nbr_off[i + 1]; q++) {
        int j = T.nbr[q];
        if (j < i) continue;
        const int nj = int(t->leaf_off[j + 1] - t->leaf_off[j]);
        double* blk = S->arena.alloc_n<double>(size_t(ni) * nj);
        S->leaf_p2p[size_t(i) * W + T.slot(i, j)] = blk;
        kb.push_back(KBlockDesc{t->leaf_off[i], t->leaf_off[j], ni, nj, blk, j == i});
      }
    }
    launch_kblocks(kb, t->d_pts, dim, kp, ws, st, s);
  }
  // child offsets (prefix of child initial ranks) for non-leaf levels
  for (int k = 2; k < K; k++) {
    InitLevel& L = S->lv[k];
    L.child_off.resize(size_t(L.nc) * ((1 << dim) + 1));
    for (int i = 0; i < L.nc; i++) {
      int64_t o = 0;
      for (int c = 0; c <= (1 << dim); c++) {
        L.child_off[size_t(i) * ((1 << dim) + 1) + c] = o;
        if (c < (1 << dim)) o += S->lv[k + 1].r0[(i << dim) + c];
      }
    }
  }
  CK(cudaStreamSynchronize(s));
  return S.release();
}

}  // namespace ifmm
