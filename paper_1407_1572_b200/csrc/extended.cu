// The extended sparse system of the initial operator store, materialised by a
// device scatter: the verification / export path of the reference
// (ifmm/operators.py:333-486 -- extended_layout, assemble_extended_dense).
//
// Unknown slots (the reference's order): every leaf contributes (x_i, z_i) in
// Morton order; then, level by level upwards (kappa-1 .. 1), every cluster
// contributes its children's multipole slots y followed by its own local slot
// z (none at level 1).  Equation rows sit at the same positions:
//   x_i rows  particle equations      sum_j P2P_ij x_j + U_i z_i
//   z_i rows  charge lumping          U_i^T (x_i | children's y) - y_i
//   y_i rows  local definition        -z_i + sum_{j in IL(i)} M2L_ij y_j + U_par[slice_i] z_par
// The slot table is built on the host from the store's dimensions; every
// block (P2P, U, U^T, child slices of U, M2L, -I) becomes one descriptor of the
// batched copy kernel writing straight into a column-major device matrix.
#include <algorithm>
#include <string>

#include "batched.cuh"
#include "core.cuh"

namespace ifmm {

namespace {

__global__ void neg_identity_kernel(double* I, int n) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += gridDim.x * blockDim.x)
    I[e] = (e % n == e / n) ? -1.0 : 0.0;
}

}  // namespace

// slot kinds
constexpr int SLOT_X = 0, SLOT_Y = 1, SLOT_Z = 2;

struct ExtLayout {
  std::vector<ExtSlot> slots;
  int64_t dim = 0;
  std::vector<int64_t> ox;                         // leaf x slot offset
  std::vector<std::vector<int64_t>> oy, oz;        // [k][i]
};

static ExtLayout build_layout(const StoreH* S) {
  const TreeH* t = S->tree;
  const int K = t->depth, nch = 1 << t->dim;
  ExtLayout E;
  E.oy.assign(K + 1, {});
  E.oz.assign(K + 1, {});
  for (int k = 1; k <= K; k++) {
    E.oy[k].assign(size_t(1) << (t->dim * k), -1);
    E.oz[k].assign(size_t(1) << (t->dim * k), -1);
  }
  auto push = [&](int sym, int k, int i, int d) {
    E.slots.push_back(ExtSlot{sym, k, i, d});
    const int64_t at = E.dim;
    E.dim += d;
    return at;
  };
  const InitLevel& LK = S->lv[K];
  E.ox.assign(LK.nc, 0);
  for (int i = 0; i < LK.nc; i++) {
    E.ox[i] = push(SLOT_X, K, i, int(t->leaf_off[i + 1] - t->leaf_off[i]));
    E.oz[K][i] = push(SLOT_Z, K, i, LK.r0[i]);
  }
  for (int k = K - 1; k >= 1; k--) {
    const int nc = 1 << (t->dim * k);
    for (int i = 0; i < nc; i++) {
      for (int c = 0; c < nch; c++) {
        const int ch = i * nch + c;
        E.oy[k + 1][ch] = push(SLOT_Y, k + 1, ch, S->lv[k + 1].r0[ch]);
      }
      if (k >= 2) E.oz[k][i] = push(SLOT_Z, k, i, S->lv[k].r0[i]);
    }
  }
  return E;
}

std::vector<ExtSlot> extended_layout(const StoreH* S) { return build_layout(S).slots; }

int64_t extended_dense(StoreH* S, int64_t cap, double* host_out) {
  ExtLayout E = build_layout(S);
  const int64_t m = E.dim;
  if (m > cap) invalid("extended dimension " + std::to_string(m) + " exceeds cap " + std::to_string(cap));
  if (!host_out) return m;
  const TreeH* t = S->tree;
  const int K = t->depth, nch = 1 << t->dim;
  cudaStream_t s = S->stream ? S->stream : default_stream();
  Arena ws(size_t(8) << 20);
  Staging st;
  double* A = ws.alloc_n<double>(size_t(std::max<int64_t>(1, m)) * std::max<int64_t>(1, m));
  CK(cudaMemsetAsync(A, 0, sizeof(double) * size_t(m) * m, s));
  int rmax = 1;
  for (int k = 2; k <= K; k++)
    for (int r : S->lv[k].r0) rmax = std::max(rmax, r);
  double* negI = ws.alloc_n<double>(size_t(rmax) * rmax);
  neg_identity_kernel<<<std::max(1, std::min(1024, (rmax * rmax + 255) / 256)), 256, 0, s>>>(negI, rmax);
  CK_LAUNCH();
  CopyBatch cb;
  auto at = [&](int64_t r, int64_t c) { return A + r + size_t(c) * m; };
  // particle equations: near field and the leaf bases
  {
    const Topo& T = t->lv[K];
    const InitLevel& L = S->lv[K];
    for (int i = 0; i < T.nc; i++) {
      for (int q = T.nbr_off[i]; q < T.nbr_off[i + 1]; q++) {
        const int j = T.nbr[q], a = std::min(i, j), b = std::max(i, j);
        const double* blk = S->leaf_p2p[size_t(a) * T.win() + T.slot(a, b)];
        // stored once as (a, b), n_a x n_b (ld n_a)
        cb.add(blk, L.n[a], at(E.ox[i], E.ox[j]), int(m), L.n[i], L.n[j], i != a);
      }
      cb.add(L.U[i], L.n[i], at(E.ox[i], E.oz[K][i]), int(m), L.n[i], L.r0[i]);
    }
  }
  // charge lumping: U^T onto the particle slots (leaves) or the children's y slots
  for (int k = K; k >= 2; k--) {
    const InitLevel& L = S->lv[k];
    for (int i = 0; i < L.nc; i++) {
      const int r = L.r0[i];
      const int64_t row = E.oz[k][i];
      if (k == K) {
        cb.add(L.U[i], L.n[i], at(row, E.ox[i]), int(m), r, L.n[i], true);
      } else {
        for (int c = 0; c < nch; c++) {
          const int64_t lo = L.child_off[size_t(i) * (nch + 1) + c];
          const int ch = i * nch + c;
          cb.add(L.U[i] + lo, L.n[i], at(row, E.oy[k + 1][ch]), int(m), r, S->lv[k + 1].r0[ch], true);
        }
      }
      cb.add(negI, rmax, at(row, E.oy[k][i]), int(m), r, r, false, 1.0, true);
    }
  }
  // local definitions: -I on z, M2L over the interaction list, the parent's transfer rows
  for (int k = 2; k <= K; k++) {
    const Topo& T = t->lv[k];
    const InitLevel& L = S->lv[k];
    for (int i = 0; i < L.nc; i++) {
      const int r = L.r0[i];
      const int64_t row = E.oy[k][i];
      cb.add(negI, rmax, at(row, E.oz[k][i]), int(m), r, r, false, 1.0, true);
      for (int q = T.il_off[i]; q < T.il_off[i + 1]; q++) {
        const int j = T.il[q];
        cb.add(L.m2l[size_t(L.m2l_off[i] + (q - T.il_off[i]))], r, at(row, E.oy[k][j]), int(m), r, L.r0[j]);
      }
      if (k > 2) {
        const InitLevel& P = S->lv[k - 1];
        const int par = i / nch;
        const int64_t lo = P.child_off[size_t(par) * (nch + 1) + (i % nch)];
        cb.add(P.U[par] + lo, P.n[par], at(row, E.oz[k - 1][par]), int(m), r, P.r0[par]);
      }
    }
  }
  launch_copies(cb, ws, st, s);
  CK(cudaMemcpyAsync(host_out, A, sizeof(double) * size_t(m) * m, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return m;
}

}  // namespace ifmm
