// Rank-growth control (the reference's unused
// _maybe_consolidate, ifmm/solver.py:437-492, made to work).
//
// Fill compression only ever appends directions to a live cluster's basis, so
// ranks creep toward the particle dimension.  Right before cluster q is
// eliminated its basis is final: every reference to its multipoles / locals
// (its M2L blocks and the rows of its parent's basis -- a live cluster has no
// other couplings of rank dimension) is gathered into one coupling row
// Rw (r x W), re-truncated jointly at rank_tol relative to its largest
// singular value, and the basis rotated onto the surviving directions T:
//   U_q <- U_q T,  M2L(q, l) <- T^T M2L(q, l),  parent rows <- T^T rows.
// q's elimination then runs with m = n + r' and its parent sees r' particles
// for it.  The solve is unchanged (the rotation happens before any record
// refers to q's multipoles).
//
// Per batch: G = Rw Rw^T for every pivot (grouped DMMA GEMM); one CTA per pivot
// runs a pivoted Cholesky G ~= L L^T (the Gram form of a column-pivoted QR of
// Rw^T), stopped at the first remaining diagonal below rank_tol^2 times the
// largest one, and takes T = the orthonormal factor of the r x r' matrix L
// (Householder), zero-padded to r x r;  ||(I - T T^T) Rw||_F <= sqrt(r - r')
// rank_tol max_i ||Rw(i, :)||.  Rw2 = T^T Rw (rows beyond r' come out zero) and
// U2 = U T follow as grouped GEMMs; the caller's copy batch scatters them back.
// The Gram matrix resolves diagonals down to ~1e-16 of the largest, so rank_tol
// is effective down to ~3e-8.
#include "consolidate.cuh"

#include "cta_la.cuh"
#include "gemm.cuh"

namespace ifmm {

namespace {

__global__ void __launch_bounds__(1024, 1)
    consolidate_kernel(const ConsDesc* __restrict__ descs, double rank_tol, int* __restrict__ d_rank,
                       int* __restrict__ newrank) {
  __shared__ CtaShared sh;
  __shared__ int s_rn;
  const CtaGroup g{sh};
  const ConsDesc D = descs[blockIdx.x];
  const int r = D.r;
  const double* G = D.G;                   // r x r
  double* T = D.T;                         // r x r out
  double* L = D.scratch;                   // r x r: Cholesky columns, then the Householder reflectors
  double* R = L + (size_t)r * r;           // r x r
  double* d = R + (size_t)r * r;           // r: remaining diagonal
  double* vv = d + r;                      // r
  int* used = reinterpret_cast<int*>(vv + r);  // r ints
  for (int i = threadIdx.x; i < r; i += blockDim.x) {
    d[i] = G[i + (size_t)i * r];
    used[i] = 0;
  }
  __syncthreads();
  int rc = 0;
  double cut = 0.0;
  for (int j = 0; j < r; j++) {
    ArgMax am{-1.0, -1};
    for (int i = threadIdx.x; i < r; i += blockDim.x)
      if (!used[i]) am = argmax_merge(am, ArgMax{fmax(d[i], 0.0), i});
    am = g.argmax(am);
    if (j == 0) cut = rank_tol * rank_tol * am.a;
    if (am.i < 0 || !(am.a > cut) || am.a <= 0.0) break;
    const int p = am.i;
    const double piv = sqrt(am.a);
    for (int i = threadIdx.x; i < r; i += blockDim.x) {
      double v = 0.0;
      if (i == p) {
        v = piv;
        used[i] = 1;
      } else if (!used[i]) {
        v = G[i + (size_t)p * r];
        for (int t = 0; t < j; t++) v = fma(-L[i + (size_t)t * r], L[p + (size_t)t * r], v);
        v /= piv;
        d[i] -= v * v;
      }
      L[i + (size_t)j * r] = v;
    }
    __syncthreads();
    rc++;
  }
  if (threadIdx.x == 0) {
    const int rn = rc > 0 ? rc : r;  // an all-zero row: nothing to decide
    s_rn = rn;
    newrank[blockIdx.x] = rn;
    if (rn < r) d_rank[D.cluster] = rn;
  }
  __syncthreads();
  const int rn = s_rn;
  if (rn >= r) {  // nothing to drop: T = I
    for (int e = threadIdx.x; e < r * r; e += blockDim.x) T[e] = (e % r == e / r) ? 1.0 : 0.0;
    return;
  }
  g_qr(g, L, r, rn, r, R, T, r, vv);  // T(:, :rn): orthonormal basis of span(L)
  for (int e = r * rn + threadIdx.x; e < r * r; e += blockDim.x) T[e] = 0.0;
}

}  // namespace

void launch_consolidate(std::vector<ConsDesc>& h, double rank_tol, int* d_rank, int* d_newrank, Arena& ws,
                        Staging& st, cudaStream_t s, int shape_maxr) {
  if (h.empty()) return;
  int maxr = std::max(1, shape_maxr);
  GemmBatch gram, rot, bas;
  for (ConsDesc& D : h) {
    maxr = std::max(maxr, D.r);
    const size_t rr = size_t(D.r) * D.r;
    D.G = ws.alloc_n<double>(rr);
    D.T = ws.alloc_n<double>(rr);
    D.scratch = ws.alloc_n<double>(2 * rr + 3 * size_t(D.r) + 8);
    D.U2 = ws.alloc_n<double>(size_t(D.n) * D.r);
    // G = Rw Rw^T;  Rw2 = T^T Rw;  U2 = U T
    gram.add(D.row, D.r, D.row, D.r, D.G, D.r, D.r, D.r, D.W, 1.0, 0.0);
    rot.add(D.T, D.r, D.row, D.r, D.row2, D.r, D.r, D.W, D.r, 1.0, 0.0);
    bas.add(D.U, D.n, D.T, D.r, D.U2, D.n, D.n, D.r, D.r, 1.0, 0.0);
  }
  const ConsDesc* dd = upload(ws, h, s, st);
  launch_grouped_gemm(gram, false, true, ws, st, s);
  const int threads = maxr <= 64 ? 128 : maxr <= 128 ? 256 : 512;
  consolidate_kernel<<<unsigned(h.size()), threads, 0, s>>>(dd, rank_tol, d_rank, d_newrank);
  CK_LAUNCH();
  launch_grouped_gemm(rot, true, false, ws, st, s);
  launch_grouped_gemm(bas, false, false, ws, st, s);
}

}  // namespace ifmm
