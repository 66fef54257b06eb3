// Batched fill-in compression kernels K1..K4 (see compress.cuh).
#include <algorithm>

#include "compress.cuh"

namespace ifmm {
__device__ int g_prof_on = 0;
__device__ double g_gram_piv = 1e-14;  // K1 Gram route: scaled pivots^2 >= g_gram_piv / tol
__device__ int g_full_rank_ok = 0;  // sparse trees: a full-rank ACA is absorbed, not kept dense
__device__ int g_gram = 1;    // 1: Gram routes (K1 recompression, coarse new directions); 0: Householder QRs
__device__ unsigned long long g_cyc[16];  // debug stage cycle counters (IFMM_PROF)
}  // namespace ifmm
// debug: Jacobi sweep statistics (sweeps, calls, columns) under IFMM_PROF
#define IFMM_JACOBI_STATS(sw, ncol, leader)                       \
  do {                                                            \
    if (g_prof_on && (leader)) {                                  \
      atomicAdd(&g_cyc[8], (unsigned long long)(sw));             \
      atomicAdd(&g_cyc[9], 1ull);                                 \
      atomicAdd(&g_cyc[10], (unsigned long long)(ncol));          \
    }                                                             \
  } while (0)
#include "cta_la.cuh"

namespace ifmm {
#define PROF_T0() long long _pt = g_prof_on ? clock64() : 0
#define PROF_ACC(i) \
  do {                                                                  \
    if (g_prof_on) {                                                    \
      const long long _n = clock64();                                   \
      if (g.rank() == 0) atomicAdd(&g_cyc[i], (unsigned long long)(_n - _pt)); \
      _pt = _n;                                                         \
    }                                                                   \
  } while (0)

constexpr int CTMAX = 512;  // compression CTAs: 128 threads for small fills, 512 at coarse levels
constexpr int WARP_KCAP = 32;  // ACA crosses a warp worker holds; fills needing more are redone by a CTA

// Worker = the group that owns one fill / chain / pivot: a whole CTA, or one
// warp of it (fine levels).  id/count enumerate workers over the grid.
template <class G> struct Worker;
template <> struct Worker<CtaGroup> {
  __device__ static int id() { return blockIdx.x; }
  __device__ static int count() { return gridDim.x; }
  __device__ static CtaGroup make(CtaShared& sh) { return CtaGroup{sh}; }
};
template <> struct Worker<WarpGroup> {
  __device__ static int id() { return blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); }
  __device__ static int count() { return gridDim.x * (blockDim.x >> 5); }
  __device__ static WarpGroup make(CtaShared&) { return WarpGroup{}; }
};

// ------------------------------------------------------------------ Gram recompression
// Column-scaled Cholesky of a k x k Gram matrix G (ld ldg, k <= 96) by ONE
// warp, in place: with d = sqrt(diag(G)) (precomputed by the caller),
// Ghat = G / (d_i d_j) = Lhat Lhat^T; on exit the lower triangle holds Lhat
// (upper triangle zeroed).  Returns false when Ghat is numerically singular
// (pivot^2 <= 1e-12, i.e. cond of the scaled factor > 1e6); the caller then
// falls back to Householder QR.  The result is identical on every lane.
__device__ bool warp_chol_scaled(double* Gm, int k, int ldg, const double* d, double min_piv2 = 1e-12) {
  const int lane = threadIdx.x & 31;
  for (int i = 0; i < k; i++)
    if (!(d[i] > 0.0)) return false;
  for (int e = lane; e < k * k; e += 32) {
    const int i = e % k, j = e / k;
    Gm[i + (size_t)j * ldg] /= d[i] * d[j];
  }
  __syncwarp();
  for (int j = 0; j < k; j++) {
    double t[3];
#pragma unroll
    for (int q = 0; q < 3; q++) {
      const int i = lane + 32 * q;
      double v = 0.0;
      if (i < k && i >= j) {
        v = Gm[i + (size_t)j * ldg];
        for (int p = 0; p < j; p++) v -= Gm[i + (size_t)p * ldg] * Gm[j + (size_t)p * ldg];
      }
      t[q] = v;
    }
    const int qj = j >> 5;
    const double mine = qj == 0 ? t[0] : (qj == 1 ? t[1] : t[2]);
    const double dj = __shfl_sync(0xffffffffu, mine, j & 31);
    if (!(dj > min_piv2)) return false;  // uniform across the warp
    const double piv = sqrt(dj);
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 3; q++) {
      const int i = lane + 32 * q;
      if (i < k && i >= j) Gm[i + (size_t)j * ldg] = (i == j) ? piv : t[q] / piv;
    }
    __syncwarp();
  }
  for (int e = lane; e < k * k; e += 32) {
    const int i = e % k, j = e / k;
    if (i < j) Gm[i + (size_t)j * ldg] = 0.0;
  }
  __syncwarp();
  return true;
}

// Recompression of the ACA crosses F ~= Uc Vc^T through their Gram matrices:
// Gu = Lu Lu^T, Gv = Lv Lv^T (column-scaled Cholesky), core = Lu^T Lv,
// core V = X (one-sided Jacobi), left = Uc Lu^-T X(:, ord), right =
// Vc Lv^-T V(:, ord) -- the same factors as QR(Uc), QR(Vc), SVD(R_u R_v^T)
// (ifmm/lowrank.py:137-171) without the two Householder QRs.  Returns the
// truncated rank, or -1 when a Gram matrix is too ill-conditioned.
template <class G>
__device__ int gram_recompress(const G& g, const double* Uc, const double* Vc, int rows, int cols, int k,
                               double* Gu, double* Gv, int ldg, double* core, double* Jv, double* sig, int* ord,
                               double tol, double* Zl, double* Zr, double* left, double* right, double* sv,
                               double* du, double* dv) {
  const int warp = g.warp(), nw = g.nwarps();
  // diagonal scales (kept: the Cholesky overwrites the Gram in place)
  for (int i = g.rank(); i < k; i += g.size()) {
    du[i] = sqrt(fmax(Gu[i + (size_t)i * ldg], 0.0));
    dv[i] = sqrt(fmax(Gv[i + (size_t)i * ldg], 0.0));
  }
  g.sync();
  bool ok = true;
  if (k > 96) return -1;
  // The factors carry ~eps * cond^2 of the column-scaled crosses: accept the
  // Gram route only while that stays 100x below the truncation tolerance
  // (scaled pivots^2 >= 1e-14 / tol; clustered inputs produce ill-conditioned
  // crosses whose Gram factors otherwise corrupt the augmented bases)
  const double min_piv2 = fmax(1e-12, g_gram_piv / tol);
  if (nw >= 2) {
    if (warp == 0) ok = warp_chol_scaled(Gu, k, ldg, du, min_piv2);
    else if (warp == 1) ok = warp_chol_scaled(Gv, k, ldg, dv, min_piv2);
  } else {
    ok = warp_chol_scaled(Gu, k, ldg, du, min_piv2) && warp_chol_scaled(Gv, k, ldg, dv, min_piv2);
  }
  if (g.any(!ok)) return -1;
  // unscale: L = D^-1 Lhat (row i times the original sqrt(G_ii))
  for (int e = g.rank(); e < k * k; e += g.size()) {
    const int i = e % k, j = e / k;
    Gu[i + (size_t)j * ldg] *= du[i];
    Gv[i + (size_t)j * ldg] *= dv[i];
  }
  g.sync();
  // core = Lu^T Lv (k x k)
  g_gemm(g, k, k, k, 1.0, Gu, ldg, true, Gv, ldg, false, 0.0, core, k);
  g_jacobi(g, core, k, k, k, Jv, k, sig, ord);
  const int r = trunc_rank_dev(sig, ord, k, tol);
  // Zl = Lu^-T X(:, ord[:r]),  Zr = Lv^-T V(:, ord[:r]): one thread per column
  for (int c = g.rank(); c < 2 * r; c += g.size()) {
    const bool isl = c < r;
    const int cc = isl ? c : c - r;
    const double* L = isl ? Gu : Gv;
    const double* B = (isl ? core : Jv) + (size_t)ord[cc] * k;
    double* Z = (isl ? Zl : Zr) + (size_t)cc * k;
    for (int i = k - 1; i >= 0; i--) {  // L^T Z = B, back substitution
      double v = B[i];
      for (int p = i + 1; p < k; p++) v -= L[p + (size_t)i * ldg] * Z[p];
      Z[i] = v / L[i + (size_t)i * ldg];
    }
  }
  g.sync();
  if (r > 0) {
    g_gemm(g, rows, r, k, 1.0, Uc, rows, false, Zl, k, false, 0.0, left, rows);
    g_gemm(g, cols, r, k, 1.0, Vc, cols, false, Zr, k, false, 0.0, right, cols);
  }
  for (int c = g.rank(); c < r; c += g.size()) sv[c] = sig[ord[c]];
  g.sync();
  return r;
}

// ------------------------------------------------------------------ K1
// ACA of the redirected fill, QR of both cross factors, Jacobi SVD of the
// k x k core, truncation (ifmm/lowrank.py:174-263, :137-144).  kcap < Kf
// (warp workers): a fill whose ACA reaches kcap crosses unconverged is marked
// status 2 and redone by the CTA pass (redo = true) with the full Kf.
template <class G>
__global__ void __launch_bounds__(G::kMaxThreads, G::kMinBlocks) aca_recompress_kernel(const FillDesc* __restrict__ fills, int nf,
                                                            FillState* state, double tol, const int* probes,
                                                            int probe_maxm, double* scratch, size_t slot,
                                                            int MR, int MC, int KK, int redo, int phase,
                                                            const int* __restrict__ order = nullptr) {
  __shared__ CtaShared sh;
  const G g = Worker<G>::make(sh);
  double* s = scratch + slot * Worker<G>::id();
  double* Uc = s; s += (size_t)MR * KK;
  double* Ql = s; s += (size_t)MR * KK;
  double* Vc = s; s += (size_t)MC * KK;
  double* Qr = s; s += (size_t)MC * KK;
  double* Rl = s; s += (size_t)KK * KK;
  double* Rr = s; s += (size_t)KK * KK;
  double* core = s; s += (size_t)KK * KK;
  double* Jv = s; s += (size_t)KK * KK;
  double* rr = s; s += MC;
  double* cc = s; s += MR;
  double* dots = s; s += KK;
  double* vv = s; s += KK;
  double* sig = s; s += KK;
  int* usedr = reinterpret_cast<int*>(s); s += MR;
  int* usedc = reinterpret_cast<int*>(s); s += MC;
  int* ord = reinterpret_cast<int*>(s);
  for (int u = Worker<G>::id(); u < nf; u += Worker<G>::count()) {
    const int f = order ? order[u] : u;
    if (redo && state[f].status != 2) continue;
    const FillDesc D = fills[f];
    const int rows = D.rows, cols = D.cols;
    int k;
    FillState S{0, 0, 0, 0, 0, 0.0};
    PROF_T0();
    if (phase == 1) {
      // recompression pass: crosses staged in the output factors by phase 0
      S = state[f];
      if (S.status != 0 || S.r != -1) continue;
      k = S.k;
      const double* gu = D.out + (size_t)rows * k;
      const double* gv = D.out + (size_t)rows * D.Kf + (size_t)cols * k;
      for (int e = g.rank(); e < rows * k; e += g.size()) Uc[e] = D.out[e];
      for (int e = g.rank(); e < cols * k; e += g.size()) Vc[e] = D.out[(size_t)rows * D.Kf + e];
      if (g_gram)
        for (int e = g.rank(); e < k * k; e += g.size()) {
          const int i = e % k, j = e / k;
          Rl[i + (size_t)j * KK] = gu[e];
          Rr[i + (size_t)j * KK] = gv[e];
        }
      g.sync();
    } else {
    if (rows == 0 || cols == 0) {
      if (g.rank() == 0) state[f] = S;
      g.sync();
      continue;
    }
    if (tol == 0.0) {  // exact mode: the redirected fill is F itself (bases are identities)
      double nz = 0.0;
      for (int e = g.rank(); e < rows * cols; e += g.size()) {
        const int a = e % rows, b = e / rows;
        nz += Fat(D.F, D.ldF, D.transF, a, b) != 0.0;
      }
      nz = g.sum(nz);
      S.r = nz > 0.0 ? min(rows, cols) : 0;
      if (g.rank() == 0) state[f] = S;
      g.sync();
      continue;
    }
    const int mrow = rows < probe_maxm ? rows : probe_maxm;
    const int kmax = min(D.Kf, KK);
    if (g_prof_on) _pt = clock64();
    AcaOut ao = g_aca(g, D.F, D.ldF, D.transF, rows, cols, tol, probes + (size_t)mrow * ACA_PROBE_STRIDE, min(10, rows), Uc, Vc,
                      kmax, rr, cc, usedr, usedc, dots, g_gram ? Rl : nullptr, g_gram ? Rr : nullptr, KK);
    PROF_ACC(0);
    k = ao.k;
    S.k = k;
    if (!ao.converged && k >= kmax && k < min(rows, cols) && (kmax < D.Kf || D.Kf < D.kfull)) {
      S.status = 2;  // needs more crosses than this worker holds
      if (g.rank() == 0) state[f] = S;
      g.sync();
      continue;
    }
    if (!ao.converged && (k >= min(rows, cols) || k >= D.Kf) && !(g_full_rank_ok && k >= min(rows, cols))) {
      S.status = 1;
      if (g.rank() == 0) state[f] = S;
      g.sync();
      continue;
    }
    // ACA pass: stage the crosses and their Gram matrices (ld k) in the output
    // factors for phase 1 (r = -1 marks a staged fill); a fill whose Gram
    // matrices do not fit behind its crosses is finished here
    if (phase == 0 && k > 0 && (size_t)k * k <= (size_t)rows * (D.Kf - k) &&
        (size_t)k * k <= (size_t)cols * (D.Kf - k) + D.Kf) {
      double* gu = D.out + (size_t)rows * k;
      double* gv = D.out + (size_t)rows * D.Kf + (size_t)cols * k;
      for (int e = g.rank(); e < rows * k; e += g.size()) D.out[e] = Uc[e];
      for (int e = g.rank(); e < cols * k; e += g.size()) D.out[(size_t)rows * D.Kf + e] = Vc[e];
      if (g_gram)
        for (int e = g.rank(); e < k * k; e += g.size()) {
          const int i = e % k, j = e / k;
          gu[e] = Rl[i + (size_t)j * KK];
          gv[e] = Rr[i + (size_t)j * KK];
        }
      S.r = -1;
      if (g.rank() == 0) state[f] = S;
      g.sync();
      continue;
    }
    }  // phase != 1
    int r = 0;
    double* left = D.out;
    double* right = D.out + (size_t)rows * D.Kf;
    double* sv = right + (size_t)cols * D.Kf;
    int rg = -1;
    if (k > 0 && g_gram) {
      rg = gram_recompress(g, Uc, Vc, rows, cols, k, Rl, Rr, KK, core, Jv, sig, ord, tol, Ql, Qr, left, right, sv,
                           rr, cc);
      PROF_ACC(1);
    }
    if (rg >= 0) {
      r = rg;
    } else if (k > 0) {
      g_qr(g, Uc, rows, k, rows, Rl, Ql, rows, vv);
      g_qr(g, Vc, cols, k, cols, Rr, Qr, cols, vv);
      PROF_ACC(1);
      g_gemm(g, k, k, k, 1.0, Rl, k, false, Rr, k, true, 0.0, core, k);
      g_jacobi(g, core, k, k, k, Jv, k, sig, ord);
      r = trunc_rank_dev(sig, ord, k, tol);
      PROF_ACC(2);
      for (int e = g.rank(); e < rows * r; e += g.size()) {
        const int i = e % rows, c = e / rows;
        const int col = ord[c];
        double acc = 0.0;
        for (int t = 0; t < k; t++) acc = fma(Ql[i + (size_t)t * rows], core[t + (size_t)col * k], acc);
        left[i + (size_t)c * rows] = acc;
      }
      for (int e = g.rank(); e < cols * r; e += g.size()) {
        const int i = e % cols, c = e / cols;
        const int col = ord[c];
        double acc = 0.0;
        for (int t = 0; t < k; t++) acc = fma(Qr[i + (size_t)t * cols], Jv[t + (size_t)col * k], acc);
        right[i + (size_t)c * cols] = acc;
      }
      for (int c = g.rank(); c < r; c += g.size()) sv[c] = sig[ord[c]];
      g.sync();
    }
    double fro = 0.0;
    for (int e = g.rank(); e < rows * r; e += g.size()) fro += left[e] * left[e];
    fro = sqrt(g.sum(fro));
    PROF_ACC(3);
    S.r = r;
    S.fro = fro;
    if (g.rank() == 0) state[f] = S;
    g.sync();
  }
}

// ------------------------------------------------------------------ new directions
// H (nU x r): directions to add (already weighted).  Appends w <= cap columns
// to U (nU x cap, ld nU) after its first rU columns; ifmm/solver.py:334-358.
// Two-pass projection, then QR + Jacobi on the small R factor.
template <class G>
__device__ int new_dirs(const G& g, double* H, int nU, int r, const double* wsig, double* U, int rU, double cutoff,
                        double* Q, double* R, double* E, double* sig, int* ord, double* vv, int pre = 0) {
  const int cap = nU - rU;
  if (cap <= 0 || r == 0) return 0;
  PROF_T0();
  // the first `pre` columns of U were projected out (twice) by the parallel
  // pre-pass; (I - W W^T)(I - U0 U0^T) = I - U U^T for W orthogonal to U0
  if (rU > pre) {
    g_project_out(g, H, nU, nU, r, U + (size_t)pre * nU, nU, rU - pre, E);
    g_project_out(g, H, nU, nU, r, U + (size_t)pre * nU, nU, rU - pre, E);
  }
  PROF_ACC(4);
  if (wsig) {
    for (int e = g.rank(); e < nU * r; e += g.size()) H[e] *= wsig[e / nU];
    g.sync();
  }
  {
    // sigma_max(H) <= ||H||_F: if the projected, weighted directions are all
    // below the cutoff there is nothing to add (exact; ~30% of the fine-level
    // steps), skip the QR and SVD
    double f2 = 0.0;
    for (int e = g.rank(); e < nU * r; e += g.size()) f2 += H[e] * H[e];
    f2 = g.sum(f2);
    if (g_prof_on && g.rank() == 0) {
      atomicAdd(&g_cyc[11], 1ull);
      if (sqrt(f2) <= cutoff) atomicAdd(&g_cyc[13], 1ull);
    }
    if (sqrt(f2) <= cutoff) return 0;
  }
  double* W = U + (size_t)rU * nU;
  int w = 0;
  if (g_gram == 1 && r <= 96 && nU >= 128) {  // measured: slower than Householder for the small leaf bases
    // Gram route: G = H^T H = L L^T (column-scaled Cholesky), H = Q L^T with
    // Q = H L^-T never formed.  Jacobi on L (= R^T) gives V (left singular
    // vectors of R) and sigma; W = Q V(:, kept) = H (L^-T V(:, kept)).
    // Only for a well-conditioned scaled factor (pivot^2 >= 1e-8): the kept
    // directions are then orthonormal to ~1e-8 before the final projection.
    g_gemm(g, r, r, nU, 1.0, H, nU, true, H, nU, false, 0.0, R, r);  // G -> R (r x r, ld r)
    for (int i = g.rank(); i < r; i += g.size()) vv[i] = sqrt(fmax(R[i + (size_t)i * r], 0.0));
    g.sync();
    bool ok = true;
    if (g.warp() == 0) ok = warp_chol_scaled(R, r, r, vv, 1e-8);
    if (!g.any(!ok)) {
      for (int e = g.rank(); e < r * r; e += g.size()) {  // unscale: L = D^-1 Lhat ; E = L (Jacobi input)
        const int i = e % r;
        R[e] *= vv[i];
        E[e] = R[e];
      }
      g.sync();
      PROF_ACC(5);
      g_jacobi(g, E, r, r, r, Q, r, sig, ord);  // V -> Q (r x r)
      PROF_ACC(6);
      for (int t = 0; t < r; t++) w += (sig[ord[t]] > cutoff);
      w = min(w, cap);
      // Z = L^-T V(:, ord[:w]) into E (r x w), one thread per column
      for (int c = g.rank(); c < w; c += g.size()) {
        const double* B = Q + (size_t)ord[c] * r;
        double* Z = E + (size_t)c * r;
        for (int i = r - 1; i >= 0; i--) {
          double v = B[i];
          for (int p = i + 1; p < r; p++) v -= R[p + (size_t)i * r] * Z[p];
          Z[i] = v / R[i + (size_t)i * r];
        }
      }
      g.sync();
      if (w > 0) g_gemm(g, nU, w, r, 1.0, H, nU, false, E, r, false, 0.0, W, nU);
      if (g_prof_on && g.rank() == 0 && w == 0) atomicAdd(&g_cyc[12], 1ull);
      g.sync();
      if (w > 0) g_project_out(g, W, nU, nU, w, U, nU, rU, E);
      PROF_ACC(7);
      return w;
    }
  }
  g_qr(g, H, nU, r, nU, R, Q, nU, vv);  // H = Q R
  PROF_ACC(5);
  // one-sided Jacobi on R^T with the rotations accumulated: R^T V = X, so V
  // holds the left singular vectors of R and ||X(:,j)|| its singular values.
  // The rows of the triangular R are far closer to orthogonal than its
  // columns (QR-preconditioned Jacobi): fewer sweeps, and W = Q V needs no
  // division by sigma.
  for (int e = g.rank(); e < r * r; e += g.size()) E[e] = R[(e / r) + (size_t)(e % r) * r];
  g.sync();
  g_jacobi(g, E, r, r, r, R, r, sig, ord);  // V -> R
  PROF_ACC(6);
  for (int t = 0; t < r; t++) w += (sig[ord[t]] > cutoff);
  w = min(w, cap);
  for (int e = g.rank(); e < nU * w; e += g.size()) {
    const int i = e % nU, c = e / nU;
    const double* v = R + (size_t)ord[c] * r;
    double acc = 0.0;
    for (int t = 0; t < r; t++) acc = fma(Q[i + (size_t)t * nU], v[t], acc);
    W[i + (size_t)c * nU] = acc;
  }
  if (g_prof_on && g.rank() == 0 && w == 0) atomicAdd(&g_cyc[12], 1ull);
  g.sync();
  if (w > 0) g_project_out(g, W, nU, nU, w, U, nU, rU, E);
  PROF_ACC(7);
  return w;
}

struct DirScratch {
  double *H, *Q, *R, *E, *sig, *vv;
  int* ord;
};
__device__ inline DirScratch carve_dirs(double* s, int MX, int KK) {
  DirScratch d;
  d.H = s; s += (size_t)MX * KK;
  d.Q = s; s += (size_t)MX * KK;
  d.E = s; s += (size_t)MX * KK;
  d.R = s; s += (size_t)KK * KK;
  d.sig = s; s += KK;
  d.vv = s; s += KK;
  d.ord = reinterpret_cast<int*>(s);
  return d;
}

// ------------------------------------------------------------------ K2+K3
// Basis augmentation, one chain per cluster c of the batch.  A hybrid fill
// (q = c) and the q side of a P2P fill (a, c) append directions of the fill's
// weighted right factor to U_c; the p side of a P2P fill (c, b) appends
// directions of its left factor.  Each step depends only on the earlier steps
// of the same cluster, so chains run in parallel and a P2P fill's two sides
// proceed independently -- the reference's sequential order restricted to
// each basis (ifmm/solver.py:334-358, 495-520).  Task = fill * 2 + side
// (0: q side, 1: p side).
// Pre-pass of the augmentation: for every task, H = the fill factor that
// task appends (right factor weighted by sigma for a q side, left factor for
// a p side) with the cluster's batch-initial basis U0 = U(:, :rank0) projected
// out twice.  Independent across tasks (the serial chains then only project
// against the columns appended during the batch).  Hbuf[t] holds nU x Kf.
template <class G>
__global__ void __launch_bounds__(G::kMaxThreads, G::kMinBlocks)
    augment_prep_kernel(const FillDesc* __restrict__ fills, const int* __restrict__ aug, int ntasks,
                        const FillState* __restrict__ state, const int* __restrict__ rank, double tol,
                        double* const* __restrict__ Hbuf, double* scratch, size_t slot,
                        double* const* __restrict__ Ebuf, int* __restrict__ r0buf) {
  __shared__ CtaShared sh;
  const G g = Worker<G>::make(sh);
  double* E = scratch + slot * Worker<G>::id();
  for (int u = Worker<G>::id(); u < ntasks; u += Worker<G>::count()) {
    const int f = aug[u] >> 1, side = aug[u] & 1;
    const FillDesc D = fills[f];
    const int r = state[f].r, status = state[f].status;
    if (status != 0 || r == 0 || tol <= 0.0) continue;
    const int nU = side ? D.rows : D.cols;
    const int cl = side ? D.p : D.q;
    const int r0 = rank[cl];
    double* H = Hbuf[u];
    const double* right = D.out + (size_t)D.rows * D.Kf;
    const double* src = side ? D.out : right;
    const double* wsig = side ? nullptr : right + (size_t)D.cols * D.Kf;
    for (int e = g.rank(); e < nU * r; e += g.size()) H[e] = src[e];
    g.sync();
    // project the UNweighted factor (the weights commute with the projection)
    // so the first-pass coefficients U0^T F are exactly what K4 needs for the
    // M2L absorption: saved in Ebuf (r0 x r), K4 only computes the rows of
    // columns appended during the batch
    const bool proj = r0 > 0 && r0 < nU;
    if (proj) {
      const double* U = side ? D.Up : D.Uq;
      double* E1 = Ebuf[u];
      g_gemm(g, r0, r, nU, 1.0, U, nU, true, H, nU, false, 0.0, E1, r0);
      g_gemm(g, nU, r, r0, -1.0, U, nU, false, E1, r0, false, 1.0, H, nU);
      g_project_out(g, H, nU, nU, r, U, nU, r0, E);
    }
    if (wsig) {
      for (int e = g.rank(); e < nU * r; e += g.size()) H[e] *= wsig[e / nU];
    }
    if (g.rank() == 0) r0buf[u] = proj ? r0 : 0;
    g.sync();
  }
}

template <class G>
__global__ void __launch_bounds__(G::kMaxThreads, G::kMinBlocks)
    augment_kernel(const FillDesc* __restrict__ fills, const int* __restrict__ aug_off, const int* __restrict__ aug,
                   int nchains, FillState* state, int* rank, double tol, double* scratch, size_t slot, int MX, int KK,
                   int debug, double* const* __restrict__ Hbuf) {
  __shared__ CtaShared sh;
  const G g = Worker<G>::make(sh);
  DirScratch d = carve_dirs(scratch + slot * Worker<G>::id(), MX, KK);
  for (int c = Worker<G>::id(); c < nchains; c += Worker<G>::count()) {
    const int t0 = aug_off[c], t1 = aug_off[c + 1];
    const int side0 = aug[t0] & 1;
    const int cl = side0 ? fills[aug[t0] >> 1].p : fills[aug[t0] >> 1].q;
    const int r0 = rank[cl];  // batch-initial rank: already projected out by the pre-pass
    int rc = r0;
    for (int u = t0; u < t1; u++) {
      const int f = aug[u] >> 1, side = aug[u] & 1;
      const FillDesc D = fills[f];
      const int r = state[f].r, status = state[f].status;
      const double fro = state[f].fro;
      if (status == 0 && r > 0 && tol > 0.0) {
        const int nU = side ? D.rows : D.cols;
        // r0 == nU: the pre-pass skipped (no room); new_dirs returns 0 anyway
        const int w = new_dirs(g, Hbuf[u], nU, r, nullptr, side ? D.Up : D.Uq, rc, tol * fro, d.Q, d.R, d.E, d.sig,
                               d.ord, d.vv, r0 < nU ? r0 : 0);
        if (debug && g.rank() == 0)
          printf("aug kind=%d side=%d p=%d q=%d r=%d +%d -> %d\n", D.kind, side, D.p, D.q, r, w, rc + w);
        rc += w;
      }
      if (g.rank() == 0) {
        if (side) state[f].rp = rc;
        else state[f].rq = rc;
      }
      g.sync();
    }
    if (g.rank() == 0) rank[cl] = rc;
    g.sync();
  }
}

// ------------------------------------------------------------------ K4
template <class G>
__global__ void __launch_bounds__(G::kMaxThreads, G::kMinBlocks) delta_kernel(const FillDesc* __restrict__ fills, int nf,
                                                   const FillState* __restrict__ state, double tol, double* scratch,
                                                   size_t slot, int MX, int KK, int* stats,
                                                   const int* __restrict__ taskq, const int* __restrict__ taskp,
                                                   double* const* __restrict__ Ebuf, const int* __restrict__ r0buf) {
  __shared__ CtaShared sh;
  const G g = Worker<G>::make(sh);
  double* Eq = scratch + slot * Worker<G>::id();
  double* Ep = Eq + (size_t)MX * KK;
  for (int f = Worker<G>::id(); f < nf; f += Worker<G>::count()) {
    const FillDesc D = fills[f];
    const FillState S = state[f];
    if (S.status != 0) {
      if (g.rank() == 0) atomicAdd(&stats[1], 1);
      continue;
    }
    const int rows = D.rows, cols = D.cols;
    if (tol == 0.0) {
      for (int e = g.rank(); e < rows * cols; e += g.size()) {
        const int a = e % rows, b = e / rows;
        const double v = Fat(D.F, D.ldF, D.transF, a, b);
        if (D.transM) D.M[b + (size_t)a * D.ldM] += v;
        else D.M[a + (size_t)b * D.ldM] += v;
      }
    } else if (S.r > 0) {
      const int r = S.r, rq = S.rq;
      const double* left = D.out;
      const double* right = D.out + (size_t)rows * D.Kf;
      // Uq^T B: rows of the batch-initial basis come from the augmentation
      // pre-pass (Ebuf), only the rows of appended columns are computed here
      auto coeffs = [&](const double* Ub, int ld, const double* Fx, int rr, int t, double* Eo) {
        const int r0 = (t >= 0 && Ebuf) ? min(r0buf[t], rr) : 0;
        if (r0 > 0) {
          const double* E1 = Ebuf[t];
          for (int e = g.rank(); e < r0 * r; e += g.size()) Eo[(e % r0) + (size_t)(e / r0) * rr] = E1[e];
        }
        if (rr > r0) g_gemm(g, rr - r0, r, ld, 1.0, Ub + (size_t)r0 * ld, ld, true, Fx, ld, false, 0.0, Eo + r0, rr);
        g.sync();
      };
      coeffs(D.Uq, cols, right, rq, taskq ? taskq[f] : -1, Eq);
      const double* X = left;
      int rx = rows, ldx = rows;
      if (D.kind == FILL_P2P) {
        coeffs(D.Up, rows, left, S.rp, taskp ? taskp[f] : -1, Ep);  // Up^T A
        X = Ep;
        rx = S.rp;
        ldx = S.rp;
      }
      // M2L(p,q) += X Eq^T   (owner stores (q,p): M += Eq X^T)
      if (D.transM) g_gemm(g, rq, rx, r, 1.0, Eq, rq, false, X, ldx, true, 1.0, D.M, D.ldM);
      else g_gemm(g, rx, rq, r, 1.0, X, ldx, false, Eq, rq, true, 1.0, D.M, D.ldM);
    }
    g.sync();
    for (int e = g.rank(); e < rows * cols; e += g.size()) {
      const int a = e % rows, b = e / rows;
      if (D.transF) D.F[b + (size_t)a * D.ldF] = 0.0;
      else D.F[a + (size_t)b * D.ldF] = 0.0;
    }
    if (g.rank() == 0) {
      atomicAdd(&stats[0], 1);
      atomicMax(&stats[2], S.r);
    }
    g.sync();
  }
}

// ------------------------------------------------------------------ test hook
// K1 on one fill F (m x n, column-major, device): gram = 1 through the Gram
// matrices (with the Householder fallback), 0 through the Householder QRs.
void test_recompress_one(const double* dF, int m, int n, double tol, const int* d_probes, int probe_maxm, int gram,
                         double* d_out, FillState* d_state, Arena& ws, Staging& st, cudaStream_t s) {
  const int g0 = gram;
  CK(cudaMemcpyToSymbolAsync(g_gram, &g0, sizeof(int), 0, cudaMemcpyHostToDevice, s));
  FillDesc D{};
  D.kind = FILL_P2P;
  D.F = const_cast<double*>(dF);
  D.ldF = m;
  D.transF = 0;
  D.rows = m;
  D.cols = n;
  D.n_p = m;
  D.n_q = n;
  D.Kf = std::max(1, std::min(96, std::min(m, n)));
  D.kfull = D.Kf;
  D.out = d_out;
  std::vector<FillDesc> v(1, D);
  const FillDesc* dfd = upload(ws, v, s, st);
  const int KK = D.Kf;
  const size_t slot = 2 * size_t(m) * KK + 2 * size_t(n) * KK + 4 * size_t(KK) * KK + 2 * size_t(m + n) +
                      4 * size_t(KK) + 64;
  double* scr = ws.alloc_n<double>(slot);
  aca_recompress_kernel<CtaGroup><<<1, 128, 0, s>>>(dfd, 1, d_state, tol, d_probes, probe_maxm, scr, slot, m, n, KK, 0, 2);
  CK_LAUNCH();
  const int one = 1;  // restore the default
  CK(cudaMemcpyToSymbolAsync(g_gram, &one, sizeof(int), 0, cudaMemcpyHostToDevice, s));
}

// ------------------------------------------------------------------ host
static int resident_grid(int work, int per_sm) { return std::max(1, std::min(work, 148 * per_sm)); }

void run_compression(CompressBatch& cb, double tol, const int* d_probes, int probe_maxm, int* d_rank,
                     FillState* d_state, int* d_stats, Arena& ws, Staging& st, cudaStream_t s, int debug) {
  const int nf = int(cb.fills.size());
  if (nf == 0) return;
  int MR = 1, MC = 1, KK = 1, MX = 1;
  for (const FillDesc& D : cb.fills) {
    MR = std::max(MR, D.rows);
    MC = std::max(MC, D.cols);
    KK = std::max(KK, D.Kf);
    MX = std::max(MX, std::max(D.n_p, D.n_q));
  }
  MX = std::max(MX, std::max(MR, MC));
  MX = std::max(MX, cb.shape_mx);
  const int nf_shape = std::max(nf, cb.shape_nf);
  // Worker shape.  Fine levels (thousands of fills of a few dozen rows): one
  // warp per fill / chain / pivot, 4 warps per CTA -- no block barriers and
  // many fills in flight per SM.  Coarse levels (few, large fills): one wide
  // CTA per fill shortens each step of the dependent chains.
  // (warp workers -- one warp per fill -- exist for the test hooks; measured
  // slower than small CTAs on the C3 leaf level, so production uses CTAs)
  const bool wmode = false;
  // fine levels: small CTAs, many fills in flight per SM
  constexpr int bs_small = 128;
  const int per_sm = 8 * 128 / bs_small;  // resident CTAs per SM at 64 registers
  // coarse levels: per-step latency of few long chains dominates -> widest CTAs
  // for the largest blocks (measured: 1024 wins for MX >= ~800, loses at 265-570)
  const int bs_big = MX >= 700 ? 1024 : 512;
  constexpr int nf_big = 2048;
  const int bs_fill = (MX >= 256 && nf_shape < nf_big) ? bs_big : (MX >= 128 ? 256 : bs_small);
  // level-6-sized bases (256 <= MX < 400): 256-thread chains measured best (112 -> 102 ms)
  const int bs_dirs = (MX >= 256 && MX < 400) ? 256 : MX >= 256 ? bs_big : (MX >= 128 ? 256 : bs_small);
  constexpr int WPB = 4;  // warps per CTA in warp mode
  static const bool prof = getenv("IFMM_PROF") != nullptr;
  {
    // The Gram routes (K1 recompression through the cross Gram matrices, new
    // directions through H^T H) lose accuracy ~ eps * cond^2; that is far below
    // the truncation for tol >= 1e-9, but at tolerances near machine precision
    // (the reference default 1e-14) the duplicated directions make pivots
    // singular, so the Householder routes run there.
    const int gram = tol >= 1e-9 ? 1 : 0;
    CK(cudaMemcpyToSymbolAsync(g_gram, &gram, sizeof(int), 0, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyToSymbolAsync(g_full_rank_ok, &cb.full_rank_ok, sizeof(int), 0, cudaMemcpyHostToDevice, s));
    const double gpiv = 1e-14;
    CK(cudaMemcpyToSymbolAsync(g_gram_piv, &gpiv, sizeof(double), 0, cudaMemcpyHostToDevice, s));
    // Jacobi rotation threshold from the truncation tolerance: singular values
    // then carry ~(1e-4 tol)^2 relative error -- far below the truncation decisions
    // (1e-2 tol measured: 15 ms faster at C3 but a C3-parameter pivot crossed the
    // 1e12 condition limit; 1e-4 tol: 10 ms faster, all gates green)
    const double jt = tol > 0.0 ? std::max(1e-15, std::min(1e-8, tol * 1e-4)) : 1e-15;
    CK(cudaMemcpyToSymbolAsync(g_jac_tol, &jt, sizeof(double), 0, cudaMemcpyHostToDevice, s));
  }
  if (prof) {
    const int one = 1;
    unsigned long long z[16] = {0};
    CK(cudaMemcpyToSymbolAsync(g_prof_on, &one, sizeof(int), 0, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyToSymbolAsync(g_cyc, z, sizeof z, 0, cudaMemcpyHostToDevice, s));
  }
  const FillDesc* dfd = upload(ws, cb.fills, s, st);
  bool may_redo = false;  // fills whose reference cross cap exceeds this pass's buffers
  for (const FillDesc& D : cb.fills) may_redo |= D.kfull > D.Kf;
  // grid for `work` items: CTA workers, or warp workers packed WPB per CTA
  auto grid_for = [&](int work, int cta_per_sm, int warps_per_sm) {
    return wmode ? resident_grid(ceil_div(work, WPB), warps_per_sm / WPB) : resident_grid(work, cta_per_sm);
  };
  auto workers = [&](int grid) { return wmode ? grid * WPB : grid; };
  // K1
  {
    auto k1_slot = [&](int kk) {
      return 2 * size_t(MR) * kk + 2 * size_t(MC) * kk + 4 * size_t(kk) * kk + 2 * size_t(MR + MC) +
             4 * size_t(kk) + 64;
    };
    if (wmode) {
      const int kw = std::min(KK, WARP_KCAP);
      const size_t slot = k1_slot(kw);
      const int grid = grid_for(nf, 8, 32);
      double* scr = ws.alloc_n<double>(slot * workers(grid));
      aca_recompress_kernel<WarpGroup><<<grid, 32 * WPB, 0, s>>>(dfd, nf, d_state, tol, d_probes, probe_maxm, scr,
                                                                   slot, MR, MC, kw, 0, 2);
      CK_LAUNCH();
      if (KK > kw) {  // fills whose ACA outgrew the warp's cross cap
        const size_t cslot = k1_slot(KK);
        const int cgrid = resident_grid(nf, 2);
        double* cscr = ws.alloc_n<double>(cslot * cgrid);
        aca_recompress_kernel<CtaGroup><<<cgrid, 128, 0, s>>>(dfd, nf, d_state, tol, d_probes, probe_maxm, cscr,
                                                               cslot, MR, MC, KK, 1, 2);
        CK_LAUNCH();
      }
    } else {
      const size_t slot = k1_slot(KK);
      const int grid = resident_grid(nf, bs_fill == bs_small ? per_sm : 8);
      double* scr = ws.alloc_n<double>(slot * grid);
      // ACA and recompression as two passes over the fills: every CTA on an SM
      // then runs the same (smaller) code region
      if (bs_fill == bs_small) {  // measured: a gain at the leaf level only
        // fills of one kind (P2P, then hybrid) run side by side (batch order instead:
        // measured 100 -> 98 ms at the C3 leaf level; largest-first within a kind: 107 ms)
        const int* dorder = nullptr;
        {
          std::vector<int> ord;
          ord.reserve(nf);
          for (int f = 0; f < nf; f++)
            if (cb.fills[f].kind == FILL_P2P) ord.push_back(f);
          for (int f = 0; f < nf; f++)
            if (cb.fills[f].kind != FILL_P2P) ord.push_back(f);
          dorder = upload(ws, ord, s, st);
        }
        for (int ph = 0; ph < 2; ph++) {
          aca_recompress_kernel<CtaGroup><<<grid, bs_fill, 0, s>>>(dfd, nf, d_state, tol, d_probes, probe_maxm, scr,
                                                                   slot, MR, MC, KK, 0, ph, dorder);
          CK_LAUNCH();
        }
      } else {
        aca_recompress_kernel<CtaGroup><<<grid, bs_fill, 0, s>>>(dfd, nf, d_state, tol, d_probes, probe_maxm, scr,
                                                                 slot, MR, MC, KK, 0, 2);
        CK_LAUNCH();
      }
    }
  }
  // Fills that used all Kf (<= 96) crosses of the first pass without
  // converging continue up to the reference's min(m, n) crosses with buffers of
  // that size (few fills, coarse levels at high accuracy).  Checked after the
  // host has prepared the augmentation launches (the readback waits for K1).
  std::vector<char> redone;
  bool redo_checked = false;
  auto redo_pass = [&]() {
    if (!may_redo || redo_checked) return false;
    redo_checked = true;
    std::vector<FillState> hs(nf);
    CK(cudaMemcpyAsync(hs.data(), d_state, sizeof(FillState) * nf, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    int nredo = 0;
    redone.assign(nf, 0);
    for (int f = 0; f < nf; f++) {
      FillDesc& D = cb.fills[f];
      if (hs[f].status != 2 || D.kfull <= D.Kf) continue;
      D.Kf = D.kfull;
      D.out = ws.alloc_n<double>(size_t(D.rows + D.cols + 1) * D.Kf);
      KK = std::max(KK, D.Kf);
      redone[f] = 1;
      nredo++;
    }
    if (nredo == 0) return false;
    dfd = upload(ws, cb.fills, s, st);
    const size_t slot = 2 * size_t(MR) * KK + 2 * size_t(MC) * KK + 4 * size_t(KK) * KK + 2 * size_t(MR + MC) +
                        4 * size_t(KK) + 64;
    const int grid = std::max(1, std::min(nredo, 148));
    double* scr = ws.alloc_n<double>(slot * grid);
    aca_recompress_kernel<CtaGroup><<<grid, bs_big, 0, s>>>(dfd, nf, d_state, tol, d_probes, probe_maxm, scr, slot,
                                                            MR, MC, KK, 1, 2);
    CK_LAUNCH();
    return true;
  };
  size_t dslot = 0;
  const int bs_d = wmode ? 32 * WPB : bs_dirs;
  std::vector<int> tq, tp;  // fill -> q-side / p-side augmentation task (-1: none)
  double* const* d_eb = nullptr;
  int* d_r0 = nullptr;
  // K2+K3: per-cluster augmentation chains.  Order inside a chain: the
  // cluster's hybrid fills (sorted), then the P2P fills touching it in the
  // pivot's pair order; clusters of different pivots of a batch are disjoint.
  {
    int maxc = 0;
    for (const FillDesc& D : cb.fills) maxc = std::max(maxc, std::max(D.p, D.q));
    std::vector<int> cid(size_t(maxc) + 1, -1);
    std::vector<std::vector<int>> tasks;
    auto push = [&](int cl, int task) {
      int& c = cid[cl];
      if (c < 0) {
        c = int(tasks.size());
        tasks.emplace_back();
      }
      tasks[c].push_back(task);
    };
    const int nch = int(cb.chain_off.size()) - 1;
    for (int c = 0; c < nch; c++)
      for (int u = cb.chain_off[c]; u < cb.chain_off[c + 1]; u++) push(cb.fills[cb.chain[u]].q, cb.chain[u] * 2);
    for (int f : cb.p2p) {
      push(cb.fills[f].q, f * 2);
      push(cb.fills[f].p, f * 2 + 1);
    }
    if (prof && !tasks.empty()) {
      size_t mx = 0, tot = 0;
      for (auto& t : tasks) { mx = std::max(mx, t.size()); tot += t.size(); }
      fprintf(stderr, "chains %zu tasks %zu max len %zu avg %.2f\n", tasks.size(), tot, mx, double(tot) / tasks.size());
    }
    if (!tasks.empty()) {
      std::vector<int> off(1, 0), lst;
      lst.reserve(2 * cb.fills.size());
      for (auto& t : tasks) {
        lst.insert(lst.end(), t.begin(), t.end());
        off.push_back(int(lst.size()));
      }
      const int* doff = upload(ws, off, s, st);
      const int* dlst = upload(ws, lst, s, st);
      const int n = int(tasks.size());
      const int ntask = int(lst.size());
      // per-task direction buffers (nU x Kf: the fill's rank is only known on the device)
      std::vector<double*> hb(lst.size());
      for (size_t u = 0; u < lst.size(); u++) {
        const FillDesc& D = cb.fills[lst[u] >> 1];
        hb[u] = ws.alloc_n<double>(size_t((lst[u] & 1) ? D.rows : D.cols) * D.Kf);
      }
      double* const* dhb = upload(ws, hb, s, st);  // re-uploaded if a fill is redone
      // first-pass coefficients U0^T F per task (r0 x Kf, r0 = batch-initial
      // rank from the host copy) + the fill -> task maps for K4
      std::vector<double*> eb(lst.size(), nullptr);
      tq.assign(cb.fills.size(), -1);
      tp.assign(cb.fills.size(), -1);
      for (size_t u = 0; u < lst.size(); u++) {
        const int f = lst[u] >> 1, side = lst[u] & 1;
        const FillDesc& D = cb.fills[f];
        const int r0 = cb.rank_host ? cb.rank_host[side ? D.p : D.q] : 0;
        if (r0 > 0) eb[u] = ws.alloc_n<double>(size_t(r0) * D.Kf);
        (side ? tp : tq)[f] = int(u);
      }
      d_eb = upload(ws, eb, s, st);
      d_r0 = ws.alloc_n<int>(lst.size());
      CK(cudaMemsetAsync(d_r0, 0, sizeof(int) * lst.size(), s));
      if (redo_pass()) {  // grown fills need larger direction / coefficient buffers
        for (size_t u = 0; u < lst.size(); u++) {
          const int f = lst[u] >> 1, side = lst[u] & 1;
          if (!redone[f]) continue;
          const FillDesc& D = cb.fills[f];
          hb[u] = ws.alloc_n<double>(size_t(side ? D.rows : D.cols) * D.Kf);
          const int r0 = cb.rank_host ? cb.rank_host[side ? D.p : D.q] : 0;
          if (r0 > 0) eb[u] = ws.alloc_n<double>(size_t(r0) * D.Kf);
        }
        dhb = upload(ws, hb, s, st);
        d_eb = upload(ws, eb, s, st);
      }
      dslot = 3 * size_t(MX) * KK + size_t(KK) * KK + 3 * size_t(KK) + 64;
      {
        const size_t pslot = size_t(MX) * KK + 64;
        const int pgrid = grid_for(ntask, bs_d == bs_small ? per_sm : 8, 32);
        double* pscr = ws.alloc_n<double>(pslot * workers(pgrid));
        if (wmode)
          augment_prep_kernel<WarpGroup><<<pgrid, bs_d, 0, s>>>(dfd, dlst, ntask, d_state, d_rank, tol, dhb, pscr,
                                                                  pslot, d_eb, d_r0);
        else
          augment_prep_kernel<CtaGroup><<<pgrid, bs_d, 0, s>>>(dfd, dlst, ntask, d_state, d_rank, tol, dhb, pscr,
                                                                 pslot, d_eb, d_r0);
        CK_LAUNCH();
      }
      const int grid = grid_for(n, bs_d == bs_small ? per_sm : 8, 32);
      double* scr = ws.alloc_n<double>(dslot * workers(grid));
      if (wmode)
        augment_kernel<WarpGroup><<<grid, bs_d, 0, s>>>(dfd, doff, dlst, n, d_state, d_rank, tol, scr, dslot, MX, KK,
                                                          debug, dhb);
      else
        augment_kernel<CtaGroup><<<grid, bs_d, 0, s>>>(dfd, doff, dlst, n, d_state, d_rank, tol, scr, dslot, MX, KK,
                                                         debug, dhb);
      CK_LAUNCH();
    }
  }
  redo_pass();  // batches without augmentation tasks
  // K4
  {
    const size_t slot = 2 * size_t(MX) * KK + 64;
    const int grid = grid_for(nf, bs_fill == bs_small ? per_sm : 8, 32);
    double* scr = ws.alloc_n<double>(slot * workers(grid));
    const int* dtq = tq.empty() ? nullptr : upload(ws, tq, s, st);
    const int* dtp = tp.empty() ? nullptr : upload(ws, tp, s, st);
    if (wmode)
      delta_kernel<WarpGroup><<<grid, 32 * WPB, 0, s>>>(dfd, nf, d_state, tol, scr, slot, MX, KK, d_stats, dtq, dtp,
                                                          d_eb, d_r0);
    else
      delta_kernel<CtaGroup><<<grid, bs_fill, 0, s>>>(dfd, nf, d_state, tol, scr, slot, MX, KK, d_stats, dtq, dtp,
                                                        d_eb, d_r0);
    CK_LAUNCH();
  }
  if (prof) {
    unsigned long long c[16];
    CK(cudaMemcpyFromSymbolAsync(c, g_cyc, sizeof c, 0, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    fprintf(stderr, "prof MX=%d nf=%d chains=%zu p2p=%zu | aca %.1f qr %.1f core %.1f rest %.1f | proj %.1f qr %.1f jac %.1f W %.1f Mcyc | jacobi calls %llu avg sweeps %.2f avg cols %.1f | aug steps %llu w=0 %llu fro<=cut %llu\n",
            MX, nf, cb.chain_off.size() - 1, cb.p2p.size(), c[0] / 1e6, c[1] / 1e6, c[2] / 1e6, c[3] / 1e6, c[4] / 1e6,
            c[5] / 1e6, c[6] / 1e6, c[7] / 1e6, c[9], c[9] ? double(c[8]) / c[9] : 0.0, c[9] ? double(c[10]) / c[9] : 0.0, c[11], c[12], c[13]);
  }
}

}  // namespace ifmm
