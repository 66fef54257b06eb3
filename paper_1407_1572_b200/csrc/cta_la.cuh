// Cooperative dense linear algebra on column-major matrices held in global
// (L1/L2-resident) scratch: DMMA GEMM, Householder QR, one-sided Jacobi SVD,
// partially pivoted ACA.  Every routine is a template over an execution group
// G -- a whole CTA (CtaGroup) or a single warp (WarpGroup) -- and must be
// called by all threads of the group.  The compression kernels run one warp
// per fill for the many small fills of the fine levels (no block barriers,
// 4-16x more fills in flight per SM) and one CTA per fill at coarse levels;
// the Chebyshev basis construction uses CTAs.
#pragma once
#include "common.cuh"

namespace ifmm {

// Off-diagonal threshold of the one-sided Jacobi SVDs: a pair is rotated while
// |x.y| > tol_rot * |x| |y|.  Column norms then match the singular values to
// ~tol_rot^2 relative to the largest, so the compression sets it from its
// truncation tolerance (compress.cu); elsewhere it stays at rounding level.
__device__ double g_jac_tol = 1e-15;

struct CtaShared {
  double red[32];
  double red2[32];
  double pmax[32 * 10];  // per-warp probe-row maxima (ACA start row)
  ArgMax am[32];
  int flag;
  int ival[4];
  double dval[4];
};

__device__ __forceinline__ ArgMax warp_argmax(ArgMax v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ArgMax w;
    w.a = __shfl_xor_sync(0xffffffffu, v.a, o);
    w.i = __shfl_xor_sync(0xffffffffu, v.i, o);
    v = argmax_merge(v, w);
  }
  return v;
}

struct CtaGroup {
  static constexpr int kMaxThreads = 1024, kMinBlocks = 1;  // launch bounds of kernels templated on the group (64 registers)
  CtaShared& sh;
  __device__ int rank() const { return threadIdx.x; }
  __device__ int size() const { return blockDim.x; }
  __device__ int lane() const { return threadIdx.x & 31; }
  __device__ int warp() const { return threadIdx.x >> 5; }
  __device__ int nwarps() const { return blockDim.x >> 5; }
  __device__ void sync() const { __syncthreads(); }
  __device__ double sum(double v) const { return block_sum(v, sh.red); }
  __device__ ArgMax argmax(ArgMax v) const { return block_argmax(v, sh.am); }
  __device__ bool any(bool p) const { return __syncthreads_or(p) != 0; }
  // combine warp-reduced partials (identical in every lane) over the group:
  // two sums and an argmax in one publish/reduce round (two barriers)
  __device__ void combine(double& a, double& b, ArgMax& c) const {
    __syncthreads();
    if (lane() == 0) {
      sh.red[warp()] = a;
      sh.red2[warp()] = b;
      sh.am[warp()] = c;
    }
    __syncthreads();
    a = 0.0;
    b = 0.0;
    c = ArgMax{-1.0, -1};
    for (int w = 0; w < nwarps(); w++) {
      a += sh.red[w];
      b += sh.red2[w];
      c = argmax_merge(c, sh.am[w]);
    }
  }
  // max over the group of v[0..np) (warp-reduced first), identical everywhere
  __device__ void max10(double (&v)[10], int np) const {
    __syncthreads();
    if (lane() == 0)
      for (int t = 0; t < np; t++) sh.pmax[warp() * 10 + t] = v[t];
    __syncthreads();
    for (int t = 0; t < np; t++) {
      double m = -1.0;
      for (int w = 0; w < nwarps(); w++) m = fmax(m, sh.pmax[w * 10 + t]);
      v[t] = m;
    }
  }
  __device__ static CtaGroup make_for_test(CtaShared& sh) { return CtaGroup{sh}; }
};

struct WarpGroup {
  static constexpr int kMaxThreads = 128, kMinBlocks = 4;
  __device__ int rank() const { return threadIdx.x & 31; }
  __device__ int size() const { return 32; }
  __device__ int lane() const { return threadIdx.x & 31; }
  __device__ int warp() const { return 0; }
  __device__ int nwarps() const { return 1; }
  __device__ void sync() const { __syncwarp(); }
  __device__ double sum(double v) const { return warp_sum(v); }
  __device__ ArgMax argmax(ArgMax v) const { return warp_argmax(v); }
  __device__ bool any(bool p) const { return __any_sync(0xffffffffu, p) != 0; }
  __device__ void combine(double&, double&, ArgMax&) const { __syncwarp(); }  // already warp-reduced
  __device__ void max10(double (&)[10], int) const {}                          // already warp-reduced
  __device__ static WarpGroup make_for_test(CtaShared&) { return WarpGroup{}; }
};

// ------------------------------------------------------------- small helpers
// CTA-cooperative DMMA GEMM (mma.sync.m8n8k4.f64): every warp owns 16x16
// output tiles (2x2 fragments); fragments are loaded straight from L1/L2.
// One DMMA does 512 flops for 2 loads per lane, vs 2 flops per 2 loads for a
// scalar loop -- the projections and deltas of the compression are otherwise
// L1-throughput bound.
template <bool TA, bool TB, class G>
__device__ inline void g_mma_gemm(const G& g, int rows, int cols, int kk, double alpha, const double* __restrict__ A, int lda,
                                    const double* __restrict__ B, int ldb, double beta, double* Y, int ldy) {
  const int lane = g.lane(), warp = g.warp(), nw = g.nwarps();
  const int tm = (rows + 15) >> 4, tn = (cols + 15) >> 4;
  const int fr = lane >> 2, fk = lane & 3;
  for (int tile = warp; tile < tm * tn; tile += nw) {
    const int i0 = (tile % tm) << 4, j0 = (tile / tm) << 4;
    double acc[2][2][2] = {{{0, 0}, {0, 0}}, {{0, 0}, {0, 0}}};
    for (int k0 = 0; k0 < kk; k0 += 4) {
      const int k = k0 + fk;
      double a[2], b[2];
#pragma unroll
      for (int m = 0; m < 2; m++) {
        const int i = i0 + m * 8 + fr;
        a[m] = (i < rows && k < kk) ? (TA ? A[k + (size_t)i * lda] : A[i + (size_t)k * lda]) : 0.0;
      }
#pragma unroll
      for (int n = 0; n < 2; n++) {
        const int j = j0 + n * 8 + fr;
        b[n] = (j < cols && k < kk) ? (TB ? B[j + (size_t)k * ldb] : B[k + (size_t)j * ldb]) : 0.0;
      }
#pragma unroll
      for (int m = 0; m < 2; m++)
#pragma unroll
        for (int n = 0; n < 2; n++)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(acc[m][n][0]), "+d"(acc[m][n][1])
                       : "d"(a[m]), "d"(b[n]));
    }
#pragma unroll
    for (int m = 0; m < 2; m++)
#pragma unroll
      for (int n = 0; n < 2; n++)
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int i = i0 + m * 8 + fr, j = j0 + n * 8 + 2 * fk + h;
          if (i < rows && j < cols) {
            double* y = Y + i + (size_t)j * ldy;
            *y = (beta == 0.0 ? 0.0 : beta * *y) + alpha * acc[m][n][h];
          }
        }
  }
  g.sync();
}

// Y(rows x cols, ldy) = alpha * op(A) * op(B) + beta*Y for the small products
// inside compression; DMMA tiles when the shape is worth it.
// opA: A is (rows x kk) if !ta else stored (kk x rows).
template <class G>
__device__ inline void g_gemm(const G& g, int rows, int cols, int kk, double alpha, const double* A, int lda, bool ta,
                                const double* B, int ldb, bool tb, double beta, double* Y, int ldy) {
  if (rows >= 8 && cols >= 8 && kk >= 8) {
    if (ta) {
      if (tb) g_mma_gemm<true, true>(g, rows, cols, kk, alpha, A, lda, B, ldb, beta, Y, ldy);
      else g_mma_gemm<true, false>(g, rows, cols, kk, alpha, A, lda, B, ldb, beta, Y, ldy);
    } else {
      if (tb) g_mma_gemm<false, true>(g, rows, cols, kk, alpha, A, lda, B, ldb, beta, Y, ldy);
      else g_mma_gemm<false, false>(g, rows, cols, kk, alpha, A, lda, B, ldb, beta, Y, ldy);
    }
    return;
  }
  if (ta && !tb) {
    // Y = A^T B: both operands are read down contiguous columns -> one warp per
    // output, lanes stride the contraction (coalesced), warp-shuffle reduction
    const int lane = g.lane(), warp = g.warp(), nw = g.nwarps();
    for (int o = warp; o < rows * cols; o += nw) {
      const int i = o % rows, j = o / rows;
      const double* a = A + (size_t)i * lda;
      const double* b = B + (size_t)j * ldb;
      double s = 0.0;
      for (int t = lane; t < kk; t += 32) s = fma(a[t], b[t], s);
      s = warp_sum(s);
      if (lane == 0) {
        double* y = Y + i + (size_t)j * ldy;
        *y = (beta == 0.0 ? 0.0 : beta * *y) + alpha * s;
      }
    }
    g.sync();
    return;
  }
  for (int e = g.rank(); e < rows * cols; e += g.size()) {
    const int i = e % rows, j = e / rows;
    double s = 0.0;
    for (int t = 0; t < kk; t++) {
      const double a = ta ? A[t + (size_t)i * lda] : A[i + (size_t)t * lda];
      const double b = tb ? B[j + (size_t)t * ldb] : B[t + (size_t)j * ldb];
      s = fma(a, b, s);
    }
    double* y = Y + i + (size_t)j * ldy;
    *y = (beta == 0.0 ? 0.0 : beta * *y) + alpha * s;
  }
  g.sync();
}

// X(n x k) -= U (U^T X), U n x r.  Scratch E >= r*k.
template <class G>
__device__ inline void g_project_out(const G& g, double* X, int ldx, int n, int k, const double* U, int ldu, int r,
                                       double* E) {
  if (r == 0 || k == 0) return;
  g_gemm(g, r, k, n, 1.0, U, ldu, true, X, ldx, false, 0.0, E, r);
  g_gemm(g, n, k, r, -1.0, U, ldu, false, E, r, false, 1.0, X, ldx);
}

// ------------------------------------------------------------- Householder QR
// A (m x k, lda) is overwritten by the reflectors.  Outputs R (k x k, ld k,
// upper) and, if Q != nullptr, the thin Q (m x k, ldq).  vv: scratch >= k.
template <class G>
__device__ inline void g_qr(const G& g, double* A, int m, int k, int lda, double* R, double* Q, int ldq, double* vv) {
  const int lane = g.lane(), warp = g.warp(), nw = g.nwarps();
  for (int j = 0; j < k && j < m; j++) {
    double* x = A + j + (size_t)j * lda;
    const int len = m - j;
    double s = 0.0;
    for (int i = g.rank(); i < len; i += g.size()) s += x[i] * x[i];
    s = g.sum(s);
    const double alpha = sqrt(s);
    const double x0 = x[0];
    double beta = 0.0, vtv = 0.0;
    if (alpha > 0.0) {
      beta = x0 >= 0.0 ? -alpha : alpha;
      // v = x - beta e1 ; vtv = s - x0^2 + (x0-beta)^2
      vtv = s - x0 * x0 + (x0 - beta) * (x0 - beta);
    }
    g.sync();
    if (g.rank() == 0) {
      x[0] = x0 - beta;
      vv[j] = vtv;
      R[j + (size_t)j * k] = alpha > 0.0 ? beta : x0;
    }
    g.sync();
    if (vtv > 0.0) {
      for (int c = j + 1 + warp; c < k; c += nw) {
        double* y = A + j + (size_t)c * lda;
        double d = 0.0;
        for (int i = lane; i < len; i += 32) d += x[i] * y[i];
        d = warp_sum(d);
        const double f = 2.0 * d / vtv;
        for (int i = lane; i < len; i += 32) y[i] -= f * x[i];
      }
    }
    g.sync();
  }
  // R strictly-upper part
  for (int e = g.rank(); e < k * k; e += g.size()) {
    const int i = e % k, c = e / k;
    if (i < c) R[i + (size_t)c * k] = (i < m) ? A[i + (size_t)c * lda] : 0.0;
    else if (i > c) R[i + (size_t)c * k] = 0.0;
    else if (i >= m) R[i + (size_t)c * k] = 0.0;
  }
  g.sync();
  if (Q == nullptr) return;
  for (int e = g.rank(); e < m * k; e += g.size()) {
    const int i = e % m, c = e / m;
    Q[i + (size_t)c * ldq] = (i == c) ? 1.0 : 0.0;
  }
  g.sync();
  for (int j = min(k, m) - 1; j >= 0; j--) {
    const double vtv = vv[j];
    if (vtv <= 0.0) continue;
    const double* x = A + j + (size_t)j * lda;
    const int len = m - j;
    for (int c = warp; c < k; c += nw) {
      double* y = Q + j + (size_t)c * ldq;
      double d = 0.0;
      for (int i = lane; i < len; i += 32) d += x[i] * y[i];
      d = warp_sum(d);
      const double f = 2.0 * d / vtv;
      for (int i = lane; i < len; i += 32) y[i] -= f * x[i];
    }
    g.sync();
  }
}

// ------------------------------------------------------------- Jacobi SVD
// One-sided (Hestenes) Jacobi on A (m x n, lda): on exit the columns of A are
// mutually orthogonal (A_out = A V), V (n x n, ldv) accumulates the rotations
// if non-null, sig[j] = ||A_out(:,j)||, ord[0..n) = column indices sorted by
// decreasing sig (ties: lower index first).  Round-robin pairing; warps own
// disjoint column pairs.
template <class G>
__device__ inline void g_jacobi(const G& g, double* A, int m, int n, int lda, double* V, int ldv, double* sig,
                                int* ord, int max_sweeps = 40) {
  const int lane = g.lane(), warp = g.warp(), nw = g.nwarps();
  if (V)
    for (int e = g.rank(); e < n * n; e += g.size()) V[(e % n) + (size_t)(e / n) * ldv] = (e % n == e / n);
  const int nn = n + (n & 1);  // even number of players (dummy = n)
  // segment width: next power of two >= m (4..32); short columns leave most
  // of a warp idle otherwise
  const int W = m <= 4 ? 4 : m <= 8 ? 8 : m <= 16 ? 16 : 32;
  const int spw = 32 / W, seg = lane / W, sl = lane & (W - 1);
  g.sync();
  for (int sweep = 0; sweep < max_sweeps && n > 1; sweep++) {
    bool rot = false;
    for (int round = 0; round < nn - 1; round++) {
      // each warp runs spw pairs at once, one per W-lane segment
      for (int base = warp * spw; base < nn / 2; base += nw * spw) {
        const int pr = base + seg;
        // circle method: player nn-1 fixed, others rotate.
        // (round + pr) and (round + nn - 1 - pr) are < 2 (nn - 1): one
        // conditional subtraction instead of an integer modulo
        int a = round + pr, b = round + nn - 1 - pr;
        if (a >= nn - 1) a -= nn - 1;
        if (b >= nn - 1) b -= nn - 1;
        if (pr == 0) {
          a = nn - 1;
          b = round;
        }
        const bool valid = pr < nn / 2 && a < n && b < n && a != b;
        if (a > b) { int t = a; a = b; b = t; }
        double* x = A + (size_t)a * lda;
        double* y = A + (size_t)b * lda;
        double al = 0.0, be = 0.0, ga = 0.0;
        if (valid)
          for (int i = sl; i < m; i += W) {
            const double xi = x[i], yi = y[i];
            al += xi * xi;
            be += yi * yi;
            ga += xi * yi;
          }
        for (int o = W >> 1; o > 0; o >>= 1) {  // all lanes: segment-local butterflies
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        if (!valid || ga == 0.0 || fabs(ga) <= g_jac_tol * sqrt(al * be)) continue;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        // a rotation below rounding level changes nothing: columns of very
        // different norms otherwise keep |ga|/sqrt(al*be) ~ eps*sqrt(al/be)
        // and never pass the relative test
        if (fabs(t) < 1e-16) continue;
        const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        for (int i = sl; i < m; i += W) {
          const double xi = x[i], yi = y[i];
          x[i] = c * xi - s * yi;
          y[i] = s * xi + c * yi;
        }
        if (V) {
          double* vx = V + (size_t)a * ldv;
          double* vy = V + (size_t)b * ldv;
          for (int i = sl; i < n; i += W) {
            const double xi = vx[i], yi = vy[i];
            vx[i] = c * xi - s * yi;
            vy[i] = s * xi + c * yi;
          }
        }
        rot = true;
      }
      g.sync();
    }
    if (!g.any(rot)) {
#ifdef IFMM_JACOBI_STATS
      IFMM_JACOBI_STATS(sweep + 1, n, g.rank() == 0);
#endif
      break;
    }
  }
  for (int c = warp; c < n; c += nw) {
    const double* x = A + (size_t)c * lda;
    double s = 0.0;
    for (int i = lane; i < m; i += 32) s += x[i] * x[i];
    s = warp_sum(s);
    if (lane == 0) sig[c] = sqrt(s);
  }
  g.sync();
  for (int c = g.rank(); c < n; c += g.size()) {
    int rank = 0;
    const double sc = sig[c];
    for (int o = 0; o < n; o++) rank += (sig[o] > sc) || (sig[o] == sc && o < c);
    ord[rank] = c;
  }
  g.sync();
}

// Smallest r with s[r]/s[0] < tol (s sorted decreasing); ifmm/lowrank.py:137-144
__device__ inline int trunc_rank_dev(const double* sig, const int* ord, int n, double tol) {
  if (n == 0) return 0;
  const double s0 = sig[ord[0]];
  if (s0 == 0.0) return 0;
  if (tol <= 0.0) return n;
  for (int r = 0; r < n; r++)
    if (sig[ord[r]] / s0 < tol) return r;
  return n;
}

// ------------------------------------------------------------- ACA
// Partially pivoted ACA of F (m x n; F(a,b) = trans ? F[b + a*ld] : F[a + b*ld])
// following ifmm/lowrank.py:174-263: probe rows (seeded table), residual
// row/column crosses, running Frobenius estimate, 3-strike tiny-pivot rule.
// Crosses are stored as columns of Uc (m x kmax, ld m) and Vc (n x kmax, ld n).
// Returns number of crosses; *converged per the reference's flag.
// scratch: rr (n), cc (m), usedr (m ints), usedc (n ints), dots (2*kmax).
struct AcaOut {
  int k;
  int converged;
};

__device__ inline double Fat(const double* F, int ld, int trans, int a, int b) {
  return trans ? F[b + (size_t)a * ld] : F[a + (size_t)b * ld];
}

// numpy's PCG64 (the reference's np.random.default_rng(0) stream, continued
// after the probe-row draw): 128-bit LCG step, XSL-RR output, 32-bit draws
// buffered from 64-bit outputs, and Generator.integers(0, k)'s Lemire bounded
// draw.  Every thread steps its own copy identically.
struct Pcg64 {
  unsigned long long shi, slo, ihi, ilo;
  unsigned long long has, u;
  __device__ unsigned long long next64() {
    const unsigned long long mhi = 0x2360ed051fc65da4ull, mlo = 0x4385df649fccf645ull;
    const unsigned long long lo = slo * mlo;
    const unsigned long long hi = __umul64hi(slo, mlo) + slo * mhi + shi * mlo;
    slo = lo + ilo;
    shi = hi + ihi + (slo < lo ? 1ull : 0ull);
    const unsigned long long x = shi ^ slo;
    const unsigned r = unsigned(shi >> 58);
    return (x >> r) | (x << ((64u - r) & 63u));
  }
  __device__ unsigned next32() {
    if (has) {
      has = 0;
      return unsigned(u);
    }
    const unsigned long long v = next64();
    has = 1;
    u = v >> 32;
    return unsigned(v & 0xffffffffull);
  }
  // Generator.integers(0, k), k <= 2^32 (rng.choice over a list of k rows)
  __device__ unsigned bounded(unsigned k) {
    const unsigned rng = k - 1;
    if (rng == 0) return 0;
    const unsigned long long ex = (unsigned long long)rng + 1ull;
    unsigned long long mm = (unsigned long long)next32() * ex;
    unsigned long long left = mm & 0xffffffffull;
    if (left < ex) {
      const unsigned long long thr = (0xffffffffull - rng) % ex;
      while (left < thr) {
        mm = (unsigned long long)next32() * ex;
        left = mm & 0xffffffffull;
      }
    }
    return unsigned(mm >> 32);
  }
};

// probes: one row of the ACA probe table (ACA_PROBE_STRIDE ints): the 10
// probe rows, then the PCG64 state after drawing them (6 x 64 bits)
template <class G>
__device__ inline AcaOut g_aca(const G& g, const double* F, int ld, int trans, int m, int n, double tol,
                                 const int* probes, int nprobe, double* Uc, double* Vc, int kmax, double* rr,
                                 double* cc, int* usedr, int* usedc, double* dots, double* Gu = nullptr,
                                 double* Gv = nullptr, int ldg = 0) {
  // Gu/Gv (optional, ld ldg): Gram matrices U_c^T U_c and V_c^T V_c of the
  // crosses, filled from the products the Frobenius estimate computes anyway
  const int lane = g.lane(), warp = g.warp(), nw = g.nwarps();
  const int full = min(m, n);
  AcaOut out{0, 0};
  if (m == 0 || n == 0) {
    out.converged = 0;
    return out;
  }
  for (int i = g.rank(); i < m; i += g.size()) usedr[i] = 0;
  for (int j = g.rank(); j < n; j += g.size()) usedc[j] = 0;
  // first row: probe with the largest max-abs entry (first in probe order on ties)
  int next;
  {
    // the probe row with the largest max-abs entry (first in probe order on
    // ties): all probe maxima in one pass and one group reduction
    double pm[10];
#pragma unroll
    for (int t = 0; t < 10; t++) pm[t] = -1.0;
#pragma unroll
    for (int t = 0; t < 10; t++)
      if (t < nprobe) {
        const int i = probes[t];
        for (int j = g.rank(); j < n; j += g.size()) pm[t] = fmax(pm[t], fabs(Fat(F, ld, trans, i, j)));
        for (int o = 16; o > 0; o >>= 1) pm[t] = fmax(pm[t], __shfl_xor_sync(0xffffffffu, pm[t], o));
      }
    g.max10(pm, nprobe);
    double best = -1.0;
    int bi = probes[0];
    for (int t = 0; t < nprobe; t++)
      if (pm[t] > best) {
        best = pm[t];
        bi = probes[t];
      }
    next = bi;  // identical in every thread
  }
  int k = 0, strikes = 0, nused = 0;
  double nsq = 0.0;
  bool done = false;
  Pcg64 rng;
  {
    const unsigned long long* w = reinterpret_cast<const unsigned long long*>(probes + 10);
    rng = Pcg64{w[0], w[1], w[2], w[3], w[4], w[5]};
  }
  const int kcap = min(full, kmax);
  while (k < kcap) {
    const int i = next;
    if (g.rank() == 0) usedr[i] = 1;
    nused++;
    // residual row (sequential subtraction over crosses, as the reference)
    for (int j = g.rank(); j < n; j += g.size()) {
      double v = Fat(F, ld, trans, i, j);
      for (int t = 0; t < k; t++) v = __dsub_rn(v, __dmul_rn(Uc[i + (size_t)t * m], Vc[j + (size_t)t * n]));
      rr[j] = usedc[j] ? 0.0 : v;
    }
    g.sync();
    ArgMax am{-1.0, -1};
    for (int j = g.rank(); j < n; j += g.size()) am = argmax_merge(am, ArgMax{fabs(rr[j]), j});
    am = g.argmax(am);
    const int j = am.i;
    const double piv = rr[j];
    const double tiny = nsq > 0.0 ? 1e-15 * sqrt(nsq) : 1e-300;
    if (fabs(piv) <= tiny) {
      strikes++;
      if (strikes >= 3 || nused >= m) {
        done = true;
        break;
      }
      // the reference's random restart row (ifmm/lowrank.py:224-226):
      // rng.choice over the unused rows in ascending order, drawn from the
      // same PCG64 stream -> the idx-th unused row
      const unsigned idx = rng.bounded(unsigned(m - nused));
      ArgMax lo{-1.0, -1};
      if (g.rank() == 0) {
        unsigned c = 0;
        for (int r = 0; r < m; r++)
          if (!usedr[r] && c++ == idx) {
            lo = ArgMax{1.0, r};
            break;
          }
      }
      lo = g.argmax(lo);
      next = lo.i;
      if (next < 0) {
        done = true;
        break;
      }
      continue;
    }
    strikes = 0;
    if (g.rank() == 0) usedc[j] = 1;
    // residual column, new cross
    double* u = Uc + (size_t)k * m;
    double* v = Vc + (size_t)k * n;
    for (int r = g.rank(); r < m; r += g.size()) {
      double x = Fat(F, ld, trans, r, j);
      for (int t = 0; t < k; t++) x = __dsub_rn(x, __dmul_rn(Vc[j + (size_t)t * n], Uc[r + (size_t)t * m]));
      u[r] = x / piv;
    }
    for (int c = g.rank(); c < n; c += g.size()) v[c] = rr[c];
    g.sync();
    // one combined reduction: ||u||^2, ||v||^2, the next row (largest |u|
    // among unused rows) and the cross terms |u.u_t||v.v_t| of the estimate
    double su = 0.0, sv = 0.0;
    ArgMax nx{-1.0, -1};
    for (int r = g.rank(); r < m; r += g.size()) {
      su += u[r] * u[r];
      const double a = (usedr[r] || r == i) ? -1.0 : fabs(u[r]);
      nx = argmax_merge(nx, ArgMax{a, r});
    }
    for (int c = g.rank(); c < n; c += g.size()) sv += v[c] * v[c];
    su = warp_sum(su);
    sv = warp_sum(sv);
    nx = warp_argmax(nx);
    for (int t = warp; t < k; t += nw) {
      double du = 0.0, dv = 0.0;
      const double* ut = Uc + (size_t)t * m;
      const double* vt = Vc + (size_t)t * n;
      for (int r = lane; r < m; r += 32) du += u[r] * ut[r];
      for (int c = lane; c < n; c += 32) dv += v[c] * vt[c];
      du = warp_sum(du);
      dv = warp_sum(dv);
      if (lane == 0) {
        dots[t] = fabs(du) * fabs(dv);
        if (Gu) {
          Gu[t + (size_t)k * ldg] = Gu[k + (size_t)t * ldg] = du;
          Gv[t + (size_t)k * ldg] = Gv[k + (size_t)t * ldg] = dv;
        }
      }
    }
    g.combine(su, sv, nx);  // also publishes dots[]
    if (Gu && g.rank() == 0) {
      Gu[k + (size_t)k * ldg] = su;
      Gv[k + (size_t)k * ldg] = sv;
    }
    const double csq = su * sv;
    if (k > 0) {
      double cross = 0.0;
      for (int t = 0; t < k; t++) cross += dots[t];
      nsq += csq + 2.0 * cross;
    } else {
      nsq = csq;
    }
    k++;
    if (tol > 0.0 && csq <= tol * tol * nsq) {
      done = true;
      break;
    }
    if (nx.i < 0 || nx.a < 0.0) {
      done = true;
      break;
    }
    next = nx.i;
  }
  g.sync();
  out.k = k;
  out.converged = done ? 1 : 0;
  // not converged below full rank because of the kmax cap -> report as not converged
  return out;
}

// CTA-wide entry points (basis construction, test hooks)
__device__ inline void cta_gemm(int rows, int cols, int kk, double alpha, const double* A, int lda, bool ta,
                                const double* B, int ldb, bool tb, double beta, double* Y, int ldy, CtaShared& sh) {
  g_gemm(CtaGroup{sh}, rows, cols, kk, alpha, A, lda, ta, B, ldb, tb, beta, Y, ldy);
}
__device__ inline void cta_qr(double* A, int m, int k, int lda, double* R, double* Q, int ldq, double* vv,
                              CtaShared& sh) {
  g_qr(CtaGroup{sh}, A, m, k, lda, R, Q, ldq, vv);
}
__device__ inline void cta_jacobi(double* A, int m, int n, int lda, double* V, int ldv, double* sig, int* ord,
                                  CtaShared& sh, int max_sweeps = 40) {
  g_jacobi(CtaGroup{sh}, A, m, n, lda, V, ldv, sig, ord, max_sweeps);
}
__device__ inline AcaOut cta_aca(const double* F, int ld, int trans, int m, int n, double tol, const int* probes,
                                 int nprobe, double* Uc, double* Vc, int kmax, double* rr, double* cc, int* usedr,
                                 int* usedc, double* dots, CtaShared& sh) {
  return g_aca(CtaGroup{sh}, F, ld, trans, m, n, tol, probes, nprobe, Uc, Vc, kmax, rr, cc, usedr, usedc, dots);
}

}  // namespace ifmm
