// CTA-cooperative dense linear algebra on column-major matrices held in global
// (L1/L2-resident) scratch: Householder QR, one-sided Jacobi SVD, partially
// pivoted ACA.  Every routine must be called by all threads of the block.
// Used by the fill-in compression kernel (one CTA per pivot) and the
// Chebyshev basis construction (one CTA per cluster).
#pragma once
#include "common.cuh"

namespace ifmm {

struct CtaShared {
  double red[32];
  ArgMax am[32];
  int flag;
  int ival[4];
  double dval[4];
};

// ------------------------------------------------------------- small helpers
// CTA-cooperative DMMA GEMM (mma.sync.m8n8k4.f64): every warp owns 16x16
// output tiles (2x2 fragments); fragments are loaded straight from L1/L2.
// One DMMA does 512 flops for 2 loads per lane, vs 2 flops per 2 loads for a
// scalar loop -- the projections and deltas of the compression are otherwise
// L1-throughput bound.
template <bool TA, bool TB>
__device__ inline void cta_mma_gemm(int rows, int cols, int kk, double alpha, const double* __restrict__ A, int lda,
                                    const double* __restrict__ B, int ldb, double beta, double* Y, int ldy) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
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
  __syncthreads();
}

// Y(rows x cols, ldy) = alpha * op(A) * op(B) + beta*Y for the small products
// inside compression; DMMA tiles when the shape is worth it.
// opA: A is (rows x kk) if !ta else stored (kk x rows).
__device__ inline void cta_gemm(int rows, int cols, int kk, double alpha, const double* A, int lda, bool ta,
                                const double* B, int ldb, bool tb, double beta, double* Y, int ldy) {
  if (rows >= 8 && cols >= 8 && kk >= 8) {
    if (ta) {
      if (tb) cta_mma_gemm<true, true>(rows, cols, kk, alpha, A, lda, B, ldb, beta, Y, ldy);
      else cta_mma_gemm<true, false>(rows, cols, kk, alpha, A, lda, B, ldb, beta, Y, ldy);
    } else {
      if (tb) cta_mma_gemm<false, true>(rows, cols, kk, alpha, A, lda, B, ldb, beta, Y, ldy);
      else cta_mma_gemm<false, false>(rows, cols, kk, alpha, A, lda, B, ldb, beta, Y, ldy);
    }
    return;
  }
  if (ta && !tb) {
    // Y = A^T B: both operands are read down contiguous columns -> one warp per
    // output, lanes stride the contraction (coalesced), warp-shuffle reduction
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
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
    __syncthreads();
    return;
  }
  for (int e = threadIdx.x; e < rows * cols; e += blockDim.x) {
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
  __syncthreads();
}

// X(n x k) -= U (U^T X), U n x r.  Scratch E >= r*k.
__device__ inline void cta_project_out(double* X, int ldx, int n, int k, const double* U, int ldu, int r,
                                       double* E) {
  if (r == 0 || k == 0) return;
  cta_gemm(r, k, n, 1.0, U, ldu, true, X, ldx, false, 0.0, E, r);
  cta_gemm(n, k, r, -1.0, U, ldu, false, E, r, false, 1.0, X, ldx);
}

// ------------------------------------------------------------- Householder QR
// A (m x k, lda) is overwritten by the reflectors.  Outputs R (k x k, ld k,
// upper) and, if Q != nullptr, the thin Q (m x k, ldq).  vv: scratch >= k.
__device__ inline void cta_qr(double* A, int m, int k, int lda, double* R, double* Q, int ldq, double* vv,
                              CtaShared& sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = 0; j < k && j < m; j++) {
    double* x = A + j + (size_t)j * lda;
    const int len = m - j;
    double s = 0.0;
    for (int i = threadIdx.x; i < len; i += blockDim.x) s += x[i] * x[i];
    s = block_sum(s, sh.red);
    const double alpha = sqrt(s);
    const double x0 = x[0];
    double beta = 0.0, vtv = 0.0;
    if (alpha > 0.0) {
      beta = x0 >= 0.0 ? -alpha : alpha;
      // v = x - beta e1 ; vtv = s - x0^2 + (x0-beta)^2
      vtv = s - x0 * x0 + (x0 - beta) * (x0 - beta);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      x[0] = x0 - beta;
      vv[j] = vtv;
      R[j + (size_t)j * k] = alpha > 0.0 ? beta : x0;
    }
    __syncthreads();
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
    __syncthreads();
  }
  // R strictly-upper part
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
    const int i = e % k, c = e / k;
    if (i < c) R[i + (size_t)c * k] = (i < m) ? A[i + (size_t)c * lda] : 0.0;
    else if (i > c) R[i + (size_t)c * k] = 0.0;
    else if (i >= m) R[i + (size_t)c * k] = 0.0;
  }
  __syncthreads();
  if (Q == nullptr) return;
  for (int e = threadIdx.x; e < m * k; e += blockDim.x) {
    const int i = e % m, c = e / m;
    Q[i + (size_t)c * ldq] = (i == c) ? 1.0 : 0.0;
  }
  __syncthreads();
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
    __syncthreads();
  }
}

// ------------------------------------------------------------- Jacobi SVD
// One-sided (Hestenes) Jacobi on A (m x n, lda): on exit the columns of A are
// mutually orthogonal (A_out = A V), V (n x n, ldv) accumulates the rotations
// if non-null, sig[j] = ||A_out(:,j)||, ord[0..n) = column indices sorted by
// decreasing sig (ties: lower index first).  Round-robin pairing; warps own
// disjoint column pairs.
__device__ inline void cta_jacobi(double* A, int m, int n, int lda, double* V, int ldv, double* sig, int* ord,
                                  CtaShared& sh, int max_sweeps = 40) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (V)
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) V[(e % n) + (size_t)(e / n) * ldv] = (e % n == e / n);
  const int nn = n + (n & 1);  // even number of players (dummy = n)
  __syncthreads();
  for (int sweep = 0; sweep < max_sweeps && n > 1; sweep++) {
    if (threadIdx.x == 0) sh.flag = 0;
    __syncthreads();
    for (int round = 0; round < nn - 1; round++) {
      for (int pr = warp; pr < nn / 2; pr += nw) {
        // circle method: player nn-1 fixed, others rotate
        int a = (pr == 0) ? nn - 1 : (round + pr) % (nn - 1);
        int b = (round + nn - 1 - pr) % (nn - 1);
        if (pr == 0) b = round % (nn - 1);
        if (a >= n || b >= n || a == b) continue;
        if (a > b) { int t = a; a = b; b = t; }
        double* x = A + (size_t)a * lda;
        double* y = A + (size_t)b * lda;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int i = lane; i < m; i += 32) {
          const double xi = x[i], yi = y[i];
          al += xi * xi;
          be += yi * yi;
          ga += xi * yi;
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum(ga);
        if (ga == 0.0 || fabs(ga) <= 1e-15 * sqrt(al * be)) continue;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        // a rotation below rounding level changes nothing: columns of very
        // different norms otherwise keep |ga|/sqrt(al*be) ~ eps*sqrt(al/be)
        // and never pass the relative test
        if (fabs(t) < 1e-16) continue;
        const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        for (int i = lane; i < m; i += 32) {
          const double xi = x[i], yi = y[i];
          x[i] = c * xi - s * yi;
          y[i] = s * xi + c * yi;
        }
        if (V) {
          double* vx = V + (size_t)a * ldv;
          double* vy = V + (size_t)b * ldv;
          for (int i = lane; i < n; i += 32) {
            const double xi = vx[i], yi = vy[i];
            vx[i] = c * xi - s * yi;
            vy[i] = s * xi + c * yi;
          }
        }
        if (lane == 0) sh.flag = 1;
      }
      __syncthreads();
    }
    const int rotated = sh.flag;
    __syncthreads();
    if (!rotated) {
#ifdef IFMM_JACOBI_STATS
      IFMM_JACOBI_STATS(sweep + 1, n);
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
  __syncthreads();
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    int rank = 0;
    const double sc = sig[c];
    for (int o = 0; o < n; o++) rank += (sig[o] > sc) || (sig[o] == sc && o < c);
    ord[rank] = c;
  }
  __syncthreads();
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

__device__ inline AcaOut cta_aca(const double* F, int ld, int trans, int m, int n, double tol,
                                 const int* probes, int nprobe, double* Uc, double* Vc, int kmax, double* rr,
                                 double* cc, int* usedr, int* usedc, double* dots, CtaShared& sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int full = min(m, n);
  AcaOut out{0, 0};
  if (m == 0 || n == 0) {
    out.converged = 0;
    return out;
  }
  for (int i = threadIdx.x; i < m; i += blockDim.x) usedr[i] = 0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) usedc[j] = 0;
  // first row: probe with the largest max-abs entry (first in probe order on ties)
  if (threadIdx.x == 0) sh.ival[0] = probes[0];
  __syncthreads();
  {
    double best = -1.0;
    int bi = probes[0];
    for (int t = 0; t < nprobe; t++) {
      const int i = probes[t];
      ArgMax am{-1.0, -1};
      for (int j = threadIdx.x; j < n; j += blockDim.x) am = argmax_merge(am, ArgMax{fabs(Fat(F, ld, trans, i, j)), j});
      am = block_argmax(am, sh.am);
      if (am.a > best) {
        best = am.a;
        bi = i;
      }
    }
    if (threadIdx.x == 0) sh.ival[0] = bi;
  }
  __syncthreads();
  int next = sh.ival[0];
  int k = 0, strikes = 0, nused = 0;
  double nsq = 0.0;
  bool done = false;
  const int kcap = min(full, kmax);
  while (k < kcap) {
    const int i = next;
    if (threadIdx.x == 0) usedr[i] = 1;
    nused++;
    // residual row (sequential subtraction over crosses, as the reference)
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      double v = Fat(F, ld, trans, i, j);
      for (int t = 0; t < k; t++) v = __dsub_rn(v, __dmul_rn(Uc[i + (size_t)t * m], Vc[j + (size_t)t * n]));
      rr[j] = usedc[j] ? 0.0 : v;
    }
    __syncthreads();
    ArgMax am{-1.0, -1};
    for (int j = threadIdx.x; j < n; j += blockDim.x) am = argmax_merge(am, ArgMax{fabs(rr[j]), j});
    am = block_argmax(am, sh.am);
    const int j = am.i;
    const double piv = rr[j];
    const double tiny = nsq > 0.0 ? 1e-15 * sqrt(nsq) : 1e-300;
    if (fabs(piv) <= tiny) {
      strikes++;
      if (strikes >= 3 || nused >= m) {
        done = true;
        break;
      }
      // deterministic substitute for the reference's random restart row:
      // the lowest-index unused row
      ArgMax lo{-1.0, -1};
      for (int r = threadIdx.x; r < m; r += blockDim.x)
        if (!usedr[r]) lo = argmax_merge(lo, ArgMax{1.0, r});
      lo = block_argmax(lo, sh.am);
      next = lo.i;
      if (next < 0) {
        done = true;
        break;
      }
      continue;
    }
    strikes = 0;
    if (threadIdx.x == 0) usedc[j] = 1;
    // residual column, new cross
    double* u = Uc + (size_t)k * m;
    double* v = Vc + (size_t)k * n;
    for (int r = threadIdx.x; r < m; r += blockDim.x) {
      double x = Fat(F, ld, trans, r, j);
      for (int t = 0; t < k; t++) x = __dsub_rn(x, __dmul_rn(Vc[j + (size_t)t * n], Uc[r + (size_t)t * m]));
      u[r] = x / piv;
    }
    for (int c = threadIdx.x; c < n; c += blockDim.x) v[c] = rr[c];
    __syncthreads();
    double su = 0.0, sv = 0.0;
    for (int r = threadIdx.x; r < m; r += blockDim.x) su += u[r] * u[r];
    for (int c = threadIdx.x; c < n; c += blockDim.x) sv += v[c] * v[c];
    su = block_sum(su, sh.red);
    sv = block_sum(sv, sh.red);
    const double csq = su * sv;
    if (k > 0) {
      for (int t = warp; t < k; t += nw) {
        double du = 0.0, dv = 0.0;
        const double* ut = Uc + (size_t)t * m;
        const double* vt = Vc + (size_t)t * n;
        for (int r = lane; r < m; r += 32) du += u[r] * ut[r];
        for (int c = lane; c < n; c += 32) dv += v[c] * vt[c];
        du = warp_sum(du);
        dv = warp_sum(dv);
        if (lane == 0) dots[t] = fabs(du) * fabs(dv);
      }
      __syncthreads();
      double cross = 0.0;
      for (int t = 0; t < k; t++) cross += dots[t];
      nsq += csq + 2.0 * cross;
      __syncthreads();
    } else {
      nsq = csq;
    }
    k++;
    if (tol > 0.0 && csq <= tol * tol * nsq) {
      done = true;
      break;
    }
    ArgMax nx{-1.0, -1};
    for (int r = threadIdx.x; r < m; r += blockDim.x) {
      const double a = (usedr[r] || r == i) ? -1.0 : fabs(u[r]);
      nx = argmax_merge(nx, ArgMax{a, r});
    }
    nx = block_argmax(nx, sh.am);
    if (nx.i < 0 || nx.a < 0.0) {
      done = true;
      break;
    }
    next = nx.i;
  }
  __syncthreads();
  out.k = k;
  out.converged = done ? 1 : 0;
  // not converged below full rank because of the kmax cap -> report as not converged
  return out;
}

}  // namespace ifmm
