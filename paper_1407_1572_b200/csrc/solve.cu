// Solve with the factored IFMM (ifmm/solver.py:549-626), level-wise and
// batch-parallel: for every colour batch one CTA per eliminated cluster.
//   forward : g_i = Sinv_nn b_i ; v[pos] -= X_top^T b_i     (z rows start at 0)
//   top     : y = T^-1 v_top
//   backward: x_i = g_i - X_top v[pos]     (batches and levels in reverse)
// Using X_top = (S^-1 C)_top for both sweeps (S symmetric) means a record is
// only Sinv_nn (n x n) + X_top (n x w): the solve streams each record twice
// and is HBM-bound.  The GEMVs keep all warps busy: warps split the columns,
// lanes own rows with register accumulators, partial sums meet in shared
// memory.  Vectors are (positions x nrhs) row-major; right-hand sides are
// processed in chunks of RC; a level's y slots alias the next level's x slots.
#include <algorithm>
#include <cmath>
#include <thread>

#include "comm.cuh"
#include "core.cuh"
#include "gemm.cuh"

namespace ifmm {

void launch_permute(const double* in, double* out, const int64_t* perm, int64_t n, int nrhs, bool inverse,
                    cudaStream_t s);

constexpr int SB = 256;       // threads per solve CTA
constexpr int SWARPS = SB / 32;
constexpr int RCMAX = 4;      // right-hand sides per pass (RC = 1 for a single rhs)
constexpr int MAXJ = 8;       // rows per lane per pass (256 rows per row block)

// y[t, q] (t < n, q < nq) = sum_c A[t + c*lda] x(c, q)  (A column-major n x w);
// x(c, q) from the `xat` accessor, result written by `emit(t, q, value)`.
template <int RC, class XAt, class Emit>
__device__ inline void cta_gemv_cols(const double* __restrict__ A, int n, int w, size_t lda, XAt xat, int nq,
                                     double* red, Emit emit) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int t0 = 0; t0 < n; t0 += 32 * MAXJ) {
    double acc[MAXJ][RC];
#pragma unroll
    for (int j = 0; j < MAXJ; j++)
#pragma unroll
      for (int q = 0; q < RC; q++) acc[j][q] = 0.0;
    // warps take chunks of 32 columns; the chunk's x values are fetched once
    // (lane u loads column cb+u) and broadcast with shuffles
    for (int cb = warp * 32; cb < w; cb += SWARPS * 32) {
      double xl[RC];
#pragma unroll
      for (int q = 0; q < RC; q++) xl[q] = (cb + lane < w && q < nq) ? xat(cb + lane, q) : 0.0;
      const int cmax = min(32, w - cb);
#pragma unroll 8
      for (int u = 0; u < cmax; u++) {
        const double* col = A + (size_t)(cb + u) * lda;
        double xv[RC];
#pragma unroll
        for (int q = 0; q < RC; q++) xv[q] = __shfl_sync(0xffffffffu, xl[q], u);
#pragma unroll
        for (int j = 0; j < MAXJ; j++) {
          const int t = t0 + lane + 32 * j;
          if (t < n) {
            const double a = col[t];
#pragma unroll
            for (int q = 0; q < RC; q++) acc[j][q] = fma(a, xv[q], acc[j][q]);
          }
        }
      }
    }
    // cross-warp reduction: red[warp][row][q]
#pragma unroll
    for (int j = 0; j < MAXJ; j++) {
      const int tl = lane + 32 * j;
#pragma unroll
      for (int q = 0; q < RC; q++) if (t0 + tl < n) red[(tl * SWARPS + warp) * RC + q] = acc[j][q];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 32 * MAXJ * nq; e += SB) {
      const int tl = e / nq, q = e % nq;
      const int t = t0 + tl;
      if (t < n) {
        double s = 0.0;
        for (int w2 = 0; w2 < SWARPS; w2++) s += red[(tl * SWARPS + w2) * RC + q];
        emit(t, q, s);
      }
    }
    __syncthreads();
  }
}

// Records are split over gridDim.y CTAs (coarse levels have few, large
// records): chunk y of the forward sweep computes rows [r0, r1) of Sinv b and
// columns [c0, c1) of X_top^T b; chunk y of the backward sweep rows [r0, r1)
// of x.  Every output has exactly one writer (deterministic).
__device__ __forceinline__ void chunk_range(int len, int y, int ny, int gran, int& lo, int& hi) {
  const int per = ((len + ny - 1) / ny + gran - 1) / gran * gran;
  lo = min(len, y * per);
  hi = min(len, lo + per);
}

template <int RC>
__global__ void __launch_bounds__(SB, RC == 1 ? 4 : 2) solve_fwd_kernel(const RecordH* __restrict__ recs, int rec0,
                                                       const int64_t* __restrict__ g_off, double* V, double* G,
                                                       int nrhs, int red_rows) {
  extern __shared__ double sm[];
  double* red = sm;                         // min(maxn, 256) x SWARPS x RC
  double* bsh = red + red_rows * SWARPS * RC;  // n x RC
  const RecordH R = recs[blockIdx.x];
  const int n = R.n, w = R.w;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int r0, r1, c0, c1;
  chunk_range(n, blockIdx.y, gridDim.y, 32, r0, r1);
  chunk_range(w, blockIdx.y, gridDim.y, 8, c0, c1);
  double* g = G + g_off[rec0 + blockIdx.x] * nrhs;
  // segment of W lanes per X_top column (short columns: several per warp)
  const int W = n > 128 ? 32 : (n > 64 ? 16 : 8);
  const int seg = lane / W, sl = lane & (W - 1), spw = 32 / W;
  for (int q0 = 0; q0 < nrhs; q0 += RC) {
    const int nq = min(RC, nrhs - q0);
    for (int e = threadIdx.x; e < n * RC; e += SB) {
      const int c = e / RC, q = e % RC;
      bsh[e] = q < nq ? V[(R.xoff + c) * nrhs + q0 + q] : 0.0;
    }
    __syncthreads();
    // g[r0:r1] = Sinv[r0:r1, :] b
    if (r1 > r0)
      cta_gemv_cols<RC>(R.sinv + r0, r1 - r0, n, (size_t)n, [&](int c, int q) { return bsh[c * RC + q]; }, nq, red,
                    [&](int t, int q, double v) { g[(size_t)(r0 + t) * nrhs + q0 + q] = v; });
    // v[pos[c]] -= X_top(:, c)^T b for c in [c0, c1)
    for (int cb = c0 + warp * spw; cb < c1; cb += SWARPS * spw) {
      const int c = cb + seg;
      const bool ok = c < c1;
      const double* x = R.xtop + (size_t)(ok ? c : c0) * n;
      double s[RC];
#pragma unroll
      for (int q = 0; q < RC; q++) s[q] = 0.0;
      if (ok)
#pragma unroll 8
        for (int t = sl; t < n; t += W) {
          const double a = x[t];
#pragma unroll
          for (int q = 0; q < RC; q++)
            if (q < nq) s[q] = fma(a, bsh[t * RC + q], s[q]);
        }
#pragma unroll
      for (int q = 0; q < RC; q++)
        if (q < nq)
          for (int o = W >> 1; o > 0; o >>= 1) s[q] += __shfl_xor_sync(0xffffffffu, s[q], o);
      if (ok && sl < nq) {
        double sv = s[0];
#pragma unroll
        for (int q = 1; q < RC; q++)
          if (sl == q) sv = s[q];
        V[(int64_t)R.pos[c] * nrhs + q0 + sl] -= sv;
      }
    }
    __syncthreads();
  }
}

// Single right-hand side forward sweep.  S (hence S^-1 and its block
// S^-1_nn) is symmetric, so g = S^-1_nn b is a set of column dots as well:
// the record [S^-1_nn | X_top] is one n x (n + w) column block and every
// output is the dot of one column with b -- W-lane segments per column, no
// cross-warp reduction, one barrier.  Chunk y of gridDim.y owns a range of
// the n + w columns.
__global__ void __launch_bounds__(SB, 3) solve_fwd1_kernel(const RecordH* __restrict__ recs, int rec0,
                                                           const int64_t* __restrict__ g_off, double* V, double* G) {
  extern __shared__ double sm[];
  double* bsh = sm;  // n
  const RecordH R = recs[blockIdx.x];
  const int n = R.n, w = R.w, nc = n + w;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int c0, c1;
  chunk_range(nc, blockIdx.y, gridDim.y, 8, c0, c1);
  if (c1 <= c0) return;
  double* g = G + g_off[rec0 + blockIdx.x];
  for (int e = threadIdx.x; e < n; e += SB) bsh[e] = V[R.xoff + e];
  __syncthreads();
  const int W = n > 128 ? 32 : (n > 64 ? 16 : 8);
  const int seg = lane / W, sl = lane & (W - 1), spw = 32 / W;
  // two columns per segment and step: 16 loads per lane in flight (the sweep
  // is latency-bound on long-scoreboard stalls with one)
  const int stride = SWARPS * spw;
  auto colp = [&](int c) { return c < n ? R.sinv + (size_t)c * n : R.xtop + (size_t)(c - n) * n; };
  for (int cb = c0 + warp * spw; cb < c1; cb += 2 * stride) {
    const int c = cb + seg, c2 = c + stride;
    const bool ok = c < c1, ok2 = c2 < c1;
    const double* x = colp(ok ? c : c0);
    const double* x2 = colp(ok2 ? c2 : c0);
    // all of the lane's elements of both columns in flight at once (W is
    // chosen so that 8 W >= n up to n = 256), streaming loads: read once
    double a[8], a2[8];
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int t = sl + u * W;
      a[u] = (ok && t < n) ? __ldcs(x + t) : 0.0;
      a2[u] = (ok2 && t < n) ? __ldcs(x2 + t) : 0.0;
    }
    double s0 = 0.0, s1 = 0.0, r0 = 0.0, r1 = 0.0;
#pragma unroll
    for (int u = 0; u < 8; u += 2) {
      const int t = sl + u * W;
      if (t < n) {
        const double bt = bsh[t];
        s0 = fma(a[u], bt, s0);
        r0 = fma(a2[u], bt, r0);
      }
      if (t + W < n) {
        const double bt = bsh[t + W];
        s1 = fma(a[u + 1], bt, s1);
        r1 = fma(a2[u + 1], bt, r1);
      }
    }
    for (int t = sl + 8 * W; t < n; t += W) {
      if (ok) s0 = fma(__ldcs(x + t), bsh[t], s0);
      if (ok2) r0 = fma(__ldcs(x2 + t), bsh[t], r0);
    }
    double sv = s0 + s1, sv2 = r0 + r1;
    for (int o = W >> 1; o > 0; o >>= 1) {
      sv += __shfl_xor_sync(0xffffffffu, sv, o);
      sv2 += __shfl_xor_sync(0xffffffffu, sv2, o);
    }
    if (sl == 0) {
      if (ok) {
        if (c < n) g[c] = sv;
        else V[(int64_t)R.pos[c - n]] -= sv;
      }
      if (ok2) {
        if (c2 < n) g[c2] = sv2;
        else V[(int64_t)R.pos[c2 - n]] -= sv2;
      }
    }
  }
}

template <int RC>
__global__ void __launch_bounds__(SB, RC == 1 ? 4 : 2) solve_bwd_kernel(const RecordH* __restrict__ recs, int rec0,
                                                       const int64_t* __restrict__ g_off, double* V,
                                                       const double* G, int nrhs, int red_rows) {
  extern __shared__ double sm[];
  double* red = sm;                         // min(maxn, 256) x SWARPS x RC
  const RecordH R = recs[blockIdx.x];
  const int n = R.n, w = R.w;
  int r0, r1;
  chunk_range(n, blockIdx.y, gridDim.y, 32, r0, r1);
  if (r1 <= r0) return;
  const double* g = G + g_off[rec0 + blockIdx.x] * nrhs;
  for (int q0 = 0; q0 < nrhs; q0 += RC) {
    const int nq = min(RC, nrhs - q0);
    // partner values are gathered on the fly (the coupling width can exceed shared memory)
    cta_gemv_cols<RC>(R.xtop + r0, r1 - r0, w, (size_t)n,
                  [&](int c, int q) { return V[(int64_t)R.pos[c] * nrhs + q0 + q]; }, nq, red,
                  [&](int t, int q, double v) {
                    V[(R.xoff + r0 + t) * nrhs + q0 + q] = g[(size_t)(r0 + t) * nrhs + q0 + q] - v;
                  });
  }
}

// Single right-hand side backward sweep: x = g - X_top v[pos] for the rows
// [r0, r1) of chunk blockIdx.y.  Lanes own rows (J per lane), warps split the
// columns; CB columns of loads are issued before their FMAs (streaming loads,
// J x CB in flight per lane) -- the generic GEMV keeps too few bytes in flight
// for the 64-row leaf records.  Partial sums meet in shared memory.
template <int J>
__global__ void __launch_bounds__(SB, J <= 4 ? 3 : 2) solve_bwd1_kernel(const RecordH* __restrict__ recs, int rec0,
                                                                       const int64_t* __restrict__ g_off, double* V,
                                                                       const double* __restrict__ G) {
  constexpr int CB = J <= 2 ? 8 : (J <= 4 ? 4 : 2);
  extern __shared__ double red[];  // (32 J) x SWARPS
  const RecordH R = recs[blockIdx.x];
  const int n = R.n, w = R.w;
  int r0, r1;
  chunk_range(n, blockIdx.y, gridDim.y, 32, r0, r1);
  if (r1 <= r0) return;
  const double* g = G + g_off[rec0 + blockIdx.x];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int t0 = r0; t0 < r1; t0 += 32 * J) {
    double acc[J];
#pragma unroll
    for (int j = 0; j < J; j++) acc[j] = 0.0;
    for (int cb = warp * 32; cb < w; cb += SWARPS * 32) {
      const double xl = (cb + lane < w) ? V[(int64_t)R.pos[cb + lane]] : 0.0;
      const int cmax = min(32, w - cb);
      for (int u0 = 0; u0 < cmax; u0 += CB) {
        double a[CB][J];
#pragma unroll
        for (int u = 0; u < CB; u++) {
          const double* col = R.xtop + (size_t)(cb + u0 + u) * n;
#pragma unroll
          for (int j = 0; j < J; j++) {
            const int t = t0 + lane + 32 * j;
            a[u][j] = (u0 + u < cmax && t < r1) ? __ldcs(col + t) : 0.0;
          }
        }
#pragma unroll
        for (int u = 0; u < CB; u++) {
          const double xv = __shfl_sync(0xffffffffu, xl, (u0 + u) & 31);
#pragma unroll
          for (int j = 0; j < J; j++) acc[j] = fma(a[u][j], xv, acc[j]);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < J; j++) red[(lane + 32 * j) * SWARPS + warp] = acc[j];
    __syncthreads();
    for (int e = threadIdx.x; e < 32 * J && t0 + e < r1; e += SB) {
      double s = 0.0;
#pragma unroll
      for (int w2 = 0; w2 < SWARPS; w2++) s += red[e * SWARPS + w2];
      V[R.xoff + t0 + e] = g[t0 + e] - s;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ many rhs
// Multi-rhs sweeps as DMMA GEMMs: each record is read once
// per chunk of up to 32 right-hand sides instead of once per 4, which turns the
// HBM-bound sweeps compute-bound (8 flop/B at 32 rhs).  64 x 32 output tiles,
// 4 warps x (16 x 32), cp.async-staged operands (layouts as in gemm.cuh).
constexpr int MQ = 32;             // rhs per chunk
constexpr int QP = MQ + 4;         // pitch of the [k][q] operand tile (== 4 mod 16)
constexpr int MM_STAGES = 3;
constexpr int MM_A = GBM * KP;     // A tile doubles ([row][k], pitch KP)
constexpr int MM_B = GBK * QP;     // B tile doubles ([k][q], pitch QP)
constexpr size_t MM_SMEM = sizeof(double) * size_t(MM_STAGES) * (MM_A + MM_B);

__device__ __forceinline__ void mm_mma(const double* As, const double* Bs, double (&acc)[2][4][2], int warp,
                                       int lane) {
#pragma unroll
  for (int kk = 0; kk < GBK; kk += 4) {
    double fa[2], fb[4];
#pragma unroll
    for (int m = 0; m < 2; m++) fa[m] = As[(warp * 16 + m * 8 + (lane >> 2)) * KP + kk + (lane & 3)];
#pragma unroll
    for (int n = 0; n < 4; n++) fb[n] = Bs[(kk + (lane & 3)) * QP + n * 8 + (lane >> 2)];
#pragma unroll
    for (int m = 0; m < 2; m++)
#pragma unroll
      for (int n = 0; n < 4; n++)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[m][n][0]), "+d"(acc[m][n][1])
                     : "d"(fa[m]), "d"(fb[n]));
  }
}

// forward: Out = [S^-1_nn | X_top]^T B (rows c < n -> G, c >= n -> V[pos] -= ),
// B = V(xoff : xoff + n, q0 : q0 + nq).  grid (record, 64-row tile, rhs chunk)
__global__ void __launch_bounds__(GTHREADS) solve_fwd_mm_kernel(const RecordH* __restrict__ recs, int rec0,
                                                                const int64_t* __restrict__ g_off, double* V,
                                                                double* G, int nrhs) {
  extern __shared__ double msm[];
  const RecordH R = recs[blockIdx.x];
  const int n = R.n, w = R.w, nc = n + w;
  const int c0 = blockIdx.y * GBM;
  if (c0 >= nc || n == 0) return;
  const int q0 = blockIdx.z * MQ, nq = min(MQ, nrhs - q0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* g = G + g_off[rec0 + blockIdx.x] * nrhs;
  const double* Bv = V + R.xoff * nrhs + q0;
  auto load = [&](int st, int k0) {
    double* As = msm + (size_t)st * (MM_A + MM_B);
    double* Bs = As + MM_A;
#pragma unroll
    for (int e = 0; e < (GBM * GBK) / GTHREADS; e++) {  // A: column c of [S^-1 | X_top], k-contiguous
      const int cidx = tid + e * GTHREADS, k = cidx & (GBK - 1), r = cidx / GBK;
      const int c = c0 + r, gk = k0 + k;
      const bool ok = c < nc && gk < n;
      const double* src = c < n ? R.sinv + gk + (size_t)c * n : R.xtop + gk + (size_t)(c - n) * n;
      cp_async8(As + r * KP + k, src, ok);
    }
#pragma unroll
    for (int e = 0; e < (GBK * MQ) / GTHREADS; e++) {  // B: rows of V, q-contiguous
      const int cidx = tid + e * GTHREADS, q = cidx & (MQ - 1), k = cidx / MQ;
      const int gk = k0 + k;
      cp_async8(Bs + k * QP + q, Bv + (size_t)gk * nrhs + q, gk < n && q < nq);
    }
  };
  double acc[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; a++)
#pragma unroll
    for (int b = 0; b < 4; b++) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int nk = (n + GBK - 1) / GBK;
#pragma unroll
  for (int st = 0; st < MM_STAGES - 1; st++) {
    if (st < nk) load(st, st * GBK);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; kt++) {
    cp_async_wait<MM_STAGES - 2>();
    __syncthreads();
    if (kt + MM_STAGES - 1 < nk) load((kt + MM_STAGES - 1) % MM_STAGES, (kt + MM_STAGES - 1) * GBK);
    cp_async_commit();
    const double* As = msm + (size_t)(kt % MM_STAGES) * (MM_A + MM_B);
    mm_mma(As, As + MM_A, acc, warp, lane);
  }
  cp_async_wait<0>();
#pragma unroll
  for (int m = 0; m < 2; m++) {
    const int c = c0 + warp * 16 + m * 8 + (lane >> 2);
    if (c >= nc) continue;
    double* row = c < n ? g + (size_t)c * nrhs + q0 : V + (int64_t)R.pos[c - n] * nrhs + q0;
    const bool sub = c >= n;
    double old[8];
#pragma unroll
    for (int e = 0; e < 8; e++) {
      const int q = (e >> 1) * 8 + 2 * (lane & 3) + (e & 1);
      old[e] = (sub && q < nq) ? row[q] : 0.0;
    }
#pragma unroll
    for (int e = 0; e < 8; e++) {
      const int q = (e >> 1) * 8 + 2 * (lane & 3) + (e & 1);
      if (q < nq) row[q] = sub ? old[e] - acc[m][e >> 1][e & 1] : acc[m][e >> 1][e & 1];
    }
  }
}

// backward: x(t, q) = G(t, q) - sum_c X_top(t, c) V(pos[c], q).
// grid (record, 64-row tile of n, rhs chunk); K = w with row-gathered B
__global__ void __launch_bounds__(GTHREADS) solve_bwd_mm_kernel(const RecordH* __restrict__ recs, int rec0,
                                                                const int64_t* __restrict__ g_off, double* V,
                                                                const double* G, int nrhs) {
  extern __shared__ double msm[];
  const RecordH R = recs[blockIdx.x];
  const int n = R.n, w = R.w;
  const int t0 = blockIdx.y * GBM;
  if (t0 >= n) return;
  const int q0 = blockIdx.z * MQ, nq = min(MQ, nrhs - q0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* g = G + g_off[rec0 + blockIdx.x] * nrhs;
  auto load = [&](int st, int k0) {
    double* As = msm + (size_t)st * (MM_A + MM_B);
    double* Bs = As + MM_A;
#pragma unroll
    for (int e = 0; e < (GBM * GBK) / GTHREADS; e++) {  // A: X_top(t, c), t-contiguous -> stored [t][k]
      const int cidx = tid + e * GTHREADS, r = cidx & (GBM - 1), k = cidx / GBM;
      const int t = t0 + r, gk = k0 + k;
      cp_async8(As + r * KP + k, R.xtop + t + (size_t)gk * n, t < n && gk < w);
    }
#pragma unroll
    for (int e = 0; e < (GBK * MQ) / GTHREADS; e++) {  // B: V(pos[c], q)
      const int cidx = tid + e * GTHREADS, q = cidx & (MQ - 1), k = cidx / MQ;
      const int gk = k0 + k;
      const bool ok = gk < w && q < nq;
      const double* src = ok ? V + (int64_t)R.pos[gk] * nrhs + q0 + q : V;
      cp_async8(Bs + k * QP + q, src, ok);
    }
  };
  double acc[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; a++)
#pragma unroll
    for (int b = 0; b < 4; b++) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int nk = (w + GBK - 1) / GBK;
#pragma unroll
  for (int st = 0; st < MM_STAGES - 1; st++) {
    if (st < nk) load(st, st * GBK);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; kt++) {
    cp_async_wait<MM_STAGES - 2>();
    __syncthreads();
    if (kt + MM_STAGES - 1 < nk) load((kt + MM_STAGES - 1) % MM_STAGES, (kt + MM_STAGES - 1) * GBK);
    cp_async_commit();
    const double* As = msm + (size_t)(kt % MM_STAGES) * (MM_A + MM_B);
    mm_mma(As, As + MM_A, acc, warp, lane);
  }
  cp_async_wait<0>();
#pragma unroll
  for (int m = 0; m < 2; m++) {
    const int t = t0 + warp * 16 + m * 8 + (lane >> 2);
    if (t >= n) continue;
#pragma unroll
    for (int e = 0; e < 8; e++) {
      const int q = (e >> 1) * 8 + 2 * (lane & 3) + (e & 1);
      if (q < nq)
        V[(R.xoff + t) * nrhs + q0 + q] = g[(size_t)t * nrhs + q0 + q] - acc[m][e >> 1][e & 1];
    }
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

// CTAs per record: enough to fill the GPU (~4 per SM) for batches of few,
// large records, at least 32 rows per chunk
static int solve_chunks(const BatchH& b) {
  const int nrec = std::max(1, b.rec1 - b.rec0);
  const int want = (148 * 4 + nrec - 1) / nrec;
  return std::max(1, std::min(want, (b.maxn + 31) / 32));
}

// Sharded solve: after a batch every rank holds the solve-vector entries its
// own pivots wrote; ship them to every other rank (the vector stays
// replicated, so later batches and the top solve read current values).
static void share_runs(FactorH* F, double* V, int nr, const std::vector<int64_t>& runs, const std::vector<int>& off,
                       Arena& ws, Staging& st, cudaStream_t s) {
  Comm& C = *F->comm;
  const int me = C.rank(), nq = C.size();
  auto len = [&](int q) {
    int64_t t = 0;
    for (int u = off[q]; u < off[q + 1]; u++) t += runs[2 * size_t(u) + 1];
    return t * nr;
  };
  CopyBatch pack, unpack;
  std::vector<Msg> sm, rm;
  const int64_t mine = len(me);
  double* sbuf = nullptr;
  if (mine > 0) {
    sbuf = ws.alloc_n<double>(size_t(mine));
    int64_t o = 0;
    for (int u = off[me]; u < off[me + 1]; u++) {
      const int64_t b = runs[2 * size_t(u)], l = runs[2 * size_t(u) + 1] * nr;
      pack.add(V + b * nr, int(l), sbuf + o, int(l), int(l), 1);
      o += l;
    }
    for (int q = 0; q < nq; q++)
      if (q != me) sm.push_back(Msg{q, sbuf, size_t(mine) * sizeof(double)});
  }
  for (int q = 0; q < nq; q++) {
    const int64_t l = q == me ? 0 : len(q);
    if (l <= 0) continue;
    double* rbuf = ws.alloc_n<double>(size_t(l));
    rm.push_back(Msg{q, rbuf, size_t(l) * sizeof(double)});
    int64_t o = 0;
    for (int u = off[q]; u < off[q + 1]; u++) {
      const int64_t b = runs[2 * size_t(u)], rl = runs[2 * size_t(u) + 1] * nr;
      unpack.add(rbuf + o, int(rl), V + b * nr, int(rl), int(rl), 1);
      o += rl;
    }
  }
  launch_copies(pack, ws, st, s);
  C.exchange(sm, rm, s);
  launch_copies(unpack, ws, st, s);
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
    CK(cudaFuncSetAttribute(solve_fwd_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(solve_bwd_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(solve_fwd_kernel<RCMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(solve_bwd_kernel<RCMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  const int RC = nr == 1 ? 1 : RCMAX;
  // many right-hand sides: DMMA sweeps (IFMM_SOLVE_MM_MIN: tuning / debug)
  static const int mm_min = getenv("IFMM_SOLVE_MM_MIN") ? atoi(getenv("IFMM_SOLVE_MM_MIN")) : 2;
  const bool mm = nr >= mm_min;
  static bool mm_attr = false;
  if (mm && !mm_attr) {
    CK(cudaFuncSetAttribute(solve_fwd_mm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(MM_SMEM)));
    CK(cudaFuncSetAttribute(solve_bwd_mm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(MM_SMEM)));
    mm_attr = true;
  }
  const int nqc = (nr + MQ - 1) / MQ;
  const bool dist = F->comm && F->comm->size() > 1;
  // sharded: descriptor staging for the run exchanges (reset per call; the
  // stream is synchronised at the end of every solve)
  static thread_local Staging xst;
  xst.reset();
  for (const BatchH& b : F->batches) {
    if (dist && b.rec1 == b.rec0) {
      share_runs(F, V, nr, b.fwd_runs, b.fwd_off, ws, xst, s);
      continue;
    }
    if (mm) {
      const dim3 grid(b.rec1 - b.rec0, (b.maxn + b.maxw + GBM - 1) / GBM, nqc);
      solve_fwd_mm_kernel<<<grid, GTHREADS, MM_SMEM, s>>>(b.d_recs, b.rec0, F->d_g_off, V, G, nr);
      CK_LAUNCH();
      if (dist) share_runs(F, V, nr, b.fwd_runs, b.fwd_off, ws, xst, s);
      continue;
    }
    const int rr = std::min(32 * MAXJ, (b.maxn + 31) / 32 * 32);
    const size_t smem = sizeof(double) * (size_t(rr) * SWARPS * RC + size_t(b.maxn) * RC);
    if (smem > 200 * 1024) invalid("solve: pivot block too large for the solve kernel");
    const dim3 grid(b.rec1 - b.rec0, solve_chunks(b));
    static const bool fwd_old = getenv("IFMM_SOLVE_FWD_GEMV") != nullptr;  // debug: S^-1 b as a GEMV
    if (RC == 1 && !fwd_old) {
      // column dots split finely: >= 8 CTAs per SM in total (few large records
      // at coarse levels would otherwise leave most SMs idle), >= 32 columns each
      const int nrec = std::max(1, b.rec1 - b.rec0);
      const int want = std::max(2, (148 * 8 + nrec - 1) / nrec);
      const dim3 g1(b.rec1 - b.rec0, std::max(1, std::min(want, (b.maxn + b.maxw) / 32)));
      solve_fwd1_kernel<<<g1, SB, sizeof(double) * size_t(b.maxn), s>>>(b.d_recs, b.rec0, F->d_g_off, V, G);
    }
    else if (RC == 1) solve_fwd_kernel<1><<<grid, SB, smem, s>>>(b.d_recs, b.rec0, F->d_g_off, V, G, nr, rr);
    else solve_fwd_kernel<RCMAX><<<grid, SB, smem, s>>>(b.d_recs, b.rec0, F->d_g_off, V, G, nr, rr);
    CK_LAUNCH();
    if (dist) share_runs(F, V, nr, b.fwd_runs, b.fwd_off, ws, xst, s);
  }
  // top: y = T^-1 b on the level-1 slots (viewed column-major as nrhs x M)
  if (F->top_dim > 0) {
    const int M = F->top_dim;
    double* vt = V + F->lvl_base[1] * nr;
    double* tmp = ws.alloc_n<double>(size_t(M) * nr);
    CK(cudaMemcpyAsync(tmp, vt, sizeof(double) * M * nr, cudaMemcpyDeviceToDevice, s));
    GemmBatch gb;
    // pinned staging for the GEMM descriptors: kept across calls (a fresh
    // cudaMallocHost per solve costs milliseconds and its free synchronises)
    static thread_local Staging st;
    st.reset();
    gb.add(tmp, nr, F->top_inv, M, vt, nr, nr, M, M, 1.0, 0.0);
    launch_grouped_gemm(gb, false, true, ws, st, s);
    CK(cudaStreamSynchronize(s));
  }
  for (auto it = F->batches.rbegin(); it != F->batches.rend(); ++it) {
    const BatchH& b = *it;
    if (dist && b.rec1 == b.rec0) {
      share_runs(F, V, nr, b.bwd_runs, b.bwd_off, ws, xst, s);
      continue;
    }
    if (mm) {
      const dim3 grid(b.rec1 - b.rec0, (b.maxn + GBM - 1) / GBM, nqc);
      solve_bwd_mm_kernel<<<grid, GTHREADS, MM_SMEM, s>>>(b.d_recs, b.rec0, F->d_g_off, V, G, nr);
      CK_LAUNCH();
      if (dist) share_runs(F, V, nr, b.bwd_runs, b.bwd_off, ws, xst, s);
      continue;
    }
    const int rr = std::min(32 * MAXJ, (b.maxn + 31) / 32 * 32);
    const size_t smem = sizeof(double) * size_t(rr) * SWARPS * RC;
    const dim3 grid(b.rec1 - b.rec0, solve_chunks(b));
    static const bool bwd_old = getenv("IFMM_SOLVE_BWD_OLD") != nullptr;  // debug: generic GEMV
    if (RC == 1 && !bwd_old) {
      // rows per lane from the chunk height (<= 64 rows: 2, <= 128: 4, else 8)
      const int rows = (b.maxn + grid.y - 1) / grid.y;
      if (rows <= 64)
        solve_bwd1_kernel<2><<<grid, SB, sizeof(double) * 64 * SWARPS, s>>>(b.d_recs, b.rec0, F->d_g_off, V, G);
      else if (rows <= 128)
        solve_bwd1_kernel<4><<<grid, SB, sizeof(double) * 128 * SWARPS, s>>>(b.d_recs, b.rec0, F->d_g_off, V, G);
      else
        solve_bwd1_kernel<8><<<grid, SB, sizeof(double) * 256 * SWARPS, s>>>(b.d_recs, b.rec0, F->d_g_off, V, G);
    } else if (RC == 1) solve_bwd_kernel<1><<<grid, SB, smem, s>>>(b.d_recs, b.rec0, F->d_g_off, V, G, nr, rr);
    else solve_bwd_kernel<RCMAX><<<grid, SB, smem, s>>>(b.d_recs, b.rec0, F->d_g_off, V, G, nr, rr);
    CK_LAUNCH();
    if (dist) share_runs(F, V, nr, b.bwd_runs, b.bwd_off, ws, xst, s);
  }
  launch_permute(V + F->lvl_base[t->depth] * nr, dout, t->d_perm, N, nr, true, s);
  if (!device_ptr) CK(cudaMemcpyAsync(x, dout, sizeof(double) * N * nr, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
}

}  // namespace ifmm

namespace ifmm {

void solve_emulated(const std::vector<FactorH*>& f, const double* rhs, const std::vector<double*>& x, int64_t nrhs,
                    bool device_ptr) {
  const int n = int(f.size());
  if (n < 1 || x.size() != f.size()) invalid("solve_emulated: one output per virtual rank");
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::vector<std::exception_ptr> errs(n);
  std::vector<std::thread> th;
  for (int r = 0; r < n; r++)
    th.emplace_back([&, r] {
      try {
        CK(cudaSetDevice(dev));
        solve(f[r], rhs, x[r], nrhs, device_ptr);
      } catch (...) {
        errs[r] = std::current_exception();
        if (auto* lc = dynamic_cast<LocalComm*>(f[r]->comm.get())) lc->world().fail();
      }
    });
  for (auto& t : th) t.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

}  // namespace ifmm
