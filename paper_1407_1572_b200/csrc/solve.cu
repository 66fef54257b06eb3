// Solve with the factored IFMM (ifmm/solver.py:549-626), level-wise and
// batch-parallel, with the LU factors of every pivot (the reference's
// lu_solve, :583,613):
//   forward : g = S^-1 [b_i; 0] (LU solves); g_top -> G, g_bot -> own z slots;
//             v[pos] -= C^T g_top (partner slots, ifmm/solver.py:586-589)
//   top     : y = T^-1 v_top (LU of the level-2 system)
//   backward: t = C v[pos]; x_i = g_top - (S^-1 [t; -y_i])_top
// The record is the LU of S (m x m), its row permutation and the coupling
// panel C (n x w): each sweep streams both once.  Vectors are (positions x
// nrhs) row-major; a level's y slots alias the next level's x slots.
#include <algorithm>
#include <cmath>
#include <thread>

#include "comm.cuh"
#include "core.cuh"
#include "gemm.cuh"
#include "lu.cuh"

namespace ifmm {

void launch_permute(const double* in, double* out, const int64_t* perm, int64_t n, int nrhs, bool inverse,
                    cudaStream_t s);

constexpr int SB = 256;       // threads per solve CTA
constexpr int SWARPS = SB / 32;

// ------------------------------------------------------------------ pivot solves
// g = S^-1 [b; 0] (forward) and h = S^-1 [t; -y_i] (backward) with the LU
// factors of the record (ifmm/solver.py:583,613: lu_solve).  One CTA per
// record (and chunk of right-hand sides); rows are gathered in pivot order.
//   forward : g_top -> G, g_bot -> own z slots (V[pos[wl + t]] += g[n + t])
//   backward: x_i = g_top - h_top -> V[xoff + t]
__device__ __forceinline__ double rec_rhs(const RecordH& R, bool fwd, int i, int wl, const double* V,
                                          const double* T, int64_t nrhs, int q) {
  if (fwd) return i < R.n ? V[(R.xoff + i) * nrhs + q] : 0.0;
  return i < R.n ? T[(size_t)i * nrhs + q] : -V[(int64_t)R.pos[wl + i - R.n] * nrhs + q];
}

// Triangular solves of one shared-memory vector with the record's inverted
// 64 x 64 diagonal blocks (RecordH::dinv): per block a 64 x 64 mat-vec (four
// threads per row, partial sums combined in shared memory) instead of two
// 32-step substitution chains on one warp, then the block's column strip
// updates the remaining rows (thread per row, coalesced column reads).  The
// coarse levels -- a few records of several hundred rows per batch -- are
// bound by exactly that chain.  part: SB doubles of shared memory.
__device__ __forceinline__ double blk_matvec_part(const double* __restrict__ Ti, const double* x, int kb, int bb,
                                                  int row, int part) {
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < LU_XB / 4; c++) {
    const int cc = part * (LU_XB / 4) + c;
    s = fma(Ti[row + LU_XB * cc], cc < bb ? x[kb + cc] : 0.0, s);
  }
  return s;
}
__device__ __forceinline__ void blk_row_update(const double* __restrict__ LU, int ld, int r, int kb, int bb, double* x) {
  double s = 0.0;
#pragma unroll
  for (int h = 0; h < 2; h++) {  // 32 loads in flight at a time
    double a[32];
#pragma unroll
    for (int c = 0; c < 32; c++) a[c] = 32 * h + c < bb ? LU[r + (size_t)(kb + 32 * h + c) * ld] : 0.0;
#pragma unroll
    for (int c = 0; c < 32; c++) s = fma(a[c], 32 * h + c < bb ? x[kb + 32 * h + c] : 0.0, s);
  }
  x[r] -= s;
}
__device__ inline void cta_trsv_lower_unit_blk(const double* __restrict__ LU, int ld, int m, double* x,
                                               const double* __restrict__ dinv, double* part) {
  const int tid = threadIdx.x, row = tid & (LU_XB - 1), q = tid >> 6;
  for (int kb = 0, k = 0; kb < m; kb += LU_XB, k++) {
    const int bb = min(LU_XB, m - kb);
    part[q * LU_XB + row] = blk_matvec_part(dinv + (size_t)k * 2 * LU_XB * LU_XB, x, kb, bb, row, q);
    __syncthreads();
    if (tid < bb) x[kb + tid] = (part[tid] + part[LU_XB + tid]) + (part[2 * LU_XB + tid] + part[3 * LU_XB + tid]);
    __syncthreads();
    for (int r = kb + bb + tid; r < m; r += blockDim.x) blk_row_update(LU, ld, r, kb, bb, x);
    __syncthreads();
  }
}
__device__ inline void cta_trsv_upper_blk(const double* __restrict__ LU, int ld, int m, double* x,
                                          const double* __restrict__ dinv, double* part) {
  const int tid = threadIdx.x, row = tid & (LU_XB - 1), q = tid >> 6;
  for (int k = (m - 1) / LU_XB; k >= 0; k--) {
    const int kb = k * LU_XB, bb = min(LU_XB, m - kb);
    part[q * LU_XB + row] =
        blk_matvec_part(dinv + (size_t)k * 2 * LU_XB * LU_XB + LU_XB * LU_XB, x, kb, bb, row, q);
    __syncthreads();
    if (tid < bb) x[kb + tid] = (part[tid] + part[LU_XB + tid]) + (part[2 * LU_XB + tid] + part[3 * LU_XB + tid]);
    __syncthreads();
    for (int r = tid; r < kb; r += blockDim.x) blk_row_update(LU, ld, r, kb, bb, x);
    __syncthreads();
  }
}

template <bool FWD>
__global__ void __launch_bounds__(SB, 3) rec_solve_vec_kernel(const RecordH* __restrict__ recs, int rec0,
                                                           const int64_t* __restrict__ g_off, double* V, double* G,
                                                           const double* __restrict__ T) {
  extern __shared__ double y[];
  const RecordH R = recs[blockIdx.x];
  const int n = R.n, r = R.r, m = n + r, wl = R.w - r;
  if (m == 0) return;
  const int64_t go = g_off[rec0 + blockIdx.x];
  for (int l = threadIdx.x; l < m; l += blockDim.x) y[l] = rec_rhs(R, FWD, R.perm[l], wl, V, T + go, 1, 0);
  __syncthreads();
  if (R.dinv != nullptr && *R.pflag == 0) {  // uniform over the CTA
    __shared__ double part[SB];
    cta_trsv_lower_unit_blk(R.lu, m, m, y, R.dinv, part);
    cta_trsv_upper_blk(R.lu, m, m, y, R.dinv, part);
  } else {
    cta_trsv_lower_unit(R.lu, m, m, y);
    cta_trsv_upper(R.lu, m, m, y);
  }
  if (FWD) {
    for (int t = threadIdx.x; t < n; t += blockDim.x) G[go + t] = y[t];
    for (int t = threadIdx.x; t < r; t += blockDim.x) V[R.pos[wl + t]] += y[n + t];
  } else {
    for (int t = threadIdx.x; t < n; t += blockDim.x) V[R.xoff + t] = G[go + t] - y[t];
  }
}

// nrhs >= 2: TW right-hand sides per CTA, DMMA tile solves (lu.cuh)
template <int TW, bool FWD>
__global__ void __launch_bounds__(SB, 3) rec_solve_tile_kernel(const RecordH* __restrict__ recs, int rec0,
                                                            const int64_t* __restrict__ g_off, double* V, double* G,
                                                            const double* __restrict__ T, int nrhs, double* scratch,
                                                            size_t per) {
  extern __shared__ double sm[];
  const RecordH R = recs[blockIdx.x];
  const int n = R.n, r = R.r, m = n + r, wl = R.w - r;
  if (m == 0) return;
  const int q0 = blockIdx.y * TW, nq = min(TW, nrhs - q0);
  const int xm = m | 1;
  double* X = scratch ? scratch + per * (blockIdx.x * (size_t)gridDim.y + blockIdx.y) : sm;
  const int64_t go = g_off[rec0 + blockIdx.x];
  for (int e = threadIdx.x; e < TW * m; e += blockDim.x) {
    const int c = e / m, l = e - c * m;
    X[(size_t)c * xm + l] = c < nq ? rec_rhs(R, FWD, R.perm[l], wl, V, T + go * nrhs, nrhs, q0 + c) : 0.0;
  }
  __syncthreads();
  cta_tile_lu_solve<TW>(R.lu, m, m, X, xm);
  for (int e = threadIdx.x; e < TW * m; e += blockDim.x) {
    const int c = e / m, l = e - c * m;
    if (c >= nq) continue;
    const double v = X[(size_t)c * xm + l];
    if (FWD) {
      if (l < n) G[(go + l) * nrhs + q0 + c] = v;
      else V[(int64_t)R.pos[wl + l - n] * nrhs + q0 + c] += v;
    } else if (l < n) {
      double* o = V + (R.xoff + l) * nrhs + q0 + c;
      *o = G[(go + l) * nrhs + q0 + c] - v;
    }
  }
}

// Top-level system y = T^-1 v (ifmm/solver.py:592-598), in place on the
// level-1 slots (M x nrhs row-major)
__global__ void __launch_bounds__(SB) top_solve_vec_kernel(const double* __restrict__ LU, const int* __restrict__ perm,
                                                           int M, double* v) {
  extern __shared__ double y[];
  for (int l = threadIdx.x; l < M; l += blockDim.x) y[l] = v[perm[l]];
  __syncthreads();
  cta_trsv_lower_unit(LU, M, M, y);
  cta_trsv_upper(LU, M, M, y);
  for (int l = threadIdx.x; l < M; l += blockDim.x) v[l] = y[l];
}
template <int TW>
__global__ void __launch_bounds__(SB) top_solve_tile_kernel(const double* __restrict__ LU,
                                                            const int* __restrict__ perm, int M, const double* vin,
                                                            double* vout, int nrhs, double* scratch, size_t per) {
  extern __shared__ double sm[];
  const int q0 = blockIdx.x * TW, nq = min(TW, nrhs - q0);
  const int xm = M | 1;
  double* X = scratch ? scratch + per * blockIdx.x : sm;
  for (int e = threadIdx.x; e < TW * M; e += blockDim.x) {
    const int c = e / M, l = e - c * M;
    X[(size_t)c * xm + l] = c < nq ? vin[(size_t)perm[l] * nrhs + q0 + c] : 0.0;
  }
  __syncthreads();
  cta_tile_lu_solve<TW>(LU, M, M, X, xm);
  for (int e = threadIdx.x; e < TW * M; e += blockDim.x) {
    const int c = e / M, l = e - c * M;
    if (c < nq) vout[(size_t)l * nrhs + q0 + c] = X[(size_t)c * xm + l];
  }
}

// ------------------------------------------------------------------ coupling GEMVs (one rhs)
// Records are split over gridDim.y CTAs (coarse levels have few, large
// records).  Every output has exactly one writer (deterministic).
__device__ __forceinline__ void chunk_range(int len, int y, int ny, int gran, int& lo, int& hi) {
  const int per = ((len + ny - 1) / ny + gran - 1) / gran * gran;
  lo = min(len, y * per);
  hi = min(len, lo + per);
}

// forward partner update: V[pos[c]] -= C(:, c)^T g_top for c < wl.  Column
// dots, W-lane segments per column (short columns: several per warp), two
// columns per segment in flight (streaming loads).
__global__ void __launch_bounds__(SB, 3) cpl_fwd1_kernel(const RecordH* __restrict__ recs, int rec0,
                                                         const int64_t* __restrict__ g_off, double* V,
                                                         const double* __restrict__ G) {
  extern __shared__ double bsh[];  // n
  const RecordH R = recs[blockIdx.x];
  const int n = R.n, wl = R.w - R.r;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int c0, c1;
  chunk_range(wl, blockIdx.y, gridDim.y, 8, c0, c1);
  if (c1 <= c0 || n == 0) return;
  const double* g = G + g_off[rec0 + blockIdx.x];
  for (int e = threadIdx.x; e < n; e += SB) bsh[e] = g[e];
  __syncthreads();
  const int W = n > 128 ? 32 : (n > 64 ? 16 : 8);
  const int seg = lane / W, sl = lane & (W - 1), spw = 32 / W;
  const int stride = SWARPS * spw;
  for (int cb = c0 + warp * spw; cb < c1; cb += 2 * stride) {
    const int c = cb + seg, c2 = c + stride;
    const bool ok = c < c1, ok2 = c2 < c1;
    const double* x = R.c + (size_t)(ok ? c : c0) * n;
    const double* x2 = R.c + (size_t)(ok2 ? c2 : c0) * n;
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
      if (ok) V[(int64_t)R.pos[c]] -= sv;
      if (ok2) V[(int64_t)R.pos[c2]] -= sv2;
    }
  }
}

// backward coupling product: T[t] = sum_{c < wl} C(t, c) V[pos[c]] for the
// rows [r0, r1) of chunk blockIdx.y.  Lanes own rows (J per lane), warps split
// the columns; CB columns of loads are issued before their FMAs.
template <int J>
__global__ void __launch_bounds__(SB, J <= 4 ? 3 : 2) cpl_bwd1_kernel(const RecordH* __restrict__ recs, int rec0,
                                                                     const int64_t* __restrict__ g_off,
                                                                     const double* __restrict__ V, double* T) {
  constexpr int CB = J <= 2 ? 8 : (J <= 4 ? 4 : 2);
  extern __shared__ double red[];  // (32 J) x SWARPS
  const RecordH R = recs[blockIdx.x];
  const int n = R.n, wl = R.w - R.r;
  int r0, r1;
  chunk_range(n, blockIdx.y, gridDim.y, 32, r0, r1);
  if (r1 <= r0) return;
  double* tout = T + g_off[rec0 + blockIdx.x];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int t0 = r0; t0 < r1; t0 += 32 * J) {
    double acc[J];
#pragma unroll
    for (int j = 0; j < J; j++) acc[j] = 0.0;
    for (int cb = warp * 32; cb < wl; cb += SWARPS * 32) {
      const double xl = (cb + lane < wl) ? V[(int64_t)R.pos[cb + lane]] : 0.0;
      const int cmax = min(32, wl - cb);
      for (int u0 = 0; u0 < cmax; u0 += CB) {
        double a[CB][J];
#pragma unroll
        for (int u = 0; u < CB; u++) {
          const double* col = R.c + (size_t)(cb + u0 + u) * n;
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
      tout[t0 + e] = s;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ many rhs
// Multi-rhs coupling products as DMMA GEMMs: each record's
// coupling panel is read once per chunk of up to 32 right-hand sides.
// 64 x 32 output tiles, 4 warps x (16 x 32), cp.async-staged operands.
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

// forward: V[pos[c], q] -= (C^T G)(c, q) for c < wl.  grid (record, 64-row tile, rhs chunk)
__global__ void __launch_bounds__(GTHREADS) cpl_fwd_mm_kernel(const RecordH* __restrict__ recs, int rec0,
                                                              const int64_t* __restrict__ g_off, double* V,
                                                              const double* G, int nrhs) {
  extern __shared__ double msm[];
  const RecordH R = recs[blockIdx.x];
  const int n = R.n, wl = R.w - R.r;
  const int c0 = blockIdx.y * GBM;
  if (c0 >= wl || n == 0) return;
  const int q0 = blockIdx.z * MQ, nq = min(MQ, nrhs - q0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* Bv = G + g_off[rec0 + blockIdx.x] * nrhs + q0;
  auto load = [&](int st, int k0) {
    double* As = msm + (size_t)st * (MM_A + MM_B);
    double* Bs = As + MM_A;
#pragma unroll
    for (int e = 0; e < (GBM * GBK) / GTHREADS; e++) {  // A: column c of C, k-contiguous
      const int cidx = tid + e * GTHREADS, k = cidx & (GBK - 1), r = cidx / GBK;
      const int c = c0 + r, gk = k0 + k;
      cp_async8(As + r * KP + k, R.c + gk + (size_t)c * n, c < wl && gk < n);
    }
#pragma unroll
    for (int e = 0; e < (GBK * MQ) / GTHREADS; e++) {  // B: rows of G, q-contiguous
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
    if (c >= wl) continue;
    double* row = V + (int64_t)R.pos[c] * nrhs + q0;
    double old[8];
#pragma unroll
    for (int e = 0; e < 8; e++) {
      const int q = (e >> 1) * 8 + 2 * (lane & 3) + (e & 1);
      old[e] = q < nq ? row[q] : 0.0;
    }
#pragma unroll
    for (int e = 0; e < 8; e++) {
      const int q = (e >> 1) * 8 + 2 * (lane & 3) + (e & 1);
      if (q < nq) row[q] = old[e] - acc[m][e >> 1][e & 1];
    }
  }
}

// backward: T(t, q) = sum_{c < wl} C(t, c) V(pos[c], q).  grid (record, 64-row tile of n, rhs chunk)
__global__ void __launch_bounds__(GTHREADS) cpl_bwd_mm_kernel(const RecordH* __restrict__ recs, int rec0,
                                                              const int64_t* __restrict__ g_off, const double* V,
                                                              double* T, int nrhs) {
  extern __shared__ double msm[];
  const RecordH R = recs[blockIdx.x];
  const int n = R.n, wl = R.w - R.r;
  const int t0 = blockIdx.y * GBM;
  if (t0 >= n) return;
  const int q0 = blockIdx.z * MQ, nq = min(MQ, nrhs - q0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* tout = T + g_off[rec0 + blockIdx.x] * nrhs;
  auto load = [&](int st, int k0) {
    double* As = msm + (size_t)st * (MM_A + MM_B);
    double* Bs = As + MM_A;
#pragma unroll
    for (int e = 0; e < (GBM * GBK) / GTHREADS; e++) {  // A: C(t, c), t-contiguous -> stored [t][k]
      const int cidx = tid + e * GTHREADS, r = cidx & (GBM - 1), k = cidx / GBM;
      const int t = t0 + r, gk = k0 + k;
      cp_async8(As + r * KP + k, R.c + t + (size_t)gk * n, t < n && gk < wl);
    }
#pragma unroll
    for (int e = 0; e < (GBK * MQ) / GTHREADS; e++) {  // B: V(pos[c], q)
      const int cidx = tid + e * GTHREADS, q = cidx & (MQ - 1), k = cidx / MQ;
      const int gk = k0 + k;
      const bool ok = gk < wl && q < nq;
      const double* src = ok ? V + (int64_t)R.pos[gk] * nrhs + q0 + q : V;
      cp_async8(Bs + k * QP + q, src, ok);
    }
  };
  double acc[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; a++)
#pragma unroll
    for (int b = 0; b < 4; b++) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int nk = (wl + GBK - 1) / GBK;
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
      if (q < nq) tout[(size_t)t * nrhs + q0 + q] = acc[m][e >> 1][e & 1];
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

// Launch one colour batch's pivot solves (forward or backward sweep).
static void launch_rec_solves(const BatchH& b, FactorH* F, double* V, double* G, const double* T, int nr, bool fwd,
                              Arena& ws, cudaStream_t s) {
  const int nrec = b.rec1 - b.rec0;
  if (nrec <= 0) return;
  if (nr == 1) {
    const size_t smem = sizeof(double) * size_t(std::max(1, b.maxm));
    if (smem > LU_TILE_SMEM_MAX) invalid("solve: pivot block too large for the solve kernel");
    if (fwd) rec_solve_vec_kernel<true><<<nrec, SB, smem, s>>>(b.d_recs, b.rec0, F->d_g_off, V, G, T);
    else rec_solve_vec_kernel<false><<<nrec, SB, smem, s>>>(b.d_recs, b.rec0, F->d_g_off, V, G, T);
    CK_LAUNCH();
    return;
  }
  int tw = lu_tile_width(b.maxm);
  const bool global = tw == 0;
  if (global) tw = 8;
  if (nr <= 8) tw = 8;
  else if (nr <= 16 && tw > 16) tw = 16;
  const size_t per = size_t(tw) * size_t(b.maxm | 1);
  const dim3 grid(nrec, (nr + tw - 1) / tw);
  double* scratch = global ? ws.alloc_n<double>(per * grid.x * grid.y) : nullptr;
  const size_t smem = global ? 0 : sizeof(double) * per;
#define IFMM_REC_TILE(TWV)                                                                                   \
  if (fwd) rec_solve_tile_kernel<TWV, true><<<grid, SB, smem, s>>>(b.d_recs, b.rec0, F->d_g_off, V, G, T, nr, \
                                                                    scratch, per);                          \
  else rec_solve_tile_kernel<TWV, false><<<grid, SB, smem, s>>>(b.d_recs, b.rec0, F->d_g_off, V, G, T, nr,    \
                                                                 scratch, per);
  if (tw == 32) { IFMM_REC_TILE(32) }
  else if (tw == 16) { IFMM_REC_TILE(16) }
  else { IFMM_REC_TILE(8) }
#undef IFMM_REC_TILE
  CK_LAUNCH();
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
  double* T = ws.alloc_n<double>(std::max<int64_t>(1, F->g_size) * nr);
  CK(cudaMemsetAsync(V, 0, sizeof(double) * std::max<int64_t>(1, F->vec_size) * nr, s));
  launch_permute(din, V + F->lvl_base[t->depth] * nr, t->d_perm, N, nr, false, s);
  static bool attr = false;
  if (!attr) {
    const int mx = int(LU_TILE_SMEM_MAX);
    CK(cudaFuncSetAttribute(rec_solve_vec_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CK(cudaFuncSetAttribute(rec_solve_vec_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CK(cudaFuncSetAttribute(rec_solve_tile_kernel<32, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CK(cudaFuncSetAttribute(rec_solve_tile_kernel<32, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CK(cudaFuncSetAttribute(rec_solve_tile_kernel<16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CK(cudaFuncSetAttribute(rec_solve_tile_kernel<16, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CK(cudaFuncSetAttribute(rec_solve_tile_kernel<8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CK(cudaFuncSetAttribute(rec_solve_tile_kernel<8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CK(cudaFuncSetAttribute(top_solve_vec_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CK(cudaFuncSetAttribute(top_solve_tile_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CK(cudaFuncSetAttribute(top_solve_tile_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CK(cudaFuncSetAttribute(top_solve_tile_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CK(cudaFuncSetAttribute(cpl_fwd_mm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(MM_SMEM)));
    CK(cudaFuncSetAttribute(cpl_bwd_mm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(MM_SMEM)));
    attr = true;
  }
  const bool mm = nr >= 2;
  const int nqc = (nr + MQ - 1) / MQ;
  const bool dist = F->comm && F->comm->size() > 1;
  // sharded: descriptor staging for the run exchanges (reset per call; the
  // stream is synchronised at the end of every solve)
  static thread_local Staging xst;
  xst.reset();
  // ---- forward replay (ifmm/solver.py:573-590)
  for (const BatchH& b : F->batches) {
    if (dist && b.rec1 == b.rec0) {
      share_runs(F, V, nr, b.fwd_runs, b.fwd_off, ws, xst, s);
      continue;
    }
    launch_rec_solves(b, F, V, G, T, nr, true, ws, s);
    const int nrec = b.rec1 - b.rec0;
    if (mm) {
      cpl_fwd_mm_kernel<<<dim3(nrec, std::max(1, (b.maxw + GBM - 1) / GBM), nqc), GTHREADS, MM_SMEM, s>>>(b.d_recs, b.rec0,
                                                                                             F->d_g_off, V, G, nr);
    } else {
      // column dots split finely: >= 8 CTAs per SM in total (few large records
      // at coarse levels would otherwise leave most SMs idle), >= 32 columns each
      const int want = std::max(2, (148 * 8 + nrec - 1) / std::max(1, nrec));
      const dim3 g1(nrec, std::max(1, std::min(want, b.maxw / 32)));
      cpl_fwd1_kernel<<<g1, SB, sizeof(double) * size_t(std::max(1, b.maxn)), s>>>(b.d_recs, b.rec0, F->d_g_off, V,
                                                                                    G);
    }
    CK_LAUNCH();
    if (dist) share_runs(F, V, nr, b.fwd_runs, b.fwd_off, ws, xst, s);
  }
  // ---- top: y = T^-1 v on the level-1 slots (ifmm/solver.py:592-598)
  if (F->top_dim > 0) {
    const int M = F->top_dim;
    double* vt = V + F->lvl_base[1] * nr;
    if (nr == 1) {
      if (sizeof(double) * size_t(M) > LU_TILE_SMEM_MAX) invalid("solve: top-level system too large");
      top_solve_vec_kernel<<<1, SB, sizeof(double) * M, s>>>(F->top_lu, F->top_perm, M, vt);
    } else {
      double* tmp = ws.alloc_n<double>(size_t(M) * nr);
      CK(cudaMemcpyAsync(tmp, vt, sizeof(double) * M * nr, cudaMemcpyDeviceToDevice, s));
      int tw = lu_tile_width(M);
      const bool global = tw == 0;
      if (global) tw = 8;
      if (nr <= 8) tw = 8;
      else if (nr <= 16 && tw > 16) tw = 16;
      const size_t per = size_t(tw) * size_t(M | 1);
      const int grid = (nr + tw - 1) / tw;
      double* scratch = global ? ws.alloc_n<double>(per * grid) : nullptr;
      const size_t smem = global ? 0 : sizeof(double) * per;
      if (tw == 32) top_solve_tile_kernel<32><<<grid, SB, smem, s>>>(F->top_lu, F->top_perm, M, tmp, vt, nr, scratch, per);
      else if (tw == 16) top_solve_tile_kernel<16><<<grid, SB, smem, s>>>(F->top_lu, F->top_perm, M, tmp, vt, nr, scratch, per);
      else top_solve_tile_kernel<8><<<grid, SB, smem, s>>>(F->top_lu, F->top_perm, M, tmp, vt, nr, scratch, per);
    }
    CK_LAUNCH();
  }
  // ---- back-substitution, levels 2..kappa, batches reversed (ifmm/solver.py:604-618)
  for (auto it = F->batches.rbegin(); it != F->batches.rend(); ++it) {
    const BatchH& b = *it;
    if (dist && b.rec1 == b.rec0) {
      share_runs(F, V, nr, b.bwd_runs, b.bwd_off, ws, xst, s);
      continue;
    }
    const int nrec = b.rec1 - b.rec0;
    if (mm) {
      cpl_bwd_mm_kernel<<<dim3(nrec, std::max(1, (b.maxn + GBM - 1) / GBM), nqc), GTHREADS, MM_SMEM, s>>>(b.d_recs, b.rec0,
                                                                                             F->d_g_off, V, T, nr);
    } else {
      const dim3 grid(nrec, solve_chunks(b));
      const int rows = (b.maxn + grid.y - 1) / grid.y;
      if (rows <= 64)
        cpl_bwd1_kernel<2><<<grid, SB, sizeof(double) * 64 * SWARPS, s>>>(b.d_recs, b.rec0, F->d_g_off, V, T);
      else if (rows <= 128)
        cpl_bwd1_kernel<4><<<grid, SB, sizeof(double) * 128 * SWARPS, s>>>(b.d_recs, b.rec0, F->d_g_off, V, T);
      else
        cpl_bwd1_kernel<8><<<grid, SB, sizeof(double) * 256 * SWARPS, s>>>(b.d_recs, b.rec0, F->d_g_off, V, T);
    }
    CK_LAUNCH();
    launch_rec_solves(b, F, V, G, T, nr, false, ws, s);
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
