// Batched LU with partial pivoting, LU-based X = S^-1 C and the dlacn2
// condition estimate (see lu.cuh).  The reference factors every pivot with
// scipy lu_factor (LAPACK dgetrf), tests it with dgecon and applies it with
// lu_solve (dgetrs) (ifmm/solver.py:214-218,246); these kernels do the same
// on a whole colour batch at once.
#include <algorithm>
#include <mutex>
#include <set>
#include <string>

#include "gemm.cuh"
#include "lu.cuh"

namespace ifmm {

namespace {

constexpr int XB = LU_XB;

struct RowMove {
  int dst, src;
};

__global__ void lu_perm_init_kernel(const MatDesc* __restrict__ desc) {
  const MatDesc D = desc[blockIdx.x];
  for (int l = threadIdx.x; l < D.m; l += blockDim.x) D.ipiv[l] = l;
}

// Panel factorization of columns [j, j+bb), rows [j, m) (shared memory, row
// stride bb+1).  Pivoting is tracked as a position <-> row map of the panel
// rows; the pivot of a column is the largest |entry| among the rows at
// positions >= the column, ties to the smallest position (idamax on the
// swapped order).  Writes the panel back in final row order, updates perm,
// and lists the row moves new[dst] = old[src] (<= 2 bb) for the other columns.
__global__ void __launch_bounds__(512) lu_panel_kernel(const MatDesc* __restrict__ desc, int j, int b, int* info,
                                                       RowMove* moves, int* nmoves) {
  extern __shared__ double sm[];
  __shared__ double candv[32];
  __shared__ int candr[32], candp[32];
  __shared__ double prow[32];
  __shared__ double s_inv;
  __shared__ int s_cnt;
  __shared__ int mv_dst[64], mv_src[64], mv_perm[64];
  const MatDesc D = desc[blockIdx.x];
  const int m = D.m;
  if (m <= j) return;
  const int bb = min(b, m - j), nr = m - j, ld = bb + 1;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  double* P = sm;                                           // P[r*ld + c] = A(j + r, j + c)
  int* pos = reinterpret_cast<int*>(P + (size_t)nr * ld);  // panel row -> position (relative to j)
  int* at = pos + nr;                                       // position -> panel row
  for (int r = tid; r < nr; r += nt) {
    const double* src = D.A + j + r;
#pragma unroll 4
    for (int c = 0; c < bb; c++) P[r * ld + c] = src[(size_t)(j + c) * D.lda];
    pos[r] = r;
    at[r] = r;
  }
  if (tid == 0) s_cnt = 0;
  __syncthreads();
  for (int c = 0; c < bb; c++) {
    double bv = -1.0;
    int br = -1, bp = 0x7fffffff;
    for (int r = tid; r < nr; r += nt) {
      const int pr = pos[r];
      if (pr < c) continue;
      const double v = fabs(P[r * ld + c]);
      if (v > bv || (v == bv && pr < bp)) { bv = v; br = r; bp = pr; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int orr = __shfl_xor_sync(0xffffffffu, br, o), op = __shfl_xor_sync(0xffffffffu, bp, o);
      if (ov > bv || (ov == bv && op < bp)) { bv = ov; br = orr; bp = op; }
    }
    if (lane == 0) { candv[warp] = bv; candr[warp] = br; candp[warp] = bp; }
    __syncthreads();
    if (warp == 0) {
      bv = lane < nw ? candv[lane] : -1.0;
      br = lane < nw ? candr[lane] : -1;
      bp = lane < nw ? candp[lane] : 0x7fffffff;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int orr = __shfl_xor_sync(0xffffffffu, br, o), op = __shfl_xor_sync(0xffffffffu, bp, o);
        if (ov > bv || (ov == bv && op < bp)) { bv = ov; br = orr; bp = op; }
      }
      if (br < 0) {  // cannot happen (row c itself is a candidate); keep the map consistent
        br = at[c];
        bp = c;
      }
      const double pv = P[br * ld + c];
      const bool sing = (pv == 0.0 || pv != pv);
      for (int cc = lane; cc < bb; cc += 32) prow[cc] = P[br * ld + cc];
      if (lane == 0) {
        s_inv = sing ? 0.0 : 1.0 / pv;
        if (sing && info[blockIdx.x] == 0) info[blockIdx.x] = j + c + 1;
        const int q = at[c];  // swap positions c <-> bp
        at[bp] = q;
        pos[q] = bp;
        at[c] = br;
        pos[br] = c;
      }
    }
    __syncthreads();
    const double inv = s_inv;
    for (int r = tid; r < nr; r += nt) {
      if (pos[r] <= c) continue;
      double* row = P + r * ld;
      const double f = row[c] * inv;
      row[c] = f;
      if (f != 0.0)
        for (int cc = c + 1; cc < bb; cc++) row[cc] = fma(-f, prow[cc], row[cc]);
    }
    __syncthreads();
  }
  // write back in final order; moves and the permutation update
  for (int l = tid; l < nr; l += nt) {
    const int r = at[l];
    double* dst = D.A + j + l;
#pragma unroll 4
    for (int c = 0; c < bb; c++) dst[(size_t)(j + c) * D.lda] = P[r * ld + c];
    if (r != l) {
      const int k = atomicAdd(&s_cnt, 1);
      mv_dst[k] = j + l;
      mv_src[k] = j + r;
    }
  }
  __syncthreads();
  const int cnt = s_cnt;
  if (tid < cnt) mv_perm[tid] = D.ipiv[mv_src[tid]];
  __syncthreads();
  if (tid < cnt) {
    D.ipiv[mv_dst[tid]] = mv_perm[tid];
    moves[(size_t)blockIdx.x * 2 * b + tid] = RowMove{mv_dst[tid], mv_src[tid]};
  }
  if (tid == 0) nmoves[blockIdx.x] = cnt;
}

// The same panel factorization with the panel in registers: 256 threads,
// thread t owns panel rows t + 256 q (q < RPT), all 32 of their panel values.
// One barrier per column: every warp posts its best candidate (|value|,
// position, row) and, from the candidate's owner, the candidate's whole panel
// row into a per-warp slot (double-buffered by column parity); after the
// barrier every thread reduces the <= 8 candidates itself and reads the pivot
// row from the winning slot.  Positions are tracked per row in registers (the
// row at position c and the pivot row trade positions).  Same pivot choices
// (ties to the smallest position) and the same fma sequence as lu_panel_kernel,
// so both give identical factors.  b == 32 only.
template <int RPT>
__global__ void __launch_bounds__(256) lu_panel_reg_kernel(const MatDesc* __restrict__ desc, int j, int* info,
                                                           RowMove* moves, int* nmoves) {
  constexpr int B = 32, NT = 256, NW = NT / 32;
  __shared__ double cv[2][NW], crow[2][NW][B];
  __shared__ int cp[2][NW], cr[2][NW];
  __shared__ int s_cnt;
  __shared__ int mv_dst[2 * B], mv_src[2 * B], mv_perm[2 * B];
  const MatDesc D = desc[blockIdx.x];
  const int m = D.m;
  if (m <= j) return;
  const int bb = min(B, m - j), nr = m - j;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double v[RPT][B];
  int pos[RPT];
#pragma unroll
  for (int q = 0; q < RPT; q++) {
    const int r = tid + NT * q;
    pos[q] = r < nr ? r : 0x7fffffff;
#pragma unroll
    for (int c = 0; c < B; c++) v[q][c] = (r < nr && c < bb) ? D.A[(j + r) + (size_t)(j + c) * D.lda] : 0.0;
  }
  if (tid == 0) s_cnt = 0;
  bool sing_seen = false;
#pragma unroll
  for (int c = 0; c < B; c++) {
    if (c >= bb) break;
    const int par = c & 1;
    // local candidate among own rows at positions >= c
    double bv = -1.0;
    int bp = 0x7fffffff, bq = -1;
#pragma unroll
    for (int q = 0; q < RPT; q++) {
      const double a = fabs(v[q][c]);
      if (pos[q] >= c && pos[q] != 0x7fffffff && (a > bv || (a == bv && pos[q] < bp))) {
        bv = a;
        bp = pos[q];
        bq = q;
      }
    }
    int br = bq >= 0 ? tid + NT * bq : -1;
    double wv = bv;
    int wp = bp, wr = br;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, wv, o);
      const int op = __shfl_xor_sync(0xffffffffu, wp, o), orr = __shfl_xor_sync(0xffffffffu, wr, o);
      if (ov > wv || (ov == wv && op < wp)) { wv = ov; wp = op; wr = orr; }
    }
    // the warp's winner posts its row
    if (br >= 0 && br == wr) {
#pragma unroll
      for (int q = 0; q < RPT; q++)
        if (q == bq)
#pragma unroll
          for (int cc = 0; cc < B; cc++) crow[par][warp][cc] = v[q][cc];
    }
    if (lane == 0) {
      cv[par][warp] = wv;
      cp[par][warp] = wp;
      cr[par][warp] = wr;
    }
    __syncthreads();
    double gv = -1.0;
    int gp = 0x7fffffff, gw = 0;
#pragma unroll
    for (int w = 0; w < NW; w++) {
      const double a = cv[par][w];
      const int p = cp[par][w];
      if (a > gv || (a == gv && p < gp)) { gv = a; gp = p; gw = w; }
    }
    const int grow = cr[par][gw];
    const double pv = crow[par][gw][c];
    const bool sing = (pv == 0.0 || pv != pv);
    if (sing && tid == 0 && !sing_seen && info[blockIdx.x] == 0) info[blockIdx.x] = j + c + 1;
    sing_seen |= sing;
    const double inv = sing ? 0.0 : 1.0 / pv;
    // positions: the pivot row moves to c, the row at c to the pivot's old position
#pragma unroll
    for (int q = 0; q < RPT; q++) {
      const int r = tid + NT * q;
      if (r == grow) pos[q] = c;
      else if (pos[q] == c) pos[q] = gp;
    }
    // eliminate below the pivot
#pragma unroll
    for (int q = 0; q < RPT; q++) {
      if (pos[q] > c && pos[q] != 0x7fffffff) {
        const double f = v[q][c] * inv;
        v[q][c] = f;
        if (f != 0.0)
#pragma unroll
          for (int cc = c + 1; cc < B; cc++) v[q][cc] = fma(-f, crow[par][gw][cc], v[q][cc]);
      }
    }
  }
  // write back in final order; moves and the permutation update
  int oldperm[RPT];
#pragma unroll
  for (int q = 0; q < RPT; q++) {
    const int r = tid + NT * q;
    oldperm[q] = r < nr ? D.ipiv[j + r] : 0;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < RPT; q++) {
    const int r = tid + NT * q;
    if (r >= nr) continue;
    const int l = pos[q];
    double* dst = D.A + j + l;
#pragma unroll
    for (int c = 0; c < B; c++)
      if (c < bb) dst[(size_t)(j + c) * D.lda] = v[q][c];
    if (l != r) {
      D.ipiv[j + l] = oldperm[q];
      const int k = atomicAdd(&s_cnt, 1);
      mv_dst[k] = j + l;
      mv_src[k] = j + r;
    }
  }
  __syncthreads();
  const int cnt = s_cnt;
  if (tid < cnt) moves[(size_t)blockIdx.x * 2 * B + tid] = RowMove{mv_dst[tid], mv_src[tid]};
  if (tid == 0) nmoves[blockIdx.x] = cnt;
  (void)mv_perm;
}

// Row moves on every column outside the panel, then U12 = L11^-1 A12 on the
// columns right of it (forward substitution with the unit lower panel block,
// lanes own rows).  One warp per column.
__global__ void __launch_bounds__(256) lu_swap_trsm_kernel(const MatDesc* __restrict__ desc, int j, int b,
                                                           const RowMove* __restrict__ moves,
                                                           const int* __restrict__ nmoves) {
  const MatDesc D = desc[blockIdx.x];
  const int m = D.m;
  if (m <= j) return;
  const int bb = min(b, m - j);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cnt = nmoves[blockIdx.x];
  const RowMove* mv = moves + (size_t)blockIdx.x * 2 * b;
  RowMove m0{-1, -1}, m1{-1, -1};
  if (lane < cnt) m0 = mv[lane];
  if (lane + 32 < cnt) m1 = mv[lane + 32];
  double lrow[32];
#pragma unroll
  for (int c = 0; c < 32; c++)
    lrow[c] = (c < lane && lane < bb) ? D.A[(j + lane) + (size_t)(j + c) * D.lda] : 0.0;
  for (int col = warp + blockIdx.y * 8; col < m; col += 8 * gridDim.y) {
    if (col >= j && col < j + bb) continue;
    double* a = D.A + (size_t)col * D.lda;
    const double v0 = m0.dst >= 0 ? a[m0.src] : 0.0;
    const double v1 = m1.dst >= 0 ? a[m1.src] : 0.0;
    __syncwarp();
    if (m0.dst >= 0) a[m0.dst] = v0;
    if (m1.dst >= 0) a[m1.dst] = v1;
    __syncwarp();
    if (col < j + bb) continue;
    double v = lane < bb ? a[j + lane] : 0.0;
#pragma unroll
    for (int c = 0; c < 31; c++) {
      const double xc = __shfl_sync(0xffffffffu, v, c);
      v = fma(-lrow[c], xc, v);
    }
    if (lane < bb) a[j + lane] = v;
  }
}

// Trailing update A22 -= L21 U12 (rows and columns [j+bb, m)), grid (matrix,
// 64x64 tile); operands on the cp.async pipeline of gemm.cuh (L21 i-contiguous,
// U12 k-contiguous), DMMA m8n8k4.
// Column tiles [ct_lo, ct_hi) of the trailing matrix (ct_hi < 0: all), all row tiles.
__global__ void __launch_bounds__(GTHREADS, 3) lu_update_kernel(const MatDesc* __restrict__ desc, int j, int b,
                                                                 int ct_lo, int ct_hi) {
  extern __shared__ double gsm[];
  const MatDesc D = desc[blockIdx.x];
  const int m = D.m;
  if (m <= j) return;
  const int bb = min(b, m - j);
  const int t0 = j + bb, nt = m - t0;
  if (nt <= 0) return;
  const int tiles = (nt + GBM - 1) / GBM;
  const int ctn = (ct_hi < 0 ? tiles : min(ct_hi, tiles)) - ct_lo;
  const int tl = blockIdx.y;
  if (ctn <= 0 || tl >= tiles * ctn) return;
  const int i0 = (tl % tiles) * GBM, c0 = (ct_lo + tl / tiles) * GBN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
  auto Asm = [&](int st) { return gsm + (size_t)st * 2 * GTILE_D; };
  auto Bsm = [&](int st) { return gsm + (size_t)st * 2 * GTILE_D + GTILE_D; };
  const double* L21 = D.A + t0 + (size_t)j * D.lda;
  const double* U12 = D.A + j + (size_t)t0 * D.lda;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; a++)
#pragma unroll
    for (int c = 0; c < 4; c++) acc[a][c][0] = acc[a][c][1] = 0.0;
  const int nk = (bb + GBK - 1) / GBK;
#pragma unroll
  for (int st = 0; st < GSTAGES - 1; st++) {
    if (st < nk) {
      load_operand<false>(Asm(st), L21, D.lda, nt, bb, i0, st * GBK, tid);
      load_operand<true>(Bsm(st), U12, D.lda, nt, bb, c0, st * GBK, tid);
    }
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; kt++) {
    cp_async_wait<GSTAGES - 2>();
    __syncthreads();
    {
      const int ntile = kt + GSTAGES - 1;
      if (ntile < nk) {
        const int st = ntile % GSTAGES;
        load_operand<false>(Asm(st), L21, D.lda, nt, bb, i0, ntile * GBK, tid);
        load_operand<true>(Bsm(st), U12, D.lda, nt, bb, c0, ntile * GBK, tid);
      }
      cp_async_commit();
    }
    const double* As = Asm(kt % GSTAGES);
    const double* Bs = Bsm(kt % GSTAGES);
#pragma unroll
    for (int kk = 0; kk < GBK; kk += 4) {
      double fa[4], fb[4];
#pragma unroll
      for (int q = 0; q < 4; q++) fa[q] = frag<false>(As, wm + q * 8 + (lane >> 2), kk + (lane & 3));
#pragma unroll
      for (int q = 0; q < 4; q++) fb[q] = frag<true>(Bs, wn + q * 8 + (lane >> 2), kk + (lane & 3));
#pragma unroll
      for (int x = 0; x < 4; x++)
#pragma unroll
        for (int y = 0; y < 4; y++)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(acc[x][y][0]), "+d"(acc[x][y][1])
                       : "d"(fa[x]), "d"(fb[y]));
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int x = 0; x < 4; x++) {
    const int gi = i0 + wm + x * 8 + (lane >> 2);
    double* ptr[8];
    double old[8];
#pragma unroll
    for (int e = 0; e < 8; e++) {
      const int gc = c0 + wn + (e >> 1) * 8 + 2 * (lane & 3) + (e & 1);
      ptr[e] = (gi < nt && gc < nt) ? D.A + (t0 + gi) + (size_t)(t0 + gc) * D.lda : nullptr;
    }
#pragma unroll
    for (int e = 0; e < 8; e++) old[e] = ptr[e] ? *ptr[e] : 0.0;
#pragma unroll
    for (int e = 0; e < 8; e++)
      if (ptr[e]) *ptr[e] = old[e] - acc[x][e >> 1][e & 1];
  }
}

// ------------------------------------------------------------------ diagonal-block inverses
// Inverses of the XB x XB diagonal blocks of L (unit lower) and U: the
// triangular solves below are then blocked GEMM-shaped steps -- the classic
// batched-TRSM scheme -- with no serial substitution chain left in them.
// grid (matrix, block), 128 threads: thread t < 64 inverts column t of L_kk,
// t >= 64 column t - 64 of U_kk.  Blocks past m are padded with the identity.
__global__ void __launch_bounds__(128) lu_diag_inv_kernel(const MatDesc* __restrict__ desc,
                                                          const int64_t* __restrict__ doff,
                                                          const int64_t* __restrict__ foff, double* dinv,
                                                          unsigned char* flags, unsigned char* pflag,
                                                          double kappa_max) {
  __shared__ double T[XB][XB + 1];
  __shared__ double cn[2][XB][2];  // per inverted column: 1-norm of T_kk's column, of the inverse's column
  const MatDesc D = desc[blockIdx.x];
  const int nb = (D.m + XB - 1) / XB, k = blockIdx.y;
  if (k >= nb) return;
  const int kb = XB * k, bb = min(XB, D.m - kb);
  for (int e = threadIdx.x; e < XB * XB; e += 128) {
    const int r = e % XB, c = e / XB;
    T[r][c] = (r < bb && c < bb) ? D.A[(kb + r) + (size_t)(kb + c) * D.lda] : (r == c ? 1.0 : 0.0);
  }
  __syncthreads();
  const int t = threadIdx.x & (XB - 1);
  double x[XB];
  double* out = dinv + doff[blockIdx.x] + (size_t)k * 2 * XB * XB;
  if (threadIdx.x < XB) {  // L_kk^-1 e_t, forward
#pragma unroll
    for (int i = 0; i < XB; i++) {
      double v = (i == t) ? 1.0 : 0.0;
#pragma unroll
      for (int j = 0; j < i; j++) v = fma(-T[i][j], x[j], v);
      x[i] = v;
    }
  } else {  // U_kk^-1 e_t, backward
#pragma unroll
    for (int i = XB - 1; i >= 0; i--) {
      double v = (i == t) ? 1.0 : 0.0;
#pragma unroll
      for (int j = i + 1; j < XB; j++) v = fma(-T[i][j], x[j], v);
      x[i] = v / T[i][i];
    }
    out += XB * XB;
  }
  double inv1 = 0.0, t1 = 0.0;
#pragma unroll
  for (int i = 0; i < XB; i++) {
    out[i + XB * t] = x[i];
    inv1 += fabs(x[i]);
  }
  const bool up = threadIdx.x >= XB;
  for (int i = 0; i < XB; i++)  // column t of the triangle itself (unit diagonal for L)
    if (up ? i <= t : i >= t) t1 += (!up && i == t) ? 1.0 : fabs(T[i][t]);
  cn[up][t][0] = t1;
  cn[up][t][1] = inv1;
  __syncthreads();
  if (threadIdx.x < 2) {
    // kappa_1(T_kk) = ||T_kk||_1 ||T_kk^-1||_1 exactly; refine the block solve
    // when an inverted block's error, ~ kappa eps, is not far below the tolerance
    double a = 0.0, b = 0.0;
    for (int c = 0; c < XB; c++) {
      a = fmax(a, cn[threadIdx.x][c][0]);
      b = fmax(b, cn[threadIdx.x][c][1]);
    }
    const bool refine = !(a * b <= kappa_max);
    const size_t f = (size_t)foff[blockIdx.x] + k;
    if (threadIdx.x == 0) flags[2 * f] = refine;
    else flags[2 * f + 1] = refine;
    if (refine) pflag[blockIdx.x] = 1;
  }
}

// ------------------------------------------------------------------ condition estimate
// Blocked triangular solves of one shared-memory vector v (length padded to
// XB nb, zeros past m) by a 256-thread CTA, left-looking: per XB-row block the
// coupling to the solved part is a coalesced mat-vec split over the 8 warps
// (several independent loads in flight per thread), then the block is finished
// by its inverted diagonal block.  part: 8 XB doubles, rb: XB doubles.
//   v := L^-1 v, U^-1 v, U^-T v, L^-T v   (dg: this matrix's diagonal inverses)
template <int KIND>  // 0 L, 1 U, 2 U^T, 3 L^T
__device__ inline void blk_trsv(const MatDesc& D, const double* __restrict__ dg, double* v, double* part,
                                double* rb) {
  const int m = D.m, ld = D.lda, nb = (m + XB - 1) / XB;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool fwd = (KIND == 0 || KIND == 2);
  for (int s = 0; s < nb; s++) {
    const int k = fwd ? s : nb - 1 - s, kb = XB * k;
    const int j0 = fwd ? 0 : min(m, kb + XB), j1 = fwd ? kb : m;  // solved part
    if (KIND == 0 || KIND == 1) {
      // rows kb + lane and kb + 32 + lane, columns j of the factor (coalesced per column)
      const int r0 = kb + lane, r1 = r0 + 32;
      const bool ok0 = r0 < m, ok1 = r1 < m;
      double c0 = 0.0, c1 = 0.0;
      int j = j0 + warp;
      for (; j + 24 < j1; j += 32) {
        double a[4], b[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
          a[u] = ok0 ? D.A[r0 + (size_t)(j + 8 * u) * ld] : 0.0;
          b[u] = ok1 ? D.A[r1 + (size_t)(j + 8 * u) * ld] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; u++) {
          c0 = fma(a[u], v[j + 8 * u], c0);
          c1 = fma(b[u], v[j + 8 * u], c1);
        }
      }
      for (; j < j1; j += 8) {
        if (ok0) c0 = fma(D.A[r0 + (size_t)j * ld], v[j], c0);
        if (ok1) c1 = fma(D.A[r1 + (size_t)j * ld], v[j], c1);
      }
      part[warp * XB + lane] = c0;
      part[warp * XB + 32 + lane] = c1;
    } else {
      // transposed: output i of the block is the dot product of factor column
      // kb + i (rows j0..j1, contiguous) with v
#pragma unroll
      for (int q = 0; q < XB / 8; q++) {
        const int i = warp + 8 * q, col = kb + i;
        double d = 0.0;
        if (col < m) {
          const double* c = D.A + (size_t)col * ld;
          int j = j0 + lane;
          for (; j + 96 < j1; j += 128) {
            const double a0 = c[j], a1 = c[j + 32], a2 = c[j + 64], a3 = c[j + 96];
            d = fma(a0, v[j], d);
            d = fma(a1, v[j + 32], d);
            d = fma(a2, v[j + 64], d);
            d = fma(a3, v[j + 96], d);
          }
          for (; j < j1; j += 32) d = fma(c[j], v[j], d);
        }
        d = warp_sum(d);
        if (lane == 0) part[i] = d;
      }
    }
    __syncthreads();
    if (tid < XB) {
      double r = v[kb + tid];
      if (KIND == 0 || KIND == 1) {
#pragma unroll
        for (int w = 0; w < 8; w++) r -= part[w * XB + tid];
      } else {
        r -= part[tid];
      }
      rb[tid] = r;
    }
    __syncthreads();
    if (tid < XB) {
      // block inverse: L (KIND 0, 3) or U (1, 2); transposed for 2, 3
      const double* Bi = dg + (size_t)k * 2 * XB * XB + ((KIND == 1 || KIND == 2) ? XB * XB : 0);
      double o = 0.0;
#pragma unroll 8
      for (int c = 0; c < XB; c++) o = fma((KIND <= 1) ? Bi[tid + XB * c] : Bi[c + XB * tid], rb[c], o);
      v[kb + tid] = (kb + tid < m) ? o : 0.0;
    }
    __syncthreads();
  }
}
__device__ inline double vasum(const double* v, int n, double* red) {
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += fabs(v[i]);
  return block_sum(s, red);
}
__device__ inline int viamax(const double* v, int n, ArgMax* red) {
  ArgMax a{-1.0, -1};
  for (int i = threadIdx.x; i < n; i += blockDim.x) a = argmax_merge(a, ArgMax{fabs(v[i]), i});
  return block_argmax(a, red).i;
}

// LAPACK dlacn2 (Hager/Higham) on B = U^-1 L^-1, as dgecon runs it: dgecon
// estimates ||A^-1||_1 through the triangular factors alone (the row
// permutation only permutes columns of A^-1 and leaves the 1-norm unchanged),
// so the estimator's iterates, hence the estimate, follow LAPACK's.
__global__ void __launch_bounds__(256) lu_inv_norm1_kernel(const MatDesc* __restrict__ desc,
                                                          const int64_t* __restrict__ doff,
                                                          const double* __restrict__ dinv, double* out) {
  extern __shared__ double sm[];
  __shared__ double red[32];
  __shared__ double part[8 * XB];
  __shared__ double rb[XB];
  __shared__ ArgMax ared[32];
  __shared__ int s_flag;
  const MatDesc D = desc[blockIdx.x];
  const int n = D.m, np = XB * ((n + XB - 1) / XB);
  if (n == 0) {
    if (threadIdx.x == 0) out[blockIdx.x] = 0.0;
    return;
  }
  const double* dg = dinv + doff[blockIdx.x];
  double* x = sm;
  double* sgn = x + np;
  auto apply = [&]() {  // x := U^-1 L^-1 x
    blk_trsv<0>(D, dg, x, part, rb);
    blk_trsv<1>(D, dg, x, part, rb);
  };
  auto apply_t = [&]() {  // x := L^-T U^-T x
    blk_trsv<2>(D, dg, x, part, rb);
    blk_trsv<3>(D, dg, x, part, rb);
  };
  for (int i = threadIdx.x; i < np; i += blockDim.x) x[i] = i < n ? 1.0 / n : 0.0;
  __syncthreads();
  apply();
  double est = vasum(x, n, red);
  if (n == 1) {
    if (threadIdx.x == 0) out[blockIdx.x] = est;
    return;
  }
  for (int i = threadIdx.x; i < np; i += blockDim.x) {
    sgn[i] = x[i] >= 0.0 ? 1.0 : -1.0;
    x[i] = i < n ? sgn[i] : 0.0;
  }
  __syncthreads();
  apply_t();
  int jj = viamax(x, n, ared);
  for (int iter = 2;; iter++) {
    for (int i = threadIdx.x; i < np; i += blockDim.x) x[i] = (i == jj) ? 1.0 : 0.0;
    __syncthreads();
    apply();
    const double old = est;
    est = vasum(x, n, red);
    if (threadIdx.x == 0) s_flag = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x)
      if ((x[i] >= 0.0 ? 1.0 : -1.0) != sgn[i]) s_flag = 1;
    __syncthreads();
    if (!s_flag || est <= old) break;
    for (int i = threadIdx.x; i < np; i += blockDim.x) {
      sgn[i] = x[i] >= 0.0 ? 1.0 : -1.0;
      x[i] = i < n ? sgn[i] : 0.0;
    }
    __syncthreads();
    apply_t();
    const int jlast = jj;
    jj = viamax(x, n, ared);
    // every thread reads x before any thread overwrites it for the next iterate
    const bool again = x[jlast] != fabs(x[jj]) && iter < 5;
    __syncthreads();
    if (!again) break;
  }
  for (int i = threadIdx.x; i < np; i += blockDim.x)
    x[i] = i < n ? ((i & 1) ? -1.0 : 1.0) * (1.0 + double(i) / double(n - 1)) : 0.0;
  __syncthreads();
  apply();
  const double temp = 2.0 * vasum(x, n, red) / (3.0 * n);
  if (threadIdx.x == 0) out[blockIdx.x] = temp > est ? temp : est;
}

// ------------------------------------------------------------------ X = S^-1 C
// One CTA per (pivot, TW-column tile of C_full): the permuted tile P C_full
// lives in shared memory (m x TW, column pitch == 4 mod 16 doubles), and the
// two triangular solves run left-looking by XB-row blocks:
//   X_k <- D_k^-1 (X_k - F[k, solved] X[solved])   (F = L forward, U backward)
// Factor blocks F[k, j] and the inverted diagonal blocks D_k^-1 stream through
// an S-stage cp.async pipeline in XB x 32 halves (one barrier per half); every
// product is DMMA m8n8k4 from shared memory.  8 warps: warp w owns rows
// 16 (w & 3) .. +16 of the block and TW / 16 16-column slabs -> 2 x (TW / 8)
// 8 x 8 tiles, so each fragment read from shared memory feeds two MMAs.
constexpr int XS_AP = XB + 4;  // A stage: [k][row], pitch == 4 mod 16
struct XChunk {
  // factor block (k, j), j != k; or, for j == k, step p of the diagonal block's
  // solve (0: D_k^-1; if the block is flagged for refinement, 1: T_kk, 2: D_k^-1
  // again); half h of its columns
  int bwd, k, j, p, h;
};
// fl: the matrix's refinement flags, fl[2 k + bwd]; sk: the last column
// block holds <= 32 valid columns (m - XB (nb - 1) <= 32), its second halves
// multiply zero padding and are skipped
__device__ __forceinline__ void xchunk_next(XChunk& c, int nb, const unsigned char* fl, bool sk) {
  if (c.h == 0 && !(sk && c.j == nb - 1)) {
    c.h = 1;
    return;
  }
  c.h = 0;
  if (fl && c.j == c.k && c.p < 2 && fl[2 * c.k + c.bwd]) {
    c.p++;
    return;
  }
  c.p = 0;
  if (!c.bwd) {
    if (c.j < c.k) c.j++;
    else if (c.k + 1 < nb) { c.k++; c.j = 0; }
    else { c.bwd = 1; c.k = nb - 1; c.j = nb - 1; }  // backward starts with the last block's diagonal
  } else {
    if (c.j > c.k) c.j--;  // walks j = nb-1 .. k+1, then the diagonal
    else { c.k--; c.j = nb - 1; }
  }
}
__device__ __forceinline__ void cp_async16(double* smem, const double* gmem, bool pred) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(pred ? gmem : nullptr), "r"(n));
}
// Stage half h of block (k, j) -- a 64-row x 32-column slab -- as As[kk * XS_AP + row].
// Thread t copies rows 2 (t & 31), +1 of columns (t >> 5) + NW q, q < 32 / NW: 16-byte
// copies when both rows are in range and the pair is 16-byte aligned (always for
// the diagonal inverses; for the factor when m or the column is even), else two
// 8-byte copies.  Address arithmetic is incremental in q.
template <int NW>
__device__ __forceinline__ void xchunk_load(double* As, const XChunk& c, const double* __restrict__ LU,
                                            const double* __restrict__ dg, int m, int tid) {
  constexpr int NQ = 32 / NW;  // columns per thread
  const int r = 2 * (tid & 31), kk0 = tid >> 5;
  double* dst = As + kk0 * XS_AP + r;
  if (c.j == c.k && c.p != 1) {
    const double* src = dg + (size_t)c.k * 2 * XB * XB + (c.bwd ? XB * XB : 0) + r + (size_t)XB * (32 * c.h + kk0);
#pragma unroll
    for (int q = 0; q < NQ; q++) cp_async16(dst + NW * q * XS_AP, src + NW * q * XB, true);
    return;
  }
  // a factor block, or the diagonal block T_kk itself (p == 1)
  const int row = XB * c.k + r, col0 = XB * c.j + 32 * c.h + kk0;
  const bool r0ok = row < m, r1ok = row + 1 < m;
  const bool diag = c.j == c.k;
  const double* src = LU + row + (size_t)col0 * m;
#pragma unroll
  for (int q = 0; q < NQ; q++) {
    const int col = col0 + NW * q;
    const double* s_ = src + (size_t)NW * q * m;
    double* d_ = dst + NW * q * XS_AP;
    bool ok0 = r0ok && col < m, ok1 = r1ok && col < m;
    if (diag) {
      // T_kk is triangular: keep only its own part (L strictly below / U on and above);
      // the unit diagonal of L is implicit in the LU storage
      if (c.bwd) {
        ok0 &= row <= col;
        ok1 &= row + 1 <= col;
      } else {
        ok0 &= row >= col;
        ok1 &= row + 1 >= col;
      }
    }
    if (diag && !c.bwd) {  // L_kk: the unit diagonal is stored directly (no copy to that slot)
      if (row == col) d_[0] = ok0 ? 1.0 : 0.0;
      else cp_async8(d_, s_, ok0);
      if (row + 1 == col) d_[1] = ok1 ? 1.0 : 0.0;
      else cp_async8(d_ + 1, s_ + 1, ok1);
    } else if (ok0 && ok1 && ((reinterpret_cast<uintptr_t>(s_) & 15) == 0)) {
      cp_async16(d_, s_, true);
    } else {
      cp_async8(d_, s_, ok0);
      cp_async8(d_ + 1, s_ + 1, ok1);
    }
  }
}

// One CTA per (pivot, TW-column tile of C_full); 8 warps, warp w owns rows
// 16 (w & 3) .. +16 of the XB-row block and TW / 16 8-column tiles.  Diagonal
// blocks: x1 = D_k^-1 R; for blocks flagged by lu_diag_inv (kappa(T_kk) eps not
// far below the fill tolerance) one step of refinement x = x1 + D_k^-1 (R - T_kk x1)
// follows -- the inverted block alone costs kappa(T_kk) eps, which tol = 1e-14
// fill compression cannot absorb (measured: the reference-default N = 8,000
// system matches the reference only with it); refined, the block solve is as
// accurate as substitution while every step stays a DMMA product.
template <int TW, int XS_STAGES, bool REFINE, int NW = 8>
__global__ void __launch_bounds__(32 * NW) lu_xsolve_kernel(const XSolveDesc* __restrict__ descs,
                                                            const int* __restrict__ tile_map) {
  constexpr int NT = 32 * NW;
  constexpr int NC = TW / (2 * NW);  // 8-column tiles per warp (NW / 4 column groups)
  static_assert(NC >= 1 && NC * 2 * NW == TW, "tile width / warp count");
  extern __shared__ double sm[];
  const XSolveDesc D = descs[tile_map[blockIdx.x]];
  const int c0 = (blockIdx.x - D.tile0) * TW;
  const int m = D.m, n = D.n, wl = D.wl, w = D.w;
  // each pivot is solved by one of the two instantiations: with refinement
  // support iff one of its diagonal blocks is flagged (the refinement state
  // costs registers that slow the common path by half, measured)
  if (m == 0 || (*D.pflag != 0) != REFINE) return;
  const int nb = (m + XB - 1) / XB, mp = XB * nb, xm = mp + 4;
  double* X = sm;
  double* As = sm + (size_t)TW * xm;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // gather the permuted panel asynchronously (one cp.async per element, all in
  // flight together; the first pipeline wait covers it): rows of C (top, in
  // pivot order), the -I block of the local slots (bottom), zeros elsewhere
  for (int l = tid; l < mp; l += NT) {
    const int i = l < m ? D.perm[l] : -1;
    const double* src = D.C + (i >= 0 && i < n ? i : 0);
#pragma unroll 8
    for (int c = 0; c < TW; c++) {
      const int cc = c0 + c;
      double* dst = X + (size_t)c * xm + l;
      if (i >= n && cc < w && cc >= wl && i - n == cc - wl) *dst = -1.0;
      else cp_async8(dst, src + (size_t)cc * n, i >= 0 && i < n && cc < wl);  // zero-fill otherwise
    }
  }
  cp_async_commit();
  const unsigned char* fl = REFINE ? D.dflag : nullptr;
  int T = 2 * nb * (nb - 1) + 4 * nb;  // off-diagonal halves + 2 halves per diagonal block, both sweeps
  if (REFINE)
    for (int q = 0; q < 2 * nb; q++) T += fl[q] ? 4 : 0;  // + 4 halves per refined diagonal block
  const bool sk = m - XB * (nb - 1) <= 32;
  if (sk) {  // skipped second halves of the last column block (backward off-diagonals, both diagonals)
    T -= nb + 1;
    if (REFINE) T -= 2 * (fl[2 * (nb - 1)] + fl[2 * (nb - 1) + 1]);
  }
  XChunk ci{0, 0, 0, 0, 0}, cc{0, 0, 0, 0, 0};
  auto issue = [&](int t) {
    if (t < T) {
      xchunk_load<NW>(As + (size_t)(t % XS_STAGES) * 32 * XS_AP, ci, D.LU, D.dinv, m, tid);
      xchunk_next(ci, nb, fl, sk);
    }
    cp_async_commit();
  };
  for (int t = 0; t < XS_STAGES - 1; t++) issue(t);
  double acc[2][NC][2];
#pragma unroll
  for (int a = 0; a < 2; a++)
#pragma unroll
    for (int b = 0; b < NC; b++) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int fk = lane & 3, fq = lane >> 2;
  // first row of the warp, first 8-column tile.  Warps w and w + 4 share an SM
  // sub-partition: they take complementary row groups (0/3, 1/2), so the rows
  // of a partly padded last block (skipped below) leave no sub-partition idle
  const int r0 = 16 * (warp & 3), cb = NC * (warp >> 2);
  // the refinement keeps R and x1 of the warp's own tiles in registers
  double rv[REFINE ? 2 : 1][NC][2], xv[REFINE ? 2 : 1][NC][2];
  // f(pointer into X_k at an owned accumulator element, that element's (a, b, e))
  auto own = [&](int kb, auto f) {
#pragma unroll
    for (int a = 0; a < 2; a++)
#pragma unroll
      for (int b = 0; b < NC; b++) {
        double* x0 = X + (size_t)(8 * (cb + b) + 2 * fk) * xm + kb + r0 + 8 * a + fq;
        f(x0, a, b, 0);
        f(x0 + xm, a, b, 1);
        acc[a][b][0] = acc[a][b][1] = 0.0;
      }
  };
  for (int t = 0; t < T; t++) {
    cp_async_wait<XS_STAGES - 2>();
    __syncthreads();
    issue(t + XS_STAGES - 1);
    const int kb = XB * cc.k;
    const bool diag = cc.j == cc.k;
    if (diag && cc.p == 0 && cc.h == 0) {  // R = X_k - acc
      if constexpr (REFINE) own(kb, [&](double* x, int a, int b, int e) { *x = rv[a][b][e] = *x - acc[a][b][e]; });
      else own(kb, [&](double* x, int a, int b, int e) { *x -= acc[a][b][e]; });
      __syncthreads();
    }
    const double* A = As + (size_t)(t % XS_STAGES) * 32 * XS_AP + fk * XS_AP + r0 + fq;
    const double* B = X + (size_t)(8 * cb + fq) * xm + XB * cc.j + 32 * cc.h + fk;
    const int bld = xm;
#pragma unroll
    for (int s = 0; s < 8; s++) {
      double fa[2], fb[NC];
#pragma unroll
      for (int a = 0; a < 2; a++) fa[a] = A[4 * s * XS_AP + 8 * a];
#pragma unroll
      for (int b = 0; b < NC; b++) fb[b] = B[(size_t)8 * b * bld + 4 * s];
#pragma unroll
      for (int a = 0; a < 2; a++)
#pragma unroll
        for (int b = 0; b < NC; b++)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(acc[a][b][0]), "+d"(acc[a][b][1])
                       : "d"(fa[a]), "d"(fb[b]));
    }
    if (diag && (cc.h == 1 || (sk && cc.j == nb - 1))) {
      __syncthreads();  // every warp has read X_k
      if (!REFINE || !fl[2 * cc.k + cc.bwd]) {  // unrefined: X_k = D R
        own(kb, [&](double* x, int a, int b, int e) { *x = acc[a][b][e]; });
      } else if constexpr (REFINE) {
        if (cc.p == 0) {  // x1 = D R
          own(kb, [&](double* x, int a, int b, int e) { *x = xv[a][b][e] = acc[a][b][e]; });
        } else if (cc.p == 1) {  // the residual R - T x1
          own(kb, [&](double* x, int a, int b, int e) { *x = rv[a][b][e] - acc[a][b][e]; });
        } else {  // x = x1 + D (R - T x1)
          own(kb, [&](double* x, int a, int b, int e) { *x = xv[a][b][e] + acc[a][b][e]; });
        }
      }
    }
    xchunk_next(cc, nb, fl, sk);
  }
  cp_async_wait<0>();
  __syncthreads();
  // a thread owns a row: its column stores are coalesced across the CTA and
  // independent of each other
  const int nc = min(TW, w - c0);
  for (int l = tid; l < m; l += NT) {
    const bool top = l < n;
    double* dst = (top ? D.Xtop + l : D.Xbot + (l - n)) + (size_t)c0 * (top ? n : D.r);
    const size_t ld = top ? n : D.r;
#pragma unroll 8
    for (int c = 0; c < TW; c++)
      if (c < nc) dst[(size_t)c * ld] = X[(size_t)c * xm + l];
  }
}

}  // namespace

int lu_tile_width(int m) {
  const size_t xm = size_t(m | 1);
  for (int tw = 32; tw >= 8; tw /= 2)
    if (size_t(tw) * xm * sizeof(double) <= LU_TILE_SMEM_MAX) return tw;
  return 0;
}

static size_t xsolve_smem(int tw, int stages, int m) {
  const size_t mp = size_t(XB) * ((m + XB - 1) / XB);
  return sizeof(double) * (size_t(tw) * (mp + 4) + size_t(stages) * 32 * XS_AP);
}

LuDiag launch_lu_diag_inv(const std::vector<MatDesc>& h, const MatDesc* d_desc, Arena& ws, Staging& st,
                          cudaStream_t s, double tol, Arena* keep, int keep_min_m) {
  std::vector<int64_t> off(h.size() + 1, 0), foff(h.size() + 1, 0);
  int maxnb = 0;
  int64_t tot = 0;
  for (size_t p = 0; p < h.size(); p++) {
    const int nb = (h[p].m + XB - 1) / XB;
    maxnb = std::max(maxnb, nb);
    foff[p + 1] = foff[p] + nb;
    const bool kept = keep != nullptr && h[p].m >= keep_min_m;
    off[p] = kept ? -1 : tot;
    if (!kept) tot += int64_t(nb) * 2 * XB * XB;
  }
  LuDiag dg;
  dg.dinv = ws.alloc_n<double>(size_t(std::max<int64_t>(1, tot)));
  for (size_t p = 0; p < h.size(); p++)
    if (off[p] < 0) {  // kept with the records: its own allocation, addressed relative to dinv
      const int nb = (h[p].m + XB - 1) / XB;
      const double* kp = keep->alloc_n<double>(size_t(nb) * 2 * XB * XB);
      off[p] = (int64_t(reinterpret_cast<intptr_t>(kp)) - int64_t(reinterpret_cast<intptr_t>(dg.dinv))) /
               int64_t(sizeof(double));
    }
  dg.flags = ws.alloc_n<unsigned char>(size_t(std::max<int64_t>(1, 2 * foff.back())));
  dg.pflag = (keep ? *keep : ws).alloc_n<unsigned char>(std::max<size_t>(1, h.size()));
  CK(cudaMemsetAsync(dg.pflag, 0, std::max<size_t>(1, h.size()), s));
  dg.d_off = upload(ws, off, s, st);
  dg.h_off = off;
  dg.d_foff = upload(ws, foff, s, st);
  dg.h_foff = foff;
  // refine a block solve when its inverted block's error kappa eps could reach
  // a hundredth of the tolerance (tol <= 0: always)
  const double kappa_max = tol > 0 ? 1e-2 * tol / 2.220446049250313e-16 : 0.0;
  if (!h.empty() && maxnb > 0) {
    lu_diag_inv_kernel<<<dim3(unsigned(h.size()), unsigned(maxnb)), 128, 0, s>>>(d_desc, dg.d_off, dg.d_foff, dg.dinv,
                                                                                dg.flags, dg.pflag, kappa_max);
    CK_LAUNCH();
  }
  return dg;
}

void batched_lu(const std::vector<MatDesc>& h, const MatDesc* d_desc, int* d_info, Arena& ws, Staging& st,
                cudaStream_t s, int shape_maxm, SideStream* la) {
  (void)st;
  const int n = int(h.size());
  if (n == 0) return;
  int maxm = shape_maxm;
  for (auto& d : h) maxm = std::max(maxm, d.m);
  // panel width: the shared-memory panel (maxm x (b+1)) must fit
  int b = 32;
  auto smem_for = [&](int bw) { return size_t(maxm) * (bw + 1) * 8 + size_t(maxm) * 8; };
  while (b > 1 && smem_for(b) > 220 * 1024) b /= 2;
  if (smem_for(b) > 220 * 1024) invalid("pivot block too large for the LU panel");
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(lu_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 * 1024));
    CK(cudaFuncSetAttribute(lu_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(GSMEM)));
    attr = true;
  }
  CK(cudaMemsetAsync(d_info, 0, sizeof(int) * n, s));
  RowMove* moves = static_cast<RowMove*>(ws.alloc(sizeof(RowMove) * size_t(n) * 2 * b));
  int* nmoves = ws.alloc_n<int>(n);
  lu_perm_init_kernel<<<n, 256, 0, s>>>(d_desc);
  CK_LAUNCH();
  const int pthreads = std::min(512, std::max(64, (maxm + 31) / 32 * 32));
  const int gy = std::max(1, std::min(16, (maxm + 63) / 64));
  auto panel = [&](int j, cudaStream_t ps) {
    const size_t smem = size_t(maxm - j) * (std::min(b, maxm - j) + 1) * 8 + size_t(maxm - j) * 8;
    // register panel while the tallest panel fits 3 rows per thread (b = 32)
    const int rows = maxm - j;
    if (b == 32 && rows <= 256) lu_panel_reg_kernel<1><<<n, 256, 0, ps>>>(d_desc, j, d_info, moves, nmoves);
    else if (b == 32 && rows <= 512) lu_panel_reg_kernel<2><<<n, 256, 0, ps>>>(d_desc, j, d_info, moves, nmoves);
    else if (b == 32 && rows <= 768) lu_panel_reg_kernel<3><<<n, 256, 0, ps>>>(d_desc, j, d_info, moves, nmoves);
    else lu_panel_kernel<<<n, pthreads, smem, ps>>>(d_desc, j, b, d_info, moves, nmoves);
    CK_LAUNCH();
  };
  // Look-ahead for batches of few matrices (the coarse levels, where the
  // single-CTA panel chain is the critical path): after step j's row moves,
  // the trailing update of the first column tile (it holds panel j+1) runs
  // first, panel j+1 then factors on the side stream while the rest of the
  // update proceeds; step j+1's moves wait for both.  Same kernels, same
  // arithmetic on disjoint columns: identical factors.
  const bool ahead = la != nullptr && n < 148 && b == 32 && GBN >= 2 * b;
  if (ahead) la->ensure();
  panel(0, s);
  for (int j = 0; j < maxm; j += b) {
    lu_swap_trsm_kernel<<<dim3(n, gy), 256, 0, s>>>(d_desc, j, b, moves, nmoves);
    CK_LAUNCH();
    int rt = 0;
    for (auto& d : h)
      if (d.m > j + b) rt = std::max(rt, ceil_div(d.m - j - b, GBM));
    const bool next = j + b < maxm;
    if (rt == 0) {
      if (next) panel(j + b, s);
      continue;
    }
    if (ahead && next) {
      lu_update_kernel<<<dim3(n, rt), GTHREADS, GSMEM, s>>>(d_desc, j, b, 0, 1);
      CK_LAUNCH();
      CK(cudaEventRecord(la->fork, s));
      CK(cudaStreamWaitEvent(la->s, la->fork, 0));
      panel(j + b, la->s);
      CK(cudaEventRecord(la->join, la->s));
      if (rt > 1) {
        lu_update_kernel<<<dim3(n, rt * (rt - 1)), GTHREADS, GSMEM, s>>>(d_desc, j, b, 1, -1);
        CK_LAUNCH();
      }
      CK(cudaStreamWaitEvent(s, la->join, 0));
    } else {
      lu_update_kernel<<<dim3(n, rt * rt), GTHREADS, GSMEM, s>>>(d_desc, j, b, 0, -1);
      CK_LAUNCH();
      if (next) panel(j + b, s);
    }
  }
}

void launch_lu_inv_norm1(const MatDesc* d_desc, int n, int maxm, const LuDiag& dg, double* out, cudaStream_t s) {
  if (n <= 0) return;
  const size_t smem = sizeof(double) * 2 * size_t(XB * ((std::max(1, maxm) + XB - 1) / XB));
  if (smem > 200 * 1024) invalid("pivot block too large for the condition estimate");
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(lu_inv_norm1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  lu_inv_norm1_kernel<<<n, 256, smem, s>>>(d_desc, dg.d_off, dg.dinv, out);
  CK_LAUNCH();
}

void launch_lu_solve_x(const std::vector<XSolveDesc>& hin, Arena& ws, Staging& st, cudaStream_t s) {
  if (hin.empty()) return;
  // Configuration per pivot, from its own m (the columns of X do not depend on
  // it: every element accumulates the same DMMA sequence): 32-column tiles at
  // two CTAs per SM with 3 stages while the tile is small, else one CTA with 4
  // stages -- the prefetch distance must cover the L2 latency with one CTA's
  // compute; 16-column tiles for the largest pivots.  Pivots of one
  // configuration share a launch sized for their largest m (a batch mixes m
  // from ~100 to ~1,000 at the coarse levels: one shared configuration would
  // give every pivot the largest pivot's shared memory and tile width).
  auto cfg_of = [](int m) {
    if (xsolve_smem(32, 3, m) <= 110 * 1024) return 0;
    if (xsolve_smem(32, 4, m) <= 220 * 1024) return 1;
    if (xsolve_smem(16, 4, m) <= 220 * 1024) return 2;
    if (xsolve_smem(16, 3, m) <= 220 * 1024) return 3;
    if (xsolve_smem(16, 2, m) <= 220 * 1024) return 4;  // the dense leaves of clustered inputs
    if (xsolve_smem(8, 2, m) <= 220 * 1024) return 5;   // (m up to 2,944: 8-column tiles, 4 warps)
    return -1;
  };
  std::vector<XSolveDesc> h(hin);
  std::vector<int> maps[6];
  int maxm[6] = {0, 0, 0, 0, 0, 0};
  for (size_t p = 0; p < h.size(); p++) {
    if (h[p].m <= 0) continue;
    const int cfg = cfg_of(h[p].m);
    if (cfg < 0) invalid("pivot block too large for the X solve (m = " + std::to_string(h[p].m) + ")");
    const int tw = cfg == 5 ? 8 : cfg >= 2 ? 16 : 32;
    std::vector<int>& map = maps[cfg];
    h[p].tile0 = int(map.size());
    maxm[cfg] = std::max(maxm[cfg], h[p].m);
    for (int t = 0, tiles = ceil_div(h[p].w, tw); t < tiles; t++) map.push_back(int(p));
  }
  bool any = false;
  for (auto& mp_ : maps) any |= !mp_.empty();
  if (!any) return;
  const XSolveDesc* dd = upload(ws, h, s, st);
  for (int cfg = 0; cfg < 6; cfg++) {
    if (maps[cfg].empty()) continue;
    const int tw = cfg == 5 ? 8 : cfg >= 2 ? 16 : 32;
    const int stages = cfg >= 4 ? 2 : (cfg == 0 || cfg == 3) ? 3 : 4;
    const int threads = cfg == 5 ? 128 : 256;
    const int* dm = upload(ws, maps[cfg], s, st);
    const size_t smem = xsolve_smem(tw, stages, maxm[cfg]);
    const unsigned grid = unsigned(maps[cfg].size());
    auto go = [&](void (*kern)(const XSolveDesc*, const int*)) {
      static std::mutex mu;
      static std::set<const void*> ready;  // kernels whose shared-memory limit is raised
      {
        std::lock_guard<std::mutex> lk(mu);
        if (ready.insert(reinterpret_cast<const void*>(kern)).second)
          CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
      }
      kern<<<grid, threads, smem, s>>>(dd, dm);
      CK_LAUNCH();
    };
    // every pivot is handled by exactly one of the two launches (lu_xsolve_kernel)
    if (cfg == 0) { go(lu_xsolve_kernel<32, 3, false>); go(lu_xsolve_kernel<32, 3, true>); }
    else if (cfg == 1) { go(lu_xsolve_kernel<32, 4, false>); go(lu_xsolve_kernel<32, 4, true>); }
    else if (cfg == 2) { go(lu_xsolve_kernel<16, 4, false>); go(lu_xsolve_kernel<16, 4, true>); }
    else if (cfg == 3) { go(lu_xsolve_kernel<16, 3, false>); go(lu_xsolve_kernel<16, 3, true>); }
    else if (cfg == 4) { go(lu_xsolve_kernel<16, 2, false>); go(lu_xsolve_kernel<16, 2, true>); }
    else { go(lu_xsolve_kernel<8, 2, false, 4>); go(lu_xsolve_kernel<8, 2, true, 4>); }
  }
}

}  // namespace ifmm
