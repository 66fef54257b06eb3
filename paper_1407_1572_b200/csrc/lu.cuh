// Batched LU with partial pivoting for the IFMM pivot blocks
// S_i = [[P2P_ii, U_i], [U_i^T, 0]] and the level-2 top system -- the
// reference's lu_factor / dgecon / lu_solve (ifmm/solver.py:214-218,246,
// 545,583,594,613), backward-stable where explicit inverses are not.
//
//   batched_lu      blocked right-looking getrf, 32-column panels: panel
//                   factorization (pivot search in shared memory) -> row moves
//                   + U12 = L11^-1 A12 (one warp per column) -> DMMA trailing
//                   update A22 -= L21 U12, all matrices of a batch per launch.
//                   Rows are tracked as a permutation `perm` (row l of P S is
//                   row perm[l] of S), kept with the factors for the solves.
//   lu_diag_inv     inverses of the 64 x 64 diagonal blocks of L and U, which
//                   make the blocked triangular solves GEMM-shaped.
//   lu_solve_x      X = S^-1 C for the pivot's coupling panel: one CTA per
//                   (matrix, column tile), the tile resident in shared memory,
//                   factor blocks streamed from L2 by cp.async; left-looking
//                   64-row blocks, every product on DMMA (diagonal blocks by
//                   their inverse plus one refinement step).
//   lu_inv_norm1    dlacn2 estimate of ||S^-1||_1 with blocked LU solves (the
//                   estimator dgecon runs, ifmm/solver.py:216).
#pragma once
#include "batched.cuh"
#include "core.cuh"

namespace ifmm {

// ------------------------------------------------------------------ device helpers
// Triangular solves of one shared-memory vector by a whole CTA, blocked by 32
// rows: warp 0 substitutes the diagonal block (lanes own rows, shuffles carry
// the solved entries), every thread then updates the remaining rows (thread
// per row, coalesced column reads of the factor).  Barriers at block borders.
__device__ inline void cta_trsv_lower_unit(const double* __restrict__ LU, int ld, int m, double* x) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int kb = 0; kb < m; kb += 32) {
    const int bb = min(32, m - kb);
    if (warp == 0) {
      double lrow[32];
#pragma unroll
      for (int c = 0; c < 32; c++) lrow[c] = (c < lane && lane < bb) ? LU[(kb + lane) + (size_t)(kb + c) * ld] : 0.0;
      double v = lane < bb ? x[kb + lane] : 0.0;
#pragma unroll
      for (int c = 0; c < 31; c++) {
        const double xc = __shfl_sync(0xffffffffu, v, c);
        v = fma(-lrow[c], xc, v);
      }
      if (lane < bb) x[kb + lane] = v;
    }
    __syncthreads();
    // all 32 loads of a row in flight (a runtime-bound loop issues them one L2 latency apart)
    for (int r = kb + bb + threadIdx.x; r < m; r += blockDim.x) {
      double a[32];
#pragma unroll
      for (int c = 0; c < 32; c++) a[c] = c < bb ? LU[r + (size_t)(kb + c) * ld] : 0.0;
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < 32; c++) s = fma(a[c], c < bb ? x[kb + c] : 0.0, s);
      x[r] -= s;
    }
    __syncthreads();
  }
}

__device__ inline void cta_trsv_upper(const double* __restrict__ LU, int ld, int m, double* x) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int kb = ((m - 1) / 32) * 32; kb >= 0; kb -= 32) {
    const int bb = min(32, m - kb);
    if (warp == 0) {
      double urow[32];
#pragma unroll
      for (int c = 0; c < 32; c++) urow[c] = (c >= lane && c < bb) ? LU[(kb + lane) + (size_t)(kb + c) * ld] : 0.0;
      // one reciprocal per row, off the dependency chain (a full-range f64
      // division inside the substitution loop runs the slow division path)
      const double rinv = lane < bb ? 1.0 / LU[(kb + lane) + (size_t)(kb + lane) * ld] : 0.0;
      double v = lane < bb ? x[kb + lane] : 0.0;
#pragma unroll
      for (int c = 31; c >= 0; c--) {
        if (lane == c) v *= rinv;
        const double xc = __shfl_sync(0xffffffffu, v, c);
        if (lane < c) v = fma(-urow[c], xc, v);
      }
      if (lane < bb) x[kb + lane] = v;
    }
    __syncthreads();
    for (int r = threadIdx.x; r < kb; r += blockDim.x) {
      double a[32];
#pragma unroll
      for (int c = 0; c < 32; c++) a[c] = c < bb ? LU[r + (size_t)(kb + c) * ld] : 0.0;
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < 32; c++) s = fma(a[c], c < bb ? x[kb + c] : 0.0, s);
      x[r] -= s;
    }
    __syncthreads();
  }
}

// U^T y = x (forward): left-looking, block dot products over U's columns
// (contiguous), then the transposed diagonal block by substitution.
__device__ inline void cta_trsv_upper_t(const double* __restrict__ LU, int ld, int m, double* x) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int kb = 0; kb < m; kb += 32) {
    const int bb = min(32, m - kb);
    for (int t = warp; t < bb; t += nw) {
      const double* col = LU + (size_t)(kb + t) * ld;
      double s = 0.0;
#pragma unroll 4
      for (int c = lane; c < kb; c += 32) s = fma(col[c], x[c], s);
      s = warp_sum(s);
      if (lane == 0) x[kb + t] -= s;
    }
    __syncthreads();
    if (warp == 0) {
      const double rinv = lane < bb ? 1.0 / LU[(kb + lane) + (size_t)(kb + lane) * ld] : 0.0;
      double v = lane < bb ? x[kb + lane] : 0.0;
      for (int c = 0; c < bb; c++) {
        if (lane == c) v *= rinv;
        const double yc = __shfl_sync(0xffffffffu, v, c);
        if (lane > c && lane < bb) v = fma(-LU[(kb + c) + (size_t)(kb + lane) * ld], yc, v);
      }
      if (lane < bb) x[kb + lane] = v;
    }
    __syncthreads();
  }
}

// L^T z = y (backward, unit diagonal)
__device__ inline void cta_trsv_lower_unit_t(const double* __restrict__ LU, int ld, int m, double* x) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int kb = ((m - 1) / 32) * 32; kb >= 0; kb -= 32) {
    const int bb = min(32, m - kb);
    for (int t = warp; t < bb; t += nw) {
      const double* col = LU + (size_t)(kb + t) * ld;
      double s = 0.0;
#pragma unroll 4
      for (int c = kb + bb + lane; c < m; c += 32) s = fma(col[c], x[c], s);
      s = warp_sum(s);
      if (lane == 0) x[kb + t] -= s;
    }
    __syncthreads();
    if (warp == 0) {
      double v = lane < bb ? x[kb + lane] : 0.0;
      for (int c = bb - 1; c >= 0; c--) {
        const double zc = __shfl_sync(0xffffffffu, v, c);
        if (lane < c) v = fma(-LU[(kb + c) + (size_t)(kb + lane) * ld], zc, v);
      }
      if (lane < bb) x[kb + lane] = v;
    }
    __syncthreads();
  }
}

// Tile solve X <- U^-1 L^-1 X for a shared-memory tile of TW columns (column
// c at X + c*xm), rows already in pivot order.  TW in {8, 16, 32}, 8 warps.
// Per 32-row block: the diagonal block by substitution, every warp taking
// TW/8 columns (lanes own rows, the block's factor column values sit in
// registers, shuffles carry the solved entries -- no barriers inside); then
// the off-diagonal update on DMMA (m8n8k4): warps own 8-row strips of all TW
// columns, the factor operand's 8 k-steps are loaded before the MMAs.  Kept
// under 85 registers so three 256-thread CTAs share an SM.
template <int TW>
__device__ inline void cta_tile_lu_solve(const double* __restrict__ LU, int ld, int m, double* X, int xm) {
  static_assert(TW == 8 || TW == 16 || TW == 32, "tile width");
  constexpr int NS = TW / 8;   // 8-column strips of the tile
  constexpr int NQW = TW / 8;  // columns per warp in the diagonal solves (8 warps)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // rows [r_lo, r_hi) of X -= F[rows, kb:kb+bb] X[kb:kb+bb]  (F = L below / U above)
  // two 8-row strips per warp pass: every tile-operand fragment read from
  // shared memory feeds two MMAs (the kernel is L1/shared-bandwidth bound)
  auto update = [&](int kb, int bb, int r_lo, int r_hi) {
    const int nstrips = (r_hi - r_lo + 7) / 8;
    for (int sp = 2 * warp; sp < nstrips; sp += 16) {
      const int rr0 = r_lo + sp * 8 + (lane >> 2), rr1 = rr0 + 8;
      double af0[8], af1[8];
#pragma unroll
      for (int s = 0; s < 8; s++) {
        const int kk = 4 * s + (lane & 3);
        af0[s] = (rr0 < r_hi && kk < bb) ? LU[rr0 + (size_t)(kb + kk) * ld] : 0.0;
        af1[s] = (rr1 < r_hi && kk < bb) ? LU[rr1 + (size_t)(kb + kk) * ld] : 0.0;
      }
      double acc0[NS][2], acc1[NS][2];
#pragma unroll
      for (int q = 0; q < NS; q++) acc0[q][0] = acc0[q][1] = acc1[q][0] = acc1[q][1] = 0.0;
#pragma unroll
      for (int s = 0; s < 8; s++) {
        const int kk = 4 * s + (lane & 3);
#pragma unroll
        for (int q = 0; q < NS; q++) {
          const double bq = kk < bb ? X[(size_t)(q * 8 + (lane >> 2)) * xm + kb + kk] : 0.0;
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(acc0[q][0]), "+d"(acc0[q][1])
                       : "d"(af0[s]), "d"(bq));
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(acc1[q][0]), "+d"(acc1[q][1])
                       : "d"(af1[s]), "d"(bq));
        }
      }
#pragma unroll
      for (int q = 0; q < NS; q++) {
        const int c = q * 8 + 2 * (lane & 3);
        if (rr0 < r_hi) {
          X[(size_t)c * xm + rr0] -= acc0[q][0];
          X[(size_t)(c + 1) * xm + rr0] -= acc0[q][1];
        }
        if (rr1 < r_hi) {
          X[(size_t)c * xm + rr1] -= acc1[q][0];
          X[(size_t)(c + 1) * xm + rr1] -= acc1[q][1];
        }
      }
    }
  };
  // ---- forward: unit lower
  for (int kb = 0; kb < m; kb += 32) {
    const int bb = min(32, m - kb);
    {
      double lr[32];
#pragma unroll
      for (int c = 0; c < 32; c++) lr[c] = (c < lane && lane < bb) ? LU[(kb + lane) + (size_t)(kb + c) * ld] : 0.0;
      double v[NQW];
#pragma unroll
      for (int u = 0; u < NQW; u++) v[u] = lane < bb ? X[(size_t)(warp + 8 * u) * xm + kb + lane] : 0.0;
#pragma unroll
      for (int c = 0; c < 31; c++)
#pragma unroll
        for (int u = 0; u < NQW; u++) v[u] = fma(-lr[c], __shfl_sync(0xffffffffu, v[u], c), v[u]);
      if (lane < bb)
#pragma unroll
        for (int u = 0; u < NQW; u++) X[(size_t)(warp + 8 * u) * xm + kb + lane] = v[u];
    }
    __syncthreads();
    update(kb, bb, kb + bb, m);
    __syncthreads();
  }
  // ---- backward: upper, non-unit
  for (int kb = ((m - 1) / 32) * 32; kb >= 0; kb -= 32) {
    const int bb = min(32, m - kb);
    {
      double ur[32];
#pragma unroll
      for (int c = 0; c < 32; c++) ur[c] = (c > lane && c < bb) ? LU[(kb + lane) + (size_t)(kb + c) * ld] : 0.0;
      const double rinv = lane < bb ? 1.0 / LU[(kb + lane) + (size_t)(kb + lane) * ld] : 0.0;
      double v[NQW];
#pragma unroll
      for (int u = 0; u < NQW; u++) v[u] = lane < bb ? X[(size_t)(warp + 8 * u) * xm + kb + lane] : 0.0;
#pragma unroll
      for (int c = 31; c >= 0; c--) {
#pragma unroll
        for (int u = 0; u < NQW; u++) {
          if (lane == c) v[u] *= rinv;
          const double xc = __shfl_sync(0xffffffffu, v[u], c);
          if (lane < c) v[u] = fma(-ur[c], xc, v[u]);
        }
      }
      if (lane < bb)
#pragma unroll
        for (int u = 0; u < NQW; u++) X[(size_t)(warp + 8 * u) * xm + kb + lane] = v[u];
    }
    __syncthreads();
    update(kb, bb, 0, kb);
    __syncthreads();
  }
}

// Column-by-column fallback (nq < 8 columns, or tiles that are not multiples of 8)
__device__ inline void cta_tile_lu_solve_cols(const double* __restrict__ LU, int ld, int m, double* X, int xm,
                                              int nq) {
  for (int q = 0; q < nq; q++) {
    cta_trsv_lower_unit(LU, ld, m, X + (size_t)q * xm);
    cta_trsv_upper(LU, ld, m, X + (size_t)q * xm);
  }
}

// ------------------------------------------------------------------ host entry points
// In-place LU of every matrix (partial pivoting, LAPACK getrf semantics).
// D.ipiv receives the row permutation `perm` (row l of P S = row perm[l] of S);
// info[p] = 0, or 1 + the first column with an exact zero pivot.
// shape_maxm: largest matrix of the whole colour batch (across ranks) so the
// panel width -- hence the arithmetic -- does not depend on the sharding.
// la: a side stream for the panel look-ahead of batches of few matrices (null: none).
void batched_lu(const std::vector<MatDesc>& h, const MatDesc* d_desc, int* d_info, Arena& ws, Staging& st,
                cudaStream_t s, int shape_maxm = 0, SideStream* la = nullptr);

// Inverses of the 64x64 diagonal blocks of every factored matrix (L_kk^-1 and
// U_kk^-1, column-major 64 x 64 each, identity-padded past m): matrix p's
// block k pair starts at dinv + h_off[p] + 8192 k.  They make the blocked
// triangular solves GEMM-shaped (the X solve refines each block solve once).
constexpr int SOLVE_BLK_MIN_M = 192;  // pivots from this size keep inverted diagonal blocks for the solve
constexpr int LU_XB = 64;  // block size of the blocked triangular solves (X solve, condition estimate)
struct LuDiag {
  double* dinv = nullptr;
  unsigned char* flags = nullptr;  // per block: [L, U] refine the block solve (lu.cu)
  unsigned char* pflag = nullptr;  // per matrix: any block flagged
  const int64_t* d_off = nullptr;
  std::vector<int64_t> h_off;   // per matrix: offset of its blocks from dinv, in doubles (matrices kept
                                // with the solve records live in another arena: the offset may be negative)
  const int64_t* d_foff = nullptr;
  std::vector<int64_t> h_foff;  // per matrix: index of its first block (flags: 2 per block)
};
// tol: the fill tolerance the X solve must support (decides which block solves
// get a refinement step); <= 0 refines every block.
// keep: arena for what must outlive the batch workspace (solve records): the per-matrix flags, and the
// inverted blocks of the matrices with m >= keep_min_m
LuDiag launch_lu_diag_inv(const std::vector<MatDesc>& h, const MatDesc* d_desc, Arena& ws, Staging& st,
                          cudaStream_t s, double tol, Arena* keep = nullptr, int keep_min_m = 1 << 30);

// out[p] = dlacn2 estimate of ||S_p^-1||_1 from the LU factors of S_p.
void launch_lu_inv_norm1(const MatDesc* d_desc, int n, int maxm, const LuDiag& dg, double* out, cudaStream_t s);

// X = S^-1 C_full for the coupling panel of a pivot, C_full = [[C, 0], [0, -I_r]]
// (m = n + r rows, w = wl + r columns; C is n x wl, ld n).  Rows [0, n) of X
// go to Xtop (ld n), rows [n, m) to Xbot (ld r).
struct XSolveDesc {
  const double* LU;
  const int* perm;
  const double* C;
  double* Xtop;
  double* Xbot;
  const double* dinv;           // the pivot's diagonal-block inverses (LuDiag)
  const unsigned char* dflag;   // and their refinement flags
  const unsigned char* pflag;   // any of them set
  int m, n, r, wl, w;
  int tile0;  // first tile of this matrix in the launch
};
void launch_lu_solve_x(const std::vector<XSolveDesc>& h, Arena& ws, Staging& st, cudaStream_t s);

// Largest tile width (columns) of cta_tile_lu_solve whose m x TW tile fits the
// shared-memory budget; 0 if even 8 columns do not fit.
int lu_tile_width(int m);
constexpr size_t LU_TILE_SMEM_MAX = 216 * 1024;

}  // namespace ifmm
