// Batched LU with partial pivoting, LU-based X = S^-1 C and the dlacn2
// condition estimate (see lu.cuh).  The reference factors every pivot with
// scipy lu_factor (LAPACK dgetrf), tests it with dgecon and applies it with
// lu_solve (dgetrs) (ifmm/solver.py:214-218,246); these kernels do the same
// on a whole colour batch at once.
#include <algorithm>

#include "gemm.cuh"
#include "lu.cuh"

namespace ifmm {

namespace {

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
__global__ void __launch_bounds__(GTHREADS, 3) lu_update_kernel(const MatDesc* __restrict__ desc, int j, int b) {
  extern __shared__ double gsm[];
  const MatDesc D = desc[blockIdx.x];
  const int m = D.m;
  if (m <= j) return;
  const int bb = min(b, m - j);
  const int t0 = j + bb, nt = m - t0;
  if (nt <= 0) return;
  const int tiles = (nt + GBM - 1) / GBM;
  const int tl = blockIdx.y;
  if (tl >= tiles * tiles) return;
  const int i0 = (tl % tiles) * GBM, c0 = (tl / tiles) * GBN;
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

// ------------------------------------------------------------------ condition estimate
// dgecon estimates ||A^-1||_1 as ||U^-1 L^-1||_1 (the row permutation only
// permutes columns of A^-1, which leaves the 1-norm unchanged) and runs the
// estimator on the triangular factors alone; so do these, so that the
// estimator's iterates -- hence the estimate -- follow LAPACK's.
// y = U^-1 L^-1 x (x, y distinct shared vectors)
__device__ inline void lu_apply(const MatDesc& D, const double* x, double* y) {
  for (int l = threadIdx.x; l < D.m; l += blockDim.x) y[l] = x[l];
  __syncthreads();
  cta_trsv_lower_unit(D.A, D.lda, D.m, y);
  cta_trsv_upper(D.A, D.lda, D.m, y);
}
// y = L^-T U^-T x
__device__ inline void lu_apply_t(const MatDesc& D, const double* x, double* y) {
  for (int l = threadIdx.x; l < D.m; l += blockDim.x) y[l] = x[l];
  __syncthreads();
  cta_trsv_upper_t(D.A, D.lda, D.m, y);
  cta_trsv_lower_unit_t(D.A, D.lda, D.m, y);
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

// LAPACK dlacn2 (Hager/Higham) on B = S^-1, as dgecon runs it
__global__ void __launch_bounds__(256, 3) lu_inv_norm1_kernel(const MatDesc* __restrict__ desc, double* out) {
  extern __shared__ double sm[];
  __shared__ double red[32];
  __shared__ ArgMax ared[32];
  __shared__ int s_flag;
  const MatDesc D = desc[blockIdx.x];
  const int n = D.m;
  if (n == 0) {
    if (threadIdx.x == 0) out[blockIdx.x] = 0.0;
    return;
  }
  double* x = sm;
  double* y = x + n;
  double* sgn = y + n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = 1.0 / n;
  __syncthreads();
  lu_apply(D, x, y);
  double est = vasum(y, n, red);
  if (n == 1) {
    if (threadIdx.x == 0) out[blockIdx.x] = est;
    return;
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) sgn[i] = y[i] >= 0.0 ? 1.0 : -1.0;
  __syncthreads();
  lu_apply_t(D, sgn, x);
  int jj = viamax(x, n, ared);
  for (int iter = 2;; iter++) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = (i == jj) ? 1.0 : 0.0;
    __syncthreads();
    lu_apply(D, x, y);
    const double old = est;
    est = vasum(y, n, red);
    if (threadIdx.x == 0) s_flag = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x)
      if ((y[i] >= 0.0 ? 1.0 : -1.0) != sgn[i]) s_flag = 1;
    __syncthreads();
    if (!s_flag || est <= old) break;
    for (int i = threadIdx.x; i < n; i += blockDim.x) sgn[i] = y[i] >= 0.0 ? 1.0 : -1.0;
    __syncthreads();
    lu_apply_t(D, sgn, x);
    const int jlast = jj;
    jj = viamax(x, n, ared);
    // every thread reads x before any thread overwrites it for the next iterate
    const bool again = x[jlast] != fabs(x[jj]) && iter < 5;
    __syncthreads();
    if (!again) break;
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    x[i] = ((i & 1) ? -1.0 : 1.0) * (1.0 + double(i) / double(n - 1));
  __syncthreads();
  lu_apply(D, x, y);
  const double temp = 2.0 * vasum(y, n, red) / (3.0 * n);
  if (threadIdx.x == 0) out[blockIdx.x] = temp > est ? temp : est;
}

// ------------------------------------------------------------------ X = S^-1 C
template <int TW, bool SCRATCH>
__global__ void __launch_bounds__(256, 3) lu_solve_x_kernel(const XSolveDesc* __restrict__ descs,
                                                         const int* __restrict__ tile_map, double* scratch,
                                                         size_t scratch_per_tile) {
  extern __shared__ double sm[];
  const XSolveDesc D = descs[tile_map[blockIdx.x]];
  const int c0 = (blockIdx.x - D.tile0) * TW;
  const int m = D.m, n = D.n, wl = D.wl, w = D.w;
  const int xm = m | 1;
  // (the shared-memory instantiation addresses X as shared: LDS/STS, not generic)
  double* X = SCRATCH ? scratch + scratch_per_tile * blockIdx.x : sm;
  for (int e = threadIdx.x; e < TW * m; e += blockDim.x) {
    const int c = e / m, l = e - c * m;
    const int i = D.perm[l], cc = c0 + c;
    double v = 0.0;
    if (cc < w) {
      if (i < n) v = cc < wl ? D.C[i + (size_t)cc * n] : 0.0;
      else v = (cc >= wl && i - n == cc - wl) ? -1.0 : 0.0;
    }
    X[(size_t)c * xm + l] = v;
  }
  __syncthreads();
  cta_tile_lu_solve<TW>(D.LU, m, m, X, xm);
  for (int e = threadIdx.x; e < TW * m; e += blockDim.x) {
    const int c = e / m, l = e - c * m;
    const int cc = c0 + c;
    if (cc >= w) continue;
    const double v = X[(size_t)c * xm + l];
    if (l < n) D.Xtop[l + (size_t)cc * n] = v;
    else D.Xbot[(l - n) + (size_t)cc * D.r] = v;
  }
}

}  // namespace

int lu_tile_width(int m) {
  const size_t xm = size_t(m | 1);
  for (int tw = 32; tw >= 8; tw /= 2)
    if (size_t(tw) * xm * sizeof(double) <= LU_TILE_SMEM_MAX) return tw;
  return 0;
}

// Tile width for the X solve: the widest tile that still lets three CTAs share
// an SM (the solve is latency-bound: occupancy beats operand reuse; measured at
// C3 level 5, m ~ 450: 32-column tiles leave one CTA per SM).
static int x_tile_width(int m) {
  const size_t xm = size_t(m | 1);
  for (int tw = 32; tw >= 8; tw /= 2)
    if (size_t(tw) * xm * sizeof(double) <= 72 * 1024) return tw;
  return lu_tile_width(m);
}

void batched_lu(const std::vector<MatDesc>& h, const MatDesc* d_desc, int* d_info, Arena& ws, Staging& st,
                cudaStream_t s, int shape_maxm) {
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
  for (int j = 0; j < maxm; j += b) {
    const size_t smem = size_t(maxm - j) * (std::min(b, maxm - j) + 1) * 8 + size_t(maxm - j) * 8;
    lu_panel_kernel<<<n, pthreads, smem, s>>>(d_desc, j, b, d_info, moves, nmoves);
    CK_LAUNCH();
    lu_swap_trsm_kernel<<<dim3(n, gy), 256, 0, s>>>(d_desc, j, b, moves, nmoves);
    CK_LAUNCH();
    int mt = 0;
    for (auto& d : h)
      if (d.m > j + b) mt = std::max(mt, ceil_div(d.m - j - b, GBM) * ceil_div(d.m - j - b, GBM));
    if (mt > 0) {
      lu_update_kernel<<<dim3(n, mt), GTHREADS, GSMEM, s>>>(d_desc, j, b);
      CK_LAUNCH();
    }
  }
}

void launch_lu_inv_norm1(const MatDesc* d_desc, int n, int maxm, double* out, cudaStream_t s) {
  if (n <= 0) return;
  const size_t smem = sizeof(double) * 3 * size_t(std::max(1, maxm));
  if (smem > 224 * 1024) invalid("pivot block too large for the condition estimate");
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(lu_inv_norm1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 * 1024));
    attr = true;
  }
  lu_inv_norm1_kernel<<<n, 256, smem, s>>>(d_desc, out);
  CK_LAUNCH();
}

void launch_lu_solve_x(const std::vector<XSolveDesc>& hin, Arena& ws, Staging& st, cudaStream_t s) {
  if (hin.empty()) return;
  int maxm = 0;
  for (auto& d : hin) maxm = std::max(maxm, d.m);
  int tw = x_tile_width(maxm);
  const bool global = tw == 0;
  if (global) tw = 8;
  std::vector<XSolveDesc> h(hin);
  std::vector<int> map;
  for (size_t p = 0; p < h.size(); p++) {
    h[p].tile0 = int(map.size());
    const int tiles = ceil_div(h[p].w, tw);
    for (int t = 0; t < tiles; t++) map.push_back(int(p));
  }
  if (map.empty()) return;
  const XSolveDesc* dd = upload(ws, h, s, st);
  const int* dm = upload(ws, map, s, st);
  const size_t per = size_t(tw) * size_t(maxm | 1);
  double* scratch = global ? ws.alloc_n<double>(per * map.size()) : nullptr;
  const size_t smem = global ? 0 : sizeof(double) * per;
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(lu_solve_x_kernel<32, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(LU_TILE_SMEM_MAX)));
    CK(cudaFuncSetAttribute(lu_solve_x_kernel<16, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(LU_TILE_SMEM_MAX)));
    CK(cudaFuncSetAttribute(lu_solve_x_kernel<8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(LU_TILE_SMEM_MAX)));
    attr = true;
  }
  const unsigned grid = unsigned(map.size());
  if (global) lu_solve_x_kernel<8, true><<<grid, 256, 0, s>>>(dd, dm, scratch, per);
  else if (tw == 32) lu_solve_x_kernel<32, false><<<grid, 256, smem, s>>>(dd, dm, scratch, per);
  else if (tw == 16) lu_solve_x_kernel<16, false><<<grid, 256, smem, s>>>(dd, dm, scratch, per);
  else lu_solve_x_kernel<8, false><<<grid, 256, smem, s>>>(dd, dm, scratch, per);
  CK_LAUNCH();
}

}  // namespace ifmm
