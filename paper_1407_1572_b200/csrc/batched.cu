// Batched block copies, grouped DGEMM launch, 1-norms and the blocked
// Gauss-Jordan inverse (Quintana-Orti et al. GJE formulation: an m x b panel is
// transformed in shared memory, the rest of the matrix is updated with six
// rank-b DMMA GEMMs per panel, row swaps are undone as column swaps at the end).
#include <algorithm>

#include "batched.cuh"

namespace ifmm {

// ------------------------------------------------------------------ copies
__global__ void __launch_bounds__(256) copy_kernel(const CopyDesc* __restrict__ desc) {
  __shared__ double tile[32][33];
  const CopyDesc D = desc[blockIdx.x];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  if (!D.trans || D.src == nullptr) {
    // four independent elements per lane in flight: loads first, then stores
    // (a load behind an unrelated store would wait for it)
    for (int j = ty; j < D.cols; j += 8) {
      double* dcol = D.dst + (size_t)j * D.ldd;
      const double* scol = D.src ? D.src + (size_t)j * D.lds : nullptr;
      for (int i0 = tx; i0 < D.rows; i0 += 128) {
        double v[4], o[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const int i = i0 + 32 * u;
          v[u] = (scol && i < D.rows) ? scol[i] : 0.0;
          o[u] = (D.accumulate && i < D.rows) ? dcol[i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const int i = i0 + 32 * u;
          if (i < D.rows) dcol[i] = o[u] + D.alpha * v[u];
        }
      }
    }
    return;
  }
  // transposed: dst(i,j) = src(j,i); go through 32x32 smem tiles
  for (int j0 = 0; j0 < D.cols; j0 += 32)
    for (int i0 = 0; i0 < D.rows; i0 += 32) {
      // src(j,i): column i of src, rows j -> coalesced along j
      for (int r = ty; r < 32; r += 8) {
        int i = i0 + r, j = j0 + tx;
        tile[r][tx] = (i < D.rows && j < D.cols) ? D.src[j + (size_t)i * D.lds] : 0.0;
      }
      __syncthreads();
      for (int r = ty; r < 32; r += 8) {
        int j = j0 + r, i = i0 + tx;
        if (i < D.rows && j < D.cols) {
          double v = D.alpha * tile[tx][r];
          double* d = D.dst + i + (size_t)j * D.ldd;
          if (D.accumulate) *d += v; else *d = v;
        }
      }
      __syncthreads();
    }
}

void launch_copies(CopyBatch& b, Arena& ws, Staging& st, cudaStream_t s) {
  if (b.d.empty()) return;
  // one CTA per descriptor: split large blocks into column chunks (<= 16K
  // elements, multiples of 32 columns) so big gathers spread over the GPU
  constexpr long long kChunk = 16384;
  bool split = false;
  for (const CopyDesc& D : b.d) split |= (long long)D.rows * D.cols > kChunk;
  if (split) {
    std::vector<CopyDesc> out;
    out.reserve(b.d.size());
    for (const CopyDesc& D : b.d) {
      if ((long long)D.rows * D.cols <= kChunk) {
        out.push_back(D);
        continue;
      }
      int cw = int(std::max<long long>(32, kChunk / std::max(1, D.rows) / 32 * 32));
      for (int j0 = 0; j0 < D.cols; j0 += cw) {
        CopyDesc C = D;
        C.cols = std::min(cw, D.cols - j0);
        C.dst = D.dst + (size_t)j0 * D.ldd;
        if (D.src) C.src = D.trans ? D.src + j0 : D.src + (size_t)j0 * D.lds;
        out.push_back(C);
      }
    }
    b.d.swap(out);
  }
  const CopyDesc* dd = upload(ws, b.d, s, st);
  size_t n = b.d.size();
  for (size_t off = 0; off < n; off += 2147483647u) {
    unsigned g = unsigned(std::min<size_t>(n - off, 2147483647u));
    copy_kernel<<<g, 256, 0, s>>>(dd + off);
    CK_LAUNCH();
  }
  b.clear();
}

// ------------------------------------------------------------------ positions
__global__ void pos_expand_kernel(const PosRun* __restrict__ runs, int n, int* pos) {
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += gridDim.x * (blockDim.x >> 5)) {
    const PosRun R = runs[r];
    for (int u = threadIdx.x & 31; u < R.dim; u += 32) pos[R.out + u] = int(R.base + u);
  }
}
void launch_pos_expand(const PosRun* d_runs, int n, int* pos, cudaStream_t s) {
  if (n <= 0) return;
  pos_expand_kernel<<<std::min(148 * 8, (n + 7) / 8), 256, 0, s>>>(d_runs, n, pos);
  CK_LAUNCH();
}

// ------------------------------------------------------------------ gemm launch
void launch_grouped_gemm(GemmBatch& b, bool transA, bool transB, Arena& ws, Staging& st, cudaStream_t s) {
  if (b.probs.empty()) return;
  const GemmProb* dp = upload(ws, b.probs, s, st);
  int np = int(b.probs.size());
  static const bool v1 = getenv("IFMM_GEMM_V1") != nullptr;  // debug: register-staged kernel
  if (v1) {
    if (!transA && !transB) grouped_dgemm_kernel<false, false><<<b.tiles, GTHREADS, 0, s>>>(dp, np);
    else if (transA && !transB) grouped_dgemm_kernel<true, false><<<b.tiles, GTHREADS, 0, s>>>(dp, np);
    else if (!transA && transB) grouped_dgemm_kernel<false, true><<<b.tiles, GTHREADS, 0, s>>>(dp, np);
    else grouped_dgemm_kernel<true, true><<<b.tiles, GTHREADS, 0, s>>>(dp, np);
    CK_LAUNCH();
    b.clear();
    return;
  }
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(grouped_dgemm_v2_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(GSMEM)));
    CK(cudaFuncSetAttribute(grouped_dgemm_v2_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(GSMEM)));
    CK(cudaFuncSetAttribute(grouped_dgemm_v2_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(GSMEM)));
    CK(cudaFuncSetAttribute(grouped_dgemm_v2_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(GSMEM)));
    attr = true;
  }
  const int* dtp = upload(ws, b.tile_prob, s, st);
  if (!transA && !transB) grouped_dgemm_v2_kernel<false, false><<<b.tiles, GTHREADS, GSMEM, s>>>(dp, dtp);
  else if (transA && !transB) grouped_dgemm_v2_kernel<true, false><<<b.tiles, GTHREADS, GSMEM, s>>>(dp, dtp);
  else if (!transA && transB) grouped_dgemm_v2_kernel<false, true><<<b.tiles, GTHREADS, GSMEM, s>>>(dp, dtp);
  else grouped_dgemm_v2_kernel<true, true><<<b.tiles, GTHREADS, GSMEM, s>>>(dp, dtp);
  CK_LAUNCH();
  b.clear();
}

// Concatenated Schur update kernel (see gemm.cuh, SchurBatch)
__device__ __forceinline__ int tri_index(int a, int b, int ns) { return a * ns - (a * (a - 1)) / 2 + (b - a); }

__global__ void __launch_bounds__(GTHREADS, 3)
    schur_concat_kernel(const SchurPiv* __restrict__ pivs, const int2* __restrict__ tiles,
                        const int* __restrict__ soff_pool, const SchurTgt* __restrict__ tab_pool) {
  extern __shared__ double gsm[];
  __shared__ int rslot[GBM], roff[GBM], cslot[GBN], coff[GBN];
  const int2 tt = tiles[blockIdx.x];
  const SchurPiv P = pivs[tt.x];
  const int i0 = (tt.y >> 16) * GBM, j0 = (tt.y & 0xffff) * GBN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // slot offsets staged in shared memory (one coalesced load) so the
  // per-thread binary searches below do not chain global-memory latencies
  __shared__ int s_soff[129];
  const int* soff = soff_pool + P.soff0;
  const bool stage = P.ns < 128;
  if (stage)
    for (int a = tid; a <= P.ns; a += GTHREADS) s_soff[a] = soff[a];
  __syncthreads();
  const int* so = stage ? s_soff : soff;
  {  // slot and in-slot offset of the tile's rows (threads 0..63) and columns (64..127)
    const int e = tid & 63;
    const int g = (tid < 64 ? i0 : j0) + e;
    int lo = 0, hi = P.ns - 1;  // largest a with soff[a] <= g
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (so[mid] <= g) lo = mid; else hi = mid - 1;
    }
    if (tid < 64) { rslot[e] = lo; roff[e] = g - so[lo]; }
    else { cslot[e] = lo; coff[e] = g - so[lo]; }
  }
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
  auto Asm = [&](int st) { return gsm + (size_t)st * 2 * GTILE_D; };
  auto Bsm = [&](int st) { return gsm + (size_t)st * 2 * GTILE_D + GTILE_D; };
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; a++)
#pragma unroll
    for (int b = 0; b < 4; b++) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int nk = (P.n + GBK - 1) / GBK;
#pragma unroll
  for (int st = 0; st < GSTAGES - 1; st++) {
    if (st < nk) {
      load_operand<true>(Asm(st), P.C, P.n, P.wr, P.n, i0, st * GBK, tid);
      load_operand<true>(Bsm(st), P.X, P.n, P.w, P.n, j0, st * GBK, tid);
    }
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; kt++) {
    cp_async_wait<GSTAGES - 2>();
    __syncthreads();
    {
      const int nt = kt + GSTAGES - 1;
      if (nt < nk) {
        const int st = nt % GSTAGES;
        load_operand<true>(Asm(st), P.C, P.n, P.wr, P.n, i0, nt * GBK, tid);
        load_operand<true>(Bsm(st), P.X, P.n, P.w, P.n, j0, nt * GBK, tid);
      }
      cp_async_commit();
    }
    const double* As = Asm(kt % GSTAGES);
    const double* Bs = Bsm(kt % GSTAGES);
#pragma unroll
    for (int kk = 0; kk < GBK; kk += 4) {
      double fa[4], fb[4];
#pragma unroll
      for (int m = 0; m < 4; m++) fa[m] = frag<true>(As, wm + m * 8 + (lane >> 2), kk + (lane & 3));
#pragma unroll
      for (int n = 0; n < 4; n++) fb[n] = frag<true>(Bs, wn + n * 8 + (lane >> 2), kk + (lane & 3));
#pragma unroll
      for (int m = 0; m < 4; m++)
#pragma unroll
        for (int n = 0; n < 4; n++)
          asm volatile(
              "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
              : "+d"(acc[m][n][0]), "+d"(acc[m][n][1])
              : "d"(fa[m]), "d"(fb[n]));
    }
  }
  cp_async_wait<0>();
  __syncthreads();  // rslot/cslot (written before the main loop) visible
  const SchurTgt* tab = tab_pool + P.tab0;
  // per row group: resolve the 8 target addresses and issue their loads
  // together, then the stores (a load behind an unrelated store would wait
  // for it: the compiler cannot prove the targets distinct)
#pragma unroll
  for (int m = 0; m < 4; m++) {
    const int li = wm + m * 8 + (lane >> 2);
    const bool rok = i0 + li < P.wr;
    const int a = rslot[li], ia = roff[li];
    double* ptr[8];
    double old[8];
#pragma unroll
    for (int e = 0; e < 8; e++) {
      const int lj = wn + (e >> 1) * 8 + 2 * (lane & 3) + (e & 1);
      const int b = cslot[lj];
      ptr[e] = nullptr;
      if (rok && j0 + lj < P.w && a <= b) {
        const SchurTgt T = tab[tri_index(a, b, P.ns)];
        const int jb = coff[lj];
        ptr[e] = T.trans ? T.p + jb + (size_t)ia * T.ld : T.p + ia + (size_t)jb * T.ld;
      }
    }
#pragma unroll
    for (int e = 0; e < 8; e++) old[e] = ptr[e] ? *ptr[e] : 0.0;
#pragma unroll
    for (int e = 0; e < 8; e++)
      if (ptr[e]) *ptr[e] = old[e] - acc[m][e >> 1][e & 1];
  }
}

void launch_schur(SchurBatch& b, Arena& ws, Staging& st, cudaStream_t s) {
  if (b.tiles.empty()) {
    b.clear();
    return;
  }
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(schur_concat_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(GSMEM)));
    attr = true;
  }
  const SchurPiv* dp = upload(ws, b.pivs, s, st);
  const int2* dt = upload(ws, b.tiles, s, st);
  const int* dso = upload(ws, b.soff, s, st);
  const SchurTgt* dtab = upload(ws, b.tab, s, st);
  for (size_t off = 0; off < b.tiles.size(); off += 2147483647u) {
    const unsigned g = unsigned(std::min<size_t>(b.tiles.size() - off, 2147483647u));
    schur_concat_kernel<<<g, GTHREADS, GSMEM, s>>>(dp, dt + off, dso, dtab);
    CK_LAUNCH();
  }
  b.clear();
}

// ------------------------------------------------------------------ norms
// 1-norm (max column abs sum) of every matrix: grid (matrix, 64-column chunk);
// chunk maxima merge with an integer atomicMax on the bit patterns, which
// orders non-negative doubles exactly (and lets a NaN column win)
__global__ void __launch_bounds__(256) norm1_kernel(const MatDesc* __restrict__ desc, double* out) {
  const MatDesc D = desc[blockIdx.x];
  const int c0 = blockIdx.y * 64;
  if (c0 >= D.m) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double best = 0.0;
  for (int c = c0 + wid; c < min(D.m, c0 + 64); c += 8) {
    double s = 0.0;
    for (int r = lane; r < D.m; r += 32) s += fabs(D.A[r + (size_t)c * D.lda]);
    s = warp_sum(s);
    best = (s != s || best != best) ? __longlong_as_double(0x7ff8000000000000ll) : fmax(best, s);
  }
  if (lane == 0)
    atomicMax(reinterpret_cast<unsigned long long*>(out + blockIdx.x),
              static_cast<unsigned long long>(__double_as_longlong(best)));
}


void launch_norm1(const MatDesc* d_desc, int n, int maxm, double* out, cudaStream_t s) {
  if (n <= 0) return;
  CK(cudaMemsetAsync(out, 0, sizeof(double) * n, s));
  norm1_kernel<<<dim3(n, std::max(1, (maxm + 63) / 64)), 256, 0, s>>>(d_desc, out);
  CK_LAUNCH();
}

// ------------------------------------------------------------------ 1-norm estimate
// Hager/Higham estimate of ||B||_1 (LAPACK dlacn2, the estimator dgecon uses,
// ifmm/solver.py:216) applied to the explicit inverse B = S^-1: the reference's
// rcond test sees this estimate (<= the exact norm), so the GPU raises
// SingularPivotError under the same criterion.
__device__ inline void gemv_n(const MatDesc& D, const double* x, double* y) {  // y = B x
  for (int i = threadIdx.x; i < D.m; i += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < D.m; j++) s = fma(D.A[i + (size_t)j * D.lda], x[j], s);
    y[i] = s;
  }
  __syncthreads();
}
__device__ inline void gemv_t(const MatDesc& D, const double* x, double* y) {  // y = B^T x
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = warp; j < D.m; j += nw) {
    const double* c = D.A + (size_t)j * D.lda;
    double s = 0.0;
    for (int i = lane; i < D.m; i += 32) s = fma(c[i], x[i], s);
    s = warp_sum(s);
    if (lane == 0) y[j] = s;
  }
  __syncthreads();
}
__device__ inline double asum(const double* v, int n, double* red) {
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += fabs(v[i]);
  return block_sum(s, red);
}
__device__ inline int iamax(const double* v, int n, ArgMax* red) {
  ArgMax a{-1.0, -1};
  for (int i = threadIdx.x; i < n; i += blockDim.x) a = argmax_merge(a, ArgMax{fabs(v[i]), i});
  return block_argmax(a, red).i;
}

__global__ void __launch_bounds__(256) norm1_est_kernel(const MatDesc* __restrict__ desc, double* out,
                                                        const double* __restrict__ normA, double limit) {
  extern __shared__ double sm[];
  __shared__ double red[32];
  __shared__ ArgMax ared[32];
  __shared__ int s_flag;
  const MatDesc D = desc[blockIdx.x];
  const int n = D.m;
  // out holds the exact ||B||_1 on entry; the estimate never exceeds it, so a
  // pivot that passes with the exact norm passes with the estimate too
  if (out[blockIdx.x] * normA[blockIdx.x] < limit) return;
  double* x = sm;
  double* y = x + n;
  double* sgn = y + n;
  if (n == 0) {
    if (threadIdx.x == 0) out[blockIdx.x] = 0.0;
    return;
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = 1.0 / n;
  __syncthreads();
  gemv_n(D, x, y);
  double est = asum(y, n, red);
  if (n == 1) {
    if (threadIdx.x == 0) out[blockIdx.x] = est;
    return;
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) sgn[i] = y[i] >= 0.0 ? 1.0 : -1.0;
  __syncthreads();
  gemv_t(D, sgn, x);
  int j = iamax(x, n, ared);
  for (int iter = 2;; iter++) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = (i == j) ? 1.0 : 0.0;
    __syncthreads();
    gemv_n(D, x, y);
    const double old = est;
    est = asum(y, n, red);
    if (threadIdx.x == 0) s_flag = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x)
      if ((y[i] >= 0.0 ? 1.0 : -1.0) != sgn[i]) s_flag = 1;
    __syncthreads();
    if (!s_flag || est <= old) break;  // repeated sign vector or no increase
    for (int i = threadIdx.x; i < n; i += blockDim.x) sgn[i] = y[i] >= 0.0 ? 1.0 : -1.0;
    __syncthreads();
    gemv_t(D, sgn, x);
    const int jlast = j;
    j = iamax(x, n, ared);
    if (!(x[jlast] != fabs(x[j]) && iter < 5)) break;
  }
  // alternating-sign test vector
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    x[i] = ((i & 1) ? -1.0 : 1.0) * (1.0 + double(i) / double(n - 1));
  __syncthreads();
  gemv_n(D, x, y);
  const double temp = 2.0 * asum(y, n, red) / (3.0 * n);
  if (threadIdx.x == 0) out[blockIdx.x] = temp > est ? temp : est;
}

void launch_norm1_estimate(const MatDesc* d_desc, int n, int maxm, double* out, const double* normA, double limit,
                           cudaStream_t s) {
  if (n <= 0) return;
  const size_t smem = sizeof(double) * 3 * size_t(std::max(1, maxm));
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(norm1_est_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  norm1_est_kernel<<<n, 256, smem, s>>>(d_desc, out, normA, limit);
  CK_LAUNCH();
}

// ------------------------------------------------------------------ Gauss-Jordan
// Panel transform: columns [j, j+b) of every matrix with m > j.
// Rows of the panel live in shared memory in their panel-start order; pivoting
// is tracked as a position <-> row map (no physical swaps), so a column step
// costs three barriers: candidate argmax, pivot-row preparation, elimination.
// Outputs: the transformed panel in final row order, ipiv (LAPACK sequential
// swap semantics, used for the final column unswap), and the list of row
// moves new[dst] = old[src] (at most 2b) that the other columns must apply.
struct RowMove {
  int dst, src;
};

__global__ void __launch_bounds__(512) gj_panel_kernel(const MatDesc* __restrict__ desc, int j, int b, int* info,
                                                       RowMove* moves, int* nmoves) {
  extern __shared__ double sm[];
  __shared__ double candv[32];
  __shared__ int candr[32], candp[32];
  __shared__ double prow[64];
  __shared__ int s_cnt;
  const MatDesc D = desc[blockIdx.x];
  const int m = D.m;
  if (m <= j) return;
  const int bb = min(b, m - j);
  const int ld = bb + 1;  // odd row stride: conflict-free per-row access
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  double* P = sm;                                   // P[r*ld + c] = A(r, j+c), r = panel-start row
  int* pos = reinterpret_cast<int*>(P + (size_t)m * ld);  // row -> current position
  int* at = pos + m;                                // position -> row
  // load: every thread issues all bb loads of its rows back to back
  for (int r = tid; r < m; r += nt) {
    const double* src = D.A + r;
#pragma unroll 8
    for (int c = 0; c < bb; c++) P[r * ld + c] = src[(size_t)(j + c) * D.lda];
    pos[r] = r;
    at[r] = r;
  }
  if (tid == 0) s_cnt = 0;
  __syncthreads();
  for (int c = 0; c < bb; c++) {
    const int jc = j + c;
    // (1) candidates among rows not yet used as pivots (position >= jc);
    // ties -> smallest position (idamax on the swapped order)
    double bv = -1.0;
    int br = -1, bp = 0x7fffffff;
    for (int r = tid; r < m; r += nt) {
      const int pr = pos[r];
      if (pr < jc) continue;
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
    // (2) every warp reduces the warp candidates with shuffles (no extra barrier)
    bv = lane < nw ? candv[lane] : -1.0;
    br = lane < nw ? candr[lane] : -1;
    bp = lane < nw ? candp[lane] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int orr = __shfl_xor_sync(0xffffffffu, br, o), op = __shfl_xor_sync(0xffffffffu, bp, o);
      if (ov > bv || (ov == bv && op < bp)) { bv = ov; br = orr; bp = op; }
    }
    if (warp == 0) {  // pivot row: scaled copy in prow (prow[c] = 1/pivot), broadcast after the barrier
      const double pv = br >= 0 ? P[br * ld + c] : 0.0;
      const bool sing = (pv == 0.0 || pv != pv);
      const double inv = sing ? 0.0 : 1.0 / pv;
      __syncwarp();
      for (int cc = lane; cc < bb; cc += 32) {
        const double v = (cc == c) ? inv : P[br * ld + cc] * inv;
        prow[cc] = v;
        P[br * ld + cc] = v;
      }
      if (lane == 0) {
        if (sing && info[blockIdx.x] == 0) info[blockIdx.x] = jc + 1;
        D.ipiv[jc] = bp;  // swap positions jc <-> bp
        const int q = at[jc];
        at[bp] = q;
        pos[q] = bp;
        at[jc] = br;
        pos[br] = jc;
      }
    }
    __syncthreads();
    const double inv = prow[c];
    // (3) eliminate column c from every other row
    for (int r = tid; r < m; r += nt) {
      if (r == br) continue;
      double* row = P + r * ld;
      const double f = row[c];
      if (f != 0.0) {
#pragma unroll 4
        for (int cc = 0; cc < bb; cc++) row[cc] -= f * prow[cc];
      }
      row[c] = -f * inv;
    }
    __syncthreads();
  }
  // write back in final order; record the row moves (positions >= j only)
  for (int l = tid; l < m; l += nt) {
    const int r = at[l];
    double* dst = D.A + l;
#pragma unroll 8
    for (int c = 0; c < bb; c++) dst[(size_t)(j + c) * D.lda] = P[r * ld + c];
    if (r != l) {
      const int k = atomicAdd(&s_cnt, 1);
      moves[(size_t)blockIdx.x * 2 * b + k] = RowMove{l, r};
    }
  }
  __syncthreads();
  if (tid == 0) nmoves[blockIdx.x] = s_cnt;
}

// Register-resident variant: thread t owns panel rows t, t+nt (R rows, B
// columns in registers).  Per column: local candidate -> warp shuffle ->
// barrier -> owner publishes the scaled pivot row -> barrier -> register
// elimination (no barrier: every thread reads only its own rows next).
// Ties are broken by row index; thread 0 keeps the position bookkeeping.
template <int B, int R>
__global__ void __launch_bounds__(R == 1 ? (B <= 16 ? 1024 : 512) : (R == 2 ? 384 : 256)) gj_panel_reg_kernel(
    const MatDesc* __restrict__ desc, int j, int* info, RowMove* moves, int* nmoves) {
  extern __shared__ int smi[];
  __shared__ double candv[32];
  __shared__ int candr[32];
  __shared__ __align__(16) double prow[B];
  __shared__ int s_cnt;
  const MatDesc D = desc[blockIdx.x];
  const int m = D.m;
  if (m <= j) return;
  const int bb = min(B, m - j);
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  int* pos = smi;     // row -> position
  int* at = pos + m;  // position -> row
  double v[R][B];
  bool used[R];
#pragma unroll
  for (int k = 0; k < R; k++) {
    const int r = tid + k * nt;
    used[k] = !(r < m) || r < j;  // rows above the panel are already pivot rows
#pragma unroll
    for (int c = 0; c < B; c++) v[k][c] = (r < m && c < bb) ? D.A[r + (size_t)(j + c) * D.lda] : 0.0;
  }
  for (int r = tid; r < m; r += nt) {
    pos[r] = r;
    at[r] = r;
  }
  if (tid == 0) s_cnt = 0;
  __syncthreads();
#pragma unroll
  for (int c = 0; c < B; c++) {
    if (c >= bb) break;
    const int jc = j + c;
    double bv = -1.0;
    int br = 0x7fffffff;
#pragma unroll
    for (int k = 0; k < R; k++) {
      const double a = fabs(v[k][c]);
      if (!used[k] && (a > bv)) { bv = a; br = tid + k * nt; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int orr = __shfl_xor_sync(0xffffffffu, br, o);
      if (ov > bv || (ov == bv && orr < br)) { bv = ov; br = orr; }
    }
    if (lane == 0) { candv[warp] = bv; candr[warp] = br; }
    __syncthreads();
    // every warp reduces the nw candidates with shuffles (same result everywhere)
    bv = lane < nw ? candv[lane] : -1.0;
    br = lane < nw ? candr[lane] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int orr = __shfl_xor_sync(0xffffffffu, br, o);
      if (ov > bv || (ov == bv && orr < br)) { bv = ov; br = orr; }
    }
    if (br == 0x7fffffff) br = -1;
    // owner of the pivot row publishes it scaled; thread 0 does the bookkeeping
    const int kown = br >= 0 ? br / nt : -1;
    if (br >= 0 && br % nt == tid) {
#pragma unroll
      for (int k = 0; k < R; k++)
        if (k == kown) {
          const double pv = v[k][c];
          const bool sing = (pv == 0.0 || pv != pv);
          const double inv = sing ? 0.0 : 1.0 / pv;
          if (sing && info[blockIdx.x] == 0) info[blockIdx.x] = jc + 1;
#pragma unroll
          for (int cc = 0; cc < B; cc++) {
            const double s = (cc == c) ? inv : v[k][cc] * inv;
            prow[cc] = s;
            v[k][cc] = s;
          }
          used[k] = true;
        }
    }
    if (tid == 0) {
      if (br < 0) {  // no candidate left (cannot happen for m > jc): keep identity
        if (info[blockIdx.x] == 0) info[blockIdx.x] = jc + 1;
        D.ipiv[jc] = jc;
      } else {
        const int bp = pos[br];
        D.ipiv[jc] = bp;
        const int q = at[jc];
        at[bp] = q;
        pos[q] = bp;
        at[jc] = br;
        pos[br] = jc;
      }
    }
    __syncthreads();
    if (R == 1) {
      double pr[B];  // pivot row in registers, 16-byte broadcast reads
#pragma unroll
      for (int cc = 0; cc < B; cc += 2) {
        const double2 t2 = *reinterpret_cast<const double2*>(&prow[cc]);
        pr[cc] = t2.x;
        pr[cc + 1] = t2.y;
      }
      const double inv = pr[c];
      const int r = tid;
      if (r != br && r < m) {
        const double f = v[0][c];
#pragma unroll
        for (int cc = 0; cc < B; cc++)
          if (cc != c) v[0][cc] = fma(-f, pr[cc], v[0][cc]);
        v[0][c] = -f * inv;
      }
    } else {  // two rows per thread: no room for a register copy of the row
      const double inv = prow[c];
#pragma unroll
      for (int k = 0; k < R; k++) {
        const int r = tid + k * nt;
        if (r == br || r >= m) continue;
        const double f = v[k][c];
#pragma unroll
        for (int cc = 0; cc < B; cc++)
          if (cc != c) v[k][cc] = fma(-f, prow[cc], v[k][cc]);
        v[k][c] = -f * inv;
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < R; k++) {
    const int r = tid + k * nt;
    if (r >= m) continue;
    const int l = pos[r];
    double* dst = D.A + l;
#pragma unroll
    for (int c = 0; c < B; c++)
      if (c < bb) dst[(size_t)(j + c) * D.lda] = v[k][c];
    if (r != l) {
      const int q = atomicAdd(&s_cnt, 1);
      moves[(size_t)blockIdx.x * 2 * B + q] = RowMove{l, r};
    }
  }
  __syncthreads();
  if (tid == 0) nmoves[blockIdx.x] = s_cnt;
}

// Apply the panel's row moves to every column outside the panel and copy the
// pivot-row block W = A[j:j+bb, :] (after the moves).  One warp per column.
__global__ void __launch_bounds__(256) gj_move_copy_kernel(const MatDesc* __restrict__ desc, int j, int b,
                                                           const RowMove* __restrict__ moves,
                                                           const int* __restrict__ nmoves, double* const* W) {
  const MatDesc D = desc[blockIdx.x];
  if (D.m <= j) return;
  const int bb = min(b, D.m - j);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cnt = nmoves[blockIdx.x];
  const RowMove* mv = moves + (size_t)blockIdx.x * 2 * b;
  double* w = W[blockIdx.x];
  for (int col = warp + blockIdx.y * 8; col < D.m; col += 8 * gridDim.y) {
    if (col >= j && col < j + bb) continue;
    double* a = D.A + (size_t)col * D.lda;
    double v0 = 0.0, v1 = 0.0;
    RowMove m0{-1, -1}, m1{-1, -1};
    if (lane < cnt) { m0 = mv[lane]; v0 = a[m0.src]; }
    if (lane + 32 < cnt) { m1 = mv[lane + 32]; v1 = a[m1.src]; }
    __syncwarp();
    if (m0.dst >= 0) a[m0.dst] = v0;
    if (m1.dst >= 0) a[m1.dst] = v1;
    __syncwarp();
    for (int t = lane; t < bb; t += 32) w[t + (size_t)col * bb] = a[j + t];
  }
}

// Two-level variant of the row moves + W copy: columns [c_lo, c_hi) of every
// matrix (c relative to j0: c_lo = j0 + lo_off ... ), minus [x_lo, x_hi),
// get the row moves of list 1 then (if nl == 2) list 2 applied; W (wb x m,
// ld wb) receives rows [j0 + w_off, j0 + w_off + wb) of those columns.
// Offsets are relative to the outer panel start j0; widths are clipped per
// matrix (wb = min(wwant, m - j0 - w_off)).
__global__ void __launch_bounds__(256) gj_move_copy2_kernel(const MatDesc* __restrict__ desc, int j0, int c_lo_off,
                                                            int c_hi_off, int x_lo_off, int x_hi_off, int b,
                                                            const RowMove* __restrict__ mv1,
                                                            const int* __restrict__ nm1,
                                                            const RowMove* __restrict__ mv2,
                                                            const int* __restrict__ nm2, int w_off, int wwant,
                                                            double* const* W, int g1_off, int g2_off) {
  const MatDesc D = desc[blockIdx.x];
  if (D.m <= j0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // column range; negative offsets mean "from 0" / positive >= m mean "to m"
  const int c_lo = c_lo_off < 0 ? 0 : min(D.m, j0 + c_lo_off);
  const int c_hi = c_hi_off < 0 ? D.m : min(D.m, j0 + c_hi_off);
  const int x_lo = min(D.m, j0 + x_lo_off), x_hi = min(D.m, j0 + x_hi_off);
  const int wr0 = j0 + w_off;
  const int wb = max(0, min(wwant, D.m - wr0));
  // a list only exists for a matrix whose panel at j0 + g*_off exists (the
  // panel kernel leaves the move counts of smaller matrices untouched)
  const int c1 = (nm1 && D.m > j0 + g1_off) ? nm1[blockIdx.x] : 0;
  const int c2 = (nm2 && D.m > j0 + g2_off) ? nm2[blockIdx.x] : 0;
  const RowMove* l1 = mv1 ? mv1 + (size_t)blockIdx.x * 2 * b : nullptr;
  const RowMove* l2 = mv2 ? mv2 + (size_t)blockIdx.x * 2 * b : nullptr;
  double* w = W[blockIdx.x];
  for (int col = c_lo + warp + blockIdx.y * 8; col < c_hi; col += 8 * gridDim.y) {
    if (col >= x_lo && col < x_hi) continue;
    double* a = D.A + (size_t)col * D.lda;
#pragma unroll
    for (int li = 0; li < 2; li++) {
      const RowMove* mv = li == 0 ? l1 : l2;
      const int cnt = li == 0 ? c1 : c2;
      if (cnt == 0) continue;
      double v0 = 0.0, v1 = 0.0;
      RowMove m0{-1, -1}, m1{-1, -1};
      if (lane < cnt) { m0 = mv[lane]; v0 = a[m0.src]; }
      if (lane + 32 < cnt) { m1 = mv[lane + 32]; v1 = a[m1.src]; }
      __syncwarp();
      if (m0.dst >= 0) a[m0.dst] = v0;
      if (m1.dst >= 0) a[m1.dst] = v1;
      __syncwarp();
    }
    for (int t = lane; t < wb; t += 32) w[t + (size_t)col * wb] = a[wr0 + t];
  }
}

// Trailing update of one Gauss-Jordan panel step, all matrices of the batch in
// one launch, indexed on the device (no per-step host descriptors):
//   A[i, c] = [i not in R1] A[i, c] + sum_k A[i, j+k] W[k, c]   for c outside the panel
// (rows R1 = [j, j+bb) hold A11^-1 in the panel columns, so the same formula
// covers the overwrite A[R1, c] = A11^-1 W[:, c]).  64x64 DMMA tiles; the
// virtual column index skips the panel columns.
__global__ void __launch_bounds__(GTHREADS) gj_update_kernel(const MatDesc* __restrict__ desc,
                                                             const int* __restrict__ tile0, int np, int j, int b,
                                                             double* const* __restrict__ Wp) {
  __shared__ double As[2][GBK][GPAD];
  __shared__ double Bs[2][GBK][GPAD];
  int lo = 0, hi = np - 1;
  const int t = blockIdx.x;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (tile0[mid] <= t) lo = mid; else hi = mid - 1;
  }
  const MatDesc D = desc[lo];
  const int m = D.m;
  const int bb = min(b, m - j);
  const int ncol = m - bb;  // virtual columns
  const int tl = t - tile0[lo];
  const int tilesM = (m + GBM - 1) / GBM;
  const int i0 = (tl % tilesM) * GBM, v0 = (tl / tilesM) * GBN;
  const double* __restrict__ W = Wp[lo];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; a++)
#pragma unroll
    for (int c = 0; c < 4; c++) acc[a][c][0] = acc[a][c][1] = 0.0;
  double ra[8], rb[8];
  auto load = [&](int k0) {
#pragma unroll
    for (int e = 0; e < 8; e++) {
      const int idx = tid + e * GTHREADS;
      int i = idx & 63, k = idx >> 6;
      int gi = i0 + i, gk = k0 + k;
      ra[e] = (gi < m && gk < bb) ? D.A[gi + (size_t)(j + gk) * D.lda] : 0.0;
      k = idx & 15;
      const int vc = v0 + (idx >> 4);
      gk = k0 + k;
      const int col = vc < j ? vc : vc + bb;
      rb[e] = (vc < ncol && gk < bb) ? W[gk + (size_t)col * bb] : 0.0;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int e = 0; e < 8; e++) {
      const int idx = tid + e * GTHREADS;
      As[buf][idx >> 6][idx & 63] = ra[e];
      Bs[buf][idx & 15][idx >> 4] = rb[e];
    }
  };
  const int nk = (bb + GBK - 1) / GBK;
  load(0);
  store(0);
  __syncthreads();
  for (int kt = 0; kt < nk; kt++) {
    const int buf = kt & 1;
    if (kt + 1 < nk) load((kt + 1) * GBK);
#pragma unroll
    for (int kk = 0; kk < GBK; kk += 4) {
      double fa[4], fb[4];
#pragma unroll
      for (int q = 0; q < 4; q++) fa[q] = As[buf][kk + (lane & 3)][wm + q * 8 + (lane >> 2)];
#pragma unroll
      for (int q = 0; q < 4; q++) fb[q] = Bs[buf][kk + (lane & 3)][wn + q * 8 + (lane >> 2)];
#pragma unroll
      for (int x = 0; x < 4; x++)
#pragma unroll
        for (int y = 0; y < 4; y++)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(acc[x][y][0]), "+d"(acc[x][y][1])
                       : "d"(fa[x]), "d"(fb[y]));
    }
    if (kt + 1 < nk) {
      store(buf ^ 1);
      __syncthreads();
    }
  }
#pragma unroll
  for (int x = 0; x < 4; x++) {
    const int gi = i0 + wm + x * 8 + (lane >> 2);
    if (gi >= m) continue;
    const bool r1 = gi >= j && gi < j + bb;
#pragma unroll
    for (int y = 0; y < 4; y++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int vc = v0 + wn + y * 8 + 2 * (lane & 3) + h;
        if (vc >= ncol) continue;
        const int col = vc < j ? vc : vc + bb;
        double* c = D.A + gi + (size_t)col * D.lda;
        *c = r1 ? acc[x][y][h] : *c + acc[x][y][h];
      }
  }
}

// Undo the row pivoting of the inverted matrix: inv(A) = inv(PA) P, i.e. the
// column swaps of ipiv in reverse order -- composed into one column gather.
__global__ void gj_colperm_kernel(const MatDesc* __restrict__ desc, int* perm, int stride) {
  const MatDesc D = desc[blockIdx.x];
  if (threadIdx.x != 0) return;
  int* src = perm + (size_t)blockIdx.x * stride;
  for (int c = 0; c < D.m; c++) src[c] = c;
  for (int c = D.m - 1; c >= 0; c--) {
    const int p = D.ipiv[c];
    const int t = src[c];
    src[c] = src[p];
    src[p] = t;
  }
}

__global__ void __launch_bounds__(256) gj_colgather_kernel(const MatDesc* __restrict__ desc, const int* perm,
                                                           int stride, double* const* T, int back) {
  const MatDesc D = desc[blockIdx.x];
  const int* src = perm + (size_t)blockIdx.x * stride;
  double* t = T[blockIdx.x];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int col = warp + blockIdx.y * 8; col < D.m; col += 8 * gridDim.y) {
    if (!back) {
      const double* a = D.A + (size_t)src[col] * D.lda;
      double* o = t + (size_t)col * D.m;
      for (int r = lane; r < D.m; r += 32) o[r] = a[r];
    } else {
      const double* a = t + (size_t)col * D.m;
      double* o = D.A + (size_t)col * D.lda;
      for (int r = lane; r < D.m; r += 32) o[r] = a[r];
    }
  }
}

// v2 trailing update (see gemm.cuh for the cp.async operand layouts): grid
// (matrix, tile); the rank-b update A(:, v) += P W(:, v) over the virtual
// columns v (all but the panel), P = A(:, j:j+b) i-contiguous, W k-contiguous.
// Rows of the pivot block are overwritten (beta = 0), the others accumulated.
// mode 0: all columns but the panel; 1: only the next panel's columns (the
// look-ahead part); 2: all but the panel and the next panel; 4: only the
// previous panel's columns [j - b, j) (two-level scheme).  Column u of the
// mode's range maps to matrix column colmap(u).
__device__ __forceinline__ int gj_cols(int mode, int j, int bb, int b2, int m) {
  return mode == 0 ? m - bb : (mode == 1 ? b2 : m - bb - b2);
}
__device__ __forceinline__ int gj_colmap(int mode, int u, int j, int bb, int b2) {
  if (mode == 1) return j + bb + u;
  if (u < j) return u;
  return u + bb + (mode == 2 ? b2 : 0);
}

__global__ void __launch_bounds__(GTHREADS, 3) gj_update_v2_kernel(const MatDesc* __restrict__ desc, int j, int b,
                                                                   double* const* __restrict__ Wp, int mode) {
  extern __shared__ double gsm[];
  const MatDesc D = desc[blockIdx.x];
  const int m = D.m;
  if (m <= j) return;
  const int bb = min(b, m - j);
  const int b2 = min(b, m - j - bb);  // width of the next panel
  // mode 4: the previous inner panel's columns [j - b, j)
  const int ncol = mode == 4 ? min(b, j) : gj_cols(mode, j, bb, b2, m);
  if (ncol <= 0) return;
  const int tilesM = (m + GBM - 1) / GBM;
  const int tl = blockIdx.y;
  if (tl >= tilesM * ((ncol + GBN - 1) / GBN)) return;
  const int i0 = (tl % tilesM) * GBM, v0 = (tl / tilesM) * GBN;
  const double* __restrict__ W = Wp[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
  auto Asm = [&](int st) { return gsm + (size_t)st * 2 * GTILE_D; };
  auto Bsm = [&](int st) { return gsm + (size_t)st * 2 * GTILE_D + GTILE_D; };
  const double* Pan = D.A + (size_t)j * D.lda;
  auto load_w = [&](double* sm, int k0) {
#pragma unroll
    for (int e = 0; e < (GBN * GBK) / GTHREADS; e++) {
      const int c = tid + e * GTHREADS;
      const int k = c & (GBK - 1), r = c / GBK;
      const int vc = v0 + r, gk = k0 + k;
      const int col = mode == 4 ? j - min(b, j) + vc : gj_colmap(mode, vc, j, bb, b2);
      const bool ok = vc < ncol && gk < bb;
      cp_async8(sm + r * KP + k, W + gk + (size_t)col * bb, ok);
    }
  };
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; a++)
#pragma unroll
    for (int c = 0; c < 4; c++) acc[a][c][0] = acc[a][c][1] = 0.0;
  const int nk = (bb + GBK - 1) / GBK;
#pragma unroll
  for (int st = 0; st < GSTAGES - 1; st++) {
    if (st < nk) {
      load_operand<false>(Asm(st), Pan, D.lda, m, bb, i0, st * GBK, tid);
      load_w(Bsm(st), st * GBK);
    }
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; kt++) {
    cp_async_wait<GSTAGES - 2>();
    __syncthreads();
    {
      const int nt = kt + GSTAGES - 1;
      if (nt < nk) {
        const int st = nt % GSTAGES;
        load_operand<false>(Asm(st), Pan, D.lda, m, bb, i0, nt * GBK, tid);
        load_w(Bsm(st), nt * GBK);
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
    const bool r1 = gi >= j && gi < j + bb;
    double* ptr[8];
    double old[8];
#pragma unroll
    for (int e = 0; e < 8; e++) {
      const int vc = v0 + wn + (e >> 1) * 8 + 2 * (lane & 3) + (e & 1);
      const int col = mode == 4 ? j - min(b, j) + vc : gj_colmap(mode, vc, j, bb, b2);
      ptr[e] = (gi < m && vc < ncol) ? D.A + gi + (size_t)col * D.lda : nullptr;
    }
#pragma unroll
    for (int e = 0; e < 8; e++) old[e] = (ptr[e] && !r1) ? *ptr[e] : 0.0;
#pragma unroll
    for (int e = 0; e < 8; e++)
      if (ptr[e]) *ptr[e] = old[e] + acc[x][e >> 1][e & 1];
  }
}

void batched_gj_inverse(const std::vector<MatDesc>& h, const MatDesc* d_desc, int* d_info, Arena& ws,
                        Staging& st, cudaStream_t s, const GjSide* side, int shape_n, int shape_maxm) {
  const int n = int(h.size());
  if (n == 0) return;
  int maxm = shape_maxm;
  for (auto& d : h) maxm = std::max(maxm, d.m);
  // panel variant: registers (one or two rows per thread) up to m = 1024,
  // shared memory beyond (the top-level system)
  int variant, b, threads;
  size_t smem;
  static const int reg1_max = getenv("IFMM_GJ_R1_MAX") ? atoi(getenv("IFMM_GJ_R1_MAX")) : 512;  // tuning
  if (maxm <= reg1_max) {
    variant = 0;
    b = 32;
    threads = std::max(64, (maxm + 31) / 32 * 32);
    smem = size_t(maxm) * 8;
  } else if (maxm <= 768) {
    variant = 1;
    b = 32;
    threads = ((maxm + 1) / 2 + 31) / 32 * 32;
    smem = size_t(maxm) * 8;
  } else if (maxm <= 1024 && !getenv("IFMM_GJ_SMEM_PANEL")) {
    // one row per thread in registers, 16-wide panels (the shared-memory
    // panel rewrites m x b entries per pivot step)
    variant = 4;
    b = 16;
    threads = (maxm + 31) / 32 * 32;
    smem = size_t(maxm) * 8;
  } else {
    variant = 2;
    auto smem_for = [&](int bw) { return size_t(maxm) * (bw + 1) * 8 + size_t(maxm) * 8; };
    // narrow panels: the shared-memory panel rewrites m x b entries per pivot
    // step, so its traffic grows with b (the wider update is cheap here)
    static const int bsm = getenv("IFMM_GJ_SMEM_B") ? atoi(getenv("IFMM_GJ_SMEM_B")) : 16;
    b = bsm;
    while (b > 1 && smem_for(b) > 224 * 1024) b /= 2;  // very large pivots (3-D top levels): narrower panels
    if (smem_for(b) > 224 * 1024) invalid("pivot block too large for the Gauss-Jordan panel");
    smem = smem_for(b);
    threads = 512;
  }
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(gj_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 * 1024));
    CK(cudaFuncSetAttribute(gj_update_v2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(GSMEM)));
    attr = true;
  }
  CK(cudaMemsetAsync(d_info, 0, sizeof(int) * n, s));
  // pivot-row block W (b x m per matrix), row moves, column-unswap scratch
  std::vector<double*> W(n);
  for (int p = 0; p < n; p++) W[p] = ws.alloc_n<double>(size_t(b) * h[p].m);
  double* const* dW = upload(ws, W, s, st);
  RowMove* moves = static_cast<RowMove*>(ws.alloc(sizeof(RowMove) * size_t(n) * 2 * b));
  int* nmoves = ws.alloc_n<int>(n);
  std::vector<int> tile_pref[2];
  const int gy = std::max(1, std::min(16, (maxm + 63) / 64));
  auto panel = [&](int j, cudaStream_t ps) {
    if (variant == 0) gj_panel_reg_kernel<32, 1><<<n, threads, smem, ps>>>(d_desc, j, d_info, moves, nmoves);
    else if (variant == 4) gj_panel_reg_kernel<16, 1><<<n, threads, smem, ps>>>(d_desc, j, d_info, moves, nmoves);
    else if (variant == 1) gj_panel_reg_kernel<32, 2><<<n, threads, smem, ps>>>(d_desc, j, d_info, moves, nmoves);
    else gj_panel_kernel<<<n, threads, smem, ps>>>(d_desc, j, b, d_info, moves, nmoves);
    CK_LAUNCH();
  };
  // tiles of the largest matrix for an update mode at step j
  auto max_tiles = [&](int j, int mode) {
    int mt = 0;
    for (int p = 0; p < n; p++) {
      const int m = h[p].m;
      if (m <= j) continue;
      const int bb = std::min(b, m - j), b2 = std::min(b, m - j - bb);
      const int nc = mode == 0 ? m - bb : (mode == 1 ? b2 : m - bb - b2);
      if (nc > 0) mt = std::max(mt, ceil_div(m, GBM) * ceil_div(nc, GBN));
    }
    return mt;
  };
  auto update = [&](int j, int mode) {
    const int mt = max_tiles(j, mode);
    if (mt > 0) {
      gj_update_v2_kernel<<<dim3(n, mt), GTHREADS, GSMEM, s>>>(d_desc, j, b, dW, mode);
      CK_LAUNCH();
    }
  };
  static const bool v1 = getenv("IFMM_GJ_UPDATE_V1") != nullptr;  // debug: register-staged update
  static const bool no_la = getenv("IFMM_GJ_NO_LOOKAHEAD") != nullptr;  // debug: serial panel/update
  static const bool one_level = getenv("IFMM_GJ_ONE_LEVEL") != nullptr;  // debug: rank-b updates only
  const bool look = side && side->s && !v1 && !no_la;
  // two-level for large batches (bandwidth-bound updates); few large matrices
  // are panel-latency-bound and keep the one-level look-ahead (measured)
  if (!v1 && !one_level && variant != 2 && std::max(n, shape_n) >= 64) {
    // Two-level blocking: an outer panel of 2b columns is processed as two
    // inner panels (each inner step updates only the other inner panel), then
    // the rest of the matrix gets ONE rank-2b update with the processed outer
    // panel and the original pivot rows (blocked Gauss-Jordan: the composed
    // transform is x + (P - E) x_piv).  Half the trailing-update traffic.
    const int B2 = 2 * b;
    RowMove* moves2 = static_cast<RowMove*>(ws.alloc(sizeof(RowMove) * size_t(n) * 2 * b));
    int* nmoves2 = ws.alloc_n<int>(n);
    std::vector<double*> Wo(n);
    for (int p = 0; p < n; p++) Wo[p] = ws.alloc_n<double>(size_t(B2) * h[p].m);
    double* const* dWo = upload(ws, Wo, s, st);
    auto panel_to = [&](int j, RowMove* mv, int* nm) {
      if (variant == 0) gj_panel_reg_kernel<32, 1><<<n, threads, smem, s>>>(d_desc, j, d_info, mv, nm);
      else if (variant == 4) gj_panel_reg_kernel<16, 1><<<n, threads, smem, s>>>(d_desc, j, d_info, mv, nm);
      else gj_panel_reg_kernel<32, 2><<<n, threads, smem, s>>>(d_desc, j, d_info, mv, nm);
      CK_LAUNCH();
    };
    auto upd = [&](int j, int bw, double* const* dw, int mode) {
      int mt = 0;
      for (int p = 0; p < n; p++) {
        const int m = h[p].m;
        if (m <= j) continue;
        const int bb = std::min(bw, m - j), b2 = std::min(bw, m - j - bb);
        const int nc = mode == 4 ? std::min(bw, j) : (mode == 0 ? m - bb : (mode == 1 ? b2 : m - bb - b2));
        if (nc > 0) mt = std::max(mt, ceil_div(m, GBM) * ceil_div(nc, GBN));
      }
      if (mt > 0) {
        gj_update_v2_kernel<<<dim3(n, mt), GTHREADS, GSMEM, s>>>(d_desc, j, bw, dw, mode);
        CK_LAUNCH();
      }
    };
    for (int J = 0; J < maxm; J += B2) {
      panel_to(J, moves, nmoves);
      const bool second = J + b < maxm;
      if (second) {
        // moves 1 on inner panel 2 + its pivot rows; inner update of panel 2
        gj_move_copy2_kernel<<<dim3(n, 1), 256, 0, s>>>(d_desc, J, b, B2, 0, 0, b, moves, nmoves, nullptr, nullptr,
                                                        0, b, dW, 0, 0);
        CK_LAUNCH();
        upd(J, b, dW, 1);
        panel_to(J + b, moves2, nmoves2);
        // moves 2 on inner panel 1 + its pivot rows; inner update of panel 1
        gj_move_copy2_kernel<<<dim3(n, 1), 256, 0, s>>>(d_desc, J, 0, b, 0, 0, b, moves2, nmoves2, nullptr,
                                                        nullptr, b, b, dW, b, 0);
        CK_LAUNCH();
        upd(J + b, b, dW, 4);
      }
      // the rest: moves 1 then 2, original pivot rows (2b of them), one rank-2b update
      gj_move_copy2_kernel<<<dim3(n, gy), 256, 0, s>>>(d_desc, J, -1, -1, 0, B2, b, moves, nmoves,
                                                       second ? moves2 : nullptr, second ? nmoves2 : nullptr, 0, B2,
                                                       dWo, 0, b);
      CK_LAUNCH();
      upd(J, B2, dWo, 0);
    }
  } else {
  panel(0, s);
  for (int j = 0; j < maxm; j += b) {
    gj_move_copy_kernel<<<dim3(n, gy), 256, 0, s>>>(d_desc, j, b, moves, nmoves, dW);
    CK_LAUNCH();
    const bool more = j + b < maxm;
    if (v1) {
      // tile prefix of this step (matrices with m <= j contribute nothing)
      std::vector<int>& t0 = tile_pref[(j / b) & 1];
      t0.assign(n + 1, 0);
      for (int p = 0; p < n; p++) {
        const int m = h[p].m;
        const int tiles = m > j ? ceil_div(m, GBM) * ceil_div(m - std::min(b, m - j), GBN) : 0;
        t0[p + 1] = t0[p] + tiles;
      }
      if (t0[n] > 0) {
        const int* dt0 = upload(ws, t0, s, st);
        gj_update_kernel<<<t0[n], GTHREADS, 0, s>>>(d_desc, dt0, n, j, b, dW);
        CK_LAUNCH();
      }
      if (more) panel(j + b, s);
    } else if (look && more) {
      // look-ahead: the next panel's columns first, then that panel on the
      // high-priority side stream concurrently with the rest of the update
      update(j, 1);
      CK(cudaEventRecord(side->e_cols, s));
      CK(cudaStreamWaitEvent(side->s, side->e_cols, 0));
      panel(j + b, side->s);
      CK(cudaEventRecord(side->e_panel, side->s));
      update(j, 2);
      CK(cudaStreamWaitEvent(s, side->e_panel, 0));
    } else {
      update(j, 0);
      if (more) panel(j + b, s);
    }
  }
  }  // one-level path
  // undo the row pivoting as one column gather per matrix (through scratch)
  int* perm = ws.alloc_n<int>(size_t(n) * maxm);
  std::vector<double*> T(n);
  for (int p = 0; p < n; p++) T[p] = ws.alloc_n<double>(size_t(h[p].m) * h[p].m);
  double* const* dT = upload(ws, T, s, st);
  gj_colperm_kernel<<<n, 32, 0, s>>>(d_desc, perm, maxm);
  CK_LAUNCH();
  gj_colgather_kernel<<<dim3(n, gy), 256, 0, s>>>(d_desc, perm, maxm, dT, 0);
  CK_LAUNCH();
  gj_colgather_kernel<<<dim3(n, gy), 256, 0, s>>>(d_desc, perm, maxm, dT, 1);
  CK_LAUNCH();
}

}  // namespace ifmm
