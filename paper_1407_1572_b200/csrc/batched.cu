// Batched block copies, grouped DGEMM and Schur-update launches, 1-norms.
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

}  // namespace ifmm
