// Grouped variable-size FP64 GEMM on the B200 FP64 tensor pipe (DMMA,
// mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4; tcgen05 has no f64 kind).
//
//   C_p = alpha_p * op(A_p) * op(B_p) + beta_p * C_p      for every problem p
//
// One launch covers a whole colour batch: problems are laid out as a flat
// tile space (64x64 output tiles, prefix-summed on the host) and every CTA
// binary-searches its problem.  C may be stored transposed (`transC`): the
// IFMM stores every symmetric block pair once, so Schur updates land in
// whichever orientation the owner block uses.  Operands are staged through
// double-buffered shared memory with a bank-conflict-free k-major layout
// (row stride 68 doubles == 4 mod 16).
#pragma once
#include "common.cuh"

namespace ifmm {

struct GemmProb {
  const double* A;
  const double* B;
  double* C;
  int M, N, K;
  int lda, ldb, ldc;
  double alpha, beta;
  int transC;
  int tile0;  // first global tile index of this problem
};

constexpr int GBM = 64, GBN = 64, GBK = 16, GPAD = 68, GTHREADS = 128;

template <bool TA, bool TB>
__global__ void __launch_bounds__(GTHREADS, 4)
    grouped_dgemm_kernel(const GemmProb* __restrict__ probs, int nprob) {
  __shared__ double As[2][GBK][GPAD];
  __shared__ double Bs[2][GBK][GPAD];
  // locate problem: largest p with tile0 <= blockIdx.x
  int lo = 0, hi = nprob - 1;
  const int t = blockIdx.x;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (probs[mid].tile0 <= t) lo = mid; else hi = mid - 1;
  }
  const GemmProb P = probs[lo];
  const int tl = t - P.tile0;
  const int tilesM = (P.M + GBM - 1) / GBM;
  const int i0 = (tl % tilesM) * GBM, j0 = (tl / tilesM) * GBN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;

  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; a++)
#pragma unroll
    for (int b = 0; b < 4; b++) acc[a][b][0] = acc[a][b][1] = 0.0;

  double ra[8], rb[8];
  auto load_tiles = [&](int k0) {
#pragma unroll
    for (int e = 0; e < 8; e++) {
      int idx = tid + e * GTHREADS;
      int i, k;
      if (!TA) { i = idx & 63; k = idx >> 6; } else { k = idx & 15; i = idx >> 4; }
      int gi = i0 + i, gk = k0 + k;
      double v = 0.0;
      if (gi < P.M && gk < P.K) v = TA ? P.A[gk + (size_t)gi * P.lda] : P.A[gi + (size_t)gk * P.lda];
      ra[e] = v;
      int j;
      if (!TB) { k = idx & 15; j = idx >> 4; } else { j = idx & 63; k = idx >> 6; }
      int gj = j0 + j;
      gk = k0 + k;
      v = 0.0;
      if (gj < P.N && gk < P.K) v = TB ? P.B[gj + (size_t)gk * P.ldb] : P.B[gk + (size_t)gj * P.ldb];
      rb[e] = v;
    }
  };
  auto store_tiles = [&](int buf) {
#pragma unroll
    for (int e = 0; e < 8; e++) {
      int idx = tid + e * GTHREADS;
      int i, k, j;
      if (!TA) { i = idx & 63; k = idx >> 6; } else { k = idx & 15; i = idx >> 4; }
      As[buf][k][i] = ra[e];
      if (!TB) { k = idx & 15; j = idx >> 4; } else { j = idx & 63; k = idx >> 6; }
      Bs[buf][k][j] = rb[e];
    }
  };

  const int nk = (P.K + GBK - 1) / GBK;
  if (nk > 0) {
    load_tiles(0);
    store_tiles(0);
    __syncthreads();
  }
  for (int kt = 0; kt < nk; kt++) {
    const int buf = kt & 1;
    if (kt + 1 < nk) load_tiles((kt + 1) * GBK);
#pragma unroll
    for (int kk = 0; kk < GBK; kk += 4) {
      double fa[4], fb[4];
#pragma unroll
      for (int m = 0; m < 4; m++) fa[m] = As[buf][kk + (lane & 3)][wm + m * 8 + (lane >> 2)];
#pragma unroll
      for (int n = 0; n < 4; n++) fb[n] = Bs[buf][kk + (lane & 3)][wn + n * 8 + (lane >> 2)];
#pragma unroll
      for (int m = 0; m < 4; m++)
#pragma unroll
        for (int n = 0; n < 4; n++)
          asm volatile(
              "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
              : "+d"(acc[m][n][0]), "+d"(acc[m][n][1])
              : "d"(fa[m]), "d"(fb[n]));
    }
    if (kt + 1 < nk) {
      store_tiles(buf ^ 1);
      __syncthreads();
    }
  }
  // epilogue: C = alpha*acc + beta*C
  const double alpha = P.alpha, beta = P.beta;
#pragma unroll
  for (int m = 0; m < 4; m++) {
    const int gi = i0 + wm + m * 8 + (lane >> 2);
    if (gi >= P.M) continue;
#pragma unroll
    for (int n = 0; n < 4; n++) {
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int gj = j0 + wn + n * 8 + 2 * (lane & 3) + h;
        if (gj >= P.N) continue;
        double* c = P.transC ? P.C + gj + (size_t)gi * P.ldc : P.C + gi + (size_t)gj * P.ldc;
        double v = alpha * acc[m][n][h];
        if (beta != 0.0) v += beta * *c;
        *c = v;
      }
    }
  }
}

// Host side: accumulate problems, then launch once.
struct GemmBatch {
  std::vector<GemmProb> probs;
  int tiles = 0;
  void add(const double* A, int lda, const double* B, int ldb, double* C, int ldc, int M, int N, int K,
           double alpha, double beta, bool transC = false) {
    if (M <= 0 || N <= 0) return;
    GemmProb p{A, B, C, M, N, K, lda, ldb, ldc, alpha, beta, transC ? 1 : 0, tiles};
    probs.push_back(p);
    tiles += ceil_div(M, GBM) * ceil_div(N, GBN);
  }
  void clear() {
    probs.clear();
    tiles = 0;
  }
};

void launch_grouped_gemm(GemmBatch& b, bool transA, bool transB, Arena& ws, Staging& st, cudaStream_t s);

}  // namespace ifmm
