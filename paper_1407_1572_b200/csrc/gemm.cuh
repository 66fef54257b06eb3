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
#include <algorithm>

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

// ---------------------------------------------------------------------------
// v2: cp.async pipeline.  Tiles go straight from global to shared memory
// (8-byte cp.async: leading dimensions are arbitrary) into a layout that keeps
// the operand's contiguous direction contiguous in shared memory:
//   k-contiguous operand (A^T, B)   -> [i][k], pitch KP = GBK + 4 (== 4 mod 16)
//   i-contiguous operand (A, B^T)   -> [k][i], pitch IP = GBM + 4 (== 4 mod 16)
// Both the copies (consecutive threads -> consecutive addresses) and the DMMA
// fragment reads (lanes 0-15 hit 16 distinct 8-byte banks) are conflict-free;
// out-of-range elements are zero-filled by the copy itself.
constexpr int KP = GBK + 4, IP = GBM + 4;
constexpr int GSTAGES = 3;
constexpr int GTILE_D = (GBM * KP > GBK * IP ? GBM * KP : GBK * IP);  // doubles per operand tile
constexpr size_t GSMEM = sizeof(double) * 2 * GTILE_D * GSTAGES;

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool pred) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int n = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(pred ? gmem : nullptr), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Copy the (GBM x GBK) op(X) tile at (r0, k0) of an operand with `rows` rows:
// KCONT: element (r, k) at X[k + r*ld] (k-contiguous), else X[r + k*ld].
template <bool KCONT>
__device__ __forceinline__ void load_operand(double* sm, const double* X, int ld, int rows, int K, int r0, int k0,
                                             int tid) {
#pragma unroll
  for (int e = 0; e < (GBM * GBK) / GTHREADS; e++) {
    const int c = tid + e * GTHREADS;
    int r, k;
    if (KCONT) { k = c & (GBK - 1); r = c / GBK; } else { r = c & (GBM - 1); k = c / GBM; }
    const int gr = r0 + r, gk = k0 + k;
    const bool ok = gr < rows && gk < K;
    const double* src = KCONT ? X + gk + (size_t)gr * ld : X + gr + (size_t)gk * ld;
    double* dst = KCONT ? sm + r * KP + k : sm + k * IP + r;
    cp_async8(dst, src, ok);
  }
}
template <bool KCONT>
__device__ __forceinline__ double frag(const double* sm, int r, int k) {
  return KCONT ? sm[r * KP + k] : sm[k * IP + r];
}

template <bool TA, bool TB>
__global__ void __launch_bounds__(GTHREADS, 3)
    grouped_dgemm_v2_kernel(const GemmProb* __restrict__ probs, const int* __restrict__ tile_prob) {
  extern __shared__ double gsm[];
  const int t = blockIdx.x;
  const GemmProb P = probs[tile_prob[t]];  // host-built map: one load, no search
  const int tl = t - P.tile0;
  const int tilesM = (P.M + GBM - 1) / GBM;
  const int i0 = (tl % tilesM) * GBM, j0 = (tl / tilesM) * GBN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
  // op(A) (M x K): k-contiguous iff TA;  op(B)^T (N x K): k-contiguous iff !TB
  constexpr bool AK = TA, BK = !TB;
  auto Asm = [&](int st) { return gsm + (size_t)st * 2 * GTILE_D; };
  auto Bsm = [&](int st) { return gsm + (size_t)st * 2 * GTILE_D + GTILE_D; };

  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; a++)
#pragma unroll
    for (int b = 0; b < 4; b++) acc[a][b][0] = acc[a][b][1] = 0.0;

  const int nk = (P.K + GBK - 1) / GBK;
#pragma unroll
  for (int st = 0; st < GSTAGES - 1; st++) {
    if (st < nk) {
      load_operand<AK>(Asm(st), P.A, P.lda, P.M, P.K, i0, st * GBK, tid);
      load_operand<BK>(Bsm(st), P.B, P.ldb, P.N, P.K, j0, st * GBK, tid);
    }
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; kt++) {
    cp_async_wait<GSTAGES - 2>();
    __syncthreads();  // tile kt visible to all; buffer of kt-1 free
    {
      const int nt = kt + GSTAGES - 1;
      if (nt < nk) {
        const int st = nt % GSTAGES;
        load_operand<AK>(Asm(st), P.A, P.lda, P.M, P.K, i0, nt * GBK, tid);
        load_operand<BK>(Bsm(st), P.B, P.ldb, P.N, P.K, j0, nt * GBK, tid);
      }
      cp_async_commit();
    }
    const double* As = Asm(kt % GSTAGES);
    const double* Bs = Bsm(kt % GSTAGES);
#pragma unroll
    for (int kk = 0; kk < GBK; kk += 4) {
      double fa[4], fb[4];
#pragma unroll
      for (int m = 0; m < 4; m++) fa[m] = frag<AK>(As, wm + m * 8 + (lane >> 2), kk + (lane & 3));
#pragma unroll
      for (int n = 0; n < 4; n++) fb[n] = frag<BK>(Bs, wn + n * 8 + (lane >> 2), kk + (lane & 3));
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
  const double alpha = P.alpha, beta = P.beta;
  // loads of a row group issued together, then its stores (see schur_concat_kernel)
#pragma unroll
  for (int m = 0; m < 4; m++) {
    const int gi = i0 + wm + m * 8 + (lane >> 2);
    double* ptr[8];
    double old[8];
#pragma unroll
    for (int e = 0; e < 8; e++) {
      const int gj = j0 + wn + (e >> 1) * 8 + 2 * (lane & 3) + (e & 1);
      ptr[e] = (gi < P.M && gj < P.N) ? (P.transC ? P.C + gj + (size_t)gi * P.ldc : P.C + gi + (size_t)gj * P.ldc)
                                      : nullptr;
    }
    if (beta != 0.0) {
#pragma unroll
      for (int e = 0; e < 8; e++) old[e] = ptr[e] ? beta * *ptr[e] : 0.0;
    } else {
#pragma unroll
      for (int e = 0; e < 8; e++) old[e] = 0.0;
    }
#pragma unroll
    for (int e = 0; e < 8; e++)
      if (ptr[e]) *ptr[e] = old[e] + alpha * acc[m][e >> 1][e & 1];
  }
}

// ---------------------------------------------------------------------------
// Schur update of one colour batch as one concatenated product per pivot:
//   T = C^T X   (C = C_top, X = X_top, both n x w with the w columns grouped in
//               slots: neighbours' particles, interaction-list ranks, own rank)
// and T's block (a, b), a <= b, is subtracted from the target block of the
// slot pair (P2P, hybrid or M2L storage, possibly transposed).  Tiles run over
// the concatenated w dimension, so slot sizes that are not multiples of the
// tile no longer pad every block to 64x64; tiles entirely below the block
// diagonal are never launched, and the epilogue scatters each element to its
// target (elements with slot(i) > slot(j) are skipped).  Rows of the own-rank
// slot are excluded: C is zero there and (own, own) is handled separately.
struct SchurTgt {
  double* p;
  int ld;
  int trans;
};
struct SchurPiv {
  const double* C;  // n x w, ld n
  const double* X;  // n x w, ld n
  int n, w, wr, ns;  // wr = rows taken (all slots but the own-rank one)
  int soff0, tab0;   // offsets into the slot-offset and target pools
};

// Host side of the concatenated Schur update.
struct SchurBatch {
  std::vector<SchurPiv> pivs;
  std::vector<int2> tiles;
  std::vector<int> soff;
  std::vector<SchurTgt> tab;
  // soff: slot offsets (ns + 1) of this pivot; call set_target for every a <= b
  // with both slots non-empty (others may stay null), then finish_pivot.
  int begin_pivot(const double* C, const double* X, int n, const std::vector<int>& so) {
    SchurPiv P{C, X, n, so.back(), so[so.size() - 2], int(so.size()) - 1, int(soff.size()), int(tab.size())};
    soff.insert(soff.end(), so.begin(), so.end());
    tab.resize(tab.size() + size_t(P.ns) * (P.ns + 1) / 2, SchurTgt{nullptr, 0, 0});
    pivs.push_back(P);
    return int(pivs.size()) - 1;
  }
  void set_target(int pv, int a, int b, double* p, int ld, bool trans) {
    const SchurPiv& P = pivs[pv];
    tab[P.tab0 + a * P.ns - (a * (a - 1)) / 2 + (b - a)] = SchurTgt{p, ld, trans ? 1 : 0};
  }
  void finish_pivot(int pv) {
    const SchurPiv& P = pivs[pv];
    if (P.n == 0 || P.wr == 0) return;
    const int* so = soff.data() + P.soff0;
    const int tm = ceil_div(P.wr, GBM), tn = ceil_div(P.w, GBN);
    auto slot_of = [&](int g) { return int(std::upper_bound(so, so + P.ns + 1, g) - so) - 1; };
    for (int ti = 0; ti < tm; ti++) {
      const int a0 = slot_of(ti * GBM);
      for (int tj = 0; tj < tn; tj++) {
        const int b1 = slot_of(std::min(P.w, (tj + 1) * GBN) - 1);
        if (a0 <= b1) tiles.push_back(make_int2(pv, (ti << 16) | tj));
      }
    }
  }
  void clear() {
    pivs.clear();
    tiles.clear();
    soff.clear();
    tab.clear();
  }
};

// Host side: accumulate problems, then launch once.
struct GemmBatch {
  std::vector<GemmProb> probs;
  int tiles = 0;
  void add(const double* A, int lda, const double* B, int ldb, double* C, int ldc, int M, int N, int K,
           double alpha, double beta, bool transC = false) {
    if (M <= 0 || N <= 0) return;
    GemmProb p{A, B, C, M, N, K, lda, ldb, ldc, alpha, beta, transC ? 1 : 0, tiles};
    const int nt = ceil_div(M, GBM) * ceil_div(N, GBN);
    tile_prob.insert(tile_prob.end(), size_t(nt), int(probs.size()));
    probs.push_back(p);
    tiles += nt;
  }
  void clear() {
    probs.clear();
    tile_prob.clear();
    tiles = 0;
  }
  std::vector<int> tile_prob;  // problem of every output tile
};

void launch_grouped_gemm(GemmBatch& b, bool transA, bool transB, Arena& ws, Staging& st, cudaStream_t s);
void launch_schur(SchurBatch& b, Arena& ws, Staging& st, cudaStream_t s);

}  // namespace ifmm
