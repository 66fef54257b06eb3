// Batched fill-in compression kernels K1..K4 (see compress.cuh).
#include <algorithm>

#include "compress.cuh"

namespace ifmm {
__device__ int g_prof_on = 0;
__device__ unsigned long long g_cyc[16];  // debug stage cycle counters (IFMM_PROF)
}  // namespace ifmm
// debug: Jacobi sweep statistics (sweeps, calls, columns) under IFMM_PROF
#define IFMM_JACOBI_STATS(sw, ncol)                               \
  do {                                                            \
    if (g_prof_on && threadIdx.x == 0) {                          \
      atomicAdd(&g_cyc[8], (unsigned long long)(sw));             \
      atomicAdd(&g_cyc[9], 1ull);                                 \
      atomicAdd(&g_cyc[10], (unsigned long long)(ncol));          \
    }                                                             \
  } while (0)
#include "cta_la.cuh"

namespace ifmm {
#define PROF_T0() long long _pt = g_prof_on ? clock64() : 0
#define PROF_ACC(i) \
  do {                                                                  \
    if (g_prof_on) {                                                    \
      const long long _n = clock64();                                   \
      if (threadIdx.x == 0) atomicAdd(&g_cyc[i], (unsigned long long)(_n - _pt)); \
      _pt = _n;                                                         \
    }                                                                   \
  } while (0)

constexpr int CTMAX = 512;  // compression CTAs: 128 threads for small fills, 512 at coarse levels

// ------------------------------------------------------------------ K1
__global__ void __launch_bounds__(CTMAX) aca_recompress_kernel(const FillDesc* __restrict__ fills, int nf,
                                                            FillState* state, double tol, const int* probes,
                                                            int probe_maxm, double* scratch, size_t slot,
                                                            int MR, int MC, int KK) {
  __shared__ CtaShared sh;
  double* s = scratch + slot * blockIdx.x;
  double* Uc = s; s += (size_t)MR * KK;
  double* Ql = s; s += (size_t)MR * KK;
  double* Vc = s; s += (size_t)MC * KK;
  double* Qr = s; s += (size_t)MC * KK;
  double* Rl = s; s += (size_t)KK * KK;
  double* Rr = s; s += (size_t)KK * KK;
  double* core = s; s += (size_t)KK * KK;
  double* Jv = s; s += (size_t)KK * KK;
  double* rr = s; s += MC;
  double* cc = s; s += MR;
  double* dots = s; s += KK;
  double* vv = s; s += KK;
  double* sig = s; s += KK;
  int* usedr = reinterpret_cast<int*>(s); s += MR;
  int* usedc = reinterpret_cast<int*>(s); s += MC;
  int* ord = reinterpret_cast<int*>(s);
  for (int f = blockIdx.x; f < nf; f += gridDim.x) {
    const FillDesc D = fills[f];
    const int rows = D.rows, cols = D.cols;
    FillState S{0, 0, 0, 0, 0, 0.0};
    if (rows == 0 || cols == 0) {
      if (threadIdx.x == 0) state[f] = S;
      __syncthreads();
      continue;
    }
    if (tol == 0.0) {  // exact mode: the redirected fill is F itself (bases are identities)
      double nz = 0.0;
      for (int e = threadIdx.x; e < rows * cols; e += blockDim.x) {
        const int a = e % rows, b = e / rows;
        nz += Fat(D.F, D.ldF, D.transF, a, b) != 0.0;
      }
      nz = block_sum(nz, sh.red);
      S.r = nz > 0.0 ? min(rows, cols) : 0;
      if (threadIdx.x == 0) state[f] = S;
      __syncthreads();
      continue;
    }
    const int mrow = rows < probe_maxm ? rows : probe_maxm;
    PROF_T0();
    AcaOut ao = cta_aca(D.F, D.ldF, D.transF, rows, cols, tol, probes + (size_t)mrow * 10, min(10, rows), Uc, Vc,
                        D.Kf, rr, cc, usedr, usedc, dots, sh);
    PROF_ACC(0);
    const int k = ao.k;
    S.k = k;
    if (!ao.converged && (k >= min(rows, cols) || k >= D.Kf)) {
      S.status = 1;
      if (threadIdx.x == 0) state[f] = S;
      __syncthreads();
      continue;
    }
    int r = 0;
    double* left = D.out;
    double* right = D.out + (size_t)rows * D.Kf;
    double* sv = right + (size_t)cols * D.Kf;
    if (k > 0) {
      cta_qr(Uc, rows, k, rows, Rl, Ql, rows, vv, sh);
      cta_qr(Vc, cols, k, cols, Rr, Qr, cols, vv, sh);
      PROF_ACC(1);
      cta_gemm(k, k, k, 1.0, Rl, k, false, Rr, k, true, 0.0, core, k);
      cta_jacobi(core, k, k, k, Jv, k, sig, ord, sh);
      r = trunc_rank_dev(sig, ord, k, tol);
      PROF_ACC(2);
      for (int e = threadIdx.x; e < rows * r; e += blockDim.x) {
        const int i = e % rows, c = e / rows;
        const int col = ord[c];
        double acc = 0.0;
        for (int t = 0; t < k; t++) acc = fma(Ql[i + (size_t)t * rows], core[t + (size_t)col * k], acc);
        left[i + (size_t)c * rows] = acc;
      }
      for (int e = threadIdx.x; e < cols * r; e += blockDim.x) {
        const int i = e % cols, c = e / cols;
        const int col = ord[c];
        double acc = 0.0;
        for (int t = 0; t < k; t++) acc = fma(Qr[i + (size_t)t * cols], Jv[t + (size_t)col * k], acc);
        right[i + (size_t)c * cols] = acc;
      }
      for (int c = threadIdx.x; c < r; c += blockDim.x) sv[c] = sig[ord[c]];
      __syncthreads();
    }
    double fro = 0.0;
    for (int e = threadIdx.x; e < rows * r; e += blockDim.x) fro += left[e] * left[e];
    fro = sqrt(block_sum(fro, sh.red));
    PROF_ACC(3);
    S.r = r;
    S.fro = fro;
    if (threadIdx.x == 0) state[f] = S;
    __syncthreads();
  }
}

// ------------------------------------------------------------------ new directions
// H (nU x r): directions to add (already weighted).  Appends w <= cap columns
// to U (nU x cap, ld nU) after its first rU columns; ifmm/solver.py:334-358.
// Two-pass projection, then QR + Jacobi on the small R factor.
__device__ int new_dirs(double* H, int nU, int r, const double* wsig, double* U, int rU, double cutoff, double* Q,
                        double* R, double* E, double* sig, int* ord, double* vv, CtaShared& sh) {
  const int cap = nU - rU;
  if (cap <= 0 || r == 0) return 0;
  PROF_T0();
  cta_project_out(H, nU, nU, r, U, nU, rU, E);
  cta_project_out(H, nU, nU, r, U, nU, rU, E);
  PROF_ACC(4);
  if (wsig) {
    for (int e = threadIdx.x; e < nU * r; e += blockDim.x) H[e] *= wsig[e / nU];
    __syncthreads();
  }
  cta_qr(H, nU, r, nU, R, Q, nU, vv, sh);  // H = Q R
  PROF_ACC(5);
  cta_jacobi(R, r, r, r, nullptr, 0, sig, ord, sh);  // R V = U_R S
  PROF_ACC(6);
  int w = 0;
  for (int t = 0; t < r; t++) w += (sig[ord[t]] > cutoff);
  w = min(w, cap);
  double* W = U + (size_t)rU * nU;
  for (int e = threadIdx.x; e < nU * w; e += blockDim.x) {
    const int i = e % nU, c = e / nU;
    const int col = ord[c];
    double acc = 0.0;
    for (int t = 0; t < r; t++) acc = fma(Q[i + (size_t)t * nU], R[t + (size_t)col * r], acc);
    W[i + (size_t)c * nU] = acc / sig[col];
  }
  __syncthreads();
  if (w > 0) cta_project_out(W, nU, nU, w, U, nU, rU, E);
  PROF_ACC(7);
  return w;
}

struct DirScratch {
  double *H, *Q, *R, *E, *sig, *vv;
  int* ord;
};
__device__ inline DirScratch carve_dirs(double* s, int MX, int KK) {
  DirScratch d;
  d.H = s; s += (size_t)MX * KK;
  d.Q = s; s += (size_t)MX * KK;
  d.E = s; s += (size_t)MX * KK;
  d.R = s; s += (size_t)KK * KK;
  d.sig = s; s += KK;
  d.vv = s; s += KK;
  d.ord = reinterpret_cast<int*>(s);
  return d;
}

// ------------------------------------------------------------------ K2
__global__ void __launch_bounds__(CTMAX) hybrid_dirs_kernel(const FillDesc* __restrict__ fills,
                                                         const int* __restrict__ chain_off,
                                                         const int* __restrict__ chain, int nchains,
                                                         FillState* state, int* rank, double tol, double* scratch,
                                                         size_t slot, int MX, int KK, int debug) {
  __shared__ CtaShared sh;
  DirScratch d = carve_dirs(scratch + slot * blockIdx.x, MX, KK);
  for (int c = blockIdx.x; c < nchains; c += gridDim.x) {
    const int f0 = chain_off[c], f1 = chain_off[c + 1];
    const int q = fills[chain[f0]].q;
    int rq = rank[q];
    for (int u = f0; u < f1; u++) {
      const int f = chain[u];
      const FillDesc D = fills[f];
      const FillState S = state[f];
      if (S.status == 0 && S.r > 0 && tol > 0.0) {
        const double* right = D.out + (size_t)D.rows * D.Kf;
        const double* sv = right + (size_t)D.cols * D.Kf;
        for (int e = threadIdx.x; e < D.cols * S.r; e += blockDim.x) d.H[e] = right[e];
        __syncthreads();
        const int w = new_dirs(d.H, D.cols, S.r, sv, D.Uq, rq, tol * S.fro, d.Q, d.R, d.E, d.sig, d.ord, d.vv, sh);
        if (debug && threadIdx.x == 0) printf("augq kind=0 p=%d q=%d r=%d +%d -> %d\n", D.p, q, S.r, w, rq + w);
        rq += w;
      }
      if (threadIdx.x == 0) state[f].rq = rq;
      __syncthreads();
    }
    if (threadIdx.x == 0) rank[q] = rq;
    __syncthreads();
  }
}

// ------------------------------------------------------------------ K3
__global__ void __launch_bounds__(CTMAX) p2p_dirs_kernel(const FillDesc* __restrict__ fills,
                                                      const int* __restrict__ p2p_off, const int* __restrict__ p2p,
                                                      int ngroups, FillState* state, int* rank, double tol,
                                                      double* scratch, size_t slot, int MX, int KK, int debug) {
  __shared__ CtaShared sh;
  DirScratch d = carve_dirs(scratch + slot * blockIdx.x, MX, KK);
  for (int g = blockIdx.x; g < ngroups; g += gridDim.x) {
    for (int u = p2p_off[g]; u < p2p_off[g + 1]; u++) {
      const int f = p2p[u];
      const FillDesc D = fills[f];
      const FillState S = state[f];
      int rq = rank[D.q], rp = rank[D.p];
      if (S.status == 0 && S.r > 0 && tol > 0.0) {
        const double* left = D.out;
        const double* right = D.out + (size_t)D.rows * D.Kf;
        const double* sv = right + (size_t)D.cols * D.Kf;
        for (int e = threadIdx.x; e < D.cols * S.r; e += blockDim.x) d.H[e] = right[e];
        __syncthreads();
        const int wq = new_dirs(d.H, D.cols, S.r, sv, D.Uq, rq, tol * S.fro, d.Q, d.R, d.E, d.sig, d.ord, d.vv, sh);
        rq += wq;
        for (int e = threadIdx.x; e < D.rows * S.r; e += blockDim.x) d.H[e] = left[e];
        __syncthreads();
        const int wp = new_dirs(d.H, D.rows, S.r, nullptr, D.Up, rp, tol * S.fro, d.Q, d.R, d.E, d.sig, d.ord, d.vv,
                                sh);
        rp += wp;
        if (debug && threadIdx.x == 0)
          printf("augq kind=1 p=%d q=%d r=%d +%d -> %d | p +%d -> %d\n", D.p, D.q, S.r, wq, rq, wp, rp);
      }
      if (threadIdx.x == 0) {
        state[f].rq = rq;
        state[f].rp = rp;
        rank[D.q] = rq;
        rank[D.p] = rp;
      }
      __syncthreads();
    }
  }
}

// ------------------------------------------------------------------ K4
__global__ void __launch_bounds__(CTMAX) delta_kernel(const FillDesc* __restrict__ fills, int nf,
                                                   const FillState* __restrict__ state, double tol, double* scratch,
                                                   size_t slot, int MX, int KK, int* stats) {
  double* Eq = scratch + slot * blockIdx.x;
  double* Ep = Eq + (size_t)MX * KK;
  for (int f = blockIdx.x; f < nf; f += gridDim.x) {
    const FillDesc D = fills[f];
    const FillState S = state[f];
    if (S.status != 0) {
      if (threadIdx.x == 0) atomicAdd(&stats[1], 1);
      continue;
    }
    const int rows = D.rows, cols = D.cols;
    if (tol == 0.0) {
      for (int e = threadIdx.x; e < rows * cols; e += blockDim.x) {
        const int a = e % rows, b = e / rows;
        const double v = Fat(D.F, D.ldF, D.transF, a, b);
        if (D.transM) D.M[b + (size_t)a * D.ldM] += v;
        else D.M[a + (size_t)b * D.ldM] += v;
      }
    } else if (S.r > 0) {
      const int r = S.r, rq = S.rq;
      const double* left = D.out;
      const double* right = D.out + (size_t)rows * D.Kf;
      cta_gemm(rq, r, cols, 1.0, D.Uq, cols, true, right, cols, false, 0.0, Eq, rq);  // Uq^T B
      const double* X = left;
      int rx = rows, ldx = rows;
      if (D.kind == FILL_P2P) {
        cta_gemm(S.rp, r, rows, 1.0, D.Up, rows, true, left, rows, false, 0.0, Ep, S.rp);  // Up^T A
        X = Ep;
        rx = S.rp;
        ldx = S.rp;
      }
      // M2L(p,q) += X Eq^T   (owner stores (q,p): M += Eq X^T)
      if (D.transM) cta_gemm(rq, rx, r, 1.0, Eq, rq, false, X, ldx, true, 1.0, D.M, D.ldM);
      else cta_gemm(rx, rq, r, 1.0, X, ldx, false, Eq, rq, true, 1.0, D.M, D.ldM);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < rows * cols; e += blockDim.x) {
      const int a = e % rows, b = e / rows;
      if (D.transF) D.F[b + (size_t)a * D.ldF] = 0.0;
      else D.F[a + (size_t)b * D.ldF] = 0.0;
    }
    if (threadIdx.x == 0) {
      atomicAdd(&stats[0], 1);
      atomicMax(&stats[2], S.r);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ host
static int resident_grid(int work, int per_sm) { return std::max(1, std::min(work, 148 * per_sm)); }

void run_compression(CompressBatch& cb, double tol, const int* d_probes, int probe_maxm, int* d_rank,
                     FillState* d_state, int* d_stats, Arena& ws, Staging& st, cudaStream_t s, int debug) {
  const int nf = int(cb.fills.size());
  if (nf == 0) return;
  int MR = 1, MC = 1, KK = 1, MX = 1;
  for (const FillDesc& D : cb.fills) {
    MR = std::max(MR, D.rows);
    MC = std::max(MC, D.cols);
    KK = std::max(KK, D.Kf);
    MX = std::max(MX, std::max(D.n_p, D.n_q));
  }
  MX = std::max(MX, std::max(MR, MC));
  // block size: small fills (leaf level, thousands of them) want many small
  // CTAs; coarse levels have few, large fills -> wide CTAs shorten each step
  static const bool narrow = getenv("IFMM_BS128") != nullptr;  // debug: force 128-thread CTAs
  const int bs_fill = narrow ? 128 : (MX >= 256 && nf < 2048) ? 512 : (MX >= 128 ? 256 : 128);
  const int bs_dirs = narrow ? 128 : MX >= 256 ? 512 : (MX >= 128 ? 256 : 128);
  static const bool prof = getenv("IFMM_PROF") != nullptr;
  if (prof) {
    const int one = 1;
    unsigned long long z[16] = {0};
    CK(cudaMemcpyToSymbolAsync(g_prof_on, &one, sizeof(int), 0, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyToSymbolAsync(g_cyc, z, sizeof z, 0, cudaMemcpyHostToDevice, s));
  }
  const FillDesc* dfd = upload(ws, cb.fills, s, st);
  // K1
  {
    const size_t slot = 2 * size_t(MR) * KK + 2 * size_t(MC) * KK + 4 * size_t(KK) * KK + 2 * size_t(MR + MC) +
                        4 * size_t(KK) + 64;
    const int grid = resident_grid(nf, 8);
    double* scr = ws.alloc_n<double>(slot * grid);
    aca_recompress_kernel<<<grid, bs_fill, 0, s>>>(dfd, nf, d_state, tol, d_probes, probe_maxm, scr, slot, MR, MC,
                                                   KK);
    CK_LAUNCH();
  }
  const size_t dslot = 3 * size_t(MX) * KK + size_t(KK) * KK + 3 * size_t(KK) + 64;
  // K2
  const int nch = int(cb.chain_off.size()) - 1;
  if (nch > 0) {
    const int* dco = upload(ws, cb.chain_off, s, st);
    const int* dch = upload(ws, cb.chain, s, st);
    const int grid = resident_grid(nch, 8);
    double* scr = ws.alloc_n<double>(dslot * grid);
    hybrid_dirs_kernel<<<grid, bs_dirs, 0, s>>>(dfd, dco, dch, nch, d_state, d_rank, tol, scr, dslot, MX, KK, debug);
    CK_LAUNCH();
  }
  // K3: P2P fills in dependency waves.  Within a pivot, a fill waits only for
  // earlier fills sharing one of its two clusters (they augment the same
  // basis); fills of different pivots never share clusters.
  const int ng = int(cb.p2p_off.size()) - 1;
  if (ng > 0 && !cb.p2p.empty()) {
    std::vector<int> wave(cb.p2p.size(), 0);
    int nwave = 0;
    static const bool serial = getenv("IFMM_P2P_SERIAL") != nullptr;  // debug: one P2P fill per wave and pivot
    for (int g = 0; g < ng; g++)
      for (int u = cb.p2p_off[g]; u < cb.p2p_off[g + 1]; u++) {
        const FillDesc& D = cb.fills[cb.p2p[u]];
        int w = 0;
        for (int v = cb.p2p_off[g]; v < u; v++) {
          const FillDesc& E = cb.fills[cb.p2p[v]];
          if (E.p == D.p || E.p == D.q || E.q == D.p || E.q == D.q || serial) w = std::max(w, wave[v] + 1);
        }
        wave[u] = w;
        nwave = std::max(nwave, w + 1);
      }
    const int grid_max = resident_grid(int(cb.p2p.size()), 8);
    double* scr = ws.alloc_n<double>(dslot * grid_max);
    for (int w = 0; w < nwave; w++) {
      std::vector<int> off(1, 0), lst;
      for (size_t u = 0; u < cb.p2p.size(); u++)
        if (wave[u] == w) {
          lst.push_back(cb.p2p[u]);
          off.push_back(int(lst.size()));
        }
      const int* dpo = upload(ws, off, s, st);
      const int* dpp = upload(ws, lst, s, st);
      const int n = int(lst.size());
      p2p_dirs_kernel<<<std::min(n, grid_max), bs_dirs, 0, s>>>(dfd, dpo, dpp, n, d_state, d_rank, tol, scr, dslot,
                                                                 MX, KK, debug);
      CK_LAUNCH();
    }
  }
  // K4
  {
    const size_t slot = 2 * size_t(MX) * KK + 64;
    const int grid = resident_grid(nf, 8);
    double* scr = ws.alloc_n<double>(slot * grid);
    delta_kernel<<<grid, bs_fill, 0, s>>>(dfd, nf, d_state, tol, scr, slot, MX, KK, d_stats);
    CK_LAUNCH();
  }
  if (prof) {
    unsigned long long c[16];
    CK(cudaMemcpyFromSymbolAsync(c, g_cyc, sizeof c, 0, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    fprintf(stderr, "prof MX=%d nf=%d chains=%zu p2p=%zu | aca %.1f qr %.1f core %.1f rest %.1f | proj %.1f qr %.1f jac %.1f W %.1f Mcyc | jacobi calls %llu avg sweeps %.2f avg cols %.1f\n",
            MX, nf, cb.chain_off.size() - 1, cb.p2p.size(), c[0] / 1e6, c[1] / 1e6, c[2] / 1e6, c[3] / 1e6, c[4] / 1e6,
            c[5] / 1e6, c[6] / 1e6, c[7] / 1e6, c[9], c[9] ? double(c[8]) / c[9] : 0.0, c[9] ? double(c[10]) / c[9] : 0.0);
  }
}

}  // namespace ifmm
