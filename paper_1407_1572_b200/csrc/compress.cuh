// Batched fill-in compression (ifmm/solver.py:319-434, 495-520).
//
// The reference compresses the fills of one elimination sequentially.  Their
// true dependencies are narrower, and the batch is split along them:
//   K1 ACA + QR/SVD recompression         -- every fill independent
//   K2+K3 basis augmentation               -- serial only per cluster: chain c
//                                            holds the steps that append to U_c
//                                            (hybrid fills into c, then the
//                                            sides of the P2P fills touching c)
//   K4 M2L absorption + drop               -- every fill independent: the basis
//                                            prefix each fill saw is recorded
// K1..K4 reproduce the reference's sequential order exactly (augmentation only
// appends columns, so "U_q after fill f" is a prefix of the final U_q).
#pragma once
#include "common.cuh"

namespace ifmm {

enum FillKind : int { FILL_HYBRID = 0, FILL_P2P = 1 };

// One row per fill height m of the ACA probe table: the reference's 10 probe
// rows (np.random.default_rng(0).choice(m, min(10, m), replace=False),
// ifmm/lowrank.py:196-197), then that generator's PCG64 state after the draw
// (6 x 64 bits: state hi/lo, increment hi/lo, has_uint32, uinteger) for the
// random restart rows (ifmm/lowrank.py:224-226).
constexpr int ACA_PROBE_STRIDE = 22;

struct FillDesc {
  int kind, p, q;
  double* F;    // fill block; F(a,b) = transF ? F[b + a*ldF] : F[a + b*ldF]
  int ldF, transF;
  int rows, cols;  // hybrid: r_p x n_q ; P2P: n_p x n_q
  int n_p, n_q;
  double* Up;   // n_p x cap (ld n_p)
  double* Uq;   // n_q x cap (ld n_q)
  double* M;    // M2L(p,q) storage
  int ldM, transM;
  double* out;  // left (rows x Kf) | right (cols x Kf) | sig (Kf)
  int Kf;       // max crosses / stored rank of this pass (buffer capacity of `out`)
  int kfull;    // the reference's cap: min(rows, cols) (ifmm/lowrank.py:188-191); a fill whose
                // ACA reaches Kf < kfull crosses unconverged is redone with a kfull buffer
};

struct FillState {
  int status;  // 0 compressed, 1 kept dense
  int k, r;    // ACA crosses, recompressed rank
  int rq, rp;  // basis ranks of q / p right after this fill's augmentation
  double fro;  // ||left||_F
};

struct CompressBatch {
  std::vector<FillDesc> fills;
  std::vector<int> chain_off, chain;  // hybrid chains (fill indices, sorted by p)
  std::vector<int> p2p_off, p2p;      // per pivot P2P fills (sorted)
  std::vector<int> chain_q;           // q of each chain
  const int* rank_host = nullptr;     // host copy of the level's ranks at batch start
  // sharded runs: largest fill dimension and fill count of the whole colour
  // batch across ranks; worker shapes are chosen from them so every fill is
  // compressed with the same arithmetic as on one GPU
  int shape_mx = 0, shape_nf = 0;
  // Trees with empty / sparse cells (build_tree(..., allow_empty_leaves=True)): a fill whose ACA
  // runs to the full rank min(m, n) is an exact factorization and is absorbed into the bases at
  // that rank instead of being kept dense (the reference keeps it dense, ifmm/solver.py:319-325;
  // between the few-point clusters of a sparse region that chains dense couplings across the
  // whole region)
  int full_rank_ok = 0;
};

// Runs K1..K4 on stream s.  rank: device ranks of the level (updated);
// state: device FillState per fill (out); stats: [compressed, dense_kept, max_rank].
void run_compression(CompressBatch& cb, double tol, const int* d_probes, int probe_maxm, int* d_rank,
                     FillState* d_state, int* d_stats, Arena& ws, Staging& st, cudaStream_t s, int debug);

// test hook: K1 (ACA + recompression) on one m x n fill; d_out holds
// left (m x Kf) | right (n x Kf) | sv (Kf), Kf = min(96, m, n)
void test_recompress_one(const double* dF, int m, int n, double tol, const int* d_probes, int probe_maxm, int gram,
                         double* d_out, FillState* d_state, Arena& ws, Staging& st, cudaStream_t s);

}  // namespace ifmm
