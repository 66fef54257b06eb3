// Rank-growth control: joint re-truncation of a cluster's coupling row right
// before its elimination (see consolidate.cu).
#pragma once
#include <vector>

#include "common.cuh"

namespace ifmm {

struct ConsDesc {
  int cluster;      // index into the level's device rank table
  int n, r, W;      // particle dim, current rank, coupling-row width
  const double* U;  // n x r basis (ld n)
  const double* row;  // gathered coupling row Rw (r x W, ld r)
  double* row2;     // out: T^T Rw, zero rows beyond the kept rank (r x W, ld r)
  // set by launch_consolidate (batch workspace):
  double* U2;       // out: U T, zero columns beyond the kept rank (n x r, ld n)
  double *G, *T, *scratch;
};

// newrank[p] = rank kept for descs[p] (== r when nothing is dropped); d_rank[cluster] is updated.
// On return every desc's row2 / U2 are queued on the stream: copy them back over the blocks / the basis.
// shape_maxr: largest rank of the whole colour batch across ranks (the CTA width follows it, so a
// sharded run uses the same arithmetic as one GPU)
void launch_consolidate(std::vector<ConsDesc>& h, double rank_tol, int* d_rank, int* d_newrank, Arena& ws,
                        Staging& st, cudaStream_t s, int shape_maxr = 0);

}  // namespace ifmm
