// Block-upper-triangle work partition shared by the symmetric applies (symv.cu:
// the stored K / P; otf_sym.cu: K recomputed on the fly).  Block-rows of BR rows;
// tiles of BR rows x TC columns; block-row I owns the tiles with column index
// jt >= (BR/TC) I, linearised row-major; persistent CTA b takes the contiguous
// range [T b/G, T (b+1)/G).  A tile on the diagonal block contributes to its rows
// only, every other tile (I, J) to its rows (K_IJ x_J) and to the rows of block J
// (K_IJ^T x_I = K_JI x_I):
//   rowpart[I][s][r]   the unrounded Dot2 pair of block-row I's segment s (the
//                      s-th CTA covering it), row r;
//   colpart[I][j]      the pair of column j from the tiles (I, J(j)), J(j) > I;
// the finalize kernel forms y_i = RN(sum_{I < J(i)} colpart[I][i] +
// sum_s rowpart[J(i)][s][i mod BR] + lambda x_i) in that fixed order, the Dot2
// pair x.y per CTA, and the last CTA runs the PCG scalar epilogue.
#pragma once
#include "laker_internal.h"

namespace laker {

struct SymvArgs {
  int64_t n;
  int32_t nb, nct, maxseg;
  int64_t T;
  const int64_t *toff;      // [nb + 1] first tile of each block-row
  const int32_t *segfirst;  // [nb] first CTA covering block-row I
  const int32_t *nseg;      // [nb]
  const double *x;          // symv: padded to >= nct * TC (zeros past n)
  double *y;
  double lambda;
  PcgState *state;
  int epi;
  double *dot_out;
  dd_pair *pair_out;
  dd_pair *colpart;  // [nb][ldcp]
  int64_t ldcp;
  dd_pair *rowpart;  // [nb][maxseg][BR]
  dd_pair *partials;  // finalize: per-CTA pairs
  unsigned int *counter;
  int evict_first;
  // symv: per-row max |A_ij| (padded with zeros to nct * TC) and per-CTA maxima of |x_j|
  // (max over nxparts values = max |x|): the offsets of dot2_step_off
  const double *rowmax;
  const double *xparts;
  int nxparts;
};

// partition of an n x n symmetric apply into BR x TC tiles over `grid` CTAs
cudaError_t tri_plan(SymvPlan *&p, int64_t n, int br, int tc, int grid);
// the plan's partition fields of SymvArgs
void tri_fill(const SymvPlan *p, SymvArgs &a);
int tri_grid(const SymvPlan *p);
int64_t tri_n(const SymvPlan *p);
int tri_br(const SymvPlan *p);
// otf_tc2.cu: the FAST symmetric on-the-fly tiles of a (128, 128) plan
cudaError_t launch_otf_tc2_sym(const OzSlices &E, int64_t n, double scale, const double *w, double2 *cf,
                               const SymvArgs &ta, int grid, cudaStream_t s);
// y (and the epilogue of a.epi) from the partials written by a tile kernel of this plan
void launch_tri_finalize(const SymvPlan *p, const SymvArgs &a, cudaStream_t s);

// CTA b's first block-row: the largest I with toff[I] <= t
__device__ __forceinline__ int find_block_row(const int64_t *toff, int nb, int64_t t) {
  int lo = 0, hi = nb - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (toff[mid] <= t) lo = mid; else hi = mid - 1;
  }
  return lo;
}

}  // namespace laker
