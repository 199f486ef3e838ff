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
#include <vector>

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
  // row-sharded plans (tri_plan_dist): block-rows are the local ones, global index I0 + I;
  // the tiles of a block-row are listed explicitly (jt_of) and every column tile jt has
  // its column partials in the local block-rows [cr_lo[jt], cr_hi[jt]); the finalize then
  // writes the unrounded pair of every row i < n to ypair (no lambda term, no epilogue)
  // for the exchange (pcg_dist.cu).  Single-rank plans: I0 = 0, jt_of = null.
  int32_t I0;
  const int32_t *jt_of;
  const int32_t *cr_lo, *cr_hi;
  dd_pair *ypair;
  int64_t own0, own1;  // global rows whose row partials this rank holds
  FusedUpdate upd;     // single-rank K apply inside the PCG: the update step fused (symv.cu)
  // the exact tensor-core apply (symv_tc.cu): per row, the 8 exact int64 level-group sums
  // [8][ldy] accumulated by the tile kernel (integer atomics: exact, order-free), turned
  // into the row's pair by the finalize with scale 2^(tc_exp[0] + tc_exp[1] + 2 - 14)
  // (eK, F), which also zeroes them for the next apply
  long long *yacc;
  int64_t ldy;
  const int *tc_exp;
};

// The exact tensor-core apply's level groups: group g holds levels L = 3g .. 3g + 2 as
// G_g = sum_{L in g} D_L 2^(7(3g+2-L)), |G_g| < 2^48 (exact in fp64); the value is
// sum_g G_g 2^(-7(3g+2)) 2^escale, folded by a TwoSum chain into an unrounded pair.
constexpr int kTcGroups = 8;
__device__ __forceinline__ double tc_pow2(int e) { return __longlong_as_double((long long)(1023 + e) << 52); }
__device__ __forceinline__ dd_pair tc_groups_to_pair(const long long (&G)[kTcGroups], int escale) {
  dd_pair r = {__dmul_rn((double)G[0], tc_pow2(-14)), 0.0};
#pragma unroll
  for (int g = 1; g < kTcGroups; ++g) {
    const double t = __dmul_rn((double)G[g], tc_pow2(-7 * (3 * g + 2)));
    double s, e;
    two_sum(r.s, t, s, e);
    r.s = s;
    r.c = __dadd_rn(r.c, e);
  }
  r.s = ldexp(r.s, escale);
  r.c = ldexp(r.c, escale);
  return r;
}

// partition of an n x n symmetric apply into BR x TC tiles over `grid` CTAs
cudaError_t tri_plan(SymvPlan *&p, int64_t n, int br, int tc, int grid);
// the row-sharded version: rank `rank` of `world` owns rows [rank n/W, (rank+1) n/W) and
// takes the tiles of dist_tiles() (each pair of symmetric entries once over all ranks)
cudaError_t tri_plan_dist(SymvPlan *&p, int64_t n, int br, int tc, int grid, int rank, int world);
bool tri_is_dist(const SymvPlan *p);
// Host: the tile lists of the row-sharded symmetric apply (n / world a multiple of 2 br).
// Rank w's block-rows I (local, global w L + I, L = n / (world br)) take, in this order:
//   the tiles of its own diagonal block from the diagonal on (jt >= (br/tc)(w L + I));
//   every tile of the blocks c = w + d (mod W), d = 1 .. D  (D = (W - 1) / 2, W odd;
//   W / 2 - 1, W even);
//   W even, c = w + W/2: rank min(w, c) takes block c for its first L/2 block-rows,
//   rank max(w, c) takes the second half of block c's columns for all its block-rows.
// Every off-diagonal block pair is then streamed once (its transpose never), so each rank
// streams (n/W)^2/2 + (W/2 - 1/2)(n/W)^2 ... = n^2 / (2 W) entries: the single-GPU
// triangle divided by W.  toff [L + 1], jt [T] (global column tiles), cr_lo / cr_hi [nct]
// (local block-rows with column partials for column tile jt: off-diagonal-block tiles).
bool dist_tiles(int64_t n, int br, int tc, int rank, int world, std::vector<int64_t> &toff,
                std::vector<int32_t> &jt, std::vector<int32_t> &cr_lo, std::vector<int32_t> &cr_hi);
// ranks that receive this rank's column partials: w + d (mod W), d = 1 .. nsend
inline int dist_nsend(int world) { return world / 2; }
// the plan's partition fields of SymvArgs
void tri_fill(const SymvPlan *p, SymvArgs &a);
int tri_grid(const SymvPlan *p);
int64_t tri_n(const SymvPlan *p);
int tri_br(const SymvPlan *p);
// otf_tc2.cu: the FAST symmetric on-the-fly tiles of a (128, 128) plan
cudaError_t launch_otf_tc2_sym(const OzSlices &E, int64_t n, double scale, const double *w, double2 *cf,
                               const SymvArgs &ta, int grid, cudaStream_t s);
// symv_tc.cu: x's digit slices, then the exact tensor-core tile pass writing a's column
// partials and its own row segments (a's nseg / maxseg / rowpart are set to them)
void launch_symv_tc(SymvTc *p, SymvArgs &a, cudaStream_t s);
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
