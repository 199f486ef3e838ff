// fp64 tensor-core GEMM for the dense contractions of the CCCP fit
// (U = (lambda I + K) Z, Gram matrices of the
// directions, T = a I + R diag(b) R^T, Newton-Schulz products, P formation)
// and the multi-RHS operator (row a10).
//
//   C = alpha * A op(B) + beta * Cin + diag * [row - col == diag_offset]
//   A: M x K row-major (k contiguous); op(B): B_KN ? B is K x N row-major
//   (n contiguous) : B is N x K row-major (k contiguous, i.e. A B^T).
//
// mma.sync m8n8k4 .f64 (SASS DMMA) -- tcgen05 has no fp64 kind on sm_100a.
// 128 x 128 x 16 CTA tile, 8 warps (2 x 4) of 64 x 32, 3-stage cp.async
// pipeline, shared-memory strides chosen so every fragment load is
// conflict-free (row stride = 8 words mod 32 for the 4 x 4 lane pattern of a
// half warp).  M and N may be ragged (zero-filled loads, masked stores);
// K must be a multiple of 16 (callers keep operands zero padded).
#include <algorithm>

#include "laker_internal.h"

namespace laker {
namespace {

constexpr int BK = 16, ST = 3;
constexpr int AS = BK + 4;       // As[m][k] row stride (doubles): 8 words mod 32
constexpr int BS_NK = BK + 4;    // Bs[n][k]

// CTA tile BM x BN, WM x WN warps, warp tile (BM/WM) x (BN/WN) of 8 x 8 DMMA fragments.
template <int BM_, int BN_, int WM_, int WN_>
struct Tile {
  static constexpr int BM = BM_, BN = BN_, WM = WM_, WN = WN_;
  static constexpr int THREADS = 32 * WM * WN;
  static constexpr int MI = BM / WM / 8, NJ = BN / WN / 8;
  static constexpr int BS_KN = BN + 4;  // Bs[k][n] stride: BN + 4 = 4 mod 16 doubles
  static constexpr int A_ELEMS = BM * AS;
  static constexpr int B_ELEMS_NK = BN * BS_NK;
  static constexpr int B_ELEMS_KN = BK * BS_KN;
  static constexpr size_t smem(bool kn) { return (size_t)ST * (A_ELEMS + (kn ? B_ELEMS_KN : B_ELEMS_NK)) * 8; }
};
using TileL = Tile<128, 128, 2, 4>;  // 256 threads, 64 x 32 per warp
using TileS = Tile<64, 64, 2, 2>;    // 128 threads, 32 x 32 per warp (skinny / small problems)

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void cp_async16(void *dst, const void *src, bool valid) {
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(su32(dst)), "l"(src), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <class TL, bool B_KN>
__global__ void __launch_bounds__(TL::THREADS) dgemm_kernel(const GemmArgs g) {
  constexpr int BM = TL::BM, BN = TL::BN, MI = TL::MI, NJ = TL::NJ, NT = TL::THREADS;
  const int bm = blockIdx.y, bn = blockIdx.x;
  if (g.lower_only && (int64_t)bn * BN > (int64_t)bm * BM + BM - 1) return;
  if (g.tri == 1 && (int64_t)bm * BM + BM - 1 + g.tri_off < (int64_t)bn * BN) return;
  if (g.tri == 2 && (int64_t)bm * BM + g.tri_off >= (int64_t)bn * BN + BN - 1) return;
  extern __shared__ __align__(16) double sm[];
  double *As = sm;
  double *Bs = sm + ST * TL::A_ELEMS;
  constexpr int BSZ = B_KN ? TL::B_ELEMS_KN : TL::B_ELEMS_NK;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = (warp / TL::WN) * (BM / TL::WM), wn = (warp % TL::WN) * (BN / TL::WN);
  const int fr = lane >> 2, fk = lane & 3;
  const int64_t row0 = (int64_t)bm * BM, col0 = (int64_t)bn * BN;

  auto load_stage = [&](int st, int k0) {
    double *as = As + st * TL::A_ELEMS;
    double *bs = Bs + st * BSZ;
#pragma unroll
    for (int c = tid; c < BM * BK / 2; c += NT) {
      const int r = c / (BK / 2), cc = (c % (BK / 2)) * 2;
      const bool ok = row0 + r < g.M;
      cp_async16(as + r * AS + cc, g.A + (ok ? (row0 + r) : 0) * g.lda + k0 + cc, ok);
    }
    if (B_KN) {
#pragma unroll
      for (int c = tid; c < BK * BN / 2; c += NT) {
        const int r = c / (BN / 2), cc = (c % (BN / 2)) * 2;
        const bool ok = col0 + cc < g.N;
        cp_async16(bs + r * TL::BS_KN + cc, g.B + (int64_t)(k0 + r) * g.ldb + (ok ? col0 + cc : 0), ok);
      }
    } else {
#pragma unroll
      for (int c = tid; c < BN * BK / 2; c += NT) {
        const int r = c / (BK / 2), cc = (c % (BK / 2)) * 2;
        const bool ok = col0 + r < g.N;
        cp_async16(bs + r * BS_NK + cc, g.B + (ok ? (col0 + r) : 0) * g.ldb + k0 + cc, ok);
      }
    }
  };

  double acc[MI][NJ][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int64_t kbase = (int64_t)blockIdx.z * g.kchunk;  // split-K: this CTA's K range
  const int64_t kend = gridDim.z > 1 ? (kbase + g.kchunk < g.K ? kbase + g.kchunk : g.K) : g.K;
  const int KT = (int)((kend - kbase) / BK);
#pragma unroll
  for (int s = 0; s < ST - 1; ++s) {
    if (s < KT) load_stage(s, (int)(kbase + s * BK));
    cp_commit();
  }
  for (int kt = 0; kt < KT; ++kt) {
    cp_wait<ST - 2>();
    __syncthreads();
    const int nk = kt + ST - 1;
    if (nk < KT) load_stage(nk % ST, (int)(kbase + nk * BK));
    cp_commit();
    const double *as = As + (kt % ST) * TL::A_ELEMS;
    const double *bs = Bs + (kt % ST) * BSZ;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[MI], b[NJ];
#pragma unroll
      for (int i = 0; i < MI; ++i) a[i] = as[(wm + 8 * i + fr) * AS + kk + fk];
#pragma unroll
      for (int j = 0; j < NJ; ++j)
        b[j] = B_KN ? bs[(kk + fk) * TL::BS_KN + wn + 8 * j + fr] : bs[(wn + 8 * j + fr) * BS_NK + kk + fk];
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma(acc[i][j], a[i], b[j]);
    }
  }
  cp_wait<0>();

  if (gridDim.z > 1) {  // split-K partial: raw sums, the reduction applies the epilogue
    double *w = g.ws + (int64_t)blockIdx.z * g.M * g.N;
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int64_t r = row0 + wm + 8 * i + fr;
      if (r >= g.M) continue;
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int64_t c = col0 + wn + 8 * j + 2 * fk;
        if (c >= g.N) continue;
        w[r * g.N + c] = acc[i][j][0];
        if (c + 1 < g.N) w[r * g.N + c + 1] = acc[i][j][1];
      }
    }
    return;
  }
  // epilogue
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int64_t r = row0 + wm + 8 * i + fr;
    if (r >= g.M) continue;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int64_t c = col0 + wn + 8 * j + 2 * fk;
      if (c >= g.N) continue;
      double v0 = g.alpha * acc[i][j][0], v1 = g.alpha * acc[i][j][1];
      if (g.beta != 0.0) {
        const double2 ci = *reinterpret_cast<const double2 *>(g.Cin + r * g.ldcin + c);
        v0 = v0 + g.beta * ci.x;
        v1 = v1 + g.beta * ci.y;
      }
      if (g.diag != 0.0) {
        if (r - c == g.diag_offset) v0 = v0 + g.diag;
        if (r - (c + 1) == g.diag_offset) v1 = v1 + g.diag;
      }
      if (g.tri == 0) {
        *reinterpret_cast<double2 *>(g.C + r * g.ldc + c) = make_double2(v0, v1);
      } else {
        const int64_t gr = r + g.tri_off;
        const bool k0 = g.tri == 1 ? gr >= c : gr < c;
        const bool k1 = g.tri == 1 ? gr >= c + 1 : gr < c + 1;
        if (k0) g.C[r * g.ldc + c] = v0;
        if (k1 && c + 1 < g.N) g.C[r * g.ldc + c + 1] = v1;
      }
    }
  }
}

// C = alpha sum_z ws[z] (z in order) + beta Cin (+ diag): the split-K epilogue
__global__ void splitk_reduce_kernel(const GemmArgs g, int ks) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= g.M * g.N) return;
  const int64_t r = e / g.N, c = e % g.N;
  double v = g.ws[e];
  for (int z = 1; z < ks; ++z) v += g.ws[(int64_t)z * g.M * g.N + e];
  v = g.alpha * v;
  if (g.beta != 0.0) v = v + g.beta * g.Cin[r * g.ldcin + c];
  if (g.diag != 0.0 && r - c == g.diag_offset) v = v + g.diag;
  g.C[r * g.ldc + c] = v;
}

double *g_splitk_ws = nullptr;
constexpr size_t kSplitWsDoubles = (size_t)4 << 20;  // 32 MiB

__global__ void mirror_lower_kernel(double *A, int64_t lda, int64_t n) {
  __shared__ double t[32][33];
  const int64_t bi = blockIdx.y, bj = blockIdx.x;  // tile (bi, bj) with bj > bi: upper tile <- lower tile (bj, bi)
  if (bj < bi) return;
  const int64_t r0 = bj * 32, c0 = bi * 32;  // source lower tile rows r0.., cols c0..
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = r0 + k, c = c0 + threadIdx.x;
    t[k][threadIdx.x] = (r < n && c < n) ? A[r * lda + c] : 0.0;
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = c0 + k, c = r0 + threadIdx.x;  // A[r][c] = A[c][r] for c > r
    if (r < n && c < n && c > r) A[r * lda + c] = t[threadIdx.x][k];
  }
}

}  // namespace

void launch_mirror_lower(double *A, int64_t lda, int64_t n, cudaStream_t s) {
  const unsigned nt = (unsigned)((n + 31) / 32);
  mirror_lower_kernel<<<dim3(nt, nt), dim3(32, 8), 0, s>>>(A, lda, n);
}

void dgemm_init() {
  if (!g_splitk_ws) cudaMalloc(&g_splitk_ws, kSplitWsDoubles * sizeof(double));
  cudaFuncSetAttribute(dgemm_kernel<TileL, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TileL::smem(false));
  cudaFuncSetAttribute(dgemm_kernel<TileL, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TileL::smem(true));
  cudaFuncSetAttribute(dgemm_kernel<TileS, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TileS::smem(false));
  cudaFuncSetAttribute(dgemm_kernel<TileS, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TileS::smem(true));
}

void launch_dgemm(const GemmArgs &g, bool b_kn, cudaStream_t s) {
  if (g.M <= 0 || g.N <= 0) return;
  // large contractions: fp64 emulated on the int8 tcgen05 tensor cores (ozaki.cu)
  if (ozaki_eligible(g) && launch_ozaki_gemm(g, b_kn, g.oz_slices, s) == cudaSuccess) return;
  static int sms = 0;
  if (!sms) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t tiles_l = ((g.N + 127) / 128) * ((g.M + 127) / 128);
  // (lower_only -- the Cholesky updates -- included: a small K = 64 update of ~100 128 x 128
  // tiles is one latency-bound wave; 64 x 64 tiles put 4x the CTAs on the SMs.  Each entry's
  // DMMA k order is the tile's own, so C is the same for either tile)
  if (tiles_l >= 2 * sms) {
    dim3 grid((unsigned)((g.N + 127) / 128), (unsigned)((g.M + 127) / 128));
    if (b_kn)
      dgemm_kernel<TileL, true><<<grid, TileL::THREADS, TileL::smem(true), s>>>(g);
    else
      dgemm_kernel<TileL, false><<<grid, TileL::THREADS, TileL::smem(false), s>>>(g);
  } else {  // skinny or small: 64 x 64 tiles, 4 warps (more CTAs in flight)
    const int64_t tiles_s = ((g.N + 63) / 64) * ((g.M + 63) / 64);
    // skinny products with a long K (the block solve's Q^T R, M Z: 64 output tiles on 148
    // SMs): split K over ks CTAs per tile, partials summed in a fixed order
    int ks = 1;
    if (g.N <= 256 && g.tri == 0 && !g.lower_only && g.K >= 2048 && tiles_s < sms && g_splitk_ws) {
      ks = (int)std::min<int64_t>({(2 * sms + tiles_s - 1) / tiles_s, g.K / 1024,
                                   (int64_t)(kSplitWsDoubles / (size_t)(g.M * g.N))});
      if (ks < 2) ks = 1;
    }
    GemmArgs gs = g;
    if (ks > 1) {
      gs.ws = g_splitk_ws;
      gs.kchunk = (g.K / ks + BK - 1) / BK * BK;
      ks = (int)((g.K + gs.kchunk - 1) / gs.kchunk);
    }
    dim3 grid((unsigned)((g.N + 63) / 64), (unsigned)((g.M + 63) / 64), (unsigned)ks);
    if (b_kn)
      dgemm_kernel<TileS, true><<<grid, TileS::THREADS, TileS::smem(true), s>>>(gs);
    else
      dgemm_kernel<TileS, false><<<grid, TileS::THREADS, TileS::smem(false), s>>>(gs);
    if (ks > 1)
      splitk_reduce_kernel<<<(unsigned)((g.M * g.N + 255) / 256), 256, 0, s>>>(gs, ks);
  }
}

}  // namespace laker
