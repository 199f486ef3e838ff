// FAST-mode kernel matvec, second generation (d <= 64): the on-the-fly operator
// q = lambda p + K p (row a11; the symmetric form of SURVEY §8(f)
// NEXT-3), the radio-map prediction out = exp(scale Eq E^T) alpha (P:164-172,
// row a12) and the FAST assembly (row a1), all with the QK^T on the tcgen05
// tensor cores as fp64 emulated by S int8 digit slices (Ozaki scheme, ozaki.cu).
//
// Changes from otf_tc.cu (measured there: XU pipe saturated by the int -> fp64
// conversions, tensor and fp64 pipes ~27% busy, 2 TMEM level buffers):
//  * slices are K = 64 wide (d <= 64) with 64-byte swizzled rows: no zero half
//    in every MMA, half the shared memory;
//  * 4 TMEM level buffers (512 columns): the MMAs of the next tile's first four
//    levels overlap the exp phase of the current one;
//  * two adjacent digit levels are combined exactly in int32 (v_{h-1} 2^7 + v_h,
//    |v| <= 7 * 64 * 64^2 < 2^21): 4 int -> fp64 conversions per entry, not 7
//    (the XU pipe that runs them is then ~20% busy instead of saturated);
//  * exp by a 16-entry table of 2^(j/16) and a degree-7 polynomial (12 fp64 ops);
//  * per-column factors {scale 2^(e_j), w_j} read as one broadcast 16-byte load;
//  * kSym: the tiles of the block upper triangle over a persistent grid (tri.cuh):
//    each off-diagonal tile gives its rows K_IJ w_J and, by a shuffle
//    reduce-scatter over the tile rows, its columns K_IJ^T w_I -- half the QK^T
//    and half the exps of the full square.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "laker_internal.h"
#include "tc_int8.cuh"
#include "tri.cuh"

namespace laker {
bool make_tmap_s8_k64(CUtensorMap *tm, const int8_t *base, int64_t rows, int64_t K, int64_t ld, int box_rows);
namespace {

constexpr int kQM = 128;                  // tile rows = tile columns
constexpr int kQK = 64;                   // slice width (bytes per row of a chunk)
constexpr int kQSmax = 7;
constexpr uint32_t kQChunk = kQM * kQK;   // 8 KiB
constexpr int kQBufs = 4;                 // TMEM level buffers of 128 columns
constexpr int kQEpiWarps = 16;
constexpr int kQThreads = (2 + kQEpiWarps) * 32;
constexpr size_t kQRedOff = 2 * kQSmax * kQChunk;          // red[4][128] pairs
constexpr size_t kQCredOff = kQRedOff + 4 * kQM * 16;       // cred[2][4][128] pairs
constexpr size_t kQTabOff = kQCredOff + 2 * 4 * kQM * 16;   // exp table [16] doubles
constexpr size_t kQBarOff = kQTabOff + 16 * 8;
constexpr size_t kQSmem = 1024 + kQBarOff + 256;

enum { kRectSum = 0, kSym = 2 };

struct Q2Args {
  SymvArgs t;           // kSym: partition and partial buffers
  int64_t a0, m, n;     // rect: query rows [a0, a0 + m) of the A slices; n points
  int S;
  const int32_t *ea;    // A row exponents
  const double2 *cf;    // per point column {scale 2^(e_j), w_j}; zero past n (nJ * 128 entries)
  const double *wrow;   // kSym: the weights of the rows (= w)
  double lambda;
  const double *xdiag;
  double *out;          // kRectSum
  const int32_t *done;
};

__constant__ double c_exp2_16[16] = {
    0x1.0000000000000p+0, 0x1.0b5586cf9890fp+0, 0x1.172b83c7d517bp+0, 0x1.2387a6e756238p+0,
    0x1.306fe0a31b715p+0, 0x1.3dea64c123422p+0, 0x1.4bfdad5362a27p+0, 0x1.5ab07dd485429p+0,
    0x1.6a09e667f3bcdp+0, 0x1.7a11473eb0187p+0, 0x1.8ace5422aa0dbp+0, 0x1.9c49182a3f090p+0,
    0x1.ae89f995ad3adp+0, 0x1.c199bdd85529cp+0, 0x1.d5818dcfba487p+0, 0x1.ea4afa2a490dap+0};

// exp(x), |x| < 700 (guaranteed by the Cauchy-Schwarz guard at assembly): x = (16 e + j)
// ln2/16 + r, |r| <= ln2/32, exp(x) = 2^e 2^(j/16) P7(r); <= 2 ulp, no special cases.
__device__ __forceinline__ double exp_tab(double x, const double *tab) {
  const double t = fma(x, 0x1.71547652b82fep+4, 0x1.8p52);  // 1.5 2^52 + rint(16 x / ln2)
  const double kd = t - 0x1.8p52;
  const int k = __double2loint(t);
  double r = fma(-kd, 0x1.62e42fee00000p-5, x);  // ln2/16 = hi + lo, kd hi exact
  r = fma(-kd, 0x1.a39ef35793c76p-37, r);
  double p = 1.0 / 5040.0;
  p = fma(p, r, 1.0 / 720.0);
  p = fma(p, r, 1.0 / 120.0);
  p = fma(p, r, 1.0 / 24.0);
  p = fma(p, r, 1.0 / 6.0);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const double tj = tab[k & 15];
  const double sc = __hiloint2double(__double2hiint(tj) + ((k >> 4) << 20), __double2loint(tj));
  return p * sc;
}

__device__ __forceinline__ double pow2d(int k) {
  return (k >= -1022 && k <= 1023) ? __longlong_as_double((long long)(k + 1023) << 52) : scalbn(1.0, k);
}

// broadcast 16-byte load kept in program order (the compiler would otherwise hoist all
// 32 of an unrolled loop and spill: 96 registers per thread at 18 warps)
__device__ __forceinline__ double2 ld_cf(const double2 *p) {
  double2 v;
  asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <int KIND>
__global__ void __launch_bounds__(kQThreads, 1)
    otf_q2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const Q2Args f) {
  if (f.done != nullptr && *(volatile const int32_t *)f.done) return;
  const int64_t nJ = (f.n + kQM - 1) / kQM;
  int64_t t0, t1;
  if (KIND == kSym) {
    t0 = f.t.T * blockIdx.x / gridDim.x;
    t1 = f.t.T * (blockIdx.x + 1) / gridDim.x;
  } else {
    t0 = (int64_t)blockIdx.x * nJ;
    t1 = t0 + nJ;
  }
  if (t0 >= t1) return;
  extern __shared__ unsigned char smem_raw[];
  const uint32_t base_s = smem_u32(smem_raw);
  unsigned char *smem = smem_raw + ((1024 - (base_s & 1023)) & 1023);
  unsigned char *sA = smem;
  unsigned char *sB = smem + kQSmax * kQChunk;
  dd_pair *red = reinterpret_cast<dd_pair *>(smem + kQRedOff);
  dd_pair *cred = reinterpret_cast<dd_pair *>(smem + kQCredOff);
  double *tab = reinterpret_cast<double *>(smem + kQTabOff);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + kQBarOff);  // [7]
  uint64_t *empty = full + kQSmax;                                  // [7]
  uint64_t *tfull = empty + kQSmax;                                 // [4]
  uint64_t *tempty = tfull + kQBufs;                                // [4]
  uint64_t *afull = tempty + kQBufs;
  uint64_t *aempty = afull + 1;
  uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(aempty + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = f.S;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kQSmax; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < kQBufs; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kQEpiWarps);
    }
    mbar_init(afull, 1);
    mbar_init(aempty, 1);
    fence_mbar_init();
  }
  if (threadIdx.x >= 64 && threadIdx.x < 80) tab[threadIdx.x - 64] = c_exp2_16[threadIdx.x - 64];
  if (warp == 1) tc::tmem_alloc(tmem_holder, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_holder;

  // tile t -> (I, J): kSym walks the block upper triangle (J >= I), rect one query block
  int I = KIND == kSym ? find_block_row(f.t.toff, f.t.nb, t0) : (int)blockIdx.x;
  int64_t rbeg = KIND == kSym ? f.t.toff[I] : t0;
  int64_t rend = KIND == kSym ? f.t.toff[I + 1] : t1;
  const int64_t arow0 = KIND == kSym ? 0 : f.a0;

  if (warp == 0) {
    if (lane == 0) {
      int aload = 0;
      for (int64_t t = t0; t < t1; ++t) {
        bool newI = (t == t0);
        while (t >= rend) {
          ++I;
          rbeg = rend;
          rend = f.t.toff[I + 1];
          newI = true;
        }
        const int64_t J = KIND == kSym ? I + (t - rbeg) : t - t0;
        if (newI) {
          if (aload > 0) mbar_wait_sleep(aempty, (uint32_t)((aload - 1) & 1));
          mbar_arrive_expect_tx(afull, (uint32_t)S * kQChunk);
          for (int c = 0; c < S; ++c)
            tc::tma_load_2d(sA + c * kQChunk, &tmA, c * kQK, (int32_t)(arow0 + (int64_t)I * kQM), afull);
          ++aload;
        }
        const int64_t lt = t - t0;
        for (int s = S - 1; s >= 0; --s) {
          if (lt > 0) mbar_wait_sleep(&empty[s], (uint32_t)((lt - 1) & 1));
          mbar_arrive_expect_tx(&full[s], kQChunk);
          tc::tma_load_2d(sB + s * kQChunk, &tmB, s * kQK, (int32_t)(J * kQM), &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_i8(kQM, kQM);
      int aload = 0;
      int64_t job = 0;
      for (int64_t t = t0; t < t1; ++t) {
        bool newI = (t == t0);
        while (t >= rend) {
          ++I;
          rbeg = rend;
          rend = f.t.toff[I + 1];
          newI = true;
        }
        if (newI) {
          if (aload > 0) tc::mma_commit(aempty);  // every MMA on the previous query block issued
          mbar_wait_sleep(afull, (uint32_t)(aload & 1));
          ++aload;
        }
        const int64_t lt = t - t0;
        for (int h = S - 1; h >= 0; --h, ++job) {
          const int b = (int)(job & (kQBufs - 1));
          if (job >= kQBufs) mbar_wait_sleep(&tempty[b], (uint32_t)(((job / kQBufs) - 1) & 1));
          tc::fence_after();
          const uint32_t td = tmem + (uint32_t)(b * kQM);
          for (int c = 0; c <= h; ++c) {
            const int tt = h - c;
            mbar_wait_sleep(&full[tt], (uint32_t)(lt & 1));
            tc::fence_after();
            const uint32_t a0s = smem_u32(sA + c * kQChunk), b0s = smem_u32(sB + tt * kQChunk);
#pragma unroll
            for (int kk = 0; kk < kQK / 32; ++kk)
              tc::mma_i8(td, tc::sdesc_k_sw64(a0s + kk * 32), tc::sdesc_k_sw64(b0s + kk * 32), idesc,
                         (c > 0 || kk > 0) ? 1u : 0u);
          }
          tc::mma_commit(&tfull[b]);
          tc::mma_commit(&empty[h]);  // slot h: no later level of this tile reads it
        }
      }
    }
  } else {
    const int q = warp & 3, qt = (warp - 2) >> 2;  // TMEM lane quadrant, column quarter
    const int rl = q * 32 + lane;
    const int64_t rows = KIND == kSym ? f.n : f.m;
    int64_t row = 0;
    bool rok = false;
    int ea = 0;
    double wr = 0.0;
    // compensated sums (Dot2: TwoProd + TwoSum, pairs combined by TwoSum): the operator's
    // rounding error stays ~u |K p| instead of ~u |K| |p|, which in the late CG iterations
    // (|K| |p| / |K p| up to ~kappa) cost +38% Jacobi iterations at the C5 regime (n = 8192,
    // lambda = 1e-5) with plain fp64 sums; the entries themselves stay FAST (tcgen05 + exp_tab)
    dd_pair rsum = {0.0, 0.0};
    int64_t job = 0;
    int cbuf = 0;
    auto flush_rows = [&](int Iblk) {
      // the four column quarters' row sums of block-row Iblk, in quarter order
      red[qt * kQM + rl] = rsum;
      named_bar(1, kQEpiWarps * 32);
      if (qt == 0) {
        dd_pair v = red[rl];
        pair_add(v, red[kQM + rl]);
        pair_add(v, red[2 * kQM + rl]);
        pair_add(v, red[3 * kQM + rl]);
        if (KIND == kSym) {
          const int s = (int)blockIdx.x - f.t.segfirst[Iblk];
          f.t.rowpart[((int64_t)Iblk * f.t.maxseg + s) * kQM + rl] = v;
        } else if (rok) {
          if (f.lambda != 0.0) dot2_step(v, f.lambda, f.xdiag[row]);
          f.out[row] = pair_value(v);
        }
      }
      named_bar(1, kQEpiWarps * 32);
      rsum = dd_pair{0.0, 0.0};
    };
    for (int64_t t = t0; t < t1; ++t) {
      bool newI = (t == t0);
      while (t >= rend) {
        flush_rows(I);
        ++I;
        rbeg = rend;
        rend = f.t.toff[I + 1];
        newI = true;
      }
      const int64_t J = KIND == kSym ? I + (t - rbeg) : t - t0;
      if (newI) {
        row = (int64_t)I * kQM + rl;
        rok = row < rows;
        ea = rok ? f.ea[arow0 + row] : 0;
        if (KIND == kSym) wr = rok ? f.wrow[row] : 0.0;
      }
      // ---- digit levels S-1 .. 0, two at a time: v_{h-1} 2^7 + v_h exact in int32
      double acc[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] = 0.0;
      for (int h = S - 1; h >= 0; h -= 2) {
        const bool two = h >= 1;
        const int b0 = (int)(job & (kQBufs - 1)), b1 = (int)((job + 1) & (kQBufs - 1));
        mbar_wait_sleep(&tfull[b0], (uint32_t)((job / kQBufs) & 1));
        if (two) mbar_wait_sleep(&tfull[b1], (uint32_t)(((job + 1) / kQBufs) & 1));
        tc::fence_after();
        const double sc = pow2d(ea - 12 - 7 * h);  // 2^(e_row) folded into the level scale
#pragma unroll
        for (int hh = 0; hh < 4; ++hh) {  // 8 columns at a time (96 registers per thread at 18 warps)
          uint32_t v0[8], v1[8];
          const uint32_t col = (uint32_t)(qt * 32 + hh * 8) + ((uint32_t)(q * 32) << 16);
          tc::tmem_ld8(tmem + (uint32_t)(b0 * kQM) + col, v0);
          if (two) tc::tmem_ld8(tmem + (uint32_t)(b1 * kQM) + col, v1);
          tc::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int32_t w = two ? (int32_t)v1[j] * 128 + (int32_t)v0[j] : (int32_t)v0[j];
            acc[hh * 8 + j] = fma((double)w, sc, acc[hh * 8 + j]);
          }
        }
        tc::fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&tempty[b0]);
          if (two) mbar_arrive(&tempty[b1]);
        }
        job += two ? 2 : 1;
      }
      // ---- entries exp(scale 2^(e_i + e_j) acc), row sums, column sums
      const int64_t cb = J * kQM + qt * 32;
      const bool cols = KIND == kSym && J != I;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const double2 cf = ld_cf(f.cf + cb + j);
        const double kv = exp_tab(acc[j] * cf.x, tab);
        dot2_step(rsum, kv, cf.y);
        acc[j] = kv;
      }
      if (cols) {
        // reduce-scatter over the warp's 32 rows of the exact products kv w_row (TwoProd
        // pairs, combined by TwoSum): lane l ends with column qt*32 + l
        dd_pair pr[16];
        {
          const bool up = (lane & 16) != 0;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            dd_pair lo, hi;
            two_prod(acc[i], wr, lo.s, lo.c);
            two_prod(acc[i + 16], wr, hi.s, hi.c);
            const dd_pair snd = up ? lo : hi;
            dd_pair rcv;
            rcv.s = __shfl_xor_sync(0xffffffffu, snd.s, 16);
            rcv.c = __shfl_xor_sync(0xffffffffu, snd.c, 16);
            pr[i] = up ? hi : lo;
            pair_add(pr[i], rcv);
          }
        }
#pragma unroll
        for (int off = 8; off >= 1; off >>= 1) {
          const bool up = (lane & off) != 0;
#pragma unroll
          for (int i = 0; i < off; ++i) {
            const dd_pair lo = pr[i], hi = pr[i + off];
            const dd_pair snd = up ? lo : hi;
            dd_pair rcv;
            rcv.s = __shfl_xor_sync(0xffffffffu, snd.s, off);
            rcv.c = __shfl_xor_sync(0xffffffffu, snd.c, off);
            pr[i] = up ? hi : lo;
            pair_add(pr[i], rcv);
          }
        }
        dd_pair *cr = cred + cbuf * 4 * kQM;
        cr[q * kQM + qt * 32 + lane] = pr[0];
        named_bar(2 + qt, 128);  // the four lane quadrants of this column quarter
        if (q == 0) {
          const int c = qt * 32 + lane;
          dd_pair v = cr[c];
          pair_add(v, cr[kQM + c]);
          pair_add(v, cr[2 * kQM + c]);
          pair_add(v, cr[3 * kQM + c]);
          f.t.colpart[(int64_t)I * f.t.ldcp + J * kQM + c] = v;
        }
        cbuf ^= 1;
      }
    }
    flush_rows(I);
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

// cf[j] = {scale 2^(e_j), w_j} for j < n, {0, 0} up to the padded length
__global__ void colfac_kernel(const int32_t *__restrict__ eb, const double *__restrict__ w, int64_t n, int64_t np,
                              double scale, double2 *__restrict__ cf) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= np) return;
  cf[j] = j < n ? make_double2(scale * pow2d(eb[j]), w ? w[j] : 0.0) : make_double2(0.0, 0.0);
}

template <int KIND>
cudaError_t launch_q2(const OzSlices &A, const OzSlices &B, const Q2Args &f, unsigned grid, cudaStream_t s) {
  CUtensorMap ta, tb;
  const int64_t ld = (int64_t)A.S * A.Kp;
  if (!make_tmap_s8_k64(&ta, A.s, A.rows, ld, ld, kQM) || !make_tmap_s8_k64(&tb, B.s, B.rows, ld, ld, kQM))
    return cudaErrorInvalidValue;
  otf_q2_kernel<KIND><<<grid, kQThreads, kQSmem, s>>>(ta, tb, f);
  return cudaGetLastError();
}

}  // namespace

void otf_tc2_init() {
  cudaFuncSetAttribute(otf_q2_kernel<kRectSum>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kQSmem);
  cudaFuncSetAttribute(otf_q2_kernel<kSym>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kQSmem);
}

bool otf_tc2_eligible(const OzSlices &A, const OzSlices &B) {
  return A.Kp == kQK && B.Kp == kQK && A.S == B.S && A.S <= kQSmax && A.S >= 1;
}

// per-column factors, padded to whole 128-column tiles (buffer: >= ceil(n/128)*128 double2)
void launch_colfac(const OzSlices &B, int64_t n, double scale, const double *w, double2 *cf, cudaStream_t s) {
  const int64_t np = (n + kQM - 1) / kQM * kQM;
  colfac_kernel<<<(unsigned)((np + 255) / 256), 256, 0, s>>>(B.e, w, n, np, scale, cf);
}

// out[a] = [lambda xdiag[a] +] sum_j exp(scale <eq_a, e_j>) w_j, a in [0, m): query rows a0.. of A
cudaError_t launch_otf_tc2_rect(const OzSlices &A, int64_t a0, int64_t m, const OzSlices &B, int64_t n, double scale,
                                const double *w, double2 *cf, double lambda, const double *xdiag, double *out,
                                const int32_t *done, cudaStream_t s) {
  if (m <= 0) return cudaSuccess;
  launch_colfac(B, n, scale, w, cf, s);
  Q2Args f{};
  f.a0 = a0;
  f.m = m;
  f.n = n;
  f.S = A.S;
  f.ea = A.e;
  f.cf = cf;
  f.lambda = lambda;
  f.xdiag = xdiag;
  f.out = out;
  f.done = done;
  return launch_q2<kRectSum>(A, B, f, (unsigned)((m + kQM - 1) / kQM), s);
}


// symmetric operator: tiles of the plan (BR = TC = 128) -> rowpart / colpart of ta
cudaError_t launch_otf_tc2_sym(const OzSlices &E, int64_t n, double scale, const double *w, double2 *cf,
                               const SymvArgs &ta, int grid, cudaStream_t s) {
  launch_colfac(E, n, scale, w, cf, s);
  Q2Args f{};
  f.t = ta;
  f.n = n;
  f.m = n;
  f.S = E.S;
  f.ea = E.e;
  f.cf = cf;
  f.wrow = w;
  f.done = ta.state ? &ta.state->done : nullptr;
  return launch_q2<kSym>(E, E, f, (unsigned)grid, s);
}

}  // namespace laker
