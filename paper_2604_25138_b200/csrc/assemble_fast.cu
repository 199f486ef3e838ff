// FAST-mode kernel assembly: the QK^T contraction of K = exp(scale E E^T)
// (Eq. sc-exp-kernel) on the fp64 tensor cores (mma.sync
// m8n8k4 .f64 -> SASS DMMA; tcgen05 has no fp64 kind), with the
// scale + exp epilogue fused.  Entries are within ~1 ulp of the EXACT mode's
// correctly rounded ones (tests/test_gpu_assemble.py).
//
// 64 x 64 tile per CTA (4 warps x 32 x 32, 16 DMMA accumulators per warp), E
// staged through shared memory in 32-wide k chunks (row stride 36 doubles:
// conflict-free fragment loads), tile written through a shared-memory
// transpose so both K[I,J] and its mirror K[J,I] are stored coalesced.
#include "laker_internal.h"

namespace laker {
namespace {

constexpr int kT = 64;
constexpr int kKC = 32;
constexpr int kS = 36;  // smem row stride (doubles)

__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(128) assemble_fast_kernel(const double *__restrict__ E, int64_t n,
                                                            int d, double scale, int64_t r0,
                                                            int64_t r1, double *__restrict__ K,
                                                            int64_t ld, int sym,
                                                            unsigned long long *flags) {
  constexpr int kBuf = (2 * kT * kS > kT * (kT + 1)) ? 2 * kT * kS : kT * (kT + 1);
  __shared__ double buf[kBuf];  // E tiles during the k loop, then the output tile
  double *Ei = buf;
  double *Ej = buf + kT * kS;
  if (sym && blockIdx.x < blockIdx.y) return;
  const int64_t I0 = sym ? (int64_t)blockIdx.y * kT : r0 + (int64_t)blockIdx.y * kT;
  const int64_t J0 = (int64_t)blockIdx.x * kT;
  const int64_t rowEnd = sym ? n : r1;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wr = (warp >> 1) * 32, wc = (warp & 1) * 32;
  const int fr = lane >> 2, fk = lane & 3;

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int k0 = 0; k0 < d; k0 += kKC) {
    const int kc = min(kKC, d - k0);
    for (int idx = tid; idx < kT * kKC; idx += 128) {
      const int r = idx / kKC, c = idx % kKC;
      const int64_t gi = I0 + r, gj = J0 + r;
      Ei[r * kS + c] = (gi < rowEnd && c < kc) ? E[gi * d + k0 + c] : 0.0;
      Ej[r * kS + c] = (gj < n && c < kc) ? E[gj * d + k0 + c] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kKC; kk += 4) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = Ei[(wr + 8 * i + fr) * kS + kk + fk];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Ej[(wc + 8 * j + fr) * kS + kk + fk];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j], a[i], b[j]);
    }
    __syncthreads();
  }

  // epilogue: exp(scale * dot) into the shared tile
  double(*tr)[kT + 1] = reinterpret_cast<double(*)[kT + 1]>(buf);
  unsigned int ovf = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double arg = scale * acc[i][j][h];
        ovf += arg > 709.782712893383973096;
        tr[wr + 8 * i + fr][wc + 8 * j + 2 * fk + h] = exp(arg);
      }
  if (ovf) atomicAdd(&flags[1], (unsigned long long)ovf);
  __syncthreads();
  const int64_t rowBase = sym ? 0 : r0;
  const int cc = tid & 63;
  for (int rr = tid >> 6; rr < kT; rr += 2) {
    const int64_t gi = I0 + rr, gj = J0 + cc;
    if (gi < rowEnd && gj < n) K[(gi - rowBase) * ld + gj] = tr[rr][cc];
  }
  if (sym && blockIdx.x != blockIdx.y) {
    for (int rr = tid >> 6; rr < kT; rr += 2) {
      const int64_t gi = J0 + rr, gj = I0 + cc;
      if (gi < n && gj < n) K[gi * ld + gj] = tr[cc][rr];
    }
  }
}

}  // namespace

void launch_assemble_fast(const double *E, int64_t n, int32_t d, double scale, int64_t r0,
                          int64_t r1, double *K, int64_t ld, unsigned long long *flags,
                          cudaStream_t s) {
  const bool sym = (r0 == 0 && r1 == n);
  const unsigned ntc = (unsigned)((n + kT - 1) / kT);
  const unsigned ntr = (unsigned)((r1 - r0 + kT - 1) / kT);
  assemble_fast_kernel<<<dim3(ntc, sym ? ntc : ntr), 128, 0, s>>>(E, n, d, scale, r0, r1, K, ld,
                                                                   sym ? 1 : 0, flags);
}

}  // namespace laker
