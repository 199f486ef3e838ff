// Microbenchmark: single-thread issue cost of tcgen05.mma kind::i8 (M = 128, N = 16) with
// descriptors computed at run time as in csrc/symv_tc.cu (ring slot base + constant
// offsets, accumulator column from a TMEM base read from shared memory), for two issue
// styles:
//   lane0: the loop runs in `if (lane == 0)` (the compiler moves each operand to uniform
//          registers with an ELECT / R2UR.BROADCAST sequence per MMA);
//   warp:  all 32 lanes run the loop; the MMA asm block elects one lane (elect.sync);
//   tile:  as warp, with the per-slice pattern of the apply: 4 row MMAs (K-major A) + 4
//          column MMAs (MN-major A spanning two halves) into separate accumulators, then a
//          commit to a ring mbarrier (variants: no commit; all K-major).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2604_25138_b200/csrc tools/mma_issue.cu
#include <cuda_runtime.h>

#include <cstdio>

#include "tc_int8.cuh"

using namespace laker;

__device__ __forceinline__ void mma_i8_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void commit_elect(uint64_t *bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ uint64_t sdesc_mn(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFFu) >> 4);
  d |= (uint64_t)(8192 >> 4) << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}

template <int STYLE>
__global__ void __launch_bounds__(128, 1) issue(int R, long long *cyc) {
  extern __shared__ unsigned char smem_raw[];
  const uint32_t base_s = smem_u32(smem_raw);
  unsigned char *smem = smem_raw + ((1024 - (base_s & 1023)) & 1023);
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 200704);  // [0] done, [8..20) ring
  uint32_t *holder = reinterpret_cast<uint32_t *>(bar + 1);
  for (int i = threadIdx.x; i < 200704 / 4; i += blockDim.x) reinterpret_cast<int *>(smem)[i] = i * 2654435761u;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tc::tmem_alloc(holder, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *holder;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr uint32_t idr = tc::idesc_i8(128, 16);
  long long c0 = 0;
  if (STYLE >= 2 && warp == 0) {
    // per-slice pattern of csrc/symv_tc.cu; STYLE 2: as the kernel, 3: no commits, 4: all K-major
    if (threadIdx.x == 0) {
      for (int k = 0; k < 12; ++k) mbar_init(bar + 8 + k, 1);
      fence_mbar_init();
    }
    __syncwarp();
    constexpr uint32_t idc = tc::idesc_i8(128, 16) | (STYLE == 4 ? 0u : (1u << 15));
    const uint64_t dK0 = tc::sdesc_k_sw64(smem_u32(smem));
    const uint64_t dKt0 = STYLE == 4 ? dK0 : sdesc_mn(smem_u32(smem));
    const uint64_t dX0 = tc::sdesc_k_sw128(smem_u32(smem + 196608));
    c0 = clock64();
    int slot = 0;
    for (int r = 0; r < R; ++r) {
      const uint32_t trow = tmem + (uint32_t)((r & 1) * 128), tcol = tmem + 256 + (uint32_t)((r & 1) * 128);
#pragma unroll 1
      for (int s = 0; s < 8; ++s) {
        const uint64_t so = (uint64_t)((slot * 16384) >> 4);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_i8_elect(trow + 16 * s, dK0 + so + (uint64_t)(((kk >> 1) * 8192 + (kk & 1) * 32) >> 4),
                       dX0 + (uint64_t)((kk * 32) >> 4), idr, kk > 0 ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_i8_elect(tcol + 16 * s, dKt0 + so + (uint64_t)((kk * 2048) >> 4), dX0 + 128 + (uint64_t)((kk * 32) >> 4),
                       idc, kk > 0 ? 1u : 0u);
        if (STYLE != 3) commit_elect(bar + 8 + slot);
        if (++slot == 12) slot = 0;
      }
    }
    commit_elect(bar);
    mbar_wait(bar, 0);
    if (lane == 0) cyc[blockIdx.x] = clock64() - c0;
  } else if (warp == 0 && (STYLE == 1 || lane == 0)) {
    const uint64_t dK0 = tc::sdesc_k_sw64(smem_u32(smem));
    const uint64_t dX0 = tc::sdesc_k_sw128(smem_u32(smem + 196608));
    c0 = clock64();
    int sc = 0;
    for (int r = 0; r < R; ++r) {
      const uint32_t trow = tmem + (uint32_t)((r & 1) * 128);
#pragma unroll 1
      for (int s = 0; s < 8; ++s, ++sc) {
        const int slot = sc % 12;
        const uint64_t so = (uint64_t)((slot * 16384) >> 4);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t ad = dK0 + so + (uint64_t)((((kk & 3) >> 1) * 8192 + (kk & 1) * 32) >> 4);
          const uint64_t bd = dX0 + (uint64_t)(((kk & 3) * 32) >> 4);
          if (STYLE == 1)
            mma_i8_elect(trow + 16 * s, ad, bd, idr, kk > 0 ? 1u : 0u);
          else
            tc::mma_i8(trow + 16 * s, ad, bd, idr, kk > 0 ? 1u : 0u);
        }
      }
    }
    if (STYLE == 1)
      commit_elect(bar);
    else
      tc::mma_commit(bar);
    mbar_wait(bar, 0);
    if (lane == 0) cyc[blockIdx.x] = clock64() - c0;
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc(tmem, 512);
}

template <int STYLE>
void run(long long *d) {
  const int R = 64;
  cudaFuncSetAttribute(issue<STYLE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200704 + 2048);
  issue<STYLE><<<148, 128, 200704 + 2048>>>(R, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148.0;
  const char *names[] = {"lane0", "warp", "tile", "tile_nocommit", "tile_all_kmajor"};
  printf("{\"style\": \"%s\", \"cycles_per_mma\": %.2f, \"err\": \"%s\"}\n", names[STYLE], avg / (R * 64.0),
         cudaGetErrorString(e));
}

int main() {
  long long *d;
  cudaMalloc(&d, 148 * sizeof(long long));
  run<0>(d);
  run<1>(d);
  run<2>(d);
  run<3>(d);
  run<4>(d);
  return 0;
}
