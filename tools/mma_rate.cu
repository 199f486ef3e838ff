// Microbenchmark: tensor-pipe time of tcgen05.mma kind::i8 for the shapes of the exact
// tensor-core symmetric apply (csrc/symv_tc.cu).  One thread per CTA (one CTA per SM, all
// SMs) issues R blocks of 32 fully unrolled MMAs with precomputed descriptors on resident
// shared-memory operands (the issue loop is not the limit), round-robin over NACC
// accumulators; cycles per MMA from clock64 around issue + commit + wait.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2604_25138_b200/csrc tools/mma_rate.cu
#include <cuda_runtime.h>

#include <cstdio>

#include "tc_int8.cuh"

using namespace laker;

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFFu) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

template <int M, int N, int MN, int NACC, int NISS>
__global__ void __launch_bounds__(128, 1) rate(int R, long long *cyc) {
  extern __shared__ unsigned char smem_raw[];
  const uint32_t base_s = smem_u32(smem_raw);
  unsigned char *smem = smem_raw + ((1024 - (base_s & 1023)) & 1023);
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 196608);
  uint32_t *holder = reinterpret_cast<uint32_t *>(bar + 1);  // bar + 2: second issuer
  for (int i = threadIdx.x; i < 196608 / 4; i += blockDim.x) reinterpret_cast<int *>(smem)[i] = i * 2654435761u;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 2, 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tc::tmem_alloc(holder, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *holder;
  if (threadIdx.x % 32 == 0 && threadIdx.x / 32 < NISS) {
    const int w = threadIdx.x / 32;
    constexpr uint32_t id = tc::idesc_i8(M, N) | ((uint32_t)MN << 15);
    const uint64_t a0 = MN ? sdesc(smem_u32(smem), 8192, 512, 4) : sdesc(smem_u32(smem), 16, 512, 4);
    const uint64_t b0 = sdesc(smem_u32(smem + 131072), 16, 1024, 2);
    const long long c0 = clock64();
    for (int r = 0; r < R / NISS; ++r) {
#pragma unroll
      for (int k = 0; k < 32; ++k)
        tc::mma_i8(tmem + (uint32_t)(((k + w) % NACC) * (512 / NACC)), a0 + (uint64_t)(((k & 7) * 16384 + (k >> 3) * 32) >> 4),
                   b0 + (uint64_t)(((k & 3) * 32) >> 4), id, 1u);
    }
    tc::mma_commit(bar + 2 * w);
    mbar_wait(bar + 2 * w, 0);
    const long long c1 = clock64();
    if (w == 0) cyc[blockIdx.x] = c1 - c0;
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc(tmem, 512);
}

template <int M, int N, int MN, int NACC, int NISS = 1>
void run(long long *d) {
  const int R = 256;
  cudaFuncSetAttribute(rate<M, N, MN, NACC, NISS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  rate<M, N, MN, NACC, NISS><<<148, 128, 200 * 1024>>>(R, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148.0;
  printf("{\"M\": %d, \"N\": %d, \"a_mn_major\": %d, \"accumulators\": %d, \"issuers\": %d, \"cycles_per_mma\": %.2f, "
         "\"err\": \"%s\"}\n", M, N, MN, NACC, NISS, avg / (R * 32.0), cudaGetErrorString(e));
}

int main() {
  long long *d;
  cudaMalloc(&d, 148 * sizeof(long long));
  run<128, 16, 0, 1>(d);
  run<128, 16, 0, 8>(d);
  run<128, 32, 0, 8>(d);
  run<128, 64, 0, 8>(d);
  run<128, 128, 0, 4>(d);
  run<128, 256, 0, 2>(d);
  run<64, 16, 1, 8>(d);
  run<64, 64, 1, 8>(d);
  run<128, 16, 1, 8>(d);
  run<128, 64, 1, 8>(d);
  run<128, 16, 1, 1>(d);
  run<128, 16, 0, 8, 2>(d);
  run<128, 16, 1, 8, 2>(d);
  run<128, 64, 0, 8, 2>(d);
  return 0;
}
