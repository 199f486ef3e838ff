// Probe: may a tcgen05.mma kind::i8 accumulator start at an arbitrary TMEM column?  The
// exact tensor-core apply could then add slice s's products into columns shifted by s
// (level L = s + t in one column).  D = A B^T, M = 128, N = 16, K = 32, written at column
// offset c (c = 0..9, 16) after zeroing 64 columns; checks every column against the host.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2604_25138_b200/csrc tools/mma_dshift_test.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_int8.cuh"

using namespace laker;

__global__ void __launch_bounds__(128, 1) probe(const int8_t *gA, const int8_t *gB, int coff, int32_t *D) {
  extern __shared__ unsigned char smem_raw[];
  const uint32_t base_s = smem_u32(smem_raw);
  unsigned char *smem = smem_raw + ((1024 - (base_s & 1023)) & 1023);
  unsigned char *sA = smem;          // 128 rows x 32 B, SWIZZLE_NONE K-major core matrices
  unsigned char *sB = smem + 4096;   // 16 rows x 32 B
  uint64_t *mbar = reinterpret_cast<uint64_t *>(smem + 8192);
  uint32_t *holder = reinterpret_cast<uint32_t *>(mbar + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // canonical no-swizzle K-major layout: core matrix (8 rows x 16 B) at ((r / 8) * 2 + k / 16) * 128,
  // row r % 8 at 16 B stride
  for (int e = threadIdx.x; e < 128 * 32; e += 128) {
    const int r = e / 32, k = e % 32;
    sA[((r / 8) * 2 + k / 16) * 128 + (r % 8) * 16 + k % 16] = gA[e];
  }
  for (int e = threadIdx.x; e < 16 * 32; e += 128) {
    const int r = e / 32, k = e % 32;
    sB[((r / 8) * 2 + k / 16) * 128 + (r % 8) * 16 + k % 16] = gB[e];
  }
  if (threadIdx.x == 0) {
    mbar_init(mbar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(holder, 128);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *holder;
  {  // zero columns 0..63 of every lane
    uint32_t z[16] = {0};
    for (int c = 0; c < 64; c += 16)
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
          "%15, %16};" ::"r"(tmem + c + ((uint32_t)(warp * 32) << 16)),
          "r"(z[0]), "r"(z[1]), "r"(z[2]), "r"(z[3]), "r"(z[4]), "r"(z[5]), "r"(z[6]), "r"(z[7]), "r"(z[8]), "r"(z[9]),
          "r"(z[10]), "r"(z[11]), "r"(z[12]), "r"(z[13]), "r"(z[14]), "r"(z[15]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (threadIdx.x == 0) {
    // no-swizzle K-major: LBO = stride between the two K core matrices (128 B), SBO = stride
    // between 8-row groups (256 B)
    auto desc = [](uint32_t addr) {
      uint64_t d = 0;
      d |= (uint64_t)((addr & 0x3FFFFu) >> 4);
      d |= (uint64_t)(128 >> 4) << 16;
      d |= (uint64_t)(256 >> 4) << 32;
      d |= (uint64_t)1 << 46;
      return d;
    };
    tc::mma_i8(tmem + (uint32_t)coff, desc(smem_u32(sA)), desc(smem_u32(sB)), tc::idesc_i8(128, 16), 1u);
    tc::mma_commit(mbar);
  }
  __syncthreads();
  mbar_wait(mbar, 0);
  tc::fence_after();
  for (int c = 0; c < 64; c += 16) {
    uint32_t v[16];
    tc::tmem_ld16(tmem + c + ((uint32_t)(warp * 32) << 16), v);
    tc::tmem_ld_wait();
    for (int t = 0; t < 16; ++t) D[(warp * 32 + lane) * 64 + c + t] = (int32_t)v[t];
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 128);
}

int main() {
  std::vector<int8_t> A(128 * 32), B(16 * 32);
  srand(5);
  for (auto &v : A) v = (int8_t)(rand() % 129 - 64);
  for (auto &v : B) v = (int8_t)(rand() % 129 - 64);
  int8_t *dA, *dB;
  int32_t *dD;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dD, 128 * 64 * 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  int offs[] = {0, 1, 2, 3, 4, 5, 7, 8, 9, 16};
  for (int coff : offs) {
    probe<<<1, 128, 16384>>>(dA, dB, coff, dD);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<int> G(128 * 64);
    cudaMemcpy(G.data(), dD, G.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < 128; ++i)
      for (int c = 0; c < 64; ++c) {
        int ref = 0;
        const int t = c - coff;
        if (t >= 0 && t < 16)
          for (int k = 0; k < 32; ++k) ref += A[i * 32 + k] * B[t * 32 + k];
        bad += G[i * 64 + c] != ref;
      }
    printf("{\"column_offset\": %d, \"err\": \"%s\", \"bad\": %d}\n", coff, cudaGetErrorString(e), bad);
    if (e != cudaSuccess) break;
  }
  return 0;
}
