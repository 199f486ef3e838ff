// Probe for the 128 x 128 tile of the exact tensor-core symmetric apply (csrc/symv_tc.cu):
// a row-major int8 tile of 128 rows i x 128 columns j held as two SWIZZLE_64B halves
// (columns 0..63 at sT, 64..127 at sT + 8192) feeds
//   D1[i][t] = sum_j T[i][j] X1[t][j]   (M = 128, N = 16, K = 128: K-major A, two halves)
//   D2[j][t] = sum_i T[i][j] X2[t][i]   (M = 128, N = 16, K = 128: MN-major A spanning both
//                                        halves, LBO = the half stride, SBO = 512)
// X1 and X2 are 16 x 128 int8 (SWIZZLE_128B).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2604_25138_b200/csrc tools/mma_mn128_test.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

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

struct Params {
  uint32_t lbo2, sbo2;
};

__global__ void __launch_bounds__(128, 1) probe(const __grid_constant__ CUtensorMap tmT,
                                                const __grid_constant__ CUtensorMap tmX, int32_t *D1, int32_t *D2,
                                                Params pr) {
  extern __shared__ unsigned char smem_raw[];
  const uint32_t base_s = smem_u32(smem_raw);
  unsigned char *smem = smem_raw + ((1024 - (base_s & 1023)) & 1023);
  unsigned char *sT = smem;            // 2 x 8 KiB (SW64 halves)
  unsigned char *sX1 = smem + 16384;   // 16 x 128 B (SW128)
  unsigned char *sX2 = smem + 18432;   // 16 x 128 B (SW128)
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 20480);
  uint64_t *mbar = bar + 1;
  uint32_t *holder = reinterpret_cast<uint32_t *>(bar + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(mbar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(holder, 64);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *holder;
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(bar, 16384 + 2048 + 2048);
    tc::tma_load_2d(sT, &tmT, 0, 0, bar);
    tc::tma_load_2d(sT + 8192, &tmT, 64, 0, bar);
    tc::tma_load_2d(sX1, &tmX, 0, 0, bar);
    tc::tma_load_2d(sX2, &tmX, 0, 16, bar);
    mbar_wait(bar, 0);
    tc::fence_after();
    const uint32_t id = tc::idesc_i8(128, 16);
    for (int kk = 0; kk < 4; ++kk)  // j = 32 kk .. : half kk / 2, offset 32 (kk % 2)
      tc::mma_i8(tmem, tc::sdesc_k_sw64(smem_u32(sT) + (kk >> 1) * 8192 + (kk & 1) * 32),
                 tc::sdesc_k_sw128(smem_u32(sX1) + kk * 32), id, kk > 0);
    for (int kk = 0; kk < 4; ++kk)  // i = 32 kk .. : rows 32 kk at 2048 kk in each half
      tc::mma_i8(tmem + 32, sdesc(smem_u32(sT) + kk * 2048, pr.lbo2, pr.sbo2, 4),
                 tc::sdesc_k_sw128(smem_u32(sX2) + kk * 32), id | (1u << 15), kk > 0);
    tc::mma_commit(mbar);
  }
  __syncthreads();
  mbar_wait(mbar, 0);
  tc::fence_after();
  uint32_t v[16];
  tc::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16), v);
  tc::tmem_ld_wait();
  for (int t = 0; t < 16; ++t) D1[(warp * 32 + lane) * 16 + t] = (int32_t)v[t];
  tc::tmem_ld16(tmem + 32 + ((uint32_t)(warp * 32) << 16), v);
  tc::tmem_ld_wait();
  for (int t = 0; t < 16; ++t) D2[(warp * 32 + lane) * 16 + t] = (int32_t)v[t];
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 64);
}

typedef CUresult (*PFN_enc)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static void tmap(PFN_enc enc, CUtensorMap *tm, void *p, int rows, int cols, int box_cols, int box_rows,
                 CUtensorMapSwizzle sw) {
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows}, strides[1] = {(cuuint64_t)cols};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows}, es[2] = {1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("tmap error %d\n", (int)r);
}

int main() {
  std::vector<int8_t> T(128 * 128), X(32 * 128);
  srand(11);
  for (auto &v : T) v = (int8_t)(rand() % 129 - 64);
  for (auto &v : X) v = (int8_t)(rand() % 129 - 64);
  int8_t *dT, *dX;
  int32_t *dD1, *dD2;
  cudaMalloc(&dT, T.size());
  cudaMalloc(&dX, X.size());
  cudaMalloc(&dD1, 128 * 16 * 4);
  cudaMalloc(&dD2, 128 * 16 * 4);
  cudaMemcpy(dT, T.data(), T.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dX, X.data(), X.size(), cudaMemcpyHostToDevice);
  void *fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  PFN_enc enc = (PFN_enc)fp;
  CUtensorMap tT, tX;
  tmap(enc, &tT, dT, 128, 128, 64, 128, CU_TENSOR_MAP_SWIZZLE_64B);
  tmap(enc, &tX, dX, 32, 128, 128, 16, CU_TENSOR_MAP_SWIZZLE_128B);
  std::vector<int> R1(128 * 16, 0), R2(128 * 16, 0);
  for (int i = 0; i < 128; ++i)
    for (int t = 0; t < 16; ++t)
      for (int j = 0; j < 128; ++j) R1[i * 16 + t] += T[i * 128 + j] * X[t * 128 + j];
  for (int j = 0; j < 128; ++j)
    for (int t = 0; t < 16; ++t)
      for (int i = 0; i < 128; ++i) R2[j * 16 + t] += T[i * 128 + j] * X[(16 + t) * 128 + i];
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  Params vars[] = {{8192, 512}, {512, 8192}, {16, 512}};
  for (auto &pr : vars) {
    cudaMemset(dD1, 0, 128 * 16 * 4);
    cudaMemset(dD2, 0, 128 * 16 * 4);
    probe<<<1, 128, 32768>>>(tT, tX, dD1, dD2, pr);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<int> G1(128 * 16), G2(128 * 16);
    cudaMemcpy(G1.data(), dD1, G1.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(G2.data(), dD2, G2.size() * 4, cudaMemcpyDeviceToHost);
    int bad1 = 0, bad2 = 0, bad2lo = 0;
    for (size_t k = 0; k < G1.size(); ++k) bad1 += G1[k] != R1[k];
    for (size_t k = 0; k < G2.size(); ++k) bad2 += G2[k] != R2[k];
    for (size_t k = 0; k < G2.size() / 2; ++k) bad2lo += G2[k] != R2[k];
    printf("{\"lbo\": %u, \"sbo\": %u, \"err\": \"%s\", \"rows_bad\": %d, \"cols_bad\": %d, \"cols_bad_first64\": %d}\n",
           pr.lbo2, pr.sbo2, cudaGetErrorString(e), bad1, bad2, bad2lo);
    if (e != cudaSuccess) break;
  }
  return 0;
}
