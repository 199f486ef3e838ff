// Feasibility probe for an exact int8 tensor-core symmetric apply: can one row-major
// int8 tile in shared memory (128 rows i x 64 bytes j, TMA SWIZZLE_64B) feed tcgen05
// kind::i8 both as a K-major A operand (row products, contraction over j) and as an
// MN-major A operand (column products, contraction over i)?
//   D1[i][t] = sum_j T[i][j] X1[t][j]   (M = 128, N = 16, K = 64: K-major A)
//   D2[j][t] = sum_i T[i][j] X2[t][i]   (M = 64,  N = 16, K = 128: MN-major A, "transpose A")
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2604_25138_b200/csrc -lcuda tools/mma_mn_major_test.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <string>
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
  uint32_t lbo2, sbo2, layout2, tbit;
};

__global__ void __launch_bounds__(128, 1) probe(const __grid_constant__ CUtensorMap tmT,
                                                const __grid_constant__ CUtensorMap tmX1,
                                                const __grid_constant__ CUtensorMap tmX2, int32_t *D1, int32_t *D2,
                                                Params pr) {
  extern __shared__ unsigned char smem_raw[];
  const uint32_t base_s = smem_u32(smem_raw);
  unsigned char *smem = smem_raw + ((1024 - (base_s & 1023)) & 1023);
  unsigned char *sT = smem;              // 128 x 64 B = 8 KiB (SW64)
  unsigned char *sX1 = smem + 8192;      // 16 x 64 B = 1 KiB (SW64)
  unsigned char *sX2 = smem + 9216 + 1024 - 9216 % 1024 + 0;  // aligned below
  sX2 = smem + 10240;                    // 16 x 128 B = 2 KiB (SW128)
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 16384);
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
    mbar_arrive_expect_tx(bar, 8192 + 1024 + 2048);
    tc::tma_load_2d(sT, &tmT, 0, 0, bar);
    tc::tma_load_2d(sX1, &tmX1, 0, 0, bar);
    tc::tma_load_2d(sX2, &tmX2, 0, 0, bar);
    mbar_wait(bar, 0);
    tc::fence_after();
    // D1 (columns 0..15): K-major A (T), K-major B (X1), K = 64 in two steps of 32
    const uint32_t id1 = tc::idesc_i8(128, 16);
    for (int kk = 0; kk < 2; ++kk)
      tc::mma_i8(tmem, tc::sdesc_k_sw64(smem_u32(sT) + kk * 32), tc::sdesc_k_sw64(smem_u32(sX1) + kk * 32), id1,
                 kk > 0);
    // D2 (columns 32..47): MN-major A (T^T: M = j, K = i), K-major B (X2, K = 128), four K steps
    // of 32 rows i (32 rows x 64 B = 2048 B of the swizzled tile each)
    const uint32_t id2 = tc::idesc_i8(64, 16) | (pr.tbit << 15);
    for (int kk = 0; kk < 4; ++kk)
      tc::mma_i8(tmem + 32, sdesc(smem_u32(sT) + kk * 2048, pr.lbo2, pr.sbo2, pr.layout2),
                 tc::sdesc_k_sw128(smem_u32(sX2) + kk * 32), id2, kk > 0);
    tc::mma_commit(mbar);
  }
  __syncthreads();
  mbar_wait(mbar, 0);
  tc::fence_after();
  uint32_t v[16];
  tc::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16), v);
  tc::tmem_ld_wait();
  for (int t = 0; t < 16; ++t) D1[(warp * 32 + lane) * 16 + t] = (int32_t)v[t];
  {  // M = 64 accumulator: rows 16 w .. 16 w + 15 in lanes 32 w .. 32 w + 15
    tc::tmem_ld16(tmem + 32 + ((uint32_t)(warp * 32) << 16), v);
    tc::tmem_ld_wait();
    if (lane < 16)
      for (int t = 0; t < 16; ++t) D2[(warp * 16 + lane) * 16 + t] = (int32_t)v[t];
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 64);
}

typedef CUresult (*PFN_enc)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static void tmap(PFN_enc enc, CUtensorMap *tm, void *p, int rows, int cols, int box_cols, CUtensorMapSwizzle sw) {
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows}, strides[1] = {(cuuint64_t)cols};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)rows}, es[2] = {1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("tmap error %d\n", (int)r);
}

int main() {
  std::vector<int8_t> T(128 * 64), X1(16 * 64), X2(16 * 128);
  srand(7);
  for (auto &v : T) v = (int8_t)(rand() % 129 - 64);
  for (auto &v : X1) v = (int8_t)(rand() % 129 - 64);
  for (auto &v : X2) v = (int8_t)(rand() % 129 - 64);
  int8_t *dT, *dX1, *dX2;
  int32_t *dD1, *dD2;
  cudaMalloc(&dT, T.size());
  cudaMalloc(&dX1, X1.size());
  cudaMalloc(&dX2, X2.size());
  cudaMalloc(&dD1, 128 * 16 * 4);
  cudaMalloc(&dD2, 64 * 16 * 4);
  cudaMemcpy(dT, T.data(), T.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dX1, X1.data(), X1.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dX2, X2.data(), X2.size(), cudaMemcpyHostToDevice);
  void *fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  PFN_enc enc = (PFN_enc)fp;
  CUtensorMap tT, t1, t2;
  tmap(enc, &tT, dT, 128, 64, 64, CU_TENSOR_MAP_SWIZZLE_64B);
  tmap(enc, &t1, dX1, 16, 64, 64, CU_TENSOR_MAP_SWIZZLE_64B);
  tmap(enc, &t2, dX2, 16, 128, 128, CU_TENSOR_MAP_SWIZZLE_128B);
  std::vector<int> R1(128 * 16, 0), R2(64 * 16, 0);
  for (int i = 0; i < 128; ++i)
    for (int t = 0; t < 16; ++t)
      for (int j = 0; j < 64; ++j) R1[i * 16 + t] += T[i * 64 + j] * X1[t * 64 + j];
  for (int j = 0; j < 64; ++j)
    for (int t = 0; t < 16; ++t)
      for (int i = 0; i < 128; ++i) R2[j * 16 + t] += T[i * 64 + j] * X2[t * 128 + i];
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  // variants of the MN-major A descriptor: (lbo, sbo, layout, transpose bit)
  Params vars[] = {{16, 512, 4, 1}, {128, 512, 4, 1}, {256, 512, 4, 1}, {2048, 512, 4, 1}, {16, 256, 4, 1},
                   {16, 512, 2, 1}, {16, 1024, 2, 1}};
  for (auto &pr : vars) {
    cudaMemset(dD1, 0, 128 * 16 * 4);
    cudaMemset(dD2, 0, 64 * 16 * 4);
    probe<<<1, 128, 32768>>>(tT, t1, t2, dD1, dD2, pr);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<int> G1(128 * 16), G2(64 * 16);
    cudaMemcpy(G1.data(), dD1, G1.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(G2.data(), dD2, G2.size() * 4, cudaMemcpyDeviceToHost);
    int bad1 = 0, bad2 = 0;
    for (size_t k = 0; k < G1.size(); ++k) bad1 += G1[k] != R1[k];
    for (size_t k = 0; k < G2.size(); ++k) bad2 += G2[k] != R2[k];
    {
      std::string okj;
      for (int j = 0; j < 64; ++j) {
        int ok = 1;
        for (int t = 0; t < 16; ++t) ok &= G2[j * 16 + t] == R2[j * 16 + t];
        okj += ok ? '1' : '0';
      }
      // which K-ranges of i would explain entry (0,0)? partial sums over i-blocks of 32
      printf("okj=%s\n", okj.c_str());
    }
    printf("{\"lbo\": %u, \"sbo\": %u, \"layout\": %u, \"tbit\": %u, \"err\": \"%s\", \"rows_bad\": %d, \"cols_bad\": %d, "
           "\"d2_0\": %d, \"r2_0\": %d}\n",
           pr.lbo2, pr.sbo2, pr.layout2, pr.tbit, cudaGetErrorString(e), bad1, bad2, G2[0], R2[0]);
    if (e != cudaSuccess) break;
  }
  return 0;
}
