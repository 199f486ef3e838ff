// Microbenchmark: HBM read rate of the symmetric apply's tile stream (128 x 64 fp64 tiles of
// the block upper triangle of an n x n matrix, one persistent CTA per SM, TMA producer warp,
// 3-stage mbarrier ring, consumer warps that only touch the tile) for two storage layouts:
//   rowmajor: the matrix row-major (ld = n), each tile one 2-D TMA (128 rows x 512 B);
//   tiled:    each tile's 64 KiB contiguous (tile-major storage), each tile 4 x 16 KiB 1-D bulk copies.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2604_25138_b200/csrc -lcuda tools/tile_read_bw.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "tma.cuh"

using namespace laker;

constexpr int kSR = 128, kSC = 64, kStages = 3, kCons = 16;
constexpr uint32_t kTile = kSR * kSC * 8;

__device__ __forceinline__ void tma2d(void *dst, const CUtensorMap *tm, int c0, int c1, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

template <bool TILED>
__global__ void __launch_bounds__((kCons + 1) * 32, 1)
    stream_kernel(const __grid_constant__ CUtensorMap tm, const double *base, const int *tI, const int *tJ, int64_t T,
                  double *sink) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + kStages * kTile);
  uint64_t *empty = full + kStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t0 = T * blockIdx.x / gridDim.x, t1 = T * (blockIdx.x + 1) / gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCons);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == kCons) {
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_first();
      int slot = 0;
      uint32_t ph = 0;
      bool first = true;
      for (int64_t t = t0; t < t1; ++t) {
        if (!first) mbar_wait(&empty[slot], ph ^ 1u);
        unsigned char *st = smem + slot * kTile;
        mbar_arrive_expect_tx(&full[slot], kTile);
        if (TILED) {
          for (int q = 0; q < 4; ++q)
            bulk_g2s(st + q * (kTile / 4), reinterpret_cast<const unsigned char *>(base) + t * kTile + q * (kTile / 4),
                     kTile / 4, &full[slot], pol);
        } else {
          tma2d(st, &tm, tJ[t] * kSC, tI[t] * kSR, &full[slot]);
        }
        if (++slot == kStages) {
          slot = 0;
          ph ^= 1u;
          first = false;
        }
      }
    }
    return;
  }
  double acc = 0.0;
  int slot = 0;
  uint32_t ph = 0;
  for (int64_t t = t0; t < t1; ++t) {
    mbar_wait(&full[slot], ph);
    const double *tile = reinterpret_cast<const double *>(smem + slot * kTile);
    acc += tile[threadIdx.x];
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
    if (++slot == kStages) {
      slot = 0;
      ph ^= 1u;
    }
  }
  if (acc == 12345.678) sink[0] = acc;
}

typedef CUresult (*PFN_enc)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int64_t n = 16384;
  const int nb = n / kSR, nct = n / kSC;
  std::vector<int> I, J;
  for (int b = 0; b < nb; ++b)
    for (int j = 2 * b; j < nct; ++j) {
      I.push_back(b);
      J.push_back(j);
    }
  const int64_t T = I.size();
  double *A = nullptr, *sink = nullptr;
  int *dI, *dJ;
  cudaMalloc(&A, (size_t)n * n * 8);
  cudaMemset(A, 0, (size_t)n * n * 8);
  cudaMalloc(&sink, 8);
  cudaMalloc(&dI, T * 4);
  cudaMalloc(&dJ, T * 4);
  cudaMemcpy(dI, I.data(), T * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dJ, J.data(), T * 4, cudaMemcpyHostToDevice);
  void *fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)n}, strides[1] = {(cuuint64_t)n * 8};
  cuuint32_t box[2] = {kSC, kSR}, es[2] = {1, 1};
  ((PFN_enc)fp)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, A, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const size_t smem = kStages * kTile + 64;
  cudaFuncSetAttribute(stream_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(stream_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = (double)T * kTile;
  for (int tiled = 0; tiled < 2; ++tiled) {
    float best = 1e9f;
    for (int r = 0; r < 12; ++r) {
      cudaEventRecord(e0);
      if (tiled)
        stream_kernel<true><<<sms, (kCons + 1) * 32, smem>>>(tm, A, dI, dJ, T, sink);
      else
        stream_kernel<false><<<sms, (kCons + 1) * 32, smem>>>(tm, A, dI, dJ, T, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 2 && ms < best) best = ms;
    }
    printf("{\"layout\": \"%s\", \"tiles\": %lld, \"bytes\": %.0f, \"best_us\": %.1f, \"gbs\": %.1f, \"err\": \"%s\"}\n",
           tiled ? "tiled" : "rowmajor", (long long)T, bytes, best * 1e3, bytes / (best * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
