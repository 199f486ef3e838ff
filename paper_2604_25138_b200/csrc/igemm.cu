// int8 x int8 -> int32 GEMM on the 5th-generation tensor cores (tcgen05.mma
// kind::i8, accumulators in TMEM), the building block of the fp64 emulation
// (Ozaki scheme, ozaki.cu) that puts the fp64 contractions of the method --
// QK^T, the multi-RHS products and the fit's GEMMs -- on tcgen05
// (tcgen05 has no fp64 kind on sm_100a).
//
//   C[m][n] = sum_k A[m][k] B[n][k]    A: M x K, B: N x K int8, both K-contiguous
//
// Tile 128 x 256 per CTA, K staged in 128-byte chunks (one 128B-swizzle atom
// row) by 2-D TMA into a 4-stage ring; warp 0 produces, one thread of warp 1
// issues 4 MMAs (K = 32 each) per stage and commits them to the stage's
// "empty" barrier, then to "tmem full"; warps 2-5 (one per TMEM lane quadrant)
// drain the 128 x 256 s32 accumulator with tcgen05.ld and run the epilogue.
#include <cuda.h>

#include <cstdlib>

#include "laker_internal.h"
#include "tc_int8.cuh"

namespace laker {
namespace {

constexpr int kBM = 128, kBN = 256, kBK = 128;
constexpr int kIStages = 4;
constexpr uint32_t kABytes = kBM * kBK, kBBytes = kBN * kBK;
constexpr size_t kIgemmSmem = 1024 + kIStages * (kABytes + kBBytes) + 256;
constexpr int kIThreads = 6 * 32;

__global__ void __launch_bounds__(kIThreads, 1)
    igemm_s8_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const IgemmEpi e, int64_t K) {
  const int64_t M = e.M, N = e.N;
  const int64_t m0 = (int64_t)blockIdx.y * kBM, n0 = (int64_t)blockIdx.x * kBN;
  // tiles with no kept entry of a triangular product are skipped entirely
  if (e.tri == 1 && m0 + kBM - 1 + e.tri_off < n0) return;
  if (e.tri == 2 && m0 + e.tri_off >= n0 + kBN - 1) return;
  extern __shared__ unsigned char smem_raw[];
  // 1024-byte alignment for the 128B-swizzle atoms (TMA destination and UMMA descriptors)
  const uint32_t base_s = smem_u32(smem_raw);
  unsigned char *smem = smem_raw + ((1024 - (base_s & 1023)) & 1023);
  unsigned char *sA = smem;
  unsigned char *sB = smem + kIStages * kABytes;
  uint64_t *full = reinterpret_cast<uint64_t *>(sB + kIStages * kBBytes);
  uint64_t *empty = full + kIStages;
  uint64_t *tfull = empty + kIStages;
  uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(tfull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = (int)((K + kBK - 1) / kBK);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kIStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_holder, 256);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % kIStages;
        if (kb >= kIStages) mbar_wait(&empty[s], (uint32_t)(((kb / kIStages) - 1) & 1));
        mbar_arrive_expect_tx(&full[s], kABytes + kBBytes);
        tc::tma_load_2d(sA + s * kABytes, &tmA, kb * kBK, (int32_t)m0, &full[s]);
        tc::tma_load_2d(sB + s * kBBytes, &tmB, kb * kBK, (int32_t)n0, &full[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_i8(kBM, kBN);
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % kIStages;
        mbar_wait(&full[s], (uint32_t)((kb / kIStages) & 1));
        tc::fence_after();
        const uint32_t a0 = smem_u32(sA + s * kABytes), b0 = smem_u32(sB + s * kBBytes);
#pragma unroll
        for (int kk = 0; kk < kBK / 32; ++kk)
          tc::mma_i8(tmem, tc::sdesc_k_sw128(a0 + kk * 32), tc::sdesc_k_sw128(b0 + kk * 32), idesc,
                     (kb > 0 || kk > 0) ? 1u : 0u);
        tc::mma_commit(&empty[s]);
      }
      tc::mma_commit(tfull);
    }
  } else {
    // epilogue: warp w reads TMEM lanes 32 (w % 4) .. + 31 = tile rows
    const int q = warp & 3;
    const int64_t row = m0 + q * 32 + lane;
    mbar_wait(tfull, 0);
    tc::fence_after();
    const int ea = (e.mode != kIgemmStoreS32 && row < M) ? e.ea[row] : 0;
#pragma unroll 1
    for (int c = 0; c < kBN; c += 32) {
      if (n0 + c >= N) break;
      uint32_t v[32];
      tc::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c, v);
      tc::tmem_ld_wait();
      if (row >= M) continue;
      if (e.mode == kIgemmStoreS32) {
        int32_t *dst = e.Ci + row * e.ldci + n0 + c;
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (n0 + c + j < N) dst[j] = (int32_t)v[j];
        continue;
      }
      // x = v 2^(shift + ea_row + eb_col): exact (|v| < 2^31, power-of-two scale)
#pragma unroll 8
      for (int j = 0; j < 32; ++j) {
        const int64_t col = n0 + c + j;
        if (col >= N) break;
        const double x = scalbn((double)(int32_t)v[j], e.shift + ea + e.eb[col]);
        double *w = e.W + row * e.ldw + col;
        if (e.mode == kIgemmAccInit) {
          *w = x;
        } else if (e.mode == kIgemmAccAdd) {
          *w = __dadd_rn(*w, x);
        } else {  // final: C = alpha (W + x) + beta Cin + diag
          if (e.tri != 0) {
            const int64_t gr = row + e.tri_off;
            if (e.tri == 1 ? gr < col : gr >= col) continue;
          }
          const double tot = e.has_w ? __dadd_rn(*w, x) : x;
          double out = __dmul_rn(e.alpha, tot);
          if (e.beta != 0.0) out = __dadd_rn(out, __dmul_rn(e.beta, e.Cin[row * e.ldcin + col]));
          if (e.diag != 0.0 && row - col == e.diag_offset) out = __dadd_rn(out, e.diag);
          e.C[row * e.ldc + col] = out;
        }
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 256);
}

typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                       const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                                       CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                       CUtensorMapFloatOOBfill);

PFN_encodeTiled_t encode_fn() {
  static PFN_encodeTiled_t fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled_t>(p);
  }
  return fn;
}

}  // namespace

// K-contiguous int8 matrix rows x K (row stride ld bytes), box 128 (K) x box_rows, 128B swizzle
bool make_tmap_s8(CUtensorMap *tm, const int8_t *base, int64_t rows, int64_t K, int64_t ld, int box_rows) {
  PFN_encodeTiled_t enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld};
  cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t *>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 64-byte rows (K = 64 int8 per box row), SWIZZLE_64B: the K = 64 digit slices of otf_tc2.cu
bool make_tmap_s8_k64(CUtensorMap *tm, const int8_t *base, int64_t rows, int64_t K, int64_t ld, int box_rows) {
  PFN_encodeTiled_t enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld};
  cuuint32_t box[2] = {64u, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t *>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

void igemm_init() {
  cudaFuncSetAttribute(igemm_s8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kIgemmSmem);
}

// C (M x N, ldc) = A (M x K) B (N x K)^T; A, B device int8 with row strides lda, ldb
// (multiples of 16 bytes); K padded by the TMA zero fill.
cudaError_t launch_igemm_s8(const int8_t *A, int64_t lda, const int8_t *B, int64_t ldb, int32_t *C, int64_t ldc,
                            int64_t M, int64_t N, int64_t K, cudaStream_t s) {
  CUtensorMap ta, tb;
  if (!make_tmap_s8(&ta, A, M, K, lda, kBM) || !make_tmap_s8(&tb, B, N, K, ldb, kBN)) return cudaErrorInvalidValue;
  IgemmEpi e{};
  e.mode = kIgemmStoreS32;
  e.Ci = C;
  e.ldci = ldc;
  e.M = M;
  e.N = N;
  dim3 grid((unsigned)((N + kBN - 1) / kBN), (unsigned)((M + kBM - 1) / kBM));
  igemm_s8_kernel<<<grid, kIThreads, kIgemmSmem, s>>>(ta, tb, e, K);
  return cudaGetLastError();
}

cudaError_t launch_igemm_epi(const int8_t *A, int64_t lda, const int8_t *B, int64_t ldb, int64_t K,
                             const IgemmEpi &e, cudaStream_t s) {
  CUtensorMap ta, tb;
  if (!make_tmap_s8(&ta, A, e.M, K, lda, kBM) || !make_tmap_s8(&tb, B, e.N, K, ldb, kBN)) return cudaErrorInvalidValue;
  dim3 grid((unsigned)((e.N + kBN - 1) / kBN), (unsigned)((e.M + kBM - 1) / kBM));
  igemm_s8_kernel<<<grid, kIThreads, kIgemmSmem, s>>>(ta, tb, e, K);
  return cudaGetLastError();
}

}  // namespace laker

extern "C" laker_status laker_debug_igemm_s8(const int8_t *A, const int8_t *B, int32_t *C, int64_t M, int64_t N,
                                             int64_t K) {
  if (!A || !B || !C || M < 1 || N < 1 || K < 1 || K % 16 != 0) return LAKER_ERR_INVALID_ARGUMENT;
  static bool inited = false;
  if (!inited) {
    laker::igemm_init();
    inited = true;
  }
  if (laker::launch_igemm_s8(A, K, B, K, C, N, M, N, K, 0) != cudaSuccess) return LAKER_ERR_CUDA;
  if (cudaDeviceSynchronize() != cudaSuccess) return LAKER_ERR_CUDA;
  return LAKER_OK;
}
