// Box characterization: sustained fp64 DFMA and DMMA
// (mma.sync m8n8k4 .f64) throughput, and a read-only HBM stream, on one B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
//   ./tools/fp64_peak      -> one JSON line
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double *out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void dmma_kernel(double *out, int iters) {
  double c[8][2];
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  double a = 1e-3 * threadIdx.x, b = 1.0 - 1e-3 * threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void read_kernel(const double2 *__restrict__ in, size_t n4, double *out) {
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldcs(in + i);
    s += v.x + v.y;
  }
  if (s == 12345.678) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *out;
  cudaMalloc(&out, sizeof(double) * 1 << 22);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  // DFMA: blocks x 256 threads x iters x 16 x 8 fma
  const int blocks = sms * 8, threads = 256, it = 4000;
  dfma_kernel<<<blocks, threads>>>(out, 10);
  cudaEventRecord(e0);
  dfma_kernel<<<blocks, threads>>>(out, it);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double dfma_tf = 2.0 * blocks * threads * (double)it * 128 / (ms * 1e-3) / 1e12;
  // DMMA: each mma = 8*8*4 FMA = 512 flop per warp instruction
  const int dit = 4000;
  dmma_kernel<<<blocks, threads>>>(out, 10);
  cudaEventRecord(e0);
  dmma_kernel<<<blocks, threads>>>(out, dit);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double dmma_tf = 512.0 * (blocks * threads / 32) * (double)dit * 8 / (ms * 1e-3) / 1e12;
  // read-only stream of 4 GiB
  const size_t bytes = (size_t)4 << 30;
  double2 *buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 0, bytes);
  read_kernel<<<sms * 8, 512>>>(buf, bytes / 16, out);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    read_kernel<<<sms * 8, 512>>>(buf, bytes / 16, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double read_gbs = bytes / (best * 1e-3) / 1e9;
  printf("{\"dfma_tflops\": %.3f, \"dmma_tflops\": %.3f, \"read_stream_gbs\": %.1f, \"sms\": %d}\n", dfma_tf, dmma_tf,
         read_gbs, sms);
  return 0;
}
