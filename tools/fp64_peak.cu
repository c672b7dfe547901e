// FP64 peak microbenchmark for B200 (sm_100a): DFMA pipe vs DMMA (mma.sync m8n8k4 f64).
// Output: one JSON line with measured TFLOP/s for each; used as the roofline
// denominator for the frontal factorisation (MEASURED_PEAKS.json has no FP64 entry).
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void dmma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-6, b = 0.999;
  double c[CHAINS][2];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) { c[k][0] = 0; c[k][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < CHAINS; ++k) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* d; CK(cudaMalloc(&d, 64));
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int threads = 256, blocks = sms * 8, iters = 20000;
  float ms;
  // DFMA
  dfma_kernel<8><<<blocks, threads>>>(d, 100, 1.0000001, 1e-9);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  dfma_kernel<8><<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1);
  double dfma_tf = 2.0 * 8 * (double)iters * threads * blocks / (ms * 1e-3) / 1e12;
  // DMMA: each mma = 8*8*4 FMAs per warp
  dmma_kernel<8><<<blocks, threads>>>(d, 100);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  dmma_kernel<8><<<blocks, threads>>>(d, iters);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  float ms2; cudaEventElapsedTime(&ms2, e0, e1);
  double dmma_tf = 2.0 * 256 * 8 * (double)iters * (threads / 32) * blocks / (ms2 * 1e-3) / 1e12;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"dfma_tflops\": %.3f, \"dmma_tflops\": %.3f, \"sms\": %d, \"dfma_ms\": %.3f, \"dmma_ms\": %.3f, \"clock_khz\": %d}\n",
         dfma_tf, dmma_tf, sms, ms, ms2, clk);
  return 0;
}
