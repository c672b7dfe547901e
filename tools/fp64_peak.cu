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

// larger f64 MMA shapes (PTX 7.8+, sm_90+): m16n8k4 / m16n8k8 / m16n8k16
template <int K, int CHAINS>
__global__ void dmma16_kernel(double* out, int iters) {
  double a[K / 2], b[K / 4];
#pragma unroll
  for (int i = 0; i < K / 2; ++i) a[i] = 1.0 + threadIdx.x * 1e-6 + i * 1e-7;
#pragma unroll
  for (int i = 0; i < K / 4; ++i) b[i] = 0.999 - i * 1e-7;
  double c[CHAINS][4];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) c[k][0] = c[k][1] = c[k][2] = c[k][3] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < CHAINS; ++k) {
      if (K == 4)
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                     : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3]) : "d"(a[0]), "d"(a[1 % (K / 2)]), "d"(b[0]));
      else if (K == 8)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3])
                     : "d"(a[0]), "d"(a[1 % (K / 2)]), "d"(a[2 % (K / 2)]), "d"(a[3 % (K / 2)]), "d"(b[0]), "d"(b[1 % (K / 4)]));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                     : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3])
                     : "d"(a[0]), "d"(a[1 % (K / 2)]), "d"(a[2 % (K / 2)]), "d"(a[3 % (K / 2)]),
                       "d"(a[4 % (K / 2)]), "d"(a[5 % (K / 2)]), "d"(a[6 % (K / 2)]), "d"(a[7 % (K / 2)]),
                       "d"(b[0]), "d"(b[1 % (K / 4)]), "d"(b[2 % (K / 4)]), "d"(b[3 % (K / 4)]));
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  if (s == 12345.678) out[0] = s;
}

// mixed: even warps run DMMA chains, odd warps DFMA chains -- do the two
// share one FP64 datapath (combined rate ~ one peak) or not (~ the sum)?
__global__ void mixed_kernel(double* out, int it_mma, int it_fma) {
  const int warp = threadIdx.x >> 5;
  double s = 0;
  if (warp & 1) {
    double acc[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] = threadIdx.x * 1e-3 + c;
    for (int it = 0; it < it_fma; ++it) {
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[c] = fma(acc[c], 1.0000001, 1e-9);
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) s += acc[c];
  } else {
    double a = 1.0 + threadIdx.x * 1e-6, b = 0.999;
    double c[8][2];
#pragma unroll
    for (int k = 0; k < 8; ++k) { c[k][0] = 0; c[k][1] = 0; }
    for (int it = 0; it < it_mma; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  }
  if (s == 12345.678) out[0] = s;
}

template <int K>
static double time16(double* d, int blocks, int threads, int iters) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  dmma16_kernel<K, 4><<<blocks, threads>>>(d, 100);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  dmma16_kernel<K, 4><<<blocks, threads>>>(d, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return 2.0 * 16 * 8 * K * 4 * (double)iters * (threads / 32) * blocks / (ms * 1e-3) / 1e12;
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
  const double t4 = time16<4>(d, blocks, threads, iters / 4);
  const double t8 = time16<8>(d, blocks, threads, iters / 8);
  const double t16 = time16<16>(d, blocks, threads, iters / 16);
  // mixed: DMMA iterations scaled so each half alone would take about the same time
  const int it_mma = iters, it_fma = (int)(iters * 8.0 * dfma_tf / dmma_tf);
  mixed_kernel<<<blocks, threads>>>(d, 100, 100);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  mixed_kernel<<<blocks, threads>>>(d, it_mma, it_fma);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  float ms3; cudaEventElapsedTime(&ms3, e0, e1);
  const double half_warps = (threads / 64.0) * blocks;
  const double mixed_tf = (2.0 * 256 * 8 * (double)it_mma * half_warps +
                           2.0 * 8 * (double)it_fma * 32 * half_warps) / (ms3 * 1e-3) / 1e12;
  printf("{\"mixed_dmma_dfma_tflops\": %.3f, ", mixed_tf);
  printf("\"dfma_tflops\": %.3f, \"dmma_tflops\": %.3f, \"dmma_m16n8k4_tflops\": %.3f, \"dmma_m16n8k8_tflops\": %.3f, \"dmma_m16n8k16_tflops\": %.3f, \"sms\": %d, \"dfma_ms\": %.3f, \"dmma_ms\": %.3f, \"clock_khz\": %d}\n",
         dfma_tf, dmma_tf, t4, t8, t16, sms, ms, ms2, clk);
  return 0;
}
