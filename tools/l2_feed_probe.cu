// L2 -> shared-memory feed rate of the Ozaki GEMM's load pattern, with and
// without cluster multicast of the A operand.
//   mode 0: every CTA bulk-copies A (28 KB) + B (14 KB) per step (unicast; the
//           two CTAs of a pair read the SAME A block, different B blocks)
//   mode 1: cluster of 2: each CTA copies HALF of A with .multicast::cluster to
//           both CTAs, plus its own B (14 KB)
// Stages are recycled as soon as they have landed (no MMAs): the number is the
// ceiling of the feed, in bytes per clock per SM landed in shared memory.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_feed_probe l2_feed_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int AB = 28672, BB = 14336, NST = 4;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
                 " selp.u32 %0, 1, 0, p;\n}\n" : "=r"(done) : "r"(su32(bar)), "r"(parity) : "memory");
  } while (!done);
}

struct Smem {
  unsigned char st[NST][AB + BB];
  uint64_t full[NST], empty[NST];
};

template <int MODE>
__global__ void __launch_bounds__(64, 1) k_feed(const unsigned char* __restrict__ buf, size_t nblk, int steps,
                                                long long* clk) {
  extern __shared__ __align__(1024) unsigned char raw[];
  Smem& S = *reinterpret_cast<Smem*>(raw);
  const int tid = threadIdx.x;
  uint32_t rank = 0;
  if (MODE == 1) asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(rank));
  const int pair = blockIdx.x >> 1;
  if (tid == 0) {
    for (int q = 0; q < NST; ++q) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" :: "r"(su32(&S.full[q])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" :: "r"(su32(&S.empty[q])), "r"(MODE == 1 ? 2 : 1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (MODE == 1) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  const long long c0 = clock64();
  if (tid == 0) {
    // producer
    for (int g = 0; g < steps; ++g) {
      const int q = g % NST;
      if (g >= NST) mbar_wait(&S.empty[q], ((g / NST) - 1) & 1);
      const size_t ia = ((size_t)pair * 977 + (size_t)g) % nblk;          // A: shared by the pair
      const size_t ib = ((size_t)blockIdx.x * 1453 + (size_t)g + 7) % nblk;  // B: own
      const unsigned char* srcA = buf + ia * (AB + BB);
      const unsigned char* srcB = buf + ib * (AB + BB) + AB;
      const uint32_t bar = su32(&S.full[q]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" :: "r"(bar), "r"(AB + BB) : "memory");
      if (MODE == 0) {
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                     :: "r"(su32(S.st[q])), "l"(srcA), "r"(AB), "r"(bar) : "memory");
      } else {
        const uint32_t half = AB / 2;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;\n"
                     :: "r"(su32(S.st[q]) + rank * half), "l"(srcA + rank * half), "r"(half), "r"(bar), "h"((unsigned short)3)
                     : "memory");
      }
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                   :: "r"(su32(S.st[q] + AB)), "l"(srcB), "r"(BB), "r"(bar) : "memory");
    }
  } else if (tid == 32) {
    // consumer: release each stage as soon as it has landed
    for (int g = 0; g < steps; ++g) {
      const int q = g % NST;
      mbar_wait(&S.full[q], (g / NST) & 1);
      if (MODE == 0) {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" :: "r"(su32(&S.empty[q])) : "memory");
      } else {
        for (uint32_t r = 0; r < 2; ++r) {
          uint32_t rem;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(rem) : "r"(su32(&S.empty[q])), "r"(r));
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" :: "r"(rem) : "memory");
        }
      }
    }
  }
  __syncthreads();
  if (MODE == 1) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  if (tid == 0) clk[blockIdx.x] = clock64() - c0;
}

int main() {
  const size_t nblk = 1400;   // 60 MB of digit blocks: L2 resident
  unsigned char* buf;
  cudaMalloc(&buf, nblk * (AB + BB));
  cudaMemset(buf, 1, nblk * (AB + BB));
  long long* clk;
  cudaMalloc(&clk, 148 * sizeof(long long));
  const int steps = 20000;
  const size_t smem = sizeof(Smem) + 1024;
  cudaFuncSetAttribute(k_feed<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_feed<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      if (mode == 0) {
        k_feed<0><<<148, 64, smem>>>(buf, nblk, steps, clk);
      } else {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(148);
        cfg.blockDim = dim3(64);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, k_feed<1>, (const unsigned char*)buf, nblk, steps, clk);
      }
      cudaEventRecord(e1);
      cudaError_t err = cudaDeviceSynchronize();
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      long long h[148];
      cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; ++i) avg += (double)h[i] / 148;
      printf("mode %d rep %d: %s  %.2f ms, %.0f clk per step, %.1f B/clk/SM landed, %.2f TB/s landed (chip)\n", mode, rep,
             cudaGetErrorString(err), ms, avg / steps, (AB + BB) / (avg / steps),
             148.0 * steps * (AB + BB) / (ms * 1e-3) / 1e12);
    }
  }
  return 0;
}
