// Probe: A operand of tcgen05.mma kind::i8 from TMEM (filled by tcgen05.cp
// from shared memory, shape 128x256b = one 128-row x 32-byte A slice),
// B from shared memory.  Correctness + rate with 7 level accumulators.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t mdesc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t db, int acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %3, 0;\n"
               " tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %4, p;\n}\n"
               :: "r"(d), "r"(a), "l"(db), "r"(acc), "r"(IDESC));
}
__device__ __forceinline__ void cp_a(uint32_t taddr, uint64_t sd) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;\n" :: "r"(taddr), "l"(sd));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  uint32_t done = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(su(b)), "r"(ph) : "memory");
  } while (!done);
}
__device__ __forceinline__ void ld16(uint32_t t, int32_t* v) {
  uint32_t r[16];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(t));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
  for (int i = 0; i < 16; ++i) v[i] = (int32_t)r[i];
}
// D = A B^T with A (128 x K) staged through TMEM, K = 32 per slice step
template <int K>
__global__ void k_ts(const int8_t* A, const int8_t* B, int32_t* D) {
  extern __shared__ __align__(1024) unsigned char sm[];
  int8_t* As = (int8_t*)sm;          // [K/16][128][16]
  int8_t* Bs = As + 128 * K;         // [K/16][64][16]
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < 128 * K; e += blockDim.x) { int r = e / K, k = e % K; As[(k / 16) * 2048 + r * 16 + k % 16] = A[e]; }
  for (int e = tid; e < 64 * K; e += blockDim.x) { int r = e / K, k = e % K; Bs[(k / 16) * 1024 + r * 16 + k % 16] = B[e]; }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" :: "r"(su(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" :: "r"(su(&bar)));
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tb = tbase;
  if (tid == 0) {
    for (int kk = 0; kk < K / 32; ++kk) {
      const uint32_t ta = tb + 448 + (kk & 1) * 8;
      cp_a(ta, mdesc(su(As + kk * 2 * 2048), 2048, 128));
      mma_ts(tb, ta, mdesc(su(Bs + kk * 2 * 1024), 1024, 128), kk > 0);
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" :: "r"(su(&bar)) : "memory");
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const int row = warp * 32 + (tid & 31);
  for (int c0 = 0; c0 < 64; c0 += 16) {
    int32_t v[16];
    ld16(tb + c0 + ((uint32_t)(warp * 32) << 16), v);
    for (int i = 0; i < 16; ++i) D[row * 64 + c0 + i] = v[i];
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" :: "r"(tb));
}
// rate: per stage 7 tcgen05.cp (A slices into TMEM) + 28 TS MMAs
__global__ void k_rate(int iters, int32_t* sink, int with_cp) {
  extern __shared__ __align__(1024) unsigned char sm[];
  int8_t* As = (int8_t*)sm;          // 7 x [2][128][16]
  int8_t* Bs = As + 7 * 4096;        // 7 x [2][64][16]
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < 7 * 4096 + 7 * 2048; e += blockDim.x) As[e] = (int8_t)((e * 37) & 7) - 3;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" :: "r"(su(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" :: "r"(su(&bar)));
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tb = tbase;
  if (tid == 0) {
    for (int t = 0; t < 7; ++t) cp_a(tb + 448 + t * 8, mdesc(su(As + t * 4096), 2048, 128));
    for (int it = 0; it < iters; ++it) {
      if (with_cp) for (int t = 0; t < 7; ++t) cp_a(tb + 448 + t * 8, mdesc(su(As + t * 4096), 2048, 128));
      for (int d = 2; d <= 8; ++d)
        for (int t = 1; t < d; ++t)
          mma_ts(tb + (d - 2) * 64, tb + 448 + (t - 1) * 8, mdesc(su(Bs + (d - t - 1) * 2048), 1024, 128),
                 it > 0 || t > 1);
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" :: "r"(su(&bar)) : "memory");
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  int32_t v[16];
  ld16(tb + ((uint32_t)(warp * 32) << 16), v);
  if (v[0] == 123456789) sink[0] = v[1];
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" :: "r"(tb));
}
int main() {
  constexpr int K = 128;
  std::vector<int8_t> A(128 * K), B(64 * K);
  srand(3);
  for (auto& a : A) a = (int8_t)(rand() % 255 - 127);
  for (auto& b : B) b = (int8_t)(rand() % 255 - 127);
  int8_t *dA, *dB; int32_t* dD;
  CK(cudaMalloc(&dA, A.size())); CK(cudaMalloc(&dB, B.size())); CK(cudaMalloc(&dD, 128 * 64 * 4));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(k_ts<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, 192 * K));
  k_ts<K><<<1, 128, 192 * K>>>(dA, dB, dD);
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  std::vector<int32_t> D(128 * 64);
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  long bad = 0;
  for (int i = 0; i < 128; ++i) for (int j = 0; j < 64; ++j) {
    long s = 0; for (int k = 0; k < K; ++k) s += (long)A[i * K + k] * B[j * K + k];
    if (s != D[i * 64 + j]) { if (bad < 5) printf("mismatch %d %d got %d want %ld\n", i, j, D[i * 64 + j], s); ++bad; }
  }
  printf("TS correctness: %ld mismatches of %d\n", bad, 128 * 64);
  CK(cudaFuncSetAttribute(k_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024));
  int32_t* sink; CK(cudaMalloc(&sink, 4));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int wc : {1, 0}) {
    const int ctas = 148;
    const int iters = 2000;
    k_rate<<<ctas, 128, 120 * 1024>>>(10, sink, wc); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); k_rate<<<ctas, 128, 120 * 1024>>>(iters, sink, wc); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double ops = 2.0 * ctas * (double)iters * 28 * 128 * 64 * 32;
    printf("TS rate with_cp=%d: %.3f ms, %.1f TOPS int8\n", wc, ms, ops / (ms * 1e-3) / 1e12);
  }
  return 0;
}
