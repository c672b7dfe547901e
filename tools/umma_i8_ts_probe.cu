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
// wide MMAs (A digit x up to 4 consecutive B digits, N <= 256; B as [chunk][digit][64 rows]):
// mode 0 = A from shared memory (SS), 1 = A from TMEM without the per-stage copies, 2 = with them
__device__ __forceinline__ uint32_t idesc_n(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__global__ void k_rate_wide(int iters, int32_t* sink, int mode) {
  extern __shared__ __align__(1024) unsigned char sm[];
  int8_t* As = (int8_t*)sm;          // 7 x [2][128][16]
  int8_t* Bs = As + 7 * 4096;        // [2][7][64][16]
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
    const long long c0 = clock64();
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int t = 1; t <= 7; ++t) {
        if (mode == 2) cp_a(tb + 448 + (t - 1) * 8, mdesc(su(As + (t - 1) * 4096), 2048, 128));
#pragma unroll
        for (int u0 = 1; u0 <= 8 - t; u0 += 4) {
          const int nu = (8 - t - u0 + 1) < 4 ? (8 - t - u0 + 1) : 4;
          const uint64_t db = mdesc(su(Bs + (u0 - 1) * 1024), 7 * 1024, 128);
          const uint32_t d = tb + (t + u0 - 2) * 64;
          const int acc = it > 0 || t > 1;
          if (mode == 0) {
            const uint64_t da = mdesc(su(As + (t - 1) * 4096), 2048, 128);
            asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                         " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                         :: "r"(d), "l"(da), "l"(db), "r"(idesc_n(64 * nu)), "r"(acc));
          } else {
            asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                         " tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n"
                         :: "r"(d), "r"(tb + 448 + (t - 1) * 8), "l"(db), "r"(idesc_n(64 * nu)), "r"(acc));
          }
        }
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" :: "r"(su(&bar)) : "memory");
    mbar_wait(&bar, 0);
    if (blockIdx.x == 0) sink[1] = (int32_t)((clock64() - c0) / iters);
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

// the same wide MMAs (A from shared memory) in different ORDERS: consecutive MMAs
// that touch the same accumulator columns may serialise in the tensor pipe
#define WMMA(t, u0, nu)                                                                              \
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"                                         \
               " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"                         \
               :: "r"(tb + ((t) + (u0) - 2) * 64), "l"(mdesc(abase + ((t) - 1) * 4096, 2048, 128)),     \
                  "l"(mdesc(bbase + ((u0) - 1) * 1024, 7 * 1024, 128)), "r"(idesc_n(64 * (nu))), "r"(1))
#define TMMA(t, u0, nu)                                                                              \
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"                                         \
               " tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n"                       \
               :: "r"(tb + ((t) + (u0) - 2) * 64), "r"(tb + 448 + ((t) - 1) * 8),                       \
                  "l"(mdesc(bbase + ((u0) - 1) * 1024, 7 * 1024, 128)), "r"(idesc_n(64 * (nu))), "r"(1))
#define TCP(t) cp_a(tb + 448 + ((t) - 1) * 8, mdesc(abase + ((t) - 1) * 4096, 2048, 128))
#define MA WMMA(1, 1, 4)
#define MB WMMA(1, 5, 3)
#define MC WMMA(2, 1, 4)
#define MD WMMA(2, 5, 2)
#define ME WMMA(3, 1, 4)
#define MF WMMA(3, 5, 1)
#define MG WMMA(4, 1, 4)
#define MH WMMA(5, 1, 3)
#define MI WMMA(6, 1, 2)
#define MJ WMMA(7, 1, 1)
template <int ORDER>
__global__ void k_rate_order(int iters, int32_t* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  int8_t* As = (int8_t*)sm;
  int8_t* Bs = As + 7 * 4096;
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
    const uint32_t abase = su(As), bbase = su(Bs);
    for (int t = 1; t <= 7; ++t) TCP(t);
    const long long c0 = clock64();
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
      if (ORDER == 0) { MA; MB; MC; MD; ME; MF; MG; MH; MI; MJ; }          // digit-major (kernel)
      if (ORDER == 1) { MB; MA; MD; MC; MF; ME; MJ; MI; MH; MG; }          // low / high alternating first
      if (ORDER == 2) { MA; MB; MA; MB; MA; MB; MA; MB; }                  // disjoint only (28 pairs)
      if (ORDER == 3) { MA; MA; MA; MA; MA; MA; MA; }                      // same columns (28 pairs)
      if (ORDER == 4) { MJ; MJ; MJ; MJ; MJ; MJ; MJ; MJ; }                  // N = 64, same columns (8 pairs)
      if (ORDER == 5) { MA; MJ; MA; MF; MA; MJ; MA; MF; }                  // disjoint 256 / 64 (20 pairs)
      if (ORDER == 6) { MG; MG; MG; MG; MG; MG; MG; }                      // N = 256 on [192,448) same columns
      if (ORDER == 7) { MA; MG; MA; MG; MA; MG; MA; }                      // [0,256) / [192,448): partial overlap
      if (ORDER == 8) {   // A from TMEM (copied once before the loop)
        TMMA(1, 1, 4); TMMA(1, 5, 3); TMMA(2, 1, 4); TMMA(2, 5, 2); TMMA(3, 1, 4); TMMA(3, 5, 1);
        TMMA(4, 1, 4); TMMA(5, 1, 3); TMMA(6, 1, 2); TMMA(7, 1, 1);
      }
      if (ORDER == 9) {   // A from TMEM, one tcgen05.cp per digit and k step
        TCP(1); TMMA(1, 1, 4); TMMA(1, 5, 3); TCP(2); TMMA(2, 1, 4); TMMA(2, 5, 2); TCP(3); TMMA(3, 1, 4);
        TMMA(3, 5, 1); TCP(4); TMMA(4, 1, 4); TCP(5); TMMA(5, 1, 3); TCP(6); TMMA(6, 1, 2); TCP(7); TMMA(7, 1, 1);
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" :: "r"(su(&bar)) : "memory");
    mbar_wait(&bar, 0);
    if (blockIdx.x == 0) sink[1] = (int32_t)((clock64() - c0) / iters);
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
template <int ORDER>
static void run_order(const char* name, int pairs, int32_t* sk) {
  CK(cudaFuncSetAttribute(k_rate_order<ORDER>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
  k_rate_order<ORDER><<<148, 128, 100 * 1024>>>(10, sk); CK(cudaDeviceSynchronize());
  k_rate_order<ORDER><<<148, 128, 100 * 1024>>>(2000, sk); CK(cudaDeviceSynchronize());
  int32_t hk[2];
  CK(cudaMemcpy(hk, sk, 8, cudaMemcpyDeviceToHost));
  printf("order %-34s %2d digit pairs: %5d clk per step (%.3f of the 32 clk/pair peak)\n", name, pairs, hk[1],
         32.0 * pairs / hk[1]);
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
  {
    int32_t* sk;
    CK(cudaMalloc(&sk, 8));
    CK(cudaFuncSetAttribute(k_rate_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int mode = 0; mode < 3; ++mode) {
      const int iters = 2000;
      k_rate_wide<<<148, 128, 100 * 1024>>>(10, sk, mode); CK(cudaDeviceSynchronize());
      cudaEventRecord(a); k_rate_wide<<<148, 128, 100 * 1024>>>(iters, sk, mode); cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms; cudaEventElapsedTime(&ms, a, b);
      int32_t hk[2];
      CK(cudaMemcpy(hk, sk, 8, cudaMemcpyDeviceToHost));
      printf("wide mode %d (%s): %d clk per k step; %.3f ms, %.1f TOPS int8\n", mode,
             mode == 0 ? "A from smem" : (mode == 1 ? "A from TMEM" : "A from TMEM + copies"), hk[1], ms,
             2.0 * 148 * iters * 28.0 * 128 * 64 * 32 / (ms * 1e-3) / 1e12);
    }
  }
  {
    int32_t* sk;
    CK(cudaMalloc(&sk, 8));
    run_order<0>("digit-major (kernel)", 28, sk);
    run_order<1>("b a d c f e j i h g", 28, sk);
    run_order<2>("a b a b (disjoint)", 28, sk);
    run_order<3>("a x7 (same columns, N=256)", 28, sk);
    run_order<4>("j x8 (same columns, N=64)", 8, sk);
    run_order<5>("a j a f (disjoint 256/64)", 20, sk);
    run_order<6>("g x7 (same columns, N=256)", 28, sk);
    run_order<7>("a g a g (partial overlap)", 28, sk);
    run_order<8>("digit-major, A from TMEM", 28, sk);
    run_order<9>("digit-major, A from TMEM + copies", 28, sk);
  }
  return 0;
}
