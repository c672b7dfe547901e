// Probe of the tcgen05 kind::i8 path used by the Ozaki-scheme Schur GEMM:
// (1) correctness of the smem descriptors (K-major, no swizzle: 8-row x 16 B
//     core matrices, chunk-major [k16][row][16 B]) and of the TMEM read-back,
// (2) issue-limited int8 MMA throughput with 7 level accumulators (M=128,
//     N=64, K=32 per instruction, 28 instructions per stage).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_i8_probe tools/umma_i8_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major, SWIZZLE_NONE descriptor: start, LBO (K-direction core-matrix
// stride), SBO (8-row group stride), version 1 (sm_100)
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;           // version
  return d;                          // base offset 0, lbo mode 0, layout 0 (none)
}
// instruction descriptor: s32 accum, s8 x s8, K-major both, M=128, N
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t dtmem, uint64_t da, uint64_t db, uint32_t idesc, int acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
               " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
               :: "r"(dtmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
               :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" :: "r"(smem_u32(bar)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  } while (!done);
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int32_t* v) {
  uint32_t r[16];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
  for (int i = 0; i < 16; ++i) v[i] = (int32_t)r[i];
}

// A: M=128 rows x K bytes (row-major in global), B: N=64 rows x K bytes.
// D[level][128][64] = sum over the level's slice pairs (here: level l uses
// A shifted by l rows cyclically, to give distinct results per accumulator).
template <int K>
__global__ void k_probe(const int8_t* A, const int8_t* B, int32_t* D, int nlev) {
  extern __shared__ __align__(1024) unsigned char sm[];
  int8_t* As = (int8_t*)sm;                 // [K/16][128][16]
  int8_t* Bs = As + 128 * K;                // [K/16][64][16]
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < 128 * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    As[(k / 16) * 128 * 16 + r * 16 + (k % 16)] = A[e];
  }
  for (int e = tid; e < 64 * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    Bs[(k / 16) * 64 * 16 + r * 16 + (k % 16)] = B[e];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" :: "r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) mbar_init(&bar, 1);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tb = tbase;
  if (tid == 0) {
    const uint32_t idesc = idesc_i8(128, 64);
    for (int l = 0; l < nlev; ++l)
      for (int kk = 0; kk < K / 32; ++kk) {
        // level l: B rows shifted by nothing, A rows as is; scale via repetition l+1
        for (int rep = 0; rep <= l; ++rep) {
          const uint64_t da = make_desc(smem_u32(As + kk * 2 * 128 * 16), 128 * 16, 128);
          const uint64_t db = make_desc(smem_u32(Bs + kk * 2 * 64 * 16), 64 * 16, 128);
          mma_i8(tb + l * 64, da, db, idesc, (kk | rep) ? 1 : 0);
        }
      }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const int row = (warp & 3) * 32 + (tid & 31);
  for (int l = 0; l < nlev; ++l)
    for (int c0 = 0; c0 < 64; c0 += 16) {
      int32_t v[16];
      tmem_ld16(tb + l * 64 + c0 + ((uint32_t)((warp & 3) * 32) << 16), v);
      for (int i = 0; i < 16; ++i) D[((size_t)l * 128 + row) * 64 + c0 + i] = v[i];
    }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" :: "r"(tb));
}

// throughput: every CTA issues `iters` stages of 28 MMAs (7 accumulators)
__global__ void k_rate(int iters, int32_t* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  int8_t* As = (int8_t*)sm;                 // 7 slices x [2][128][16]
  int8_t* Bs = As + 7 * 32 * 128;           // 7 slices x [2][64][16]
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < 7 * 32 * 128 + 7 * 32 * 64; e += blockDim.x) As[e] = (int8_t)((e * 37) & 7) - 3;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" :: "r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) mbar_init(&bar, 1);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tb = tbase;
  if (tid == 0) {
    const uint32_t idesc = idesc_i8(128, 64);
    for (int it = 0; it < iters; ++it)
      for (int d = 2; d <= 8; ++d)
        for (int t = 1; t < d; ++t) {
          const int u = d - t;
          const uint64_t da = make_desc(smem_u32(As + (t - 1) * 32 * 128), 128 * 16, 128);
          const uint64_t db = make_desc(smem_u32(Bs + (u - 1) * 32 * 64), 64 * 16, 128);
          mma_i8(tb + (d - 2) * 64, da, db, idesc, it > 0 || t > 1);
        }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  int32_t v[16];
  tmem_ld16(tb + ((uint32_t)((warp & 3) * 32) << 16), v);
  if (v[0] == 123456789) sink[0] = v[1];
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" :: "r"(tb));
}


template <int N, int NACC>
__global__ void k_rateN(int iters, int32_t* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  int8_t* As = (int8_t*)sm;                 // 4 slices x [2][128][16]
  int8_t* Bs = As + 4 * 32 * 128;           // 4 slices x [2][N][16]
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < 4 * 32 * 128 + 4 * 32 * N; e += blockDim.x) As[e] = (int8_t)((e * 37) & 7) - 3;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" :: "r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) mbar_init(&bar, 1);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tb = tbase;
  if (tid == 0) {
    const uint32_t idesc = idesc_i8(128, N);
    for (int it = 0; it < iters; ++it)
      for (int q = 0; q < 28; ++q) {
        const uint64_t da = make_desc(smem_u32(As + (q % 4) * 32 * 128), 128 * 16, 128);
        const uint64_t db = make_desc(smem_u32(Bs + ((q / 4) % 4) * 32 * N), N * 16, 128);
        mma_i8(tb + (q % NACC) * N, da, db, idesc, it > 0 || q >= NACC);
      }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  int32_t v[16];
  tmem_ld16(tb + ((uint32_t)((warp & 3) * 32) << 16), v);
  if (v[0] == 123456789) sink[0] = v[1];
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" :: "r"(tb));
}
// Sustained rate: the same N = 256 loop with pseudo-random operand bytes (the
// burst loop above uses 3-bit values), launched back to back for several
// seconds; SM clock from %globaltimer against clock64 inside the kernel.  This
// is the roofline denominator for an INT8 kernel timed inside a long step:
// the board power cap, not the issue rate, sets it.
template <int N, int NACC>
__global__ void k_rateS(int iters, int32_t* sink, unsigned long long* clk) {
  extern __shared__ __align__(1024) unsigned char sm[];
  int8_t* As = (int8_t*)sm;
  int8_t* Bs = As + 4 * 32 * 128;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < 4 * 32 * 128 + 4 * 32 * N; e += blockDim.x) {
    uint32_t h = (uint32_t)e * 2654435761u + blockIdx.x * 40503u;
    h ^= h >> 15; h *= 2246822519u; h ^= h >> 13;
    As[e] = (int8_t)(h & 0xFF);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" :: "r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) mbar_init(&bar, 1);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tb = tbase;
  unsigned long long n0 = 0, n1 = 0;
  long long c0 = 0, c1 = 0;
  if (tid == 0) {
    asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(n0));
    c0 = clock64();
    const uint32_t idesc = idesc_i8(128, N);
    for (int it = 0; it < iters; ++it)
      for (int q = 0; q < 28; ++q) {
        const uint64_t da = make_desc(smem_u32(As + (q % 4) * 32 * 128), 128 * 16, 128);
        const uint64_t db = make_desc(smem_u32(Bs + ((q / 4) % 4) * 32 * N), N * 16, 128);
        mma_i8(tb + (q % NACC) * N, da, db, idesc, it > 0 || q >= NACC);
      }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  if (tid == 0) {
    c1 = clock64();
    asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(n1));
    if (blockIdx.x == 0) { clk[0] = (unsigned long long)(c1 - c0); clk[1] = n1 - n0; }
  }
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  int32_t v[16];
  tmem_ld16(tb + ((uint32_t)((warp & 3) * 32) << 16), v);
  if (v[0] == 123456789) sink[0] = v[1];
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" :: "r"(tb));
}
void sustained(int32_t* sink) {
  CK(cudaFuncSetAttribute(k_rateS<256, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024));
  unsigned long long* clk;
  CK(cudaMalloc(&clk, 16));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 100000, ctas = 148;      // ~0.2 s per launch
  for (int rep = 0; rep < 30; ++rep) {
    cudaEventRecord(e0); k_rateS<256, 2><<<ctas, 128, 120 * 1024>>>(iters, sink, clk); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[2];
    CK(cudaMemcpy(h, clk, 16, cudaMemcpyDeviceToHost));
    if (rep % 3 == 2 || rep == 0)
      printf("sustained rep %2d: %.1f ms, %.1f TOPS, SM clock %.0f MHz\n", rep, ms,
             2.0 * ctas * iters * 28.0 * 128 * 256 * 32 / (ms * 1e-3) / 1e12, 1e3 * (double)h[0] / (double)h[1]);
  }
}

template <int N, int NACC>
void rateN(int32_t* sink) {
  CK(cudaFuncSetAttribute(k_rateN<N, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 1000, ctas = 148;
  k_rateN<N, NACC><<<ctas, 128, 120 * 1024>>>(10, sink); CK(cudaDeviceSynchronize());
  cudaEventRecord(e0); k_rateN<N, NACC><<<ctas, 128, 120 * 1024>>>(iters, sink); cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("N=%d acc=%d: %.1f TOPS\n", N, NACC, 2.0 * ctas * iters * 28.0 * 128 * N * 32 / (ms * 1e-3) / 1e12);
}

int main(int argc, char** argv) {
  if (argc > 1 && argv[1][0] == 's') {
    int32_t* sk;
    CK(cudaMalloc(&sk, 4));
    sustained(sk);
    return 0;
  }
  constexpr int K = 128;
  const int nlev = 7;
  std::vector<int8_t> A(128 * K), B(64 * K);
  srand(1);
  for (auto& a : A) a = (int8_t)(rand() % 255 - 127);
  for (auto& b : B) b = (int8_t)(rand() % 255 - 127);
  int8_t *dA, *dB;
  int32_t* dD;
  CK(cudaMalloc(&dA, A.size()));
  CK(cudaMalloc(&dB, B.size()));
  CK(cudaMalloc(&dD, (size_t)nlev * 128 * 64 * 4));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
  const int smem = 192 * K;
  CK(cudaFuncSetAttribute(k_probe<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k_probe<K><<<1, 128, smem>>>(dA, dB, dD, nlev);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<int32_t> D((size_t)nlev * 128 * 64);
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  long bad = 0;
  for (int l = 0; l < nlev; ++l)
    for (int i = 0; i < 128; ++i)
      for (int j = 0; j < 64; ++j) {
        long s = 0;
        for (int k = 0; k < K; ++k) s += (long)A[i * K + k] * B[j * K + k];
        s *= (l + 1);
        if (s != D[((size_t)l * 128 + i) * 64 + j]) {
          if (bad < 5) printf("mismatch l=%d i=%d j=%d got %d want %ld\n", l, i, j, D[((size_t)l * 128 + i) * 64 + j], s);
          ++bad;
        }
      }
  printf("correctness: %ld mismatches of %d\n", bad, nlev * 128 * 64);
  // throughput
  const int smem2 = 7 * 32 * 192;
  CK(cudaFuncSetAttribute(k_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
  int32_t* sink;
  CK(cudaMalloc(&sink, 4));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int ctas : {148, 296}) {
    const int iters = 2000;
    k_rate<<<ctas, 128, 100 * 1024>>>(10, sink);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    k_rate<<<ctas, 128, 100 * 1024>>>(iters, sink);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = 2.0 * ctas * (double)iters * 28 * 128 * 64 * 32;
    printf("ctas %d: %.3f ms, %.1f TOPS int8 (dense)\n", ctas, ms, ops / (ms * 1e-3) / 1e12);
  }
  (void)smem2;
  rateN<64, 7>(sink);
  rateN<128, 4>(sink);
  rateN<256, 2>(sink);
  rateN<128, 1>(sink);
  return 0;
}
