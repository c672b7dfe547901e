// Schur-complement update of the large fronts on the INT8 tensor cores
// (tcgen05.mma kind::i8, TMEM accumulators): an Ozaki-scheme FP64 GEMM.
//
// The Schur update of a front with p pivots and b = nf - p border rows is
//     C (b x b, complex symmetric, packed lower)  -=  L' L'^T,   L' = L'[p:nf, 0:p]
// (L' = L D^{1/2}, fronts.cuh).  Each complex row r of L' is scaled by its own
// power of two 2^-e_r (max_k max(|Re|, |Im|) < 2^e_r) and written as 7 balanced
// base-256 digits d_1..d_7 in [-128, 127] of Y = rint(L'_rk 2^(54 - e_r)):
//     L'_rk = 2^(e_r - 54) sum_t d_t 256^(7 - t)   (exact up to the rint, 2^-55
// relative to the row maximum).  Then
//     (L' L'^T)_ij = 2^(e_i + e_j - 108) sum_{t,u} 256^(14 - t - u) sum_k d_t(ik) d_u(jk)
// and the 28 most significant digit pairs (t + u <= 8) are kept; every inner
// sum is an exact int8 x int8 -> int32 tensor-core product (K <= 18,000 cannot
// overflow).  Complex arithmetic rides a real embedding (4 real products): the
// 128 accumulator lanes of a tile hold the real parts of 64 complex rows
// (A row = (Re, -Im) interleaved along k) and their imaginary parts
// (A row = (Im, Re)); the B rows are (Re, Im).  k_oz_split writes all three
// digit layouts once per factorisation step, so the GEMM only streams them.
//
// The GEMM CTA (one 64 x 64 complex tile of one front of one pole) keeps the 7
// digit levels d = t + u = 2..8 in 7 TMEM accumulators of 64 columns (448 of
// 512), streams 16 complex k per stage (A_big 28 KB + B 14 KB digit blocks, bulk
// copies by a producer thread into a 4-stage ring), issues 28 MMAs (M=128,
// N=64, K=32) per stage from one thread, and combines the levels in FP64 in
// the epilogue:  C_ij -= 2^(e_i + e_j - 108) sum_{d=8..2} 256^(14 - d) acc_d(ij)
// (all scalings exact powers of two).
// Deterministic: fixed k order, fixed level order, one CTA per C tile.
// Accuracy: normwise like an FP64 GEMM (2^-54 of row max x column max per
// term); the device factor is checked against the reference's SuperLU
// backward error and the parity goldens (tests/test_gpu_verify.py).
#include "fronts.cuh"
#include "kernels.h"

namespace rba {

namespace {
constexpr int OZ_S = 7;                    // digits per value
constexpr int OZ_KS = 16;                  // complex k per stage (= one MMA-K32)
constexpr int OZ_ABYTES = OZ_S * 2 * 128 * 16;  // A_big digits of one (row tile, k step)
constexpr int OZ_BBYTES = OZ_S * 2 * 64 * 16;   // B digits
constexpr int OZ_BLK = OZ_ABYTES + OZ_BBYTES;   // one (row tile, k step) block
constexpr int OZ_NLD = 4;                  // stages of the load ring
constexpr int OZ_LEV = 7;                  // accumulator levels d = 2..8

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;                  // sm_100 descriptor version; no swizzle
  return d;
}
// s32 accumulator, s8 x s8, both K-major, M = 128, N = 64
constexpr uint32_t OZ_IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(64 >> 3) << 17) |
                              ((uint32_t)(128 >> 4) << 24);

__device__ __forceinline__ void mma_i8(uint32_t dtmem, uint64_t da, uint64_t db, int acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
               " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
               :: "r"(dtmem), "l"(da), "l"(db), "r"(OZ_IDESC), "r"(acc));
}
__device__ __forceinline__ void mbar_init_(uint64_t* bar, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" :: "r"(su32(bar)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_wait_(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  long long t0 = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                 " selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(su32(bar)), "r"(parity) : "memory");
    if (!done) {                       // a lost copy / commit must not hang the device
      if (t0 == 0) t0 = clock64();
      else if (clock64() - t0 > 40000000000LL) __trap();
    }
  } while (!done);
}
// the same with cluster-scope acquire: arrivals released by the peer CTA
__device__ __forceinline__ void mbar_wait_cl_(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  long long t0 = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
                 " selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(su32(bar)), "r"(parity) : "memory");
    if (!done) {
      if (t0 == 0) t0 = clock64();
      else if (clock64() - t0 > 40000000000LL) __trap();
    }
  } while (!done);
}
}  // namespace

// ---------------------------------------------------------------------------
// digit split: one CTA per (front task, row tile of 64 border rows, pole).
// Balanced base-256 digits without carries: U = Y + 0x80808080808080 is
// non-negative for |Y| < 2^54 and byte j of U, XOR 0x80, is the signed digit
// of weight 256^j.  -Im gets its own digits (a negated -128 would overflow).
// Per (row tile, k step) block: A_big [slice][chunk][128 rows][16 B] with rows
// 0..63 = (Re, -Im) and 64..127 = (Im, Re), then B [slice][chunk][64][16 B]
// = (Re, Im); k interleaved with the real/imaginary part inside each 16 B.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long oz_u(double v, int e) {
  return (unsigned long long)(__double2ll_rn(ldexp(v, 54 - e)) + 0x80808080808080LL);
}
// digit byte (signed, as raw bits) of slice t (t = 0: most significant, 256^6)
__device__ __forceinline__ uint32_t oz_dig(unsigned long long u, int t) {
  return (uint32_t)((u >> (8 * (OZ_S - 1 - t))) & 0xFFu) ^ 0x80u;
}

__global__ void __launch_bounds__(128) k_oz_split(const OzTask* __restrict__ tasks, int ntasks,
                                                  FrontsDev F, PoleBatch pb,
                                                  unsigned char* __restrict__ split,
                                                  int64_t split_pole, int* __restrict__ expo,
                                                  int64_t exp_pole, int bhalf) {
  __shared__ int s_e[64];
  __shared__ double s_m[2][64];
  const int slot = blockIdx.y;
  int ti = 0;
  {
    int lo = 0, hi = ntasks - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (tasks[mid].rt_start <= (int)blockIdx.x) lo = mid; else hi = mid - 1;
    }
    ti = lo;
  }
  const OzTask tk = tasks[ti];
  const int rt = blockIdx.x - tk.rt_start;
  const int s = tk.s, nf = tk.nf, c_lo = tk.c_lo, t0 = tk.t0, t1 = tk.t1;
  const int b = nf - c_lo;                     // rows of the region
  const cplx* __restrict__ panel = pb.factor[slot] + F.panel_off[s];
  const int tid = threadIdx.x, r = tid & 63, h = tid >> 6;
  const int row = rt * 64 + r;                 // region row (0-based)
  const bool on = row < b;
  // pass 1: row maximum over the k range
  double m = 0.0;
  if (on)
    for (int k = t0 + h; k < t1; k += 2) {
      const cplx v = __ldg(panel + (int64_t)k * nf + c_lo + row);
      m = fmax(m, fmax(fabs(v.x), fabs(v.y)));
    }
  s_m[h][r] = m;
  __syncthreads();
  if (h == 0) {
    const double mm = fmax(s_m[0][r], s_m[1][r]);
    s_e[r] = mm > 0.0 ? ilogb(mm) + 1 : 0;     // mm < 2^e
    if (on) expo[(int64_t)slot * exp_pole + tk.exp_off + row] = s_e[r];
  }
  __syncthreads();
  const int e = s_e[r];
  // pass 2: digits, thread = (row r, chunk h of 8 complex k) per k step
  unsigned char* out = split + (int64_t)slot * split_pole + tk.split_off + (int64_t)rt * tk.nks * OZ_BLK;
  for (int ks = 0; ks < tk.nks; ++ks) {
    unsigned long long ure[8], uim[8], unim[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int k = t0 + ks * OZ_KS + h * 8 + j;
      cplx v = cmk(0.0, 0.0);
      if (on && k < t1) v = __ldg(panel + (int64_t)k * nf + c_lo + row);
      ure[j] = oz_u(v.x, e);
      uim[j] = oz_u(v.y, e);
      unim[j] = oz_u(-v.y, e);
    }
    unsigned char* blk = out + (int64_t)ks * OZ_BLK;
#pragma unroll
    for (int t = 0; t < OZ_S; ++t) {
      uint4 wre, wim, wb;
      uint32_t* pre = &wre.x;
      uint32_t* pim = &wim.x;
      uint32_t* pb_ = &wb.x;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t r0 = oz_dig(ure[2 * q], t), r1 = oz_dig(ure[2 * q + 1], t);
        const uint32_t i0 = oz_dig(uim[2 * q], t), i1 = oz_dig(uim[2 * q + 1], t);
        const uint32_t n0 = oz_dig(unim[2 * q], t), n1 = oz_dig(unim[2 * q + 1], t);
        pre[q] = r0 | (n0 << 8) | (r1 << 16) | (n1 << 24);   // (Re, -Im)
        pim[q] = i0 | (r0 << 8) | (i1 << 16) | (r1 << 24);   // (Im, Re)
        pb_[q] = r0 | (i0 << 8) | (r1 << 16) | (i1 << 24);   // (Re, Im)
      }
      *reinterpret_cast<uint4*>(blk + ((t * 2 + h) * 128 + r) * 16) = wre;
      *reinterpret_cast<uint4*>(blk + ((t * 2 + h) * 128 + 64 + r) * 16) = wim;
      // B rows: [slice][chunk][64 rows] (one CTA per tile) or, for the
      // cluster-pair kernel, [row half][slice][chunk][32 rows] (each CTA of
      // the pair streams its half of the columns contiguously)
      const int boff = bhalf ? (((r >> 5) * OZ_S + t) * 2 + h) * 32 + (r & 31) : (t * 2 + h) * 64 + r;
      *reinterpret_cast<uint4*>(blk + OZ_ABYTES + boff * 16) = wb;
    }
  }
}

// ---------------------------------------------------------------------------
// INT8 tensor-core GEMM, persistent and warp-specialised (192 threads):
// warp 0 / lane 0 streams the digit blocks (bulk copies into a 4-stage
// mbarrier ring, straight across tile boundaries), warp 1 / lane 0 issues the
// 28 digit-pair MMAs per k step into the 7 TMEM level accumulators, warps 2..5
// (TMEM lanes 32 (w mod 4) ...) read the accumulators, hand TMEM back to the
// MMA warp and only then do the read-modify-write of C -- so the global
// epilogue of one tile overlaps the MMAs of the next.  CTA b takes the items
// (pole, tile) b, b + G, b + 2G, ...: each tile is still computed by exactly
// one CTA in a fixed k and level order (deterministic).
// ---------------------------------------------------------------------------
struct OzSmem {
  unsigned char st[OZ_NLD][OZ_BLK];          // [stage][A_big | B] digit blocks
  uint64_t full[OZ_NLD], empty[OZ_NLD];
  uint64_t tfull, tempty;                    // accumulators: MMA -> epilogue -> MMA
  uint64_t aslot[8];                         // TS: A digit slot in TMEM free again
  uint32_t tbase;
};
// TS variant: the A digit of each (k step, t) is copied once into one of 8
// TMEM slots of 8 columns (448..511, next to the 7 level accumulators) by
// tcgen05.cp and the 8 - t MMAs that use it read A from TMEM, so the MMAs
// read only B (2 KB) from shared memory instead of A + B (6 KB).  A slot is
// rewritten 8 digits later, after the commit of the MMAs that read it.
__device__ __forceinline__ void mma_i8_ts(uint32_t dtmem, uint32_t atmem, uint64_t db, int acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
               " tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n"
               :: "r"(dtmem), "r"(atmem), "l"(db), "r"(OZ_IDESC), "r"(acc));
}

__device__ __forceinline__ void oz_item(const OzTask* __restrict__ tasks, int ntasks,
                                        const int2* __restrict__ tiles, int ntiles, int item,
                                        int& slot, OzTask& tk, int& tr, int& tj) {
  slot = item / ntiles;
  const int tile = item - slot * ntiles;
  int lo = 0, hi = ntasks - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (tasks[mid].tile_start <= tile) lo = mid; else hi = mid - 1;
  }
  tk = tasks[lo];
  const int2 tt = __ldg(tiles + tile);
  tr = tt.x;
  tj = tt.y;
}

template <bool TS>
__global__ void __launch_bounds__(192, 1) k_oz_gemm(const OzTask* __restrict__ tasks, int ntasks,
                                                    const int2* __restrict__ tiles, int ntiles,
                                                    FrontsDev F, PoleBatch pb,
                                                    const unsigned char* __restrict__ split,
                                                    int64_t split_pole, const int* __restrict__ expo,
                                                    int64_t exp_pole) {
  extern __shared__ __align__(1024) unsigned char oz_raw[];
  OzSmem& S = *reinterpret_cast<OzSmem*>(oz_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nitems = ntiles * pb.count;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" :: "r"(su32(&S.tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 32) {
    for (int q = 0; q < OZ_NLD; ++q) {
      mbar_init_(&S.full[q], 1);
      mbar_init_(&S.empty[q], 1);
    }
    mbar_init_(&S.tfull, 1);
    mbar_init_(&S.tempty, 128);
    for (int q = 0; q < 8; ++q) mbar_init_(&S.aslot[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tb = S.tbase;

  if (tid == 0) {
    // ---- producer ----
    int g = 0;
    for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
      int slot, tr, tj;
      OzTask tk;
      oz_item(tasks, ntasks, tiles, ntiles, item, slot, tk, tr, tj);
      const unsigned char* sp = split + (int64_t)slot * split_pole + tk.split_off;
      const unsigned char* srcA = sp + (int64_t)tr * tk.nks * OZ_BLK;
      const unsigned char* srcB = sp + (int64_t)tj * tk.nks * OZ_BLK + OZ_ABYTES;
      for (int ks = 0; ks < tk.nks; ++ks, ++g) {
        const int q = g % OZ_NLD;
        if (g >= OZ_NLD) mbar_wait_(&S.empty[q], ((g / OZ_NLD) - 1) & 1);
        const uint32_t bar = su32(&S.full[q]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" :: "r"(bar), "r"(OZ_ABYTES + OZ_BBYTES) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                     :: "r"(su32(S.st[q])), "l"(srcA + (int64_t)ks * OZ_BLK), "r"(OZ_ABYTES), "r"(bar) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                     :: "r"(su32(S.st[q] + OZ_ABYTES)), "l"(srcB + (int64_t)ks * OZ_BLK), "r"(OZ_BBYTES), "r"(bar) : "memory");
      }
    }
  } else if (tid == 32) {
    // ---- MMA issuer ----
    int g = 0, it = 0;
    for (int item = blockIdx.x; item < nitems; item += gridDim.x, ++it) {
      int slot, tr, tj;
      OzTask tk;
      oz_item(tasks, ntasks, tiles, ntiles, item, slot, tk, tr, tj);
      if (it > 0) mbar_wait_(&S.tempty, (it - 1) & 1);     // epilogue drained TMEM
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      for (int ks = 0; ks < tk.nks; ++ks, ++g) {
        const int q = g % OZ_NLD;
        mbar_wait_(&S.full[q], (g / OZ_NLD) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        const uint32_t abase = su32(S.st[q]), bbase = abase + OZ_ABYTES;
        if constexpr (TS) {
          // digit-major order (integer sums: the order does not change the result)
#pragma unroll
          for (int t = 1; t <= OZ_S; ++t) {
            const int n = g * OZ_S + (t - 1);          // global A digit counter
            const int sl = n & 7;
            if (n >= 8) {
              mbar_wait_(&S.aslot[sl], ((n >> 3) - 1) & 1);
              asm volatile("tcgen05.fence::after_thread_sync;\n");
            }
            const uint32_t ta = tb + 448 + sl * 8;
            asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;\n"
                         :: "r"(ta), "l"(umma_desc(abase + (t - 1) * 2 * 128 * 16, 128 * 16, 128)));
#pragma unroll
            for (int u = 1; u <= 8 - t; ++u) {
              const uint64_t db = umma_desc(bbase + (u - 1) * 2 * 64 * 16, 64 * 16, 128);
              mma_i8_ts(tb + (t + u - 2) * 64, ta, db, (ks > 0 || t > 1) ? 1 : 0);
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
                         :: "r"(su32(&S.aslot[sl])) : "memory");
          }
        } else {
#pragma unroll
        for (int d = 2; d <= 8; ++d)
#pragma unroll
          for (int t = 1; t < d; ++t) {
            const int u = d - t;
            if (t > OZ_S || u > OZ_S) continue;
            const uint64_t da = umma_desc(abase + (t - 1) * 2 * 128 * 16, 128 * 16, 128);
            const uint64_t db = umma_desc(bbase + (u - 1) * 2 * 64 * 16, 64 * 16, 128);
            mma_i8(tb + (d - 2) * 64, da, db, (ks > 0 || t > 1) ? 1 : 0);
          }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
                     :: "r"(su32(&S.empty[q])) : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
                   :: "r"(su32(&S.tfull)) : "memory");
    }
  } else if (warp >= 2) {
    // ---- epilogue: warp w reads TMEM lanes 32 (w mod 4) .. +31 ----
    const int wq = warp & 3;
    const int arow = wq * 32 + lane;
    const bool imag = arow >= 64;
    const int lr = arow & 63;
    int it = 0;
    for (int item = blockIdx.x; item < nitems; item += gridDim.x, ++it) {
      int slot, tr, tj;
      OzTask tk;
      oz_item(tasks, ntasks, tiles, ntiles, item, slot, tk, tr, tj);
      mbar_wait_(&S.tfull, it & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      double acc[64];
#pragma unroll
      for (int i = 0; i < 64; ++i) acc[i] = 0.0;
#pragma unroll
      for (int c0 = 0; c0 < 64; c0 += 16) {
#pragma unroll
        for (int d = 8; d >= 2; --d) {            // smallest terms first
          uint32_t v[16];
          const uint32_t taddr = tb + (uint32_t)((d - 2) * 64 + c0) + ((uint32_t)(wq * 32) << 16);
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                       : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                         "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
                         "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                       : "r"(taddr));
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
          const double w = ldexp(1.0, 8 * (14 - d));
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[c0 + i] = fma((double)(int32_t)v[i], w, acc[c0 + i]);
        }
      }
      // TMEM is free for the next tile's MMAs
      asm volatile("tcgen05.fence::before_thread_sync;\n");
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" :: "r"(su32(&S.tempty)) : "memory");
      const int s = tk.s, nf = tk.nf, c_lo = tk.c_lo, c_hi = tk.c_hi;
      const int p = F.npiv[s];
      const int b = nf - c_lo;
      const int grow = tr * 64 + lr;                // region row of this accumulator row
      if (grow < b) {
        const int* ex = expo + (int64_t)slot * exp_pole + tk.exp_off;
        const int ei = __ldg(ex + grow);
        cplx* panel = pb.factor[slot] + F.panel_off[s];
        cplx* upd = pb.upd[slot] + (F.upd_off[s] >= 0 ? F.upd_off[s] : 0);
        const int r = c_lo + grow;                   // front row
#pragma unroll
        for (int c0 = 0; c0 < 64; c0 += 16) {
          double* dst[16];
          double cur[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int gcol = tj * 64 + c0 + i;
            const int c = c_lo + gcol;               // front column
            dst[i] = (c < c_hi && gcol <= grow)
                         ? reinterpret_cast<double*>(faddr(panel, upd, p, nf, r, c)) + (imag ? 1 : 0)
                         : nullptr;
            cur[i] = dst[i] ? __ldcg(dst[i]) : 0.0;
          }
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (dst[i]) *dst[i] = cur[i] - ldexp(acc[c0 + i], ei + __ldg(ex + tj * 64 + c0 + i) - 108);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" :: "r"(tb));
}

// ---------------------------------------------------------------------------
// Cluster-pair variant (RBA_OZ_2CTA=1): two CTAs on the two SMs of a TPC run
// one tcgen05.mma.cta_group::2 (M = 256: 128 complex rows, N = 64): each CTA
// streams its own 64-row A block and HALF of the 64 B columns, so per SM the
// MMAs read 5 KB instead of 6 KB of shared memory per 262k MACs and the L2
// traffic drops by a sixth.  The leader issues the MMAs; both CTAs' bulk
// copies complete on the leader's stage barrier; the commits are multicast to
// both CTAs; each CTA drains its own TMEM lanes and arrives on the leader's
// "TMEM empty" barrier.  A non-tensor bulk copy completes only on a barrier of
// its own CTA, so the peer's copies land on the peer's stage barrier and a
// relay thread there forwards each completed stage to the leader's (count 2).
// Same digits, same order, same results as k_oz_gemm.
// ---------------------------------------------------------------------------
constexpr int OZ_BH = OZ_S * 2 * 32 * 16;        // half of a B block (32 rows)
constexpr uint32_t OZ_IDESC2 = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(64 >> 3) << 17) |
                               ((uint32_t)(256 >> 4) << 24);
constexpr int OZ_NLD2 = 6;                         // deeper ring: hides the relay hop
struct OzSmem2 {
  unsigned char st[OZ_NLD2][OZ_ABYTES + OZ_BH];
  uint64_t full[OZ_NLD2], empty[OZ_NLD2];
  uint64_t tfull, tempty;
  uint32_t tbase;
};

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t map_to_leader(uint32_t saddr) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;\n" : "=r"(r) : "r"(saddr));
  return r;
}
__device__ __forceinline__ void cluster_sync_() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
k_oz_gemm2(const OzTask* __restrict__ tasks, int ntasks, const int2* __restrict__ tiles, int ntiles,
           FrontsDev F, PoleBatch pb, const unsigned char* __restrict__ split, int64_t split_pole,
           const int* __restrict__ expo, int64_t exp_pole) {
  extern __shared__ __align__(1024) unsigned char oz_raw2[];
  OzSmem2& S = *reinterpret_cast<OzSmem2*>(oz_raw2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cta_rank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int nitems = ntiles * pb.count;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" :: "r"(su32(&S.tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  if (tid == 32) {
    for (int q = 0; q < OZ_NLD2; ++q) {
      mbar_init_(&S.full[q], rank == 0 ? 2 : 1);
      mbar_init_(&S.empty[q], 1);
    }
    mbar_init_(&S.tfull, 1);
    mbar_init_(&S.tempty, 256);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  cluster_sync_();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tb = S.tbase;

  if (tid == 0) {
    // ---- producer (both CTAs): own A block + own half of B ----
    int g = 0;
    for (int item = pair; item < nitems; item += npairs) {
      int slot, tr2, tj;
      OzTask tk;
      oz_item(tasks, ntasks, tiles, ntiles, item, slot, tk, tr2, tj);
      const int tr = 2 * tr2 + (int)rank;
      const unsigned char* sp = split + (int64_t)slot * split_pole + tk.split_off;
      const unsigned char* srcA = sp + (int64_t)tr * tk.nks * OZ_BLK;
      const unsigned char* srcB = sp + (int64_t)tj * tk.nks * OZ_BLK + OZ_ABYTES + rank * OZ_BH;
      for (int ks = 0; ks < tk.nks; ++ks, ++g) {
        const int q = g % OZ_NLD2;
        if (g >= OZ_NLD2) mbar_wait_(&S.empty[q], ((g / OZ_NLD2) - 1) & 1);
        const uint32_t bar = su32(&S.full[q]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n"
                     :: "r"(bar), "r"(OZ_ABYTES + OZ_BH) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                     :: "r"(su32(S.st[q])), "l"(srcA + (int64_t)ks * OZ_BLK), "r"(OZ_ABYTES), "r"(bar) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                     :: "r"(su32(S.st[q] + OZ_ABYTES)), "l"(srcB + (int64_t)ks * OZ_BLK), "r"(OZ_BH), "r"(bar) : "memory");
      }
    }
  } else if (tid == 32 && rank == 1) {
    // ---- relay (peer): forward each landed stage to the leader's barrier ----
    int g = 0;
    for (int item = pair; item < nitems; item += npairs) {
      int slot, tr2, tj;
      OzTask tk;
      oz_item(tasks, ntasks, tiles, ntiles, item, slot, tk, tr2, tj);
      for (int ks = 0; ks < tk.nks; ++ks, ++g) {
        const int q = g % OZ_NLD2;
        mbar_wait_(&S.full[q], (g / OZ_NLD2) & 1);
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n"
                     :: "r"(map_to_leader(su32(&S.full[q]))) : "memory");
      }
    }
  } else if (tid == 32 && rank == 0) {
    // ---- MMA issuer (leader) ----
    int g = 0, it = 0;
    for (int item = pair; item < nitems; item += npairs, ++it) {
      int slot, tr2, tj;
      OzTask tk;
      oz_item(tasks, ntasks, tiles, ntiles, item, slot, tk, tr2, tj);
      if (it > 0) mbar_wait_cl_(&S.tempty, (it - 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      for (int ks = 0; ks < tk.nks; ++ks, ++g) {
        const int q = g % OZ_NLD2;
        mbar_wait_cl_(&S.full[q], (g / OZ_NLD2) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        const uint32_t abase = su32(S.st[q]), bbase = abase + OZ_ABYTES;
#pragma unroll
        for (int d = 2; d <= 8; ++d)
#pragma unroll
          for (int t = 1; t < d; ++t) {
            const int u = d - t;
            if (t > OZ_S || u > OZ_S) continue;
            const uint64_t da = umma_desc(abase + (t - 1) * 2 * 128 * 16, 128 * 16, 128);
            const uint64_t db = umma_desc(bbase + (u - 1) * 2 * 32 * 16, 32 * 16, 128);
            asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                         " tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                         :: "r"(tb + (uint32_t)((d - 2) * 64)), "l"(da), "l"(db), "r"(OZ_IDESC2),
                            "r"((ks > 0 || t > 1) ? 1 : 0));
          }
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n"
                     :: "r"(su32(&S.empty[q])), "h"((unsigned short)3) : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n"
                   :: "r"(su32(&S.tfull)), "h"((unsigned short)3) : "memory");
    }
  } else if (warp >= 2) {
    // ---- epilogue (both CTAs): own 128 TMEM lanes = own 64 complex rows ----
    const int wq = warp & 3;
    const int arow = wq * 32 + lane;
    const bool imag = arow >= 64;
    const int lr = arow & 63;
    const uint32_t tempty_leader = map_to_leader(su32(&S.tempty));
    int it = 0;
    for (int item = pair; item < nitems; item += npairs, ++it) {
      int slot, tr2, tj;
      OzTask tk;
      oz_item(tasks, ntasks, tiles, ntiles, item, slot, tk, tr2, tj);
      const int tr = 2 * tr2 + (int)rank;
      mbar_wait_(&S.tfull, it & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      double acc[64];
#pragma unroll
      for (int i = 0; i < 64; ++i) acc[i] = 0.0;
#pragma unroll
      for (int c0 = 0; c0 < 64; c0 += 16) {
#pragma unroll
        for (int d = 8; d >= 2; --d) {
          uint32_t v[16];
          const uint32_t taddr = tb + (uint32_t)((d - 2) * 64 + c0) + ((uint32_t)(wq * 32) << 16);
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                       : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                         "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
                         "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                       : "r"(taddr));
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
          const double w = ldexp(1.0, 8 * (14 - d));
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[c0 + i] = fma((double)(int32_t)v[i], w, acc[c0 + i]);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n");
      asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" :: "r"(tempty_leader) : "memory");
      const int s = tk.s, nf = tk.nf, c_lo = tk.c_lo, c_hi = tk.c_hi;
      const int p = F.npiv[s];
      const int b = nf - c_lo;
      const int grow = tr * 64 + lr;
      if (tr < tk.nrt && grow < b) {
        const int* ex = expo + (int64_t)slot * exp_pole + tk.exp_off;
        const int ei = __ldg(ex + grow);
        cplx* panel = pb.factor[slot] + F.panel_off[s];
        cplx* upd = pb.upd[slot] + (F.upd_off[s] >= 0 ? F.upd_off[s] : 0);
        const int r = c_lo + grow;
#pragma unroll
        for (int c0 = 0; c0 < 64; c0 += 16) {
          double* dst[16];
          double cur[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int gcol = tj * 64 + c0 + i;
            const int c = c_lo + gcol;
            dst[i] = (c < c_hi && gcol <= grow)
                         ? reinterpret_cast<double*>(faddr(panel, upd, p, nf, r, c)) + (imag ? 1 : 0)
                         : nullptr;
            cur[i] = dst[i] ? __ldcg(dst[i]) : 0.0;
          }
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (dst[i]) *dst[i] = cur[i] - ldexp(acc[c0 + i], ei + __ldg(ex + tj * 64 + c0 + i) - 108);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  cluster_sync_();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" :: "r"(tb));
}

void launch_oz_schur(cudaStream_t st, const OzTask* tasks, int ntasks, const int2* tiles,
                     int nrowtiles, int ntiles, const FrontsDev& F, const PoleBatch& pb,
                     unsigned char* split, int64_t split_pole, int* expo, int64_t exp_pole,
                     int pair) {
  if (ntasks <= 0 || ntiles <= 0) return;
  k_oz_split<<<dim3(nrowtiles, pb.count), 128, 0, st>>>(tasks, ntasks, F, pb, split,
                                                        split_pole, expo, exp_pole, pair == 1);
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  const int items = ntiles * pb.count;
  if (pair == 1) {
    const size_t smem = sizeof(OzSmem2) + 1024;
    static bool attr2 = false;
    if (!attr2) {
      cudaFuncSetAttribute(k_oz_gemm2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr2 = true;
    }
    const int npairs = std::min(items, nsm / 2);
    k_oz_gemm2<<<2 * npairs, 192, smem, st>>>(tasks, ntasks, tiles, ntiles, F, pb, split, split_pole,
                                               expo, exp_pole);
    return;
  }
  const size_t smem = sizeof(OzSmem) + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_oz_gemm<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_oz_gemm<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  if (pair == 2)
    k_oz_gemm<true><<<std::min(items, nsm), 192, smem, st>>>(tasks, ntasks, tiles, ntiles, F, pb, split,
                                                             split_pole, expo, exp_pole);
  else
    k_oz_gemm<false><<<std::min(items, nsm), 192, smem, st>>>(tasks, ntasks, tiles, ntiles, F, pb, split,
                                                              split_pole, expo, exp_pole);
}

}  // namespace rba
