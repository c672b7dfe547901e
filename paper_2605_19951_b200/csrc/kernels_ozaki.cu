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
// copies by a producer thread into a 4-stage ring), issues the 28 digit-pair
// products of a stage as 10 wide MMAs from one thread (M = 128, K = 32, N =
// 64 x the number of consecutive B digits that pair with one A digit: the 7
// level accumulators are consecutive TMEM columns and the B digits consecutive
// shared-memory rows, so A digit t times B digits u0..u1 is ONE MMA of N =
// 64 (u1 - u0 + 1) <= 256 into levels t + u0 .. t + u1 -- each A digit block is
// read from shared memory 10 times per stage instead of 28), and combines
// the levels in FP64 in the epilogue:  C_ij -= 2^(e_i + e_j - 108) sum_{d=8..2} 256^(14 - d) acc_d(ij)
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
constexpr int OZ_LEV = 7;                  // accumulator levels d = 2..8
// cluster-pair kernel: per-CTA B arrangement (see k_oz_gemm2), bytes per (row tile, k step)
constexpr int OZ_B2 = 12288;
constexpr int OZ_BLK2 = OZ_ABYTES + 2 * OZ_B2;
// B groups of the pair kernel: byte offset inside the rank's B arrangement and rows per chunk
constexpr int OZ_G1 = 0, OZ_G2 = 4096, OZ_G3 = 6144, OZ_G4 = 7168, OZ_G5 = 8192, OZ_G6 = 10240, OZ_G7 = 11264;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;                  // sm_100 descriptor version; no swizzle
  return d;
}
// s32 accumulator, s8 x s8, both K-major, M = 128, N = n
__host__ __device__ constexpr uint32_t oz_idesc(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t dtmem, uint64_t da, uint64_t db, uint32_t idesc, int acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
               " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
               :: "r"(dtmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
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
}  // namespace

// ---------------------------------------------------------------------------
// digit split: one CTA per (front task, row tile of 64 border rows, pole).
// Balanced base-256 digits without carries: U = Y + 0x80808080808080 is
// non-negative for |Y| < 2^54 and byte j of U, XOR 0x80, is the signed digit
// of weight 256^j.  -Im gets its own digits (a negated -128 would overflow).
// Per (row tile, k step) block: A_big [slice][chunk][128 rows][16 B] with row
// 2 r = (Re, -Im) and row 2 r + 1 = (Im, Re) of complex row r (accumulator
// lanes 2 r, 2 r + 1 = real and imaginary part of C row r: a warp of the
// epilogue covers 16 complex rows = 256 contiguous bytes of a C column), then
// B = (Re, Im) as
// [chunk][slice][64 rows][16 B] (bwide: the rows of consecutive digits are
// consecutive, so one MMA descriptor spans several digits) or
// [slice][chunk][64][16 B] (one MMA per digit pair, RBA_OZ_WIDE=0);
// k interleaved with the real/imaginary part inside each 16 B.
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
                                                  int64_t split_pole, double* __restrict__ scl,
                                                  int64_t exp_pole, int bwide, int* __restrict__ ticket) {
  __shared__ int s_e[64];
  __shared__ double s_m[2][64];
  const int slot = blockIdx.y;
  // the next (pole, tile) item of the k_oz_gemm launch that follows on this stream
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *ticket = 0;
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
    if (on) scl[(int64_t)slot * exp_pole + tk.exp_off + row] = ldexp(1.0, s_e[r] - 54);   // 2^(e_r - 54)
  }
  __syncthreads();
  const int e = s_e[r];
  // pass 2: digits, thread = (row r, chunk h of 8 complex k) per k step
  const int blkb = bwide == 2 ? OZ_BLK2 : OZ_BLK;
  // the B view is only streamed for column tiles (rows c_lo .. c_hi - 1 of the region)
  const bool need_b = rt * 64 < tk.c_hi - c_lo;
  unsigned char* out = split + (int64_t)slot * split_pole + tk.split_off + (int64_t)rt * tk.nks * blkb;
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
    unsigned char* blk = out + (int64_t)ks * blkb;
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
      *reinterpret_cast<uint4*>(blk + ((t * 2 + h) * 128 + 2 * r) * 16) = wre;
      *reinterpret_cast<uint4*>(blk + ((t * 2 + h) * 128 + 2 * r + 1) * 16) = wim;
      if (!need_b) continue;
      if (bwide == 2) {
        // cluster pair: rank q holds, per group of consecutive B digits that one
        // cta_group::2 MMA spans, ITS half of the group's rows ([chunk][rows]):
        // {1234}: digits 1,2 | 3,4; {56}: 5 | 6; {12}: 1 | 2; {7},{5},{3},{1}: rows 0-31 | 32-63
        unsigned char* b0 = blk + OZ_ABYTES;
        unsigned char* b1 = b0 + OZ_B2;
        unsigned char* bh = (r >> 5) ? b1 : b0;          // half-row groups
        const int r5 = r & 31;
        auto put = [&](unsigned char* base, int goff, int nrows, int row) {
          *reinterpret_cast<uint4*>(base + goff + (h * nrows + row) * 16) = wb;
        };
        switch (t) {
          case 0: put(b0, OZ_G1, 128, r); put(b0, OZ_G5, 64, r); put(bh, OZ_G7, 32, r5); break;
          case 1: put(b0, OZ_G1, 128, 64 + r); put(b1, OZ_G5, 64, r); break;
          case 2: put(b1, OZ_G1, 128, r); put(bh, OZ_G6, 32, r5); break;
          case 3: put(b1, OZ_G1, 128, 64 + r); break;
          case 4: put(b0, OZ_G2, 64, r); put(bh, OZ_G4, 32, r5); break;
          case 5: put(b1, OZ_G2, 64, r); break;
          default: put(bh, OZ_G3, 32, r5); break;
        }
      } else {
        const int boff = bwide ? (h * OZ_S + t) * 64 + r : (t * 2 + h) * 64 + r;
        *reinterpret_cast<uint4*>(blk + OZ_ABYTES + boff * 16) = wb;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// INT8 tensor-core GEMM, persistent and warp-specialised (192 threads):
// warp 0 / lane 0 streams the digit blocks (bulk copies into a 4-stage
// mbarrier ring, straight across tile boundaries), warp 1 / lane 0 issues the
// 28 digit-pair MMAs per k step into the 7 TMEM level accumulators, warps 2..9
// (TMEM lanes 32 (w mod 4) ..., columns 32 ((w - 2) / 4) ...) read the
// accumulators, hand TMEM back to the MMA warp and only then do the
// read-modify-write of C -- so the global epilogue of one tile overlaps the
// MMAs of the next.  Items (pole, tile) are
// handed out by a global ticket (the producer draws it and passes the item to
// the other roles through a shared-memory ring), so the ~148 tiles in flight
// are always consecutive in the super-block tile order and share their digit
// streams in L2 even when the CTAs drift apart; each tile is still computed
// by exactly one CTA in a fixed k and level order (deterministic).
// ---------------------------------------------------------------------------
template <int OZ_NLD>                        // stages of the load ring
struct OzSmem {
  unsigned char st[OZ_NLD][OZ_BLK];          // [stage][A_big | B] digit blocks
  uint64_t full[OZ_NLD], empty[OZ_NLD];
  uint64_t tfull, tempty;                    // accumulators: MMA -> epilogue -> MMA
  uint32_t tbase;
  // items drawn by the producer: (sequence number << 32) | item, item -1 = no more
  volatile unsigned long long itemq[8];
};
__device__ __forceinline__ unsigned long long oz_qent(int seq, int item) {
  return ((unsigned long long)(uint32_t)seq << 32) | (uint32_t)item;
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

#ifndef OZ_PF
#define OZ_PF 1   // L2 prefetch of the C tile by the epilogue threads while the tile's MMAs run
#endif
// Epilogue of one tile for one thread (TMEM lane 32 wq + lane, columns 32 ch ..):
// wait for the accumulators, drain them, hand TMEM back, update C.
template <bool REMOTE>
__device__ __forceinline__ void oz_tile_epilogue(const OzTask& tk, int slot, int tr, int tj, bool rows_on,
                                                 const FrontsDev& F, const PoleBatch& pb,
                                                 const double* __restrict__ scl, int64_t exp_pole,
                                                 uint32_t tb, int wq, int ch, int lane, uint64_t* tfull,
                                                 uint32_t tfull_parity, uint32_t tempty_addr,
                                                 long long& w_acc, long long& t_drain, long long& t_rmw) {
    const int arow = wq * 32 + lane;
    const int imag = arow & 1;
    const int lr = arow >> 1;
    // this thread's part of the C tile: row grow, columns gc0 .. gc0 + jm - 1
    // (lower triangle, inside [c_lo, c_hi)); columns < npiv live in the
    // panel (stride nf), the others in the packed update block (column j + 1
    // starts b - j - 1 elements after column j at the same row)
    const int s = tk.s, nf = tk.nf, c_lo = tk.c_lo, c_hi = tk.c_hi;
    const int p = F.npiv[s];
    const int b = nf - c_lo;
    const int grow = tr * 64 + lr, gc0 = tj * 64 + ch * 32;
    const int jm = (rows_on && grow < b) ? min(32, min(c_hi - c_lo - gc0, grow - gc0 + 1)) : 0;
    const double* sc = scl + (int64_t)slot * exp_pole + tk.exp_off;
    const double si = jm > 0 ? __ldg(sc + grow) : 0.0;
    const bool inpanel = c_hi <= p;
    double* const ptr0 =
        reinterpret_cast<double*>(faddr(pb.factor[slot] + F.panel_off[s],
                                        pb.upd[slot] + (F.upd_off[s] >= 0 ? F.upd_off[s] : 0), p, nf,
                                        c_lo + grow, c_lo + gc0)) + imag;
    const int64_t step0 = inpanel ? 2 * (int64_t)nf : 2 * (int64_t)(nf - (c_lo + gc0) - 1);
    const int64_t dstep = inpanel ? 0 : -2;
    if (OZ_PF) {  // pull this thread's part of the tile into L2 while its MMAs run
      double* pf = ptr0;
      int64_t st = step0;
      for (int j = 0; j < jm; ++j) {
        asm volatile("prefetch.global.L2 [%0];\n" :: "l"(pf));
        pf += st;
        st += dstep;
      }
    }
    const long long c0 = clock64();
    mbar_wait_(tfull, tfull_parity);
    const long long c1 = clock64();
    w_acc += c1 - c0;
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    // sum_d 256^(14 - d) acc_d: levels (2,3,4), (5,6), (7,8) are combined exactly in
    // int64 (< 2^48) and converted by the 2^52 + 2^51 offset (exact), then three FP64 terms
    double acc[32];
#pragma unroll
    for (int cb = 0; cb < 32; cb += 8) {
      uint32_t v[OZ_LEV][8];
#pragma unroll
      for (int d = 0; d < OZ_LEV; ++d) {
        const uint32_t taddr = tb + (uint32_t)(d * 64 + ch * 32 + cb) + ((uint32_t)(wq * 32) << 16);
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                     : "=r"(v[d][0]), "=r"(v[d][1]), "=r"(v[d][2]), "=r"(v[d][3]), "=r"(v[d][4]),
                       "=r"(v[d][5]), "=r"(v[d][6]), "=r"(v[d][7])
                     : "r"(taddr));
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      constexpr long long MAGIC = 0x4338000000000000LL;       // bits of 2^52 + 2^51
      constexpr double MAGICD = 6755399441055744.0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const long long hi = (long long)(int32_t)v[0][i] * 65536 + (long long)(int32_t)v[1][i] * 256 +
                             (long long)(int32_t)v[2][i];
        const long long mid = (long long)(int32_t)v[3][i] * 256 + (long long)(int32_t)v[4][i];
        const long long lo = (long long)(int32_t)v[5][i] * 256 + (long long)(int32_t)v[6][i];
        const double dhi = __longlong_as_double(hi + MAGIC) - MAGICD;
        const double dmid = __longlong_as_double(mid + MAGIC) - MAGICD;
        const double dlo = __longlong_as_double(lo + MAGIC) - MAGICD;
        // weights 256^10, 256^8, 256^6
        acc[cb + i] = fma(dhi, 1208925819614629174706176.0, fma(dmid, 18446744073709551616.0, dlo * 281474976710656.0)) * si;
      }
    }
    // TMEM is free for the next tile's MMAs
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    if (REMOTE)
      asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" :: "r"(tempty_addr) : "memory");
    else
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" :: "r"(tempty_addr) : "memory");
    const long long c2 = clock64();
    t_drain += c2 - c1;
    if (jm > 0) {
      double* pl = ptr0;
      double* ps = ptr0;
      int64_t stl = step0, sts = step0;
#pragma unroll
      for (int cb = 0; cb < 32; cb += 16) {
        double cur[16], sj[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const bool on = cb + i < jm;
          cur[i] = on ? __ldcg(pl) : 0.0;
          sj[i] = on ? __ldg(sc + gc0 + cb + i) : 0.0;
          pl += stl;
          stl += dstep;
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          if (cb + i < jm) *ps = fma(-acc[cb + i], sj[i], cur[i]);
          ps += sts;
          sts += dstep;
        }
      }
    }
    t_rmw += clock64() - c2;
}

// cycle counters of the three roles, summed over CTAs (rba_oz_prof): [0] MMA
// issuer loop, [1] its waits for data, [2] its waits for TMEM, [3] producer
// waits for a free stage, [4] epilogue waits for accumulators, [5] TMEM drain,
// [6] global read-modify-write, [7] k steps, [8] tiles, [9] issuer loop in ns
__device__ unsigned long long g_oz_prof[10];

constexpr int OZ_THREADS = 320;
// TS = true: the A digit of each (k step, t) is copied once from shared memory
// into one of 8 TMEM slots of 8 columns (448..511, beside the 7 level
// accumulators) by tcgen05.cp and its 1-2 wide MMAs read A from TMEM: per k
// step the shared-memory port then carries 56 KB of B reads + 28 KB of copy
// reads + 42 KB of bulk-copy writes = 126 KB instead of 138 KB, and -- what
// matters -- only 86 B/clk while the MMAs run, which leaves the bulk copies the
// 42 B/clk they need (with A from shared memory the MMAs take 104 of the 128
// B/clk and the copies starve: 15 % of the issuer's time went into waiting
// for data).  tcgen05.cp and tcgen05.mma of one thread execute in issue order
// (one pipeline), so the copy that rewrites a slot 8 digits later runs after
// the MMAs that read it: no barrier (with a commit + wait per digit the
// issuer lost its run-ahead and the k step took 2,660 clocks).  Same integer
// sums: bitwise equal.
template <bool WIDE, int OZ_NLD, bool TS = false>
__global__ void __launch_bounds__(OZ_THREADS, 1) k_oz_gemm(const OzTask* __restrict__ tasks, int ntasks,
                                                    const int2* __restrict__ tiles, int ntiles,
                                                    FrontsDev F, PoleBatch pb,
                                                    const unsigned char* __restrict__ split,
                                                    int64_t split_pole, const double* __restrict__ scl,
                                                    int64_t exp_pole, int* __restrict__ ticket) {
  extern __shared__ __align__(1024) unsigned char oz_raw[];
  OzSmem<OZ_NLD>& S = *reinterpret_cast<OzSmem<OZ_NLD>*>(oz_raw);
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
    mbar_init_(&S.tempty, OZ_THREADS - 64);
    for (int q = 0; q < 8; ++q) S.itemq[q] = ~0ull;   // no sequence number matches
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tb = S.tbase;

  if (tid == 0) {
    // ---- producer ----
    int g = 0;
    long long w_empty = 0;
    for (int n = 0;; ++n) {
      int item = atomicAdd(ticket, 1);
      if (item >= nitems) item = -1;
      S.itemq[n & 7] = oz_qent(n, item);   // released by the arrive on the item's first stage
      if (item < 0) {                      // an empty stage carries the end marker
        const int q = g % OZ_NLD;
        if (g >= OZ_NLD) mbar_wait_(&S.empty[q], ((g / OZ_NLD) - 1) & 1);
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" :: "r"(su32(&S.full[q])) : "memory");
        break;
      }
      int slot, tr, tj;
      OzTask tk;
      oz_item(tasks, ntasks, tiles, ntiles, item, slot, tk, tr, tj);
      const unsigned char* sp = split + (int64_t)slot * split_pole + tk.split_off;
      const unsigned char* srcA = sp + (int64_t)tr * tk.nks * OZ_BLK;
      const unsigned char* srcB = sp + (int64_t)tj * tk.nks * OZ_BLK + OZ_ABYTES;
      for (int ks = 0; ks < tk.nks; ++ks, ++g) {
        const int q = g % OZ_NLD;
        if (g >= OZ_NLD) {
          const long long c0 = clock64();
          mbar_wait_(&S.empty[q], ((g / OZ_NLD) - 1) & 1);
          w_empty += clock64() - c0;
        }
        const uint32_t bar = su32(&S.full[q]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" :: "r"(bar), "r"(OZ_ABYTES + OZ_BBYTES) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                     :: "r"(su32(S.st[q])), "l"(srcA + (int64_t)ks * OZ_BLK), "r"(OZ_ABYTES), "r"(bar) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                     :: "r"(su32(S.st[q] + OZ_ABYTES)), "l"(srcB + (int64_t)ks * OZ_BLK), "r"(OZ_BBYTES), "r"(bar) : "memory");
      }
    }
    atomicAdd(&g_oz_prof[3], (unsigned long long)w_empty);
  } else if (tid == 32) {
    // ---- MMA issuer ----
    int g = 0, it = 0;
    long long w_full = 0, w_tmem = 0;
    const long long cstart = clock64();
    unsigned long long nstart;
    asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(nstart));
    for (;; ++it) {
      {  // the item arrives with its first stage
        const long long c0 = clock64();
        mbar_wait_(&S.full[g % OZ_NLD], (g / OZ_NLD) & 1);
        w_full += clock64() - c0;
      }
      const int item = (int)(uint32_t)S.itemq[it & 7];
      if (it > 0) {
        const long long c0 = clock64();
        mbar_wait_(&S.tempty, (it - 1) & 1);     // epilogue drained TMEM
        w_tmem += clock64() - c0;
      }
      if (item < 0) break;
      int slot, tr, tj;
      OzTask tk;
      oz_item(tasks, ntasks, tiles, ntiles, item, slot, tk, tr, tj);
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      for (int ks = 0; ks < tk.nks; ++ks, ++g) {
        const int q = g % OZ_NLD;
        if (ks > 0) {
          const long long c0 = clock64();
          mbar_wait_(&S.full[q], (g / OZ_NLD) & 1);
          w_full += clock64() - c0;
        }
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        const uint32_t abase = su32(S.st[q]), bbase = abase + OZ_ABYTES;
        if constexpr (WIDE && TS) {
#pragma unroll
          for (int t = 1; t <= OZ_S; ++t) {
            const int n = g * OZ_S + (t - 1);          // global A digit counter
            const int sl = n & 7;
            const uint32_t ta = tb + 448 + sl * 8;
            asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;\n"
                         :: "r"(ta), "l"(umma_desc(abase + (t - 1) * 2 * 128 * 16, 128 * 16, 128)));
#pragma unroll
            for (int u0 = 1; u0 <= 8 - t; u0 += 4) {
              const int nu = (8 - t - u0 + 1) < 4 ? (8 - t - u0 + 1) : 4;
              const uint64_t db = umma_desc(bbase + (u0 - 1) * 64 * 16, OZ_S * 64 * 16, 128);
              asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                           " tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n"
                           :: "r"(tb + (uint32_t)((t + u0 - 2) * 64)), "r"(ta), "l"(db), "r"(oz_idesc(64 * nu)),
                              "r"((ks > 0 || t > 1) ? 1 : 0));
            }
          }
        } else if constexpr (WIDE) {
          // A digit t x B digits u0..u1 -> levels t + u0 .. t + u1 (TMEM columns
          // 64 (t + u0 - 2) ...): integer sums, so the order does not matter
#pragma unroll
          for (int t = 1; t <= OZ_S; ++t) {
            const uint64_t da = umma_desc(abase + (t - 1) * 2 * 128 * 16, 128 * 16, 128);
#pragma unroll
            for (int u0 = 1; u0 <= 8 - t; u0 += 4) {
              const int nu = (8 - t - u0 + 1) < 4 ? (8 - t - u0 + 1) : 4;
              const uint64_t db = umma_desc(bbase + (u0 - 1) * 64 * 16, OZ_S * 64 * 16, 128);
              mma_i8(tb + (t + u0 - 2) * 64, da, db, oz_idesc(64 * nu), (ks > 0 || t > 1) ? 1 : 0);
            }
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
              mma_i8(tb + (d - 2) * 64, da, db, oz_idesc(64), (ks > 0 || t > 1) ? 1 : 0);
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
                     :: "r"(su32(&S.empty[q])) : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
                   :: "r"(su32(&S.tfull)) : "memory");
    }
    atomicAdd(&g_oz_prof[0], (unsigned long long)(clock64() - cstart));
    atomicAdd(&g_oz_prof[1], (unsigned long long)w_full);
    atomicAdd(&g_oz_prof[2], (unsigned long long)w_tmem);
    atomicAdd(&g_oz_prof[7], (unsigned long long)g);
    atomicAdd(&g_oz_prof[8], (unsigned long long)it);
    unsigned long long nend;
    asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(nend));
    atomicAdd(&g_oz_prof[9], nend - nstart);
  } else if (warp >= 2) {
    // ---- epilogue: warp w reads TMEM lanes 32 (w mod 4) .. +31, columns 32 ch .. +31 ----
    // lane 2 r / 2 r + 1 = real / imaginary part of complex row r of the tile
    const int wq = warp & 3;
    const int ch = (warp - 2) >> 2;
    int it = 0;
    long long w_acc = 0, t_drain = 0, t_rmw = 0;
    for (;; ++it) {
      // the item is published by the producer well before its MMAs finish
      unsigned long long qe;
      do qe = S.itemq[it & 7]; while ((int)(qe >> 32) != it);
      const int item = (int)(uint32_t)qe;
      if (item < 0) break;
      int slot, tr, tj;
      OzTask tk;
      oz_item(tasks, ntasks, tiles, ntiles, item, slot, tk, tr, tj);
      oz_tile_epilogue<false>(tk, slot, tr, tj, true, F, pb, scl, exp_pole, tb, wq, ch, lane, &S.tfull,
                              (uint32_t)(it & 1), su32(&S.tempty), w_acc, t_drain, t_rmw);
    }
    if (tid == 64) {
      atomicAdd(&g_oz_prof[4], (unsigned long long)w_acc);
      atomicAdd(&g_oz_prof[5], (unsigned long long)t_drain);
      atomicAdd(&g_oz_prof[6], (unsigned long long)t_rmw);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" :: "r"(tb));
}

// ---------------------------------------------------------------------------
// Cluster-pair GEMM (RBA_OZ_2CTA=1): the two CTAs of a cluster (two SMs) run
// tcgen05.mma.cta_group::2 (M = 256: row tiles 2 i and 2 i + 1, one column
// tile): each CTA streams its own A block and only ITS HALF of the B rows of
// every MMA, so per SM and k step the MMAs read 48 KB of A + 28 KB of B from
// shared memory (one-SM kernel: 40 + 56 KB) and the bulk copies write 40 KB
// (42 KB): 116 KB instead of 138 KB through the 128 B/clk shared-memory port
// that bounds the one-SM kernel.  The 28 digit pairs are 12 MMAs: A digit t x
// B digit groups {1234},{56},{7} (t = 1), {1234},{56} (2), {1234},{5} (3),
// {1234} (4), {12},{3} (5), {12} (6), {1} (7); a group's first half of rows
// (in digit-major order) lives in rank 0, the second in rank 1, at the same
// shared-memory offset (k_oz_split writes both arrangements).
// The leader issues the MMAs; a bulk copy completes only on a barrier of its
// own CTA, so a relay thread of the peer forwards each landed stage to the
// leader's stage barrier (count 2); commits are multicast to both CTAs; both
// CTAs' epilogues arrive on the leader's "TMEM free" barrier.  The leader's
// producer draws the ticket and publishes the item in both CTAs.
// Same exact integer sums as k_oz_gemm: bitwise equal results.
// ---------------------------------------------------------------------------
constexpr int OZ_NLD2 = 5;
struct OzSmem2 {
  unsigned char st[OZ_NLD2][OZ_ABYTES + OZ_B2];
  uint64_t full[OZ_NLD2], empty[OZ_NLD2];
  uint64_t pfull[OZ_NLD2];                   // leader: the peer's stage has landed
  uint64_t tfull, tempty;
  uint32_t tbase;
  volatile unsigned long long itemq[8];
};
__host__ __device__ constexpr uint32_t oz_idesc2(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}
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
__device__ __forceinline__ uint32_t map_to_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void mma_i8_2(uint32_t dtmem, uint64_t da, uint64_t db, uint32_t idesc, int acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
               " tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n"
               :: "r"(dtmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(OZ_THREADS, 1)
k_oz_gemm2(const OzTask* __restrict__ tasks, int ntasks, const int2* __restrict__ tiles, int ntiles,
           FrontsDev F, PoleBatch pb, const unsigned char* __restrict__ split, int64_t split_pole,
           const double* __restrict__ scl, int64_t exp_pole, int* __restrict__ ticket) {
  extern __shared__ __align__(1024) unsigned char oz_raw2[];
  OzSmem2& S = *reinterpret_cast<OzSmem2*>(oz_raw2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(rank));
  const int nitems = ntiles * pb.count;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" :: "r"(su32(&S.tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  if (tid == 32) {
    for (int q = 0; q < OZ_NLD2; ++q) {
      mbar_init_(&S.full[q], 1);
      mbar_init_(&S.pfull[q], 1);
      mbar_init_(&S.empty[q], 1);
    }
    mbar_init_(&S.tfull, 1);
    mbar_init_(&S.tempty, 2 * (OZ_THREADS - 64));
    for (int q = 0; q < 8; ++q) S.itemq[q] = ~0ull;
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  cluster_sync_();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tb = S.tbase;
  // item n of this pair: published by the leader's producer in both CTAs
  auto get_item = [&](int n) -> int {
    unsigned long long qe;
    do qe = S.itemq[n & 7]; while ((int)(qe >> 32) != n);
    return (int)(uint32_t)qe;
  };

  if (tid == 0) {
    // ---- producer (both CTAs): own A block + own B arrangement ----
    int g = 0;
    for (int n = 0;; ++n) {
      int item;
      if (rank == 0) {
        item = atomicAdd(ticket, 1);
        if (item >= nitems) item = -1;
        const unsigned long long qe = oz_qent(n, item);
        asm volatile("st.shared::cluster.u64 [%0], %1;\n" :: "r"(map_to_rank(su32((const void*)&S.itemq[n & 7]), 1)), "l"(qe) : "memory");
        S.itemq[n & 7] = qe;
      } else {
        item = get_item(n);
      }
      if (item < 0) break;
      int slot, tr2, tj;
      OzTask tk;
      oz_item(tasks, ntasks, tiles, ntiles, item, slot, tk, tr2, tj);
      const int tr = 2 * tr2 + (int)rank;
      const unsigned char* sp = split + (int64_t)slot * split_pole + tk.split_off;
      const unsigned char* srcA = sp + (int64_t)tr * tk.nks * OZ_BLK2;
      const unsigned char* srcB = sp + (int64_t)tj * tk.nks * OZ_BLK2 + OZ_ABYTES + rank * OZ_B2;
      for (int ks = 0; ks < tk.nks; ++ks, ++g) {
        const int q = g % OZ_NLD2;
        if (g >= OZ_NLD2) mbar_wait_(&S.empty[q], ((g / OZ_NLD2) - 1) & 1);
        const uint32_t bar = su32(&S.full[q]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n"
                     :: "r"(bar), "r"(OZ_ABYTES + OZ_B2) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                     :: "r"(su32(S.st[q])), "l"(srcA + (int64_t)ks * OZ_BLK2), "r"(OZ_ABYTES), "r"(bar) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                     :: "r"(su32(S.st[q] + OZ_ABYTES)), "l"(srcB + (int64_t)ks * OZ_BLK2), "r"(OZ_B2), "r"(bar) : "memory");
      }
    }
  } else if (tid == 32 && rank == 1) {
    // ---- relay (peer): forward each landed stage to the leader's barrier ----
    int g = 0;
    for (int n = 0;; ++n) {
      const int item = get_item(n);
      if (item < 0) break;
      int slot, tr2, tj;
      OzTask tk;
      oz_item(tasks, ntasks, tiles, ntiles, item, slot, tk, tr2, tj);
      for (int ks = 0; ks < tk.nks; ++ks, ++g) {
        const int q = g % OZ_NLD2;
        mbar_wait_(&S.full[q], (g / OZ_NLD2) & 1);
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n"
                     :: "r"(map_to_rank(su32(&S.pfull[q]), 0)) : "memory");
      }
    }
  } else if (tid == 32 && rank == 0) {
    // ---- MMA issuer (leader) ----
    int g = 0, it = 0;
    long long w_full = 0, w_tmem = 0, w_peer = 0;
    const long long cstart = clock64();
    unsigned long long nstart;
    asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(nstart));
    for (;; ++it) {
      const int item = get_item(it);
      if (it > 0) {
        const long long c0 = clock64();
        mbar_wait_cl_(&S.tempty, (it - 1) & 1);
        w_tmem += clock64() - c0;
      }
      if (item < 0) break;
      int slot, tr2, tj;
      OzTask tk;
      oz_item(tasks, ntasks, tiles, ntiles, item, slot, tk, tr2, tj);
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      for (int ks = 0; ks < tk.nks; ++ks, ++g) {
        const int q = g % OZ_NLD2;
        {
          const long long c0 = clock64();
          mbar_wait_(&S.full[q], (g / OZ_NLD2) & 1);
          const long long c1 = clock64();
          mbar_wait_cl_(&S.pfull[q], (g / OZ_NLD2) & 1);
          w_full += c1 - c0;
          w_peer += clock64() - c1;
        }
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        const uint32_t abase = su32(S.st[q]), bbase = abase + OZ_ABYTES;
        const int acc0 = ks > 0 ? 1 : 0;
        auto A = [&](int t) { return umma_desc(abase + (t - 1) * 2 * 128 * 16, 128 * 16, 128); };
        auto B = [&](int goff, int nrows) { return umma_desc(bbase + goff, nrows * 16, 128); };
        auto D = [&](int t, int u) { return tb + (uint32_t)((t + u - 2) * 64); };
        mma_i8_2(D(1, 1), A(1), B(OZ_G1, 128), oz_idesc2(256), acc0);
        mma_i8_2(D(1, 5), A(1), B(OZ_G2, 64), oz_idesc2(128), acc0);
        mma_i8_2(D(1, 7), A(1), B(OZ_G3, 32), oz_idesc2(64), acc0);
        mma_i8_2(D(2, 1), A(2), B(OZ_G1, 128), oz_idesc2(256), 1);
        mma_i8_2(D(2, 5), A(2), B(OZ_G2, 64), oz_idesc2(128), 1);
        mma_i8_2(D(3, 1), A(3), B(OZ_G1, 128), oz_idesc2(256), 1);
        mma_i8_2(D(3, 5), A(3), B(OZ_G4, 32), oz_idesc2(64), 1);
        mma_i8_2(D(4, 1), A(4), B(OZ_G1, 128), oz_idesc2(256), 1);
        mma_i8_2(D(5, 1), A(5), B(OZ_G5, 64), oz_idesc2(128), 1);
        mma_i8_2(D(5, 3), A(5), B(OZ_G6, 32), oz_idesc2(64), 1);
        mma_i8_2(D(6, 1), A(6), B(OZ_G5, 64), oz_idesc2(128), 1);
        mma_i8_2(D(7, 1), A(7), B(OZ_G7, 32), oz_idesc2(64), 1);
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n"
                     :: "r"(su32(&S.empty[q])), "h"((unsigned short)3) : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n"
                   :: "r"(su32(&S.tfull)), "h"((unsigned short)3) : "memory");
    }
    atomicAdd(&g_oz_prof[0], (unsigned long long)(clock64() - cstart));
    atomicAdd(&g_oz_prof[1], (unsigned long long)w_full);
    atomicAdd(&g_oz_prof[2], (unsigned long long)w_tmem);
    atomicAdd(&g_oz_prof[3], (unsigned long long)w_peer);       // (pair kernel: waits for the peer's stage)
    atomicAdd(&g_oz_prof[7], (unsigned long long)(2 * g));      // k steps of two tiles
    atomicAdd(&g_oz_prof[8], (unsigned long long)(2 * it));
    unsigned long long nend;
    asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(nend));
    atomicAdd(&g_oz_prof[9], nend - nstart);
  } else if (warp >= 2) {
    // ---- epilogue (both CTAs): own 128 TMEM lanes = own 64 complex rows ----
    const int wq = warp & 3;
    const int ch = (warp - 2) >> 2;
    const uint32_t tempty_leader = map_to_rank(su32(&S.tempty), 0);
    int it = 0;
    long long w_acc = 0, t_drain = 0, t_rmw = 0;
    for (;; ++it) {
      const int item = get_item(it);
      if (item < 0) break;
      int slot, tr2, tj;
      OzTask tk;
      oz_item(tasks, ntasks, tiles, ntiles, item, slot, tk, tr2, tj);
      const int tr = 2 * tr2 + (int)rank;
      oz_tile_epilogue<true>(tk, slot, tr, tj, tr < tk.nrt, F, pb, scl, exp_pole, tb, wq, ch, lane, &S.tfull,
                             (uint32_t)(it & 1), tempty_leader, w_acc, t_drain, t_rmw);
    }
    if (tid == 64 && rank == 0) {
      atomicAdd(&g_oz_prof[4], (unsigned long long)w_acc);
      atomicAdd(&g_oz_prof[5], (unsigned long long)(2 * t_drain));
      atomicAdd(&g_oz_prof[6], (unsigned long long)(2 * t_rmw));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  cluster_sync_();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" :: "r"(tb));
}

void oz_prof_read(unsigned long long* out, bool reset) {
  cudaMemcpyFromSymbol(out, g_oz_prof, sizeof(unsigned long long) * 10);
  if (reset) {
    unsigned long long z[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_oz_prof, z, sizeof(z));
  }
}

void launch_oz_schur(cudaStream_t st, const OzTask* tasks, int ntasks, const int2* tiles,
                     int nrowtiles, int ntiles, const FrontsDev& F, const PoleBatch& pb,
                     unsigned char* split, int64_t split_pole, double* scl, int64_t exp_pole,
                     int wide, int* ticket) {
  if (ntasks <= 0 || ntiles <= 0) return;
  k_oz_split<<<dim3(nrowtiles, pb.count), 128, 0, st>>>(tasks, ntasks, F, pb, split,
                                                        split_pole, scl, exp_pole, wide == 3 ? 2 : (wide != 0), ticket);
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  const int items = ntiles * pb.count;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_oz_gemm<false, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(OzSmem<4>) + 1024);
    cudaFuncSetAttribute(k_oz_gemm<true, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(OzSmem<4>) + 1024);
    cudaFuncSetAttribute(k_oz_gemm<true, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(OzSmem<5>) + 1024);
    cudaFuncSetAttribute(k_oz_gemm<true, 4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(OzSmem<4>) + 1024);
    cudaFuncSetAttribute(k_oz_gemm<true, 5, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(OzSmem<5>) + 1024);
    attr = true;
  }
  const int grid = std::min(items, nsm);
  if (wide == 3) {
    const size_t smem2 = sizeof(OzSmem2) + 1024;
    static bool attr2 = false;
    if (!attr2) {
      cudaFuncSetAttribute(k_oz_gemm2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
      attr2 = true;
    }
    const int npairs = std::min(items, nsm / 2);
    k_oz_gemm2<<<2 * npairs, OZ_THREADS, smem2, st>>>(tasks, ntasks, tiles, ntiles, F, pb, split, split_pole,
                                                     scl, exp_pole, ticket);
    return;
  }
  if (wide == 4)
    k_oz_gemm<true, 4, true><<<grid, OZ_THREADS, sizeof(OzSmem<4>) + 1024, st>>>(tasks, ntasks, tiles, ntiles, F, pb,
                                                                                split, split_pole, scl, exp_pole, ticket);
  else if (wide == 5)
    k_oz_gemm<true, 5, true><<<grid, OZ_THREADS, sizeof(OzSmem<5>) + 1024, st>>>(tasks, ntasks, tiles, ntiles, F, pb,
                                                                                split, split_pole, scl, exp_pole, ticket);
  else if (wide == 2)
    k_oz_gemm<true, 5><<<grid, OZ_THREADS, sizeof(OzSmem<5>) + 1024, st>>>(tasks, ntasks, tiles, ntiles, F, pb, split,
                                                                          split_pole, scl, exp_pole, ticket);
  else if (wide)
    k_oz_gemm<true, 4><<<grid, OZ_THREADS, sizeof(OzSmem<4>) + 1024, st>>>(tasks, ntasks, tiles, ntiles, F, pb, split,
                                                                          split_pole, scl, exp_pole, ticket);
  else
    k_oz_gemm<false, 4><<<grid, OZ_THREADS, sizeof(OzSmem<4>) + 1024, st>>>(tasks, ntasks, tiles, ntiles, F, pb, split,
                                                                           split_pole, scl, exp_pole, ticket);
}

}  // namespace rba
