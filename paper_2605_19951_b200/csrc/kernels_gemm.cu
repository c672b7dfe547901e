// K4 on the FP64 tensor cores: the panel TRSM and the complex trailing / Schur
// update of the fronts
//     C[r,c] -= sum_t L'[r,t] L'[c,t]        (lower triangle, r >= c)
// with L' = L D^{1/2} (factor format, fronts.cuh), using warp-level DMMA
// (mma.sync.m8n8k4.f64 -> SASS DMMA.8 on sm_100a; the tcgen05 UMMA has no f64
// kind).  Kernels: v3 (k_gemm3: cp.async pipeline; MODE 1 is the
// default TRSM), v5 (k_gemm5: bulk copies into an mbarrier ring, 4-multiply
// complex products), v6/v8 (k_gemm6: 3-multiply complex products, v8 = TMA
// tensor-map operands, the default update).  All tile lists come from the
// same GemmTask / PanelTask descriptors as the DFMA reference kernel
// (kernels_factor.cu, k_gemm_update).
#include "fronts.cuh"
#include "kernels.h"

#include <cstdlib>

namespace rba {

namespace {
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ int find_task(const GemmTask* tasks, int n, int b) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (tasks[mid].tile_start <= b) lo = mid; else hi = mid - 1;
  }
  return lo;
}

}  // namespace

// ---------------------------------------------------------------------------
// v3: 64x64 CTA tile, 8 warps of 32x16 (<=128 registers: 2 CTAs = 16 warps/SM), interleaved complex [row][k]
// shared-memory tiles filled by cp.async (16 B, zero-fill out of range) in a
// 3-stage pipeline with one barrier per stage; one LDS.128 yields both the re
// and im DMMA fragments.  The d_t scaling (MODE 0) and the unit-triangular
// mask of X (MODE 1) are applied to the B fragments in registers.
// ---------------------------------------------------------------------------
namespace {
constexpr int BM3 = 64, BN3 = 64;
constexpr int NT3 = 256;

__device__ __forceinline__ void cp_async16_3(void* smem, const void* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz)
               : "memory");
}
__device__ __forceinline__ void cp_commit3() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait3() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// T3K: k per stage (complex); row stride T3K + 4 (x 16 B) keeps the LDS.128
// fragment loads conflict-free
template <int T3K>
struct Stage3 {
  static constexpr int L3K = T3K + 4;
  cplx a[BM3 * L3K];
  cplx b[BN3 * L3K];
};
}  // namespace

template <int MODE, int T3K, int NS3>
__global__ void __launch_bounds__(NT3, 2) k_gemm3(const GemmTask* __restrict__ tasks, int ntasks,
                                                  const PanelTask* __restrict__ ptasks,
                                                  FrontsDev F, PoleBatch pb) {
  extern __shared__ __align__(16) unsigned char smraw3[];
  using St = Stage3<T3K>;
  constexpr int L3K = St::L3K;
  St* st = reinterpret_cast<St*>(smraw3);
  __shared__ cplx dinv[BN3];
  const int slot = blockIdx.y;
  int s, t0, t1, r0, cc0, cmax, kbase = 0;
  if (MODE == 0) {
    const int ti = find_task(tasks, ntasks, blockIdx.x);
    const GemmTask tk = tasks[ti];
    int local = blockIdx.x - tk.tile_start;
    int j = 0;
    while (local >= tk.ntr - j) { local -= tk.ntr - j; ++j; }
    const int i = j + local;
    s = tk.s; t0 = tk.t0; t1 = tk.t1;
    r0 = tk.c_lo + i * GT;
    cc0 = tk.c_lo + j * GT;
    cmax = min(cc0 + GT, tk.c_hi);
  } else {
    const PanelTask pt = ptasks[blockIdx.x];
    s = pt.s;
    t0 = 0;
    t1 = min(GT, F.npiv[s] - pt.k0);
    kbase = pt.k0;
    r0 = pt.r0;
    cc0 = 0;
    cmax = t1;
  }
  const int nf = F.nf[s], p = F.npiv[s];
  const cplx* __restrict__ panel = pb.factor[slot] + F.panel_off[s];
  cplx* pw = pb.factor[slot] + F.panel_off[s];
  cplx* upd = pb.upd[slot] + (F.upd_off[s] >= 0 ? F.upd_off[s] : 0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 16;
  const int g = lane >> 2, t4 = lane & 3;

  double cre[4][2][2], cim[4][2][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      cre[a][b][0] = cre[a][b][1] = 0.0;
      cim[a][b][0] = cim[a][b][1] = 0.0;
    }
  if (MODE == 1 && tid < BN3)
    dinv[tid] = tid < cmax ? cinv(__ldg(panel + (int64_t)(kbase + tid) * nf + kbase + tid))
                           : cmk(0.0, 0.0);

  const int nchunks = (t1 - t0 + T3K - 1) / T3K;
  auto issue = [&](int ch) {
    if (ch < nchunks) {
      St& S = st[ch % NS3];
      const int kt = t0 + ch * T3K;
#pragma unroll
      for (int q = 0; q < (BM3 * T3K) / NT3; ++q) {
        const int e = tid + q * NT3;
        const int rr = e % BM3, kk = e / BM3;
        const int t = kt + kk;
        const int row = r0 + rr;
        const bool ok = t < t1 && row < nf;
        const int64_t col = MODE == 0 ? (int64_t)t : (int64_t)(kbase + t);
        cp_async16_3(&S.a[rr * L3K + kk], panel + (ok ? col * nf + row : 0), ok);
      }
#pragma unroll
      for (int q = 0; q < (BN3 * T3K) / NT3; ++q) {
        const int e = tid + q * NT3;
        const int rr = e % BN3, kk = e / BN3;
        const int t = kt + kk;
        bool ok;
        const cplx* src;
        if (MODE == 0) {
          ok = t < t1 && cc0 + rr < cmax;
          src = panel + (ok ? (int64_t)t * nf + cc0 + rr : 0);
        } else {
          // X[c][t] at (row kbase+t, col kbase+c); masked to t < c in registers
          ok = t < t1 && rr < cmax;
          src = panel + (ok ? (int64_t)(kbase + rr) * nf + kbase + t : 0);
        }
        cp_async16_3(&S.b[rr * L3K + kk], src, ok);
      }
    }
    cp_commit3();
  };
  for (int c = 0; c < NS3 - 1; ++c) issue(c);
  for (int ch = 0; ch < nchunks; ++ch) {
    cp_wait3<NS3 - 2>();
    __syncthreads();
    issue(ch + NS3 - 1);
    const St& S = st[ch % NS3];
    const int kt = t0 + ch * T3K;
    // warp's 16 columns all past the block / tile edge, or 32 rows past the front
    if (cc0 + wn >= cmax || r0 + wm >= nf) continue;
    // TRSM: X is unit lower triangular (X[c][t] = 0 for t > c), so the k
    // range past the warp's last column contributes nothing
    if (MODE == 1 && kt > wn + 15) continue;
#pragma unroll
    for (int k4 = 0; k4 < T3K; k4 += 4) {
      if (MODE == 1 && kt + k4 > wn + 15) break;
      double ar[4], ai[4], an[4], br[2], bi[2];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const cplx v = S.a[(wm + a * 8 + g) * L3K + k4 + t4];
        ar[a] = v.x;
        ai[a] = v.y;
        an[a] = -v.y;
      }
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        cplx v = S.b[(wn + b * 8 + g) * L3K + k4 + t4];
        if (MODE == 1) {
          const int c = wn + b * 8 + g, t = kt + k4 + t4;
          v = t < c ? v : (t == c ? cmk(1.0, 0.0) : cmk(0.0, 0.0));
        }
        br[b] = v.x;
        bi[b] = v.y;
      }
      // four passes of independent DMMAs: back-to-back MMAs never share an
      // accumulator (the DMMA result latency would stall the warp otherwise)
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) dmma(cre[a][b][0], cre[a][b][1], ar[a], br[b]);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) dmma(cim[a][b][0], cim[a][b][1], ar[a], bi[b]);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) dmma(cre[a][b][0], cre[a][b][1], an[a], bi[b]);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) dmma(cim[a][b][0], cim[a][b][1], ai[a], br[b]);
    }
  }
  cp_wait3<0>();
  __syncthreads();
  if (MODE == 0) {
    // batched read-modify-write: all C loads of two m-tiles in flight at once
#pragma unroll
    for (int a0 = 0; a0 < 4; a0 += 2) {
      cplx* dst[2][2][2];
      cplx cv[2][2][2];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = r0 + wm + (a0 + a) * 8 + g;
            const int c = cc0 + wn + b * 8 + t4 * 2 + h;
            dst[a][b][h] = (r < nf && c < cmax && r >= c) ? faddr(pw, upd, p, nf, r, c) : nullptr;
            cv[a][b][h] = dst[a][b][h] ? __ldcg(dst[a][b][h]) : cmk(0.0, 0.0);
          }
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            if (dst[a][b][h])
              *dst[a][b][h] = cmk(cv[a][b][h].x - cre[a0 + a][b][h], cv[a][b][h].y - cim[a0 + a][b][h]);
    }
  } else {
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = r0 + wm + a * 8 + g;
          const int c = cc0 + wn + b * 8 + t4 * 2 + h;
          if (r < nf && c < cmax)
            pw[(int64_t)(kbase + c) * nf + r] = cmul(cmk(cre[a][b][h], cim[a][b][h]), dinv[c]);
        }
  }
}

template <int MODE, int T3K, int NS3>
static void launch_g3(cudaStream_t st, dim3 grid, const GemmTask* tasks, int ntasks,
                      const PanelTask* ptasks, const FrontsDev& F, const PoleBatch& pb) {
  const size_t smem = NS3 * sizeof(Stage3<T3K>);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_gemm3<MODE, T3K, NS3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    attr = true;
  }
  k_gemm3<MODE, T3K, NS3><<<grid, NT3, smem, st>>>(tasks, ntasks, ptasks, F, pb);
}

// variant 0: 8 k per stage, 3 stages; variant 1: 16 k per stage, 2 stages
void launch_gemm3(cudaStream_t st, const GemmTask* tasks, int ntasks, int nctas,
                  const FrontsDev& F, const PoleBatch& pb, int variant) {
  if (ntasks <= 0 || nctas <= 0) return;
  dim3 grid(nctas, pb.count);
  if (variant == 1) launch_g3<0, 16, 2>(st, grid, tasks, ntasks, nullptr, F, pb);
  else launch_g3<0, 8, 3>(st, grid, tasks, ntasks, nullptr, F, pb);
}

void launch_trsm3(cudaStream_t st, const PanelTask* tasks, int ntasks, const FrontsDev& F,
                  const PoleBatch& pb, int variant) {
  if (ntasks <= 0) return;
  dim3 grid(ntasks, pb.count);
  if (variant == 1) launch_g3<1, 16, 2>(st, grid, nullptr, 0, tasks, F, pb);
  else launch_g3<1, 8, 3>(st, grid, nullptr, 0, tasks, F, pb);
}


// ---------------------------------------------------------------------------
// v5 (trailing/Schur update only): the same 64x64 tile and 8 warps of 32x16 as
// v3, but the operands move by bulk async copies (cp.async.bulk, one 1 KB
// copy per k column of A and of B -- the panel is column-major, so a
// column's 64 rows are contiguous) completing on a per-stage "full" mbarrier.
// There is no CTA-wide barrier in the main loop: each warp waits only for
// its stage's bytes, and the last warp to finish a stage (shared-memory
// counter) refills it.  Smem layout [k][row] with a 66-complex column stride
// keeps the LDS.128 fragment loads conflict-free.  Out-of-range k columns
// are copied from a zero buffer (so they contribute exactly 0); rows and
// columns past the tile edge only feed discarded outputs.
// ---------------------------------------------------------------------------
namespace {
constexpr int G5LD = 66;    // column stride (complex)
constexpr int G5W = 8;      // warps
template <int G5K>          // k per stage (complex)
struct Stage5 {
  cplx a[G5K * G5LD];
  cplx b[G5K * G5LD];
};

}  // namespace

template <int G5K, int NS>
__global__ void __launch_bounds__(32 * G5W, 2) k_gemm5(const GemmTask* __restrict__ tasks, int ntasks,
                                                     FrontsDev F, PoleBatch pb,
                                                     const cplx* __restrict__ zeros) {
  extern __shared__ __align__(128) unsigned char smraw5[];
  using St = Stage5<G5K>;
  St* st = reinterpret_cast<St*>(smraw5);
  __shared__ __align__(8) unsigned long long full[NS];
  __shared__ int cnt[NS];
  const int slot = blockIdx.y;
  const int ti = find_task(tasks, ntasks, blockIdx.x);
  const GemmTask tk = tasks[ti];
  int local = blockIdx.x - tk.tile_start;
  int j = 0;
  while (local >= tk.ntr - j) { local -= tk.ntr - j; ++j; }
  const int i = j + local;
  const int s = tk.s, t0 = tk.t0, t1 = tk.t1;
  const int r0 = tk.c_lo + i * GT;
  const int cc0 = tk.c_lo + j * GT;
  const int cmax = min(cc0 + GT, tk.c_hi);
  const int nf = F.nf[s], p = F.npiv[s];
  const cplx* __restrict__ panel = pb.factor[slot] + F.panel_off[s];
  cplx* pw = pb.factor[slot] + F.panel_off[s];
  cplx* upd = pb.upd[slot] + (F.upd_off[s] >= 0 ? F.upd_off[s] : 0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 16;
  const int g = lane >> 2, t4 = lane & 3;
  const int nchunks = (t1 - t0 + G5K - 1) / G5K;
  const unsigned na = (unsigned)min(GT, nf - r0) * 16u;     // valid A rows (bytes)
  const unsigned nb = (unsigned)min(GT, nf - cc0) * 16u;    // valid B rows (bytes)
  // one warp: lane 0 arms stage ch % NS, the lanes split the copies of chunk ch
  auto issue = [&](int ch) {
    St& S = st[ch % NS];
    const unsigned bar = smem_u32(&full[ch % NS]);
    const int kt = t0 + ch * G5K;
    const int nval = max(0, min(G5K, t1 - kt));
    if (lane == 0)
      mbar_expect_tx(bar, (unsigned)nval * (na + nb) + (unsigned)(G5K - nval) * 2048u);
    for (int q = lane; q < 2 * G5K; q += 32) {
      const int kk = q >> 1;
      const int t = kt + kk;
      cplx* dst = (q & 1) ? &S.b[kk * G5LD] : &S.a[kk * G5LD];
      if (t < t1)
        bulk_g2s(smem_u32(dst), panel + (int64_t)t * nf + ((q & 1) ? cc0 : r0), (q & 1) ? nb : na, bar);
      else
        bulk_g2s(smem_u32(dst), zeros, 1024u, bar);
    }
  };
  if (tid == 0) {
#pragma unroll
    for (int q = 0; q < NS; ++q) {
      mbar_init(smem_u32(&full[q]), 1);
      cnt[q] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == 0)
    for (int ch = 0; ch < min(NS, nchunks); ++ch) issue(ch);

  double cre[4][2][2], cim[4][2][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      cre[a][b][0] = cre[a][b][1] = 0.0;
      cim[a][b][0] = cim[a][b][1] = 0.0;
    }
  for (int ch = 0; ch < nchunks; ++ch) {
    const int sidx = ch % NS;
    mbar_wait(smem_u32(&full[sidx]), (unsigned)((ch / NS) & 1));
    const St& S = st[sidx];
#pragma unroll
    for (int k4 = 0; k4 < G5K; k4 += 4) {
      double ar[4], ai[4], br[2], bi[2];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const cplx v = S.a[(k4 + t4) * G5LD + wm + a * 8 + g];
        ar[a] = v.x;
        ai[a] = v.y;
      }
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const cplx v = S.b[(k4 + t4) * G5LD + wn + b * 8 + g];
        br[b] = v.x;
        bi[b] = v.y;
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) dmma(cre[a][b][0], cre[a][b][1], ar[a], br[b]);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) dmma(cim[a][b][0], cim[a][b][1], ar[a], bi[b]);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) dmma(cre[a][b][0], cre[a][b][1], -ai[a], bi[b]);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) dmma(cim[a][b][0], cim[a][b][1], ai[a], br[b]);
    }
    // stage consumed by this warp; the last warp refills it
    __syncwarp();
    if (ch + NS < nchunks) {
      int last = 0;
      if (lane == 0) {
        __threadfence_block();
        last = atomicAdd(&cnt[sidx], 1) == G5W - 1;
        if (last) {
          __threadfence_block();
          cnt[sidx] = 0;
        }
      }
      if (__shfl_sync(0xffffffffu, last, 0)) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        issue(ch + NS);
      }
    }
  }
  // batched read-modify-write epilogue (as v3)
#pragma unroll
  for (int a0 = 0; a0 < 4; a0 += 2) {
    cplx* dst[2][2][2];
    cplx cv[2][2][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = r0 + wm + (a0 + a) * 8 + g;
          const int c = cc0 + wn + b * 8 + t4 * 2 + h;
          dst[a][b][h] = (r < nf && c < cmax && r >= c) ? faddr(pw, upd, p, nf, r, c) : nullptr;
          cv[a][b][h] = dst[a][b][h] ? __ldcg(dst[a][b][h]) : cmk(0.0, 0.0);
        }
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (dst[a][b][h])
            *dst[a][b][h] = cmk(cv[a][b][h].x - cre[a0 + a][b][h], cv[a][b][h].y - cim[a0 + a][b][h]);
  }
}

template <int G5K, int NS>
static void launch_g5(cudaStream_t st, dim3 grid, const GemmTask* tasks, int ntasks,
                      const FrontsDev& F, const PoleBatch& pb, const cplx* zeros) {
  const size_t smem = NS * sizeof(Stage5<G5K>);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_gemm5<G5K, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  k_gemm5<G5K, NS><<<grid, 32 * G5W, smem, st>>>(tasks, ntasks, F, pb, zeros);
}

// variant 0: 16 k x 3 stages; 1: 8 k x 6 stages
void launch_gemm5(cudaStream_t st, const GemmTask* tasks, int ntasks, int nctas,
                  const FrontsDev& F, const PoleBatch& pb, const cplx* zeros, int variant) {
  if (ntasks <= 0 || nctas <= 0) return;
  dim3 grid(nctas, pb.count);
  if (variant == 1) launch_g5<8, 6>(st, grid, tasks, ntasks, F, pb, zeros);
  else launch_g5<16, 3>(st, grid, tasks, ntasks, F, pb, zeros);
}


// ---------------------------------------------------------------------------
// v6 (trailing/Schur update only): three real DMMA products per complex
// multiply-add instead of four (Gauss / "3M"):
//     P = sum Are Bre,  Q = sum Aim Bim,  T = sum (Are + Aim)(Bre + Bim)
//     Cre -= P - Q,     Cim -= T - P - Q
// 25 % fewer tensor-core instructions for the same result; the real part is
// bit-for-bit the 4M sum, the imaginary part differs by rounding only
// (normwise backward stable; checked against the 4M kernels and the
// reference goldens in tests/test_gpu_factor_structure.py and
// tests/test_gpu_parity.py).  Three accumulator sets cost 96 registers per
// 32x16 warp tile, so the CTA is 4 warps on a 64x32 tile (two CTAs per 64x64
// task tile, blockIdx.x = 2*tile + half) with up to 255 registers, 2 CTAs/SM.
// Operand movement is v5's: bulk async copies (one per k column of A and of
// B) into an mbarrier ring, last warp through a stage refills it.
// ---------------------------------------------------------------------------
namespace {
constexpr int G6LA = 66;    // A column stride (complex): 64 rows + pad
template <int G6K, int NCOL>
struct Stage6 {
  cplx a[G6K * G6LA];
  cplx b[G6K * (NCOL + 2)];  // B column stride: NCOL cols + pad
};
}  // namespace

// NCOL = 32: 4 warps on a 64x32 half tile (2-3 CTAs/SM); NCOL = 64: 8 warps
// on the whole 64x64 tile, up to 255 registers, one CTA/SM.
template <int G6K, int NS, int NCOL, bool TMAP>
__global__ void __launch_bounds__(NCOL * 4, NCOL == 32 ? 2 : 1) k_gemm6(
    const GemmTask* __restrict__ tasks, int ntasks, FrontsDev F, PoleBatch pb,
    const cplx* __restrict__ zeros) {
  constexpr int G6W = NCOL / 8;
  constexpr int G6LB = NCOL + 2;
  constexpr int SPLIT = NCOL == 32 ? 2 : 1;
  extern __shared__ __align__(128) unsigned char smraw6[];
  using St = Stage6<G6K, NCOL>;
  St* st = reinterpret_cast<St*>(smraw6);
  __shared__ __align__(8) unsigned long long full[NS];
  __shared__ int cnt[NS];
  const int slot = blockIdx.y;
  const int tile = blockIdx.x / SPLIT, half = blockIdx.x % SPLIT;
  const int ti = find_task(tasks, ntasks, tile);
  const GemmTask tk = tasks[ti];
  int local = tile - tk.tile_start;
  int j = 0;
  while (local >= tk.ntr - j) { local -= tk.ntr - j; ++j; }
  const int i = j + local;
  const int s = tk.s, t0 = tk.t0, t1 = tk.t1;
  const int r0 = tk.c_lo + i * GT;
  const int cc0 = tk.c_lo + j * GT + half * NCOL;
  const int cmax = min(cc0 + NCOL, tk.c_hi);
  if (cc0 >= cmax) return;                       // right half beyond the column range
  const int nf = F.nf[s], p = F.npiv[s];
  if (cc0 >= nf) return;
  const cplx* __restrict__ panel = pb.factor[slot] + F.panel_off[s];
  cplx* pw = pb.factor[slot] + F.panel_off[s];
  cplx* upd = pb.upd[slot] + (F.upd_off[s] >= 0 ? F.upd_off[s] : 0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 16;
  const int g = lane >> 2, t4 = lane & 3;
  // a warp whose 32x16 block lies strictly above the diagonal only keeps the
  // stage protocol going
  const bool active = r0 + wm + 31 >= cc0 + wn && r0 + wm < nf && cc0 + wn < cmax;
  const int nchunks = (t1 - t0 + G6K - 1) / G6K;
  const unsigned na = (unsigned)min(GT, nf - r0) * 16u;
  const unsigned nb = (unsigned)min(NCOL, nf - cc0) * 16u;

  const TMap* tm = TMAP ? pb.tmap[slot] + 2 * s : nullptr;
  auto issue = [&](int ch) {
    St& S = st[ch % NS];
    const unsigned bar = smem_u32(&full[ch % NS]);
    const int kt = t0 + ch * G6K;
    const int nval = max(0, min(G6K, t1 - kt));
    if (TMAP) {
      // one tensor copy per operand: boxes of 66 (A) / 34 (B) rows x G6K
      // columns land in the padded [k][row] layout; rows past nf and columns
      // past npiv are zero-filled by the TMA unit (chunks never straddle t1
      // except at t1 = npiv, see build_plans)
      if (lane == 0) {
        mbar_expect_tx(bar, (unsigned)G6K * (G6LA + G6LB) * 16u);
        tma_2d(smem_u32(&S.a[0]), tm, 2 * r0, kt, bar);
        tma_2d(smem_u32(&S.b[0]), tm + 1, 2 * cc0, kt, bar);
      }
      return;
    }
    if (lane == 0)
      mbar_expect_tx(bar, (unsigned)nval * (na + nb) + (unsigned)(G6K - nval) * (1024u + NCOL * 16u));
    for (int q = lane; q < 2 * G6K; q += 32) {
      const int kk = q >> 1;
      const int t = kt + kk;
      if (q & 1) {
        cplx* dst = &S.b[kk * G6LB];
        if (t < t1) bulk_g2s(smem_u32(dst), panel + (int64_t)t * nf + cc0, nb, bar);
        else bulk_g2s(smem_u32(dst), zeros, NCOL * 16u, bar);
      } else {
        cplx* dst = &S.a[kk * G6LA];
        if (t < t1) bulk_g2s(smem_u32(dst), panel + (int64_t)t * nf + r0, na, bar);
        else bulk_g2s(smem_u32(dst), zeros, 1024u, bar);
      }
    }
  };
  if (tid == 0) {
#pragma unroll
    for (int q = 0; q < NS; ++q) {
      mbar_init(smem_u32(&full[q]), 1);
      cnt[q] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == 0)
    for (int ch = 0; ch < min(NS, nchunks); ++ch) issue(ch);

  double cp[4][2][2], cq[4][2][2], ct[4][2][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) cp[a][b][h] = cq[a][b][h] = ct[a][b][h] = 0.0;
  for (int ch = 0; ch < nchunks; ++ch) {
    const int sidx = ch % NS;
    mbar_wait(smem_u32(&full[sidx]), (unsigned)((ch / NS) & 1));
    const St& S = st[sidx];
    if (active) {
#pragma unroll
      for (int k4 = 0; k4 < G6K; k4 += 4) {
        double ar[4], ai[4], br[2], bi[2];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const cplx v = S.a[(k4 + t4) * G6LA + wm + a * 8 + g];
          ar[a] = v.x;
          ai[a] = v.y;
        }
        // boxes wider than the 64-column task boundaries (G6K not dividing 64)
        // read real columns past t1: mask them in the B fragment
        const bool kin = !(TMAP && (64 % G6K) != 0) || t0 + ch * G6K + k4 + t4 < t1;
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          const cplx v = S.b[(k4 + t4) * G6LB + wn + b * 8 + g];
          br[b] = kin ? v.x : 0.0;
          bi[b] = kin ? v.y : 0.0;
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 2; ++b) dmma(cp[a][b][0], cp[a][b][1], ar[a], br[b]);
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 2; ++b) dmma(cq[a][b][0], cq[a][b][1], ai[a], bi[b]);
#pragma unroll
        for (int a = 0; a < 4; ++a) ar[a] += ai[a];
#pragma unroll
        for (int b = 0; b < 2; ++b) br[b] += bi[b];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 2; ++b) dmma(ct[a][b][0], ct[a][b][1], ar[a], br[b]);
      }
    }
    __syncwarp();
    if (ch + NS < nchunks) {
      int last = 0;
      if (lane == 0) {
        __threadfence_block();
        last = atomicAdd(&cnt[sidx], 1) == G6W - 1;
        if (last) {
          __threadfence_block();
          cnt[sidx] = 0;
        }
      }
      if (__shfl_sync(0xffffffffu, last, 0)) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        issue(ch + NS);
      }
    }
  }
  if (!active) return;
#pragma unroll
  for (int a0 = 0; a0 < 4; a0 += 2) {
    cplx* dst[2][2][2];
    cplx cv[2][2][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = r0 + wm + (a0 + a) * 8 + g;
          const int c = cc0 + wn + b * 8 + t4 * 2 + h;
          dst[a][b][h] = (r < nf && c < cmax && r >= c) ? faddr(pw, upd, p, nf, r, c) : nullptr;
          cv[a][b][h] = dst[a][b][h] ? __ldcg(dst[a][b][h]) : cmk(0.0, 0.0);
        }
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (dst[a][b][h]) {
            const double P = cp[a0 + a][b][h], Q = cq[a0 + a][b][h], T = ct[a0 + a][b][h];
            *dst[a][b][h] = cmk(cv[a][b][h].x - (P - Q), cv[a][b][h].y - (T - P - Q));
          }
  }
}

template <int G6K, int NS, int NCOL, bool TMAP = false>
static void launch_g6(cudaStream_t st, dim3 grid, const GemmTask* tasks, int ntasks,
                      const FrontsDev& F, const PoleBatch& pb, const cplx* zeros) {
  const size_t smem = NS * sizeof(Stage6<G6K, NCOL>);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_gemm6<G6K, NS, NCOL, TMAP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    attr = true;
  }
  k_gemm6<G6K, NS, NCOL, TMAP><<<grid, NCOL * 4, smem, st>>>(tasks, ntasks, F, pb, zeros);
}

// variant 0: 16 k x 4 stages (2 CTAs/SM); 1: 8 k x 8 stages (2 CTAs/SM);
// 2: 8 k x 5 stages (65 KB, 3 CTAs/SM); 3: 12 k x 3 stages (3 CTAs/SM);
// 4: whole 64x64 tile, 8 warps, 16 k x 6 stages (1 CTA/SM); 5: 64x64, 16 k x 4
// (1 CTA/SM); 6: as 2 with the operands moved by two TMA tensor copies per
// stage (tensor maps per front, make_tmaps) instead of one bulk copy per column
void launch_gemm6(cudaStream_t st, const GemmTask* tasks, int ntasks, int nctas,
                  const FrontsDev& F, const PoleBatch& pb, const cplx* zeros, int variant) {
  if (ntasks <= 0 || nctas <= 0) return;
  dim3 grid(2 * nctas, pb.count), grid1(nctas, pb.count);
  if (variant == 1) launch_g6<8, 8, 32>(st, grid, tasks, ntasks, F, pb, zeros);
  else if (variant == 2) launch_g6<8, 5, 32>(st, grid, tasks, ntasks, F, pb, zeros);
  else if (variant == 3) launch_g6<12, 3, 32>(st, grid, tasks, ntasks, F, pb, zeros);
  else if (variant == 4) launch_g6<16, 6, 64>(st, grid1, tasks, ntasks, F, pb, zeros);
  else if (variant == 5) launch_g6<16, 4, 64>(st, grid1, tasks, ntasks, F, pb, zeros);
  else if (variant == 6) launch_g6<G8K, 5, 32, true>(st, grid, tasks, ntasks, F, pb, zeros);
  else if (variant == 7) launch_g6<12, 3, 32, true>(st, grid, tasks, ntasks, F, pb, zeros);
  else if (variant == 8) launch_g6<16, 2, 32, true>(st, grid, tasks, ntasks, F, pb, zeros);
  else launch_g6<16, 4, 32>(st, grid, tasks, ntasks, F, pb, zeros);
}

// ---------------------------------------------------------------------------
// Schur update of the small fronts (one pivot block, p <= 64): one CTA of 4
// warps per (front, pole); a warp takes 16 x 8 blocks of the lower triangle of
// C (b x b, b = nf - p) and accumulates C -= L' L'^T over the p pivots with
// mma.sync m8n8k4 on exact 8 x 8 x 4 fragments (4 real MMAs per complex
// product).  The 64 x 32 tiles of k_gemm6 are mostly padding on these fronts
// (C4 level 0: b ~ 70, p ~ 33 -> ~20 % useful MMAs).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_schur_small(const int32_t* __restrict__ fronts, FrontsDev F,
                                                     PoleBatch pb) {
  const int slot = blockIdx.y;
  const int s = fronts[blockIdx.x];
  const int nf = F.nf[s], p = F.npiv[s];
  const int b = nf - p;
  const cplx* __restrict__ panel = pb.factor[slot] + F.panel_off[s];
  cplx* upd = pb.upd[slot] + F.upd_off[s];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int kq = lane & 3, mq = lane >> 2;
  const int nb8 = (b + 7) >> 3, nb16 = (b + 15) >> 4;
  const int p4 = (p + 3) & ~3;
  // blocks (I16, J8): rows 16 I16 .. +15, columns 8 J8 .. +7, J8 <= 2 I16 + 1
  int q = warp;
  for (int I = 0; I < nb16; ++I) {
    const int jmax = min(2 * I + 1, nb8 - 1);
    for (int J = 0; J <= jmax; ++J, ++q) {
      if ((q & 3) != 0) continue;          // round-robin over the 4 warps (q starts at warp)
      double re[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, im[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
      const int r0 = p + 16 * I + mq, r1 = r0 + 8;       // A rows of this lane (two fragments)
      const int cr = p + 8 * J + mq;                       // B row (= C column) of this lane
#pragma unroll 2
      for (int k0 = 0; k0 < p4; k0 += 4) {
        const int k = k0 + kq;
        const bool kon = k < p;
        const cplx* col = panel + (int64_t)k * nf;
        const cplx a0 = (kon && r0 < nf) ? __ldg(col + r0) : cmk(0.0, 0.0);
        const cplx a1 = (kon && r1 < nf) ? __ldg(col + r1) : cmk(0.0, 0.0);
        const cplx bb = (kon && cr < nf) ? __ldg(col + cr) : cmk(0.0, 0.0);
        dmma(re[0][0], re[0][1], a0.x, bb.x);
        dmma(re[1][0], re[1][1], a1.x, bb.x);
        dmma(im[0][0], im[0][1], a0.x, bb.y);
        dmma(im[1][0], im[1][1], a1.x, bb.y);
        dmma(re[0][0], re[0][1], -a0.y, bb.y);
        dmma(re[1][0], re[1][1], -a1.y, bb.y);
        dmma(im[0][0], im[0][1], a0.y, bb.x);
        dmma(im[1][0], im[1][1], a1.y, bb.x);
      }
      // fragment element (row mq, columns 2 kq, 2 kq + 1)
#pragma unroll
      for (int f = 0; f < 2; ++f)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = 16 * I + 8 * f + mq, c = 8 * J + 2 * kq + h;
          if (r < b && c <= r) {
            cplx* dst = upd + ucol(c, b) + (r - c);
            const cplx v = *dst;
            *dst = cmk(v.x - re[f][h], v.y - im[f][h]);
          }
        }
    }
  }
}

void launch_schur_small(cudaStream_t st, const int32_t* fronts, int nfr, const FrontsDev& F,
                        const PoleBatch& pb) {
  if (nfr <= 0) return;
  k_schur_small<<<dim3(nfr, pb.count), 128, 0, st>>>(fronts, F, pb);
}

}  // namespace rba
