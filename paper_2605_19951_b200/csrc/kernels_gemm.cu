// K4b on the FP64 tensor cores: complex trailing / Schur update of the fronts
//     C[r,c] -= sum_t (L[r,t] d_t) L[c,t]        (lower triangle, r >= c)
// with warp-level DMMA (mma.sync.m8n8k4.f64 -> SASS DMMA.8 on sm_100a; the
// tcgen05 UMMA has no f64 kind).  A complex product is four real
// DMMAs on split re/im planes: Cre += Are*Bre - Aim*Bim, Cim += Are*Bim + Aim*Bre.
//
// CTA tile 64x64 complex, 4 warps each 32x32 (4x4 DMMA tiles x {re,im}).
// K is staged in chunks of 16 through shared memory in [row][k] planes padded
// to 20 doubles (conflict-free 8-byte fragment loads), with a register
// prefetch of the next chunk (software pipeline) and the d_t scaling of the A
// operand fused into the staging.  Tiles are listed per task exactly as the
// DFMA reference kernel (k_gemm_update) and both share FrontsDev addressing.
#include "fronts.cuh"
#include "kernels.h"

namespace rba {

namespace {
constexpr int TK = 16;          // k-chunk (complex)
constexpr int LDK = TK + 4;     // padded row stride of the smem planes (doubles)
constexpr int NT = 128;         // threads per CTA

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
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

struct Stage {
  double are[GT * LDK], aim[GT * LDK], bre[GT * LDK], bim[GT * LDK];
};
}  // namespace

__global__ void __launch_bounds__(NT) k_gemm_dmma(const GemmTask* __restrict__ tasks, int ntasks,
                                                  FrontsDev F, PoleBatch pb) {
  extern __shared__ __align__(16) double smraw[];
  Stage* st = reinterpret_cast<Stage*>(smraw);     // st[0], st[1]
  __shared__ cplx ds[2][TK];
  const int slot = blockIdx.y;
  const int ti = find_task(tasks, ntasks, blockIdx.x);
  const GemmTask tk = tasks[ti];
  int local = blockIdx.x - tk.tile_start;
  int j = 0;
  while (local >= tk.ntr - j) { local -= tk.ntr - j; ++j; }
  const int i = j + local;
  const int s = tk.s;
  const int nf = F.nf[s], p = F.npiv[s];
  const int r0 = tk.c_lo + i * GT, cc0 = tk.c_lo + j * GT;
  const int cmax = min(cc0 + GT, tk.c_hi);
  const cplx* __restrict__ panel = pb.factor[slot] + F.panel_off[s];
  cplx* pw = pb.factor[slot] + F.panel_off[s];
  cplx* upd = pb.upd[slot] + (F.upd_off[s] >= 0 ? F.upd_off[s] : 0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;   // warp tile origin
  const int g = lane >> 2, t4 = lane & 3;

  // accumulators: [mi][ni] 8x8 tiles, re and im, 2 doubles each
  double cre[4][4][2], cim[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      cre[a][b][0] = cre[a][b][1] = 0.0;
      cim[a][b][0] = cim[a][b][1] = 0.0;
    }

  // staging: each thread loads 8 A and 8 B complex per chunk:
  // element e = tid + q*NT (q < 8) -> row = e % 64, k = e / 64
  cplx pa[8], pbv[8];
  auto gload = [&](int kt) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = tid + q * NT;
      const int rr = e & (GT - 1), kk = e >> 6;
      const int t = kt + kk;
      cplx a = cmk(0.0, 0.0), b = cmk(0.0, 0.0);
      if (t < tk.t1) {
        const cplx* col = panel + (int64_t)t * nf;
        if (r0 + rr < nf) a = __ldg(col + r0 + rr);
        if (cc0 + rr < cmax) b = __ldg(col + cc0 + rr);
      }
      pa[q] = a;
      pbv[q] = b;
    }
  };
  auto dload = [&](int kt, int buf) {
    if (tid < TK) {
      const int t = kt + tid;
      ds[buf][tid] = t < tk.t1 ? __ldg(panel + (int64_t)t * nf + t) : cmk(0.0, 0.0);
    }
  };
  auto sstore = [&](int buf) {
    Stage& S = st[buf];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = tid + q * NT;
      const int rr = e & (GT - 1), kk = e >> 6;
      const cplx a = cmul(pa[q], ds[buf][kk]);
      S.are[rr * LDK + kk] = a.x;
      S.aim[rr * LDK + kk] = a.y;
      S.bre[rr * LDK + kk] = pbv[q].x;
      S.bim[rr * LDK + kk] = pbv[q].y;
    }
  };

  const int nchunks = (tk.t1 - tk.t0 + TK - 1) / TK;
  dload(tk.t0, 0);
  gload(tk.t0);
  __syncthreads();
  sstore(0);
  __syncthreads();
  for (int ch = 0; ch < nchunks; ++ch) {
    const int buf = ch & 1;
    const bool more = ch + 1 < nchunks;
    if (more) {
      dload(tk.t0 + (ch + 1) * TK, buf ^ 1);
      gload(tk.t0 + (ch + 1) * TK);
    }
    const Stage& S = st[buf];
#pragma unroll
    for (int k4 = 0; k4 < TK; k4 += 4) {
      double ar[4], ai[4], an[4], br[4], bi[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int idx = (wm + a * 8 + g) * LDK + k4 + t4;
        ar[a] = S.are[idx];
        ai[a] = S.aim[idx];
        an[a] = -ai[a];
      }
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int idx = (wn + b * 8 + g) * LDK + k4 + t4;
        br[b] = S.bre[idx];
        bi[b] = S.bim[idx];
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          dmma(cre[a][b][0], cre[a][b][1], ar[a], br[b]);
          dmma(cre[a][b][0], cre[a][b][1], an[a], bi[b]);
          dmma(cim[a][b][0], cim[a][b][1], ar[a], bi[b]);
          dmma(cim[a][b][0], cim[a][b][1], ai[a], br[b]);
        }
    }
    if (more) {
      __syncthreads();            // ds[buf^1] visible; st[buf^1] free (read 2 chunks ago)
      sstore(buf ^ 1);
    }
    __syncthreads();
  }
  // epilogue: C -= acc  (lower triangle only)
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = r0 + wm + a * 8 + g;
        const int c = cc0 + wn + b * 8 + t4 * 2 + h;
        if (r < nf && c < cmax && r >= c) {
          cplx* dst = faddr(pw, upd, p, nf, r, c);
          cplx v = *dst;
          v.x -= cre[a][b][h];
          v.y -= cim[a][b][h];
          *dst = v;
        }
      }
}

void launch_gemm_dmma(cudaStream_t st, const GemmTask* tasks, int ntasks, int ntiles,
                      const FrontsDev& F, const PoleBatch& pb) {
  if (ntasks <= 0 || ntiles <= 0) return;
  const size_t smem = 2 * sizeof(Stage);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_gemm_dmma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  dim3 grid(ntiles, pb.count);
  k_gemm_dmma<<<grid, NT, smem, st>>>(tasks, ntasks, F, pb);
}

}  // namespace rba
