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

// MODE 0: trailing/Schur update  C[r,c] -= sum_t (L[r,t] d_t) L[c,t]  (r >= c)
// MODE 1: panel TRSM  L[r, k0+c] = (sum_{t<=c} F[r, k0+t] X[c][t]) / d_c, with
//         X = L_kk^{-1} read from the diagonal block's upper triangle (k_diag).
template <int MODE>
__global__ void __launch_bounds__(NT) k_gemm_dmma(const GemmTask* __restrict__ tasks, int ntasks,
                                                  const PanelTask* __restrict__ ptasks,
                                                  FrontsDev F, PoleBatch pb) {
  extern __shared__ __align__(16) double smraw[];
  Stage* st = reinterpret_cast<Stage*>(smraw);     // st[0], st[1]
  __shared__ cplx ds[2][TK];
  __shared__ cplx dinv[GT];
  const int slot = blockIdx.y;
  GemmTask tk;
  int r0, cc0, cmax, kbase = 0;
  if (MODE == 0) {
    const int ti = find_task(tasks, ntasks, blockIdx.x);
    tk = tasks[ti];
    int local = blockIdx.x - tk.tile_start;
    int j = 0;
    while (local >= tk.ntr - j) { local -= tk.ntr - j; ++j; }
    const int i = j + local;
    r0 = tk.c_lo + i * GT;
    cc0 = tk.c_lo + j * GT;
    cmax = min(cc0 + GT, tk.c_hi);
  } else {
    const PanelTask pt = ptasks[blockIdx.x];
    const int p_ = F.npiv[pt.s];
    tk.s = pt.s;
    tk.t0 = 0;
    tk.t1 = min(GT, p_ - pt.k0);         // kb
    kbase = pt.k0;
    r0 = pt.r0;
    cc0 = 0;
    cmax = tk.t1;
  }
  const int s = tk.s;
  const int nf = F.nf[s], p = F.npiv[s];
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
        if (MODE == 0) {
          const cplx* col = panel + (int64_t)t * nf;
          if (r0 + rr < nf) a = __ldg(col + r0 + rr);
          if (cc0 + rr < cmax) b = __ldg(col + cc0 + rr);
        } else {
          // A = F[r0+rr, kbase+t]; B[c=rr][t] = X[c][t] (t < c), 1 (t == c), 0 (t > c)
          if (r0 + rr < nf) a = __ldg(panel + (int64_t)(kbase + t) * nf + r0 + rr);
          if (rr < cmax) {
            if (t < rr) b = __ldg(panel + (int64_t)(kbase + rr) * nf + kbase + t);
            else if (t == rr) b = cmk(1.0, 0.0);
          }
        }
      }
      pa[q] = a;
      pbv[q] = b;
    }
  };
  auto dload = [&](int kt, int buf) {
    if (tid < TK) {
      const int t = kt + tid;
      ds[buf][tid] = MODE == 1 ? cmk(1.0, 0.0)
                   : (t < tk.t1 ? __ldg(panel + (int64_t)t * nf + t) : cmk(0.0, 0.0));
    }
  };
  if (MODE == 1 && tid < GT) {
    dinv[tid] = tid < cmax ? cinv(__ldg(panel + (int64_t)(kbase + tid) * nf + kbase + tid))
                           : cmk(0.0, 0.0);
  }
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
  if (MODE == 0) {
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
  } else {
    // epilogue: L = (F X^T) D^{-1}, written in place (every A element of this
    // tile was staged before any write: the K loop ended with a barrier)
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = r0 + wm + a * 8 + g;
          const int c = wn + b * 8 + t4 * 2 + h;
          if (r < nf && c < cmax)
            pw[(int64_t)(kbase + c) * nf + r] = cmul(cmk(cre[a][b][h], cim[a][b][h]), dinv[c]);
        }
  }
}

void launch_gemm_dmma(cudaStream_t st, const GemmTask* tasks, int ntasks, int ntiles,
                      const FrontsDev& F, const PoleBatch& pb) {
  if (ntasks <= 0 || ntiles <= 0) return;
  const size_t smem = 2 * sizeof(Stage);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_gemm_dmma<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  dim3 grid(ntiles, pb.count);
  k_gemm_dmma<0><<<grid, NT, smem, st>>>(tasks, ntasks, nullptr, F, pb);
}

void launch_trsm_dmma(cudaStream_t st, const PanelTask* tasks, int ntasks, const FrontsDev& F,
                      const PoleBatch& pb) {
  if (ntasks <= 0) return;
  const size_t smem = 2 * sizeof(Stage);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_gemm_dmma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  dim3 grid(ntasks, pb.count);
  k_gemm_dmma<1><<<grid, NT, smem, st>>>(nullptr, 0, tasks, F, pb);
}

}  // namespace rba
