// Multi-RHS triangular solves with the stored multifrontal factors (K6/K7):
// forward L y = b per level (row-block tasks), D^{-1}, backward L^T x = z per
// level (column-block tasks).  Replaces `_Factor.solve`
// (/root/reference/pkg/src/rbainv/shifted.py:58-61); A_i is complex symmetric,
// so trans 'T' uses the same sweeps (sensitivity.py:8-13,91).
//
// Inside one launch, tasks of the same front depend on one another (the
// triangular chain).  CTAs take tasks through an atomic ticket in dependency
// order and wait on per-block flags (acquire/release); a task only waits on
// tasks with smaller tickets, which are already resident, so no deadlock.
// Child contributions enter through a deterministic gather (ucon lists), so
// results are bitwise reproducible.
#include "fronts.cuh"
#include "kernels.h"

namespace rba {

struct SolveBatchDev {
  const cplx* factor[32];
  cplx* x[32];
  cplx* uvec[32];
  int* flags[32];
};

__device__ __forceinline__ cplx ldcg_c(const cplx* p) { return __ldcg(p); }

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <int NR>
__global__ void __launch_bounds__(256) k_fwd(const SolveTask* __restrict__ tasks, int nslots,
                                             FrontsDev F, SolveBatchDev sb, int* ticket,
                                             int epoch) {
  __shared__ int s_t;
  extern __shared__ cplx dsm[];
  cplx(*v)[NR] = reinterpret_cast<cplx(*)[NR]>(dsm);
  cplx(*ys)[NR] = reinterpret_cast<cplx(*)[NR]>(dsm + PB * NR);
  cplx(*red)[PB][NR] = reinterpret_cast<cplx(*)[PB][NR]>(dsm + 2 * PB * NR);
  cplx(*Lb)[PB + 1] = reinterpret_cast<cplx(*)[PB + 1]>(dsm + 6 * PB * NR);
  const int tid = threadIdx.x;
  if (tid == 0) s_t = atomicAdd(ticket, 1);
  __syncthreads();
  const int t = s_t;
  const int slot = t % nslots;
  const SolveTask tk = tasks[t / nslots];
  const int s = tk.s, blk = tk.blk;
  const int p = F.npiv[s], nf = F.nf[s], first = F.first[s];
  const int npb = (p + PB - 1) / PB;
  const cplx* panel = sb.factor[slot] + F.panel_off[s];
  cplx* x = sb.x[slot];
  const cplx* uvec = sb.uvec[slot];
  int* flags = sb.flags[slot] + F.blk_off[s];
  const bool pivot = blk < npb;
  const int r0 = pivot ? blk * PB : p + (blk - npb) * PB;
  const int nr = pivot ? min(PB, p - r0) : min(PB, nf - r0);
  const int jmax = pivot ? blk : npb;
  const int row = tid & (PB - 1), cg = tid >> 6;

  if (cg == 0 && row < nr) {
    const int rho = r0 + row;
    cplx val[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r)
      val[r] = pivot ? x[(int64_t)(first + rho) * NR + r] : cmk(0.0, 0.0);
    const int64_t fr = F.rows_off[s] + rho;
    for (int64_t q = F.ucon_ptr[fr]; q < F.ucon_ptr[fr + 1]; ++q) {
      const int64_t u = F.ucon_idx[q];
#pragma unroll
      for (int r = 0; r < NR; ++r) val[r] = cadd(val[r], uvec[u * NR + r]);
    }
#pragma unroll
    for (int r = 0; r < NR; ++r) v[row][r] = val[r];
  }
  cplx acc[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) acc[r] = cmk(0.0, 0.0);
  for (int j = 0; j < jmax; ++j) {
    const int c0 = j * PB, ncol = min(PB, p - c0);
    if (tid == 0) {
      while (ld_acquire(flags + j) < epoch) { __nanosleep(64); }
    }
    __syncthreads();
    for (int q = tid; q < ncol * NR; q += blockDim.x)
      ys[q / NR][q % NR] = ldcg_c(x + (int64_t)(first + c0) * NR + q);
    __syncthreads();
    if (row < nr) {
      const cplx* col = panel + (int64_t)c0 * nf + r0 + row;
#pragma unroll 4
      for (int c = cg; c < ncol; c += 4) {
        const cplx l = __ldg(col + (int64_t)c * nf);
#pragma unroll
        for (int r = 0; r < NR; ++r) acc[r] = cfma(l, ys[c][r], acc[r]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < NR; ++r) red[cg][row][r] = acc[r];
  if (pivot) {
    for (int idx = tid; idx < nr * nr; idx += blockDim.x) {
      const int i = idx % nr, c = idx / nr;
      if (i > c) Lb[i][c] = panel[(int64_t)(r0 + c) * nf + r0 + i];
    }
  }
  __syncthreads();
  if (cg == 0 && row < nr) {
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      cplx sacc = cadd(cadd(red[0][row][r], red[1][row][r]), cadd(red[2][row][r], red[3][row][r]));
      v[row][r] = csub(v[row][r], sacc);
    }
  }
  __syncthreads();
  if (pivot) {
    // unit-lower solve, threads 0..63 own one row each
    if (tid < PB) {
      for (int c = 0; c < nr; ++c) {
        named_bar(1, PB);
        if (tid > c && tid < nr) {
#pragma unroll
          for (int r = 0; r < NR; ++r) v[tid][r] = cfms(Lb[tid][c], v[c][r], v[tid][r]);
        }
      }
      named_bar(1, PB);
      if (tid < nr) {
#pragma unroll
        for (int r = 0; r < NR; ++r) x[(int64_t)(first + r0 + tid) * NR + r] = v[tid][r];
      }
      __threadfence();
    }
    __syncthreads();
    if (tid == 0) st_release(flags + blk, epoch);
  } else {
    if (cg == 0 && row < nr) {
      cplx* u = sb.uvec[slot] + (F.uvec_off[s] + (r0 - p) + row) * NR;
#pragma unroll
      for (int r = 0; r < NR; ++r) u[r] = v[row][r];
    }
  }
}

// Backward: column block of pivots; x_c = L_cc^{-T} (y_c / d_c - sum_{rows below} L^T x).
template <int NR>
__global__ void __launch_bounds__(512) k_bwd(const SolveTask* __restrict__ tasks, int nslots,
                                             FrontsDev F, SolveBatchDev sb, int* ticket,
                                             int epoch) {
  __shared__ int s_t;
  extern __shared__ cplx dsm[];
  cplx(*red)[NR] = reinterpret_cast<cplx(*)[NR]>(dsm);
  cplx(*tv)[NR] = reinterpret_cast<cplx(*)[NR]>(dsm + PB * NR);
  cplx(*Lb)[PB + 1] = reinterpret_cast<cplx(*)[PB + 1]>(dsm + 2 * PB * NR);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_t = atomicAdd(ticket, 1);
  __syncthreads();
  const int t = s_t;
  const int slot = t % nslots;
  const SolveTask tk = tasks[t / nslots];
  const int s = tk.s, cb = tk.blk;
  const int p = F.npiv[s], nf = F.nf[s], first = F.first[s];
  const int npb = (p + PB - 1) / PB;
  const cplx* panel = sb.factor[slot] + F.panel_off[s];
  cplx* x = sb.x[slot];
  int* flags = sb.flags[slot] + F.blk_off[s];
  const int c0 = cb * PB, ncol = min(PB, p - c0);
  const int* rows = F.rows + F.rows_off[s];
  // warp w owns columns c0 + 4w .. c0 + 4w + 3
  cplx acc[4][NR];
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int r = 0; r < NR; ++r) acc[k][r] = cmk(0.0, 0.0);
  const int cw = 4 * warp;
  // border rows (ancestor pivots: final)
  for (int rho = p + lane; rho < nf; rho += 32) {
    const int g = rows[rho];
    cplx xv[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) xv[r] = ldcg_c(x + (int64_t)g * NR + r);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (cw + k < ncol) {
        const cplx l = __ldg(panel + (int64_t)(c0 + cw + k) * nf + rho);
#pragma unroll
        for (int r = 0; r < NR; ++r) acc[k][r] = cfma(l, xv[r], acc[k][r]);
      }
    }
  }
  // later pivot blocks of this front (produced by earlier tickets)
  for (int rb = npb - 1; rb > cb; --rb) {
    if (tid == 0) {
      while (ld_acquire(flags + rb) < epoch) { __nanosleep(64); }
    }
    __syncthreads();
    const int q0 = rb * PB, q1 = min(q0 + PB, p);
    for (int rho = q0 + lane; rho < q1; rho += 32) {
      cplx xv[NR];
#pragma unroll
      for (int r = 0; r < NR; ++r) xv[r] = ldcg_c(x + (int64_t)(first + rho) * NR + r);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (cw + k < ncol) {
          const cplx l = __ldg(panel + (int64_t)(c0 + cw + k) * nf + rho);
#pragma unroll
          for (int r = 0; r < NR; ++r) acc[k][r] = cfma(l, xv[r], acc[k][r]);
        }
      }
    }
  }
  // in-block strictly-lower part handled by the triangular solve below
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      double a = acc[k][r].x, b = acc[k][r].y;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
      }
      acc[k][r] = cmk(a, b);
    }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (cw + k < ncol)
#pragma unroll
        for (int r = 0; r < NR; ++r) red[cw + k][r] = acc[k][r];
  }
  for (int idx = tid; idx < ncol * ncol; idx += blockDim.x) {
    const int i = idx % ncol, c = idx / ncol;
    if (i > c) Lb[i][c] = panel[(int64_t)(c0 + c) * nf + c0 + i];
  }
  __syncthreads();
  if (tid < PB) {
    if (tid < ncol) {
      const cplx d = panel[(int64_t)(c0 + tid) * nf + c0 + tid];
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const cplx y = x[(int64_t)(first + c0 + tid) * NR + r];
        tv[tid][r] = csub(cdiv(y, d), red[tid][r]);
      }
    }
    for (int c = ncol - 1; c >= 0; --c) {
      named_bar(1, PB);
      if (tid < c) {
#pragma unroll
        for (int r = 0; r < NR; ++r) tv[tid][r] = cfms(Lb[c][tid], tv[c][r], tv[tid][r]);
      }
    }
    named_bar(1, PB);
    if (tid < ncol) {
#pragma unroll
      for (int r = 0; r < NR; ++r) x[(int64_t)(first + c0 + tid) * NR + r] = tv[tid][r];
    }
    __threadfence();
  }
  __syncthreads();
  if (tid == 0) st_release(flags + cb, epoch);
}

template <int NR>
static void fwd_nr(cudaStream_t st, const SolveTask* tasks, int ntasks, int nslots,
                   const FrontsDev& F, const SolveBatchDev& sb, int* ticket, int epoch) {
  const size_t smem = (6 * PB * NR + PB * (PB + 1)) * sizeof(cplx);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_fwd<NR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  k_fwd<NR><<<ntasks * nslots, 256, smem, st>>>(tasks, nslots, F, sb, ticket, epoch);
}
template <int NR>
static void bwd_nr(cudaStream_t st, const SolveTask* tasks, int ntasks, int nslots,
                   const FrontsDev& F, const SolveBatchDev& sb, int* ticket, int epoch) {
  const size_t smem = (2 * PB * NR + PB * (PB + 1)) * sizeof(cplx);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_bwd<NR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  k_bwd<NR><<<ntasks * nslots, 512, smem, st>>>(tasks, nslots, F, sb, ticket, epoch);
}

void launch_solve_level(cudaStream_t st, bool forward, int nr, const SolveTask* tasks,
                        int ntasks, int nslots, const FrontsDev& F, const SolveBatch& b,
                        int* ticket, int epoch) {
  if (ntasks <= 0) return;
  SolveBatchDev sb;
  for (int i = 0; i < nslots; ++i) {
    sb.factor[i] = b.factor[i];
    sb.x[i] = b.x[i];
    sb.uvec[i] = b.uvec[i];
    sb.flags[i] = forward ? b.flags_f[i] : b.flags_b[i];
  }
  switch (nr) {
    case 1: forward ? fwd_nr<1>(st, tasks, ntasks, nslots, F, sb, ticket, epoch)
                    : bwd_nr<1>(st, tasks, ntasks, nslots, F, sb, ticket, epoch); break;
    case 2: forward ? fwd_nr<2>(st, tasks, ntasks, nslots, F, sb, ticket, epoch)
                    : bwd_nr<2>(st, tasks, ntasks, nslots, F, sb, ticket, epoch); break;
    case 4: forward ? fwd_nr<4>(st, tasks, ntasks, nslots, F, sb, ticket, epoch)
                    : bwd_nr<4>(st, tasks, ntasks, nslots, F, sb, ticket, epoch); break;
    default: forward ? fwd_nr<8>(st, tasks, ntasks, nslots, F, sb, ticket, epoch)
                     : bwd_nr<8>(st, tasks, ntasks, nslots, F, sb, ticket, epoch); break;
  }
}

// original-order (column-major N x nrhs complex) <-> permuted padded layout
__global__ void k_perm_in(int64_t n, int nrhs, int NR, const int32_t* __restrict__ perm,
                          const cplx* __restrict__ b, int64_t ldb, cplx* __restrict__ x) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = perm[k];
    for (int r = 0; r < NR; ++r) x[k * NR + r] = r < nrhs ? b[r * ldb + o] : cmk(0.0, 0.0);
  }
}
__global__ void k_perm_out(int64_t n, int nrhs, int NR, const int32_t* __restrict__ perm,
                           const cplx* __restrict__ x, cplx* __restrict__ b, int64_t ldb) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = perm[k];
    for (int r = 0; r < nrhs; ++r) b[r * ldb + o] = x[k * NR + r];
  }
}
void launch_perm_in(cudaStream_t st, int64_t n, int nrhs, int NR, const int32_t* perm,
                    const cplx* b, int64_t ldb, cplx* x) {
  k_perm_in<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 8), 256, 0, st>>>(n, nrhs, NR, perm,
                                                                              b, ldb, x);
}
void launch_perm_out(cudaStream_t st, int64_t n, int nrhs, int NR, const int32_t* perm,
                     const cplx* x, cplx* b, int64_t ldb) {
  k_perm_out<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 8), 256, 0, st>>>(n, nrhs, NR, perm,
                                                                               x, b, ldb);
}

}  // namespace rba
