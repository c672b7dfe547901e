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
#include <cstdlib>
#include "fronts.cuh"
#include "kernels.h"

namespace rba {

struct SolveBatchDev {
  const cplx* factor[32];
  cplx* x[32];
  cplx* uvec[32];
  int* flags[32];
  int* done[32];      // fused sweeps: per-front completion counters (monotonic)
  int epoch[32];      // per-slot solve count: flags hold it, counters reach epoch*need
};

// Cross-front dependencies of the fused (single-launch) sweeps.
struct SweepDeps {
  const int32_t* parent;   // front parent (-1 root)
  const int32_t* need_u;   // forward: border tasks of all children of the front
  int fused;
};

__device__ __forceinline__ cplx ldcg_c(const cplx* p) { return __ldcg(p); }

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Forward task (front s, row block blk): rows [r0, r0+nr) of the front vector.
//   pivot block  : y_blk = S^{-1} X_blk (v_blk - sum_{j<blk} L'[blk, j] y_j)
//                  (X = L_bb^{-1}, S = diag sqrt(d): factor format, fronts.cuh)
//   border block : u     = v - sum_{j<npb} L'[rows, j] y_j             -> parent
// Warps split the pivot columns (column c handled by warp c % 8), lanes own
// rows lane and lane+32, so every L load is a coalesced 2 x 512 B column
// segment; each warp fetches the y values of its 8 columns of a block with one
// L2 load per lane (they were produced by other CTAs) and broadcasts them with
// shuffles.  16 L loads per lane are in flight per block.
template <int NR, bool STAGEX>
__global__ void __launch_bounds__(256, NR >= 8 ? 1 : 2) k_fwd(const SolveTask* __restrict__ tasks, int nslots,
                                             FrontsDev F, SolveBatchDev sb, int* ticket,
                                             int /*unused*/, SweepDeps dep) {
  __shared__ int s_t;
  extern __shared__ cplx dsm[];
  cplx(*v)[NR] = reinterpret_cast<cplx(*)[NR]>(dsm);
  cplx(*red)[PB][NR] = reinterpret_cast<cplx(*)[PB][NR]>(dsm + PB * NR);   // [8][PB][NR]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_t = atomicAdd(ticket, 1);
  __syncthreads();
  const int t = s_t;
  const int slot = t % nslots;
  const int epoch = sb.epoch[slot];
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
  cplx* Xs = dsm + 9 * PB * NR;      // [PB][PB+1]: column r0+i of the diagonal block in row i
  if (STAGEX && pivot) {
    for (int e = tid; e < nr * nr; e += blockDim.x) {
      const int i = e / nr, c = e - i * nr;
      const unsigned sa = (unsigned)__cvta_generic_to_shared(Xs + i * (PB + 1) + c);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(sa),
                   "l"(panel + (int64_t)(r0 + i) * nf + r0 + c) : "memory");
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  if (dep.fused) {
    // every child's border (u-vector) tasks must have completed
    const int need = dep.need_u[s];
    if (need > 0) {
      if (tid == 0)
        spin_wait_geq(sb.done[slot] + s, epoch * need);
      __syncthreads();
    }
  }

  if (tid < nr) {
    const int rho = r0 + tid;
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
    for (int r = 0; r < NR; ++r) v[tid][r] = val[r];
  }
  cplx acc0[NR], acc1[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) acc0[r] = acc1[r] = cmk(0.0, 0.0);
  const bool ok0 = lane < nr, ok1 = lane + 32 < nr;
  const cplx* rowp = panel + r0 + lane;
  if (!pivot && jmax > 0) {
    // border rows need every pivot block: one wait (block npb-1 implies all)
    if (lane == 0)
      spin_wait_geq(flags + jmax - 1, epoch);
    __syncwarp();
  }
  constexpr int YPL = (8 * NR + 31) / 32;   // y values per lane per block
  for (int j = 0; j < jmax; ++j) {
    const int c0 = j * PB, ncol = min(PB, p - c0);
    // L does not depend on y: issue its loads before waiting for block j
    cplx l0[8], l1[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int c = warp + 8 * q;
      const cplx* colp = rowp + (int64_t)(c0 + c) * nf;
      l0[q] = (c < ncol && ok0) ? __ldg(colp) : cmk(0.0, 0.0);
      l1[q] = (c < ncol && ok1) ? __ldg(colp + 32) : cmk(0.0, 0.0);
    }
    if (pivot) {
      if (lane == 0)
        spin_wait_geq(flags + j, epoch);
      __syncwarp();
    }
    // y of this warp's 8 columns (c0 + warp + 8q), NR each
    cplx yv[YPL];
#pragma unroll
    for (int h = 0; h < YPL; ++h) {
      const int e = lane + 32 * h;
      const int q = e / NR, r = e % NR;
      const int c = warp + 8 * q;
      yv[h] = (e < 8 * NR && c < ncol) ? ldcg_c(x + (int64_t)(first + c0 + c) * NR + r)
                                       : cmk(0.0, 0.0);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q)
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const int e = q * NR + r;
        const cplx y = cmk(__shfl_sync(0xffffffffu, yv[e / 32].x, e % 32),
                           __shfl_sync(0xffffffffu, yv[e / 32].y, e % 32));
        acc0[r] = cfma(l0[q], y, acc0[r]);
        acc1[r] = cfma(l1[q], y, acc1[r]);
      }
  }
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    red[warp][lane][r] = acc0[r];
    red[warp][lane + 32][r] = acc1[r];
  }
  __syncthreads();
  if (tid < nr) {
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      cplx sacc = red[0][tid][r];
#pragma unroll
      for (int w = 1; w < 8; ++w) sacc = cadd(sacc, red[w][tid][r]);
      v[tid][r] = csub(v[tid][r], sacc);
    }
  }
  __syncthreads();
  if (pivot) {
    // y_i = t_i + sum_{c<i} X[i][c] t_c ; X[i][c] sits at (row r0+c, col r0+i),
    // staged in shared memory at the start of the task.
    // 4 threads per output row (c = k mod 4), shuffle-reduced.
    if (STAGEX) {
      asm volatile("cp.async.wait_all;\n" ::: "memory");
      __syncthreads();
    }
    const int i = tid >> 2, k = tid & 3;
    cplx yv[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) yv[r] = cmk(0.0, 0.0);
    if (i < nr) {
      const cplx* xcol = STAGEX ? Xs + i * (PB + 1) : panel + (int64_t)(r0 + i) * nf + r0;
#pragma unroll 8
      for (int c = k; c < i; c += 4) {
        const cplx xv = xcol[c];
#pragma unroll
        for (int r = 0; r < NR; ++r) yv[r] = cfma(xv, v[c][r], yv[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      double a = yv[r].x, b = yv[r].y;
      a += __shfl_xor_sync(0xffffffffu, a, 1);
      b += __shfl_xor_sync(0xffffffffu, b, 1);
      a += __shfl_xor_sync(0xffffffffu, a, 2);
      b += __shfl_xor_sync(0xffffffffu, b, 2);
      yv[r] = cmk(a, b);
    }
    if (i < nr && k == 0) {
      // y' = S^{-1} X t  (s_i = sqrt(d_i) on the diagonal, fronts.cuh)
      const cplx si = cinv(STAGEX ? Xs[i * (PB + 1) + i] : panel[(int64_t)(r0 + i) * nf + r0 + i]);
#pragma unroll
      for (int r = 0; r < NR; ++r)
        x[(int64_t)(first + r0 + i) * NR + r] = cmul(cadd(v[i][r], yv[r]), si);
      __threadfence();
    }
    __syncthreads();
    if (tid == 0) st_release(flags + blk, epoch);
  } else {
    if (tid < nr) {
      cplx* u = sb.uvec[slot] + (F.uvec_off[s] + (r0 - p) + tid) * NR;
#pragma unroll
      for (int r = 0; r < NR; ++r) u[r] = v[tid][r];
      if (dep.fused) __threadfence();
    }
    if (dep.fused) {
      __syncthreads();
      if (tid == 0) atomicAdd(sb.done[slot] + dep.parent[s], 1);
    }
  }
}

// Backward task (front s, pivot column block cb), blocks processed from the
// last one down:  x_cb = X^T S^{-1} (y_cb - sum_{rho beyond block} L'[rho, cb]^T x_rho).
// NW warps x 64/NW columns, lanes stride the rows; no block barrier in the main
// loop (the pivot-block waits are per warp).
template <int NR, int NW>
__global__ void __launch_bounds__(32 * NW) k_bwd(const SolveTask* __restrict__ tasks, int nslots,
                                             FrontsDev F, SolveBatchDev sb, int* ticket,
                                             int /*unused*/, SweepDeps dep) {
  __shared__ int s_t;
  extern __shared__ cplx dsm[];
  cplx(*red)[NR] = reinterpret_cast<cplx(*)[NR]>(dsm);
  cplx(*tv)[NR] = reinterpret_cast<cplx(*)[NR]>(dsm + PB * NR);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_t = atomicAdd(ticket, 1);
  __syncthreads();
  const int t = s_t;
  const int slot = t % nslots;
  const int epoch = sb.epoch[slot];
  const SolveTask tk = tasks[t / nslots];
  const int s = tk.s, cb = tk.blk;
  const int p = F.npiv[s], nf = F.nf[s], first = F.first[s];
  const int npb = (p + PB - 1) / PB;
  const cplx* panel = sb.factor[slot] + F.panel_off[s];
  cplx* x = sb.x[slot];
  int* flags = sb.flags[slot] + F.blk_off[s];
  const int c0 = cb * PB, ncol = min(PB, p - c0);
  const int* rows = F.rows + F.rows_off[s];
  // stage the diagonal block (X^T in its upper triangle) for the final GEMV
  cplx* Xs = dsm + 2 * PB * NR;       // [PB][PB+1]: Xs[i][c] = panel(row c0+c, col c0+i)
  for (int e = tid; e < ncol * ncol; e += blockDim.x) {
    const int i = e / ncol, c = e - i * ncol;
    const unsigned sa = (unsigned)__cvta_generic_to_shared(Xs + i * (PB + 1) + c);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(sa),
                 "l"(panel + (int64_t)(c0 + i) * nf + c0 + c) : "memory");
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  // columns per warp per pass: 64 / NW, halved (in two passes) when the
  // NR accumulators would not fit in registers
  constexpr int CW = PB / NW;
  constexpr int CPW = (NR * CW > 16) ? CW / 2 : CW;
  constexpr int NPASS = CW / CPW;
  if (dep.fused && nf > p) {
    // border rows are final once the parent front is complete (its own tasks
    // waited for every owner of its border)
    const int par = dep.parent[s];
    const int need = (F.npiv[par] + PB - 1) / PB;
    if (tid == 0)
      spin_wait_geq(sb.done[slot] + par, epoch * need);
    __syncthreads();
  }

  for (int pass = 0; pass < NPASS; ++pass) {
  cplx acc[CPW][NR];
#pragma unroll
  for (int k = 0; k < CPW; ++k)
#pragma unroll
    for (int r = 0; r < NR; ++r) acc[k][r] = cmk(0.0, 0.0);
  const int cw = (pass * NW + warp) * CPW;
  const int nk = max(0, min(CPW, ncol - cw));
  const cplx* colp = panel + (int64_t)(c0 + cw) * nf;
  // border rows: pivots of ancestors, final before this launch (L1 is
  // invalidated at launch, so the read-only path is safe); the 16 warps of
  // the CTA read the same x rows, which therefore hit in L1.
#pragma unroll 2
  for (int rho = p + lane; rho < nf; rho += 32) {
    const int g = __ldg(rows + rho);
    cplx lv[CPW];
#pragma unroll
    for (int k = 0; k < CPW; ++k)
      lv[k] = k < nk ? __ldg(colp + (int64_t)k * nf + rho) : cmk(0.0, 0.0);
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const cplx xv = __ldg(x + (int64_t)g * NR + r);
#pragma unroll
      for (int k = 0; k < CPW; ++k) acc[k][r] = cfma(lv[k], xv, acc[k][r]);
    }
  }
  // later pivot blocks of this front (produced by earlier tickets in this
  // launch): per-warp wait, L2 reads
  // with two column passes the dependent block cb+1 is handled after both
  // passes (below), so the second pass does not re-stream every later block
  // after the chain wait
  for (int rb = npb - 1; rb > (NPASS > 1 ? cb + 1 : cb); --rb) {
    const int q0 = rb * PB, q1 = min(q0 + PB, p);
    // the block's 64 rows = 2 per lane: load L before waiting for x
    cplx lv[2][CPW];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int rho = q0 + lane + 32 * h;
#pragma unroll
      for (int k = 0; k < CPW; ++k)
        lv[h][k] = (k < nk && rho < q1) ? __ldg(colp + (int64_t)k * nf + rho) : cmk(0.0, 0.0);
    }
    if (lane == 0)
      spin_wait_geq(flags + rb, epoch);
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int rho = q0 + lane + 32 * h;
      if (rho < q1) {
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          const cplx xv = ldcg_c(x + (int64_t)(first + rho) * NR + r);
#pragma unroll
          for (int k = 0; k < CPW; ++k) acc[k][r] = cfma(lv[h][k], xv, acc[k][r]);
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < CPW; ++k)
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
    for (int k = 0; k < CPW; ++k)
      if (k < nk)
#pragma unroll
        for (int r = 0; r < NR; ++r) red[cw + k][r] = acc[k][r];
  }
  __syncthreads();
  }
  if (NPASS > 1 && cb + 1 < npb) {
    const int q0 = (cb + 1) * PB, q1 = min(q0 + PB, p);
    if (lane == 0)
      spin_wait_geq(flags + cb + 1, epoch);
    __syncwarp();
    for (int pass = 0; pass < NPASS; ++pass) {
      const int cw = (pass * NW + warp) * CPW;
      const int nk = max(0, min(CPW, ncol - cw));
      const cplx* colp = panel + (int64_t)(c0 + cw) * nf;
      cplx acc[CPW][NR];
#pragma unroll
      for (int k = 0; k < CPW; ++k)
#pragma unroll
        for (int r = 0; r < NR; ++r) acc[k][r] = cmk(0.0, 0.0);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int rho = q0 + lane + 32 * h;
        if (rho < q1) {
          cplx lv[CPW];
#pragma unroll
          for (int k = 0; k < CPW; ++k)
            lv[k] = k < nk ? __ldg(colp + (int64_t)k * nf + rho) : cmk(0.0, 0.0);
#pragma unroll
          for (int r = 0; r < NR; ++r) {
            const cplx xv = ldcg_c(x + (int64_t)(first + rho) * NR + r);
#pragma unroll
            for (int k = 0; k < CPW; ++k) acc[k][r] = cfma(lv[k], xv, acc[k][r]);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < CPW; ++k)
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          double re = acc[k][r].x, im = acc[k][r].y;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            re += __shfl_xor_sync(0xffffffffu, re, o);
            im += __shfl_xor_sync(0xffffffffu, im, o);
          }
          acc[k][r] = cmk(re, im);
        }
      if (lane == 0) {
#pragma unroll
        for (int k = 0; k < CPW; ++k)
          if (k < nk)
#pragma unroll
            for (int r = 0; r < NR; ++r) red[cw + k][r] = cadd(red[cw + k][r], acc[k][r]);
      }
    }
    __syncthreads();
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  if (tid < ncol) {
    const cplx sc = Xs[tid * (PB + 1) + tid];   // s_c = sqrt(d_c)
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const cplx y = x[(int64_t)(first + c0 + tid) * NR + r];
      tv[tid][r] = cdiv(csub(y, red[tid][r]), sc);
    }
  }
  __syncthreads();
  // x_c = t_c + sum_{i>c} X[i][c] t_i ; X[i][c] sits at (row c0+c, col c0+i).
  // 8 threads per column (i = c+1+k mod 8), shuffle-reduced.
  {
    const int c = tid >> 3, k = tid & 7;
    cplx xv[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) xv[r] = cmk(0.0, 0.0);
    if (c < ncol) {
#pragma unroll 4
      for (int i = c + 1 + k; i < ncol; i += 8) {
        const cplx w = Xs[i * (PB + 1) + c];
#pragma unroll
        for (int r = 0; r < NR; ++r) xv[r] = cfma(w, tv[i][r], xv[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      double a = xv[r].x, b = xv[r].y;
#pragma unroll
      for (int o = 1; o < 8; o <<= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
      }
      xv[r] = cmk(a, b);
    }
    if (c < ncol && k == 0) {
#pragma unroll
      for (int r = 0; r < NR; ++r)
        x[(int64_t)(first + c0 + c) * NR + r] = cadd(tv[c][r], xv[r]);
      __threadfence();
    }
  }
  __syncthreads();
  if (tid == 0) {
    st_release(flags + cb, epoch);
    if (dep.fused) atomicAdd(sb.done[slot] + s, 1);
  }
}

// ---------------------------------------------------------------------------
// 4 right-hand sides: the row reduction sum_rho L'[rho, c] x_rho of the
// backward sweep on the FP64 tensor cores (mma.sync m8n8k4).  A = 8 columns x
// 4 rows of L' (one 16-byte load per lane: lane = (column lane / 4, row
// lane % 4)), B = the 4 rows x [Re x (4 RHS) | Im x (4 RHS)], two MMAs per
// 4 rows (Re L' with (Re x | Im x), Im L' with (-Im x | Re x)); the 8 x 8
// accumulator holds [Re | Im] of the 8 columns x 4 RHS sums, so there is no
// shuffle reduction, one x load per lane per 4 rows instead of 4 per row, and
// 2 accumulator registers instead of 32: the sweep stays on the HBM stream.
// ---------------------------------------------------------------------------
constexpr int BCH = 512;   // border rows gathered per shared-memory chunk (k_bwd_mma4)
struct BwdFrag {
  double c0 = 0.0, c1 = 0.0;
  __device__ __forceinline__ void mac(cplx l, cplx xv, bool hi) {
    dmma_f64(c0, c1, l.x, hi ? xv.y : xv.x);
    dmma_f64(c0, c1, l.y, hi ? xv.x : -xv.y);
  }
};

// Backward task (front s, pivot column block cb) for NR = 4: 8 warps x 8 columns.
__global__ void __launch_bounds__(256, 2) k_bwd_mma4(const SolveTask* __restrict__ tasks, int nslots,
                                                     FrontsDev F, SolveBatchDev sb, int* ticket,
                                                     SweepDeps dep) {
  constexpr int NR = 4;
  __shared__ int s_t;
  extern __shared__ cplx dsm[];
  cplx(*red)[NR] = reinterpret_cast<cplx(*)[NR]>(dsm);
  cplx(*tv)[NR] = reinterpret_cast<cplx(*)[NR]>(dsm + PB * NR);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_t = atomicAdd(ticket, 1);
  __syncthreads();
  const int t = s_t;
  const int slot = t % nslots;
  const int epoch = sb.epoch[slot];
  const SolveTask tk = tasks[t / nslots];
  const int s = tk.s, cb = tk.blk;
  const int p = F.npiv[s], nf = F.nf[s], first = F.first[s];
  const int npb = (p + PB - 1) / PB;
  const cplx* panel = sb.factor[slot] + F.panel_off[s];
  cplx* x = sb.x[slot];
  int* flags = sb.flags[slot] + F.blk_off[s];
  const int c0 = cb * PB, ncol = min(PB, p - c0);
  const int* rows = F.rows + F.rows_off[s];
  cplx* Xs = dsm + 2 * PB * NR;       // [PB][PB+1]: Xs[i][c] = panel(row c0+c, col c0+i)
  for (int e = tid; e < ncol * ncol; e += blockDim.x) {
    const int i = e / ncol, c = e - i * ncol;
    const unsigned sa = (unsigned)__cvta_generic_to_shared(Xs + i * (PB + 1) + c);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(sa),
                 "l"(panel + (int64_t)(c0 + i) * nf + c0 + c) : "memory");
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  if (dep.fused && nf > p) {
    const int par = dep.parent[s];
    const int need = (F.npiv[par] + PB - 1) / PB;
    if (tid == 0) spin_wait_geq(sb.done[slot] + par, epoch * need);
    __syncthreads();
  }
  const int kq = lane & 3, cq = lane >> 2;
  const int col = warp * 8 + cq;                 // this lane's column of the block
  const bool con = col < ncol;
  const cplx* colp = panel + (int64_t)(c0 + (con ? col : 0)) * nf;
  const int rhs = cq & 3;
  const bool hi = cq >= 4;
  BwdFrag acc, acc2;
  // border rows (pivots of ancestors, final before this launch): the x rows
  // are gathered once per CTA into shared memory in chunks of BCH rows, then
  // every warp streams its 8 columns of L' against them
  cplx(*xs)[NR] = reinterpret_cast<cplx(*)[NR]>(dsm + 2 * PB * NR + PB * (PB + 1));
  const bool won = warp * 8 < ncol;
  for (int ch0 = p; ch0 < nf; ch0 += BCH) {
    const int nch = min(BCH, nf - ch0);
    // first L' loads of the chunk go out before the gather and the barrier
    cplx lv[8];
#pragma unroll
    for (int h = 0; h < 8; ++h) {
      const int rho = ch0 + 4 * h + kq;
      lv[h] = (won && con && rho < nf) ? __ldg(colp + rho) : cmk(0.0, 0.0);
    }
    __syncthreads();                               // previous chunk consumed
    for (int e = tid; e < nch * NR; e += blockDim.x) {
      const int rr = e >> 2, r = e & 3;
      const int g = __ldg(rows + ch0 + rr);
      xs[rr][r] = __ldg(x + (int64_t)g * NR + r);
    }
    for (int e = nch * NR + tid; e < ((nch + 3) & ~3) * NR; e += blockDim.x) xs[e >> 2][e & 3] = cmk(0.0, 0.0);
    __syncthreads();
    if (won) {
      for (int g0 = 0; g0 < nch; g0 += 32) {
        cplx ln[8];
#pragma unroll
        for (int h = 0; h < 8; ++h) {              // next 32 rows in flight
          const int rho = ch0 + g0 + 32 + 4 * h + kq;
          ln[h] = (con && g0 + 32 < nch && rho < nf) ? __ldg(colp + rho) : cmk(0.0, 0.0);
        }
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          const int rr = g0 + 4 * h + kq;
          const cplx xv = rr < ((nch + 3) & ~3) ? xs[rr][rhs] : cmk(0.0, 0.0);
          if (h & 1) acc2.mac(lv[h], xv, hi); else acc.mac(lv[h], xv, hi);
        }
#pragma unroll
        for (int h = 0; h < 8; ++h) lv[h] = ln[h];
      }
    }
  }
  if (won) {
    // later pivot blocks of this front (earlier tickets of this launch): L'
    // is loaded before the wait, x with L2 loads after it
    for (int rb = npb - 1; rb > cb; --rb) {
      const int q0 = rb * PB, q1 = min(q0 + PB, p);
      cplx lv[16];
#pragma unroll
      for (int h = 0; h < 16; ++h) {
        const int rho = q0 + 4 * h + kq;
        lv[h] = (con && rho < q1) ? __ldg(colp + rho) : cmk(0.0, 0.0);
      }
      if (lane == 0) spin_wait_geq(flags + rb, epoch);
      __syncwarp();
      cplx xv[16];
#pragma unroll
      for (int h = 0; h < 16; ++h) {
        const int rho = q0 + 4 * h + kq;
        xv[h] = rho < q1 ? ldcg_c(x + (int64_t)(first + rho) * NR + rhs) : cmk(0.0, 0.0);
      }
#pragma unroll
      for (int h = 0; h < 16; ++h) { if (h & 1) acc2.mac(lv[h], xv[h], hi); else acc.mac(lv[h], xv[h], hi); }
    }
    // accumulator (column cq, n = 2 kq, 2 kq + 1): n < 4 real part of RHS n, else imaginary of n - 4
    if (con) {
      double* rd = reinterpret_cast<double*>(&red[col][0]);
      const int n0 = 2 * kq;
      rd[2 * (n0 & 3) + (n0 >> 2)] = acc.c0 + acc2.c0;
      rd[2 * ((n0 + 1) & 3) + ((n0 + 1) >> 2)] = acc.c1 + acc2.c1;
    }
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  if (tid < ncol) {
    const cplx sc = Xs[tid * (PB + 1) + tid];   // s_c = sqrt(d_c)
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const cplx y = x[(int64_t)(first + c0 + tid) * NR + r];
      tv[tid][r] = cdiv(csub(y, red[tid][r]), sc);
    }
  }
  __syncthreads();
  // x_c = t_c + sum_{i>c} X[i][c] t_i ; 4 threads per column, shuffle-reduced
  {
    const int c = tid >> 2, k = tid & 3;
    cplx xv[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) xv[r] = cmk(0.0, 0.0);
    if (c < ncol) {
#pragma unroll 4
      for (int i = c + 1 + k; i < ncol; i += 4) {
        const cplx w = Xs[i * (PB + 1) + c];
#pragma unroll
        for (int r = 0; r < NR; ++r) xv[r] = cfma(w, tv[i][r], xv[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      double a = xv[r].x, b = xv[r].y;
#pragma unroll
      for (int o = 1; o < 4; o <<= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
      }
      xv[r] = cmk(a, b);
    }
    if (c < ncol && k == 0) {
#pragma unroll
      for (int r = 0; r < NR; ++r)
        x[(int64_t)(first + c0 + c) * NR + r] = cadd(tv[c][r], xv[r]);
      __threadfence();
    }
  }
  __syncthreads();
  if (tid == 0) {
    st_release(flags + cb, epoch);
    if (dep.fused) atomicAdd(sb.done[slot] + s, 1);
  }
}

// Small fronts (npiv <= 64), NR = 4: one warp per (front, pole), up to 8
// column groups of 8 with one accumulator fragment each.
__global__ void __launch_bounds__(256) k_bwd_small_mma4(const int32_t* __restrict__ fronts, int nfr,
                                                        int nslots, FrontsDev F, SolveBatchDev sb) {
  constexpr int NR = 4;
  extern __shared__ cplx dsm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int item = blockIdx.x * 8 + warp;
  if (item >= nfr * nslots) return;
  const int slot = item % nslots;
  const int s = fronts[item / nslots];
  cplx(*tv)[NR] = reinterpret_cast<cplx(*)[NR]>(dsm + warp * PB * NR);
  const int p = F.npiv[s], nf = F.nf[s], first = F.first[s];
  const cplx* panel = sb.factor[slot] + F.panel_off[s];
  cplx* x = sb.x[slot];
  const int* rows = F.rows + F.rows_off[s];
  const int kq = lane & 3, cq = lane >> 2;
  const int rhs = cq & 3;
  const bool hi = cq >= 4;
  const int ncg = (p + 7) >> 3;
  BwdFrag acc[8];
  const cplx* colp = panel + (int64_t)cq * nf;      // column cq of group 0
#pragma unroll 2
  for (int r0 = p; r0 < nf; r0 += 4) {
    const int rho = r0 + kq;
    const bool ron = rho < nf;
    const int g = ron ? __ldg(rows + rho) : 0;
    cplx l[8];
#pragma unroll
    for (int cg = 0; cg < 8; ++cg)
      l[cg] = (cg < ncg && ron && cg * 8 + cq < p) ? __ldg(colp + (int64_t)cg * 8 * nf + rho) : cmk(0.0, 0.0);
    const cplx xv = ron ? x[(int64_t)g * NR + rhs] : cmk(0.0, 0.0);
#pragma unroll
    for (int cg = 0; cg < 8; ++cg)
      if (cg < ncg) acc[cg].mac(l[cg], xv, hi);
  }
  // tv[c] = sum (before the diagonal solve)
#pragma unroll
  for (int cg = 0; cg < 8; ++cg) {
    const int col = cg * 8 + cq;
    if (cg < ncg && col < p) {
      double* rd = reinterpret_cast<double*>(&tv[col][0]);
      const int n0 = 2 * kq;
      rd[2 * (n0 & 3) + (n0 >> 2)] = acc[cg].c0;
      rd[2 * ((n0 + 1) & 3) + ((n0 + 1) >> 2)] = acc[cg].c1;
    }
  }
  __syncwarp();
  // t = (y - sum) / s, then x = X^T t  (X[i][c] at (row c, col i), i > c)
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int c = lane + 32 * h;
    if (c < p) {
      const cplx sc = panel[(int64_t)c * nf + c];   // s_c = sqrt(d_c)
#pragma unroll
      for (int r = 0; r < NR; ++r)
        tv[c][r] = cdiv(csub(x[(int64_t)(first + c) * NR + r], tv[c][r]), sc);
    }
  }
  __syncwarp();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int c = lane + 32 * h;
    if (c < p) {
      cplx xv[NR];
#pragma unroll
      for (int r = 0; r < NR; ++r) xv[r] = tv[c][r];
      for (int i = c + 1; i < p; ++i) {
        const cplx w = __ldg(panel + (int64_t)i * nf + c);
#pragma unroll
        for (int r = 0; r < NR; ++r) xv[r] = cfma(w, tv[i][r], xv[r]);
      }
#pragma unroll
      for (int r = 0; r < NR; ++r) x[(int64_t)(first + c) * NR + r] = xv[r];
    }
  }
}

// ---------------------------------------------------------------------------
// Small fronts (one pivot block, npiv <= 64): one WARP per (front, pole) does
// the whole front -- no tickets, flags or block barriers.  The bottom levels
// of the tree (C4: levels 0-4, ~20k fronts per pole) are all of this kind.
// ---------------------------------------------------------------------------
template <int NR, int MB>
__global__ void __launch_bounds__(256) k_fwd_small(const int32_t* __restrict__ fronts, int nfr,
                                                   int nslots, FrontsDev F, SolveBatchDev sb) {
  extern __shared__ cplx dsm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int item = blockIdx.x * 8 + warp;
  if (item >= nfr * nslots) return;
  const int slot = item % nslots;
  const int s = fronts[item / nslots];
  cplx(*vy)[NR] = reinterpret_cast<cplx(*)[NR]>(dsm + warp * MB * PB * NR);   // [MB*PB][NR]
  const int p = F.npiv[s], nf = F.nf[s], first = F.first[s];
  const cplx* panel = sb.factor[slot] + F.panel_off[s];
  cplx* x = sb.x[slot];
  const cplx* uvec = sb.uvec[slot];
  const int64_t ro = F.rows_off[s];
  // pivot rows: v = b + child contributions
  for (int c = lane; c < p; c += 32) {
    cplx val[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) val[r] = x[(int64_t)(first + c) * NR + r];
    for (int64_t q = F.ucon_ptr[ro + c]; q < F.ucon_ptr[ro + c + 1]; ++q) {
      const int64_t u = F.ucon_idx[q];
#pragma unroll
      for (int r = 0; r < NR; ++r) val[r] = cadd(val[r], uvec[u * NR + r]);
    }
#pragma unroll
    for (int r = 0; r < NR; ++r) vy[c][r] = val[r];
  }
  __syncwarp();
  for (int c0 = 0; c0 < p; c0 += PB) {
    const int pb = min(PB, p - c0);
    // y = X v on this pivot block (X = L_bb^{-1}; X[c][t] sits at (row t, col c))
    cplx yv[2][NR];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = lane + 32 * h;
#pragma unroll
      for (int r = 0; r < NR; ++r) yv[h][r] = cmk(0.0, 0.0);
      if (c < pb) {
        const cplx* xc = panel + (int64_t)(c0 + c) * nf + c0;
#pragma unroll
        for (int r = 0; r < NR; ++r) yv[h][r] = vy[c0 + c][r];
        for (int t = 0; t < c; ++t) {
          const cplx w = __ldg(xc + t);
#pragma unroll
          for (int r = 0; r < NR; ++r) yv[h][r] = cfma(w, vy[c0 + t][r], yv[h][r]);
        }
      }
    }
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = lane + 32 * h;
      if (c < pb) {
        const cplx si = cinv(panel[(int64_t)(c0 + c) * nf + c0 + c]);   // 1 / sqrt(d_c)
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          const cplx y = cmul(yv[h][r], si);
          vy[c0 + c][r] = y;
          x[(int64_t)(first + c0 + c) * NR + r] = y;
        }
      }
    }
    __syncwarp();
    if (MB > 1) {
      // later pivot rows: v -= L[rows, block] y_block
      for (int rho = c0 + PB + lane; rho < p; rho += 32) {
        cplx acc[NR];
#pragma unroll
        for (int r = 0; r < NR; ++r) acc[r] = vy[rho][r];
        const cplx* lrow = panel + (int64_t)c0 * nf + rho;
#pragma unroll 4
        for (int c = 0; c < pb; ++c) {
          const cplx l = __ldg(lrow + (int64_t)c * nf);
#pragma unroll
          for (int r = 0; r < NR; ++r) acc[r] = cfms(l, vy[c0 + c][r], acc[r]);
        }
#pragma unroll
        for (int r = 0; r < NR; ++r) vy[rho][r] = acc[r];
      }
      __syncwarp();
    }
  }
  // border rows: u = contributions - L21 y
  cplx* uout = sb.uvec[slot] + F.uvec_off[s] * NR;
  for (int rho = p + lane; rho < nf; rho += 32) {
    cplx acc[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) acc[r] = cmk(0.0, 0.0);
    for (int64_t q = F.ucon_ptr[ro + rho]; q < F.ucon_ptr[ro + rho + 1]; ++q) {
      const int64_t u = F.ucon_idx[q];
#pragma unroll
      for (int r = 0; r < NR; ++r) acc[r] = cadd(acc[r], uvec[u * NR + r]);
    }
    const cplx* lrow = panel + rho;
#pragma unroll 4
    for (int c = 0; c < p; ++c) {
      const cplx l = __ldg(lrow + (int64_t)c * nf);
#pragma unroll
      for (int r = 0; r < NR; ++r) acc[r] = cfms(l, vy[c][r], acc[r]);
    }
#pragma unroll
    for (int r = 0; r < NR; ++r) uout[(int64_t)(rho - p) * NR + r] = acc[r];
  }
}

template <int NR>
__global__ void __launch_bounds__(256) k_bwd_small(const int32_t* __restrict__ fronts, int nfr,
                                                   int nslots, FrontsDev F, SolveBatchDev sb) {
  extern __shared__ cplx dsm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int item = blockIdx.x * 8 + warp;
  if (item >= nfr * nslots) return;
  const int slot = item % nslots;
  const int s = fronts[item / nslots];
  cplx(*xs)[NR] = reinterpret_cast<cplx(*)[NR]>(dsm + warp * 2 * 32 * NR);   // [32][NR] chunk
  cplx(*tv)[NR] = reinterpret_cast<cplx(*)[NR]>(dsm + 16 * 32 * NR + warp * PB * NR);
  const int p = F.npiv[s], nf = F.nf[s], first = F.first[s];
  const cplx* panel = sb.factor[slot] + F.panel_off[s];
  cplx* x = sb.x[slot];
  const int* rows = F.rows + F.rows_off[s];
  // pivot blocks from the last one down; rows beyond the block are final
  // (ancestors: before this launch; later blocks: written by this warp, so
  // read with coherent loads)
  for (int c0 = ((p - 1) / PB) * PB; c0 >= 0; c0 -= PB) {
    const int pb = min(PB, p - c0);
    cplx acc[2][NR];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int r = 0; r < NR; ++r) acc[h][r] = cmk(0.0, 0.0);
    // rows beyond the block in chunks of 32: gather x then stream L columns
    for (int q0 = c0 + pb; q0 < nf; q0 += 32) {
      const int n = min(32, nf - q0);
      if (lane < n) {
        const int g = __ldg(rows + q0 + lane);
#pragma unroll
        for (int r = 0; r < NR; ++r) xs[lane][r] = x[(int64_t)g * NR + r];
      }
      __syncwarp();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = lane + 32 * h;
        if (c < pb) {
          const cplx* lc = panel + (int64_t)(c0 + c) * nf + q0;
          for (int i = 0; i < n; ++i) {
            const cplx l = __ldg(lc + i);
#pragma unroll
            for (int r = 0; r < NR; ++r) acc[h][r] = cfma(l, xs[i][r], acc[h][r]);
          }
        }
      }
      __syncwarp();
    }
    // t = y / d - acc, then x = X^T t  (X[i][c] at (row c, col i), i > c)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = lane + 32 * h;
      if (c < pb) {
        const cplx sc = panel[(int64_t)(c0 + c) * nf + c0 + c];   // s_c = sqrt(d_c)
#pragma unroll
        for (int r = 0; r < NR; ++r)
          tv[c][r] = cdiv(csub(x[(int64_t)(first + c0 + c) * NR + r], acc[h][r]), sc);
      }
    }
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = lane + 32 * h;
      if (c < pb) {
        cplx xv[NR];
#pragma unroll
        for (int r = 0; r < NR; ++r) xv[r] = tv[c][r];
        for (int i = c + 1; i < pb; ++i) {
          const cplx w = __ldg(panel + (int64_t)(c0 + i) * nf + c0 + c);
#pragma unroll
          for (int r = 0; r < NR; ++r) xv[r] = cfma(w, tv[i][r], xv[r]);
        }
#pragma unroll
        for (int r = 0; r < NR; ++r) x[(int64_t)(first + c0 + c) * NR + r] = xv[r];
      }
    }
    __syncwarp();
  }
}

// RBA_BWD_MMA: 0 = scalar (DFMA) backward kernels for 4 right-hand sides too,
// 1 (default) = tensor-core kernel for the small fronts (C4 levels 0-4:
// 8.5 -> 6.6 ms per 16-pole sweep), 2 = also for the large fronts (measured
// slower, 27 -> 32 ms: the 8 x 64 B segments of an A fragment load keep fewer
// bytes in flight per register than the scalar kernel's 512 B row segments;
// it needs a TMA-fed shared-memory ring to pay)
static int g_bwd_mma = -1;
static int bwd_mma_mode() {
  if (g_bwd_mma < 0) {
    const char* e = getenv("RBA_BWD_MMA");
    g_bwd_mma = e ? atoi(e) : 1;
  }
  return g_bwd_mma;
}
// re-read the environment (every rba_ctx_create: the tests switch variants per context)
void solve_env_refresh() { g_bwd_mma = -1; }
static bool bwd_mma_on() { return bwd_mma_mode() >= 1; }

template <int NR>
static void small_nr(cudaStream_t st, bool forward, const int32_t* fronts, int nfr, int nslots,
                     const FrontsDev& F, const SolveBatchDev& sb, int mb) {
  const int items = nfr * nslots;
  const int grid = (items + 7) / 8;
  if (forward) {
    if (mb <= 1) {
      const size_t smem = 8 * PB * NR * sizeof(cplx);
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(k_fwd_small<NR, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
      }
      k_fwd_small<NR, 1><<<grid, 256, smem, st>>>(fronts, nfr, nslots, F, sb);
    } else {
      const size_t smem = 8 * 2 * PB * NR * sizeof(cplx);
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(k_fwd_small<NR, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
      }
      k_fwd_small<NR, 2><<<grid, 256, smem, st>>>(fronts, nfr, nslots, F, sb);
    }
  } else if (NR == 4 && mb <= 1 && bwd_mma_on()) {   // one pivot block per front
    k_bwd_small_mma4<<<grid, 256, 8 * PB * NR * sizeof(cplx), st>>>(fronts, nfr, nslots, F, sb);
  } else {
    const size_t smem = (16 * 32 * NR + 8 * PB * NR) * sizeof(cplx);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_bwd_small<NR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr = true;
    }
    k_bwd_small<NR><<<grid, 256, smem, st>>>(fronts, nfr, nslots, F, sb);
  }
}

void launch_solve_small(cudaStream_t st, bool forward, int nr, const int32_t* fronts, int nfr,
                        int nslots, const FrontsDev& F, const SolveBatch& b, int mb) {
  if (nfr <= 0) return;
  SolveBatchDev sb;
  for (int i = 0; i < nslots; ++i) {
    sb.factor[i] = b.factor[i];
    sb.x[i] = b.x[i];
    sb.uvec[i] = b.uvec[i];
    sb.flags[i] = nullptr;
    sb.done[i] = nullptr;
    sb.epoch[i] = 0;
  }
  switch (nr) {
    case 1: small_nr<1>(st, forward, fronts, nfr, nslots, F, sb, mb); break;
    case 2: small_nr<2>(st, forward, fronts, nfr, nslots, F, sb, mb); break;
    case 4: small_nr<4>(st, forward, fronts, nfr, nslots, F, sb, mb); break;
    default: small_nr<8>(st, forward, fronts, nfr, nslots, F, sb, mb); break;
  }
}

template <int NR>
static void fwd_nr(cudaStream_t st, const SolveTask* tasks, int ntasks, int nslots,
                   const FrontsDev& F, const SolveBatchDev& sb, int* ticket, int epoch,
                   const SweepDeps& dep, bool stagex) {
  const size_t smem0 = (9 * PB * NR) * sizeof(cplx);
  const size_t smem1 = smem0 + PB * (PB + 1) * sizeof(cplx);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_fwd<NR, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem0);
    cudaFuncSetAttribute(k_fwd<NR, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1);
    attr = true;
  }
  // staging the diagonal block only pays where the pivot chain dominates
  if (stagex)
    k_fwd<NR, true><<<ntasks * nslots, 256, smem1, st>>>(tasks, nslots, F, sb, ticket, epoch, dep);
  else
    k_fwd<NR, false><<<ntasks * nslots, 256, smem0, st>>>(tasks, nslots, F, sb, ticket, epoch, dep);
}
template <int NR, int NW>
static void bwd_nw(cudaStream_t st, const SolveTask* tasks, int ntasks, int nslots,
                   const FrontsDev& F, const SolveBatchDev& sb, int* ticket, int epoch,
                   const SweepDeps& dep) {
  const size_t smem = (2 * PB * NR + PB * (PB + 1)) * sizeof(cplx);  // + staged X
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_bwd<NR, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  k_bwd<NR, NW><<<ntasks * nslots, 32 * NW, smem, st>>>(tasks, nslots, F, sb, ticket, epoch, dep);
}
static int g_bwd_nw = -1;
template <int NR>
static void bwd_nr(cudaStream_t st, const SolveTask* tasks, int ntasks, int nslots,
                   const FrontsDev& F, const SolveBatchDev& sb, int* ticket, int epoch,
                   const SweepDeps& dep) {
  if (NR == 4 && bwd_mma_mode() >= 2) {
    const size_t smem = (2 * PB * NR + PB * (PB + 1) + BCH * NR) * sizeof(cplx);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_bwd_mma4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr = true;
    }
    k_bwd_mma4<<<ntasks * nslots, 256, smem, st>>>(tasks, nslots, F, sb, ticket, dep);
    return;
  }
  if (g_bwd_nw < 0) {
    const char* e = getenv("RBA_BWD_NW");
    g_bwd_nw = (e && atoi(e) == 32) ? 32 : 16;
  }
  if (g_bwd_nw == 16) bwd_nw<NR, 16>(st, tasks, ntasks, nslots, F, sb, ticket, epoch, dep);
  else bwd_nw<NR, 32>(st, tasks, ntasks, nslots, F, sb, ticket, epoch, dep);
}

void launch_solve_level(cudaStream_t st, bool forward, int nr, const SolveTask* tasks,
                        int ntasks, int nslots, const FrontsDev& F, const SolveBatch& b,
                        int* ticket, int epoch, const int32_t* parent, const int32_t* need_u,
                        bool fused, bool stagex) {
  if (ntasks <= 0) return;
  SolveBatchDev sb;
  for (int i = 0; i < nslots; ++i) {
    sb.factor[i] = b.factor[i];
    sb.x[i] = b.x[i];
    sb.uvec[i] = b.uvec[i];
    sb.flags[i] = forward ? b.flags_f[i] : b.flags_b[i];
    sb.done[i] = forward ? b.done_f[i] : b.done_b[i];
    sb.epoch[i] = b.epoch[i];
  }
  SweepDeps dep{parent, need_u, fused ? 1 : 0};
  switch (nr) {
    case 1: forward ? fwd_nr<1>(st, tasks, ntasks, nslots, F, sb, ticket, epoch, dep, stagex)
                    : bwd_nr<1>(st, tasks, ntasks, nslots, F, sb, ticket, epoch, dep); break;
    case 2: forward ? fwd_nr<2>(st, tasks, ntasks, nslots, F, sb, ticket, epoch, dep, stagex)
                    : bwd_nr<2>(st, tasks, ntasks, nslots, F, sb, ticket, epoch, dep); break;
    case 4: forward ? fwd_nr<4>(st, tasks, ntasks, nslots, F, sb, ticket, epoch, dep, stagex)
                    : bwd_nr<4>(st, tasks, ntasks, nslots, F, sb, ticket, epoch, dep); break;
    default: forward ? fwd_nr<8>(st, tasks, ntasks, nslots, F, sb, ticket, epoch, dep, stagex)
                     : bwd_nr<8>(st, tasks, ntasks, nslots, F, sb, ticket, epoch, dep); break;
  }
}

// ---------------------------------------------------------------------------
// Backward sweep of the receiver-Green build as FP64 tensor-core GEMMs: Z holds
// y' = L'^{-1} Q^T (N x Mr, row-major, from the pruned forward sweeps); each
// task (front s, pivot block cb) computes, for all Mr columns at once,
//   T   = Z[block rows] - L'[rows beyond block, block]^T Z[rows beyond block]
//   Z[block rows] = X^T S^{-1} T
// i.e. the k_bwd recurrence with Mr right-hand sides, where the row reduction
// is a DMMA GEMM (K = rows beyond the block) instead of a GEMV per RHS.  CTA
// tile 64 (block columns) x 32 (receivers), 4 warps of 32x16, 4 real DMMAs per
// complex product, operands staged by cp.async in a 3-stage pipeline; the CTA
// walks the receiver chunks.  Rows beyond the block: border rows (ancestor
// pivots, final before this launch) first, then the later pivot blocks of the
// same front from the last one down (earlier tickets; flag waits).
// ---------------------------------------------------------------------------
namespace {
constexpr int ZMC = 32;           // receiver columns per chunk
template <int ZK>                 // k (rows) per stage
struct ZStage {
  static constexpr int ZLK = ZK + 4;   // padded [row][k] stride (complex): conflict-free LDS.128
  cplx a[PB * ZLK];               // [block column i][k]
  cplx b[ZMC * ZLK];              // [receiver n][k]
};
}  // namespace

template <int ZK, int ZNS>
__global__ void __launch_bounds__(128) k_zbwd(const SolveTask* __restrict__ tasks, int nslots,
                                              FrontsDev F, SolveBatchDev sb, int* ticket, int Mr,
                                              SlotPtrs Zp) {
  using ZStage = ::rba::ZStage<ZK>;
  constexpr int ZLK = ZStage::ZLK;
  extern __shared__ __align__(16) unsigned char zsm[];
  ZStage* st = reinterpret_cast<ZStage*>(zsm);
  cplx(*Ts)[ZMC + 1] = reinterpret_cast<cplx(*)[ZMC + 1]>(zsm);   // overlays the stages
  __shared__ int s_t;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_t = atomicAdd(ticket, 1);
  __syncthreads();
  const int t = s_t;
  const int slot = t % nslots;
  const int epoch = sb.epoch[slot];
  const SolveTask tk = tasks[t / nslots];
  const int s = tk.s, cb = tk.blk;
  const int p = F.npiv[s], nf = F.nf[s], first = F.first[s];
  const int npb = (p + PB - 1) / PB;
  const cplx* panel = sb.factor[slot] + F.panel_off[s];
  cplx* Z = Zp.p[slot];
  // completion flags per (pivot block, receiver chunk): a chunk of block cb
  // only waits for the same chunk of the later blocks, so the chains of the
  // chunks pipeline
  const int nmc = (Mr + ZMC - 1) / ZMC;
  int* flags = sb.flags[slot] + F.blk_off[s] * nmc;
  const int c0 = cb * PB, kb = min(PB, p - c0);
  const int* rows = F.rows + F.rows_off[s];
  const int nbord = nf - p;                    // border rows p .. nf-1
  const int kbord = (nbord + ZK - 1) / ZK;     // border chunks (last one partial)
  // later pivot blocks cb+1 .. npb-1, last (possibly partial) block first
  const int clast = cb < npb - 1 ? (p - (npb - 1) * PB + ZK - 1) / ZK : 0;
  const int nchunk = kbord + clast + (cb < npb - 1 ? (npb - 2 - cb) * (PB / ZK) : 0);
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 16;
  const int g = lane >> 2, t4 = lane & 3;

  for (int m0 = 0; m0 < Mr; m0 += ZMC) {
    const int nm = min(ZMC, Mr - m0), mc = m0 / ZMC;
    // stage chunk ch: k rows rho_k, A[i][k] = L'[rho_k, c0+i], B[n][k] = Z[idx(rho_k)][m0+n]
    auto issue = [&](int ch) {
      if (ch >= nchunk) {
        asm volatile("cp.async.commit_group;\n" ::: "memory");
        return;
      }
      ZStage& S = st[ch % ZNS];
      int rho0, nval;
      if (ch < kbord) {
        rho0 = p + ch * ZK;
        nval = min(ZK, nf - rho0);
      } else {
        const int q = ch - kbord;
        int rb, sub;
        if (q < clast) {
          rb = npb - 1;
          sub = q;
        } else {
          rb = npb - 2 - (q - clast) / (PB / ZK);
          sub = (q - clast) % (PB / ZK);
        }
        rho0 = rb * PB + sub * ZK;
        nval = min(ZK, min(p, rb * PB + PB) - rho0);
        if (sub == 0) {
          // first chunk of block rb: its Z rows must be final
          if (tid == 0) spin_wait_geq(flags + rb * nmc + mc, epoch);
          __syncthreads();
        }
      }
#pragma unroll
      for (int q = 0; q < (PB * ZK) / 128; ++q) {
        const int e = tid + q * 128;
        const int kk = e % ZK, i = e / ZK;
        const bool ok = kk < nval && i < kb;
        cp_async16(&S.a[i * ZLK + kk], panel + (ok ? (int64_t)(c0 + i) * nf + rho0 + kk : 0), ok);
      }
#pragma unroll
      for (int q = 0; q < (ZMC * ZK) / 128; ++q) {
        const int e = tid + q * 128;
        const int n = e % ZMC, kk = e / ZMC;
        const bool ok = kk < nval && n < nm;
        const int rho = rho0 + kk;
        const int64_t zr = ok ? (rho < p ? (int64_t)(first + rho) : (int64_t)__ldg(rows + rho)) : 0;
        cp_async16(&S.b[n * ZLK + kk], Z + (ok ? zr * Mr + m0 + n : 0), ok);
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    double cre[4][2][2], cim[4][2][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        cre[a][b][0] = cre[a][b][1] = 0.0;
        cim[a][b][0] = cim[a][b][1] = 0.0;
      }
    for (int c = 0; c < ZNS - 1; ++c) issue(c);
    for (int ch = 0; ch < nchunk; ++ch) {
      asm volatile("cp.async.wait_group %0;\n" ::"n"(ZNS - 2) : "memory");
      __syncthreads();
      issue(ch + ZNS - 1);
      const ZStage& S = st[ch % ZNS];
      if (wm >= kb || wn >= nm) continue;   // warp tile entirely outside the block / chunk
#pragma unroll
      for (int k4 = 0; k4 < ZK; k4 += 4) {
        double ar[4], ai[4], an[4], br[2], bi[2];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const cplx v = S.a[(wm + a * 8 + g) * ZLK + k4 + t4];
          ar[a] = v.x;
          ai[a] = v.y;
          an[a] = -v.y;
        }
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          const cplx v = S.b[(wn + b * 8 + g) * ZLK + k4 + t4];
          br[b] = v.x;
          bi[b] = v.y;
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 2; ++b) dmma_f64(cre[a][b][0], cre[a][b][1], ar[a], br[b]);
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 2; ++b) dmma_f64(cim[a][b][0], cim[a][b][1], ar[a], bi[b]);
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 2; ++b) dmma_f64(cre[a][b][0], cre[a][b][1], an[a], bi[b]);
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 2; ++b) dmma_f64(cim[a][b][0], cim[a][b][1], ai[a], br[b]);
      }
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    // T = (Z[block rows] - acc) / s  -> shared memory
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int i = wm + a * 8 + g, n = wn + b * 8 + t4 * 2 + h;
          if (i < kb && n < nm) {
            const cplx y = Z[(int64_t)(first + c0 + i) * Mr + m0 + n];
            const cplx sc = __ldg(panel + (int64_t)(c0 + i) * nf + c0 + i);
            Ts[i][n] = cdiv(cmk(y.x - cre[a][b][h], y.y - cim[a][b][h]), sc);
          }
        }
    __syncthreads();
    // Z[block rows] = X^T T :  out_i = T_i + sum_{j > i} X[j][i] T_j, X[j][i] at (row c0+i, col c0+j)
    {
      const int n = tid % ZMC, ig = tid / ZMC;
      for (int i = ig; i < kb; i += 128 / ZMC) {
        cplx acc = Ts[i][n];
        const cplx* xr = panel + (int64_t)c0 * nf + c0 + i;
        for (int j = i + 1; j < kb; ++j) acc = cfma(__ldg(xr + (int64_t)j * nf), Ts[j][n], acc);
        if (n < nm) Z[(int64_t)(first + c0 + i) * Mr + m0 + n] = acc;
      }
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) st_release(flags + cb * nmc + mc, epoch);
  }
}

template <int ZK, int ZNS>
static void zbwd_go(cudaStream_t st, const SolveTask* tasks, int ntasks, int nslots,
                    const FrontsDev& F, const SolveBatchDev& sb, int* ticket, int Mr,
                    const SlotPtrs& Z) {
  const size_t smem = std::max(ZNS * sizeof(ZStage<ZK>), PB * (ZMC + 1) * sizeof(cplx));
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_zbwd<ZK, ZNS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  k_zbwd<ZK, ZNS><<<ntasks * nslots, 128, smem, st>>>(tasks, nslots, F, sb, ticket, Mr, Z);
}

void launch_zbwd(cudaStream_t st, const SolveTask* tasks, int ntasks, int nslots,
                 const FrontsDev& F, const SolveBatch& b, int* ticket, int Mr, const SlotPtrs& Z) {
  if (ntasks <= 0) return;
  SolveBatchDev sb;
  for (int i = 0; i < nslots; ++i) {
    sb.factor[i] = b.factor[i];
    sb.x[i] = b.x[i];
    sb.uvec[i] = b.uvec[i];
    sb.flags[i] = b.flags_b[i];
    sb.done[i] = b.done_b[i];
    sb.epoch[i] = b.epoch[i];
  }
  static int var = -1;
  if (var < 0) {
    const char* e = getenv("RBA_ZBWD");
    var = e ? atoi(e) : 1;
  }
  // 1 (default): 16 rows x 2 stages; 0: 8 x 3; 2: 16 x 3
  if (var == 1) zbwd_go<16, 2>(st, tasks, ntasks, nslots, F, sb, ticket, Mr, Z);
  else if (var == 2) zbwd_go<16, 3>(st, tasks, ntasks, nslots, F, sb, ticket, Mr, Z);
  else zbwd_go<8, 3>(st, tasks, ntasks, nslots, F, sb, ticket, Mr, Z);
}

// ---------------------------------------------------------------------------
// Forward sweep of the large fronts with NR (8) right-hand sides as FP64
// tensor-core GEMM tasks -- the k_fwd recurrence (task = front s, 64-row block
// blk; see k_fwd) with the row reduction done by DMMA:
//   T = L'[rows of blk, pivot columns < jmax] Y[pivot columns < jmax]   (GEMM,
//       K = the previous pivot columns, NR columns of y)
//   pivot block : y_blk = S^{-1} X_blk (v_blk - T)    (v = rhs + child u-vectors)
//   border block: u     = (child u-vectors) - T       -> parent
// CTA tile 64 rows x ZMC columns (the NR used ones), 4 warps of 32 x 16, 4 real
// DMMAs per complex product, cp.async 2-stage pipeline over k; the flag of
// pivot block j is awaited at the first k chunk of block j (earlier tickets).
// ---------------------------------------------------------------------------
template <int ZK, int ZNS>
__global__ void __launch_bounds__(128) k_zfwd(const SolveTask* __restrict__ tasks, int nslots,
                                              FrontsDev F, SolveBatchDev sb, int* ticket, int NR) {
  using ZStage = ::rba::ZStage<ZK>;
  constexpr int ZLK = ZStage::ZLK;
  extern __shared__ __align__(16) unsigned char zsm[];
  ZStage* st = reinterpret_cast<ZStage*>(zsm);
  cplx(*Vs)[ZMC + 1] = reinterpret_cast<cplx(*)[ZMC + 1]>(zsm);   // overlays the stages
  __shared__ int s_t;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_t = atomicAdd(ticket, 1);
  __syncthreads();
  const int t = s_t;
  const int slot = t % nslots;
  const int epoch = sb.epoch[slot];
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
  const int jmax = pivot ? blk : npb;                 // pivot blocks entering the product
  const int kend = min(jmax * PB, p);
  const int nchunk = (kend + ZK - 1) / ZK;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 16;
  const int g = lane >> 2, t4 = lane & 3;
  auto issue = [&](int ch) {
    if (ch >= nchunk) {
      asm volatile("cp.async.commit_group;\n" ::: "memory");
      return;
    }
    ZStage& S = st[ch % ZNS];
    const int k0 = ch * ZK;
    const int nval = min(ZK, kend - k0);
    if (k0 % PB == 0) {
      // first chunk of pivot block k0 / PB: its y rows must be final
      if (tid == 0) spin_wait_geq(flags + k0 / PB, epoch);
      __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < (PB * ZK) / 128; ++q) {
      const int e = tid + q * 128;
      const int i = e % PB, kk = e / PB;              // A[i][k] = L'[r0 + i, k0 + kk]
      const bool ok = kk < nval && i < nr;
      cp_async16(&S.a[i * ZLK + kk], panel + (ok ? (int64_t)(k0 + kk) * nf + r0 + i : 0), ok);
    }
#pragma unroll
    for (int q = 0; q < (ZMC * ZK) / 128; ++q) {
      const int e = tid + q * 128;
      const int n = e % ZMC, kk = e / ZMC;            // B[n][k] = y[first + k0 + kk][n]
      const bool ok = kk < nval && n < NR;
      cp_async16(&S.b[n * ZLK + kk], x + (ok ? (int64_t)(first + k0 + kk) * NR + n : 0), ok);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  double cre[4][2][2], cim[4][2][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int bb = 0; bb < 2; ++bb) {
      cre[a][bb][0] = cre[a][bb][1] = 0.0;
      cim[a][bb][0] = cim[a][bb][1] = 0.0;
    }
  for (int c = 0; c < ZNS - 1; ++c) issue(c);
  for (int ch = 0; ch < nchunk; ++ch) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(ZNS - 2) : "memory");
    __syncthreads();
    issue(ch + ZNS - 1);
    const ZStage& S = st[ch % ZNS];
    if (wm >= nr || wn >= NR) continue;               // warp tile outside the rows / columns
#pragma unroll
    for (int k4 = 0; k4 < ZK; k4 += 4) {
      double ar[4], ai[4], an[4], br[2], bi[2];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const cplx v = S.a[(wm + a * 8 + g) * ZLK + k4 + t4];
        ar[a] = v.x;
        ai[a] = v.y;
        an[a] = -v.y;
      }
#pragma unroll
      for (int bb = 0; bb < 2; ++bb) {
        const cplx v = S.b[(wn + bb * 8 + g) * ZLK + k4 + t4];
        br[bb] = v.x;
        bi[bb] = v.y;
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int bb = 0; bb < 2; ++bb) dmma_f64(cre[a][bb][0], cre[a][bb][1], ar[a], br[bb]);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int bb = 0; bb < 2; ++bb) dmma_f64(cim[a][bb][0], cim[a][bb][1], ar[a], bi[bb]);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int bb = 0; bb < 2; ++bb) dmma_f64(cre[a][bb][0], cre[a][bb][1], an[a], bi[bb]);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int bb = 0; bb < 2; ++bb) dmma_f64(cim[a][bb][0], cim[a][bb][1], ai[a], br[bb]);
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  // v = (rhs for pivot rows) + child u-vectors, in shared memory
  for (int e = tid; e < nr * NR; e += 128) {
    const int i = e / NR, r = e % NR;
    const int rho = r0 + i;
    cplx val = pivot ? x[(int64_t)(first + rho) * NR + r] : cmk(0.0, 0.0);
    const int64_t fr = F.rows_off[s] + rho;
    for (int64_t q = F.ucon_ptr[fr]; q < F.ucon_ptr[fr + 1]; ++q)
      val = cadd(val, uvec[F.ucon_idx[q] * NR + r]);
    Vs[i][r] = val;
  }
  __syncthreads();
  // v - T
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int bb = 0; bb < 2; ++bb)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = wm + a * 8 + g, n = wn + bb * 8 + t4 * 2 + h;
        if (i < nr && n < NR) Vs[i][n] = cmk(Vs[i][n].x - cre[a][bb][h], Vs[i][n].y - cim[a][bb][h]);
      }
  __syncthreads();
  if (!pivot) {
    cplx* u = sb.uvec[slot] + (F.uvec_off[s] + (r0 - p)) * NR;
    for (int e = tid; e < nr * NR; e += 128) u[e] = Vs[e / NR][e % NR];
    return;
  }
  // y_i = s_i^{-1} (v_i + sum_{c < i} X[i][c] v_c); X[i][c] sits at (row r0+c, col r0+i)
  for (int e = tid; e < nr * NR; e += 128) {
    const int i = e / NR, r = e % NR;
    const cplx* xcol = panel + (int64_t)(r0 + i) * nf + r0;
    cplx acc = Vs[i][r];
    for (int c = 0; c < i; ++c) acc = cfma(__ldg(xcol + c), Vs[c][r], acc);
    x[(int64_t)(first + r0 + i) * NR + r] = cmul(acc, cinv(__ldg(xcol + i)));
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) st_release(flags + blk, epoch);
}

void launch_zfwd(cudaStream_t st, const SolveTask* tasks, int ntasks, int nslots,
                 const FrontsDev& F, const SolveBatch& b, int* ticket, int NR) {
  if (ntasks <= 0) return;
  SolveBatchDev sb;
  for (int i = 0; i < nslots; ++i) {
    sb.factor[i] = b.factor[i];
    sb.x[i] = b.x[i];
    sb.uvec[i] = b.uvec[i];
    sb.flags[i] = b.flags_f[i];
    sb.done[i] = b.done_f[i];
    sb.epoch[i] = b.epoch[i];
  }
  constexpr int ZK = 16, ZNS = 2;
  const size_t smem = std::max(ZNS * sizeof(ZStage<ZK>), PB * (ZMC + 1) * sizeof(cplx));
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_zfwd<ZK, ZNS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  k_zfwd<ZK, ZNS><<<ntasks * nslots, 128, smem, st>>>(tasks, nslots, F, sb, ticket, NR);
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
