// Numeric factorisation kernels: M(sigma) assembly (K1), shifted values
// scattered into the fronts (K2), multifrontal extend-add (K3), dense
// partial complex-symmetric LDL^T of the fronts (K4: diagonal block + panel
// TRSM, then GEMM updates).  Replaces SuperLU's numeric factorisation
// (/root/reference/pkg/src/rbainv/shifted.py:54) and assemble_M
// (/root/reference/pkg/src/rbainv/mesh.py:348-355).
#include "fronts.cuh"
#include "kernels.h"

namespace rba {

// ---------------------------------------------------------------------------
// K1: M values in the fixed lower-triangle pattern, deterministic gather.
// Mv[e] = sum_{q in contrib(e)} mass[off_q] * exp(m[cell_q]) (list order).
// ---------------------------------------------------------------------------
__global__ void k_exp(int64_t n, const double* __restrict__ m, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = exp(m[i]);
}

__global__ void k_assemble_M(int64_t nnz, const int64_t* __restrict__ cptr,
                             const int64_t* __restrict__ coff, const double* __restrict__ mass,
                             const double* __restrict__ expm, int k2, double* __restrict__ Mv) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    const int64_t q1 = cptr[e + 1];
    for (int64_t q = cptr[e]; q < q1; ++q) {
      const int64_t off = coff[q];
      acc = __dadd_rn(acc, __dmul_rn(__ldg(mass + off), __ldg(expm + off / k2)));
    }
    Mv[e] = acc;
  }
}

void launch_assemble_M(cudaStream_t st, int64_t nnz, const int64_t* cptr, const int64_t* coff,
                       const double* mass, const double* m, double* expm, int64_t P, int k2,
                       double* Mv) {
  k_exp<<<(int)std::min<int64_t>((P + 255) / 256, 148 * 16), 256, 0, st>>>(P, m, expm);
  k_assemble_M<<<(int)std::min<int64_t>((nnz + 255) / 256, 148 * 32), 256, 0, st>>>(
      nnz, cptr, coff, mass, expm, k2, Mv);
}

// ---------------------------------------------------------------------------
// K2: A_i = K - xi_i M scattered into the pivot columns of the fronts.
// ---------------------------------------------------------------------------
__global__ void k_scatter_A(int64_t nnz, const int64_t* __restrict__ tgt,
                            const double* __restrict__ Kv, const double* __restrict__ Mv,
                            PoleBatch pb) {
  const int slot = blockIdx.y;
  cplx* fac = pb.factor[slot];
  const cplx xi = pb.xi[slot];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double k = Kv[e], m = Mv[e];
    fac[tgt[e]] = cmk(k - xi.x * m, -xi.y * m);
  }
}

void launch_scatter_A(cudaStream_t st, int64_t nnz, const int64_t* tgt, const double* Kv,
                      const double* Mv, const PoleBatch& pb) {
  dim3 grid((unsigned)std::min<int64_t>((nnz + 255) / 256, 148 * 16), pb.count);
  k_scatter_A<<<grid, 256, 0, st>>>(nnz, tgt, Kv, Mv, pb);
}

// ---------------------------------------------------------------------------
// K3: extend-add.  One CTA per (front, 32-column tile): zero the update-block
// columns of the tile, then add every child's update block restricted to the
// tile, children in ascending order (deterministic, no atomics).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int lower_bound_i32(const int32_t* a, int n, int v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(256) k_extend_add(const int2* __restrict__ tasks, FrontsDev F,
                                                    PoleBatch pb) {
  const int slot = blockIdx.y;
  const int2 tk = tasks[blockIdx.x];
  const int s = tk.x;
  const int nf = F.nf[s], p = F.npiv[s];
  cplx* panel = pb.factor[slot] + F.panel_off[s];
  cplx* upd = pb.upd[slot] + (F.upd_off[s] >= 0 ? F.upd_off[s] : 0);
  if (tk.y < 0) {
    // whole (small) front in one CTA: zero the packed update block, then
    // add each child's packed block column by column
    const int r = nf - p;
    for (int64_t q = threadIdx.x; q < (int64_t)r * (r + 1) / 2; q += blockDim.x)
      upd[q] = cmk(0.0, 0.0);
    __syncthreads();
    for (int ci = F.child_ptr[s]; ci < F.child_ptr[s + 1]; ++ci) {
      const int ch = F.child_list[ci];
      const int rc = F.nf[ch] - F.npiv[ch];
      const int32_t* rm = F.relmap + F.rel_off[ch];
      const cplx* U = pb.upd[slot] + F.upd_off[ch];
      // all (column, row) pairs of the child's block at once: a small child has
      // fewer rows than the CTA has threads (each parent entry still receives
      // exactly one addend per child, children in order: same sums)
      for (int q = threadIdx.x; q < rc * rc; q += blockDim.x) {
        const int j = q / rc, i = q - j * rc;
        if (i >= j) {
          cplx* dst = faddr(panel, upd, p, nf, rm[i], rm[j]);
          *dst = cadd(*dst, U[ucol(j, rc) + (i - j)]);
        }
      }
      __syncthreads();
    }
    return;
  }
  const int c0 = tk.y * 32, c1 = min(c0 + 32, nf);
  // zero update-block columns (rows >= column)
  for (int c = max(c0, p); c < c1; ++c)
    for (int r = c + threadIdx.x; r < nf; r += blockDim.x)
      upd[ucol(c - p, nf - p) + (r - c)] = cmk(0.0, 0.0);
  __syncthreads();
  for (int ci = F.child_ptr[s]; ci < F.child_ptr[s + 1]; ++ci) {
    const int ch = F.child_list[ci];
    const int rc = F.nf[ch] - F.npiv[ch];
    const int32_t* rm = F.relmap + F.rel_off[ch];
    const int j0 = lower_bound_i32(rm, rc, c0), j1 = lower_bound_i32(rm, rc, c1);
    const cplx* U = pb.upd[slot] + F.upd_off[ch];
    for (int j = j0; j < j1; ++j) {
      const int tc = rm[j];
      const cplx* Uc = U + ucol(j, rc);
      for (int i = j + threadIdx.x; i < rc; i += blockDim.x) {
        cplx* dst = faddr(panel, upd, p, nf, rm[i], tc);
        *dst = cadd(*dst, Uc[i - j]);
      }
    }
    __syncthreads();
  }
}

void launch_extend_add(cudaStream_t st, const int2* tasks, int ntasks, const FrontsDev& F,
                       const PoleBatch& pb) {
  if (ntasks <= 0) return;
  dim3 grid(ntasks, pb.count);
  k_extend_add<<<grid, 256, 0, st>>>(tasks, F, pb);
}

// ---------------------------------------------------------------------------
// K4a: diagonal block LDL^T (one CTA per front, shared memory), written back
// in place: unit-lower L below the diagonal, D on the diagonal, and the
// inverse X = L^{-1} (unit lower) stored TRANSPOSED in the otherwise unused
// strictly-upper triangle (X[i][j] at row j, column i).  The inverse turns the
// panel TRSM into a tensor-core GEMM and the solve's diagonal-block
// substitutions into GEMVs (no sequential chains inside a block).
// ---------------------------------------------------------------------------
constexpr int LDS = PB + 1;

__global__ void __launch_bounds__(256) k_diag(const PanelTask* __restrict__ tasks, FrontsDev F,
                                              PoleBatch pb, int* err) {
  extern __shared__ cplx sm[];
  cplx* Dg = sm;  // [PB][LDS] row-major
  const int slot = blockIdx.y;
  const PanelTask tk = tasks[blockIdx.x];
  const int s = tk.s, k0 = tk.k0;
  const int nf = F.nf[s], p = F.npiv[s];
  const int kb = min(PB, p - k0);
  cplx* panel = pb.factor[slot] + F.panel_off[s];
  const int tid = threadIdx.x;
  for (int idx = tid; idx < kb * kb; idx += blockDim.x) {
    int i = idx % kb, j = idx / kb;
    if (i >= j) Dg[i * LDS + j] = panel[(int64_t)(k0 + j) * nf + k0 + i];
  }
  __syncthreads();
  for (int j = 0; j < kb; ++j) {
    const cplx d = Dg[j * LDS + j];
    const bool bad = !(isfinite(d.x) && isfinite(d.y)) || (d.x == 0.0 && d.y == 0.0);
    if (bad && tid == 0) atomicCAS(err, 0, 1 + s);
    const cplx dinv = cinv(d);
    const int rem = kb - j - 1;
    for (int q = tid; q < rem * rem; q += blockDim.x) {
      int c = j + 1 + q / rem, i = j + 1 + q % rem;
      if (i >= c) {
        cplx w = Dg[i * LDS + j];
        cplx l = cmul(Dg[c * LDS + j], dinv);
        Dg[i * LDS + c] = cfms(w, l, Dg[i * LDS + c]);
      }
    }
    __syncthreads();
    for (int i = j + 1 + tid; i < kb; i += blockDim.x) Dg[i * LDS + j] = cmul(Dg[i * LDS + j], dinv);
    __syncthreads();
  }
  // X = L^{-1}: one column per thread, forward substitution down the column
  cplx* Xs = sm + PB * LDS;
  if (tid < kb) {
    const int j = tid;
    for (int i = j + 1; i < kb; ++i) {
      cplx acc = Dg[i * LDS + j];
      for (int t = j + 1; t < i; ++t) acc = cfma(Dg[i * LDS + t], Xs[t * LDS + j], acc);
      Xs[i * LDS + j] = cmk(-acc.x, -acc.y);
    }
  }
  __syncthreads();
  // diagonal slot: s_j = sqrt(d_j) (factor format, see fronts.cuh)
  for (int idx = tid; idx < kb * kb; idx += blockDim.x) {
    int i = idx % kb, j = idx / kb;
    panel[(int64_t)(k0 + j) * nf + k0 + i] =
        i > j ? Dg[i * LDS + j] : (i == j ? csqrt_c(Dg[i * LDS + i]) : Xs[j * LDS + i]);
  }
}

// K4a (v2): the same diagonal-block LDL^T + inverse, blocked by 16 so that
// only ~20 block barriers remain (v1: two per pivot).  Warp 0 factors each
// 16x16 diagonal sub-block with warp barriers, all threads do the sub-panel
// TRSM and the trailing update; the inverse is built block-row by block-row
// (X_ij = -X_ii sum_k L_ik X_kj).
constexpr int SB = 16;

template <int BK>   // maximum block size: 64 (PB), or 32 (small fronts: 128 threads,
                   // 4x less shared memory, several more CTAs per SM)
__global__ void __launch_bounds__(BK <= 48 ? 128 : 256) k_diag2(const PanelTask* __restrict__ tasks, FrontsDev F,
                                               PoleBatch pb, int* err) {
  // Dg holds L (lower) and, transposed in the free upper triangle, X = L^{-1}
  // (X[i][j], i > j, at Dg[j][i]) -- exactly the panel layout written back.
  // Ts is one 16-row block row of T; 85 KB in all -> 2 CTAs per SM.
  constexpr int LDS = BK + 1;
  extern __shared__ cplx sm[];
  cplx* Dg = sm;                   // [BK][LDS]
  cplx* Ts = sm + BK * LDS;        // [SB][LDS]
  cplx* dv = Ts + SB * LDS;        // [BK]
  cplx* di = dv + BK;              // [BK]
  const int slot = blockIdx.y;
  const PanelTask tk = tasks[blockIdx.x];
  const int s = tk.s, k0 = tk.k0;
  const int nf = F.nf[s], p = F.npiv[s];
  const int kb = min(BK, p - k0);
  cplx* panel = pb.factor[slot] + F.panel_off[s];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int idx = tid; idx < kb * kb; idx += blockDim.x) {
    int i = idx % kb, j = idx / kb;
    if (i >= j) Dg[i * LDS + j] = panel[(int64_t)(k0 + j) * nf + k0 + i];
  }
  __syncthreads();
  const int nsub = (kb + SB - 1) / SB;
  for (int sbk = 0; sbk < nsub; ++sbk) {
    const int b0 = sbk * SB, b1 = min(b0 + SB, kb);
    if (warp == 0) {
      for (int j = b0; j < b1; ++j) {
        if (lane == 0) {
          const cplx d = Dg[j * LDS + j];
          const bool bad = !(isfinite(d.x) && isfinite(d.y)) || (d.x == 0.0 && d.y == 0.0);
          if (bad) atomicCAS(err, 0, 1 + s);
          dv[j] = d;
          di[j] = cinv(d);
        }
        __syncwarp();
        const cplx dij = di[j];
        const int rem = b1 - j - 1;
        for (int q = lane; q < rem * rem; q += 32) {
          const int c = j + 1 + q / rem, i = j + 1 + q % rem;
          if (i >= c) Dg[i * LDS + c] = cfms(Dg[i * LDS + j], cmul(Dg[c * LDS + j], dij), Dg[i * LDS + c]);
        }
        __syncwarp();
        for (int i = j + 1 + lane; i < b1; i += 32) Dg[i * LDS + j] = cmul(Dg[i * LDS + j], dij);
        __syncwarp();
      }
    }
    __syncthreads();
    // sub-panel TRSM: rows [b1, kb), columns [b0, b1)
    for (int i = b1 + tid; i < kb; i += blockDim.x) {
      cplx w[SB];
#pragma unroll
      for (int jj = 0; jj < SB; ++jj) {
        if (b0 + jj < b1) {
          cplx acc = Dg[i * LDS + b0 + jj];
#pragma unroll
          for (int tt = 0; tt < jj; ++tt) acc = cfms(w[tt], Dg[(b0 + jj) * LDS + b0 + tt], acc);
          w[jj] = acc;
        }
      }
#pragma unroll
      for (int jj = 0; jj < SB; ++jj)
        if (b0 + jj < b1) Dg[i * LDS + b0 + jj] = cmul(w[jj], di[b0 + jj]);
    }
    __syncthreads();
    // trailing update of [b1, kb)^2 (lower) with the sub-block's columns
    const int rem = kb - b1;
    for (int q = tid; q < rem * rem; q += blockDim.x) {
      const int c = b1 + q / rem, i = b1 + q % rem;
      if (i >= c) {
        cplx acc = Dg[i * LDS + c];
        for (int t = b0; t < b1; ++t) acc = cfms(cmul(Dg[i * LDS + t], dv[t]), Dg[c * LDS + t], acc);
        Dg[i * LDS + c] = acc;
      }
    }
    __syncthreads();
  }
  // X = L^{-1}: diagonal 16x16 blocks (one warp each, one column per lane)
  if (warp < nsub) {
    const int b0 = warp * SB, b1 = min(b0 + SB, kb);
    const int j = b0 + lane;
    if (j < b1) {
      for (int i = j + 1; i < b1; ++i) {
        cplx acc = Dg[i * LDS + j];
        for (int t = j + 1; t < i; ++t) acc = cfma(Dg[i * LDS + t], Dg[j * LDS + t], acc);
        Dg[j * LDS + i] = cmk(-acc.x, -acc.y);
      }
    }
  }
  __syncthreads();
  for (int bi = 1; bi < nsub; ++bi) {
    const int i0 = bi * SB, i1 = min(i0 + SB, kb), ni = i1 - i0;
    // T = L[bi, :i0] X[:i0, :i0]  (X[t][j] at Dg[j][t])
    for (int q = tid; q < ni * i0; q += blockDim.x) {
      const int i = i0 + q % ni, j = q / ni;
      cplx acc = Dg[i * LDS + j];
      for (int t = j + 1; t < i0; ++t) acc = cfma(Dg[i * LDS + t], Dg[j * LDS + t], acc);
      Ts[(i - i0) * LDS + j] = acc;
    }
    __syncthreads();
    // X[bi, :i0] = -X[bi, bi] T   (X[i][t] at Dg[t][i])
    for (int q = tid; q < ni * i0; q += blockDim.x) {
      const int i = i0 + q % ni, j = q / ni;
      cplx acc = Ts[(i - i0) * LDS + j];
      for (int t = i0; t < i; ++t) acc = cfma(Dg[t * LDS + i], Ts[(t - i0) * LDS + j], acc);
      Dg[j * LDS + i] = cmk(-acc.x, -acc.y);
    }
    __syncthreads();
  }
  // diagonal slot: s_j = sqrt(d_j) (factor format, see fronts.cuh)
  for (int idx = tid; idx < kb * kb; idx += blockDim.x) {
    int i = idx % kb, j = idx / kb;
    panel[(int64_t)(k0 + j) * nf + k0 + i] = i == j ? csqrt_c(Dg[i * LDS + j]) : Dg[i * LDS + j];
  }
}

template <int BK>
static void diag2_go(cudaStream_t st, const PanelTask* tasks, int ntasks, const FrontsDev& F,
                     const PoleBatch& pb, int* err) {
  if (ntasks <= 0) return;
  const size_t smem = ((BK + SB) * (BK + 1) + 2 * BK) * sizeof(cplx);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_diag2<BK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  dim3 grid(ntasks, pb.count);
  k_diag2<BK><<<grid, BK <= 48 ? 128 : 256, smem, st>>>(tasks, F, pb, err);
}

// the first nsmall tasks have blocks of at most 32 pivots, the next nmid of 33..48 (build_plans)
void launch_diag2(cudaStream_t st, const PanelTask* tasks, int ntasks, const FrontsDev& F,
                  const PoleBatch& pb, int* err, int nsmall, int nmid) {
  diag2_go<32>(st, tasks, nsmall, F, pb, err);
  diag2_go<48>(st, tasks + nsmall, nmid, F, pb, err);
  diag2_go<PB>(st, tasks + nsmall + nmid, ntasks - nsmall - nmid, F, pb, err);
}

// K4a': panel TRSM  L_r = F_r L_kk^{-T} D^{-1}  for one 64-row tile per CTA
// (rows below the diagonal block), reading the factored diagonal block.
__global__ void __launch_bounds__(256) k_trsm(const PanelTask* __restrict__ tasks, FrontsDev F,
                                              PoleBatch pb) {
  extern __shared__ cplx sm[];
  cplx* Dg = sm;               // [PB][LDS]
  cplx* X = sm + PB * LDS;     // [PB][LDS]
  const int slot = blockIdx.y;
  const PanelTask tk = tasks[blockIdx.x];
  const int s = tk.s, k0 = tk.k0, r0 = tk.r0;
  const int nf = F.nf[s], p = F.npiv[s];
  const int kb = min(PB, p - k0);
  cplx* panel = pb.factor[slot] + F.panel_off[s];
  const int tid = threadIdx.x;
  const int nr = min(PB, nf - r0);
  for (int idx = tid; idx < kb * kb; idx += blockDim.x) {
    int i = idx % kb, j = idx / kb;
    if (i >= j) Dg[i * LDS + j] = panel[(int64_t)(k0 + j) * nf + k0 + i];
  }
  for (int idx = tid; idx < nr * kb; idx += blockDim.x) {
    int i = idx % nr, j = idx / nr;
    X[i * LDS + j] = panel[(int64_t)(k0 + j) * nf + r0 + i];
  }
  __syncthreads();
  // W L_kk^T = X  (column sweep), then L = W D^{-1}
  for (int t = 0; t < kb; ++t) {
    const int rem = kb - t - 1;
    for (int q = tid; q < nr * rem; q += blockDim.x) {
      int i = q % nr, j = t + 1 + q / nr;
      X[i * LDS + j] = cfms(X[i * LDS + t], Dg[j * LDS + t], X[i * LDS + j]);
    }
    __syncthreads();
  }
  for (int idx = tid; idx < nr * kb; idx += blockDim.x) {
    int i = idx % nr, j = idx / nr;
    panel[(int64_t)(k0 + j) * nf + r0 + i] = cdiv(X[i * LDS + j], Dg[j * LDS + j]);
  }
}

void launch_diag(cudaStream_t st, const PanelTask* tasks, int ntasks, const FrontsDev& F,
                 const PoleBatch& pb, int* err) {
  if (ntasks <= 0) return;
  size_t smem = 2 * PB * LDS * sizeof(cplx);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  dim3 grid(ntasks, pb.count);
  k_diag<<<grid, 256, smem, st>>>(tasks, F, pb, err);
}

void launch_trsm(cudaStream_t st, const PanelTask* tasks, int ntasks, const FrontsDev& F,
                 const PoleBatch& pb) {
  if (ntasks <= 0) return;
  size_t smem = 2 * PB * LDS * sizeof(cplx);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_trsm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  dim3 grid(ntasks, pb.count);
  k_trsm<<<grid, 256, smem, st>>>(tasks, F, pb);
}

// ---------------------------------------------------------------------------
// K4b: trailing update  C[r,c] -= sum_t L'[r,t] L'[c,t]  (r >= c), one
// 64x64 complex tile per CTA, tiles listed per task (front, k-range, column
// range).  v1: DFMA register tiling (4x4 complex per thread).
// ---------------------------------------------------------------------------
constexpr int KC = 16;

__device__ __forceinline__ int find_task(const GemmTask* tasks, int n, int b) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (tasks[mid].tile_start <= b) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(256) k_gemm_update(const GemmTask* __restrict__ tasks, int ntasks,
                                                     FrontsDev F, PoleBatch pb) {
  __shared__ cplx As[KC][GT];
  __shared__ cplx Bs[KC][GT];
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
  cplx* panel = pb.factor[slot] + F.panel_off[s];
  cplx* upd = pb.upd[slot] + (F.upd_off[s] >= 0 ? F.upd_off[s] : 0);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  cplx acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = cmk(0.0, 0.0);
  for (int kt = tk.t0; kt < tk.t1; kt += KC) {
    const int kn = min(KC, tk.t1 - kt);
    __syncthreads();
    for (int idx = threadIdx.x; idx < KC * GT; idx += 256) {
      const int rr = idx % GT, kk = idx / GT;
      cplx a = cmk(0.0, 0.0), b = cmk(0.0, 0.0);
      if (kk < kn) {
        const cplx* col = panel + (int64_t)(kt + kk) * nf;
        if (r0 + rr < nf) a = col[r0 + rr];
        if (cc0 + rr < cmax) b = col[cc0 + rr];
      }
      As[kk][rr] = a;
      Bs[kk][rr] = b;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < KC; ++kk) {
      cplx av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = As[kk][tx + 16 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = Bs[kk][ty + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = cfma(av[a], bv[b], acc[a][b]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int r = r0 + tx + 16 * a, c = cc0 + ty + 16 * b;
      if (r < nf && c < cmax && r >= c) {
        cplx* dst = faddr(panel, upd, p, nf, r, c);
        *dst = csub(*dst, acc[a][b]);
      }
    }
}

void launch_gemm_update(cudaStream_t st, const GemmTask* tasks, int ntasks, int ntiles,
                        const FrontsDev& F, const PoleBatch& pb) {
  if (ntasks <= 0 || ntiles <= 0) return;
  dim3 grid(ntiles, pb.count);
  k_gemm_update<<<grid, 256, 0, st>>>(tasks, ntasks, F, pb);
}

}  // namespace rba
