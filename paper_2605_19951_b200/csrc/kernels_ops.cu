// Element, observation, reduction and vector kernels around the solves:
//  K8  J v right-hand sides   (dM_contract(g) @ v, mesh.py:358-370 / sensitivity.py:73)
//  K9  J^T w cell kernel      (dM[i].T @ z, sensitivity.py:92)
//  K10 Q apply + residue/time combination in ascending pole order
//      (forward.py:61-63, sensitivity.py:74-78,85-96)
//  K11 CSR SpMV for the regulariser square root R / R^T (inversion.py:144,147)
//  K12 LSQR vector kernels with deterministic two-stage reductions
// All reductions run in a fixed order, so results do not depend on the GPU
// count or on launch timing.
#include "fronts.cuh"
#include "kernels.h"

namespace rba {

static inline int grid_for(int64_t n, int per = 256, int cap = 148 * 16) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + per - 1) / per, cap));
}

// out[k][r] = sum_{(c,a) in dofcells(k)} e^{m_c} v_c (M_c g|_c)_a
template <int NR>
__global__ void k_jvp_rhs(ElemDev E, const double* __restrict__ v, SlotPtrs g, SlotPtrs out,
                          int S) {
  const int slot = blockIdx.y;
  const cplx* gs = g.p[slot];
  cplx* o = out.p[slot];
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < E.N;
       k += (int64_t)gridDim.x * blockDim.x) {
    cplx acc[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) acc[r] = cmk(0.0, 0.0);
    for (int64_t q = E.dc_ptr[k]; q < E.dc_ptr[k + 1]; ++q) {
      const int item = E.dc_item[q];
      const int c = item / 6, a = item - 6 * c;
      const int32_t* dofs = E.cell_dofs + (int64_t)c * 6;
      const double* Mrow = E.mass + (int64_t)c * 36 + a * 6;
      cplx loc[NR];
#pragma unroll
      for (int r = 0; r < NR; ++r) loc[r] = cmk(0.0, 0.0);
#pragma unroll
      for (int b = 0; b < 6; ++b) {
        const int d = __ldg(dofs + b);
        if (d < 0) continue;
        const double mab = __ldg(Mrow + b);
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          if (r < S) {
            const cplx gv = gs[(int64_t)d * NR + r];
            loc[r].x = fma(mab, gv.x, loc[r].x);
            loc[r].y = fma(mab, gv.y, loc[r].y);
          }
        }
      }
      const double sc = __ldg(E.expm + c) * __ldg(v + c);
      // rounded product, then add (no FMA contraction): bit-identical to the
      // two-pass k_jvp_cells + k_jvp_gather, so the choice between the two
      // (it depends on free memory, i.e. on the poles per GPU) never changes
      // J v -- results stay bitwise independent of the GPU count
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        acc[r].x = __dadd_rn(acc[r].x, __dmul_rn(loc[r].x, sc));
        acc[r].y = __dadd_rn(acc[r].y, __dmul_rn(loc[r].y, sc));
      }
    }
#pragma unroll
    for (int r = 0; r < NR; ++r) o[k * NR + r] = acc[r];
  }
}

// Two-pass variant (a workspace of nslots*P*6*NR complex is given):
// pass 1, one thread per cell: w[c][a][r] = e^{m_c} v_c (M_c g|_c)_a -- the
// cell's g rows are gathered once (the dof-parallel kernel gathers them once
// per cell dof, 6x); pass 2, one thread per dof: the item sum in dc order.
template <int NR>
__global__ void k_jvp_cells(ElemDev E, const double* __restrict__ v, SlotPtrs g, cplx* __restrict__ w,
                            int S) {
  const int slot = blockIdx.y;
  const cplx* gs = g.p[slot];
  cplx* ws = w + (int64_t)slot * E.P * 6 * NR;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < E.P;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int32_t* dofs = E.cell_dofs + c * 6;
    const double* M = E.mass + c * 36;
    int dd[6];
#pragma unroll
    for (int b = 0; b < 6; ++b) dd[b] = __ldg(dofs + b);
    const double sc = __ldg(E.expm + c) * __ldg(v + c);
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      cplx gl[6];
#pragma unroll
      for (int b = 0; b < 6; ++b)
        gl[b] = (dd[b] >= 0 && r < S) ? gs[(int64_t)dd[b] * NR + r] : cmk(0.0, 0.0);
#pragma unroll
      for (int a = 0; a < 6; ++a) {
        cplx loc = cmk(0.0, 0.0);
#pragma unroll
        for (int b = 0; b < 6; ++b) {
          const double mab = __ldg(M + a * 6 + b);
          loc.x = fma(mab, gl[b].x, loc.x);
          loc.y = fma(mab, gl[b].y, loc.y);
        }
        ws[(c * 6 + a) * NR + r] = cmk(__dmul_rn(loc.x, sc), __dmul_rn(loc.y, sc));
      }
    }
  }
}

template <int NR>
__global__ void k_jvp_gather(ElemDev E, const cplx* __restrict__ w, SlotPtrs out) {
  const int slot = blockIdx.y;
  const cplx* ws = w + (int64_t)slot * E.P * 6 * NR;
  cplx* o = out.p[slot];
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < E.N;
       k += (int64_t)gridDim.x * blockDim.x) {
    cplx acc[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) acc[r] = cmk(0.0, 0.0);
    for (int64_t q = E.dc_ptr[k]; q < E.dc_ptr[k + 1]; ++q) {
      const cplx* wi = ws + (int64_t)E.dc_item[q] * NR;
#pragma unroll
      for (int r = 0; r < NR; ++r)
        acc[r] = cmk(__dadd_rn(acc[r].x, wi[r].x), __dadd_rn(acc[r].y, wi[r].y));
    }
#pragma unroll
    for (int r = 0; r < NR; ++r) o[k * NR + r] = acc[r];
  }
}

template <int NR>
static void jvp2_nr(cudaStream_t st, int nslots, const ElemDev& E, const double* v,
                    const SlotPtrs& g, const SlotPtrs& out, int S, cplx* w) {
  k_jvp_cells<NR><<<dim3(grid_for(E.P), nslots), 256, 0, st>>>(E, v, g, w, S);
  k_jvp_gather<NR><<<dim3(grid_for(E.N), nslots), 256, 0, st>>>(E, w, out);
}

void launch_jvp_rhs2(cudaStream_t st, int nslots, const ElemDev& E, const double* v,
                     const SlotPtrs& g, const SlotPtrs& out, int NR, int S, cplx* w) {
  switch (NR) {
    case 1: jvp2_nr<1>(st, nslots, E, v, g, out, S, w); break;
    case 2: jvp2_nr<2>(st, nslots, E, v, g, out, S, w); break;
    case 4: jvp2_nr<4>(st, nslots, E, v, g, out, S, w); break;
    default: jvp2_nr<8>(st, nslots, E, v, g, out, S, w); break;
  }
}

void launch_jvp_rhs(cudaStream_t st, int nslots, const ElemDev& E, const double* v,
                    const SlotPtrs& g, const SlotPtrs& out, int NR, int S) {
  dim3 grid(grid_for(E.N), nslots);
  switch (NR) {
    case 1: k_jvp_rhs<1><<<grid, 256, 0, st>>>(E, v, g, out, S); break;
    case 2: k_jvp_rhs<2><<<grid, 256, 0, st>>>(E, v, g, out, S); break;
    case 4: k_jvp_rhs<4><<<grid, 256, 0, st>>>(E, v, g, out, S); break;
    default: k_jvp_rhs<8><<<grid, 256, 0, st>>>(E, v, g, out, S); break;
  }
}

// qpart[slot][s][r] = sum_e Q[r,e] h[col_e][s]
__global__ void k_q_apply(int64_t Mr, const int64_t* __restrict__ qptr,
                          const int32_t* __restrict__ qcol, const double* __restrict__ qval,
                          SlotPtrs h, int NR, int S, cplx* __restrict__ qpart) {
  const int slot = blockIdx.y;
  const cplx* hs = h.p[slot];
  const int64_t total = Mr * S;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t % Mr;
    const int s = (int)(t / Mr);
    cplx acc = cmk(0.0, 0.0);
    for (int64_t e = qptr[r]; e < qptr[r + 1]; ++e) {
      const cplx hv = hs[(int64_t)qcol[e] * NR + s];
      acc.x = fma(qval[e], hv.x, acc.x);
      acc.y = fma(qval[e], hv.y, acc.y);
    }
    qpart[((int64_t)slot * S + s) * Mr + r] = acc;
  }
}

void launch_q_apply(cudaStream_t st, int nslots, int64_t Mr, const int64_t* qptr,
                    const int32_t* qcol, const double* qval, const SlotPtrs& h, int NR, int S,
                    cplx* qpart) {
  if (Mr <= 0) return;
  dim3 grid(grid_for(Mr * S), nslots);
  k_q_apply<<<grid, 256, 0, st>>>(Mr, qptr, qcol, qval, h, NR, S, qpart);
}

// d[s][j][r] = sum_i 2 Re( (alpha_ij q_i,s,r) [* xi_i] ), i ascending
__global__ void k_combine_data(int m, int S, int Kt, int64_t Mr, const cplx* __restrict__ qall,
                               const int32_t* __restrict__ slot_of_pole,
                               const cplx* __restrict__ res, const cplx* __restrict__ poles,
                               bool times_pole, double* __restrict__ d) {
  const int64_t total = (int64_t)S * Kt * Mr;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t % Mr;
    const int j = (int)((t / Mr) % Kt);
    const int s = (int)(t / (Mr * Kt));
    double acc = 0.0;
    for (int i = 0; i < m; ++i) {
      const cplx q = qall[((int64_t)slot_of_pole[i] * S + s) * Mr + r];
      cplx z = cmul(res[(int64_t)i * Kt + j], q);
      if (times_pole) z = cmul(poles[i], z);
      acc += 2.0 * z.x;
    }
    d[t] = acc;
  }
}

void launch_combine_data(cudaStream_t st, int m, int S, int Kt, int64_t Mr, const cplx* qall,
                         const int32_t* slot_of_pole, const cplx* residues, const cplx* poles,
                         bool times_pole, double* d) {
  const int64_t total = (int64_t)S * Kt * Mr;
  if (total <= 0) return;
  k_combine_data<<<grid_for(total), 256, 0, st>>>(m, S, Kt, Mr, qall, slot_of_pole, residues,
                                                  poles, times_pole, d);
}

// wa[slot][s][r] = sum_j alpha_{i,j} w[s][j][r]
__global__ void k_walpha(int nslots, const int32_t* __restrict__ pole_of_slot, int S, int Kt,
                         int64_t Mr, const double* __restrict__ w, const cplx* __restrict__ res,
                         cplx* __restrict__ wa) {
  const int64_t total = (int64_t)nslots * S * Mr;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t % Mr;
    const int s = (int)((t / Mr) % S);
    const int slot = (int)(t / (Mr * S));
    const int i = pole_of_slot[slot];
    cplx acc = cmk(0.0, 0.0);
    for (int j = 0; j < Kt; ++j) {
      const double wv = w[((int64_t)s * Kt + j) * Mr + r];
      const cplx a = res[(int64_t)i * Kt + j];
      acc.x = fma(a.x, wv, acc.x);
      acc.y = fma(a.y, wv, acc.y);
    }
    wa[t] = acc;
  }
}

// out[slot][k][s] = sum_{e in QT row k} QT[k,e] wa[slot][s][col_e]   (all N rows)
__global__ void k_qt_apply(int64_t N, int S, int64_t Mr, const int64_t* __restrict__ qtptr,
                           const int32_t* __restrict__ qtcol, const double* __restrict__ qtval,
                           const cplx* __restrict__ wa, SlotPtrs out, int NR) {
  const int slot = blockIdx.y;
  cplx* o = out.p[slot];
  const cplx* was = wa + (int64_t)slot * S * Mr;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < N;
       k += (int64_t)gridDim.x * blockDim.x) {
    for (int s = 0; s < NR; ++s) {
      cplx acc = cmk(0.0, 0.0);
      if (s < S) {
        for (int64_t e = qtptr[k]; e < qtptr[k + 1]; ++e) {
          const cplx a = was[(int64_t)s * Mr + qtcol[e]];
          acc.x = fma(qtval[e], a.x, acc.x);
          acc.y = fma(qtval[e], a.y, acc.y);
        }
      }
      o[k * NR + s] = acc;
    }
  }
}

void launch_vjp_rhs(cudaStream_t st, int nslots, const int32_t* pole_of_slot, int S, int Kt,
                    int64_t Mr, int64_t N, const double* w, const cplx* residues,
                    const int64_t* qtptr, const int32_t* qtcol, const double* qtval, cplx* wa,
                    const SlotPtrs& out, int NR) {
  const int64_t total = (int64_t)nslots * S * Mr;
  if (total > 0)
    k_walpha<<<grid_for(total), 256, 0, st>>>(nslots, pole_of_slot, S, Kt, Mr, w, residues, wa);
  dim3 grid(grid_for(N), nslots);
  k_qt_apply<<<grid, 256, 0, st>>>(N, S, Mr, qtptr, qtcol, qtval, wa, out, NR);
}

// ---------------------------------------------------------------------------
// Receiver Green's functions Z_i = A_i^{-1} Q^T (N x Mr per pole, permuted
// rows, row-major [j][m]).  With A_i complex symmetric,
//   Q A_i^{-1} h    = Z_i^T h      (J v,  sensitivity.py:73-74)
//   A_i^{-T} Q^T z  = Z_i z        (J^T w, sensitivity.py:89-91)
// so once Z_i is built (Mr/NR multi-RHS solves per factorisation), every
// LSQR action streams Z_i (N*Mr*16 bytes) instead of two triangular sweeps
// over the factor (2*nnz(L)*16 bytes each way).
// ---------------------------------------------------------------------------

// x[slot][k][r] = Q^T[k, m0 + r]  (r < nb), 0 otherwise
__global__ void k_green_rhs(int64_t N, int64_t m0, int nb, int NR, const int64_t* __restrict__ qtptr,
                            const int32_t* __restrict__ qtcol, const double* __restrict__ qtval,
                            SlotPtrs x) {
  cplx* o = x.p[blockIdx.y];
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < N;
       k += (int64_t)gridDim.x * blockDim.x) {
    for (int r = 0; r < NR; ++r) {
      double a = 0.0;
      if (r < nb)
        for (int64_t e = qtptr[k]; e < qtptr[k + 1]; ++e)
          if (qtcol[e] == m0 + r) a += qtval[e];
      o[k * NR + r] = cmk(a, 0.0);
    }
  }
}

// Z[slot][k][m0 + r] = x[slot][k][r]
__global__ void k_green_store(int64_t N, int64_t Mr, int64_t m0, int nb, int NR, SlotPtrs x,
                              SlotPtrs Z) {
  const cplx* xs = x.p[blockIdx.y];
  cplx* z = Z.p[blockIdx.y];
  const int64_t total = N * nb;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = t / nb;
    const int r = (int)(t - k * nb);
    z[k * Mr + m0 + r] = xs[k * NR + r];
  }
}

// part[chunk][slot][s][m] = sum_{j in chunk} Z[slot][j][m] h[slot][j][s]
// Thread per m (coalesced Z rows); the chunk's h rows are staged in shared
// memory 128 at a time, 8 Z loads in flight per thread.
template <int NR>
__global__ void __launch_bounds__(128) k_green_jvp(int64_t N, int Mr, int S, int64_t rows_per_chunk,
                                                   SlotPtrs Z, SlotPtrs h, cplx* __restrict__ part) {
  constexpr int TR = 128;
  __shared__ cplx hs[TR][NR];
  const int slot = blockIdx.y, nslots = gridDim.y, chunk = blockIdx.x;
  const cplx* z = Z.p[slot];
  const cplx* hg = h.p[slot];
  const int64_t j0 = chunk * rows_per_chunk, j1 = min(N, j0 + rows_per_chunk);
  for (int mb = 0; mb < Mr; mb += blockDim.x) {
    const int m = mb + threadIdx.x;
    const bool on = m < Mr;
    cplx acc[NR];
#pragma unroll
    for (int s = 0; s < NR; ++s) acc[s] = cmk(0.0, 0.0);
    for (int64_t t0 = j0; t0 < j1; t0 += TR) {
      const int nt = (int)min((int64_t)TR, j1 - t0);
      __syncthreads();
      for (int e = threadIdx.x; e < nt * NR; e += blockDim.x)
        hs[e / NR][e % NR] = __ldg(hg + t0 * NR + e);
      __syncthreads();
      if (on) {
        const cplx* zp = z + t0 * Mr + m;
        int jj = 0;
        for (; jj + 8 <= nt; jj += 8) {
          cplx zv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) zv[u] = __ldg(zp + (int64_t)(jj + u) * Mr);
#pragma unroll
          for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int s = 0; s < NR; ++s)
              if (s < S) acc[s] = cfma(zv[u], hs[jj + u][s], acc[s]);
        }
        for (; jj < nt; ++jj) {
          const cplx zv = __ldg(zp + (int64_t)jj * Mr);
#pragma unroll
          for (int s = 0; s < NR; ++s)
            if (s < S) acc[s] = cfma(zv, hs[jj][s], acc[s]);
        }
      }
    }
    if (on)
      for (int s = 0; s < S; ++s)
        part[(((int64_t)chunk * nslots + slot) * S + s) * Mr + m] = acc[s];
  }
}

// qpart[slot][s][m] = sum_chunk part[chunk][slot][s][m], chunks ascending
__global__ void k_green_reduce(int nchunk, int64_t per_chunk, const cplx* __restrict__ part,
                               cplx* __restrict__ qpart) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < per_chunk;
       t += (int64_t)gridDim.x * blockDim.x) {
    cplx a = cmk(0.0, 0.0);
    for (int c = 0; c < nchunk; ++c) a = cadd(a, part[c * per_chunk + t]);
    qpart[t] = a;
  }
}

// x[slot][j][s] = sum_m Z[slot][j][m] wa[slot][s][m]
// A warp takes 8 rows at a time: lane = (row jr, m-group mg of 4), so each
// load instruction reads 8 row segments of 4 consecutive m (64 B each); the
// four m-groups are reduced with two shuffle levels.
template <int NR>
__global__ void __launch_bounds__(256) k_green_vjp(int64_t N, int Mr, int S, SlotPtrs Z,
                                                   const cplx* __restrict__ wa, SlotPtrs x) {
  extern __shared__ cplx wsm[];   // [S][Mr]
  const int slot = blockIdx.y;
  const cplx* z = Z.p[slot];
  cplx* xs = x.p[slot];
  for (int e = threadIdx.x; e < S * Mr; e += blockDim.x) wsm[e] = wa[(int64_t)slot * S * Mr + e];
  __syncthreads();
  const int lane = threadIdx.x & 31, jr = lane >> 2, mg = lane & 3;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t j0 = (blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5)) * 8; j0 < N;
       j0 += nw * 8) {
    const int64_t j = j0 + jr;
    cplx acc[NR];
#pragma unroll
    for (int s = 0; s < NR; ++s) acc[s] = cmk(0.0, 0.0);
    if (j < N) {
      const cplx* zp = z + j * Mr;
#pragma unroll 5
      for (int m = mg; m < Mr; m += 4) {
        const cplx zv = __ldg(zp + m);
#pragma unroll
        for (int s = 0; s < NR; ++s)
          if (s < S) acc[s] = cfma(zv, wsm[s * Mr + m], acc[s]);
      }
    }
#pragma unroll
    for (int s = 0; s < NR; ++s) {
      double a = acc[s].x, b = acc[s].y;
      a += __shfl_xor_sync(0xffffffffu, a, 1);
      b += __shfl_xor_sync(0xffffffffu, b, 1);
      a += __shfl_xor_sync(0xffffffffu, a, 2);
      b += __shfl_xor_sync(0xffffffffu, b, 2);
      acc[s] = cmk(a, b);
    }
    if (j < N) {
#pragma unroll
      for (int s = mg; s < NR; s += 4) {
        cplx v = cmk(0.0, 0.0);
#pragma unroll
        for (int q = 0; q < NR; ++q)
          if (q == s && q < S) v = acc[q];
        xs[j * NR + s] = v;
      }
    }
  }
}

void launch_green_rhs(cudaStream_t st, int nslots, int64_t N, int64_t m0, int nb, int NR,
                      const int64_t* qtptr, const int32_t* qtcol, const double* qtval,
                      const SlotPtrs& x) {
  dim3 grid(grid_for(N), nslots);
  k_green_rhs<<<grid, 256, 0, st>>>(N, m0, nb, NR, qtptr, qtcol, qtval, x);
}
void launch_green_store(cudaStream_t st, int nslots, int64_t N, int64_t Mr, int64_t m0, int nb,
                        int NR, const SlotPtrs& x, const SlotPtrs& Z) {
  dim3 grid(grid_for(N * nb), nslots);
  k_green_store<<<grid, 256, 0, st>>>(N, Mr, m0, nb, NR, x, Z);
}
void launch_green_jvp(cudaStream_t st, int nslots, int64_t N, int Mr, int S, int NR, int nchunk,
                      const SlotPtrs& Z, const SlotPtrs& h, cplx* part, cplx* qpart) {
  const int64_t rpc = (N + nchunk - 1) / nchunk;
  dim3 grid(nchunk, nslots);
  switch (NR) {
    case 1: k_green_jvp<1><<<grid, 128, 0, st>>>(N, Mr, S, rpc, Z, h, part); break;
    case 2: k_green_jvp<2><<<grid, 128, 0, st>>>(N, Mr, S, rpc, Z, h, part); break;
    case 4: k_green_jvp<4><<<grid, 128, 0, st>>>(N, Mr, S, rpc, Z, h, part); break;
    default: k_green_jvp<8><<<grid, 128, 0, st>>>(N, Mr, S, rpc, Z, h, part); break;
  }
  const int64_t per = (int64_t)nslots * S * Mr;
  k_green_reduce<<<grid_for(per), 256, 0, st>>>(nchunk, per, part, qpart);
}
void launch_walpha(cudaStream_t st, int nslots, const int32_t* pole_of_slot, int S, int Kt,
                   int64_t Mr, const double* w, const cplx* residues, cplx* wa) {
  const int64_t total = (int64_t)nslots * S * Mr;
  if (total > 0)
    k_walpha<<<grid_for(total), 256, 0, st>>>(nslots, pole_of_slot, S, Kt, Mr, w, residues, wa);
}
void launch_green_vjp(cudaStream_t st, int nslots, int64_t N, int Mr, int S, int NR,
                      const SlotPtrs& Z, const cplx* wa, const SlotPtrs& x) {
  dim3 grid(148 * 4, nslots);
  const size_t smem = (size_t)S * Mr * sizeof(cplx);
  if (smem > 48 * 1024) {
    cudaFuncSetAttribute(k_green_vjp<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_green_vjp<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_green_vjp<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_green_vjp<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  switch (NR) {
    case 1: k_green_vjp<1><<<grid, 256, smem, st>>>(N, Mr, S, Z, wa, x); break;
    case 2: k_green_vjp<2><<<grid, 256, smem, st>>>(N, Mr, S, Z, wa, x); break;
    case 4: k_green_vjp<4><<<grid, 256, smem, st>>>(N, Mr, S, Z, wa, x); break;
    default: k_green_vjp<8><<<grid, 256, smem, st>>>(N, Mr, S, Z, wa, x); break;
  }
}

// tpart[slot][c] = sum_s 2 Re( xi_i * e^{m_c} sum_a z_a (M_c g)_a )
template <int NR>
__global__ void k_vjp_cells(const int32_t* __restrict__ pole_of_slot,
                            const cplx* __restrict__ poles, ElemDev E, SlotPtrs z, SlotPtrs g,
                            int S, double* __restrict__ tpart) {
  const int slot = blockIdx.y;
  const cplx xi = poles[pole_of_slot[slot]];
  const cplx* zs = z.p[slot];
  const cplx* gs = g.p[slot];
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < E.P;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int32_t* dofs = E.cell_dofs + c * 6;
    const double* M = E.mass + c * 36;
    int dd[6];
#pragma unroll
    for (int a = 0; a < 6; ++a) dd[a] = __ldg(dofs + a);
    const double em = __ldg(E.expm + c);
    double tot = 0.0;
#pragma unroll
    for (int s = 0; s < NR; ++s) {
      if (s >= S) break;
      cplx gl[6], zl[6];
#pragma unroll
      for (int a = 0; a < 6; ++a) {
        gl[a] = dd[a] >= 0 ? gs[(int64_t)dd[a] * NR + s] : cmk(0.0, 0.0);
        zl[a] = dd[a] >= 0 ? zs[(int64_t)dd[a] * NR + s] : cmk(0.0, 0.0);
      }
      cplx part = cmk(0.0, 0.0);
#pragma unroll
      for (int a = 0; a < 6; ++a) {
        cplx mg = cmk(0.0, 0.0);
#pragma unroll
        for (int b = 0; b < 6; ++b) {
          const double mab = __ldg(M + a * 6 + b);
          mg.x = fma(mab, gl[b].x, mg.x);
          mg.y = fma(mab, gl[b].y, mg.y);
        }
        mg.x *= em;
        mg.y *= em;
        part = cfma(mg, zl[a], part);
      }
      tot += 2.0 * cmul(xi, part).x;
    }
    tpart[(int64_t)slot * E.P + c] = tot;
  }
}

void launch_vjp_cells(cudaStream_t st, int nslots, const int32_t* pole_of_slot,
                      const cplx* poles, const ElemDev& E, const SlotPtrs& z,
                      const SlotPtrs& g, int NR, int S, double* tpart) {
  dim3 grid(grid_for(E.P), nslots);
  switch (NR) {
    case 1: k_vjp_cells<1><<<grid, 256, 0, st>>>(pole_of_slot, poles, E, z, g, S, tpart); break;
    case 2: k_vjp_cells<2><<<grid, 256, 0, st>>>(pole_of_slot, poles, E, z, g, S, tpart); break;
    case 4: k_vjp_cells<4><<<grid, 256, 0, st>>>(pole_of_slot, poles, E, z, g, S, tpart); break;
    default: k_vjp_cells<8><<<grid, 256, 0, st>>>(pole_of_slot, poles, E, z, g, S, tpart); break;
  }
}

__global__ void k_combine_cells(int m, int64_t P, const double* __restrict__ tall,
                                const int32_t* __restrict__ slot_of_pole, double* __restrict__ out) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < P;
       c += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int i = 0; i < m; ++i) acc += tall[(int64_t)slot_of_pole[i] * P + c];
    out[c] = acc;
  }
}

void launch_combine_cells(cudaStream_t st, int m, int64_t P, const double* tall,
                          const int32_t* slot_of_pole, double* out) {
  k_combine_cells<<<grid_for(P), 256, 0, st>>>(m, P, tall, slot_of_pole, out);
}

__global__ void k_spmv(int64_t nrows, const int64_t* __restrict__ ptr,
                       const int32_t* __restrict__ idx, const double* __restrict__ val,
                       const double* __restrict__ x, double alpha, double* __restrict__ y,
                       bool accumulate) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows;
       r += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int64_t e = ptr[r]; e < ptr[r + 1]; ++e) acc = fma(val[e], __ldg(x + idx[e]), acc);
    y[r] = accumulate ? fma(alpha, acc, y[r]) : alpha * acc;
  }
}

void launch_spmv(cudaStream_t st, int64_t nrows, const int64_t* ptr, const int32_t* idx,
                 const double* val, const double* x, double alpha, double* y, bool accumulate) {
  if (nrows <= 0) return;
  k_spmv<<<grid_for(nrows), 256, 0, st>>>(nrows, ptr, idx, val, x, alpha, y, accumulate);
}

// ---------------------------------------------------------------------------
// vector kernels
// ---------------------------------------------------------------------------
constexpr int RED_BLOCKS = 296;

__global__ void k_axpby(int64_t n, double a, const double* __restrict__ x, double b,
                        const double* __restrict__ y, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a * x[i] + (b == 0.0 ? 0.0 : b * y[i]);
}
void launch_axpby(cudaStream_t st, int64_t n, double a, const double* x, double b,
                  const double* y, double* out) {
  if (n <= 0) return;
  k_axpby<<<grid_for(n), 256, 0, st>>>(n, a, x, b, y, out);
}

__global__ void k_mul(int64_t n, const double* __restrict__ a, const double* __restrict__ x,
                      double alpha, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = alpha * (a[i] * x[i]);
}
void launch_mul(cudaStream_t st, int64_t n, const double* a, const double* x, double alpha,
                double* out) {
  if (n <= 0) return;
  k_mul<<<grid_for(n), 256, 0, st>>>(n, a, x, alpha, out);
}

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double sh[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += sh[k];
  return t;
}

__global__ void k_dot_part(int64_t n, const double* __restrict__ x, const double* __restrict__ y,
                           double* __restrict__ part) {
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    acc = fma(x[i], y[i], acc);
  acc = block_sum(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}
__global__ void k_sum_part(int nb, const double* __restrict__ part, double* __restrict__ result) {
  double acc = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) acc += part[i];
  acc = block_sum(acc);
  if (threadIdx.x == 0) *result = acc;
}
void launch_dot(cudaStream_t st, int64_t n, const double* x, const double* y, double* part,
                double* result) {
  k_dot_part<<<RED_BLOCKS, 256, 0, st>>>(n, x, y, part);
  k_sum_part<<<1, 256, 0, st>>>(RED_BLOCKS, part, result);
}

// ddn += |w|^2 (old w); x += t1 w; w = v + t2 w
__global__ void k_lsqr_xw(int64_t n, double t1, double t2, const double* __restrict__ v,
                          double* __restrict__ w, double* __restrict__ x,
                          double* __restrict__ part) {
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double wi = w[i];
    acc = fma(wi, wi, acc);
    x[i] = x[i] + t1 * wi;
    w[i] = v[i] + t2 * wi;
  }
  acc = block_sum(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}
void launch_lsqr_xw(cudaStream_t st, int64_t n, double t1, double t2, const double* v,
                    double* w, double* x, double* part, double* result) {
  k_lsqr_xw<<<RED_BLOCKS, 256, 0, st>>>(n, t1, t2, v, w, x, part);
  k_sum_part<<<1, 256, 0, st>>>(RED_BLOCKS, part, result);
}

__global__ void k_zero_c(int64_t n, cplx* p) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = cmk(0.0, 0.0);
}
void launch_zero_c(cudaStream_t st, int64_t n, cplx* p) {
  if (n <= 0) return;
  k_zero_c<<<grid_for(n), 256, 0, st>>>(n, p);
}

__global__ void k_scatter_vals(int64_t nnz, const int64_t* __restrict__ tgt,
                               const cplx* __restrict__ vals, cplx* __restrict__ fac) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x)
    fac[tgt[e]] = vals[e];
}
void launch_scatter_vals(cudaStream_t st, int64_t nnz, const int64_t* tgt, const cplx* vals,
                         cplx* factor) {
  k_scatter_vals<<<grid_for(nnz), 256, 0, st>>>(nnz, tgt, vals, factor);
}

// dst = conj(src)  (trans 'H' solves: A^{-H} b = conj(A^{-1} conj(b)))
__global__ void k_conj(int64_t n, const cplx* __restrict__ src, cplx* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const cplx v = src[i];
    dst[i] = cmk(v.x, -v.y);
  }
}
void launch_conj(cudaStream_t st, int64_t n, const cplx* src, cplx* dst) {
  if (n <= 0) return;
  k_conj<<<grid_for(n), 256, 0, st>>>(n, src, dst);
}

// Factor statistics of one pole (stability report of the pivot-free LDL^T):
// out[0] = max |L'| over the stored factor (L' = L D^{1/2}; inside a diagonal
// block |L'(r,c)| = |L_bb(r,c)| |s_c|), out[1] = min |s_c|, out[2] = max |s_c|
// (s_c = sqrt(d_c), so |d_c| = |s_c|^2), out[3] = non-finite entries.
// Non-negative doubles order like their bit patterns, so max/min are 64-bit
// integer atomics.
__global__ void k_factor_stats(FrontsDev F, int nfront, const cplx* __restrict__ fac,
                               double* __restrict__ out) {
  double mx = 0.0, mn = __longlong_as_double(0x7ff0000000000000LL), ms = 0.0, bad = 0.0;
  const int nsplit = gridDim.y;
  for (int s = blockIdx.x; s < nfront; s += gridDim.x) {
    const int p = F.npiv[s], nf = F.nf[s];
    const cplx* pan = fac + F.panel_off[s];
    for (int c = blockIdx.y; c < p; c += nsplit) {
      const cplx* col = pan + (int64_t)c * nf;
      const cplx sc = col[c];
      const double as = hypot(sc.x, sc.y);
      const int bend = min(p, (c / PB + 1) * PB);
      for (int r = c + threadIdx.x; r < nf; r += blockDim.x) {
        const cplx v = col[r];
        double a;
        if (r == c) {
          a = as;
          mn = fmin(mn, as);
          ms = fmax(ms, as);
        } else {
          a = hypot(v.x, v.y);
          if (r < bend) a *= as;
        }
        if (!isfinite(a)) bad += 1.0;
        else mx = fmax(mx, a);
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    ms = fmax(ms, __shfl_xor_sync(0xffffffffu, ms, o));
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax((unsigned long long*)out, (unsigned long long)__double_as_longlong(mx));
    atomicMin((unsigned long long*)(out + 1), (unsigned long long)__double_as_longlong(mn));
    atomicMax((unsigned long long*)(out + 2), (unsigned long long)__double_as_longlong(ms));
    if (bad > 0) atomicAdd(out + 3, bad);
  }
}
void launch_factor_stats(cudaStream_t st, const FrontsDev& F, int nfront, const cplx* fac,
                         double* out) {
  k_factor_stats<<<dim3(std::min(nfront, 148 * 8), 16), 256, 0, st>>>(F, nfront, fac, out);
}

}  // namespace rba
