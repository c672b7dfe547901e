// Device view of the symbolic structure (see symbolic.h) plus the task
// descriptors of the level-scheduled factorisation and solves.
#pragma once
#include "common.cuh"

namespace rba {

struct FrontsDev {
  const int32_t* first;
  const int32_t* npiv;
  const int32_t* nf;
  const int64_t* panel_off;
  const int64_t* upd_off;
  const int64_t* rows_off;
  const int32_t* rows;
  const int32_t* child_ptr;
  const int32_t* child_list;
  const int64_t* rel_off;
  const int32_t* relmap;
  const int64_t* uvec_off;
  const int64_t* ucon_ptr;   // per front-row (rows_off indexing) -> uvec contributions
  const int64_t* ucon_idx;
  const int64_t* blk_off;    // per front: offset of its pivot-block flags
};

// TMA tensor map (CUtensorMap, 128 B) as stored in device memory.
struct alignas(64) TMap { unsigned char b[128]; };
// per front: [0] A operand (66-row x G8K-column box of the panel),
//            [1] B operand (34-row x G8K-column box)
constexpr int G8K = 8;

// Batch of poles processed by one launch (gridDim.y or ticket modulo).
struct PoleBatch {
  const TMap* tmap[32]; // per slot: tensor maps of the slot's factor panels (or null)
  cplx* factor[32];     // per slot: factor storage base
  cplx* upd[32];        // per slot: update arena base
  cplx xi[32];          // per slot: pole value
  int32_t count;
};

// Factor format (per front panel, column-major nf x npiv): A_front = L' L'^T
// with L' = L D^{1/2} (complex-symmetric LDL^T with the pivot square roots
// folded into the columns, so no GEMM carries a d scaling):
//   * rows below a column's 64-pivot diagonal block: L'[r,c] = L[r,c] s_c
//   * diagonal slot: s_c = sqrt(d_c) (principal root)
//   * strictly lower part of each 64x64 diagonal block: unit L_bb
//   * strictly upper part of each diagonal block: X = L_bb^{-1}, transposed
//     (X[i][j], i > j, stored at (row j, col i))
// Block forms: y_b = S_b^{-1} X_b (v_b - sum L'_bj y_j);
//              x_b = X_b^T S_b^{-1} (y_b - sum L'_rb^T x_r).
constexpr int PB = 64;   // pivot block (factorisation) and solve row block
constexpr int GT = 64;   // GEMM tile (complex)

// Packed lower-triangular update block of order n: column j holds rows j..n-1.
__host__ __device__ __forceinline__ int64_t ucol(int64_t j, int64_t n) {
  return j * n - j * (j - 1) / 2;
}
// element address in front s (r >= c): columns < p live in the factor panel
// (ld = nf), columns >= p in the packed lower-triangular update block.
__device__ __forceinline__ cplx* faddr(cplx* panel, cplx* upd, int p, int nf, int r, int c) {
  return c < p ? panel + (int64_t)c * nf + r : upd + ucol(c - p, nf - p) + (r - c);
}

struct PanelTask { int32_t s, k0, r0, pad; };
struct GemmTask { int32_t s, t0, t1, c_lo, c_hi, tile_start, ntr, pad; };
struct SolveTask { int32_t s, blk; };
// One INT8-tensor-core (Ozaki scheme) update of front s (kernels_ozaki.cu):
//   C[r, c] -= sum_{t0 <= k < t1} L'[r, k] L'[c, k],  c_lo <= c < c_hi, c <= r < nf
// (front coordinates; columns >= npiv live in the update block).  The Schur
// update is c_lo = npiv, c_hi = nf, [t0, t1) = [0, npiv); an aggregated panel
// update is c_lo = panel end, c_hi = npiv, [t0, t1) = the panel.  nrt row
// tiles of 64 rows from c_lo, nks k steps of 16; digit blocks at split_off
// (bytes, per pole), row exponents at exp_off (rows, per pole).
struct OzTask {
  int32_t s, nf, c_lo, c_hi, t0, t1, nrt, nks, tile_start, rt_start;
  int64_t split_off, exp_off;
};

}  // namespace rba
