/* rba_b200.h -- C ABI of the B200-native shifted-solve Gauss-Newton path.
 *
 * The reference (arXiv 2605.19951 analog, /root/reference/pkg/src/rbainv) has
 * no FFI: its seams are duck-typed Python objects.  Each entry
 * point below replaces the reference operation named in its comment; the
 * Python host layer (paper_2605_19951_b200/) binds them with ctypes and keeps
 * the reference's names, argument meaning and exceptions.
 *
 * Conventions
 *  - plain pointers and sizes only; complex numbers are interleaved doubles
 *    (re, im), matching numpy complex128;
 *  - "_h" arguments are HOST pointers, borrowed for the duration of the call;
 *    "_d" arguments are DEVICE pointers (e.g. from torch tensors);
 *  - every function returns a status code; rba_last_error() gives the message
 *    (thread-local).  Codes map to the reference's exceptions:
 *      RBA_ERR_INVALID    -> ValueError
 *      RBA_ERR_SOLVE      -> SolveError        (shifted.py:40-41,55-56)
 *      RBA_ERR_CACHE_MISS -> CacheMissError    (shifted.py:36-37,111-112)
 *      RBA_ERR_STATE      -> RuntimeError      (sensitivity.py:61-63)
 *      RBA_ERR_CUDA / RBA_ERR_OOM -> RuntimeError / MemoryError
 *  - a context owns all device buffers (factors, fields, work vectors) and
 *    one CUDA stream; calls on one context must not overlap.
 */
#ifndef RBA_B200_H
#define RBA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  RBA_OK = 0,
  RBA_ERR_INVALID = 1,
  RBA_ERR_CUDA = 2,
  RBA_ERR_SOLVE = 3,
  RBA_ERR_CACHE_MISS = 4,
  RBA_ERR_STATE = 5,
  RBA_ERR_OOM = 6
};

typedef struct rba_ctx rba_ctx;
typedef struct rba_symbolic rba_symbolic;
typedef struct rba_box rba_box;

const char* rba_last_error(void);
int rba_version(void);

/* ---- host symbolic analysis (no GPU needed) ------------------------------
 * Replaces the ordering + symbolic phase inside spla.splu (shifted.py:54):
 * nested dissection (geometric when coords != NULL) and the supernodal
 * assembly tree.  pattern: symmetric CSR, both triangles. */
int rba_symbolic_analyze(int64_t n, const int64_t* indptr_h, const int32_t* indices_h,
                         const double* coords_h, int32_t leaf, rba_symbolic** out);
/* istats[16]: n, nfront, nlevels, nnzL, panel_total, upd_total, uvec_total,
 *             max_nf, max_npiv, nblocks;  dstats[4]: flops (SURVEY §8d formula) */
int rba_symbolic_stats(const rba_symbolic* s, int64_t* istats_h, double* dstats_h);
/* copy an array by name ("perm","first","npiv","nf","parent","level","rows_off",
 * "rows","rel_off","relmap","panel_off","upd_off") into out_h; *nbytes = size */
int rba_symbolic_array(const rba_symbolic* s, const char* name, void* out_h,
                       int64_t capacity_bytes, int64_t* nbytes);
void rba_symbolic_destroy(rba_symbolic* s);
/* Host-only dry run of rba_set_mesh's preparation (pattern, symbolic,
 * scatter plan) for validation without a GPU.  out[4]: nnz(lower A),
 * M contributions, fronts, panel entries. */
int rba_mesh_prepare(int64_t N, int64_t P, int32_t k, const int32_t* cell_dofs_h,
                     const double* mass_local_h, const int64_t* K_indptr_h,
                     const int32_t* K_indices_h, const double* K_data_h, const double* coords_h,
                     int32_t leaf, int64_t* out_h);

/* ---- 3-D operator generation on the GPU (mesh_gen.cu) ----------------------
 * The lowest-order Nedelec problem on a Kuhn-split n^3 hex box with PEC
 * boundary, the 3-D counterpart of the reference's build_problem
 * (/root/reference/pkg/src/rbainv/mesh.py:294-345): edge dofs in (low, high)
 * vertex order, per-tet dofs and vertices, the curl-curl K (CSR, duplicates
 * summed in element order; stiff6 = the 6 Kuhn-tet local matrices, 6x36),
 * edge midpoints, interior-face adjacency and measures (RT0 regulariser).
 * info[6]: N, P, nnz(K), faces, edges, vertices.  Arrays by name: "cell_dofs"
 * (i32 P*6), "cells" (i64 P*4), "indptr" (i64 N+1), "indices" (i32), "data"
 * (f64), "face_cells" (i32 F*2), "face_measure" (f64 F), "dof_of_edge" (i64 E),
 * "dof_coords" (f64 N*3), "dof_offset" (i64 vertices+1: first dof of the edges
 * leaving each vertex). */
int rba_box_generate(int32_t n, double h, const double* stiff6_h, rba_box** out);
int rba_box_info(const rba_box* box, int64_t* info_h);
int rba_box_get(const rba_box* box, const char* name, void* out_h, int64_t capacity_bytes);
void rba_box_destroy(rba_box* box);
const char* rba_box_last_error(void);
/* Largest generalised eigenvalue over the element pencils (K_c, e^{m_c} M_c),
 * P cells of 6x6 matrices (mesh.py:406-421 spectral_bound): one Cholesky +
 * power iteration per cell on the device, max over cells. */
int rba_spectral_bound(int64_t P, const double* mass_local_h, const double* stiff_local_h,
                       const double* m_h, double* out_h);

/* ---- context ------------------------------------------------------------ */
int rba_ctx_create(int device, void* cuda_stream, rba_ctx** out);
void rba_ctx_destroy(rba_ctx* ctx);

/* Static operators of one mesh: Problem.K (CSR), cell_dofs (P,k),
 * mass_local (P,k,k) (mesh.py:127-162).  Builds the A pattern, runs the
 * symbolic analysis and uploads everything.  k must be 6 (edge elements) or
 * any k <= 6 for the reference's 1-D/2-D problems. */
int rba_set_mesh(rba_ctx* ctx, int64_t N, int64_t P, int32_t k, const int32_t* cell_dofs_h,
                 const double* mass_local_h, const int64_t* K_indptr_h,
                 const int32_t* K_indices_h, const double* K_data_h, const double* coords_h,
                 int32_t leaf);
/* Observation operator Q (M_r x N CSR) and the S source vectors (S x N). */
int rba_set_observation(rba_ctx* ctx, int64_t Mr, const int64_t* Q_indptr_h,
                        const int32_t* Q_indices_h, const double* Q_data_h);
int rba_set_sources(rba_ctx* ctx, int32_t S, const double* F_h);
/* Complex right-hand sides (S x N complex) -- e.g. the C2 random-RHS solves. */
int rba_set_sources_complex(rba_ctx* ctx, int32_t S, const double* F_h);
/* Poles xi_i (m complex) and residues alpha (m x K_t complex, row-major);
 * local_poles: the global pole indices this context factorises (sharding
 * i mod G, shifted.py:147-149). */
int rba_set_poles(rba_ctx* ctx, int32_t m, const double* poles_h, int32_t Kt,
                  const double* residues_h, int32_t n_local, const int32_t* local_poles_h);
/* Model m (P log-conductivities): M(m) assembly on the device
 * (assemble_M, mesh.py:348-355); invalidates factors (cache.activate). */
int rba_set_model(rba_ctx* ctx, const double* m_h);
int rba_set_model_d(rba_ctx* ctx, const double* m_d);
/* Factorise every local pole at the current model (factorize_all_poles,
 * shifted.py:158-173).  RBA_ERR_SOLVE on a zero / non-finite pivot. */
int rba_factor(rba_ctx* ctx);
/* Factorise local slot `slot` from explicit values of A in the lower pattern
 * returned by rba_pattern (ShiftedFactorCache.factorize(i, A), shifted.py:98-105). */
int rba_factor_values(rba_ctx* ctx, int32_t slot, const double* values_h);
/* Lower-triangle pattern of A (original numbering, row >= col): nnz, then
 * rows/cols (int32) and the assembled K / M values in that order. */
int rba_pattern(rba_ctx* ctx, int64_t* nnz, int32_t* rows_h, int32_t* cols_h, double* K_h,
                double* M_h);
/* x = A_i^{-1} rhs, trans 0 'N' / 1 'T' (identical: A_i is complex symmetric)
 * or 2 'H' (conj(A_i^{-1} conj(rhs))); other values -> RBA_ERR_INVALID
 * (_Factor.solve(rhs, trans), shifted.py:58-61; cache.solve :107-116).
 * rhs/out: column-major N x nrhs complex. */
int rba_solve(rba_ctx* ctx, int32_t slot, const double* rhs_h, double* out_h, int32_t nrhs,
              int32_t trans);
int rba_solve_d(rba_ctx* ctx, int32_t slot, const double* rhs_d, double* out_d, int32_t nrhs,
                int32_t trans);
/* Forward pass (solve_all_poles with the sources + Q): stores g_i per local
 * pole and writes q_part_d[slot][S][M_r] (complex) = Q g_i. */
int rba_forward_partial(rba_ctx* ctx, double* qpart_d);
/* J v partials (sensitivity.py:65-79): q_part_d[slot][S][M_r] = Q A_i^{-1}(dM(g_i) v).
 * Receiver-Green mode (env RBA_GREEN, default on when memory allows): the
 * first J v / J^T w after a factorisation builds Z_i = A_i^{-1} Q^T with
 * M_r / NR multi-RHS solves; then Q A_i^{-1} h = Z_i^T h and
 * A_i^{-T} Q^T z = Z_i z (A_i complex symmetric) stream Z_i instead of the
 * two triangular sweeps.  Same mathematics, rounding-level differences. */
int rba_jvp_partial(rba_ctx* ctx, const double* v_d, double* qpart_d);
/* J^T w partials (sensitivity.py:81-97): t_part_d[slot][P] = 2 Re xi_i dM_i^T A_i^{-T} Q^T(sum_j alpha_ij w_j). */
int rba_vjp_partial(rba_ctx* ctx, const double* w_d, double* tpart_d);
/* g_i of local slot `slot` after rba_forward_partial: column-major N x S
 * complex, original dof order (ForwardResult fields / pole_solutions). */
int rba_get_g(rba_ctx* ctx, int32_t slot, double* out_h);
/* Same into a device buffer (N x S complex, column-major): the per-rank
 * pole solutions all-gathered by solve_all_poles at G > 1 (shifted.py:176-199). */
int rba_get_g_d(rba_ctx* ctx, int32_t slot, double* out_d);
/* Replace g_i of a local slot by caller-supplied pole solutions (host,
 * N x S complex column-major, original order): JacobianOperator built from
 * given pole_solutions (sensitivity.py:43-59) contracts dM with those. */
int rba_set_g(rba_ctx* ctx, int32_t slot, const double* g_h);
/* Stability report of a local slot's pivot-free LDL^T (no SciPy analogue;
 * SuperLU pivots, shifted.py:54): out[4] = max |L'| (L' = L D^{1/2}),
 * min |sqrt(d)|, max |sqrt(d)|, number of non-finite factor entries.
 * Growth = max|L'|^2 / max|A|, smallest pivot = min|sqrt(d)|^2 / max|A|. */
int rba_factor_stats(rba_ctx* ctx, int32_t slot, double* out_h);
/* Copy the factor storage of a local slot (panel_total complex entries;
 * per-front nf x npiv column-major panels at symbolic panel_off) -- used by
 * the structure-level parity tests against the host emulation.  Format
 * (A_front = L' L'^T, L' = L D^{1/2}): rows below a column's 64-pivot diagonal
 * block hold L' = L sqrt(d), the diagonal holds sqrt(d), the strictly lower
 * part of each 64x64 diagonal block the unit L, its strictly upper part
 * X = L_bb^{-1} transposed (tests/mf_emulator.py: device_panel_to_ldl). */
int rba_get_factor(rba_ctx* ctx, int32_t slot, double* out_h, int64_t count);
/* Ordered pole sums (forward.py:61-63; sensitivity.py:77-78,95-96):
 *   data: d[s][j][r] = sum_i 2 Re(alpha_ij q_i [* xi_i])  (times_pole = 1 for J v)
 *   cells: out[c] = sum_i t_i[c]
 * slot_of_pole_h[i] = row of pole i in the gathered partial array. */
int rba_combine_data(rba_ctx* ctx, const double* qall_d, const int32_t* slot_of_pole_h,
                     int32_t times_pole, double* d_d);
int rba_combine_cells(rba_ctx* ctx, const double* tall_d, const int32_t* slot_of_pole_h,
                      double* out_d);
/* Regulariser square root R (nrows x P CSR) -- dense-Cholesky factor of the
 * reference (regularization.py:65-66) or the face-based root. */
int rba_set_reg(rba_ctx* ctx, int64_t nrows, const int64_t* indptr_h, const int32_t* indices_h,
                const double* data_h);
/* y = alpha R x (+ y if accumulate), transpose=1: y = alpha R^T x (+ y) */
int rba_reg_apply(rba_ctx* ctx, int32_t transpose, const double* x_d, double alpha, double* y_d,
                  int32_t accumulate);
/* The regulariser operator L = D Mdiv^-1 D^T + eps diag(meas) (P x P CSR,
 * regularization.py:55-63) and y = alpha L x (+ y): reg_value_grad
 * (regularization.py:71-75) and the GN gradient term lambda L (m - m_ref)
 * (inversion.py:250) on the device. */
int rba_set_reg_L(rba_ctx* ctx, int64_t n, const int64_t* indptr_h, const int32_t* indices_h,
                  const double* data_h);
int rba_reg_L_apply(rba_ctx* ctx, const double* x_d, double alpha, double* y_d,
                    int32_t accumulate);
/* LSQR vector kernels (SciPy lsqr recurrences, inversion.py:153) */
int rba_vec_axpby(rba_ctx* ctx, int64_t n, double a, const double* x_d, double b,
                  const double* y_d, double* out_d);
int rba_vec_mul(rba_ctx* ctx, int64_t n, const double* a_d, const double* x_d, double alpha,
                double* out_d);
int rba_vec_dot(rba_ctx* ctx, int64_t n, const double* x_d, const double* y_d, double* result_h);
int rba_vec_lsqr_xw(rba_ctx* ctx, int64_t n, double t1, double t2, const double* v_d,
                    double* w_d, double* x_d, double* wnorm2_h);
/* counters (CacheCounters, shifted.py:64-70) and sizes:
 * out[10]: factorizations, solves, N, P, Mr, S, m, n_local,
 *          receiver-Green mode on (1/0), Green builds (slots) */
int rba_info(rba_ctx* ctx, int64_t* out_h);
/* bytes of device memory held by the context: factors, workspace, other */
int rba_memory(rba_ctx* ctx, int64_t* out_h);
int rba_sync(rba_ctx* ctx);
/* Context options:
 *  "green" 0|1        -- 0 disables the receiver-Green mode (per-action
 *                        sweeps); ranks of one job agree on the mode
 *  "lazy_factors" 0|1 -- allocate a slot's factor storage on its first
 *                        factorisation (generic mode: the reference's
 *                        cache.factorize(i, A), shifted.py:98-105, where the
 *                        pole count is not known up front); set before
 *                        rba_set_poles. */
int rba_set_option(rba_ctx* ctx, const char* name, int64_t value);
/* The Ozaki-scheme INT8 Schur updates (kernels_ozaki.cu; env RBA_OZAKI=0
 * turns them off): out[5] = on (1/0), executed int8 ops and FP64-equivalent
 * flops per pole factorisation, poles per launch, minimum pivots per front. */
int rba_oz_stats(rba_ctx* ctx, double* out_h);
/* Cycle counters of the Ozaki GEMM's roles summed over CTAs since the last
   reset (profiling aid): out_h[10] = MMA-issuer loop, its waits for data, its
   waits for TMEM, producer waits for a free stage, epilogue waits for the
   accumulators, TMEM drain, global read-modify-write, k steps, tiles, issuer loop in ns. */
int rba_oz_prof(rba_ctx* ctx, double* out_h, int reset);
/* Device time per kernel class (ms, CUDA events around every launch while
 * timing is enabled), out[16]: scatter, extend-add, diag, trsm, gemm (DMMA),
 * solve-fwd, solve-bwd, element/observation, vector/SpMV, M assembly,
 * receiver-Green, Ozaki INT8 Schur (digit split + GEMM), ...,
 * out[15] = kernel launches issued by this context (always counted).
 * rba_set_timing: 1 on, 0 off, 2 reset the accumulators. */
int rba_timings(rba_ctx* ctx, double* out_h);
int rba_set_timing(rba_ctx* ctx, int32_t enabled);
/* out[128]: out[0..15] as rba_timings; out[16+L] forward-sweep ms of level L,
 * out[48+L] backward-sweep ms of level L (L < 32). */
int rba_timings_detail(rba_ctx* ctx, double* out_h);

#ifdef __cplusplus
}
#endif
#endif
