// Host-side launch wrappers of the sm_100a kernels.
#pragma once
#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>

#include "fronts.cuh"

namespace rba {

struct SlotPtrs {
  cplx* p[32];
};

struct SolveBatch {
  const cplx* factor[32];
  cplx* x[32];
  cplx* uvec[32];
  int* flags_f[32];
  int* flags_b[32];
  int* done_f[32];
  int* done_b[32];
  int epoch[32];
};

// factorisation
void launch_assemble_M(cudaStream_t st, int64_t nnz, const int64_t* cptr, const int64_t* coff,
                       const double* mass, const double* m, double* expm, int64_t P, int k2,
                       double* Mv);
void launch_scatter_A(cudaStream_t st, int64_t nnz, const int64_t* tgt, const double* Kv,
                      const double* Mv, const PoleBatch& pb);
void launch_scatter_vals(cudaStream_t st, int64_t nnz, const int64_t* tgt, const cplx* vals,
                         cplx* factor);
void launch_extend_add(cudaStream_t st, const int2* tasks, int ntasks, const FrontsDev& F,
                       const PoleBatch& pb);
void launch_diag(cudaStream_t st, const PanelTask* tasks, int ntasks, const FrontsDev& F,
                 const PoleBatch& pb, int* err);
void launch_diag2(cudaStream_t st, const PanelTask* tasks, int ntasks, const FrontsDev& F,
                  const PoleBatch& pb, int* err, int nsmall = 0, int nmid = 0);
void launch_trsm(cudaStream_t st, const PanelTask* tasks, int ntasks, const FrontsDev& F,
                 const PoleBatch& pb);
void launch_gemm_update(cudaStream_t st, const GemmTask* tasks, int ntasks, int ntiles,
                        const FrontsDev& F, const PoleBatch& pb);
void launch_gemm3(cudaStream_t st, const GemmTask* tasks, int ntasks, int nctas,
                  const FrontsDev& F, const PoleBatch& pb, int variant);
void launch_gemm5(cudaStream_t st, const GemmTask* tasks, int ntasks, int nctas,
                  const FrontsDev& F, const PoleBatch& pb, const cplx* zeros, int variant);
void launch_schur_small(cudaStream_t st, const int32_t* fronts, int nfr, const FrontsDev& F,
                        const PoleBatch& pb);
void launch_gemm6(cudaStream_t st, const GemmTask* tasks, int ntasks, int nctas,
                  const FrontsDev& F, const PoleBatch& pb, const cplx* zeros, int variant);
// Schur update of large fronts on the INT8 tensor cores (Ozaki scheme)
void oz_prof_read(unsigned long long* out, bool reset);
void launch_oz_schur(cudaStream_t st, const OzTask* tasks, int ntasks, const int2* tiles,
                     int nrowtiles, int ntiles,
                     const FrontsDev& F, const PoleBatch& pb, unsigned char* split,
                     int64_t split_pole, double* scl, int64_t exp_pole, int wide, int* ticket);
void launch_trsm3(cudaStream_t st, const PanelTask* tasks, int ntasks, const FrontsDev& F,
                  const PoleBatch& pb, int variant);

// solves
void launch_solve_level(cudaStream_t st, bool forward, int nr, const SolveTask* tasks,
                        int ntasks, int nslots, const FrontsDev& F, const SolveBatch& b,
                        int* ticket, int epoch, const int32_t* parent, const int32_t* need_u,
                        bool fused, bool stagex = false);
void solve_env_refresh();
void launch_solve_small(cudaStream_t st, bool forward, int nr, const int32_t* fronts, int nfr,
                        int nslots, const FrontsDev& F, const SolveBatch& b, int mb);
// receiver-Green build: backward sweep over Z (N x Mr) as DMMA GEMMs
void launch_zbwd(cudaStream_t st, const SolveTask* tasks, int ntasks, int nslots,
                 const FrontsDev& F, const SolveBatch& b, int* ticket, int Mr, const SlotPtrs& Z);
// forward sweep of the large fronts as DMMA GEMM tasks (NR right-hand sides)
void launch_zfwd(cudaStream_t st, const SolveTask* tasks, int ntasks, int nslots,
                 const FrontsDev& F, const SolveBatch& b, int* ticket, int NR);
void launch_perm_in(cudaStream_t st, int64_t n, int nrhs, int NR, const int32_t* perm,
                    const cplx* b, int64_t ldb, cplx* x);
void launch_perm_out(cudaStream_t st, int64_t n, int nrhs, int NR, const int32_t* perm,
                     const cplx* x, cplx* b, int64_t ldb);

// element / observation / reduction operators
struct ElemDev {
  int64_t N, P;
  const int32_t* cell_dofs;  // P*6, permuted dofs, -1 eliminated
  const double* mass;        // P*36
  const double* expm;        // P
  const int64_t* dc_ptr;     // N+1 (permuted dof -> items)
  const int32_t* dc_item;    // c*6 + a
};
void launch_jvp_rhs2(cudaStream_t st, int nslots, const ElemDev& E, const double* v,
                     const SlotPtrs& g, const SlotPtrs& out, int NR, int S, cplx* w);
void launch_jvp_rhs(cudaStream_t st, int nslots, const ElemDev& E, const double* v,
                    const SlotPtrs& g, const SlotPtrs& out, int NR, int S);
void launch_q_apply(cudaStream_t st, int nslots, int64_t Mr, const int64_t* qptr,
                    const int32_t* qcol, const double* qval, const SlotPtrs& h, int NR, int S,
                    cplx* qpart /* [slot][S][Mr] */);
void launch_combine_data(cudaStream_t st, int m, int S, int Kt, int64_t Mr, const cplx* qall,
                         const int32_t* slot_of_pole, const cplx* residues, const cplx* poles,
                         bool times_pole, double* d /* [S][Kt][Mr] */);
void launch_vjp_rhs(cudaStream_t st, int nslots, const int32_t* pole_of_slot, int S, int Kt,
                    int64_t Mr, int64_t N, const double* w, const cplx* residues,
                    const int64_t* qtptr, const int32_t* qtcol, const double* qtval,
                    cplx* wa /* [slot][S][Mr] */, const SlotPtrs& out, int NR);
// receiver Green's functions (kernels_ops.cu)
void launch_green_rhs(cudaStream_t st, int nslots, int64_t N, int64_t m0, int nb, int NR,
                      const int64_t* qtptr, const int32_t* qtcol, const double* qtval,
                      const SlotPtrs& x);
void launch_green_store(cudaStream_t st, int nslots, int64_t N, int64_t Mr, int64_t m0, int nb,
                        int NR, const SlotPtrs& x, const SlotPtrs& Z);
void launch_green_jvp(cudaStream_t st, int nslots, int64_t N, int Mr, int S, int NR, int nchunk,
                      const SlotPtrs& Z, const SlotPtrs& h, cplx* part, cplx* qpart);
void launch_walpha(cudaStream_t st, int nslots, const int32_t* pole_of_slot, int S, int Kt,
                   int64_t Mr, const double* w, const cplx* residues, cplx* wa);
void launch_green_vjp(cudaStream_t st, int nslots, int64_t N, int Mr, int S, int NR,
                      const SlotPtrs& Z, const cplx* wa, const SlotPtrs& x);
void launch_vjp_cells(cudaStream_t st, int nslots, const int32_t* pole_of_slot,
                      const cplx* poles, const ElemDev& E, const SlotPtrs& z,
                      const SlotPtrs& g, int NR, int S, double* tpart /* [slot][P] */);
void launch_combine_cells(cudaStream_t st, int m, int64_t P, const double* tall,
                          const int32_t* slot_of_pole, double* out);
void launch_spmv(cudaStream_t st, int64_t nrows, const int64_t* ptr, const int32_t* idx,
                 const double* val, const double* x, double alpha, double* y, bool accumulate);
// vector kernels (deterministic reductions); partial buffer >= 1024 doubles
void launch_axpby(cudaStream_t st, int64_t n, double a, const double* x, double b,
                  const double* y, double* out);
void launch_mul(cudaStream_t st, int64_t n, const double* a, const double* x, double alpha,
                double* out);
void launch_dot(cudaStream_t st, int64_t n, const double* x, const double* y, double* part,
                double* result);
void launch_lsqr_xw(cudaStream_t st, int64_t n, double t1, double t2, const double* v,
                    double* w, double* x, double* part, double* result);
void launch_zero_c(cudaStream_t st, int64_t n, cplx* p);
void launch_conj(cudaStream_t st, int64_t n, const cplx* src, cplx* dst);
void launch_factor_stats(cudaStream_t st, const FrontsDev& F, int nfront, const cplx* fac,
                         double* out /* [4] */);

}  // namespace rba
