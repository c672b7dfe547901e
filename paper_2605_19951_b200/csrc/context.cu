// C-ABI implementation: device context, setup (pattern, symbolic, plans),
// factorisation driver, solves and the operator entry points.
// See include/rba_b200.h for the contract and the reference functions each
// entry point replaces.
#include <cstdio>
#include <cstring>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "../../include/rba_b200.h"
#include "kernels.h"
#include "mesh_prep.h"
#include "symbolic.h"

using rba::cplx;

namespace {
thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(e_ == cudaErrorMemoryAllocation ? RBA_ERR_OOM : RBA_ERR_CUDA,           \
                  std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #call);   \
  } while (0)

#define CKL()                                                                             \
  do {                                                                                    \
    cudaError_t e_ = cudaGetLastError();                                                  \
    if (e_ != cudaSuccess)                                                                \
      return fail(RBA_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e_)); \
  } while (0)

enum StepKind { ST_EA = 0, ST_DIAG = 1, ST_TRSM = 2, ST_GEMM = 3, ST_OZ = 4, ST_SSCHUR = 5 };
struct Step {
  int kind;
  int64_t off;
  int n;
  int ntiles;
  int schur;   // ST_GEMM: 1 = Schur-complement update (K = npiv), 0 = panel update;
               // ST_DIAG: blocks of 33..48 pivots (after the ntiles blocks of <= 32);
               // ST_OZ: row tiles of the step (digit-split CTAs)
  int level;
  int64_t oz_split = 0;   // ST_OZ: digit-block bytes per pole
  int64_t oz_rows = 0;    // ST_OZ: border rows (row exponents) per pole
  int64_t oz_tile_off = 0;  // ST_OZ: offset of the step's tile list
};
constexpr int64_t OZ_BLK_BYTES = 7 * 2 * 192 * 16;  // kernels_ozaki.cu OZ_BLK (A_big + B)
constexpr int64_t OZ_BLK2_BYTES = 7 * 2 * 128 * 16 + 2 * 12288;  // OZ_BLK2 (A_big + two B arrangements)

int nr_pad(int s) { return s <= 1 ? 1 : s <= 2 ? 2 : s <= 4 ? 4 : 8; }
}  // namespace

struct rba_symbolic {
  rba::Symbolic S;
};

struct rba_ctx {
  int device = 0;
  cudaStream_t st = nullptr;
  // second lane of the factorisation (rba_factor): the two halves of a pole
  // batch run the same plan on two streams, so the DRAM-bound steps of one
  // half (extend-add, digit split) overlap the tensor-bound steps of the other
  cudaStream_t st2 = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int fstreams = 1;            // RBA_FACTOR_STREAMS=2: two lanes (measured no gain at C4, 1.888 vs
                               // 1.893 s per 16 poles: the INT8 phases run at the board power cap and
                               // the Ozaki GEMM CTA leaves registers for one extend-add CTA per SM)
  int* oz_ticket = nullptr;    // [2] tile tickets of the Ozaki GEMM launches, one per lane
  bool own_stream = false;
  std::vector<void*> allocs;       // persistent (mesh-level) device allocations
  size_t mem_other = 0, mem_factor = 0, mem_work = 0;
  // mesh
  bool have_mesh = false;
  int64_t N = 0, P = 0;
  int k = 0;
  rba::Symbolic sym;
  int64_t nnzA = 0;
  std::vector<int32_t> a_rows, a_cols;
  std::vector<double> Kv_h;
  double *Kv = nullptr, *Mv = nullptr, *mass = nullptr, *mdev = nullptr, *expm = nullptr;
  int64_t *tgt = nullptr, *cptr = nullptr, *coff = nullptr;
  int32_t* cell_dofs_p = nullptr;
  int64_t* dc_ptr = nullptr;
  int32_t* dc_item = nullptr;
  int32_t* perm_d = nullptr;
  rba::FrontsDev F{};
  std::vector<Step> plan;
  int2* ea_tasks = nullptr;
  rba::PanelTask* pt_tasks = nullptr;
  rba::GemmTask* gm_tasks = nullptr;
  int32_t* ss_fronts = nullptr;   // ST_SSCHUR: small fronts (one pivot block) per level
  bool schur_small = true;        // RBA_SCHUR_SMALL=0: k_gemm6 tiles for the small fronts too
  int schur_small_b = 288;        // largest border of a front taken by k_schur_small (RBA_SCHUR_SMALL_B)
  // Ozaki-scheme INT8 tensor-core Schur updates (RBA_OZAKI, kernels_ozaki.cu)
  bool ozaki = true;           // RBA_OZAKI=0: DMMA for every Schur update
  int oz_stages = 4;           // RBA_OZ_STAGES: load-ring depth of the wide GEMM (4 or 5; 5 measured
                               // the same: the feed is L2-bandwidth, not latency bound)
  int oz_kmax = 1 << 20;       // RBA_OZ_KMAX: pivots per pass of a Schur update (passes of 1024
                               // measured 4 % slower: one more epilogue per tile)
  int oz_min_k = 128;          // Schur updates of fronts with at least this many pivots (RBA_OZ_MINK)
  bool oz_trail = true;        // RBA_OZ_TRAIL=0: aggregated panel updates stay on the DMMA GEMM
  int oz_min_rows = 256;       // aggregated panel updates with at least this many rows (RBA_OZ_MINROWS)
  rba::OzTask* oz_tasks = nullptr;
  int2* oz_tiles = nullptr;    // (row tile, column tile) per CTA, L2-friendly order
  int64_t oz_split_max = 0, oz_rows_max = 0;
  double oz_int8_ops = 0, oz_flops = 0;   // per pole factorisation: executed int8 ops,
                                          // FP64-equivalent (4-multiply) flops
  int oz_sub = 1;              // poles per Ozaki launch (digit-buffer budget)
  int oz_ts = 0;               // RBA_OZ_TS=1: A digits staged in TMEM (tcgen05.cp), wide MMAs read A from TMEM
                               // (bitwise equal; 981 clk per k step alone, tools/umma_i8_ts_probe.cu, but
                               // 1,380 vs 1,189 in the kernel: off)
  int oz_pair = 0;             // RBA_OZ_2CTA=1: cluster-pair GEMM (cta_group::2, M = 256)
  int oz_wide = 1;             // RBA_OZ_WIDE=0: one N = 64 MMA per digit pair (28 per k step)
                               // instead of 10 wide ones (same integer sums, bitwise equal)
  unsigned char* oz_buf = nullptr;
  double* oz_exp = nullptr;   // row scales 2^(e_r - 54) of the Ozaki digit blocks
  std::vector<std::pair<int64_t, int>> fwd_lv, bwd_lv, fwdb_lv, bwdb_lv, small_lv;
  std::vector<int> small_mb;   // per level: pivot blocks of the largest warp-per-front front
  // host copies for the pruned forward sweeps of the receiver-Green build
  std::vector<int32_t> smallf_h;
  std::vector<rba::SolveTask> ftb_h;
  std::vector<int64_t> q_ptr_h;
  std::vector<int32_t> q_col_h;
  int prune_nb = 0;                                            // batch width of the lists
  std::vector<std::pair<int64_t, int>> pr_small_lv, pr_fwdb_lv;  // [batch * nlevels + L]
  int32_t* pr_small = nullptr;
  rba::SolveTask* pr_fwdb = nullptr;
  rba::SolveTask *fwdb_tasks = nullptr, *bwdb_tasks = nullptr;
  int32_t* small_fronts = nullptr;
  rba::SolveTask *fwd_tasks = nullptr, *bwd_tasks = nullptr, *bwd_all = nullptr;
  int64_t n_fwd_tasks = 0, n_bwd_tasks = 0;
  int32_t *parent_d = nullptr, *need_u_d = nullptr;
  int epoch_limit = 1 << 20;  // flags/counters are monotonic in the epoch; reset before overflow
  bool fused_sweep = false;   // RBA_SWEEP=fused: one launch per sweep (cross-front counters)
  bool diag_v1 = false;       // RBA_DIAG=v1: unblocked diagonal-block kernel
  int fwd_gemm = -1;          // RBA_FWD_GEMM: as RBA_BWD_GEMM for the forward tasks
  int bwd_gemm = -1;          // RBA_BWD_GEMM: 1 / 0 force the DMMA-GEMM / GEMV backward
                              // tasks; default: GEMM for 8 right-hand sides
  int* tickets = nullptr;
  int64_t nblocks = 0;
  // observation / sources
  int64_t Mr = 0;
  int64_t *q_ptr = nullptr, *qt_ptr = nullptr;
  int32_t *q_col = nullptr, *qt_col = nullptr;
  double *q_val = nullptr, *qt_val = nullptr;
  std::vector<void*> obs_allocs;
  int S = 0, NRs = 1;
  cplx* Fsrc = nullptr;
  // poles
  int m = 0, Kt = 0;
  std::vector<cplx> poles_h, res_h;
  cplx *poles_d = nullptr, *res_d = nullptr;
  std::vector<int> local;
  int32_t* pole_of_slot = nullptr;
  int32_t* slot_map = nullptr;   // m entries, staging for combine
  std::vector<void*> pole_allocs;
  // per local slot
  std::vector<cplx*> factor, g, x, uvec;
  std::vector<rba::TMap*> tmaps;  // per slot: [nfront][2] tensor maps of the factor panels
  // receiver Green's functions Z = A^{-1} Q^T per slot (RBA_GREEN, default on
  // when they fit): J v / J^T w stream Z instead of sweeping the factor
  bool green_req = true;
  bool green = false;
  std::vector<cplx*> Z;
  std::vector<char> green_valid;
  std::vector<int*> zflags;       // per slot: [nblocks][Mr/32] completion flags of k_zbwd
  std::vector<int> zepoch;
  cplx* green_part = nullptr;
  cplx* jvp_w = nullptr;          // two-pass J v workspace (in the pool, past Z), or null
  int green_chunks = 64;
  bool green_prune = true;        // RBA_GREEN_PRUNE=0: full forward sweeps in the Z build
  bool green_gemm = true;         // RBA_GREEN_GEMM=0: per-batch backward sweeps in the Z build
  int64_t n_green = 0;            // Z builds (slots)
  std::vector<int*> flf, flb, dnf, dnb;
  std::vector<int> slot_epoch;    // solves issued per local slot (flags / counters)
  std::vector<char> valid;
  int NRw = 1;
  std::vector<cplx*> upd;
  int fbatch = 1;
  cplx* wa = nullptr;
  cplx* stage = nullptr;
  int64_t stage_n = 0;
  // regulariser
  int64_t R_rows = 0;
  int64_t *r_ptr = nullptr, *rt_ptr = nullptr;
  int32_t *r_idx = nullptr, *rt_idx = nullptr;
  double *r_val = nullptr, *rt_val = nullptr;
  std::vector<void*> reg_allocs;
  // regulariser operator L (P x P CSR): reg_value_grad on the device
  int64_t L_n = 0;
  int64_t* l_ptr = nullptr;
  int32_t* l_idx = nullptr;
  double* l_val = nullptr;
  std::vector<void*> regl_allocs;
  // factor buffers allocated on first use of a slot (generic mode: the
  // reference's factorize(i, A) with an unknown pole count); one update arena
  bool lazy = false;
  // misc
  double* red_part = nullptr;
  double* red_res = nullptr;
  cplx* zeros = nullptr;      // 1 KB of zeros: source of out-of-range bulk-copy columns
  int* err_d = nullptr;
  int64_t n_fact = 0, n_solve = 0;
  int epoch = 0;
  bool model_set = false;
  bool timing = false;
  double t_ms[8] = {0};
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  // per-kernel-class device time (CUDA events around every launch, enabled
  // by rba_set_timing) and the launch count of this context's kernels
  double cls_ms[128] = {0};   // 0-15 kernel classes; 16+L fwd, 48+L bwd, 80+L factor,
                              // 112+L GEMM per level
  bool gemm_dfma = false;     // RBA_GEMM=dfma selects the DFMA reference kernels
  int gemm_v = 6;             // default 3M DMMA kernel (k_gemm6); RBA_GEMM=v3..v7b select
                              // the earlier kernels for A/B tests
  int small_p = 2 * rba::PB;  // warp-per-front solves up to this npiv (RBA_SMALLP=64|128)
  int gemm5_var = 8;          // v5/v6 stage shape (see launch_gemm5 / launch_gemm6); default
                              // v8c = 64x32 half tiles, 16 k x 2 stages, 3 CTAs/SM,
                              // operands by TMA tensor copies
  int panel_v = 0;            // RBA_GEMM_PANEL: kernel for the panel updates (0 = as RBA_GEMM)
  int panel_var = 0;
  int gemm_var = 0;           // k_gemm3 stage shape (TRSM; the v3/v4 GEMM): 0 (default TRSM,
                              // RBA_GEMM=v3) = 8 k x 3 stages, 1 (RBA_GEMM=v4) = 16 k x 2;
                              // RBA_TRSM_VAR overrides
  int64_t launches = 0;
  std::vector<cudaEvent_t> evpool;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
};

namespace {

enum KClass { KC_SCATTER = 0, KC_EA = 1, KC_DIAG = 2, KC_TRSM = 3, KC_GEMM = 4, KC_FWD = 5,
              KC_BWD = 6, KC_ELEM = 7, KC_VEC = 8, KC_ASSEMBLY = 9, KC_GREEN = 10, KC_OZ = 11 };

struct Timed {
  rba_ctx* c;
  int cls;
  cudaEvent_t b = nullptr;
  Timed(rba_ctx* c_, int cls_, int nlaunch = 1) : c(c_), cls(cls_) {
    c->launches += nlaunch;
    if (!c->timing) return;
    cudaEvent_t a;
    if (c->evpool.size() < 2) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      c->evpool.push_back(e0);
      c->evpool.push_back(e1);
    }
    a = c->evpool.back(); c->evpool.pop_back();
    b = c->evpool.back(); c->evpool.pop_back();
    cudaEventRecord(a, c->st);
    c->pending.push_back({cls, {a, b}});
  }
  ~Timed() {
    if (b) cudaEventRecord(b, c->st);
  }
};

void flush_timing(rba_ctx* c) {
  if (c->pending.empty()) return;
  cudaStreamSynchronize(c->st);
  for (auto& p : c->pending) {
    float ms = 0;
    cudaEventElapsedTime(&ms, p.second.first, p.second.second);
    c->cls_ms[p.first] += ms;
    c->evpool.push_back(p.second.first);
    c->evpool.push_back(p.second.second);
  }
  c->pending.clear();
}

template <class T>
int dalloc(rba_ctx* c, std::vector<void*>& list, T** out, size_t count, size_t* acct) {
  *out = nullptr;
  if (count == 0) count = 1;
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, count * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(RBA_ERR_OOM, "device allocation of " + std::to_string(count * sizeof(T)) +
                                 " bytes failed: " + cudaGetErrorString(e));
  }
  list.push_back(p);
  if (acct) *acct += count * sizeof(T);
  *out = (T*)p;
  (void)c;
  return RBA_OK;
}

template <class T>
int upload(rba_ctx* c, std::vector<void*>& list, T** out, const T* h, size_t count) {
  int rc = dalloc(c, list, out, count, &c->mem_other);
  if (rc) return rc;
  if (count) CK(cudaMemcpyAsync(*out, h, count * sizeof(T), cudaMemcpyHostToDevice, c->st));
  return RBA_OK;
}

void free_list(std::vector<void*>& list) {
  for (void* p : list) cudaFree(p);
  list.clear();
}

void free_slots(rba_ctx* c) {
  free_list(c->pole_allocs);
  c->factor.clear(); c->g.clear(); c->x.clear(); c->uvec.clear();
  c->flf.clear(); c->flb.clear(); c->valid.clear(); c->upd.clear();
  c->dnf.clear(); c->dnb.clear(); c->slot_epoch.clear();
  c->wa = nullptr;
  c->pole_of_slot = nullptr;
  c->slot_map = nullptr;
  c->oz_buf = nullptr;
  c->oz_exp = nullptr;
  c->poles_d = nullptr;
  c->res_d = nullptr;
  c->mem_factor = 0;
  c->mem_work = 0;
}

int ensure_stage(rba_ctx* c, int64_t n) {
  if (c->stage_n >= n) return RBA_OK;
  if (c->stage) { cudaFree(c->stage); c->stage = nullptr; }
  cudaError_t e = cudaMalloc(&c->stage, n * sizeof(cplx));
  if (e != cudaSuccess) { cudaGetLastError(); c->stage_n = 0; return fail(RBA_ERR_OOM, "stage alloc"); }
  c->stage_n = n;
  return RBA_OK;
}

// ---------------------------------------------------------------------------
// plans
// ---------------------------------------------------------------------------
int build_plans(rba_ctx* c) {
  const rba::Symbolic& S = c->sym;
  int panel = 4;                  // 64-column blocks per trailing-update panel
  if (const char* e = getenv("RBA_PANEL")) panel = std::max(1, atoi(e));
  std::vector<int2> ea;
  std::vector<rba::PanelTask> pt;
  std::vector<rba::GemmTask> gm;
  std::vector<rba::OzTask> oz;
  std::vector<int32_t> ssf;
  std::vector<int2> ozt;
  c->plan.clear();
  c->oz_split_max = c->oz_rows_max = 0;
  c->oz_int8_ops = c->oz_flops = 0;
  // one plan step of Ozaki (INT8 tensor-core) updates: C[r, c] -= L'[r, t0:t1]
  // L'[c, t0:t1]^T for clo <= c < chi, c <= r < nf, per front
  struct OzStep { int64_t ooff = 0, otoff = 0, bytes = 0, rows = 0; int tiles = 0, rt = 0; };
  auto oz_begin = [&]() { OzStep o; o.ooff = (int64_t)oz.size(); o.otoff = (int64_t)ozt.size(); return o; };
  auto oz_add = [&](OzStep& o, int s, int nf, int clo, int chi, int t0, int t1) {
    const int nrt = (nf - clo + 63) / 64, ntc = (chi - clo + 63) / 64, nks = (t1 - t0 + 15) / 16;
    rba::OzTask t{};
    t.s = s; t.nf = nf; t.c_lo = clo; t.c_hi = chi; t.t0 = t0; t.t1 = t1;
    t.nrt = nrt; t.nks = nks; t.tile_start = o.tiles; t.rt_start = o.rt;
    t.split_off = o.bytes; t.exp_off = o.rows;
    oz.push_back(t);
    // lower-triangle 64 x 64 tiles in 12 x 12 super-blocks (column-major
    // inside): the ~148 CTAs resident at a time reuse each other's digit
    // blocks in L2
    constexpr int SB = 12;
    int nt = 0;
    if (c->oz_pair) {
      // cluster pairs own two row tiles (2 i, 2 i + 1) x one column tile
      const int np = (nrt + 1) / 2;
      for (int I = 0; I < np; I += SB / 2)
        for (int J = 0; J < ntc && J <= 2 * (I + SB / 2) - 1; J += SB)
          for (int j = J; j < std::min(J + SB, ntc); ++j)
            for (int i = std::max(I, j / 2); i < std::min(I + SB / 2, np); ++i) {
              ozt.push_back(make_int2(i, j));
              ++nt;
            }
    } else
    for (int I = 0; I < nrt; I += SB)
      for (int J = 0; J < ntc && J <= I + SB - 1; J += SB)
        for (int j = J; j < std::min(J + SB, ntc); ++j)
          for (int i = std::max(I, j); i < std::min(I + SB, nrt); ++i) {
            ozt.push_back(make_int2(i, j));
            ++nt;
          }
    o.tiles += nt;
    o.rt += nrt;
    o.bytes += c->oz_pair ? (int64_t)((nrt + 1) / 2 * 2) * nks * OZ_BLK2_BYTES : (int64_t)nrt * nks * OZ_BLK_BYTES;
    o.rows += nf - clo;
    const double w = chi - clo;
    c->oz_int8_ops += 2.0 * 28 * ((c->oz_pair ? 256.0 : 128.0) * 64 * 32) * nks * nt;
    c->oz_flops += 8.0 * (w * (nf - clo) - 0.5 * w * (w - 1)) * (t1 - t0);
  };
  auto oz_end = [&](OzStep& o, int level) {
    if ((int64_t)oz.size() == o.ooff) return;
    Step st{ST_OZ, o.ooff, (int)((int64_t)oz.size() - o.ooff), o.tiles, o.rt, level};
    st.oz_split = o.bytes;
    st.oz_rows = o.rows;
    st.oz_tile_off = o.otoff;
    c->plan.push_back(st);
    c->oz_split_max = std::max(c->oz_split_max, o.bytes);
    c->oz_rows_max = std::max(c->oz_rows_max, o.rows);
  };
  for (int L = 0; L < S.nlevels; ++L) {
    const size_t plan0 = c->plan.size();
    const int q0 = S.level_ptr[L], q1 = S.level_ptr[L + 1];
    // extend-add / zeroing
    int64_t off = ea.size();
    for (int q = q0; q < q1; ++q) {
      int s = S.level_fronts[q];
      bool kids = S.child_ptr[s + 1] > S.child_ptr[s];
      if (!kids && S.nf[s] == S.npiv[s]) continue;
      if (S.nf[s] <= 384) {
        ea.push_back(make_int2(s, -1));      // small front: one CTA does it all
        continue;
      }
      int c0 = kids ? 0 : S.npiv[s] / 32;
      for (int ct = c0; ct * 32 < S.nf[s]; ++ct) ea.push_back(make_int2(s, ct));
    }
    if ((int64_t)ea.size() > off) c->plan.push_back({ST_EA, off, (int)(ea.size() - off), 0});
    int kmax = 0;
    for (int q = q0; q < q1; ++q) kmax = std::max(kmax, (S.npiv[S.level_fronts[q]] + rba::PB - 1) / rba::PB);
    for (int kk = 0; kk < kmax; ++kk) {
      const int k0 = kk * rba::PB;
      // diagonal blocks of at most 32 pivots first (k_diag2<32>: 128 threads,
      // 4x less shared memory), then the full ones
      int64_t doff = pt.size();
      for (int q = q0; q < q1; ++q) {
        int s = S.level_fronts[q];
        if (S.npiv[s] > k0 && S.npiv[s] - k0 <= 32) pt.push_back({s, k0, k0, 0});
      }
      const int nsmall = (int)(pt.size() - doff);
      // then the blocks of 33..48 pivots (k_diag2<48>: 52 KB, 4 CTAs per SM instead of 2)
      for (int q = q0; q < q1; ++q) {
        int s = S.level_fronts[q];
        if (S.npiv[s] - k0 > 32 && S.npiv[s] - k0 <= 48) pt.push_back({s, k0, k0, 0});
      }
      const int nmid = (int)(pt.size() - doff) - nsmall;
      for (int q = q0; q < q1; ++q) {
        int s = S.level_fronts[q];
        if (S.npiv[s] - k0 > 48) pt.push_back({s, k0, k0, 0});
      }
      if ((int64_t)pt.size() > doff)
        c->plan.push_back({ST_DIAG, doff, (int)(pt.size() - doff), c->diag_v1 ? 0 : nsmall,
                           c->diag_v1 ? 0 : nmid});
      int64_t toff = pt.size();
      for (int q = q0; q < q1; ++q) {
        int s = S.level_fronts[q];
        if (S.npiv[s] <= k0) continue;
        int kb = std::min(rba::PB, S.npiv[s] - k0);
        for (int r0 = k0 + kb; r0 < S.nf[s]; r0 += rba::PB) pt.push_back({s, k0, r0, 0});
      }
      if ((int64_t)pt.size() > toff) c->plan.push_back({ST_TRSM, toff, (int)(pt.size() - toff), 0});
      // trailing update after block kk: inside a panel of `panel` blocks only
      // the rest of the panel is updated (K = 64, look-ahead); at the panel's
      // last block all columns beyond the panel get one update with
      // K = the whole panel (fewer, fatter tensor-core GEMM passes).
      int64_t goff = gm.size();
      int tiles = 0;
      OzStep otr = oz_begin();
      for (int q = q0; q < q1; ++q) {
        int s = S.level_fronts[q];
        const int p = S.npiv[s];
        if (p <= k0) continue;
        const int kb = std::min(rba::PB, p - k0);
        const int pstart = (kk / panel) * panel * rba::PB;
        const int pend = std::min(p, (kk / panel + 1) * panel * rba::PB);
        int t0, t1, clo, chi;
        if (k0 + kb < pend) {            // in-panel look-ahead update
          t0 = k0; t1 = k0 + kb; clo = k0 + kb; chi = pend;
        } else {                         // end of panel: aggregated update
          t0 = pstart; t1 = pend; clo = pend; chi = p;
        }
        if (chi <= clo) continue;
        // aggregated panel updates of tall fronts on the INT8 tensor cores
        if (c->ozaki && c->oz_trail && t1 - t0 >= std::min(256, c->oz_min_k) &&
            S.nf[s] - clo >= c->oz_min_rows) {
          oz_add(otr, s, S.nf[s], clo, chi, t0, t1);
          continue;
        }
        int ntr = (S.nf[s] - clo + rba::GT - 1) / rba::GT;
        int ntc = (chi - clo + rba::GT - 1) / rba::GT;
        int nt = 0;
        for (int j = 0; j < ntc; ++j) nt += ntr - j;
        gm.push_back({s, t0, t1, clo, chi, tiles, ntr, 0});
        tiles += nt;
      }
      if ((int64_t)gm.size() > goff) c->plan.push_back({ST_GEMM, goff, (int)(gm.size() - goff), tiles});
      oz_end(otr, L);
    }
    // Schur complement of each front with a border: large fronts on the INT8
    // tensor cores (Ozaki scheme), the rest with the DMMA GEMM
    int64_t goff = gm.size();
    const int64_t ssoff = ssf.size();
    int tiles = 0;
    // the pivots of a wide front are taken in passes of at most oz_kmax (one
    // plan step per pass): the digit streams of the ~148 tiles in flight
    // (12 x 12 super-block: 18 row-tile streams of K / 16 x 28 KB) then stay
    // L2-resident while the tiles that share them catch up
    int opass = 1;
    for (int q = q0; q < q1; ++q) {
      int s = S.level_fronts[q];
      int p = S.npiv[s], nf = S.nf[s];
      if (nf > p && c->ozaki && p >= c->oz_min_k && p <= 16384)
        opass = std::max(opass, (p + c->oz_kmax - 1) / c->oz_kmax);
    }
    std::vector<OzStep> osc(opass);
    for (auto& o : osc) o = oz_begin();
    for (int q = q0; q < q1; ++q) {
      int s = S.level_fronts[q];
      int p = S.npiv[s], nf = S.nf[s];
      if (nf <= p || p == 0) continue;
      if (c->ozaki && p >= c->oz_min_k && p <= 16384) {
        if (opass == 1) oz_add(osc[0], s, nf, p, nf, 0, p);
        continue;
      }
      if (c->schur_small && p <= rba::PB && nf - p <= c->schur_small_b) {   // one pivot block: fragment-exact kernel
        ssf.push_back(s);
        continue;
      }
      int ntr = (nf - p + rba::GT - 1) / rba::GT;
      gm.push_back({s, 0, p, p, nf, tiles, ntr, 0});
      tiles += ntr * (ntr + 1) / 2;
    }
    if ((int64_t)gm.size() > goff) c->plan.push_back({ST_GEMM, goff, (int)(gm.size() - goff), tiles, 1});
    if ((int64_t)ssf.size() > ssoff) c->plan.push_back({ST_SSCHUR, ssoff, (int)(ssf.size() - ssoff), 0});
    oz_end(osc[0], L);
    // tasks of one plan step are contiguous in `oz`, so the passes of a
    // multi-pass level are built one after the other
    for (int j = 0; opass > 1 && j < opass; ++j) {
      OzStep o = oz_begin();
      for (int q = q0; q < q1; ++q) {
        int s = S.level_fronts[q];
        int p = S.npiv[s], nf = S.nf[s];
        if (nf <= p || !(c->ozaki && p >= c->oz_min_k && p <= 16384)) continue;
        const int np = (p + c->oz_kmax - 1) / c->oz_kmax;           // this front's passes
        const int len = ((p + np - 1) / np + 15) / 16 * 16;
        const int t0 = j * len, t1 = std::min(p, (j + 1) * len);
        if (t0 < t1) oz_add(o, s, nf, p, nf, t0, t1);
      }
      oz_end(o, L);
    }
    for (size_t q = plan0; q < c->plan.size(); ++q) c->plan[q].level = L;
  }
  int rc;
  if ((rc = upload(c, c->allocs, &c->ea_tasks, ea.data(), ea.size()))) return rc;
  if ((rc = upload(c, c->allocs, &c->pt_tasks, pt.data(), pt.size()))) return rc;
  if ((rc = upload(c, c->allocs, &c->gm_tasks, gm.data(), gm.size()))) return rc;
  if (!ssf.empty() && (rc = upload(c, c->allocs, &c->ss_fronts, ssf.data(), ssf.size()))) return rc;
  if (!oz.empty() && (rc = upload(c, c->allocs, &c->oz_tasks, oz.data(), oz.size()))) return rc;
  if (!ozt.empty() && (rc = upload(c, c->allocs, &c->oz_tiles, ozt.data(), ozt.size()))) return rc;

  // solve plans
  std::vector<rba::SolveTask> ft, bt, ftb, btb;
  std::vector<int32_t> smallf;
  c->fwd_lv.assign(S.nlevels, {0, 0});
  c->bwd_lv.assign(S.nlevels, {0, 0});
  c->fwdb_lv.assign(S.nlevels, {0, 0});
  c->bwdb_lv.assign(S.nlevels, {0, 0});
  c->small_lv.assign(S.nlevels, {0, 0});
  c->small_mb.assign(S.nlevels, 1);
  std::vector<int64_t> blk_off(S.nfront + 1, 0);
  for (int s = 0; s < S.nfront; ++s) blk_off[s + 1] = blk_off[s] + (S.npiv[s] + rba::PB - 1) / rba::PB;
  c->nblocks = blk_off[S.nfront];
  for (int L = 0; L < S.nlevels; ++L) {
    const int q0 = S.level_ptr[L], q1 = S.level_ptr[L + 1];
    int bmax = 0;
    for (int q = q0; q < q1; ++q) {
      int s = S.level_fronts[q];
      int npb = (S.npiv[s] + rba::PB - 1) / rba::PB;
      int nbb = (S.nf[s] - S.npiv[s] + rba::PB - 1) / rba::PB;
      bmax = std::max(bmax, npb + nbb);
    }
    int64_t off = ft.size();
    for (int b = 0; b < bmax; ++b)
      for (int q = q0; q < q1; ++q) {
        int s = S.level_fronts[q];
        int npb = (S.npiv[s] + rba::PB - 1) / rba::PB;
        int nbb = (S.nf[s] - S.npiv[s] + rba::PB - 1) / rba::PB;
        if (b < npb + nbb) ft.push_back({s, b});
      }
    c->fwd_lv[L] = {off, (int)(ft.size() - off)};
    // split for the per-level path: fronts with at most two pivot blocks go
    // to the warp-per-front kernels, the rest keep the block-task kernels
    {
      int64_t so = smallf.size();
      for (int q = q0; q < q1; ++q)
        if (S.npiv[S.level_fronts[q]] <= c->small_p) {
          smallf.push_back(S.level_fronts[q]);
          if (S.npiv[S.level_fronts[q]] > rba::PB) c->small_mb[L] = 2;
        }
      c->small_lv[L] = {so, (int)(smallf.size() - so)};
      int64_t bo = ftb.size();
      for (int b = 0; b < bmax; ++b)
        for (int q = q0; q < q1; ++q) {
          int s = S.level_fronts[q];
          if (S.npiv[s] <= c->small_p) continue;
          int npb = (S.npiv[s] + rba::PB - 1) / rba::PB;
          int nbb = (S.nf[s] - S.npiv[s] + rba::PB - 1) / rba::PB;
          if (b < npb + nbb) ftb.push_back({s, b});
        }
      c->fwdb_lv[L] = {bo, (int)(ftb.size() - bo)};
    }
    off = bt.size();
    int pmax = 0;
    for (int q = q0; q < q1; ++q) pmax = std::max(pmax, (S.npiv[S.level_fronts[q]] + rba::PB - 1) / rba::PB);
    for (int key = 0; key < pmax; ++key)
      for (int q = q0; q < q1; ++q) {
        int s = S.level_fronts[q];
        int npb = (S.npiv[s] + rba::PB - 1) / rba::PB;
        if (key < npb) bt.push_back({s, npb - 1 - key});
      }
    c->bwd_lv[L] = {off, (int)(bt.size() - off)};
    {
      int64_t bo = btb.size();
      for (int key = 0; key < pmax; ++key)
        for (int q = q0; q < q1; ++q) {
          int s = S.level_fronts[q];
          if (S.npiv[s] <= c->small_p) continue;
          int npb = (S.npiv[s] + rba::PB - 1) / rba::PB;
          if (key < npb) btb.push_back({s, npb - 1 - key});
        }
      c->bwdb_lv[L] = {bo, (int)(btb.size() - bo)};
    }
  }
  if ((rc = upload(c, c->allocs, &c->fwd_tasks, ft.data(), ft.size()))) return rc;
  if ((rc = upload(c, c->allocs, &c->bwd_tasks, bt.data(), bt.size()))) return rc;
  if ((rc = upload(c, c->allocs, &c->fwdb_tasks, ftb.data(), ftb.size()))) return rc;
  if ((rc = upload(c, c->allocs, &c->bwdb_tasks, btb.data(), btb.size()))) return rc;
  if ((rc = upload(c, c->allocs, &c->small_fronts, smallf.data(), smallf.size()))) return rc;
  c->smallf_h = smallf;
  c->ftb_h = ftb;
  c->prune_nb = 0;
  {
    // fused backward: levels top-down in one task list
    std::vector<rba::SolveTask> ba;
    for (int L = S.nlevels - 1; L >= 0; --L)
      ba.insert(ba.end(), bt.begin() + c->bwd_lv[L].first,
                bt.begin() + c->bwd_lv[L].first + c->bwd_lv[L].second);
    if ((rc = upload(c, c->allocs, &c->bwd_all, ba.data(), ba.size()))) return rc;
    c->n_fwd_tasks = ft.size();
    c->n_bwd_tasks = ba.size();
    std::vector<int32_t> need(S.nfront, 0);
    for (int ch = 0; ch < S.nfront; ++ch)
      if (S.parent[ch] >= 0) need[S.parent[ch]] += (S.nf[ch] - S.npiv[ch] + rba::PB - 1) / rba::PB;
    if ((rc = upload(c, c->allocs, &c->need_u_d, need.data(), need.size()))) return rc;
    int mx = 1;
    for (int s2 = 0; s2 < S.nfront; ++s2) mx = std::max({mx, need[s2], (S.npiv[s2] + rba::PB - 1) / rba::PB});
    c->epoch_limit = std::max(1, (1 << 30) / mx);
    if ((rc = upload(c, c->allocs, &c->parent_d, S.parent.data(), S.parent.size()))) return rc;
  }
  if ((rc = dalloc(c, c->allocs, &c->tickets, 2 * (size_t)S.nlevels + 2, &c->mem_other))) return rc;

  // solve gather lists (child u-vector rows -> parent front rows), child order
  const int64_t nrows_tot = S.rows_off[S.nfront];
  std::vector<int64_t> ucnt(nrows_tot + 1, 0);
  for (int ch = 0; ch < S.nfront; ++ch) {
    int s = S.parent[ch];
    if (s < 0) continue;
    for (int64_t kk = 0; kk < S.nf[ch] - S.npiv[ch]; ++kk)
      ucnt[S.rows_off[s] + S.relmap[S.rel_off[ch] + kk] + 1]++;
  }
  for (int64_t i = 0; i < nrows_tot; ++i) ucnt[i + 1] += ucnt[i];
  std::vector<int64_t> uidx(ucnt[nrows_tot]);
  std::vector<int64_t> pos(ucnt.begin(), ucnt.end() - 1);
  for (int s = 0; s < S.nfront; ++s)
    for (int ci = S.child_ptr[s]; ci < S.child_ptr[s + 1]; ++ci) {
      int ch = S.child_list[ci];
      for (int64_t kk = 0; kk < S.nf[ch] - S.npiv[ch]; ++kk)
        uidx[pos[S.rows_off[s] + S.relmap[S.rel_off[ch] + kk]]++] = S.uvec_off[ch] + kk;
    }
  int64_t *ucp, *uci, *bo;
  if ((rc = upload(c, c->allocs, &ucp, ucnt.data(), ucnt.size()))) return rc;
  if ((rc = upload(c, c->allocs, &uci, uidx.data(), uidx.size()))) return rc;
  if ((rc = upload(c, c->allocs, &bo, blk_off.data(), blk_off.size()))) return rc;
  c->F.ucon_ptr = ucp;
  c->F.ucon_idx = uci;
  c->F.blk_off = bo;
  return RBA_OK;
}

// One lane of the factorisation: its poles, its stream, its share of the Ozaki
// digit buffers (poles [oz0, oz0 + ozn) of the buffer) and its tile ticket.
struct Lane {
  rba::PoleBatch pb;
  cudaStream_t st;
  int oz0, ozn, id;
};

static void run_step(rba_ctx* c, const Step& s, const Lane& ln) {
  const rba::PoleBatch& pb = ln.pb;
  cudaStream_t st = ln.st;
  switch (s.kind) {
    case ST_EA: { Timed t(c, KC_EA); rba::launch_extend_add(st, c->ea_tasks + s.off, s.n, c->F, pb); break; }
    case ST_DIAG: {
      Timed t(c, KC_DIAG, (s.ntiles > 0) + (s.schur > 0) + (s.ntiles + s.schur < s.n));
      if (c->diag_v1)
        rba::launch_diag(st, c->pt_tasks + s.off, s.n, c->F, pb, c->err_d);
      else
        rba::launch_diag2(st, c->pt_tasks + s.off, s.n, c->F, pb, c->err_d, s.ntiles, s.schur);
      break;
    }
    case ST_TRSM: {
      Timed t(c, KC_TRSM);
      if (c->gemm_dfma)
        rba::launch_trsm(st, c->pt_tasks + s.off, s.n, c->F, pb);
      else
        rba::launch_trsm3(st, c->pt_tasks + s.off, s.n, c->F, pb, c->gemm_var);
      break;
    }
    case ST_OZ: {
      Timed t(c, KC_OZ);
      Timed tg(c, 112 + std::min(s.level, 15), 0);
      for (int g0 = 0; g0 < pb.count; g0 += ln.ozn) {
        rba::PoleBatch sub{};
        sub.count = std::min(ln.ozn, pb.count - g0);
        for (int i = 0; i < sub.count; ++i) {
          sub.factor[i] = pb.factor[g0 + i];
          sub.upd[i] = pb.upd[g0 + i];
          sub.tmap[i] = pb.tmap[g0 + i];
          sub.xi[i] = pb.xi[g0 + i];
        }
        c->launches += 1;
        rba::launch_oz_schur(st, c->oz_tasks + s.off, s.n, c->oz_tiles + s.oz_tile_off, s.schur,
                             s.ntiles, c->F, sub,
                             c->oz_buf + (size_t)ln.oz0 * c->oz_split_max, s.oz_split,
                             c->oz_exp + (size_t)ln.oz0 * c->oz_rows_max, s.oz_rows,
                             c->oz_pair ? 3 : (c->oz_wide ? (c->oz_ts ? (c->oz_stages == 5 ? 5 : 4) : (c->oz_stages == 5 ? 2 : 1)) : 0),
                             c->oz_ticket + ln.id);
      }
      break;
    }
    case ST_SSCHUR: {
      Timed t(c, KC_GEMM);
      Timed tg(c, 112 + std::min(s.level, 15), 0);
      rba::launch_schur_small(st, c->ss_fronts + s.off, s.n, c->F, pb);
      break;
    }
    case ST_GEMM: {
      Timed t(c, KC_GEMM);
      Timed tg(c, 112 + std::min(s.level, 15), 0);   // GEMM time per level
      if (!s.schur && c->panel_v > 0) {
        // panel (look-ahead / aggregated) updates: short K, own kernel choice
        if (c->panel_v == 5)
          rba::launch_gemm5(st, c->gm_tasks + s.off, s.n, s.ntiles, c->F, pb, c->zeros, c->panel_var);
        else
          rba::launch_gemm6(st, c->gm_tasks + s.off, s.n, s.ntiles, c->F, pb, c->zeros, c->panel_var);
        break;
      }
      if (c->gemm_dfma)
        rba::launch_gemm_update(st, c->gm_tasks + s.off, s.n, s.ntiles, c->F, pb);
      else if (c->gemm_v == 3)
        rba::launch_gemm3(st, c->gm_tasks + s.off, s.n, s.ntiles, c->F, pb, c->gemm_var);
      else if (c->gemm_v == 5)
        rba::launch_gemm5(st, c->gm_tasks + s.off, s.n, s.ntiles, c->F, pb, c->zeros, c->gemm5_var);
      else
        rba::launch_gemm6(st, c->gm_tasks + s.off, s.n, s.ntiles, c->F, pb, c->zeros, c->gemm5_var);
      break;
    }
  }
}

// The plan, step by step, for one or two lanes (the launches of the lanes are
// interleaved on the host so neither stream's queue runs dry).
int run_plan(rba_ctx* c, const Lane* lanes, int nlanes) {
  for (const Step& s : c->plan) {
    Timed tl(c, 80 + std::min(s.level, 31), 0);   // factor time per level
    for (int l = 0; l < nlanes; ++l) run_step(c, s, lanes[l]);
    CKL();
  }
  return RBA_OK;
}

int check_err(rba_ctx* c, int pole) {
  int h = 0;
  CK(cudaMemcpyAsync(&h, c->err_d, sizeof(int), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  if (h) {
    CK(cudaMemsetAsync(c->err_d, 0, sizeof(int), c->st));
    return fail(RBA_ERR_SOLVE, "factorization of shifted matrix failed: zero or non-finite pivot "
                               "in front " + std::to_string(h - 1) + " (pole " +
                               std::to_string(pole) + ")");
  }
  return RBA_OK;
}

// TMA tensor maps of every front panel of one factor buffer (GEMM v6 with
// RBA_GEMM=v8 / default): the panel is a column-major nf x npiv complex
// matrix = a 2-D FLOAT64 tensor {2*nf, npiv} with row pitch nf*16 bytes.
// Boxes: 66 complex rows (A operand) and 34 (B operand) by G8K columns, so a
// box lands in shared memory with the padded strides the kernel reads
// conflict-free.  Out-of-range rows / columns are zero-filled.
int make_tmaps(rba_ctx* c, const cplx* base, rba::TMap** out, int boxk) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return fail(RBA_ERR_CUDA, "cuTensorMapEncodeTiled not available");
    encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }
  const rba::Symbolic& S = c->sym;
  std::vector<rba::TMap> h((size_t)2 * S.nfront);
  std::memset(h.data(), 0, h.size() * sizeof(rba::TMap));
  for (int s = 0; s < S.nfront; ++s) {
    const int nf = S.nf[s], p = S.npiv[s];
    if (nf <= p || p == 0) {
      // no trailing/Schur GEMM can touch a front without a border unless it
      // has several pivot blocks; encode those too (panel updates)
      if (p <= rba::PB) continue;
    }
    const cuuint64_t dims[2] = {(cuuint64_t)2 * nf, (cuuint64_t)p};
    const cuuint64_t strides[1] = {(cuuint64_t)nf * sizeof(cplx)};
    const cuuint32_t estr[2] = {1, 1};
    for (int w = 0; w < 2; ++w) {
      const cuuint32_t box[2] = {(cuuint32_t)(w == 0 ? 132 : 68), (cuuint32_t)boxk};
      CUresult r = encode(reinterpret_cast<CUtensorMap*>(&h[2 * s + w]), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                          (void*)(base + S.panel_off[s]), dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS)
        return fail(RBA_ERR_CUDA, "cuTensorMapEncodeTiled failed for front " + std::to_string(s) +
                                      " (code " + std::to_string((int)r) + ")");
    }
  }
  int rc;
  if ((rc = upload(c, c->pole_allocs, out, h.data(), h.size()))) return rc;
  return RBA_OK;
}

// k-width of the TMA boxes for the selected tensor-map GEMM variant
// (launch_gemm6: 6 -> 8 columns, 7 -> 12, 8 -> 16)
int tmap_boxk(const rba_ctx* c) {
  const int v = std::max(c->gemm_v == 6 ? c->gemm5_var : 0, c->panel_v == 6 ? c->panel_var : 0);
  return v == 7 ? 12 : v == 8 ? 16 : rba::G8K;
}

int ensure_factor(rba_ctx* c, int l) {
  if (c->factor[l]) return RBA_OK;
  const rba::Symbolic& S = c->sym;
  int rc;
  if ((rc = dalloc(c, c->pole_allocs, &c->factor[l], S.panel_off[S.nfront], &c->mem_factor))) return rc;
  if ((c->gemm_v == 6 && c->gemm5_var >= 6) || (c->panel_v == 6 && c->panel_var >= 6))
    if ((rc = make_tmaps(c, c->factor[l], &c->tmaps[l], tmap_boxk(c)))) return rc;
  return RBA_OK;
}

int ensure_slots(rba_ctx* c) {
  if (!c->factor.empty()) return RBA_OK;
  const int nl = (int)c->local.size();
  if (nl == 0) return RBA_OK;
  const rba::Symbolic& S = c->sym;
  int rc;
  c->factor.assign(nl, nullptr); c->g.assign(nl, nullptr); c->x.assign(nl, nullptr);
  c->tmaps.assign(nl, nullptr);
  c->uvec.assign(nl, nullptr); c->flf.assign(nl, nullptr); c->flb.assign(nl, nullptr);
  c->dnf.assign(nl, nullptr); c->dnb.assign(nl, nullptr);
  c->slot_epoch.assign(nl, 0);
  c->valid.assign(nl, 0);
  c->NRw = c->NRs;
  for (int l = 0; l < nl; ++l) {
    if (!c->lazy && (rc = ensure_factor(c, l))) return rc;
    if ((rc = dalloc(c, c->pole_allocs, &c->g[l], (size_t)c->N * c->NRw, &c->mem_work))) return rc;
    if ((rc = dalloc(c, c->pole_allocs, &c->x[l], (size_t)c->N * c->NRw, &c->mem_work))) return rc;
    if ((rc = dalloc(c, c->pole_allocs, &c->uvec[l], (size_t)std::max<int64_t>(S.uvec_off[S.nfront], 1) * c->NRw, &c->mem_work))) return rc;
    if ((rc = dalloc(c, c->pole_allocs, &c->flf[l], (size_t)c->nblocks + 1, &c->mem_work))) return rc;
    if ((rc = dalloc(c, c->pole_allocs, &c->flb[l], (size_t)c->nblocks + 1, &c->mem_work))) return rc;
    if ((rc = dalloc(c, c->pole_allocs, &c->dnf[l], (size_t)S.nfront + 1, &c->mem_work))) return rc;
    if ((rc = dalloc(c, c->pole_allocs, &c->dnb[l], (size_t)S.nfront + 1, &c->mem_work))) return rc;
    CK(cudaMemsetAsync(c->dnf[l], 0, (S.nfront + 1) * sizeof(int), c->st));
    CK(cudaMemsetAsync(c->dnb[l], 0, (S.nfront + 1) * sizeof(int), c->st));
    CK(cudaMemsetAsync(c->flf[l], 0, (c->nblocks + 1) * sizeof(int), c->st));
    CK(cudaMemsetAsync(c->flb[l], 0, (c->nblocks + 1) * sizeof(int), c->st));
    CK(cudaMemsetAsync(c->g[l], 0, (size_t)c->N * c->NRw * sizeof(cplx), c->st));
  }
  {
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    // more poles per factor launch fill the GPU at the top of the tree;
    // each needs its own update arena
    const size_t need = (size_t)S.upd_total * sizeof(cplx);
    c->fbatch = 1;
    for (int k = 2; k <= 8 && k <= nl; ++k)
      if (fr > k * need + ((size_t)8 << 30)) c->fbatch = k;
    if (const char* e = getenv("RBA_FACTOR_BATCH")) c->fbatch = std::max(1, std::min(atoi(e), nl));
    if (c->lazy) c->fbatch = 1;
    // The receiver Green's functions Z_l (needed between a factorisation and
    // the next one: J v / J^T w) and the update arenas (needed only inside a
    // factorisation) are never live together, so they share one allocation;
    // any factorisation invalidates every Z_l.
    const size_t arenas = (size_t)c->fbatch * S.upd_total;
    const size_t zsz = (size_t)c->N * std::max<int64_t>(c->Mr, 1);
    const size_t zall = (size_t)nl * zsz;
    const size_t extra = zall > arenas ? (zall - arenas) * sizeof(cplx) : 0;
    c->green = c->green_req && !c->lazy && c->Mr > 0 &&
               fr > (size_t)c->fbatch * need + extra + ((size_t)8 << 30);
    cplx* pool = nullptr;
    if ((rc = dalloc(c, c->pole_allocs, &pool, c->green ? std::max(arenas, zall) : arenas, &c->mem_work)))
      return rc;
    c->upd.assign(c->fbatch, nullptr);
    for (int b = 0; b < c->fbatch; ++b) c->upd[b] = pool + (size_t)b * S.upd_total;
    c->Z.assign(nl, nullptr);
    c->green_valid.assign(nl, 0);
    // the J v cell workspace also lives in the pool (not live during a
    // factorisation), past Z when Green mode is on
    {
      const size_t wn = (size_t)nl * c->P * 6 * c->NRs;
      const size_t z0 = c->green ? zall : 0;
      const size_t cap = c->green ? std::max(arenas, zall) : arenas;
      const char* e = getenv("RBA_JVP2");
      c->jvp_w = (z0 + wn <= cap && !(e && std::string(e) == "0")) ? pool + z0 : nullptr;
    }
    if (c->green) {
      // J v row chunks of a fixed 2048 rows: the partial-sum order depends on
      // N only, never on the poles per GPU, so J v is bitwise independent of
      // the GPU count (C4: 324 chunks -> 648 CTAs with 2 poles per GPU)
      c->green_chunks = (int)std::max<int64_t>(1, (c->N + 2047) / 2048);
      for (int l = 0; l < nl; ++l) c->Z[l] = pool + (size_t)l * zsz;
      const size_t nzf = (size_t)(c->nblocks + 1) * ((c->Mr + 31) / 32);
      c->zflags.assign(nl, nullptr);
      c->zepoch.assign(nl, 0);
      for (int l = 0; l < nl; ++l) {
        if ((rc = dalloc(c, c->pole_allocs, &c->zflags[l], nzf, &c->mem_work))) return rc;
        CK(cudaMemsetAsync(c->zflags[l], 0, nzf * sizeof(int), c->st));
      }
      if ((rc = dalloc(c, c->pole_allocs, &c->green_part,
                       (size_t)c->green_chunks * nl * std::max(c->S, 1) * c->Mr, &c->mem_work)))
        return rc;
    }
  }
  if ((rc = dalloc(c, c->pole_allocs, &c->wa, (size_t)nl * std::max(c->S, 1) * std::max<int64_t>(c->Mr, 1), &c->mem_work))) return rc;
  if (c->ozaki && c->oz_split_max > 0) {
    // digit blocks of one Ozaki Schur step for oz_sub poles at a time, sized
    // to the memory left after the factors, arenas and work vectors
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    const size_t margin = (size_t)3 << 29;        // 1.5 GB
    const size_t per = (size_t)c->oz_split_max;
    int sub = fr > margin + per ? (int)((fr - margin) / per) : 1;
    c->oz_sub = std::max(1, std::min(sub, c->fbatch));
    if (const char* e = getenv("RBA_OZ_SUB")) c->oz_sub = std::max(1, std::min(atoi(e), c->fbatch));
    if ((rc = dalloc(c, c->pole_allocs, &c->oz_buf, per * c->oz_sub, &c->mem_work))) return rc;
    if ((rc = dalloc(c, c->pole_allocs, &c->oz_exp, (size_t)c->oz_rows_max * c->oz_sub, &c->mem_work))) return rc;
  }
  std::vector<int32_t> pos(c->local.begin(), c->local.end());
  if ((rc = dalloc(c, c->pole_allocs, &c->pole_of_slot, nl, &c->mem_other))) return rc;
  CK(cudaMemcpyAsync(c->pole_of_slot, pos.data(), nl * sizeof(int32_t), cudaMemcpyHostToDevice, c->st));
  return RBA_OK;
}

// prune_b >= 0: forward sweep only over the fronts on the paths of receiver
// batch prune_b (right-hand sides Q^T e_m are zero elsewhere; see build_prune)
int solve_slots(rba_ctx* c, const std::vector<int>& slots, int NR, int prune_b = -1,
                bool fwd_only = false) {
  const int ns = (int)slots.size();
  if (ns == 0) return RBA_OK;
  rba::SolveBatch b;
  for (int i = 0; i < ns; ++i) {
    int l = slots[i];
    if (!c->valid[l]) return fail(RBA_ERR_CACHE_MISS, "no factorization for pole " +
                                                         std::to_string(c->local[l]));
    b.factor[i] = c->factor[l];
    b.x[i] = c->x[l];
    b.uvec[i] = c->uvec[l];
    b.flags_f[i] = c->flf[l];
    b.flags_b[i] = c->flb[l];
    b.done_f[i] = c->dnf[l];
    b.done_b[i] = c->dnb[l];
  }
  const rba::Symbolic& S = c->sym;
  for (int i = 0; i < ns; ++i) {
    const int l = slots[i];
    if (c->slot_epoch[l] + 1 >= c->epoch_limit) {
      CK(cudaMemsetAsync(c->flf[l], 0, (c->nblocks + 1) * sizeof(int), c->st));
      CK(cudaMemsetAsync(c->flb[l], 0, (c->nblocks + 1) * sizeof(int), c->st));
      CK(cudaMemsetAsync(c->dnf[l], 0, (S.nfront + 1) * sizeof(int), c->st));
      CK(cudaMemsetAsync(c->dnb[l], 0, (S.nfront + 1) * sizeof(int), c->st));
      c->slot_epoch[l] = 0;
    }
    b.epoch[i] = ++c->slot_epoch[l];
  }
  c->epoch++;
  CK(cudaMemsetAsync(c->tickets, 0, (2 * (size_t)S.nlevels + 2) * sizeof(int), c->st));
  if (c->timing) cudaEventRecord(c->ev[0], c->st);
  if (c->fused_sweep) {
    {
      Timed tm(c, KC_FWD);
      rba::launch_solve_level(c->st, true, NR, c->fwd_tasks, (int)c->n_fwd_tasks, ns, c->F, b,
                              c->tickets, c->epoch, c->parent_d, c->need_u_d, true);
    }
    CKL();
    if (c->timing) cudaEventRecord(c->ev[1], c->st);
    {
      Timed tm(c, KC_BWD);
      rba::launch_solve_level(c->st, false, NR, c->bwd_all, (int)c->n_bwd_tasks, ns, c->F, b,
                              c->tickets + 1, c->epoch, c->parent_d, c->need_u_d, true);
    }
    CKL();
  } else {
    // forward sweeps of the large fronts: GEMV tasks of k_fwd, or DMMA GEMM
    // tasks (k_zfwd) with RBA_FWD_GEMM=1
    const bool fgemm = c->fwd_gemm > 0;      // measured neutral at NR = 8 (C5): off by default
    for (int L = 0; L < S.nlevels; ++L) {
      Timed tl(c, 16 + std::min(L, 31), 0);
      const bool pr = prune_b >= 0;
      const auto sl = pr ? c->pr_small_lv[(size_t)prune_b * S.nlevels + L] : c->small_lv[L];
      const auto fl = pr ? c->pr_fwdb_lv[(size_t)prune_b * S.nlevels + L] : c->fwdb_lv[L];
      if (sl.second > 0) {
        Timed tm(c, KC_FWD);
        rba::launch_solve_small(c->st, true, NR, (pr ? c->pr_small : c->small_fronts) + sl.first,
                                sl.second, ns, c->F, b, c->small_mb[L]);
        CKL();
      }
      if (fl.second > 0) {
        Timed tm(c, KC_FWD);
        const int nfr_lv = S.level_ptr[L + 1] - S.level_ptr[L];
        if (fgemm)
          rba::launch_zfwd(c->st, (pr ? c->pr_fwdb : c->fwdb_tasks) + fl.first, fl.second, ns, c->F, b,
                           c->tickets + L, NR);
        else
          rba::launch_solve_level(c->st, true, NR, (pr ? c->pr_fwdb : c->fwdb_tasks) + fl.first,
                                  fl.second, ns, c->F, b, c->tickets + L, c->epoch,
                                  c->parent_d, c->need_u_d, false, nfr_lv <= 2);
        CKL();
      }
    }
    if (c->timing) cudaEventRecord(c->ev[1], c->st);
    // backward sweeps of the large fronts: with 8 right-hand sides as FP64
    // tensor-core GEMM tasks (k_zbwd on x: the block's rows-beyond product
    // L'^T x is a DMMA GEMM with N = 8), else the GEMV tasks of k_bwd
    const bool bgemm = c->bwd_gemm > 0 ? true : c->bwd_gemm == 0 ? false : NR >= 8;
    rba::SlotPtrs xz{};
    for (int i = 0; i < ns; ++i) xz.p[i] = b.x[i];
    for (int L = S.nlevels - 1; L >= 0 && !fwd_only; --L) {
      Timed tl(c, 48 + std::min(L, 31), 0);
      if (c->bwdb_lv[L].second > 0) {
        Timed tm(c, KC_BWD);
        if (bgemm)
          rba::launch_zbwd(c->st, c->bwdb_tasks + c->bwdb_lv[L].first, c->bwdb_lv[L].second, ns, c->F, b,
                           c->tickets + S.nlevels + L, NR, xz);
        else
          rba::launch_solve_level(c->st, false, NR, c->bwdb_tasks + c->bwdb_lv[L].first,
                                  c->bwdb_lv[L].second, ns, c->F, b, c->tickets + S.nlevels + L,
                                  c->epoch, c->parent_d, c->need_u_d, false);
        CKL();
      }
      if (c->small_lv[L].second > 0) {
        Timed tm(c, KC_BWD);
        rba::launch_solve_small(c->st, false, NR, c->small_fronts + c->small_lv[L].first,
                                c->small_lv[L].second, ns, c->F, b, c->small_mb[L]);
        CKL();
      }
    }
  }
  if (c->timing) {
    cudaEventRecord(c->ev[2], c->st);
    cudaEventSynchronize(c->ev[2]);
    float a = 0, bb = 0;
    cudaEventElapsedTime(&a, c->ev[0], c->ev[1]);
    cudaEventElapsedTime(&bb, c->ev[1], c->ev[2]);
    c->t_ms[4] = a;
    c->t_ms[5] = bb;
  }
  c->n_solve += ns;
  return RBA_OK;
}

rba::ElemDev elem(rba_ctx* c) {
  rba::ElemDev E;
  E.N = c->N;
  E.P = c->P;
  E.cell_dofs = c->cell_dofs_p;
  E.mass = c->mass;
  E.expm = c->expm;
  E.dc_ptr = c->dc_ptr;
  E.dc_item = c->dc_item;
  return E;
}

}  // namespace

extern "C" {

const char* rba_last_error(void) { return g_err.c_str(); }
int rba_version(void) { return 1; }

int rba_symbolic_analyze(int64_t n, const int64_t* indptr, const int32_t* indices,
                         const double* coords, int32_t leaf, rba_symbolic** out) {
  if (!out || !indptr || !indices) return fail(RBA_ERR_INVALID, "null argument");
  auto* s = new rba_symbolic();
  std::string e = rba::analyze(n, indptr, indices, coords, leaf, s->S);
  if (!e.empty()) { delete s; return fail(RBA_ERR_INVALID, e); }
  *out = s;
  return RBA_OK;
}

int rba_symbolic_stats(const rba_symbolic* s, int64_t* is, double* ds) {
  if (!s) return fail(RBA_ERR_INVALID, "null symbolic");
  const rba::Symbolic& S = s->S;
  int64_t nb = 0;
  for (int f = 0; f < S.nfront; ++f) nb += (S.npiv[f] + rba::PB - 1) / rba::PB;
  int64_t v[16] = {S.n, S.nfront, S.nlevels, S.nnzL, S.panel_off[S.nfront], S.upd_total,
                   S.uvec_off[S.nfront], S.max_nf, S.max_npiv, nb, 0, 0, 0, 0, 0, 0};
  if (is) memcpy(is, v, sizeof(v));
  if (ds) { ds[0] = S.flops; ds[1] = ds[2] = ds[3] = 0; }
  return RBA_OK;
}

int rba_symbolic_array(const rba_symbolic* s, const char* name, void* out, int64_t cap,
                       int64_t* nbytes) {
  if (!s || !name) return fail(RBA_ERR_INVALID, "null argument");
  const rba::Symbolic& S = s->S;
  const void* src = nullptr;
  int64_t nb = 0;
  auto pick32 = [&](const std::vector<int32_t>& v) { src = v.data(); nb = v.size() * 4; };
  auto pick64 = [&](const std::vector<int64_t>& v) { src = v.data(); nb = v.size() * 8; };
  std::string n(name);
  if (n == "perm") pick32(S.perm);
  else if (n == "first") pick32(S.first);
  else if (n == "npiv") pick32(S.npiv);
  else if (n == "nf") pick32(S.nf);
  else if (n == "parent") pick32(S.parent);
  else if (n == "level") pick32(S.level);
  else if (n == "rows") pick32(S.rows);
  else if (n == "relmap") pick32(S.relmap);
  else if (n == "rows_off") pick64(S.rows_off);
  else if (n == "rel_off") pick64(S.rel_off);
  else if (n == "panel_off") pick64(S.panel_off);
  else if (n == "upd_off") pick64(S.upd_off);
  else return fail(RBA_ERR_INVALID, "unknown symbolic array " + n);
  if (nbytes) *nbytes = nb;
  if (out) {
    if (cap < nb) return fail(RBA_ERR_INVALID, "buffer too small");
    memcpy(out, src, nb);
  }
  return RBA_OK;
}

void rba_symbolic_destroy(rba_symbolic* s) { delete s; }

int rba_mesh_prepare(int64_t N, int64_t P, int32_t k, const int32_t* cell_dofs,
                     const double* mass_local, const int64_t* Kp, const int32_t* Ki,
                     const double* Kx, const double* coords, int32_t leaf, int64_t* out) {
  if (!Kp || !Ki || !Kx || (P > 0 && (!cell_dofs || !mass_local)))
    return fail(RBA_ERR_INVALID, "null argument");
  rba::MeshPrep MP;
  std::string err = rba::prepare_mesh(N, P, k, cell_dofs, mass_local, Kp, Ki, Kx, coords, leaf, MP);
  if (!err.empty()) return fail(RBA_ERR_INVALID, err);
  if (out) {
    out[0] = MP.nnzA;
    out[1] = (int64_t)MP.moff.size();
    out[2] = MP.sym.nfront;
    out[3] = MP.sym.panel_off[MP.sym.nfront];
  }
  return RBA_OK;
}

int rba_ctx_create(int device, void* stream, rba_ctx** out) {
  if (!out) return fail(RBA_ERR_INVALID, "null out");
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(RBA_ERR_INVALID, "bad device index");
  CK(cudaSetDevice(device));
  auto* c = new rba_ctx();
  c->device = device;
  if (stream) {
    c->st = (cudaStream_t)stream;
  } else {
    cudaError_t e = cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking);
    if (e != cudaSuccess) { delete c; return fail(RBA_ERR_CUDA, cudaGetErrorString(e)); }
    c->own_stream = true;
  }
  for (auto& e : c->ev) cudaEventCreate(&e);
  cudaStreamCreateWithFlags(&c->st2, cudaStreamNonBlocking);
  cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming);
  if (cudaMalloc(&c->oz_ticket, 2 * sizeof(int)) != cudaSuccess) { delete c; return fail(RBA_ERR_OOM, "ticket allocation"); }
  cudaMemset(c->oz_ticket, 0, 2 * sizeof(int));
  if (const char* e = getenv("RBA_FACTOR_STREAMS")) c->fstreams = atoi(e) == 2 ? 2 : 1;
  if (const char* e = getenv("RBA_GEMM")) {
    c->gemm_dfma = std::string(e) == "dfma";
    if (std::string(e) == "v3") { c->gemm_v = 3; c->gemm_var = 0; }
    if (std::string(e) == "v4") { c->gemm_v = 3; c->gemm_var = 1; }
    if (std::string(e) == "v5") { c->gemm_v = 5; c->gemm5_var = 0; }
    if (std::string(e) == "v5b") { c->gemm_v = 5; c->gemm5_var = 1; }
    if (std::string(e) == "v6") { c->gemm_v = 6; c->gemm5_var = 0; }
    if (std::string(e) == "v6b") { c->gemm_v = 6; c->gemm5_var = 1; }
    if (std::string(e) == "v6c") { c->gemm_v = 6; c->gemm5_var = 2; }
    if (std::string(e) == "v6d") { c->gemm_v = 6; c->gemm5_var = 3; }
    if (std::string(e) == "v7") { c->gemm_v = 6; c->gemm5_var = 4; }
    if (std::string(e) == "v7b") { c->gemm_v = 6; c->gemm5_var = 5; }
    if (std::string(e) == "v8") { c->gemm_v = 6; c->gemm5_var = 6; }
    if (std::string(e) == "v8b") { c->gemm_v = 6; c->gemm5_var = 7; }
    if (std::string(e) == "v8c") { c->gemm_v = 6; c->gemm5_var = 8; }
  }
  if (const char* e = getenv("RBA_GEMM_PANEL")) {
    const std::string v(e);
    const char* names[] = {"v6", "v6b", "v6c", "v6d", "v7", "v7b", "v8"};
    for (int q = 0; q < 7; ++q)
      if (v == names[q]) { c->panel_v = 6; c->panel_var = q; }
    if (v == "v5") { c->panel_v = 5; c->panel_var = 0; }
    // the per-front tensor maps have one box width: two tensor-map variants
    // with different boxes cannot share them -> the panel updates follow RBA_GEMM
    auto boxk = [](int var) { return var == 7 ? 12 : var == 8 ? 16 : var == 6 ? 8 : 0; };
    if (c->panel_v == 6 && c->gemm_v == 6 && boxk(c->panel_var) && boxk(c->gemm5_var) &&
        boxk(c->panel_var) != boxk(c->gemm5_var))
      c->panel_v = 0;
  }
  if (const char* e = getenv("RBA_GREEN")) c->green_req = std::string(e) != "0";
  if (const char* e = getenv("RBA_TRSM_VAR")) c->gemm_var = atoi(e) ? 1 : 0;
  if (const char* e = getenv("RBA_GREEN_PRUNE")) c->green_prune = std::string(e) != "0";
  if (const char* e = getenv("RBA_GREEN_GEMM")) c->green_gemm = std::string(e) != "0";
  if (const char* e = getenv("RBA_SWEEP")) c->fused_sweep = std::string(e) == "fused";
  if (const char* e = getenv("RBA_SMALLP")) c->small_p = std::string(e) == "64" ? rba::PB : 2 * rba::PB;
  if (const char* e = getenv("RBA_DIAG")) c->diag_v1 = std::string(e) == "v1";
  if (const char* e = getenv("RBA_BWD_GEMM")) c->bwd_gemm = atoi(e) ? 1 : 0;
  if (const char* e = getenv("RBA_FWD_GEMM")) c->fwd_gemm = atoi(e) ? 1 : 0;
  rba::solve_env_refresh();
  if (const char* e = getenv("RBA_OZAKI")) c->ozaki = std::string(e) != "0";
  if (const char* e = getenv("RBA_OZ_MINK")) c->oz_min_k = std::max(16, atoi(e));
  if (const char* e = getenv("RBA_OZ_TRAIL")) c->oz_trail = std::string(e) != "0";
  if (const char* e = getenv("RBA_OZ_KMAX")) c->oz_kmax = std::max(64, atoi(e) / 16 * 16);
  if (const char* e = getenv("RBA_SCHUR_SMALL")) c->schur_small = std::string(e) != "0";
  if (const char* e = getenv("RBA_SCHUR_SMALL_B")) c->schur_small_b = std::max(8, atoi(e));
  if (const char* e = getenv("RBA_OZ_TS")) c->oz_ts = std::string(e) == "1";
  if (const char* e = getenv("RBA_OZ_2CTA")) c->oz_pair = std::string(e) == "1";
  if (const char* e = getenv("RBA_OZ_WIDE")) c->oz_wide = std::string(e) != "0";
  if (const char* e = getenv("RBA_OZ_STAGES")) c->oz_stages = atoi(e) == 4 ? 4 : 5;
  if (const char* e = getenv("RBA_OZ_MINROWS")) c->oz_min_rows = std::max(64, atoi(e));
  int rc;
  if ((rc = dalloc(c, c->allocs, &c->err_d, 1, &c->mem_other)) ||
      (rc = dalloc(c, c->allocs, &c->red_part, 1024, &c->mem_other)) ||
      (rc = dalloc(c, c->allocs, &c->red_res, 8, &c->mem_other)) ||
      (rc = dalloc(c, c->allocs, &c->zeros, 64, &c->mem_other))) {
    rba_ctx_destroy(c);
    return rc;
  }
  cudaMemsetAsync(c->err_d, 0, sizeof(int), c->st);
  cudaMemsetAsync(c->zeros, 0, 64 * sizeof(cplx), c->st);
  *out = c;
  return RBA_OK;
}

void rba_ctx_destroy(rba_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->st) cudaStreamSynchronize(c->st);
  free_slots(c);
  free_list(c->obs_allocs);
  free_list(c->reg_allocs);
  free_list(c->regl_allocs);
  free_list(c->allocs);
  if (c->stage) cudaFree(c->stage);
  for (auto& e : c->ev) if (e) cudaEventDestroy(e);
  if (c->own_stream && c->st) cudaStreamDestroy(c->st);
  if (c->st2) cudaStreamDestroy(c->st2);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->oz_ticket) cudaFree(c->oz_ticket);
  delete c;
}

int rba_set_mesh(rba_ctx* c, int64_t N, int64_t P, int32_t k, const int32_t* cell_dofs,
                 const double* mass_local, const int64_t* Kp, const int32_t* Ki, const double* Kx,
                 const double* coords, int32_t leaf) {
  if (!c || !Kp || !Ki || !Kx || (P > 0 && (!cell_dofs || !mass_local)))
    return fail(RBA_ERR_INVALID, "null argument");
  if (N <= 0 || P < 0 || k <= 0 || k > 6) return fail(RBA_ERR_INVALID, "bad mesh sizes");
  if (c->have_mesh) return fail(RBA_ERR_STATE, "mesh already set on this context");
  CK(cudaSetDevice(c->device));
  c->N = N; c->P = P; c->k = k;
  rba::MeshPrep MP;
  {
    std::string err = rba::prepare_mesh(N, P, k, cell_dofs, mass_local, Kp, Ki, Kx, coords, leaf, MP);
    if (!err.empty()) return fail(RBA_ERR_INVALID, err);
  }
  c->sym = std::move(MP.sym);
  c->a_rows = std::move(MP.a_rows);
  c->a_cols = std::move(MP.a_cols);
  c->Kv_h = std::move(MP.Kv);
  c->nnzA = MP.nnzA;
  const rba::Symbolic& S = c->sym;
  std::vector<int64_t>& tgt = MP.tgt;
  std::vector<int64_t>& mcnt = MP.mcnt;
  std::vector<int64_t>& moff = MP.moff;
  std::vector<int32_t>& cdp = MP.cdp;
  std::vector<double>& mass36 = MP.mass36;
  std::vector<int64_t>& pdcp = MP.pdcp;
  std::vector<int32_t>& pdci = MP.pdci;
  // uploads
  int rc;
  auto up32 = [&](int32_t** d, const std::vector<int32_t>& v) { return upload(c, c->allocs, d, v.data(), v.size()); };
  auto up64 = [&](int64_t** d, const std::vector<int64_t>& v) { return upload(c, c->allocs, d, v.data(), v.size()); };
  int32_t *d_first, *d_npiv, *d_nf, *d_rows, *d_cp, *d_cl, *d_rel;
  int64_t *d_po, *d_uo, *d_ro, *d_relo, *d_uvo;
  if ((rc = up32(&d_first, S.first)) || (rc = up32(&d_npiv, S.npiv)) || (rc = up32(&d_nf, S.nf)) ||
      (rc = up32(&d_rows, S.rows)) || (rc = up32(&d_cp, S.child_ptr)) ||
      (rc = up32(&d_cl, S.child_list)) || (rc = up32(&d_rel, S.relmap)) ||
      (rc = up64(&d_po, S.panel_off)) || (rc = up64(&d_uo, S.upd_off)) ||
      (rc = up64(&d_ro, S.rows_off)) || (rc = up64(&d_relo, S.rel_off)) ||
      (rc = up64(&d_uvo, S.uvec_off)))
    return rc;
  c->F.first = d_first; c->F.npiv = d_npiv; c->F.nf = d_nf; c->F.rows = d_rows;
  c->F.child_ptr = d_cp; c->F.child_list = d_cl; c->F.relmap = d_rel;
  c->F.panel_off = d_po; c->F.upd_off = d_uo; c->F.rows_off = d_ro; c->F.rel_off = d_relo;
  c->F.uvec_off = d_uvo;
  if ((rc = upload(c, c->allocs, &c->Kv, c->Kv_h.data(), c->Kv_h.size())) ||
      (rc = dalloc(c, c->allocs, &c->Mv, c->nnzA, &c->mem_other)) ||
      (rc = up64(&c->tgt, tgt)) || (rc = up64(&c->cptr, mcnt)) || (rc = up64(&c->coff, moff)) ||
      (rc = upload(c, c->allocs, &c->mass, mass36.data(), mass36.size())) ||
      (rc = dalloc(c, c->allocs, &c->mdev, P, &c->mem_other)) ||
      (rc = dalloc(c, c->allocs, &c->expm, P, &c->mem_other)) ||
      (rc = up32(&c->cell_dofs_p, cdp)) || (rc = up64(&c->dc_ptr, pdcp)) ||
      (rc = up32(&c->dc_item, pdci)) || (rc = up32(&c->perm_d, S.perm)))
    return rc;
  if ((rc = build_plans(c))) return rc;
  CK(cudaStreamSynchronize(c->st));
  c->have_mesh = true;
  return RBA_OK;
}

int rba_set_observation(rba_ctx* c, int64_t Mr, const int64_t* qp, const int32_t* qi,
                        const double* qx) {
  if (!c || !c->have_mesh) return fail(RBA_ERR_STATE, "set_mesh first");
  if (Mr < 0 || (Mr > 0 && (!qp || !qi || !qx))) return fail(RBA_ERR_INVALID, "bad Q");
  CK(cudaSetDevice(c->device));
  free_list(c->obs_allocs);
  free_slots(c);
  c->Mr = Mr;
  const rba::Symbolic& S = c->sym;
  int64_t nnz = Mr > 0 ? qp[Mr] : 0;
  std::vector<int64_t> ptr(qp, qp + Mr + 1);
  if (Mr == 0) ptr.assign(1, 0);
  std::vector<int32_t> col(nnz);
  std::vector<double> val(qx, qx + nnz);
  for (int64_t e = 0; e < nnz; ++e) {
    if (qi[e] < 0 || qi[e] >= c->N) return fail(RBA_ERR_INVALID, "Q index out of range");
    col[e] = S.iperm[qi[e]];
  }
  std::vector<int64_t> tp(c->N + 1, 0);
  for (int64_t e = 0; e < nnz; ++e) tp[col[e] + 1]++;
  for (int64_t i = 0; i < c->N; ++i) tp[i + 1] += tp[i];
  std::vector<int32_t> tc(nnz);
  std::vector<double> tv(nnz);
  {
    std::vector<int64_t> pos(tp.begin(), tp.end() - 1);
    for (int64_t r = 0; r < Mr; ++r)
      for (int64_t e = ptr[r]; e < ptr[r + 1]; ++e) {
        int64_t q = pos[col[e]]++;
        tc[q] = (int32_t)r;
        tv[q] = val[e];
      }
  }
  int rc;
  if ((rc = upload(c, c->obs_allocs, &c->q_ptr, ptr.data(), ptr.size())) ||
      (rc = upload(c, c->obs_allocs, &c->q_col, col.data(), col.size())) ||
      (rc = upload(c, c->obs_allocs, &c->q_val, val.data(), val.size())) ||
      (rc = upload(c, c->obs_allocs, &c->qt_ptr, tp.data(), tp.size())) ||
      (rc = upload(c, c->obs_allocs, &c->qt_col, tc.data(), tc.size())) ||
      (rc = upload(c, c->obs_allocs, &c->qt_val, tv.data(), tv.size())))
    return rc;
  c->S = 0;       // sources live in obs_allocs: set them again
  c->Fsrc = nullptr;
  c->q_ptr_h = ptr;
  c->q_col_h = col;
  c->prune_nb = 0;
  return RBA_OK;
}

int rba_set_sources(rba_ctx* c, int32_t S_, const double* F) {
  if (!c || !c->have_mesh) return fail(RBA_ERR_STATE, "set_mesh first");
  if (S_ < 1 || S_ > 8 || !F) return fail(RBA_ERR_INVALID, "1 <= S <= 8 sources required");
  if (!c->q_ptr) return fail(RBA_ERR_STATE, "set_observation first");
  CK(cudaSetDevice(c->device));
  free_slots(c);
  c->S = S_;
  c->NRs = nr_pad(S_);
  std::vector<cplx> h((size_t)c->N * c->NRs, rba::cmk(0.0, 0.0));
  for (int64_t kk = 0; kk < c->N; ++kk) {
    int32_t o = c->sym.perm[kk];
    for (int s = 0; s < S_; ++s) h[kk * c->NRs + s] = rba::cmk(F[(int64_t)s * c->N + o], 0.0);
  }
  return upload(c, c->obs_allocs, &c->Fsrc, h.data(), h.size());
}

int rba_set_sources_complex(rba_ctx* c, int32_t S_, const double* F) {
  if (!c || !c->have_mesh) return fail(RBA_ERR_STATE, "set_mesh first");
  if (S_ < 1 || S_ > 8 || !F) return fail(RBA_ERR_INVALID, "1 <= S <= 8 sources required");
  if (!c->q_ptr) return fail(RBA_ERR_STATE, "set_observation first");
  CK(cudaSetDevice(c->device));
  free_slots(c);
  c->S = S_;
  c->NRs = nr_pad(S_);
  const cplx* Fc = (const cplx*)F;
  std::vector<cplx> h((size_t)c->N * c->NRs, rba::cmk(0.0, 0.0));
  for (int64_t kk = 0; kk < c->N; ++kk) {
    int32_t o = c->sym.perm[kk];
    for (int s = 0; s < S_; ++s) h[kk * c->NRs + s] = Fc[(int64_t)s * c->N + o];
  }
  return upload(c, c->obs_allocs, &c->Fsrc, h.data(), h.size());
}

int rba_set_poles(rba_ctx* c, int32_t m, const double* poles, int32_t Kt, const double* res,
                  int32_t nl, const int32_t* local) {
  if (!c || !c->have_mesh) return fail(RBA_ERR_STATE, "set_mesh first");
  if (m < 1 || Kt < 1 || !poles || !res || nl < 0 || nl > 32 || (nl > 0 && !local))
    return fail(RBA_ERR_INVALID, "bad poles (need 1 <= m, 0 <= n_local <= 32)");
  if (c->S < 1) return fail(RBA_ERR_STATE, "set_sources first");
  CK(cudaSetDevice(c->device));
  free_slots(c);
  c->m = m;
  c->Kt = Kt;
  c->poles_h.assign((const cplx*)poles, (const cplx*)poles + m);
  c->res_h.assign((const cplx*)res, (const cplx*)res + (size_t)m * Kt);
  c->local.assign(local, local + nl);
  for (int l : c->local)
    if (l < 0 || l >= m) return fail(RBA_ERR_INVALID, "local pole index out of range");
  int rc;
  if ((rc = upload(c, c->pole_allocs, &c->poles_d, c->poles_h.data(), c->poles_h.size())) ||
      (rc = upload(c, c->pole_allocs, &c->res_d, c->res_h.data(), c->res_h.size())) ||
      (rc = dalloc(c, c->pole_allocs, &c->slot_map, (size_t)m, &c->mem_other)))
    return rc;
  return ensure_slots(c);
}

int rba_set_model_d(rba_ctx* c, const double* m_d) {
  if (!c || !c->have_mesh) return fail(RBA_ERR_STATE, "set_mesh first");
  CK(cudaSetDevice(c->device));
  if (m_d != c->mdev) CK(cudaMemcpyAsync(c->mdev, m_d, c->P * sizeof(double), cudaMemcpyDeviceToDevice, c->st));
  {
    Timed t(c, KC_ASSEMBLY, 2);
    rba::launch_assemble_M(c->st, c->nnzA, c->cptr, c->coff, c->mass, c->mdev, c->expm, c->P, 36, c->Mv);
  }
  CKL();
  for (auto& v : c->valid) v = 0;
  for (auto& v : c->green_valid) v = 0;   // Z_i belong to the previous model
  c->model_set = true;
  return RBA_OK;
}

int rba_set_model(rba_ctx* c, const double* m_h) {
  if (!c || !c->have_mesh || !m_h) return fail(RBA_ERR_STATE, "set_mesh first");
  CK(cudaSetDevice(c->device));
  CK(cudaMemcpyAsync(c->mdev, m_h, c->P * sizeof(double), cudaMemcpyHostToDevice, c->st));
  int rc = rba_set_model_d(c, c->mdev);
  if (rc) return rc;
  CK(cudaStreamSynchronize(c->st));   // m_h is only borrowed for the call
  return RBA_OK;
}

int rba_factor(rba_ctx* c) {
  if (!c || !c->model_set) return fail(RBA_ERR_STATE, "set_model first");
  if (c->local.empty()) return RBA_OK;
  CK(cudaSetDevice(c->device));
  int rc;
  if ((rc = ensure_slots(c))) return rc;
  const rba::Symbolic& S = c->sym;
  const int nl = (int)c->local.size();
  if (c->timing) cudaEventRecord(c->ev[0], c->st);
  for (auto& v : c->green_valid) v = 0;   // the update arenas overlay Z
  for (int b0 = 0; b0 < nl; b0 += c->fbatch) {
    const int count = std::min(c->fbatch, nl - b0);
    // two lanes when nothing is being timed per launch (the Timed events sit on
    // the main stream) and every lane gets a pole and a share of the digit buffers
    const bool dual = c->fstreams == 2 && !c->timing && count >= 2 && (!c->ozaki || c->oz_sub >= 2);
    Lane lanes[2];
    const int nlanes = dual ? 2 : 1;
    const int half = dual ? (count + 1) / 2 : count;
    for (int l = 0; l < nlanes; ++l) {
      Lane& ln = lanes[l];
      ln.id = l;
      ln.st = l == 0 ? c->st : c->st2;
      const int ozh = dual ? c->oz_sub / 2 : c->oz_sub;
      ln.oz0 = l * ozh;
      ln.ozn = std::max(1, dual && l == 1 ? c->oz_sub - ozh : ozh);
      ln.pb = rba::PoleBatch{};
      ln.pb.count = l == 0 ? half : count - half;
    }
    if (dual) {
      CK(cudaEventRecord(c->ev_fork, c->st));
      CK(cudaStreamWaitEvent(c->st2, c->ev_fork, 0));
    }
    for (int i = 0; i < count; ++i) {
      int l = b0 + i;
      if ((rc = ensure_factor(c, l))) return rc;
      c->valid[l] = 0;
      Lane& ln = lanes[i < half ? 0 : 1];
      const int k = i < half ? i : i - half;
      ln.pb.factor[k] = c->factor[l];
      ln.pb.tmap[k] = c->tmaps[l];
      ln.pb.upd[k] = c->upd[i];
      ln.pb.xi[k] = c->poles_h[c->local[l]];
      CK(cudaMemsetAsync(c->factor[l], 0, S.panel_off[S.nfront] * sizeof(cplx), ln.st));
    }
    for (int l = 0; l < nlanes; ++l) {
      Timed t(c, KC_SCATTER);
      rba::launch_scatter_A(lanes[l].st, c->nnzA, c->tgt, c->Kv, c->Mv, lanes[l].pb);
    }
    CKL();
    if ((rc = run_plan(c, lanes, nlanes))) return rc;
    if (dual) {
      CK(cudaEventRecord(c->ev_join, c->st2));
      CK(cudaStreamWaitEvent(c->st, c->ev_join, 0));
    }
    if ((rc = check_err(c, c->local[b0]))) return rc;
    for (int i = 0; i < count; ++i) c->valid[b0 + i] = 1;
    c->n_fact += count;
  }
  if (c->timing) {
    cudaEventRecord(c->ev[1], c->st);
    cudaEventSynchronize(c->ev[1]);
    float a = 0;
    cudaEventElapsedTime(&a, c->ev[0], c->ev[1]);
    c->t_ms[0] = a;
  }
  return RBA_OK;
}

int rba_factor_values(rba_ctx* c, int32_t slot, const double* vals) {
  if (!c || !c->have_mesh || !vals) return fail(RBA_ERR_STATE, "set_mesh first");
  if (slot < 0 || slot >= (int)c->local.size()) return fail(RBA_ERR_INVALID, "bad slot");
  CK(cudaSetDevice(c->device));
  int rc;
  if ((rc = ensure_slots(c))) return rc;
  if ((rc = ensure_stage(c, c->nnzA))) return rc;
  if ((rc = ensure_factor(c, slot))) return rc;
  const rba::Symbolic& S = c->sym;
  CK(cudaMemcpyAsync(c->stage, vals, c->nnzA * sizeof(cplx), cudaMemcpyHostToDevice, c->st));
  CK(cudaMemsetAsync(c->factor[slot], 0, S.panel_off[S.nfront] * sizeof(cplx), c->st));
  rba::launch_scatter_vals(c->st, c->nnzA, c->tgt, c->stage, c->factor[slot]);
  CKL();
  rba::PoleBatch pb;
  pb.count = 1;
  pb.factor[0] = c->factor[slot];
  pb.tmap[0] = c->tmaps[slot];
  pb.upd[0] = c->upd[0];
  pb.xi[0] = rba::cmk(0.0, 0.0);
  c->valid[slot] = 0;
  for (auto& v : c->green_valid) v = 0;   // the update arenas overlay Z
  Lane ln{pb, c->st, 0, std::max(1, c->oz_sub), 0};
  if ((rc = run_plan(c, &ln, 1))) return rc;
  if ((rc = check_err(c, c->local[slot]))) return rc;
  c->valid[slot] = 1;
  c->n_fact += 1;
  return RBA_OK;
}

int rba_pattern(rba_ctx* c, int64_t* nnz, int32_t* rows, int32_t* cols, double* Kh, double* Mh) {
  if (!c || !c->have_mesh) return fail(RBA_ERR_STATE, "set_mesh first");
  if (nnz) *nnz = c->nnzA;
  if (rows) memcpy(rows, c->a_rows.data(), c->nnzA * 4);
  if (cols) memcpy(cols, c->a_cols.data(), c->nnzA * 4);
  if (Kh) memcpy(Kh, c->Kv_h.data(), c->nnzA * 8);
  if (Mh) {
    if (!c->model_set) return fail(RBA_ERR_STATE, "set_model first");
    CK(cudaMemcpyAsync(Mh, c->Mv, c->nnzA * 8, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
  }
  return RBA_OK;
}

static int solve_common(rba_ctx* c, int32_t slot, const cplx* rhs_d, cplx* out_d, int32_t nrhs) {
  if (slot < 0 || slot >= (int)c->local.size()) return fail(RBA_ERR_INVALID, "bad slot");
  if (!c->valid[slot]) return fail(RBA_ERR_CACHE_MISS, "no factorization for pole " +
                                                         std::to_string(c->local[slot]));
  int rc;
  for (int r0 = 0; r0 < nrhs; r0 += c->NRw) {
    int nr = std::min(c->NRw, nrhs - r0);
    rba::launch_perm_in(c->st, c->N, nr, c->NRw, c->perm_d, rhs_d + (int64_t)r0 * c->N, c->N, c->x[slot]);
    CKL();
    if ((rc = solve_slots(c, {slot}, c->NRw))) return rc;
    rba::launch_perm_out(c->st, c->N, nr, c->NRw, c->perm_d, c->x[slot], out_d + (int64_t)r0 * c->N, c->N);
    CKL();
  }
  return RBA_OK;
}

// trans: 0 'N', 1 'T' (A complex symmetric: A^T = A, same solve), 2 'H'
// (A^{-H} b = conj(A^{-1} conj(b))); anything else is invalid.
int rba_solve_d(rba_ctx* c, int32_t slot, const double* rhs_d, double* out_d, int32_t nrhs,
                int32_t trans) {
  if (!c || !rhs_d || !out_d || nrhs < 1) return fail(RBA_ERR_INVALID, "bad arguments");
  if (trans < 0 || trans > 2) return fail(RBA_ERR_INVALID, "trans must be 'N', 'T' or 'H'");
  CK(cudaSetDevice(c->device));
  if (trans != 2) return solve_common(c, slot, (const cplx*)rhs_d, (cplx*)out_d, nrhs);
  const int64_t n = c->N * (int64_t)nrhs;
  int rc;
  if ((rc = ensure_stage(c, n))) return rc;
  rba::launch_conj(c->st, n, (const cplx*)rhs_d, c->stage);
  CKL();
  if ((rc = solve_common(c, slot, c->stage, (cplx*)out_d, nrhs))) return rc;
  rba::launch_conj(c->st, n, (const cplx*)out_d, (cplx*)out_d);
  CKL();
  return RBA_OK;
}

int rba_solve(rba_ctx* c, int32_t slot, const double* rhs_h, double* out_h, int32_t nrhs,
              int32_t trans) {
  if (!c || !rhs_h || !out_h || nrhs < 1) return fail(RBA_ERR_INVALID, "bad arguments");
  if (trans < 0 || trans > 2) return fail(RBA_ERR_INVALID, "trans must be 'N', 'T' or 'H'");
  CK(cudaSetDevice(c->device));
  int rc;
  const int64_t n = c->N * (int64_t)nrhs;
  if ((rc = ensure_stage(c, 2 * n))) return rc;
  CK(cudaMemcpyAsync(c->stage, rhs_h, n * sizeof(cplx), cudaMemcpyHostToDevice, c->st));
  if (trans == 2) rba::launch_conj(c->st, n, c->stage, c->stage);
  if ((rc = solve_common(c, slot, c->stage, c->stage + n, nrhs))) return rc;
  if (trans == 2) rba::launch_conj(c->st, n, c->stage + n, c->stage + n);
  CK(cudaMemcpyAsync(out_h, c->stage + n, n * sizeof(cplx), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  return RBA_OK;
}

static std::vector<int> all_slots(rba_ctx* c) {
  std::vector<int> v(c->local.size());
  std::iota(v.begin(), v.end(), 0);
  return v;
}

static rba::SlotPtrs slot_ptrs(const std::vector<cplx*>& v) {
  rba::SlotPtrs p;
  for (size_t i = 0; i < v.size() && i < 32; ++i) p.p[i] = v[i];
  return p;
}

int rba_forward_partial(rba_ctx* c, double* qpart) {
  if (!c || !c->model_set) return fail(RBA_ERR_STATE, "set_model first");
  CK(cudaSetDevice(c->device));
  const int nl = (int)c->local.size();
  for (int l = 0; l < nl; ++l)
    CK(cudaMemcpyAsync(c->x[l], c->Fsrc, (size_t)c->N * c->NRs * sizeof(cplx), cudaMemcpyDeviceToDevice, c->st));
  int rc;
  if ((rc = solve_slots(c, all_slots(c), c->NRs))) return rc;
  for (int l = 0; l < nl; ++l)
    CK(cudaMemcpyAsync(c->g[l], c->x[l], (size_t)c->N * c->NRs * sizeof(cplx), cudaMemcpyDeviceToDevice, c->st));
  if (qpart && c->Mr > 0) {
    Timed t(c, KC_ELEM);
    rba::launch_q_apply(c->st, nl, c->Mr, c->q_ptr, c->q_col, c->q_val, slot_ptrs(c->g), c->NRs, c->S, (cplx*)qpart);
    CKL();
  }
  return RBA_OK;
}

static rba::SlotPtrs slot_sub(const std::vector<cplx*>& v, const std::vector<int>& slots) {
  rba::SlotPtrs p;
  for (size_t i = 0; i < slots.size() && i < 32; ++i) p.p[i] = v[slots[i]];
  return p;
}

// Forward-sweep pruning for the Z build: the right-hand sides of receiver
// batch b (columns m0..m0+nb of Q^T) are nonzero only in the fronts holding
// those receivers' dofs, so L^{-1} Q^T is nonzero only on the paths from those
// fronts to the root (C4: ~25% of the factor bytes per batch of 4).
static int build_prune(rba_ctx* c, int nb) {
  const rba::Symbolic& S = c->sym;
  std::vector<int32_t> fr_of(c->N, -1);
  for (int s = 0; s < S.nfront; ++s)
    for (int k = 0; k < S.npiv[s]; ++k) fr_of[S.first[s] + k] = s;
  const int nbat = (int)((c->Mr + nb - 1) / nb);
  std::vector<int32_t> ps;
  std::vector<rba::SolveTask> pf;
  c->pr_small_lv.assign((size_t)nbat * S.nlevels, {0, 0});
  c->pr_fwdb_lv.assign((size_t)nbat * S.nlevels, {0, 0});
  std::vector<char> act(S.nfront);
  for (int b = 0; b < nbat; ++b) {
    std::fill(act.begin(), act.end(), 0);
    for (int64_t m = (int64_t)b * nb; m < std::min<int64_t>(c->Mr, (int64_t)(b + 1) * nb); ++m)
      for (int64_t e = c->q_ptr_h[m]; e < c->q_ptr_h[m + 1]; ++e)
        for (int s = fr_of[c->q_col_h[e]]; s >= 0 && !act[s]; s = S.parent[s]) act[s] = 1;
    for (int L = 0; L < S.nlevels; ++L) {
      const int64_t o1 = ps.size(), o2 = pf.size();
      for (int q = 0; q < c->small_lv[L].second; ++q) {
        const int32_t f = c->smallf_h[c->small_lv[L].first + q];
        if (act[f]) ps.push_back(f);
      }
      for (int q = 0; q < c->fwdb_lv[L].second; ++q) {
        const rba::SolveTask t = c->ftb_h[c->fwdb_lv[L].first + q];
        if (act[t.s]) pf.push_back(t);
      }
      c->pr_small_lv[(size_t)b * S.nlevels + L] = {o1, (int)(ps.size() - o1)};
      c->pr_fwdb_lv[(size_t)b * S.nlevels + L] = {o2, (int)(pf.size() - o2)};
    }
  }
  int rc;
  if (ps.empty()) ps.push_back(0);   // keep the device lists non-empty
  if (pf.empty()) pf.push_back({0, 0});
  if ((rc = upload(c, c->obs_allocs, &c->pr_small, ps.data(), ps.size()))) return rc;
  if ((rc = upload(c, c->obs_allocs, &c->pr_fwdb, pf.data(), pf.size()))) return rc;
  c->prune_nb = nb;
  return RBA_OK;
}

// Build Z = A^{-1} Q^T for every local slot whose factor changed: Mr/NRw
// multi-RHS solves over all such slots at once, columns stored row-major.
static int ensure_green(rba_ctx* c) {
  std::vector<int> slots;
  for (int l = 0; l < (int)c->local.size(); ++l)
    if (!c->green_valid[l]) {
      if (!c->valid[l]) return fail(RBA_ERR_CACHE_MISS, "no factorization for pole " +
                                                           std::to_string(c->local[l]));
      slots.push_back(l);
    }
  if (slots.empty()) return RBA_OK;
  const int ns = (int)slots.size(), nb = c->NRw;
  const rba::SlotPtrs xs = slot_sub(c->x, slots), zs = slot_sub(c->Z, slots);
  int rc;
  const bool prune = !c->fused_sweep && c->green_prune;
  const bool zg = !c->fused_sweep && c->green_gemm;
  if (prune && c->prune_nb != nb && (rc = build_prune(c, nb))) return rc;
  const rba::Symbolic& S = c->sym;
  const size_t uvn = (size_t)std::max<int64_t>(S.uvec_off[S.nfront], 1) * c->NRw;
  for (int64_t m0 = 0; m0 < c->Mr; m0 += nb) {
    const int n = (int)std::min<int64_t>(nb, c->Mr - m0);
    if (prune)   // skipped fronts must contribute zero u-vectors to active parents
      for (int l : slots) CK(cudaMemsetAsync(c->uvec[l], 0, uvn * sizeof(cplx), c->st));
    {
      Timed t(c, KC_GREEN);
      rba::launch_green_rhs(c->st, ns, c->N, m0, n, nb, c->qt_ptr, c->qt_col, c->qt_val, xs);
    }
    CKL();
    // forward sweep only (y' = L'^{-1} Q^T); the backward runs once over all
    // receivers below, unless RBA_GREEN_GEMM=0
    if ((rc = solve_slots(c, slots, nb, prune ? (int)(m0 / nb) : -1, zg))) return rc;
    {
      Timed t(c, KC_GREEN);
      rba::launch_green_store(c->st, ns, c->N, c->Mr, m0, n, nb, xs, zs);
    }
    CKL();
  }
  if (zg) {
    // Z := L'^{-T} Z, level by level from the root, all receivers per task
    rba::SolveBatch b;
    for (int i = 0; i < ns; ++i) {
      const int l = slots[i];
      b.factor[i] = c->factor[l];
      b.x[i] = c->x[l];
      b.uvec[i] = c->uvec[l];
      b.flags_f[i] = nullptr;
      b.flags_b[i] = c->zflags[l];
      b.done_f[i] = nullptr;
      b.done_b[i] = nullptr;
      if (c->zepoch[l] + 1 >= (1 << 30)) {
        CK(cudaMemsetAsync(c->zflags[l], 0, (size_t)(c->nblocks + 1) * ((c->Mr + 31) / 32) * sizeof(int), c->st));
        c->zepoch[l] = 0;
      }
      b.epoch[i] = ++c->zepoch[l];
    }
    CK(cudaMemsetAsync(c->tickets, 0, (2 * (size_t)S.nlevels + 2) * sizeof(int), c->st));
    for (int L = S.nlevels - 1; L >= 0; --L) {
      Timed t(c, KC_GREEN);
      rba::launch_zbwd(c->st, c->bwd_tasks + c->bwd_lv[L].first, c->bwd_lv[L].second, ns, c->F, b,
                       c->tickets + S.nlevels + L, (int)c->Mr, zs);
      CKL();
    }
  }
  for (int l : slots) c->green_valid[l] = 1;
  c->n_green += ns;
  return RBA_OK;
}

int rba_jvp_partial(rba_ctx* c, const double* v_d, double* qpart) {
  if (!c || !c->model_set || !v_d || !qpart) return fail(RBA_ERR_STATE, "bad state/arguments");
  CK(cudaSetDevice(c->device));
  const int nl = (int)c->local.size();
  int rc;
  if (c->green && (rc = ensure_green(c))) return rc;
  {
    Timed t(c, KC_ELEM, c->jvp_w ? 2 : 1);
    if (c->jvp_w)
      rba::launch_jvp_rhs2(c->st, nl, elem(c), v_d, slot_ptrs(c->g), slot_ptrs(c->x), c->NRs, c->S,
                           c->jvp_w);
    else
      rba::launch_jvp_rhs(c->st, nl, elem(c), v_d, slot_ptrs(c->g), slot_ptrs(c->x), c->NRs, c->S);
  }
  CKL();
  if (c->green) {
    Timed t(c, KC_GREEN, 2);
    rba::launch_green_jvp(c->st, nl, c->N, (int)c->Mr, c->S, c->NRs, c->green_chunks,
                          slot_ptrs(c->Z), slot_ptrs(c->x), c->green_part, (cplx*)qpart);
    CKL();
    return RBA_OK;
  }
  if ((rc = solve_slots(c, all_slots(c), c->NRs))) return rc;
  if (c->Mr > 0) {
    Timed t(c, KC_ELEM);
    rba::launch_q_apply(c->st, nl, c->Mr, c->q_ptr, c->q_col, c->q_val, slot_ptrs(c->x), c->NRs, c->S, (cplx*)qpart);
    CKL();
  }
  return RBA_OK;
}

int rba_vjp_partial(rba_ctx* c, const double* w_d, double* tpart) {
  if (!c || !c->model_set || !w_d || !tpart) return fail(RBA_ERR_STATE, "bad state/arguments");
  CK(cudaSetDevice(c->device));
  const int nl = (int)c->local.size();
  int rc;
  if (c->green) {
    if ((rc = ensure_green(c))) return rc;
    {
      Timed t0(c, KC_GREEN, 2);
      rba::launch_walpha(c->st, nl, c->pole_of_slot, c->S, c->Kt, c->Mr, w_d, c->res_d, c->wa);
      rba::launch_green_vjp(c->st, nl, c->N, (int)c->Mr, c->S, c->NRs, slot_ptrs(c->Z), c->wa,
                            slot_ptrs(c->x));
    }
    CKL();
  } else {
  Timed t0(c, KC_ELEM, 2);
  rba::launch_vjp_rhs(c->st, nl, c->pole_of_slot, c->S, c->Kt, c->Mr, c->N, w_d, c->res_d, c->qt_ptr,
                      c->qt_col, c->qt_val, c->wa, slot_ptrs(c->x), c->NRs);
  }
  CKL();
  if (!c->green && (rc = solve_slots(c, all_slots(c), c->NRs))) return rc;
  Timed t1(c, KC_ELEM);
  rba::launch_vjp_cells(c->st, nl, c->pole_of_slot, c->poles_d, elem(c), slot_ptrs(c->x), slot_ptrs(c->g),
                        c->NRs, c->S, tpart);
  CKL();
  return RBA_OK;
}

int rba_combine_data(rba_ctx* c, const double* qall, const int32_t* som, int32_t times_pole,
                     double* d) {
  if (!c || !qall || !som || !d) return fail(RBA_ERR_INVALID, "null argument");
  CK(cudaSetDevice(c->device));
  CK(cudaMemcpyAsync(c->slot_map, som, c->m * sizeof(int32_t), cudaMemcpyHostToDevice, c->st));
  {
  Timed t(c, KC_ELEM);
  rba::launch_combine_data(c->st, c->m, c->S, c->Kt, c->Mr, (const cplx*)qall, c->slot_map, c->res_d,
                           c->poles_d, times_pole != 0, d);
  }
  CKL();
  CK(cudaStreamSynchronize(c->st));  // som is borrowed
  return RBA_OK;
}

int rba_combine_cells(rba_ctx* c, const double* tall, const int32_t* som, double* out) {
  if (!c || !tall || !som || !out) return fail(RBA_ERR_INVALID, "null argument");
  CK(cudaSetDevice(c->device));
  CK(cudaMemcpyAsync(c->slot_map, som, c->m * sizeof(int32_t), cudaMemcpyHostToDevice, c->st));
  {
    Timed t(c, KC_ELEM);
    rba::launch_combine_cells(c->st, c->m, c->P, tall, c->slot_map, out);
  }
  CKL();
  CK(cudaStreamSynchronize(c->st));
  return RBA_OK;
}

int rba_set_reg(rba_ctx* c, int64_t nrows, const int64_t* rp, const int32_t* ri, const double* rx) {
  if (!c || !c->have_mesh || nrows < 0 || (nrows > 0 && (!rp || !ri || !rx)))
    return fail(RBA_ERR_INVALID, "bad regulariser");
  CK(cudaSetDevice(c->device));
  free_list(c->reg_allocs);
  c->R_rows = nrows;
  const int64_t nnz = rp[nrows];
  std::vector<int64_t> tp(c->P + 1, 0);
  for (int64_t e = 0; e < nnz; ++e) {
    if (ri[e] < 0 || ri[e] >= c->P) return fail(RBA_ERR_INVALID, "R index out of range");
    tp[ri[e] + 1]++;
  }
  for (int64_t i = 0; i < c->P; ++i) tp[i + 1] += tp[i];
  std::vector<int32_t> tc(nnz);
  std::vector<double> tv(nnz);
  {
    std::vector<int64_t> pos(tp.begin(), tp.end() - 1);
    for (int64_t r = 0; r < nrows; ++r)
      for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {
        int64_t q = pos[ri[e]]++;
        tc[q] = (int32_t)r;
        tv[q] = rx[e];
      }
  }
  int rc;
  if ((rc = upload(c, c->reg_allocs, &c->r_ptr, rp, nrows + 1)) ||
      (rc = upload(c, c->reg_allocs, &c->r_idx, ri, nnz)) ||
      (rc = upload(c, c->reg_allocs, &c->r_val, rx, nnz)) ||
      (rc = upload(c, c->reg_allocs, &c->rt_ptr, tp.data(), tp.size())) ||
      (rc = upload(c, c->reg_allocs, &c->rt_idx, tc.data(), tc.size())) ||
      (rc = upload(c, c->reg_allocs, &c->rt_val, tv.data(), tv.size())))
    return rc;
  CK(cudaStreamSynchronize(c->st));
  return RBA_OK;
}

int rba_reg_apply(rba_ctx* c, int32_t transpose, const double* x, double alpha, double* y,
                  int32_t accumulate) {
  if (!c || !c->r_ptr || !x || !y) return fail(RBA_ERR_STATE, "set_reg first");
  Timed t(c, KC_VEC);
  if (transpose)
    rba::launch_spmv(c->st, c->P, c->rt_ptr, c->rt_idx, c->rt_val, x, alpha, y, accumulate != 0);
  else
    rba::launch_spmv(c->st, c->R_rows, c->r_ptr, c->r_idx, c->r_val, x, alpha, y, accumulate != 0);
  CKL();
  return RBA_OK;
}

int rba_vec_axpby(rba_ctx* c, int64_t n, double a, const double* x, double b, const double* y,
                  double* out) {
  Timed t(c, KC_VEC);
  rba::launch_axpby(c->st, n, a, x, b, y, out);
  CKL();
  return RBA_OK;
}

int rba_vec_mul(rba_ctx* c, int64_t n, const double* a, const double* x, double alpha,
                double* out) {
  Timed t(c, KC_VEC);
  rba::launch_mul(c->st, n, a, x, alpha, out);
  CKL();
  return RBA_OK;
}

int rba_vec_dot(rba_ctx* c, int64_t n, const double* x, const double* y, double* result) {
  { Timed t(c, KC_VEC, 2); rba::launch_dot(c->st, n, x, y, c->red_part, c->red_res); }
  CKL();
  CK(cudaMemcpyAsync(result, c->red_res, sizeof(double), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  return RBA_OK;
}

int rba_vec_lsqr_xw(rba_ctx* c, int64_t n, double t1, double t2, const double* v, double* w,
                    double* x, double* wn2) {
  { Timed t(c, KC_VEC, 2); rba::launch_lsqr_xw(c->st, n, t1, t2, v, w, x, c->red_part, c->red_res); }
  CKL();
  CK(cudaMemcpyAsync(wn2, c->red_res, sizeof(double), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  return RBA_OK;
}

int rba_get_g(rba_ctx* c, int32_t slot, double* out_h) {
  if (!c || !out_h || slot < 0 || slot >= (int)c->local.size()) return fail(RBA_ERR_INVALID, "bad slot");
  CK(cudaSetDevice(c->device));
  int rc;
  const int64_t n = c->N * (int64_t)c->S;
  if ((rc = ensure_stage(c, n))) return rc;
  rba::launch_perm_out(c->st, c->N, c->S, c->NRs, c->perm_d, c->g[slot], c->stage, c->N);
  CKL();
  CK(cudaMemcpyAsync(out_h, c->stage, n * sizeof(cplx), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  return RBA_OK;
}

int rba_get_factor(rba_ctx* c, int32_t slot, double* out_h, int64_t count) {
  if (!c || !out_h || slot < 0 || slot >= (int)c->local.size()) return fail(RBA_ERR_INVALID, "bad slot");
  const int64_t tot = c->sym.panel_off[c->sym.nfront];
  if (count < tot) return fail(RBA_ERR_INVALID, "buffer too small");
  if (!c->factor[slot]) return fail(RBA_ERR_CACHE_MISS, "slot has no factor storage yet");
  CK(cudaSetDevice(c->device));
  CK(cudaMemcpyAsync(out_h, c->factor[slot], tot * sizeof(cplx), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  return RBA_OK;
}

int rba_get_g_d(rba_ctx* c, int32_t slot, double* out_d) {
  if (!c || !out_d || slot < 0 || slot >= (int)c->local.size()) return fail(RBA_ERR_INVALID, "bad slot");
  CK(cudaSetDevice(c->device));
  rba::launch_perm_out(c->st, c->N, c->S, c->NRs, c->perm_d, c->g[slot], (cplx*)out_d, c->N);
  CKL();
  return RBA_OK;
}

int rba_set_g(rba_ctx* c, int32_t slot, const double* g_h) {
  if (!c || !g_h || slot < 0 || slot >= (int)c->local.size()) return fail(RBA_ERR_INVALID, "bad slot");
  CK(cudaSetDevice(c->device));
  int rc;
  const int64_t n = c->N * (int64_t)c->S;
  if ((rc = ensure_stage(c, n))) return rc;
  CK(cudaMemcpyAsync(c->stage, g_h, n * sizeof(cplx), cudaMemcpyHostToDevice, c->st));
  CK(cudaMemsetAsync(c->g[slot], 0, (size_t)c->N * c->NRs * sizeof(cplx), c->st));
  rba::launch_perm_in(c->st, c->N, c->S, c->NRs, c->perm_d, c->stage, c->N, c->g[slot]);
  CKL();
  CK(cudaStreamSynchronize(c->st));
  return RBA_OK;
}

int rba_factor_stats(rba_ctx* c, int32_t slot, double* out_h) {
  if (!c || !out_h || slot < 0 || slot >= (int)c->local.size()) return fail(RBA_ERR_INVALID, "bad slot");
  if (c->valid.empty() || !c->valid[slot])
    return fail(RBA_ERR_CACHE_MISS, "no factorization for pole " + std::to_string(c->local[slot]));
  CK(cudaSetDevice(c->device));
  const double init[4] = {0.0, __builtin_inf(), 0.0, 0.0};
  CK(cudaMemcpyAsync(c->red_part, init, sizeof(init), cudaMemcpyHostToDevice, c->st));
  rba::launch_factor_stats(c->st, c->F, c->sym.nfront, c->factor[slot], c->red_part);
  CKL();
  CK(cudaMemcpyAsync(out_h, c->red_part, 4 * sizeof(double), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  return RBA_OK;
}

int rba_set_option(rba_ctx* c, const char* name, int64_t value) {
  if (!c || !name) return fail(RBA_ERR_INVALID, "null argument");
  const std::string n(name);
  if (n == "green") {
    // 0: stream per-action sweeps instead of the receiver Green's functions
    // (ranks of a multi-GPU job agree on the mode so J v / J^T w round the
    // same way everywhere); 1: request Green mode (only if it was allocated)
    if (value == 0) { c->green = false; c->green_req = false; return RBA_OK; }
    if (!c->factor.empty() && !c->green)
      return fail(RBA_ERR_STATE, "receiver-Green storage was not allocated (memory)");
    c->green_req = true;
    return RBA_OK;
  }
  if (n == "lazy_factors") {
    if (!c->factor.empty()) return fail(RBA_ERR_STATE, "set lazy_factors before set_poles");
    c->lazy = value != 0;
    return RBA_OK;
  }
  return fail(RBA_ERR_INVALID, "unknown option " + n);
}

int rba_set_reg_L(rba_ctx* c, int64_t n, const int64_t* lp, const int32_t* li, const double* lx) {
  if (!c || !c->have_mesh || n != c->P || !lp || !li || !lx)
    return fail(RBA_ERR_INVALID, "L must be P x P CSR");
  CK(cudaSetDevice(c->device));
  free_list(c->regl_allocs);
  const int64_t nnz = lp[n];
  for (int64_t e = 0; e < nnz; ++e)
    if (li[e] < 0 || li[e] >= c->P) return fail(RBA_ERR_INVALID, "L index out of range");
  int rc;
  if ((rc = upload(c, c->regl_allocs, &c->l_ptr, lp, n + 1)) ||
      (rc = upload(c, c->regl_allocs, &c->l_idx, li, nnz)) ||
      (rc = upload(c, c->regl_allocs, &c->l_val, lx, nnz)))
    return rc;
  c->L_n = n;
  CK(cudaStreamSynchronize(c->st));
  return RBA_OK;
}

int rba_reg_L_apply(rba_ctx* c, const double* x, double alpha, double* y, int32_t accumulate) {
  if (!c || !c->l_ptr || !x || !y) return fail(RBA_ERR_STATE, "set_reg_L first");
  Timed t(c, KC_VEC);
  rba::launch_spmv(c->st, c->L_n, c->l_ptr, c->l_idx, c->l_val, x, alpha, y, accumulate != 0);
  CKL();
  return RBA_OK;
}

int rba_oz_stats(rba_ctx* c, double* out) {
  if (!c || !out) return fail(RBA_ERR_INVALID, "null argument");
  out[0] = c->ozaki ? 1.0 : 0.0;
  out[1] = c->oz_int8_ops;
  out[2] = c->oz_flops;
  out[3] = (double)c->oz_sub;
  out[4] = (double)c->oz_min_k;
  return RBA_OK;
}

int rba_oz_prof(rba_ctx* c, double* out, int reset) {
  if (!c || !out) return fail(RBA_ERR_INVALID, "null argument");
  CK(cudaStreamSynchronize(c->st));
  unsigned long long v[10];
  rba::oz_prof_read(v, reset != 0);
  for (int i = 0; i < 10; ++i) out[i] = (double)v[i];
  return RBA_OK;
}

int rba_info(rba_ctx* c, int64_t* out) {
  if (!c || !out) return fail(RBA_ERR_INVALID, "null argument");
  out[0] = c->n_fact; out[1] = c->n_solve; out[2] = c->N; out[3] = c->P;
  out[4] = c->Mr; out[5] = c->S; out[6] = c->m; out[7] = (int64_t)c->local.size();
  out[8] = c->green ? 1 : 0; out[9] = c->n_green;
  return RBA_OK;
}

int rba_memory(rba_ctx* c, int64_t* out) {
  if (!c || !out) return fail(RBA_ERR_INVALID, "null argument");
  out[0] = (int64_t)c->mem_factor; out[1] = (int64_t)c->mem_work; out[2] = (int64_t)c->mem_other;
  return RBA_OK;
}

int rba_sync(rba_ctx* c) {
  CK(cudaStreamSynchronize(c->st));
  return RBA_OK;
}

int rba_timings(rba_ctx* c, double* out) {
  flush_timing(c);
  for (int i = 0; i < 16; ++i) out[i] = c->cls_ms[i];
  out[15] = (double)c->launches;
  return RBA_OK;
}

int rba_timings_detail(rba_ctx* c, double* out) {
  flush_timing(c);
  for (int i = 0; i < 128; ++i) out[i] = c->cls_ms[i];
  return RBA_OK;
}

int rba_set_timing(rba_ctx* c, int32_t en) {
  flush_timing(c);
  if (en == 2) {
    for (double& v : c->cls_ms) v = 0;
    c->launches = 0;
    return RBA_OK;
  }
  c->timing = en != 0;
  return RBA_OK;
}

}  // extern "C"
