// 3-D operator generation on the GPU: the lowest-order
// Nedelec problem on a Kuhn-split n^3 hex box -- edge numbering with the PEC
// boundary eliminated, per-tet dofs, the curl-curl stiffness K (CSR, duplicates
// summed in element order), tet vertices, edge midpoints, the interior-face
// adjacency and face measures of the RT0 regulariser -- plus the element-pencil
// spectral bound.  Device restatement of paper_2605_19951_b200/mesh3d.py
// (build_box_problem, spectral_bound), the 3-D counterpart of the reference's
// build_problem / spectral_bound (/root/reference/pkg/src/rbainv/mesh.py:294-345,
// 406-421).  Same numbering as the host builder: edges sorted by (low vertex,
// high vertex) -- from a vertex v the seven edge directions of the Kuhn split,
// +x, +y, +x+y, +z, +x+z, +y+z, +x+y+z, have increasing vertex offsets -- so
// the dof of an edge is a prefix count over vertices.
#include <cub/cub.cuh>

#include <string>
#include <vector>

#include "../../include/rba_b200.h"

namespace {

__constant__ int c_dir[7][3] = {{1, 0, 0}, {0, 1, 0}, {1, 1, 0}, {0, 0, 1},
                                {1, 0, 1}, {0, 1, 1}, {1, 1, 1}};
__constant__ int c_perm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
__constant__ int c_ledge[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
__constant__ double c_stiff[6][36];     // per Kuhn tet type (mesh3d._local_matrices)

__device__ __forceinline__ int dir_of(int dx, int dy, int dz) {
  // inverse of c_dir
  const int code = dx + 2 * dy + 4 * dz;   // 1,2,3,4,5,6,7 for the 7 directions
  const int map[8] = {-1, 0, 1, 2, 3, 4, 5, 6};
  return map[code];
}

// bit d of the result: edge (v, dir d) exists (in the box) / is interior (not PEC)
__device__ __forceinline__ void edge_masks(int n, int x, int y, int z, unsigned& valid,
                                           unsigned& inter) {
  valid = inter = 0;
#pragma unroll
  for (int d = 0; d < 7; ++d) {
    const int dx = c_dir[d][0], dy = c_dir[d][1], dz = c_dir[d][2];
    if (x + dx > n || y + dy > n || z + dz > n) continue;
    valid |= 1u << d;
    const bool bnd = (dx == 0 && (x == 0 || x == n)) || (dy == 0 && (y == 0 || y == n)) ||
                     (dz == 0 && (z == 0 || z == n));
    if (!bnd) inter |= 1u << d;
  }
}

__global__ void k_edge_count(int n, int64_t nvt, int64_t* cnt_valid, int64_t* cnt_inter) {
  const int64_t nv1 = n + 1;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvt;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(v % nv1), y = (int)((v / nv1) % nv1), z = (int)(v / (nv1 * nv1));
    unsigned va, in;
    edge_masks(n, x, y, z, va, in);
    cnt_valid[v] = __popc(va);
    cnt_inter[v] = __popc(in);
  }
}

// dof_of_edge (edges in key order, -1 on the PEC boundary), edge midpoints of the dofs
__global__ void k_edges(int n, double h, int64_t nvt, const int64_t* eoff, const int64_t* doff,
                        int64_t* dof_of_edge, double* dof_coords) {
  const int64_t nv1 = n + 1;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvt;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(v % nv1), y = (int)((v / nv1) % nv1), z = (int)(v / (nv1 * nv1));
    unsigned va, in;
    edge_masks(n, x, y, z, va, in);
    int64_t e = eoff[v], dd = doff[v];
    for (int d = 0; d < 7; ++d) {
      if (!(va >> d & 1u)) continue;
      if (in >> d & 1u) {
        dof_of_edge[e] = dd;
        dof_coords[dd * 3 + 0] = (x + 0.5 * c_dir[d][0]) * h;
        dof_coords[dd * 3 + 1] = (y + 0.5 * c_dir[d][1]) * h;
        dof_coords[dd * 3 + 2] = (z + 0.5 * c_dir[d][2]) * h;
        ++dd;
      } else {
        dof_of_edge[e] = -1;
      }
      ++e;
    }
  }
}

// tets: vertices, dofs, stiffness COO entries (key = row * N + col, invalid -> max)
__global__ void k_tets(int n, int64_t N, int64_t P, const int64_t* doff, int64_t* cells,
                       int32_t* cell_dofs, unsigned long long* keys, double* vals,
                       uint32_t* idx, int64_t* fkeys, uint32_t* fidx) {
  const int64_t nv1 = n + 1, nvt = nv1 * nv1 * nv1;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < P;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t hex = c / 6;
    const int t = (int)(c % 6);
    int co[4][3];
    co[0][0] = (int)(hex % n);
    co[0][1] = (int)((hex / n) % n);
    co[0][2] = (int)(hex / ((int64_t)n * n));
    for (int sidx = 0; sidx < 3; ++sidx) {
      for (int a = 0; a < 3; ++a) co[sidx + 1][a] = co[sidx][a];
      co[sidx + 1][c_perm[t][sidx]] += 1;
    }
    int64_t vid[4];
    for (int k = 0; k < 4; ++k) {
      vid[k] = co[k][0] + nv1 * (co[k][1] + nv1 * co[k][2]);
      cells[c * 4 + k] = vid[k];
    }
    int32_t dofs[6];
    for (int a = 0; a < 6; ++a) {
      const int i = c_ledge[a][0], j = c_ledge[a][1];   // vertex ids increase: i -> j is low -> high
      const int d = dir_of(co[j][0] - co[i][0], co[j][1] - co[i][1], co[j][2] - co[i][2]);
      unsigned va, in;
      edge_masks(n, co[i][0], co[i][1], co[i][2], va, in);
      dofs[a] = (in >> d & 1u) ? (int32_t)(doff[vid[i]] + __popc(in & ((1u << d) - 1u))) : -1;
      cell_dofs[c * 6 + a] = dofs[a];
    }
    for (int a = 0; a < 6; ++a)
      for (int b = 0; b < 6; ++b) {
        const int64_t q = c * 36 + a * 6 + b;
        const bool ok = dofs[a] >= 0 && dofs[b] >= 0;
        keys[q] = ok ? (unsigned long long)dofs[a] * (unsigned long long)N + (unsigned long long)dofs[b]
                     : ~0ull;
        vals[q] = c_stiff[t][a * 6 + b];
        idx[q] = (uint32_t)q;
      }
    // faces (0,1,2), (0,1,3), (0,2,3), (1,2,3): vertex ids already ascending
    const int fl[4][3] = {{0, 1, 2}, {0, 1, 3}, {0, 2, 3}, {1, 2, 3}};
    for (int f = 0; f < 4; ++f) {
      fkeys[c * 4 + f] = (vid[fl[f][0]] * nvt + vid[fl[f][1]]) * nvt + vid[fl[f][2]];
      fidx[c * 4 + f] = (uint32_t)(c * 4 + f);
    }
  }
}

// segment heads of the sorted keys (1 where a new (row, col) starts)
__global__ void k_heads(int64_t m, const unsigned long long* keys, int64_t* head) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    head[i] = (keys[i] != ~0ull && (i == 0 || keys[i] != keys[i - 1])) ? 1 : 0;
}

// one thread per (row, col) segment: sequential sum in element order
__global__ void k_reduce(int64_t m, int64_t N, const unsigned long long* keys, const double* vals,
                         const uint32_t* idx, const int64_t* hscan, const int64_t* head,
                         int32_t* colv, double* valv, int64_t* rowcnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (!head[i]) continue;
    const unsigned long long k = keys[i];
    double acc = 0.0;
    for (int64_t j = i; j < m && keys[j] == k; ++j) acc += vals[idx[j]];
    const int64_t out = hscan[i];
    colv[out] = (int32_t)(k % (unsigned long long)N);
    valv[out] = acc;
    atomicAdd(reinterpret_cast<unsigned long long*>(rowcnt + (k / (unsigned long long)N)), 1ull);
  }
}

// interior faces: adjacent equal keys after the stable sort
__global__ void k_face_marks(int64_t m, const int64_t* fk, int64_t* mark) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    mark[i] = (i + 1 < m && fk[i] == fk[i + 1]) ? 1 : 0;
}
__global__ void k_faces(int64_t m, int n, double h, const int64_t* fk, const uint32_t* fidx,
                        const int64_t* mark, const int64_t* mscan, int32_t* face_cells,
                        double* face_measure) {
  const int64_t nv1 = n + 1, nvt = nv1 * nv1 * nv1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (!mark[i]) continue;
    const int64_t f = mscan[i];
    face_cells[2 * f] = (int32_t)(fidx[i] / 4);
    face_cells[2 * f + 1] = (int32_t)(fidx[i + 1] / 4);
    const int64_t k = fk[i];
    const int64_t a = k / (nvt * nvt), b = (k / nvt) % nvt, cc = k % nvt;
    double p[3][3];
    const int64_t vv[3] = {a, b, cc};
    for (int q = 0; q < 3; ++q) {
      p[q][0] = (double)(vv[q] % nv1) * h;
      p[q][1] = (double)((vv[q] / nv1) % nv1) * h;
      p[q][2] = (double)(vv[q] / (nv1 * nv1)) * h;
    }
    const double u0 = p[1][0] - p[0][0], u1 = p[1][1] - p[0][1], u2 = p[1][2] - p[0][2];
    const double w0 = p[2][0] - p[0][0], w1 = p[2][1] - p[0][1], w2 = p[2][2] - p[0][2];
    const double c0 = u1 * w2 - u2 * w1, c1 = u2 * w0 - u0 * w2, c2 = u0 * w1 - u1 * w0;
    face_measure[f] = 0.5 * sqrt(c0 * c0 + c1 * c1 + c2 * c2);
  }
}

// per cell: largest eigenvalue of M_c^{-1/2} K_c M_c^{-1/2} (Cholesky of the
// 6x6 mass, power iteration on the symmetric 6x6)
__host__ __device__ inline double cell_lmax(const double* M, const double* S) {
  double L[6][6] = {}, A[6][6], B[6][6];
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = M[i * 6 + j];
      for (int k = 0; k < j; ++k) s -= L[i][k] * L[j][k];
      L[i][j] = i == j ? sqrt(s) : s / L[j][j];
    }
  // B = L^{-1} S, A = B L^{-T}
  for (int col = 0; col < 6; ++col)
    for (int i = 0; i < 6; ++i) {
      double s = S[i * 6 + col];
      for (int k = 0; k < i; ++k) s -= L[i][k] * B[k][col];
      B[i][col] = s / L[i][i];
    }
  for (int row = 0; row < 6; ++row)
    for (int i = 0; i < 6; ++i) {
      double s = B[row][i];
      for (int k = 0; k < i; ++k) s -= L[i][k] * A[row][k];
      A[row][i] = s / L[i][i];
    }
  // largest eigenvalue of the symmetric PSD A: power iteration + Rayleigh
  // quotient (ratio lambda_2 / lambda_1 ~ 0.4 on the Kuhn tets; 200 steps)
  double x[6] = {1.0, 0.75, 0.5, -0.25, 0.6, 0.9}, lam = 0.0;
  for (int it = 0; it < 200; ++it) {
    double y[6], nrm = 0.0;
    for (int i = 0; i < 6; ++i) {
      double acc = 0.0;
      for (int k = 0; k < 6; ++k) acc += A[i][k] * x[k];
      y[i] = acc;
      nrm += acc * acc;
    }
    nrm = sqrt(nrm);
    if (nrm == 0.0) return 0.0;
    for (int i = 0; i < 6; ++i) x[i] = y[i] / nrm;
  }
  for (int i = 0; i < 6; ++i) {
    double acc = 0.0;
    for (int k = 0; k < 6; ++k) acc += A[i][k] * x[k];
    lam += x[i] * acc;
  }
  return lam;
}

// max over cells of cell_lmax / e^{m_c}
__global__ void k_spectral(int64_t P, const double* mass, const double* stiff, const double* m,
                           double* out) {
  double best = 0.0;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < P;
       c += (int64_t)gridDim.x * blockDim.x)
    best = fmax(best, cell_lmax(mass + c * 36, stiff + c * 36) / exp(m[c]));
  for (int o = 16; o > 0; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0)
    atomicMax(reinterpret_cast<unsigned long long*>(out), (unsigned long long)__double_as_longlong(best));
}

thread_local std::string g_gen_err;
int gfail(const std::string& m) { g_gen_err = m; return RBA_ERR_CUDA; }
#define GK(x)                                                                     \
  do {                                                                            \
    cudaError_t e_ = (x);                                                         \
    if (e_ != cudaSuccess) return gfail(std::string(cudaGetErrorString(e_)) + " at " #x); \
  } while (0)

int grid_of(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }

}  // namespace

struct rba_box {
  int n = 0;
  int64_t nvt = 0, P = 0, N = 0, E = 0, nnz = 0, F = 0;
  std::vector<void*> bufs;
  int64_t* dof_of_edge = nullptr;
  double* dof_coords = nullptr;
  int64_t* cells = nullptr;
  int32_t* cell_dofs = nullptr;
  int64_t* indptr = nullptr;
  int32_t* indices = nullptr;
  double* data = nullptr;
  int32_t* face_cells = nullptr;
  double* face_measure = nullptr;
  int64_t* doff = nullptr;
};

namespace {
template <class T>
int galloc(rba_box* b, T** p, size_t count) {
  void* q = nullptr;
  cudaError_t e = cudaMalloc(&q, std::max<size_t>(count, 1) * sizeof(T));
  if (e != cudaSuccess) { cudaGetLastError(); return gfail("device allocation failed"); }
  b->bufs.push_back(q);
  *p = (T*)q;
  return RBA_OK;
}
}  // namespace

extern "C" {

const char* rba_box_last_error(void) { return g_gen_err.c_str(); }

int rba_box_generate(int32_t n, double h, const double* stiff6_h, rba_box** out) {
  if (n < 1 || !stiff6_h || !out) { g_gen_err = "bad arguments"; return RBA_ERR_INVALID; }
  auto* b = new rba_box();
  b->n = n;
  const int64_t nv1 = n + 1;
  b->nvt = nv1 * nv1 * nv1;
  b->P = (int64_t)n * n * n * 6;
  int rc = RBA_OK;
  auto fin = [&](int r) { if (r) { rba_box_destroy(b); } return r; };
  GK(cudaMemcpyToSymbol(c_stiff, stiff6_h, sizeof(double) * 6 * 36));
  int64_t *cv, *ci, *eoff;
  if ((rc = galloc(b, &cv, b->nvt + 1)) || (rc = galloc(b, &ci, b->nvt + 1)) ||
      (rc = galloc(b, &eoff, b->nvt + 1)) || (rc = galloc(b, &b->doff, b->nvt + 1)))
    return fin(rc);
  GK(cudaMemset(cv + b->nvt, 0, 8));
  GK(cudaMemset(ci + b->nvt, 0, 8));
  k_edge_count<<<grid_of(b->nvt), 256>>>(n, b->nvt, cv, ci);
  size_t tmp = 0;
  void* tbuf = nullptr;
  auto scan = [&](const int64_t* in, int64_t* o, int64_t cnt) -> int {
    size_t need = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, need, in, o, cnt);
    if (need > tmp) {
      if (tbuf) cudaFree(tbuf);
      if (cudaMalloc(&tbuf, need) != cudaSuccess) { cudaGetLastError(); return gfail("scan temp"); }
      tmp = need;
    }
    cub::DeviceScan::ExclusiveSum(tbuf, tmp, in, o, cnt);
    return RBA_OK;
  };
  if ((rc = scan(cv, eoff, b->nvt + 1)) || (rc = scan(ci, b->doff, b->nvt + 1))) return fin(rc);
  GK(cudaMemcpy(&b->E, eoff + b->nvt, 8, cudaMemcpyDeviceToHost));
  GK(cudaMemcpy(&b->N, b->doff + b->nvt, 8, cudaMemcpyDeviceToHost));
  if ((rc = galloc(b, &b->dof_of_edge, b->E)) || (rc = galloc(b, &b->dof_coords, b->N * 3)) ||
      (rc = galloc(b, &b->cells, b->P * 4)) || (rc = galloc(b, &b->cell_dofs, b->P * 6)))
    return fin(rc);
  k_edges<<<grid_of(b->nvt), 256>>>(n, h, b->nvt, eoff, b->doff, b->dof_of_edge, b->dof_coords);
  // stiffness and face entries
  const int64_t m = b->P * 36, mf = b->P * 4;
  unsigned long long *keys, *keys2;
  double* vals;
  uint32_t *idx, *idx2, *fidx, *fidx2;
  int64_t *fkeys, *fkeys2, *head, *hscan;
  if ((rc = galloc(b, &keys, m)) || (rc = galloc(b, &keys2, m)) || (rc = galloc(b, &vals, m)) ||
      (rc = galloc(b, &idx, m)) || (rc = galloc(b, &idx2, m)) || (rc = galloc(b, &fkeys, mf)) ||
      (rc = galloc(b, &fkeys2, mf)) || (rc = galloc(b, &fidx, mf)) || (rc = galloc(b, &fidx2, mf)) ||
      (rc = galloc(b, &head, m + 1)) || (rc = galloc(b, &hscan, m + 1)))
    return fin(rc);
  k_tets<<<grid_of(b->P), 256>>>(n, b->N, b->P, b->doff, b->cells, b->cell_dofs, keys, vals, idx,
                                 fkeys, fidx);
  // stable radix sorts (equal keys keep element order)
  {
    size_t need = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, need, keys, keys2, idx, idx2, (int)m);
    size_t need2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, need2, fkeys, fkeys2, fidx, fidx2, (int)mf);
    need = std::max(need, need2);
    if (need > tmp) {
      if (tbuf) cudaFree(tbuf);
      if (cudaMalloc(&tbuf, need) != cudaSuccess) { cudaGetLastError(); return fin(gfail("sort temp")); }
      tmp = need;
    }
    cub::DeviceRadixSort::SortPairs(tbuf, tmp, keys, keys2, idx, idx2, (int)m);
    cub::DeviceRadixSort::SortPairs(tbuf, tmp, fkeys, fkeys2, fidx, fidx2, (int)mf);
  }
  GK(cudaMemset(head + m, 0, 8));
  k_heads<<<grid_of(m), 256>>>(m, keys2, head);
  if ((rc = scan(head, hscan, m + 1))) return fin(rc);
  GK(cudaMemcpy(&b->nnz, hscan + m, 8, cudaMemcpyDeviceToHost));
  int64_t* rowcnt;
  if ((rc = galloc(b, &b->indices, b->nnz)) || (rc = galloc(b, &b->data, b->nnz)) ||
      (rc = galloc(b, &rowcnt, b->N + 1)) || (rc = galloc(b, &b->indptr, b->N + 1)))
    return fin(rc);
  GK(cudaMemset(rowcnt, 0, (b->N + 1) * 8));
  k_reduce<<<grid_of(m), 256>>>(m, b->N, keys2, vals, idx2, hscan, head, b->indices, b->data, rowcnt);
  if ((rc = scan(rowcnt, b->indptr, b->N + 1))) return fin(rc);
  // faces
  GK(cudaMemset(head + mf, 0, 8));
  k_face_marks<<<grid_of(mf), 256>>>(mf, fkeys2, head);
  if ((rc = scan(head, hscan, mf + 1))) return fin(rc);
  GK(cudaMemcpy(&b->F, hscan + mf, 8, cudaMemcpyDeviceToHost));
  if ((rc = galloc(b, &b->face_cells, b->F * 2)) || (rc = galloc(b, &b->face_measure, b->F)))
    return fin(rc);
  k_faces<<<grid_of(mf), 256>>>(mf, n, h, fkeys2, fidx2, head, hscan, b->face_cells, b->face_measure);
  GK(cudaGetLastError());
  GK(cudaDeviceSynchronize());
  if (tbuf) cudaFree(tbuf);
  *out = b;
  return RBA_OK;
}

int rba_box_info(const rba_box* b, int64_t* out_h) {
  if (!b || !out_h) return RBA_ERR_INVALID;
  out_h[0] = b->N; out_h[1] = b->P; out_h[2] = b->nnz; out_h[3] = b->F; out_h[4] = b->E;
  out_h[5] = b->nvt;
  return RBA_OK;
}

int rba_box_get(const rba_box* b, const char* name, void* out_h, int64_t capacity_bytes) {
  if (!b || !name || !out_h) { g_gen_err = "null argument"; return RBA_ERR_INVALID; }
  const std::string s(name);
  const void* src = nullptr;
  int64_t nb = 0;
  if (s == "cell_dofs") { src = b->cell_dofs; nb = b->P * 6 * 4; }
  else if (s == "cells") { src = b->cells; nb = b->P * 4 * 8; }
  else if (s == "indptr") { src = b->indptr; nb = (b->N + 1) * 8; }
  else if (s == "indices") { src = b->indices; nb = b->nnz * 4; }
  else if (s == "data") { src = b->data; nb = b->nnz * 8; }
  else if (s == "face_cells") { src = b->face_cells; nb = b->F * 2 * 4; }
  else if (s == "face_measure") { src = b->face_measure; nb = b->F * 8; }
  else if (s == "dof_of_edge") { src = b->dof_of_edge; nb = b->E * 8; }
  else if (s == "dof_coords") { src = b->dof_coords; nb = b->N * 3 * 8; }
  else if (s == "dof_offset") { src = b->doff; nb = (b->nvt + 1) * 8; }
  else { g_gen_err = "unknown array " + s; return RBA_ERR_INVALID; }
  if (capacity_bytes < nb) { g_gen_err = "buffer too small"; return RBA_ERR_INVALID; }
  if (cudaMemcpy(out_h, src, nb, cudaMemcpyDeviceToHost) != cudaSuccess) {
    g_gen_err = "copy failed";
    return RBA_ERR_CUDA;
  }
  return RBA_OK;
}

void rba_box_destroy(rba_box* b) {
  if (!b) return;
  for (void* p : b->bufs) cudaFree(p);
  delete b;
}

int rba_spectral_bound(int64_t P, const double* mass_local_h, const double* stiff_local_h,
                       const double* m_h, double* out_h) {
  if (P < 1 || !mass_local_h || !stiff_local_h || !m_h || !out_h) {
    g_gen_err = "bad arguments";
    return RBA_ERR_INVALID;
  }
  double *dm, *ds, *dmm, *dout;
  if (cudaMalloc(&dm, P * 36 * 8) != cudaSuccess || cudaMalloc(&ds, P * 36 * 8) != cudaSuccess ||
      cudaMalloc(&dmm, P * 8) != cudaSuccess || cudaMalloc(&dout, 8) != cudaSuccess) {
    cudaGetLastError();
    g_gen_err = "device allocation failed";
    return RBA_ERR_OOM;
  }
  cudaMemcpy(dm, mass_local_h, P * 36 * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(ds, stiff_local_h, P * 36 * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dmm, m_h, P * 8, cudaMemcpyHostToDevice);
  cudaMemset(dout, 0, 8);
  k_spectral<<<grid_of(P), 256>>>(P, dm, ds, dmm, dout);
  const cudaError_t e = cudaMemcpy(out_h, dout, 8, cudaMemcpyDeviceToHost);
  cudaFree(dm); cudaFree(ds); cudaFree(dmm); cudaFree(dout);
  if (e != cudaSuccess) { g_gen_err = cudaGetErrorString(e); return RBA_ERR_CUDA; }
  return RBA_OK;
}

}  // extern "C"
