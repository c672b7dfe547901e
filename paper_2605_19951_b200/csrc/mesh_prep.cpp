// See mesh_prep.h.
#include "mesh_prep.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace rba {

std::string prepare_mesh(int64_t N, int64_t P, int32_t k, const int32_t* cell_dofs,
                         const double* mass_local, const int64_t* Kp, const int32_t* Ki,
                         const double* Kx, const double* coords, int32_t leaf, MeshPrep& M) {
  // dof -> (cell, slot) lists
  std::vector<int64_t> dcp(N + 1, 0);
  for (int64_t i = 0; i < P * k; ++i) {
    int32_t d = cell_dofs[i];
    if (d >= N) return std::string("cell_dofs entry out of range");
    if (d >= 0) dcp[d + 1]++;
  }
  for (int64_t i = 0; i < N; ++i) dcp[i + 1] += dcp[i];
  std::vector<int32_t> dci(dcp[N]);
  {
    std::vector<int64_t> pos(dcp.begin(), dcp.end() - 1);
    for (int64_t cidx = 0; cidx < P; ++cidx)
      for (int a = 0; a < k; ++a) {
        int32_t d = cell_dofs[cidx * k + a];
        if (d >= 0) dci[pos[d]++] = (int32_t)(cidx * 6 + a);
      }
  }
  // full symmetric pattern: element pattern U K pattern
  std::vector<int64_t> ap(N + 1, 0);
  std::vector<int32_t> ai;
  {
    std::vector<int32_t> mark(N, -1), row;
    ai.reserve((size_t)dcp[N] * k);
    for (int64_t r = 0; r < N; ++r) {
      row.clear();
      for (int64_t q = dcp[r]; q < dcp[r + 1]; ++q) {
        int64_t cidx = dci[q] / 6;
        for (int b = 0; b < k; ++b) {
          int32_t cc = cell_dofs[cidx * k + b];
          if (cc >= 0 && mark[cc] != r) { mark[cc] = (int32_t)r; row.push_back(cc); }
        }
      }
      for (int64_t e = Kp[r]; e < Kp[r + 1]; ++e) {
        int32_t cc = Ki[e];
        if (cc < 0 || cc >= N) return std::string("K index out of range");
        if (mark[cc] != r) { mark[cc] = (int32_t)r; row.push_back(cc); }
      }
      if (mark[r] != r) { mark[r] = (int32_t)r; row.push_back((int32_t)r); }
      std::sort(row.begin(), row.end());
      ai.insert(ai.end(), row.begin(), row.end());
      ap[r + 1] = ai.size();
    }
  }
  // lower triangle (row >= col), K values, M contribution lists
  std::vector<int64_t> lp(N + 1, 0);
  M.a_rows.clear(); M.a_cols.clear(); M.Kv.clear();
  for (int64_t r = 0; r < N; ++r) {
    for (int64_t e = ap[r]; e < ap[r + 1]; ++e) {
      int32_t cc = ai[e];
      if (cc > r) break;
      M.a_rows.push_back((int32_t)r);
      M.a_cols.push_back(cc);
    }
    lp[r + 1] = M.a_rows.size();
  }
  M.nnzA = M.a_rows.size();
  M.Kv.assign(M.nnzA, 0.0);
  for (int64_t r = 0; r < N; ++r)
    for (int64_t e = Kp[r]; e < Kp[r + 1]; ++e) {
      int32_t cc = Ki[e];
      if (cc > r) continue;
      const int32_t* b0 = M.a_cols.data() + lp[r];
      const int32_t* b1 = M.a_cols.data() + lp[r + 1];
      const int32_t* it = std::lower_bound(b0, b1, cc);
      M.Kv[lp[r] + (it - b0)] += Kx[e];
    }
  M.mcnt.assign(M.nnzA + 1, 0);
  std::vector<int64_t>& mcnt = M.mcnt;
  std::vector<int64_t> me;  // (e, off) pairs flattened
  me.reserve((size_t)P * k * (k + 1));
  for (int64_t cidx = 0; cidx < P; ++cidx)
    for (int a = 0; a < k; ++a) {
      int32_t r = cell_dofs[cidx * k + a];
      if (r < 0) continue;
      for (int b = 0; b < k; ++b) {
        int32_t cc = cell_dofs[cidx * k + b];
        if (cc < 0 || cc > r) continue;
        const int32_t* b0 = M.a_cols.data() + lp[r];
        const int32_t* b1 = M.a_cols.data() + lp[r + 1];
        int64_t e = lp[r] + (std::lower_bound(b0, b1, cc) - b0);
        me.push_back(e);
        me.push_back(cidx * 36 + a * 6 + b);
        mcnt[e + 1]++;
      }
    }
  for (int64_t e = 0; e < M.nnzA; ++e) mcnt[e + 1] += mcnt[e];
  M.moff.assign(mcnt[M.nnzA], 0);
  std::vector<int64_t>& moff = M.moff;
  {
    std::vector<int64_t> pos(mcnt.begin(), mcnt.end() - 1);
    for (size_t q = 0; q < me.size(); q += 2) moff[pos[me[q]]++] = me[q + 1];
  }
  std::vector<int64_t>().swap(me);
  // symbolic analysis
  std::string err = rba::analyze(N, ap.data(), ai.data(), coords, leaf > 0 ? leaf : 64, M.sym);
  if (!err.empty()) return std::string("symbolic analysis: " + err);
  const rba::Symbolic& S = M.sym;
  // scatter targets of A entries into the front panels
  std::vector<int32_t> front_of(N);
  for (int s = 0; s < S.nfront; ++s)
    for (int q = 0; q < S.npiv[s]; ++q) front_of[S.first[s] + q] = s;
  M.tgt.assign(M.nnzA, 0);
  std::vector<int64_t>& tgt = M.tgt;
  for (int64_t e = 0; e < M.nnzA; ++e) {
    int32_t pr = S.iperm[M.a_rows[e]], pc = S.iperm[M.a_cols[e]];
    int32_t hi = std::max(pr, pc), lo = std::min(pr, pc);
    int s = front_of[lo];
    const int32_t* rb = S.rows.data() + S.rows_off[s];
    const int32_t* it = std::lower_bound(rb, rb + S.nf[s], hi);
    if (it == rb + S.nf[s] || *it != hi) {
      if (getenv("RBA_DEBUG"))
        fprintf(stderr, "e=%ld row=%d col=%d pr=%d pc=%d s=%d first=%d npiv=%d nf=%d nnzpat=%ld\n",
                (long)e, M.a_rows[e], M.a_cols[e], pr, pc, s, S.first[s], S.npiv[s], S.nf[s], (long)ap[N]);
      return std::string("internal: A entry outside front");
    }
    tgt[e] = S.panel_off[s] + (int64_t)(lo - S.first[s]) * S.nf[s] + (it - rb);
  }
  // permuted element data
  M.cdp.assign((size_t)P * 6, -1);
  std::vector<int32_t>& cdp = M.cdp;
  M.mass36.assign((size_t)P * 36, 0.0);
  std::vector<double>& mass36 = M.mass36;
  for (int64_t cidx = 0; cidx < P; ++cidx)
    for (int a = 0; a < k; ++a) {
      int32_t d = cell_dofs[cidx * k + a];
      cdp[cidx * 6 + a] = d >= 0 ? S.iperm[d] : -1;
      for (int b = 0; b < k; ++b) mass36[cidx * 36 + a * 6 + b] = mass_local[(cidx * k + a) * k + b];
    }
  // dof lists re-indexed by permuted dof, element mass offsets rebased to 36
  M.pdcp.assign(N + 1, 0);
  std::vector<int64_t>& pdcp = M.pdcp;
  M.pdci.assign(dci.size(), 0);
  std::vector<int32_t>& pdci = M.pdci;
  for (int64_t kk = 0; kk < N; ++kk) {
    int32_t o = S.perm[kk];
    pdcp[kk + 1] = pdcp[kk] + (dcp[o + 1] - dcp[o]);
  }
  for (int64_t kk = 0; kk < N; ++kk) {
    int32_t o = S.perm[kk];
    std::copy(dci.begin() + dcp[o], dci.begin() + dcp[o + 1], pdci.begin() + pdcp[kk]);
  }
  return "";
}

}  // namespace rba
