// Host symbolic analysis: nested dissection, assembly tree, front structures,
// level schedule and memory plans.  See symbolic.h.
#include "symbolic.h"

#include <algorithm>
#include <cmath>
#include <map>
#include <numeric>

namespace rba {
namespace {

struct ND {
  int64_t n;
  const int64_t* ip;
  const int32_t* ix;
  const double* xyz;
  int32_t leaf;
  std::vector<int32_t> order;            // new -> old
  std::vector<int32_t> node_first, node_npiv;
  std::vector<std::vector<int32_t>> node_children;
  std::vector<int32_t> stamp, side, dist;
  int32_t cur = 0;

  ND(int64_t n_, const int64_t* ip_, const int32_t* ix_, const double* xyz_, int32_t leaf_)
      : n(n_), ip(ip_), ix(ix_), xyz(xyz_), leaf(leaf_), stamp(n_, -1), side(n_, 0),
        dist(n_, -1) {}

  int32_t new_node(const std::vector<int32_t>& piv, std::vector<int32_t> kids) {
    int32_t id = (int32_t)node_first.size();
    node_first.push_back((int32_t)order.size());
    node_npiv.push_back((int32_t)piv.size());
    node_children.push_back(std::move(kids));
    order.insert(order.end(), piv.begin(), piv.end());
    return id;
  }

  // side: 0 left, 1 right, 2 separator.  Returns true on a usable split.
  bool split_geometric(const std::vector<int32_t>& V, std::vector<int32_t>& L,
                       std::vector<int32_t>& R, std::vector<int32_t>& Ssep) {
    double lo[3], hi[3];
    for (int a = 0; a < 3; ++a) { lo[a] = 1e300; hi[a] = -1e300; }
    for (int32_t v : V)
      for (int a = 0; a < 3; ++a) {
        lo[a] = std::min(lo[a], xyz[3 * (int64_t)v + a]);
        hi[a] = std::max(hi[a], xyz[3 * (int64_t)v + a]);
      }
    int ax = 0;
    for (int a = 1; a < 3; ++a)
      if (hi[a] - lo[a] > hi[ax] - lo[ax]) ax = a;
    double ext = hi[ax] - lo[ax];
    if (ext <= 0) return false;
    std::vector<double> xs(V.size());
    for (size_t k = 0; k < V.size(); ++k) xs[k] = xyz[3 * (int64_t)V[k] + ax];
    std::vector<double> srt = xs;
    std::sort(srt.begin(), srt.end());
    srt.erase(std::unique(srt.begin(), srt.end()), srt.end());
    // candidate planes: distinct coordinates nearest the median value
    double med;
    {
      std::vector<double> tmp = xs;
      std::nth_element(tmp.begin(), tmp.begin() + tmp.size() / 2, tmp.end());
      med = tmp[tmp.size() / 2];
    }
    size_t mi = std::lower_bound(srt.begin(), srt.end(), med) - srt.begin();
    std::vector<double> cands;
    for (int d = -4; d <= 4; ++d) {
      long k = (long)mi + d;
      if (k > 0 && k < (long)srt.size() - 1) cands.push_back(srt[k]);
    }
    const double tol = 1e-9 * std::max(1.0, ext);
    size_t best = SIZE_MAX;
    double best_bal = 0, best_c = 0;
    for (double c : cands) {
      // label
      ++cur;
      size_t nl = 0, nr = 0, nm = 0;
      for (size_t k = 0; k < V.size(); ++k) {
        int32_t v = V[k];
        stamp[v] = cur;
        if (xs[k] < c - tol) { side[v] = 0; ++nl; }
        else if (xs[k] > c + tol) { side[v] = 1; ++nr; }
        else { side[v] = 2; ++nm; }
      }
      size_t ncov = 0;
      for (int32_t v : V) {
        if (side[v] != 0) continue;
        for (int64_t e = ip[v]; e < ip[v + 1]; ++e) {
          int32_t u = ix[e];
          if (stamp[u] == cur && side[u] == 1) { ++ncov; break; }
        }
      }
      size_t sep = nm + ncov;
      size_t a = nl - ncov, b = nr;
      double bal = (double)std::min(a, b) / (double)V.size();
      if (bal < 0.2) continue;
      if (sep < best || (sep == best && bal > best_bal)) {
        best = sep; best_bal = bal; best_c = c;
      }
    }
    if (best == SIZE_MAX) return false;
    ++cur;
    for (size_t k = 0; k < V.size(); ++k) {
      int32_t v = V[k];
      stamp[v] = cur;
      side[v] = xs[k] < best_c - tol ? 0 : (xs[k] > best_c + tol ? 1 : 2);
    }
    for (int32_t v : V) {
      if (side[v] != 0) continue;
      for (int64_t e = ip[v]; e < ip[v + 1]; ++e) {
        int32_t u = ix[e];
        if (stamp[u] == cur && side[u] == 1) { side[v] = 3; break; }  // cover
      }
    }
    for (int32_t v : V) {
      int s = side[v];
      if (s == 0) L.push_back(v);
      else if (s == 1) R.push_back(v);
      else Ssep.push_back(v);
    }
    return !L.empty() && !R.empty();
  }

  int32_t bfs_far(const std::vector<int32_t>& V, int32_t src, std::vector<int32_t>& q) {
    for (int32_t v : V) dist[v] = -1;
    q.clear();
    q.push_back(src);
    dist[src] = 0;
    for (size_t h = 0; h < q.size(); ++h) {
      int32_t v = q[h];
      for (int64_t e = ip[v]; e < ip[v + 1]; ++e) {
        int32_t u = ix[e];
        if (stamp[u] == cur && dist[u] < 0) { dist[u] = dist[v] + 1; q.push_back(u); }
      }
    }
    return q.back();
  }

  bool split_bfs(const std::vector<int32_t>& V, std::vector<int32_t>& L,
                 std::vector<int32_t>& R, std::vector<int32_t>& Ssep) {
    ++cur;
    for (int32_t v : V) stamp[v] = cur;
    std::vector<int32_t> q;
    int32_t a = bfs_far(V, V[0], q);
    a = bfs_far(V, a, q);
    (void)a;
    int32_t D = dist[q.back()];
    if (D < 2) return false;
    std::vector<size_t> cnt(D + 1, 0);
    for (int32_t v : q) cnt[dist[v]]++;
    size_t acc = 0;
    int32_t lev = 1;
    for (int32_t d = 0; d <= D; ++d) {
      acc += cnt[d];
      if (acc * 2 >= q.size()) { lev = std::max(1, std::min(d, D - 1)); break; }
    }
    for (int32_t v : V) {
      int32_t d = dist[v];
      if (d < 0) R.push_back(v);          // other components: not adjacent to L
      else if (d < lev) L.push_back(v);
      else if (d > lev) R.push_back(v);
      else Ssep.push_back(v);
    }
    return !L.empty() && !R.empty();
  }

  std::vector<int32_t> build(std::vector<int32_t>& V) {
    if (V.empty()) return {};
    if ((int32_t)V.size() <= leaf) return {new_node(V, {})};
    std::vector<int32_t> L, R, Ssep;
    bool ok = xyz ? split_geometric(V, L, R, Ssep) : false;
    if (!ok) {
      L.clear(); R.clear(); Ssep.clear();
      ok = split_bfs(V, L, R, Ssep);
    }
    if (!ok) return {new_node(V, {})};
    std::vector<int32_t>().swap(V);
    std::vector<int32_t> kids = build(L);
    std::vector<int32_t> kr = build(R);
    kids.insert(kids.end(), kr.begin(), kr.end());
    if (Ssep.empty()) return kids;
    return {new_node(Ssep, kids)};
  }
};

struct FreeList {
  std::map<int64_t, int64_t> fl;  // off -> len
  int64_t top = 0;
  int64_t alloc(int64_t len) {
    for (auto it = fl.begin(); it != fl.end(); ++it) {
      if (it->second >= len) {
        int64_t off = it->first, rem = it->second - len;
        fl.erase(it);
        if (rem > 0) fl[off + len] = rem;
        return off;
      }
    }
    // extend, merging with a free tail block
    if (!fl.empty()) {
      auto last = std::prev(fl.end());
      if (last->first + last->second == top) {
        int64_t off = last->first;
        fl.erase(last);
        top = off + len;
        return off;
      }
    }
    int64_t off = top;
    top += len;
    return off;
  }
  void release(int64_t off, int64_t len) {
    auto it = fl.emplace(off, len).first;
    if (it != fl.begin()) {
      auto pv = std::prev(it);
      if (pv->first + pv->second == it->first) {
        pv->second += it->second;
        fl.erase(it);
        it = pv;
      }
    }
    auto nx = std::next(it);
    if (nx != fl.end() && it->first + it->second == nx->first) {
      it->second += nx->second;
      fl.erase(nx);
    }
  }
};

inline int64_t align16(int64_t x) { return (x + 15) & ~int64_t(15); }

}  // namespace

std::string analyze(int64_t n, const int64_t* indptr, const int32_t* indices,
                    const double* coords, int32_t leaf, Symbolic& S) {
  if (n <= 0) return "empty matrix";
  if (n > INT32_MAX - 1) return "n exceeds 32-bit index range";
  if (leaf < 1) leaf = 1;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e)
      if (indices[e] < 0 || indices[e] >= n) return "pattern index out of range";

  ND nd(n, indptr, indices, coords, leaf);
  std::vector<int32_t> V(n);
  std::iota(V.begin(), V.end(), 0);
  std::vector<int32_t> roots = nd.build(V);
  if ((int64_t)nd.order.size() != n) return "internal: dissection lost vertices";

  S = Symbolic();
  S.n = n;
  S.perm = nd.order;
  S.iperm.assign(n, 0);
  for (int64_t k = 0; k < n; ++k) S.iperm[S.perm[k]] = (int32_t)k;
  const int32_t nfr = (int32_t)nd.node_first.size();
  S.nfront = nfr;
  S.first = nd.node_first;
  S.npiv = nd.node_npiv;
  S.parent.assign(nfr, -1);
  S.child_ptr.assign(nfr + 1, 0);
  for (int32_t s = 0; s < nfr; ++s) {
    std::vector<int32_t> kids = nd.node_children[s];
    std::sort(kids.begin(), kids.end());
    for (int32_t c : kids) S.parent[c] = s;
    S.child_ptr[s + 1] = S.child_ptr[s] + (int32_t)kids.size();
    S.child_list.insert(S.child_list.end(), kids.begin(), kids.end());
  }
  (void)roots;

  // front row structures (postorder: node ids are created children-first)
  std::vector<int32_t> mk(n, -1);
  S.rows_off.assign(nfr + 1, 0);
  S.nf.assign(nfr, 0);
  std::vector<int32_t> border;
  for (int32_t s = 0; s < nfr; ++s) {
    const int32_t f0 = S.first[s], p = S.npiv[s], last = f0 + p - 1;
    border.clear();
    for (int32_t k = f0; k <= last; ++k) {
      int32_t old = S.perm[k];
      for (int64_t e = indptr[old]; e < indptr[old + 1]; ++e) {
        int32_t r = S.iperm[indices[e]];
        if (r > last && mk[r] != s) { mk[r] = s; border.push_back(r); }
      }
    }
    for (int32_t ci = S.child_ptr[s]; ci < S.child_ptr[s + 1]; ++ci) {
      int32_t c = S.child_list[ci];
      for (int64_t q = S.rows_off[c] + S.npiv[c]; q < S.rows_off[c + 1]; ++q) {
        int32_t r = S.rows[q];
        if (r > last && mk[r] != s) { mk[r] = s; border.push_back(r); }
        if (r >= f0 && r <= last) continue;
        if (r < f0) return "internal: child border below parent pivots";
      }
    }
    std::sort(border.begin(), border.end());
    for (int32_t k = f0; k <= last; ++k) S.rows.push_back(k);
    S.rows.insert(S.rows.end(), border.begin(), border.end());
    S.nf[s] = p + (int32_t)border.size();
    S.rows_off[s + 1] = S.rows_off[s] + S.nf[s];
  }
  // relative maps child -> parent
  S.rel_off.assign(nfr + 1, 0);
  for (int32_t s = 0; s < nfr; ++s) S.rel_off[s + 1] = S.rel_off[s] + (S.nf[s] - S.npiv[s]);
  S.relmap.assign(S.rel_off[nfr], 0);
  for (int32_t c = 0; c < nfr; ++c) {
    int32_t s = S.parent[c];
    if (s < 0) {
      if (S.nf[c] != S.npiv[c]) return "internal: root front with a border";
      continue;
    }
    const int32_t* prow = S.rows.data() + S.rows_off[s];
    const int32_t pnf = S.nf[s];
    for (int32_t k = 0; k < S.nf[c] - S.npiv[c]; ++k) {
      int32_t r = S.rows[S.rows_off[c] + S.npiv[c] + k];
      const int32_t* it = std::lower_bound(prow, prow + pnf, r);
      if (it == prow + pnf || *it != r) return "internal: child row missing from parent";
      S.relmap[S.rel_off[c] + k] = (int32_t)(it - prow);
    }
  }
  // levels
  S.level.assign(nfr, 0);
  int32_t maxlev = 0;
  for (int32_t s = 0; s < nfr; ++s) {
    int32_t lv = 0;
    for (int32_t ci = S.child_ptr[s]; ci < S.child_ptr[s + 1]; ++ci)
      lv = std::max(lv, S.level[S.child_list[ci]] + 1);
    S.level[s] = lv;
    maxlev = std::max(maxlev, lv);
  }
  S.nlevels = maxlev + 1;
  S.level_ptr.assign(S.nlevels + 1, 0);
  for (int32_t s = 0; s < nfr; ++s) S.level_ptr[S.level[s] + 1]++;
  for (int32_t l = 0; l < S.nlevels; ++l) S.level_ptr[l + 1] += S.level_ptr[l];
  S.level_fronts.assign(nfr, 0);
  {
    std::vector<int32_t> pos(S.level_ptr.begin(), S.level_ptr.end() - 1);
    for (int32_t s = 0; s < nfr; ++s) S.level_fronts[pos[S.level[s]]++] = s;
  }
  // memory plans and statistics
  S.panel_off.assign(nfr + 1, 0);
  S.uvec_off.assign(nfr + 1, 0);
  S.upd_off.assign(nfr, -1);
  double fl = 0;
  int64_t nnzL = 0;
  for (int32_t s = 0; s < nfr; ++s) {
    int64_t p = S.npiv[s], f = S.nf[s], r = f - p;
    S.panel_off[s + 1] = S.panel_off[s] + align16(f * p);
    S.uvec_off[s + 1] = S.uvec_off[s] + r;
    double pd = (double)p, rd = (double)r;
    fl += 8.0 * (pd * pd * pd / 6.0 + rd * pd * pd / 2.0 + rd * rd * pd / 2.0);
    nnzL += p * f - p * (p - 1) / 2;
    S.max_nf = std::max<int32_t>(S.max_nf, (int32_t)f);
    S.max_npiv = std::max<int32_t>(S.max_npiv, (int32_t)p);
  }
  S.flops = fl;
  S.nnzL = nnzL;
  FreeList fls;
  for (int32_t l = 0; l < S.nlevels; ++l) {
    for (int32_t q = S.level_ptr[l]; q < S.level_ptr[l + 1]; ++q) {
      int32_t s = S.level_fronts[q];
      if (S.parent[s] < 0) continue;
      int64_t r = S.nf[s] - S.npiv[s];
      S.upd_off[s] = fls.alloc(align16(std::max<int64_t>(r * (r + 1) / 2, 1)));
    }
    for (int32_t q = S.level_ptr[l]; q < S.level_ptr[l + 1]; ++q) {
      int32_t s = S.level_fronts[q];
      for (int32_t ci = S.child_ptr[s]; ci < S.child_ptr[s + 1]; ++ci) {
        int32_t c = S.child_list[ci];
        int64_t r = S.nf[c] - S.npiv[c];
        fls.release(S.upd_off[c], align16(std::max<int64_t>(r * (r + 1) / 2, 1)));
      }
    }
  }
  S.upd_total = std::max<int64_t>(fls.top, 16);
  return "";
}

}  // namespace rba
