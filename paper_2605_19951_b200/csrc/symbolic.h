// Host symbolic analysis for the supernodal multifrontal complex-symmetric
// LDL^T of A_i = K - xi_i M(m)  (replaces SuperLU's COLAMD + symbolic phase
// inside spla.splu, /root/reference/pkg/src/rbainv/shifted.py:54).
//
// Nested dissection (geometric when dof coordinates are given, BFS level-set
// otherwise) -> assembly tree whose nodes are the dissection nodes (relaxed
// supernodes: a separator or a leaf block is one dense front) -> front row
// structures, child->parent relative maps, level schedule, and memory plans.
// The same structure is shared by every pole and every model (only values
// change), so it is computed once per mesh.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace rba {

struct Symbolic {
  int64_t n = 0;
  std::vector<int32_t> perm;    // perm[new] = old
  std::vector<int32_t> iperm;   // iperm[old] = new
  int32_t nfront = 0;
  // per front, postorder (children before parents)
  std::vector<int32_t> first, npiv, nf, parent, level;
  std::vector<int64_t> rows_off;   // nfront + 1
  std::vector<int32_t> rows;       // permuted indices, sorted; first npiv are pivots
  std::vector<int32_t> child_ptr;  // nfront + 1
  std::vector<int32_t> child_list; // ascending front id
  std::vector<int64_t> rel_off;    // nfront + 1 ; (nf - npiv) entries per front
  std::vector<int32_t> relmap;     // local row in parent of rows[npiv + k]
  std::vector<int64_t> panel_off;  // nfront + 1 ; nf*npiv complex entries per front
  std::vector<int64_t> upd_off;    // per front offset into the update arena (-1: root);
                                   // packed lower-triangular blocks of order nf - npiv
  int64_t upd_total = 0;           // complex entries
  std::vector<int64_t> uvec_off;   // nfront + 1 ; (nf - npiv) per front (solve arena)
  int32_t nlevels = 0;
  std::vector<int32_t> level_ptr;  // nlevels + 1
  std::vector<int32_t> level_fronts;
  // statistics
  double flops = 0;       // SURVEY §8d formula, real flops per factorisation
  int64_t nnzL = 0;       // lower incl. diagonal, dense fronts
  int32_t max_nf = 0, max_npiv = 0;
};

// pattern: symmetric CSR (both triangles; diagonal optional), n x n.
// coords: n*3 doubles or nullptr.  leaf: max pivots in a leaf block.
// Returns empty string on success, else an error message.
std::string analyze(int64_t n, const int64_t* indptr, const int32_t* indices,
                    const double* coords, int32_t leaf, Symbolic& S);

}  // namespace rba
