// Host preparation of a mesh for the device path: the symmetric pattern of
// A = K - xi M (element pattern U K), its lower triangle with K values and the
// M-assembly contribution lists, the symbolic analysis, the scatter targets of
// A entries into the front panels, and the permuted element data.  Pure host
// code (no CUDA), so it is testable without a GPU (rba_mesh_prepare).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "symbolic.h"

namespace rba {

struct MeshPrep {
  int64_t nnzA = 0;
  std::vector<int32_t> a_rows, a_cols;   // lower pattern, original numbering
  std::vector<double> Kv;                // K values on it
  std::vector<int64_t> mcnt, moff;       // M contributions (CSR over e, offsets c*36+a*6+b)
  std::vector<int64_t> tgt;              // panel offset of each lower entry
  std::vector<int32_t> cdp;              // P*6 permuted cell dofs
  std::vector<double> mass36;            // P*36
  std::vector<int64_t> pdcp;             // permuted dof -> items
  std::vector<int32_t> pdci;
  Symbolic sym;
};

std::string prepare_mesh(int64_t N, int64_t P, int32_t k, const int32_t* cell_dofs,
                         const double* mass_local, const int64_t* Kp, const int32_t* Ki,
                         const double* Kx, const double* coords, int32_t leaf, MeshPrep& M);

}  // namespace rba
