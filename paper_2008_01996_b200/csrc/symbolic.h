// Host-side symbolic analysis for the batched multifrontal LDL^T.
//
// Replaces the reference's `sparse_direct.analyze` (pkg/src/kronheat/
// sparse_direct.py:112-152: MMD ordering via SuperLU on a stand-in matrix +
// etree postorder) with a graph nested dissection whose separators become
// dense supernodal fronts. One analysis is shared by every shift
// M_x + lambda_k A_x (solvers.py:379), as in the reference.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace kh {

struct Front {
  int64_t first;   // first pivot position in the permuted order
  int32_t p;       // pivots (contiguous: first .. first+p-1)
  int32_t q;       // update rows (ancestor positions, sorted)
  int32_t depth;   // root = 0
  int32_t parent;  // -1 for roots
  int64_t rows_begin;   // into Symbolic::urows (q entries, permuted positions)
  int64_t relind_begin; // into Symbolic::relind (q entries, local index in parent)
  int64_t orig_begin, orig_end;  // into orig_src / orig_dst
  int64_t panel_off;    // complex offset of the m x p panel in per-shift factor storage
  int64_t upd_off;      // complex offset of the q x q update in its depth-parity buffer
  int64_t rupd_off;     // complex offset of the q rhs-update in its depth-parity buffer
  int64_t cmap_begin;   // into Symbolic::cmap: parent's m local rows -> this front's update index or -1
  int32_t m() const { return p + q; }
};

struct Symbolic {
  int64_t n = 0;
  int64_t nnz = 0;                 // entries of the analyzed CSR (values arrays are aligned to it)
  // the analyzed CSR: the input pattern made symmetric (A | A^T), with the
  // full diagonal, rows sorted, no duplicates
  std::vector<int64_t> pat_ptr, pat_idx;
  std::vector<int64_t> perm;       // perm[k] = original index eliminated k-th
  std::vector<int64_t> iperm;      // iperm[orig] = k
  std::vector<Front> fronts;       // postorder (children before parents)
  std::vector<int32_t> child_ptr;  // fronts.size()+1
  std::vector<int32_t> child_list;
  std::vector<int64_t> urows;      // update-row positions per front
  std::vector<int32_t> relind;     // child update row -> parent local row
  std::vector<int32_t> cmap;       // inverse of relind per child, over the parent's m rows (-1 = absent)
  std::vector<int64_t> orig_src;   // CSR entry index
  std::vector<int32_t> orig_dst;   // local (row + col*m) inside the front panel
  std::vector<std::vector<int32_t>> levels;  // levels[d] = fronts at depth d
  int32_t max_depth = 0;
  int64_t panel_total = 0;         // complex entries per shift (all panels)
  int64_t upd_size[2] = {0, 0};    // complex entries per shift, per parity buffer
  int64_t rupd_size[2] = {0, 0};
  int64_t factor_nnz = 0;          // lower-triangle entries of L incl. diagonal
  double flops = 0.0;              // real flops per shift for complex LDL^T
  int32_t max_front = 0;
  int32_t leaf_size = 0;
};

// Builds the analysis. Pattern is a square CSR (any symmetry; union-
// symmetrized internally). Returns empty string on success, else a message.
std::string analyze(int64_t n, const int64_t* indptr, const int64_t* indices,
                    int32_t leaf_size, Symbolic& out);

}  // namespace kh
