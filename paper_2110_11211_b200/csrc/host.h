// Host-side setup structures: sparse patterns, the supernodal block-inverse
// factor and the ordering / factorization entry points (host C++, threaded).
#pragma once
#include <cstdint>
#include <vector>

namespace sfcdd {

// full symmetric sparsity pattern (both triangles; diagonal optional)
struct SymPattern {
  int64_t n = 0;
  std::vector<int64_t> indptr;
  std::vector<int32_t> indices;
};

// full symmetric matrix in CSR (both triangles)
struct CsrMatrix {
  int64_t n = 0;
  std::vector<int64_t> indptr;
  std::vector<int32_t> indices;
  std::vector<double> data;
};

std::vector<int32_t> amd_order(const SymPattern& A);
// hybrid nested dissection (BFS level-set separators, AMD on parts <= leaf)
std::vector<int32_t> nd_order(const SymPattern& A, int32_t leaf);

// One supernode of the block-inverse factor.  Columns col0..col0+s-1 of the
// permuted matrix; m below rows.  The stored block is
//     M = [ L_JJ^{-1} ; L_BJ L_JJ^{-1} ]      ((s+m) x s, lower trapezoid)
// packed column-major: column k holds rows k..s+m-1 (s+m-k values).
// Forward:  out = M f_J;  y_J = out[:s];  u_J = f_B - out[s:]
// Backward: x_J = M^T [y_J ; -x_B]
struct Supernode {
  int32_t s = 0, m = 0;
  int64_t col0 = 0;
  int64_t rows_off = 0;  // into HostFactor::rows (m entries, permuted indices)
  int64_t val_off = 0;   // into HostFactor::val
  int64_t rel_off = 0;   // into HostFactor::rel: positions of rows in parent's frontal
  int32_t parent = -1;
  int32_t level = 0;     // height above the leaves (0 = leaf)
};

#ifdef __CUDACC__
#define SFCDD_HD __host__ __device__
#else
#define SFCDD_HD
#endif
SFCDD_HD inline int64_t packed_size(int64_t s, int64_t m) { return s * (s + 1) / 2 + s * m; }
SFCDD_HD inline int64_t packed_col_off(int64_t s, int64_t m, int64_t k) {
  return k * (s + m) - k * (k - 1) / 2;
}

struct HostFactor {
  int64_t n = 0;
  std::vector<int32_t> perm;   // perm[new] = original index
  std::vector<Supernode> sn;   // postorder: children precede parents
  std::vector<int32_t> rows;   // below rows (permuted numbering), ascending
  std::vector<int32_t> rel;    // per supernode: m positions in the parent's frontal
  std::vector<double> val;     // packed M blocks
  std::vector<int32_t> child_ptr, child_list;
  int64_t nnz_l = 0;   // nnz(L) incl. diagonal, fundamental supernodes (no zeros)
  int64_t stored = 0;  // stored entries (with amalgamation zeros)
  int32_t max_front = 0;
};

struct FactorOptions {
  // relaxed amalgamation: merge child into parent when the merged block has
  // at most `relax_small` columns and zero fraction <= relax_small_frac, or
  // zero fraction <= relax_frac.  Environment overrides (tuning):
  // SFCDD_RELAX_SMALL, SFCDD_RELAX_SMALL_FRAC, SFCDD_RELAX_FRAC.
  int32_t relax_small = 16;
  double relax_small_frac = 0.30;
  double relax_frac = 0.02;
  // fill-reducing ordering: 0 = AMD, 1 = hybrid nested dissection (SFCDD_ORDER=amd|nd,
  // SFCDD_ND_LEAF = part size below which AMD takes over)
  int32_t ordering = 1;
  int32_t nd_leaf = 64;
  FactorOptions();
};

// order + symbolic + numeric; throws Error(SFCDD_EFACTOR) if not SPD
HostFactor factorize_host(const CsrMatrix& A, const FactorOptions& opt);
// symbolic only (sizes, structure); val left empty
HostFactor analyze_host(const CsrMatrix& A, const FactorOptions& opt);
void numeric_host(const CsrMatrix& A, HostFactor& F);
// x = A^{-1} b with the block-inverse factor, same arithmetic order as the
// device DAG kernel (test hook / coarse inverse)
void host_block_solve(const HostFactor& F, const double* b, double* x);

int hardware_threads();

// partition.cpp (partition.py:64-157)
void partition_ranges(int64_t n, int32_t p, int64_t gnum, int64_t gden, std::vector<int64_t>& dj_start,
                      std::vector<int64_t>& dj_len, std::vector<int64_t>& ov_start, std::vector<int64_t>& ov_len);
void partition_weights(int64_t n, int32_t p, const int64_t* ov_start, const int64_t* ov_len, int32_t* counts,
                       double* omega);

}  // namespace sfcdd
