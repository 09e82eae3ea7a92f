// Small dense kernels the setup needs and the reference delegated to Eigen
// (absent here, SURVEY.md §7 hard part 2): Cholesky, triangular solves,
// cyclic-Jacobi symmetric eigensolver. Row-major n x n, n <= a few hundred.
#pragma once

#include <vector>

namespace aspamg {

// In-place lower Cholesky of row-major SPD `a` (n x n). Returns the index of
// the first non-positive pivot, or -1 on success. The strict upper part is
// zeroed.
long cholesky_lower(int n, double* a);
// sum_k a[k] b[k] in the order of a 32-lane warp reduction: 32 strided partial
// sums combined by the xor butterfly (deterministic; the device aFSAI's order).
double dot_w32(const double* a, const double* b, int n);
// Solve L y = b in place (L row-major lower, leading dimension ld), in 32-row
// blocks: sequential panel products, right-looking inside the block (a warp's order).
void trsv_lower(int n, const double* L, int ld, double* b);
// Solve L' y = b in place, right-looking (b_k -= L_ik b_i, i descending).
void trsv_lower_t(int n, const double* L, int ld, double* b);

// Symmetric eigen-decomposition by cyclic Jacobi. `a` (row-major n x n) is
// destroyed; eigenvalues ascending in w, eigenvectors as columns of v
// (row-major, v[i*n + k] = component i of vector k).
void sym_eig(int n, double* a, double* w, double* v);

}  // namespace aspamg
