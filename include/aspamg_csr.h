/* aspamg_csr.h — the CSR view shared by both C-ABIs: the reference's
 * SparseMatrix layout verbatim (sparse_matrix.hpp:27-33): int64 offsets and
 * column indices (sorted, duplicate-free per row), fp64 values. Borrowed
 * pointers only. */
#ifndef ASPAMG_CSR_H
#define ASPAMG_CSR_H

#include <stdint.h>

typedef struct aspamg_csr_view {
    int64_t n_rows;
    int64_t n_cols;
    int64_t nnz;
    const int64_t* row_offsets; /* n_rows + 1 */
    const int64_t* col_indices; /* nnz, sorted per row */
    const double* values;       /* nnz */
} aspamg_csr_view;

/* Output allocator for producers of a CSR whose size is known only after the
 * product (the GPU Galerkin backend): returns 0 and n_rows + 1 / nnz / nnz
 * writable buffers owned by `sink`. */
typedef int (*aspamg_csr_alloc_fn)(void* sink, int64_t n_rows, int64_t n_cols, int64_t nnz,
                                   int64_t** row_offsets, int64_t** col_indices, double** values);

#endif
