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

/* Parameters of the adaptive FSAI smoother set-up (fsai.hpp:27-42, SPEC.md:166-169,
 * 218-219,231): initial build (k0, rho0, eps0), refinement passes (ki, rhoi, epsi)
 * while omega < omega_bar and nnz/row < rho_bar (already resolved: > 0), Lanczos
 * steps and seed for lambda_max. */
typedef struct aspamg_smoother_params {
    int64_t k0, rho0;
    double eps0;
    int64_t ki, rhoi;
    double epsi;
    double omega_bar, rho_bar;
    int64_t lanczos_steps;
    uint64_t seed;
} aspamg_smoother_params;

#endif
