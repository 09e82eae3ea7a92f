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

/* Mesh description handed to an assembly backend (aspamg_set_assembly_backend,
 * aspamg_host.h; aspamg_gpu_assemble_hex, aspamg_gpu.h). */
typedef struct aspamg_hex_assembly {
    int64_t nx, ny, nz;        /* elements per axis; nodes are (nx+1)(ny+1)(nz+1), node = i + (nx+1)(j + (ny+1)k) */
    int64_t n_free;            /* free (unclamped) nodes; K is 3 n_free x 3 n_free, dofs interleaved */
    int32_t cube;              /* 1: undistorted cubes of spacing h, one stiffness per table entry (fem.cpp:153-158);
                                  0: one stiffness per element from its 8 node coordinates */
    double h;
    const double* node_xyz;    /* all nodes, row-major x y z */
    const int64_t* free_index; /* node -> free node id, or -1 (clamped) */
    const int64_t* free_node;  /* free node id -> node */
    const int32_t* el_ke;      /* element (ex + nx (ey + ny ez)) -> stiffness-table entry */
    int64_t n_ke;              /* stiffness-table entries (distinct materials, or elements) */
    const double* young;       /* per table entry */
    const double* poisson;
} aspamg_hex_assembly;

#endif
