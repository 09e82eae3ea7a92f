// ref_shim.cpp — extern "C" handle API over the reference's OWN compiled
// sparse kernels (TEST INFRASTRUCTURE ONLY). Built by oracle/Makefile together
// with the unmodified /root/reference/proj/core/src/sparse_matrix.cpp into
// oracle/_ref/libaspamg_ref.so. Nothing from the reference is copied: this
// file only includes its header and calls its functions
// (sparse_matrix.hpp:27-84).
#include "aspamg/parallel.hpp"
#include "aspamg/sparse_matrix.hpp"

#include <cstdint>
#include <exception>

using aspamg::SparseMatrix;

extern "C" {

void* ref_csr_create(int64_t n_rows, int64_t n_cols, const int64_t* rp, const int64_t* ci, const double* v) {
    auto* m = new SparseMatrix;
    m->n_rows = n_rows;
    m->n_cols = n_cols;
    m->row_offsets.assign(rp, rp + n_rows + 1);
    m->col_indices.assign(ci, ci + rp[n_rows]);
    m->values.assign(v, v + rp[n_rows]);
    return m;
}

void* ref_csr_from_triplets(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* r, const int64_t* c,
                            const double* v, int symmetric) {
    std::vector<aspamg::Triplet> t(static_cast<size_t>(nnz));
    for (int64_t k = 0; k < nnz; ++k) t[static_cast<size_t>(k)] = {r[k], c[k], v[k]};
    return new SparseMatrix(SparseMatrix::from_triplets(n_rows, n_cols, t, symmetric != 0));
}

void ref_csr_free(void* h) { delete static_cast<SparseMatrix*>(h); }

void ref_csr_shape(void* h, int64_t* n_rows, int64_t* n_cols, int64_t* nnz) {
    auto* m = static_cast<SparseMatrix*>(h);
    *n_rows = m->n_rows;
    *n_cols = m->n_cols;
    *nnz = m->nnz();
}

void ref_csr_copy(void* h, int64_t* rp, int64_t* ci, double* v) {
    auto* m = static_cast<SparseMatrix*>(h);
    std::copy(m->row_offsets.begin(), m->row_offsets.end(), rp);
    std::copy(m->col_indices.begin(), m->col_indices.end(), ci);
    std::copy(m->values.begin(), m->values.end(), v);
}

void ref_set_threads(int n) { aspamg::set_num_threads(n); }

// 0 ok, 1 DimensionError, 5 other
int ref_spmv_checked(void* h, const double* x, int64_t nx, double* y, int64_t ny) {
    auto* m = static_cast<SparseMatrix*>(h);
    try {
        aspamg::spmv(*m, std::span<const double>(x, static_cast<size_t>(nx)), std::span<double>(y, static_cast<size_t>(ny)));
        return 0;
    } catch (const aspamg::DimensionError&) { return 1; } catch (...) { return 5; }
}

// oracle hook signature: void(void* ref, const double* x, double* y)
void ref_spmv(void* h, const double* x, double* y) {
    auto* m = static_cast<SparseMatrix*>(h);
    aspamg::spmv(*m, std::span<const double>(x, static_cast<size_t>(m->n_cols)),
                 std::span<double>(y, static_cast<size_t>(m->n_rows)));
}

void ref_spmv_transpose(void* h, const double* x, double* y) {
    auto* m = static_cast<SparseMatrix*>(h);
    aspamg::spmv_transpose(*m, std::span<const double>(x, static_cast<size_t>(m->n_rows)),
                           std::span<double>(y, static_cast<size_t>(m->n_cols)));
}

void* ref_transpose(void* h) { return new SparseMatrix(aspamg::transpose(*static_cast<SparseMatrix*>(h))); }

void* ref_galerkin_triple(void* P, void* A) {
    return new SparseMatrix(aspamg::galerkin_triple(*static_cast<SparseMatrix*>(P), *static_cast<SparseMatrix*>(A)));
}

void* ref_sparse_multiply(void* A, void* B) {
    return new SparseMatrix(aspamg::sparse_multiply(*static_cast<SparseMatrix*>(A), *static_cast<SparseMatrix*>(B)));
}

int ref_lower_tri_solve_t(void* G, const double* x, double* y) {
    auto* m = static_cast<SparseMatrix*>(G);
    try {
        auto r = aspamg::lower_triangular_solve_transposed(*m, std::span<const double>(x, static_cast<size_t>(m->n_rows)));
        std::copy(r.begin(), r.end(), y);
        return 0;
    } catch (...) { return 3; }
}

}  // extern "C"
