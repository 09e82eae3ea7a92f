// Host-side core types for the aSP-AMG setup that feeds the B200 solve.
//
// CSR carrier, error hierarchy and seeded RNG restated from the reference's
// runtime layer so the hierarchy handed to the GPU has exactly the reference
// layout:
//   * CSR (int64 offsets/cols, fp64 values, full symmetric pattern):
//     /root/reference/proj/core/include/aspamg/sparse_matrix.hpp:27-59
//   * errors: types.hpp:15-41 ; index_t = int64: types.hpp:13
//   * Rng (mt19937_64, top-53-bit uniform) + splitmix64 derive_seed:
//     random.hpp:13-38
// Threads: OpenMP static row partitions; every per-row reduction keeps a fixed
// order so results are bit-identical at any thread count (parallel.hpp:4-6).
#pragma once

#include <cmath>
#include <cstdint>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace aspamg {

using index_t = std::int64_t;

struct DimensionError : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct NotSpdError : std::runtime_error { using std::runtime_error::runtime_error; };
struct NumericalError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ConfigError : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct IoError : std::runtime_error {
    index_t line = 0;
    IoError(const std::string& m, index_t l = 0)
        : std::runtime_error(l > 0 ? m + " (line " + std::to_string(l) + ")" : m), line(l) {}
};

// CSR with sorted, duplicate-free columns per row.
struct Csr {
    index_t n_rows = 0;
    index_t n_cols = 0;
    std::vector<index_t> rowptr;  // n_rows + 1
    std::vector<index_t> col;
    std::vector<double> val;
    bool symmetric = false;

    index_t nnz() const { return static_cast<index_t>(col.size()); }
    double nnz_per_row() const { return n_rows ? double(nnz()) / double(n_rows) : 0.0; }
    index_t row_begin(index_t i) const { return rowptr[static_cast<size_t>(i)]; }
    index_t row_end(index_t i) const { return rowptr[static_cast<size_t>(i) + 1]; }
    double at(index_t i, index_t j) const;  // 0 if not stored

    static Csr identity(index_t n);
    static Csr diagonal(const std::vector<double>& d);
};

// y = A x, ascending column order per row (sparse_matrix.cpp:96-107 semantics).
void spmv(const Csr& A, const double* x, double* y);
// Counting-sort transpose (sparse_matrix.cpp:168-189 semantics: deterministic).
Csr transpose(const Csr& A);
void transpose_into(const Csr& A, Csr& T);  // same, reusing T's buffers
// C = A B, per-row accumulator; first-touch order; sorted output
// (sparse_matrix.cpp:132-166 semantics, row-parallel).
Csr sparse_multiply(const Csr& A, const Csr& B);
// A_c = P' (A P) (sparse_matrix.cpp:191-199 semantics).
Csr galerkin_triple(const Csr& P, const Csr& A);

// Rng stream identical to random.hpp:13-27 (std::mt19937_64 is fully specified).
class Rng {
public:
    explicit Rng(std::uint64_t seed) : engine_(seed) {}
    std::uint64_t next_u64() { return engine_(); }
    double uniform() { return static_cast<double>(engine_() >> 11) * 0x1.0p-53; }
    double symmetric() { return 2.0 * uniform() - 1.0; }
    // Box-Muller on uniform() (the reference RNG has no Gaussian).
    double gaussian() {
        if (has_spare_) { has_spare_ = false; return spare_; }
        const double u1 = 1.0 - uniform();  // (0, 1]
        const double u2 = uniform();
        const double rad = std::sqrt(-2.0 * std::log(u1));
        const double ang = 6.283185307179586476925286766559 * u2;
        spare_ = rad * std::sin(ang);
        has_spare_ = true;
        return rad * std::cos(ang);
    }

private:
    std::mt19937_64 engine_;
    bool has_spare_ = false;
    double spare_ = 0.0;
};

inline std::uint64_t derive_seed(std::uint64_t seed, std::uint64_t salt) {
    std::uint64_t z = seed + salt * 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

int num_threads();
void set_num_threads(int n);

// Dense column-major block (test spaces, RBMs): n_rows x n_cols.
struct Dense {
    index_t n_rows = 0, n_cols = 0;
    std::vector<double> v;
    Dense() = default;
    Dense(index_t r, index_t c) : n_rows(r), n_cols(c), v(static_cast<size_t>(r * c), 0.0) {}
    double& operator()(index_t i, index_t j) { return v[static_cast<size_t>(i + j * n_rows)]; }
    double operator()(index_t i, index_t j) const { return v[static_cast<size_t>(i + j * n_rows)]; }
    double* colp(index_t j) { return v.data() + j * n_rows; }
    const double* colp(index_t j) const { return v.data() + j * n_rows; }
    void resize_cols(index_t c) { n_cols = c; v.resize(static_cast<size_t>(n_rows * c)); }
};

// Modified Gram-Schmidt with one re-orthogonalization pass; columns whose
// remainder is <= drop_tol * original norm are dropped (dense.cpp:5-23
// semantics). Returns the number of dropped columns.
index_t orthonormalize_columns(Dense& B, double drop_tol = 1e-12);

double dot(index_t n, const double* a, const double* b);
double norm2(index_t n, const double* a);

}  // namespace aspamg
