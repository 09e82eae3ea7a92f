// Host CSR kernels used by the setup (Galerkin products, transposes, the
// Lanczos / SRQCG operator applications). Semantics follow
// /root/reference/proj/core/src/sparse_matrix.cpp (cited per function); the
// row loops are OpenMP-parallel but every per-row reduction keeps the
// reference's order, so outputs are bit-identical to the sequential reference.
#include "core.hpp"

#include <algorithm>
#include <numeric>
#include <omp.h>

namespace aspamg {

namespace {
int g_threads = 0;  // 0 = OpenMP default
}

int num_threads() { return g_threads > 0 ? g_threads : omp_get_max_threads(); }
void set_num_threads(int n) {
    g_threads = n < 1 ? 0 : n;
    if (n >= 1) omp_set_num_threads(n);
}

double Csr::at(index_t i, index_t j) const {
    auto b = col.begin() + row_begin(i), e = col.begin() + row_end(i);
    auto it = std::lower_bound(b, e, j);
    if (it == e || *it != j) return 0.0;
    return val[static_cast<size_t>(it - col.begin())];
}

Csr Csr::identity(index_t n) {
    Csr m;
    m.n_rows = m.n_cols = n;
    m.symmetric = true;
    m.rowptr.resize(static_cast<size_t>(n) + 1);
    m.col.resize(static_cast<size_t>(n));
    m.val.assign(static_cast<size_t>(n), 1.0);
    std::iota(m.rowptr.begin(), m.rowptr.end(), index_t{0});
    std::iota(m.col.begin(), m.col.end(), index_t{0});
    return m;
}

Csr Csr::diagonal(const std::vector<double>& d) {
    Csr m = identity(static_cast<index_t>(d.size()));
    m.val = d;
    return m;
}

// sparse_matrix.cpp:96-107
void spmv(const Csr& A, const double* x, double* y) {
    const index_t n = A.n_rows;
    const index_t* rp = A.rowptr.data();
    const index_t* ci = A.col.data();
    const double* v = A.val.data();
#pragma omp parallel for schedule(static) num_threads(num_threads()) if (n > 4096)
    for (index_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (index_t k = rp[i]; k < rp[i + 1]; ++k) s += v[k] * x[ci[k]];
        y[i] = s;
    }
}

// sparse_matrix.cpp:168-189 (counting sort; rows of T in ascending source row).
// Parallel over contiguous source-row chunks: chunk t's entries of column c go
// after those of chunks < t, so every row of T is still in ascending source row
// (the same T as the sequential counting sort).
Csr transpose(const Csr& A) {
    Csr T;
    transpose_into(A, T);
    return T;
}

void transpose_into(const Csr& A, Csr& T) {
    T.n_rows = A.n_cols;
    T.n_cols = A.n_rows;
    T.symmetric = A.symmetric;
    const size_t nc = static_cast<size_t>(A.n_cols);
    T.rowptr.assign(nc + 1, 0);
    T.col.resize(A.col.size());
    T.val.resize(A.val.size());
    const size_t nnz = A.col.size();
    int nt = (nnz < (1u << 20) || nc == 0) ? 1 : std::min(num_threads(), 16);
    // chunk boundaries by nnz
    std::vector<index_t> rb(static_cast<size_t>(nt) + 1, A.n_rows);
    rb[0] = 0;
    for (int t = 1; t < nt; ++t) {
        const index_t target = static_cast<index_t>(nnz * static_cast<size_t>(t) / static_cast<size_t>(nt));
        rb[static_cast<size_t>(t)] = std::lower_bound(A.rowptr.begin(), A.rowptr.end(), target) - A.rowptr.begin();
        rb[static_cast<size_t>(t)] = std::min(std::max(rb[static_cast<size_t>(t)], rb[static_cast<size_t>(t) - 1]), A.n_rows);
    }
    std::vector<std::vector<index_t>> cnt(static_cast<size_t>(nt));
#pragma omp parallel num_threads(nt)
    {
        const int tid = omp_get_thread_num(), nthr = omp_get_num_threads();
        for (int t = tid; t < nt; t += nthr) {  // chunk t (the team may be smaller than nt)
            std::vector<index_t>& c = cnt[static_cast<size_t>(t)];
            c.assign(nc, 0);
            for (index_t k = A.row_begin(rb[static_cast<size_t>(t)]); k < A.row_begin(rb[static_cast<size_t>(t) + 1]); ++k)
                ++c[static_cast<size_t>(A.col[static_cast<size_t>(k)])];
        }
#pragma omp barrier
#pragma omp for schedule(static)
        for (size_t j = 0; j < nc; ++j) {  // per column: chunk offsets (exclusive), total
            index_t s = 0;
            for (int u = 0; u < nt; ++u) {
                const index_t v = cnt[static_cast<size_t>(u)][j];
                cnt[static_cast<size_t>(u)][j] = s;
                s += v;
            }
            T.rowptr[j + 1] = s;
        }
#pragma omp single
        std::partial_sum(T.rowptr.begin(), T.rowptr.end(), T.rowptr.begin());
        for (int t = tid; t < nt; t += nthr) {
            std::vector<index_t>& c = cnt[static_cast<size_t>(t)];
            for (index_t i = rb[static_cast<size_t>(t)]; i < rb[static_cast<size_t>(t) + 1]; ++i)
                for (index_t k = A.row_begin(i); k < A.row_end(i); ++k) {
                    const size_t j = static_cast<size_t>(A.col[static_cast<size_t>(k)]);
                    const index_t p = T.rowptr[j] + c[j]++;
                    T.col[static_cast<size_t>(p)] = i;
                    T.val[static_cast<size_t>(p)] = A.val[static_cast<size_t>(k)];
                }
        }
    }
}

// sparse_matrix.cpp:132-166. Row-parallel: each thread owns a dense
// accumulator; the per-row accumulation order (A row ascending, then B row
// ascending, first touch resets to 0.0) is the reference's, so the result is
// bit-identical to the sequential reference.
Csr sparse_multiply(const Csr& A, const Csr& B) {
    if (A.n_cols != B.n_rows) throw DimensionError("product A*B: A has " + std::to_string(A.n_cols) + " columns but B has " + std::to_string(B.n_rows) + " rows");
    Csr C;
    C.n_rows = A.n_rows;
    C.n_cols = B.n_cols;
    const index_t n = A.n_rows;
    const int nt = num_threads();
    // Pass 1: row counts. Pass 2: fill. Chunked so each thread keeps one accumulator.
    std::vector<index_t> counts(static_cast<size_t>(n) + 1, 0);
    std::vector<std::vector<index_t>> tcols(static_cast<size_t>(nt));
    std::vector<std::vector<double>> tvals(static_cast<size_t>(nt));
    std::vector<index_t> tbeg(static_cast<size_t>(nt) + 1, 0);
    const index_t chunk = (n + nt - 1) / std::max(nt, 1);
#pragma omp parallel num_threads(nt)
    {
        const int t = omp_get_thread_num();
        const index_t lo = std::min(n, t * chunk), hi = std::min(n, lo + chunk);
        std::vector<double> acc(static_cast<size_t>(B.n_cols), 0.0);
        std::vector<char> mark(static_cast<size_t>(B.n_cols), 0);
        std::vector<index_t> cols;
        auto& oc = tcols[static_cast<size_t>(t)];
        auto& ov = tvals[static_cast<size_t>(t)];
        for (index_t i = lo; i < hi; ++i) {
            cols.clear();
            for (index_t ka = A.row_begin(i); ka < A.row_end(i); ++ka) {
                const index_t tt = A.col[static_cast<size_t>(ka)];
                const double a = A.val[static_cast<size_t>(ka)];
                for (index_t kb = B.row_begin(tt); kb < B.row_end(tt); ++kb) {
                    const index_t j = B.col[static_cast<size_t>(kb)];
                    if (!mark[static_cast<size_t>(j)]) {
                        mark[static_cast<size_t>(j)] = 1;
                        acc[static_cast<size_t>(j)] = 0.0;
                        cols.push_back(j);
                    }
                    acc[static_cast<size_t>(j)] += a * B.val[static_cast<size_t>(kb)];
                }
            }
            std::sort(cols.begin(), cols.end());
            for (index_t j : cols) {
                oc.push_back(j);
                ov.push_back(acc[static_cast<size_t>(j)]);
                mark[static_cast<size_t>(j)] = 0;
            }
            counts[static_cast<size_t>(i) + 1] = static_cast<index_t>(cols.size());
        }
    }
    std::partial_sum(counts.begin(), counts.end(), counts.begin());
    C.rowptr = std::move(counts);
    C.col.resize(static_cast<size_t>(C.rowptr.back()));
    C.val.resize(static_cast<size_t>(C.rowptr.back()));
#pragma omp parallel num_threads(nt)
    {
        const int t = omp_get_thread_num();
        const index_t lo = std::min(n, t * chunk);
        const auto& oc = tcols[static_cast<size_t>(t)];
        const auto& ov = tvals[static_cast<size_t>(t)];
        if (!oc.empty()) {
            std::copy(oc.begin(), oc.end(), C.col.begin() + C.rowptr[static_cast<size_t>(lo)]);
            std::copy(ov.begin(), ov.end(), C.val.begin() + C.rowptr[static_cast<size_t>(lo)]);
        }
    }
    return C;
}

// sparse_matrix.cpp:191-199
Csr galerkin_triple(const Csr& P, const Csr& A) {
    if (P.n_rows != A.n_rows || A.n_rows != A.n_cols)
        throw DimensionError("Galerkin product: A must be square with as many rows as P");
    const Csr AP = sparse_multiply(A, P);
    const Csr Pt = transpose(P);
    Csr C = sparse_multiply(Pt, AP);
    C.symmetric = A.symmetric;
    return C;
}

// dense.cpp:5-23 semantics (2-pass MGS, drop on small remainder, order kept).
index_t orthonormalize_columns(Dense& B, double drop_tol) {
    const index_t n = B.n_rows, m = B.n_cols;
    index_t kept = 0;
    std::vector<double> v(static_cast<size_t>(n));
    for (index_t j = 0; j < m; ++j) {
        std::copy(B.colp(j), B.colp(j) + n, v.begin());
        const double original = norm2(n, v.data());
        for (int pass = 0; pass < 2; ++pass)
            for (index_t q = 0; q < kept; ++q) {
                const double c = dot(n, B.colp(q), v.data());
                const double* bq = B.colp(q);
#pragma omp parallel for schedule(static) num_threads(num_threads()) if (n > 65536)
                for (index_t i = 0; i < n; ++i) v[static_cast<size_t>(i)] -= c * bq[i];
            }
        const double rem = norm2(n, v.data());
        if (original == 0.0 || rem <= drop_tol * original) continue;
        double* dst = B.colp(kept);
        for (index_t i = 0; i < n; ++i) dst[i] = v[static_cast<size_t>(i)] / rem;
        ++kept;
    }
    const index_t dropped = m - kept;
    B.resize_cols(kept);
    return dropped;
}

// Deterministic parallel dot: fixed 8192-element chunks summed sequentially
// within a chunk, chunk partials summed in index order -> independent of the
// thread count.
double dot(index_t n, const double* a, const double* b) {
    constexpr index_t CH = 8192;
    const index_t nc = (n + CH - 1) / CH;
    if (nc <= 1) {
        double s = 0.0;
        for (index_t i = 0; i < n; ++i) s += a[i] * b[i];
        return s;
    }
    std::vector<double> part(static_cast<size_t>(nc));
#pragma omp parallel for schedule(static) num_threads(num_threads())
    for (index_t c = 0; c < nc; ++c) {
        double s = 0.0;
        const index_t e = std::min(n, (c + 1) * CH);
        for (index_t i = c * CH; i < e; ++i) s += a[i] * b[i];
        part[static_cast<size_t>(c)] = s;
    }
    double s = 0.0;
    for (double p : part) s += p;
    return s;
}

double norm2(index_t n, const double* a) { return std::sqrt(dot(n, a, a)); }

}  // namespace aspamg
