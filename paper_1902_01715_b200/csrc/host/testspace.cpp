// Test space: RBM/random seeding and SRQCG (Alg. 4
// :522-563). test_space.cpp is missing from the reference.
#include "amg.hpp"
#include "smalldense.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>
#include <omp.h>

namespace aspamg {

namespace {

struct SOp {  // x -> G A G' x
    const Csr& A;
    const Csr& G;
    const Csr& Gt;
    mutable std::vector<double> t1, t2;
    SOp(const Csr& a, const Csr& g, const Csr& gt)
        : A(a), G(g), Gt(gt), t1(static_cast<size_t>(a.n_rows)), t2(static_cast<size_t>(a.n_rows)) {}
    void apply(const double* x, double* y) const {
        spmv(Gt, x, t1.data());
        spmv(A, t1.data(), t2.data());
        spmv(G, t2.data(), y);
    }
};

void axpy(index_t n, double a, const double* x, double* y) {
#pragma omp parallel for schedule(static) num_threads(num_threads()) if (n > 65536)
    for (index_t i = 0; i < n; ++i) y[i] += a * x[i];
}

}  // namespace

// SPEC.md:249-257
Dense seed_space(const Dense* rbms, index_t n_tv, index_t n, std::uint64_t seed) {
    const index_t r = rbms ? rbms->n_cols : 0;
    if (n_tv < r) throw ConfigError("seed_space: n_tv smaller than the number of RBMs");
    if (rbms && rbms->n_rows != n) throw DimensionError("seed_space: RBM rows mismatch");
    Dense V(n, n_tv);
    for (index_t j = 0; j < r; ++j) std::copy(rbms->colp(j), rbms->colp(j) + n, V.colp(j));
    Rng rng(seed);
    for (index_t j = r; j < n_tv; ++j)
        for (index_t i = 0; i < n; ++i) V(i, j) = rng.symmetric();
    return V;
}

// Alg. 4 on S = G A G'. q_i is the true Rayleigh quotient e/f (the algorithm
// keeps Z_i unnormalised between Ritz projections; its alpha formula already
// carries f = Z_i'Z_i). Fallback: Delta < 0 or |bc - ad| < 1e-300
// -> steepest-descent exact line search for that vector this iteration.
TestSpace srqcg(const Csr& A, const Csr& G, const Csr& Gt, const Dense& V0, const SrqcgConfig& cfg) {
    const index_t n = A.n_rows;
    if (V0.n_rows != n) throw DimensionError("srqcg: V0 rows mismatch");
    SOp S(A, G, Gt);
    TestSpace out;
    // Z0 = (I - S) V0, orthonormalised; lost columns replaced by seeded randoms.
    Dense Z(n, V0.n_cols);
    for (index_t j = 0; j < V0.n_cols; ++j) {
        S.apply(V0.colp(j), Z.colp(j));
        const double* v = V0.colp(j);
        double* z = Z.colp(j);
        for (index_t i = 0; i < n; ++i) z[i] = v[i] - z[i];
    }
    const index_t want = V0.n_cols;
    index_t dropped = orthonormalize_columns(Z);
    if (dropped > 0) {
        out.rank_collapse = true;
        Rng rng(derive_seed(cfg.seed, 77));
        Dense Z2(n, want);
        std::copy(Z.v.begin(), Z.v.end(), Z2.v.begin());
        for (index_t j = Z.n_cols; j < want; ++j)
            for (index_t i = 0; i < n; ++i) Z2(i, j) = rng.symmetric();
        Z = std::move(Z2);
        orthonormalize_columns(Z);
    }
    const index_t nt = Z.n_cols;
    Dense SZ(n, nt), P(n, nt), SP(n, nt), R(n, nt);
    std::vector<double> q(static_cast<size_t>(nt)), f(static_cast<size_t>(nt), 1.0);
    std::vector<char> conv(static_cast<size_t>(nt), 0);
    auto residual = [&](index_t i) {  // R_i = S Z_i - q Z_i, returns ||R_i|| <= tol |q| ||Z_i||
        const double e = dot(n, Z.colp(i), SZ.colp(i));
        f[static_cast<size_t>(i)] = dot(n, Z.colp(i), Z.colp(i));
        q[static_cast<size_t>(i)] = e / f[static_cast<size_t>(i)];
        const double qi = q[static_cast<size_t>(i)];
        const double* z = Z.colp(i);
        const double* sz = SZ.colp(i);
        double* r = R.colp(i);
#pragma omp parallel for schedule(static) num_threads(num_threads()) if (n > 65536)
        for (index_t k = 0; k < n; ++k) r[k] = sz[k] - qi * z[k];
        return norm2(n, r) <= cfg.residual_tol * std::fabs(qi) * std::sqrt(f[static_cast<size_t>(i)]);
    };
    for (index_t i = 0; i < nt; ++i) {
        S.apply(Z.colp(i), SZ.colp(i));
        conv[static_cast<size_t>(i)] = residual(i);
        double* p = P.colp(i);
        const double* r = R.colp(i);
        for (index_t k = 0; k < n; ++k) p[k] = 2.0 * r[k];
        f[static_cast<size_t>(i)] = 1.0;
        S.apply(P.colp(i), SP.colp(i));
    }
    bool all_conv = std::all_of(conv.begin(), conv.end(), [](char c) { return c != 0; });
    std::vector<double> gi(static_cast<size_t>(n));
    for (index_t k = 1; !all_conv && cfg.k_max > 0; ++k) {
        if (cfg.k_ritz > 0 && k % cfg.k_ritz == 0) {
            // Ritz projection (ZᵀSZ) U = (ZᵀZ) U Λ, Z <- Z U. Solved on an orthonormal
            // basis of span(Z): two-pass MGS of Z with the same column operations on
            // SZ (SZ stays S·Z without new S products); a column that collapses (the
            // per-vector minimisations drifting onto one eigenvector) is replaced by a
            // seeded random vector — the same rank-collapse rule as the entry step.
            const int m = static_cast<int>(nt);
            for (int j = 0; j < m; ++j) {
                double* zj = Z.colp(j);
                double* szj = SZ.colp(j);
                const double orig = norm2(n, zj);
                for (int pass = 0; pass < 2; ++pass)
                    for (int q = 0; q < j; ++q) {
                        const double cq = dot(n, Z.colp(q), zj);
                        axpy(n, -cq, Z.colp(q), zj);
                        axpy(n, -cq, SZ.colp(q), szj);
                    }
                double nr = norm2(n, zj);
                if (!(nr > 1e-10 * orig)) {
                    out.rank_collapse = true;
                    Rng rng(derive_seed(cfg.seed, 1000 + static_cast<std::uint64_t>(k) * 64 + static_cast<std::uint64_t>(j)));
                    for (index_t i = 0; i < n; ++i) zj[i] = rng.symmetric();
                    for (int pass = 0; pass < 2; ++pass)
                        for (int q = 0; q < j; ++q) axpy(n, -dot(n, Z.colp(q), zj), Z.colp(q), zj);
                    nr = norm2(n, zj);
                    S.apply(zj, szj);
                }
                const double inv = 1.0 / nr;
#pragma omp parallel for schedule(static) num_threads(num_threads()) if (n > 65536)
                for (index_t i = 0; i < n; ++i) {
                    zj[i] *= inv;
                    szj[i] *= inv;
                }
            }
            std::vector<double> M1(static_cast<size_t>(m) * m);
            for (int a1 = 0; a1 < m; ++a1)
                for (int b1 = 0; b1 <= a1; ++b1) {
                    const double v = 0.5 * (dot(n, Z.colp(a1), SZ.colp(b1)) + dot(n, Z.colp(b1), SZ.colp(a1)));
                    M1[static_cast<size_t>(a1) * m + b1] = M1[static_cast<size_t>(b1) * m + a1] = v;
                }
            std::vector<double> w(static_cast<size_t>(m)), U(static_cast<size_t>(m) * m);
            sym_eig(m, M1.data(), w.data(), U.data());
            Dense Zn(n, nt), SZn(n, nt);
#pragma omp parallel for schedule(static) num_threads(num_threads())
            for (index_t i = 0; i < n; ++i)
                for (int c = 0; c < m; ++c) {
                    double s1 = 0.0, s2 = 0.0;
                    for (int r = 0; r < m; ++r) {
                        s1 += Z(i, r) * U[static_cast<size_t>(r) * m + c];
                        s2 += SZ(i, r) * U[static_cast<size_t>(r) * m + c];
                    }
                    Zn(i, c) = s1;
                    SZn(i, c) = s2;
                }
            Z = std::move(Zn);
            SZ = std::move(SZn);
        }
        all_conv = true;
        for (index_t i = 0; i < nt; ++i) {
            double* z = Z.colp(i);
            double* sz = SZ.colp(i);
            double* p = P.colp(i);
            double* sp = SP.colp(i);
            double fi = dot(n, z, z);
            double a = 0, b = 0, c = 0, d = 0, e = 0, disc = 0, den = 0;
            auto coeffs = [&]() {
                a = dot(n, p, sz); b = dot(n, p, sp); c = dot(n, p, z); d = dot(n, p, p); e = dot(n, z, sz);
                den = b * c - a * d;
                disc = (d * e - b * fi) * (d * e - b * fi) - 4.0 * den * (a * fi - c * e);
            };
            coeffs();
            bool ok = disc >= 0.0 && std::fabs(den) >= 1e-300;
            if (!ok) {  // steepest descent along the current gradient
                const double qi = e / fi;
#pragma omp parallel for schedule(static) num_threads(num_threads()) if (n > 65536)
                for (index_t kk = 0; kk < n; ++kk) p[kk] = 2.0 * (sz[kk] - qi * z[kk]) / fi;
                S.apply(p, sp);
                coeffs();
                ok = disc >= 0.0 && std::fabs(den) >= 1e-300;
            }
            if (ok) {
                const double alpha = (d * e - b * fi + std::sqrt(disc)) / (2.0 * den);
                axpy(n, alpha, p, z);
                axpy(n, alpha, sp, sz);
            }
            conv[static_cast<size_t>(i)] = residual(i);
            if (!conv[static_cast<size_t>(i)]) all_conv = false;
            // gradient G_i = 2 R_i / f_i ; beta = -G_i' S P_i / b ; P_i = G_i + beta P_i
            const double inv = 2.0 / f[static_cast<size_t>(i)];
            const double* r = R.colp(i);
#pragma omp parallel for schedule(static) num_threads(num_threads()) if (n > 65536)
            for (index_t kk = 0; kk < n; ++kk) gi[static_cast<size_t>(kk)] = inv * r[kk];
            const double bb = dot(n, p, sp);
            const double beta = bb != 0.0 ? -dot(n, gi.data(), sp) / bb : 0.0;
#pragma omp parallel for schedule(static) num_threads(num_threads()) if (n > 65536)
            for (index_t kk = 0; kk < n; ++kk) p[kk] = gi[static_cast<size_t>(kk)] + beta * p[kk];
            S.apply(p, sp);
        }
        out.iterations = k;
        if (k >= cfg.k_max) break;
    }
    // Order by ascending quotient, V = G' Z, orthonormalise.
    std::vector<index_t> ord(static_cast<size_t>(nt));
    std::iota(ord.begin(), ord.end(), index_t{0});
    std::stable_sort(ord.begin(), ord.end(), [&](index_t x, index_t y) { return q[static_cast<size_t>(x)] < q[static_cast<size_t>(y)]; });
    Dense V(n, nt);
    for (index_t c = 0; c < nt; ++c) {
        spmv(Gt, Z.colp(ord[static_cast<size_t>(c)]), V.colp(c));
        out.quotients.push_back(q[static_cast<size_t>(ord[static_cast<size_t>(c)])]);
    }
    if (orthonormalize_columns(V) > 0) out.rank_collapse = true;
    out.quotients.resize(static_cast<size_t>(V.n_cols));
    out.V = std::move(V);
    return out;
}

}  // namespace aspamg
