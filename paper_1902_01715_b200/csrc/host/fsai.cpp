// Adaptive FSAI smoother set-up (Alg. 3 :374-387).
// The reference declares this module (fsai.hpp:27-83) but fsai.cpp is missing.
#include "amg.hpp"
#include "smalldense.hpp"

#include <algorithm>
#include <cmath>
#include <omp.h>

namespace aspamg {

namespace {

struct RowWork {
    std::vector<double> dense;     // scatter buffer for one row of A (size n)
    std::vector<double> grad;      // gradient accumulator (size n)
    std::vector<char> gmark;       // touched flag for grad
    std::vector<index_t> touched;
    std::vector<double> L;         // incremental Cholesky of A[pat, pat], row-major, ld = cap
    int cap = 0;
    explicit RowWork(index_t n) : dense(static_cast<size_t>(n), 0.0), grad(static_cast<size_t>(n), 0.0),
                                  gmark(static_cast<size_t>(n), 0) {}
    void ensure(int m) {
        if (m <= cap) return;
        int nc = std::max(64, cap * 2);
        while (nc < m) nc *= 2;
        std::vector<double> nl(static_cast<size_t>(nc) * nc, 0.0);
        for (int i = 0; i < cap; ++i)
            for (int j = 0; j <= i; ++j) nl[static_cast<size_t>(i) * nc + j] = L[static_cast<size_t>(i) * cap + j];
        L.swap(nl);
        cap = nc;
    }
};

// Append index j to the pattern factor: row m of L from A[j, pat[0..m)].
bool chol_append(const Csr& A, RowWork& w, const std::vector<index_t>& pat, int m, index_t j) {
    w.ensure(m + 1);
    for (index_t k = A.row_begin(j); k < A.row_end(j); ++k)
        w.dense[static_cast<size_t>(A.col[static_cast<size_t>(k)])] = A.val[static_cast<size_t>(k)];
    double* row = &w.L[static_cast<size_t>(m) * w.cap];
    for (int q = 0; q < m; ++q) row[q] = w.dense[static_cast<size_t>(pat[static_cast<size_t>(q)])];
    const double ajj = w.dense[static_cast<size_t>(j)];
    for (index_t k = A.row_begin(j); k < A.row_end(j); ++k)
        w.dense[static_cast<size_t>(A.col[static_cast<size_t>(k)])] = 0.0;
    trsv_lower(m, w.L.data(), w.cap, row);
    const double d = ajj - dot_fixed4(row, row, m);
    if (!(d > 0.0)) return false;
    row[m] = std::sqrt(d);
    return true;
}

}  // namespace

// SPEC.md:172-180. Per row i: pattern P_i (< i) grows by up to rho entries
// per step for at most k steps, choosing the candidates j < i adjacent to
// P_i + {i} with the largest |(A g~)_j| (ties: smaller index); the row stops
// once the relative decrease of psi_i = 1/g~_last is <= eps. Final row is
// g~ / sqrt(g~_last), so diag(G A G') = 1.
Csr afsai_build(const Csr& A, const Csr* G_start, index_t k, index_t rho, double eps,
                std::vector<double>* psi_out) {
    if (A.n_rows != A.n_cols) throw DimensionError("afsai_build: A must be square");
    const index_t n = A.n_rows;
    if (G_start && G_start->n_rows != n) throw DimensionError("afsai_build: G_start size mismatch");
    std::vector<std::vector<index_t>> rcol(static_cast<size_t>(n));
    std::vector<std::vector<double>> rval(static_cast<size_t>(n));
    std::vector<double> psi_all(static_cast<size_t>(n), 0.0);
    index_t bad_row = -1;
#pragma omp parallel num_threads(num_threads())
    {
        RowWork w(n);
        std::vector<index_t> pat;     // insertion order (factor order)
        std::vector<double> y;
        std::vector<std::pair<double, index_t>> cand;
#pragma omp for schedule(dynamic, 256)
        for (index_t i = 0; i < n; ++i) {
            pat.clear();
            if (G_start) {
                for (index_t q = G_start->row_begin(i); q < G_start->row_end(i); ++q) {
                    const index_t c = G_start->col[static_cast<size_t>(q)];
                    if (c < i) pat.push_back(c);
                }
            }
            int m = 0;
            bool ok = true;
            for (index_t c : pat) {
                if (!chol_append(A, w, pat, m, c)) { ok = false; break; }
                ++m;
            }
            const double aii = A.at(i, i);
            double psi_prev = 0.0, psi = 0.0;
            for (index_t step = 0; ok; ++step) {
                // Bordered solve: y = A_PP^{-1} a, psi = a_ii - a'y (Schur complement = 1/g~_last).
                y.assign(static_cast<size_t>(m), 0.0);
                for (index_t q = A.row_begin(i); q < A.row_end(i); ++q)
                    w.dense[static_cast<size_t>(A.col[static_cast<size_t>(q)])] = A.val[static_cast<size_t>(q)];
                for (int q = 0; q < m; ++q) y[static_cast<size_t>(q)] = w.dense[static_cast<size_t>(pat[static_cast<size_t>(q)])];
                for (index_t q = A.row_begin(i); q < A.row_end(i); ++q)
                    w.dense[static_cast<size_t>(A.col[static_cast<size_t>(q)])] = 0.0;
                std::vector<double> a(y);
                trsv_lower(m, w.L.data(), w.cap, y.data());
                trsv_lower_t(m, w.L.data(), w.cap, y.data());
                psi = aii - dot_fixed4(a.data(), y.data(), m);
                if (!(psi > 0.0)) { ok = false; break; }
                if (step > 0 && (psi_prev - psi) <= eps * psi_prev) break;  // (c)
                if (step == k) break;
                psi_prev = psi;
                // (d) gradient (A g~)_j over rows of A in P + {i}; g~ = (-y, 1)/psi (scale irrelevant).
                w.touched.clear();
                auto scatter = [&](index_t mrow, double gm) {
                    for (index_t q = A.row_begin(mrow); q < A.row_end(mrow); ++q) {
                        const index_t j = A.col[static_cast<size_t>(q)];
                        if (j >= i) continue;
                        if (!w.gmark[static_cast<size_t>(j)]) {
                            w.gmark[static_cast<size_t>(j)] = 1;
                            w.grad[static_cast<size_t>(j)] = 0.0;
                            w.touched.push_back(j);
                        }
                        w.grad[static_cast<size_t>(j)] += A.val[static_cast<size_t>(q)] * gm;
                    }
                };
                // fixed order: pattern in insertion order, then i
                for (int q = 0; q < m; ++q) scatter(pat[static_cast<size_t>(q)], -y[static_cast<size_t>(q)]);
                scatter(i, 1.0);
                for (int q = 0; q < m; ++q) w.gmark[static_cast<size_t>(pat[static_cast<size_t>(q)])] = 2;  // exclude P
                cand.clear();
                for (index_t j : w.touched)
                    if (w.gmark[static_cast<size_t>(j)] == 1) cand.emplace_back(std::fabs(w.grad[static_cast<size_t>(j)]), j);
                for (index_t j : w.touched) w.gmark[static_cast<size_t>(j)] = 0;
                for (int q = 0; q < m; ++q) w.gmark[static_cast<size_t>(pat[static_cast<size_t>(q)])] = 0;
                if (cand.empty()) break;
                const size_t take = std::min(cand.size(), static_cast<size_t>(rho));
                std::partial_sort(cand.begin(), cand.begin() + static_cast<long>(take), cand.end(),
                                  [](const auto& x, const auto& z) {
                                      return x.first > z.first || (x.first == z.first && x.second < z.second);
                                  });
                std::sort(cand.begin(), cand.begin() + static_cast<long>(take),
                          [](const auto& x, const auto& z) { return x.second < z.second; });
                for (size_t c = 0; c < take && ok; ++c) {
                    pat.push_back(cand[c].second);
                    if (!chol_append(A, w, pat, m, cand[c].second)) ok = false;
                    else ++m;
                }
            }
            if (!ok) {
#pragma omp critical
                if (bad_row < 0 || i < bad_row) bad_row = i;
                continue;
            }
            // Row = g~ / sqrt(g~_last) = (-y, 1) * (1/psi) * sqrt(psi) = (-y, 1) / sqrt(psi)
            const double s = 1.0 / std::sqrt(psi);
            std::vector<std::pair<index_t, double>> e;
            e.reserve(static_cast<size_t>(m) + 1);
            for (int q = 0; q < m; ++q) e.emplace_back(pat[static_cast<size_t>(q)], -y[static_cast<size_t>(q)] * s);
            e.emplace_back(i, s);
            std::sort(e.begin(), e.end());
            auto& rc = rcol[static_cast<size_t>(i)];
            auto& rv = rval[static_cast<size_t>(i)];
            rc.resize(e.size());
            rv.resize(e.size());
            for (size_t q = 0; q < e.size(); ++q) { rc[q] = e[q].first; rv[q] = e[q].second; }
            psi_all[static_cast<size_t>(i)] = psi;
        }
    }
    if (bad_row >= 0)
        throw NotSpdError("afsai_build: non-positive local pivot at row " + std::to_string(bad_row));
    Csr G;
    G.n_rows = G.n_cols = n;
    G.rowptr.assign(static_cast<size_t>(n) + 1, 0);
    for (index_t i = 0; i < n; ++i) G.rowptr[static_cast<size_t>(i) + 1] = G.rowptr[static_cast<size_t>(i)] + static_cast<index_t>(rcol[static_cast<size_t>(i)].size());
    G.col.resize(static_cast<size_t>(G.rowptr.back()));
    G.val.resize(static_cast<size_t>(G.rowptr.back()));
#pragma omp parallel for schedule(static) num_threads(num_threads())
    for (index_t i = 0; i < n; ++i) {
        std::copy(rcol[static_cast<size_t>(i)].begin(), rcol[static_cast<size_t>(i)].end(), G.col.begin() + G.rowptr[static_cast<size_t>(i)]);
        std::copy(rval[static_cast<size_t>(i)].begin(), rval[static_cast<size_t>(i)].end(), G.val.begin() + G.rowptr[static_cast<size_t>(i)]);
    }
    if (psi_out) *psi_out = std::move(psi_all);
    return G;
}

// Lanczos on x -> G A G' x from a fixed-seed random start;
// largest Ritz value x 1.05; breakdown returns the Ritz value reached.
double estimate_lambda_max(const Csr& G, const Csr& Gt, const Csr& A, index_t steps, std::uint64_t seed) {
    const index_t n = A.n_rows;
    if (n == 0) return 1.05;
    Rng rng(seed);
    std::vector<double> v(static_cast<size_t>(n)), vp(static_cast<size_t>(n), 0.0), w(static_cast<size_t>(n)),
        t1(static_cast<size_t>(n)), t2(static_cast<size_t>(n));
    for (auto& x : v) x = rng.symmetric();
    double nv = norm2(n, v.data());
    for (auto& x : v) x /= nv;
    std::vector<double> alpha, beta;
    double beta_prev = 0.0;
    for (index_t j = 0; j < steps; ++j) {
        spmv(Gt, v.data(), t1.data());
        spmv(A, t1.data(), t2.data());
        spmv(G, t2.data(), w.data());
        const double a = dot(n, w.data(), v.data());
        alpha.push_back(a);
#pragma omp parallel for schedule(static) num_threads(num_threads()) if (n > 65536)
        for (index_t i = 0; i < n; ++i) w[static_cast<size_t>(i)] -= a * v[static_cast<size_t>(i)] + beta_prev * vp[static_cast<size_t>(i)];
        const double b = norm2(n, w.data());
        if (j + 1 == steps || !(b > 1e-12 * std::fabs(a))) break;
        beta.push_back(b);
        beta_prev = b;
        vp.swap(v);
        for (index_t i = 0; i < n; ++i) v[static_cast<size_t>(i)] = w[static_cast<size_t>(i)] / b;
    }
    const int m = static_cast<int>(alpha.size());
    std::vector<double> T(static_cast<size_t>(m) * m, 0.0), ev(static_cast<size_t>(m)), evec(static_cast<size_t>(m) * m);
    for (int i = 0; i < m; ++i) {
        T[static_cast<size_t>(i) * m + i] = alpha[static_cast<size_t>(i)];
        if (i + 1 < m) T[static_cast<size_t>(i) * m + i + 1] = T[static_cast<size_t>(i + 1) * m + i] = beta[static_cast<size_t>(i)];
    }
    sym_eig(m, T.data(), ev.data(), evec.data());
    return 1.05 * ev[static_cast<size_t>(m - 1)];
}

double compute_omega(double lambda_hat) {
    if (!(lambda_hat > 0.0)) throw ConfigError("compute_omega: lambda_hat must be positive");
    return std::min(1.0, 2.0 / lambda_hat);
}

// Alg. 3 / SPEC.md:194-202.
FsaiSmoother smoother_setup(const Csr& A, const SmootherConfig& cfg) {
    FsaiSmoother s;
    double rho_bar = cfg.rho_bar;
    if (rho_bar <= 0.0) {
        index_t lower = 0;
        for (index_t i = 0; i < A.n_rows; ++i)
            for (index_t q = A.row_begin(i); q < A.row_end(i); ++q)
                if (A.col[static_cast<size_t>(q)] <= i) ++lower;
        rho_bar = A.n_rows ? 2.0 * double(lower) / double(A.n_rows) : 1.0;
    }
    std::vector<double> psi;
    const int ext = smoother_backend_set() ? smoother_external(A, cfg, rho_bar, psi, s) : 0;
    if (ext != 1) {
        Csr Gt;
        if (ext == 0) {
            s.G = afsai_build(A, nullptr, cfg.k0, cfg.rho0, cfg.eps0, &psi);
            Gt = transpose(s.G);
            s.lambda_hat = estimate_lambda_max(s.G, Gt, A, cfg.lanczos_steps, cfg.seed);
            s.omega = compute_omega(s.lambda_hat);
            s.exit_reason = SmootherExit::omega_reached;
        }  // ext == 2: the backend finished some passes; continue its loop from there
        while (s.omega < cfg.omega_bar) {
            if (!(s.G.nnz_per_row() < rho_bar)) { s.exit_reason = SmootherExit::density_bound; break; }
            std::vector<double> psi2;
            Csr G2 = afsai_build(A, &s.G, cfg.ki, cfg.rhoi, cfg.epsi, &psi2);
            if (G2.nnz() == s.G.nnz()) { s.exit_reason = SmootherExit::pattern_stagnation; break; }
            s.G = std::move(G2);
            psi.swap(psi2);
            Gt = transpose(s.G);
            s.lambda_hat = estimate_lambda_max(s.G, Gt, A, cfg.lanczos_steps, cfg.seed);
            s.omega = compute_omega(s.lambda_hat);
            ++s.refinement_passes;
            s.exit_reason = SmootherExit::omega_reached;
        }
    }
    // Kaporin gain (prod A_ii / prod psi_i)^(1/n) in log domain (fsai.hpp:49-51).
    double lg = 0.0;
    for (index_t i = 0; i < A.n_rows; ++i) lg += std::log(A.at(i, i)) - std::log(psi[static_cast<size_t>(i)]);
    s.kaporin_estimate = A.n_rows ? std::exp(lg / double(A.n_rows)) : 1.0;
    return s;
}

std::vector<double> apply_smoothing_step(const Csr& G, const Csr& Gt, double omega, const Csr& A,
                                         const std::vector<double>& b, const std::vector<double>& x) {
    const index_t n = A.n_rows;
    if (static_cast<index_t>(b.size()) != n || static_cast<index_t>(x.size()) != n)
        throw DimensionError("apply_smoothing_step: size mismatch");
    std::vector<double> r(static_cast<size_t>(n)), t(static_cast<size_t>(n)), u(static_cast<size_t>(n)), out(x);
    spmv(A, x.data(), r.data());
    for (index_t i = 0; i < n; ++i) r[static_cast<size_t>(i)] = b[static_cast<size_t>(i)] - r[static_cast<size_t>(i)];
    spmv(G, r.data(), t.data());
    spmv(Gt, t.data(), u.data());
    for (index_t i = 0; i < n; ++i) out[static_cast<size_t>(i)] += omega * u[static_cast<size_t>(i)];
    return out;
}

}  // namespace aspamg
