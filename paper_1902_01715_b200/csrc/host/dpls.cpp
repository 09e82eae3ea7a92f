// Dynamic-Pattern Least-Squares prolongation (Alg. 5
// :659-685). prolongation.cpp is missing from the reference.
#include "amg.hpp"

#include <algorithm>
#include <cmath>
#include <omp.h>

namespace aspamg {

// For each fine node i: candidates J_i = coarse nodes within d_p hops in the
// filtered SoC graph (ascending index). Greedily add the candidate whose
// Householder-transformed test row has maximal affinity with the current
// residual; R's diagonal-ratio condition estimate is checked before accepting
// (empty R has cond 1); stop on eps_p relative residual, kappa_p, n_max or
// exhausted candidates; weights w = R^{-1} (Q r)[0:k].
Prolongation dpls_build(const Csr& soc, const CfSplit& split, const Dense& V, const DplsConfig& cfg) {
    const index_t n = soc.n_rows, m = V.n_cols;
    if (V.n_rows != n) throw DimensionError("dpls_build: V rows mismatch");
    if (cfg.d_p < 1 || !(cfg.kappa_p > 1.0) || cfg.n_max < 1) throw ConfigError("dpls_build: bad config");
    std::vector<std::vector<std::pair<index_t, double>>> rows(static_cast<size_t>(n));
    Prolongation out;
    out.stop.assign(static_cast<size_t>(n), DplsStop::coarse);
#pragma omp parallel num_threads(num_threads())
    {
        std::vector<char> seen(static_cast<size_t>(n), 0);
        std::vector<index_t> touched, frontier, next, J;
        std::vector<double> W, r, Rm, vi;
        std::vector<char> used;
        std::vector<index_t> sel;
#pragma omp for schedule(dynamic, 512)
        for (index_t i = 0; i < n; ++i) {
            auto& row = rows[static_cast<size_t>(i)];
            if (split.is_coarse[static_cast<size_t>(i)]) {
                row.emplace_back(split.coarse_index[static_cast<size_t>(i)], 1.0);
                continue;
            }
            // BFS to depth d_p
            touched.clear(); frontier.clear(); J.clear();
            seen[static_cast<size_t>(i)] = 1; touched.push_back(i); frontier.push_back(i);
            for (index_t d = 0; d < cfg.d_p && !frontier.empty(); ++d) {
                next.clear();
                for (index_t u : frontier)
                    for (index_t q = soc.row_begin(u); q < soc.row_end(u); ++q) {
                        const index_t v = soc.col[static_cast<size_t>(q)];
                        if (seen[static_cast<size_t>(v)]) continue;
                        seen[static_cast<size_t>(v)] = 1; touched.push_back(v); next.push_back(v);
                        if (split.is_coarse[static_cast<size_t>(v)]) J.push_back(v);
                    }
                frontier.swap(next);
            }
            for (index_t t : touched) seen[static_cast<size_t>(t)] = 0;
            std::sort(J.begin(), J.end());
            const size_t nc = J.size();
            W.assign(nc * static_cast<size_t>(m), 0.0);
            for (size_t c = 0; c < nc; ++c)
                for (index_t k = 0; k < m; ++k) W[c * static_cast<size_t>(m) + static_cast<size_t>(k)] = V(J[c], k);
            r.assign(static_cast<size_t>(m), 0.0);
            for (index_t k = 0; k < m; ++k) r[static_cast<size_t>(k)] = V(i, k);
            double vn = 0.0;
            for (double x : r) vn += x * x;
            vn = std::sqrt(vn);
            Rm.assign(static_cast<size_t>(m * m), 0.0);  // column-major upper, R(a,b) = Rm[a + b*m]
            used.assign(nc, 0);
            sel.clear();
            index_t k = 0;
            double dmax = 0.0, dmin = 0.0;
            DplsStop why = DplsStop::exhausted;
            for (;;) {
                double rr = 0.0;
                for (index_t t = k; t < m; ++t) rr += r[static_cast<size_t>(t)] * r[static_cast<size_t>(t)];
                if (std::sqrt(rr) <= cfg.eps_p * vn) { why = DplsStop::tolerance; break; }
                if (k >= cfg.n_max) { why = DplsStop::n_max; break; }
                // best candidate by affinity on the trailing components
                long best = -1;
                double best_aff = -1.0;
                for (size_t c = 0; c < nc; ++c) {
                    if (used[c]) continue;
                    const double* w = &W[c * static_cast<size_t>(m)];
                    double d = 0.0, ww = 0.0;
                    for (index_t t = k; t < m; ++t) { d += w[t] * r[static_cast<size_t>(t)]; ww += w[t] * w[t]; }
                    const double aff = (ww > 0.0 && rr > 0.0) ? (d * d) / (ww * rr) : 0.0;
                    if (aff > best_aff) { best_aff = aff; best = static_cast<long>(c); }
                }
                if (best < 0) { why = DplsStop::exhausted; break; }
                double* x = &W[static_cast<size_t>(best) * static_cast<size_t>(m)];
                double sig = 0.0;
                for (index_t t = k; t < m; ++t) sig += x[t] * x[t];
                sig = std::sqrt(sig);
                if (!(sig > 0.0)) { why = DplsStop::condition; break; }
                const double sgn = x[k] >= 0.0 ? 1.0 : -1.0;
                const double rkk = -sgn * sig;
                const double nmax = std::max(dmax, std::fabs(rkk)), nmin = k == 0 ? std::fabs(rkk) : std::min(dmin, std::fabs(rkk));
                if (nmax / nmin > cfg.kappa_p) { why = DplsStop::condition; break; }
                dmax = nmax; dmin = nmin;
                for (index_t t = 0; t < k; ++t) Rm[static_cast<size_t>(t + k * m)] = x[t];
                Rm[static_cast<size_t>(k + k * m)] = rkk;
                // Householder u = x[k:] - rkk e0 applied to r and remaining candidates
                std::vector<double> u(static_cast<size_t>(m - k));
                for (index_t t = k; t < m; ++t) u[static_cast<size_t>(t - k)] = x[t];
                u[0] -= rkk;
                double uu = 0.0;
                for (double z : u) uu += z * z;
                used[static_cast<size_t>(best)] = 1;
                sel.push_back(J[static_cast<size_t>(best)]);
                if (uu > 0.0) {
                    auto reflect = [&](double* y) {
                        double s = 0.0;
                        for (index_t t = k; t < m; ++t) s += u[static_cast<size_t>(t - k)] * y[t];
                        s = 2.0 * s / uu;
                        for (index_t t = k; t < m; ++t) y[t] -= s * u[static_cast<size_t>(t - k)];
                    };
                    reflect(r.data());
                    for (size_t c = 0; c < nc; ++c)
                        if (!used[c]) reflect(&W[c * static_cast<size_t>(m)]);
                }
                ++k;
            }
            out.stop[static_cast<size_t>(i)] = why;
            // back substitution R w = r[0:k]
            std::vector<double> w(static_cast<size_t>(k));
            for (index_t a = k - 1; a >= 0; --a) {
                double s = r[static_cast<size_t>(a)];
                for (index_t b = a + 1; b < k; ++b) s -= Rm[static_cast<size_t>(a + b * m)] * w[static_cast<size_t>(b)];
                w[static_cast<size_t>(a)] = s / Rm[static_cast<size_t>(a + a * m)];
            }
            for (index_t a = 0; a < k; ++a)
                row.emplace_back(split.coarse_index[static_cast<size_t>(sel[static_cast<size_t>(a)])], w[static_cast<size_t>(a)]);
            std::sort(row.begin(), row.end());
        }
    }
    Csr& P = out.P;
    P.n_rows = n;
    P.n_cols = split.n_coarse;
    P.rowptr.assign(static_cast<size_t>(n) + 1, 0);
    for (index_t i = 0; i < n; ++i) P.rowptr[static_cast<size_t>(i) + 1] = P.rowptr[static_cast<size_t>(i)] + static_cast<index_t>(rows[static_cast<size_t>(i)].size());
    P.col.resize(static_cast<size_t>(P.rowptr.back()));
    P.val.resize(static_cast<size_t>(P.rowptr.back()));
    for (index_t i = 0; i < n; ++i) {
        index_t o = P.rowptr[static_cast<size_t>(i)];
        for (const auto& e : rows[static_cast<size_t>(i)]) {
            P.col[static_cast<size_t>(o)] = e.first;
            P.val[static_cast<size_t>(o)] = e.second;
            ++o;
        }
    }
    return out;
}

}  // namespace aspamg
