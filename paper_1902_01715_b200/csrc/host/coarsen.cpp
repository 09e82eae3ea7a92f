// Affinity SoC, theta-filtering and greedy MIS (PAPER.md
// :565-594). coarsening.cpp is missing from the reference.
#include "amg.hpp"

#include <algorithm>
#include <numeric>
#include <omp.h>

namespace aspamg {

// SoC[i,j] = (v_i.v_j)^2 / ((v_i.v_i)(v_j.v_j)) on A's off-diagonal pattern;
// zero-norm rows give 0.
Csr affinity_soc(const Csr& A, const Dense& V) {
    if (V.n_rows != A.n_rows) throw DimensionError("affinity_soc: V rows mismatch");
    const index_t n = A.n_rows, m = V.n_cols;
    std::vector<double> nrm(static_cast<size_t>(n), 0.0);
#pragma omp parallel for schedule(static) num_threads(num_threads())
    for (index_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (index_t c = 0; c < m; ++c) s += V(i, c) * V(i, c);
        nrm[static_cast<size_t>(i)] = s;
    }
    Csr S;
    S.n_rows = S.n_cols = n;
    S.symmetric = true;
    S.rowptr.assign(static_cast<size_t>(n) + 1, 0);
    for (index_t i = 0; i < n; ++i) {
        index_t c = 0;
        for (index_t q = A.row_begin(i); q < A.row_end(i); ++q)
            if (A.col[static_cast<size_t>(q)] != i) ++c;
        S.rowptr[static_cast<size_t>(i) + 1] = S.rowptr[static_cast<size_t>(i)] + c;
    }
    S.col.resize(static_cast<size_t>(S.rowptr.back()));
    S.val.resize(static_cast<size_t>(S.rowptr.back()));
#pragma omp parallel for schedule(static) num_threads(num_threads())
    for (index_t i = 0; i < n; ++i) {
        index_t o = S.rowptr[static_cast<size_t>(i)];
        for (index_t q = A.row_begin(i); q < A.row_end(i); ++q) {
            const index_t j = A.col[static_cast<size_t>(q)];
            if (j == i) continue;
            double d = 0.0;
            for (index_t c = 0; c < m; ++c) d += V(i, c) * V(j, c);
            const double den = nrm[static_cast<size_t>(i)] * nrm[static_cast<size_t>(j)];
            S.col[static_cast<size_t>(o)] = j;
            S.val[static_cast<size_t>(o)] = den > 0.0 ? (d * d) / den : 0.0;
            ++o;
        }
    }
    return S;
}

// Per row keep the theta largest affinities (ties -> smaller column), then
// symmetrise by union. Kept values are the SoC values.
Csr filter_soc(const Csr& soc, index_t theta) {
    if (theta < 1) throw ConfigError("filter_soc: theta must be >= 1");
    const index_t n = soc.n_rows;
    std::vector<std::vector<index_t>> keep(static_cast<size_t>(n));
#pragma omp parallel for schedule(static) num_threads(num_threads())
    for (index_t i = 0; i < n; ++i) {
        std::vector<std::pair<double, index_t>> e;
        for (index_t q = soc.row_begin(i); q < soc.row_end(i); ++q)
            e.emplace_back(soc.val[static_cast<size_t>(q)], soc.col[static_cast<size_t>(q)]);
        const size_t t = std::min(e.size(), static_cast<size_t>(theta));
        std::partial_sort(e.begin(), e.begin() + static_cast<long>(t), e.end(), [](const auto& a, const auto& b) {
            return a.first > b.first || (a.first == b.first && a.second < b.second);
        });
        auto& k = keep[static_cast<size_t>(i)];
        for (size_t c = 0; c < t; ++c) k.push_back(e[c].second);
    }
    // union: edge (i,j) kept if i kept j or j kept i
    std::vector<index_t> cnt(static_cast<size_t>(n) + 1, 0);
    for (index_t i = 0; i < n; ++i)
        for (index_t j : keep[static_cast<size_t>(i)]) { ++cnt[static_cast<size_t>(i) + 1]; ++cnt[static_cast<size_t>(j) + 1]; }
    std::partial_sum(cnt.begin(), cnt.end(), cnt.begin());
    std::vector<index_t> adj(static_cast<size_t>(cnt.back()));
    std::vector<index_t> cur(cnt.begin(), cnt.end() - 1);
    for (index_t i = 0; i < n; ++i)
        for (index_t j : keep[static_cast<size_t>(i)]) {
            adj[static_cast<size_t>(cur[static_cast<size_t>(i)]++)] = j;
            adj[static_cast<size_t>(cur[static_cast<size_t>(j)]++)] = i;
        }
    Csr F;
    F.n_rows = F.n_cols = n;
    F.symmetric = true;
    F.rowptr.assign(static_cast<size_t>(n) + 1, 0);
    std::vector<std::vector<index_t>> rows(static_cast<size_t>(n));
#pragma omp parallel for schedule(static) num_threads(num_threads())
    for (index_t i = 0; i < n; ++i) {
        auto& r = rows[static_cast<size_t>(i)];
        r.assign(adj.begin() + cnt[static_cast<size_t>(i)], adj.begin() + cnt[static_cast<size_t>(i) + 1]);
        std::sort(r.begin(), r.end());
        r.erase(std::unique(r.begin(), r.end()), r.end());
    }
    for (index_t i = 0; i < n; ++i)
        F.rowptr[static_cast<size_t>(i) + 1] = F.rowptr[static_cast<size_t>(i)] + static_cast<index_t>(rows[static_cast<size_t>(i)].size());
    F.col.resize(static_cast<size_t>(F.rowptr.back()));
    F.val.resize(static_cast<size_t>(F.rowptr.back()));
#pragma omp parallel for schedule(static) num_threads(num_threads())
    for (index_t i = 0; i < n; ++i) {
        index_t o = F.rowptr[static_cast<size_t>(i)];
        for (index_t j : rows[static_cast<size_t>(i)]) {
            F.col[static_cast<size_t>(o)] = j;
            F.val[static_cast<size_t>(o)] = soc.at(i, j);
            ++o;
        }
    }
    return F;
}

// Greedy MIS: visit in descending filtered degree (ties ascending index); a
// node joins C unless a neighbour is already in C. Sequential by contract.
CfSplit select_coarse_mis(const Csr& g) {
    const index_t n = g.n_rows;
    std::vector<index_t> ord(static_cast<size_t>(n));
    std::iota(ord.begin(), ord.end(), index_t{0});
    std::stable_sort(ord.begin(), ord.end(), [&](index_t a, index_t b) {
        return (g.row_end(a) - g.row_begin(a)) > (g.row_end(b) - g.row_begin(b));
    });
    CfSplit s;
    s.is_coarse.assign(static_cast<size_t>(n), 0);
    std::vector<char> blocked(static_cast<size_t>(n), 0);
    for (index_t v : ord) {
        if (blocked[static_cast<size_t>(v)]) continue;
        s.is_coarse[static_cast<size_t>(v)] = 1;
        for (index_t q = g.row_begin(v); q < g.row_end(v); ++q) blocked[static_cast<size_t>(g.col[static_cast<size_t>(q)])] = 1;
    }
    s.coarse_index.assign(static_cast<size_t>(n), -1);
    for (index_t i = 0; i < n; ++i)
        if (s.is_coarse[static_cast<size_t>(i)]) s.coarse_index[static_cast<size_t>(i)] = s.n_coarse++;
    return s;
}

}  // namespace aspamg
