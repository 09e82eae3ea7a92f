// Adaptive FSAI smoother set-up (Alg. 3 :374-387).
// The reference declares this module (fsai.hpp:27-83) but fsai.cpp is missing.
#include "amg.hpp"
#include "smalldense.hpp"

#include <algorithm>
#include <cstdint>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <omp.h>
#include <unistd.h>

namespace aspamg {

namespace {

struct RowWork {
    std::vector<double> dense;       // scatter buffer for one row of A (size n)
    struct GradSlot {
        double g;             // gradient accumulator, valid where stamp == ep
        std::uint64_t stamp;  // gradient epoch of the last touch of the column
    };
    std::vector<GradSlot> grad;  // size n: one cache access per touched column
    std::vector<std::uint32_t> pstamp;  // row epoch in which column j entered the pattern
    std::uint64_t ep = 0;
    std::uint32_t rep = 0;
    std::vector<index_t> touched;
    std::vector<double> L;         // incremental Cholesky of A[pat, pat], row-major, ld = cap
    int cap = 0;
    explicit RowWork(index_t n) : dense(static_cast<size_t>(n), 0.0), grad(static_cast<size_t>(n), GradSlot{0.0, 0}),
                                  pstamp(static_cast<size_t>(n), 0) {}
    void next_step() { ++ep; }
    void next_row() {
        if (++rep == 0) { std::fill(pstamp.begin(), pstamp.end(), 0u); rep = 1; }
    }
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
    const double d = ajj - dot_w32(row, row, m);
    if (!(d > 0.0)) return false;
    row[m] = std::sqrt(d);
    return true;
}

}  // namespace

// ------------------------------------------------------------ afsai passes
//
// SPEC.md:172-180 per row i: pattern P_i (< i) grows by up to rho entries per
// step for at most k steps, choosing the candidates j < i adjacent to P_i + {i}
// with the largest |(A g~)_j| (ties: smaller index); the row stops once the
// relative decrease of psi_i = 1/g~_last is <= eps. Final row is
// g~ / sqrt(g~_last), so diag(G A G') = 1.
//
// The factor of A[P_i, P_i] is kept in the pattern's insertion order, and a
// refinement pass (Alg. 3 line 5, "aFSAI(A, G, k_i, rho_i, eps_i)") restarts
// from the previous pass's pattern in that same order. The factor a pass
// rebuilds is therefore exactly the one the previous pass ended with, and the
// last bordered solve of a pass is exactly the first solve of the next one:
// a row's successive passes form ONE continuous sequence of steps. run_passes
// exploits that: it runs several passes of a row back to back (one factor
// build per batch instead of one per pass) and records the row of G after
// each pass; smoother_setup consumes them pass by pass (Lanczos, omega, the
// loop guards), so the result is the one pass-at-a-time execution gives.
namespace {

struct PassParams {
    index_t k, rho;
    double eps;
};

// One row's output of a batch of passes.
struct RowRun {
    std::vector<index_t> pat;  // final pattern, insertion order
    std::vector<double> y;     // per pass p: y_p[0..m_p) (the bordered solve), concatenated
    std::vector<int> m;        // per pass: pattern size
    std::vector<double> psi;   // per pass: Schur complement psi_i = 1/g~_last
    std::vector<int> perm;     // positions of pat in ascending column order
};

// Runs npass passes of row i (pass 0 with p0, the others with pr) from the
// start pattern st[0..ns) (insertion order). false: non-positive pivot.
bool run_row(const Csr& A, RowWork& w, index_t i, const index_t* st, index_t ns, int npass, const PassParams& p0,
             const PassParams& pr, RowRun& out, std::vector<double>& y, std::vector<double>& a,
             std::vector<std::pair<double, index_t>>& cand) {
    std::vector<index_t>& pat = out.pat;
    pat.clear();
    out.y.clear();
    out.m.clear();
    out.psi.clear();
    w.next_row();
    for (index_t q = 0; q < ns; ++q)
        if (st[q] < i) {
            pat.push_back(st[q]);
            w.pstamp[static_cast<size_t>(st[q])] = w.rep;
        }
    int m = 0;
    for (index_t c : pat) {
        if (!chol_append(A, w, pat, m, c)) return false;
        ++m;
    }
    const double aii = A.at(i, i);
    double psi = 0.0;
    bool have = false;  // y / psi hold the bordered solve of the current pattern
    for (int pass = 0; pass < npass; ++pass) {
        const PassParams& pp = pass == 0 ? p0 : pr;
        double psi_prev = 0.0;
        for (index_t step = 0;; ++step) {
            if (!have) {
                // Bordered solve: y = A_PP^{-1} a, psi = a_ii - a'y (Schur complement = 1/g~_last).
                y.assign(static_cast<size_t>(m), 0.0);
                for (index_t q = A.row_begin(i); q < A.row_end(i); ++q)
                    w.dense[static_cast<size_t>(A.col[static_cast<size_t>(q)])] = A.val[static_cast<size_t>(q)];
                for (int q = 0; q < m; ++q) y[static_cast<size_t>(q)] = w.dense[static_cast<size_t>(pat[static_cast<size_t>(q)])];
                for (index_t q = A.row_begin(i); q < A.row_end(i); ++q)
                    w.dense[static_cast<size_t>(A.col[static_cast<size_t>(q)])] = 0.0;
                a.assign(y.begin(), y.end());
                trsv_lower(m, w.L.data(), w.cap, y.data());
                trsv_lower_t(m, w.L.data(), w.cap, y.data());
                psi = aii - dot_w32(a.data(), y.data(), m);
                if (!(psi > 0.0)) return false;
                have = true;
            }
            if (step > 0 && (psi_prev - psi) <= pp.eps * psi_prev) break;  // (c)
            if (step == pp.k) break;
            psi_prev = psi;
            // (d) gradient (A g~)_j over rows of A in P + {i}; g~ = (-y, 1)/psi (scale irrelevant).
            // Each (A g~)_j is summed over the rows in the fixed order below (pattern in
            // insertion order, then i); a first touch starts from 0 (epoch stamps).
            w.next_step();
            w.touched.clear();
            const std::uint64_t ep = w.ep;
            auto scatter = [&](index_t mrow, double gm) {
                const index_t b = A.row_begin(mrow);
                const index_t* cb = A.col.data() + b;
                const index_t len = std::lower_bound(cb, cb + (A.row_end(mrow) - b), i) - cb;  // columns < i
                const double* vb = A.val.data() + b;
                for (index_t q = 0; q < len; ++q) {
                    const size_t j = static_cast<size_t>(cb[q]);
                    const double t = vb[q] * gm;
                    RowWork::GradSlot& g = w.grad[j];
                    if (g.stamp != ep) {
                        g.stamp = ep;
                        g.g = 0.0 + t;
                        w.touched.push_back(static_cast<index_t>(j));
                    } else {
                        g.g += t;
                    }
                }
            };
            for (int q = 0; q < m; ++q) scatter(pat[static_cast<size_t>(q)], -y[static_cast<size_t>(q)]);
            scatter(i, 1.0);
            cand.clear();
            for (index_t j : w.touched)
                if (w.pstamp[static_cast<size_t>(j)] != w.rep) cand.emplace_back(std::fabs(w.grad[static_cast<size_t>(j)].g), j);
            if (cand.empty()) break;
            const size_t take = std::min(cand.size(), static_cast<size_t>(pp.rho));
            std::partial_sort(cand.begin(), cand.begin() + static_cast<long>(take), cand.end(),
                              [](const auto& x, const auto& z) {
                                  return x.first > z.first || (x.first == z.first && x.second < z.second);
                              });
            std::sort(cand.begin(), cand.begin() + static_cast<long>(take),
                      [](const auto& x, const auto& z) { return x.second < z.second; });
            for (size_t c = 0; c < take; ++c) {
                pat.push_back(cand[c].second);
                w.pstamp[static_cast<size_t>(cand[c].second)] = w.rep;
                if (!chol_append(A, w, pat, m, cand[c].second)) return false;
                ++m;
            }
            have = false;
        }
        out.m.push_back(m);
        out.psi.push_back(psi);
        out.y.insert(out.y.end(), y.begin(), y.begin() + m);
    }
    out.perm.resize(pat.size());
    for (size_t q = 0; q < pat.size(); ++q) out.perm[q] = static_cast<int>(q);
    std::sort(out.perm.begin(), out.perm.end(), [&](int x, int z) { return pat[static_cast<size_t>(x)] < pat[static_cast<size_t>(z)]; });
    return true;
}

// Runs npass passes of every row; start: insertion-ordered start pattern
// (rows may hold i itself, which is skipped), nullptr = identity start.
std::vector<RowRun> run_passes(const Csr& A, const Csr* start, int npass, const PassParams& p0,
                               const PassParams& pr) {
    const index_t n = A.n_rows;
    std::vector<RowRun> rr(static_cast<size_t>(n));
    index_t bad_row = -1;
#pragma omp parallel num_threads(num_threads())
    {
        RowWork w(n);
        std::vector<double> y, a;
        std::vector<std::pair<double, index_t>> cand;
#pragma omp for schedule(dynamic, 64)
        for (index_t i = 0; i < n; ++i) {
            const index_t* st = start ? start->col.data() + start->row_begin(i) : nullptr;
            const index_t ns = start ? start->row_end(i) - start->row_begin(i) : 0;
            if (!run_row(A, w, i, st, ns, npass, p0, pr, rr[static_cast<size_t>(i)], y, a, cand)) {
#pragma omp critical
                if (bad_row < 0 || i < bad_row) bad_row = i;
            }
        }
    }
    if (bad_row >= 0)
        throw NotSpdError("afsai_build: non-positive local pivot at row " + std::to_string(bad_row));
    return rr;
}

// G after pass p of a batch (sorted rows), its insertion-ordered twin (the
// pattern then i; the start pattern of the next pass) and psi. The pattern's
// columns are all < i, so i closes both rows. G and ord may hold buffers of an
// earlier pass (reused, not reallocated).
void pass_matrix(const std::vector<RowRun>& rr, index_t n, int p, Csr& G, Csr& ord, std::vector<double>& psi) {
    G.n_rows = G.n_cols = n;
    G.symmetric = false;
    G.rowptr.resize(static_cast<size_t>(n) + 1);
    G.rowptr[0] = 0;
    for (index_t i = 0; i < n; ++i)
        G.rowptr[static_cast<size_t>(i) + 1] = G.rowptr[static_cast<size_t>(i)] + rr[static_cast<size_t>(i)].m[static_cast<size_t>(p)] + 1;
    const size_t nnz = static_cast<size_t>(G.rowptr.back());
    G.col.resize(nnz);
    G.val.resize(nnz);
    ord.n_rows = ord.n_cols = n;
    ord.rowptr = G.rowptr;
    ord.col.resize(nnz);
    ord.val.clear();
    psi.resize(static_cast<size_t>(n));
#pragma omp parallel for schedule(dynamic, 1024) num_threads(num_threads())
    for (index_t i = 0; i < n; ++i) {
        const RowRun& r = rr[static_cast<size_t>(i)];
        size_t yoff = 0;
        for (int q = 0; q < p; ++q) yoff += static_cast<size_t>(r.m[static_cast<size_t>(q)]);
        const int m = r.m[static_cast<size_t>(p)];
        const double ps = r.psi[static_cast<size_t>(p)];
        // Row = g~ / sqrt(g~_last) = (-y, 1) * (1/psi) * sqrt(psi) = (-y, 1) / sqrt(psi)
        const double s = 1.0 / std::sqrt(ps);
        const size_t b = static_cast<size_t>(G.rowptr[static_cast<size_t>(i)]);
        for (int q = 0; q < m; ++q) ord.col[b + static_cast<size_t>(q)] = r.pat[static_cast<size_t>(q)];
        ord.col[b + static_cast<size_t>(m)] = i;
        size_t o = b;
        for (int q : r.perm)
            if (q < m) {
                G.col[o] = r.pat[static_cast<size_t>(q)];
                G.val[o++] = -r.y[yoff + static_cast<size_t>(q)] * s;
            }
        G.col[o] = i;
        G.val[o] = s;
        psi[static_cast<size_t>(i)] = ps;
    }
}

// Passes per batch: doubling, bounded by the memory the batch's recorded rows
// take (ASPAMG_SETUP_MEM_GB, default a quarter of the host's memory).
double batch_budget_bytes() {
    if (const char* e = std::getenv("ASPAMG_SETUP_MEM_GB")) {
        const double gb = std::atof(e);
        if (gb > 0) return gb * 1e9;
    }
    const double phys = double(sysconf(_SC_PHYS_PAGES)) * double(sysconf(_SC_PAGE_SIZE));
    return phys > 0 ? 0.25 * phys : 8e9;
}

}  // namespace

Csr afsai_build(const Csr& A, const Csr* G_start, index_t k, index_t rho, double eps,
                std::vector<double>* psi_out) {
    if (A.n_rows != A.n_cols) throw DimensionError("afsai_build: A must be square");
    const index_t n = A.n_rows;
    if (G_start && G_start->n_rows != n) throw DimensionError("afsai_build: G_start size mismatch");
    const PassParams pp{k, rho, eps};
    std::vector<RowRun> rr = run_passes(A, G_start, 1, pp, pp);
    Csr G, ord;
    std::vector<double> psi;
    pass_matrix(rr, n, 0, G, ord, psi);
    if (psi_out) *psi_out = std::move(psi);
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

// Alg. 3 / SPEC.md:194-202. Passes are computed in batches (run_passes) and
// consumed one at a time, so the loop guards see exactly the pass sequence.
FsaiSmoother smoother_setup(const Csr& A, const SmootherConfig& cfg) {
    FsaiSmoother s;
    const index_t n = A.n_rows;
    double rho_bar = cfg.rho_bar;
    if (rho_bar <= 0.0) {
        index_t lower = 0;
        for (index_t i = 0; i < n; ++i)
            for (index_t q = A.row_begin(i); q < A.row_end(i); ++q)
                if (A.col[static_cast<size_t>(q)] <= i) ++lower;
        rho_bar = n ? 2.0 * double(lower) / double(n) : 1.0;
    }
    std::vector<double> psi;
    Csr ord;  // insertion-ordered twin of s.G (start pattern of the next pass)
    const int ext = smoother_backend_set() ? smoother_external(A, cfg, rho_bar, psi, s, &ord) : 0;
    if (ext != 1) {
        const PassParams p0{cfg.k0, cfg.rho0, cfg.eps0}, pr{cfg.ki, cfg.rhoi, cfg.epsi};
        std::vector<RowRun> batch;
        std::vector<double> lam_hist, nnzr_hist;  // per finished pass (batch-size prediction only)
        Csr spareG, spareO;
        std::vector<double> psi2;
        int next = 0, nbatch = 0, last_batch = 1;
        Csr Gt;
        auto take_pass = [&](Csr& G, Csr& O, std::vector<double>& ps) {
            if (next >= nbatch) {  // compute the next batch of passes from the current pattern
                batch.clear();
                batch.shrink_to_fit();
                const bool first = ext == 0 && s.G.n_rows == 0 && n > 0;
                // Batch size: the passes the loop is predicted to still run (linear
                // extrapolation of lambda_hat towards 2 / omega_bar and of nnz_r(G)
                // towards rho_bar over the last two passes), at most double the last
                // batch, within the memory the recorded rows may take (~8 B per
                // entry per pass). A misprediction costs time, never changes G.
                const double per = 8.0 * (double(ord.col.size()) + double(n) * double(cfg.ki * cfg.rhoi + 1)) + 1.0;
                const int fit = static_cast<int>(std::max(1.0, batch_budget_bytes() / per));
                int want = 2 * last_batch;
                const size_t h = lam_hist.size();
                if (h >= 2) {
                    const double dl = lam_hist[h - 2] - lam_hist[h - 1];
                    const double dz = nnzr_hist[h - 1] - nnzr_hist[h - 2];
                    double pred = 1e9;
                    if (dl > 0) pred = std::min(pred, (lam_hist[h - 1] - 2.0 / cfg.omega_bar) / dl);
                    if (dz > 0) pred = std::min(pred, (rho_bar - nnzr_hist[h - 1]) / dz);
                    if (pred < 1e9) want = std::min(want, static_cast<int>(std::ceil(std::max(pred, 0.0))) + 1);
                }
                nbatch = first ? 1 : std::max(1, std::min(want, std::min(fit, 16)));
                last_batch = nbatch;
                const double t0 = omp_get_wtime();
                batch = run_passes(A, first ? nullptr : &ord, nbatch, first ? p0 : pr, pr);
                next = 0;
                if (std::getenv("ASPAMG_SETUP_TRACE"))
                    std::fprintf(stderr, "[smoother n=%lld] batch of %d passes: %.2f s\n", (long long)n, nbatch,
                                 omp_get_wtime() - t0);
            }
            pass_matrix(batch, n, next++, G, O, ps);
        };
        if (ext == 0) {
            take_pass(s.G, ord, psi);
            Gt = transpose(s.G);
            s.lambda_hat = estimate_lambda_max(s.G, Gt, A, cfg.lanczos_steps, cfg.seed);
            s.omega = compute_omega(s.lambda_hat);
            s.exit_reason = SmootherExit::omega_reached;
        }  // ext == 2: the backend finished some passes; continue its loop from there
        while (s.omega < cfg.omega_bar) {
            if (!(s.G.nnz_per_row() < rho_bar)) { s.exit_reason = SmootherExit::density_bound; break; }
            Csr G2 = std::move(spareG), O2 = std::move(spareO);
            const double t0 = omp_get_wtime();
            take_pass(G2, O2, psi2);
            if (G2.nnz() == s.G.nnz()) { s.exit_reason = SmootherExit::pattern_stagnation; break; }
            std::swap(s.G, G2);
            std::swap(ord, O2);
            spareG = std::move(G2);  // the previous pass's buffers, reused by the next one
            spareO = std::move(O2);
            psi.swap(psi2);
            const double t1 = omp_get_wtime();
            transpose_into(s.G, Gt);
            const double t2 = omp_get_wtime();
            s.lambda_hat = estimate_lambda_max(s.G, Gt, A, cfg.lanczos_steps, cfg.seed);
            if (std::getenv("ASPAMG_SETUP_TRACE"))
                std::fprintf(stderr, "  pass: take %.2f transpose %.2f lanczos %.2f\n", t1 - t0, t2 - t1, omp_get_wtime() - t2);
            s.omega = compute_omega(s.lambda_hat);
            lam_hist.push_back(s.lambda_hat);
            nnzr_hist.push_back(s.G.nnz_per_row());
            ++s.refinement_passes;
            s.exit_reason = SmootherExit::omega_reached;
        }
    }
    // Kaporin gain (prod A_ii / prod psi_i)^(1/n) in log domain (fsai.hpp:49-51).
    double lg = 0.0;
    for (index_t i = 0; i < n; ++i) lg += std::log(A.at(i, i)) - std::log(psi[static_cast<size_t>(i)]);
    s.kaporin_estimate = n ? std::exp(lg / double(n)) : 1.0;
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
