// Recursive AMG setup (Alg. 1),
// complexities and a binary hierarchy dump (SURVEY.md §5:
// the CPU setup is not redone per measurement). hierarchy.cpp is missing from
// the reference.
#include "amg.hpp"
#include "fem.hpp"
#include "smalldense.hpp"

#include <chrono>
#include <cstdio>
#include <cstring>
#include <memory>

namespace aspamg {

namespace {
double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

void dense_cholesky_coarse(const Csr& A, index_t level, std::vector<double>& Lcm) {
    const index_t n = A.n_rows;
    if (n > 20000) throw NumericalError("amg_setup: coarsest level too large for a dense factor (level " + std::to_string(level) + ")");
    std::vector<double> a(static_cast<size_t>(n * n), 0.0);
    for (index_t i = 0; i < n; ++i)  // dense.cpp:25-33 row-major fill
        for (index_t q = A.row_begin(i); q < A.row_end(i); ++q)
            a[static_cast<size_t>(i * n + A.col[static_cast<size_t>(q)])] = A.val[static_cast<size_t>(q)];
    const long bad = cholesky_lower(static_cast<int>(n), a.data());
    if (bad >= 0)
        throw NotSpdError("amg_setup: dense Cholesky failed at level " + std::to_string(level) +
                          " (pivot " + std::to_string(bad) + ")");
    Lcm.assign(static_cast<size_t>(n * n), 0.0);
    for (index_t i = 0; i < n; ++i)
        for (index_t j = 0; j <= i; ++j) Lcm[static_cast<size_t>(i + j * n)] = a[static_cast<size_t>(i * n + j)];
}
}  // namespace

void compute_complexities(Hierarchy& h) {
    if (h.levels.empty()) return;
    const double n0 = double(h.levels[0].A.n_rows), z0 = double(h.levels[0].A.nnz());
    double gd = 0, op = 0, fs = 0;
    for (const auto& L : h.levels) {
        gd += double(L.A.n_rows);
        op += double(L.A.nnz());
        fs += double(L.smoother.G.nnz());
    }
    h.C_gd = n0 > 0 ? gd / n0 : 1.0;
    h.C_op = z0 > 0 ? op / z0 : 1.0;
    h.C_fs = z0 > 0 ? fs / z0 : 0.0;
}

Hierarchy amg_setup(const Csr& A0, const std::vector<double>& coords, const HierarchyConfig& cfg) {
    if (A0.n_rows != A0.n_cols) throw DimensionError("amg_setup: A must be square");
    if (cfg.max_levels < 1 || cfg.nu1 < 0 || cfg.nu2 < 0 || cfg.nu1 + cfg.nu2 < 1)
        throw ConfigError("amg_setup: invalid hierarchy config");
    const double t0 = now_s();
    Hierarchy h;
    h.nu1 = cfg.nu1;
    h.nu2 = cfg.nu2;
    Dense V;
    Csr A = A0;
    for (index_t lvl = 0;; ++lvl) {
        Level L;
        const index_t n = A.n_rows;
        const bool last = n <= cfg.min_coarse_size || lvl == cfg.max_levels - 1;
        if (last) {
            L.A = std::move(A);
            dense_cholesky_coarse(L.A, lvl, h.coarse_L);
            h.n_coarse = L.A.n_rows;
            h.levels.push_back(std::move(L));
            break;
        }
        double t = now_s();
        L.smoother = smoother_setup(A, cfg.smoother);
        L.Gt = transpose(L.smoother.G);
        L.t_smoother = now_s() - t;
        h.t.T_sm += L.t_smoother;
        if (lvl == 0) {
            t = now_s();
            Dense rbm;
            bool have_rbm = false;
            if (!coords.empty() && static_cast<index_t>(coords.size()) == n) {
                bool rd = false;
                rbm = rigid_body_modes(coords, n / 3, &rd);
                have_rbm = rbm.n_cols > 0 && rbm.n_cols <= cfg.srqcg.n_tv;
            }
            Dense V0 = seed_space(have_rbm ? &rbm : nullptr, cfg.srqcg.n_tv, n, derive_seed(cfg.srqcg.seed, 6));
            TestSpace ts = srqcg_backend_set() ? srqcg_external(A, L.smoother.G, L.Gt, V0, cfg.srqcg)
                                              : srqcg(A, L.smoother.G, L.Gt, V0, cfg.srqcg);
            V = std::move(ts.V);
            h.t.T_ts += now_s() - t;
        }
        L.n_tv = V.n_cols;
        t = now_s();
        Csr soc = affinity_soc(A, V);
        Csr filt = filter_soc(soc, cfg.theta);
        CfSplit split = select_coarse_mis(filt);
        h.t.T_cs += now_s() - t;
        if (split.n_coarse == 0 || split.n_coarse >= n) {  // no coarsening progress: stop here
            L.smoother = FsaiSmoother{};
            L.Gt = Csr{};
            L.A = std::move(A);
            dense_cholesky_coarse(L.A, lvl, h.coarse_L);
            h.n_coarse = L.A.n_rows;
            h.levels.push_back(std::move(L));
            break;
        }
        t = now_s();
        Prolongation pr = dpls_build(filt, split, V, cfg.dpls);
        L.P = std::move(pr.P);
        L.Pt = transpose(L.P);
        h.t.T_pl += now_s() - t;
        t = now_s();
        Csr Ac = galerkin_backend_set() ? galerkin_external(L.P, L.Pt, A) : galerkin_triple(L.P, A);
        h.t.T_rap += now_s() - t;
        // Injected, re-orthonormalised coarse test space.
        Dense Vc(split.n_coarse, V.n_cols);
        for (index_t i = 0; i < n; ++i)
            if (split.is_coarse[static_cast<size_t>(i)])
                for (index_t c = 0; c < V.n_cols; ++c) Vc(split.coarse_index[static_cast<size_t>(i)], c) = V(i, c);
        orthonormalize_columns(Vc);
        V = std::move(Vc);
        L.A = std::move(A);
        h.levels.push_back(std::move(L));
        A = std::move(Ac);
    }
    compute_complexities(h);
    h.t.T_p = now_s() - t0;
    return h;
}

// ------------------------------------------------------------------ dump/load
namespace {
constexpr std::uint64_t kMagic = 0x4250414d47423230ULL;  // "BPAMGB20"
struct File {
    std::FILE* f;
    explicit File(const std::string& p, const char* mode) : f(std::fopen(p.c_str(), mode)) {
        if (!f) throw IoError("hierarchy: cannot open " + p);
    }
    ~File() { if (f) std::fclose(f); }
    void w(const void* p, size_t n) { if (n && std::fwrite(p, 1, n, f) != n) throw IoError("hierarchy: write failed"); }
    void r(void* p, size_t n) { if (n && std::fread(p, 1, n, f) != n) throw IoError("hierarchy: truncated file"); }
    template <class T> void wv(const std::vector<T>& v) { std::uint64_t n = v.size(); w(&n, 8); w(v.data(), n * sizeof(T)); }
    template <class T> void rv(std::vector<T>& v) { std::uint64_t n; r(&n, 8); v.resize(n); r(v.data(), n * sizeof(T)); }
    template <class T> void ws(const T& x) { w(&x, sizeof(T)); }
    template <class T> void rs(T& x) { r(&x, sizeof(T)); }
    void wcsr(const Csr& m) { ws(m.n_rows); ws(m.n_cols); ws(static_cast<int>(m.symmetric)); wv(m.rowptr); wv(m.col); wv(m.val); }
    void rcsr(Csr& m) { int s; rs(m.n_rows); rs(m.n_cols); rs(s); m.symmetric = s; rv(m.rowptr); rv(m.col); rv(m.val); }
};
}  // namespace

void hierarchy_save(const Hierarchy& h, const std::string& path) {
    File f(path, "wb");
    f.ws(kMagic);
    std::uint64_t nl = h.levels.size();
    f.ws(nl); f.ws(h.nu1); f.ws(h.nu2); f.ws(h.n_coarse);
    f.ws(h.C_gd); f.ws(h.C_op); f.ws(h.C_fs); f.ws(h.t);
    for (const auto& L : h.levels) {
        f.wcsr(L.A); f.wcsr(L.smoother.G); f.wcsr(L.Gt); f.wcsr(L.P); f.wcsr(L.Pt);
        f.ws(L.smoother.omega); f.ws(L.smoother.lambda_hat); f.ws(L.smoother.kaporin_estimate);
        f.ws(L.smoother.refinement_passes); f.ws(static_cast<int>(L.smoother.exit_reason)); f.ws(L.n_tv);
    }
    f.wv(h.coarse_L);
}

Hierarchy hierarchy_load(const std::string& path) {
    File f(path, "rb");
    std::uint64_t magic, nl;
    f.rs(magic);
    if (magic != kMagic) throw IoError("hierarchy: bad magic in " + path);
    Hierarchy h;
    f.rs(nl); f.rs(h.nu1); f.rs(h.nu2); f.rs(h.n_coarse);
    f.rs(h.C_gd); f.rs(h.C_op); f.rs(h.C_fs); f.rs(h.t);
    h.levels.resize(nl);
    for (auto& L : h.levels) {
        int ex;
        f.rcsr(L.A); f.rcsr(L.smoother.G); f.rcsr(L.Gt); f.rcsr(L.P); f.rcsr(L.Pt);
        f.rs(L.smoother.omega); f.rs(L.smoother.lambda_hat); f.rs(L.smoother.kaporin_estimate);
        f.rs(L.smoother.refinement_passes); f.rs(ex); f.rs(L.n_tv);
        L.smoother.exit_reason = static_cast<SmootherExit>(ex);
    }
    f.rv(h.coarse_L);
    return h;
}

}  // namespace aspamg
