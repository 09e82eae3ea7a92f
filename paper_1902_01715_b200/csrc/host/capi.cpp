// C-ABI over the host setup (include/aspamg_host.h).
#include "../../../include/aspamg_host.h"

#include "amg.hpp"
#include "fem.hpp"

#include <algorithm>
#include <new>
#include <string>

using namespace aspamg;

struct aspamg_problem {
    GeneratedProblem p;
    std::vector<double> rhs;
};
struct aspamg_hierarchy {
    Hierarchy h;
};
struct aspamg_csr_owned {
    Csr m;
};

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const DimensionError& e) { g_err = e.what(); return 1; }
    catch (const NotSpdError& e) { g_err = e.what(); return 2; }
    catch (const NumericalError& e) { g_err = e.what(); return 3; }
    catch (const ConfigError& e) { g_err = e.what(); return 4; }
    catch (const IoError& e) { g_err = e.what(); return 7; }
    catch (const std::bad_alloc&) { g_err = "out of host memory"; return 5; }
    catch (const std::exception& e) { g_err = e.what(); return 5; }
    catch (...) { g_err = "unknown error"; return 5; }
}

aspamg_csr_view view(const Csr& m) {
    aspamg_csr_view v{};
    v.n_rows = m.n_rows;
    v.n_cols = m.n_cols;
    v.nnz = m.nnz();
    v.row_offsets = m.rowptr.empty() ? nullptr : m.rowptr.data();
    v.col_indices = m.col.data();
    v.values = m.val.data();
    return v;
}

Csr from_view(const aspamg_csr_view& v) {
    if (v.n_rows < 0 || v.n_cols < 0) throw DimensionError("csr view: negative size");
    if (!v.row_offsets) throw DimensionError("csr view: null row_offsets");
    Csr m;
    m.n_rows = v.n_rows;
    m.n_cols = v.n_cols;
    m.rowptr.assign(v.row_offsets, v.row_offsets + v.n_rows + 1);
    const index_t nnz = m.rowptr.back();
    if (m.rowptr[0] != 0 || nnz < 0) throw DimensionError("csr view: bad row_offsets");
    for (index_t i = 0; i < m.n_rows; ++i)
        if (m.rowptr[static_cast<size_t>(i) + 1] < m.rowptr[static_cast<size_t>(i)])
            throw DimensionError("csr view: row_offsets not non-decreasing");
    m.col.assign(v.col_indices, v.col_indices + nnz);
    m.val.assign(v.values, v.values + nnz);
    for (index_t i = 0; i < m.n_rows; ++i)
        for (index_t q = m.rowptr[static_cast<size_t>(i)]; q < m.rowptr[static_cast<size_t>(i) + 1]; ++q) {
            const index_t c = m.col[static_cast<size_t>(q)];
            if (c < 0 || c >= m.n_cols) throw DimensionError("csr view: column index out of range");
            if (q > m.rowptr[static_cast<size_t>(i)] && c <= m.col[static_cast<size_t>(q) - 1])
                throw DimensionError("csr view: columns must be sorted and unique per row");
        }
    return m;
}
}  // namespace

extern "C" {

const char* aspamg_host_last_error(void) { return g_err.c_str(); }
int aspamg_host_set_threads(int n) { set_num_threads(n); return 0; }
int aspamg_host_get_threads(void) { return num_threads(); }

int aspamg_problem_config(int cfg, int64_t scale, aspamg_problem** out) {
    return guard([&] {
        auto* p = new aspamg_problem;
        try { p->p = make_config(cfg, scale, p->rhs); } catch (...) { delete p; throw; }
        *out = p;
    });
}

int aspamg_problem_hex(int64_t nx, int64_t ny, int64_t nz, double spacing, double young, double poisson,
                       uint32_t clamp_faces, aspamg_problem** out) {
    return guard([&] {
        MeshSpec m;
        m.nx = nx; m.ny = ny; m.nz = nz;
        m.hx = m.hy = m.hz = spacing;
        m.clamped = clamp_faces;
        if (nx < 1 || ny < 1 || nz < 1) throw ConfigError("assembly: element counts must be >= 1");
        std::vector<Material> mats(static_cast<size_t>(nx * ny * nz), Material{young, poisson});
        auto* p = new aspamg_problem;
        try {
            p->p = assemble_hex(m, mats);
            p->rhs = rhs_ones(p->p);
        } catch (...) { delete p; throw; }
        *out = p;
    });
}

int aspamg_problem_matrix(const aspamg_problem* p, aspamg_csr_view* out) {
    return guard([&] { *out = view(p->p.stiffness); });
}
int aspamg_problem_rhs(const aspamg_problem* p, const double** rhs, int64_t* n) {
    return guard([&] { *rhs = p->rhs.data(); *n = static_cast<int64_t>(p->rhs.size()); });
}
int aspamg_problem_coords(const aspamg_problem* p, const double** xyz, int64_t* n_nodes) {
    return guard([&] { *xyz = p->p.coords.data(); *n_nodes = p->p.n_free; });
}
void aspamg_problem_free(aspamg_problem* p) { delete p; }

int aspamg_setup_config_default(aspamg_setup_config* c) {
    return guard([&] {
        HierarchyConfig h;
        c->k0 = h.smoother.k0; c->rho0 = h.smoother.rho0; c->eps0 = h.smoother.eps0;
        c->ki = h.smoother.ki; c->rhoi = h.smoother.rhoi; c->epsi = h.smoother.epsi;
        c->omega_bar = h.smoother.omega_bar; c->rho_bar = h.smoother.rho_bar;
        c->lanczos_steps = h.smoother.lanczos_steps;
        c->n_tv = h.srqcg.n_tv; c->n_rq = h.srqcg.k_max; c->k_ritz = h.srqcg.k_ritz; c->srqcg_tol = h.srqcg.residual_tol;
        c->theta = h.theta; c->d_p = h.dpls.d_p; c->n_max = h.dpls.n_max; c->eps_p = h.dpls.eps_p; c->kappa_p = h.dpls.kappa_p;
        c->max_levels = h.max_levels; c->min_coarse_size = h.min_coarse_size; c->nu1 = h.nu1; c->nu2 = h.nu2;
        c->seed = h.smoother.seed;
    });
}

int aspamg_setup(const aspamg_csr_view* A, const double* coords, int64_t n_nodes, const aspamg_setup_config* c,
                 aspamg_hierarchy** out) {
    return guard([&] {
        if (!A || !c || !out) throw ConfigError("aspamg_setup: null argument");
        HierarchyConfig h;
        h.smoother.k0 = c->k0; h.smoother.rho0 = c->rho0; h.smoother.eps0 = c->eps0;
        h.smoother.ki = c->ki; h.smoother.rhoi = c->rhoi; h.smoother.epsi = c->epsi;
        h.smoother.omega_bar = c->omega_bar; h.smoother.rho_bar = c->rho_bar;
        h.smoother.lanczos_steps = c->lanczos_steps; h.smoother.seed = c->seed;
        h.srqcg.n_tv = c->n_tv; h.srqcg.k_max = c->n_rq; h.srqcg.k_ritz = c->k_ritz;
        h.srqcg.residual_tol = c->srqcg_tol; h.srqcg.seed = c->seed;
        h.theta = c->theta;
        h.dpls.d_p = c->d_p; h.dpls.n_max = c->n_max; h.dpls.eps_p = c->eps_p; h.dpls.kappa_p = c->kappa_p;
        h.max_levels = c->max_levels; h.min_coarse_size = c->min_coarse_size; h.nu1 = c->nu1; h.nu2 = c->nu2;
        if (h.srqcg.n_tv < 1 || h.srqcg.k_ritz < 1 || h.smoother.lanczos_steps < 1)
            throw ConfigError("aspamg_setup: n_tv, k_ritz, lanczos_steps must be >= 1");
        Csr K = from_view(*A);
        K.symmetric = true;
        std::vector<double> xyz;
        if (coords && n_nodes > 0) {
            if (3 * n_nodes != K.n_rows) throw DimensionError("aspamg_setup: coordinates do not match 3 dofs per node");
            xyz.assign(coords, coords + 3 * n_nodes);
        }
        auto* hh = new aspamg_hierarchy;
        try { hh->h = amg_setup(K, xyz, h); } catch (...) { delete hh; throw; }
        *out = hh;
    });
}

int aspamg_hierarchy_info_get(const aspamg_hierarchy* hh, aspamg_hierarchy_info* o) {
    return guard([&] {
        const Hierarchy& h = hh->h;
        o->n_levels = static_cast<int64_t>(h.levels.size());
        o->n_coarse = h.n_coarse; o->nu1 = h.nu1; o->nu2 = h.nu2;
        o->C_gd = h.C_gd; o->C_op = h.C_op; o->C_fs = h.C_fs;
        o->T_ts = h.t.T_ts; o->T_cs = h.t.T_cs; o->T_sm = h.t.T_sm; o->T_pl = h.t.T_pl; o->T_rap = h.t.T_rap; o->T_p = h.t.T_p;
    });
}

int aspamg_hierarchy_level(const aspamg_hierarchy* hh, int64_t l, aspamg_level_view* o) {
    return guard([&] {
        const Hierarchy& h = hh->h;
        if (l < 0 || l >= static_cast<int64_t>(h.levels.size())) throw DimensionError("hierarchy: level out of range");
        const Level& L = h.levels[static_cast<size_t>(l)];
        o->A = view(L.A); o->G = view(L.smoother.G); o->Gt = view(L.Gt); o->P = view(L.P); o->Pt = view(L.Pt);
        o->omega = L.smoother.omega; o->lambda_hat = L.smoother.lambda_hat; o->kaporin_estimate = L.smoother.kaporin_estimate;
        o->refinement_passes = L.smoother.refinement_passes;
        o->smoother_exit = static_cast<int32_t>(L.smoother.exit_reason);
        o->n_tv = L.n_tv;
        o->t_smoother = L.t_smoother;
    });
}

int aspamg_hierarchy_coarse(const aspamg_hierarchy* hh, int64_t* n_c, const double** L) {
    return guard([&] { *n_c = hh->h.n_coarse; *L = hh->h.coarse_L.data(); });
}

int aspamg_hierarchy_save(const aspamg_hierarchy* hh, const char* path) {
    return guard([&] { hierarchy_save(hh->h, path); });
}

int aspamg_hierarchy_load(const char* path, aspamg_hierarchy** out) {
    return guard([&] {
        auto* hh = new aspamg_hierarchy;
        try { hh->h = hierarchy_load(path); } catch (...) { delete hh; throw; }
        *out = hh;
    });
}

void aspamg_hierarchy_free(aspamg_hierarchy* h) { delete h; }

int aspamg_srqcg(const aspamg_csr_view* A, const aspamg_csr_view* G, const double* V0, int64_t m, int64_t k_max,
                 int64_t k_ritz, double tol, uint64_t seed, double* V, double* quotients, int64_t* m_out) {
    return guard([&] {
        Csr a = from_view(*A), g = from_view(*G);
        Csr gt = transpose(g);
        Dense v0(a.n_rows, m);
        std::copy(V0, V0 + a.n_rows * m, v0.v.begin());
        SrqcgConfig cfg;
        cfg.n_tv = m; cfg.k_max = k_max; cfg.k_ritz = k_ritz; cfg.residual_tol = tol; cfg.seed = seed;
        TestSpace ts = srqcg(a, g, gt, v0, cfg);
        std::copy(ts.V.v.begin(), ts.V.v.end(), V);
        std::copy(ts.quotients.begin(), ts.quotients.end(), quotients);
        *m_out = ts.V.n_cols;
    });
}

int aspamg_afsai_build(const aspamg_csr_view* A, int64_t k, int64_t rho, double eps, aspamg_csr_owned** G,
                       aspamg_csr_view* G_view) {
    return guard([&] {
        Csr a = from_view(*A);
        auto* o = new aspamg_csr_owned;
        try { o->m = afsai_build(a, nullptr, k, rho, eps); } catch (...) { delete o; throw; }
        *G = o;
        *G_view = view(o->m);
    });
}

int aspamg_smoother_setup(const aspamg_csr_view* A, const aspamg_setup_config* c, aspamg_csr_owned** G,
                          aspamg_csr_view* G_view, double* omega, double* lambda_hat, int64_t* passes,
                          int* exit_reason) {
    return guard([&] {
        if (!A || !c || !G || !G_view || !omega || !lambda_hat || !passes || !exit_reason)
            throw ConfigError("aspamg_smoother_setup: null argument");
        SmootherConfig sc;
        sc.k0 = c->k0; sc.rho0 = c->rho0; sc.eps0 = c->eps0;
        sc.ki = c->ki; sc.rhoi = c->rhoi; sc.epsi = c->epsi;
        sc.omega_bar = c->omega_bar; sc.rho_bar = c->rho_bar;
        sc.lanczos_steps = c->lanczos_steps; sc.seed = c->seed;
        Csr a = from_view(*A);
        auto* o = new aspamg_csr_owned;
        try {
            FsaiSmoother sm = smoother_setup(a, sc);
            o->m = std::move(sm.G);
            *omega = sm.omega;
            *lambda_hat = sm.lambda_hat;
            *passes = sm.refinement_passes;
            *exit_reason = static_cast<int>(sm.exit_reason);
        } catch (...) { delete o; throw; }
        *G = o;
        *G_view = view(o->m);
    });
}

int aspamg_estimate_lambda_max(const aspamg_csr_view* G, const aspamg_csr_view* A, int64_t steps, uint64_t seed,
                               double* lambda_hat) {
    return guard([&] {
        Csr g = from_view(*G), a = from_view(*A);
        Csr gt = transpose(g);
        *lambda_hat = estimate_lambda_max(g, gt, a, steps, seed);
    });
}

void aspamg_csr_free(aspamg_csr_owned* m) { delete m; }

}  // extern "C"

// ------------------------------------------------ external test-space backend
namespace {
aspamg_srqcg_fn g_srqcg_fn = nullptr;
void* g_srqcg_user = nullptr;
}  // namespace

namespace aspamg {

bool srqcg_backend_set() { return g_srqcg_fn != nullptr; }

TestSpace srqcg_external(const Csr& A, const Csr& G, const Csr& Gt, const Dense& V0, const SrqcgConfig& cfg) {
    const aspamg_csr_view a = view(A), g = view(G), gt = view(Gt);
    const index_t n = A.n_rows, m = V0.n_cols;
    TestSpace ts;
    ts.V = Dense(n, m);
    ts.quotients.assign(static_cast<size_t>(m), 0.0);
    int64_t m_out = 0, iters = 0;
    int collapse = 0;
    const int st = g_srqcg_fn(g_srqcg_user, &a, &g, &gt, V0.v.data(), m, cfg.k_max, cfg.k_ritz, cfg.residual_tol,
                              cfg.seed, ts.V.v.data(), ts.quotients.data(), &m_out, &iters, &collapse);
    if (st != 0) {
        const std::string msg = "srqcg backend failed with status " + std::to_string(st);
        if (st == 1) throw DimensionError(msg);
        if (st == 3) throw NumericalError(msg);
        if (st == 4) throw ConfigError(msg);
        throw std::runtime_error(msg);
    }
    ts.V.resize_cols(m_out);
    ts.quotients.resize(static_cast<size_t>(m_out));
    ts.iterations = iters;
    ts.rank_collapse = collapse != 0;
    return ts;
}

}  // namespace aspamg

int aspamg_set_srqcg_backend(aspamg_srqcg_fn fn, void* user) {
    g_srqcg_fn = fn;
    g_srqcg_user = user;
    return 0;
}

// ------------------------------------------------------ external Galerkin backend
namespace {
aspamg_galerkin_fn g_galerkin_fn = nullptr;
void* g_galerkin_user = nullptr;

int csr_sink_alloc(void* sink, int64_t n_rows, int64_t n_cols, int64_t nnz, int64_t** rp, int64_t** ci, double** v) {
    auto* m = static_cast<aspamg::Csr*>(sink);
    try {
        m->n_rows = n_rows;
        m->n_cols = n_cols;
        m->rowptr.assign(static_cast<size_t>(n_rows) + 1, 0);
        m->col.assign(static_cast<size_t>(nnz), 0);
        m->val.assign(static_cast<size_t>(nnz), 0.0);
    } catch (...) {
        return 5;
    }
    *rp = m->rowptr.data();
    *ci = m->col.data();
    *v = m->val.data();
    return 0;
}
}  // namespace

namespace aspamg {

bool galerkin_backend_set() { return g_galerkin_fn != nullptr; }

Csr galerkin_external(const Csr& P, const Csr& Pt, const Csr& A) {
    const aspamg_csr_view p = view(P), pt = view(Pt), a = view(A);
    Csr C;
    const int st = g_galerkin_fn(g_galerkin_user, &p, &pt, &a, csr_sink_alloc, &C);
    if (st != 0) {
        const std::string msg = "galerkin backend failed with status " + std::to_string(st);
        if (st == 1) throw DimensionError(msg);
        if (st == 3) throw NumericalError(msg);
        if (st == 4) throw ConfigError(msg);
        throw std::runtime_error(msg);
    }
    C.symmetric = A.symmetric;
    return C;
}

}  // namespace aspamg

int aspamg_set_galerkin_backend(aspamg_galerkin_fn fn, void* user) {
    g_galerkin_fn = fn;
    g_galerkin_user = user;
    return 0;
}

// ------------------------------------------------------ external assembly backend
namespace {
aspamg_assembly_fn g_assembly_fn = nullptr;
void* g_assembly_user = nullptr;
}  // namespace

namespace aspamg {

bool assembly_backend_set() { return g_assembly_fn != nullptr; }

void assemble_external(const aspamg_hex_assembly& in, Csr& K) {
    const index_t n = K.n_rows;
    const bool sym = K.symmetric;
    const int st = g_assembly_fn(g_assembly_user, &in, csr_sink_alloc, &K);
    if (st != 0) {
        const std::string msg = "assembly backend failed with status " + std::to_string(st);
        if (st == 3) throw NumericalError("assembly: inverted or degenerate element");
        if (st == 4) throw ConfigError(msg);
        throw std::runtime_error(msg);
    }
    if (K.n_rows != n || K.n_cols != n) throw DimensionError("assembly backend returned a matrix of the wrong size");
    K.symmetric = sym;
}

}  // namespace aspamg

int aspamg_set_assembly_backend(aspamg_assembly_fn fn, void* user) {
    g_assembly_fn = fn;
    g_assembly_user = user;
    return 0;
}

int aspamg_galerkin(const aspamg_csr_view* P, const aspamg_csr_view* A, aspamg_csr_owned** out,
                    aspamg_csr_view* out_view) {
    return guard([&] {
        Csr p = from_view(*P), a = from_view(*A);
        auto* o = new aspamg_csr_owned;
        try { o->m = galerkin_triple(p, a); } catch (...) { delete o; throw; }
        *out = o;
        *out_view = view(o->m);
    });
}

// ------------------------------------------------------ external smoother backend
namespace {
aspamg_smoother_fn g_smoother_fn = nullptr;
void* g_smoother_user = nullptr;
}  // namespace

namespace aspamg {

bool smoother_backend_set() { return g_smoother_fn != nullptr; }

int smoother_external(const Csr& A, const SmootherConfig& cfg, double rho_bar, std::vector<double>& psi,
                      FsaiSmoother& out, Csr* ord) {
    const aspamg_csr_view a = view(A);
    aspamg_smoother_params prm{cfg.k0, cfg.rho0, cfg.eps0, cfg.ki, cfg.rhoi, cfg.epsi,
                               cfg.omega_bar, rho_bar, cfg.lanczos_steps, cfg.seed};
    FsaiSmoother s;
    psi.assign(static_cast<size_t>(A.n_rows), 0.0);
    int64_t passes = 0;
    int exit_reason = 0;
    const int st = g_smoother_fn(g_smoother_user, &a, &prm, csr_sink_alloc, &s.G, psi.data(), &s.omega,
                                 &s.lambda_hat, &passes, &exit_reason);
    if (st == -1) return 0;  // declined: the host computes this level
    if (st != 0 && st != -2) {
        const std::string msg = "smoother backend failed with status " + std::to_string(st);
        if (st == 1) throw DimensionError(msg);
        if (st == 2) throw NotSpdError(msg);
        if (st == 3) throw NumericalError(msg);
        if (st == 4) throw ConfigError(msg);
        throw std::runtime_error(msg);
    }
    s.refinement_passes = passes;
    s.exit_reason = static_cast<SmootherExit>(exit_reason);
    if (st == -2) {  // handed back: rows arrive in insertion order (the pattern, then i)
        Csr& G = s.G;
        if (ord) {
            ord->n_rows = ord->n_cols = G.n_rows;
            ord->rowptr = G.rowptr;
            ord->col = G.col;
            ord->val.clear();
        }
#pragma omp parallel num_threads(num_threads())
        {
            std::vector<std::pair<index_t, double>> e;
#pragma omp for schedule(dynamic, 1024)
            for (index_t i = 0; i < G.n_rows; ++i) {
                e.clear();
                for (index_t q = G.row_begin(i); q < G.row_end(i); ++q)
                    e.emplace_back(G.col[static_cast<size_t>(q)], G.val[static_cast<size_t>(q)]);
                std::sort(e.begin(), e.end());
                for (size_t q = 0; q < e.size(); ++q) {
                    G.col[static_cast<size_t>(G.row_begin(i)) + q] = e[q].first;
                    G.val[static_cast<size_t>(G.row_begin(i)) + q] = e[q].second;
                }
            }
        }
    }
    out = std::move(s);
    return st == -2 ? 2 : 1;
}

}  // namespace aspamg

int aspamg_set_smoother_backend(aspamg_smoother_fn fn, void* user) {
    g_smoother_fn = fn;
    g_smoother_user = user;
    return 0;
}
