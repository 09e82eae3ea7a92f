// aspamg_b200.hpp — C++ host API of the B200 solve path, mirroring the
// reference's solver interface on top of the two C-ABIs (header-only).
//
// Reference surface mirrored (same names, argument meaning, error behaviour):
//   SparseMatrix                  sparse_matrix.hpp:27-59 (int64 CSR, fp64 values)
//   DimensionError / NotSpdError / NumericalError / ConfigError / IoError
//                                 types.hpp:15-41
//   amg_setup(A, coordinates, cfg) -> Hierarchy
//   vcycle_apply(h, y) -> z
//   pcg(A, b, precond, rel_tol, max_it, x0) -> (x, SolveReport)
//   SolveReport {iterations, residual_history, converged, timings, complexities}
//                                 SPEC.md:498-501
// The setup runs on the CPU (lib/libaspamg_host.so); every per-iteration
// operation of vcycle_apply / pcg runs on the GPU (lib/libaspamg_gpu.so). There
// is no CPU fallback: without a device, GpuVcycle's constructor throws.
#pragma once

#include <array>
#include <cstdint>
#include <cstring>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

extern "C" {
#include "aspamg_gpu.h"
#include "aspamg_host.h"
}

namespace aspamg::b200 {

using index_t = std::int64_t;

struct DimensionError : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct NotSpdError : std::runtime_error { using std::runtime_error::runtime_error; };
struct NumericalError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ConfigError : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct IoError : std::runtime_error { using std::runtime_error::runtime_error; };
struct CudaError : std::runtime_error { using std::runtime_error::runtime_error; };

namespace detail {
inline void raise(int st, const char* msg) {
    const std::string m = msg ? msg : "";
    switch (st) {
        case 0: return;
        case 1: throw DimensionError(m);
        case 2: throw NotSpdError(m);
        case 3: throw NumericalError(m);
        case 4: throw ConfigError(m);
        case 7: throw IoError(m);
        default: throw CudaError(m);
    }
}
inline void host(int st) {
    if (st != 0) raise(st, aspamg_host_last_error());
}
}  // namespace detail

// sparse_matrix.hpp:27-59
struct SparseMatrix {
    index_t n_rows = 0;
    index_t n_cols = 0;
    std::vector<index_t> row_offsets;
    std::vector<index_t> col_indices;
    std::vector<double> values;
    bool symmetric = false;

    index_t nnz() const { return static_cast<index_t>(col_indices.size()); }
    aspamg_csr_view view() const {
        return {n_rows, n_cols, nnz(), row_offsets.data(), col_indices.data(), values.data()};
    }
    static SparseMatrix from_view(const aspamg_csr_view& v) {
        SparseMatrix m;
        m.n_rows = v.n_rows;
        m.n_cols = v.n_cols;
        if (v.row_offsets) m.row_offsets.assign(v.row_offsets, v.row_offsets + v.n_rows + 1);
        m.col_indices.assign(v.col_indices, v.col_indices + v.nnz);
        m.values.assign(v.values, v.values + v.nnz);
        return m;
    }
};

// BASELINE.json configs 1..5 (generator restated from fem.cpp, extended per SURVEY.md §8d).
struct GeneratedProblem {
    SparseMatrix stiffness;
    std::vector<double> rhs;
    std::vector<double> coordinates;  // n_nodes x 3, row-major
};

inline GeneratedProblem generate_config(int cfg, index_t scale = 1) {
    aspamg_problem* p = nullptr;
    detail::host(aspamg_problem_config(cfg, scale, &p));
    std::unique_ptr<aspamg_problem, void (*)(aspamg_problem*)> guard(p, aspamg_problem_free);
    GeneratedProblem out;
    aspamg_csr_view v;
    detail::host(aspamg_problem_matrix(p, &v));
    out.stiffness = SparseMatrix::from_view(v);
    out.stiffness.symmetric = true;
    const double* r = nullptr;
    index_t n = 0;
    detail::host(aspamg_problem_rhs(p, &r, &n));
    out.rhs.assign(r, r + n);
    detail::host(aspamg_problem_coords(p, &r, &n));
    out.coordinates.assign(r, r + 3 * n);
    return out;
}

inline aspamg_setup_config default_config() {  // Table-3 / SPEC defaults
    aspamg_setup_config c;
    detail::host(aspamg_setup_config_default(&c));
    return c;
}

// SPEC.md:430-433 (owns the CPU-side hierarchy)
class Hierarchy {
public:
    explicit Hierarchy(aspamg_hierarchy* h) : h_(h, aspamg_hierarchy_free) {}
    aspamg_hierarchy* get() const { return h_.get(); }
    aspamg_hierarchy_info info() const {
        aspamg_hierarchy_info i;
        detail::host(aspamg_hierarchy_info_get(h_.get(), &i));
        return i;
    }
    aspamg_level_view level(index_t l) const {
        aspamg_level_view v;
        detail::host(aspamg_hierarchy_level(h_.get(), l, &v));
        return v;
    }
    std::pair<index_t, const double*> coarse_factor() const {
        index_t n = 0;
        const double* L = nullptr;
        detail::host(aspamg_hierarchy_coarse(h_.get(), &n, &L));
        return {n, L};
    }
    void save(const std::string& path) const { detail::host(aspamg_hierarchy_save(h_.get(), path.c_str())); }
    static Hierarchy load(const std::string& path) {
        aspamg_hierarchy* h = nullptr;
        detail::host(aspamg_hierarchy_load(path.c_str(), &h));
        return Hierarchy(h);
    }

private:
    std::unique_ptr<aspamg_hierarchy, void (*)(aspamg_hierarchy*)> h_;
};

// SPEC.md:436-444
inline Hierarchy amg_setup(const SparseMatrix& A, std::span<const double> coordinates = {},
                           const aspamg_setup_config& cfg = default_config()) {
    aspamg_hierarchy* h = nullptr;
    const aspamg_csr_view v = A.view();
    detail::host(aspamg_setup(&v, coordinates.empty() ? nullptr : coordinates.data(),
                              static_cast<index_t>(coordinates.size() / 3), &cfg, &h));
    return Hierarchy(h);
}

// SPEC.md:498-501
struct SolveReport {
    index_t iterations = 0;
    std::vector<double> residual_history;  // ||r_k|| / ||b||, k = 1..iterations
    bool converged = false;
    double true_relative_residual = 0.0;
    double T_s = 0.0;  // device time of the solve (s)
    std::array<double, 3> complexities{1.0, 1.0, 0.0};  // C_gd, C_op, C_fs
};

// The uploaded hierarchy on one GPU: usable as pcg's `precond` operator.
class GpuVcycle {
public:
    explicit GpuVcycle(const Hierarchy& h, int device = 0) : h_(&h) {
        const int st = aspamg_gpu_ctx_create(device, &ctx_);  // status first, then its message
        detail::raise(st, aspamg_gpu_last_error(nullptr));
        try {
            const aspamg_hierarchy_info info = h.info();
            cx_ = {info.C_gd, info.C_op, info.C_fs};
            check(aspamg_gpu_set_cycle(ctx_, info.nu1, info.nu2));
            for (index_t l = 0; l < info.n_levels; ++l) {
                const aspamg_level_view lv = h.level(l);
                check(aspamg_gpu_upload_level(ctx_, l, &lv.A, &lv.G, &lv.Gt, &lv.P, &lv.Pt,
                                              l + 1 < info.n_levels ? lv.omega : 1.0));
                if (l == 0) n_ = lv.A.n_rows;
            }
            const auto [nc, L] = h.coarse_factor();
            check(aspamg_gpu_upload_coarse(ctx_, nc, L));
            check(aspamg_gpu_finalize(ctx_));
        } catch (...) {
            aspamg_gpu_ctx_destroy(ctx_);
            throw;
        }
    }
    GpuVcycle(const GpuVcycle&) = delete;
    GpuVcycle& operator=(const GpuVcycle&) = delete;
    ~GpuVcycle() { aspamg_gpu_ctx_destroy(ctx_); }

    index_t size() const { return n_; }
    const Hierarchy& hierarchy() const { return *h_; }
    // vcycle_apply(h, y)
    std::vector<double> operator()(std::span<const double> y) const {
        if (static_cast<index_t>(y.size()) != n_) throw DimensionError("vcycle_apply: y length mismatch");
        std::vector<double> z(y.size());
        check(aspamg_gpu_vcycle(ctx_, y.data(), z.data()));
        return z;
    }
    std::pair<std::vector<double>, SolveReport> solve(std::span<const double> b, double rel_tol, index_t max_it,
                                                      const std::vector<double>* x0) const {
        if (static_cast<index_t>(b.size()) != n_) throw DimensionError("pcg: b length mismatch");
        if (x0 && static_cast<index_t>(x0->size()) != n_) throw DimensionError("pcg: x0 length mismatch");
        std::vector<double> x(b.size());
        SolveReport rep;
        rep.residual_history.resize(static_cast<size_t>(std::max<index_t>(max_it, 1)));
        index_t n_it = 0;
        int conv = 0;
        double trr = 0.0;
        const int st = aspamg_gpu_pcg(ctx_, b.data(), x0 ? x0->data() : nullptr, rel_tol, max_it, x.data(),
                                      rep.residual_history.data(), &n_it, &conv, &trr);
        if (st != 6) check(st);  // 6 = not converged: a report, not an exception
        rep.iterations = n_it;
        rep.residual_history.resize(static_cast<size_t>(n_it));
        rep.converged = conv != 0;
        rep.true_relative_residual = trr;
        double ms = 0.0;
        aspamg_gpu_last_solve_ms(ctx_, &ms);
        rep.T_s = ms * 1e-3;
        rep.complexities = cx_;
        return {std::move(x), std::move(rep)};
    }

private:
    void check(int st) const {
        if (st != 0) detail::raise(st, aspamg_gpu_last_error(ctx_));
    }
    const Hierarchy* h_;
    aspamg_gpu_ctx* ctx_ = nullptr;
    index_t n_ = 0;
    std::array<double, 3> cx_{};
};

inline std::vector<double> vcycle_apply(const GpuVcycle& h, std::span<const double> y) { return h(y); }

// True when two CSR views hold the same matrix (same sizes, same arrays bit for
// bit); borrowed views of one buffer compare by pointer.
inline bool same_matrix(const aspamg_csr_view& a, const aspamg_csr_view& b) {
    if (a.n_rows != b.n_rows || a.n_cols != b.n_cols || a.nnz != b.nnz) return false;
    auto eq = [](const void* p, const void* q, size_t bytes) {
        return p == q || bytes == 0 || std::memcmp(p, q, bytes) == 0;
    };
    return eq(a.row_offsets, b.row_offsets, sizeof(int64_t) * static_cast<size_t>(a.n_rows + 1)) &&
           eq(a.col_indices, b.col_indices, sizeof(int64_t) * static_cast<size_t>(a.nnz)) &&
           eq(a.values, b.values, sizeof(double) * static_cast<size_t>(a.nnz));
}

// SPEC.md:504-512. The Krylov operator lives on the device as the finest level
// of `precond`'s hierarchy, so A must be that matrix: a different A of the same
// size (e.g. a stale cached hierarchy) would silently solve another system.
inline std::pair<std::vector<double>, SolveReport> pcg(const SparseMatrix& A, std::span<const double> b,
                                                       const GpuVcycle& precond, double rel_tol = 1e-8,
                                                       index_t max_it = 1000,
                                                       const std::vector<double>* x0 = nullptr) {
    if (A.n_rows != A.n_cols || A.n_rows != precond.size())
        throw DimensionError("pcg: operator does not match the preconditioner's finest level");
    if (!same_matrix(A.view(), precond.hierarchy().level(0).A))
        throw DimensionError("pcg: A differs from the finest operator of the preconditioner's hierarchy");
    return precond.solve(b, rel_tol, max_it, x0);
}

}  // namespace aspamg::b200
