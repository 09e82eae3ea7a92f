// aspamg_solve — the `solve` command of SPEC.md:619-624 on the B200 path,
// written against the C++ host API (include/aspamg_b200.hpp).
//
//   aspamg_solve (--config N [--scale S] | --matrix K.mtx [--coords xyz.txt] [--rhs ones])
//                [--rel-tol 1e-8] [--max-it 1000] [--device 0] [--threads T]
//                [--hierarchy cache.bin] [--report out.json] [key=value ...]
//
// key=value overrides use the paper's parameter names: k_g, rho_g, eps_g, n_tv, n_rq,
// theta, n_max, kappa_p, d_p, eps_p, omega_bar, rho_bar, nu1, nu2, max_levels, min_coarse_size, seed.
// Exit codes: 0 ok, 1 config error, 2 I/O error, 3 non-convergence, 4 numerical failure,
// 5 CUDA/runtime failure (no device: the path has no CPU fallback).
#include "../../../include/aspamg_b200.hpp"

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <map>
#include <sstream>
#include <string>
#include <vector>

using namespace aspamg::b200;

namespace {

// Matrix Market coordinate real {general,symmetric}: 1-based,
// symmetric storage expanded to the full pattern, duplicates summed in order.
SparseMatrix read_matrix_market(const std::string& path) {
    std::ifstream f(path);
    if (!f) throw IoError("cannot open " + path);
    std::string line;
    if (!std::getline(f, line)) throw IoError("empty file " + path);
    std::istringstream hs(line);
    std::string banner, object, format, field, symmetry;
    hs >> banner >> object >> format >> field >> symmetry;
    if (banner != "%%MatrixMarket" || object != "matrix" || format != "coordinate")
        throw IoError("unsupported Matrix Market header (line 1)");
    if (field != "real" && field != "double" && field != "integer") throw IoError("non-real field (line 1)");
    const bool sym = symmetry == "symmetric";
    if (!sym && symmetry != "general") throw IoError("unsupported symmetry " + symmetry + " (line 1)");
    long long lineno = 1;
    while (std::getline(f, line)) {
        ++lineno;
        if (!line.empty() && line[0] != '%') break;
    }
    std::istringstream ss(line);
    long long nr = 0, nc = 0, nz = 0;
    if (!(ss >> nr >> nc >> nz) || nr <= 0 || nc <= 0 || nz < 0)
        throw IoError("bad size line (line " + std::to_string(lineno) + ")");
    std::vector<std::vector<std::pair<index_t, double>>> rows(static_cast<size_t>(nr));
    for (long long k = 0; k < nz; ++k) {
        if (!std::getline(f, line)) throw IoError("truncated entries (line " + std::to_string(lineno + 1) + ")");
        ++lineno;
        std::istringstream es(line);
        long long i, j;
        double v;
        if (!(es >> i >> j >> v)) throw IoError("bad entry (line " + std::to_string(lineno) + ")");
        if (i < 1 || i > nr || j < 1 || j > nc) throw IoError("index out of bounds (line " + std::to_string(lineno) + ")");
        rows[static_cast<size_t>(i - 1)].emplace_back(j - 1, v);
        if (sym && i != j) rows[static_cast<size_t>(j - 1)].emplace_back(i - 1, v);
    }
    SparseMatrix A;
    A.n_rows = nr;
    A.n_cols = nc;
    A.symmetric = sym;
    A.row_offsets.assign(static_cast<size_t>(nr) + 1, 0);
    for (index_t i = 0; i < nr; ++i) {
        auto& r = rows[static_cast<size_t>(i)];
        std::stable_sort(r.begin(), r.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
        for (size_t k = 0; k < r.size(); ++k) {
            double s = r[k].second;
            while (k + 1 < r.size() && r[k + 1].first == r[k].first) s += r[++k].second;
            A.col_indices.push_back(r[k].first);
            A.values.push_back(s);
        }
        A.row_offsets[static_cast<size_t>(i) + 1] = A.nnz();
    }
    return A;
}

std::vector<double> read_coordinates(const std::string& path, index_t n_nodes) {
    std::ifstream f(path);
    if (!f) throw IoError("cannot open " + path);
    std::vector<double> xyz;
    double a, b, c;
    while (f >> a >> b >> c) xyz.insert(xyz.end(), {a, b, c});
    if (static_cast<index_t>(xyz.size()) != 3 * n_nodes) throw IoError("coordinate count mismatch in " + path);
    return xyz;
}

void apply_override(aspamg_setup_config& c, const std::string& key, const std::string& val) {
    const double v = std::stod(val);
    const std::map<std::string, std::function<void(double)>> set = {
        {"k_g", [&](double x) { c.k0 = (int64_t)x; }},        {"rho_g", [&](double x) { c.rho0 = (int64_t)x; }},
        {"eps_g", [&](double x) { c.eps0 = x; }},              {"n_tv", [&](double x) { c.n_tv = (int64_t)x; }},
        {"n_rq", [&](double x) { c.n_rq = (int64_t)x; }},      {"theta", [&](double x) { c.theta = (int64_t)x; }},
        {"n_max", [&](double x) { c.n_max = (int64_t)x; }},    {"kappa_p", [&](double x) { c.kappa_p = x; }},
        {"d_p", [&](double x) { c.d_p = (int64_t)x; }},        {"eps_p", [&](double x) { c.eps_p = x; }},
        {"omega_bar", [&](double x) { c.omega_bar = x; }},     {"rho_bar", [&](double x) { c.rho_bar = x; }},
        {"nu1", [&](double x) { c.nu1 = (int64_t)x; }},        {"nu2", [&](double x) { c.nu2 = (int64_t)x; }},
        {"max_levels", [&](double x) { c.max_levels = (int64_t)x; }},
        {"min_coarse_size", [&](double x) { c.min_coarse_size = (int64_t)x; }},
        {"seed", [&](double x) { c.seed = (uint64_t)x; }},
    };
    auto it = set.find(key);
    if (it == set.end()) throw ConfigError("unknown config key " + key);
    it->second(v);
}

double seconds_since(std::chrono::steady_clock::time_point t) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t).count();
}

}  // namespace

int main(int argc, char** argv) {
    try {
        int cfg_id = 0, device = 0, threads = 0;
        index_t scale = 1, max_it = 1000;
        double rel_tol = 1e-8;
        std::string matrix, coords, report, hier_path, rhs_kind;
        aspamg_setup_config cfg = default_config();
        for (int i = 1; i < argc; ++i) {
            const std::string a = argv[i];
            auto next = [&]() -> std::string {
                if (i + 1 >= argc) throw ConfigError("missing value for " + a);
                return argv[++i];
            };
            if (a == "--config") cfg_id = std::stoi(next());
            else if (a == "--scale") scale = std::stoll(next());
            else if (a == "--matrix") matrix = next();
            else if (a == "--coords") coords = next();
            else if (a == "--rhs") rhs_kind = next();
            else if (a == "--rel-tol") rel_tol = std::stod(next());
            else if (a == "--max-it") max_it = std::stoll(next());
            else if (a == "--device") device = std::stoi(next());
            else if (a == "--threads") threads = std::stoi(next());
            else if (a == "--hierarchy") hier_path = next();
            else if (a == "--report") report = next();
            else if (a.find('=') != std::string::npos) apply_override(cfg, a.substr(0, a.find('=')), a.substr(a.find('=') + 1));
            else throw ConfigError("unknown argument " + a);
        }
        if ((cfg_id == 0) == matrix.empty()) throw ConfigError("give exactly one of --config N or --matrix file");
        aspamg_host_set_threads(threads);
        const auto t0 = std::chrono::steady_clock::now();
        SparseMatrix A;
        std::vector<double> b, xyz;
        if (cfg_id) {
            GeneratedProblem p = generate_config(cfg_id, scale);
            A = std::move(p.stiffness);
            b = std::move(p.rhs);
            xyz = std::move(p.coordinates);
        } else {
            A = read_matrix_market(matrix);
            if (!coords.empty()) xyz = read_coordinates(coords, A.n_rows / 3);
            b.assign(static_cast<size_t>(A.n_rows), 1.0);  // SPEC.md:622 default rhs: ones
        }
        if (rhs_kind == "ones") b.assign(static_cast<size_t>(A.n_rows), 1.0);
        const auto ts = std::chrono::steady_clock::now();
        std::optional<Hierarchy> h;
        if (!hier_path.empty()) {
            std::ifstream probe(hier_path);
            if (probe) {
                h.emplace(Hierarchy::load(hier_path));
                // a cached hierarchy must have been built from this very matrix
                if (!same_matrix(A.view(), h->level(0).A))
                    throw ConfigError("--hierarchy " + hier_path + " was built from a different matrix");
            }
        }
        if (!h) {
            h.emplace(amg_setup(A, xyz, cfg));
            if (!hier_path.empty()) h->save(hier_path);
        }
        const double T_p = seconds_since(ts);
        GpuVcycle M(*h, device);
        const auto [x, rep] = pcg(A, b, M, rel_tol, max_it);
        const double T_t = seconds_since(t0);
        const aspamg_hierarchy_info info = h->info();
        std::ostringstream js;
        js.precision(17);
        js << "{\"n\": " << A.n_rows << ", \"nnz\": " << A.nnz() << ", \"levels\": " << info.n_levels
           << ", \"iterations\": " << rep.iterations << ", \"converged\": " << (rep.converged ? "true" : "false")
           << ", \"true_relative_residual\": " << rep.true_relative_residual << ", \"T_ts\": " << info.T_ts
           << ", \"T_cs\": " << info.T_cs << ", \"T_sm\": " << info.T_sm << ", \"T_pl\": " << info.T_pl
           << ", \"T_rap\": " << info.T_rap << ", \"T_p\": " << T_p << ", \"T_s\": " << rep.T_s
           << ", \"T_t\": " << T_t << ", \"C_gd\": " << info.C_gd << ", \"C_op\": " << info.C_op
           << ", \"C_fs\": " << info.C_fs << ", \"residual_history\": [";
        for (size_t k = 0; k < rep.residual_history.size(); ++k) js << (k ? ", " : "") << rep.residual_history[k];
        js << "]}";
        if (!report.empty()) {
            std::ofstream o(report);
            if (!o) throw IoError("cannot write " + report);
            o << js.str() << "\n";
        }
        std::printf("%s\n", js.str().c_str());
        std::fprintf(stderr, "n=%lld levels=%lld C_gd=%.3f C_op=%.3f C_fs=%.3f n_it=%lld T_p=%.3fs T_s=%.4fs T_t=%.3fs %s\n",
                     (long long)A.n_rows, (long long)info.n_levels, info.C_gd, info.C_op, info.C_fs,
                     (long long)rep.iterations, T_p, rep.T_s, T_t, rep.converged ? "converged" : "NOT converged");
        return rep.converged ? 0 : 3;
    } catch (const ConfigError& e) {
        std::fprintf(stderr, "config error: %s\n", e.what());
        return 1;
    } catch (const IoError& e) {
        std::fprintf(stderr, "I/O error: %s\n", e.what());
        return 2;
    } catch (const NotSpdError& e) {
        std::fprintf(stderr, "numerical failure (not SPD): %s\n", e.what());
        return 4;
    } catch (const NumericalError& e) {
        std::fprintf(stderr, "numerical failure: %s\n", e.what());
        return 4;
    } catch (const DimensionError& e) {
        std::fprintf(stderr, "config error (dimension): %s\n", e.what());
        return 1;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "runtime error: %s\n", e.what());
        return 5;
    }
}
