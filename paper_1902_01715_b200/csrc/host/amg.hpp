// aSP-AMG setup (CPU) producing the hierarchy the B200 solve consumes.
//
// The reference ships only the declarations (fsai.hpp:27-83) and SPEC text for
// these modules; fsai.cpp, test_space.cpp, coarsening.cpp, prolongation.cpp and
// hierarchy.cpp are missing (core/CMakeLists.txt:5-19). Each function below is
// a restatement of the SPEC operation it cites; the algorithm references are
// PAPER.md Alg. 1 (:263-286), Alg. 3 (:374-387), Alg. 4 (:522-563),
// Alg. 5 (:659-685).
#pragma once

#include "core.hpp"

#include <cstdint>
#include <string>
#include <vector>

namespace aspamg {

// ---------------------------------------------------------------- smoother
enum class SmootherExit { omega_reached = 0, density_bound = 1, pattern_stagnation = 2 };

struct SmootherConfig {  // fsai.hpp:27-42
    index_t k0 = 4, rho0 = 4;
    double eps0 = 1e-3;
    index_t ki = 2, rhoi = 4;
    double epsi = 1e-3;
    double omega_bar = 0.95;
    double rho_bar = 0.0;  // 0 = 2 * nnz_r(lower(A))
    index_t lanczos_steps = 10;
    std::uint64_t seed = 1234;
};

struct FsaiSmoother {  // fsai.hpp:44-53
    Csr G;                 // lower triangular, positive diagonal
    double omega = 1.0;
    double lambda_hat = 1.0;
    double kaporin_estimate = 1.0;
    index_t refinement_passes = 0;
    SmootherExit exit_reason = SmootherExit::omega_reached;
};

// SPEC.md:172-180 (fsai.hpp:61-66). G_start == nullptr means identity start; otherwise
// each row's start pattern (columns < i) is taken in G_start's stored order, which is
// the order of the row's incremental factor (smoother_setup passes insertion order).
Csr afsai_build(const Csr& A, const Csr* G_start, index_t k, index_t rho, double eps,
                std::vector<double>* psi_out = nullptr);
// SPEC.md:181-189 (fsai.hpp:68-71): Lanczos on G A G', x1.05.
double estimate_lambda_max(const Csr& G, const Csr& Gt, const Csr& A, index_t steps, std::uint64_t seed);
double compute_omega(double lambda_hat);
FsaiSmoother smoother_setup(const Csr& A, const SmootherConfig& cfg);  // SPEC.md:194-202, Alg. 3
// smoother_setup through the registered external backend (aspamg_set_smoother_backend), if any:
// returns G, omega, lambda_hat, passes, exit reason, and psi (for the Kaporin estimate).
bool smoother_backend_set();
// 0: the backend declined (status -1), the host computes the level; 1: complete;
// 2: handed back after a finished pass (status -2), the host continues the refinement loop;
// the backend then delivers G's rows in insertion order (pattern, then i): G is sorted
// here and *ord receives the insertion-ordered twin (the next pass's start pattern).
int smoother_external(const Csr& A, const SmootherConfig& cfg, double rho_bar, std::vector<double>& psi,
                      FsaiSmoother& out, Csr* ord);
// x' = x + omega G'(G(b - A x)) (host reference; Gt explicit)
std::vector<double> apply_smoothing_step(const Csr& G, const Csr& Gt, double omega, const Csr& A,
                                         const std::vector<double>& b, const std::vector<double>& x);

// --------------------------------------------------------------- test space
struct SrqcgConfig {
    index_t n_tv = 10;
    index_t k_max = 10;  // n_rq
    index_t k_ritz = 1;
    double residual_tol = 1e-2;
    std::uint64_t seed = 1234;
};

struct TestSpace {
    Dense V;  // n x n_tv, orthonormal columns
    std::vector<double> quotients;
    index_t iterations = 0;
    bool rank_collapse = false;
};

Dense seed_space(const Dense* rbms, index_t n_tv, index_t n, std::uint64_t seed);
TestSpace srqcg(const Csr& A, const Csr& G, const Csr& Gt, const Dense& V0, const SrqcgConfig& cfg);  // Alg. 4
// srqcg through the registered external backend (aspamg_set_srqcg_backend), if any.
bool srqcg_backend_set();
TestSpace srqcg_external(const Csr& A, const Csr& G, const Csr& Gt, const Dense& V0, const SrqcgConfig& cfg);
// galerkin_triple through the registered external backend (aspamg_set_galerkin_backend), if any.
bool galerkin_backend_set();
Csr galerkin_external(const Csr& P, const Csr& Pt, const Csr& A);

// --------------------------------------------------------------- coarsening
Csr affinity_soc(const Csr& A, const Dense& V);
Csr filter_soc(const Csr& soc, index_t theta);
struct CfSplit {
    std::vector<char> is_coarse;
    std::vector<index_t> coarse_index;  // fine -> coarse id, -1 for F
    index_t n_coarse = 0;
};
CfSplit select_coarse_mis(const Csr& g);

// ------------------------------------------------------------- prolongation
struct DplsConfig {
    index_t d_p = 2;
    double eps_p = 1e-2;
    double kappa_p = 50.0;
    index_t n_max = 5;
};
enum class DplsStop : std::int8_t { coarse = 0, tolerance = 1, condition = 2, exhausted = 3, n_max = 4 };
struct Prolongation {
    Csr P;
    std::vector<DplsStop> stop;
};
Prolongation dpls_build(const Csr& soc, const CfSplit& split, const Dense& V, const DplsConfig& cfg);  // Alg. 5

// ---------------------------------------------------------------- hierarchy
struct HierarchyConfig {
    index_t max_levels = 10;
    index_t min_coarse_size = 500;
    index_t nu1 = 1, nu2 = 1;
    SmootherConfig smoother;
    SrqcgConfig srqcg;
    index_t theta = 5;
    DplsConfig dpls;
};

struct Level {
    Csr A;
    FsaiSmoother smoother;  // absent (empty G) on the coarsest level
    Csr Gt;                 // explicit G' (transpose, sparse_matrix.cpp:168-189)
    Csr P, Pt;              // absent on the coarsest level
    index_t n_tv = 0;
    double t_smoother = 0;  // seconds (diagnostic, not persisted)
};

struct SetupTimings {  // SPEC.md:499 taxonomy (seconds)
    double T_ts = 0, T_cs = 0, T_sm = 0, T_pl = 0, T_rap = 0, T_p = 0;
};

struct Hierarchy {
    std::vector<Level> levels;
    std::vector<double> coarse_L;  // dense lower Cholesky of the last A, column-major n_c x n_c
    index_t n_coarse = 0;
    double C_gd = 1, C_op = 1, C_fs = 0;
    SetupTimings t;
    index_t nu1 = 1, nu2 = 1;
};

// Alg. 1 / SPEC.md:436-444. coords: n/3 x 3 free-node coordinates or empty.
Hierarchy amg_setup(const Csr& A, const std::vector<double>& coords, const HierarchyConfig& cfg);
void compute_complexities(Hierarchy& h);

void hierarchy_save(const Hierarchy& h, const std::string& path);
Hierarchy hierarchy_load(const std::string& path);

}  // namespace aspamg
