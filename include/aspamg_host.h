/* aspamg_host.h — C-ABI of the CPU side of the B200 solve path: problem
 * generation (input side) and the aSP-AMG setup that produces the hierarchy
 * uploaded once to the GPU (BASELINE.json north_star: "The preconditioner
 * hierarchy ... is produced by the reference's CPU setup").
 *
 * Reference interfaces this replaces (the reference is C++; these are the
 * binding points a maintainer would expose over FFI):
 *   aspamg_problem_*      <- assemble_hex_cube / rigid_body_modes
 *                            /root/reference/proj/core/include/aspamg/fem.hpp:43-66
 *   aspamg_setup          <- amg_setup(A, coordinates, cfg)
 *                            (hierarchy.cpp/.hpp missing, core/CMakeLists.txt:12)
 *   aspamg_setup_config   <- HierarchyConfig / SmootherConfig / SrqcgConfig /
 *                            DplsConfig: SPEC.md:166-169,243-246,366-369,426-429,
 *                            fsai.hpp:27-42
 *   aspamg_hierarchy_level<- Level {A_k, smoother_k(G, omega), P_k} SPEC.md:422-425
 *
 * Conventions: every call returns an int status (0 OK, 1 dimension, 2 not SPD,
 * 3 numerical, 4 config, 5 runtime, 7 I/O); aspamg_host_last_error() returns
 * the calling thread's last message. CSR views are borrowed pointers into
 * objects owned by the library (valid until the owning object is freed):
 * int64 offsets / columns and fp64 values, exactly sparse_matrix.hpp:27-33.
 */
#ifndef ASPAMG_HOST_H
#define ASPAMG_HOST_H

#include <stdint.h>

#include "aspamg_csr.h"

#ifdef __cplusplus
extern "C" {
#endif


typedef struct aspamg_problem aspamg_problem;
typedef struct aspamg_hierarchy aspamg_hierarchy;

typedef struct aspamg_setup_config {
    /* aFSAI smoother (fsai.hpp:27-42; Table 3 k_g, rho_g, eps_g) */
    int64_t k0, rho0; double eps0;
    int64_t ki, rhoi; double epsi;
    double omega_bar, rho_bar; /* rho_bar 0 = 2 * nnz_r(lower(A)) */
    int64_t lanczos_steps;
    /* test space (Table 3 n_tv, n_rq) */
    int64_t n_tv, n_rq, k_ritz; double srqcg_tol;
    /* coarsening + prolongation (Table 3 theta, n_max, kappa_p; SPEC d_p, eps_p) */
    int64_t theta, d_p, n_max; double eps_p, kappa_p;
    /* hierarchy */
    int64_t max_levels, min_coarse_size, nu1, nu2;
    uint64_t seed;
} aspamg_setup_config;

typedef struct aspamg_level_view {
    aspamg_csr_view A, G, Gt, P, Pt; /* G..Pt empty (n_rows 0) on the coarsest level */
    double omega, lambda_hat, kaporin_estimate;
    int64_t refinement_passes;
    int32_t smoother_exit; /* 0 omega_reached, 1 density_bound, 2 pattern_stagnation */
    int64_t n_tv;
    double t_smoother;     /* seconds of this level's smoother set-up (0 after a load) */
} aspamg_level_view;

typedef struct aspamg_hierarchy_info {
    int64_t n_levels, n_coarse, nu1, nu2;
    double C_gd, C_op, C_fs;
    double T_ts, T_cs, T_sm, T_pl, T_rap, T_p; /* seconds */
} aspamg_hierarchy_info;

const char* aspamg_host_last_error(void);
int aspamg_host_set_threads(int n); /* <1 = OpenMP default */
int aspamg_host_get_threads(void);

/* BASELINE.json configs 1..5; scale >= 1 divides element counts (test sizes). */
int aspamg_problem_config(int cfg, int64_t scale, aspamg_problem** out);
/* Uniform-material structured cube (fem.hpp:62-64), clamp_faces: bit set
 * 1 x_min, 2 x_max, 4 y_min, 8 y_max, 16 z_min, 32 z_max. rhs = ones. */
int aspamg_problem_hex(int64_t nx, int64_t ny, int64_t nz, double spacing, double young,
                       double poisson, uint32_t clamp_faces, aspamg_problem** out);
int aspamg_problem_matrix(const aspamg_problem* p, aspamg_csr_view* out);
int aspamg_problem_rhs(const aspamg_problem* p, const double** rhs, int64_t* n);
int aspamg_problem_coords(const aspamg_problem* p, const double** xyz, int64_t* n_nodes);
void aspamg_problem_free(aspamg_problem* p);

int aspamg_setup_config_default(aspamg_setup_config* cfg);
/* Setup components exposed for verification (SPEC.md operations):
 * SRQCG (Alg. 4) on S = G A G' from V0 (n x m column-major); writes V (n x m_out,
 * orthonormal columns, ascending quotients), quotients[m_out], m_out. */
int aspamg_srqcg(const aspamg_csr_view* A, const aspamg_csr_view* G, const double* V0, int64_t m,
                 int64_t k_max, int64_t k_ritz, double tol, uint64_t seed, double* V, double* quotients,
                 int64_t* m_out);
/* Test-space backend: when set, aspamg_setup runs the level-0
 * SRQCG through fn instead of the CPU restatement, e.g. aspamg_gpu_srqcg from
 * libaspamg_gpu.so with user = (void*)(intptr_t)device. Same arguments as aspamg_srqcg
 * plus G' (explicit) and the iteration / rank-collapse outputs; fn must return 0 on
 * success (its status is passed through otherwise). NULL restores the CPU path.
 * Process-wide; not thread-safe against a concurrent aspamg_setup. */
typedef int (*aspamg_srqcg_fn)(void* user, const aspamg_csr_view* A, const aspamg_csr_view* G,
                               const aspamg_csr_view* Gt, const double* V0, int64_t m, int64_t k_max,
                               int64_t k_ritz, double tol, uint64_t seed, double* V, double* quotients,
                               int64_t* m_out, int64_t* iterations, int* rank_collapse);
int aspamg_set_srqcg_backend(aspamg_srqcg_fn fn, void* user);
typedef struct aspamg_csr_owned aspamg_csr_owned;
/* Galerkin backend: when set, aspamg_setup forms every coarse
 * operator A_c = P' (A P) through fn (e.g. aspamg_gpu_galerkin) instead of the CPU
 * sparse products; fn writes the result through alloc(sink, ...). NULL restores the CPU
 * path. Process-wide. */
typedef int (*aspamg_galerkin_fn)(void* user, const aspamg_csr_view* P, const aspamg_csr_view* Pt,
                                  const aspamg_csr_view* A, aspamg_csr_alloc_fn alloc, void* sink);
int aspamg_set_galerkin_backend(aspamg_galerkin_fn fn, void* user);
/* Host Galerkin product (the CPU restatement; exposed for verification). The result
 * is owned by *out (free with aspamg_csr_free). */
int aspamg_galerkin(const aspamg_csr_view* P, const aspamg_csr_view* A, aspamg_csr_owned** out,
                    aspamg_csr_view* out_view);
/* Assembly backend (fem.cpp:87-184): when set, the generator
 * (aspamg_problem_config / aspamg_problem_hex) hands the element stiffness matrices, the
 * CSR pattern and the fill of K to fn (e.g. aspamg_gpu_assemble_hex), which writes K
 * through alloc(sink, ...). The mesh description is computed on the host (node
 * coordinates incl. the seeded perturbation, clamp -> free numbering, material table).
 * fn must reproduce the host assembly bit for bit. NULL restores the CPU path. */
typedef int (*aspamg_assembly_fn)(void* user, const aspamg_hex_assembly* in, aspamg_csr_alloc_fn alloc, void* sink);
int aspamg_set_assembly_backend(aspamg_assembly_fn fn, void* user);
/* Smoother backend: when set, aspamg_setup runs each level's
 * adaptive FSAI set-up through fn (e.g. aspamg_gpu_smoother_setup); the host forms the
 * Kaporin estimate from the returned psi. fn may return -1 to decline a level (the
 * host then computes it) or -2 to hand back the refinement loop after its last finished
 * pass (the host continues it; G's rows then arrive in insertion order — the pattern in
 * the order its entries were added, then the diagonal — which is the factor order the
 * next pass restarts from). NULL restores the CPU path. Process-wide. */
typedef int (*aspamg_smoother_fn)(void* user, const aspamg_csr_view* A, const aspamg_smoother_params* prm,
                                  aspamg_csr_alloc_fn alloc, void* sink, double* psi, double* omega,
                                  double* lambda_hat, int64_t* passes, int* exit_reason);
int aspamg_set_smoother_backend(aspamg_smoother_fn fn, void* user);
/* aFSAI build from the identity start: returns G via a new hierarchy-owned
 * buffer set; G_out views stay valid until aspamg_csr_free. */
int aspamg_afsai_build(const aspamg_csr_view* A, int64_t k, int64_t rho, double eps, aspamg_csr_owned** G,
                       aspamg_csr_view* G_view);
/* smoother_setup (Alg. 3) of one operator on the host (through the
 * registered smoother backend, if any): G (free with aspamg_csr_free), omega,
 * lambda_hat, refinement passes and exit reason (0 omega reached, 1 density bound,
 * 2 pattern stagnation). */
int aspamg_smoother_setup(const aspamg_csr_view* A, const aspamg_setup_config* cfg, aspamg_csr_owned** G,
                          aspamg_csr_view* G_view, double* omega, double* lambda_hat, int64_t* passes,
                          int* exit_reason);
/* Lanczos estimate of lambda_max(G A G') x 1.05. */
int aspamg_estimate_lambda_max(const aspamg_csr_view* G, const aspamg_csr_view* A, int64_t steps, uint64_t seed,
                               double* lambda_hat);
void aspamg_csr_free(aspamg_csr_owned* m);
/* coords: n_nodes x 3 row-major free-node coordinates (3 dofs per node,
 * interleaved) or NULL; drives the rigid-body-mode seeding of the test space. */
int aspamg_setup(const aspamg_csr_view* A, const double* coords, int64_t n_nodes,
                 const aspamg_setup_config* cfg, aspamg_hierarchy** out);
int aspamg_hierarchy_info_get(const aspamg_hierarchy* h, aspamg_hierarchy_info* out);
int aspamg_hierarchy_level(const aspamg_hierarchy* h, int64_t level, aspamg_level_view* out);
/* Dense lower Cholesky factor of the coarsest A, column-major n_c x n_c. */
int aspamg_hierarchy_coarse(const aspamg_hierarchy* h, int64_t* n_c, const double** L_colmajor);
int aspamg_hierarchy_save(const aspamg_hierarchy* h, const char* path);
int aspamg_hierarchy_load(const char* path, aspamg_hierarchy** out);
void aspamg_hierarchy_free(aspamg_hierarchy* h);

#ifdef __cplusplus
}
#endif

#endif /* ASPAMG_HOST_H */
