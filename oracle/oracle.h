/* oracle.h — CPU oracle for the B200 solve path. TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this library, and only as the checker / the CPU
 * baseline. The product path (paper_1902_01715_b200, lib/libaspamg_gpu.so)
 * never links or calls it.
 *
 * What it restates (plain C, sequential order of the reference):
 *   orc_spmv          sparse_matrix.cpp:96-107 (ascending column order per row)
 *   orc_smooth        apply_smoothing_step, fsai.hpp:78-80 / SPEC.md:203-206
 *   orc_coarse_solve  "Forward and Backward solve" L L' z = y, PAPER.md:291-292,
 *                     SPEC.md:448,478
 *   orc_vcycle        vcycle_apply, SPEC.md:445-453 / Alg. 2
 *   orc_pcg           pcg, SPEC.md:504-512,518-525 / PAPER.md:760-762
 * Parity status: spmv/transpose are pinned bit-exactly against the reference's
 * own compiled sparse_matrix.cpp (oracle/_ref, tests/golden). The V-cycle, the
 * smoother step and PCG have no reference code (fsai.cpp, hierarchy.cpp,
 * krylov.cpp are missing, core/CMakeLists.txt:9-14); they are pinned by the
 * SPEC known-answer examples in tests/.
 *
 * The spmv used inside smooth/vcycle/pcg can be routed through the
 * reference's own spmv (oracle/_ref/libaspamg_ref.so) with orc_set_spmv_hook;
 * that is the "reference" CPU baseline of bench.py.
 */
#ifndef ASPAMG_ORACLE_H
#define ASPAMG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_csr {
    int64_t n_rows, n_cols;
    const int64_t* rp;
    const int64_t* ci;
    const double* v;
    void* ref; /* optional handle into oracle/_ref for the spmv hook */
} orc_csr;

typedef struct orc_level {
    orc_csr A, G, Gt, P, Pt;
    double omega;
} orc_level;

typedef struct orc_hier {
    int64_t n_levels;
    const orc_level* levels;
    int64_t n_c;
    const double* Lcm; /* coarsest Cholesky factor, column-major n_c x n_c */
    int64_t nu1, nu2;
} orc_hier;

typedef void (*orc_spmv_hook)(void* ref, const double* x, double* y);

void orc_set_threads(int n);
void orc_set_dot_mode(int mode); /* 0 sequential (default); 1 blocked (sensitivity studies only) */
void orc_set_spmv_hook(orc_spmv_hook fn); /* NULL = the oracle's own loop */

int orc_spmv(const orc_csr* A, const double* x, double* y);
int orc_smooth(const orc_hier* h, int64_t level, const double* b, const double* x, double* out);
int orc_coarse_solve(const orc_hier* h, const double* y, double* z);
int orc_vcycle(const orc_hier* h, const double* y, double* z);
/* status: 0 ok, 2 not SPD (p'q <= 0); n_it = len(history), history[k-1] = ||r_k||/||b|| */
int orc_pcg(const orc_hier* h, const double* b, const double* x0, double rel_tol, int64_t max_it,
            double* x, double* history, int64_t* n_it, int* converged, double* true_rel_res);

#ifdef __cplusplus
}
#endif

#endif
