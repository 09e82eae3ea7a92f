/* oracle.c — CPU oracle of the B200 solve path. TEST INFRASTRUCTURE ONLY
 * (see oracle.h for what it restates and who may call it). Plain C, fp64,
 * every reduction in index order; OpenMP only splits independent rows of a
 * product, which leaves results bit-identical to one thread
 * (parallel.hpp:4-6 contract).
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static int g_threads = 1;
static orc_spmv_hook g_hook = NULL;

void orc_set_threads(int n) { g_threads = n < 1 ? 1 : n; }
void orc_set_spmv_hook(orc_spmv_hook fn) { g_hook = fn; }

/* sparse_matrix.cpp:96-107: y_i = sum_k v_k x_{c_k}, ascending k */
int orc_spmv(const orc_csr* A, const double* x, double* y) {
    if (g_hook && A->ref) {
        g_hook(A->ref, x, y);
        return 0;
    }
    const int64_t n = A->n_rows;
#pragma omp parallel for schedule(static) num_threads(g_threads) if (g_threads > 1 && n > 2048)
    for (int64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int64_t k = A->rp[i]; k < A->rp[i + 1]; ++k) s += A->v[k] * x[A->ci[k]];
        y[i] = s;
    }
    return 0;
}

/* dot_mode 0 (default): one sequential sum in index order (the reference's
 * single-thread order). dot_mode 1: 4096-element blocks summed sequentially,
 * block partials summed in index order — an equally valid fixed order, used
 * only to measure how sensitive a solve's iteration count is to the dot's
 * summation order. */
static int g_dot_mode = 0;
void orc_set_dot_mode(int m) { g_dot_mode = m; }

static double dotp(int64_t n, const double* a, const double* b) {
    if (g_dot_mode == 1) {
        /* block partials (computed in parallel when threads > 1), summed in index order:
         * the same bits for every thread count */
        const int64_t nb = (n + 4095) / 4096;
        double* part = (double*)malloc((size_t)(nb > 0 ? nb : 1) * sizeof(double));
#pragma omp parallel for schedule(static) num_threads(g_threads) if (g_threads > 1 && nb > 8)
        for (int64_t bk = 0; bk < nb; ++bk) {
            const int64_t i0 = bk * 4096, i1 = i0 + 4096 < n ? i0 + 4096 : n;
            double t = 0.0;
            for (int64_t i = i0; i < i1; ++i) t += a[i] * b[i];
            part[bk] = t;
        }
        double s = 0.0;
        for (int64_t bk = 0; bk < nb; ++bk) s += part[bk];
        free(part);
        return s;
    }
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

/* x' = x + w G'(G(b - A x)); x == NULL means x = 0 (then x' = w G'(G b)). */
static void smooth_into(const orc_level* L, const double* b, const double* x, double* out, double* r, double* t) {
    const int64_t n = L->A.n_rows;
    if (x) {
        orc_spmv(&L->A, x, r);
        for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
    } else {
        memcpy(r, b, (size_t)n * sizeof(double));
    }
    orc_spmv(&L->G, r, t);
    orc_spmv(&L->Gt, t, r);
    if (x) {
        for (int64_t i = 0; i < n; ++i) out[i] = x[i] + L->omega * r[i];
    } else {
        for (int64_t i = 0; i < n; ++i) out[i] = L->omega * r[i];
    }
}

int orc_smooth(const orc_hier* h, int64_t level, const double* b, const double* x, double* out) {
    if (level < 0 || level >= h->n_levels - 1) return 1;
    const orc_level* L = &h->levels[level];
    const int64_t n = L->A.n_rows;
    double* r = (double*)malloc((size_t)n * sizeof(double));
    double* t = (double*)malloc((size_t)n * sizeof(double));
    smooth_into(L, b, x, out, r, t);
    free(r);
    free(t);
    return 0;
}

/* L L' z = y, L column-major lower (column-oriented forward, then backward). */
int orc_coarse_solve(const orc_hier* h, const double* y, double* z) {
    const int64_t n = h->n_c;
    const double* L = h->Lcm;
    if (z != y) memcpy(z, y, (size_t)n * sizeof(double));
    for (int64_t j = 0; j < n; ++j) {
        const double zj = z[j] / L[j + j * n];
        z[j] = zj;
        for (int64_t i = j + 1; i < n; ++i) z[i] -= L[i + j * n] * zj;
    }
    for (int64_t j = n - 1; j >= 0; --j) {
        const double zj = z[j] / L[j + j * n];
        z[j] = zj;
        for (int64_t i = 0; i < j; ++i) z[i] -= L[j + i * n] * zj;
    }
    return 0;
}

static void vcycle_rec(const orc_hier* h, int64_t k, const double* y, double* z) {
    if (k == h->n_levels - 1) {
        orc_coarse_solve(h, y, z);
        return;
    }
    const orc_level* L = &h->levels[k];
    const int64_t n = L->A.n_rows, nc = L->P.n_cols;
    double* s = z; /* s accumulates in z */
    /* per-level workspace kept between V-cycles (a fresh 50-MB malloc per vector per
     * cycle costs page faults that are not part of the algorithm) */
    static double* ws[64][5];
    static int64_t wsn[64], wsc[64];
    if (k < 64 && (wsn[k] < n || wsc[k] < nc)) {
        for (int j = 0; j < 5; ++j) free(ws[k][j]);
        for (int j = 0; j < 3; ++j) ws[k][j] = (double*)malloc((size_t)n * sizeof(double));
        for (int j = 3; j < 5; ++j) ws[k][j] = (double*)malloc((size_t)(nc > 0 ? nc : 1) * sizeof(double));
        wsn[k] = n;
        wsc[k] = nc;
    }
    double *r = ws[k][0], *t = ws[k][1], *u = ws[k][2], *rc = ws[k][3], *hc = ws[k][4];
    /* nu1 pre-smoothing steps from s = 0 */
    for (int64_t it = 0; it < h->nu1; ++it) {
        if (it == 0) smooth_into(L, y, NULL, s, r, t);
        else { smooth_into(L, y, s, u, r, t); memcpy(s, u, (size_t)n * sizeof(double)); }
    }
    if (h->nu1 == 0) memset(s, 0, (size_t)n * sizeof(double));
    /* r = y - A s ; r_c = P' r */
    orc_spmv(&L->A, s, r);
    for (int64_t i = 0; i < n; ++i) r[i] = y[i] - r[i];
    orc_spmv(&L->Pt, r, rc);
    vcycle_rec(h, k + 1, rc, hc);
    /* s += P h_c */
    orc_spmv(&L->P, hc, t);
    for (int64_t i = 0; i < n; ++i) s[i] = s[i] + t[i];
    /* nu2 post-smoothing steps from s */
    for (int64_t it = 0; it < h->nu2; ++it) {
        smooth_into(L, y, s, u, r, t);
        memcpy(s, u, (size_t)n * sizeof(double));
    }
}

int orc_vcycle(const orc_hier* h, const double* y, double* z) {
    if (h->n_levels < 1) return 1;
    vcycle_rec(h, 0, y, z);
    return 0;
}

/* SPEC.md:504-512 standard PCG; history[k-1] = ||r_k|| / ||b||. */
int orc_pcg(const orc_hier* h, const double* b, const double* x0, double rel_tol, int64_t max_it,
            double* x, double* history, int64_t* n_it, int* converged, double* true_rel_res) {
    const orc_csr* A = &h->levels[0].A;
    const int64_t n = A->n_rows;
    double* r = (double*)malloc((size_t)n * sizeof(double));
    double* z = (double*)malloc((size_t)n * sizeof(double));
    double* p = (double*)malloc((size_t)n * sizeof(double));
    double* q = (double*)malloc((size_t)n * sizeof(double));
    int status = 0;
    *n_it = 0;
    *converged = 0;
    const double bnorm = sqrt(dotp(n, b, b));
    if (x0) {
        memcpy(x, x0, (size_t)n * sizeof(double));
        orc_spmv(A, x, q);
        for (int64_t i = 0; i < n; ++i) r[i] = b[i] - q[i];
    } else {
        memset(x, 0, (size_t)n * sizeof(double));
        memcpy(r, b, (size_t)n * sizeof(double));
    }
    if (bnorm == 0.0) {
        memset(x, 0, (size_t)n * sizeof(double));
        *converged = 1;
        *true_rel_res = 0.0;
        goto done;
    }
    if (sqrt(dotp(n, r, r)) <= rel_tol * bnorm) {
        *converged = 1;
    } else {
        orc_vcycle(h, r, z);
        memcpy(p, z, (size_t)n * sizeof(double));
        double rz = dotp(n, r, z);
        for (int64_t k = 1; k <= max_it; ++k) {
            orc_spmv(A, p, q);
            const double pq = dotp(n, p, q);
            if (!(pq > 0.0)) { status = 2; break; }
            const double alpha = rz / pq;
                for (int64_t i = 0; i < n; ++i) {
                x[i] = x[i] + alpha * p[i];
                r[i] = r[i] - alpha * q[i];
            }
            const double rn = sqrt(dotp(n, r, r));
            history[k - 1] = rn / bnorm;
            *n_it = k;
            if (rn <= rel_tol * bnorm) { *converged = 1; break; }
            orc_vcycle(h, r, z);
            const double rz_new = dotp(n, r, z);
            const double beta = rz_new / rz;
            rz = rz_new;
                for (int64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
        }
    }
    /* true residual recheck */
    orc_spmv(A, x, q);
    for (int64_t i = 0; i < n; ++i) q[i] = b[i] - q[i];
    *true_rel_res = sqrt(dotp(n, q, q)) / bnorm;
    if (*converged && !(*true_rel_res <= 10.0 * rel_tol)) *converged = 0;
done:
    free(r); free(z); free(p); free(q);
    return status;
}
