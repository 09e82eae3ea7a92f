/* aspamg_gpu.h — C-ABI of the B200 (sm_100a) solve phase: PCG with one
 * aSP-AMG V(nu1,nu2)-cycle per iteration, every per-iteration operation in
 * hand-written CUDA (lib/libaspamg_gpu.so). No cuSPARSE/cuBLAS, no CPU
 * fallback: without a CUDA device every call fails with status 5.
 *
 * Reference interfaces each entry point replaces (the reference declares the
 * path in C++ and SPEC text; hierarchy.cpp / krylov.cpp / fsai.cpp are
 * missing, core/CMakeLists.txt:9-14):
 *   aspamg_gpu_upload_level   <- Level {A_k, FsaiSmoother{G, omega}, P_k}
 *                                SPEC.md:422-425, fsai.hpp:44-53; CSR exactly
 *                                as SparseMatrix (sparse_matrix.hpp:27-33);
 *                                G' and P' explicit (transpose, sparse_matrix.cpp:168-189)
 *   aspamg_gpu_upload_coarse  <- Hierarchy::coarse_factor (dense Cholesky),
 *                                SPEC.md:430-433,478
 *   aspamg_gpu_vcycle         <- vcycle_apply(h, y)  SPEC.md:445-453, Alg. 2
 *   aspamg_gpu_smooth         <- apply_smoothing_step(s, A, b, x) fsai.hpp:78-80
 *   aspamg_gpu_spmv           <- spmv(A, x) sparse_matrix.hpp:61-63 (on any uploaded operand)
 *   aspamg_gpu_pcg            <- pcg(A, b, precond, rel_tol, max_it, x0) SPEC.md:504-512,
 *                                A = finest A_0, precond = the uploaded V-cycle;
 *                                SolveReport fields n_it / residual_history /
 *                                converged
 *
 * Status codes: 0 OK, 1 dimension mismatch (DimensionError),
 * 2 not SPD: p'Ap <= 0 (NotSpdError), 3 numerical (NumericalError), 4 config
 * (ConfigError), 5 CUDA/runtime, 6 not converged (converged = 0, x valid).
 * Ownership: host buffers are borrowed for the duration of a call; all device
 * memory belongs to the context. Threading: one context = one CUDA stream,
 * calls on one context must be serialized; distinct contexts may run
 * concurrently.
 */
#ifndef ASPAMG_GPU_H
#define ASPAMG_GPU_H

#include <stdint.h>

#include "aspamg_csr.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct aspamg_gpu_ctx aspamg_gpu_ctx;

typedef struct aspamg_gpu_level_stats {
    int64_t n;
    int32_t a_format;     /* 0 CSR (thread group per row), 1 sliced 3x3 BSR, 2 SELL-32, 3 tile-local SELL */
    int64_t a_nnz, a_nnzb;
    double a_fill;        /* stored values / true nnz (1.0 = exact) */
    int64_t g_nnz, p_nnz;
    double omega;
    double alg_bytes_A, alg_bytes_G, alg_bytes_Gt, alg_bytes_P, alg_bytes_Pt; /* one product each */
    double device_bytes;
    int32_t fmt[5];       /* formats of A, G, G', P, P' (same codes as a_format) */
    double fill[5];       /* stored slots / true nnz per operand (padding of sliced formats) */
} aspamg_gpu_level_stats;

typedef struct aspamg_gpu_kernel_time {
    char name[48];
    int32_t level;
    double ms;
    double alg_bytes;
} aspamg_gpu_kernel_time;

const char* aspamg_gpu_last_error(const aspamg_gpu_ctx* ctx); /* ctx may be NULL (thread's last) */
int aspamg_gpu_device_count(int* n);
int aspamg_gpu_ctx_create(int device, aspamg_gpu_ctx** out);
int aspamg_gpu_ctx_destroy(aspamg_gpu_ctx* ctx);
/* keys (set before the first upload; unknown keys -> status 4):
 *   "bsr"          1 auto (exactly 3x3-blocked operands -> sliced BSR3), 0 never
 *   "device_loop"  1 CUDA-graph while-loop (default), 0 host loop
 *   "stream_bytes" operators above this many bytes use evict-first loads
 *   "keep_bytes"   coarsest levels up to this many bytes load with evict-last
 *   "coarse_mode"  1 explicit inverse-factor triangles (default), 0 one-CTA substitution
 *   "idx16"        16-bit column offsets where rows span < 2^16 columns (default 1)
 *   "sell_*"       SELL layout / kernel choices (chunk height, sorting window, unroll)
 *   "csr_per_thread", "csr_pf", "csr_long"  CSR kernel group size (entries per thread of the
 *                  mean row), row-pointer prefetch (1 = groups <= 16, default; 2 = also warp-per-row),
 *                  long-row split threshold (0 = off)
 *   "csr_max_group" (32) threads per row cap for operands with >= 600k / cap rows: one warp per
 *                  row, no shared-memory combine
 *   "csrw"         (4) pipelined warp-per-row CSR kernel for group-32 operands: column indices one
 *                  round ahead across row boundaries; value = columns per lane per round (4 / 8), 0 off
 *   "csr_blocked"  (250000) k_csrw operands with at least this many rows: a contiguous row block per
 *                  CTA instead of rows interleaved over the grid (L1 reuse of the x gathers); 0 = off
 *   "csr_noalloc"  (0) k_csrw matrix loads bypass L1 (measured slower)
 *   "xsell", "xsell_*"  tile-local SELL (x footprint staged in shared memory, 16-bit local columns):
 *                  role mask (1 A, 2 G, 4 G', 8 P, 16 P'; default 0 = off) and its layout choices
 *   "fuse_rr"      (0) restriction fused with the residual: one cooperative launch per level computes
 *                  r = y - A s, crosses a grid barrier, gathers r_c = P' r (measured slower)
 *   "tail_dense"   (1500) levels below the first one with <= this many rows collapse into one dense operator
 *   "tail_rows"    levels below this many rows run as one persistent cooperative kernel (0 = off)
 *   "pdl"          programmatic dependent launch (default 1)
 * Every variant sums in a fixed order (deterministic); the sliced formats (BSR3, SELL, tile-local
 * SELL) are bit-identical to the reference spmv (tests/test_gpu_parity.py). */
int aspamg_gpu_set_option(aspamg_gpu_ctx* ctx, const char* key, int64_t value);
int aspamg_gpu_set_cycle(aspamg_gpu_ctx* ctx, int64_t nu1, int64_t nu2);
/* Levels 0..L-2 carry A, G, G', P, P' and omega; the coarsest level L-1 carries
 * A only (G..Pt may be NULL or empty). Levels must be uploaded in order. */
int aspamg_gpu_upload_level(aspamg_gpu_ctx* ctx, int64_t level, const aspamg_csr_view* A,
                            const aspamg_csr_view* G, const aspamg_csr_view* Gt,
                            const aspamg_csr_view* P, const aspamg_csr_view* Pt, double omega);
int aspamg_gpu_upload_coarse(aspamg_gpu_ctx* ctx, int64_t n_c, const double* L_colmajor);
int aspamg_gpu_finalize(aspamg_gpu_ctx* ctx);

int aspamg_gpu_num_levels(aspamg_gpu_ctx* ctx, int64_t* n);
int aspamg_gpu_level_info(aspamg_gpu_ctx* ctx, int64_t level, aspamg_gpu_level_stats* out);

/* host buffers */
int aspamg_gpu_vcycle(aspamg_gpu_ctx* ctx, const double* y, double* z);
int aspamg_gpu_spmv(aspamg_gpu_ctx* ctx, int64_t level, int which /*0 A,1 G,2 G',3 P,4 P'*/,
                    const double* x, double* y);
int aspamg_gpu_smooth(aspamg_gpu_ctx* ctx, int64_t level, const double* b, const double* x, double* out);
int aspamg_gpu_coarse_solve(aspamg_gpu_ctx* ctx, const double* y, double* z);
int aspamg_gpu_pcg(aspamg_gpu_ctx* ctx, const double* b, const double* x0_or_null, double rel_tol,
                   int64_t max_it, double* x, double* history, int64_t* n_it, int* converged,
                   double* true_rel_res);
/* device buffers (b, x0, x on the context's device); history is a host buffer */
int aspamg_gpu_vcycle_device(aspamg_gpu_ctx* ctx, const double* y_dev, double* z_dev);
int aspamg_gpu_pcg_device(aspamg_gpu_ctx* ctx, const double* b_dev, const double* x0_dev_or_null,
                          double rel_tol, int64_t max_it, double* x_dev, double* history,
                          int64_t* n_it, int* converged, double* true_rel_res);

/* GPU setup: SRQCG (Alg. 4) on S = G A G' with the
 * solve's SpMV kernels; bit-identical to the host aspamg_srqcg (same operation order).
 * Signature = aspamg_srqcg_fn of aspamg_host.h (pass it to aspamg_set_srqcg_backend);
 * device = (void*)(intptr_t)device_index. V0, V: n x m column-major host buffers,
 * quotients[m]; m <= 64. Creates and destroys its own context. */
int aspamg_gpu_srqcg(void* device, const aspamg_csr_view* A, const aspamg_csr_view* G,
                     const aspamg_csr_view* Gt, const double* V0, int64_t m, int64_t k_max, int64_t k_ritz,
                     double tol, uint64_t seed, double* V, double* quotients, int64_t* m_out,
                     int64_t* iterations, int* rank_collapse);

/* GPU setup: Galerkin A_c = P' (A P) with the host's summation
 * order (bit-identical to aspamg's galerkin_triple); the result is written into buffers
 * obtained from alloc(sink, ...). Signature = aspamg_galerkin_fn of aspamg_host.h.
 * device = (void*)(intptr_t)device_index. */
int aspamg_gpu_galerkin(void* device, const aspamg_csr_view* P, const aspamg_csr_view* Pt,
                        const aspamg_csr_view* A, aspamg_csr_alloc_fn alloc, void* sink);

/* GPU setup: adaptive FSAI smoother set-up (aFSAI build,
 * Lanczos lambda_max x 1.05, omega = min(1, 2/lambda), refinement passes; fsai.hpp:27-83,
 * SPEC.md:157-232) with the host's operation order — bit-identical G, omega, lambda.
 * G is written through alloc(sink, ...); psi[n] receives the final pass's Schur
 * complements; exit_reason 0 omega reached, 1 density bound, 2 pattern stagnation.
 * Signature = aspamg_smoother_fn of aspamg_host.h. device = (void*)(intptr_t)index. */
int aspamg_gpu_smoother_setup(void* device, const aspamg_csr_view* A, const aspamg_smoother_params* prm,
                              aspamg_csr_alloc_fn alloc, void* sink, double* psi, double* omega,
                              double* lambda_hat, int64_t* passes, int* exit_reason);
/* Level policy of aspamg_gpu_smoother_setup (process-wide):
 *   "smoother_max_mean_row" (300), "smoother_min_rows" (50000): operators with longer mean
 *      rows or fewer rows are declined (returns -1, nothing written);
 *   "smoother_max_pattern" (64): before a refinement pass whose pattern bound exceeds it,
 *      returns -2 with the state after the last finished pass (G, psi, omega, lambda,
 *      passes); the caller continues the refinement loop. <= 0 disables a rule. */
int aspamg_gpu_set_setup_policy(const char* key, double value);
/* aFSAI build alone from the identity start, for verification. */
int aspamg_gpu_afsai_build(void* device, const aspamg_csr_view* A, int64_t k, int64_t rho, double eps,
                           aspamg_csr_alloc_fn alloc, void* sink, double* psi);

/* GPU setup: assembly of the structured-hex elasticity stiffness
 * (fem.cpp:87-184: 2x2x2-Gauss element stiffness, pattern, element-order fill) on the
 * device, bit-identical to the host generator's K (same element-stiffness source, no FMA
 * contraction, every entry summed in element order). K is written through alloc(sink, ...)
 * as the reference-layout CSR. Signature = aspamg_assembly_fn of aspamg_host.h.
 * device = (void*)(intptr_t)index. Status 3: inverted / degenerate element. */
int aspamg_gpu_assemble_hex(void* device, const aspamg_hex_assembly* in, aspamg_csr_alloc_fn alloc, void* sink);

/* Layout self-check of the tile-local SELL format ("xsell") — host only, no
 * device needed: builds the format's arrays for A exactly as upload does and walks them on
 * the CPU with the kernel's indexing (staged x window, 16-bit local columns, quads, tile
 * permutation). y must equal spmv(A, x) (sparse_matrix.cpp:96-107) bit for bit. */
int aspamg_gpu_xsell_layout_spmv(const aspamg_csr_view* A, int64_t tile_rows, int64_t fold, int64_t gran,
                                 const double* x, double* y);

/* measurement helpers */
int aspamg_gpu_last_solve_ms(aspamg_gpu_ctx* ctx, double* ms);      /* device time of the last pcg */
int aspamg_gpu_launch_count(aspamg_gpu_ctx* ctx, int64_t* n);       /* kernels launched by the last pcg */
int aspamg_gpu_profile_iteration(aspamg_gpu_ctx* ctx, aspamg_gpu_kernel_time* out, int cap, int* count);
int aspamg_gpu_time_vcycle(aspamg_gpu_ctx* ctx, int reps, double* avg_ms); /* standalone V-cycle graph */
/* graph-mode per-op time: each op of the PCG body replayed `reps` times inside one CUDA graph */
int aspamg_gpu_profile_ops(aspamg_gpu_ctx* ctx, int reps, aspamg_gpu_kernel_time* out, int cap, int* count);
int aspamg_gpu_time_kernel(aspamg_gpu_ctx* ctx, const char* name, int64_t level, int reps,
                           double* avg_ms, double* alg_bytes);
int aspamg_gpu_stream(aspamg_gpu_ctx* ctx, void** stream);
int aspamg_gpu_alloc_pinned(int64_t bytes, void** out);
int aspamg_gpu_free_pinned(void* p);
int aspamg_gpu_alloc_device(aspamg_gpu_ctx* ctx, int64_t bytes, void** out);
int aspamg_gpu_free_device(aspamg_gpu_ctx* ctx, void* p);
int aspamg_gpu_memcpy(aspamg_gpu_ctx* ctx, void* dst, const void* src, int64_t bytes); /* any direction, synchronous */

#ifdef __cplusplus
}
#endif

#endif /* ASPAMG_GPU_H */
