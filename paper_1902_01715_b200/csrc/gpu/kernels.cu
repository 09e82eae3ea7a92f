// sm_100a kernels of the solve path (PCG + V(nu1,nu2)-cycle), fp64.
//
// Replaces, per SURVEY.md §2 kernel table:
//   k_bsr3   <- spmv sparse_matrix.cpp:96-107 on K (exact 3x3 blocks)
//   k_csr    <- spmv / spmv_transpose sparse_matrix.cpp:96-124 on G, G', P, P', A_l
//              (G', P' stored explicitly -> every product is a row gather)
//   epilogues fuse the V-cycle vector updates (Alg. 2):
//              s = w G't, r = y - A s, s += P e_c, z = s + w G't
//   k_pcg_*  <- pcg SPEC.md:504-512 vector updates with fused dots
//   k_coarse <- "Forward and Backward solve" PAPER.md:291-292
// All dots are deterministic two-pass reductions (fixed per-CTA tree, last CTA
// sums the partials in index order): no floating-point atomics, run-to-run
// bit-identical (SPEC.md:77 determinism contract).
#include "kernels.cuh"

#include <cuda_runtime.h>

namespace aspamg_gpu {

namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Fixed-tree CTA sum; result valid in every thread.
__device__ __forceinline__ double block_sum(double v, double* sh) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double t = lane < (blockDim.x >> 5) ? sh[lane] : 0.0;
    t = warp_sum(t);
    return t;
}

__device__ void finalize(const Red& red, double s, double s2) {
    PcgState* st = red.st;
    switch (red.fin) {
        case FIN_STORE:
            red.out[0] = s;
            break;
        case FIN_PQ:
            st->pq = s;
            if (!(s > 0.0)) {
                st->notspd = 1;
                st->done = 1;
            } else {
                st->alpha = st->rz / s;
            }
            break;
        case FIN_RZ:
            st->beta = st->k == 0 ? 0.0 : s / st->rz;
            st->rz = s;
            break;
        case FIN_RR: {
            st->rr = s;
            const double rn = sqrt(s);
            st->history[st->k] = rn / st->bnorm;
            st->k += 1;
            const int conv = rn <= st->tol * st->bnorm;
            st->converged = conv;
            st->done = conv || st->k >= st->max_it;
            if (red.use_cond) cudaGraphSetConditional(red.cond, st->done ? 0u : 1u);
            break;
        }
        case FIN_INIT: {
            st->bnorm = sqrt(s);
            st->rr = s2;
            st->k = 0;
            st->notspd = 0;
            st->beta = 0.0;
            const int conv = st->bnorm == 0.0 || sqrt(s2) <= st->tol * st->bnorm;
            st->converged = conv;
            st->done = conv || st->max_it <= 0;
            break;
        }
        default:
            break;
    }
}

// Per-CTA partial -> partials[blockIdx]; last CTA reduces in index order.
__device__ void reduce_finish(double v, const Red& red) {
    __shared__ double sh[32];
    __shared__ int last;
    const double t = block_sum(v, sh);
    if (threadIdx.x == 0) {
        red.partials[blockIdx.x] = t;
        __threadfence();
        const unsigned ticket = atomicAdd(red.counter, 1u);
        last = ticket == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double s = 0.0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) s += __ldcg(red.partials + i);
    s = block_sum(s, sh);
    if (threadIdx.x == 0) {
        finalize(red, s, 0.0);
        *red.counter = 0;
    }
}

__device__ void reduce_finish2(double v, double v2, const Red& red) {
    __shared__ double sh[32];
    __shared__ int last;
    const double t = block_sum(v, sh);
    const double t2 = block_sum(v2, sh);
    if (threadIdx.x == 0) {
        red.partials[blockIdx.x] = t;
        red.partials[gridDim.x + blockIdx.x] = t2;
        __threadfence();
        const unsigned ticket = atomicAdd(red.counter, 1u);
        last = ticket == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double s = 0.0, s2 = 0.0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) {
        s += __ldcg(red.partials + i);
        s2 += __ldcg(red.partials + gridDim.x + i);
    }
    s = block_sum(s, sh);
    s2 = block_sum(s2, sh);
    if (threadIdx.x == 0) {
        finalize(red, s, s2);
        *red.counter = 0;
    }
}

__device__ __forceinline__ double epilogue(int epi, double s, const double* aux, int row, double omega) {
    switch (epi) {
        case EPI_SCALE: return omega * s;
        case EPI_RESID: return aux[row] - s;
        case EPI_ADD: return aux[row] + s;
        case EPI_ADDSCALE: return aux[row] + omega * s;
        default: return s;
    }
}

template <bool STREAM, class T>
__device__ __forceinline__ T ld_mat(const T* p) {
    if constexpr (STREAM) return __ldcs(p);
    else return __ldg(p);
}

__device__ __forceinline__ bool is_done(const int* done) {
    return done != nullptr && *reinterpret_cast<const volatile int*>(done) != 0;
}

// ---------------------------------------------------------------- CSR SpMV
// G threads per row (warp-uniform loop so sub-warp shuffles stay converged);
// each lane sums its strided entries in ascending order, then a fixed
// shuffle tree. Loads of values/columns are coalesced across the group.
template <int G, bool STREAM>
__global__ void __launch_bounds__(kBlock) k_csr(DCsr M, int epi, const double* __restrict__ x, double* y,
                                                 const double* aux, double omega, const double* dotw, Red red,
                                                 const int* done) {
    if (is_done(done)) return;
    constexpr int GPW = 32 / G;
    const int lane = threadIdx.x & 31;
    const int gl = lane % G, gw = lane / G;
    const int warp = (blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * kBlock) >> 5;
    double dacc = 0.0;
    for (int base = warp * GPW; base < M.n_rows; base += nwarps * GPW) {
        const int row = base + gw;
        double s = 0.0;
        if (row < M.n_rows) {
            const int b = __ldg(M.rp + row), e = __ldg(M.rp + row + 1);
#pragma unroll 4
            for (int k = b + gl; k < e; k += G) {
                const double v = ld_mat<STREAM>(M.v + k);
                const int c = ld_mat<STREAM>(M.ci + k);
                s = fma(v, __ldg(x + c), s);
            }
        }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o, G);
        if (gl == 0 && row < M.n_rows) {
            const double out = epilogue(epi, s, aux, row, omega);
            y[row] = out;
            if (dotw) dacc = fma(out, dotw[row], dacc);
        }
    }
    if (red.fin != FIN_NONE) reduce_finish(dacc, red);
}

// --------------------------------------------------------------- BSR3 SpMV
// One warp per block row. The block row's values are one contiguous run of
// 9*nnzb doubles; lane l takes flat positions l, l+32, ... (perfectly
// coalesced 256-B warp loads), tracking (block, entry) incrementally
// (32 = 3*9 + 5), and accumulates into the block's row r = entry/3 with the
// gathered x[3*col + entry%3]. Three fixed shuffle trees finish the rows.
template <bool STREAM>
__global__ void __launch_bounds__(kBlock) k_bsr3(DBsr3 M, int epi, const double* __restrict__ x, double* y,
                                                  const double* aux, double omega, const double* dotw, Red red,
                                                  const int* done) {
    if (is_done(done)) return;
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * kBlock) >> 5;
    double dacc = 0.0;
    for (int br = warp; br < M.nb; br += nwarps) {
        const int b0 = __ldg(M.rp + br), b1 = __ldg(M.rp + br + 1);
        const int nval = 9 * (b1 - b0);
        const double* vb = M.v + 9ll * b0;
        const int* cb = M.ci + b0;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
        int blk = lane / 9, e = lane - 9 * (lane / 9);
#pragma unroll 4
        for (int p = lane; p < nval; p += 32) {
            const double v = ld_mat<STREAM>(vb + p);
            const int c = ld_mat<STREAM>(cb + blk);
            const int r = e >= 6 ? 2 : (e >= 3 ? 1 : 0);
            const double xv = __ldg(x + 3 * c + (e - 3 * r));
            if (r == 0) a0 = fma(v, xv, a0);
            else if (r == 1) a1 = fma(v, xv, a1);
            else a2 = fma(v, xv, a2);
            blk += 3;
            e += 5;
            if (e >= 9) { e -= 9; blk += 1; }
        }
        a0 = warp_sum(a0);
        a1 = warp_sum(a1);
        a2 = warp_sum(a2);
        if (lane < 3) {
            const double s = lane == 0 ? a0 : (lane == 1 ? a1 : a2);
            const int row = 3 * br + lane;
            const double out = epilogue(epi, s, aux, row, omega);
            y[row] = out;
            if (dotw) dacc = fma(out, dotw[row], dacc);
        }
    }
    if (red.fin != FIN_NONE) reduce_finish(dacc, red);
}

// ------------------------------------------------------------- PCG vectors
__global__ void __launch_bounds__(kBlock) k_pcg_p(int n, const double* __restrict__ z, double* __restrict__ p,
                                                   const PcgState* st, const int* done) {
    if (is_done(done)) return;
    const bool first = st->k == 0;
    const double beta = st->beta;
    for (int i = blockIdx.x * kBlock + threadIdx.x; i < n; i += gridDim.x * kBlock)
        p[i] = first ? z[i] : fma(beta, p[i], z[i]);
}

__global__ void __launch_bounds__(kBlock) k_pcg_xr(int n, double* __restrict__ x, double* __restrict__ r,
                                                    const double* __restrict__ p, const double* __restrict__ q,
                                                    Red red, const int* done) {
    if (is_done(done)) {
        if (red.use_cond && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(red.cond, 0u);
        return;
    }
    const double alpha = red.st->alpha;
    double acc = 0.0;
    for (int i = blockIdx.x * kBlock + threadIdx.x; i < n; i += gridDim.x * kBlock) {
        x[i] = fma(alpha, p[i], x[i]);
        const double ri = fma(-alpha, q[i], r[i]);
        r[i] = ri;
        acc = fma(ri, ri, acc);
    }
    reduce_finish(acc, red);
}

__global__ void __launch_bounds__(kBlock) k_pcg_init(int n, const double* __restrict__ b, const double* __restrict__ r,
                                                      Red red) {
    double s = 0.0, s2 = 0.0;
    for (int i = blockIdx.x * kBlock + threadIdx.x; i < n; i += gridDim.x * kBlock) {
        s = fma(b[i], b[i], s);
        s2 = fma(r[i], r[i], s2);
    }
    reduce_finish2(s, s2, red);
}

__global__ void __launch_bounds__(kBlock) k_zero(int n, double* y, const int* done) {
    if (is_done(done)) return;
    for (int i = blockIdx.x * kBlock + threadIdx.x; i < n; i += gridDim.x * kBlock) y[i] = 0.0;
}

// ---------------------------------------------------------- coarse solve
// One CTA of 1024 threads; z lives in shared memory. Blocked substitution
// with 32-wide panels: the diagonal 32x32 triangle is applied through its
// precomputed inverse (one warp, 32 independent FMAs per lane), then all 32
// warps update the remaining rows from the panel (row-contiguous loads:
// Lrm for the forward sweep, Lcm == row-major L' for the backward sweep).
constexpr int kCoarseThreads = 1024;

__global__ void __launch_bounds__(kCoarseThreads) k_coarse(int n, const double* __restrict__ Lrm,
                                                            const double* __restrict__ Lcm,
                                                            const double* __restrict__ Dinv_f,
                                                            const double* __restrict__ Dinv_b,
                                                            const double* __restrict__ y, double* z,
                                                            const double* dotw, Red red, const int* done) {
    if (is_done(done)) return;
    extern __shared__ double zs[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int i = threadIdx.x; i < n; i += blockDim.x) zs[i] = y[i];
    __syncthreads();
    const int nb = (n + 31) / 32;
    // forward: L w = y
    for (int jb = 0; jb < nb; ++jb) {
        const int j0 = 32 * jb, bs = min(32, n - j0);
        if (w == 0) {
            const double* D = Dinv_f + 1024ll * jb;
            double acc = 0.0;
            if (lane < bs)
                for (int j = 0; j <= lane; ++j) acc = fma(D[32 * lane + j], zs[j0 + j], acc);
            __syncwarp();
            if (lane < bs) zs[j0 + lane] = acc;
        }
        __syncthreads();
        const double zl = lane < bs ? zs[j0 + lane] : 0.0;
        for (int i = j0 + bs + w; i < n; i += nw) {
            double t = lane < bs ? Lrm[(long long)i * n + j0 + lane] * zl : 0.0;
            t = warp_sum(t);
            if (lane == 0) zs[i] -= t;
        }
        __syncthreads();
    }
    // backward: L' z = w
    for (int jb = nb - 1; jb >= 0; --jb) {
        const int j0 = 32 * jb, bs = min(32, n - j0);
        if (w == 0) {
            const double* D = Dinv_b + 1024ll * jb;
            double acc = 0.0;
            if (lane < bs)
                for (int j = lane; j < bs; ++j) acc = fma(D[32 * lane + j], zs[j0 + j], acc);
            __syncwarp();
            if (lane < bs) zs[j0 + lane] = acc;
        }
        __syncthreads();
        const double zl = lane < bs ? zs[j0 + lane] : 0.0;
        for (int i = w; i < j0; i += nw) {
            double t = lane < bs ? Lcm[(long long)i * n + j0 + lane] * zl : 0.0;
            t = warp_sum(t);
            if (lane == 0) zs[i] -= t;
        }
        __syncthreads();
    }
    double acc = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        z[i] = zs[i];
        if (dotw) acc = fma(zs[i], dotw[i], acc);
    }
    if (red.fin != FIN_NONE) reduce_finish(acc, red);
}

int g_num_sms = 0;
int num_sms() {
    if (g_num_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    return g_num_sms;
}

template <class K>
int occ_grid(K kern, long long work_units_per_cta_needed) {
    static int cache[64];
    (void)cache;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBlock, 0);
    if (per_sm <= 0) per_sm = 1;
    long long g = (long long)num_sms() * per_sm;
    if (work_units_per_cta_needed < g) g = work_units_per_cta_needed;
    return (int)(g < 1 ? 1 : g);
}

}  // namespace

// ------------------------------------------------------------------ host API
int spmv_grid(const DMat& M) {
    if (M.fmt == 1) {
        const long long warps = M.bsr.nb;
        return M.bsr.stream ? occ_grid(k_bsr3<true>, (warps + 7) / 8) : occ_grid(k_bsr3<false>, (warps + 7) / 8);
    }
    const int G = M.csr.group;
    const long long warps = ((long long)M.csr.n_rows * G + 31) / 32;
    return occ_grid(k_csr<32, false>, (warps + 7) / 8);
}

void spmv(const DMat& M, Epi epi, const double* x, double* y, const double* aux, double omega, const double* dotw,
          const Red& red, const int* done, const Launch& L) {
    const int grid = L.grid > 0 ? L.grid : spmv_grid(M);
    if (M.fmt == 1) {
        if (M.bsr.stream)
            k_bsr3<true><<<grid, kBlock, 0, L.stream>>>(M.bsr, epi, x, y, aux, omega, dotw, red, done);
        else
            k_bsr3<false><<<grid, kBlock, 0, L.stream>>>(M.bsr, epi, x, y, aux, omega, dotw, red, done);
        return;
    }
#define ASPAMG_CSR_CASE(GG)                                                                                   \
    case GG:                                                                                                  \
        if (M.csr.stream)                                                                                     \
            k_csr<GG, true><<<grid, kBlock, 0, L.stream>>>(M.csr, epi, x, y, aux, omega, dotw, red, done);   \
        else                                                                                                  \
            k_csr<GG, false><<<grid, kBlock, 0, L.stream>>>(M.csr, epi, x, y, aux, omega, dotw, red, done);  \
        break;
    switch (M.csr.group) {
        ASPAMG_CSR_CASE(1)
        ASPAMG_CSR_CASE(2)
        ASPAMG_CSR_CASE(4)
        ASPAMG_CSR_CASE(8)
        ASPAMG_CSR_CASE(16)
        default:
        ASPAMG_CSR_CASE(32)
    }
#undef ASPAMG_CSR_CASE
}

int vec_grid(int n) {
    const long long need = ((long long)n + kBlock - 1) / kBlock;
    return occ_grid(k_pcg_xr, need);
}

void pcg_p(int n, const double* z, double* p, const PcgState* st, const int* done, const Launch& L) {
    k_pcg_p<<<L.grid > 0 ? L.grid : vec_grid(n), kBlock, 0, L.stream>>>(n, z, p, st, done);
}

void pcg_xr(int n, double* x, double* r, const double* p, const double* q, const Red& red, const int* done,
            const Launch& L) {
    k_pcg_xr<<<L.grid > 0 ? L.grid : vec_grid(n), kBlock, 0, L.stream>>>(n, x, r, p, q, red, done);
}

void pcg_init_dots(int n, const double* b, const double* r, const Red& red, const Launch& L) {
    k_pcg_init<<<L.grid > 0 ? L.grid : vec_grid(n), kBlock, 0, L.stream>>>(n, b, r, red);
}

void coarse_solve(int n, const double* Lrm, const double* Lcm, const double* Dinv_f, const double* Dinv_b,
                  const double* y, double* z, const double* dotw, const Red& red, const int* done,
                  const Launch& L) {
    const size_t smem = sizeof(double) * (size_t)(n > 0 ? n : 1);
    k_coarse<<<1, kCoarseThreads, smem, L.stream>>>(n, Lrm, Lcm, Dinv_f, Dinv_b, y, z, dotw, red, done);
}

void coarse_prepare(int n) {
    const size_t smem = sizeof(double) * (size_t)(n > 0 ? n : 1);
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_coarse, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

void fill_zero(int n, double* y, const int* done, const Launch& L) {
    k_zero<<<L.grid > 0 ? L.grid : vec_grid(n), kBlock, 0, L.stream>>>(n, y, done);
}

}  // namespace aspamg_gpu
