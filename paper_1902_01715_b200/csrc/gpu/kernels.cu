// sm_100a kernels of the solve path (PCG + V(nu1,nu2)-cycle), fp64.
//
// Replaces, per SURVEY.md §2 kernel table:
//   k_sbsr3  <- spmv sparse_matrix.cpp:96-107 on K (exact 3x3 blocks, sliced, lane per block row)
//   k_sell   <- spmv on short-row operands (SELL-32, lane per row)
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

// Epilogues are written with explicit _rn intrinsics (no FMA contraction) so
// they round exactly like the oracle's separate multiply / add.
__device__ __forceinline__ double epilogue(int epi, double s, const double* aux, int row, double omega) {
    switch (epi) {
        case EPI_SCALE: return __dmul_rn(omega, s);
        case EPI_RESID: return __dsub_rn(aux[row], s);
        case EPI_ADD: return __dadd_rn(aux[row], s);
        case EPI_ADDSCALE: return __dadd_rn(aux[row], __dmul_rn(omega, s));
        default: return s;
    }
}

// Matrix-stream load with an L2 policy: POL 0 default, 1 evict-first
// (operators much larger than L2 stream through it), 2 evict-last (the small
// coarse levels stay L2-resident across V-cycles).
__device__ __forceinline__ unsigned long long l2_keep_policy() {
    unsigned long long pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ double ld_keep(const double* p) {
    double r;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(l2_keep_policy()));
    return r;
}
__device__ __forceinline__ int ld_keep(const int* p) {
    int r;
    asm("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(l2_keep_policy()));
    return r;
}
__device__ __forceinline__ unsigned short ld_keep(const unsigned short* p) {
    unsigned short r;
    asm("ld.global.nc.L2::cache_hint.u16 %0, [%1], %2;" : "=h"(r) : "l"(p), "l"(l2_keep_policy()));
    return r;
}
__device__ __forceinline__ double2 ld_keep(const double2* p) {
    double2 r;
    asm("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(r.x), "=d"(r.y) : "l"(p), "l"(l2_keep_policy()));
    return r;
}
__device__ __forceinline__ uint2 ld_keep(const uint2* p) {
    uint2 r;
    asm("ld.global.nc.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;" : "=r"(r.x), "=r"(r.y) : "l"(p), "l"(l2_keep_policy()));
    return r;
}
// POL 3: stream past L1 (no_allocate) with an L2 evict-first hint — the matrix stream of the
// warp-per-row kernels then leaves L1 to the x gathers.
__device__ __forceinline__ unsigned long long l2_first_policy() {
    unsigned long long pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ double ld_na(const double* p) {
    double r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(l2_first_policy()));
    return r;
}
__device__ __forceinline__ int ld_na(const int* p) {
    int r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(l2_first_policy()));
    return r;
}
__device__ __forceinline__ double ld_na(const double* p, unsigned long long pol) {
    double r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ int ld_na(const int* p, unsigned long long pol) {
    int r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ double ld_hint(const double* p, unsigned long long pol) {
    double r;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ int ld_hint(const int* p, unsigned long long pol) {
    int r;
    asm("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
    return r;
}
template <int POL, class T>
__device__ __forceinline__ T ld_mat(const T* p) {
    if constexpr (POL == 3) return ld_na(p);
    else if constexpr (POL == 1) return __ldcs(p);
    else if constexpr (POL == 2) return ld_keep(p);
    else return __ldg(p);
}

__device__ __forceinline__ bool is_done(const int* done) {
    return done != nullptr && *reinterpret_cast<const volatile int*>(done) != 0;
}

// Programmatic dependent launch (sm_90+): every kernel first waits for its
// predecessor grid's completion + memory flush (no-op when launched without the
// PDL attribute), then immediately allows its own successor to start launching,
// so launch latency overlaps the previous kernel's tail instead of adding to it.
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---------------------------------------------------------------- CSR SpMV
// T threads per row (power of two, 1..256); a CTA owns 256/T consecutive rows
// per step (CTA-uniform loop, so barriers are legal). Each thread walks its
// strided entries in groups of CSR_U predicated loads issued before use, then
// a fixed shuffle tree (and, for T > 32, a fixed smem combine of the warp sums).
constexpr int CSR_U = 4;

// PF: the row pointers (and 16-bit base) of the thread's NEXT row are loaded
// one step ahead, so a step costs two dependent memory round trips (values,
// then x) instead of three.
template <int T, int STREAM, bool I16, int CSR_U = 4, bool PF = false>
__global__ void __launch_bounds__(kBlock) k_csr(DCsr M, int epi, const double* __restrict__ x, double* y,
                                                 const double* aux, double omega, const double* dotw, Red red,
                                                 const int* done) {
    pdl_enter();
    if (is_done(done)) return;
    constexpr int RPC = kBlock / T;  // rows per CTA step
    __shared__ double wsum[kBlock / 32];
    const int t = threadIdx.x % T;
    const int lr = threadIdx.x / T;
    const int lane = threadIdx.x & 31;
    double dacc = 0.0;
    if ((int)blockIdx.x < M.nlctas) {
        // Long-row CTAs: one warp per row of the long-row list (rows longer than
        // lthr), 32 lanes x CSR_U loads per round, fixed shuffle tree.
        const int nw = M.nlctas * (kBlock / 32);
        for (int q = blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5); q < M.nlong; q += nw) {
            const int row = __ldg(M.lrows + q);
            const int b = __ldg(M.rp + row), e = __ldg(M.rp + row + 1);
            const double* xr = I16 ? x + __ldg(M.cb + row) : x;
            double s = 0.0;
            for (int k0 = b + lane; k0 < e; k0 += 32 * CSR_U) {
                double v[CSR_U], xv[CSR_U];
                int c[CSR_U];
#pragma unroll
                for (int u = 0; u < CSR_U; ++u) {
                    const int k = k0 + u * 32;
                    v[u] = 0.0;
                    c[u] = 0;
                    if (k < e) {
                        v[u] = ld_mat<STREAM>(M.v + k);
                        if constexpr (I16) c[u] = ld_mat<STREAM>(M.ci16 + k);
                        else c[u] = ld_mat<STREAM>(M.ci + k);
                    }
                }
#pragma unroll
                for (int u = 0; u < CSR_U; ++u) xv[u] = (k0 + u * 32 < e) ? __ldg(xr + c[u]) : 0.0;
#pragma unroll
                for (int u = 0; u < CSR_U; ++u) s = fma(v[u], xv[u], s);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
            if (lane == 0) {
                const double out = epilogue(epi, s, aux, row, omega);
                y[row] = out;
                if (dotw) dacc = fma(out, dotw[row], dacc);
            }
        }
        if (red.fin != FIN_NONE) reduce_finish(dacc, red);
        return;
    }
    const int bid = (int)blockIdx.x - M.nlctas;
    const int stride = ((int)gridDim.x - M.nlctas) * RPC;
    int pb = 0, pe = 0, pc = 0;
    if constexpr (PF) {
        const int row = bid * RPC + lr;
        if (row < M.n_rows) {
            pb = __ldg(M.rp + row);
            pe = __ldg(M.rp + row + 1);
            if constexpr (I16) pc = __ldg(M.cb + row);
        }
    }
    for (int rbase = bid * RPC; rbase < M.n_rows; rbase += stride) {
        const int row = rbase + lr;
        double s = 0.0;
        int b = 0, e = 0, cbase = 0;
        if constexpr (PF) {
            b = pb;
            e = pe;
            cbase = pc;
            const int nrow = row + stride;
            if (nrow < M.n_rows) {
                pb = __ldg(M.rp + nrow);
                pe = __ldg(M.rp + nrow + 1);
                if constexpr (I16) pc = __ldg(M.cb + nrow);
            }
        } else if (row < M.n_rows) {
            b = __ldg(M.rp + row);
            e = __ldg(M.rp + row + 1);
            cbase = I16 ? __ldg(M.cb + row) : 0;
        }
        // rows on the long-row list are computed (and written) by the long-row CTAs
        const bool own = row < M.n_rows && (M.nlong == 0 || e - b <= M.lthr);
        if (own) {
            const double* xr = I16 ? x + cbase : x;
            for (int k0 = b + t; k0 < e; k0 += T * CSR_U) {
                double v[CSR_U], xv[CSR_U];
                int c[CSR_U];
#pragma unroll
                for (int u = 0; u < CSR_U; ++u) {
                    const int k = k0 + u * T;
                    v[u] = 0.0;
                    c[u] = 0;
                    if (k < e) {
                        v[u] = ld_mat<STREAM>(M.v + k);
                        if constexpr (I16) c[u] = ld_mat<STREAM>(M.ci16 + k);
                        else c[u] = ld_mat<STREAM>(M.ci + k);
                    }
                }
#pragma unroll
                for (int u = 0; u < CSR_U; ++u) xv[u] = (k0 + u * T < e) ? __ldg(xr + c[u]) : 0.0;
#pragma unroll
                for (int u = 0; u < CSR_U; ++u) s = fma(v[u], xv[u], s);
            }
        }
        if constexpr (T <= 32) {
#pragma unroll
            for (int o = T / 2; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o, T);
        } else {
            s = warp_sum(s);
            if (lane == 0) wsum[threadIdx.x >> 5] = s;
            __syncthreads();
            if (t == 0) {
                double a = 0.0;
#pragma unroll
                for (int w = 0; w < T / 32; ++w) a += wsum[(threadIdx.x >> 5) + w];
                s = a;
            }
            __syncthreads();
        }
        if (t == 0 && own) {
            const double out = epilogue(epi, s, aux, row, omega);
            y[row] = out;
            if (dotw) dacc = fma(out, dotw[row], dacc);
        }
    }
    if (red.fin != FIN_NONE) reduce_finish(dacc, red);
}

// ------------------------------------------------- CSR SpMV, warp per row, pipelined
// Long-row operands (Galerkin A_l, dense smoother factors: 100..2000 entries per row)
// with one warp per row. k_csr<32> spends, per row, one memory round trip on the row
// pointers and TWO per round of 32*U entries (values + columns, then the x gathers that
// need the columns): at 64 resident warps the dependent chain, not HBM, bounds it (C5
// level 1: 262 entries per row, 0.75-0.79 of the copy peak). Here the column indices
// run one round ahead — across row boundaries, the next row's first round is fetched
// during the current row's last one — and the row pointers two rows ahead, so every
// round issues its value loads and x gathers together: one round trip per round.
// Per-lane entry order, fma chain and shuffle tree are those of k_csr<32>: identical bits.
template <int STREAM, int U>
__global__ void __launch_bounds__(kBlock) k_csrw(DCsr M, int epi, const double* __restrict__ x, double* y,
                                                  const double* aux, double omega, const double* dotw, Red red,
                                                  const int* done) {
    pdl_enter();
    if (is_done(done)) return;
    // one L2 policy per thread, not per load
    const unsigned long long hint = STREAM == 3 ? l2_first_policy() : STREAM == 2 ? l2_keep_policy() : 0ull;
    auto ldm = [&](auto* p) {
        if constexpr (STREAM == 3) return ld_na(p, hint);
        else if constexpr (STREAM == 2) return ld_hint(p, hint);
        else return ld_mat<STREAM>(p);
    };
    const int lane = threadIdx.x & 31;
    // Row assignment. Interleaved (blk = 0): warp w takes rows w, w + nwarps, ... Blocked (blk = 1):
    // CTA b owns the contiguous rows [b * rpc, (b + 1) * rpc) and its 8 warps walk them together,
    // 8 adjacent rows per step — the x lines one step gathers are reused by the next steps of the
    // same CTA out of L1 (neighbouring rows share most of their columns).
    int row, n_end, nwarps;
    if (M.blk) {
        constexpr int wpc = kBlock / 32;
        const int rpc = (((M.n_rows + (int)gridDim.x - 1) / (int)gridDim.x + wpc - 1) / wpc) * wpc;
        row = min((long long)blockIdx.x * rpc, (long long)M.n_rows) + (threadIdx.x >> 5);
        n_end = (int)min((long long)(blockIdx.x + 1) * rpc, (long long)M.n_rows);
        nwarps = wpc;
    } else {
        row = (blockIdx.x * kBlock + threadIdx.x) >> 5;
        n_end = M.n_rows;
        nwarps = (gridDim.x * kBlock) >> 5;
    }
    double dacc = 0.0;
    int b = 0, e = 0, nb = 0, ne = 0;
    int cn[U];
#pragma unroll
    for (int u = 0; u < U; ++u) cn[u] = 0;
    if (row < n_end) {
        b = __ldg(M.rp + row);
        e = __ldg(M.rp + row + 1);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int k = b + lane + 32 * u;
            cn[u] = k < e ? ldm(M.ci + k) : 0;
        }
        if (row + nwarps < n_end) {
            nb = __ldg(M.rp + row + nwarps);
            ne = __ldg(M.rp + row + nwarps + 1);
        }
    }
    while (row < n_end) {
        const int nrow = row + nwarps;
        int fb = 0, fe = 0;  // pointers of the row after next
        if (nrow + nwarps < n_end) {
            fb = __ldg(M.rp + nrow + nwarps);
            fe = __ldg(M.rp + nrow + nwarps + 1);
        }
        double s = 0.0;
        int k0 = b + lane;
        do {  // at least one pass: an empty row still fetches the next row's first columns
            double v[U], xv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int k = k0 + 32 * u;
                const bool p = k < e;
                v[u] = p ? ldm(M.v + k) : 0.0;
                xv[u] = p ? __ldg(x + cn[u]) : 0.0;
            }
            const int kn = k0 + 32 * U;
            if (kn - lane < e) {  // warp-uniform: another round of this row
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int k = kn + 32 * u;
                    cn[u] = k < e ? ldm(M.ci + k) : 0;
                }
            } else if (nrow < n_end) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int k = nb + lane + 32 * u;
                    cn[u] = k < ne ? ldm(M.ci + k) : 0;
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) s = fma(v[u], xv[u], s);
            k0 = kn;
        } while (k0 - lane < e);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
        if (lane == 0) {
            const double out = epilogue(epi, s, aux, row, omega);
            y[row] = out;
            if (dotw) dacc = fma(out, dotw[row], dacc);
        }
        row = nrow;
        b = nb;
        e = ne;
        nb = fb;
        ne = fe;
    }
    if (red.fin != FIN_NONE) reduce_finish(dacc, red);
}

constexpr int SB_U = 3;    // block slots per load group (sliced BSR3)

// ------------------------------------------------------- sliced BSR3 SpMV
// One lane per block row (3 rows of K), 32 block rows per warp-chunk. Per
// block slot the warp issues one 128-B column load and nine 256-B value loads
// (all fully coalesced), then gathers x[3c..3c+2] (L1/L2-resident). The three
// row sums run sequentially in ascending column order with separate multiply
// and add — exactly the reference spmv's arithmetic (sparse_matrix.cpp:100-105),
// so y is bit-identical to it.
// The chunk loop of the sliced BSR3 product for warp `warp` of `nwarps`; the dot
// contribution of the rows it writes is added to dacc.
template <int STREAM>
__device__ __forceinline__ void sbsr3_rows(const DSbsr3& M, int epi, const double* __restrict__ x, double* y,
                                           const double* aux, double omega, const double* dotw, int warp,
                                           int nwarps, double& dacc) {
    const int lane = threadIdx.x & 31;
    for (int ch = warp; ch < M.nchunks; ch += nwarps) {
        const int br = ch * 32 + lane;
        const bool act = br < M.nb;
        const int len = act ? __ldg(M.len + br) : 0;
        const int2 mw = __ldg(M.meta + ch);
        const int* cp = M.ci + (long long)mw.x * 32 + lane;
        const double* vp = M.v + (long long)mw.x * 288 + lane;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
        // Groups of SB_U slots: every load of the group is issued (predicated,
        // never for padding) before the first use, so each lane keeps
        // 10*SB_U independent DRAM loads and then 3*SB_U gathers in flight.
        for (int j0 = 0; j0 < mw.y; j0 += SB_U) {
            int c[SB_U];
            double v[SB_U][9];
            double xv[SB_U][3];
#pragma unroll
            for (int u = 0; u < SB_U; ++u) {
                const int j = j0 + u;
                c[u] = 0;
#pragma unroll
                for (int e = 0; e < 9; ++e) v[u][e] = 0.0;
                if (j < len) {
                    c[u] = ld_mat<STREAM>(cp + 32 * j);
                    const double* vj = vp + 288ll * j;
#pragma unroll
                    for (int e = 0; e < 9; ++e) v[u][e] = ld_mat<STREAM>(vj + 32 * e);
                }
            }
#pragma unroll
            for (int u = 0; u < SB_U; ++u) {
                xv[u][0] = xv[u][1] = xv[u][2] = 0.0;
                if (j0 + u < len) {
                    xv[u][0] = __ldg(x + 3 * c[u]);
                    xv[u][1] = __ldg(x + 3 * c[u] + 1);
                    xv[u][2] = __ldg(x + 3 * c[u] + 2);
                }
            }
#pragma unroll
            for (int u = 0; u < SB_U; ++u) {
                if (j0 + u < len) {
                    a0 = __dadd_rn(a0, __dmul_rn(v[u][0], xv[u][0]));
                    a0 = __dadd_rn(a0, __dmul_rn(v[u][1], xv[u][1]));
                    a0 = __dadd_rn(a0, __dmul_rn(v[u][2], xv[u][2]));
                    a1 = __dadd_rn(a1, __dmul_rn(v[u][3], xv[u][0]));
                    a1 = __dadd_rn(a1, __dmul_rn(v[u][4], xv[u][1]));
                    a1 = __dadd_rn(a1, __dmul_rn(v[u][5], xv[u][2]));
                    a2 = __dadd_rn(a2, __dmul_rn(v[u][6], xv[u][0]));
                    a2 = __dadd_rn(a2, __dmul_rn(v[u][7], xv[u][1]));
                    a2 = __dadd_rn(a2, __dmul_rn(v[u][8], xv[u][2]));
                }
            }
        }
        if (act) {
            const int r0 = 3 * br;
            const double o0 = epilogue(epi, a0, aux, r0, omega);
            const double o1 = epilogue(epi, a1, aux, r0 + 1, omega);
            const double o2 = epilogue(epi, a2, aux, r0 + 2, omega);
            y[r0] = o0;
            y[r0 + 1] = o1;
            y[r0 + 2] = o2;
            if (dotw) {
                dacc = fma(o0, dotw[r0], dacc);
                dacc = fma(o1, dotw[r0 + 1], dacc);
                dacc = fma(o2, dotw[r0 + 2], dacc);
            }
        }
    }
}

template <int STREAM>
__global__ void __launch_bounds__(kBlock) k_sbsr3(DSbsr3 M, int epi, const double* __restrict__ x, double* y,
                                                   const double* aux, double omega, const double* dotw, Red red,
                                                   const int* done) {
    pdl_enter();
    if (is_done(done)) return;
    double dacc = 0.0;
    sbsr3_rows<STREAM>(M, epi, x, y, aux, omega, dotw, (blockIdx.x * kBlock + threadIdx.x) >> 5,
                       (gridDim.x * kBlock) >> 5, dacc);
    if (red.fin != FIN_NONE) reduce_finish(dacc, red);
}

// ----------------------------------------------------------- SELL-32 SpMV
// One lane per row; slot-major layout (coalesced); sequential ascending-column
// sum with separate multiply/add (bit-identical to the reference spmv).
// Software pipeline: column indices are fetched one load group ahead (and the
// next chunk's metadata + first column group during the current chunk), so
// each group costs ONE memory round trip — values and x gathers are issued
// together because the x addresses are already known.
struct SellChunk {
    int len, row, w, cb;
    long long base;
    double av, dw;
    bool act;
};

template <int STREAM>
__device__ __forceinline__ SellChunk sell_chunk(const DSell& M, int ch, int lane, bool need_aux, const double* aux,
                                                const double* dotw) {
    // ch = group of 32 slot rows (one warp); the layout's chunk height chh (8 or
    // 32) splits the group into 32/chh chunks, each with its own width/offset.
    SellChunk c;
    const int srow = ch * 32 + lane;
    c.act = srow < M.n_rows;
    c.len = c.act ? __ldg(M.len + srow) : 0;
    c.row = c.act ? (M.perm ? __ldg(M.perm + srow) : srow) : 0;
    const int sub = min(srow, M.n_rows - 1) / M.chh;
    const int2 mw = __ldg(M.meta + sub);
    c.w = M.chh == 32 ? mw.y : (int)__reduce_max_sync(0xffffffffu, (unsigned)mw.y);
    c.base = (long long)mw.x * M.chh + (srow % M.chh);
    c.cb = (c.act && M.ci16) ? __ldg(M.cb + srow) : 0;
    c.av = (c.act && need_aux) ? aux[c.row] : 0.0;
    c.dw = (c.act && dotw) ? dotw[c.row] : 0.0;
    return c;
}

template <bool I16>
struct SellCol {
    using T = int;
    __device__ static const T* base(const DSell& M) { return M.ci; }
};
template <>
struct SellCol<true> {
    using T = unsigned short;
    __device__ static const T* base(const DSell& M) { return M.ci16; }
};

// CHH: the layout's chunk height when known at compile time (32), 0 = runtime
// (M.chh): with a constant slot stride every load of a group addresses off one
// running pointer with an immediate offset.
template <int U, int STREAM, int MINB, bool I16, int CHH>
__global__ void __launch_bounds__(kBlock, MINB) k_sell(DSell M, int epi, const double* __restrict__ x, double* y,
                                                  const double* aux, double omega, const double* dotw, Red red,
                                                  const int* done) {
    pdl_enter();
    if (is_done(done)) return;
    using CT = typename SellCol<I16>::T;
    const CT* __restrict__ colb = SellCol<I16>::base(M);
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * kBlock) >> 5;
    const bool need_aux = epi == EPI_RESID || epi == EPI_ADD || epi == EPI_ADDSCALE;
    const int SS = CHH ? CHH : M.chh;  // slot stride
    double dacc = 0.0;
    int ch = warp;
    SellChunk nx{};
    int cn[U];
#pragma unroll
    for (int u = 0; u < U; ++u) cn[u] = 0;
    if (ch < M.nchunks) {
        nx = sell_chunk<STREAM>(M, ch, lane, need_aux, aux, dotw);
        const CT* cp = colb + nx.base;
#pragma unroll
        for (int u = 0; u < U; ++u) cn[u] = (u < nx.len) ? (int)ld_mat<STREAM>(cp + SS * u) : 0;
    }
    while (ch < M.nchunks) {
        const SellChunk cu = nx;
        const int chn = ch + nwarps;
        if (chn < M.nchunks) nx = sell_chunk<STREAM>(M, chn, lane, need_aux, aux, dotw);
        const double* vp = M.v + cu.base;  // slot j of this lane at vp[SS * j]
        const CT* cp = colb + cu.base;
        const double* xb = x + cu.cb;
        int rem = cu.len;                  // entries of this row not yet consumed
        double s = 0.0;
        for (int j0 = 0; j0 < cu.w; j0 += U, vp += SS * U, cp += SS * U, rem -= U) {
            int cc[U];
            double v[U], xv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                cc[u] = cn[u];
                const bool p = u < rem;
                v[u] = p ? ld_mat<STREAM>(vp + SS * u) : 0.0;
                xv[u] = p ? __ldg(xb + cc[u]) : 0.0;
            }
            if (j0 + U < cu.w) {
#pragma unroll
                for (int u = 0; u < U; ++u) cn[u] = (U + u < rem) ? (int)ld_mat<STREAM>(cp + SS * (U + u)) : 0;
            } else if (chn < M.nchunks) {
                const CT* np = colb + nx.base;
#pragma unroll
                for (int u = 0; u < U; ++u) cn[u] = (u < nx.len) ? (int)ld_mat<STREAM>(np + SS * u) : 0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (u < rem) s = __dadd_rn(s, __dmul_rn(v[u], xv[u]));
        }
        if (cu.w <= 0 && chn < M.nchunks) {  // all-empty group: the loop above never prefetched the next chunk
            const CT* np = colb + nx.base;
#pragma unroll
            for (int u = 0; u < U; ++u) cn[u] = (u < nx.len) ? (int)ld_mat<STREAM>(np + SS * u) : 0;
        }
        if (cu.act) {
            double out;
            switch (epi) {
                case EPI_SCALE: out = __dmul_rn(omega, s); break;
                case EPI_RESID: out = __dsub_rn(cu.av, s); break;
                case EPI_ADD: out = __dadd_rn(cu.av, s); break;
                case EPI_ADDSCALE: out = __dadd_rn(cu.av, __dmul_rn(omega, s)); break;
                default: out = s;
            }
            y[cu.row] = out;
            if (dotw) dacc = fma(out, cu.dw, dacc);
        }
        ch = chn;
    }
    if (red.fin != FIN_NONE) reduce_finish(dacc, red);
}

// ------------------------------------------------------ tile-local SELL SpMV
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// One CTA per tile, F rows per lane (F = 1: sorted rank t; F = 2, "folded":
// ranks t and R-1-t, a long row paired with a short one so the warps of a
// tile carry nearly equal work). Phases: (1) cp.async the tile's x footprint
// into shared memory; (2) meanwhile fetch the chunk metadata and the first
// load group of the matrix stream (independent of x); (3) row sums over the
// chunk's quads (row a's quads, then row b's), gathers from shared memory, the
// next group's loads issued before the current group is consumed; (4) results
// pass through shared memory back to natural row order, so the epilogue reads
// aux / writes y coalesced.
template <int Q, int STREAM, int MINB, int F>
__global__ void __launch_bounds__(kBlock, MINB) k_xsell(DXsell M, int epi, const double* __restrict__ x, double* y,
                                                       const double* aux, double omega, const double* dotw, Red red,
                                                       const int* done) {
    pdl_enter();
    if (is_done(done)) return;
    extern __shared__ __align__(16) double xsm[];
    const int tid = threadIdx.x, lane = tid & 31, T = blockDim.x, R = F * T;
    const int tile = blockIdx.x;
    double* ys = xsm + M.fp_doubles;
    const int2 tm = __ldg(M.tmeta + tile);
    {
        const int sh = M.gran - 1;  // 16-B pieces per granule = 1 << sh
        const int np = tm.y << sh;
        const int* lst = M.list + tm.x;
        for (int p = tid; p < np; p += T) {
            const int g = __ldg(lst + (p >> sh));
            const int i0 = (g << M.gran) + 2 * (p & ((1 << sh) - 1));
            if (i0 + 2 <= M.n_cols) {
                cp_async16(xsm + 2 * p, x + i0);
            } else {  // the last granule may straddle the end of x
                xsm[2 * p] = i0 < M.n_cols ? x[i0] : 0.0;
                xsm[2 * p + 1] = 0.0;
            }
        }
        cp_async_commit();
    }
    const int r0 = tile * R;
    const int lenA = M.len[r0 + tid];
    const int prA = M.perm[r0 + tid];
    const int lenB = F == 2 ? (int)M.len[r0 + R - 1 - tid] : 0;
    const int prB = F == 2 ? (int)M.perm[r0 + R - 1 - tid] : 0;
    const int2 cm = __ldg(M.cmeta + (tile * (T >> 5) + (tid >> 5)));
    const bool need_aux = epi == EPI_RESID || epi == EPI_ADD || epi == EPI_ADDSCALE;
    double av[F], dw[F];
#pragma unroll
    for (int f = 0; f < F; ++f) {
        const int orow = r0 + f * T + tid;  // this thread's output rows (natural order)
        av[f] = (orow < M.n_rows && need_aux) ? aux[orow] : 0.0;
        dw[f] = (orow < M.n_rows && dotw) ? dotw[orow] : 0.0;
    }
    const double2* vp = M.v + ((long long)cm.x * 64 + lane);
    const uint2* cp = M.lc + ((long long)cm.x * 32 + lane);
    const int qa = ((cm.y & 0xffff) + 3) >> 2;           // quads of the a rows (warp-uniform)
    const int nq = qa + ((((unsigned)cm.y >> 16) + 3) >> 2);  // + quads of the b rows
    auto rem_of = [&](int qi) { return qi < qa ? lenA - 4 * qi : lenB - 4 * (qi - qa); };
    uint2 c[Q];
    double2 v[Q][2];
#pragma unroll
    for (int u = 0; u < Q; ++u) {
        const int rem = u < nq ? rem_of(u) : 0;
        c[u] = rem > 0 ? ld_mat<STREAM>(cp + 32 * u) : make_uint2(0u, 0u);
        v[u][0] = rem > 0 ? ld_mat<STREAM>(vp + 64 * u) : make_double2(0.0, 0.0);
        v[u][1] = rem > 2 ? ld_mat<STREAM>(vp + 64 * u + 32) : make_double2(0.0, 0.0);
    }
    cp_async_wait_all();
    __syncthreads();
    double s = 0.0, sa = 0.0;
    for (int q0 = 0; q0 < nq; q0 += Q) {
        uint2 cc[Q];
        double2 vv[Q][2];
#pragma unroll
        for (int u = 0; u < Q; ++u) {
            cc[u] = c[u];
            vv[u][0] = v[u][0];
            vv[u][1] = v[u][1];
        }
        if (q0 + Q < nq) {
#pragma unroll
            for (int u = 0; u < Q; ++u) {
                const int qq = q0 + Q + u;
                const int rem = qq < nq ? rem_of(qq) : 0;
                c[u] = rem > 0 ? ld_mat<STREAM>(cp + 32 * qq) : make_uint2(0u, 0u);
                v[u][0] = rem > 0 ? ld_mat<STREAM>(vp + 64 * qq) : make_double2(0.0, 0.0);
                v[u][1] = rem > 2 ? ld_mat<STREAM>(vp + 64 * qq + 32) : make_double2(0.0, 0.0);
            }
        }
        double xv[Q][4];
#pragma unroll
        for (int u = 0; u < Q; ++u) {
            xv[u][0] = xsm[cc[u].x & 0xffffu];
            xv[u][1] = xsm[cc[u].x >> 16];
            xv[u][2] = xsm[cc[u].y & 0xffffu];
            xv[u][3] = xsm[cc[u].y >> 16];
        }
#pragma unroll
        for (int u = 0; u < Q; ++u) {
            const int qi = q0 + u;
            // row a finished, row b starts (warp-uniform). Only when b quads exist: a group's
            // trailing slot qi == nq == qa must not clear the finished sum (handled after the loop).
            if (F == 2 && qi == qa && qa < nq) {
                sa = s;
                s = 0.0;
            }
            const int rem = qi < nq ? rem_of(qi) : 0;
            if (rem > 0) s = __dadd_rn(s, __dmul_rn(vv[u][0].x, xv[u][0]));
            if (rem > 1) s = __dadd_rn(s, __dmul_rn(vv[u][0].y, xv[u][1]));
            if (rem > 2) s = __dadd_rn(s, __dmul_rn(vv[u][1].x, xv[u][2]));
            if (rem > 3) s = __dadd_rn(s, __dmul_rn(vv[u][1].y, xv[u][3]));
        }
    }
    if (F == 2) {
        if (nq == qa) {  // no b quads: s still holds row a
            sa = s;
            s = 0.0;
        }
        ys[prA] = sa;
        ys[prB] = s;
    } else {
        ys[prA] = s;
    }
    __syncthreads();
    double dacc = 0.0;
#pragma unroll
    for (int f = 0; f < F; ++f) {
        const int orow = r0 + f * T + tid;
        if (orow < M.n_rows) {
            const double r = ys[f * T + tid];
            double out;
            switch (epi) {
                case EPI_SCALE: out = __dmul_rn(omega, r); break;
                case EPI_RESID: out = __dsub_rn(av[f], r); break;
                case EPI_ADD: out = __dadd_rn(av[f], r); break;
                case EPI_ADDSCALE: out = __dadd_rn(av[f], __dmul_rn(omega, r)); break;
                default: out = r;
            }
            y[orow] = out;
            dacc = fma(out, dw[f], dacc);
        }
    }
    if (red.fin != FIN_NONE) reduce_finish(dacc, red);
}

// ------------------------------------------------------------- coarse tail
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Sense-reversing software grid barrier (all CTAs co-resident: cooperative
// launch sized to the occupancy). Thread 0's gpu-scope fences order the CTA's
// writes before the arrival and invalidate L1 after the release.
__device__ __forceinline__ void grid_barrier(GridBar* b) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = ld_acquire_u32(&b->gen);
        __threadfence();
        if (atomicAdd(&b->count, 1u) == gridDim.x - 1) {
            atomicExch(&b->count, 0u);
            __threadfence();
            atomicAdd(&b->gen, 1u);
        } else {
            while (ld_acquire_u32(&b->gen) == g) __nanosleep(20);
        }
        __threadfence();
    }
    __syncthreads();
}

// One CSR product op inside the persistent kernel: runtime T (power of two,
// 1..256) threads per row, same per-thread order and trees as k_csr. Vector
// operands written earlier in the same kernel are read through L2 (__ldcg).
__device__ void tail_csr(const TailOp& op, double* wsum) {
    const DCsr& M = op.M;
    const int T = M.group;
    const int RPC = kBlock / T;
    const int t = threadIdx.x & (T - 1);
    const int lr = threadIdx.x / T;
    const int lane = threadIdx.x & 31;
    for (int rbase = blockIdx.x * RPC; rbase < M.n_rows; rbase += gridDim.x * RPC) {
        const int row = rbase + lr;
        double s = 0.0;
        if (row < M.n_rows) {
            const int b = __ldg(M.rp + row), e = __ldg(M.rp + row + 1);
            for (int k0 = b + t; k0 < e; k0 += T * CSR_U) {
                double v[CSR_U], xv[CSR_U];
                int c[CSR_U];
#pragma unroll
                for (int u = 0; u < CSR_U; ++u) {
                    const int kk = k0 + u * T;
                    v[u] = kk < e ? __ldg(M.v + kk) : 0.0;
                    c[u] = kk < e ? (M.ci16 ? __ldg(M.cb + row) + (int)__ldg(M.ci16 + kk) : __ldg(M.ci + kk)) : 0;
                }
#pragma unroll
                for (int u = 0; u < CSR_U; ++u) xv[u] = (k0 + u * T < e) ? __ldcg(op.x + c[u]) : 0.0;
#pragma unroll
                for (int u = 0; u < CSR_U; ++u) s = fma(v[u], xv[u], s);
            }
        }
        if (T <= 32) {
            for (int o = T / 2; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o, T);
        } else {
            s = warp_sum(s);
            if (lane == 0) wsum[threadIdx.x >> 5] = s;
            __syncthreads();
            if (t == 0) {
                double a = 0.0;
                for (int w = 0; w < T / 32; ++w) a += wsum[(threadIdx.x >> 5) + w];
                s = a;
            }
            __syncthreads();
        }
        if (t == 0 && row < M.n_rows) {
            double out;
            switch (op.epi) {
                case EPI_SCALE: out = __dmul_rn(op.omega, s); break;
                case EPI_RESID: out = __dsub_rn(__ldcg(op.aux + row), s); break;
                case EPI_ADD: out = __dadd_rn(__ldcg(op.aux + row), s); break;
                case EPI_ADDSCALE: out = __dadd_rn(__ldcg(op.aux + row), __dmul_rn(op.omega, s)); break;
                default: out = s;
            }
            op.y[row] = out;
        }
    }
}

__global__ void __launch_bounds__(kBlock) k_tail(const TailOp* __restrict__ ops, int nops, GridBar* bar,
                                                  const int* done) {
    pdl_enter();
    if (is_done(done)) return;
    __shared__ double wsum[kBlock / 32];
    for (int i = 0; i < nops; ++i) {
        const TailOp op = ops[i];
        if (op.kind == 0) {
            tail_csr(op, wsum);
        } else {
            for (int r = blockIdx.x * kBlock + threadIdx.x; r < op.n; r += gridDim.x * kBlock) op.y[r] = 0.0;
        }
        if (i + 1 < nops) grid_barrier(bar);
    }
}

// Restriction fused with the fine residual (Alg. 2):
// ONE cooperative launch computes r = y - A s with the sliced BSR3 chunk loop, crosses
// a grid barrier, and gathers r_c = P' r (CSR rows, T threads each) while r is still
// L2-resident. Same per-row arithmetic and trees as the two separate kernels, so the
// results are bit-identical to the unfused path; no atomics on the data.
template <int STREAM>
__global__ void __launch_bounds__(kBlock) k_resid_restrict(DSbsr3 A, TailOp pt, const double* __restrict__ s,
                                                            double* r, const double* y, GridBar* bar,
                                                            const int* done) {
    pdl_enter();
    if (is_done(done)) return;
    __shared__ double wsum[kBlock / 32];
    double dacc = 0.0;
    sbsr3_rows<STREAM>(A, EPI_RESID, s, r, y, 1.0, nullptr, (blockIdx.x * kBlock + threadIdx.x) >> 5,
                       (gridDim.x * kBlock) >> 5, dacc);
    grid_barrier(bar);
    tail_csr(pt, wsum);
}

// ------------------------------------------------------------- PCG vectors
__global__ void __launch_bounds__(kBlock) k_pcg_p(int n, const double* __restrict__ z, double* __restrict__ p,
                                                   const PcgState* st, const int* done) {
    pdl_enter();
    if (is_done(done)) return;
    const bool first = st->k == 0;
    const double beta = st->beta;
    for (int i = blockIdx.x * kBlock + threadIdx.x; i < n; i += gridDim.x * kBlock)
        p[i] = first ? z[i] : fma(beta, p[i], z[i]);
}

__global__ void __launch_bounds__(kBlock) k_pcg_xr(int n, double* __restrict__ x, double* __restrict__ r,
                                                    const double* __restrict__ p, const double* __restrict__ q,
                                                    Red red, const int* done) {
    pdl_enter();
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
    pdl_enter();
    double s = 0.0, s2 = 0.0;
    for (int i = blockIdx.x * kBlock + threadIdx.x; i < n; i += gridDim.x * kBlock) {
        s = fma(b[i], b[i], s);
        s2 = fma(r[i], r[i], s2);
    }
    reduce_finish2(s, s2, red);
}

__global__ void __launch_bounds__(kBlock) k_zero(int n, double* y, const int* done) {
    pdl_enter();
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
    pdl_enter();
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
            const double* D = Dinv_f + 1024ll * jb + 32 * lane;
            double acc = 0.0;
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (j <= lane && lane < bs) acc = fma(__ldg(D + j), zs[j0 + j], acc);
            __syncwarp();
            if (lane < bs) zs[j0 + lane] = acc;
        }
        __syncthreads();
        const double zl = lane < bs ? zs[j0 + lane] : 0.0;
#pragma unroll 4
        for (int i = j0 + bs + w; i < n; i += nw) {
            double t = lane < bs ? __ldg(Lrm + (long long)i * n + j0 + lane) * zl : 0.0;
            t = warp_sum(t);
            if (lane == 0) zs[i] -= t;
        }
        __syncthreads();
    }
    // backward: L' z = w
    for (int jb = nb - 1; jb >= 0; --jb) {
        const int j0 = 32 * jb, bs = min(32, n - j0);
        if (w == 0) {
            const double* D = Dinv_b + 1024ll * jb + 32 * lane;
            double acc = 0.0;
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (j >= lane && j < bs && lane < bs) acc = fma(__ldg(D + j), zs[j0 + j], acc);
            __syncwarp();
            if (lane < bs) zs[j0 + lane] = acc;
        }
        __syncthreads();
        const double zl = lane < bs ? zs[j0 + lane] : 0.0;
#pragma unroll 4
        for (int i = w; i < j0; i += nw) {
            double t = lane < bs ? __ldg(Lcm + (long long)i * n + j0 + lane) * zl : 0.0;
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

bool g_pdl = true;

// Launch through cudaLaunchKernelEx so the PDL attribute can be attached; the
// attribute is recorded into CUDA graphs as a programmatic dependency edge.
template <class... KArgs, class... Args>
void launch(void (*kern)(KArgs...), int grid, int block, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = g_pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
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
int occ_grid(K kern, long long work_units_per_cta_needed, size_t smem = 0) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBlock, smem);
    if (per_sm <= 0) per_sm = 1;
    long long g = (long long)num_sms() * per_sm;
    if (work_units_per_cta_needed < g) g = work_units_per_cta_needed;
    return (int)(g < 1 ? 1 : g);
}

}  // namespace

// ------------------------------------------------------------------ host API
// Kernel pointer for an operand's index width (same signature either way).
#define SELLK(UU, P, MB)                                                                            \
    (M.sell.chh == 32 ? (M.sell.ci16 ? k_sell<UU, P, MB, true, 32> : k_sell<UU, P, MB, false, 32>)   \
                      : (M.sell.ci16 ? k_sell<UU, P, MB, true, 0> : k_sell<UU, P, MB, false, 0>))
// CSR kernel variant of an operand: pf = row-pointer prefetch (T <= 16).
using SpmvKern = void (*)(DCsr, int, const double*, double*, const double*, double, const double*, Red, const int*);
template <int GG, int P, bool I16>
SpmvKern csr_kernel_i(const DCsr& A) {
    if constexpr (GG <= 16) {
        if (A.pf) return k_csr<GG, P, I16, 4, true>;
    } else if constexpr (GG <= 64 && !I16) {
        if (A.pf >= 2) return k_csr<GG, P, I16, 4, true>;  // opt-in: prefetch for warp-per-row operands too
    }
    return k_csr<GG, P, I16, 4>;
}
template <int GG, int P>
SpmvKern csr_kernel(const DCsr& A) {
    return A.ci16 ? csr_kernel_i<GG, P, true>(A) : csr_kernel_i<GG, P, false>(A);
}
#define CSRK(GG, P) csr_kernel<GG, P>(M.csr)
// Warp-per-row pipelined variant (DCsr::wu = columns fetched per lane per round, 4 or 8).
SpmvKern csrw_kernel(const DCsr& A) {
    if (A.pol == 3) return A.wu >= 8 ? k_csrw<3, 8> : k_csrw<3, 4>;
    if (A.wu >= 8) return A.pol == 1 ? k_csrw<1, 8> : A.pol == 2 ? k_csrw<2, 8> : k_csrw<0, 8>;
    return A.pol == 1 ? k_csrw<1, 4> : A.pol == 2 ? k_csrw<2, 4> : k_csrw<0, 4>;
}
using XsellKern = void (*)(DXsell, int, const double*, double*, const double*, double, const double*, Red, const int*);
XsellKern xsell_kernel(const DXsell& X) {
#define ASPAMG_XS(QQ, MB)                                                                              \
    if (X.q == QQ * 10 + MB) {                                                                         \
        if (X.fold == 2)                                                                               \
            return X.pol == 1 ? k_xsell<QQ, 1, MB, 2> : X.pol == 2 ? k_xsell<QQ, 2, MB, 2> : k_xsell<QQ, 0, MB, 2>; \
        return X.pol == 1 ? k_xsell<QQ, 1, MB, 1> : X.pol == 2 ? k_xsell<QQ, 2, MB, 1> : k_xsell<QQ, 0, MB, 1>;     \
    }
    ASPAMG_XS(1, 4)
    ASPAMG_XS(1, 6)
    ASPAMG_XS(2, 3)
    ASPAMG_XS(2, 4)
#undef ASPAMG_XS
    if (X.fold == 2) return X.pol == 1 ? k_xsell<2, 1, 4, 2> : X.pol == 2 ? k_xsell<2, 2, 4, 2> : k_xsell<2, 0, 4, 2>;
    return X.pol == 1 ? k_xsell<2, 1, 4, 1> : X.pol == 2 ? k_xsell<2, 2, 4, 1> : k_xsell<2, 0, 4, 1>;
}
size_t xsell_smem(const DXsell& X) { return sizeof(double) * ((size_t)X.fp_doubles + (size_t)X.R); }

int spmv_grid(const DMat& M) {
    if (M.fmt == 3) return M.xs.ntiles;
    if (M.fmt == 1) {
        const long long ch = (M.sb.nchunks + 7) / 8;
        return M.sb.pol == 1 ? occ_grid(k_sbsr3<1>, ch) : M.sb.pol == 2 ? occ_grid(k_sbsr3<2>, ch) : occ_grid(k_sbsr3<0>, ch);
    }
    if (M.fmt == 2) {
        const long long ch = (M.sell.nchunks + 7) / 8;
        const int st = M.sell.pol;
#define ASPAMG_SELL_OCC(UU, MB)                                                                  \
    if (M.sell.u == UU * 10 + MB)                                                                \
        return st == 1 ? occ_grid(SELLK(UU, 1, MB), ch)                                          \
                       : st == 2 ? occ_grid(SELLK(UU, 2, MB), ch) : occ_grid(SELLK(UU, 0, MB), ch);
        ASPAMG_SELL_OCC(8, 3)
        ASPAMG_SELL_OCC(4, 1)
        ASPAMG_SELL_OCC(4, 4)
        ASPAMG_SELL_OCC(2, 1)
#undef ASPAMG_SELL_OCC
        return 1;
    }
    const int T = M.csr.group;
    const long long ctas = ((long long)M.csr.n_rows * T + kBlock - 1) / kBlock;
    const int st = M.csr.pol;
    if (M.csr.wu) {
        const int g = occ_grid(csrw_kernel(M.csr), ctas);
        // blocked rows: 4 waves of CTAs, so uneven row blocks still balance over the SMs
        return M.csr.blk ? (int)(4ll * g < ctas ? 4ll * g : ctas) : g;
    }
    // + the long-row CTAs (M.csr.nlctas, fixed at upload) ahead of the regular grid
#define ASPAMG_CSR_OCC(TT)                                                                                   \
    case TT: return M.csr.nlctas + (st == 1 ? occ_grid(CSRK(TT, 1), ctas)                                    \
                                            : st == 2 ? occ_grid(CSRK(TT, 2), ctas) : occ_grid(CSRK(TT, 0), ctas));
    switch (T) {
        ASPAMG_CSR_OCC(1)
        ASPAMG_CSR_OCC(2)
        ASPAMG_CSR_OCC(4)
        ASPAMG_CSR_OCC(8)
        ASPAMG_CSR_OCC(16)
        ASPAMG_CSR_OCC(32)
        ASPAMG_CSR_OCC(64)
        ASPAMG_CSR_OCC(128)
        default:
        ASPAMG_CSR_OCC(256)
    }
#undef ASPAMG_CSR_OCC
}

void spmv(const DMat& M, Epi epi, const double* x, double* y, const double* aux, double omega, const double* dotw,
          const Red& red, const int* done, const Launch& L) {
    const int grid = L.grid > 0 ? L.grid : spmv_grid(M);
    if (M.fmt == 3) {
        launch(xsell_kernel(M.xs), M.xs.ntiles, M.xs.R / M.xs.fold, xsell_smem(M.xs), L.stream, M.xs, epi, x, y, aux, omega, dotw,
               red, done);
        return;
    }
    if (M.fmt == 1) {
        if (M.sb.pol == 1)
            launch(k_sbsr3<1>, grid, kBlock, 0, L.stream, M.sb, epi, x, y, aux, omega, dotw, red, done);
        else if (M.sb.pol == 2)
            launch(k_sbsr3<2>, grid, kBlock, 0, L.stream, M.sb, epi, x, y, aux, omega, dotw, red, done);
        else
            launch(k_sbsr3<0>, grid, kBlock, 0, L.stream, M.sb, epi, x, y, aux, omega, dotw, red, done);
        return;
    }
    if (M.fmt == 2) {
#define ASPAMG_SELL(UU, MB)                                                                                          \
    if (M.sell.u == UU * 10 + MB) {                                                                                 \
        if (M.sell.pol == 1)                                                                                        \
            launch(SELLK(UU, 1, MB), grid, kBlock, 0, L.stream, M.sell, epi, x, y, aux, omega, dotw, red, done);      \
        else if (M.sell.pol == 2)                                                                                   \
            launch(SELLK(UU, 2, MB), grid, kBlock, 0, L.stream, M.sell, epi, x, y, aux, omega, dotw, red, done);      \
        else                                                                                                        \
            launch(SELLK(UU, 0, MB), grid, kBlock, 0, L.stream, M.sell, epi, x, y, aux, omega, dotw, red, done);      \
        return;                                                                                                     \
    }
        ASPAMG_SELL(8, 3)
        ASPAMG_SELL(4, 1)
        ASPAMG_SELL(4, 4)
        ASPAMG_SELL(2, 1)
#undef ASPAMG_SELL
        return;
    }
    if (M.csr.wu) {
        launch(csrw_kernel(M.csr), grid, kBlock, 0, L.stream, M.csr, epi, x, y, aux, omega, dotw, red, done);
        return;
    }
#define ASPAMG_CSR_CASE(GG)                                                                                   \
    case GG:                                                                                                  \
        if (M.csr.pol == 1)                                                                                   \
            launch(CSRK(GG, 1), grid, kBlock, 0, L.stream, M.csr, epi, x, y, aux, omega, dotw, red, done);       \
        else if (M.csr.pol == 2)                                                                              \
            launch(CSRK(GG, 2), grid, kBlock, 0, L.stream, M.csr, epi, x, y, aux, omega, dotw, red, done);       \
        else                                                                                                  \
            launch(CSRK(GG, 0), grid, kBlock, 0, L.stream, M.csr, epi, x, y, aux, omega, dotw, red, done);       \
        break;
    switch (M.csr.group) {
        ASPAMG_CSR_CASE(1)
        ASPAMG_CSR_CASE(2)
        ASPAMG_CSR_CASE(4)
        ASPAMG_CSR_CASE(8)
        ASPAMG_CSR_CASE(16)
        ASPAMG_CSR_CASE(32)
        ASPAMG_CSR_CASE(64)
        ASPAMG_CSR_CASE(128)
        default:
        ASPAMG_CSR_CASE(256)
    }
#undef ASPAMG_CSR_CASE
}

int vec_grid(int n) {
    const long long need = ((long long)n + kBlock - 1) / kBlock;
    return occ_grid(k_pcg_xr, need);
}

void pcg_p(int n, const double* z, double* p, const PcgState* st, const int* done, const Launch& L) {
    launch(k_pcg_p, L.grid > 0 ? L.grid : vec_grid(n), kBlock, 0, L.stream, n, z, p, st, done);
}

void pcg_xr(int n, double* x, double* r, const double* p, const double* q, const Red& red, const int* done,
            const Launch& L) {
    launch(k_pcg_xr, L.grid > 0 ? L.grid : vec_grid(n), kBlock, 0, L.stream, n, x, r, p, q, red, done);
}

void pcg_init_dots(int n, const double* b, const double* r, const Red& red, const Launch& L) {
    launch(k_pcg_init, L.grid > 0 ? L.grid : vec_grid(n), kBlock, 0, L.stream, n, b, r, red);
}

void coarse_solve(int n, const double* Lrm, const double* Lcm, const double* Dinv_f, const double* Dinv_b,
                  const double* y, double* z, const double* dotw, const Red& red, const int* done,
                  const Launch& L) {
    const size_t smem = sizeof(double) * (size_t)(n > 0 ? n : 1);
    launch(k_coarse, 1, kCoarseThreads, smem, L.stream, n, Lrm, Lcm, Dinv_f, Dinv_b, y, z, dotw, red, done);
}

void set_pdl(bool on) { g_pdl = on; }

int tail_grid() {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tail, kBlock, 0);
    if (per_sm <= 0) per_sm = 1;
    return num_sms() * per_sm;
}

void tail_run(const TailOp* ops, int nops, GridBar* bar, const int* done, int grid, cudaStream_t s) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)kBlock);
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;  // co-residency for the software grid barrier
    attr[0].val.cooperative = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = g_pdl ? 2 : 1;
    cudaLaunchKernelEx(&cfg, k_tail, ops, nops, bar, done);
}

int resid_restrict_grid(int pol) {
    int per_sm = 0;
    if (pol == 1) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_resid_restrict<1>, kBlock, 0);
    else if (pol == 2) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_resid_restrict<2>, kBlock, 0);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_resid_restrict<0>, kBlock, 0);
    if (per_sm <= 0) per_sm = 1;
    return num_sms() * per_sm;
}

void resid_restrict(const DSbsr3& A, const TailOp& pt, const double* s, double* r, const double* y, GridBar* bar,
                    const int* done, int grid, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)kBlock);
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;  // co-residency for the software grid barrier
    attr[0].val.cooperative = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = g_pdl ? 2 : 1;
    if (A.pol == 1) cudaLaunchKernelEx(&cfg, k_resid_restrict<1>, A, pt, s, r, y, bar, done);
    else if (A.pol == 2) cudaLaunchKernelEx(&cfg, k_resid_restrict<2>, A, pt, s, r, y, bar, done);
    else cudaLaunchKernelEx(&cfg, k_resid_restrict<0>, A, pt, s, r, y, bar, done);
}

// Opt in to the operand's dynamic shared memory on every variant that may run it.
void xsell_prepare(const DXsell& X) {
    const int need = (int)xsell_smem(X);
    if (need <= 48 * 1024) return;
    DXsell t = X;
    for (int pol = 0; pol < 3; ++pol)
        for (int q : {14, 16, 23, 24}) {
            t.pol = pol;
            t.q = q;
            cudaFuncSetAttribute(xsell_kernel(t), cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        }
}

void spmv_prepare() {
    static bool done = false;
    if (done) return;
    done = true;
}

void coarse_prepare(int n) {
    const size_t smem = sizeof(double) * (size_t)(n > 0 ? n : 1);
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_coarse, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

void fill_zero(int n, double* y, const int* done, const Launch& L) {
    launch(k_zero, L.grid > 0 ? L.grid : vec_grid(n), kBlock, 0, L.stream, n, y, done);
}

}  // namespace aspamg_gpu
