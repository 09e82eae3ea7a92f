// GPU setup components: the Galerkin triple product
// A_c = P' (A P) (sparse_matrix.cpp:191-199 semantics) on the device.
//
// Restates core.cpp sparse_multiply() — row-wise Gustavson, first-touch
// accumulator acc[j] = 0.0; acc[j] += a * b in ascending (row-of-A, row-of-B)
// order; explicit zeros kept; output columns ascending — with every value sum in
// the same order, so the coarse operator is bit-identical to the host's:
//   * one warp per output row (one CTA for rows whose column set overflows a
//     warp's table); the row's accumulator is an open-addressing table in shared
//     memory keyed by column;
//   * the entries of A's row are consumed one at a time (group-synchronised), the
//     lanes of the group taking distinct columns of the B row — so every
//     accumulator receives its terms in the host order;
//   * the finished table is compacted and bitonic-sorted by column in shared
//     memory and written at the row's offset (count pass + host scan + fill pass).
// Indices stay int64 as in the reference layout (no conversion of the inputs).
#include "setup_common.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdint>
#include <vector>

namespace aspamg_gpu {
namespace {

constexpr int kWarpCap = 1024;   // table entries per warp (12 KB)
constexpr int kWarpsPerCta = 8;  // 96 KB dynamic shared memory per CTA
constexpr int kBigCap = 16384;   // table entries for one CTA (192 KB dynamic)
constexpr int kBigThreads = 512;

__device__ __forceinline__ unsigned hslot(int j, int cap) { return ((unsigned)j * 2654435761u) & (unsigned)(cap - 1); }

// Group-wide helpers: GROUP = 32 (warp) or the CTA.
template <bool WARP>
__device__ __forceinline__ void gsync() {
    if (WARP) __syncwarp();
    else __syncthreads();
}

// One output row i of C = A B by a group of G threads (rank t) over a table
// (keys, vals) of cap entries. Returns the row's column count (or -1 on overflow).
// pass 0: count; pass 1: accumulate, compact, sort, write at out_off.
template <bool WARP>
__device__ long long row_product(const DCsr64 A, const DCsr64 B, long long i, int pass, int* keys, double* vals,
                                 int cap, int t, int G, int* sh_cnt, int* sh_flag, long long out_off,
                                 long long* out_ci, double* out_v) {
    gsync<WARP>();  // the previous row's readers are done with the table and counters
    for (int s = t; s < cap; s += G) keys[s] = -1;
    if (t == 0) { *sh_cnt = 0; *sh_flag = 0; }
    gsync<WARP>();
    const long long a0 = A.rp[i], a1 = A.rp[i + 1];
    for (long long ka = a0; ka < a1; ++ka) {
        const long long tt = A.ci[ka];
        const double a = A.v[ka];
        const long long b0 = B.rp[tt], b1 = B.rp[tt + 1];
        for (long long kb = b0 + t; kb < b1; kb += G) {
            const int j = (int)B.ci[kb];
            unsigned h = hslot(j, cap);
            int probes = 0;
            int slot = -1;
            while (probes < cap) {
                const int k = keys[h];
                if (k == j) { slot = (int)h; break; }
                if (k == -1) {
                    const int old = atomicCAS(&keys[h], -1, j);
                    if (old == -1) {
                        slot = (int)h;
                        atomicAdd(sh_cnt, 1);
                        if (pass == 1) vals[h] = 0.0;  // acc[j] = 0.0 on first touch
                        break;
                    }
                    if (old == j) { slot = (int)h; break; }
                }
                h = (h + 1) & (unsigned)(cap - 1);
                ++probes;
            }
            if (slot < 0) { *sh_flag = 1; continue; }
            if (pass == 1) vals[slot] = __dadd_rn(vals[slot], __dmul_rn(a, B.v[kb]));
        }
        gsync<WARP>();  // next A entry only after every term of this one landed
        if (*sh_flag) break;
    }
    gsync<WARP>();
    const int cnt = *sh_cnt;
    if (*sh_flag) return -1;
    if (pass == 0) return cnt;
    // compact in place (write index <= read index; each block read before written)
    int base = 0;
    for (int s0 = 0; s0 < cap; s0 += G) {
        const int s = s0 + t;
        const int k = s < cap ? keys[s] : -1;
        const double v = s < cap ? vals[s] : 0.0;
        const bool valid = k != -1;
        int pos, tot;
        if constexpr (WARP) {
            const unsigned m = __ballot_sync(0xffffffffu, valid);
            pos = __popc(m & ((1u << t) - 1u));
            tot = __popc(m);
        } else {
            // CTA-wide exclusive prefix via per-warp ballots
            __shared__ int wsum[kBigThreads / 32];
            const unsigned m = __ballot_sync(0xffffffffu, valid);
            const int lane = t & 31, w = t >> 5;
            if (lane == 0) wsum[w] = __popc(m);
            __syncthreads();
            int off = 0;
            tot = 0;
            for (int q = 0; q < G / 32; ++q) {
                if (q < w) off += wsum[q];
                tot += wsum[q];
            }
            pos = off + __popc(m & ((1u << lane) - 1u));
            __syncthreads();
        }
        gsync<WARP>();
        if (valid) {
            keys[base + pos] = k;
            vals[base + pos] = v;
        }
        base += tot;
        gsync<WARP>();
    }
    int P2 = 1;
    while (P2 < cnt) P2 <<= 1;
    for (int s = cnt + t; s < P2; s += G) keys[s] = INT_MAX;
    gsync<WARP>();
    // bitonic sort of (keys, vals)[0, P2) ascending by key (keys are distinct)
    for (int k = 2; k <= P2; k <<= 1)
        for (int jj = k >> 1; jj > 0; jj >>= 1) {
            for (int x = t; x < P2; x += G) {
                const int y = x ^ jj;
                if (y > x) {
                    const bool up = (x & k) == 0;
                    const int kx = keys[x], ky = keys[y];
                    if ((kx > ky) == up) {
                        keys[x] = ky;
                        keys[y] = kx;
                        const double vx = vals[x];
                        vals[x] = vals[y];
                        vals[y] = vx;
                    }
                }
            }
            gsync<WARP>();
        }
    for (int s = t; s < cnt; s += G) {
        out_ci[out_off + s] = keys[s];
        out_v[out_off + s] = vals[s];
    }
    gsync<WARP>();
    return cnt;
}

// Warp per row. pass 0 writes counts[i] (-1: overflow -> big-row kernel);
// pass 1 fills rows whose count was >= 0.
__global__ void __launch_bounds__(32 * kWarpsPerCta) k_spgemm_warp(const DCsr64 A, const DCsr64 B, int pass,
                                                                  long long* counts, const long long* out_rp,
                                                                  long long* out_ci, double* out_v) {
    extern __shared__ unsigned char dyn[];
    double (*vals)[kWarpCap] = reinterpret_cast<double (*)[kWarpCap]>(dyn);
    int (*keys)[kWarpCap] = reinterpret_cast<int (*)[kWarpCap]>(dyn + sizeof(double) * kWarpsPerCta * kWarpCap);
    __shared__ int cnt[kWarpsPerCta], flag[kWarpsPerCta];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long nw = (long long)gridDim.x * kWarpsPerCta;
    for (long long i = (long long)blockIdx.x * kWarpsPerCta + w; i < A.n_rows; i += nw) {
        if (pass == 1 && counts[i] < 0) continue;
        const long long c = row_product<true>(A, B, i, pass, keys[w], vals[w], kWarpCap, lane,
                                              32, &cnt[w], &flag[w], pass == 1 ? out_rp[i] : 0, out_ci, out_v);
        if (pass == 0 && lane == 0) counts[i] = c;
    }
}

// One CTA per overflow row (list `rows`).
__global__ void __launch_bounds__(kBigThreads) k_spgemm_big(const DCsr64 A, const DCsr64 B, int pass,
                                                            const long long* rows, long long nrows,
                                                            long long* counts, const long long* out_rp,
                                                            long long* out_ci, double* out_v) {
    extern __shared__ unsigned char dyn[];
    double* vals = reinterpret_cast<double*>(dyn);
    int* keys = reinterpret_cast<int*>(vals + kBigCap);
    __shared__ int cnt, flag;
    for (long long r = blockIdx.x; r < nrows; r += gridDim.x) {
        const long long i = rows[r];
        const long long c = row_product<false>(A, B, i, pass, keys, vals, kBigCap, threadIdx.x, kBigThreads, &cnt,
                                               &flag, pass == 1 ? out_rp[i] : 0, out_ci, out_v);
        if (pass == 0 && threadIdx.x == 0) counts[i] = c;
    }
}

// C = A B on the device (inputs device-resident); returns C device-resident.
DevCsr spgemm(aspamg_gpu_ctx* c, const DCsr64& A, const DCsr64& B) {
    cudaStream_t s = c->stream;
    const long long n = A.n_rows;
    long long* counts = dalloc<long long>(c, (size_t)n + 1);
    const size_t warp_smem = (size_t)kWarpsPerCta * kWarpCap * (sizeof(double) + sizeof(int));
    CK(cudaFuncSetAttribute(k_spgemm_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)warp_smem));
    const int gw = grid_for((const void*)k_spgemm_warp, 32 * kWarpsPerCta, warp_smem);
    const size_t big_smem = (size_t)kBigCap * (sizeof(double) + sizeof(int));
    CK(cudaFuncSetAttribute(k_spgemm_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)big_smem));
    const int gb = grid_for((const void*)k_spgemm_big, kBigThreads, big_smem);
    k_spgemm_warp<<<gw, 32 * kWarpsPerCta, warp_smem, s>>>(A, B, 0, counts, nullptr, nullptr, nullptr);
    CK(cudaGetLastError());
    std::vector<long long> h((size_t)n);
    CK(cudaMemcpyAsync(h.data(), counts, (size_t)n * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    std::vector<long long> big;
    for (long long i = 0; i < n; ++i)
        if (h[(size_t)i] < 0) big.push_back(i);
    long long* dbig = nullptr;
    if (!big.empty()) {
        dbig = dalloc<long long>(c, big.size());
        CK(cudaMemcpyAsync(dbig, big.data(), big.size() * 8, cudaMemcpyHostToDevice, s));
        k_spgemm_big<<<gb, kBigThreads, big_smem, s>>>(A, B, 0, dbig, (long long)big.size(), counts, nullptr, nullptr,
                                                       nullptr);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(h.data(), counts, (size_t)n * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        for (long long i : big)
            if (h[(size_t)i] < 0)
                throw Fail{4, "galerkin: a product row has more than 16384 distinct columns"};
    }
    std::vector<long long> rp((size_t)n + 1, 0);
    for (long long i = 0; i < n; ++i) rp[(size_t)i + 1] = rp[(size_t)i] + h[(size_t)i];
    DevCsr C;
    C.rp = dalloc<long long>(c, (size_t)n + 1);
    C.ci = dalloc<long long>(c, (size_t)std::max<long long>(rp.back(), 1));
    C.v = dalloc<double>(c, (size_t)std::max<long long>(rp.back(), 1));
    CK(cudaMemcpyAsync(C.rp, rp.data(), rp.size() * 8, cudaMemcpyHostToDevice, s));
    k_spgemm_warp<<<gw, 32 * kWarpsPerCta, warp_smem, s>>>(A, B, 1, counts, C.rp, C.ci, C.v);
    CK(cudaGetLastError());
    if (!big.empty()) {
        k_spgemm_big<<<gb, kBigThreads, big_smem, s>>>(A, B, 1, dbig, (long long)big.size(), counts, C.rp, C.ci, C.v);
        CK(cudaGetLastError());
    }
    CK(cudaStreamSynchronize(s));  // rp (host) outlives the copy
    C.view = {n, B.n_cols, rp.back(), C.rp, C.ci, C.v};
    return C;
}

}  // namespace
}  // namespace aspamg_gpu

using namespace aspamg_gpu;

extern "C" int aspamg_gpu_galerkin(void* device, const aspamg_csr_view* P, const aspamg_csr_view* Pt,
                                   const aspamg_csr_view* A, aspamg_csr_alloc_fn alloc, void* sink) {
    aspamg_gpu_ctx* c = nullptr;
    int st = aspamg_gpu_ctx_create((int)(intptr_t)device, &c);
    if (st != 0) return st;
    st = guard(c, [&] {
        if (!P || !Pt || !A || !alloc) throw Fail{4, "galerkin: null argument"};
        if (P->n_rows != A->n_rows || A->n_rows != A->n_cols || Pt->n_rows != P->n_cols || Pt->n_cols != P->n_rows)
            throw Fail{1, "Galerkin product: A must be square with as many rows as P"};
        if (P->n_cols > INT_MAX - 1 || A->n_cols > INT_MAX - 1) throw Fail{1, "galerkin: column index range"};
        const DevCsr dA = upload64(c, *A), dP = upload64(c, *P), dPt = upload64(c, *Pt);
        const DevCsr AP = spgemm(c, dA.view, dP.view);
        const DevCsr Ac = spgemm(c, dPt.view, AP.view);
        int64_t *rp = nullptr, *ci = nullptr;
        double* v = nullptr;
        if (alloc(sink, Ac.view.n_rows, Ac.view.n_cols, Ac.view.nnz, &rp, &ci, &v) != 0 || !rp ||
            (Ac.view.nnz && (!ci || !v)))
            throw Fail{5, "galerkin: output allocation failed"};
        CK(cudaMemcpyAsync(rp, Ac.rp, sizeof(int64_t) * (Ac.view.n_rows + 1), cudaMemcpyDeviceToHost, c->stream));
        if (Ac.view.nnz) {
            CK(cudaMemcpyAsync(ci, Ac.ci, sizeof(int64_t) * Ac.view.nnz, cudaMemcpyDeviceToHost, c->stream));
            CK(cudaMemcpyAsync(v, Ac.v, sizeof(double) * Ac.view.nnz, cudaMemcpyDeviceToHost, c->stream));
        }
        CK(cudaStreamSynchronize(c->stream));
    });
    aspamg_gpu_ctx_destroy(c);
    return st;
}
