// Internal: shared pieces of the GPU setup components (setup_gpu.cu,
// galerkin_gpu.cu, fsai_gpu.cu): exact device BLAS-1 in the host setup's
// operation order, int64 CSR operands in the reference layout.
#pragma once

#include "ctx.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <utility>
#include <vector>

namespace aspamg_gpu {
namespace {

constexpr int kDotChunk = 8192;  // core.cpp dot(): CH
constexpr int kDotThreads = 256;
constexpr int kDotMaxVec = 32;
constexpr int kDotMaxPairs = 256;
constexpr int kDotStage = 2048;  // doubles per shared-memory stage

struct MDot {
    const double* vec[kDotMaxVec];
    unsigned char pa[kDotMaxPairs], pb[kDotMaxPairs];
    int nvec, npairs, sb;  // sb = rows per stage (nvec * sb <= kDotStage)
    long long n;
    double* part;  // [pair][chunk]
    int nchunks;
};

// One CTA per 8192-row chunk: rows are staged (registers -> shared memory, one
// stage ahead), thread t < npairs carries chain t: s = 0; s += a_i * b_i in
// ascending i — exactly the host chunk loop.
__global__ void __launch_bounds__(kDotThreads) k_mdot(const MDot d) {
    __shared__ double buf[2][kDotStage];
    const int tid = threadIdx.x;
    const long long lo = (long long)blockIdx.x * kDotChunk;
    const long long hi = min(d.n, lo + kDotChunk);
    const int per = (d.nvec * d.sb + kDotThreads - 1) / kDotThreads;  // <= kDotStage / kDotThreads
    double reg[kDotStage / kDotThreads];
    auto load = [&](long long r0) {
#pragma unroll
        for (int k = 0; k < kDotStage / kDotThreads; ++k) {
            const int idx = tid + k * kDotThreads;
            reg[k] = 0.0;
            if (k < per && idx < d.nvec * d.sb) {
                const int v = idx / d.sb, r = idx % d.sb;
                const long long row = r0 + r;
                if (row < hi) reg[k] = __ldcs(d.vec[v] + row);
            }
        }
    };
    auto store = [&](int b) {
#pragma unroll
        for (int k = 0; k < kDotStage / kDotThreads; ++k) {
            const int idx = tid + k * kDotThreads;
            if (k < per && idx < d.nvec * d.sb) buf[b][idx] = reg[k];
        }
    };
    double s = 0.0;
    const int a = tid < d.npairs ? d.pa[tid] : 0;
    const int bq = tid < d.npairs ? d.pb[tid] : 0;
    load(lo);
    store(0);
    __syncthreads();
    int b = 0;
    for (long long r0 = lo; r0 < hi; r0 += d.sb) {
        const bool more = r0 + d.sb < hi;
        if (more) load(r0 + d.sb);
        if (tid < d.npairs) {
            const double* xa = &buf[b][a * d.sb];
            const double* xb = &buf[b][bq * d.sb];
            const int cnt = (int)min((long long)d.sb, hi - r0);
            for (int r = 0; r < cnt; ++r) s = __dadd_rn(s, __dmul_rn(xa[r], xb[r]));
        }
        if (more) store(b ^ 1);
        __syncthreads();
        b ^= 1;
    }
    if (tid < d.npairs) d.part[(size_t)tid * d.nchunks + blockIdx.x] = s;
}

enum VecOp : int {
    V_SUBFROM = 0,  // y = x - y
    V_AXPY,         // y = y + s1 x
    V_MINUS_CX,     // y = y - s1 x
    V_DIV,          // y = x / s1
    V_RESID,        // y = x - s1 w
    V_TWICE,        // y = 2 x
    V_SD,           // y = 2 (x - s1 w) / s2
    V_SCALE,        // y = s1 x
    V_PUPD,         // y = x + s1 y
    V_SCALE_IP,     // y = y s1
    V_COPY,         // y = x
};

__global__ void k_vec(int op, long long n, const double* __restrict__ x, const double* __restrict__ w, double* y,
                      double s1, double s2) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        double o;
        switch (op) {
            case V_SUBFROM: o = __dsub_rn(x[i], y[i]); break;
            case V_AXPY: o = __dadd_rn(y[i], __dmul_rn(s1, x[i])); break;
            case V_MINUS_CX: o = __dsub_rn(y[i], __dmul_rn(s1, x[i])); break;
            case V_DIV: o = __ddiv_rn(x[i], s1); break;
            case V_RESID: o = __dsub_rn(x[i], __dmul_rn(s1, w[i])); break;
            case V_TWICE: o = __dmul_rn(2.0, x[i]); break;
            case V_SD: o = __ddiv_rn(__dmul_rn(2.0, __dsub_rn(x[i], __dmul_rn(s1, w[i]))), s2); break;
            case V_SCALE: o = __dmul_rn(s1, x[i]); break;
            case V_PUPD: o = __dadd_rn(x[i], __dmul_rn(s1, y[i])); break;
            case V_SCALE_IP: o = __dmul_rn(y[i], s1); break;
            default: o = x[i];
        }
        y[i] = o;
    }
}


struct DCsr64 {
    long long n_rows = 0, n_cols = 0, nnz = 0;
    const long long* rp = nullptr;
    const long long* ci = nullptr;
    const double* v = nullptr;
};

struct DevCsr {
    long long *rp = nullptr, *ci = nullptr;
    double* v = nullptr;
    DCsr64 view;
};

DevCsr upload64(aspamg_gpu_ctx* c, const aspamg_csr_view& h) {
    DevCsr d;
    const size_t n1 = (size_t)h.n_rows + 1, nz = (size_t)h.nnz;
    d.rp = dalloc<long long>(c, n1);
    d.ci = dalloc<long long>(c, nz);
    d.v = dalloc<double>(c, nz);
    CK(cudaMemcpyAsync(d.rp, h.row_offsets, n1 * 8, cudaMemcpyHostToDevice, c->stream));
    if (nz) {
        CK(cudaMemcpyAsync(d.ci, h.col_indices, nz * 8, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(d.v, h.values, nz * 8, cudaMemcpyHostToDevice, c->stream));
    }
    d.view = {h.n_rows, h.n_cols, h.nnz, d.rp, d.ci, d.v};
    return d;
}

int grid_for(const void* fn, int threads, size_t smem) {
    int dev = 0, sms = 148, occ = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem);
    return sms * std::max(occ, 1);
}

using Pair = std::pair<const double*, const double*>;

// Exact device BLAS-1 for the setup components: one context, one stream,
// synchronous scalar read-backs (dots in core.cpp's order, elementwise ops with
// round-to-nearest intrinsics).
struct DevLA {
    aspamg_gpu_ctx* c = nullptr;
    cudaStream_t s = nullptr;
    long long n = 0;
    int nchunks = 1;
    double* part = nullptr;
    std::vector<double> hpart;
    int vgrid = 1;

    void init(aspamg_gpu_ctx* ctx, long long rows) {
        c = ctx;
        s = ctx->stream;
        n = rows;
        nchunks = (int)std::max<long long>(1, (n + kDotChunk - 1) / kDotChunk);
        part = dalloc<double>(c, (size_t)kDotMaxPairs * nchunks);
        hpart.resize((size_t)kDotMaxPairs * nchunks);
        vgrid = vec_grid((int)std::max<long long>(n, 1));
    }

    void vec(int op, const double* x, const double* w, double* y, double s1 = 0.0, double s2 = 0.0) {
        k_vec<<<vgrid, 256, 0, s>>>(op, n, x, w, y, s1, s2);
        CK(cudaGetLastError());
    }
    void copy(const double* x, double* y) { CK(cudaMemcpyAsync(y, x, sizeof(double) * n, cudaMemcpyDeviceToDevice, s)); }
    // core.cpp dot() for every pair, in one launch per <= 256 pairs.
    std::vector<double> dots(const std::vector<Pair>& pairs) {
        std::vector<double> out(pairs.size());
        size_t p0 = 0;
        while (p0 < pairs.size()) {
            MDot d{};
            d.n = n;
            d.part = part;
            d.nchunks = nchunks;
            std::vector<const double*> vs;
            size_t p = p0;
            for (; p < pairs.size() && p - p0 < (size_t)kDotMaxPairs; ++p) {
                int ia = -1, ib = -1;
                for (int k = 0; k < (int)vs.size(); ++k) {
                    if (vs[k] == pairs[p].first) ia = k;
                    if (vs[k] == pairs[p].second) ib = k;
                }
                const int need = (ia < 0) + (ib < 0 && pairs[p].second != pairs[p].first);
                if ((int)vs.size() + need > kDotMaxVec) break;
                if (ia < 0) { ia = (int)vs.size(); vs.push_back(pairs[p].first); }
                if (ib < 0) {
                    if (pairs[p].second == pairs[p].first) ib = ia;
                    else { ib = (int)vs.size(); vs.push_back(pairs[p].second); }
                }
                d.pa[p - p0] = (unsigned char)ia;
                d.pb[p - p0] = (unsigned char)ib;
            }
            d.npairs = (int)(p - p0);
            d.nvec = (int)vs.size();
            for (int k = 0; k < d.nvec; ++k) d.vec[k] = vs[k];
            int sb = kDotStage / d.nvec;
            d.sb = std::min(sb, kDotChunk);
            k_mdot<<<nchunks, kDotThreads, 0, s>>>(d);
            CK(cudaGetLastError());
            const size_t cnt = (size_t)d.npairs * nchunks;
            CK(cudaMemcpyAsync(hpart.data(), part, cnt * sizeof(double), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            for (int q = 0; q < d.npairs; ++q) {
                if (nchunks == 1) {  // dot(): single sequential sum, no partial pass
                    out[p0 + q] = hpart[(size_t)q];
                    continue;
                }
                double acc = 0.0;
                for (int ch = 0; ch < nchunks; ++ch) acc += hpart[(size_t)q * nchunks + ch];
                out[p0 + q] = acc;
            }
            p0 = p;
        }
        return out;
    }
    double dot(const double* a, const double* b) { return dots({{a, b}})[0]; }
    double norm2(const double* a) { return std::sqrt(dot(a, a)); }
};

}  // namespace
}  // namespace aspamg_gpu
