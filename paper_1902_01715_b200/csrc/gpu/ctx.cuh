// Internal: the device context shared by the solve (context.cu) and the
// GPU setup components (setup_gpu.cu). Not part of the C-ABI.
#pragma once

#include "../../../include/aspamg_gpu.h"
#include "kernels.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <functional>
#include <string>
#include <vector>

namespace aspamg_gpu {

inline thread_local std::string g_last_err;

struct Op {
    std::string name;
    int level;
    double bytes;  // algorithmic bytes (compulsory traffic)
    std::function<void(cudaStream_t)> fn;
    bool describable = false;  // expressible as a TailOp (CSR product / zero fill, no reduction)
    TailOp desc{};
};

struct GLevel {
    int n = 0;
    DMat A, G, Gt, P, Pt;
    double omega = 1.0;
    bool has_smoother = false;
    double* y = nullptr;  // input (levels > 0)
    double* z = nullptr;  // output == s accumulator (levels > 0)
    double* r = nullptr;
    double* t = nullptr;
    long long a_nnz = 0;
};

struct Site {  // one deterministic reduction site
    double* partials = nullptr;
    unsigned* counter = nullptr;
};

}  // namespace aspamg_gpu

using namespace aspamg_gpu;

struct aspamg_gpu_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::string err;
    std::vector<GLevel> lv;
    int nu1 = 1, nu2 = 1;
    // coarsest factor
    int n_c = 0;
    double *Lrm = nullptr, *Lcm = nullptr, *Dinv_f = nullptr, *Dinv_b = nullptr;
    double* cw = nullptr;  // temp between the two triangular products
    DMat Wm, Wtm;          // W = L^{-1} (lower) and W' (upper) as CSR operands
    // Collapsed coarse tail (opt "tail_dense"): the V-cycle from level tail_level
    // down is a fixed linear operator; its n x n matrix (columns = the sub-cycle
    // applied to unit vectors on the device at finalize) replaces those levels.
    int tail_level = -1;
    DMat Tm;
    bool coarse_uploaded = false;
    bool finalized = false;
    // options
    int opt_bsr = 1, opt_device_loop = 1, opt_coarse_mode = 1;
    long long opt_sell_min_rows = 65536, opt_sell_max_mean = 48, opt_sell_max_len = 64, opt_sell_sigma = 4096, opt_sell_sort_fill_pct = 110,
              opt_sell_u = 0, opt_sell_chh = 0, opt_sell_sort = 0,
              opt_sell_min_mean = 8;
    // Tile-local SELL (kernels.cuh DXsell), OFF by default: measured slower than SELL / CSR on every
    // operand role except the level-0 G' (C2: 37-45 vs 40-48 us; G 36 vs 31, P' 34 vs 12 us;
    // profiles/tune_r02_c2_xsell.json). Bit mask over operand roles (1 A, 2 G, 4 G', 8 P, 16 P'),
    // minimum rows, maximum mean row length, threads per CTA (0 = by size: 256 / 128 / 64), rows per
    // lane (fold: 1, or 2 = long rows paired with short ones; a tile has threads x fold rows),
    // footprint granule (log2 doubles), kernel variant (quads per group x 10 + min CTAs/SM),
    // shared-memory budget per CTA.
    long long opt_xsell = 0, opt_xsell_min_rows = 32768, opt_xsell_max_mean = 256, opt_xsell_min_mean = 0, opt_xsell_rows = 0,
              opt_xsell_rows256 = 400000, opt_xsell_rows128 = 100000, opt_xsell_gran = 3, opt_xsell_q = 0,
              opt_xsell_smem_kb = 100, opt_xsell_fold = 2;
    // collapse the V-cycle below the first level with <= this many rows (0 = off);
    // C2 0.995 -> 0.966 ms/it, C1 0.120 -> 0.107 ms/it (profiles/tune_r01_tail_long.log)
    long long opt_tail_dense = 1500;
    // k_csrw: operands with at least this many rows give every CTA a contiguous row block (x lines
    // gathered for rows r..r+7 are reused from L1 by the CTA's next steps); 0 = off. C5: 10.35 -> 10.01
    // ms/it (level-1/2 operands -3..-8 %); C2's 168k-row A_1 is 3 % slower with it, hence the threshold.
    long long opt_csr_blocked = 250000;
    long long opt_csr_noalloc = 0;  // k_csrw on streamed operands: matrix loads with L1::no_allocate
    long long opt_csrw = 4;  // warp-per-row pipelined CSR kernel for group == 32 operands: columns per lane per round (4 / 8), 0 = off
    long long opt_csr_max_group = 32;  // threads per row cap for operands with >= 600k / cap rows
    long long opt_fuse_rr = 0;  // restriction fused with the residual (one cooperative launch per level)
    long long opt_csr_long = 4;  // long-row split threshold in rounds (rows > long*T*4 entries; 0 = off)
    long long opt_csr_pf = 1;  // CSR (T <= 16): prefetch the next row's pointers (measured 1.4% faster per PCG iteration on C2)
    long long opt_idx16 = 1;  // 16-bit column offsets where every row spans < 2^16 columns
    long long opt_idx16_max_group = 16;  // ... and (CSR) at most this many threads per row
    long long opt_stream_bytes = 48ll << 20, opt_keep_bytes = 64ll << 20, opt_tail_rows = 0, opt_csr_per_thread = 4;
    // PCG state and vectors
    PcgState* st = nullptr;       // device
    PcgState* st_host = nullptr;  // pinned
    int* zero_flag = nullptr;     // device int 0 (done pointer for standalone calls)
    double *b = nullptr, *x = nullptr, *r = nullptr, *z = nullptr, *p = nullptr, *q = nullptr;
    double* hist = nullptr;
    long long hist_cap = 0;
    double *vy = nullptr, *vz = nullptr;  // standalone V-cycle in/out
    std::vector<void*> allocs;
    std::vector<Site> sites;
    // op lists + graphs
    std::vector<Op> body, vc_ops, init0, init1, post;
    cudaGraphExec_t pcg_exec = nullptr, body_exec = nullptr, vc_exec = nullptr;
    cudaGraph_t pcg_graph = nullptr, body_graph = nullptr, vc_graph = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    double last_ms = 0.0;
    long long last_launches = 0;
    size_t device_bytes = 0;
};

namespace aspamg_gpu {

struct CudaFail {
    std::string msg;
};

#define CK(call)                                                                                 \
    do {                                                                                         \
        cudaError_t e_ = (call);                                                                 \
        if (e_ != cudaSuccess)                                                                   \
            throw CudaFail{std::string(#call) + ": " + cudaGetErrorString(e_)};                  \
    } while (0)

struct Fail {
    int code;
    std::string msg;
};

template <class F>
inline int guard(aspamg_gpu_ctx* c, F&& f) {
    try {
        f();
        return 0;
    } catch (const Fail& e) {
        if (c) c->err = e.msg;
        g_last_err = e.msg;
        return e.code;
    } catch (const CudaFail& e) {
        if (c) c->err = e.msg;
        g_last_err = e.msg;
        return 5;
    } catch (const std::bad_alloc&) {
        if (c) c->err = "out of host memory";
        g_last_err = "out of host memory";
        return 5;
    } catch (const std::exception& e) {
        if (c) c->err = e.what();
        g_last_err = e.what();
        return 5;
    }
}

template <class T>
inline T* dalloc(aspamg_gpu_ctx* c, size_t count) {
    void* p = nullptr;
    if (count == 0) count = 1;
    CK(cudaMalloc(&p, count * sizeof(T)));
    c->allocs.push_back(p);
    c->device_bytes += count * sizeof(T);
    return static_cast<T*>(p);
}

// Free one dalloc'ed block before the context ends (setup scratch).
inline void dfree(aspamg_gpu_ctx* c, void* p) {
    if (!p) return;
    auto it = std::find(c->allocs.begin(), c->allocs.end(), p);
    if (it == c->allocs.end()) return;
    cudaFree(p);
    c->allocs.erase(it);
}

inline Red make_red(aspamg_gpu_ctx* c, int grid, int fin, double* out = nullptr) {
    Site s;
    s.partials = dalloc<double>(c, 2 * (size_t)std::max(grid, 1));
    s.counter = dalloc<unsigned>(c, 1);
    CK(cudaMemset(s.counter, 0, sizeof(unsigned)));
    c->sites.push_back(s);
    Red r;
    r.partials = s.partials;
    r.counter = s.counter;
    r.fin = fin;
    r.out = out;
    r.st = c->st;
    return r;
}


// Operand upload with per-operand format choice (sliced BSR3 / SELL / CSR).
// role: 0 A, 1 G, 2 G', 3 P, 4 P' of a hierarchy level (eligible for the tile-local SELL format by
// the "xsell" option mask), -1 anything else.
DMat upload_mat(aspamg_gpu_ctx* c, const aspamg_csr_view& v, bool allow_bsr, int role = -1);

}  // namespace aspamg_gpu
