// Device context, hierarchy upload, V-cycle / PCG orchestration (CUDA graph
// with a device-side while loop) and the C-ABI of include/aspamg_gpu.h.
//
// Orchestration restates, on the device:
//   vcycle_apply  SPEC.md:445-453 / Alg. 2 PAPER.md:287-306 (s = 0 start, so the
//                 first pre-smoothing step is s = w G'(G y) exactly)
//   pcg           SPEC.md:504-512 (x0 = 0 default, ||r|| <= tol ||b||, not-SPD on
//                 p'Ap <= 0, true-residual recheck x10)
// The iteration is rotated so the convergence test is the last kernel of the
// loop body: body = [V-cycle(r)->z (+ r.z -> beta), p = z + beta p,
// q = K p (+ p.q -> alpha), x += alpha p, r -= alpha q (+ r.r -> history,
// test -> graph condition)]. This is the reference's order of operations.
#include "ctx.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

namespace aspamg_gpu {

// ----------------------------------------------------------- format choice
bool exact_bsr3(const aspamg_csr_view& v) {
    if (v.n_rows % 3 || v.n_cols % 3 || v.n_rows == 0) return false;
    const int64_t* rp = v.row_offsets;
    const int64_t* ci = v.col_indices;
    const int64_t nb = v.n_rows / 3;
    int ok = 1;
#pragma omp parallel for schedule(static) reduction(&& : ok)
    for (int64_t br = 0; br < nb; ++br) {
        const int64_t r0 = 3 * br;
        const int64_t len = rp[r0 + 1] - rp[r0];
        bool good = len % 3 == 0;
        for (int k = 1; k < 3 && good; ++k)
            if (rp[r0 + k + 1] - rp[r0 + k] != len) good = false;
        for (int64_t t = 0; t < len && good; t += 3) {
            const int64_t c0 = ci[rp[r0] + t];
            if (c0 % 3) good = false;
            for (int k = 0; k < 3 && good; ++k)
                for (int cc = 0; cc < 3; ++cc)
                    if (ci[rp[r0 + k] + t + cc] != c0 + cc) good = false;
        }
        ok = ok && good;
    }
    return ok != 0;
}

void check_view(const aspamg_csr_view* v, const char* what) {
    if (!v) throw Fail{1, std::string(what) + ": null matrix"};
    if (v->n_rows < 0 || v->n_cols < 0) throw Fail{1, std::string(what) + ": negative size"};
    if (v->n_rows > 0 && !v->row_offsets) throw Fail{1, std::string(what) + ": null row_offsets"};
    if (v->n_rows > 0 && v->row_offsets[v->n_rows] != v->nnz) throw Fail{1, std::string(what) + ": nnz mismatch"};
    if (v->nnz >= (1ll << 31) || v->n_rows >= (1ll << 31) || v->n_cols >= (1ll << 31))
        throw Fail{4, std::string(what) + ": exceeds int32 device indexing"};
    // Columns in range and strictly ascending within each row (the SparseMatrix
    // invariant, sparse_matrix.hpp:27-33): the 16-bit column mode stores
    // col - first-col-of-row and would wrap on an unsorted row.
    int bad = 0;
#pragma omp parallel for schedule(dynamic, 4096) reduction(| : bad)
    for (int64_t i = 0; i < v->n_rows; ++i) {
        const int64_t b = v->row_offsets[i], e = v->row_offsets[i + 1];
        if (b > e || b < 0 || e > v->nnz) { bad |= 2; continue; }
        for (int64_t k = b; k < e; ++k) {
            const int64_t c = v->col_indices[k];
            bad |= (c < 0 || c >= v->n_cols);
            if (k > b && c <= v->col_indices[k - 1]) bad |= 4;
        }
    }
    if (bad & 2) throw Fail{1, std::string(what) + ": row offsets not monotone"};
    if (bad & 1) throw Fail{1, std::string(what) + ": column index out of range"};
    if (bad & 4) throw Fail{1, std::string(what) + ": column indices not strictly ascending within a row"};
}

// Threads per row for the CSR kernel: ~4+ entries per thread, widened for
// small levels so the grid still covers the GPU (>= ~150k threads).
// Threads per row for the CSR kernel: ~4+ entries per thread for the mean
// row, at most ~16 sequential entries for the longest row (its serial chain
// sets the kernel latency on small levels), and widened for small levels so
// the grid still covers the GPU (>= ~150k threads).
// Threads per row for the CSR kernel: ~8 entries per thread for the mean row;
// on small operands (< 64k rows, where the longest row's serial chain sets the
// kernel latency) also <= ~32 sequential entries for the longest row, and
// widened so the grid still covers the GPU (>= ~150k threads).
// `big_cap`: operands with enough rows to fill the GPU at `big_cap` threads per row
// (>= ~600k threads) use at most that many: with one warp per row the row sum needs
// no shared-memory combine and no CTA barrier (ncu, C5 level 1: csr64 at 0.75 of
// peak with `barrier` the second stall reason).
int group_for(double mean, int maxlen, int64_t n_rows, double per_thread = 4.0, int big_cap = 256) {
    int g = 1;
    while (g < 256 && per_thread * 2 * g <= mean) g *= 2;
    if (n_rows < 65536)
        while (g < 256 && 32 * g < maxlen) g *= 2;
    while (g < 256 && (double)n_rows * g < 150000.0 && 2.0 * g <= std::max(mean, 1.0)) g *= 2;
    if (g > big_cap && (double)n_rows * big_cap >= 600000.0) g = big_cap;
    return g;
}

// Chunk metadata of a sliced layout: rows (or block rows) in chunks of 32,
// chunk width = longest row of the chunk.
// Chunk metadata of a sliced layout: rows (or block rows) in chunks of h,
// chunk width = longest row of the chunk; `slots` counts padded slot rows of
// h entries (entry (j, r) of chunk q lives at (off_q + j) * h + r).
void slice_meta(const std::vector<int>& len, std::vector<int2>& meta, long long& slots, int h = 32) {
    const int n = (int)len.size();
    const int nch = (n + h - 1) / h;
    meta.resize((size_t)std::max(nch, 1));
    slots = 0;
    for (int ch = 0; ch < nch; ++ch) {
        int w = 0;
        for (int l = 0; l < h && ch * h + l < n; ++l) w = std::max(w, len[(size_t)ch * h + l]);
        if (slots > INT_MAX - 65536) throw Fail{4, "sliced layout exceeds int32 slot offsets"};
        meta[(size_t)ch] = make_int2((int)slots, w);
        slots += w;
    }
}

// True when every row's columns fit in [first, first + 65535] (sorted rows).
bool rows_fit_u16(const aspamg_csr_view& v) {
    int ok = 1;
#pragma omp parallel for schedule(static) reduction(&& : ok)
    for (int64_t i = 0; i < v.n_rows; ++i) {
        const int64_t b = v.row_offsets[i], e = v.row_offsets[i + 1];
        if (e > b && v.col_indices[e - 1] - v.col_indices[b] > 65535) ok = 0;
    }
    return ok != 0;
}

// Tile-local SELL build (layout in kernels.cuh, DXsell), host side. Returns
// false when the operand does not fit the format (a tile's x footprint larger
// than the shared-memory budget, a row longer than 65535 entries).
struct XsellHost {
    int R = 0, F = 1, g = 0, fp_doubles = 0;
    int64_t nt = 0;
    long long quads = 0, list_len = 0;
    std::vector<unsigned short> slen, perm;
    std::vector<int2> tmeta, cmeta;
    std::vector<int> list;
    std::vector<double2> val;
    std::vector<uint2> lc;
};

// Slot (chunk, lane, part) of sorted rank i inside a tile of R rows: fold 1 ->
// chunk i / 32, lane i % 32, part a; fold 2 -> ranks < R/2 are the a rows of
// thread i, ranks >= R/2 the b rows of thread R-1-i.
struct XsellSlot {
    int chunk, lane, part;
};
inline XsellSlot xsell_slot(int i, int R, int F) {
    if (F == 1 || i < R / 2) return {i / 32, i % 32, 0};
    const int t = R - 1 - i;
    return {t / 32, t % 32, 1};
}

bool build_xsell_host(const aspamg_csr_view& v, int R, int F, int g, size_t cap_doubles, XsellHost& H) {
    const int64_t n = v.n_rows;
    if (n <= 0 || v.nnz <= 0) return false;
    const int64_t nt = (n + R - 1) / R;
    const int cpt = R / F / 32;  // chunks (warps) per tile
    H.F = F;
    if (nt * cpt >= (1ll << 30)) return false;
    H.R = R;
    H.g = g;
    H.nt = nt;
    H.slen.assign((size_t)(nt * R), 0);
    H.perm.assign((size_t)(nt * R), 0);
    std::vector<int> cw((size_t)(nt * cpt), 0), cwb((size_t)(nt * cpt), 0);
    std::vector<std::vector<int>> fp((size_t)nt);
    int too_big = 0;
#pragma omp parallel
    {
        std::vector<int> ord((size_t)R), gl;
#pragma omp for schedule(dynamic, 16)
        for (int64_t t = 0; t < nt; ++t) {
            const int64_t r0 = t * R, r1 = std::min<int64_t>(n, r0 + R);
            const int m = (int)(r1 - r0);
            auto rlen = [&](int i) { return v.row_offsets[r0 + i + 1] - v.row_offsets[r0 + i]; };
            for (int i = 0; i < R; ++i) ord[(size_t)i] = i;
            std::stable_sort(ord.begin(), ord.begin() + m, [&](int a, int b) { return rlen(a) > rlen(b); });
            for (int i = 0; i < R; ++i) {
                H.perm[(size_t)(r0 + i)] = (unsigned short)ord[(size_t)i];
                const int64_t li = i < m ? rlen(ord[(size_t)i]) : 0;
                if (li > 65535) {
#pragma omp atomic write
                    too_big = 1;
                }
                H.slen[(size_t)(r0 + i)] = (unsigned short)std::min<int64_t>(li, 65535);
            }
            for (int w = 0; w < cpt; ++w) {  // sorted: the smallest rank of a chunk part is its longest row
                cw[(size_t)(t * cpt + w)] = H.slen[(size_t)(r0 + 32 * w)];
                if (F == 2) cwb[(size_t)(t * cpt + w)] = H.slen[(size_t)(r0 + R - 32 * w - 32)];
            }
            gl.clear();
            for (int64_t k = v.row_offsets[r0]; k < v.row_offsets[r1]; ++k) gl.push_back((int)(v.col_indices[k] >> g));
            std::sort(gl.begin(), gl.end());
            gl.erase(std::unique(gl.begin(), gl.end()), gl.end());
            if (((size_t)gl.size() << g) > cap_doubles || ((size_t)gl.size() << g) > 65536) {
#pragma omp atomic write
                too_big = 1;
            }
            fp[(size_t)t] = gl;
        }
    }
    if (too_big) return false;
    H.tmeta.resize((size_t)nt);
    H.cmeta.resize((size_t)(nt * cpt));
    long long lo = 0, qo = 0;
    size_t maxfp = 0;
    for (int64_t t = 0; t < nt; ++t) {
        H.tmeta[(size_t)t] = make_int2((int)lo, (int)fp[(size_t)t].size());
        lo += (long long)fp[(size_t)t].size();
        maxfp = std::max(maxfp, fp[(size_t)t].size());
        for (int w = 0; w < cpt; ++w) {
            const int wd = cw[(size_t)(t * cpt + w)], wb = cwb[(size_t)(t * cpt + w)];
            H.cmeta[(size_t)(t * cpt + w)] = make_int2((int)qo, wd | (wb << 16));
            qo += (wd + 3) / 4 + (wb + 3) / 4;
        }
        if (lo > INT_MAX - 65536 || qo > INT_MAX / 64 - 65536) return false;
    }
    H.list.resize((size_t)std::max<long long>(lo, 1));
    H.val.assign((size_t)std::max<long long>(qo, 1) * 64, make_double2(0.0, 0.0));
    H.lc.assign((size_t)std::max<long long>(qo, 1) * 32, make_uint2(0u, 0u));
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t t = 0; t < nt; ++t) {
        const std::vector<int>& gl = fp[(size_t)t];
        std::copy(gl.begin(), gl.end(), H.list.begin() + H.tmeta[(size_t)t].x);
        const int64_t r0 = t * R, r1 = std::min<int64_t>(n, r0 + R);
        for (int i = 0; i < (int)(r1 - r0); ++i) {
            const int64_t row = r0 + H.perm[(size_t)(r0 + i)];
            const XsellSlot sl = xsell_slot(i, R, F);
            const int2 cmw = H.cmeta[(size_t)(t * cpt + sl.chunk)];
            const long long q0 = cmw.x + (sl.part ? ((cmw.y & 0xffff) + 3) / 4 : 0);
            const int lane = sl.lane;
            const int64_t b = v.row_offsets[row], e = v.row_offsets[row + 1];
            for (int64_t k = b; k < e; ++k) {
                const int j = (int)(k - b);
                const int64_t col = v.col_indices[k];
                const int rank = (int)(std::lower_bound(gl.begin(), gl.end(), (int)(col >> g)) - gl.begin());
                const unsigned loc = ((unsigned)rank << g) | (unsigned)(col & ((1 << g) - 1));
                const long long q = q0 + j / 4;
                double2& dv = H.val[(size_t)((q * 2 + (j % 4) / 2) * 32 + lane)];
                if (j % 2 == 0) dv.x = v.values[k];
                else dv.y = v.values[k];
                uint2& dc = H.lc[(size_t)(q * 32 + lane)];
                unsigned& w = (j % 4) < 2 ? dc.x : dc.y;
                w |= (j % 2 == 0) ? loc : (loc << 16);
            }
        }
    }
    H.quads = qo;
    H.list_len = lo;
    H.fp_doubles = (int)(((maxfp << g) + 1) / 2 * 2);
    return true;
}

// CPU walk of the layout exactly as k_xsell indexes it (staged window, quads,
// per-lane sequential sums, output through the tile permutation): the layout
// check that runs without a GPU (tests/test_abi.py).
void xsell_host_spmv(const XsellHost& H, int64_t n_rows, int64_t n_cols, const double* x, double* y) {
    const int R = H.R, F = H.F, g = H.g, cpt = R / F / 32;
#pragma omp parallel
    {
        std::vector<double> win((size_t)H.fp_doubles + 2), ys((size_t)R);
#pragma omp for schedule(dynamic, 16)
        for (int64_t t = 0; t < H.nt; ++t) {
            const int2 tm = H.tmeta[(size_t)t];
            for (int q = 0; q < tm.y; ++q)
                for (int o = 0; o < (1 << g); ++o) {
                    const int64_t i = ((int64_t)H.list[(size_t)(tm.x + q)] << g) + o;
                    win[(size_t)((q << g) + o)] = i < n_cols ? x[i] : 0.0;
                }
            for (int i = 0; i < R; ++i) {
                const int64_t srow = t * R + i;
                const int len = H.slen[(size_t)srow];
                const XsellSlot sl = xsell_slot(i, R, F);
                const int2 cm = H.cmeta[(size_t)(t * cpt + sl.chunk)];
                const long long qb = cm.x + (sl.part ? ((cm.y & 0xffff) + 3) / 4 : 0);
                const int lane = sl.lane;
                double s = 0.0;
                for (int j = 0; j < len; ++j) {
                    const long long q = qb + j / 4;
                    const double2 dv = H.val[(size_t)((q * 2 + (j % 4) / 2) * 32 + lane)];
                    const uint2 dc = H.lc[(size_t)(q * 32 + lane)];
                    const unsigned w = (j % 4) < 2 ? dc.x : dc.y;
                    const unsigned loc = (j % 2 == 0) ? (w & 0xffffu) : (w >> 16);
                    const double prod = ((j % 2 == 0) ? dv.x : dv.y) * win[loc];
                    s = s + prod;
                }
                ys[(size_t)H.perm[(size_t)srow]] = s;
            }
            for (int tid = 0; tid < R; ++tid)
                if (t * R + tid < n_rows) y[t * R + tid] = ys[(size_t)tid];
        }
    }
}

// Threads per CTA: "xsell_rows" when set, else by operand size (256 / 128 / 64)
// so that mid-size operands still spread over all SMs.
int xsell_threads(const aspamg_gpu_ctx* c, int64_t n) {
    int T = (int)c->opt_xsell_rows;
    if (T <= 0) T = n >= c->opt_xsell_rows256 ? 256 : n >= c->opt_xsell_rows128 ? 128 : 64;
    return std::clamp(T / 32 * 32, 32, kBlock);
}

bool build_xsell(aspamg_gpu_ctx* c, const aspamg_csr_view& v, DXsell& X) {
    const int g = (int)std::clamp<long long>(c->opt_xsell_gran, 1, 4);
    const int F = c->opt_xsell_fold == 2 ? 2 : 1;
    int T = xsell_threads(c, v.n_rows);
    XsellHost H;
    // a tile's footprint must fit the shared-memory budget: halve the tile until it does
    for (;; T /= 2) {
        if (T < 32) return false;
        const int R = T * F;
        const size_t cap_doubles = (size_t)std::max<long long>(c->opt_xsell_smem_kb, 8) * 128 - (size_t)R;
        H = XsellHost{};
        if (build_xsell_host(v, R, F, g, cap_doubles, H)) break;
    }
    const int R = T * F;
    X.n_rows = (int)v.n_rows;
    X.n_cols = (int)v.n_cols;
    X.ntiles = (int)H.nt;
    X.R = R;
    X.fold = F;
    X.gran = g;
    X.nnz = v.nnz;
    X.quads = H.quads;
    X.list_len = H.list_len;
    X.fp_doubles = H.fp_doubles;
    auto up = [&](auto*& dst, const auto& src) {
        using T = typename std::remove_reference<decltype(src)>::type::value_type;
        dst = dalloc<T>(c, src.size());
        CK(cudaMemcpy(dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice));
    };
    up(X.tmeta, H.tmeta);
    up(X.cmeta, H.cmeta);
    up(X.len, H.slen);
    up(X.perm, H.perm);
    up(X.list, H.list);
    up(X.v, H.val);
    up(X.lc, H.lc);
    X.pol = (long long)(10.0 * v.nnz) > c->opt_stream_bytes ? 1 : 0;
    X.q = c->opt_xsell_q > 0 ? (int)c->opt_xsell_q : 24;
    xsell_prepare(X);
    CK(cudaGetLastError());
    return true;
}

DMat upload_mat(aspamg_gpu_ctx* c, const aspamg_csr_view& v, bool allow_bsr, int role) {
    DMat M;
    const long long nnz = v.nnz;
    const bool bsr = allow_bsr && c->opt_bsr && exact_bsr3(v);
    const double mean = v.n_rows ? double(nnz) / double(v.n_rows) : 0.0;
    if (bsr) {
        M.fmt = 1;
        DSbsr3& B = M.sb;
        B.nb = (int)(v.n_rows / 3);
        B.nbc = (int)(v.n_cols / 3);
        B.nnzb = nnz / 9;
        B.nchunks = (B.nb + 31) / 32;
        std::vector<int> len((size_t)B.nb);
        for (int br = 0; br < B.nb; ++br)
            len[(size_t)br] = (int)((v.row_offsets[3 * (int64_t)br + 1] - v.row_offsets[3 * (int64_t)br]) / 3);
        std::vector<int2> meta;
        slice_meta(len, meta, B.slots);
        std::vector<int> ci((size_t)B.slots * 32, 0);
        std::vector<double> val((size_t)B.slots * 288, 0.0);
#pragma omp parallel for schedule(static)
        for (int br = 0; br < B.nb; ++br) {
            const int ch = br / 32, lane = br % 32;
            const long long off = meta[(size_t)ch].x;
            const int64_t r0 = 3 * (int64_t)br;
            for (int j = 0; j < len[(size_t)br]; ++j) {
                ci[(size_t)((off + j) * 32 + lane)] = (int)(v.col_indices[v.row_offsets[r0] + 3 * j] / 3);
                for (int r = 0; r < 3; ++r)
                    for (int cc = 0; cc < 3; ++cc)
                        val[(size_t)(((off + j) * 9 + 3 * r + cc) * 32 + lane)] = v.values[v.row_offsets[r0 + r] + 3 * j + cc];
            }
        }
        B.len = dalloc<int>(c, len.size());
        B.meta = dalloc<int2>(c, meta.size());
        B.ci = dalloc<int>(c, ci.size());
        B.v = dalloc<double>(c, val.size());
        CK(cudaMemcpy(B.len, len.data(), len.size() * sizeof(int), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(B.meta, meta.data(), meta.size() * sizeof(int2), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(B.ci, ci.data(), ci.size() * sizeof(int), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(B.v, val.data(), val.size() * sizeof(double), cudaMemcpyHostToDevice));
        B.pol = (long long)(76.0 * B.nnzb) > c->opt_stream_bytes ? 1 : 0;
        return M;
    }
    std::vector<int> len((size_t)std::max<int64_t>(v.n_rows, 0), 0);
    int maxlen = 0;
    for (int64_t i = 0; i < v.n_rows; ++i) {
        len[(size_t)i] = (int)(v.row_offsets[i + 1] - v.row_offsets[i]);
        maxlen = std::max(maxlen, len[(size_t)i]);
    }
    // "fuse_rr": the restriction runs inside the residual kernel (k_resid_restrict / k_tail),
    // which walks plain CSR rows — P' then skips the sliced formats and the long-row split
    const bool plain_csr = role == 4 && c->opt_fuse_rr;
    if (!plain_csr && role >= 0 && ((c->opt_xsell >> role) & 1) && v.n_rows >= c->opt_xsell_min_rows &&
        mean <= (double)c->opt_xsell_max_mean && mean >= (double)c->opt_xsell_min_mean && build_xsell(c, v, M.xs)) {
        M.fmt = 3;
        return M;
    }
    bool sell = !plain_csr && v.n_rows >= c->opt_sell_min_rows && mean <= (double)c->opt_sell_max_mean &&
                mean >= (double)c->opt_sell_min_mean && maxlen <= c->opt_sell_max_len;
    if (sell && c->opt_sell_chh == 0 && !c->opt_sell_sort && nnz > 0) {
        // natural order only (sorted SELL loses the x-gather locality): fall back
        // to CSR when neither chunk height pads <= the limit
        std::vector<int2> m32, m8;
        long long a = 0, b = 0;
        slice_meta(len, m32, a, 32);
        slice_meta(len, m8, b, 8);
        const double lim = (double)c->opt_sell_sort_fill_pct / 100.0;
        sell = double(a) * 32.0 / double(nnz) <= lim || double(b) * 8.0 / double(nnz) <= lim;
    }
    if (sell) {
        M.fmt = 2;
        DSell& S = M.sell;
        S.n_rows = (int)v.n_rows;
        S.n_cols = (int)v.n_cols;
        S.nnz = nnz;
        S.nchunks = (S.n_rows + 31) / 32;
        // Layout choice by padded bytes, natural order preferred (x-gather locality):
        // SELL-32 natural -> SELL-8 natural -> SELL-32-sigma (rows sorted by
        // length, descending, inside windows of sigma rows).
        std::vector<int2> meta;
        long long s32 = 0, s8 = 0;
        slice_meta(len, meta, s32, 32);
        std::vector<int2> meta8;
        slice_meta(len, meta8, s8, 8);
        const double f32 = nnz ? double(s32) * 32.0 / double(nnz) : 1.0;
        const double f8 = nnz ? double(s8) * 8.0 / double(nnz) : 1.0;
        const double lim = (double)c->opt_sell_sort_fill_pct / 100.0;
        std::vector<int> perm;
        std::vector<int> slen = len;
        int h = 32;
        if (c->opt_sell_chh == 8 || (c->opt_sell_chh == 0 && f32 > lim && f8 <= lim)) {
            h = 8;
            meta.swap(meta8);
            S.slots = s8;
        } else if (c->opt_sell_chh == 0 && f32 > lim && nnz > 0) {
            const int64_t sigma = std::max<int64_t>(32, c->opt_sell_sigma);
            perm.resize((size_t)v.n_rows);
            for (int64_t i = 0; i < v.n_rows; ++i) perm[(size_t)i] = (int)i;
            for (int64_t w0 = 0; w0 < v.n_rows; w0 += sigma) {
                const int64_t w1 = std::min<int64_t>(v.n_rows, w0 + sigma);
                std::stable_sort(perm.begin() + w0, perm.begin() + w1,
                                 [&](int a, int b) { return len[(size_t)a] > len[(size_t)b]; });
            }
            for (int64_t i = 0; i < v.n_rows; ++i) slen[(size_t)i] = len[(size_t)perm[(size_t)i]];
            slice_meta(slen, meta, S.slots, 32);
        } else {
            S.slots = s32;
        }
        S.chh = h;
        // S.slots counts slot rows of h entries; store padded entries / 32 for the byte accounting
        const bool i16 = c->opt_idx16 && rows_fit_u16(v);
        const size_t nslot = (size_t)std::max<long long>(S.slots * h, 1);
        std::vector<int> ci(i16 ? 0 : nslot, 0), cb(i16 ? (size_t)std::max<int64_t>(v.n_rows, 1) : 0, 0);
        std::vector<unsigned short> c16(i16 ? nslot : 0, 0);
        std::vector<double> val(nslot, 0.0);
#pragma omp parallel for schedule(static)
        for (int64_t sr = 0; sr < v.n_rows; ++sr) {
            const int64_t i = perm.empty() ? sr : perm[(size_t)sr];
            const long long off = meta[(size_t)(sr / h)].x;
            const int r = (int)(sr % h);
            const int64_t b = v.row_offsets[i];
            const int64_t base = (i16 && v.row_offsets[i + 1] > b) ? v.col_indices[b] : 0;
            if (i16) cb[(size_t)sr] = (int)base;
            for (int64_t k = b; k < v.row_offsets[i + 1]; ++k) {
                const long long j = k - b;
                if (i16) c16[(size_t)((off + j) * h + r)] = (unsigned short)(v.col_indices[k] - base);
                else ci[(size_t)((off + j) * h + r)] = (int)v.col_indices[k];
                val[(size_t)((off + j) * h + r)] = v.values[k];
            }
        }
        S.slots = (S.slots * h + 31) / 32;  // padded entries / 32 (byte accounting, as for SELL-32)
        S.len = dalloc<int>(c, slen.size());
        S.meta = dalloc<int2>(c, meta.size());
        S.v = dalloc<double>(c, val.size());
        CK(cudaMemcpy(S.len, slen.data(), slen.size() * sizeof(int), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(S.meta, meta.data(), meta.size() * sizeof(int2), cudaMemcpyHostToDevice));
        if (i16) {
            S.ci16 = dalloc<unsigned short>(c, c16.size());
            S.cb = dalloc<int>(c, cb.size());
            CK(cudaMemcpy(S.ci16, c16.data(), c16.size() * sizeof(unsigned short), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(S.cb, cb.data(), cb.size() * sizeof(int), cudaMemcpyHostToDevice));
        } else {
            S.ci = dalloc<int>(c, ci.size());
            CK(cudaMemcpy(S.ci, ci.data(), ci.size() * sizeof(int), cudaMemcpyHostToDevice));
        }
        CK(cudaMemcpy(S.v, val.data(), val.size() * sizeof(double), cudaMemcpyHostToDevice));
        if (!perm.empty()) {
            S.perm = dalloc<int>(c, perm.size());
            CK(cudaMemcpy(S.perm, perm.data(), perm.size() * sizeof(int), cudaMemcpyHostToDevice));
        }
        S.pol = (long long)(12.0 * nnz) > c->opt_stream_bytes ? 1 : 0;
        // U*10 + min CTAs/SM. Large operators: U = 4 at 4 CTAs/SM (64 registers) keeps more
        // warps in flight (C2 level-0 G: 35 vs 40 us); smaller ones keep U = 8 (tools/tune_kernels.py)
        S.u = c->opt_sell_u > 0 ? (int)c->opt_sell_u : (maxlen <= 4 ? 41 : v.n_rows >= 400000 ? 44 : 83);
        return M;
    }
    M.fmt = 0;
    DCsr& A = M.csr;
    A.n_rows = (int)v.n_rows;
    A.n_cols = (int)v.n_cols;
    A.nnz = nnz;
    A.group = group_for(mean, maxlen, v.n_rows, (double)c->opt_csr_per_thread,
                        (int)std::clamp<long long>(c->opt_csr_max_group, 1, 256));
    A.pf = (int)c->opt_csr_pf;
    if (c->opt_csr_long > 0 && A.group <= 16 && !plain_csr) {
        const int thr = (int)c->opt_csr_long * A.group * 4;
        std::vector<int> lr;
        for (int64_t i = 0; i < v.n_rows; ++i)
            if (len[(size_t)i] > thr) lr.push_back((int)i);
        if (!lr.empty()) {
            A.nlong = (int)lr.size();
            A.lthr = thr;
            A.nlctas = (int)std::min<int64_t>((lr.size() + kBlock / 32 - 1) / (kBlock / 32), 296);
            A.lrows = dalloc<int>(c, lr.size());
            CK(cudaMemcpy(A.lrows, lr.data(), lr.size() * sizeof(int), cudaMemcpyHostToDevice));
        }
    }
    // 16-bit offsets pay off for short rows (few threads per row, index bytes a
    // larger share of the per-thread stream); long-row operands (group >= 32)
    // measured slower with them (tools/tune_kernels.py, profiles/README.md).
    const bool i16 = c->opt_idx16 && A.group <= c->opt_idx16_max_group && rows_fit_u16(v);
    const int64_t nbase = v.n_rows;
    std::vector<int> rp((size_t)v.n_rows + 1), ci(i16 ? 0 : (size_t)nnz), cb(i16 ? (size_t)std::max<int64_t>(nbase, 1) : 0);
    std::vector<unsigned short> c16(i16 ? (size_t)nnz : 0);
    for (int64_t i = 0; i <= v.n_rows; ++i) rp[(size_t)i] = (int)(v.n_rows ? v.row_offsets[i] : 0);
    if (i16) {
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < v.n_rows; ++i) {
            const int64_t b = v.row_offsets[i], e = v.row_offsets[i + 1];
            const int64_t base = e > b ? v.col_indices[b] : 0;
            cb[(size_t)i] = (int)base;
            for (int64_t k = b; k < e; ++k) c16[(size_t)k] = (unsigned short)(v.col_indices[k] - base);
        }
    } else {
#pragma omp parallel for schedule(static)
        for (int64_t k = 0; k < nnz; ++k) ci[(size_t)k] = (int)v.col_indices[k];
    }
    A.rp = dalloc<int>(c, rp.size());
    A.v = dalloc<double>(c, (size_t)nnz);
    CK(cudaMemcpy(A.rp, rp.data(), rp.size() * sizeof(int), cudaMemcpyHostToDevice));
    if (i16) {
        A.ci16 = dalloc<unsigned short>(c, std::max<size_t>(c16.size(), 1));
        A.cb = dalloc<int>(c, cb.size());
        if (nnz) CK(cudaMemcpy(A.ci16, c16.data(), c16.size() * sizeof(unsigned short), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(A.cb, cb.data(), cb.size() * sizeof(int), cudaMemcpyHostToDevice));
    } else {
        A.ci = dalloc<int>(c, std::max<size_t>(ci.size(), 1));
        if (nnz) CK(cudaMemcpy(A.ci, ci.data(), ci.size() * sizeof(int), cudaMemcpyHostToDevice));
    }
    if (nnz) CK(cudaMemcpy(A.v, v.values, (size_t)nnz * sizeof(double), cudaMemcpyHostToDevice));
    A.pol = (long long)(12.0 * nnz) > c->opt_stream_bytes ? 1 : 0;
    // warp-per-row operands run the column-pipelined kernel (k_csrw)
    if (c->opt_csrw > 0 && A.group == 32 && !i16 && !A.nlong && !plain_csr) {
        A.wu = c->opt_csrw >= 8 ? 8 : 4;
        if (A.pol == 1 && c->opt_csr_noalloc) A.pol = 3;  // streamed operand: matrix loads bypass L1
        A.blk = (c->opt_csr_blocked > 0 && v.n_rows >= c->opt_csr_blocked) ? 1 : 0;
    }
    return M;
}

// Device bytes of an operand's matrix stream (what one product reads).
double mat_bytes(const DMat& M) {
    if (M.fmt == 3)  // padded quads are predicated off: ~10 B per entry + per-row and per-tile metadata
        return 10.0 * double(M.xs.nnz) + 4.0 * double(M.xs.ntiles) * M.xs.R + 4.0 * double(M.xs.list_len) +
               8.0 * double(M.xs.ntiles) * (1 + M.xs.R / 32);
    if (M.fmt == 1) return 76.0 * 32.0 * double(M.sb.slots) + 4.0 * M.sb.nb;
    if (M.fmt == 2) return (M.sell.ci16 ? 10.0 : 12.0) * 32.0 * double(M.sell.slots) + (M.sell.ci16 ? 8.0 : 4.0) * M.sell.n_rows;
    const double nb = double(M.csr.n_rows);
    return (M.csr.ci16 ? 10.0 : 12.0) * double(M.csr.nnz) + 4.0 * (M.csr.n_rows + 1) + (M.csr.ci16 ? 4.0 * nb : 0.0);
}
void set_pol(DMat& M, int pol) {
    if (M.fmt == 1) M.sb.pol = pol;
    else if (M.fmt == 3) M.xs.pol = pol;
    else if (M.fmt == 2) M.sell.pol = pol;
    else M.csr.pol = pol;
}

// Stored (padded) entries / true nnz of an operand.
double fill_ratio(const DMat& M) {
    if (M.fmt == 3) return M.xs.nnz ? double(M.xs.quads) * 128.0 / double(M.xs.nnz) : 1.0;
    if (M.fmt == 1) return M.sb.nnzb ? double(M.sb.slots) * 32.0 / double(M.sb.nnzb) : 1.0;
    if (M.fmt == 2) return M.sell.nnz ? double(M.sell.slots) * 32.0 / double(M.sell.nnz) : 1.0;
    return 1.0;
}

// Algorithmic bytes of one product y = M x: matrix arrays
// once, x once, y once; padding never counted.
double alg_bytes(const DMat& M) {
    if (M.fmt == 1) {
        const double nnzb = double(M.sb.nnzb);
        return 72.0 * nnzb + 4.0 * nnzb + 4.0 * (M.sb.nb + 1) + 8.0 * M.cols() + 8.0 * M.rows();
    }
    if (M.fmt == 3) {
        // values + 16-bit local columns, per-row length + position (2 x 2 B), the footprint lists, x and y once
        const double nnz = double(M.xs.nnz);
        return 8.0 * nnz + 2.0 * nnz + 4.0 * M.rows() + 4.0 * double(M.xs.list_len) + 8.0 * M.cols() + 8.0 * M.rows();
    }
    const double nnz = double(M.fmt == 2 ? M.sell.nnz : M.csr.nnz);
    const bool i16 = M.fmt == 2 ? M.sell.ci16 != nullptr : M.csr.ci16 != nullptr;
    // 16-bit offsets: 2 B per entry + a 4-B base column per row
    const double nb = double(M.rows());
    const double idx = i16 ? 2.0 * nnz + 4.0 * nb : 4.0 * nnz;
    return 8.0 * nnz + idx + 4.0 * (M.rows() + 1) + 8.0 * M.cols() + 8.0 * M.rows();
}

std::string fmt_name(const DMat& M) {
    const bool h = M.fmt == 2 ? M.sell.ci16 != nullptr : M.fmt == 0 && M.csr.ci16 != nullptr;
    if (M.fmt == 3) return "xsell" + std::to_string(M.xs.R) + (M.xs.fold == 2 ? "f" : "");
    const std::string base = M.fmt == 1   ? "sbsr3"
                             : M.fmt == 2 ? (M.sell.perm ? "sells" : M.sell.chh == 8 ? "sell8" : "sell")
                                          : (M.csr.wu ? "csrw" + std::to_string(M.csr.wu) : "csr" + std::to_string(M.csr.group));
    return h ? base + "h" : base;  // h: 16-bit column offsets
}

void add_spmv(aspamg_gpu_ctx* c, std::vector<Op>& ops, const std::string& name, int level, const DMat& M, Epi epi,
              const double* x, double* y, const double* aux, double omega, const double* dotw, int fin,
              double* out, const int* done) {
    const int grid = spmv_grid(M);
    Red red;
    if (fin != FIN_NONE) red = make_red(c, grid, fin, out);
    double bytes = alg_bytes(M);
    if (aux) bytes += 8.0 * M.rows();
    if (dotw) bytes += 8.0 * M.rows();
    const DMat Mc = M;
    ops.push_back({name + "." + fmt_name(M), level, bytes, [=](cudaStream_t s) {
                       Launch L{grid, s};
                       spmv(Mc, epi, x, y, aux, omega, dotw, red, done, L);
                   }});
    if (M.fmt == 0 && !M.csr.nlong && fin == FIN_NONE && !dotw) {
        Op& o = ops.back();
        o.describable = true;
        o.desc.kind = 0;
        o.desc.epi = epi;
        o.desc.M = M.csr;
        o.desc.x = x;
        o.desc.y = y;
        o.desc.aux = aux;
        o.desc.omega = omega;
        o.desc.n = M.rows();
    }
}

// V-cycle ops at level k: input y, output z (z doubles as the s accumulator).
// dotw0/fin0: the dot fused into the last op that writes the level-0 output.
void build_vcycle(aspamg_gpu_ctx* c, std::vector<Op>& ops, int k, const double* y, double* z, const double* dotw0,
                  int fin0, const int* done, bool allow_tail = true);

// Levels k.. (all smaller than tail_rows) as one persistent cooperative kernel.
bool build_tail(aspamg_gpu_ctx* c, std::vector<Op>& ops, int k, const double* y, double* z, const int* done) {
    std::vector<Op> sub;
    build_vcycle(c, sub, k, y, z, nullptr, FIN_NONE, done, false);
    for (const Op& o : sub)
        if (!o.describable) return false;
    std::vector<TailOp> d;
    double bytes = 0.0;
    for (const Op& o : sub) {
        d.push_back(o.desc);
        bytes += o.bytes;
    }
    TailOp* dd = dalloc<TailOp>(c, d.size());
    CK(cudaMemcpy(dd, d.data(), d.size() * sizeof(TailOp), cudaMemcpyHostToDevice));
    GridBar* bar = dalloc<GridBar>(c, 1);
    CK(cudaMemset(bar, 0, sizeof(GridBar)));
    const int grid = tail_grid();
    const int nops = (int)d.size();
    ops.push_back({"tail" + std::to_string(nops), k, bytes, [=](cudaStream_t s) { tail_run(dd, nops, bar, done, grid, s); }});
    return true;
}

// "fuse_rr": r = y - A s and r_c = P' r of level k as ONE cooperative launch (grid
// barrier between the two phases, r read back through L2). Level 0 with the sliced
// BSR3 K uses k_resid_restrict; levels whose A and P' are both plain CSR use the
// op-table kernel with two ops. Returns false when the level's formats do not fit.
bool add_resid_restrict(aspamg_gpu_ctx* c, std::vector<Op>& ops, int k, const double* s, const double* y, double* yc,
                        const int* done) {
    GLevel& l = c->lv[(size_t)k];
    if (l.Pt.fmt != 0 || l.Pt.csr.nlong) return false;
    TailOp pt{};
    pt.kind = 0;
    pt.epi = EPI_PLAIN;
    pt.M = l.Pt.csr;
    pt.x = l.r;
    pt.y = yc;
    pt.omega = 1.0;
    pt.n = l.Pt.rows();
    const double bytes = alg_bytes(l.A) + 8.0 * l.n + alg_bytes(l.Pt);
    double* r = l.r;
    if (l.A.fmt == 1) {
        GridBar* bar = dalloc<GridBar>(c, 1);
        CK(cudaMemset(bar, 0, sizeof(GridBar)));
        const DSbsr3 A = l.A.sb;
        const int grid = resid_restrict_grid(A.pol);
        ops.push_back({"resid_restrict.sbsr3+" + fmt_name(l.Pt), k, bytes,
                       [=](cudaStream_t st) { resid_restrict(A, pt, s, r, y, bar, done, grid, st); }});
        return true;
    }
    if (l.A.fmt != 0 || l.A.csr.nlong) return false;
    TailOp d[2] = {};
    d[0].kind = 0;
    d[0].epi = EPI_RESID;
    d[0].M = l.A.csr;
    d[0].x = s;
    d[0].y = r;
    d[0].aux = y;
    d[0].omega = 1.0;
    d[0].n = l.n;
    d[1] = pt;
    TailOp* dd = dalloc<TailOp>(c, 2);
    CK(cudaMemcpy(dd, d, sizeof(d), cudaMemcpyHostToDevice));
    GridBar* bar = dalloc<GridBar>(c, 1);
    CK(cudaMemset(bar, 0, sizeof(GridBar)));
    const int grid = tail_grid();
    ops.push_back({"resid_restrict." + fmt_name(l.A) + "+" + fmt_name(l.Pt), k, bytes,
                   [=](cudaStream_t st) { tail_run(dd, 2, bar, done, grid, st); }});
    return true;
}

void build_vcycle(aspamg_gpu_ctx* c, std::vector<Op>& ops, int k, const double* y, double* z, const double* dotw0,
                  int fin0, const int* done, bool allow_tail) {
    const int L = (int)c->lv.size();
    const bool top = k == 0;
    if (allow_tail && k >= 1 && c->lv[(size_t)k].n <= c->opt_tail_rows && build_tail(c, ops, k, y, z, done)) return;
    if (allow_tail && k >= 1 && k == c->tail_level) {  // collapsed coarse tail: z = T y
        add_spmv(c, ops, "tail_dense", k, c->Tm, EPI_PLAIN, y, z, nullptr, 1.0, nullptr, FIN_NONE, nullptr, done);
        return;
    }
    if (k == L - 1) {  // coarsest: forward/backward solve
        Red red;
        const int n = c->n_c;
        const double* dw = top ? dotw0 : nullptr;
        if (c->opt_coarse_mode == 1) {
            add_spmv(c, ops, "coarse_fwd", k, c->Wm, EPI_PLAIN, y, c->cw, nullptr, 1.0, nullptr, FIN_NONE, nullptr, done);
            add_spmv(c, ops, "coarse_bwd", k, c->Wtm, EPI_PLAIN, c->cw, z, nullptr, 1.0, dw, top ? fin0 : FIN_NONE,
                     nullptr, done);
            return;
        }
        if (top && fin0 != FIN_NONE) red = make_red(c, 1, fin0);
        const double *Lrm = c->Lrm, *Lcm = c->Lcm, *Df = c->Dinv_f, *Db = c->Dinv_b;
        const double bytes = 2.0 * (8.0 * double(n) * (n + 1) / 2 + 16.0 * n);
        ops.push_back({"coarse_solve", k, bytes, [=](cudaStream_t s) {
                           Launch Lc{1, s};
                           coarse_solve(n, Lrm, Lcm, Df, Db, y, z, dw, red, done, Lc);
                       }});
        return;
    }
    GLevel& l = c->lv[(size_t)k];
    const int n = l.n;
    double* s = z;
    const GLevel& nx = c->lv[(size_t)k + 1];
    double* yc = nx.y;
    double* zc = nx.z;
    // pre-smoothing from s = 0
    for (int it = 0; it < c->nu1; ++it) {
        if (it == 0) {
            add_spmv(c, ops, "smooth_G", k, l.G, EPI_PLAIN, y, l.t, nullptr, 1.0, nullptr, FIN_NONE, nullptr, done);
            add_spmv(c, ops, "smooth_Gt", k, l.Gt, EPI_SCALE, l.t, s, nullptr, l.omega, nullptr, FIN_NONE, nullptr, done);
        } else {
            add_spmv(c, ops, "resid_A", k, l.A, EPI_RESID, s, l.r, y, 1.0, nullptr, FIN_NONE, nullptr, done);
            add_spmv(c, ops, "smooth_G", k, l.G, EPI_PLAIN, l.r, l.t, nullptr, 1.0, nullptr, FIN_NONE, nullptr, done);
            add_spmv(c, ops, "smooth_Gt", k, l.Gt, EPI_ADDSCALE, l.t, s, s, l.omega, nullptr, FIN_NONE, nullptr, done);
        }
    }
    if (c->nu1 == 0) {
        const int g = vec_grid(n);
        ops.push_back({"zero", k, 8.0 * n, [=](cudaStream_t st) { fill_zero(n, s, done, Launch{g, st}); }});
        ops.back().describable = true;
        ops.back().desc.kind = 1;
        ops.back().desc.y = s;
        ops.back().desc.n = n;
    }
    // r = y - A s ; r_c = P' r
    if (!(c->opt_fuse_rr && add_resid_restrict(c, ops, k, s, y, yc, done))) {
        add_spmv(c, ops, "resid_A", k, l.A, EPI_RESID, s, l.r, y, 1.0, nullptr, FIN_NONE, nullptr, done);
        add_spmv(c, ops, "restrict_Pt", k, l.Pt, EPI_PLAIN, l.r, yc, nullptr, 1.0, nullptr, FIN_NONE, nullptr, done);
    }
    build_vcycle(c, ops, k + 1, yc, zc, dotw0, fin0, done, allow_tail);
    // s += P e_c
    const bool last_is_prolong = c->nu2 == 0;
    add_spmv(c, ops, "prolong_P", k, l.P, EPI_ADD, zc, s, s, 1.0, (top && last_is_prolong) ? dotw0 : nullptr,
             (top && last_is_prolong) ? fin0 : FIN_NONE, nullptr, done);
    for (int it = 0; it < c->nu2; ++it) {
        const bool last = top && it == c->nu2 - 1;
        add_spmv(c, ops, "resid_A", k, l.A, EPI_RESID, s, l.r, y, 1.0, nullptr, FIN_NONE, nullptr, done);
        add_spmv(c, ops, "smooth_G", k, l.G, EPI_PLAIN, l.r, l.t, nullptr, 1.0, nullptr, FIN_NONE, nullptr, done);
        add_spmv(c, ops, "smooth_Gt", k, l.Gt, EPI_ADDSCALE, l.t, s, s, l.omega, last ? dotw0 : nullptr,
                 last ? fin0 : FIN_NONE, nullptr, done);
    }
}

void run_ops(const std::vector<Op>& ops, cudaStream_t s) {
    for (const auto& o : ops) o.fn(s);
}

void ensure_ready(aspamg_gpu_ctx* c) {
    if (!c) throw Fail{4, "null context"};
    if (!c->finalized) throw Fail{4, "context not finalized (upload levels + coarse factor, then finalize)"};
}

cudaGraph_t capture(aspamg_gpu_ctx* c, const std::vector<Op>& ops) {
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    run_ops(ops, c->stream);
    cudaGraph_t g = nullptr;
    const cudaError_t le = cudaGetLastError();
    const cudaError_t ce = cudaStreamEndCapture(c->stream, &g);  // always leave capture mode
    CK(le);
    CK(ce);
    return g;
}

void build_graphs(aspamg_gpu_ctx* c) {
    c->vc_graph = capture(c, c->vc_ops);  // standalone V-cycle
    CK(cudaGraphInstantiate(&c->vc_exec, c->vc_graph, 0));
    c->body_graph = capture(c, c->body);  // PCG body (host-loop fallback)
    CK(cudaGraphInstantiate(&c->body_exec, c->body_graph, 0));
}

// Device-side loop: parent graph = WHILE(cond) { body }; the last kernel of the
// body (pcg_xr) sets the condition from the convergence test.
void build_device_loop(aspamg_gpu_ctx* c) {
    CK(cudaGraphCreate(&c->pcg_graph, 0));
    cudaGraphConditionalHandle handle;
    CK(cudaGraphConditionalHandleCreate(&handle, c->pcg_graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = handle;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    CK(cudaGraphAddNode(&node, c->pcg_graph, nullptr, 0, &cp));
    cudaGraph_t bodyg = cp.conditional.phGraph_out[0];
    // rebuild the body op list with the condition handle wired into pcg_xr
    const std::vector<Op>& body = c->body;
    // pcg_xr with the conditional: its reduction site is allocated before capture
    const int n = c->lv[0].n;
    const int g = vec_grid(n);
    Red red = make_red(c, g, FIN_RR);
    red.cond = handle;
    red.use_cond = 1;
    CK(cudaStreamBeginCaptureToGraph(c->stream, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    for (size_t i = 0; i + 1 < body.size(); ++i) body[i].fn(c->stream);
    pcg_xr(n, c->x, c->r, c->p, c->q, red, &c->st->done, Launch{g, c->stream});
    cudaGraph_t out;
    const cudaError_t le = cudaGetLastError();
    const cudaError_t ce = cudaStreamEndCapture(c->stream, &out);
    CK(le);
    CK(ce);
    CK(cudaGraphInstantiate(&c->pcg_exec, c->pcg_graph, 0));
}

// Collapsed coarse tail: B_k, the V-cycle restricted to levels k..L-1, is a
// fixed linear map (SPEC.md:445-453 with fixed G, P, omega and coarse factor).
// Its matrix is formed on the device column by column — the sub-cycle's own
// kernels applied to the unit vectors e_j — and stored as a dense CSR operand,
// so the whole tail becomes one L2-resident product per V-cycle. Exact up to
// rounding (different summation order), checked by the V-cycle/PCG parity tests.
void build_dense_tail(aspamg_gpu_ctx* c) {
    const int L = (int)c->lv.size();
    int k = -1;
    for (int q = 1; q < L; ++q)
        if (c->lv[(size_t)q].n <= c->opt_tail_dense) { k = q; break; }
    if (k < 0 || k == L - 1) return;  // nothing to collapse (the coarsest alone is already one solve)
    const int n = c->lv[(size_t)k].n;
    double* y = c->lv[(size_t)k].y;
    double* z = c->lv[(size_t)k].z;
    std::vector<Op> sub;
    build_vcycle(c, sub, k, y, z, nullptr, FIN_NONE, nullptr, false);
    double* dM = dalloc<double>(c, (size_t)n * n);
    const double one = 1.0;
    for (int j = 0; j < n; ++j) {
        CK(cudaMemsetAsync(y, 0, (size_t)n * sizeof(double), c->stream));
        CK(cudaMemcpyAsync(y + j, &one, sizeof(double), cudaMemcpyHostToDevice, c->stream));
        run_ops(sub, c->stream);
        // column j of the row-major matrix: M[i][j] = z_i
        CK(cudaMemcpy2DAsync(dM + j, (size_t)n * sizeof(double), z, sizeof(double), sizeof(double), (size_t)n,
                             cudaMemcpyDeviceToDevice, c->stream));
    }
    CK(cudaGetLastError());
    std::vector<double> M((size_t)n * n);
    CK(cudaMemcpyAsync(M.data(), dM, M.size() * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    std::vector<int64_t> rp((size_t)n + 1), ci((size_t)n * n);
    for (int i = 0; i <= n; ++i) rp[(size_t)i] = (int64_t)i * n;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) ci[(size_t)i * n + j] = j;
    aspamg_csr_view v{};
    v.n_rows = n;
    v.n_cols = n;
    v.nnz = (int64_t)n * n;
    v.row_offsets = rp.data();
    v.col_indices = ci.data();
    v.values = M.data();
    c->Tm = upload_mat(c, v, false);
    set_pol(c->Tm, 2);
    c->tail_level = k;
}

void do_finalize(aspamg_gpu_ctx* c) {
    if ((int)c->lv.size() < 1) throw Fail{4, "finalize: no levels uploaded"};
    if (!c->coarse_uploaded) throw Fail{4, "finalize: coarse factor not uploaded"};
    const int L = (int)c->lv.size();
    if (c->lv.back().n != c->n_c) throw Fail{1, "finalize: coarse factor size does not match the last level"};
    for (int k = 0; k + 1 < L; ++k) {
        GLevel& l = c->lv[(size_t)k];
        if (!l.has_smoother) throw Fail{4, "finalize: level " + std::to_string(k) + " lacks G/P"};
        if (l.P.cols() != c->lv[(size_t)k + 1].n) throw Fail{1, "finalize: P columns != next level size"};
    }
    const int n0 = c->lv[0].n;
    c->st = dalloc<PcgState>(c, 1);
    CK(cudaMemset(c->st, 0, sizeof(PcgState)));
    CK(cudaMallocHost(&c->st_host, sizeof(PcgState)));
    c->zero_flag = dalloc<int>(c, 1);
    CK(cudaMemset(c->zero_flag, 0, sizeof(int)));
    c->b = dalloc<double>(c, n0);
    c->x = dalloc<double>(c, n0);
    c->r = dalloc<double>(c, n0);
    c->z = dalloc<double>(c, n0);
    c->p = dalloc<double>(c, n0);
    c->q = dalloc<double>(c, n0);
    c->vy = dalloc<double>(c, n0);
    c->vz = dalloc<double>(c, n0);
    for (int k = 0; k < L; ++k) {
        GLevel& l = c->lv[(size_t)k];
        if (k > 0) {
            l.y = dalloc<double>(c, l.n);
            l.z = dalloc<double>(c, l.n);
        }
        if (k + 1 < L) {
            l.r = dalloc<double>(c, l.n);
            l.t = dalloc<double>(c, l.n);
        }
    }
    // L2 policy: the coarsest levels (bottom-up, up to keep_bytes) are loaded
    // with evict-last so they stay L2-resident across V-cycles; everything
    // bigger than stream_bytes streams with evict-first.
    {
        double kept = mat_bytes(c->Wm) + mat_bytes(c->Wtm);
        set_pol(c->Wm, 2);
        set_pol(c->Wtm, 2);
        for (int k = L - 1; k >= 0; --k) {
            GLevel& l = c->lv[(size_t)k];
            DMat* ms[5] = {&l.A, &l.G, &l.Gt, &l.P, &l.Pt};
            double b = 0.0;
            for (int i = 0; i < 5; ++i)
                if (i == 0 || l.has_smoother) b += mat_bytes(*ms[i]);
            if (kept + b > (double)c->opt_keep_bytes) break;
            kept += b;
            for (int i = 0; i < 5; ++i)
                if (i == 0 || l.has_smoother) set_pol(*ms[i], 2);
        }
    }
    if (c->opt_tail_dense > 0) build_dense_tail(c);
    const int* done = &c->st->done;
    // standalone V-cycle: vy -> vz
    build_vcycle(c, c->vc_ops, 0, c->vy, c->vz, nullptr, FIN_NONE, c->zero_flag);
    // PCG loop body
    build_vcycle(c, c->body, 0, c->r, c->z, c->r, FIN_RZ, done);
    {
        const int g = vec_grid(n0);
        double *z = c->z, *p = c->p;
        const PcgState* st = c->st;
        c->body.push_back({"pcg_p", 0, 24.0 * n0, [=](cudaStream_t s) { pcg_p(n0, z, p, st, done, Launch{g, s}); }});
    }
    add_spmv(c, c->body, "pcg_Kp", 0, c->lv[0].A, EPI_PLAIN, c->p, c->q, nullptr, 1.0, c->p, FIN_PQ, nullptr, done);
    {
        const int g = vec_grid(n0);
        Red red = make_red(c, g, FIN_RR);
        double *x = c->x, *r = c->r, *p = c->p, *q = c->q;
        c->body.push_back({"pcg_xr", 0, 48.0 * n0, [=](cudaStream_t s) { pcg_xr(n0, x, r, p, q, red, done, Launch{g, s}); }});
    }
    // init: x0 given -> r = b - A x ; then dots b.b, r.r
    add_spmv(c, c->init1, "init_resid", 0, c->lv[0].A, EPI_RESID, c->x, c->r, c->b, 1.0, nullptr, FIN_NONE, nullptr,
             nullptr);
    {
        const int g = vec_grid(n0);
        Red red = make_red(c, g, FIN_INIT);
        double *b = c->b, *r = c->r;
        c->init0.push_back({"init_dots", 0, 16.0 * n0, [=](cudaStream_t s) { pcg_init_dots(n0, b, r, red, Launch{g, s}); }});
    }
    // post: true residual q = b - A x, ||q||^2 -> st->trr2
    add_spmv(c, c->post, "true_resid", 0, c->lv[0].A, EPI_RESID, c->x, c->q, c->b, 1.0, c->q, FIN_STORE,
             &c->st->trr2, nullptr);
    build_graphs(c);
    if (c->opt_device_loop) {
        try {
            build_device_loop(c);
        } catch (const CudaFail& e) {
            std::fprintf(stderr, "aspamg_gpu: device-side loop unavailable (%s); using host loop\n", e.msg.c_str());
            cudaGetLastError();
            c->opt_device_loop = 0;
        }
    }
    CK(cudaEventCreate(&c->ev0));
    CK(cudaEventCreate(&c->ev1));
    CK(cudaStreamSynchronize(c->stream));
    c->finalized = true;
}

// Core device PCG: b, x0 already in c->b / c->x (if has_x0). Returns status.
int run_pcg(aspamg_gpu_ctx* c, bool has_x0, double rel_tol, long long max_it, long long* n_it, int* converged,
            double* trr) {
    if (!(rel_tol >= 0.0)) throw Fail{4, "pcg: rel_tol must be >= 0"};
    if (max_it < 0) throw Fail{4, "pcg: max_it must be >= 0"};
    const int n0 = c->lv[0].n;
    if (max_it + 1 > c->hist_cap) {
        if (c->hist) cudaFree(c->hist);
        c->hist_cap = std::max<long long>(max_it + 1, 1024);
        CK(cudaMalloc(&c->hist, (size_t)c->hist_cap * sizeof(double)));
    }
    PcgState h = {};
    h.tol = rel_tol;
    h.max_it = max_it;
    h.history = c->hist;
    *c->st_host = h;
    cudaStream_t s = c->stream;
    long long launches = 0;
    CK(cudaEventRecord(c->ev0, s));
    CK(cudaMemcpyAsync(c->st, c->st_host, sizeof(PcgState), cudaMemcpyHostToDevice, s));
    if (has_x0) {
        run_ops(c->init1, s);
        launches += (long long)c->init1.size();
    } else {
        CK(cudaMemsetAsync(c->x, 0, (size_t)n0 * sizeof(double), s));
        CK(cudaMemcpyAsync(c->r, c->b, (size_t)n0 * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
    run_ops(c->init0, s);
    launches += (long long)c->init0.size();
    if (c->opt_device_loop && c->pcg_exec) {
        CK(cudaGraphLaunch(c->pcg_exec, s));
    } else {
        // host loop: launch the body graph in batches, poll the done flag
        long long it = 0;
        CK(cudaMemcpyAsync(c->st_host, c->st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        while (!c->st_host->done && it < max_it) {
            const long long batch = std::min<long long>(4, max_it - it);
            for (long long j = 0; j < batch; ++j) CK(cudaGraphLaunch(c->body_exec, s));
            it += batch;
            CK(cudaMemcpyAsync(c->st_host, c->st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
        }
    }
    CK(cudaEventRecord(c->ev1, s));
    run_ops(c->post, s);
    launches += (long long)c->post.size();
    CK(cudaMemcpyAsync(c->st_host, c->st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
    c->last_ms = ms;
    const PcgState& st = *c->st_host;
    // kernels that ran: every body op per iteration (plus the final body when already converged)
    launches += (long long)c->body.size() * std::max<long long>(st.k, st.max_it > 0 ? 1 : 0);
    c->last_launches = launches;
    *n_it = st.k;
    *converged = st.converged;
    if (st.bnorm == 0.0) {
        CK(cudaMemsetAsync(c->x, 0, (size_t)n0 * sizeof(double), s));
        CK(cudaStreamSynchronize(s));
        *trr = 0.0;
        *converged = 1;
        return 0;
    }
    *trr = std::sqrt(st.trr2) / st.bnorm;
    if (*converged && !(*trr <= 10.0 * rel_tol)) *converged = 0;
    if (st.notspd) throw Fail{2, "pcg: operator not SPD (p'Ap <= 0)"};
    return *converged ? 0 : 6;
}

}  // namespace

extern "C" {

const char* aspamg_gpu_last_error(const aspamg_gpu_ctx* c) { return c ? c->err.c_str() : g_last_err.c_str(); }

int aspamg_gpu_device_count(int* n) {
    return guard(nullptr, [&] {
        int d = 0;
        cudaError_t e = cudaGetDeviceCount(&d);
        if (e != cudaSuccess) {
            cudaGetLastError();
            d = 0;
        }
        *n = d;
    });
}

int aspamg_gpu_ctx_create(int device, aspamg_gpu_ctx** out) {
    return guard(nullptr, [&] {
        int nd = 0;
        if (cudaGetDeviceCount(&nd) != cudaSuccess || nd == 0) {
            cudaGetLastError();
            throw Fail{5, "no CUDA device: the B200 solve path has no CPU fallback"};
        }
        if (device < 0 || device >= nd) throw Fail{4, "invalid device index"};
        CK(cudaSetDevice(device));
        spmv_prepare();
        auto* c = new aspamg_gpu_ctx;
        c->device = device;
        cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) {
            delete c;
            throw CudaFail{std::string("cudaStreamCreate: ") + cudaGetErrorString(e)};
        }
        *out = c;
    });
}

int aspamg_gpu_ctx_destroy(aspamg_gpu_ctx* c) {
    if (!c) return 0;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->pcg_exec) cudaGraphExecDestroy(c->pcg_exec);
    if (c->body_exec) cudaGraphExecDestroy(c->body_exec);
    if (c->vc_exec) cudaGraphExecDestroy(c->vc_exec);
    if (c->pcg_graph) cudaGraphDestroy(c->pcg_graph);
    if (c->body_graph) cudaGraphDestroy(c->body_graph);
    if (c->vc_graph) cudaGraphDestroy(c->vc_graph);
    for (void* p : c->allocs) cudaFree(p);
    if (c->hist) cudaFree(c->hist);
    if (c->st_host) cudaFreeHost(c->st_host);
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
    return 0;
}

int aspamg_gpu_set_option(aspamg_gpu_ctx* c, const char* key, int64_t value) {
    return guard(c, [&] {
        if (!c || !key) throw Fail{4, "set_option: null argument"};
        if (c->finalized) throw Fail{4, "set_option: context already finalized"};
        const std::string k(key);
        if (k == "bsr") c->opt_bsr = (int)value;
        else if (k == "device_loop") c->opt_device_loop = (int)value;
        else if (k == "stream_bytes") c->opt_stream_bytes = value;
        else if (k == "keep_bytes") c->opt_keep_bytes = value;
        else if (k == "tail_rows") c->opt_tail_rows = value;
        else if (k == "csr_per_thread") c->opt_csr_per_thread = std::max<int64_t>(1, value);
        else if (k == "idx16") c->opt_idx16 = value;
        else if (k == "csr_pf") c->opt_csr_pf = value;
        else if (k == "csr_long") c->opt_csr_long = value;
        else if (k == "csr_max_group") c->opt_csr_max_group = value;
        else if (k == "csrw") c->opt_csrw = value;
        else if (k == "csr_noalloc") c->opt_csr_noalloc = value;
        else if (k == "csr_blocked") c->opt_csr_blocked = value;
        else if (k == "tail_dense") c->opt_tail_dense = value;
        else if (k == "idx16_max_group") c->opt_idx16_max_group = value;
        else if (k == "sell_max_mean") c->opt_sell_max_mean = value;
        else if (k == "sell_max_len") c->opt_sell_max_len = value;
        else if (k == "sell_min_rows") c->opt_sell_min_rows = value;
        else if (k == "sell_sigma") c->opt_sell_sigma = value;
        else if (k == "sell_sort_fill_pct") c->opt_sell_sort_fill_pct = value;
        else if (k == "sell_u") c->opt_sell_u = value;
        else if (k == "sell_chh") c->opt_sell_chh = value;
        else if (k == "sell_sort") c->opt_sell_sort = value;
        else if (k == "sell_min_mean") c->opt_sell_min_mean = value;
        else if (k == "xsell") c->opt_xsell = value;
        else if (k == "xsell_min_rows") c->opt_xsell_min_rows = value;
        else if (k == "xsell_max_mean") c->opt_xsell_max_mean = value;
        else if (k == "xsell_min_mean") c->opt_xsell_min_mean = value;
        else if (k == "xsell_rows") c->opt_xsell_rows = value;
        else if (k == "xsell_fold") c->opt_xsell_fold = value;
        else if (k == "xsell_rows256") c->opt_xsell_rows256 = value;
        else if (k == "xsell_rows128") c->opt_xsell_rows128 = value;
        else if (k == "xsell_gran") c->opt_xsell_gran = value;
        else if (k == "xsell_q") c->opt_xsell_q = value;
        else if (k == "xsell_smem_kb") c->opt_xsell_smem_kb = value;
        else if (k == "fuse_rr") c->opt_fuse_rr = value;
        else if (k == "pdl") set_pdl(value != 0);
        else if (k == "coarse_mode") c->opt_coarse_mode = (int)value;
        else throw Fail{4, "set_option: unknown key " + k};
    });
}

int aspamg_gpu_set_cycle(aspamg_gpu_ctx* c, int64_t nu1, int64_t nu2) {
    return guard(c, [&] {
        if (!c) throw Fail{4, "null context"};
        if (c->finalized) throw Fail{4, "set_cycle: context already finalized"};
        if (nu1 < 0 || nu2 < 0 || nu1 + nu2 < 1 || nu1 > 16 || nu2 > 16)
            throw Fail{4, "set_cycle: need nu1, nu2 >= 0, nu1 + nu2 >= 1"};
        c->nu1 = (int)nu1;
        c->nu2 = (int)nu2;
    });
}

int aspamg_gpu_upload_level(aspamg_gpu_ctx* c, int64_t level, const aspamg_csr_view* A, const aspamg_csr_view* G,
                            const aspamg_csr_view* Gt, const aspamg_csr_view* P, const aspamg_csr_view* Pt,
                            double omega) {
    return guard(c, [&] {
        if (!c) throw Fail{4, "null context"};
        if (c->finalized) throw Fail{4, "upload_level: context already finalized"};
        if (level != (int64_t)c->lv.size()) throw Fail{4, "upload_level: levels must be uploaded in order"};
        if (level >= 32) throw Fail{4, "upload_level: too many levels"};
        CK(cudaSetDevice(c->device));
        check_view(A, "A");
        if (A->n_rows != A->n_cols) throw Fail{1, "upload_level: A must be square"};
        if (level > 0) {
            const GLevel& prev = c->lv.back();
            if (prev.P.cols() != A->n_rows) throw Fail{1, "upload_level: A size != previous P columns"};
        }
        GLevel l;
        l.n = (int)A->n_rows;
        l.a_nnz = A->nnz;
        l.A = upload_mat(c, *A, true, 0);
        const bool has = G && G->n_rows > 0;
        if (has) {
            check_view(G, "G"); check_view(Gt, "Gt"); check_view(P, "P"); check_view(Pt, "Pt");
            if (G->n_rows != l.n || G->n_cols != l.n || Gt->n_rows != l.n || Gt->n_cols != l.n)
                throw Fail{1, "upload_level: G/G' must be n x n"};
            if (P->n_rows != l.n || Pt->n_cols != l.n || Pt->n_rows != P->n_cols)
                throw Fail{1, "upload_level: P must be n x n_c and P' n_c x n"};
            if (!(omega > 0.0) || !(omega <= 1.0)) throw Fail{4, "upload_level: omega must be in (0, 1]"};
            l.G = upload_mat(c, *G, false, 1);
            l.Gt = upload_mat(c, *Gt, false, 2);
            l.P = upload_mat(c, *P, false, 3);
            l.Pt = upload_mat(c, *Pt, false, 4);
            l.omega = omega;
            l.has_smoother = true;
        }
        c->lv.push_back(l);
    });
}

int aspamg_gpu_upload_coarse(aspamg_gpu_ctx* c, int64_t n_c, const double* Lc) {
    return guard(c, [&] {
        if (!c) throw Fail{4, "null context"};
        if (c->finalized) throw Fail{4, "upload_coarse: context already finalized"};
        if (n_c < 1 || n_c > 20000) throw Fail{1, "upload_coarse: n_c out of range"};
        if (!Lc) throw Fail{1, "upload_coarse: null factor"};
        CK(cudaSetDevice(c->device));
        const int n = (int)n_c;
        std::vector<double> rm((size_t)n * n, 0.0), cm((size_t)n * n, 0.0);
        for (int j = 0; j < n; ++j)
            for (int i = j; i < n; ++i) {
                const double v = Lc[(size_t)i + (size_t)j * n];
                rm[(size_t)i * n + j] = v;  // row-major L
                cm[(size_t)i + (size_t)j * n] = v;  // column-major L == row-major L'
            }
        for (int i = 0; i < n; ++i)
            if (!(rm[(size_t)i * n + i] > 0.0)) throw Fail{3, "upload_coarse: non-positive diagonal in factor"};
        // inverted 32x32 diagonal blocks (lower for L, upper for L')
        const int nb = (n + 31) / 32;
        std::vector<double> df((size_t)nb * 1024, 0.0), db((size_t)nb * 1024, 0.0);
        for (int b = 0; b < nb; ++b) {
            const int j0 = 32 * b, bs = std::min(32, n - j0);
            double inv[32][32] = {};
            for (int col = 0; col < bs; ++col) {  // solve L_b x = e_col
                double xv[32] = {};
                for (int i = 0; i < bs; ++i) {
                    double s = (i == col) ? 1.0 : 0.0;
                    for (int k = 0; k < i; ++k) s -= rm[(size_t)(j0 + i) * n + j0 + k] * xv[k];
                    xv[i] = s / rm[(size_t)(j0 + i) * n + j0 + i];
                }
                for (int i = 0; i < bs; ++i) inv[i][col] = xv[i];
            }
            for (int i = 0; i < 32; ++i)
                for (int j = 0; j < 32; ++j) {
                    df[(size_t)b * 1024 + 32 * i + j] = inv[i][j];
                    db[(size_t)b * 1024 + 32 * i + j] = inv[j][i];  // (L_b^{-1})' = (L_b')^{-1}
                }
        }
        // W = L^{-1}: column j solves L w = e_j (forward substitution from row j)
        std::vector<double> W((size_t)n * n, 0.0), Wt((size_t)n * n, 0.0);
        for (int j = 0; j < n; ++j) {
            for (int i = j; i < n; ++i) {
                double sacc = (i == j) ? 1.0 : 0.0;
                for (int k = j; k < i; ++k) sacc -= rm[(size_t)i * n + k] * W[(size_t)k * n + j];
                W[(size_t)i * n + j] = sacc / rm[(size_t)i * n + i];
            }
        }
        for (int i = 0; i < n; ++i)
            for (int j = 0; j <= i; ++j) Wt[(size_t)j * n + i] = W[(size_t)i * n + j];
        c->n_c = n;
        c->cw = dalloc<double>(c, (size_t)n);
        {  // dense triangles as CSR (row-contiguous, ascending columns)
            std::vector<int64_t> rpl((size_t)n + 1), rpu((size_t)n + 1), cil, ciu;
            std::vector<double> vl, vu;
            cil.reserve((size_t)n * (n + 1) / 2);
            ciu.reserve((size_t)n * (n + 1) / 2);
            vl.reserve(cil.capacity());
            vu.reserve(ciu.capacity());
            for (int i = 0; i < n; ++i) {
                rpl[(size_t)i] = (int64_t)cil.size();
                for (int j = 0; j <= i; ++j) { cil.push_back(j); vl.push_back(W[(size_t)i * n + j]); }
                rpu[(size_t)i] = (int64_t)ciu.size();
                for (int j = i; j < n; ++j) { ciu.push_back(j); vu.push_back(Wt[(size_t)i * n + j]); }
            }
            rpl[(size_t)n] = (int64_t)cil.size();
            rpu[(size_t)n] = (int64_t)ciu.size();
            aspamg_csr_view lv{n, n, (int64_t)cil.size(), rpl.data(), cil.data(), vl.data()};
            aspamg_csr_view uv{n, n, (int64_t)ciu.size(), rpu.data(), ciu.data(), vu.data()};
            c->Wm = upload_mat(c, lv, false);
            c->Wtm = upload_mat(c, uv, false);
        }
        c->Lrm = dalloc<double>(c, rm.size());
        c->Lcm = dalloc<double>(c, cm.size());
        c->Dinv_f = dalloc<double>(c, df.size());
        c->Dinv_b = dalloc<double>(c, db.size());
        CK(cudaMemcpy(c->Lrm, rm.data(), rm.size() * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(c->Lcm, cm.data(), cm.size() * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(c->Dinv_f, df.data(), df.size() * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(c->Dinv_b, db.data(), db.size() * 8, cudaMemcpyHostToDevice));
        coarse_prepare(n);
        CK(cudaGetLastError());
        c->coarse_uploaded = true;
    });
}

int aspamg_gpu_finalize(aspamg_gpu_ctx* c) {
    return guard(c, [&] {
        if (!c) throw Fail{4, "null context"};
        if (c->finalized) return;
        CK(cudaSetDevice(c->device));
        do_finalize(c);
    });
}

int aspamg_gpu_num_levels(aspamg_gpu_ctx* c, int64_t* n) {
    return guard(c, [&] { *n = c ? (int64_t)c->lv.size() : 0; });
}

int aspamg_gpu_level_info(aspamg_gpu_ctx* c, int64_t level, aspamg_gpu_level_stats* o) {
    return guard(c, [&] {
        if (!c || level < 0 || level >= (int64_t)c->lv.size()) throw Fail{1, "level_info: level out of range"};
        const GLevel& l = c->lv[(size_t)level];
        std::memset(o, 0, sizeof(*o));
        o->n = l.n;
        o->a_format = l.A.fmt;
        o->a_nnz = l.a_nnz;
        o->a_nnzb = l.A.fmt == 1 ? l.A.sb.nnzb : 0;
        o->a_fill = fill_ratio(l.A);
        o->g_nnz = l.has_smoother ? l.G.nnz() : 0;
        o->p_nnz = l.has_smoother ? l.P.nnz() : 0;
        o->omega = l.omega;
        o->alg_bytes_A = alg_bytes(l.A);
        if (l.has_smoother) {
            o->alg_bytes_G = alg_bytes(l.G);
            o->alg_bytes_Gt = alg_bytes(l.Gt);
            o->alg_bytes_P = alg_bytes(l.P);
            o->alg_bytes_Pt = alg_bytes(l.Pt);
        }
        o->device_bytes = (double)c->device_bytes;
        const DMat* ms[5] = {&l.A, &l.G, &l.Gt, &l.P, &l.Pt};
        for (int i = 0; i < 5; ++i) {
            const bool present = i == 0 || l.has_smoother;
            o->fmt[i] = present ? ms[i]->fmt : -1;
            o->fill[i] = present ? fill_ratio(*ms[i]) : 0.0;
        }
    });
}

int aspamg_gpu_vcycle_device(aspamg_gpu_ctx* c, const double* y, double* z) {
    return guard(c, [&] {
        ensure_ready(c);
        CK(cudaSetDevice(c->device));
        const size_t bytes = (size_t)c->lv[0].n * sizeof(double);
        CK(cudaMemcpyAsync(c->vy, y, bytes, cudaMemcpyDeviceToDevice, c->stream));
        CK(cudaGraphLaunch(c->vc_exec, c->stream));
        CK(cudaMemcpyAsync(z, c->vz, bytes, cudaMemcpyDeviceToDevice, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        CK(cudaGetLastError());
    });
}

int aspamg_gpu_vcycle(aspamg_gpu_ctx* c, const double* y, double* z) {
    return guard(c, [&] {
        ensure_ready(c);
        if (!y || !z) throw Fail{1, "vcycle: null buffer"};
        CK(cudaSetDevice(c->device));
        const size_t bytes = (size_t)c->lv[0].n * sizeof(double);
        CK(cudaMemcpyAsync(c->vy, y, bytes, cudaMemcpyHostToDevice, c->stream));
        CK(cudaGraphLaunch(c->vc_exec, c->stream));
        CK(cudaMemcpyAsync(z, c->vz, bytes, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        CK(cudaGetLastError());
    });
}

int aspamg_gpu_spmv(aspamg_gpu_ctx* c, int64_t level, int which, const double* x, double* y) {
    return guard(c, [&] {
        ensure_ready(c);
        if (level < 0 || level >= (int64_t)c->lv.size()) throw Fail{1, "spmv: level out of range"};
        const GLevel& l = c->lv[(size_t)level];
        if (which != 0 && !l.has_smoother) throw Fail{1, "spmv: operand absent on the coarsest level"};
        const DMat* M = which == 0 ? &l.A : which == 1 ? &l.G : which == 2 ? &l.Gt : which == 3 ? &l.P : which == 4 ? &l.Pt : nullptr;
        if (!M) throw Fail{4, "spmv: which must be 0..4"};
        CK(cudaSetDevice(c->device));
        double *dx = nullptr, *dy = nullptr;
        CK(cudaMalloc(&dx, sizeof(double) * std::max(1, M->cols())));
        CK(cudaMalloc(&dy, sizeof(double) * std::max(1, M->rows())));
        cudaMemcpyAsync(dx, x, sizeof(double) * M->cols(), cudaMemcpyHostToDevice, c->stream);
        spmv(*M, EPI_PLAIN, dx, dy, nullptr, 1.0, nullptr, Red{}, nullptr, Launch{0, c->stream});
        cudaMemcpyAsync(y, dy, sizeof(double) * M->rows(), cudaMemcpyDeviceToHost, c->stream);
        cudaError_t e = cudaStreamSynchronize(c->stream);
        cudaFree(dx);
        cudaFree(dy);
        CK(e);
        CK(cudaGetLastError());
    });
}

int aspamg_gpu_smooth(aspamg_gpu_ctx* c, int64_t level, const double* b, const double* x, double* out) {
    return guard(c, [&] {
        ensure_ready(c);
        if (level < 0 || level + 1 >= (int64_t)c->lv.size()) throw Fail{1, "smooth: level has no smoother"};
        GLevel& l = c->lv[(size_t)level];
        CK(cudaSetDevice(c->device));
        const size_t bytes = sizeof(double) * l.n;
        double *db = nullptr, *dx = nullptr;
        CK(cudaMalloc(&db, bytes));
        CK(cudaMalloc(&dx, bytes));
        cudaStream_t s = c->stream;
        cudaMemcpyAsync(db, b, bytes, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(dx, x, bytes, cudaMemcpyHostToDevice, s);
        // r = b - A x ; t = G r ; x' = x + w G' t (in place)
        spmv(l.A, EPI_RESID, dx, l.r, db, 1.0, nullptr, Red{}, nullptr, Launch{0, s});
        spmv(l.G, EPI_PLAIN, l.r, l.t, nullptr, 1.0, nullptr, Red{}, nullptr, Launch{0, s});
        spmv(l.Gt, EPI_ADDSCALE, l.t, dx, dx, l.omega, nullptr, Red{}, nullptr, Launch{0, s});
        cudaMemcpyAsync(out, dx, bytes, cudaMemcpyDeviceToHost, s);
        cudaError_t e = cudaStreamSynchronize(s);
        cudaFree(db);
        cudaFree(dx);
        CK(e);
        CK(cudaGetLastError());
    });
}

int aspamg_gpu_coarse_solve(aspamg_gpu_ctx* c, const double* y, double* z) {
    return guard(c, [&] {
        ensure_ready(c);
        CK(cudaSetDevice(c->device));
        const size_t bytes = sizeof(double) * c->n_c;
        double *dy = nullptr, *dz = nullptr;
        CK(cudaMalloc(&dy, bytes));
        CK(cudaMalloc(&dz, bytes));
        cudaMemcpyAsync(dy, y, bytes, cudaMemcpyHostToDevice, c->stream);
        if (c->opt_coarse_mode == 1) {
            spmv(c->Wm, EPI_PLAIN, dy, c->cw, nullptr, 1.0, nullptr, Red{}, nullptr, Launch{0, c->stream});
            spmv(c->Wtm, EPI_PLAIN, c->cw, dz, nullptr, 1.0, nullptr, Red{}, nullptr, Launch{0, c->stream});
        } else {
            coarse_solve(c->n_c, c->Lrm, c->Lcm, c->Dinv_f, c->Dinv_b, dy, dz, nullptr, Red{}, nullptr,
                         Launch{1, c->stream});
        }
        cudaMemcpyAsync(z, dz, bytes, cudaMemcpyDeviceToHost, c->stream);
        cudaError_t e = cudaStreamSynchronize(c->stream);
        cudaFree(dy);
        cudaFree(dz);
        CK(e);
        CK(cudaGetLastError());
    });
}

int aspamg_gpu_pcg(aspamg_gpu_ctx* c, const double* b, const double* x0, double rel_tol, int64_t max_it, double* x,
                   double* history, int64_t* n_it, int* converged, double* true_rel_res) {
    int status = 0;
    int code = guard(c, [&] {
        ensure_ready(c);
        if (!b || !x || !n_it || !converged || !true_rel_res) throw Fail{1, "pcg: null argument"};
        CK(cudaSetDevice(c->device));
        const size_t bytes = sizeof(double) * c->lv[0].n;
        CK(cudaMemcpyAsync(c->b, b, bytes, cudaMemcpyHostToDevice, c->stream));
        if (x0) CK(cudaMemcpyAsync(c->x, x0, bytes, cudaMemcpyHostToDevice, c->stream));
        long long it = 0;
        int conv = 0;
        double trr = 0;
        try {
            status = run_pcg(c, x0 != nullptr, rel_tol, max_it, &it, &conv, &trr);
        } catch (const Fail& f) {
            *n_it = it;
            throw;
        }
        CK(cudaMemcpyAsync(x, c->x, bytes, cudaMemcpyDeviceToHost, c->stream));
        if (history && it > 0) CK(cudaMemcpyAsync(history, c->hist, sizeof(double) * it, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        CK(cudaGetLastError());
        *n_it = it;
        *converged = conv;
        *true_rel_res = trr;
    });
    if (code != 0) return code;
    if (status == 6) c->err = "pcg: not converged";
    return status;
}

int aspamg_gpu_pcg_device(aspamg_gpu_ctx* c, const double* b, const double* x0, double rel_tol, int64_t max_it,
                          double* x, double* history, int64_t* n_it, int* converged, double* true_rel_res) {
    int status = 0;
    int code = guard(c, [&] {
        ensure_ready(c);
        if (!b || !x || !n_it || !converged || !true_rel_res) throw Fail{1, "pcg: null argument"};
        CK(cudaSetDevice(c->device));
        const size_t bytes = sizeof(double) * c->lv[0].n;
        CK(cudaMemcpyAsync(c->b, b, bytes, cudaMemcpyDeviceToDevice, c->stream));
        if (x0) CK(cudaMemcpyAsync(c->x, x0, bytes, cudaMemcpyDeviceToDevice, c->stream));
        long long it = 0;
        int conv = 0;
        double trr = 0;
        status = run_pcg(c, x0 != nullptr, rel_tol, max_it, &it, &conv, &trr);
        CK(cudaMemcpyAsync(x, c->x, bytes, cudaMemcpyDeviceToDevice, c->stream));
        if (history && it > 0) CK(cudaMemcpyAsync(history, c->hist, sizeof(double) * it, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        CK(cudaGetLastError());
        *n_it = it;
        *converged = conv;
        *true_rel_res = trr;
    });
    if (code != 0) return code;
    if (status == 6) c->err = "pcg: not converged";
    return status;
}

int aspamg_gpu_xsell_layout_spmv(const aspamg_csr_view* A, int64_t tile_rows, int64_t fold, int64_t gran, const double* x,
                                 double* y) {
    return guard(nullptr, [&] {
        check_view(A, "A");
        if (!x || !y) throw Fail{1, "xsell_layout_spmv: null vector"};
        if (fold < 1 || fold > 2 || tile_rows < 32 * fold || tile_rows > kBlock * fold || tile_rows % (32 * fold) || gran < 1 ||
            gran > 4)
            throw Fail{4, "xsell_layout_spmv: tile_rows / fold must be a multiple of 32 in [32, 256], fold 1 or 2, gran in [1, 4]"};
        XsellHost H;
        if (!build_xsell_host(*A, (int)tile_rows, (int)fold, (int)gran, (size_t)65536, H))
            throw Fail{4, "xsell_layout_spmv: operand does not fit the tile-local format"};
        xsell_host_spmv(H, A->n_rows, A->n_cols, x, y);
    });
}

int aspamg_gpu_last_solve_ms(aspamg_gpu_ctx* c, double* ms) {
    return guard(c, [&] { *ms = c ? c->last_ms : 0.0; });
}

int aspamg_gpu_launch_count(aspamg_gpu_ctx* c, int64_t* n) {
    return guard(c, [&] { *n = c ? c->last_launches : 0; });
}

// One PCG iteration's ops run eagerly with an event pair around each kernel.
int aspamg_gpu_profile_iteration(aspamg_gpu_ctx* c, aspamg_gpu_kernel_time* out, int cap, int* count) {
    return guard(c, [&] {
        ensure_ready(c);
        CK(cudaSetDevice(c->device));
        cudaStream_t s = c->stream;
        // a live, non-terminating state: k = 1 (beta path), tol 0, huge max_it
        PcgState h = {};
        CK(cudaMemcpyAsync(c->st_host, c->st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        h = *c->st_host;
        h.done = 0; h.notspd = 0; h.k = 1; h.tol = 0.0; h.max_it = 1ll << 40; h.history = c->hist;
        if (!(h.bnorm > 0)) h.bnorm = 1.0;
        if (!(h.rz != 0)) h.rz = 1.0;
        if (!c->hist) {
            c->hist_cap = 1024;
            CK(cudaMalloc(&c->hist, (size_t)c->hist_cap * sizeof(double)));
            h.history = c->hist;
        }
        *c->st_host = h;
        CK(cudaMemcpyAsync(c->st, c->st_host, sizeof(PcgState), cudaMemcpyHostToDevice, s));
        std::vector<cudaEvent_t> ev(c->body.size() + 1);
        for (auto& e : ev) CK(cudaEventCreate(&e));
        // warm the iteration once
        run_ops(c->body, s);
        CK(cudaMemcpyAsync(c->st, c->st_host, sizeof(PcgState), cudaMemcpyHostToDevice, s));
        CK(cudaEventRecord(ev[0], s));
        for (size_t i = 0; i < c->body.size(); ++i) {
            c->body[i].fn(s);
            CK(cudaEventRecord(ev[i + 1], s));
        }
        CK(cudaStreamSynchronize(s));
        int k = 0;
        for (size_t i = 0; i < c->body.size() && k < cap; ++i, ++k) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
            std::memset(&out[k], 0, sizeof(out[k]));
            std::strncpy(out[k].name, c->body[i].name.c_str(), sizeof(out[k].name) - 1);
            out[k].level = c->body[i].level;
            out[k].ms = ms;
            out[k].alg_bytes = c->body[i].bytes;
        }
        *count = k;
        for (auto& e : ev) cudaEventDestroy(e);
        CK(cudaGetLastError());
    });
}

// Device time of the standalone V-cycle graph (y = vy -> z = vz), averaged.
int aspamg_gpu_time_vcycle(aspamg_gpu_ctx* c, int reps, double* avg_ms) {
    return guard(c, [&] {
        ensure_ready(c);
        CK(cudaSetDevice(c->device));
        reps = std::max(1, reps);
        for (int i = 0; i < 3; ++i) CK(cudaGraphLaunch(c->vc_exec, c->stream));
        CK(cudaEventRecord(c->ev0, c->stream));
        for (int i = 0; i < reps; ++i) CK(cudaGraphLaunch(c->vc_exec, c->stream));
        CK(cudaEventRecord(c->ev1, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
        *avg_ms = ms / reps;
    });
}

// Graph-mode per-op timing: each body op is captured `reps` times back to back
// into its own graph; the per-launch time includes the in-graph launch gap.
int aspamg_gpu_profile_ops(aspamg_gpu_ctx* c, int reps, aspamg_gpu_kernel_time* out, int cap, int* count) {
    return guard(c, [&] {
        ensure_ready(c);
        CK(cudaSetDevice(c->device));
        cudaStream_t s = c->stream;
        reps = std::max(1, std::min(reps, 64));
        CK(cudaMemcpyAsync(c->st_host, c->st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        PcgState h = *c->st_host;
        h.done = 0; h.notspd = 0; h.k = 1; h.tol = 0.0; h.max_it = 1ll << 40;
        if (!c->hist || c->hist_cap < 4096) {
            if (c->hist) cudaFree(c->hist);
            c->hist_cap = 4096;
            CK(cudaMalloc(&c->hist, (size_t)c->hist_cap * sizeof(double)));
        }
        h.history = c->hist;
        if (!(h.bnorm > 0)) h.bnorm = 1.0;
        if (!(h.rz != 0)) h.rz = 1.0;
        int k = 0;
        for (size_t i = 0; i < c->body.size() && k < cap; ++i, ++k) {
            std::vector<Op> rep(reps, c->body[i]);
            cudaGraph_t g = capture(c, rep);
            cudaGraphExec_t ge = nullptr;
            CK(cudaGraphInstantiate(&ge, g, 0));
            h.k = 1;
            *c->st_host = h;
            CK(cudaMemcpyAsync(c->st, c->st_host, sizeof(PcgState), cudaMemcpyHostToDevice, s));
            CK(cudaGraphLaunch(ge, s));  // warm
            CK(cudaMemcpyAsync(c->st, c->st_host, sizeof(PcgState), cudaMemcpyHostToDevice, s));
            CK(cudaEventRecord(c->ev0, s));
            CK(cudaGraphLaunch(ge, s));
            CK(cudaEventRecord(c->ev1, s));
            CK(cudaStreamSynchronize(s));
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
            cudaGraphExecDestroy(ge);
            cudaGraphDestroy(g);
            std::memset(&out[k], 0, sizeof(out[k]));
            std::strncpy(out[k].name, c->body[i].name.c_str(), sizeof(out[k].name) - 1);
            out[k].level = c->body[i].level;
            out[k].ms = ms / reps;
            out[k].alg_bytes = c->body[i].bytes;
        }
        *count = k;
        CK(cudaGetLastError());
    });
}

int aspamg_gpu_time_kernel(aspamg_gpu_ctx* c, const char* name, int64_t level, int reps, double* avg_ms,
                           double* bytes) {
    return guard(c, [&] {
        ensure_ready(c);
        CK(cudaSetDevice(c->device));
        const Op* op = nullptr;
        for (const auto& o : c->body)
            if (o.level == level && (o.name == name || o.name.rfind(std::string(name) + ".", 0) == 0)) { op = &o; break; }
        if (!op) throw Fail{4, std::string("time_kernel: no op named ") + name + " at that level"};
        cudaStream_t s = c->stream;
        PcgState h = {};
        CK(cudaMemcpyAsync(c->st_host, c->st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        h = *c->st_host;
        h.done = 0; h.notspd = 0; h.k = 1; h.tol = 0.0; h.max_it = 1ll << 40;
        if (!c->hist) {
            c->hist_cap = 1024;
            CK(cudaMalloc(&c->hist, (size_t)c->hist_cap * sizeof(double)));
        }
        h.history = c->hist;
        if (!(h.bnorm > 0)) h.bnorm = 1.0;
        if (!(h.rz != 0)) h.rz = 1.0;
        *c->st_host = h;
        CK(cudaMemcpyAsync(c->st, c->st_host, sizeof(PcgState), cudaMemcpyHostToDevice, s));
        for (int i = 0; i < 3; ++i) op->fn(s);
        CK(cudaEventRecord(c->ev0, s));
        for (int i = 0; i < reps; ++i) op->fn(s);
        CK(cudaEventRecord(c->ev1, s));
        CK(cudaStreamSynchronize(s));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
        *avg_ms = ms / std::max(1, reps);
        *bytes = op->bytes;
        CK(cudaGetLastError());
    });
}

int aspamg_gpu_stream(aspamg_gpu_ctx* c, void** s) {
    return guard(c, [&] { *s = c ? (void*)c->stream : nullptr; });
}

int aspamg_gpu_alloc_pinned(int64_t bytes, void** out) {
    return guard(nullptr, [&] { CK(cudaMallocHost(out, (size_t)std::max<int64_t>(bytes, 1))); });
}

int aspamg_gpu_free_pinned(void* p) {
    return guard(nullptr, [&] { CK(cudaFreeHost(p)); });
}

int aspamg_gpu_alloc_device(aspamg_gpu_ctx* c, int64_t bytes, void** out) {
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        CK(cudaMalloc(out, (size_t)std::max<int64_t>(bytes, 1)));
    });
}

int aspamg_gpu_free_device(aspamg_gpu_ctx* c, void* p) {
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        CK(cudaFree(p));
    });
}

int aspamg_gpu_memcpy(aspamg_gpu_ctx* c, void* dst, const void* src, int64_t bytes) {
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        CK(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

}  // extern "C"
