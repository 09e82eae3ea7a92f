// GPU setup components: the adaptive FSAI smoother
// set-up — aFSAI build, Lanczos lambda_max, the omega refinement loop
// (Alg. 3 :374-387) — on the device.
//
// Restates csrc/host/fsai.cpp operation for operation, so G, omega and psi are
// bit-identical to the host's:
//   * afsai passes (fsai.cpp run_passes): one warp per row runs several
//     refinement passes back to back (the factor is kept in the pattern's
//     insertion order, so a pass continues exactly where the previous one
//     stopped) and records the row of G after each pass. The row's incremental
//     Cholesky factor of A[P, P] (packed; shared memory, or an L2-sized global
//     scratch for long patterns), the bordered solves and the gradient
//     accumulator (open addressing keyed by column) are per warp. The dense
//     arithmetic is the lane-parallel order the host restates: dot products as
//     32 strided partial sums + xor butterfly (dot_w32), the forward solve
//     left-looking with dot_w32 rows, the transposed solve right-looking (lanes
//     update b_k, k < i). The gradient takes the pattern rows in insertion order,
//     then row i. Candidate choice = the host's partial_sort order (|g|
//     descending, column ascending).
//   * transpose: counting sort by column + per-column sort by row (the unique
//     transpose, identical to core.cpp transpose()).
//   * Lanczos: exact sequential CSR products (thread per row, ascending column
//     order) and core.cpp's chunked dots; the tridiagonal eigenproblem and the
//     start vector (Rng) on the host, same code.
#include "setup_common.cuh"
#include "../host/core.hpp"
#include "../host/smalldense.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

namespace aspamg_gpu {
namespace {

constexpr unsigned FULL = 0xffffffffu;

struct AfsaiArgs {
    DCsr64 A;
    const long long* gs_rp = nullptr;  // start pattern rows in insertion order (i itself skipped), or null
    const long long* gs_ci = nullptr;
    int npass = 1;               // passes run back to back per row (fsai.cpp run_row)
    int k0 = 0, rho0 = 0;        // pass 0
    double eps0 = 0.0;
    int ki = 0, rhoi = 0;        // passes 1 .. npass-1
    double epsi = 0.0;
    int mcap = 1, hcap = 1024;   // mcap: bound of the final pattern size
    int l_global = 0;            // factor in global scratch (rows too long for shared memory)
    double* lscratch = nullptr;  // [gridDim.x * W][packed(mcap)] when l_global
    int h_global = 0;            // gradient values in global scratch (large tables)
    double* hvscratch = nullptr; // [gridDim.x * W][hcap] when h_global
    int* gscratch = nullptr;     // per warp: column hash (keys, slots), slot keys, slot maps
    long long gstride = 0;       // ints per warp in gscratch
    int smap_cap = 0;            // slot-map entries per pattern row (max entries j < i of a row)
    const long long* rows = nullptr;  // rows to process (null: all)
    long long nrows = 0;
    // outputs: pass p of row i
    int* cnt = nullptr;          // [npass][n]: m_p + 1 (row status in pass 0's slot: -1 not SPD, -2 table overflow)
    double* psi = nullptr;       // [npass][n]
    double* yout = nullptr;      // y_p[0..m_p) at yout + yoff[p] + i * ycap[p]
    const long long* yoff = nullptr;
    const int* ycap = nullptr;
    int* pout = nullptr;         // final pattern, insertion order: pout + i * mcap
    unsigned long long* bad = nullptr;  // smallest failing row
    unsigned long long* prof = nullptr; // optional: cycles per phase (ASPAMG_AFSAI_PROF)
};

__host__ __device__ inline size_t packed(long long m) { return (size_t)m * (size_t)(m + 1) / 2; }

// pattern-position table: column -> index in the pattern (power of two >= 2 mcap)
__host__ __device__ inline int pat_cap(int mcap) {
    int c = 64;
    while (c < 2 * mcap) c <<= 1;
    return c;
}

__host__ __device__ inline size_t warp_bytes(int mcap, int hcap, bool l_global, bool h_global) {
    const size_t lp = l_global ? 0 : packed(mcap);
    const size_t hc = h_global ? 0 : (size_t)hcap / 2;  // slot values (the column hash stays <= half full)
    size_t b = 8 * (lp + 2 * (size_t)mcap + hc) + 4 * (2 * (size_t)mcap + 41 + 40 + 2 * (size_t)pat_cap(mcap) + 4);
    return (b + 15) & ~(size_t)15;
}
// per-warp global ints: column hash keys + slots (2 hcap), slot keys (hcap), slot
// maps of the pattern rows and row i ((mcap + 1) smap_cap)
__host__ __device__ inline long long gscratch_ints(int mcap, int hcap, int smap_cap) {
    return 3LL * hcap + (long long)(mcap + 1) * smap_cap;
}

struct WarpMem {
    double *L, *y, *a;
    double* sv;      // gradient value per slot
    int* hk;         // column hash: keys (-1 empty)
    int* hs;         // column hash: slot of the key
    int* sk;         // slot -> column (>= 0), or -1 - column once the column is in the pattern
    int* smap;       // slot maps: pattern position q (mcap: row i) -> slots of row's entries j < i
    int* slen;       // entries j < i of the row at position q (mcap: row i)
    int* ns;         // [0] slot count, [1] overflow flag
    int *pat, *sel, *pk, *pv;
    int pcap;
};

__device__ __forceinline__ unsigned hslot(int j, int cap) { return ((unsigned)j * 2654435761u) & (unsigned)(cap - 1); }

// A(r, c) of a sorted-row CSR, 0 if not stored (the host's dense scatter).
__device__ double a_at(const DCsr64& A, long long r, long long c) {
    long long lo = A.rp[r], hi = A.rp[r + 1];
    const long long end = hi;
    while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if (A.ci[mid] < c) lo = mid + 1;
        else hi = mid;
    }
    return (lo < end && A.ci[lo] == c) ? A.v[lo] : 0.0;
}

// smalldense.cpp dot_w32: lane l sums k = l, l+32, ... (separate mul / add), then
// the xor butterfly; every lane ends with the same value (addition commutes).
__device__ __forceinline__ double dot_w32(const double* x, const double* y, int n, int lane) {
    double s = 0.0;
    for (int k = lane; k < n; k += 32) s = __dadd_rn(s, __dmul_rn(x[k], y[k]));
#pragma unroll
    for (int h = 16; h >= 1; h >>= 1) s = __dadd_rn(s, __shfl_xor_sync(FULL, s, h));
    return s;
}

// smalldense.cpp trsv_lower on the packed factor (b may be the factor's row n):
// 32-row blocks, lane l on row B + l — the panel product t = L_i[0..B) . b[0..B)
// as one sequential chain, then right-looking inside the block (lane j divides,
// broadcasts, lanes > j update).
__device__ void trsv_lower_w(int n, const double* L, double* b, int lane) {
    for (int B = 0; B < n; B += 32) {
        const int i = B + lane;
        const double* Li = L + packed(i < n ? i : 0);
        double t = 0.0;
        if (i < n) {
#pragma unroll 8
            for (int k = 0; k < B; ++k) t = __dadd_rn(t, __dmul_rn(Li[k], b[k]));
        }
        double bi = i < n ? __dsub_rn(b[i], t) : 0.0;
        const int nb = min(32, n - B);
        for (int j = 0; j < nb; ++j) {
            if (lane == j) bi = __ddiv_rn(bi, Li[i]);
            const double xj = __shfl_sync(FULL, bi, j);
            if (lane > j && i < n) bi = __dsub_rn(bi, __dmul_rn(Li[B + j], xj));
        }
        __syncwarp();
        if (i < n) b[i] = bi;
        __syncwarp();
    }
}

// smalldense.cpp trsv_lower_t (right-looking): b_i /= L_ii, then b_k -= L_ik b_i for k < i.
__device__ void trsv_lower_t_w(int n, const double* L, double* b, int lane) {
    for (int i = n - 1; i >= 0; --i) {
        const double* Li = L + packed(i);
        const double bi = __ddiv_rn(b[i], Li[i]);
        __syncwarp();
        for (int k = lane; k < i; k += 32) b[k] = __dsub_rn(b[k], __dmul_rn(Li[k], bi));
        if (lane == 0) b[i] = bi;
        __syncwarp();
    }
}

__device__ void pat_insert(const WarpMem& w, int col, int q) {  // one lane
    unsigned h = hslot(col, w.pcap);
    while (w.pk[h] != -1) h = (h + 1) & (unsigned)(w.pcap - 1);
    w.pk[h] = col;
    w.pv[h] = q;
}
__device__ int pat_find(const WarpMem& w, long long col) {
    unsigned h = hslot((int)col, w.pcap);
    for (;;) {
        const int k = w.pk[h];
        if (k == (int)col) return w.pv[h];
        if (k == -1) return -1;
        h = (h + 1) & (unsigned)(w.pcap - 1);
    }
}

// out[q] = A(r, pat[q]) for q < m (0 if not stored: the host's dense scatter),
// one coalesced pass over row r; returns A(r, d) on every lane.
__device__ double gather_row(const DCsr64& A, long long r, long long d, const WarpMem& w, int m, double* out, int lane) {
    for (int q = lane; q < m; q += 32) out[q] = 0.0;
    __syncwarp();
    double dv = 0.0;
    bool hit = false;
    const long long b = A.rp[r], e1 = A.rp[r + 1];
    for (long long e0 = b + lane; e0 < e1; e0 += 4 * 32) {  // 4 loads in flight per lane
        long long c[4];
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const long long e = e0 + 32 * u;
            c[u] = e < e1 ? A.ci[e] : -1;
            v[u] = e < e1 ? A.v[e] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (c[u] < 0) continue;
            if (c[u] == d) {
                dv = v[u];
                hit = true;
            }
            const int q = pat_find(w, c[u]);
            if (q >= 0 && q < m) out[q] = v[u];
        }
    }
    __syncwarp();
    const unsigned hb = __ballot_sync(FULL, hit);
    return hb ? __shfl_sync(FULL, dv, __ffs(hb) - 1) : 0.0;
}

// fsai.cpp chol_append: row m of the factor from A[j, pat[0..m)].
__device__ bool chol_append_w(const DCsr64& A, const WarpMem& w, int m, long long j, int lane) {
    double* row = w.L + packed(m);
    const double ajj = gather_row(A, j, j, w, m, row, lane);
    trsv_lower_w(m, w.L, row, lane);
    const double d = __dsub_rn(ajj, dot_w32(row, row, m, lane));
    if (!(d > 0.0)) return false;
    if (lane == 0) row[m] = __dsqrt_rn(d);
    __syncwarp();
    return true;
}

// Gradient support (fsai.cpp run_row step (d)). The columns j < i touched by the
// rows of P + {i} get dense slots once, when a row enters (a column hash maps j
// to its slot); each row keeps the slot of each of its entries (its slot map).
// A gradient step then zeroes the slot values and, row by row in the host's
// order (pattern in insertion order, then i), adds A(r, j) * gm into the
// entries' slots: the same sum per column as the host's accumulator, with no
// probing per step. Slot numbering is not deterministic and does not need to
// be: the candidate choice is a strict total order on (|g|, column).
__device__ int slot_of(const WarpMem& w, int hcap, int col, bool& ovf) {  // find or create
    unsigned h = hslot(col, hcap);
    for (int p = 0; p < hcap; ++p) {
        const int k = w.hk[h];
        if (k == col) return w.hs[h];  // (a row's columns are distinct: never concurrently created)
        if (k == -1) {
            const int old = atomicCAS(&w.hk[h], -1, col);
            if (old == -1) {
                const int sl = atomicAdd(&w.ns[0], 1);
                if (sl >= hcap / 2) {  // keep the table at most half full
                    ovf = true;
                    w.hs[h] = 0;
                    return -1;
                }
                w.sk[sl] = col;
                w.hs[h] = sl;
                return sl;
            }
            if (old == col) return w.hs[h];
        }
        h = (h + 1) & (unsigned)(hcap - 1);
    }
    ovf = true;
    return -1;
}

__device__ int slot_find(const WarpMem& w, int hcap, int col) {
    unsigned h = hslot(col, hcap);
    for (int p = 0; p < hcap; ++p) {
        const int k = w.hk[h];
        if (k == col) return w.hs[h];
        if (k == -1) return -1;
        h = (h + 1) & (unsigned)(hcap - 1);
    }
    return -1;
}

// Row r enters the gradient support at pattern position q (mcap: row i): slots for
// its entries j < i (new slots of columns already in P are marked at once).
__device__ void support_add(const AfsaiArgs& P, const WarpMem& w, long long r, int q, long long i, int lane,
                            bool& ovf) {
    const DCsr64& A = P.A;
    const long long b = A.rp[r], e = A.rp[r + 1];
    int* sm = w.smap + (long long)q * P.smap_cap;
    int len = (int)(e - b);  // all entries < i unless a column >= i is met
    for (long long q0 = b; q0 < e; q0 += 32) {
        const long long t = q0 + lane;
        const long long j = t < e ? A.ci[t] : LLONG_MAX;
        if (j < i) {
            const int sl = slot_of(w, P.hcap, (int)j, ovf);
            sm[t - b] = sl;
            if (sl >= 0 && pat_find(w, j) >= 0) w.sk[sl] = -1 - (int)j;
        }
        const unsigned ge = __ballot_sync(FULL, j >= i);
        if (ge) {
            len = (int)(q0 - b) + __ffs(ge) - 1;
            break;
        }
    }
    if (lane == 0) w.slen[q] = len;
    __syncwarp();
}

// grad[slot(j)] += A(r, j) * gm over row r's entries j < i (lanes take distinct j).
__device__ void grad_row(const DCsr64& A, const WarpMem& w, long long r, const int* sm, int len, double gm, int lane) {
    const double* av = A.v + A.rp[r];
    for (int t = lane; t < len; t += 32) {
        const int sl = sm[t];
        w.sv[sl] = __dadd_rn(w.sv[sl], __dmul_rn(av[t], gm));
    }
    __syncwarp();
}

// One row of fsai.cpp run_row: npass passes back to back from the start pattern.
__device__ void afsai_row(const AfsaiArgs& P, const WarpMem& w, long long i, int lane) {
    const DCsr64& A = P.A;
    const long long n = A.n_rows;
    int m = 0;
    long long tph = clock64();
    auto mark = [&](int ph) {
        if (P.prof) {
            const long long t = clock64();
            if (lane == 0) atomicAdd(P.prof + ph, (unsigned long long)(t - tph));
            tph = t;
        }
    };
    auto fail = [&](int code) {
        if (lane == 0) {
            P.cnt[i] = code;
            if (code == -1) atomicMin(P.bad, (unsigned long long)i);
        }
    };
    for (int q = lane; q < w.pcap; q += 32) w.pk[q] = -1;
    for (int q = lane; q < P.hcap; q += 32) {
        w.hk[q] = -1;
        w.hs[q] = -1;
    }
    if (lane == 0) w.ns[0] = 0;
    __syncwarp();
    if (P.gs_rp) {
        const long long b = P.gs_rp[i], e = P.gs_rp[i + 1];
        int ns = 0;
        for (long long q0 = b; q0 < e; q0 += 32) {  // columns < i, in stored order
            const long long c = q0 + lane < e ? P.gs_ci[q0 + lane] : LLONG_MAX;
            const unsigned lt = __ballot_sync(FULL, c < i);
            if (c < i) w.pat[ns + __popc(lt & ((1u << lane) - 1))] = (int)c;
            ns += __popc(lt);
        }
        __syncwarp();
        for (int q = 0; q < ns; ++q) {
            if (lane == 0) pat_insert(w, w.pat[q], q);
            __syncwarp();
            if (!chol_append_w(A, w, m, w.pat[q], lane)) return fail(-1);
            ++m;
        }
    }
    bool ovf = false;
    for (int q = 0; q < m; ++q) support_add(P, w, w.pat[q], q, i, lane, ovf);
    support_add(P, w, i, P.mcap, i, lane, ovf);
    if (__any_sync(FULL, ovf)) return fail(-2);
    mark(0);
    double aii = lane == 0 ? a_at(A, i, i) : 0.0;
    aii = __shfl_sync(FULL, aii, 0);
    double psi = 0.0;
    bool have = false;  // w.y / psi hold the bordered solve of the current pattern
    for (int pass = 0; pass < P.npass; ++pass) {
        const int k = pass ? P.ki : P.k0, rho = pass ? P.rhoi : P.rho0;
        const double eps = pass ? P.epsi : P.eps0;
        double psi_prev = 0.0;
        for (int step = 0;; ++step) {
            if (!have) {
                // bordered solve y = A_PP^{-1} a, psi = a_ii - a'y
                gather_row(A, i, i, w, m, w.a, lane);
                for (int q = lane; q < m; q += 32) w.y[q] = w.a[q];
                __syncwarp();
                mark(1);
                trsv_lower_w(m, w.L, w.y, lane);
                mark(2);
                trsv_lower_t_w(m, w.L, w.y, lane);
                mark(3);
                psi = __dsub_rn(aii, dot_w32(w.a, w.y, m, lane));
                if (!(psi > 0.0)) return fail(-1);
                have = true;
            }
            if (step > 0 && __dsub_rn(psi_prev, psi) <= __dmul_rn(eps, psi_prev)) break;
            if (step == k) break;
            psi_prev = psi;
            // gradient: rows of P (insertion order) then row i, into the support's slots
            const int T = w.ns[0];
            for (int t = lane; t < T; t += 32) w.sv[t] = 0.0;
            __syncwarp();
            for (int q = 0; q < m; ++q)
                grad_row(A, w, w.pat[q], w.smap + (long long)q * P.smap_cap, w.slen[q], -w.y[q], lane);
            grad_row(A, w, i, w.smap + (long long)P.mcap * P.smap_cap, w.slen[P.mcap], 1.0, lane);
            mark(4);
            // the rho best candidates: |g| descending, then column ascending
            int take = 0;
            for (; take < rho; ++take) {
                double bv = -1.0;
                int bj = INT_MAX, bs = -1;
                for (int t = lane; t < T; t += 32) {
                    const int key = w.sk[t];
                    if (key >= 0) {
                        const double av = fabs(w.sv[t]);
                        if (av > bv || (av == bv && key < bj)) {
                            bv = av;
                            bj = key;
                            bs = t;
                        }
                    }
                }
                for (int o = 16; o > 0; o >>= 1) {
                    const double ov = __shfl_down_sync(FULL, bv, o);
                    const int oj = __shfl_down_sync(FULL, bj, o), os = __shfl_down_sync(FULL, bs, o);
                    if (ov > bv || (ov == bv && oj < bj)) {
                        bv = ov;
                        bj = oj;
                        bs = os;
                    }
                }
                bs = __shfl_sync(FULL, bs, 0);
                bj = __shfl_sync(FULL, bj, 0);
                if (bs < 0) break;
                if (lane == 0) {
                    w.sel[take] = bj;
                    w.sk[bs] = -1 - bj;  // enters the pattern
                }
                __syncwarp();
            }
            mark(5);
            if (take == 0) break;
            if (lane == 0)  // ascending column order of the chosen candidates
                for (int a = 1; a < take; ++a) {
                    const int v = w.sel[a];
                    int b = a - 1;
                    while (b >= 0 && w.sel[b] > v) {
                        w.sel[b + 1] = w.sel[b];
                        --b;
                    }
                    w.sel[b + 1] = v;
                }
            __syncwarp();
            for (int c = 0; c < take; ++c) {
                const int j = w.sel[c];
                if (lane == 0) {
                    w.pat[m] = j;
                    pat_insert(w, j, m);
                }
                __syncwarp();
                if (!chol_append_w(A, w, m, j, lane)) return fail(-1);
                support_add(P, w, j, m, i, lane, ovf);
                ++m;
            }
            if (__any_sync(FULL, ovf)) return fail(-2);
            have = false;
            mark(6);
        }
        double* yo = P.yout + P.yoff[pass] + i * (long long)P.ycap[pass];
        for (int q = lane; q < m; q += 32) yo[q] = w.y[q];
        if (lane == 0) {
            P.cnt[pass * n + i] = m + 1;
            P.psi[pass * n + i] = psi;
        }
    }
    for (int q = lane; q < m; q += 32) P.pout[i * (long long)P.mcap + q] = w.pat[q];
    __syncwarp();
}

__global__ void k_afsai(const AfsaiArgs P) {
    extern __shared__ __align__(16) unsigned char dyn[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, W = blockDim.x >> 5;
    unsigned char* p = dyn + (size_t)wid * warp_bytes(P.mcap, P.hcap, P.l_global != 0, P.h_global != 0);
    const size_t gw = (size_t)blockIdx.x * W + wid;
    WarpMem w;
    if (P.l_global) {
        w.L = P.lscratch + gw * packed(P.mcap);
    } else {
        w.L = reinterpret_cast<double*>(p);
        p += 8 * packed(P.mcap);
    }
    w.y = reinterpret_cast<double*>(p);
    w.a = w.y + P.mcap;
    double* after = w.a + P.mcap;
    if (P.h_global) {
        w.sv = P.hvscratch + gw * (P.hcap / 2);
    } else {
        w.sv = after;
        after += P.hcap / 2;
    }
    w.ns = reinterpret_cast<int*>(after);
    w.slen = w.ns + 4;
    w.pat = w.slen + P.mcap + 1;
    int* g = P.gscratch + gw * P.gstride;
    w.hk = g;
    w.hs = g + P.hcap;
    w.sk = g + 2LL * P.hcap;
    w.smap = g + 3LL * P.hcap;
    w.sel = w.pat + P.mcap;
    w.pcap = pat_cap(P.mcap);
    w.pk = w.sel + 40;
    w.pv = w.pk + w.pcap;
    const long long total = P.rows ? P.nrows : P.A.n_rows;
    for (long long t = (long long)blockIdx.x * W + wid; t < total; t += (long long)gridDim.x * W)
        afsai_row(P, w, P.rows ? P.rows[t] : t, lane);
}

// Pass p of a batch -> G_p (rows sorted by column) and its insertion-ordered twin
// (pattern, then i) — fsai.cpp pass_matrix. Warp per row.
__global__ void k_pass_csr(long long n, const long long* __restrict__ rp, const int* __restrict__ cnt,
                           const double* __restrict__ psi, const double* __restrict__ y, int ycap,
                           const int* __restrict__ pout, int mcap, long long* ci, double* v, long long* ici,
                           double* iv) {
    const int lane = threadIdx.x & 31;
    const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long i = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += nw) {
        const int m = cnt[i] - 1;
        const double s = __ddiv_rn(1.0, __dsqrt_rn(psi[i]));
        const int* pt = pout + i * (long long)mcap;
        const double* yi = y + i * (long long)ycap;
        const long long b = rp[i];
        for (int e = lane; e <= m; e += 32) {
            const long long col = e < m ? (long long)pt[e] : i;
            const double val = e < m ? __dmul_rn(-yi[e], s) : s;
            int rank = m;  // i closes the row (pattern columns are < i)
            if (e < m) {
                rank = 0;
                for (int f = 0; f < m; ++f) rank += pt[f] < pt[e];
            }
            ci[b + rank] = col;
            v[b + rank] = val;
            ici[b + e] = col;
            iv[b + e] = val;
        }
    }
}

// ---------------------------------------------------------------- transpose
__global__ void k_colcount(long long nnz, const long long* __restrict__ ci, int* cc) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < nnz; q += (long long)gridDim.x * blockDim.x)
        atomicAdd(&cc[ci[q]], 1);
}
__global__ void k_colfill(long long n, const long long* __restrict__ rp, const long long* __restrict__ ci,
                          const double* __restrict__ v, const long long* __restrict__ trp, int* cur, long long* tci,
                          double* tv) {
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x)
        for (long long q = rp[r]; q < rp[r + 1]; ++q) {
            const long long c = ci[q];
            const long long pos = trp[c] + atomicAdd(&cur[c], 1);
            tci[pos] = r;
            tv[pos] = v[q];
        }
}
__global__ void k_segsort(long long n, const long long* __restrict__ trp, long long* tci, double* tv) {
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x) {
        const long long b = trp[c], e = trp[c + 1];
        for (long long a = b + 1; a < e; ++a) {
            const long long key = tci[a];
            const double val = tv[a];
            long long q = a - 1;
            while (q >= b && tci[q] > key) {
                tci[q + 1] = tci[q];
                tv[q + 1] = tv[q];
                --q;
            }
            tci[q + 1] = key;
            tv[q + 1] = val;
        }
    }
}

// y = M x, each row summed sequentially in ascending column order (spmv()).
__global__ void k_spmv_seq(DCsr64 M, const double* __restrict__ x, double* y) {
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < M.n_rows;
         r += (long long)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (long long q = M.rp[r]; q < M.rp[r + 1]; ++q) s = __dadd_rn(s, __dmul_rn(M.v[q], x[M.ci[q]]));
        y[r] = s;
    }
}

// w = w - (a v + b vp)   (fsai.cpp estimate_lambda_max)
__global__ void k_lanczos_upd(long long n, double* w, const double* __restrict__ v, const double* __restrict__ vp,
                              double a, double b) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        w[i] = __dsub_rn(w[i], __dadd_rn(__dmul_rn(a, v[i]), __dmul_rn(b, vp[i])));
}

struct DevG {  // a device CSR the setup owns, plus its host row offsets
    DevCsr d;
    DevCsr ins;  // the same rows in insertion order (the next pass's start pattern); shares d.rp
    std::vector<long long> rp;
};

void free_csr(aspamg_gpu_ctx* c, DevCsr& d) {
    dfree(c, d.rp);
    dfree(c, d.ci);
    dfree(c, d.v);
    d = DevCsr{};
}

void free_g(aspamg_gpu_ctx* c, DevG& g) {
    dfree(c, g.ins.ci);
    dfree(c, g.ins.v);
    g.ins = DevCsr{};
    free_csr(c, g.d);
}

int sm_count() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

// fsai.cpp run_passes on the device: npass passes of every row, back to back,
// from the insertion-ordered start pattern (null = identity start).
struct PassParams {
    int k, rho;
    double eps;
};
struct Batch {
    long long n = 0;
    int npass = 0, mcap = 1;
    int* cnt = nullptr;
    double* psi = nullptr;
    double* y = nullptr;
    int* pout = nullptr;
    long long* d_yoff = nullptr;
    int* d_ycap = nullptr;
    std::vector<long long> yoff;
    std::vector<int> ycap;
};

void free_batch(aspamg_gpu_ctx* c, Batch& b) {
    dfree(c, b.cnt);
    dfree(c, b.psi);
    dfree(c, b.y);
    dfree(c, b.pout);
    dfree(c, b.d_yoff);
    dfree(c, b.d_ycap);
    b = Batch{};
}

constexpr int kMaxPattern = 4096;

long long max_row(const DevG* g) {
    long long r = 0;
    if (g)
        for (size_t i = 0; i + 1 < g->rp.size(); ++i) r = std::max(r, g->rp[i + 1] - g->rp[i]);
    return r;
}

// device bytes of a batch of npass passes (yout + pattern + counters)
double batch_bytes(long long n, long long gs_max, int npass, const PassParams& p0, const PassParams& pr) {
    double ys = 0.0;
    long long cap = gs_max + (long long)p0.k * p0.rho;
    for (int p = 0; p < npass; ++p) {
        if (p) cap += (long long)pr.k * pr.rho;
        ys += double(cap);
    }
    return double(n) * (8.0 * ys + 4.0 * double(cap) + 12.0 * npass);
}

Batch run_passes_device(aspamg_gpu_ctx* c, const DCsr64& A, long long a_maxrow, const DevG* Gs, int npass,
                        const PassParams& p0, const PassParams& pr, int* hcap_hint = nullptr) {
    cudaStream_t s = c->stream;
    const long long n = A.n_rows;
    const long long gs_max = max_row(Gs);  // includes the diagonal: a bound of the start pattern
    Batch B;
    B.n = n;
    B.npass = npass;
    long long cap = gs_max + (long long)p0.k * p0.rho, tot = 0;
    for (int p = 0; p < npass; ++p) {
        if (p) cap += (long long)pr.k * pr.rho;
        B.ycap.push_back((int)std::max<long long>(cap, 1));
        B.yoff.push_back(tot);
        tot += (long long)B.ycap.back() * std::max<long long>(n, 1);
    }
    if (cap > kMaxPattern) throw Fail{4, "afsai (GPU): pattern bound exceeds 4096 entries per row"};
    B.mcap = (int)std::max<long long>(cap, 1);
    const int mcap = B.mcap;
    const size_t nn = (size_t)std::max<long long>(n, 1);
    B.cnt = dalloc<int>(c, nn * npass);
    B.psi = dalloc<double>(c, nn * npass);
    B.y = dalloc<double>(c, (size_t)std::max<long long>(tot, 1));
    B.pout = dalloc<int>(c, nn * mcap);
    B.d_yoff = dalloc<long long>(c, (size_t)npass);
    B.d_ycap = dalloc<int>(c, (size_t)npass);
    CK(cudaMemcpyAsync(B.d_yoff, B.yoff.data(), 8 * (size_t)npass, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(B.d_ycap, B.ycap.data(), 4 * (size_t)npass, cudaMemcpyHostToDevice, s));
    unsigned long long* bad = dalloc<unsigned long long>(c, 1);
    const unsigned long long none = ~0ull;
    CK(cudaMemcpyAsync(bad, &none, 8, cudaMemcpyHostToDevice, s));
    const int sms = sm_count();
    std::vector<int> hc((size_t)n);
    std::vector<long long> todo;
    std::vector<void*> scratch;
    // table sizes: an upper bound of the touched columns, capped; overflowing rows rerun wider
    const long long touch = (long long)(mcap + 1) * std::max<long long>(a_maxrow, 1);
    int hcap = 64;
    while (hcap < 2 * touch && hcap < 4096) hcap <<= 1;
    if (hcap_hint && *hcap_hint > hcap) hcap = *hcap_hint;  // an earlier batch of this level overflowed
    for (int attempt = 0; attempt < 4; ++attempt) {
        AfsaiArgs P;
        P.A = A;
        P.gs_rp = Gs ? Gs->d.rp : nullptr;
        P.gs_ci = Gs ? Gs->ins.ci : nullptr;  // factor order = insertion order (fsai.cpp run_row)
        P.npass = npass;
        P.k0 = p0.k;
        P.rho0 = p0.rho;
        P.eps0 = p0.eps;
        P.ki = pr.k;
        P.rhoi = pr.rho;
        P.epsi = pr.eps;
        P.mcap = mcap;
        P.hcap = hcap;
        P.cnt = B.cnt;
        P.psi = B.psi;
        P.yout = B.y;
        P.yoff = B.d_yoff;
        P.ycap = B.d_ycap;
        P.pout = B.pout;
        P.bad = bad;
        if (attempt > 0) {
            long long* drows = dalloc<long long>(c, todo.size());
            scratch.push_back(drows);
            CK(cudaMemcpyAsync(drows, todo.data(), todo.size() * 8, cudaMemcpyHostToDevice, s));
            P.rows = drows;
            P.nrows = (long long)todo.size();
        }
        // rows in flight: short factors in shared memory, longer ones in a global
        // scratch (latency hidden by more warps per SM; the factor sweeps are streams)
        const size_t budget = 200 * 1024;
        const bool lg = 8 * packed(mcap) > 24 * 1024;
        const bool hg = hcap > 4096;
        const size_t wb = warp_bytes(mcap, hcap, lg, hg);
        if (wb > budget) throw Fail{4, "afsai (GPU): row workspace exceeds shared memory"};
        const int W = (int)std::max<size_t>(1, std::min<size_t>(16, budget / wb));
        const size_t smem = wb * W;
        CK(cudaFuncSetAttribute(k_afsai, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int occ = 1;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_afsai, 32 * W, smem));
        const long long rows = attempt ? (long long)todo.size() : n;
        const long long need = (rows + W - 1) / W;
        const int grid = (int)std::max<long long>(1, std::min<long long>(need, (long long)sms * std::max(occ, 1)));
        P.l_global = lg ? 1 : 0;
        if (lg) {
            P.lscratch = dalloc<double>(c, (size_t)grid * W * packed(mcap));
            scratch.push_back(P.lscratch);
        }
        P.h_global = hg ? 1 : 0;
        if (hg) {
            P.hvscratch = dalloc<double>(c, (size_t)grid * W * (hcap / 2));
            scratch.push_back(P.hvscratch);
        }
        P.smap_cap = (int)std::max<long long>(a_maxrow, 1);
        P.gstride = gscratch_ints(mcap, hcap, P.smap_cap);
        P.gscratch = dalloc<int>(c, (size_t)grid * W * (size_t)P.gstride);
        scratch.push_back(P.gscratch);
        static const bool prof = std::getenv("ASPAMG_AFSAI_PROF") != nullptr;
        if (prof) {
            P.prof = dalloc<unsigned long long>(c, 8);
            scratch.push_back(P.prof);
            CK(cudaMemsetAsync(P.prof, 0, 64, s));
        }
        if (rows > 0) {
            k_afsai<<<grid, 32 * W, smem, s>>>(P);
            CK(cudaGetLastError());
        }
        if (prof) {
            unsigned long long h[8];
            CK(cudaMemcpyAsync(h, P.prof, 64, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            std::fprintf(stderr, "[afsai prof n=%lld npass=%d mcap=%d hcap=%d W=%d grid=%d lg=%d hg=%d] Gcyc: start %.2f gather %.2f fwd %.2f bwd %.2f grad %.2f cand %.2f append %.2f\n",
                         rows, npass, mcap, hcap, W, grid, (int)lg, (int)hg, h[0] / 1e9, h[1] / 1e9, h[2] / 1e9, h[3] / 1e9, h[4] / 1e9, h[5] / 1e9, h[6] / 1e9);
        }
        CK(cudaMemcpyAsync(hc.data(), B.cnt, (size_t)n * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        todo.clear();
        for (long long i = 0; i < n; ++i)
            if (hc[(size_t)i] == -2) todo.push_back(i);
        if (todo.empty()) break;
        if (hcap_hint && (double)todo.size() > 0.01 * (double)n) *hcap_hint = hcap * 4;  // next batches start wider
        hcap *= 4;
    }
    if (!todo.empty()) throw Fail{4, "afsai (GPU): gradient support exceeds the gradient table in a row"};
    unsigned long long hbad = 0;
    CK(cudaMemcpy(&hbad, bad, 8, cudaMemcpyDeviceToHost));
    for (void* q : scratch) dfree(c, q);
    dfree(c, bad);
    if (hbad != none) {
        free_batch(c, B);
        throw Fail{2, "afsai_build: non-positive local pivot at row " + std::to_string((long long)hbad)};
    }
    return B;
}

// Pass p of a batch as a device CSR (sorted) + its insertion-ordered twin; psi_p -> psi.
DevG pass_device(aspamg_gpu_ctx* c, const Batch& B, int p, double* psi) {
    cudaStream_t s = c->stream;
    const long long n = B.n;
    std::vector<int> hc((size_t)n);
    CK(cudaMemcpyAsync(hc.data(), B.cnt + (size_t)p * n, (size_t)n * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    DevG G;
    G.rp.assign((size_t)n + 1, 0);
    for (long long i = 0; i < n; ++i) G.rp[(size_t)i + 1] = G.rp[(size_t)i] + hc[(size_t)i];
    const long long nnz = G.rp.back();
    G.d.rp = dalloc<long long>(c, (size_t)n + 1);
    G.d.ci = dalloc<long long>(c, (size_t)std::max<long long>(nnz, 1));
    G.d.v = dalloc<double>(c, (size_t)std::max<long long>(nnz, 1));
    G.ins.ci = dalloc<long long>(c, (size_t)std::max<long long>(nnz, 1));
    G.ins.v = dalloc<double>(c, (size_t)std::max<long long>(nnz, 1));
    CK(cudaMemcpyAsync(G.d.rp, G.rp.data(), G.rp.size() * 8, cudaMemcpyHostToDevice, s));
    if (n > 0) {
        k_pass_csr<<<sm_count() * 8, 256, 0, s>>>(n, G.d.rp, B.cnt + (size_t)p * n, B.psi + (size_t)p * n,
                                                  B.y + B.yoff[(size_t)p], B.ycap[(size_t)p], B.pout, B.mcap,
                                                  G.d.ci, G.d.v, G.ins.ci, G.ins.v);
        CK(cudaGetLastError());
    }
    if (psi) CK(cudaMemcpyAsync(psi, B.psi + (size_t)p * n, (size_t)n * 8, cudaMemcpyDeviceToDevice, s));
    CK(cudaStreamSynchronize(s));  // G.rp (host) outlives the copy
    G.d.view = {n, n, nnz, G.d.rp, G.d.ci, G.d.v};
    G.ins.view = {n, n, nnz, G.d.rp, G.ins.ci, G.ins.v};
    return G;
}

DevCsr transpose_device(aspamg_gpu_ctx* c, const DevG& G) {
    cudaStream_t s = c->stream;
    const long long n = G.d.view.n_rows, m = G.d.view.n_cols, nnz = G.d.view.nnz;
    const int sms = sm_count();
    int* cc = dalloc<int>(c, (size_t)std::max<long long>(m, 1));
    CK(cudaMemsetAsync(cc, 0, (size_t)m * 4, s));
    k_colcount<<<sms * 8, 256, 0, s>>>(nnz, G.d.ci, cc);
    CK(cudaGetLastError());
    std::vector<int> h((size_t)m);
    CK(cudaMemcpyAsync(h.data(), cc, (size_t)m * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    std::vector<long long> trp((size_t)m + 1, 0);
    for (long long j = 0; j < m; ++j) trp[(size_t)j + 1] = trp[(size_t)j] + h[(size_t)j];
    DevCsr T;
    T.rp = dalloc<long long>(c, (size_t)m + 1);
    T.ci = dalloc<long long>(c, (size_t)std::max<long long>(nnz, 1));
    T.v = dalloc<double>(c, (size_t)std::max<long long>(nnz, 1));
    CK(cudaMemcpyAsync(T.rp, trp.data(), trp.size() * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(cc, 0, (size_t)m * 4, s));
    k_colfill<<<sms * 8, 256, 0, s>>>(n, G.d.rp, G.d.ci, G.d.v, T.rp, cc, T.ci, T.v);
    k_segsort<<<sms * 8, 256, 0, s>>>(m, T.rp, T.ci, T.v);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));  // trp (host) outlives the copy
    dfree(c, cc);
    T.view = {m, n, nnz, T.rp, T.ci, T.v};
    return T;
}

// fsai.cpp estimate_lambda_max on the device.
double lanczos_device(DevLA& E, const DCsr64& G, const DCsr64& Gt, const DCsr64& A, long long steps,
                      std::uint64_t seed, double* v, double* vp, double* w, double* t1, double* t2) {
    const long long n = E.n;
    if (n == 0) return 1.05;
    const int sms = sm_count();
    aspamg::Rng rng(seed);
    std::vector<double> hv((size_t)n);
    for (auto& x : hv) x = rng.symmetric();
    CK(cudaMemcpyAsync(v, hv.data(), (size_t)n * 8, cudaMemcpyHostToDevice, E.s));
    CK(cudaMemsetAsync(vp, 0, (size_t)n * 8, E.s));
    const double nv = E.norm2(v);  // synchronises: hv outlives the copy
    E.vec(V_DIV, v, nullptr, v, nv);
    std::vector<double> alpha, beta;
    double beta_prev = 0.0;
    for (long long j = 0; j < steps; ++j) {
        k_spmv_seq<<<sms * 8, 256, 0, E.s>>>(Gt, v, t1);
        k_spmv_seq<<<sms * 8, 256, 0, E.s>>>(A, t1, t2);
        k_spmv_seq<<<sms * 8, 256, 0, E.s>>>(G, t2, w);
        CK(cudaGetLastError());
        const double a = E.dot(w, v);
        alpha.push_back(a);
        k_lanczos_upd<<<E.vgrid, 256, 0, E.s>>>(n, w, v, vp, a, beta_prev);
        CK(cudaGetLastError());
        const double b = E.norm2(w);
        if (j + 1 == steps || !(b > 1e-12 * std::fabs(a))) break;
        beta.push_back(b);
        beta_prev = b;
        std::swap(vp, v);
        E.vec(V_DIV, w, nullptr, v, b);
    }
    const int m = (int)alpha.size();
    std::vector<double> T((size_t)m * m, 0.0), ev((size_t)m), evec((size_t)m * m);
    for (int i = 0; i < m; ++i) {
        T[(size_t)i * m + i] = alpha[(size_t)i];
        if (i + 1 < m) T[(size_t)i * m + i + 1] = T[(size_t)(i + 1) * m + i] = beta[(size_t)i];
    }
    aspamg::sym_eig(m, T.data(), ev.data(), evec.data());
    return 1.05 * ev[(size_t)m - 1];
}

// Level policy: operators with fewer than smoother_min_rows rows, or mean rows
// above smoother_max_mean_row (0 = no bound), are declined (status -1: the host
// computes them — small levels are latency-bound on the device); a refinement
// batch whose pattern bound would exceed smoother_max_pattern (0 = only the
// kernel's 4096 limit) is handed back (status -2, state after the last finished
// pass): the host continues the same loop from there — bit-identical either way.
double g_smoother_max_mean_row = 0.0;
double g_smoother_min_rows = 20000.0;
double g_smoother_max_pattern = 0.0;

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

double device_free_bytes() {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) return 8e9;
    return double(fr);
}

}  // namespace
}  // namespace aspamg_gpu

using namespace aspamg_gpu;

extern "C" int aspamg_gpu_set_setup_policy(const char* key, double value) {
    const std::string k = key ? key : "";
    if (k == "smoother_max_mean_row") {
        g_smoother_max_mean_row = value;
        return 0;
    }
    if (k == "smoother_min_rows") {
        g_smoother_min_rows = value;
        return 0;
    }
    if (k == "smoother_max_pattern") {
        g_smoother_max_pattern = value;
        return 0;
    }
    g_last_err = "set_setup_policy: unknown key " + k;
    return 4;
}

// fsai.cpp smoother_setup (Alg. 3) on the device, batched exactly as the host's:
// passes computed back to back per row (run_passes_device), consumed one at a
// time (Lanczos, omega, loop guards). A: host view; G written through alloc(sink,
// ...); psi[n] (host) receives the final pass's Schur complements (the host forms
// the Kaporin estimate from them).
extern "C" int aspamg_gpu_smoother_setup(void* device, const aspamg_csr_view* A, const aspamg_smoother_params* prm,
                                         aspamg_csr_alloc_fn alloc, void* sink, double* psi_out, double* omega,
                                         double* lambda_hat, int64_t* passes, int* exit_reason) {
    aspamg_gpu_ctx* c = nullptr;
    int st = aspamg_gpu_ctx_create((int)(intptr_t)device, &c);
    if (st != 0) return st;
    bool declined = false, handed = false;
    st = guard(c, [&] {
        if (!A || !prm || !alloc || !psi_out || !omega || !lambda_hat || !passes || !exit_reason)
            throw Fail{4, "smoother_setup: null argument"};
        if (A->n_rows != A->n_cols) throw Fail{1, "afsai_build: A must be square"};
        const long long n = A->n_rows;
        if (n > INT_MAX) throw Fail{1, "smoother_setup: n exceeds the int32 column range"};
        if ((g_smoother_max_mean_row > 0 && n > 0 && double(A->nnz) / double(n) > g_smoother_max_mean_row) ||
            double(n) < g_smoother_min_rows) {
            declined = true;
            return;
        }
        long long a_maxrow = 0;
        for (long long i = 0; i < n; ++i) a_maxrow = std::max<long long>(a_maxrow, A->row_offsets[i + 1] - A->row_offsets[i]);
        const DevCsr dA = upload64(c, *A);
        DevLA E;
        E.init(c, n);
        double* psi = dalloc<double>(c, (size_t)std::max<long long>(n, 1));
        double* psi2 = dalloc<double>(c, (size_t)std::max<long long>(n, 1));
        double *v = dalloc<double>(c, (size_t)n + 1), *vp = dalloc<double>(c, (size_t)n + 1),
               *w = dalloc<double>(c, (size_t)n + 1), *t1 = dalloc<double>(c, (size_t)n + 1),
               *t2 = dalloc<double>(c, (size_t)n + 1);
        auto omega_of = [](double lam) {
            if (!(lam > 0.0)) throw Fail{4, "compute_omega: lambda_hat must be positive"};
            return std::min(1.0, 2.0 / lam);
        };
        const PassParams p0{(int)prm->k0, (int)prm->rho0, prm->eps0}, pr{(int)prm->ki, (int)prm->rhoi, prm->epsi};
        Batch B;
        int next = 0, last_batch = 1, hcap_hint = 0;
        std::vector<double> lam_hist, nnzr_hist;
        const bool trace = std::getenv("ASPAMG_SETUP_TRACE") != nullptr;
        DevG G;
        // next pass from the batch (a new batch when the current one is used up);
        // false: the batch's pattern bound exceeds the policy -> hand back
        auto take = [&](bool first, DevG& out, double* ps) -> bool {
            if (next >= B.npass) {
                free_batch(c, B);
                const long long gs_max = first ? 0 : max_row(&G);
                int want = first ? 1 : 2 * last_batch;
                const size_t h = lam_hist.size();
                if (!first && h >= 2) {  // fsai.cpp take_pass: predicted remaining passes
                    const double dl = lam_hist[h - 2] - lam_hist[h - 1];
                    const double dz = nnzr_hist[h - 1] - nnzr_hist[h - 2];
                    double pred = 1e9;
                    if (dl > 0) pred = std::min(pred, (lam_hist[h - 1] - 2.0 / prm->omega_bar) / dl);
                    if (dz > 0) pred = std::min(pred, (prm->rho_bar - nnzr_hist[h - 1]) / dz);
                    if (pred < 1e9) want = std::min(want, (int)std::ceil(std::max(pred, 0.0)) + 1);
                }
                want = std::max(1, std::min(want, 16));
                const double budget = 0.5 * device_free_bytes();
                while (want > 1 && batch_bytes(n, gs_max, want, first ? p0 : pr, pr) > budget) --want;
                if (!first) {
                    const long long bound = gs_max + (long long)want * pr.k * pr.rho;
                    if ((g_smoother_max_pattern > 0 && double(gs_max + (long long)pr.k * pr.rho) > g_smoother_max_pattern) ||
                        gs_max + (long long)pr.k * pr.rho > kMaxPattern)
                        return false;
                    while (want > 1 && gs_max + (long long)want * pr.k * pr.rho > kMaxPattern) --want;
                    (void)bound;
                }
                last_batch = want;
                const double t0 = now_s();
                B = run_passes_device(c, dA.view, a_maxrow, first ? nullptr : &G, want, first ? p0 : pr, pr, &hcap_hint);
                next = 0;
                if (trace)
                    std::fprintf(stderr, "[gpu smoother n=%lld] batch of %d passes: %.2f s\n", n, want, now_s() - t0);
            }
            out = pass_device(c, B, next++, ps);
            return true;
        };
        take(true, G, psi);
        DevCsr Gt = transpose_device(c, G);
        double lam = lanczos_device(E, G.d.view, Gt.view, dA.view, prm->lanczos_steps, prm->seed, v, vp, w, t1, t2);
        double om = omega_of(lam);
        int64_t np = 0;
        int ex = 0;  // omega_reached
        while (om < prm->omega_bar) {
            const double nnz_r = n ? double(G.d.view.nnz) / double(n) : 0.0;
            if (!(nnz_r < prm->rho_bar)) { ex = 1; break; }  // density_bound
            DevG G2;
            if (!take(false, G2, psi2)) {
                handed = true;
                break;
            }
            if (G2.d.view.nnz == G.d.view.nnz) {  // pattern_stagnation
                free_g(c, G2);
                ex = 2;
                break;
            }
            free_g(c, G);
            free_csr(c, Gt);
            G = std::move(G2);
            std::swap(psi, psi2);
            Gt = transpose_device(c, G);
            lam = lanczos_device(E, G.d.view, Gt.view, dA.view, prm->lanczos_steps, prm->seed, v, vp, w, t1, t2);
            om = omega_of(lam);
            lam_hist.push_back(lam);
            nnzr_hist.push_back(n ? double(G.d.view.nnz) / double(n) : 0.0);
            ++np;
            ex = 0;
        }
        free_batch(c, B);
        int64_t *rp = nullptr, *ci = nullptr;
        double* vals = nullptr;
        const long long nnz = G.d.view.nnz;
        if (alloc(sink, n, n, nnz, &rp, &ci, &vals) != 0 || !rp || (nnz && (!ci || !vals)))
            throw Fail{5, "smoother_setup: output allocation failed"};
        // finished: sorted rows; handed back: insertion order (the host restarts from it)
        const DevCsr& out = handed ? G.ins : G.d;
        CK(cudaMemcpyAsync(rp, G.d.rp, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost, c->stream));
        if (nnz) {
            CK(cudaMemcpyAsync(ci, out.ci, sizeof(int64_t) * nnz, cudaMemcpyDeviceToHost, c->stream));
            CK(cudaMemcpyAsync(vals, out.v, sizeof(double) * nnz, cudaMemcpyDeviceToHost, c->stream));
        }
        CK(cudaMemcpyAsync(psi_out, psi, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        *omega = om;
        *lambda_hat = lam;
        *passes = np;
        *exit_reason = ex;
    });
    aspamg_gpu_ctx_destroy(c);
    return (st == 0 && declined) ? -1 : (st == 0 && handed) ? -2 : st;
}

// afsai_build alone (identity start) on the device, for verification.
extern "C" int aspamg_gpu_afsai_build(void* device, const aspamg_csr_view* A, int64_t k, int64_t rho, double eps,
                                      aspamg_csr_alloc_fn alloc, void* sink, double* psi_out) {
    aspamg_gpu_ctx* c = nullptr;
    int st = aspamg_gpu_ctx_create((int)(intptr_t)device, &c);
    if (st != 0) return st;
    st = guard(c, [&] {
        if (!A || !alloc) throw Fail{4, "afsai_build: null argument"};
        if (A->n_rows != A->n_cols) throw Fail{1, "afsai_build: A must be square"};
        const long long n = A->n_rows;
        long long a_maxrow = 0;
        for (long long i = 0; i < n; ++i) a_maxrow = std::max<long long>(a_maxrow, A->row_offsets[i + 1] - A->row_offsets[i]);
        const DevCsr dA = upload64(c, *A);
        double* psi = dalloc<double>(c, (size_t)std::max<long long>(n, 1));
        const PassParams pp{(int)k, (int)rho, eps};
        Batch B = run_passes_device(c, dA.view, a_maxrow, nullptr, 1, pp, pp);
        DevG G = pass_device(c, B, 0, psi);
        free_batch(c, B);
        int64_t *rp = nullptr, *ci = nullptr;
        double* vals = nullptr;
        const long long nnz = G.d.view.nnz;
        if (alloc(sink, n, n, nnz, &rp, &ci, &vals) != 0 || !rp || (nnz && (!ci || !vals)))
            throw Fail{5, "afsai_build: output allocation failed"};
        CK(cudaMemcpy(rp, G.d.rp, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost));
        if (nnz) {
            CK(cudaMemcpy(ci, G.d.ci, sizeof(int64_t) * nnz, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(vals, G.d.v, sizeof(double) * nnz, cudaMemcpyDeviceToHost));
        }
        if (psi_out) CK(cudaMemcpy(psi_out, psi, sizeof(double) * n, cudaMemcpyDeviceToHost));
    });
    aspamg_gpu_ctx_destroy(c);
    return st;
}
