// GPU setup components: SRQCG test-space generation
// (Alg. 4 :522-563) on the device, reusing the
// solve's bit-exact SpMV kernels for S = G A G'.
//
// The device run is a restatement of the host srqcg (csrc/host/testspace.cpp)
// with every floating-point operation in the same order:
//   * products y = M x : the sliced-BSR3 / SELL kernels (lane per row, ascending
//     sequential sums, __dmul_rn/__dadd_rn) — bit-identical to spmv() in core.cpp;
//   * dots : core.cpp dot() — 8192-element chunks summed sequentially from 0.0,
//     chunk partials summed in index order — restated by k_mdot (one CTA per
//     chunk, chunk rows staged through shared memory, one thread per dot chain)
//     with the partials summed on the host in index order;
//   * vector updates : elementwise with explicit round-to-nearest intrinsics (no
//     FMA contraction, as the host build's -ffp-contract=off);
//   * Ritz eigenproblem (m x m) and Rng reseeding: on the host, same code.
// Hence GPU and CPU test spaces are bit-identical, and so is every hierarchy
// built from them (tests/test_gpu_setup.py).
#include "setup_common.cuh"
#include "../host/core.hpp"
#include "../host/smalldense.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <vector>

namespace aspamg_gpu {
namespace {

// Zn(i, c) = sum_r Z(i, r) U[r m + c] (and the same for SZ), r ascending from 0.0.
__global__ void k_ritz_combine(long long n, int m, const double* __restrict__ Z, const double* __restrict__ SZ,
                               const double* __restrict__ U, double* Zn, double* SZn) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        for (int c = 0; c < m; ++c) {
            double s1 = 0.0, s2 = 0.0;
            for (int r = 0; r < m; ++r) {
                const double u = __ldg(U + (size_t)r * m + c);
                s1 = __dadd_rn(s1, __dmul_rn(Z[(size_t)r * n + i], u));
                s2 = __dadd_rn(s2, __dmul_rn(SZ[(size_t)r * n + i], u));
            }
            Zn[(size_t)c * n + i] = s1;
            SZn[(size_t)c * n + i] = s2;
        }
}

// Device SRQCG engine.
struct Srq : DevLA {
    DMat A, G, Gt;
    double *t1 = nullptr, *t2 = nullptr;

    void sapply(const double* x, double* y) {  // y = G A G' x (testspace.cpp SOp::apply)
        spmv(Gt, EPI_PLAIN, x, t1, nullptr, 1.0, nullptr, Red{}, nullptr, Launch{0, s});
        spmv(A, EPI_PLAIN, t1, t2, nullptr, 1.0, nullptr, Red{}, nullptr, Launch{0, s});
        spmv(G, EPI_PLAIN, t2, y, nullptr, 1.0, nullptr, Red{}, nullptr, Launch{0, s});
    }
    void gt_apply(const double* x, double* y) {
        spmv(Gt, EPI_PLAIN, x, y, nullptr, 1.0, nullptr, Red{}, nullptr, Launch{0, s});
    }
    // core.cpp orthonormalize_columns on an n x m column-major device block.
    long long orthonormalize(double* B, long long m, double* v, double drop_tol = 1e-12) {
        long long kept = 0;
        for (long long j = 0; j < m; ++j) {
            copy(B + j * n, v);
            const double original = norm2(v);
            for (int pass = 0; pass < 2; ++pass)
                for (long long q = 0; q < kept; ++q) {
                    const double cq = dot(B + q * n, v);
                    vec(V_MINUS_CX, B + q * n, nullptr, v, cq);
                }
            const double rem = norm2(v);
            if (original == 0.0 || rem <= drop_tol * original) continue;
            vec(V_DIV, v, nullptr, B + kept * n, rem);
            ++kept;
        }
        return kept;
    }
    void upload_col(double* dst, const std::vector<double>& h) {
        CK(cudaMemcpyAsync(dst, h.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));
    }
};

struct SrqOut {
    long long m_out = 0, iterations = 0;
    bool rank_collapse = false;
};

// testspace.cpp srqcg(), operation for operation.
SrqOut run_srqcg(Srq& E, const double* V0_host, long long m, long long k_max, long long k_ritz, double tol,
                 std::uint64_t seed, double* V_host, double* q_host) {
    const long long n = E.n;
    aspamg_gpu_ctx* c = E.c;
    SrqOut out;
    const size_t nm = (size_t)n * (size_t)std::max<long long>(m, 1);
    double* Z = dalloc<double>(c, nm);
    double* SZ = dalloc<double>(c, nm);
    double* P = dalloc<double>(c, nm);
    double* SP = dalloc<double>(c, nm);
    double* R = dalloc<double>(c, nm);
    double* Zn = dalloc<double>(c, nm);
    double* SZn = dalloc<double>(c, nm);
    double* V0 = dalloc<double>(c, nm);
    double* gi = dalloc<double>(c, (size_t)n);
    double* tmp = dalloc<double>(c, (size_t)n);
    double* Ud = dalloc<double>(c, (size_t)std::max<long long>(m * m, 1));
    CK(cudaMemcpyAsync(V0, V0_host, sizeof(double) * n * m, cudaMemcpyHostToDevice, E.s));
    // Z0 = (I - S) V0
    for (long long j = 0; j < m; ++j) {
        E.sapply(V0 + j * n, Z + j * n);
        E.vec(V_SUBFROM, V0 + j * n, nullptr, Z + j * n);
    }
    const long long want = m;
    long long nt = E.orthonormalize(Z, m, tmp);
    if (nt < want) {
        out.rank_collapse = true;
        aspamg::Rng rng(aspamg::derive_seed(seed, 77));
        std::vector<double> col((size_t)n);
        for (long long j = nt; j < want; ++j) {
            for (long long i = 0; i < n; ++i) col[(size_t)i] = rng.symmetric();
            E.upload_col(Z + j * n, col);
        }
        nt = E.orthonormalize(Z, want, tmp);
    }
    std::vector<double> q((size_t)nt), f((size_t)nt, 1.0);
    std::vector<char> conv((size_t)nt, 0);
    auto col = [&](double* B, long long i) { return B + i * n; };
    auto residual = [&](long long i) {
        const auto ef = E.dots({{col(Z, i), col(SZ, i)}, {col(Z, i), col(Z, i)}});
        f[(size_t)i] = ef[1];
        q[(size_t)i] = ef[0] / f[(size_t)i];
        const double qi = q[(size_t)i];
        E.vec(V_RESID, col(SZ, i), col(Z, i), col(R, i), qi);
        return E.norm2(col(R, i)) <= tol * std::fabs(qi) * std::sqrt(f[(size_t)i]);
    };
    for (long long i = 0; i < nt; ++i) {
        E.sapply(col(Z, i), col(SZ, i));
        conv[(size_t)i] = residual(i);
        E.vec(V_TWICE, col(R, i), nullptr, col(P, i));
        f[(size_t)i] = 1.0;
        E.sapply(col(P, i), col(SP, i));
    }
    bool all_conv = std::all_of(conv.begin(), conv.end(), [](char x) { return x != 0; });
    for (long long k = 1; !all_conv && k_max > 0; ++k) {
        if (k_ritz > 0 && k % k_ritz == 0) {
            const int mm = (int)nt;
            for (int j = 0; j < mm; ++j) {
                double* zj = col(Z, j);
                double* szj = col(SZ, j);
                const double orig = E.norm2(zj);
                for (int pass = 0; pass < 2; ++pass)
                    for (int qq = 0; qq < j; ++qq) {
                        const double cq = E.dot(col(Z, qq), zj);
                        E.vec(V_AXPY, col(Z, qq), nullptr, zj, -cq);
                        E.vec(V_AXPY, col(SZ, qq), nullptr, szj, -cq);
                    }
                double nr = E.norm2(zj);
                if (!(nr > 1e-10 * orig)) {
                    out.rank_collapse = true;
                    aspamg::Rng rng(aspamg::derive_seed(seed, 1000 + static_cast<std::uint64_t>(k) * 64 + static_cast<std::uint64_t>(j)));
                    std::vector<double> h((size_t)n);
                    for (long long i = 0; i < n; ++i) h[(size_t)i] = rng.symmetric();
                    E.upload_col(zj, h);
                    for (int pass = 0; pass < 2; ++pass)
                        for (int qq = 0; qq < j; ++qq) E.vec(V_AXPY, col(Z, qq), nullptr, zj, -E.dot(col(Z, qq), zj));
                    nr = E.norm2(zj);
                    E.sapply(zj, szj);
                }
                const double inv = 1.0 / nr;
                E.vec(V_SCALE_IP, nullptr, nullptr, zj, inv);
                E.vec(V_SCALE_IP, nullptr, nullptr, szj, inv);
            }
            std::vector<Pair> pr;
            for (int a1 = 0; a1 < mm; ++a1)
                for (int b1 = 0; b1 <= a1; ++b1) {
                    pr.push_back({col(Z, a1), col(SZ, b1)});
                    pr.push_back({col(Z, b1), col(SZ, a1)});
                }
            const std::vector<double> dv = E.dots(pr);
            std::vector<double> M1((size_t)mm * mm);
            size_t t = 0;
            for (int a1 = 0; a1 < mm; ++a1)
                for (int b1 = 0; b1 <= a1; ++b1, t += 2) {
                    const double v = 0.5 * (dv[t] + dv[t + 1]);
                    M1[(size_t)a1 * mm + b1] = M1[(size_t)b1 * mm + a1] = v;
                }
            std::vector<double> w((size_t)mm), U((size_t)mm * mm);
            aspamg::sym_eig(mm, M1.data(), w.data(), U.data());
            CK(cudaMemcpyAsync(Ud, U.data(), sizeof(double) * U.size(), cudaMemcpyHostToDevice, E.s));
            k_ritz_combine<<<E.vgrid, 256, 0, E.s>>>(n, mm, Z, SZ, Ud, Zn, SZn);
            CK(cudaGetLastError());
            CK(cudaStreamSynchronize(E.s));  // U (host) outlives the copy
            std::swap(Z, Zn);
            std::swap(SZ, SZn);
        }
        all_conv = true;
        for (long long i = 0; i < nt; ++i) {
            double* z = col(Z, i);
            double* sz = col(SZ, i);
            double* p = col(P, i);
            double* spp = col(SP, i);
            double fi = 0, a = 0, b = 0, cc = 0, d = 0, e = 0, disc = 0, den = 0;
            auto coeffs = [&](bool with_f) {
                std::vector<Pair> pr = {{p, sz}, {p, spp}, {p, z}, {p, p}, {z, sz}};
                if (with_f) pr.push_back({z, z});
                const auto r = E.dots(pr);
                a = r[0]; b = r[1]; cc = r[2]; d = r[3]; e = r[4];
                if (with_f) fi = r[5];
                den = b * cc - a * d;
                disc = (d * e - b * fi) * (d * e - b * fi) - 4.0 * den * (a * fi - cc * e);
            };
            coeffs(true);
            bool ok = disc >= 0.0 && std::fabs(den) >= 1e-300;
            if (!ok) {
                const double qi = e / fi;
                E.vec(V_SD, sz, z, p, qi, fi);
                E.sapply(p, spp);
                coeffs(false);
                ok = disc >= 0.0 && std::fabs(den) >= 1e-300;
            }
            if (ok) {
                const double alpha = (d * e - b * fi + std::sqrt(disc)) / (2.0 * den);
                E.vec(V_AXPY, p, nullptr, z, alpha);
                E.vec(V_AXPY, spp, nullptr, sz, alpha);
            }
            conv[(size_t)i] = residual(i);
            if (!conv[(size_t)i]) all_conv = false;
            const double inv = 2.0 / f[(size_t)i];
            E.vec(V_SCALE, col(R, i), nullptr, gi, inv);
            const auto bg = E.dots({{p, spp}, {gi, spp}});
            const double bb = bg[0];
            const double beta = bb != 0.0 ? -bg[1] / bb : 0.0;
            E.vec(V_PUPD, gi, nullptr, p, beta);
            E.sapply(p, spp);
        }
        out.iterations = k;
        if (k >= k_max) break;
    }
    std::vector<long long> ord((size_t)nt);
    std::iota(ord.begin(), ord.end(), 0LL);
    std::stable_sort(ord.begin(), ord.end(), [&](long long x, long long y) { return q[(size_t)x] < q[(size_t)y]; });
    double* V = Zn;  // free after the last Ritz swap
    std::vector<double> qs;
    for (long long cix = 0; cix < nt; ++cix) {
        E.gt_apply(col(Z, ord[(size_t)cix]), col(V, cix));
        qs.push_back(q[(size_t)ord[(size_t)cix]]);
    }
    const long long kept = E.orthonormalize(V, nt, tmp);
    if (kept < nt) out.rank_collapse = true;
    CK(cudaMemcpyAsync(V_host, V, sizeof(double) * n * kept, cudaMemcpyDeviceToHost, E.s));
    CK(cudaStreamSynchronize(E.s));
    for (long long i = 0; i < kept; ++i) q_host[i] = qs[(size_t)i];
    out.m_out = kept;
    return out;
}

}  // namespace
}  // namespace aspamg_gpu

using namespace aspamg_gpu;

extern "C" int aspamg_gpu_srqcg(void* device, const aspamg_csr_view* A, const aspamg_csr_view* G,
                                const aspamg_csr_view* Gt, const double* V0, int64_t m, int64_t k_max,
                                int64_t k_ritz, double tol, uint64_t seed, double* V, double* quotients,
                                int64_t* m_out, int64_t* iterations, int* rank_collapse) {
    aspamg_gpu_ctx* c = nullptr;
    const int dev = (int)(intptr_t)device;
    int st = aspamg_gpu_ctx_create(dev, &c);
    if (st != 0) return st;
    st = guard(c, [&] {
        if (!A || !G || !Gt || !V0 || !V || !quotients || !m_out) throw Fail{4, "srqcg: null argument"};
        const long long n = A->n_rows;
        if (A->n_cols != n || G->n_rows != n || G->n_cols != n || Gt->n_rows != n || Gt->n_cols != n)
            throw Fail{1, "srqcg: operator dimensions mismatch"};
        if (m < 1 || m > 64) throw Fail{4, "srqcg: m must be in [1, 64]"};
        if (n > (1ll << 31) - 1) throw Fail{1, "srqcg: n exceeds the int32 device index range"};
        // exact-order operands: sliced BSR3 where A is 3x3-blocked, SELL-32 in
        // natural row order otherwise (lane per row, sequential sums)
        c->opt_sell_chh = 32;
        c->opt_sell_min_rows = 0;
        c->opt_sell_min_mean = 0;
        c->opt_sell_max_mean = 1ll << 40;
        c->opt_sell_max_len = 1ll << 30;
        Srq E;
        E.init(c, n);
        E.A = upload_mat(c, *A, true);
        E.G = upload_mat(c, *G, false);
        E.Gt = upload_mat(c, *Gt, false);
        E.t1 = dalloc<double>(c, (size_t)n);
        E.t2 = dalloc<double>(c, (size_t)n);
        const SrqOut o = run_srqcg(E, V0, m, k_max, k_ritz, tol, seed, V, quotients);
        *m_out = o.m_out;
        if (iterations) *iterations = o.iterations;
        if (rank_collapse) *rank_collapse = o.rank_collapse ? 1 : 0;
    });
    aspamg_gpu_ctx_destroy(c);
    return st;
}
