#include "smalldense.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>

namespace aspamg {

long cholesky_lower(int n, double* a) {
    for (int j = 0; j < n; ++j) {
        double d = a[j * n + j];
        for (int k = 0; k < j; ++k) d -= a[j * n + k] * a[j * n + k];
        if (!(d > 0.0)) return j;
        d = std::sqrt(d);
        a[j * n + j] = d;
        for (int i = j + 1; i < n; ++i) {
            double s = a[i * n + j];
            for (int k = 0; k < j; ++k) s -= a[i * n + k] * a[j * n + k];
            a[i * n + j] = s / d;
        }
        for (int i = 0; i < j; ++i) a[i * n + j] = 0.0;
    }
    return -1;
}

// 32 strided partial sums — partial l takes k = l, l + 32, ... in ascending
// order, each term a separate multiply and add — combined by the xor butterfly
// (16, 8, 4, 2, 1) that a warp's __shfl_xor_sync reduction performs; lane 0's
// value is the result. The device aFSAI kernel (fsai_gpu.cu dot_w32) runs the
// identical sequence, so both produce the same bits.
double dot_w32(const double* a, const double* b, int n) {
    double s[32];
    for (int l = 0; l < 32; ++l) s[l] = 0.0;
    int k = 0;
    for (; k + 32 <= n; k += 32)
        for (int l = 0; l < 32; ++l) s[l] += a[k + l] * b[k + l];
    for (int l = 0; k + l < n; ++l) s[l] += a[k + l] * b[k + l];
    for (int h = 16; h >= 1; h >>= 1)  // lanes < h keep s_l + s_{l xor h} (= s_l + s_{l+h})
        for (int l = 0; l < h; ++l) s[l] = s[l] + s[l + h];
    return s[0];
}

// Blocked in 32-row blocks, the order of a warp with lane l on row B + l:
// t_i = L_i[0..B) . b[0..B) as one sequential chain, b_i -= t_i; then inside the
// block, right-looking: b_j /= L_jj, b_i -= L_ij b_j for the block's rows i > j.
void trsv_lower(int n, const double* L, int ld, double* b) {
    for (int B = 0; B < n; B += 32) {
        const int nb = std::min(32, n - B);
        double bi[32];
        for (int l = 0; l < nb; ++l) {
            const double* Li = L + (size_t)(B + l) * ld;
            double t = 0.0;
            for (int k = 0; k < B; ++k) t += Li[k] * b[k];
            bi[l] = b[B + l] - t;
        }
        for (int j = 0; j < nb; ++j) {
            bi[j] = bi[j] / L[(size_t)(B + j) * ld + B + j];
            for (int l = j + 1; l < nb; ++l) bi[l] = bi[l] - L[(size_t)(B + l) * ld + B + j] * bi[j];
        }
        for (int l = 0; l < nb; ++l) b[B + l] = bi[l];
    }
}

// Right-looking: b_i /= L_ii, then b_k -= L_ik b_i for k < i (i descending).
void trsv_lower_t(int n, const double* L, int ld, double* b) {
    for (int i = n - 1; i >= 0; --i) {
        const double* Li = L + (size_t)i * ld;
        const double bi = b[i] / Li[i];
        b[i] = bi;
        for (int k = 0; k < i; ++k) b[k] = b[k] - Li[k] * bi;
    }
}

void sym_eig(int n, double* a, double* w, double* v) {
    std::vector<double> V(static_cast<size_t>(n) * n, 0.0);
    for (int i = 0; i < n; ++i) V[static_cast<size_t>(i) * n + i] = 1.0;
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0, tot = 0.0;
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) {
                const double x = a[i * n + j] * a[i * n + j];
                tot += x;
                if (i != j) off += x;
            }
        if (off <= 1e-30 * tot || off == 0.0) break;
        for (int p = 0; p < n - 1; ++p)
            for (int q = p + 1; q < n; ++q) {
                const double apq = a[p * n + q];
                if (apq == 0.0) continue;
                const double app = a[p * n + p], aqq = a[q * n + q];
                const double theta = (aqq - app) / (2.0 * apq);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
                const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
                for (int k = 0; k < n; ++k) {  // columns p, q
                    const double akp = a[k * n + p], akq = a[k * n + q];
                    a[k * n + p] = c * akp - s * akq;
                    a[k * n + q] = s * akp + c * akq;
                }
                for (int k = 0; k < n; ++k) {  // rows p, q
                    const double apk = a[p * n + k], aqk = a[q * n + k];
                    a[p * n + k] = c * apk - s * aqk;
                    a[q * n + k] = s * apk + c * aqk;
                }
                for (int k = 0; k < n; ++k) {
                    const double vkp = V[static_cast<size_t>(k) * n + p], vkq = V[static_cast<size_t>(k) * n + q];
                    V[static_cast<size_t>(k) * n + p] = c * vkp - s * vkq;
                    V[static_cast<size_t>(k) * n + q] = s * vkp + c * vkq;
                }
            }
    }
    std::vector<int> ord(static_cast<size_t>(n));
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return a[x * n + x] < a[y * n + y]; });
    for (int k = 0; k < n; ++k) {
        w[k] = a[ord[static_cast<size_t>(k)] * n + ord[static_cast<size_t>(k)]];
        for (int i = 0; i < n; ++i) v[i * n + k] = V[static_cast<size_t>(i) * n + ord[static_cast<size_t>(k)]];
    }
}

}  // namespace aspamg
