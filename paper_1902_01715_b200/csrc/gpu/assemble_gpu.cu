// GPU setup components: assembly of the structured-hex
// elasticity stiffness K on the device (fem.cpp:87-184 semantics).
//
// Restates csrc/host/fem.cpp assemble_hex() so that K is bit-identical to the
// host's (and through tests/test_golden.py to the reference's from_triplets on
// its element-order triplet stream, sparse_matrix.cpp:18-64):
//   * element stiffness: the SAME source as the host (host/hex_stiffness.hpp),
//     this file compiled with -fmad=false (the host: -ffp-contract=off) — one
//     thread per stiffness-table entry (distinct material on undistorted cubes,
//     fem.cpp:153-158; one per element on distorted meshes);
//   * pattern: node f couples with the free nodes of its 3x3x3 neighbourhood in
//     ascending node id; degree pass on the device, node-level exclusive scan on
//     the host, rows 3f+c laid out back to back;
//   * fill: one thread per (free node, neighbour offset) owns the 3x3 block of
//     that pair and adds the contributions of the (up to 4) elements containing
//     both nodes in element order (ez, ey, ex ascending) onto -0.0 — the order in
//     which the host's direct fill and the reference's triplet sort see them.
// K leaves the device as the reference-layout CSR (int64 offsets / columns,
// fp64 values) written through the caller's allocator.
#include "ctx.cuh"
#include "../host/hex_stiffness.hpp"

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <vector>

namespace aspamg_gpu {
namespace {

struct DMesh {
    long long nx, ny, nz, mx, my, n_free, n_el;
    const double* xyz;
    const long long* free_index;
    const long long* free_node;
    const int* el_ke;
};

__global__ void k_ke_cube(int n_ke, double h, const double* __restrict__ young, const double* __restrict__ poisson,
                          double gp, double* ke) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < n_ke) aspamg::hexk::stiffness_cube(h, young[q], poisson[q], gp, ke + 576ll * q);
}

__global__ void k_ke_general(DMesh m, const double* __restrict__ young, const double* __restrict__ poisson, double gp,
                             double* ke, int* bad) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m.n_el) return;
    const long long ex = e % m.nx, ey = (e / m.nx) % m.ny, ez = e / (m.nx * m.ny);
    double xyz[8][3];
    for (int a = 0; a < 8; ++a) {
        const long long v = (ex + (a & 1)) + m.mx * ((ey + ((a >> 1) & 1)) + m.my * (ez + ((a >> 2) & 1)));
        for (int c = 0; c < 3; ++c) xyz[a][c] = m.xyz[3 * v + c];
    }
    if (!aspamg::hexk::stiffness_general(xyz, young[e], poisson[e], gp, ke + 576ll * e)) *bad = 1;
}

// Free neighbours of free node f (3x3x3 box, inside the mesh, not clamped).
__global__ void k_degree(DMesh m, int* deg) {
    const long long f = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= m.n_free) return;
    const long long v = m.free_node[f];
    const long long i = v % m.mx, j = (v / m.mx) % m.my, k = v / (m.mx * m.my);
    int d = 0;
    for (int o = 0; o < 27; ++o) {
        const long long a = i + (o % 3) - 1, b = j + ((o / 3) % 3) - 1, c = k + (o / 9) - 1;
        if (a < 0 || a > m.nx || b < 0 || b > m.ny || c < 0 || c > m.nz) continue;
        if (m.free_index[a + m.mx * (b + m.my * c)] >= 0) ++d;
    }
    deg[f] = d;
}

// Thread (f, o): the 3x3 block coupling free node f with its neighbour at
// offset o (if that node exists and is free).
__global__ void k_fill(DMesh m, const int* __restrict__ deg, const long long* __restrict__ nbase,
                       const double* __restrict__ ke, long long* col, double* val) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 27 * m.n_free) return;
    const long long f = t / 27;
    const int o = (int)(t % 27);
    const long long v = m.free_node[f];
    const long long i = v % m.mx, j = (v / m.mx) % m.my, k = v / (m.mx * m.my);
    const int di = o % 3 - 1, dj = (o / 3) % 3 - 1, dk = o / 9 - 1;
    const long long wi = i + di, wj = j + dj, wk = k + dk;
    if (wi < 0 || wi > m.nx || wj < 0 || wj > m.ny || wk < 0 || wk > m.nz) return;
    const long long g = m.free_index[wi + m.mx * (wj + m.my * wk)];
    if (g < 0) return;
    int pos = 0;  // free neighbours ahead of this one in the row (ascending node id)
    for (int q = 0; q < o; ++q) {
        const long long a = i + (q % 3) - 1, b = j + ((q / 3) % 3) - 1, c = k + (q / 9) - 1;
        if (a < 0 || a > m.nx || b < 0 || b > m.ny || c < 0 || c > m.nz) continue;
        if (m.free_index[a + m.mx * (b + m.my * c)] >= 0) ++pos;
    }
    double blk[3][3];
    for (int ca = 0; ca < 3; ++ca)
        for (int cb = 0; cb < 3; ++cb) blk[ca][cb] = -0.0;  // (-0.0) + x == x bit-exactly
    // elements containing node v, in element order; those that also contain the neighbour contribute
    for (long long ez = k - 1; ez <= k; ++ez) {
        if (ez < 0 || ez >= m.nz) continue;
        for (long long ey = j - 1; ey <= j; ++ey) {
            if (ey < 0 || ey >= m.ny) continue;
            for (long long ex = i - 1; ex <= i; ++ex) {
                if (ex < 0 || ex >= m.nx) continue;
                const long long bi = wi - ex, bj = wj - ey, bk = wk - ez;
                if (bi < 0 || bi > 1 || bj < 0 || bj > 1 || bk < 0 || bk > 1) continue;
                const long long el = ex + m.nx * (ey + m.ny * ez);
                const double* Ke = ke + 576ll * m.el_ke[el];
                const int a = (int)((i - ex) + 2 * (j - ey) + 4 * (k - ez));
                const int b = (int)(bi + 2 * bj + 4 * bk);
                for (int ca = 0; ca < 3; ++ca)
                    for (int cb = 0; cb < 3; ++cb) blk[ca][cb] += Ke[(3 * a + ca) * 24 + 3 * b + cb];
            }
        }
    }
    const long long d3 = 3ll * deg[f];
    const long long base = 9ll * nbase[f];
    for (int ca = 0; ca < 3; ++ca)
        for (int cb = 0; cb < 3; ++cb) {
            const long long at = base + ca * d3 + 3 * pos + cb;
            col[at] = 3 * g + cb;
            val[at] = blk[ca][cb];
        }
}

}  // namespace
}  // namespace aspamg_gpu

using namespace aspamg_gpu;

extern "C" int aspamg_gpu_assemble_hex(void* device, const aspamg_hex_assembly* in, aspamg_csr_alloc_fn alloc,
                                       void* sink) {
    aspamg_gpu_ctx* c = nullptr;
    int st = aspamg_gpu_ctx_create((int)(intptr_t)device, &c);
    if (st != 0) return st;
    st = guard(c, [&] {
        if (!in || !alloc) throw Fail{4, "assemble_hex: null argument"};
        if (in->nx < 1 || in->ny < 1 || in->nz < 1) throw Fail{4, "assembly: element counts must be >= 1"};
        if (in->n_free < 0 || !in->node_xyz || !in->free_index || !in->el_ke || !in->young || !in->poisson ||
            (in->n_free > 0 && !in->free_node))
            throw Fail{4, "assemble_hex: null mesh array"};
        const long long n_el = in->nx * in->ny * in->nz;
        const long long mx = in->nx + 1, my = in->ny + 1, mz = in->nz + 1;
        const long long n_nodes = mx * my * mz;
        if (in->n_ke < 1 || (!in->cube && in->n_ke != n_el)) throw Fail{4, "assemble_hex: stiffness table size"};
        if (in->cube && !(in->h > 0.0)) throw Fail{4, "hex generator: element edge lengths have to be > 0"};
        if (27 * in->n_free >= (1ll << 40)) throw Fail{4, "assemble_hex: mesh too large"};
        cudaStream_t s = c->stream;
        DMesh m{};
        m.nx = in->nx; m.ny = in->ny; m.nz = in->nz; m.mx = mx; m.my = my; m.n_free = in->n_free; m.n_el = n_el;
        double* d_xyz = dalloc<double>(c, (size_t)(3 * n_nodes));
        long long* d_fi = dalloc<long long>(c, (size_t)n_nodes);
        long long* d_fn = dalloc<long long>(c, (size_t)in->n_free);
        int* d_el = dalloc<int>(c, (size_t)n_el);
        double* d_E = dalloc<double>(c, (size_t)in->n_ke);
        double* d_nu = dalloc<double>(c, (size_t)in->n_ke);
        double* d_ke = dalloc<double>(c, (size_t)in->n_ke * 576);
        int* d_bad = dalloc<int>(c, 1);
        CK(cudaMemcpyAsync(d_xyz, in->node_xyz, sizeof(double) * 3 * n_nodes, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(d_fi, in->free_index, sizeof(long long) * n_nodes, cudaMemcpyHostToDevice, s));
        if (in->n_free)
            CK(cudaMemcpyAsync(d_fn, in->free_node, sizeof(long long) * in->n_free, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(d_el, in->el_ke, sizeof(int) * n_el, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(d_E, in->young, sizeof(double) * in->n_ke, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(d_nu, in->poisson, sizeof(double) * in->n_ke, cudaMemcpyHostToDevice, s));
        CK(cudaMemsetAsync(d_bad, 0, sizeof(int), s));
        m.xyz = d_xyz; m.free_index = d_fi; m.free_node = d_fn; m.el_ke = d_el;
        const double gp = 1.0 / std::sqrt(3.0);
        const int B = 128;
        if (in->cube)
            k_ke_cube<<<(unsigned)((in->n_ke + B - 1) / B), B, 0, s>>>((int)in->n_ke, in->h, d_E, d_nu, gp, d_ke);
        else
            k_ke_general<<<(unsigned)((n_el + B - 1) / B), B, 0, s>>>(m, d_E, d_nu, gp, d_ke, d_bad);
        CK(cudaGetLastError());
        // pattern: degrees on the device, node-level scan on the host
        std::vector<int> deg((size_t)in->n_free);
        int* d_deg = dalloc<int>(c, (size_t)in->n_free);
        if (in->n_free) {
            k_degree<<<(unsigned)((in->n_free + 255) / 256), 256, 0, s>>>(m, d_deg);
            CK(cudaGetLastError());
            CK(cudaMemcpyAsync(deg.data(), d_deg, sizeof(int) * in->n_free, cudaMemcpyDeviceToHost, s));
        }
        int bad = 0;
        CK(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (bad) throw Fail{3, "assembly: inverted or degenerate element"};
        std::vector<long long> nbase((size_t)in->n_free + 1, 0);
        for (long long f = 0; f < in->n_free; ++f) nbase[(size_t)f + 1] = nbase[(size_t)f] + deg[(size_t)f];
        const long long nnz = 9 * nbase[(size_t)in->n_free];
        int64_t *rp = nullptr, *ci = nullptr;
        double* v = nullptr;
        if (alloc(sink, 3 * in->n_free, 3 * in->n_free, nnz, &rp, &ci, &v) != 0 || !rp || (nnz && (!ci || !v)))
            throw Fail{5, "assemble_hex: output allocation failed"};
#pragma omp parallel for schedule(static)
        for (long long f = 0; f < in->n_free; ++f)
            for (int cc = 0; cc < 3; ++cc)
                rp[3 * f + cc] = 9 * nbase[(size_t)f] + 3ll * cc * deg[(size_t)f];
        rp[3 * in->n_free] = nnz;
        if (nnz) {
            long long* d_nb = dalloc<long long>(c, (size_t)in->n_free);
            long long* d_col = dalloc<long long>(c, (size_t)nnz);
            double* d_val = dalloc<double>(c, (size_t)nnz);
            CK(cudaMemcpyAsync(d_nb, nbase.data(), sizeof(long long) * in->n_free, cudaMemcpyHostToDevice, s));
            const long long nt = 27 * in->n_free;
            k_fill<<<(unsigned)((nt + 255) / 256), 256, 0, s>>>(m, d_deg, d_nb, d_ke, d_col, d_val);
            CK(cudaGetLastError());
            CK(cudaMemcpyAsync(ci, d_col, sizeof(int64_t) * nnz, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(v, d_val, sizeof(double) * nnz, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
        }
    });
    aspamg_gpu_ctx_destroy(c);
    return st;
}
