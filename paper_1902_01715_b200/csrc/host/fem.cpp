// Structured hex elasticity generator; see fem.hpp for the reference mapping.
#include "fem.hpp"
#include "hex_stiffness.hpp"

#include <algorithm>
#include <cmath>
#include <map>
#include <omp.h>

namespace aspamg {

// fem.cpp:9-14
void Material::validate() const {
    const bool e_ok = std::isfinite(young_modulus) && young_modulus > 0.0;
    const bool nu_ok = poisson_ratio > -1.0 && poisson_ratio < 0.5;  // NaN fails both comparisons
    if (!e_ok) throw ConfigError("Material: E = " + std::to_string(young_modulus) + " is not a finite positive modulus");
    if (!nu_ok) throw ConfigError("Material: nu = " + std::to_string(poisson_ratio) + " is outside the open interval (-1, 1/2)");
}

// fem.cpp:37-85 (regular grid: constant Jacobian 2/h, det h^3/8); the arithmetic
// lives in hex_stiffness.hpp, shared with the device assembler.
void hex_element_stiffness_cube(double h, const Material& m, double Ke[24][24]) {
    m.validate();
    if (!(h > 0.0)) throw ConfigError("hex generator: element edge lengths have to be > 0");
    hexk::stiffness_cube(h, m.young_modulus, m.poisson_ratio, 1.0 / std::sqrt(3.0), &Ke[0][0]);
}

// General isoparametric trilinear hex (extension for distorted meshes, C3).
void hex_element_stiffness(const double xyz[8][3], const Material& m, double Ke[24][24]) {
    m.validate();
    if (!hexk::stiffness_general(xyz, m.young_modulus, m.poisson_ratio, 1.0 / std::sqrt(3.0), &Ke[0][0]))
        throw NumericalError("assembly: inverted or degenerate element");
}

GeneratedProblem assemble_hex(const MeshSpec& mesh, const std::vector<Material>& materials) {
    const index_t nx = mesh.nx, ny = mesh.ny, nz = mesh.nz;
    if (nx < 1 || ny < 1 || nz < 1) throw ConfigError("assembly: element counts must be >= 1");
    if (!(mesh.hx > 0.0) || !(mesh.hy > 0.0) || !(mesh.hz > 0.0))
        throw ConfigError("hex generator: element edge lengths have to be > 0");
    const index_t n_el = nx * ny * nz;
    if (static_cast<index_t>(materials.size()) != n_el)
        throw ConfigError("assembly: one material per element required");
    for (const auto& m : materials) m.validate();

    const index_t mx = nx + 1, my = ny + 1, mz = nz + 1;
    const index_t n_nodes = mx * my * mz;
    auto node_id = [&](index_t i, index_t j, index_t k) { return i + mx * (j + my * k); };

    GeneratedProblem P;
    P.mesh = mesh;
    P.n_nodes = n_nodes;
    // Node coordinates (+ interior perturbation, node order, 3 draws per interior node).
    P.node_xyz.resize(static_cast<size_t>(3 * n_nodes));
    {
        Rng rng(mesh.perturb_seed);
        for (index_t k = 0; k < mz; ++k)
            for (index_t j = 0; j < my; ++j)
                for (index_t i = 0; i < mx; ++i) {
                    const index_t v = node_id(i, j, k);
                    double x = mesh.hx * double(i), y = mesh.hy * double(j), z = mesh.hz * double(k);
                    if (mesh.perturb > 0.0 && i > 0 && i < nx && j > 0 && j < ny && k > 0 && k < nz) {
                        x += rng.symmetric() * mesh.perturb * mesh.hx;
                        y += rng.symmetric() * mesh.perturb * mesh.hy;
                        z += rng.symmetric() * mesh.perturb * mesh.hz;
                    }
                    P.node_xyz[static_cast<size_t>(3 * v + 0)] = x;
                    P.node_xyz[static_cast<size_t>(3 * v + 1)] = y;
                    P.node_xyz[static_cast<size_t>(3 * v + 2)] = z;
                }
    }
    // Clamp (fem.cpp:101-117, extended to a face set) and free numbering (fem.cpp:119-122).
    auto clamped = [&](index_t i, index_t j, index_t k) {
        const unsigned c = mesh.clamped;
        return ((c & FACE_XMIN) && i == 0) || ((c & FACE_XMAX) && i == nx) ||
               ((c & FACE_YMIN) && j == 0) || ((c & FACE_YMAX) && j == ny) ||
               ((c & FACE_ZMIN) && k == 0) || ((c & FACE_ZMAX) && k == nz);
    };
    P.free_index.assign(static_cast<size_t>(n_nodes), -1);
    index_t n_free = 0;
    for (index_t k = 0; k < mz; ++k)
        for (index_t j = 0; j < my; ++j)
            for (index_t i = 0; i < mx; ++i)
                if (!clamped(i, j, k)) P.free_index[static_cast<size_t>(node_id(i, j, k))] = n_free++;
    P.n_free = n_free;
    P.coords.resize(static_cast<size_t>(3 * n_free));
    std::vector<index_t> free_node(static_cast<size_t>(n_free));
    for (index_t v = 0; v < n_nodes; ++v) {
        const index_t f = P.free_index[static_cast<size_t>(v)];
        if (f < 0) continue;
        free_node[static_cast<size_t>(f)] = v;
        for (int c = 0; c < 3; ++c)
            P.coords[static_cast<size_t>(3 * f + c)] = P.node_xyz[static_cast<size_t>(3 * v + c)];
    }

    // Element stiffness: one per distinct material on undistorted isotropic
    // cubes (the reference caches by material, fem.cpp:153-158); per element
    // on distorted / anisotropic meshes.
    const bool cube = mesh.perturb == 0.0 && mesh.hx == mesh.hy && mesh.hy == mesh.hz;
    std::vector<int> el_ke(static_cast<size_t>(n_el));
    std::vector<double> ke_young, ke_poisson;  // material of each stiffness-table entry
    if (cube) {
        std::map<std::pair<double, double>, int> seen;
        for (index_t e = 0; e < n_el; ++e) {
            const auto key = std::make_pair(materials[static_cast<size_t>(e)].young_modulus,
                                            materials[static_cast<size_t>(e)].poisson_ratio);
            auto it = seen.find(key);
            if (it == seen.end()) {
                it = seen.emplace(key, static_cast<int>(ke_young.size())).first;
                ke_young.push_back(key.first);
                ke_poisson.push_back(key.second);
            }
            el_ke[static_cast<size_t>(e)] = it->second;
        }
    } else {
        ke_young.resize(static_cast<size_t>(n_el));
        ke_poisson.resize(static_cast<size_t>(n_el));
        for (index_t e = 0; e < n_el; ++e) {
            ke_young[static_cast<size_t>(e)] = materials[static_cast<size_t>(e)].young_modulus;
            ke_poisson[static_cast<size_t>(e)] = materials[static_cast<size_t>(e)].poisson_ratio;
            el_ke[static_cast<size_t>(e)] = static_cast<int>(e);
        }
    }
    Csr& K = P.stiffness;
    K.n_rows = K.n_cols = 3 * n_free;
    K.symmetric = true;

    // Assembly backend: element stiffness, pattern and fill on
    // the device (aspamg_gpu_assemble_hex), bit-identical to the host path below.
    if (assembly_backend_set()) {
        aspamg_hex_assembly in{};
        in.nx = nx; in.ny = ny; in.nz = nz;
        in.n_free = n_free;
        in.cube = cube ? 1 : 0;
        in.h = mesh.hx;
        in.node_xyz = P.node_xyz.data();
        in.free_index = P.free_index.data();
        in.free_node = free_node.data();
        in.el_ke = el_ke.data();
        in.n_ke = static_cast<int64_t>(ke_young.size());
        in.young = ke_young.data();
        in.poisson = ke_poisson.data();
        assemble_external(in, K);
        return P;
    }

    std::vector<std::array<double, 576>> ke_table(ke_young.size());
    if (cube) {
        for (size_t q = 0; q < ke_table.size(); ++q)
            hex_element_stiffness_cube(mesh.hx, Material{ke_young[q], ke_poisson[q]},
                                       reinterpret_cast<double(*)[24]>(ke_table[q].data()));
    } else {
#pragma omp parallel for schedule(static) num_threads(num_threads())
        for (index_t e = 0; e < n_el; ++e) {
            const index_t ex = e % nx, ey = (e / nx) % ny, ez = e / (nx * ny);
            double xyz[8][3];
            for (int a = 0; a < 8; ++a) {
                const index_t v = node_id(ex + (a & 1), ey + ((a >> 1) & 1), ez + ((a >> 2) & 1));
                for (int c = 0; c < 3; ++c) xyz[a][c] = P.node_xyz[static_cast<size_t>(3 * v + c)];
            }
            hex_element_stiffness(xyz, materials[static_cast<size_t>(e)],
                                  reinterpret_cast<double(*)[24]>(ke_table[static_cast<size_t>(e)].data()));
        }
    }

    // CSR pattern: row node f couples with every free node in its 3x3x3
    // neighbourhood; neighbours ascend in node id == ascending free id.
    std::vector<index_t> deg(static_cast<size_t>(n_free));
#pragma omp parallel for schedule(static) num_threads(num_threads())
    for (index_t f = 0; f < n_free; ++f) {
        const index_t v = free_node[static_cast<size_t>(f)];
        const index_t i = v % mx, j = (v / mx) % my, k = v / (mx * my);
        index_t d = 0;
        for (index_t dk = -1; dk <= 1; ++dk)
            for (index_t dj = -1; dj <= 1; ++dj)
                for (index_t di = -1; di <= 1; ++di) {
                    const index_t a = i + di, b = j + dj, c = k + dk;
                    if (a < 0 || a > nx || b < 0 || b > ny || c < 0 || c > nz) continue;
                    if (P.free_index[static_cast<size_t>(node_id(a, b, c))] >= 0) ++d;
                }
        deg[static_cast<size_t>(f)] = d;
    }
    K.rowptr.assign(static_cast<size_t>(3 * n_free) + 1, 0);
    for (index_t f = 0; f < n_free; ++f)
        for (int c = 0; c < 3; ++c)
            K.rowptr[static_cast<size_t>(3 * f + c) + 1] = 3 * deg[static_cast<size_t>(f)];
    for (size_t r = 1; r < K.rowptr.size(); ++r) K.rowptr[r] += K.rowptr[r - 1];
    K.col.resize(static_cast<size_t>(K.rowptr.back()));
    K.val.assign(static_cast<size_t>(K.rowptr.back()), -0.0);  // (-0.0) + x == x bit-exactly

#pragma omp parallel for schedule(static) num_threads(num_threads())
    for (index_t f = 0; f < n_free; ++f) {
        const index_t v = free_node[static_cast<size_t>(f)];
        const index_t i = v % mx, j = (v / mx) % my, k = v / (mx * my);
        int slot[27];  // offset (di,dj,dk) -> neighbour position in the row, or -1
        int pos = 0;
        for (int o = 0; o < 27; ++o) {
            const index_t a = i + (o % 3) - 1, b = j + ((o / 3) % 3) - 1, c = k + (o / 9) - 1;
            slot[o] = -1;
            if (a < 0 || a > nx || b < 0 || b > ny || c < 0 || c > nz) continue;
            const index_t g = P.free_index[static_cast<size_t>(node_id(a, b, c))];
            if (g < 0) continue;
            slot[o] = pos;
            for (int cc = 0; cc < 3; ++cc) {
                const index_t base = K.rowptr[static_cast<size_t>(3 * f + cc)];
                for (int cb = 0; cb < 3; ++cb)
                    K.col[static_cast<size_t>(base + 3 * pos + cb)] = 3 * g + cb;
            }
            ++pos;
        }
        // Elements containing node v, in element order (ez, ey, ex ascending).
        for (index_t ez = k - 1; ez <= k; ++ez) {
            if (ez < 0 || ez >= nz) continue;
            for (index_t ey = j - 1; ey <= j; ++ey) {
                if (ey < 0 || ey >= ny) continue;
                for (index_t ex = i - 1; ex <= i; ++ex) {
                    if (ex < 0 || ex >= nx) continue;
                    const index_t el = ex + nx * (ey + ny * ez);
                    const double* Ke = ke_table[static_cast<size_t>(el_ke[static_cast<size_t>(el)])].data();
                    const int a = static_cast<int>((i - ex) + 2 * (j - ey) + 4 * (k - ez));
                    for (int b = 0; b < 8; ++b) {
                        const index_t bi = ex + (b & 1), bj = ey + ((b >> 1) & 1), bk = ez + ((b >> 2) & 1);
                        const int o = static_cast<int>((bi - i + 1) + 3 * (bj - j + 1) + 9 * (bk - k + 1));
                        const int p = slot[o];
                        if (p < 0) continue;  // clamped neighbour
                        for (int ca = 0; ca < 3; ++ca) {
                            const index_t base = K.rowptr[static_cast<size_t>(3 * f + ca)] + 3 * p;
                            for (int cb = 0; cb < 3; ++cb)
                                K.val[static_cast<size_t>(base + cb)] += Ke[(3 * a + ca) * 24 + 3 * b + cb];
                        }
                    }
                }
            }
        }
    }
    return P;
}

// fem.cpp:192-221
Dense rigid_body_modes(const std::vector<double>& coords, index_t n, bool* rank_deficient) {
    double cx = 0, cy = 0, cz = 0;
    if (n > 0) {  // Eigen colwise().mean(): plain sum / n
        for (index_t v = 0; v < n; ++v) {
            cx += coords[static_cast<size_t>(3 * v)];
            cy += coords[static_cast<size_t>(3 * v + 1)];
            cz += coords[static_cast<size_t>(3 * v + 2)];
        }
        cx /= double(n); cy /= double(n); cz /= double(n);
    }
    Dense M(3 * n, 6);
    for (index_t v = 0; v < n; ++v) {
        const double dx = coords[static_cast<size_t>(3 * v)] - cx;
        const double dy = coords[static_cast<size_t>(3 * v + 1)] - cy;
        const double dz = coords[static_cast<size_t>(3 * v + 2)] - cz;
        M(3 * v + 0, 0) = 1.0;
        M(3 * v + 1, 1) = 1.0;
        M(3 * v + 2, 2) = 1.0;
        M(3 * v + 1, 3) = -dz; M(3 * v + 2, 3) = dy;   // rotation-x
        M(3 * v + 0, 4) = dz;  M(3 * v + 2, 4) = -dx;  // rotation-y
        M(3 * v + 0, 5) = -dy; M(3 * v + 1, 5) = dx;   // rotation-z
    }
    const index_t dropped = orthonormalize_columns(M);
    if (rank_deficient) *rank_deficient = dropped > 0;
    return M;
}

std::vector<double> rhs_ones(const GeneratedProblem& p) {
    return std::vector<double>(static_cast<size_t>(3 * p.n_free), 1.0);
}

std::vector<double> rhs_top_nodal(const GeneratedProblem& p, double fz) {
    std::vector<double> b(static_cast<size_t>(3 * p.n_free), 0.0);
    const auto& m = p.mesh;
    const index_t mx = m.nx + 1, my = m.ny + 1;
    for (index_t j = 0; j < my; ++j)
        for (index_t i = 0; i < mx; ++i) {
            const index_t f = p.free_index[static_cast<size_t>(i + mx * (j + my * m.nz))];
            if (f >= 0) b[static_cast<size_t>(3 * f + 2)] = fz;
        }
    return b;
}

std::vector<double> rhs_top_pressure(const GeneratedProblem& p, double pressure) {
    std::vector<double> b(static_cast<size_t>(3 * p.n_free), 0.0);
    const auto& m = p.mesh;
    const index_t mx = m.nx + 1, my = m.ny + 1;
    const double share = pressure * m.hx * m.hy / 4.0;
    for (index_t ey = 0; ey < m.ny; ++ey)
        for (index_t ex = 0; ex < m.nx; ++ex)
            for (int c = 0; c < 4; ++c) {
                const index_t i = ex + (c & 1), j = ey + (c >> 1);
                const index_t f = p.free_index[static_cast<size_t>(i + mx * (j + my * m.nz))];
                if (f >= 0) b[static_cast<size_t>(3 * f + 2)] -= share;
            }
    return b;
}

std::vector<double> rhs_gaussian(const GeneratedProblem& p, std::uint64_t seed) {
    Rng rng(seed);
    std::vector<double> b(static_cast<size_t>(3 * p.n_free));
    for (auto& x : b) x = rng.gaussian();
    return b;
}

GeneratedProblem make_config(int cfg, index_t scale, std::vector<double>& rhs) {
    if (scale < 1) scale = 1;
    const std::uint64_t base = 1234;  // SPEC.md:219 global seed; salts per SURVEY.md §8d
    auto sc = [&](index_t n, index_t lo) { return std::max(lo, n / scale); };
    MeshSpec mesh;
    std::vector<Material> mats;
    switch (cfg) {
        case 1: {
            mesh.nx = mesh.ny = mesh.nz = sc(20, 2);
            mesh.hx = mesh.hy = mesh.hz = 1.0 / double(mesh.nx);
            mesh.clamped = FACE_ZMIN;
            mats.assign(static_cast<size_t>(mesh.nx * mesh.ny * mesh.nz), Material{1.0, 0.3});
            break;
        }
        case 2: {
            mesh.nx = mesh.ny = mesh.nz = sc(64, 2);
            mesh.hx = mesh.hy = mesh.hz = 1.0 / double(mesh.nx);
            mesh.clamped = FACE_ZMIN;
            const index_t nb = 8, bs = std::max<index_t>(1, mesh.nx / nb);
            const index_t nbx = (mesh.nx + bs - 1) / bs;
            Rng rng(derive_seed(base, 1));
            std::vector<double> E(static_cast<size_t>(nbx * nbx * nbx));
            for (auto& e : E) e = std::pow(10.0, 6.0 * rng.uniform());
            mats.resize(static_cast<size_t>(mesh.nx * mesh.ny * mesh.nz));
            for (index_t ez = 0; ez < mesh.nz; ++ez)
                for (index_t ey = 0; ey < mesh.ny; ++ey)
                    for (index_t ex = 0; ex < mesh.nx; ++ex) {
                        const index_t b = ex / bs + nbx * (ey / bs + nbx * (ez / bs));
                        mats[static_cast<size_t>(ex + mesh.nx * (ey + mesh.ny * ez))] =
                            Material{E[static_cast<size_t>(b)], 0.3};
                    }
            break;
        }
        case 3: {
            mesh.nx = mesh.ny = sc(96, 2);
            mesh.nz = sc(24, 2);
            mesh.hx = mesh.hy = 1.0;
            mesh.hz = 0.05;
            mesh.perturb = 0.3;
            mesh.perturb_seed = derive_seed(base, 2);
            mesh.clamped = FACE_ZMIN;
            mats.assign(static_cast<size_t>(mesh.nx * mesh.ny * mesh.nz), Material{1.0, 0.3});
            break;
        }
        case 4: {
            mesh.nx = mesh.ny = sc(400, 2);
            mesh.nz = 4;
            mesh.hx = mesh.hy = mesh.hz = 1.0;
            mesh.clamped = FACE_XMIN | FACE_XMAX | FACE_YMIN | FACE_YMAX;
            mats.assign(static_cast<size_t>(mesh.nx * mesh.ny * mesh.nz), Material{1.0, 0.49});
            break;
        }
        case 5: {
            mesh.nx = mesh.ny = mesh.nz = sc(128, 2);
            const double h = 1.0 / double(mesh.nx);
            mesh.hx = mesh.hy = mesh.hz = h;
            mesh.clamped = FACE_ZMIN;
            Rng rng(derive_seed(base, 4));
            struct Sphere { double x, y, z, r; };
            std::vector<Sphere> sp(200);
            for (auto& s : sp) {
                s.x = rng.uniform(); s.y = rng.uniform(); s.z = rng.uniform();
                s.r = (2.0 + 4.0 * rng.uniform()) * h;
            }
            mats.resize(static_cast<size_t>(mesh.nx * mesh.ny * mesh.nz));
            for (index_t ez = 0; ez < mesh.nz; ++ez)
                for (index_t ey = 0; ey < mesh.ny; ++ey)
                    for (index_t ex = 0; ex < mesh.nx; ++ex) {
                        const double cx = (double(ex) + 0.5) * h, cy = (double(ey) + 0.5) * h,
                                     cz = (double(ez) + 0.5) * h;
                        bool in = false;
                        for (const auto& s : sp) {
                            const double dx = cx - s.x, dy = cy - s.y, dz = cz - s.z;
                            if (dx * dx + dy * dy + dz * dz <= s.r * s.r) { in = true; break; }
                        }
                        mats[static_cast<size_t>(ex + mesh.nx * (ey + mesh.ny * ez))] =
                            in ? Material{1.0e4, 0.25} : Material{1.0, 0.3};
                    }
            break;
        }
        default:
            throw ConfigError("make_config: config must be 1..5");
    }
    GeneratedProblem p = assemble_hex(mesh, mats);
    if (cfg == 3) rhs = rhs_gaussian(p, derive_seed(base, 3));
    else if (cfg == 4) rhs = rhs_top_pressure(p, 1.0);
    else rhs = rhs_top_nodal(p, -1.0);
    return p;
}

}  // namespace aspamg
