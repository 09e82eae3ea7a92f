// Structured hexahedral linear-elasticity generator (input side of the solve).
//
// Restates /root/reference/proj/core/src/fem.cpp:9-221 without Eigen and
// extends it for BASELINE.json configs 3-5:
//   * per-axis spacing + interior-node perturbation -> full isoparametric
//     Jacobian per Gauss point (the reference assumes cubes, fem.cpp:38,56);
//   * a set of clamped faces (the reference supports one, fem.hpp:26,43-45);
//   * nodal / pressure / Gaussian right-hand sides.
// Assembly fills CSR directly (no triplet list): every (row, col) slot sums
// its element contributions in element order, exactly the order
// SparseMatrix::from_triplets uses for the reference's triplet stream
// (sparse_matrix.cpp:18-64, fem.cpp:148-182), and keeps all 9 entries of each
// node-pair block, so K is exactly 3x3-blocked with dofs interleaved 3f+c.
#pragma once

#include "core.hpp"
#include "../../../include/aspamg_host.h"

#include <array>
#include <vector>

namespace aspamg {

struct Material {
    double young_modulus = 1.0e6;
    double poisson_ratio = 0.3;
    void validate() const;  // fem.cpp:9-14
};

enum FaceBits : unsigned {
    FACE_NONE = 0, FACE_XMIN = 1, FACE_XMAX = 2, FACE_YMIN = 4,
    FACE_YMAX = 8, FACE_ZMIN = 16, FACE_ZMAX = 32
};

struct MeshSpec {
    index_t nx = 1, ny = 1, nz = 1;
    double hx = 1.0, hy = 1.0, hz = 1.0;
    double perturb = 0.0;          // interior nodes offset by U(-p*h_a, p*h_a) per axis
    std::uint64_t perturb_seed = 0;
    unsigned clamped = FACE_ZMIN;  // FaceBits
};

struct GeneratedProblem {
    Csr stiffness;                 // free dofs only, 3 per free node, interleaved
    std::vector<double> coords;    // n_free_nodes x 3 row-major
    std::vector<index_t> free_index;   // node -> free node id or -1
    std::vector<double> node_xyz;  // all nodes, row-major x,y,z
    index_t n_nodes = 0, n_free = 0;
    MeshSpec mesh;
};

// 24x24 unconstrained element stiffness of a (possibly distorted) hex with
// node coordinates xyz[8][3] in local order a = ia + 2 ja + 4 ka
// (fem.cpp:30-34), 2x2x2 Gauss, symmetric by mirroring (fem.cpp:81-83).
void hex_element_stiffness(const double xyz[8][3], const Material& m, double Ke[24][24]);
// The reference's regular-cube path (fem.cpp:37-85), spacing h on all axes.
void hex_element_stiffness_cube(double h, const Material& m, double Ke[24][24]);

// Assembly backend (capi.cpp, aspamg_set_assembly_backend): when set, assemble_hex
// hands the element stiffness + pattern + fill to it (the device assembler).
bool assembly_backend_set();
void assemble_external(const aspamg_hex_assembly& in, Csr& K);

GeneratedProblem assemble_hex(const MeshSpec& mesh, const std::vector<Material>& materials);

// Rigid body modes of the free nodes about their centroid, orthonormalized
// (fem.cpp:192-221). Returns 3n x r, r <= 6.
Dense rigid_body_modes(const std::vector<double>& coords, index_t n_free, bool* rank_deficient);

// Right-hand sides. All are length 3 * n_free.
std::vector<double> rhs_top_nodal(const GeneratedProblem& p, double fz);
std::vector<double> rhs_top_pressure(const GeneratedProblem& p, double pressure);
std::vector<double> rhs_gaussian(const GeneratedProblem& p, std::uint64_t seed);
std::vector<double> rhs_ones(const GeneratedProblem& p);

// BASELINE.json configs 1-5 (index 1..5); `scale` divides the element counts
// (>=1) for CPU-sized tests of the same construction. Fills rhs.
GeneratedProblem make_config(int cfg, index_t scale, std::vector<double>& rhs);

}  // namespace aspamg
