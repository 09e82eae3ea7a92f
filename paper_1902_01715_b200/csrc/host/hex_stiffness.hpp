// Element stiffness of the trilinear 8-node hex (2x2x2 Gauss, isotropic
// linear elasticity), shared by the host assembler (fem.cpp, g++
// -ffp-contract=off) and the device assembler (assemble_gpu.cu, nvcc
// -fmad=false): the same source, no contraction on either side, so both produce
// the same bits. Restates /root/reference/proj/core/src/fem.cpp:18-85 without
// Eigen (B' D B written as two explicit sequential products) and extends it to
// distorted hexes (full isoparametric Jacobian per Gauss point).
#pragma once

#if defined(__CUDACC__)
#define ASPAMG_HD __host__ __device__
#else
#define ASPAMG_HD
#endif

namespace aspamg {
namespace hexk {

// fem.cpp:30-34: local node a = ia + 2 ja + 4 ka
ASPAMG_HD inline double node_sign(int a, int axis) { return ((a >> axis) & 1) ? 1.0 : -1.0; }

// fem.cpp:18-28 (isotropic D in Voigt order xx,yy,zz,xy,yz,zx)
ASPAMG_HD inline void elastic_matrix(double E, double nu, double D[6][6]) {
    const double lambda = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
    const double mu = E / (2.0 * (1.0 + nu));
    for (int i = 0; i < 6; ++i)
        for (int j = 0; j < 6; ++j) D[i][j] = 0.0;
    D[0][0] = D[1][1] = D[2][2] = lambda + 2.0 * mu;
    D[0][1] = D[0][2] = D[1][0] = D[1][2] = D[2][0] = D[2][1] = lambda;
    D[3][3] = D[4][4] = D[5][5] = mu;
}

// Accumulate det * B' D B for one Gauss point given physical gradients
// (fem.cpp:67-79). K is row-major 24 x 24.
ASPAMG_HD inline void add_btdb(const double grad[8][3], const double D[6][6], double det, double* K) {
    double B[6][24];
    for (int r = 0; r < 6; ++r)
        for (int c = 0; c < 24; ++c) B[r][c] = 0.0;
    for (int a = 0; a < 8; ++a) {
        const double dx = grad[a][0], dy = grad[a][1], dz = grad[a][2];
        B[0][3 * a + 0] = dx;
        B[1][3 * a + 1] = dy;
        B[2][3 * a + 2] = dz;
        B[3][3 * a + 0] = dy;
        B[3][3 * a + 1] = dx;
        B[4][3 * a + 1] = dz;
        B[4][3 * a + 2] = dy;
        B[5][3 * a + 0] = dz;
        B[5][3 * a + 2] = dx;
    }
    double BtD[24][6];
    for (int i = 0; i < 24; ++i)
        for (int k = 0; k < 6; ++k) {
            double s = 0.0;
            for (int l = 0; l < 6; ++l) s += B[l][i] * D[l][k];
            BtD[i][k] = s;
        }
    for (int i = 0; i < 24; ++i)
        for (int j = 0; j < 24; ++j) {
            double s = 0.0;
            for (int k = 0; k < 6; ++k) s += BtD[i][k] * B[k][j];
            K[i * 24 + j] += det * s;
        }
}

ASPAMG_HD inline void mirror_lower(double* K) {  // fem.cpp:81-83
    for (int i = 0; i < 24; ++i)
        for (int j = 0; j < i; ++j) K[j * 24 + i] = K[i * 24 + j];
}

// Reference points of the 2-point Gauss rule; gp = 1 / sqrt(3) is passed in
// (computed once by the caller with the correctly rounded sqrt).
ASPAMG_HD inline void shape_gradients(double xi, double eta, double zeta, double dn[8][3]) {
    for (int a = 0; a < 8; ++a) {
        const double sx = node_sign(a, 0), sy = node_sign(a, 1), sz = node_sign(a, 2);
        dn[a][0] = 0.125 * sx * (1.0 + sy * eta) * (1.0 + sz * zeta);
        dn[a][1] = 0.125 * sy * (1.0 + sx * xi) * (1.0 + sz * zeta);
        dn[a][2] = 0.125 * sz * (1.0 + sx * xi) * (1.0 + sy * eta);
    }
}

// fem.cpp:37-85 (regular grid: constant Jacobian 2/h, det h^3/8).
ASPAMG_HD inline void stiffness_cube(double h, double E, double nu, double gp, double* Ke) {
    double D[6][6];
    elastic_matrix(E, nu, D);
    const double det_j = h * h * h / 8.0;
    for (int i = 0; i < 576; ++i) Ke[i] = 0.0;
    double grad[8][3];
    for (int gx = 0; gx < 2; ++gx)
        for (int gy = 0; gy < 2; ++gy)
            for (int gz = 0; gz < 2; ++gz) {
                const double xi = gp * (2 * gx - 1), eta = gp * (2 * gy - 1), zeta = gp * (2 * gz - 1);
                const double scale = 2.0 / h;
                for (int a = 0; a < 8; ++a) {
                    const double sx = node_sign(a, 0), sy = node_sign(a, 1), sz = node_sign(a, 2);
                    grad[a][0] = 0.125 * sx * (1.0 + sy * eta) * (1.0 + sz * zeta) * scale;
                    grad[a][1] = 0.125 * sy * (1.0 + sx * xi) * (1.0 + sz * zeta) * scale;
                    grad[a][2] = 0.125 * sz * (1.0 + sx * xi) * (1.0 + sy * eta) * scale;
                }
                add_btdb(grad, D, det_j, Ke);
            }
    mirror_lower(Ke);
}

// General isoparametric trilinear hex (distorted meshes, config 3). Returns
// false on an inverted or degenerate element (det J <= 0 at a Gauss point).
ASPAMG_HD inline bool stiffness_general(const double xyz[8][3], double E, double nu, double gp, double* Ke) {
    double D[6][6];
    elastic_matrix(E, nu, D);
    for (int i = 0; i < 576; ++i) Ke[i] = 0.0;
    for (int gx = 0; gx < 2; ++gx)
        for (int gy = 0; gy < 2; ++gy)
            for (int gz = 0; gz < 2; ++gz) {
                const double xi = gp * (2 * gx - 1), eta = gp * (2 * gy - 1), zeta = gp * (2 * gz - 1);
                double dn[8][3];
                shape_gradients(xi, eta, zeta, dn);
                double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};  // J[i][j] = dx_j/dxi_i
                for (int a = 0; a < 8; ++a)
                    for (int i = 0; i < 3; ++i)
                        for (int j = 0; j < 3; ++j) J[i][j] += dn[a][i] * xyz[a][j];
                const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                                   J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                                   J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
                if (!(det > 0.0)) return false;
                double Ji[3][3];
                Ji[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) / det;
                Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
                Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
                Ji[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) / det;
                Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
                Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
                Ji[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) / det;
                Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
                Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
                double grad[8][3];  // grad_x N = J^{-1} grad_xi N
                for (int a = 0; a < 8; ++a)
                    for (int i = 0; i < 3; ++i)
                        grad[a][i] = Ji[i][0] * dn[a][0] + Ji[i][1] * dn[a][1] + Ji[i][2] * dn[a][2];
                add_btdb(grad, D, det, Ke);
            }
    mirror_lower(Ke);
    return true;
}

}  // namespace hexk
}  // namespace aspamg
