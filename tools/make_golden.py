#!/usr/bin/env python3
"""Generate tests/golden/ref_kernels.npz from the REFERENCE's own compiled code.

Runs here (where /root/reference exists and oracle/_ref/libaspamg_ref.so was
built from the unmodified sparse_matrix.cpp). The GPU box never needs the
reference: tests read the committed fixture.

Fixtures (inputs + the reference's outputs):
  * SPEC.md:39-42 spmv examples, SPEC.md:49-50 galerkin examples,
    SPEC.md:57-60 transposed triangular solve examples;
  * spmv / spmv_transpose / transpose of the C1 construction at 5^3 elements
    (product generator K) with a seeded x;
  * galerkin_triple(P_0, A_0) of that problem's product setup (P from DPLS);
  * from_triplets on the reference's element-order triplet stream for a 3x2x2
    mesh built from the product's own element stiffness (pins the assembly
    summation order, fem.cpp:148-182 + sparse_matrix.cpp:18-64).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import paper_1902_01715_b200 as P  # noqa: E402
import pyoracle as O  # noqa: E402


def element_triplets(nx, ny, nz, Ke, clamp_zmin=True):
    """The reference's triplet stream order (fem.cpp:148-180) for a uniform mesh."""
    mx, my, mz = nx + 1, ny + 1, nz + 1
    node = lambda i, j, k: i + mx * (j + my * k)  # noqa: E731
    clamped = np.zeros(mx * my * mz, bool)
    if clamp_zmin:
        for j in range(my):
            for i in range(mx):
                clamped[node(i, j, 0)] = True
    free = -np.ones(mx * my * mz, np.int64)
    free[~clamped] = np.arange((~clamped).sum())
    r, c, v = [], [], []
    for ez in range(nz):
        for ey in range(ny):
            for ex in range(nx):
                conn = [node(ex + (a & 1), ey + ((a >> 1) & 1), ez + ((a >> 2) & 1)) for a in range(8)]
                for a in range(8):
                    if clamped[conn[a]]:
                        continue
                    for b in range(8):
                        if clamped[conn[b]]:
                            continue
                        for ca in range(3):
                            for cb in range(3):
                                r.append(3 * free[conn[a]] + ca)
                                c.append(3 * free[conn[b]] + cb)
                                v.append(Ke[3 * a + ca, 3 * b + cb])
    return 3 * int((~clamped).sum()), np.array(r), np.array(c), np.array(v)


def main():
    assert O.ref_available(), "build oracle/_ref first (make oracle)"
    out = {}
    # SPEC.md:41 [[2,1],[1,2]] (1,1) -> (3,3)
    A = O.RefCsr.from_arrays(2, 2, [0, 2, 4], [0, 1, 0, 1], [2.0, 1.0, 1.0, 2.0])
    out["spec41_y"] = A.spmv(np.ones(2))
    # SPEC.md:50 A = I2, P = (1,1)' -> [2]
    I2 = O.RefCsr.from_arrays(2, 2, [0, 1, 2], [0, 1], [1.0, 1.0])
    Pc = O.RefCsr.from_arrays(2, 1, [0, 1, 2], [0, 0], [1.0, 1.0])
    Ac = O.RefCsr(O.ref().ref_galerkin_triple(Pc.h, I2.h))
    out["spec50_Ac"] = Ac.arrays()[4]
    # SPEC.md:59 G = [[1,0],[-1,2]], x = (1,2) -> G'y = x, y = (2,1)
    G = O.RefCsr.from_arrays(2, 2, [0, 1, 3], [0, 0, 1], [1.0, -1.0, 2.0])
    y = np.empty(2)
    x = np.array([1.0, 2.0])
    import ctypes as C
    O.ref().ref_lower_tri_solve_t(G.h, x.ctypes.data_as(C.POINTER(C.c_double)), y.ctypes.data_as(C.POINTER(C.c_double)))
    out["spec59_y"] = y

    # C1 construction at 5^3 elements
    prob = P.Problem.config(1, 4)
    K = prob.K
    rng = np.random.default_rng(20261019)
    xk = rng.standard_normal(K.n_rows)
    RK = O.RefCsr.from_arrays(K.n_rows, K.n_cols, K.row_offsets, K.col_indices, K.values)
    out["K_rp"], out["K_ci"], out["K_v"] = K.row_offsets.copy(), K.col_indices.copy(), K.values.copy()
    out["K_x"] = xk
    out["K_y"] = RK.spmv(xk)
    out["K_yt"] = RK.spmv_transpose(xk)
    h = P.Hierarchy.setup(K, prob.coords)
    l0 = h.level(0)
    RG = O.RefCsr.from_arrays(l0.G.n_rows, l0.G.n_cols, l0.G.row_offsets, l0.G.col_indices, l0.G.values)
    out["G_rp"], out["G_ci"], out["G_v"] = l0.G.row_offsets, l0.G.col_indices, l0.G.values
    _, _, out["Gt_rp"], out["Gt_ci"], out["Gt_v"] = RG.transpose().arrays()
    RP = O.RefCsr.from_arrays(l0.P.n_rows, l0.P.n_cols, l0.P.row_offsets, l0.P.col_indices, l0.P.values)
    out["P_shape"] = np.array([l0.P.n_rows, l0.P.n_cols])
    out["P_rp"], out["P_ci"], out["P_v"] = l0.P.row_offsets, l0.P.col_indices, l0.P.values
    _, _, out["Ac_rp"], out["Ac_ci"], out["Ac_v"] = O.RefCsr(O.ref().ref_galerkin_triple(RP.h, RK.h)).arrays()

    # assembly order pin: element stiffness from the product generator (1 element, unclamped)
    one = P.Problem.hex_cube(1, spacing=0.5, young=1.0, poisson=0.3, clamp=0)
    Ke = one.K.to_scipy().toarray()
    n, r, c, v = element_triplets(3, 2, 2, Ke)
    RA = O.RefCsr.from_triplets(n, n, r, c, v, symmetric=True)
    _, _, out["asm_rp"], out["asm_ci"], out["asm_v"] = RA.arrays()
    out["asm_mesh"] = np.array([3, 2, 2])
    out["asm_Ke"] = Ke
    path = os.path.join(ROOT, "tests", "golden", "ref_kernels.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, {k: getattr(v, "shape", None) for k, v in out.items()})


if __name__ == "__main__":
    main()
